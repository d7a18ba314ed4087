import csv,sys,collections
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; ix={h:i for i,h in enumerate(hdr)}
data=[r for r in rows[2:] if len(r)>=len(hdr)]
tot=sum(int(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)) for r in data)
# windows of W instructions
W=int(sys.argv[2]) if len(sys.argv)>2 else 100
for s in range(0,len(data),W):
    blk=data[s:s+W]
    smp=sum(int(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)) for r in blk)
    if smp < tot*0.005: continue
    ops=collections.Counter()
    for r in blk:
        src=r[ix["Source"]].strip().split()
        if not src: continue
        op=src[1] if src[0].startswith('@') else src[0]
        ops[op.split('.')[0]]+=int(float(r[ix["Instructions Executed"]] or 0))
    st=collections.Counter()
    for r in blk:
        for k in ("stall_barrier","stall_wait","stall_math","stall_short_sb","stall_long_sb","stall_selected","stall_not_selected","stall_dispatch"):
            st[k]+=int(float(r[ix[k]] or 0))
    print(f"[{s:5d}-{s+W:5d}] {r[ix['Address']] if False else blk[0][ix['Address']]} samples {100*smp/tot:5.1f}%  ", " ".join(f"{k[6:]}={100*v/tot:.1f}" for k,v in st.most_common(5)), "|", " ".join(f"{o}:{n/1e6:.0f}M" for o,n in ops.most_common(5)))
