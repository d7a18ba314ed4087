import csv, sys, subprocess
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[2]
ix = {k: i for i, k in enumerate(hdr)}
S = 4
stall_cols = [i for i, k in enumerate(hdr) if k.startswith('stall_') and '(Not' not in k]
lines = []
for r in rows[3:]:
    if len(r) < len(hdr) or not r[0]:
        continue
    try:
        s = int(r[S])
    except Exception:
        continue
    st = {hdr[i]: int(r[i]) for i in stall_cols if r[i] not in ('', '-', '0')}
    lines.append((s, int(r[0]), r[1][:95], st))
tot = sum(l[0] for l in lines)
print('total samples', tot)
lines.sort(key=lambda x: -x[0])
for l in lines[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    top = sorted(l[3].items(), key=lambda kv: -kv[1])[:3]
    print(f"{l[0]*100/tot:5.1f}% L{l[1]:>5} {l[2]:95s} {[(k[6:], round(v*100/tot,1)) for k,v in top]}")
