timeout 120 python scripts/dbg_one.py 13 7 2 8 64
timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import synth, time, numpy as np
import paper_2504_21784_b200 as pk
for nx,G in ((40,64),(96,64),(512,64)):
    prob = synth.config(5, nx=nx, G=G)
    t=time.time()
    try:
        out = pk.run_problem(prob); print(nx, G, 'ok', time.time()-t, np.abs(out).max(), flush=True)
    except Exception as e: print(nx, G, 'EXC', e, time.time()-t, flush=True)
"
