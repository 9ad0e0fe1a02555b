import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2111_09512_b200 as ilug
spec = sys.argv[1]
A = ilug.Matrix.generate(spec)
for p in sys.argv[2].split(","):
    for extra in ({}, {"device.graph": "false"}):
        kv = dict({"krylov.tol": "1e-8", "schur.blocks_list": p}, **extra)
        t = time.time()
        try:
            rep = ilug.run_schur_solve(A, ilug.Config().update(kv))
            print(spec, p, extra, "ok", rep.table_rows("schur"), round(time.time() - t, 1), flush=True)
        except ilug.IlugError as e:
            print(spec, p, extra, "ERR", e, round(time.time() - t, 1), flush=True)
