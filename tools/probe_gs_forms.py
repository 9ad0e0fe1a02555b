"""Coarse-level Gauss-Seidel (K5, MODE 2) on every level of SPEC's PMIS
hierarchy under each level-set schedule: the cluster kernel (default for
narrow DAGs) vs the value-flag forms. Timing probe, not a test.

    python tools/probe_gs_forms.py [SPEC]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_09512_b200 as ilug  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "pressure27(256,256,256)"
A = ilug.Matrix.generate(spec)
H = ilug.Hierarchy(A, ilug.Config().update({"amg.coarsening": "pmis"}), host_only=True)
FORMS = {"default": {}, "sx": {"ILUG_LEVELSET": "sx"}, "cta": {"ILUG_LEVELSET": "cta"}}
for code in ("0", "1", "83", "8", "88", "164", "168", "324"):
    FORMS["vf" + code] = {"ILUG_LEVELSET": "vflags", "ILUG_VF_SUB": code}
# FORMS env var: comma-separated subset (default: all)
forms = [(k, FORMS[k]) for k in (os.environ.get("FORMS") or ",".join(FORMS)).split(",")]
for lvl in range(1, H.levels - 1):
    M = H.level_matrix(lvl, "A")
    rp, _, _ = M.csr()
    row = {"level": lvl, "n": M.rows, "nnz": M.nnz, "max_row": int(np.diff(rp).max())}
    b = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, M.rows)).cuda()
    ref_x = None
    for name, env in forms:
        for k in ("ILUG_LEVELSET", "ILUG_VF_SUB"):
            os.environ.pop(k, None)
        os.environ.update(env)
        S = ilug.Smoother(M, ilug.Config().update({"smoother.kind": "gauss_seidel", "smoother.sweeps": "1"}))
        x = torch.zeros_like(b)
        S.smooth(b, x)
        torch.cuda.synchronize()
        xs = x.cpu().numpy()
        if ref_x is None:
            ref_x = xs
        same = bool(np.array_equal(xs.view(np.int64), ref_x.view(np.int64)))
        for _ in range(2):
            S.smooth(b, x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            S.smooth(b, x)
        e1.record()
        torch.cuda.synchronize()
        row[name] = round(e0.elapsed_time(e1) / 5, 3)
        row[name + "_bitwise"] = same
        del S
    print(json.dumps(row), flush=True)
