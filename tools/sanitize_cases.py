"""Small runs of the flag- and cluster-synchronised kernels for
compute-sanitizer (memcheck / racecheck / synccheck), each checked bitwise
against the oracle so a run that "passes" the sanitizer also computed the
right answer under it.

    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py levelset_vflags

Cases:
  levelset_<schedule>  K5 lower/upper direct solves + level-scheduled GS
                       (schedule: cta = k_levels_warp on a cluster,
                       cta1 = one-CTA kernel, flags = separate flags,
                       vflags = value flags k_levels_vflags)
  ilu0_warp / ilu0_thread   device ILU(0) (k_ilu0_warp / thread-per-row)
  ilut                      device ILUT (k_ilut), incl. the overflow relaunch
  sweeps                    K1-K4 (k_rowdot family, k_row_scale_fused)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def bitwise(a, b):
    return a.shape == b.shape and np.array_equal(a.view(np.int64), b.view(np.int64))


def main(case):
    if case.startswith("levelset_"):
        os.environ["ILUG_LEVELSET"] = case.split("_", 1)[1]
    if case == "ilu0_thread":
        os.environ["ILUG_ILU0_WARP"] = "0"
    import torch
    import paper_2111_09512_b200 as ilug
    from oracle import oracle
    ref = oracle.Ref()
    torch.cuda.set_device(0)

    def dev(a):
        return torch.from_numpy(np.ascontiguousarray(a)).cuda()

    def host(t):
        torch.cuda.synchronize()
        return t.cpu().numpy()

    specs = [("poisson3d(12,12,10)", {}),
             ("pressure27(10,10,9)", {"ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5"})]
    if case.startswith("levelset_"):
        for spec, kv in specs:
            A = ilug.Matrix.generate(spec)
            L, U = ilug.ilu_factorize(A, ilug.Config().update(kv))
            f = ilug.Factors.from_csr(A.rows, L.csr(), U.csr(), scaling="row", direct=True)
            fr = ref.scale(ref.ilu(ref.mat(*A.csr()), ref.cfg(kv)), "row")
            b = np.random.default_rng(1).uniform(-1, 1, A.rows)
            y = torch.empty(A.rows, dtype=torch.float64, device="cuda")
            for _ in range(2):
                f.solve_lower(dev(b), y)
                assert bitwise(host(y), ref.solve_lower_direct(ref.mat(*L.csr()), b))
                f.solve_upper(dev(b), y)
                assert bitwise(host(y), ref.solve_upper_scaled_direct(fr, b))
            S = ilug.Smoother(A, ilug.Config().set("smoother.kind", "gauss_seidel"))
            x0 = np.random.default_rng(2).uniform(-1, 1, A.rows)
            xd = dev(x0.copy())
            S.smooth(dev(b), xd)
            Ar = ref.mat(*A.csr())
            want, _ = ref.smooth(Ar, ref.smoother(Ar, ref.cfg({"smoother.kind": "gauss_seidel"})), b, x0)
            assert bitwise(host(xd), want)
    elif case in ("ilu0_warp", "ilu0_thread", "ilut"):
        for spec, kv in specs:
            if (case == "ilut") != ("ilu.variant" in kv):
                continue
            A = ilug.Matrix.generate(spec)
            L, U = ilug.ilu_factorize_device(A, ilug.Config().update(kv))
            Lr, Ur, _, _ = ref.factors_arrays(ref.ilu(ref.mat(*A.csr()), ref.cfg(kv)))
            assert bitwise(L.csr()[2], Lr[2]) and bitwise(U.csr()[2], Ur[2])
        if case == "ilut":  # rows beyond the 256-entry shared list: the overflow relaunch
            kv = {"ilu.variant": "ilut", "ilu.droptol": "0", "ilu.lfill": "400"}
            A = ilug.Matrix.generate("poisson2d(24,24)")
            L, U = ilug.ilu_factorize_device(A, ilug.Config().update(kv))
            Lr, Ur, _, _ = ref.factors_arrays(ref.ilu(ref.mat(*A.csr()), ref.cfg(kv)))
            assert bitwise(L.csr()[2], Lr[2]) and bitwise(U.csr()[2], Ur[2])
    elif case == "sweeps":
        spec, kv = specs[1]
        A = ilug.Matrix.generate(spec)
        kv = dict(kv, **{"smoother.kind": "ilu", "trisolve.m_lower": 5, "trisolve.m_upper": 5})
        S = ilug.Smoother(A, ilug.Config().update(kv))
        Ar = ref.mat(*A.csr())
        rng = np.random.default_rng(3)
        b, x0 = rng.uniform(-1, 1, A.rows), rng.uniform(-1, 1, A.rows)
        xd = dev(x0.copy())
        S.ilu_sweep(dev(b), xd)
        assert bitwise(host(xd), ref.ilu_smooth_sweep(Ar, ref.smoother(Ar, ref.cfg(kv)), b, x0))
    else:
        raise SystemExit(f"unknown case {case}")
    print(f"{case}: OK (bitwise vs oracle/_ref)")


if __name__ == "__main__":
    main(sys.argv[1])
