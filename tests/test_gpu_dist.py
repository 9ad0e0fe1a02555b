"""GPU: the row-block distributed solve phase at p = 1, 2, 4, 8
ranks against the composed oracle.

The ranks run as host threads of this process on the one GPU, joined by the
in-process transport (ilug_dist_group: every collective synchronises the
caller's stream and meets at a host barrier, so no kernel waits on another
rank's kernel). The data path is the one the NCCL ranks run — halo plans,
pack kernels, split-gather products, rank-local smoothers, the all-gathered
coarsest solve, summed GMRES reductions — only the transport differs.

Oracle: oracle/_ref's ref_dist_* = the reference hierarchy with every level's
smoother state rebuilt from the block-diagonal part (block-Jacobi ILU factors
of blockdiag(A_k), block poly-GS, hybrid GS = residual with the off-block part
then gauss_seidel_sweep on the blocks) and cycle_level restated around them.
  * V-cycle and smoother: BITWISE (global entry order in every product).
  * GMRES: iterations +-1 (the reductions are summed per rank, then over ranks).
"""
import numpy as np
import pytest

from conftest import bitwise

pytestmark = pytest.mark.gpu

BASE = {"amg.coarsening": "pmis", "krylov.tol": "1e-8"}
CASES = [
    # C4-like: ILU(0) block-Jacobi on the finest level, hybrid GS below
    ("poisson3d(20,20,20)", {"smoother.kind": "ilu", "trisolve.m_lower": "5", "trisolve.m_upper": "5"}),
    # C2-like: ILUT, poly-GS fallback
    ("pressure27(14,14,14)", {"smoother.kind": "ilu", "ilu.variant": "ilut", "trisolve.m_lower": "5",
                              "trisolve.m_upper": "5", "smoother.fallback.kind": "poly_gs"}),
    # direct triangular solves, row/col scaling, W-cycle, l1-Jacobi below
    ("cutcell(12,12,12)", {"smoother.kind": "ilu", "trisolve.mode": "direct", "scaling": "row_col",
                           "amg.cycles_nu": "2", "smoother.fallback.kind": "l1_jacobi"}),
    # no ILU: Jacobi everywhere (global), two smoothed levels of GS
    ("poisson3d(16,16,12)", {"smoother.kind": "gauss_seidel", "smoother.levels": "2",
                             "smoother.fallback.kind": "jacobi"}),
]


def _ranks(ilug, torch, spec, kv, p, body):
    from paper_2111_09512_b200 import dist as idist
    A = ilug.Matrix.generate(spec)
    cfg = ilug.Config().update(dict(BASE, **kv))
    H = ilug.Hierarchy(A, cfg, host_only=True)
    group = idist.LocalGroup(p)

    def rank_fn(r):
        comm = group.comm(r)
        S = idist.Solver(H, comm)
        st = torch.cuda.Stream()
        return body(r, S, cfg, st)
    return A, cfg, idist.run_ranks(p, rank_fn, group)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 7, 8])  # 3, 7: uneven blocks (the last rank takes the remainder)
@pytest.mark.parametrize("spec,kv", CASES, ids=[c[0] for c in CASES])
def test_dist_vcycle_bitwise(ilug, ref, torch_cuda, spec, kv, p):
    torch = torch_cuda
    n = ilug.Matrix.generate(spec).rows
    r = np.random.default_rng(17).uniform(-1, 1, n)

    def body(rank, S, cfg, st):
        rl = torch.from_numpy(r[S.row0:S.row0 + S.nloc].copy()).cuda()
        z = torch.empty_like(rl)
        torch.cuda.synchronize()
        for _ in range(2):  # repeated cycles reuse every buffer
            S.vcycle(rl, z, stream=st)
        st.synchronize()
        return S.row0, z.cpu().numpy(), S.levels

    A, cfg, out = _ranks(ilug, torch, spec, kv, p, body)
    z = np.concatenate([o[1] for o in sorted(out, key=lambda o: o[0])])
    Ar = ref.mat(*A.csr())
    d = ref.dist_setup(Ar, ref.cfg(dict(BASE, **kv)), p)
    assert out[0][2] == ref.L.ref_dist_nlevels(d)
    want = ref.dist_vcycle(d, r, np.zeros(n))
    assert bitwise(z, want), f"max diff {np.abs(z - want).max()}"
    if p == 1:  # one rank: the composed oracle is the reference V-cycle itself
        assert bitwise(z, ref.vcycle(ref.amg(Ar, ref.cfg(dict(BASE, **kv))), r, np.zeros(n)))


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("spec,kv", CASES[:2], ids=[c[0] for c in CASES[:2]])
def test_dist_gmres_iterations(ilug, ref, torch_cuda, spec, kv, p):
    torch = torch_cuda
    A0 = ilug.Matrix.generate(spec)
    n = A0.rows
    b = np.random.default_rng(23).uniform(-1, 1, n)

    def body(rank, S, cfg, st):
        bl = torch.from_numpy(b[S.row0:S.row0 + S.nloc].copy()).cuda()
        x = torch.zeros_like(bl)
        torch.cuda.synchronize()
        res = S.gmres(cfg, bl, x, stream=st)
        st.synchronize()
        return S.row0, x.cpu().numpy(), res

    A, cfg, out = _ranks(ilug, torch, spec, kv, p, body)
    its = {o[2]["iterations"] for o in out}
    assert len(its) == 1, "ranks disagree on the iteration count"
    got = its.pop()
    Ar = ref.mat(*A.csr())
    want = ref.dist_krylov(Ar, ref.dist_setup(Ar, ref.cfg(dict(BASE, **kv)), p), ref.cfg(dict(BASE, **kv)), b)
    assert want["converged"]
    assert abs(got - want["iterations"]) <= 1, f"{got} vs composed reference {want['iterations']}"
    assert all(o[2]["status"] == 0 and o[2]["final_relres"] < 1e-8 for o in out)
    x = np.concatenate([o[1] for o in sorted(out, key=lambda o: o[0])])
    r = ref.residual(Ar, x, b)
    assert np.linalg.norm(r) / np.linalg.norm(b) < 1e-8


@pytest.mark.parametrize("p", [2, 4])
@pytest.mark.parametrize("kind", ["ilu", "gauss_seidel", "poly_gs", "l1_jacobi"])
def test_dist_smoother_bitwise(ilug, ref, torch_cuda, kind, p):
    """ilug_dist_smoother (the bench's N > 1 object) = the composed level-0 smoother."""
    from paper_2111_09512_b200 import dist as idist
    torch = torch_cuda
    spec = "pressure27(12,12,10)"
    kv = dict(BASE, **{"smoother.kind": kind, "ilu.variant": "ilut", "trisolve.m_lower": "4",
                       "trisolve.m_upper": "6"})
    A = ilug.Matrix.generate(spec)
    n = A.rows
    cfg = ilug.Config().update(kv)
    rng = np.random.default_rng(4)
    b, x0 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    starts = idist.partition(n, p)
    group = idist.LocalGroup(p)

    def rank_fn(r):
        comm = group.comm(r)
        r0, r1 = int(starts[r]), int(starts[r + 1])
        plan = idist.Plan(idist.generate_rows(spec, r0, r1), n, p, r)
        plan.exchange(comm)
        S = idist.Smoother(plan, comm, cfg)
        xl = torch.from_numpy(x0[r0:r1].copy()).cuda()
        bl = torch.from_numpy(b[r0:r1].copy()).cuda()
        torch.cuda.synchronize()
        S.smooth(bl, xl)
        torch.cuda.synchronize()
        return r0, xl.cpu().numpy()

    out = idist.run_ranks(p, rank_fn, group)
    got = np.concatenate([o[1] for o in sorted(out, key=lambda o: o[0])])
    Ar = ref.mat(*A.csr())
    want = ref.dist_smooth(ref.dist_setup(Ar, ref.cfg(kv), p), 0, b, x0)
    assert bitwise(got, want)


def test_dist_smooth_host_many_two_ranks(ilug, ref, torch_cuda):
    """The bench's host-buffer pipeline at 2 ranks = the composed smoother per step."""
    from paper_2111_09512_b200 import dist as idist
    torch = torch_cuda
    spec, p = "poisson3d(14,14,12)", 2
    kv = dict(BASE, **{"smoother.kind": "ilu", "trisolve.m_lower": "5", "trisolve.m_upper": "5"})
    A = ilug.Matrix.generate(spec)
    n = A.rows
    cfg = ilug.Config().update(kv)
    rng = np.random.default_rng(9)
    bs = [rng.uniform(-1, 1, n) for _ in range(3)]
    xs = [rng.uniform(-1, 1, n) for _ in range(3)]
    starts = idist.partition(n, p)
    group = idist.LocalGroup(p)

    def rank_fn(r):
        comm = group.comm(r)
        r0, r1 = int(starts[r]), int(starts[r + 1])
        plan = idist.Plan(idist.generate_rows(spec, r0, r1), n, p, r)
        plan.exchange(comm)
        S = idist.Smoother(plan, comm, cfg)
        bl = [bb[r0:r1].copy() for bb in bs]
        xl = [xx[r0:r1].copy() for xx in xs]
        S.smooth_host_many(bl, xl)
        return r0, xl

    out = sorted(idist.run_ranks(p, rank_fn, group), key=lambda o: o[0])
    Ar = ref.mat(*A.csr())
    d = ref.dist_setup(Ar, ref.cfg(kv), p)
    for i in range(3):
        got = np.concatenate([o[1][i] for o in out])
        assert bitwise(got, ref.dist_smooth(d, 0, bs[i], xs[i]))


SCHUR = {"smoother.kind": "schur_ilut", "krylov.method": "fgmres", "schur.ilut.droptol": "1e-3",
         "schur.ilut.lfill": "5", "schur.trisolve.mL": "10", "schur.trisolve.mU": "10"}


@pytest.mark.parametrize("p", [2, 4, 8])
def test_dist_schur_smoother_matches_reference(ilug, ref, torch_cuda, p):
    """The ILUT Schur-complement smoother across p ranks (block b = rank b,
    src/schur.cpp:158-219): B/E/F block-local, C's interface halo exchanged,
    beta^2 / h11 / h21^2 summed over the ranks — the reference's schur_smooth
    with p blocks to rounding (the three sums are the only reordering)."""
    from paper_2111_09512_b200 import dist as idist
    from conftest import rel_err
    torch = torch_cuda
    spec = "pressure27(16,16,16)"
    kv = dict(BASE, **SCHUR, **{"schur.blocks": str(p)})
    A = ilug.Matrix.generate(spec)
    n = A.rows
    cfg = ilug.Config().update(kv)
    rng = np.random.default_rng(6)
    b, x0 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    starts = idist.partition(n, p)
    group = idist.LocalGroup(p)

    def rank_fn(r):
        comm = group.comm(r)
        r0, r1 = int(starts[r]), int(starts[r + 1])
        plan = idist.Plan(idist.generate_rows(spec, r0, r1), n, p, r)
        plan.exchange(comm)
        S = idist.Smoother(plan, comm, cfg)
        xl = torch.from_numpy(x0[r0:r1].copy()).cuda()
        bl = torch.from_numpy(b[r0:r1].copy()).cuda()
        torch.cuda.synchronize()
        S.smooth(bl, xl)
        torch.cuda.synchronize()
        return r0, xl.cpu().numpy()

    out = idist.run_ranks(p, rank_fn, group)
    got = np.concatenate([o[1] for o in sorted(out, key=lambda o: o[0])])
    Ar = ref.mat(*A.csr())
    want, _ = ref.smooth(Ar, ref.smoother(Ar, ref.cfg(kv)), b, x0)
    assert rel_err(got - x0, want - x0) < 1e-12


@pytest.mark.parametrize("p", [2, 4, 8])
def test_dist_schur_fgmres_iterations(ilug, ref, torch_cuda, p):
    """C5 (BASELINE configs[4]) in miniature: FGMRES + AMG with the Schur
    smoother on the finest level across p ranks, iterations +-1 of the
    composed reference (its Schur smoother with p blocks, block smoothers below)."""
    torch = torch_cuda
    spec = "poisson3d(16,16,16)"  # reference: 5 / 8 / 9 / 9 iterations at p = 1 / 2 / 4 / 8
    kv = dict(SCHUR, **{"schur.blocks": str(p)})
    A0 = ilug.Matrix.generate(spec)
    n = A0.rows
    b = np.random.default_rng(29).uniform(-1, 1, n)

    def body(rank, S, cfg, st):
        bl = torch.from_numpy(b[S.row0:S.row0 + S.nloc].copy()).cuda()
        x = torch.zeros_like(bl)
        torch.cuda.synchronize()
        res = S.gmres(cfg, bl, x, stream=st)
        st.synchronize()
        return S.row0, x.cpu().numpy(), res

    A, cfg, out = _ranks(ilug, torch, spec, kv, p, body)
    got = out[0][2]["iterations"]
    assert all(o[2]["iterations"] == got and o[2]["status"] == 0 for o in out)
    Ar = ref.mat(*A.csr())
    kvr = dict(BASE, **kv)
    want = ref.dist_krylov(Ar, ref.dist_setup(Ar, ref.cfg(kvr), p), ref.cfg(kvr), b)
    assert want["converged"] and abs(got - want["iterations"]) <= 1, f"{got} vs {want['iterations']}"


@pytest.mark.parametrize("p", [2, 4])
def test_dist_schur_fgmres_iterations_pressure27(ilug, ref, torch_cuda, p):
    """C5 on the variable-coefficient operator, where the Schur smoother with
    p blocks needs 140-180 FGMRES iterations (the reference: 139 / 174 at
    pressure27(20^3)): the distributed solver's count stays within +-1 of the
    reference's own Schur smoother with p blocks over the long run."""
    torch = torch_cuda
    spec = "pressure27(20,20,20)"
    kv = dict(SCHUR, **{"schur.blocks": str(p)})
    A0 = ilug.Matrix.generate(spec)
    b = np.random.default_rng(29).uniform(-1, 1, A0.rows)

    def body(rank, S, cfg, st):
        bl = torch.from_numpy(b[S.row0:S.row0 + S.nloc].copy()).cuda()
        x = torch.zeros_like(bl)
        torch.cuda.synchronize()
        res = S.gmres(cfg, bl, x, stream=st)
        st.synchronize()
        return S.row0, x.cpu().numpy(), res

    A, cfg, out = _ranks(ilug, torch, spec, kv, p, body)
    got = out[0][2]["iterations"]
    assert all(o[2]["iterations"] == got and o[2]["status"] == 0 for o in out)
    Ar = ref.mat(*A.csr())
    kvr = dict(BASE, **kv)
    want = ref.dist_krylov(Ar, ref.dist_setup(Ar, ref.cfg(kvr), p), ref.cfg(kvr), b)
    assert want["converged"] and abs(got - want["iterations"]) <= 1, f"{got} vs {want['iterations']}"


def test_dist_solver_nccl_world_one_matches_local(ilug, ref, torch_cuda):
    """The NCCL transport (what torchrun ranks use) at world size 1 runs the same
    distributed solver as the in-process group: identical V-cycle bits and
    iteration count (at p = 1 both equal the reference V-cycle)."""
    from paper_2111_09512_b200 import dist as idist
    torch = torch_cuda
    spec, kv = CASES[1]
    A = ilug.Matrix.generate(spec)
    cfg = ilug.Config().update(dict(BASE, **kv))
    H = ilug.Hierarchy(A, cfg, host_only=True)
    r = np.random.default_rng(3).uniform(-1, 1, A.rows)
    rd = torch.from_numpy(r).cuda()
    outs = []
    for comm in (idist.Comm(1, 0, idist.unique_id()), idist.LocalGroup(1).comm(0)):
        S = idist.Solver(H, comm)
        z = torch.empty_like(rd)
        S.vcycle(rd, z)
        x = torch.zeros_like(rd)
        res = S.gmres(cfg, rd, x)
        torch.cuda.synchronize()
        outs.append((z.cpu().numpy(), res["iterations"], x.cpu().numpy()))
    assert bitwise(outs[0][0], outs[1][0]) and outs[0][1] == outs[1][1] and bitwise(outs[0][2], outs[1][2])
    Hr = ref.amg(ref.mat(*A.csr()), ref.cfg(dict(BASE, **kv)))
    assert bitwise(outs[0][0], ref.vcycle(Hr, r, np.zeros(A.rows)))


def test_dist_failure_on_one_rank_does_not_hang(ilug, torch_cuda):
    """A rank that fails (here: an invalid smoother configuration on rank 0
    only) aborts the in-process group, so its peer's next collective raises
    instead of waiting forever."""
    from paper_2111_09512_b200 import dist as idist
    torch = torch_cuda
    spec, p = "poisson3d(12,12,12)", 2
    A = ilug.Matrix.generate(spec)
    n = A.rows
    starts = idist.partition(n, p)
    group = idist.LocalGroup(p)
    good = {"smoother.kind": "ilu", "trisolve.m_lower": "3", "trisolve.m_upper": "3"}
    bad = dict(good, **{"scaling": "none"})  # Richardson on unscaled factors: invalid

    def rank_fn(r):
        comm = group.comm(r)
        r0, r1 = int(starts[r]), int(starts[r + 1])
        plan = idist.Plan(idist.generate_rows(spec, r0, r1), n, p, r)
        plan.exchange(comm)
        S = idist.Smoother(plan, comm, ilug.Config().update(bad if r == 0 else good))
        x = torch.zeros(r1 - r0, dtype=torch.float64, device="cuda")
        S.smooth(torch.ones_like(x), x)  # rank 1 reaches the halo exchange alone
        return r

    with pytest.raises(ilug.IlugError):
        idist.run_ranks(p, rank_fn, group)
