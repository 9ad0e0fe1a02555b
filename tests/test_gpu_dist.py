"""GPU, one rank: the distributed objects (halo plan, NCCL communicator,
block-Jacobi smoother, distributed GMRES+AMG) reduce exactly to the
single-GPU path when there is one rank — same kernels, same order — so they
are bitwise / iteration-exact against it. (More than one rank cannot run on
this one-GPU pool; the multi-rank host logic is covered by
tests/test_distributed.py with gloo.)"""
import numpy as np
import pytest

from conftest import bitwise

pytestmark = pytest.mark.gpu

KV = {"smoother.kind": "ilu", "ilu.variant": "ilut", "trisolve.m_lower": "5", "trisolve.m_upper": "5",
      "krylov.tol": "1e-8", "amg.coarsening": "pmis", "smoother.fallback.kind": "poly_gs"}


def _setup(ilug, spec):
    from paper_2111_09512_b200 import dist as idist
    A = ilug.Matrix.generate(spec)
    rows = idist.generate_rows(spec, 0, A.rows)
    plan = idist.Plan(rows, A.rows, 1, 0)
    comm = idist.Comm(1, 0, idist.unique_id())
    return idist, A, plan, comm


@pytest.mark.parametrize("spec", ["pressure27(16,16,16)", "poisson3d(20,20,20)"])
def test_dist_smoother_single_rank_bitwise(ilug, torch_cuda, spec):
    idist, A, plan, comm = _setup(ilug, spec)
    assert plan.nhalo == 0
    cfg = ilug.Config().update(KV)
    Sd = idist.Smoother(plan, comm, cfg)
    S = ilug.Smoother(A, cfg)
    rng = np.random.default_rng(3)
    b = torch_cuda.from_numpy(rng.uniform(-1, 1, A.rows)).cuda()
    x0 = torch_cuda.from_numpy(rng.uniform(-1, 1, A.rows)).cuda()
    x1, x2 = x0.clone(), x0.clone()
    Sd.smooth(b, x1)
    S.smooth(b, x2)
    torch_cuda.cuda.synchronize()
    assert bitwise(x1.cpu().numpy(), x2.cpu().numpy())
    r = torch_cuda.empty_like(b)
    Sd.residual(x1, b, r)
    D = ilug.DeviceMatrix(A)
    r2 = torch_cuda.empty_like(b)
    D.residual(x1, b, r2)
    torch_cuda.cuda.synchronize()
    assert bitwise(r.cpu().numpy(), r2.cpu().numpy())


def test_dist_gmres_single_rank_matches(ilug, torch_cuda):
    idist, A, plan, comm = _setup(ilug, "pressure27(20,20,20)")
    cfg = ilug.Config().update(dict(KV, **{"krylov.form_iterates": "false"}))
    Sol = idist.Solver(plan, comm, cfg)
    D = ilug.DeviceMatrix(A)
    ones = torch_cuda.ones(A.rows, dtype=torch_cuda.float64, device="cuda")
    b = torch_cuda.empty_like(ones)
    D.spmv(ones, b)
    x = torch_cuda.zeros_like(ones)
    out = Sol.gmres(cfg, b, x)
    H = ilug.Hierarchy(A, cfg)
    x2 = torch_cuda.zeros_like(ones)
    want = H.gmres(cfg, b, x2)
    assert out["status"] == 0 and out["iterations"] == want["iterations"]
    assert out["final_relres"] == want["final_relres"]
    assert float((x - 1).abs().max()) < 1e-5


def test_dist_plan_two_virtual_ranks_structure(ilug):
    """Two ranks' plans built in one process: requests of one are exactly what
    the other can serve, and the extended matrices keep the global entry order."""
    from paper_2111_09512_b200 import dist as idist
    spec = "pressure27(10,10,8)"
    A = ilug.Matrix.generate(spec)
    starts = idist.partition(A.rows, 2)
    plans = [idist.Plan(idist.generate_rows(spec, int(starts[r]), int(starts[r + 1])), A.rows, 2, r)
             for r in range(2)]
    need01 = plans[0].requests(1)
    need10 = plans[1].requests(0)
    assert len(need01) == plans[0].nhalo and len(need10) == plans[1].nhalo
    assert need01.min() >= starts[1] and need10.max() < starts[1]
    plans[1].set_sends(0, need01)
    plans[0].set_sends(1, need10)
    assert np.array_equal(plans[1].sends(0) + starts[1], need01)


def test_dist_smooth_host_many_single_rank(ilug, torch_cuda):
    """ilug_dist_smooth_host_many at one rank = the single-GPU smoother applied
    to each host pair, bitwise."""
    idist, A, plan, comm = _setup(ilug, "pressure27(14,14,14)")
    cfg = ilug.Config().update(KV)
    Sd = idist.Smoother(plan, comm, cfg)
    S = ilug.Smoother(A, cfg)
    rng = np.random.default_rng(8)
    bs = [rng.uniform(-1, 1, A.rows) for _ in range(3)]
    xs = [rng.uniform(-1, 1, A.rows) for _ in range(3)]
    want = []
    for b, x in zip(bs, xs):
        xd = torch_cuda.from_numpy(x.copy()).cuda()
        S.smooth(torch_cuda.from_numpy(b).cuda(), xd)
        torch_cuda.cuda.synchronize()
        want.append(xd.cpu().numpy())
    Sd.smooth_host_many(bs, xs)
    for got, w in zip(xs, want):
        assert bitwise(got, w)
