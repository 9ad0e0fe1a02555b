"""Concurrent calls on ONE handle (SURVEY.md §8b threading row): the reference
guarantees that types are immutable after construction and that concurrent
`vcycle` calls on distinct right-hand sides are safe and bitwise equal to the
serial ones (README.md:152-154, tests/test_amg.cpp:337-354). Here several
host threads, each on its own CUDA stream, drive the same hierarchy /
smoother / factors handle at once (ctypes releases the GIL during the calls);
every result must equal the serial result bit for bit."""
import threading

import numpy as np
import pytest

from conftest import bitwise

pytestmark = pytest.mark.gpu

KV = {"smoother.kind": "ilu", "ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5",
      "trisolve.m_lower": "5", "trisolve.m_upper": "5", "amg.coarsening": "pmis", "smoother.sweeps": "2"}
THREADS, REPEATS = 4, 6


def _run_concurrently(torch, fn, rhs):
    """fn(k, stream) on THREADS threads at once, each with its own stream."""
    streams = [torch.cuda.Stream() for _ in rhs]
    errors = []
    barrier = threading.Barrier(len(rhs))

    def work(k):
        try:
            barrier.wait()
            for _ in range(REPEATS):
                fn(k, streams[k])
        except BaseException as e:  # noqa: BLE001 (surface any failure in the main thread)
            errors.append(e)

    ts = [threading.Thread(target=work, args=(k,)) for k in range(len(rhs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    torch.cuda.synchronize()
    assert not errors, errors


def _rhs(torch, n, seed):
    return [torch.from_numpy(np.random.default_rng(seed + k).uniform(-1, 1, n)).cuda() for k in range(THREADS)]


@pytest.mark.parametrize("graph", [True, False])
def test_concurrent_vcycles_bitwise_serial(ilug, torch_cuda, graph):
    torch = torch_cuda
    A = ilug.Matrix.generate("pressure27(24,24,24)")
    H = ilug.Hierarchy(A, ilug.Config().update(dict(KV, **{"device.graph": str(graph).lower()})))
    rs = _rhs(torch, A.rows, 100)
    want = []
    for r in rs:
        z = torch.empty_like(r)
        H.vcycle(r, z)
        torch.cuda.synchronize()
        want.append(z.cpu().numpy())
    zs = [torch.empty_like(r) for r in rs]
    _run_concurrently(torch, lambda k, st: H.vcycle(rs[k], zs[k], stream=st), rs)
    for k in range(THREADS):
        assert bitwise(zs[k].cpu().numpy(), want[k]), f"rhs {k}"


def test_concurrent_smoothing_bitwise_serial(ilug, torch_cuda):
    """Each thread smooths its own x in place REPEATS times; the serial
    reference applies the same number of smoothing steps."""
    torch = torch_cuda
    A = ilug.Matrix.generate("pressure27(24,24,24)")
    S = ilug.Smoother(A, ilug.Config().update(KV))
    bs = _rhs(torch, A.rows, 200)
    want = []
    for b in bs:
        x = torch.zeros_like(b)
        for _ in range(REPEATS):
            S.smooth(b, x)
        torch.cuda.synchronize()
        want.append(x.cpu().numpy())
    xs = [torch.zeros_like(b) for b in bs]
    _run_concurrently(torch, lambda k, st: S.smooth(bs[k], xs[k], stream=st), bs)
    for k in range(THREADS):
        assert bitwise(xs[k].cpu().numpy(), want[k]), f"rhs {k}"


def test_concurrent_direct_solves_bitwise_serial(ilug, torch_cuda):
    """Level-scheduled direct solves (K5) share the plan's tickets / flags."""
    torch = torch_cuda
    A = ilug.Matrix.generate("pressure27(24,24,24)")
    F = ilug.Factors.create(A, ilug.Config().update(KV), scaling="row", direct=True)
    bs = _rhs(torch, A.rows, 300)
    want = []
    for b in bs:
        y, x = torch.empty_like(b), torch.empty_like(b)
        F.solve_lower(b, y)
        F.solve_upper(y, x)
        torch.cuda.synchronize()
        want.append(x.cpu().numpy())
    ys = [torch.empty_like(b) for b in bs]
    xs = [torch.empty_like(b) for b in bs]

    def both(k, st):
        F.solve_lower(bs[k], ys[k], stream=st)
        F.solve_upper(ys[k], xs[k], stream=st)

    _run_concurrently(torch, both, bs)
    for k in range(THREADS):
        assert bitwise(xs[k].cpu().numpy(), want[k]), f"rhs {k}"
