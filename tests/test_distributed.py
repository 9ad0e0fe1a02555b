"""CPU, multi-process (gloo, world sizes 2 and 3): the host side of the
multi-GPU path — row-block partition, per-rank generation, halo plans and the
request exchange — reproduces the single-process operator exactly.

Each rank builds its plan through the C ABI, exchanges requests with
torch.distributed (gloo), performs the halo exchange the device path performs
with NCCL (pack sends(q), send/recv), and evaluates its residual rows from the
extended local matrix in stored entry order; the result must be bitwise the
global residual of the C restatement oracle (same products, same order).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SPECS = ["pressure27(12,10,9)", "poisson3d(9,8,11)", "cutcell(10,10,10)"]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _csr_rows_apply(rp, ci, v, x_ext, b):
    r = np.empty(len(rp) - 1)
    for i in range(len(rp) - 1):
        s = 0.0
        for k in range(rp[i], rp[i + 1]):
            s += v[k] * x_ext[ci[k]]
        r[i] = b[i] - s
    return r


def _worker(rank, world, port, spec, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2111_09512_b200 as ilug
        from paper_2111_09512_b200 import dist as idist
        from oracle import oracle

        A = ilug.Matrix.generate(spec)
        n = A.rows
        starts = idist.partition(n, world)
        r0, r1 = int(starts[rank]), int(starts[rank + 1])
        rows = idist.generate_rows(spec, r0, r1)
        grp, gci, gv = A.csr()
        lrp, lci, lv = rows.csr()
        # per-rank generation == the global matrix's rows
        assert np.array_equal(lrp, grp[r0:r1 + 1] - grp[r0])
        assert np.array_equal(lci, gci[grp[r0]:grp[r1]]) and np.array_equal(lv, gv[grp[r0]:grp[r1]])

        plan = idist.Plan(rows, n, world, rank)
        assert (plan.row0, plan.row1) == (r0, r1)

        def all_gather(obj):
            out = [None] * world
            dist.all_gather_object(out, obj)
            return out
        plan.exchange_requests(all_gather)

        rng = np.random.default_rng(5)
        x = rng.uniform(-1, 1, n)
        b = rng.uniform(-1, 1, n)
        x_loc = x[r0:r1].copy()
        # halo exchange (the device path does this with grouped ncclSend/ncclRecv)
        halo = np.empty(plan.nhalo)
        reqs = []
        for p in range(world):
            if p == rank:
                continue
            send = plan.sends(p)
            if len(send):
                reqs.append(dist.isend(torch.from_numpy(x_loc[send].copy()), dst=p))
        offset = 0
        for p in range(world):
            if p == rank:
                continue
            need = plan.requests(p)
            if len(need):
                buf = torch.empty(len(need), dtype=torch.float64)
                dist.recv(buf, src=p)
                halo[offset:offset + len(need)] = buf.numpy()
                assert np.array_equal(halo[offset:offset + len(need)], x[need])
                offset += len(need)
        for rq in reqs:
            rq.wait()
        assert offset == plan.nhalo
        erp, eci, ev = plan.matrix("ext").csr()
        r_loc = _csr_rows_apply(erp, eci, ev, np.concatenate([x_loc, halo]), b[r0:r1])
        want = oracle.Port().residual((grp, gci, gv), x, b)[r0:r1]
        assert np.array_equal(r_loc.view(np.int64), want.view(np.int64)), "distributed residual not bitwise"
        # diagonal block = the local columns of the local rows, sorted
        drp, dci, dv = plan.matrix("diag").csr()
        M = np.zeros((r1 - r0, r1 - r0))
        for i in range(r1 - r0):
            M[i, dci[drp[i]:drp[i + 1]]] = dv[drp[i]:drp[i + 1]]
        G = np.zeros((r1 - r0, r1 - r0))
        for i in range(r0, r1):
            for k in range(grp[i], grp[i + 1]):
                if r0 <= gci[k] < r1:
                    G[i - r0, gci[k] - r0] = gv[k]
        assert np.array_equal(M, G)
        q.put((rank, "ok"))
    except Exception as e:  # surface the failure to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("spec", SPECS)
def test_distributed_residual_bitwise_gloo(world, spec):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, spec, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert results[r] == "ok", results[r]


def test_partition_rule():
    """src/schur.cpp:28-33: base = n/p, the last block absorbs the remainder."""
    import sys
    sys.path.insert(0, ROOT)
    from paper_2111_09512_b200 import dist as idist
    assert idist.partition(10, 3).tolist() == [0, 3, 6, 10]
    assert idist.partition(16, 4).tolist() == [0, 4, 8, 12, 16]
    with pytest.raises(Exception):
        idist.partition(3, 0)


# ---------------------------------------------------------------------------
# Distributed V-cycle host logic: every rank builds the global
# host hierarchy, takes its per-level plans from ilug_dist_level_plans
# (A_k / P_k rows by the level's partition, R_k rows by the next level's),
# completes the send lists over gloo, and runs the V-cycle with the C port's
# products on its extended matrices and gloo halo exchanges. Jacobi smoothing
# (a global smoother: no block approximation), the last smoothed level's
# residual all-reduced into the whole coarse rhs. Compared with the composed
# single-process oracle (oracle/_ref ref_dist_vcycle at p ranks).

def _halo(plan, world, rank, x_loc):
    """Exchange the entries of x_loc other ranks read; return this rank's halo."""
    reqs = []
    for p in range(world):
        if p != rank:
            send = plan.sends(p)
            if len(send):
                reqs.append(dist.isend(torch.from_numpy(x_loc[send].copy()), dst=p))
    halo = np.empty(plan.nhalo)
    off = 0
    for p in range(world):
        if p != rank:
            need = plan.requests(p)
            if len(need):
                buf = torch.empty(len(need), dtype=torch.float64)
                dist.recv(buf, src=p)
                halo[off:off + len(need)] = buf.numpy()
                off += len(need)
    for rq in reqs:
        rq.wait()
    return halo


def _vcycle_worker(rank, world, port, spec, kv, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2111_09512_b200 as ilug
        from paper_2111_09512_b200 import dist as idist
        from oracle import oracle
        P = oracle.Port()

        def all_gather(obj):
            out = [None] * world
            dist.all_gather_object(out, obj)
            return out

        A = ilug.Matrix.generate(spec)
        H = ilug.Hierarchy(A, ilug.Config().update(kv), host_only=True)
        L = H.levels
        LP = idist.LevelPlans(H, world, rank)
        assert LP.count == L - 1
        lev = []
        for k in range(L - 1):
            d = {"A": LP.plan(k, "A")}
            d["A"].exchange_requests(all_gather)
            last = k == L - 2
            if not last:
                for w in ("R", "P"):
                    d[w] = LP.plan(k, w)
                    d[w].exchange_requests(all_gather)
            else:
                d["R_full"] = LP.last("R").csr()
                d["P_rows"] = LP.last("P").csr()
            Aext = d["A"].matrix("ext").csr()
            diag = np.zeros(d["A"].row1 - d["A"].row0)
            drp, dci, dv = d["A"].matrix("diag").csr()
            for i in range(len(diag)):
                for t in range(drp[i], drp[i + 1]):
                    if dci[t] == i:
                        diag[i] = dv[t]
            d["Aext"], d["invd"], d["last"] = Aext, 1.0 / diag, last
            d["n"] = H.level_matrix(k, "A").rows
            lev.append(d)
        Ac = H.level_matrix(L - 1, "A")
        crp, cci, cv = Ac.csr()
        Cd = np.zeros((Ac.rows, Ac.rows))
        for i in range(Ac.rows):
            Cd[i, cci[crp[i]:crp[i + 1]]] = cv[crp[i]:crp[i + 1]]
        sweeps = int(kv.get("smoother.sweeps", 2))

        def smooth(d, b, x):
            for _ in range(sweeps):
                xe = np.concatenate([x, _halo(d["A"], world, rank, x)])
                x = x + d["invd"] * (b - P.spmv(d["Aext"], xe))
            return x

        def cycle(k, b, x):
            d = lev[k]
            x = smooth(d, b, x)
            r = P.residual(d["Aext"], np.concatenate([x, _halo(d["A"], world, rank, x)]), b)
            if not d["last"]:
                rc = P.spmv(d["R"].matrix("ext").csr(), np.concatenate([r, _halo(d["R"], world, rank, r)]))
                e = np.zeros(lev[k + 1]["A"].row1 - lev[k + 1]["A"].row0)
                e = cycle(k + 1, rc, e)
                x = x + P.spmv(d["P"].matrix("ext").csr(), np.concatenate([e, _halo(d["P"], world, rank, e)]))
            else:
                full = torch.zeros(d["n"], dtype=torch.float64)
                full[d["A"].row0:d["A"].row1] = torch.from_numpy(r)
                dist.all_reduce(full)
                bc = P.spmv(d["R_full"], full.numpy())
                xc = np.linalg.solve(Cd, bc)
                x = x + P.spmv(d["P_rows"], xc)
            return smooth(d, b, x)

        n = A.rows
        r_glob = np.random.default_rng(31).uniform(-1, 1, n)
        p0 = lev[0]["A"]
        z = cycle(0, r_glob[p0.row0:p0.row1].copy(), np.zeros(p0.row1 - p0.row0))
        zs = all_gather((p0.row0, z))
        zfull = np.concatenate([t[1] for t in sorted(zs, key=lambda t: t[0])])
        R = oracle.Ref()
        Ar = R.mat(*A.csr())
        want = R.dist_vcycle(R.dist_setup(Ar, R.cfg(kv), world), r_glob, np.zeros(n))
        err = np.linalg.norm(zfull - want) / np.linalg.norm(want)
        assert err < 1e-12, f"distributed V-cycle differs from the composed oracle: {err}"
        q.put((rank, "ok"))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("spec", ["poisson3d(10,10,9)", "pressure27(9,9,8)"])
def test_distributed_vcycle_plans_gloo(world, spec):
    from oracle import oracle
    if not os.path.exists(oracle.REF_SO):
        pytest.skip("oracle/_ref not built")
    kv = {"smoother.kind": "jacobi", "smoother.fallback.kind": "jacobi", "amg.coarsening": "pmis"}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_vcycle_worker, args=(r, world, port, spec, kv, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert results[r] == "ok", results[r]
