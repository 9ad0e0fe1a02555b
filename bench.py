#!/usr/bin/env python3
"""Benchmark of the hot path: the ILU(T) smoother application inside the AMG
V-cycle on BASELINE config 2 (27-point variable-coefficient pressure matrix
256^3, 16.7M rows, ILUT(1e-3, 5) factors, row-scaled U) on one B200.

One "step" = one ilu_smooth_sweep (src/smoother.cpp:143-159) with
m_L = m_U = 5 Richardson sweeps: residual SpMV + 4 L sweeps + 4 row-scaled U
sweeps (the first iterate of each is exact, x1 = b), fused epilogues. The
metric is achieved HBM GB/s with the fixed algorithmic-byte formula of
SURVEY.md §8(d); the roofline object covers the dominant kernel
(the scaled-U sweep). The `tts` object is the GMRES+AMG time-to-solution part
of the metric (host setup + device solve) with the direct-sptrsv comparison
(`--no-tts` skips it).

Multi-GPU (torchrun, N > 1): every rank smooths its own C2-sized row block
(weak scaling, global residual through the NCCL halo exchange),
time = max over ranks. `tts.strong` is the distributed GMRES+AMG solve of the
one global C2 matrix over the N ranks (strong scaling, every N including 1).
`--strong` switches the whole line to BASELINE configs[3]: C4 =
poisson3d(465^3), 100.5 M rows, block-Jacobi ILU(0), fixed global size over the
N GPUs (`scaling: "strong"`).

`--impl reference` times the reference's own CPU code (oracle/_ref, the
unmodified reference library; its input from the oracle-side generators, no
product library loaded) on rank 0's host cores: concurrent ilu_smooth_sweep
calls on one shared smoother state (the reference's threading contract), on
the full matrix when the host has the memory for it, else on a slab.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("NCCL_DEBUG", "WARN")  # no init banner on stdout (one JSON line)

# stdout carries exactly one JSON line: the real stdout is kept aside and fd 1
# points at stderr for everything else (library banners such as NCCL's version
# line on communicator init, prints from native code)
_JSON_OUT = None


def emit(obj):
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(obj) + "\n")
    out.flush()


def _claim_stdout():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)

METRIC = "ILU sweep GB/s (% HBM peak); GMRES+AMG time-to-solution at 1/2/4/8 B200"
SPEC = "pressure27(256,256,256)"
SAMPLE_SPEC = "pressure27(256,256,16)"  # CPU baseline sample: 16 of the 256 z-planes
ILU_KV = {"smoother.kind": "ilu", "ilu.variant": "ilut", "ilu.droptol": "1e-3", "ilu.lfill": "5",
          "scaling": "row", "trisolve.mode": "richardson", "trisolve.m_lower": "5",
          "trisolve.m_upper": "5", "smoother.sweeps": "1"}
# BASELINE configs[3] (C4): 7-point Poisson 465^3 = 100.5 M rows, block-Jacobi ILU(0) row-scaled
C4_SPEC = "poisson3d(465,465,465)"
# BASELINE configs[0] / BASELINE.md §2 (C1): the reference's CPU-runnable case, GMRES+AMG
C1_SPEC = "poisson3d(64,64,64)"
C1_KV = {"smoother.kind": "ilu", "ilu.variant": "ilu0", "scaling": "row", "trisolve.mode": "richardson",
         "trisolve.m_lower": "5", "trisolve.m_upper": "5", "smoother.sweeps": "2",
         "smoother.fallback.kind": "gauss_seidel", "amg.coarsening": "pmis", "krylov.tol": "1e-8"}
C4_KV = dict(ILU_KV, **{"ilu.variant": "ilu0"})


def sweep_bytes(n, nnz):
    """One factor sweep / SpMV over a matrix with nnz stored entries (§8d)."""
    return 12 * nnz + 28 * n + 4


def step_bytes(n, nnz_a, nnz_l, nnz_u, m_l=5, m_u=5):
    """Algorithmic bytes of one ilu_smooth_sweep: residual, (m_L-1) L sweeps
    (+8n for the fused 1/row_scale of the last), (m_U-1) U sweeps (+8n for the
    x += z read of the last)."""
    return (sweep_bytes(n, nnz_a) + (m_l - 1) * sweep_bytes(n, nnz_l) + 8 * n
            + (m_u - 1) * sweep_bytes(n, nnz_u) + 8 * n)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.p is None:
            return
        time.sleep(0.1)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=5)
        for line in out.splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 7:
                self.rows.append(f)

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def host_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    mem_gb = None
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemAvailable"):
                    mem_gb = int(line.split()[1]) / 1e6
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model, "mem_available_gb": round(mem_gb, 1) if mem_gb else None}


def spec_rows(spec):
    dims = [int(t) for t in spec[spec.index("(") + 1:spec.index(")")].split(",")[:3]]
    return dims[0] * dims[1] * dims[2]


def ref_smoother_rate(spec, kv, max_steps, budget_s, threads=None):
    """The reference's own ilu_smooth_sweep (oracle/_ref: the unmodified
    reference library, single-threaded per call) on `spec`, built with the
    oracle-side generator (no product library in the process). Each step runs
    T concurrent calls on one shared smoother state with their own b/x — the
    reference's documented threading contract — so the host's cores and memory
    bandwidth are all in use; GB/s = T x algorithmic step bytes / step wall."""
    import ctypes as C
    import threading
    import numpy as np
    from oracle import oracle
    if not os.path.exists(oracle.REF_SO):
        return None
    ref = oracle.Ref()
    info = host_info()
    n = spec_rows(spec)
    # RSS model from the 1 M-row slab (measured): ~1.3 KB/row resident, ~0.3 KB/row per concurrent call
    base_gb, per_call_gb = 1.3e-6 * n, 0.3e-6 * n
    avail = info["mem_available_gb"] or 16.0
    T = threads or max(1, min(os.cpu_count() or 1, int((0.8 * avail - base_gb) / max(per_call_gb, 1e-9))))
    t0 = time.perf_counter()
    A = ref.gen3d(spec)
    st = ref.smoother(A, ref.cfg(kv))
    setup_s = time.perf_counter() - t0
    nr, nl, nu = C.c_int64(), C.c_int64(), C.c_int64()
    ref.L.ref_smoother_factor_nnz(st, C.byref(nr), C.byref(nl), C.byref(nu))
    ni, nn, nz = C.c_int64(), C.c_int64(), C.c_int64()
    ref.L.ref_mat_info(A, C.byref(ni), C.byref(nn), C.byref(nz))
    nrows = nr.value
    B = step_bytes(nrows, nz.value, nl.value, nu.value - nrows)
    bs = [np.random.default_rng(1 + t).uniform(-1, 1, nrows) for t in range(T)]

    def one(t):
        ref.ilu_smooth_sweep(A, st, bs[t], np.zeros(nrows))

    best, steps, t_start = 1e300, 0, time.perf_counter()
    while steps < max(1, max_steps):
        th = [threading.Thread(target=one, args=(t,)) for t in range(T)]
        t = time.perf_counter()
        for x in th:
            x.start()
        for x in th:
            x.join()
        best = min(best, time.perf_counter() - t)
        steps += 1
        if time.perf_counter() - t_start > budget_s:
            break
    ref.L.ref_smoother_free(st)
    ref.free_mat(A)
    gbs = T * B / best / 1e9
    return {"value": round(gbs, 4), "unit": "GB/s", "cores": T, "kind": "reference",
            "sample": f"{spec} (n={nrows}), ILUT(1e-3,5) row-scaled, one ilu_smooth_sweep m_L=m_U=5 per call via "
                      f"the reference library; {T} concurrent calls per step on one shared state, best of {steps} "
                      f"step(s), {best:.3f} s/step; reference setup (generate + ILUT + scaling) {setup_s:.1f} s",
            "host": info, "steps_timed": steps}


def ref_sweeps_only_rate(spec, kv, budget_s=20.0):
    """SURVEY.md §8d's fairness figure beside the reference's own call: the
    reference's sweep core alone — spmv_into (src/sparse.cpp:162-174) over its
    own pre-split strict row-scaled U, without the per-call split and
    allocations of richardson_upper_scaled (src/trisolve.cpp:123-147) — T
    concurrent calls (the GIL is released in the library), GB/s on the same
    per-sweep byte formula."""
    import threading
    import numpy as np
    from oracle import oracle
    if not os.path.exists(oracle.REF_SO):
        return None
    ref = oracle.Ref()
    A = ref.gen3d(spec)
    f = ref.scale(ref.ilu(A, ref.cfg(kv)), "row")
    _, (urp, uci, uv), _, _ = ref.factors_arrays(f)
    n = len(urp) - 1
    keep = np.ones(len(uci), dtype=bool)
    keep[urp[:-1][np.diff(urp) > 0]] = False  # every U row starts with its (unit) diagonal
    rp = np.concatenate([[0], np.cumsum(np.diff(urp) - (np.diff(urp) > 0))])
    Us = ref.mat(rp, uci[keep], uv[keep])
    nnz = int(rp[-1])
    T = os.cpu_count() or 1
    xs = [np.random.default_rng(7 + t).uniform(-1, 1, n) for t in range(T)]
    best, steps, t0 = 1e300, 0, time.perf_counter()
    while steps < 3 and time.perf_counter() - t0 < budget_s:
        th = [threading.Thread(target=ref.spmv, args=(Us, xs[t], n)) for t in range(T)]
        t = time.perf_counter()
        for x in th:
            x.start()
        for x in th:
            x.join()
        best = min(best, time.perf_counter() - t)
        steps += 1
    ref.free_mat(Us)
    ref.free_mat(A)
    return {"value": round(T * (12 * nnz + 28 * n + 4) / best / 1e9, 3), "unit": "GB/s", "cores": T,
            "sample": f"{spec}: one strict-U sweep core (spmv_into, pre-split U_s, nnz {nnz}) per call, "
                      f"{T} concurrent calls, best of {steps}",
            "note": "for comparison with the device U sweep (roofline.achieved), not with the smoother step"}


def cpu_baseline():
    """Bounded sample for the GPU arm's line (~10-30 s): the 16-plane slab."""
    return ref_smoother_rate(SAMPLE_SPEC, ILU_KV, max_steps=2, budget_s=15.0)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    spec = args.spec if not args.strong else C4_SPEC
    kv = ILU_KV if not args.strong else C4_KV
    info = host_info()
    need_gb = 1.3e-6 * spec_rows(spec) * 1.6  # resident state plus one concurrent call, with margin
    full = not args.ref_sample and info["mem_available_gb"] and info["mem_available_gb"] * 0.8 > need_gb
    sample = spec if full else (SAMPLE_SPEC if not args.strong else "poisson3d(465,465,16)")
    base = ref_smoother_rate(sample, kv, max_steps=max(1, args.steps), budget_s=90.0)
    if base is None:
        emit({"impl": "reference", "unavailable": "oracle/_ref not built"})
        return
    v = base["value"]
    # the reference's own time-to-solution at C1 (run_solve, src/driver.cpp:239-260; single-threaded)
    tts_c1 = None
    try:
        from oracle import oracle
        ref = oracle.Ref()
        A1 = ref.gen3d(C1_SPEC)
        rep = ref.run_solve(ref.arrays(A1), C1_KV)
        tts_c1 = {"spec": C1_SPEC, "iterations": int(rep["iterations"]), "converged": rep["converged"] == "true",
                  "setup_s": float(rep["setup_seconds"]), "solve_s": float(rep["solve_seconds"]),
                  "final_relres": float(rep["final_relres"]), "cores": 1}
    except Exception as e:  # report, never lose the line
        tts_c1 = {"error": str(e)[:200]}
    try:
        sweeps = ref_sweeps_only_rate(SAMPLE_SPEC if not args.strong else "poisson3d(465,465,16)", kv)
    except Exception as e:  # report, never lose the line
        sweeps = {"error": str(e)[:200]}
    why = None if full else (f"full {spec} needs ~{need_gb:.0f} GB host RAM in the reference's int64 CSR layout, "
                             f"{info['mem_available_gb']} GB available (or --ref-sample): a slab of the same "
                             f"matrix family with the same per-row work is timed")
    emit({
        "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": world, "steps": base["steps_timed"],
        "warmup": 0, "higher_is_better": True, "scaling": "strong" if args.strong else "weak",
        "impl": "reference", "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"ilu_smooth_sweep (m_L=m_U=5) on {sample}", "target_workload": spec,
                   "same_config": bool(full), "why_not_same": why,
                   "parallelism": f"reference CPU code, {base['cores']} concurrent calls on rank 0's host"},
        "cpu_baseline": base, "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "sweeps_only": sweeps, "tts": {"C1": tts_c1}, "vs_baseline": None})


def build_workload(ilug, args, rank, world, local, use_dist=False):
    """The smoother of this rank: N=1 the C2 matrix; N>1 the rank's 256^3 slab of
    pressure27(256,256,256N) (weak scaling), block-Jacobi ILUT factors of the
    local diagonal block, global residual with an NCCL halo exchange."""
    import ctypes as C
    cfg = ilug.Config().update(ILU_KV)
    if not use_dist:
        A = ilug.Matrix.generate(args.spec)
        S = ilug.Smoother(A, cfg)  # host ILUT + upload + K1 row scaling on the device
        v = [C.c_longlong() for _ in range(5)]
        ilug._check(ilug.lib.ilug_smoother_stats(S.h, *[C.byref(x) for x in v]))
        n, nnz_a, nnz_l, nnz_u, pad_u = (x.value for x in v)
        smooth = S.smooth
        once = lambda which, xin, rhs, out, st: ilug._check(ilug.lib.ilug_smoother_sweep_once(
            S.h, which, xin.data_ptr(), rhs.data_ptr(), out.data_ptr(), st.cuda_stream))
        host = lambda bs, xs: S.smooth_host_many(bs, xs)
        return dict(A=A, S=S, n=n, nnz_a=nnz_a, nnz_l=nnz_l, nnz_u=nnz_u, pad_u=pad_u, smooth=smooth, once=once,
                    host=host, spec=args.spec)
    import torch.distributed as dist
    from paper_2111_09512_b200 import dist as idist
    nx, ny, nz = (int(t) for t in args.spec[args.spec.index("(") + 1:args.spec.index(")")].split(",")[:3])
    spec = f"pressure27({nx},{ny},{nz * world})"
    n_g = nx * ny * nz * world
    starts = idist.partition(n_g, world)
    rows = idist.generate_rows(spec, int(starts[rank]), int(starts[rank + 1]))
    plan = idist.Plan(rows, n_g, world, rank)
    comm = dist_comm(rank, world, local)
    plan.exchange(comm)
    S = idist.Smoother(plan, comm, cfg)
    # the smoother holds everything it needs on the device: drop this rank's host
    # rows and plan (the strong-scaling solve that follows builds a global host
    # hierarchy on every rank; host memory is shared by all the ranks of a node)
    del rows, plan
    st = S.stats()
    once = lambda which, xin, rhs, out, stm: ilug._check(ilug.lib.ilug_dist_smoother_sweep_once(
        S.h, which, xin.data_ptr(), rhs.data_ptr(), out.data_ptr(), stm.cuda_stream))
    host = lambda bs, xs: S.smooth_host_many(bs, xs)
    return dict(A=None, S=S, comm=comm, n=st["nloc"], nnz_a=st["nnz_A"], nnz_l=st["nnz_Ls"],
                nnz_u=st["nnz_Us"], pad_u=0, smooth=S.smooth, once=once, host=host, spec=spec)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--spec", default=SPEC)
    ap.add_argument("--no-tts", action="store_true", help="skip the GMRES+AMG time-to-solution part")
    ap.add_argument("--no-tts-gs", action="store_true",
                    help="skip the Gauss-Seidel coarse fallback (the reference's default) in the TTS part")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tts-strong", action="store_true",
                    help="N = 1: also run the distributed-solver time-to-solution (the strong-scaling curve's first point)")
    ap.add_argument("--dist", action="store_true",
                    help="use the distributed (N > 1) code path even with one rank (validation)")
    ap.add_argument("--strong", action="store_true",
                    help="BASELINE configs[3]: C4 poisson3d(465^3), block-Jacobi ILU(0), fixed global size over N GPUs")
    ap.add_argument("--ref-sample", action="store_true",
                    help="reference arm: time the slab sample even when the host could hold the full matrix")
    args = ap.parse_args()
    _claim_stdout()
    if args.impl == "reference":
        return run_reference(args)
    if args.strong:
        return run_strong(args)

    import ctypes as C
    import torch
    import paper_2111_09512_b200 as ilug

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    use_dist = world > 1 or args.dist
    if use_dist:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ilug.lib.ilug_set_device(local)

    t0 = time.perf_counter()
    W = build_workload(ilug, args, rank, world, local, use_dist)
    setup_s = time.perf_counter() - t0
    n, nnz_a, nnz_l, nnz_u, pad_u = W["n"], W["nnz_a"], W["nnz_l"], W["nnz_u"], W["pad_u"]
    B = step_bytes(n, nnz_a, nnz_l, nnz_u)

    stream = torch.cuda.current_stream()
    g = torch.Generator(device="cpu").manual_seed(1234 + rank)
    b = torch.rand(n, dtype=torch.float64, generator=g).cuda() * 2 - 1
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    for _ in range(args.warmup):
        W["smooth"](b, x, stream=stream)
    torch.cuda.synchronize()

    def barrier():
        if use_dist:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(v):
        if not use_dist:
            return v
        import torch.distributed as dist
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            W["smooth"](b, x, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    value = B * world / (ms * 1e-3) / 1e9

    # ---- roofline: the dominant kernel (scaled-U sweep), timed alone on the same stream
    peak, peak_kind = peaks()
    xin = torch.rand(n, dtype=torch.float64, generator=g).cuda()
    out = torch.empty_like(xin)
    reps = 50
    kern = {}
    for which, name, nnz in ((1, "u_sweep", nnz_u), (0, "l_sweep", nnz_l)):
        for _ in range(3):
            W["once"](which, xin, b, out, stream)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            W["once"](which, xin, b, out, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        kms = max_over_ranks(e0.elapsed_time(e1) / reps)
        kern[name] = {"ms": kms, "gbs": sweep_bytes(n, nnz) / (kms * 1e-3) / 1e9, "bytes": sweep_bytes(n, nnz)}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "u_sweep_traffic.json")
    if os.path.exists(tpath) and not use_dist:
        with open(tpath) as fh:
            traffic = json.load(fh).get("dram_bytes_per_launch")
    ach = kern["u_sweep"]["gbs"]
    roofline = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": traffic, "peak_source": peak_kind,
                "kernel": "k_rowdot<EpiResidual> on strict row-scaled U (SELL-32, sigma-sorted, D8-coded columns)",
                "bytes_rule": "SURVEY 8d formula 12*nnz+28n+4 (4 B per index; the 1-byte column stream is not credited)",
                "bytes_per_launch": kern["u_sweep"]["bytes"], "ms_per_launch": round(kern["u_sweep"]["ms"], 5),
                "frac_of_8TBs_nominal": round(ach / 8000.0, 4),
                "l_sweep_gbs": round(kern["l_sweep"]["gbs"], 1)}

    # ---- e2e through the public host-buffer API: every step copies its b and x
    # in from pinned host memory and its x out (ilug_smooth_host_many pipelines
    # step i's smoothing with step i+1's H2D and step i-1's D2H over three
    # device slots; three host pairs rotate, so each step's input is the output
    # of that pair's previous use, which the pipeline waits for)
    NP = 3
    pairs = [(torch.empty(n, dtype=torch.float64, pin_memory=True), torch.zeros(n, dtype=torch.float64,
                                                                               pin_memory=True)) for _ in range(NP)]
    for bh, _ in pairs:
        bh.copy_(b.cpu())
    e2e_steps = max(6, min(args.steps, 48))  # enough steps that the pipeline fill and drain amortise
    seq_b = [pairs[i % NP][0] for i in range(e2e_steps)]
    seq_x = [pairs[i % NP][1] for i in range(e2e_steps)]
    W["host"](seq_b[:NP], seq_x[:NP])  # warm-up (streams, staging slots)
    barrier()
    t = time.perf_counter()
    W["host"](seq_b, seq_x)
    e2e_s = max_over_ranks((time.perf_counter() - t) / e2e_steps)
    e2e = {"value": round(B * world / e2e_s / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": 16 * n * world,
           "d2h_bytes_per_step": 8 * n * world, "ms_per_step": round(e2e_s * 1e3, 3), "steps": e2e_steps,
           "api": "ilug_smooth_host_many / ilug_dist_smooth_host_many (pinned host b, x; copies pipelined "
                  "with the previous/next step's smoothing)"}

    res = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"ilu_smooth_sweep (m_L=m_U=5, row-scaled ILUT(1e-3,5)) on {W['spec']}"
                               + ("" if not use_dist else " (rank slabs of 256^3, block-Jacobi, NCCL halo)"),
                   "n_per_gpu": n, "nnz_A": nnz_a, "nnz_L_strict": nnz_l, "nnz_U_strict": nnz_u,
                   "sell_padding_U": round(pad_u / max(nnz_u, 1) - 1, 4) if pad_u else None, "bytes_per_step": B,
                   "l2": "inputs (>= 5 GB per step) exceed the 126 MB L2; no flush needed",
                   "parallelism": f"row-block x{world} (weak)", "host_setup_s": round(setup_s, 2)},
        "frac_of_peak": round(value / world / peak, 4),
        "roofline": roofline, "e2e": e2e, "clocks": clk.summary(),
        "gpu_launches": 9 * args.steps,
    }
    if not args.no_tts and not use_dist:
        res["tts"] = time_to_solution(ilug, W["A"], ("poly_gs",) if args.no_tts_gs else ("poly_gs", "gauss_seidel"))
    if not args.no_tts and (use_dist or args.tts_strong):
        # the distributed solve of the ONE global C2 matrix over the N ranks: the
        # strong-scaling time-to-solution curve (also at N = 1 with --tts-strong)
        kv = dict(ILU_KV, **{"smoother.sweeps": "2", "krylov.tol": "1e-8", "amg.coarsening": "pmis",
                             "krylov.form_iterates": "false", "smoother.fallback.kind": "poly_gs"})
        try:
            comm = W.get("comm") or dist_comm(rank, world, local)
            tts_s = strong_solve(ilug, args.spec, kv, (rank, world, comm), barrier, max_over_ranks)
        except Exception as e:  # report, never lose the bench line
            tts_s = {"error": str(e)[:300]}
        if rank == 0:
            res.setdefault("tts", {})["strong"] = tts_s
    if rank == 0 and not use_dist and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline()
        if not args.no_tts:
            res["tts"]["C1"] = c1_tts(ilug)
    if rank == 0:
        emit(res)
    if use_dist:
        import torch.distributed as dist
        del W
        dist.destroy_process_group()


def strong_solve(ilug, spec, kv, comm_args, barrier, max_over_ranks, hierarchy=None):
    """Distributed GMRES+AMG of ONE global matrix over the ranks (strong
    scaling): every rank holds the global host hierarchy (redundant host setup)
    and builds the device objects of its rows at every level (A/R/P halo
    plans, block-Jacobi ILU on the finest level, rank-local smoothers below,
    replicated coarsest solve); global (F)GMRES with summed CGS2 reductions.
    Setup and solve are timed as the max over ranks."""
    import torch
    from paper_2111_09512_b200 import dist as idist
    rank, world, comm = comm_args
    cfg = ilug.Config().update(kv)
    barrier()
    t = time.perf_counter()
    A = ilug.Matrix.generate(spec)
    # the global hierarchy, built on this rank's GPU (device AMG setup, PMIS + direct)
    H = hierarchy or ilug.Hierarchy(A, ilug.Config().update(dict(kv, **{"device.amg_setup": "device"})),
                                    host_only=True)
    host_s = max_over_ranks(time.perf_counter() - t)
    t = time.perf_counter()
    solver = idist.Solver(H, comm)
    torch.cuda.synchronize()
    dev_s = max_over_ranks(time.perf_counter() - t)
    # the reference driver's default right-hand side, b = A * ones (src/config.cpp:334-337)
    import numpy as np
    rp, _, v = A.csr()
    r0, r1 = solver.row0, solver.row0 + solver.nloc
    b = torch.from_numpy(np.add.reduceat(v[:rp[r1]], rp[r0:r1]) if r1 > r0 else np.zeros(0)).cuda()
    x = torch.zeros_like(b)
    # the solver keeps only device data: release this rank's copies of the global
    # matrix and hierarchy before the solve (all ranks of a node share its RAM)
    del rp, v, A, H
    # warm-up (lazy module loading) outside the timed solve
    solver.gmres(ilug.Config().update(dict(kv, **{"krylov.max_iters": "2"})), b, x)
    x.zero_()
    torch.cuda.synchronize()
    barrier()
    t = time.perf_counter()
    out = solver.gmres(cfg, b, x)
    torch.cuda.synchronize()
    solve = max_over_ranks(time.perf_counter() - t)
    return {"spec": spec, "ranks": world, "iterations": out["iterations"], "converged": out["status"] == 0,
            "final_relres": out["final_relres"], "levels": solver.levels, "host_setup_s": round(host_s, 3),
            "device_setup_s": round(dev_s, 3), "solve_s": round(solve, 4),
            "preconditioner": "row-block distributed AMG: A/R/P halo-exchanged per level, block-Jacobi "
                              f"{kv.get('ilu.variant', 'ilu0')} smoother on the finest level, "
                              f"{kv.get('smoother.fallback.kind', 'gauss_seidel')} (rank-local) below, "
                              "replicated coarsest solve"}


class stdout_to_stderr:
    """fd-level redirect: library banners (NCCL prints its version on init)
    must not reach stdout, which carries exactly one JSON line."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)

    def __exit__(self, *a):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


def dist_comm(rank, world, local):
    """NCCL communicator of this rank (torch.distributed only broadcasts the id)."""
    from paper_2111_09512_b200 import dist as idist
    with stdout_to_stderr():
        if world == 1:
            return idist.Comm(1, 0, idist.unique_id())
        import torch.distributed as dist
        uid = [idist.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        return idist.Comm(world, rank, uid[0])


def run_strong(args):
    """C4 (BASELINE configs[3]) at fixed global size over N GPUs: value = the
    aggregate GB/s of the block-Jacobi ILU(0) smoother step on the ranks' rows
    (global residual through the NCCL halo exchange), `tts` = the distributed
    GMRES+AMG solve."""
    import torch
    import paper_2111_09512_b200 as ilug
    from paper_2111_09512_b200 import dist as idist
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ilug.lib.ilug_set_device(local)
    spec = args.spec if args.spec != SPEC else C4_SPEC

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        import torch.distributed as dist
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    comm = dist_comm(rank, world, local)
    n_g = spec_rows(spec)
    starts = idist.partition(n_g, world)
    t0 = time.perf_counter()
    plan = idist.Plan(idist.generate_rows(spec, int(starts[rank]), int(starts[rank + 1])), n_g, world, rank)
    plan.exchange(comm)
    S = idist.Smoother(plan, comm, ilug.Config().update(C4_KV))
    del plan  # the smoother keeps only device data (host RAM is shared by the node's ranks)
    setup_s = max_over_ranks(time.perf_counter() - t0)
    st = S.stats()
    n, B = st["nloc"], step_bytes(st["nloc"], st["nnz_A"], st["nnz_Ls"], st["nnz_Us"])
    stream = torch.cuda.current_stream()
    g = torch.Generator(device="cpu").manual_seed(1234 + rank)
    b = torch.rand(n, dtype=torch.float64, generator=g).cuda() * 2 - 1
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    for _ in range(args.warmup):
        S.smooth(b, x, stream=stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            S.smooth(b, x, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    B_all = max_over_ranks(0.0) if False else B  # per-rank bytes; the aggregate below sums the ranks
    if world > 1:
        import torch.distributed as dist
        tb = torch.tensor([float(B)], dtype=torch.float64, device="cuda")
        dist.all_reduce(tb)
        B_all = float(tb.item())
    value = B_all / (ms * 1e-3) / 1e9
    peak, peak_kind = peaks()
    # e2e: host buffers through ilug_dist_smooth_host_many (copies inside the timed region)
    NP = 3  # three rotating host pairs: the pipeline's three device slots overlap copies and compute
    pairs = [(torch.empty(n, dtype=torch.float64, pin_memory=True), torch.zeros(n, dtype=torch.float64,
                                                                               pin_memory=True)) for _ in range(NP)]
    for bh, _ in pairs:
        bh.copy_(b.cpu())
    e2e_steps = max(6, min(args.steps, 12))
    S.smooth_host_many([pq[0] for pq in pairs], [pq[1] for pq in pairs])
    barrier()
    t = time.perf_counter()
    S.smooth_host_many([pairs[i % NP][0] for i in range(e2e_steps)], [pairs[i % NP][1] for i in range(e2e_steps)])
    e2e_s = max_over_ranks((time.perf_counter() - t) / e2e_steps)
    res = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"ilu_smooth_sweep (m_L=m_U=5, row-scaled block-Jacobi ILU(0)) on {spec} "
                               f"(BASELINE configs[3], fixed global size)", "n_global": n_g, "n_per_gpu": n,
                   "bytes_per_step_all_ranks": B_all,
                   "l2": "inputs (>= 1 GB per rank per step) exceed the 126 MB L2; no flush needed",
                   "parallelism": f"row-block x{world} (strong), NCCL halo", "smoother_setup_s": round(setup_s, 2)},
        "frac_of_peak": round(value / world / peak, 4),
        "e2e": {"value": round(B_all / e2e_s / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": 16 * n_g,
                "d2h_bytes_per_step": 8 * n_g, "ms_per_step": round(e2e_s * 1e3, 3), "steps": e2e_steps,
                "api": "ilug_dist_smooth_host_many (pinned host b, x per rank)"},
        "clocks": clk.summary(), "gpu_launches": 9 * args.steps,
    }
    del S
    if not args.no_tts:
        kv = dict(C4_KV, **{"smoother.sweeps": "2", "krylov.tol": "1e-8", "amg.coarsening": "pmis",
                            "krylov.form_iterates": "false", "smoother.fallback.kind": "poly_gs"})
        try:
            res["tts"] = {"strong": strong_solve(ilug, spec, kv, (rank, world, comm), barrier, max_over_ranks)}
        except Exception as e:  # report, never lose the bench line
            res["tts"] = {"strong": {"error": str(e)[:300]}}
    if rank == 0:
        emit(res)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def c1_tts(ilug):
    """C1 (BASELINE.md §2 keys) through iluamg_run_solve on the GPU, next to the
    reference's run_solve on one host core (oracle/_ref, the same call the
    reference arm makes). Small: ~0.3 s on the device, ~5 s on the CPU."""
    out = {}
    A = ilug.Matrix.generate(C1_SPEC)
    ilug.run_solve(A, ilug.Config().update(C1_KV))  # warm-up (module loading)
    rep = ilug.run_solve(A, ilug.Config().update(C1_KV))
    out["device"] = {"spec": C1_SPEC, "iterations": int(rep["iterations"]), "converged": rep["converged"] == "true",
                     "setup_s": float(rep["setup_seconds"]), "solve_s": float(rep["solve_seconds"]),
                     "final_relres": float(rep["final_relres"])}
    try:
        from oracle import oracle
        if os.path.exists(oracle.REF_SO):
            ref = oracle.Ref()
            r = ref.run_solve(ref.arrays(ref.gen3d(C1_SPEC)), C1_KV)
            out["reference_cpu_1core"] = {"iterations": int(r["iterations"]), "converged": r["converged"] == "true",
                                          "setup_s": float(r["setup_seconds"]),
                                          "solve_s": float(r["solve_seconds"])}
            out["speedup_solve"] = round(out["reference_cpu_1core"]["solve_s"] / out["device"]["solve_s"], 1)
            rc, dv = out["reference_cpu_1core"], out["device"]
            out["speedup_total"] = round((rc["setup_s"] + rc["solve_s"]) / (dv["setup_s"] + dv["solve_s"]), 1)
    except Exception as e:
        out["reference_cpu_1core"] = {"error": str(e)[:200]}
    return out


def time_to_solution(ilug, A, fallbacks=("poly_gs",)):
    """GMRES+AMG (relres 1e-8, PMIS, ILUT(1e-3,5) row-scaled smoother on the
    finest level, 2 sweeps) through iluamg_run_solve: iterative (m_L = m_U = 5
    Richardson sweeps) vs direct (level-scheduled) triangular solves, for each
    coarse-level fallback smoother. poly_gs is the GPU-friendly fallback (SpMV
    based); gauss_seidel is the reference default (latency-bound level
    scheduling on unstructured coarse grids). krylov.form_iterates=false: one
    V-cycle per iteration (iteration counts unchanged, see tests)."""
    out = {}
    for fb in fallbacks:
        res = {}
        base = dict(ILU_KV, **{"smoother.sweeps": "2", "krylov.tol": "1e-8", "amg.coarsening": "pmis",
                               "krylov.form_iterates": "false", "smoother.fallback.kind": fb})
        modes = ("richardson", "direct") + (("direct_cusparse",) if fb == "poly_gs" else ())
        for mode in modes:
            # direct_cusparse: the same direct solve through cuSPARSE SpSV (ILUG_DIRECT=cusparse),
            # the library comparison point for the level-scheduled K5 kernels
            kv = dict(base, **{"trisolve.mode": "direct" if mode == "direct_cusparse" else mode})
            if mode == "direct_cusparse":
                os.environ["ILUG_DIRECT"] = "cusparse"
            # warm-up on a small matrix: lazy module loading of every kernel the
            # solve uses happens here, not inside the timed solve below
            ilug.run_solve(ilug.Matrix.generate("pressure27(24,24,24)"), ilug.Config().update(kv))
            try:
                rep = ilug.run_solve(A, ilug.Config().update(kv))
            finally:
                os.environ.pop("ILUG_DIRECT", None)
            res[mode] = {"iterations": int(rep["iterations"]), "converged": rep["converged"] == "true",
                         "setup_s": float(rep["setup_seconds"]), "solve_s": float(rep["solve_seconds"]),
                         "final_relres": float(rep["final_relres"]), "levels": int(rep["levels"]),
                         "vcycles": int(rep["device_vcycles"])}
        res["speedup_iterative_vs_direct"] = round(res["direct"]["solve_s"] / res["richardson"]["solve_s"], 3)
        if "direct_cusparse" in res:
            res["speedup_iterative_vs_cusparse_direct"] = round(
                res["direct_cusparse"]["solve_s"] / res["richardson"]["solve_s"], 3)
        # against the faster direct solve, and end to end (setup + solve)
        best = min((res[m] for m in ("direct", "direct_cusparse") if m in res), key=lambda r: r["solve_s"])
        it = res["richardson"]
        res["speedup_iterative_vs_best_direct"] = round(best["solve_s"] / it["solve_s"], 3)
        res["speedup_total_vs_best_direct"] = round((best["setup_s"] + best["solve_s"]) /
                                                    (it["setup_s"] + it["solve_s"]), 3)
        out[f"fallback_{fb}"] = res
    return out


if __name__ == "__main__":
    main()
