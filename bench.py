#!/usr/bin/env python
"""VeST CD-sweep benchmark (BASELINE.json metric: observed-nnz*iter/s).

Headline workload (BASELINE.json configs[3], "config 4" -- the largest
configuration, fits one B200): 4-mode 1M^4 tensor, 200M observed entries at
uniform-random distinct coordinates, values N(0,1) rounded to fp32 (held as
fp64), Tucker ranks 8x8x8x8 with the core pruned to 10% nonzero (a seeded 90%
core mask in the initial model), lambda = 0.01 (LF),
init_random(7) factors.  A step = one CD iteration as fit() runs it
(trainer.hpp:121-127): update_all_factors + update_core + residuals/RE over all
200M entries.  Config 2 (3-mode 100k^3, 10M entries, R 10^3; the round-1
headline) is measured after it as a secondary key.  Prune events
(responsibilities + prune) are timed separately ("prune_event").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

ours:       device-resident steps, CUDA events on the library stream ("value");
            the same steps through the C-ABI with host model buffers, H2D+D2H
            inside the timed region ("e2e"); kernel-family times for the
            roofline; the reference CPU path timed on a bounded sample
            ("cpu_baseline").
reference:  the reference's own CPU implementation (oracle/_ref: the
            unmodified reference headers; the C port when _ref is absent) on a
            bounded sample of the same workload (same dims, ranks, core mask,
            lambda and value distribution; fewer entries, stated in `config`),
            all host threads.  It never loads the repo's CUDA library.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CD sweep observed-nnz*iter/s"
UNIT = "nnz*iter/s"
HEADLINE = 4
SECONDARY = 2
# CPU reference samples: entries per step (same dims/ranks/mask/distribution)
SAMPLE_NNZ = {1: 100_000, 2: 300_000, 3: 300_000, 4: 500_000, 5: 200_000}


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def synth(dims, nnz, seed, values_kind=0, zipf=None):
    from paper_1904_02603_b200 import _lib
    L = _lib.lib()
    d = np.asarray(dims, np.uint64)
    z = np.asarray(zipf if zipf else [0.0] * len(dims), np.float64)
    coords = np.empty(nnz * len(dims), np.uint32)
    vals = np.empty(nnz, np.float64)
    _lib.check(L.vest_synth(len(dims), _lib.ptr(d, _lib.u64p), nnz, _lib.ptr(z, _lib.f64p), values_kind, seed,
                            _lib.ptr(coords, _lib.u32p), _lib.ptr(vals, _lib.f64p)))
    return coords.reshape(nnz, len(dims)), vals


# --------------------------------------------------------------- algorithmic --
def contraction_fmas(ranks, n):
    """FMA count per entry of the factorised delta contraction for mode n, as
    the static kernel executes it (vest_common.cuh delta_static):
    T(k) = J_k (T(k+1) + 1) for k < N-1, T(N-1) = J_{N-1}, T(N) = 0;
    n == 0: J_1 J_0 (T(2) + 1);  n > 0: J_0 P(1) with P(k) = J_k (1 + P(k+1))
    for k < n and P(n) = J_n (T(n+1) + 1)."""
    N = len(ranks)

    def T(k):
        if k >= N:
            return 0
        if k == N - 1:
            return ranks[k]
        return ranks[k] * (T(k + 1) + 1)

    def P(k):
        if k == n:
            return ranks[n] * (T(n + 1) + 1)
        return ranks[k] * (1 + P(k + 1))

    if n == 0:
        return ranks[1] * ranks[0] * (T(2) + 1)
    return ranks[0] * P(1)


def step_flops_per_entry(ranks, core_unmasked=None):
    """SURVEY.md 8(d) F_alg: reference-equivalent flops per entry x iteration,
    sum_n [dense-factorised delta + J_n (J_n + 1) + 2 J_n] + |G_u| (N + 7) + 2,
    dense-factorised delta = 2 (|G| + |G|/J_a + ...) over the N-1 contractions
    (largest J first)."""
    N = len(ranks)
    G = 1
    for J in ranks:
        G *= J
    Gu = G if core_unmasked is None else core_unmasked
    total = 0
    for n in range(N):
        others = sorted((ranks[k] for k in range(N) if k != n), reverse=True)
        d, size = 0, G
        for Ja in others:
            d += size
            size //= Ja
        total += min(2 * d, Gu * N) + ranks[n] * (ranks[n] + 1) + 2 * ranks[n]
    return total + Gu * (N + 7) + 2


# ------------------------------------------------------------------ clocks --
class Clocks:
    FIELDS = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active," \
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index):
        self.index = index
        self.p = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}_{id(self):x}.csv")

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
            self.f.close()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines()]
        except Exception:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) < 9:
                continue
            for k, nm in enumerate(names):
                if r[5 + k].strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- workloads --
def core_mask(ranks, keep):
    """Seeded core mask ("core pruned to 10% nonzero"
    as a 90% mask in the initial model, identical for the GPU and the CPU arm)."""
    rng = np.random.default_rng(44)
    return (rng.random(int(np.prod(ranks))) >= keep).astype(np.uint8)


def model_for(c):
    """init_random(dims, ranks, 7) (tucker_model.hpp:88-108) + the config's core mask."""
    from paper_1904_02603_b200 import sparsetuck as st
    m = st.init_random(c["dims"], c["ranks"], 7)
    if c["core_keep"] < 1.0:
        mask = core_mask(c["ranks"], c["core_keep"]).reshape(m.core.shape)
        m.core[mask == 1] = 0.0
        m.core_mask = mask
    return m


def synth_numpy(dims, nnz, seed, values_kind=0):
    """Seeded sample for the CPU arms, made with numpy only (the reference arm
    must not load the repo's CUDA library): uniform distinct coordinates
    (duplicates dropped; at 1M^4 there are none in practice), values U[0,1)
    (kind 0), integers 1..5 (kind 1) or N(0,1) rounded to float (kind 2)."""
    rng = np.random.default_rng(seed)
    c = np.stack([rng.integers(0, int(d), nnz, dtype=np.int64) for d in dims], 1).astype(np.uint32)
    c = np.unique(c, axis=0)  # canonical row-major order, distinct
    n = len(c)
    if values_kind == 1:
        v = rng.integers(1, 6, n).astype(np.float64)
    elif values_kind == 2:
        v = rng.standard_normal(n).astype(np.float32).astype(np.float64)
    else:
        v = rng.random(n)
    return c, v


def cpu_session(cfg_id, nnz, threads):
    """The reference CPU path (oracle/_ref = the unmodified reference headers
    when built, else the C port) on a bounded sample of config `cfg_id`: the
    config's dims, ranks, lambda, value distribution, initial model and core
    mask, `nnz` entries."""
    from oracle import oracle as O  # test/baseline infrastructure only
    kind = "reference" if O.available("reference") else "port"
    c = CONFIGS[cfg_id]
    coords, vals = synth_numpy(c["dims"], nnz, 77 + cfg_id, c["values_kind"])
    s = O.Session(c["dims"], coords, vals, c["ranks"], kind)
    s.init_random(7)
    if c["core_keep"] < 1.0:
        core, cm, fs, ms = s.get_model()
        mask = core_mask(c["ranks"], c["core_keep"]).reshape(core.shape)
        core[mask == 1] = 0.0
        s.set_model(core, mask, fs, ms)
    return s, kind, len(vals)


def sample_desc(cfg_id, nnz):
    c = CONFIGS[cfg_id]
    return (f"config{cfg_id} shape ({'x'.join(str(d) for d in c['dims'])}, ranks {c['ranks']}, core keep "
            f"{c['core_keep']}, lambda {c['lam']}) with {nnz} uniform entries (numpy-seeded) per step; dims kept "
            f"so the factor gathers miss cache as at full size")


def cpu_reference_rate(cfg_id, steps=2):
    threads = os.cpu_count() or 1
    s, kind, nnz = cpu_session(cfg_id, SAMPLE_NNZ[cfg_id], threads)
    c = CONFIGS[cfg_id]
    s.cd_iteration(0, c["lam"], threads)  # warm-up (first touch, page-in)
    t0 = time.perf_counter()
    for _ in range(steps):
        s.cd_iteration(0, c["lam"], threads)
    dt = (time.perf_counter() - t0) / steps
    return nnz / dt, kind, threads, dt, nnz


def run_reference_arm(args, rank):
    """`--impl reference`: the reference's own CPU implementation of the path
    (oracle/_ref) on the host cores, each step one CD iteration over a bounded
    sample of the headline workload.  Rank 0 only under torchrun."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    cfg_id = args.workload
    c = CONFIGS[cfg_id]
    s, kind, nnz = cpu_session(cfg_id, SAMPLE_NNZ[cfg_id], threads)
    for _ in range(args.warmup):
        s.cd_iteration(0, c["lam"], threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s.cd_iteration(0, c["lam"], threads)
    dt = time.perf_counter() - t0
    value = nnz * args.steps / dt
    cfgd = workload_config(cfg_id, args.gpus)
    cfgd["nnz"] = nnz
    cfgd["sample"] = sample_desc(cfg_id, nnz)
    cfgd["parallelism"] = f"OpenMP, {threads} host threads"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfgd,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": sample_desc(cfg_id, nnz)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(cfg_id, n):
    c = CONFIGS[cfg_id]
    return {"workload": f"config{cfg_id}: {c['desc']}; step = update_all_factors + update_core + RE "
                        f"(trainer.hpp:121-127)",
            "nnz": c["nnz"], "ranks": c["ranks"], "dims": c["dims"], "lambda": c["lam"],
            "core_keep": c["core_keep"],
            "values": {0: "fp64 U[0,1)", 1: "integers 1..5 as fp64", 2: "N(0,1) rounded to fp32, held as fp64"}[
                c["values_kind"]],
            "parallelism": (f"rows sharded x{n} (NCCL)" if n > 1 or os.environ.get("VEST_FORCE_SHARDED") == "1"
                            else "single"),
            "l2": "inputs larger than L2 (per-mode CSF >= 600 MB vs 126 MB L2)"}


# ----------------------------------------------------------- roofline ---------
def dense_delta_flops(ranks, n):
    """dense-factorised delta cost 2 (|G| + |G|/J_a + ...) over the
    N-1 contractions of mode n (largest J first)."""
    G = int(np.prod(ranks))
    others = sorted((ranks[k] for k in range(len(ranks)) if k != n), reverse=True)
    d, size = 0, G
    for Ja in others:
        d += size
        size //= Ja
    return 2 * d


def family_models(ranks, nnz, core_live):
    """Algorithmic (reference-equivalent) flops and compulsory
    bytes per entry of the two big families: one factor-mode update (averaged
    over modes) and one whole core sweep."""
    N = len(ranks)
    f_fl = np.mean([min(dense_delta_flops(ranks, n), core_live * N) + ranks[n] * (ranks[n] + 1) + 2 * ranks[n]
                    for n in range(N)])
    f_by = (N - 1) * 4 + 8
    c_fl = core_live * (N + 7)
    c_by = 4 * N + 8 + 16
    return float(f_fl), float(f_by), float(c_fl), float(c_by)


def roofline_for(c, fams, steps, ms_total, peak_tf, hbm_peak, core_live, nnz_local, traffic_db):
    """Roofline of the dominant kernel family of the step (largest share of
    the timed region): achieved = algorithmic flops per launch / average launch
    time (CUDA events on the library stream), against the measured FP64 peak."""
    ranks = c["ranks"]
    f_fl, f_by, c_fl, c_by = family_models(ranks, nnz_local, core_live)
    fac_ms = fams["factor_update"]["ms"] + fams["factor_update_fused_residual"]["ms"]
    fac_n = fams["factor_update"]["scopes"] + fams["factor_update_fused_residual"]["scopes"]
    core_ms = fams["core_pass"]["ms"]
    core_n = fams["core_pass"]["scopes"]
    if fac_ms >= core_ms and fac_n:
        avg = fac_ms / fac_n
        fl, by = f_fl * nnz_local, f_by * nnz_local
        kernel = "factor-mode update (per mode: " + ("mask-specialised delta + statistics/solve"
                                                     if c["core_keep"] < 1.0 else "k_rowpass<kStats>") + ")"
        fam = "factor_update"
        share = fac_ms / ms_total
    else:
        avg = core_ms / max(core_n, 1)
        sweeps = steps
        fl = c_fl * nnz_local * sweeps / max(core_n, 1)
        by = c_by * nnz_local * sweeps / max(core_n, 1)
        kernel = ("core-sweep block pass (per pass; one sweep's algorithmic work spread over its passes; "
                  + ("vest_cp_* plan-specialised)" if len(ranks) > 3 else "all-prefix statistics/group passes)"))
        fam = "core_pass"
        share = core_ms / ms_total
    ach = fl / (avg * 1e-3) / 1e12
    ach_b = by / (avg * 1e-3) / 1e9
    prof = traffic_db.get(fam) or {}
    return {
        "bound": "fp64", "kernel": kernel, "family": fam, "achieved": ach, "peak": peak_tf, "unit": "TFLOP/s",
        "frac": ach / peak_tf,
        "peak_source": "measured live in this run: vest_measure_fp64_peak (DFMA microbenchmark, 1184 CTAs x 256 "
                       "threads x 8 chains x 32768 FMA, best of 5)",
        "traffic": prof.get("traffic"), "flops_per_launch": fl, "avg_launch_ms": avg, "step_share": share,
        "ncu": {k: v for k, v in prof.items() if k != "traffic"} or None,
        "hbm": {"achieved": ach_b, "peak": hbm_peak, "unit": "GB/s", "frac": ach_b / hbm_peak,
                "bytes_per_launch": by, "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
    }


# --------------------------------------------------------------- our arm ------
def measure(dev, c, steps, warmup, world, dist, local_rank, L, _lib, torch, families=True):
    """Timed region: `steps` CD iterations, device-resident, CUDA events on the
    library stream, barrier + synchronize on both sides, max over ranks."""
    stream = torch.cuda.ExternalStream(dev.stream(), device=torch.device("cuda", local_rank))
    for _ in range(warmup):
        dev.cd_iteration(0, c["lam"])
    L.vest_ctx_profile(dev.h, 1 if families else 0)
    ms_arr = np.zeros(8)
    n_arr = np.zeros(8, np.uint64)
    L.vest_ctx_profile_read(dev.h, _lib.ptr(ms_arr, _lib.f64p), _lib.ptr(n_arr, _lib.u64p), 1)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    launches0 = L.vest_launch_count()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    res = [dev.cd_iteration(0, c["lam"]) for _ in range(steps)]
    ev1.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    launches = L.vest_launch_count() - launches0
    ms = ev0.elapsed_time(ev1)
    L.vest_ctx_profile_read(dev.h, _lib.ptr(ms_arr, _lib.f64p), _lib.ptr(n_arr, _lib.u64p), 1)
    L.vest_ctx_profile(dev.h, 0)
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    fam_names = ["factor_update", "core_pass", "core_gemm", "core_solve", "residual", "resp", "prune",
                 "factor_update_fused_residual"]
    fams = {fam_names[i]: {"ms": float(ms_arr[i]), "scopes": int(n_arr[i])} for i in range(8)}
    return ms, res, fams, int(launches)


def measure_e2e(dev, c, steps, dist, torch):
    """The same iteration through the C-ABI host entry point
    (vest_cd_iteration_host): the model is copied in from pinned host memory
    and the updated core and factors are read back inside the timed region."""
    from paper_1904_02603_b200 import sparsetuck as st
    m_host = dev.get_model()
    pinned = []

    def pin(a):
        t = torch.empty(a.shape, dtype={np.float64: torch.float64, np.uint8: torch.uint8}[a.dtype.type],
                        pin_memory=True)
        t.numpy()[...] = a
        pinned.append(t)
        return t.numpy()

    m_host = st.TuckerModel(m_host.dims, m_host.ranks, pin(m_host.core), pin(m_host.core_mask),
                            [pin(f) for f in m_host.factors], [pin(k) for k in m_host.factor_masks])
    h2d = m_host.core.nbytes + m_host.core_mask.nbytes + sum(f.nbytes + k.nbytes for f, k in
                                                              zip(m_host.factors, m_host.factor_masks))
    d2h = m_host.core.nbytes + sum(f.nbytes for f in m_host.factors)  # masks are inputs only
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        dev.cd_iteration_host(m_host, 0, c["lam"])
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    return e2e_s, int(h2d), int(d2h)


def run_ours(args, rank, world, local_rank):
    import torch
    from paper_1904_02603_b200 import _lib
    from paper_1904_02603_b200 import sparsetuck as st

    torch.cuda.set_device(local_rank)
    dist = None
    # VEST_FORCE_SHARDED=1: the sharded driver + NCCL hooks even at world size 1
    # (exercises the multi-GPU plumbing on a single GPU; diagnostic only)
    sharded = world > 1 or os.environ.get("VEST_FORCE_SHARDED") == "1"
    if sharded:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    L = _lib.lib()
    cfg_id = args.workload
    c = CONFIGS[cfg_id]
    coords, vals = synth(c["dims"], c["nnz"], 1000 + cfg_id, c["values_kind"], c["zipf"])
    x = st.SparseTensor(c["dims"], coords, vals)
    del coords, vals
    if sharded:
        # rows of every mode sharded by work-balanced ranges; NCCL exchanges
        # (paper_1904_02603_b200/sharded.py)
        from paper_1904_02603_b200 import sharded as sh
        comm = sh.TorchComm("cuda") if os.environ.get("VEST_TORCH_COMM") == "1" else sh.NcclNative()
        dev = sh.ShardDevice(x, c["ranks"], rank, world, comm, local_rank)
        nnz_local = dev.local_nnz(len(c["dims"]) - 1)
    else:
        dev = st.Device(x, c["ranks"], local_rank)
        nnz_local = c["nnz"]
    m0 = model_for(c)
    core_live = int(np.count_nonzero(m0.core_mask == 0))
    gf32 = bool(c.get("gather_f32")) and not args.fp64_gathers
    alt = None
    if gf32:
        # BASELINE config 4 is the fp32 configuration: the generated kernels
        # run their fp32 mode -- fp32 copies of the gathered factor rows, fp32
        # contraction of delta and of the core passes' fiber products, fp32 delta
        # and chunk statistics between kernels; every Gram, solve, residual, the
        # factors and the core stay fp64 (north_star's stated fp32 tolerance
        # 1e-4, normwise per SURVEY 8(c); tests/test_gpu_generated.py,
        # tests/test_gpu_fullsize.py).  The same steps in the fp64 mode are
        # timed first and reported beside it.
        dev.set_gather_f32(False)
        dev.set_model(m0)
        ms64, _, fams64, _ = measure(dev, c, args.steps, args.warmup, world, dist, local_rank, L, _lib, torch)
        alt = {"value": c["nnz"] * args.steps / (ms64 * 1e-3), "ms_per_step": ms64 / args.steps,
               "gathers": "fp64", "kernel_families_ms": fams64}
        dev.set_gather_f32(True)
    dev.set_model(m0)
    clk = Clocks(local_rank).__enter__()  # sampling covers warm-up and the timed region
    ms, res, fams, launches = measure(dev, c, args.steps, args.warmup, world, dist, local_rank, L, _lib, torch)
    clk.__exit__(None, None, None)
    value = c["nnz"] * args.steps / (ms * 1e-3)  # whole job: the N ranks share the nnz

    # ---- e2e through the C-ABI with host buffers (before any prune: same mask)
    e2e_steps = max(1, min(args.steps, 5))
    e2e_s, h2d, d2h = measure_e2e(dev, c, e2e_steps, dist, torch)
    e2e_value = c["nnz"] * e2e_steps / e2e_s

    # ---- prune event (timed separately; not an iteration)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev.compute_responsibilities(want=False)
    counts = dev.prune_step(0.3)
    prune_ms = (time.perf_counter() - t0) * 1e3
    dev.close()
    del dev, x

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    peak = C.c_double()
    pclk = Clocks(local_rank).__enter__()  # the peak is quoted with the SM clock it ran at
    best, t_end = 0.0, time.perf_counter() + 0.6  # repeated for ~0.6 s so the 50 ms clock sampler sees it
    while True:
        L.vest_measure_fp64_peak(local_rank, C.byref(peak))
        best = max(best, peak.value)
        if time.perf_counter() >= t_end:
            break
    peak.value = best
    pclk.__exit__(None, None, None)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    traffic_db = {}
    prof_json = os.path.join(ROOT, "profiles", "ncu_dominant.json")
    if os.path.exists(prof_json):
        try:
            traffic_db = json.load(open(prof_json)).get(f"config{cfg_id}", {})
        except Exception:
            traffic_db = {}
    roofline = roofline_for(c, fams, args.steps, ms, peak.value, peaks.get("hbm_gbs", 6650.0), core_live,
                            nnz_local, traffic_db)
    roofline["peak_clocks"] = pclk.summary()
    # whole-iteration FMA roof: reference-equivalent flops of one
    # CD iteration over the whole job vs the measured FP64 peak of all GPUs
    f_alg = step_flops_per_entry(c["ranks"], core_live)
    step_tf = f_alg * value / 1e12
    roofline["step"] = {"flops_per_entry": f_alg, "achieved": step_tf, "peak": peak.value * world,
                        "unit": "TFLOP/s", "frac": step_tf / (peak.value * world),
                        "note": "SURVEY.md 8(d) F_alg (reference-equivalent work) at the measured rate"}
    # ---- CPU baseline (rank 0, N = 1 only): the reference on a bounded sample
    cpu = None
    if world == 1 and not args.no_cpu:
        rate, kind, thr, sec, snnz = cpu_reference_rate(cfg_id)
        cpu = {"value": rate, "unit": UNIT, "cores": thr, "kind": kind,
               "sample": f"one CD iteration ({sec:.1f} s) of " + sample_desc(cfg_id, snnz)}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": f"synthetic (seeded; BASELINE config {cfg_id} shape)",
        "config": dict(workload_config(cfg_id, world),
                       gathers=("fp32 mode of the generated kernels: fp32 copies of the gathered factor rows, fp32 "
                                "contraction of delta and of the core passes' fiber products; Grams, solves, "
                                "residuals, factors and core fp64 (north_star fp32 tolerance 1e-4, normwise)"
                                if gf32 else "fp64")),
        "fp64_gathers": alt,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "steps": e2e_steps, "path": "vest_cd_iteration_host: host model in/out (pinned)"},
        "gpu_launches": launches,
        "roofline": roofline,
        "kernel_families_ms": fams,
        "prune_event": {"ms": prune_ms, "rate": 0.3, "counts": [counts.core] + counts.factors},
        "re_trace": res,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    # ---- secondary workload (config 2, the round-1 headline), N = 1 only
    if world == 1 and args.secondary and args.secondary != cfg_id:
        c2 = CONFIGS[args.secondary]
        co, va = synth(c2["dims"], c2["nnz"], 1000 + args.secondary, c2["values_kind"], c2["zipf"])
        x2 = st.SparseTensor(c2["dims"], co, va)
        d2 = st.Device(x2, c2["ranks"], local_rank)
        d2.set_model(model_for(c2))
        ms2, _, fams2, l2 = measure(d2, c2, 20, 5, 1, None, local_rank, L, _lib, torch, families=False)
        e2s, hb, db = measure_e2e(d2, c2, 5, None, torch)
        d2.close()
        line[f"config{args.secondary}"] = {
            "workload": workload_config(args.secondary, 1)["workload"], "value": c2["nnz"] * 20 / (ms2 * 1e-3),
            "ms_per_step": ms2 / 20, "steps": 20, "warmup": 5, "gpu_launches": l2,
            "e2e": {"value": c2["nnz"] * 5 / e2s, "h2d_bytes_per_step": hb, "d2h_bytes_per_step": db},
            "step_roof_frac": step_flops_per_entry(c2["ranks"]) * c2["nnz"] * 20 / (ms2 * 1e-3) / 1e12 / peak.value}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


# ------------------------------------------------ the other BASELINE configs --
CONFIGS = {
    1: dict(desc="3-mode 1000^3, 100k uniform, fp64 U[0,1), R 5^3, lambda 0.01; 10 iterations then prune 0.5",
            dims=[1000] * 3, nnz=100_000, ranks=[5, 5, 5], lam=0.01, zipf=None, values_kind=0, iters=10,
            prune=[(10, 0.5)], core_keep=1.0),
    2: dict(desc="3-mode 100k^3, 10M uniform, fp64 U[0,1), R 10^3, lambda 0.01; 20 iterations, prune 0.3 every 5",
            dims=[100_000] * 3, nnz=10_000_000, ranks=[10, 10, 10], lam=0.01, zipf=None, values_kind=0, iters=20,
            prune=[(5, 0.3), (10, 0.3), (15, 0.3)], core_keep=1.0),
    3: dict(desc="3-mode 1M x 200k x 1000, 50M, Zipf(1.1) on modes 1-2, integers 1..5, R (10,10,5), lambda 0.1; "
                 "10 iterations", dims=[1_000_000, 200_000, 1000], nnz=50_000_000, ranks=[10, 10, 5], lam=0.1,
            zipf=[1.1, 1.1, 0.0], values_kind=1, iters=10, prune=[], core_keep=1.0),
    4: dict(desc="4-mode 1M^4, 200M uniform, N(0,1) as float, R 8^4 core pruned to 10% nonzero, lambda 0.01; "
                 "10 iterations", dims=[1_000_000] * 4, nnz=200_000_000, ranks=[8, 8, 8, 8], lam=0.01, zipf=None,
            values_kind=2, iters=10, prune=[], core_keep=0.1, gather_f32=True),
    5: dict(desc="5-mode 100k^5, 100M Zipf(1.0) per mode, fp64 U[0,1), R 5^5; 90/10 split; prune-rate sweep "
                 "0.1..0.9 with train/test RE", dims=[100_000] * 5, nnz=100_000_000, ranks=[5] * 5, lam=0.01,
            zipf=[1.0] * 5, values_kind=0, iters=5, prune=[], core_keep=1.0, sweep=True),
}


def run_shard_emulation(cfg_id, world, iters):
    """Per-GPU device time of one rank's share of the sweep at `world` GPUs
    (ranks 0 and world-1 of the nnz-balanced row partition, exchanges replaced
    by no-ops: sharded.NullComm) -- the compute side of the scaling estimate on
    one B200.  The exchange volume per iteration is reported beside it."""
    import torch
    from paper_1904_02603_b200 import sharded as sh
    from paper_1904_02603_b200 import sparsetuck as st

    c = CONFIGS[cfg_id]
    coords, vals = synth(c["dims"], c["nnz"], 1000 + cfg_id, c["values_kind"], c["zipf"])
    x = st.SparseTensor(c["dims"], coords, vals)
    if c.get("sweep"):
        x, _ = st.split_train_test(x, 0.1, 2026)
    m = st.init_random(c["dims"], c["ranks"], 7)
    if c["core_keep"] < 1.0:
        rng = np.random.default_rng(44)
        mask = (rng.random(m.core.shape) >= c["core_keep"]).astype(np.uint8)
        m.core[mask == 1] = 0.0
        m.core_mask = mask
    bounds = sh.partition(x, world)
    out = {"config": cfg_id, "world": world, "ranks": {}}
    for rank in sorted({0, world - 1}):
        dev = sh.ShardDevice(x, c["ranks"], rank, world, sh.NullComm(), bounds=bounds)
        if c.get("gather_f32") and os.environ.get("VEST_GATHER_F32") is None:
            dev.set_gather_f32(True)
        dev.set_model(m)
        stream = torch.cuda.ExternalStream(dev.stream())
        times = []
        for t in range(iters + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dev.cd_iteration(0, c["lam"])
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        out["ranks"][rank] = {"ms_per_iter": statistics.median(times[1:]), "local_nnz_last_mode":
                              dev.local_nnz(len(c["dims"]) - 1)}
        dev.close()
    # exchanges per iteration: every factor once (row all-gather) + block statistics
    out["allgather_bytes_per_iter"] = int(sum(int(d) * int(r) * 8 for d, r in zip(c["dims"], c["ranks"])))
    print(json.dumps(out), flush=True)


NO_FAMILIES = False


def run_config(cfg_id, iters_override=None):
    """Full-size run of BASELINE config `cfg_id` on one GPU: per-iteration device
    time (CUDA events on the library stream), prune events timed separately."""
    import torch
    from paper_1904_02603_b200 import sparsetuck as st

    c = CONFIGS[cfg_id]
    t0 = time.perf_counter()
    coords, vals = synth(c["dims"], c["nnz"], 1000 + cfg_id, c["values_kind"], c["zipf"])
    gen_s = time.perf_counter() - t0
    x = st.SparseTensor(c["dims"], coords, vals)
    test = None
    if c.get("sweep"):
        x, test = st.split_train_test(x, 0.1, 2026)
    t0 = time.perf_counter()
    dev = st.Device(x, c["ranks"], 0)
    build_s = time.perf_counter() - t0
    m = st.init_random(c["dims"], c["ranks"], 7)
    if c["core_keep"] < 1.0:  # seeded core mask
        rng = np.random.default_rng(44)
        mask = (rng.random(m.core.shape) >= c["core_keep"]).astype(np.uint8)
        m.core[mask == 1] = 0.0
        m.core_mask = mask
    if c.get("gather_f32") and os.environ.get("VEST_GATHER_F32") is None:
        dev.set_gather_f32(True)
    dev.set_model(m)
    stream = torch.cuda.ExternalStream(dev.stream())
    iters = iters_override or c["iters"]
    from paper_1904_02603_b200 import _lib
    L = _lib.lib()
    # kernel-family timing (per-family events) disables the iteration graphs;
    # --no-families measures the production path
    L.vest_ctx_profile(dev.h, 0 if NO_FAMILIES else 1)
    times, res, prunes = [], [], []
    ms_arr = np.zeros(8)
    n_arr = np.zeros(8, np.uint64)
    for t in range(1, iters + 1):
        if t == iters:  # kernel families of the last (steady-state) iteration only
            L.vest_ctx_profile_read(dev.h, _lib.ptr(ms_arr, _lib.f64p), _lib.ptr(n_arr, _lib.u64p), 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res.append(dev.cd_iteration(0, c["lam"]))
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        for (at, pr) in c["prune"]:
            if at == t:
                p0 = time.perf_counter()
                dev.compute_responsibilities(want=False)
                cnt = dev.prune_step(pr)
                prunes.append({"iter": t, "rate": pr, "ms": (time.perf_counter() - p0) * 1e3,
                               "counts": [cnt.core] + cnt.factors})
    L.vest_ctx_profile_read(dev.h, _lib.ptr(ms_arr, _lib.f64p), _lib.ptr(n_arr, _lib.u64p), 1)
    fam_names = ["factor_update", "core_pass", "core_gemm", "core_solve", "residual", "resp", "prune",
                 "factor_update_fused_residual"]
    fams = {fam_names[i]: {"ms": float(ms_arr[i]), "scopes": int(n_arr[i])} for i in range(8)}  # last iteration
    # steady state: the first sweep with a new core mask runs the precompiled
    # kernels and the second compiles the mask-specialised ones (NVRTC, auto
    # mode), so the median is taken from the third iteration on when there is one
    med = statistics.median(times[2:] if len(times) > 2 else (times[1:] if len(times) > 1 else times))
    line = {"config": cfg_id, "workload": c["desc"], "nnz": x.nnz(), "ms_per_iter_median": med,
            "ms_per_iter": times, "value": x.nnz() / (med * 1e-3), "unit": UNIT, "re_trace": res,
            "prune_events": prunes, "gen_s": gen_s, "ctx_build_s": build_s, "specialised": dev.specialised(),
            "device_gb": dev.device_bytes() / 1e9, "kernel_families_ms_last_iter": fams}
    if c.get("sweep"):
        p0 = time.perf_counter()
        sweep = st.auto_search(x, test, dev.get_model(), [round(0.1 * k, 1) for k in range(1, 10)], dev=dev)
        line["sweep"] = [{"rate": r.rate, "train_re": r.train_re, "test_re": r.test_re, "sparsity": r.sparsity}
                         for r in sweep]
        line["sweep_s"] = time.perf_counter() - p0
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=0, help="run BASELINE config 1..5 at full size (diagnostic)")
    ap.add_argument("--iters", type=int, default=0)
    ap.add_argument("--no-families", action="store_true",
                    help="with --config: no per-family event timing (iteration graphs stay enabled)")
    ap.add_argument("--shard-emulate", type=int, default=0,
                    help="with --config: per-GPU device time of one rank's share at W GPUs (no exchanges)")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--fp64-gathers", action="store_true", help="config 4: fp64 factor gathers only")
    ap.add_argument("--workload", type=int, default=HEADLINE, help="BASELINE config of the headline line")
    ap.add_argument("--secondary", type=int, default=SECONDARY,
                    help="BASELINE config measured after the headline as an extra key (0: none)")
    args = ap.parse_args()
    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local_rank = env_int("LOCAL_RANK", 0)
    global NO_FAMILIES
    NO_FAMILIES = args.no_families
    if args.config and args.shard_emulate:
        run_shard_emulation(args.config, args.shard_emulate, args.iters or 3)
        return
    if args.config:
        run_config(args.config, args.iters or None)
        return
    if args.impl == "reference":
        run_reference_arm(args, rank)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
