#!/usr/bin/env python
"""Benchmark: assembled nonzeros/sec (FP64, device-timed) of the weighted-Gaussian row-wise
assembly (BASELINE.json metric), one process per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A step = one pass of the whole hot path (every row of the rank's slab,
M and K fused) over the workload; inputs (rules tables, coefficient slab) are resident in HBM
when the timed region starts.  Default workload: C5 (3D C2-cubic, 256^3 elements, M+K,
gridded lognormal coefficient), the config the metric is quoted on (it fits one B200).
Rows are z-slab sharded across ranks; the total mesh is fixed, so scaling is
"strong".  Timing: CUDA events on the launching stream around each step, L2 flushed between
steps, max over ranks.  Rank 0 prints one JSON line.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import inputs  # noqa: E402

METRIC = "assembled nonzeros/sec (FP64, device-timed)"
UNIT = "nnz/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--n", "--elems", dest="n", type=int, default=None,
                    help="override elements per direction (--elems under torchrun: its parser claims --n)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ld", type=int, default=None)
    ap.add_argument("--no-extras", action="store_true", help="skip the secondary measurements (other configs, operators)")
    return ap.parse_args()


def stencil_nnz(p, n, d, rows):
    """Structural nonzeros of a set of global rows (per matrix)."""
    N = n + p
    tot = 0
    for r in rows:
        w = 1
        for a in range(d):
            i = (r // N ** a) % N
            w *= min(i + p, N - 1) - max(i - p, 0) + 1
        tot += w
    return tot


# ------------------------------------------------------------------------------------------
# the oracle on the host (cpu_baseline and --impl reference)
# ------------------------------------------------------------------------------------------
def oracle_sample_rows(cfg, budget_rows, seed=0):
    """A bounded, deterministic sample of the workload's rows: whole x-lines from the first,
    a middle and the last z-planes (every row class occurs), as (grid slab, plane0, rows)."""
    p, n, d = cfg["p"], cfg["n"], cfg["dim"]
    N = n + p
    rng = np.random.default_rng(seed)
    groups = []
    if d == 3:
        zs = [0, 1, N // 2, N - 1]
    elif d == 2:
        zs = [0, N // 2, N - 1]
    else:
        zs = [0]
    per = max(1, budget_rows // len(zs))
    for z in zs:
        if d == 1:
            rows = np.arange(N)[:per]
        else:
            lines = max(1, per // N)
            ys = rng.choice(N, size=min(lines, N), replace=False) if d == 3 else [None]
            rows = []
            for y in ys:
                base = (z * N + y) * N if d == 3 else z * N
                rows.extend(range(base, base + N))
            rows = np.array(rows[:per])
        groups.append((z, rows))
    return groups


def run_oracle(cfg, seconds, rows_hint=None):
    """Time the oracle (as it stands) on a bounded sample: returns (nnz/s, sample text, cores)."""
    from oracle import assemble as oasm
    p, n, d = cfg["p"], cfg["n"], cfg["dim"]
    desc = inputs.coefficient(cfg["coeff"], d)
    kinds = cfg["kinds"]
    oasm.tables_1d(p, n)                                  # setup, untimed
    probe = oracle_sample_rows(cfg, 64)
    g0 = _oracle_grid(cfg, probe[0][0])
    t0 = time.perf_counter()
    oasm.assemble_rows(p, n, d, probe[0][1][:16], desc, kinds, grid=g0[0], plane0=g0[1])
    per_row = (time.perf_counter() - t0) / 16
    budget = rows_hint or max(32, int(seconds / max(per_row, 1e-6)))
    groups = oracle_sample_rows(cfg, budget)
    nnz = 0
    elapsed = 0.0
    nrows = 0
    for z, rows in groups:
        grid, plane0 = _oracle_grid(cfg, z)
        t0 = time.perf_counter()
        oasm.assemble_rows(p, n, d, rows, desc, kinds, grid=grid, plane0=plane0)
        elapsed += time.perf_counter() - t0
        nnz += stencil_nnz(p, n, d, rows) * len(kinds)
        nrows += len(rows)
    sample = f"{nrows} rows of {cfg['name']} (whole x-lines of z-planes {[int(z) for z, _ in groups]}), {'+'.join(kinds)}"
    run_oracle.last_rows = nrows
    return nnz / elapsed, sample, 1, elapsed


_POOL_JOBS = None


def _oracle_job(i):
    """One block of the all-core oracle run (fork workers; the job list is inherited)."""
    from threadpoolctl import threadpool_limits

    from oracle import assemble as oasm
    threadpool_limits(1)
    cfg, desc, rows, grid, plane0 = _POOL_JOBS[i]
    t0 = time.perf_counter()
    oasm.assemble_rows(cfg["p"], cfg["n"], cfg["dim"], rows, desc, cfg["kinds"], grid=grid, plane0=plane0)
    return time.perf_counter() - t0


def cpu_baseline(cfg, seconds):
    """The oracle (as it stands: plain numpy, oracle.assemble_rows) on the host cores: a
    1-core run on a bounded sample of the workload, and the same per-core sample on every core
    at once (fork workers over row blocks) -- SURVEY §8(d) / BASELINE.md §4."""
    import multiprocessing as mp
    global _POOL_JOBS
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):                      # the 1-core figure is one core
        v1, sample, _, el1 = run_oracle(cfg, seconds / 2)
    cores = os.cpu_count() or 1
    desc = inputs.coefficient(cfg["coeff"], cfg["dim"])
    # every core gets about the 1-core sample's rows, in 2 blocks per core
    per_job = max(1, run_oracle.last_rows // 2)
    jobs = []
    for z, rows in oracle_sample_rows(cfg, cores * run_oracle.last_rows, seed=1):
        grid, plane0 = _oracle_grid(cfg, z)
        for b0 in range(0, len(rows), per_job):
            jobs.append((cfg, desc, rows[b0:b0 + per_job], grid, plane0))
    _POOL_JOBS = jobs
    from oracle import assemble as oasm
    oasm.tables_1d(cfg["p"], cfg["n"])
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(cores) as pool:
        pool.map(_oracle_job, range(len(jobs)), chunksize=1)
    wall = time.perf_counter() - t0
    nnz = sum(stencil_nnz(cfg["p"], cfg["n"], cfg["dim"], r) for _, _, r, _, _ in jobs) * len(cfg["kinds"])
    rows_all = sum(len(r) for _, _, r, _, _ in jobs)
    return {"value": nnz / wall, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{rows_all} rows of {cfg['name']} (whole x-lines of boundary and interior z-planes, "
                      f"{len(jobs)} row blocks over {cores} processes), {'+'.join(cfg['kinds'])}",
            "seconds": round(wall, 2),
            "one_core": {"value": v1, "unit": UNIT, "cores": 1, "sample": sample, "seconds": round(el1, 2)}}


def build_info():
    """git commit of the tree (the GPU box gets a snapshot without .git: build() records it)."""
    info = {}
    try:
        with open(os.path.join(ROOT, "paper_1710_01048_b200", "build_info.json")) as f:
            info = json.load(f)
    except Exception:
        pass
    try:
        r = subprocess.run(["git", "-C", ROOT, "rev-parse", "HEAD"], capture_output=True, text=True, timeout=5)
        if r.returncode == 0 and r.stdout.strip():
            info["git_sha"] = r.stdout.strip()
    except Exception:
        pass
    return info


def _oracle_grid(cfg, z):
    if cfg["coeff"]["kind"] != "grid":
        return None, 0
    p, n, d = cfg["p"], cfg["n"], cfg["dim"]
    lo, hi = max(0, z - p), min(n, z + 1)
    g = inputs.lognormal_grid(n, seed=cfg["coeff"]["seed"], sigma=cfg["coeff"]["sigma"], dim=d, plane0=lo,
                              planes=hi - lo + 1)
    return g, lo


# ------------------------------------------------------------------------------------------
# clocks during the timed region (NVML)
# ------------------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, device):
        self.samples, self.power, self.reasons, self.ok = [], [], 0, False
        self.limit_w = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
            try:
                self.limit_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(self.h) / 1e3
            except Exception:
                pass
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.power.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1e3)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": [v for k, v in self.REASONS.items() if self.reasons & k], "samples": len(self.samples),
                "power_w": round(float(np.median(self.power)), 1) if self.power else None,
                "power_limit_w": self.limit_w}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


def traffic_from_profiles(cfg_name):
    """dram bytes (read+write) per launch of the dominant kernel from a committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
        return t.get(cfg_name)
    except Exception:
        return None


# ------------------------------------------------------------------------------------------
def arm_config(cfg, world, ld=None):
    """The workload description, identical for this arm and the reference (oracle) arm."""
    p, n, d = cfg["p"], cfg["n"], cfg["dim"]
    s = 2 * p + 1
    return {"workload": cfg["name"], "p": p, "n_elems": n, "dim": d, "kinds": list(cfg["kinds"]),
            "coefficient": cfg["coeff"]["kind"], "rows": (n + p) ** d, "ld": ld or s ** d,
            "layout": "ELL", "parallelism": f"line-granular z-slabs x{world}",
            "l2": "flushed (512 MB write) between timed steps; outputs >> L2"}


def gpu_launches_per_step(cfg):
    """Kernels of one assembly call: one, except the 2D FOURIER path: factor tables, the
    device-generated GL-shell row list, then for p = 3 one fused launch (class-I interior, frame
    and shell items) and for p = 2 the per-row kernel plus the generic shell pass."""
    if cfg["dim"] == 2 and cfg["coeff"]["kind"] == "fourier_logn":
        return 3 if cfg["p"] == 3 else 4
    return 1


def main():
    args = parse()
    cfg = inputs.config(args.config, args.n)
    p, n, d = cfg["p"], cfg["n"], cfg["dim"]
    kinds = cfg["kinds"]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        vals = []
        info = None
        for i in range(args.warmup + args.steps):
            cb = cpu_baseline(cfg, min(args.cpu_seconds, 120.0 / max(1, args.steps + args.warmup)))
            if i >= args.warmup:
                vals.append(cb["value"])
                info = (cb["sample"], cb["cores"])
        value = float(np.median(vals))
        line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
                "dtype": "f64", "data": "synthetic",
                "config": arm_config(cfg, world),
                "cpu_baseline": {"value": value, "unit": UNIT, "cores": info[1], "kind": "oracle", "sample": info[0]},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "vs_baseline": None}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    from paper_1710_01048_b200 import api, wgq
    from paper_1710_01048_b200 import dist as wdist

    # WGQ_BENCH_FUNCTIONAL=1: functional check of the N>1 code path on ONE GPU (every rank on
    # cuda:0, gloo on CPU tensors); its timings are not measurements (the ranks share a GPU)
    functional = os.environ.get("WGQ_BENCH_FUNCTIONAL") == "1"
    dev = 0 if functional else local
    torch.cuda.set_device(dev)
    if world > 1:
        if functional:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    red_dev = "cpu" if functional else "cuda"
    stream = torch.cuda.current_stream()

    # setup, reported separately: host rule build, device tables, grid generation
    setup = {}
    t0 = time.perf_counter()
    rules = wgq.Rules(p, n, d)
    setup["rules_host_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
    N = rules.N
    row_begin, row_end = api.slab_rows(N, d, rank, world)
    rows = row_end - row_begin
    ld = args.ld or rules.stencil
    grid, plane0 = (None, 0)
    torch.cuda.synchronize()
    if cfg["coeff"]["kind"] == "grid":
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        grid, plane0 = api.make_grid(rules, cfg["coeff"]["seed"], cfg["coeff"]["sigma"], row_begin, row_end)
        e1.record()
        torch.cuda.synchronize()
        setup["grid_generation_ms"] = round(e0.elapsed_time(e1), 3)
    coef = api.coefficient(inputs.coefficient(cfg["coeff"], d), grid, plane0)
    t0 = time.perf_counter()
    api.assemble_load(rules, coef, row_begin, min(row_end, row_begin + 1))   # first device call: row tables
    torch.cuda.synchronize()
    setup["device_tables_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
    out = {k: api.alloc_ell(rules, row_begin, row_end, ld) for k in kinds}
    nnz_rank = wgq.wgq_nnz(rules, row_begin, row_end) * len(kinds)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")     # 512 MB > L2

    def step():
        api.assemble(rules, coef, kinds, row_begin, row_end, out=out, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(dev) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    # per-step max over ranks; the metric is taken at the median step
    t = torch.tensor(step_ms, dtype=torch.float64, device=red_dev)
    nz = torch.tensor([float(nnz_rank)], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(nz, op=dist.ReduceOp.SUM)
    step_max = [float(x) for x in t.cpu().tolist()]
    med_ms = float(np.median(step_max))
    nnz_all = float(nz.item())
    value = nnz_all / (med_ms / 1e3)

    # self-check of the result (every N): order-independent hash of each matrix's slab, summed
    # over ranks -- an N-GPU line carries the same hash as the 1-GPU line (rows are independent)
    checksum = {}
    for k in kinds:
        h = torch.zeros(3, dtype=torch.int64, device="cuda")
        wgq.wgq_checksum(rules, wgq.make_out(out[k], row_begin, row_end, ld=ld), h, stream)
        torch.cuda.synchronize()
        local = h.to(red_dev)
        if world > 1:
            hv, s1, s2 = wdist.reduce_checks(local)
        else:
            hv, s1, s2 = int(local[0].item()) & (2 ** 64 - 1), float(local[1:].view(torch.float64)[0]), \
                float(local[1:].view(torch.float64)[1])
        checksum[k] = {"hash": f"{hv:016x}", "sum": s1, "sumsq": s2}

    # roofline of the dominant (only) kernel: algorithmic bytes = rows x s^d x 8 x matrices
    alg_bytes = rows * rules.stencil * 8 * len(kinds)
    kernel_s = float(np.median(step_ms)) / 1e3
    peak, peak_src = peaks()
    achieved = alg_bytes / kernel_s / 1e9
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "peak_source": peak_src,
            "traffic": traffic_from_profiles(cfg["name"]),
            "kernel": "wgq assembly (M+K fused)", "algorithmic_bytes_per_launch": int(alg_bytes),
            "kernel_ms": round(kernel_s * 1e3, 4), "kernel_ms_stat": "median of the timed steps (this rank)",
            "step_ms": {"min": round(float(np.min(step_ms)), 4), "median": round(float(np.median(step_ms)), 4),
                        "mean": round(float(np.mean(step_ms)), 4), "max": round(float(np.max(step_ms)), 4)}}

    # end to end through the public API with HOST buffers (H2D of the coefficient slab, D2H of M, K)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, cfg, rules, row_begin, row_end, ld, world, rank, local, nnz_all, red_dev)

    extras = None
    if rank == 0 and world == 1 and not args.no_extras:
        del out
        torch.cuda.empty_cache()
        extras = run_extras(rules, coef, peak)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg, args.cpu_seconds)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": med_ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": arm_config(cfg, world, ld),
                # one assembly kernel per step; the 2D Fourier path adds its per-call factor tables
                # and the generic shell-row pass
                "gpu_launches": args.steps * gpu_launches_per_step(cfg),
                "roofline": roof, "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu, "extras": extras,
                "setup": setup, "checksum": checksum, "nnz_per_step": int(nnz_all),
                "timing": {"stat": "median over the timed steps of the per-step max over ranks",
                           "ms_mean": float(np.mean(step_max)), "ms_min": float(np.min(step_max)),
                           "ms_max": float(np.max(step_max))},
                "build": build_info(), "peaks": {"hbm_gbs": peak, "source": peak_src}}
        if functional:
            line["functional_check"] = "WGQ_BENCH_FUNCTIONAL=1: all ranks on one GPU over gloo; not a measurement"
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def apply_flops_per_row(rules):
    """Algorithmic FP64 flops per row of the matrix-free product y_M = M u, y_K = K u on the GRID
    line structure, structural zeros skipped: with the interior vertex-projected
    tables P^M, P^K (V = p+2 vertex planes x S = 2p+1 columns; entry (v, o) is nonzero iff some
    node k of the row's rule lies in element f_k = floor(tau_k) with v in {f_k, f_k+1} and o in
    [f_k, f_k+p]) of nz_M, nz_K nonzeros,
      phase A (one vertex plane per row): TT_M = P^M_y patch (nz_M V), TT_K (nz_K V),
              H_M = TT_M P^M_z (S nz_M), H_K = TT_K P^M_z + TT_M P^K_z (S nz_M + S nz_K);
      D stage: D_X(c, X) = sum_{o2,o3} H_X u (S^2 per matrix) for the n_delta distinct offsets
               X - c = o - v of the nonzeros (one (c, X) pair per offset per row);
      finish: y_M = sum P^M D_M (nz_M), y_K = sum P^K D_M + P^M D_K (nz_K + nz_M).
    Returns (flops per row, definition text)."""
    from paper_1710_01048_b200 import wgq
    p = rules.p
    V, S = p + 2, 2 * p + 1
    nz, offs = {}, set()
    for kind, kc in (("M", wgq.WGQ_MASS), ("K", wgq.WGQ_STIFFNESS)):
        tau, om, _ = wgq.wgq_rules_query(rules, p, kc)
        pat = set()
        for tk, wk in zip(tau, om):
            f = int(np.floor(tk))
            for v in (f, f + 1):
                for o in range(f, f + p + 1):
                    pat.add((v, o))
        nz[kind] = len(pat)
        offs |= {o - v for v, o in pat}
    nzM, nzK, nd = nz["M"], nz["K"], len(offs)
    fma = V * (nzM + nzK) + S * (2 * nzM + nzK) + 2 * S * S * nd + 2 * nzM + nzK
    return 2 * fma, (f"2 x FMA: phase A V(nzM+nzK)+S(2nzM+nzK) + D 2 S^2 n_delta + finish 2nzM+nzK with "
                     f"p={p}, V={V}, S={S}, nzM={nzM}, nzK={nzK}, n_delta={nd}")


def _time_ms(fn, reps=5, flush=None):
    """Median device time (CUDA events on the current stream) of fn(), L2 flushed before each."""
    import torch
    fn()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def run_extras(rules5, coef5, peak):
    """Secondary measurements (not the headline): the other BASELINE configs' assembly (parity
    cases; their kernels differ: separable, 2D tensor-core FOURIER) against the same HBM
    roofline, and the SURVEY §8(f) operators at C5 — load vector and matrix-free y = M u, K u."""
    import torch

    from paper_1710_01048_b200 import api, wgq
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    out = {"configs": {}, "operators": {}}
    for name in ("C1", "C2", "C3", "C4"):
        cfg = inputs.config(name)
        r = wgq.Rules(cfg["p"], cfg["n"], cfg["dim"])
        c = api.coefficient(inputs.coefficient(cfg["coeff"], cfg["dim"]))
        o = {k: api.alloc_ell(r, 0, r.n_rows) for k in cfg["kinds"]}
        ms = _time_ms(lambda: api.assemble(r, c, cfg["kinds"], out=o), flush=flush)
        alg = r.n_rows * r.stencil * 8 * len(cfg["kinds"])
        nnz = wgq.wgq_nnz(r, 0, r.n_rows) * len(cfg["kinds"])
        out["configs"][cfg["name"]] = {"ms": round(ms, 4), "nnz_per_s": nnz / (ms / 1e3),
                                       "hbm_gbs": round(alg / ms / 1e6, 1), "hbm_frac": round(alg / ms / 1e6 / peak, 4)}
        del o
    # C5 with a different element count per direction (eq:Gmap3 P:113-120): 256 x 256 x 192,
    # the same GRID kernel and coefficient recipe
    ra = wgq.Rules(3, (256, 256, 192), 3)
    ga, la = api.make_grid(ra, inputs.SEED, 0.5, 0, ra.n_rows)
    ca = api.coefficient({"kind": "grid"}, ga, la)
    oa = {k: api.alloc_ell(ra, 0, ra.n_rows) for k in ("mass", "stiffness")}
    ms = _time_ms(lambda: api.assemble(ra, ca, out=oa), flush=flush)
    alg = ra.n_rows * ra.stencil * 8 * 2
    nnz = wgq.wgq_nnz(ra, 0, ra.n_rows) * 2
    out["configs"]["3d_p3_n256x256x192_mk_grid"] = {"ms": round(ms, 4), "rows": ra.n_rows, "nnz_per_s": nnz / (ms / 1e3),
                                                    "hbm_gbs": round(alg / ms / 1e6, 1),
                                                    "hbm_frac": round(alg / ms / 1e6 / peak, 4)}
    del oa, ga, ca
    torch.cuda.empty_cache()
    # C5 in CSR layout (values of both matrices; the closed-form structure is built once, untimed)
    nnz5 = wgq.wgq_nnz(rules5, 0, rules5.n_rows)
    row_ptr = torch.empty(rules5.n_rows + 1, dtype=torch.int64, device="cuda")
    col_idx = torch.empty(nnz5, dtype=torch.int32, device="cuda")
    wgq.wgq_csr_structure(rules5, 0, rules5.n_rows, row_ptr, col_idx)
    del col_idx
    vals = {k: torch.empty(nnz5, dtype=torch.float64, device="cuda") for k in ("mass", "stiffness")}
    dm = wgq.make_out(vals["mass"], 0, rules5.n_rows, ld=0, layout=wgq.WGQ_CSR, row_ptr=row_ptr)
    dk = wgq.make_out(vals["stiffness"], 0, rules5.n_rows, ld=0, layout=wgq.WGQ_CSR, row_ptr=row_ptr)
    ms = _time_ms(lambda: wgq.wgq_assemble_mass_stiffness(rules5, coef5, dm, dk), flush=flush)
    csr_bytes = 2 * nnz5 * 8
    out["configs"]["3d_p3_n256_mk_grid_csr"] = {"ms": round(ms, 4), "nnz_per_s": 2 * nnz5 / (ms / 1e3),
                                                "hbm_gbs": round(csr_bytes / ms / 1e6, 1),
                                                "hbm_frac": round(csr_bytes / ms / 1e6 / peak, 4)}
    del vals, row_ptr, dm, dk
    torch.cuda.empty_cache()
    n_rows = rules5.n_rows
    # peak microbenchmarks of this box, same session (tools/peaks.cu, built by build()): the
    # FP64 denominator of the matrix-free product
    exe = os.path.join(ROOT, "tools", "peaks")
    if os.path.exists(exe):
        try:
            r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
            out["box_peaks"] = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception as e:          # the headline numbers do not depend on it
            out["box_peaks"] = {"error": str(e)[:200]}
    fp64_peak, fp64_src = out.get("box_peaks", {}).get("fp64_tflops"), "tools/peaks DFMA (this box, this run)"
    if not fp64_peak:
        fp64_peak, fp64_src = 34.2, "DFMA microbenchmark, round 1 (DESIGN.md §5)"
    b = torch.empty(n_rows, dtype=torch.float64, device="cuda")
    ms = _time_ms(lambda: api.assemble_load(rules5, coef5, out=b), flush=flush)
    nv = rules5.n + 1
    load_bytes = (nv ** 3 + n_rows) * 8                  # the vertex grid read once + b written
    out["operators"]["load_vector_C5"] = {
        "ms": round(ms, 4), "rows_per_s": n_rows / (ms / 1e3),
        "roofline": {"bound": "hbm", "achieved": round(load_bytes / (ms / 1e3) / 1e9, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(load_bytes / (ms / 1e3) / 1e9 / peak, 4),
                     "algorithmic_bytes": int(load_bytes), "bytes_def": "257^3 vertex values read once + b written"}}
    u = torch.randn(n_rows, dtype=torch.float64, device="cuda")
    ms = _time_ms(lambda: api.apply(rules5, coef5, u), flush=flush)
    fl_row, fl_def = apply_flops_per_row(rules5)
    apply_bytes = (nv ** 3 + 3 * n_rows) * 8             # grid + u read once, y_M and y_K written
    a_tf = fl_row * n_rows / (ms / 1e3) / 1e12
    a_gbs = apply_bytes / (ms / 1e3) / 1e9
    fp_frac, hbm_frac = a_tf / fp64_peak, a_gbs / peak
    # context: the time just to stream the assembled M and K (ELL) once at the copy peak
    stream_ms = n_rows * rules5.stencil * 8 * 2 / (peak * 1e9) * 1e3
    out["operators"]["apply_MK_C5"] = {
        "ms": round(ms, 4), "rows_per_s": n_rows / (ms / 1e3), "stream_assembled_ms": round(stream_ms, 3),
        "roofline": {"bound": "fp64" if fp_frac >= hbm_frac else "hbm",
                     "achieved": round(a_tf, 2) if fp_frac >= hbm_frac else round(a_gbs, 1),
                     "peak": fp64_peak if fp_frac >= hbm_frac else peak,
                     "unit": "TFLOP/s" if fp_frac >= hbm_frac else "GB/s",
                     "frac": round(max(fp_frac, hbm_frac), 4),
                     "fp64": {"achieved_tflops": round(a_tf, 2), "peak_tflops": fp64_peak, "peak_source": fp64_src,
                              "frac": round(fp_frac, 4), "algorithmic_flops_per_row": fl_row, "flops_def": fl_def},
                     "hbm": {"achieved_gbs": round(a_gbs, 1), "peak_gbs": peak, "frac": round(hbm_frac, 5),
                             "algorithmic_bytes": int(apply_bytes)}},
        "note": "matrix-free y_M = M u and y_K = K u, nothing stored; stream_assembled_ms = reading the 95 GB of "
                "assembled M, K once at the copy peak (what any assembled SpMV would need)"}
    # the paper's own cost metric (context): basis evaluations for its 2D 100x100 test
    # problem, weighted Gaussian (this library's rules) vs the weighted Newton-Cotes point sets
    out["paper_eval_counts_2d_100x100_mass"] = {}
    for pp in (2, 3):
        g, c = wgq.wgq_eval_counts(wgq.Rules(pp, 100, 2), wgq.WGQ_MASS)
        out["paper_eval_counts_2d_100x100_mass"][f"p{pp}"] = {
            "gaussian": g, "newton_cotes": c, "ratio": round(c / g, 4),
            "paper_ratio": {2: 2.08, 3: 2.44}[pp], "interior_ratio": round({2: (13 / 9) ** 2, 3: (25 / 16) ** 2}[pp], 4)}
    return out


def run_e2e(args, cfg, rules, row_begin, row_end, ld, world, rank, local, nnz_all, red_dev="cuda"):
    import torch
    import torch.distributed as dist

    from paper_1710_01048_b200 import api, wgq
    p, n, d = cfg["p"], cfg["n"], cfg["dim"]
    kinds = cfg["kinds"]
    rows = row_end - row_begin
    host = {k: wgq.PinnedArray((rows, ld)) for k in kinds}
    h2d = 0
    if cfg["coeff"]["kind"] == "grid":
        lo, hi = api.grid_planes_for(rules, row_begin, row_end)
        g = inputs.lognormal_grid(n, seed=cfg["coeff"]["seed"], sigma=cfg["coeff"]["sigma"], dim=d, plane0=lo,
                                  planes=hi - lo + 1)
        pin = wgq.PinnedArray(g.shape)
        pin.array[...] = g
        coef = wgq.make_coeff({"kind": "grid"}, grid=wgq.HostGrid(pin.array), plane0=lo)
        h2d = g.nbytes
    else:
        coef = api.coefficient(inputs.coefficient(cfg["coeff"], d))
    M = host["mass"].array if "mass" in host else None
    K = host["stiffness"].array if "stiffness" in host else None
    wgq.wgq_assemble_host(rules, coef, row_begin, row_end, M, K, ld)       # warm-up
    times = []
    for _ in range(args.e2e_steps):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        wgq.wgq_assemble_host(rules, coef, row_begin, row_end, M, K, ld)
        times.append(time.perf_counter() - t0)
    t = torch.tensor([float(np.sum(times))], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    value = nnz_all * args.e2e_steps / float(t.item())
    d2h = rows * ld * 8 * len(kinds)
    for v in host.values():
        v.close()
    return {"value": value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "steps": args.e2e_steps, "api": "wgq_assemble_host (pinned host buffers, chunked 2-stream pipeline)"}


if __name__ == "__main__":
    main()
