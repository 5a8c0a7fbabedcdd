"""Benchmark of the GPU IC(k) numeric factorization (the reference's
factor_by_blocks hot path) -- prints ONE JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

The default workload is C3 (BASELINE.json configs[2], 27-point 48^3 IC(2),
7.6 M factor entries), the largest configuration that runs on one GPU; the
other configurations are selectable and are parity-test cases.

A step is one numeric factorization of the configuration's matrix, starting
from the initialised factor U resident in HBM (the reference's
numeric_seconds region, factorize.hpp:169-227). Between steps U is restored
from its device copy and L2 is flushed (256 MiB write), both untimed.

  value  factor-nnz/s over the whole job = N * nnz_u / (max over ranks of the
         device time of one step); device time = CUDA events around the
         persistent kernel on the stream it is launched on.
  e2e    the same metric through the C ABI with host buffers
         (tcg_factor_host_a): H2D of PaP's values (the reference call's
         input) from pinned memory, init_factor_values on the device, factor
         -- with CTAs of the same launch copying each group of factor values
         to the pinned host buffer as soon as it is final, so the D2H
         overlaps the factorization --, one stream-ordered call; the symbolic
         structure (plan) stays resident, as in a refactorization.
  roofline  algorithmic bytes 20*nnz_u + 8*(n+1) per
         launch / kernel time, against the measured HBM copy bandwidth.

N > 1 (torchrun, one process per GPU): the single-matrix configs do not
shard, so every rank factors its own replica (weak scaling, no collective on
the data path); timing is the max over ranks. --config c5b is the sharded
C5 batch: the 64 members are split over the ranks (paper_1601_05871_b200/
batch.py), each rank factors its members in one launch, value = 64 * nnz_u /
max-over-ranks time (strong scaling over the fixed batch).

  parity_vs_oracle  the last factor's hash against the golden hash of the
         reference's factor_serial (tests/golden), every configuration.
  one_shot  wall time of one factor_by_blocks_gpu call (plan, context,
         upload, factor, download), the reference's unit of work.

--impl reference: times the reference's own CPU factor_by_blocks
(oracle/_ref, compiled from the unmodified reference headers) with a pooled
policy over all host threads, rank 0 only, on inputs built by the shim
(generators + the reference's analyze); factor_serial and pooled(1) beside it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

WORKLOADS = {
    "c1": "C1: 2D 5-point Laplacian 100x100 (n=10,000), IC(0), fp64, ND leaf 64",
    "c2": "C2: 3D 7-point Laplacian 64^3 (n=262,144), IC(1), fp64, ND leaf 64",
    "c3": "C3: 3D 27-point variable-coefficient 48^3 (n=110,592), IC(2), fp64, ND leaf 64",
    "c4": "C4: elasticity-like 40^3 x 3 dofs (n=192,000), IC(0), fp64, ND leaf 64",
    "c5": "C5 member: 3D 7-point log-normal diffusion 32^3 (n=32,768), IC(1), fp64",
    "c5b": "C5: batch of 64 3D 7-point log-normal diffusion 32^3 matrices (n=32,768 each), IC(1), fp64, "
           "members sharded over ranks, one launch per rank",
    "c6": "C6: 3D 7-point Laplacian 128^3 (n=2,097,152), IC(1), fp64, ND leaf 64",
}
METRIC = "ic_numeric_factor_nnz_per_s"
UNIT = "nnz/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic(config: str):
    """Per-launch DRAM bytes of the factor kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", f"ncu_{config}_factor.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch")
    return None


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the measured
    loops: NVML every 2 ms from a background thread (nvidia-smi's 50 ms loop
    as the fallback), so even a region of a few tens of ms gets samples."""

    NAMES = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
             ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
             ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
             ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []   # (sm_mhz, max_mhz, [reasons])
        self.proc = None
        self.stop = threading.Event()
        self.thread = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)

            def poll():
                while not self.stop.is_set():
                    try:
                        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((float(sm), float(mx),
                                             [n for n, attr in self.NAMES if r & getattr(nv, attr, 0)]))
                    except Exception:
                        pass
                    self.stop.wait(0.002)
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        names = [n for n, _ in self.NAMES]
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7 and parts[0].replace(".", "").isdigit():
                self.samples.append((float(parts[0]), float(parts[1]) if parts[1].replace(".", "").isdigit()
                                     else float("nan"), [names[i] for i in range(4) if parts[3 + i] == "Active"]))

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"], "samples": 0}
        sm = [x[0] for x in self.samples]
        mx = [x[1] for x in self.samples if x[1] == x[1]]
        reasons = sorted({r for x in self.samples for r in x[2]})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples), "sm_mhz_min": min(sm)}


def build_problem(config: str, member: int = 0):
    import paper_1601_05871_b200 as T
    name = "c5" if config in ("c5", "c5b") else config
    a, level = T.config_matrix(name, member)
    t0 = time.perf_counter()
    an = T.analyze(a, level=level)
    t_an = time.perf_counter() - t0
    plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
    return a, an, plan, t_an


def cpu_reference_times(an, workers: int, reps: int):
    from checkers import Reference, reference_available
    if not reference_available():
        return None
    R = Reference()
    u = an.pattern.pattern
    out = {"serial": [], "pool": []}
    for _ in range(reps):
        _, st, secs, _, _ = R.factor_serial(an.a_permuted, u)
        out["serial"].append(secs)
    for _ in range(reps):
        _, st, secs, _, _, _ = R.factor_by_blocks(an.a_permuted, u, an.ranges.bounds, workers=workers,
                                                  want_values=False)
        out["pool"].append(secs)
    # TaskPolicy::pooled(1) once (W = 1 and W = all cores)
    out["pool1"] = [R.factor_by_blocks(an.a_permuted, u, an.ranges.bounds, workers=1, want_values=False)[2]]
    return out


# generator table of the configurations (core.CONFIGS), repeated here so the
# reference arm does not import the package: (kind, p0, p1, seed, level)
REF_CONFIGS = {"c1": ("grid2d", 100, 100, 0, 0), "c2": ("lap7", 64, 0, 0, 1), "c3": ("stencil27", 48, 0, 1, 2),
               "c4": ("elasticity", 40, 0, 1, 0), "c5": ("diffusion", 32, 1000, 1, 1), "c6": ("lap7", 128, 0, 0, 1)}


class _Csr:
    def __init__(self, n, ptr, col, val=None):
        self.nrows, self.row_ptr, self.col_idx = n, ptr, col
        self.values = val if val is not None else np.ones(col.size)

    def nnz(self):
        return int(self.col_idx.size)


def run_reference(args):
    """The reference's own CPU path, nothing of this repo's product on it: the
    inputs come from the shim (the repo's seeded generators compiled into
    oracle/_ref next to the unmodified reference headers), the reference's
    analyze() orders and fills, and the timed call is its factor_by_blocks
    with TaskPolicy::pooled(all host threads) -- numeric_seconds, the same
    region as ours (factorize.hpp:169-227). factor_serial and pooled(1) are
    reported beside it. C5 batch: the 64 members' factor_serial spread over
    all host threads (the reference has no batch API), wall time."""
    rank, _, world = dist_env()
    if rank != 0:
        return
    from checkers import Reference, reference_available
    if not reference_available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref (reference compiled from /root/reference) was not built"}))
        return
    R = Reference()
    cores = os.cpu_count() or 1
    name = "c5" if args.config in ("c5", "c5b") else args.config
    kind, p0, p1, seed, level = REF_CONFIGS[name]

    def problem(sd):
        ptr, col, val = R.generate(kind, p0, p1, sd)
        n = ptr.size - 1
        ra = R.analyze(_Csr(n, ptr, col, val), level=level)
        return (n, _Csr(n, ra["a_ptr"], ra["a_col"], ra["a_val"]), _Csr(n, ra["u_ptr"], ra["u_col"]),
                ra["bounds"])

    n, ap, u, bounds = problem(seed)
    nnz = u.nnz()
    serial = [R.factor_serial(ap, u)[2] for _ in range(3)]
    pool1 = R.factor_by_blocks(ap, u, bounds, workers=1, want_values=False)[2]
    times, walls = [], []
    if args.config == "c5b":
        from concurrent.futures import ThreadPoolExecutor
        members = [ap] + [problem(b + 1)[1] for b in range(1, 64)]
        units = 64 * nnz
        with ThreadPoolExecutor(cores) as ex:
            for i in range(args.warmup + args.steps):
                t0 = time.perf_counter()
                sts = list(ex.map(lambda m: R.factor_serial(m, u)[1], members))
                dt = time.perf_counter() - t0
                if any(sts):
                    raise RuntimeError("reference factor_serial breakdown in the batch")
                if i >= args.warmup:
                    times.append(dt)
                    walls.append(dt)
        policy = f"64 x factor_serial over {cores} threads"
    else:
        units = nnz
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            _, st, secs, _, _, _ = R.factor_by_blocks(ap, u, bounds, workers=cores, want_values=False)
            wall = time.perf_counter() - t0
            if st != 0:
                raise RuntimeError(f"reference factor_by_blocks status {st}")
            if i >= args.warmup:
                times.append(secs)
                walls.append(wall)
        policy = f"TaskPolicy::pooled({cores})"
    t = statistics.mean(times)
    value = units / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.config == "c5b" else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, SURVEY.md Appendix B)",
        "config": {"workload": WORKLOADS[args.config], "n": n, "nnz_u": nnz, "policy": policy,
                   "inputs": "oracle/_ref: repo generators + the reference's analyze() (no product library)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{args.steps} full runs, {policy}; numeric_seconds"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_paths_ms": {"factor_serial_median": statistics.median(serial) * 1e3,
                               "factor_by_blocks_pooled1": pool1 * 1e3,
                               f"factor_by_blocks_pooled{cores}": t * 1e3 if args.config != "c5b" else None,
                               "one_shot_wall_median": statistics.median(walls) * 1e3},
    }
    print(json.dumps(line))


def golden_parity(got, names, aps, u):
    """'bitwise (golden hash)' when every member's factor hashes to the golden
    hash of the reference's factor_serial; else the max relative difference
    against the oracle (checker only)."""
    from checkers import Oracle
    O = Oracle()
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        golden = json.load(f)
    checked, by_oracle, bad = 0, 0, []
    for g, nm, ap in zip(got, names, aps):
        # (the single C5 matrix is member 0 of the batch)
        want = golden.get("c5_m0" if nm == "c5" else nm, {}).get("factor_values")
        if want is None:  # no fixture for this member: the oracle itself (checker only)
            ref = O.factor_serial(ap, u)[0]
            by_oracle += 1
            if not np.array_equal(np.ascontiguousarray(g).view(np.int64), ref.view(np.int64)):
                bad.append(float(np.max(np.abs(g - ref) / (np.abs(ref) + 1e-300))))
            continue
        checked += 1
        if O.hash(np.ascontiguousarray(g)) != want:
            ref = O.factor_serial(ap, u)[0]
            bad.append(float(np.max(np.abs(g - ref) / (np.abs(ref) + 1e-300))))
    if bad:
        return f"MISMATCH max_rel={max(bad):.3e}"
    how = []
    if checked:
        how.append(f"golden hash of the reference's factor_serial, {checked} checked")
    if by_oracle:
        how.append(f"the oracle's factor_serial, {by_oracle} checked")
    return "bitwise (" + "; ".join(how) + ")"


def chain_hop_us(dev: int) -> float:
    """Measured latency of one value hand-off between dependent rows: the
    factor of a 1,000-row tridiagonal matrix (IC(0), one range) is a pure
    chain of 1,000 finalising rows (SURVEY §8(d)'s latency bound)."""
    import numpy as np

    import paper_1601_05871_b200 as T
    n = 1000
    a = T.generate("path", n)
    fp = T.levelk_pattern(a, 0)
    plan = T.Plan(a, fp, T.RangeList(np.array([0, n], np.int32)))
    fz = T.GpuFactorizer(plan, T.GpuOptions(device=dev, mode=5))
    ts = []
    for _ in range(7):
        fz.restore()
        ts.append(fz.factor().device_ms)
    fz_depth = fz.flow_records()[2]  # the schedule's depth, built on the device
    fz.close()
    return statistics.median(ts) * 1e3 / fz_depth


def run_ours(args):
    import numpy as np
    import torch

    import paper_1601_05871_b200 as T

    rank, local_rank, world = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = local_rank

    a, an, plan, t_an = build_problem(args.config)
    ps = plan.stats()
    u = an.pattern.pattern
    nnz, n = u.nnz(), a.nrows
    fz = T.GpuFactorizer(plan, T.GpuOptions(device=dev, mode=args.mode, timeout_s=60))
    # the schedule's depth: built on the device at upload (or by the host plan)
    depth = (fz.flow_records()[2] if args.mode in (0, 5) else 0) or int(ps.flow_depth)
    _, prog_upd, prog_ms = fz.flow_programs() if args.mode in (0, 5) else (None, np.zeros((0, 2)), 0.0)
    nprod = len(prog_upd)
    del prog_upd
    batched = args.config == "c5b"
    nmembers_total, mine, batch_vals = 1, range(1), None
    if batched:
        from paper_1601_05871_b200 import batch as B
        nmembers_total = 64
        mine = B.shard(nmembers_total, rank, world)
        _, batch_vals, batch_perms = B.member_values(list(mine))
        fz.set_batch(batch_vals)
    per_rank = len(mine)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(dev).__enter__()  # nvidia-smi sampling spans every measured loop
    # warm-up
    for _ in range(args.warmup):
        fz.restore()
        fz.factor()
    # timed region: device time of the factor kernel per step
    dev_ms = []
    barrier()
    for _ in range(args.steps):
        fz.restore()            # untimed: U <- initialised values (D2D)
        flush.fill_(1.0)        # untimed: 256 MiB write evicts L2
        torch.cuda.synchronize()
        st = fz.factor()        # CUDA events around the persistent kernel
        dev_ms.append(st.device_ms)
    barrier()
    step_ms = statistics.mean(dev_ms)
    if world > 1:
        t = torch.tensor([step_ms], device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        step_ms = float(t.item())

    # end to end through the C ABI with host buffers (pinned): the reference's inputs,
    # PᵀAP's values, in; the factor out (tcg_factor_host_a: H2D of A, init_factor_values
    # on the device, prelude, factor, D2H)
    if batched:
        a_vals = np.stack([ap.values for ap in batch_perms]).reshape(-1)
    else:
        a_vals = an.a_permuted.values
    host_in = torch.from_numpy(np.ascontiguousarray(a_vals)).pin_memory()
    nnz_a = an.a_permuted.nnz()
    host_out = torch.empty(nnz * per_rank, dtype=torch.float64).pin_memory()
    e2e_ms = []
    barrier()
    # 9 more untimed calls: the call decides on this box how the factor leaves
    # (capi.cpp run_flow: a copy after the launch, the drain CTAs or chunked copies
    # beside the launch take turns over the first calls of a problem)
    for i in range(9 + args.warmup + args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st_e2e = fz.factor_host_a_ptr(host_in.data_ptr(), host_out.data_ptr())
        if i >= 9 + args.warmup:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
    barrier()
    if batched:  # back to the initialised batch for anything after
        fz.set_batch(batch_vals)
    clocks.__exit__(None, None, None)
    e2e = statistics.mean(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e], device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e = float(t.item())

    # parity of the last factor on every configuration: its hash against the
    # golden hash of the reference's factor_serial (tests/golden, produced by
    # the unmodified reference), i.e. bitwise equality with the reference
    parity = None
    if rank == 0:
        got = host_out.numpy().reshape(per_rank, nnz)
        names = [f"c5_m{m}" for m in mine] if batched else [args.config]
        parity = golden_parity(got, names, [an.a_permuted] if not batched else batch_perms, u)

    # one-shot drop-in call (the reference's unit of work, factorize.hpp:134-235):
    # factor_by_blocks_gpu from (PᵀAP, pattern, ranges) on the host to the factor on
    # the host -- plan, context, upload, factor, download, teardown -- wall time
    one_shot = None
    if not batched and not args.no_one_shot:
        walls, res = [], None
        for i in range(4):
            t0 = time.perf_counter()
            res = T.factor_by_blocks_gpu(an.a_permuted, an.pattern, an.ranges, T.GpuOptions(device=dev))
            if i:
                walls.append(time.perf_counter() - t0)
        one_shot = {"ms": statistics.median(walls) * 1e3, "calls": len(walls),
                    "plan_ms": res.stats.plan_seconds * 1e3, "block_build_ms": res.stats.block_build_seconds * 1e3,
                    "device_ms": res.stats.device_ms,
                    "parity": golden_parity(res.factor.values.reshape(1, -1), [args.config], [an.a_permuted], u)
                    if rank == 0 else None,
                    "call": "factor_by_blocks_gpu(a_permuted, fp, ranges): plan + tcg_create + upload + factor + "
                            "download + destroy, warm process (CUDA initialised), median of 3 after 1"}

    # CPU baseline (rank 0, N = 1): the reference's own serial factorization
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        times = cpu_reference_times(an, workers=min(os.cpu_count() or 1, 64), reps=3)
        if times:
            s_med = statistics.median(times["serial"])
            cpu = {"value": nnz / s_med, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": ("3 x factor_serial on one member (reference's fastest CPU path), median; "
                              "the batch rate on 1 core is the same per member") if batched else
                             "3 x factor_serial on the full matrix (reference's fastest CPU path), median",
                   "factor_by_blocks_pooled_s": statistics.median(times["pool"]),
                   "pooled_workers": min(os.cpu_count() or 1, 64),
                   "factor_by_blocks_pooled1_s": times["pool1"][0]}
    peak, peak_kind = measured_peak()
    hop_us = chain_hop_us(dev)
    bytes_alg = (20 * nnz + 8 * (n + 1)) * per_rank
    achieved = bytes_alg / (step_ms / 1e3) / 1e9
    launches_per_step = st.kernel_launches
    units = nmembers_total * nnz if batched else world * nnz   # factor entries per step, whole job
    line = {
        "metric": METRIC, "value": units / (step_ms / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "strong" if batched else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, SURVEY.md Appendix B)",
        "config": {"workload": WORKLOADS[args.config], "n": n, "nnz_u": nnz,
                   "tasks": int(sum(ps.tasks)),
                   "mode": {1: "task DAG / device merge", 2: "task DAG / update programs",
                            5: "value flow / static schedule of the finalising rows"}[st.mode],
                   "flow_rows": int(ps.flow_rows), "flow_depth": depth,
                   "grid_ctas": int(st.grid_ctas), "threads_per_cta": int(st.threads_per_cta),
                   "parallelism": (f"batch: {nmembers_total} members, {per_rank} on rank 0, one launch "
                                   f"per rank" if batched else
                                   f"replicas{world}" if world > 1 else "single"),
                   "l2": "flushed between steps (256 MiB write), U restored from device copy (untimed)",
                   "analysis_s": round(t_an, 3), "plan_s": round(ps.plan_seconds, 4),
                   "plan_host_threads": int(ps.host_threads),
                   "programs_device_ms": round(prog_ms, 3), "products": int(nprod),
                   "parity_vs_oracle": parity},
        "e2e": {"value": units / (e2e / 1e3), "unit": UNIT, "h2d_bytes_per_step": 8 * nnz_a * per_rank,
                "d2h_bytes_per_step": 8 * nnz * per_rank, "ms_per_step": e2e,
                "call": "tcg_factor_host_a: PaP values in (pinned host), device init_factor_values, factor, the "
                        "factor out (pinned host); how it leaves is calibrated per problem (d2h)",
                "d2h": ("copy after the launch" if st_e2e.drain_ctas == 0 else
                        f"{st_e2e.drain_ctas} drain CTAs of the launch (zero-copy stores)" if st_e2e.drain_ctas > 0 else
                        f"{-st_e2e.drain_ctas} chunks copied by the copy engine beside the launch as they become final"),
                "drain_ctas": int(st_e2e.drain_ctas),
                "launches": int(st_e2e.kernel_launches)},
        "gpu_launches": launches_per_step * args.steps,
        "launches_per_step": ({"flow_prepare (timed)": 1, "factor_flow (timed)": 1} if st.mode == 5 else
                              {"prepare (untimed)": 1, "factor": 1}),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(args.config),
                     "peak_kind": peak_kind, "algorithmic_bytes_per_launch": bytes_alg},
        # what actually binds: the dependence chain. Lower bound = value-flow depth x
        # the measured hand-off latency of a pure chain on this GPU.
        "latency_bound": {"flow_depth": depth, "hop_us": round(hop_us, 4),
                          "bound_ms": round(depth * hop_us / 1e3, 4),
                          "frac": round(depth * hop_us / 1e3 / step_ms, 4)},
        "cpu_baseline": cpu,
        "one_shot": one_shot,
        "clocks": clocks.summary(),
    }
    if rank == 0:
        print(json.dumps(line))
    fz.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def run_sharded(args):
    """C6 over N GPUs (BASELINE.json configs[4], second half): rank r owns the
    rows of the r-th level-log2(N) ND subtree; the N-1 separators above them
    go one per part (--separators spread, the default; rank0 keeps them all on
    rank 0); each rank runs its rows (mode 5) and reads the few operands other
    ranks own straight from their U through CUDA IPC peer mappings over
    NVLink (tcg_plan_part_problem / tcg_set_peers). Every rank resets its U
    (phase 1) before any rank's kernel starts (phase 2). value = nnz_u of the
    one matrix / max-over-ranks time (strong scaling)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1601_05871_b200 as T

    rank, local_rank, world = dist_env()
    dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = local_rank
    a, an, plan, t_an = build_problem(args.config)
    ps = plan.schedule().stats()  # the parts are slices of the host schedule
    u = an.pattern.pattern
    nnz, n = u.nnz(), a.nrows
    owners = an.subtree_owners(world, separators=0 if args.separators == "rank0" else "spread")
    problem = plan.part_problem(world, owners, rank)
    fz = T.GpuFactorizer(plan, T.GpuOptions(device=dev, mode=5, timeout_s=60), problem=problem)
    handle, offset = fz.ipc_handle()
    table = [None] * world
    dist.all_gather_object(table, (handle, offset))
    ptrs = [fz.values_device_ptr() if r == rank else fz.ipc_open(h, off) for r, (h, off) in enumerate(table)]
    fz.set_peers(ptrs)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")

    def barrier():
        torch.cuda.synchronize()
        dist.barrier()

    def step():
        fz.factor_phase(1)      # this part's U <- marker
        barrier()               # ... on every part before any kernel reads it
        return fz.factor_phase(2)

    clocks = ClockSampler(dev).__enter__()
    for _ in range(args.warmup):
        fz.restore()
        step()
    dev_ms = []
    for _ in range(args.steps):
        fz.restore()
        flush.fill_(1.0)
        st = step()
        dev_ms.append(st.device_ms)
    barrier()
    step_ms = max_over(statistics.mean(dev_ms), dev)
    host_in = torch.from_numpy(plan.flow_tables()["values"]).pin_memory()
    host_out = torch.empty(nnz, dtype=torch.float64).pin_memory()
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        flush.fill_(1.0)
        barrier()
        t0 = time.perf_counter()
        fz.set_values_ptr(host_in.data_ptr())   # H2D 8*nnz_u
        step()
        fz.download_ptr(host_out.data_ptr())    # D2H 8*nnz_u (this rank's rows valid)
        if i >= args.warmup:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
    clocks.__exit__(None, None, None)
    e2e = max_over(statistics.mean(e2e_ms), dev)
    # parity: every rank contributes its rows, rank 0 compares with the oracle
    own = np.repeat(owners, np.diff(u.row_ptr)) == rank
    mine = torch.from_numpy(np.where(own, host_out.numpy(), 0.0)).to(f"cuda:{dev}")
    dist.all_reduce(mine)  # rows are disjoint: the sum is the whole factor
    parity = None
    if rank == 0:
        from checkers import Oracle
        ref, _, _, _ = Oracle().factor_serial(an.a_permuted, u)
        got = mine.cpu().numpy()
        parity = "bitwise" if np.array_equal(ref.view(np.int64), got.view(np.int64)) else \
            f"max_rel={float(np.max(np.abs(got - ref) / (np.abs(ref) + 1e-300))):.3e}"
    peak, peak_kind = measured_peak()
    bytes_alg = 20 * nnz + 8 * (n + 1)
    line = {
        "metric": METRIC, "value": nnz / (step_ms / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, SURVEY.md Appendix B)",
        "config": {"workload": WORKLOADS[args.config] + f", ND subtrees sharded over {world} GPUs",
                   "n": n, "nnz_u": nnz, "flow_rows": int(ps.flow_rows), "flow_depth": int(ps.flow_depth),
                   "rows_rank0": int(problem.nflow), "remote_operands_rank0": int(problem.remote_operands),
                   "parallelism": f"ND subtrees over {world} ranks, peer reads over NVLink (CUDA IPC), separators {args.separators}",
                   "l2": "flushed between steps (256 MiB write), U restored from device copy (untimed)",
                   "analysis_s": round(t_an, 3), "parity_vs_oracle": parity},
        "e2e": {"value": nnz / (e2e / 1e3), "unit": UNIT, "h2d_bytes_per_step": 8 * nnz,
                "d2h_bytes_per_step": 8 * nnz, "ms_per_step": e2e},
        "gpu_launches": args.steps,
        "launches_per_step": {"flow_prepare (untimed, before the barrier)": 1, "factor_flow (timed)": 1},
        "roofline": {"bound": "hbm", "achieved": bytes_alg / (step_ms / 1e3) / 1e9, "peak": peak * world,
                     "unit": "GB/s", "frac": bytes_alg / (step_ms / 1e3) / 1e9 / (peak * world),
                     "traffic": None, "peak_kind": peak_kind + f" x {world}",
                     "algorithmic_bytes_per_launch": bytes_alg},
        "cpu_baseline": None,
        "clocks": clocks.summary(),
    }
    if rank == 0:
        print(json.dumps(line))
    fz.close()
    dist.destroy_process_group()


def run_symbolic(args):
    """--path symbolic: the level-k fill pattern on the device (tcg_sym_*, the
    reference's levelk_pattern_bfs, symbolic.hpp:57-120)
    on the config's PᵀAP. A step = count pass + scan + fill pass; value =
    nnz_u / device time; e2e = upload of PᵀAP's pattern + the step + download
    of the pattern through the C ABI from host buffers. Replicas for N > 1."""
    import numpy as np
    import torch

    import paper_1601_05871_b200 as T

    rank, local_rank, world = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = local_rank
    name = "c5" if args.config in ("c5", "c5b") else args.config
    a, level = T.config_matrix(name)
    an = T.analyze(a, level=level)
    ap_ = an.a_permuted
    n, nnz_a = ap_.nrows, ap_.nnz()
    g = T.GpuSymbolic(ap_, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(dev).__enter__()
    for _ in range(args.warmup):
        g.levelk(level)
    dev_ms = []
    barrier()
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        fp, st = g.levelk(level)
        dev_ms.append(st.device_ms)
    barrier()
    step_ms = statistics.mean(dev_ms)
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g.upload(ap_)                         # H2D: PᵀAP's row_ptr + col_idx
        fp_e, _ = g.levelk(level)             # D2H: U's row_ptr + col_idx
        if i >= args.warmup:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
    clocks.__exit__(None, None, None)
    e2e = statistics.mean(e2e_ms)
    g.close()
    if world > 1:
        step_ms, e2e = max_over(step_ms, dev), max_over(e2e, dev)
    same_e2e = np.array_equal(fp_e.pattern.col_idx, fp.pattern.col_idx)
    u = fp.pattern
    nnz_u = u.nnz()
    parity = None
    if rank == 0:
        same = np.array_equal(u.row_ptr, an.pattern.pattern.row_ptr) and \
            np.array_equal(u.col_idx, an.pattern.pattern.col_idx)
        parity = ("bit-exact vs host levelk (pinned to the reference's golden hashes)"
                  if same and same_e2e else "MISMATCH")
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from checkers import Reference, reference_available
        if reference_available():
            R = Reference()
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                R.levelk(ap_, level)
                ts.append(time.perf_counter() - t0)
            cpu = {"value": nnz_u / statistics.median(ts), "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": "3 x levelk_pattern_bfs on the full PaP (reference, oracle/_ref), median"}
    peak, peak_kind = measured_peak()
    bytes_alg = 8 * (n + 1) + 4 * nnz_a + 8 * (n + 1) + 4 * nnz_u
    achieved = bytes_alg / (step_ms / 1e3) / 1e9
    line = {
        "metric": "levelk_pattern_nnz_per_s", "value": world * nnz_u / (step_ms / 1e3), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic (seeded generator, SURVEY.md Appendix B)",
        "config": {"workload": WORKLOADS[args.config] + ": level-k symbolic of PaP", "path": "symbolic",
                   "n": n, "nnz_a": nnz_a, "nnz_u": nnz_u, "level": level, "slow_rows": st.slow_rows,
                   "grid_ctas": st.grid_ctas,
                   "l2": "flushed before every step (256 MiB write)", "parity": parity},
        "e2e": {"value": world * nnz_u / (e2e / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": 8 * (n + 1) + 4 * nnz_a, "d2h_bytes_per_step": 8 * (n + 1) + 4 * nnz_u,
                "ms_per_step": e2e},
        "gpu_launches": st.kernel_launches * args.steps,
        "launches_per_step": {"levelk_fast (tier 1, count + rows into scratch)": 1,
                              "levelk_fast (tier 2, rows past tier 1)": 1, "device scan": 1, "levelk_copy": 1},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "peak_kind": peak_kind, "algorithmic_bytes_per_launch": bytes_alg,
                     "note": "whole symbolic step (4 launches): PaP pattern read once, U pattern written once"},
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
    }
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


def run_solve(args):
    """--path solve: the IC(k) preconditioner apply z = (UᵀU)⁻¹ r with the GPU
    factor (tcg_solve_*): forward Uᵀ y = r then
    backward U z = y in one launch. A step = one apply with r resident in HBM;
    e2e = the apply through the C ABI from host buffers (H2D r, D2H z)."""
    import numpy as np
    import torch

    import paper_1601_05871_b200 as T

    rank, local_rank, world = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = local_rank
    a, an, plan, t_an = build_problem(args.config)
    u = an.pattern.pattern
    n, nnz = u.nrows, u.nnz()
    fz = T.GpuFactorizer(plan, T.GpuOptions(device=dev, timeout_s=60))
    fz.factor()
    s = T.GpuTriSolve(fz)
    r = np.random.default_rng(11).standard_normal(n)
    rd = torch.from_numpy(r).to(f"cuda:{dev}")
    zd = torch.empty_like(rd)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(dev).__enter__()
    for _ in range(args.warmup):
        s.apply_device_ptr(rd.data_ptr(), zd.data_ptr(), 3)
    dev_ms = []
    barrier()
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        st = s.apply_device_ptr(rd.data_ptr(), zd.data_ptr(), 3)
        dev_ms.append(st.device_ms)
    barrier()
    step_ms = statistics.mean(dev_ms)
    host_r = torch.from_numpy(r).pin_memory()
    host_z = torch.empty(n, dtype=torch.float64).pin_memory()
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.apply_host_ptr(host_r.data_ptr(), host_z.data_ptr(), 3)
        if i >= args.warmup:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
    clocks.__exit__(None, None, None)
    e2e = statistics.mean(e2e_ms)
    if world > 1:
        step_ms, e2e = max_over(step_ms, dev), max_over(e2e, dev)
    parity, cpu = None, None
    if rank == 0:
        from checkers import Oracle
        O = Oracle()
        vals = fz.download()
        t0 = time.perf_counter()
        ref = O.trisolve(u, vals, r, 3)
        t_cpu = time.perf_counter() - t0
        got = host_z.numpy()
        parity = "bitwise vs oracle orc_trisolve" if np.array_equal(got.view(np.int64), ref.view(np.int64)) \
            else f"max_rel={float(np.max(np.abs(got - ref) / (np.abs(ref) + 1e-300))):.3e}"
        if world == 1 and not args.no_cpu:
            ts = [t_cpu]
            for _ in range(2):
                t0 = time.perf_counter()
                O.trisolve(u, vals, r, 3)
                ts.append(time.perf_counter() - t0)
            cpu = {"value": nnz / statistics.median(ts), "unit": UNIT, "cores": 1, "kind": "port",
                   "sample": "3 x orc_trisolve (oracle's sequential forward + backward substitution; the "
                             "reference has no solve), median"}
    s.close()
    fz.close()
    peak, peak_kind = measured_peak()
    bytes_alg = 2 * 12 * nnz + 32 * n
    achieved = bytes_alg / (step_ms / 1e3) / 1e9
    line = {
        "metric": "ic_apply_factor_nnz_per_s", "value": world * nnz / (step_ms / 1e3), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, SURVEY.md Appendix B); r ~ N(0,1) seed 11",
        "config": {"workload": WORKLOADS[args.config] + ": preconditioner apply (UᵀU)^-1 r", "path": "solve",
                   "n": n, "nnz_u": nnz, "depth_forward": st.depth_forward, "depth_backward": st.depth_backward,
                   "grid_ctas": st.grid_ctas, "l2": "flushed before every step (256 MiB write)",
                   "parity_vs_oracle": parity},
        "e2e": {"value": world * nnz / (e2e / 1e3), "unit": UNIT, "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n, "ms_per_step": e2e},
        "gpu_launches": st.kernel_launches * args.steps,
        "launches_per_step": {"trisolve_flow": 1, "memset (marker)": 2, "copy (result)": 1},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "peak_kind": peak_kind, "algorithmic_bytes_per_launch": bytes_alg,
                     "note": "U values + an int32 index per entry, once per direction; 4 vectors of n"},
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
    }
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


def run_reference_symbolic(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    from checkers import Reference, reference_available

    import paper_1601_05871_b200 as T
    if not reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref was not built"}))
        return
    name = "c5" if args.config in ("c5", "c5b") else args.config
    a, level = T.config_matrix(name)
    an = T.analyze(a, level=level)
    R = Reference()
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        ptr, _ = R.levelk(an.a_permuted, level)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    nnz_u = int(ptr[-1])
    t = statistics.mean(times)
    print(json.dumps({
        "impl": "reference", "metric": "levelk_pattern_nnz_per_s", "value": nnz_u / t, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config] + ": level-k symbolic of PaP", "path": "symbolic",
                   "nnz_u": nnz_u},
        "cpu_baseline": {"value": nnz_u / t, "unit": UNIT, "cores": 1, "kind": "reference",
                         "sample": f"{args.steps} x levelk_pattern_bfs (sequential in the reference)"},
        "e2e": {"value": nnz_u / t, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


def max_over(x, dev):
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{dev}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(WORKLOADS),
                    help="c3 (default): the largest single-GPU configuration of BASELINE.json")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", type=int, default=0, help="0 auto (5: value flow), 1/2 task DAG")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--separators", default="spread", choices=["spread", "rank0"],
                    help="C6 over N GPUs: ND separators spread over the parts (one each) or all on rank 0")
    ap.add_argument("--no-one-shot", action="store_true", help="skip the one-shot drop-in calls")
    ap.add_argument("--path", default="factor", choices=["factor", "symbolic", "solve"],
                    help="factor: the numeric factorization (headline); symbolic: level-k pattern on the "
                         "device; solve: the preconditioner apply with the factor")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warm-up raised to 3 (timing rule)")
        args.warmup = 3
    if args.path == "symbolic":
        run_reference_symbolic(args) if args.impl == "reference" else run_symbolic(args)
    elif args.path == "solve":
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "path": "solve",
                              "unavailable": "the reference has no triangular solve (SPEC.md:477); "
                                             "bench --path solve reports the oracle port as cpu_baseline"}))
        else:
            run_solve(args)
    elif args.impl == "reference":
        run_reference(args)
    elif args.config == "c6" and dist_env()[2] > 1:
        run_sharded(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
