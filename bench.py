#!/usr/bin/env python
"""bench.py -- vertex-updates/s of the LMS sweep and % of HBM roofline on B200.

Metric (BASELINE.json): "vertex-updates/sec per LMS sweep and % of HBM roofline
at 1/2/4/8 B200".  Workload at N=1: configs[3] (C4, 2D jittered grid 4096^2,
16.8 M vertices, 50 sweeps, 738 MB CSR+coords -- larger than the 126 MB L2, so
no L2 flush is needed between steps), best ordering (original, row-major).

One timed STEP = lms_smooth(mesh, 50 sweeps) on the HBM-resident relabelled
mesh (A9, the hot loop).  The preparation rows of the path (A2-A8: CSR build,
fixed mask, colouring, ordering, relabelling, schedule) are timed separately in
the same run ("setup_ms"), and the end-to-end number ("e2e") runs the WHOLE
path per step through the public API from pinned host buffers: H2D of
coordinates + elements, build_csr, order, permute, smooth(50), D2H of the
smoothed coordinates.

value = V_free * sweeps * steps / t  (t = max over ranks of the CUDA-event time).
roofline.achieved = B_sweep * sweeps / (sweep-kernel time per step),
B_sweep = 4(V+1) + 4 nnz + 8 d V + 8 d V_free bytes.

--impl reference: the CPU oracle (oracle/, test infrastructure) timed as it
stands on the host cores, each step one colour-GS sweep of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import meshgen  # noqa: E402

FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
# BASELINE.json's metric, printed verbatim by both arms (the driver divides
# the two lines only when the strings match)
METRIC = "vertex-updates/sec per LMS sweep and % of HBM roofline at 1/2/4/8 B200"


def l2_note(V, nnz, dim):
    mb = (4 * (V + 1) + 4 * nnz + 8 * dim * V) / 1e6
    if mb > 126:
        return "inputs larger than L2 (resident CSR+coords %.0f MB > 126 MB); no flush" % mb
    return "L2-resident (CSR+coords %.0f MB <= 126 MB): effective bandwidth, not an HBM figure" % mb


def workload_config(args, cfg, sweeps, V, vfree, nnz, C, dim, world=1, how=None):
    """The `config` object both arms print (identical for the same workload)."""
    return {"workload": f"{args.config}: {cfg['desc']}, {args.ordering} ordering, "
                        f"{sweeps} colour-GS sweeps per step",
            "config": args.config, "ordering": args.ordering, "sweeps_per_step": sweeps,
            "V": V, "V_free": vfree, "nnz": nnz, "colours": C,
            "l2": l2_note(V, nnz, dim),
            "parallelism": how or (f"contiguous vertex ranges x{world}" if world > 1 else "1 GPU")}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C4")
    p.add_argument("--ordering", default="original")
    p.add_argument("--sweeps", type=int, default=0, help="0 = the config's sweep count")
    p.add_argument("--schedule", default="auto", choices=["auto", "s1", "s3", "gz"])
    p.add_argument("--tile", type=int, default=0)
    p.add_argument("--lag", type=int, default=0)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--jobs-in-flight", type=int, default=4,
                   help="e2e: jobs kept in flight on as many streams (job k on stream k %% N)")
    p.add_argument("--cpu-sweeps", type=int, default=2)
    p.add_argument("--force-dist", action="store_true",
                   help="take the multi-GPU path even at one rank (tests its plumbing under torchrun)")
    return p.parse_args()


def b_sweep(dim, V, nnz, vfree):
    return 4 * (V + 1) + 4 * nnz + 8 * dim * V + 8 * dim * vfree


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy test)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.maxclk = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.maxclk = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def record(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.maxclk, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.maxclk,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def load_traffic(config, ordering, kernel):
    """ncu DRAM bytes per launch of the sweep kernel from the committed capture
    (profiles/ncu_summary.json), or None.  The capture records the sha256 of
    the kernel's source file; a capture of another version of the kernel is
    stale and not reported."""
    import hashlib
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    src = os.path.join(ROOT, "paper_1606_00803_b200", "csrc", "gz.cu")
    try:
        with open(path) as f:
            d = json.load(f)
        with open(src, "rb") as f:
            sha = hashlib.sha256(f.read()).hexdigest()
        for rec in d.get("kernels", []):
            if rec.get("config") == config and rec.get("ordering") == ordering and rec.get("kernel") == kernel:
                return rec if rec.get("gz_cu_sha256") == sha else None
    except Exception:
        pass
    return None


# --------------------------------------------------------------------------- reference arm
def _oracle_mesh(args, m):
    import oracle
    om = oracle.prepare(m)
    if args.ordering != "original":
        om = oracle.permute_mesh(om, oracle.order(om, args.ordering, meshgen.RANDOM_ORDER_SEED))
    return om


def _oracle_rate(om, sweeps, threads):
    """vertex-updates/s of `sweeps` oracle sweeps in one call (colour lists built
    once per call, coordinates smoothed in place: the sweep loop is what is
    timed); returns (rate, threads used, seconds)."""
    import oracle
    X = [np.array(c, dtype=np.float64, copy=True) for c in om["coords"]]
    vfree = int((om["fixed"] == 0).sum())
    t0 = time.perf_counter()
    r = oracle.smooth(X, om["row_ptr"], om["col"], om["colour"], om["C"], sweeps, threads=threads, inplace=True)
    dt = time.perf_counter() - t0
    used = r[1] if threads > 0 else 1
    return vfree * sweeps / dt, used, dt


def run_reference(args):
    """The CPU oracle as it stands, on the host cores (o_smooth_omp, all cores),
    timed on a bounded sample of our arm's workload: each step is ONE
    colour-GS sweep of the same mesh (the metric is a rate)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = meshgen.CONFIGS[args.config]
    sweeps = args.sweeps or cfg["sweeps"]
    m = meshgen.make_config(args.config)
    om = _oracle_mesh(args, m)
    V = om["coords"][0].shape[0]
    vfree = int((om["fixed"] == 0).sum())
    cores = len(os.sched_getaffinity(0))
    _oracle_rate(om, max(1, args.warmup), cores)  # warm-up sweeps (untimed)
    value, used, dt = _oracle_rate(om, args.steps, cores)
    sample = (f"{args.steps} sweeps of the full {args.config} mesh ({V} vertices, {args.ordering} ordering), "
              f"one sweep per step, o_smooth_omp on {used} threads, sweep loop only")
    line = {"impl": "reference", "metric": METRIC, "value": value,
            "unit": "vertex-updates/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, cfg, sweeps, V, vfree, int(om["row_ptr"][-1]), int(om["C"]), m["dim"]),
            "cpu_baseline": {"value": value, "unit": "vertex-updates/s", "cores": used, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "vertex-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- our arm
def cpu_baseline(args, m):
    """the oracle on 1 host core (o_smooth) and on all N host
    cores (o_smooth_omp, bit-identical), sweep loop only."""
    t0 = time.perf_counter()
    om = _oracle_mesh(args, m)
    prep = time.perf_counter() - t0
    cores = len(os.sched_getaffinity(0))
    n = args.cpu_sweeps
    v1, _, t1 = _oracle_rate(om, n, 0)
    vn, used, tn = _oracle_rate(om, n, cores)
    try:
        import cpuinfo
        cpu_model = cpuinfo.get_cpu_info().get("brand_raw")
    except Exception:
        cpu_model = None
    return {"value": vn, "unit": "vertex-updates/s", "cores": used, "kind": "oracle",
            "value_1core": v1, "cpu_model": cpu_model,
            "sample": f"{n} colour-GS sweeps of the full {args.config} mesh ({args.ordering}) on 1 core "
                      f"({t1:.2f} s, o_smooth) and on {used} cores ({tn:.2f} s, o_smooth_omp), sweep loop only "
                      f"(oracle prep {prep:.1f}s untimed)"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1606_00803_b200 as lms

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or args.force_dist:
        # communicator sizes in the log (the library's own NCCL communicator included)
        os.environ["NCCL_DEBUG"] = "INFO"
        os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    cfg = meshgen.CONFIGS[args.config]
    sweeps = args.sweeps or cfg["sweeps"]
    m = meshgen.make_config(args.config)
    dim = m["dim"]
    V = m.V
    if world > 1 or args.force_dist:
        return run_ours_dist(args, m, cfg, sweeps, world, rank, dev)

    # ---------------- setup phases (A2-A8), each timed with CUDA events
    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e
    coords_d = [torch.from_numpy(c).to(dev) for c in m["coords"]]
    elems_d = torch.from_numpy(m["elems"]).to(dev)
    torch.cuda.synchronize()
    setup = {}
    e0 = ev()
    gm = lms.Mesh.build_csr(coords_d, elems_d)
    e1 = ev()
    perm = gm.order(args.ordering, meshgen.RANDOM_ORDER_SEED if args.ordering == "random" else 0)
    e2 = ev()
    gm.permute(perm)
    e3 = ev()
    gm.set_schedule(args.schedule, args.tile, args.lag)
    gm.smooth(0)
    # schedule build happens lazily on the first non-zero smooth: time it via 1 sweep minus a sweep
    torch.cuda.synchronize()
    setup["build_csr+boundary+colour"] = e0.elapsed_time(e1)
    setup["order_" + args.ordering] = e1.elapsed_time(e2)
    setup["permute"] = e2.elapsed_time(e3)
    e4 = ev()
    gm.smooth(1)  # builds the schedule + 1 sweep
    e5 = ev()
    torch.cuda.synchronize()
    setup["schedule+1sweep"] = e4.elapsed_time(e5)
    info = gm.info()
    sinfo = gm.schedule_info()
    nnz, C, vfree = info["nnz"], info["C"], sinfo["n_free"]
    bsw = b_sweep(dim, V, nnz, vfree)

    # ---------------- timed steps: lms_smooth(sweeps)
    for _ in range(args.warmup):
        gm.smooth(sweeps)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lms.kernel_launches()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for i in range(args.steps):
            starts[i].record(stream)
            gm.smooth(sweeps)
            ends[i].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
    launches = lms.kernel_launches() - launches0
    t_ms = t_start.elapsed_time(t_end)
    if world > 1:
        tt = torch.tensor([t_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    step_mean = statistics.mean(step_ms)
    value = vfree * sweeps * args.steps / (t_ms / 1e3) * world
    peak, peak_src = peaks()
    # the dominant kernel and its launches per step: GZ = one launch per pass of
    # P sweeps; S3 = one persistent launch per step; S1 = C launches per sweep
    kind = sinfo["kind"]
    if kind == "gz":
        kname, per_launch_sweeps = "k_sweep_gz", max(1, sinfo["lag"])
    elif kind == "s3":
        kname, per_launch_sweeps = "k_sweep_s3", sweeps
    else:
        kname, per_launch_sweeps = "k_sweep_s1", 1
    n_launch = max(1, -(-sweeps // per_launch_sweeps))
    launch_ms = step_mean / n_launch
    achieved = bsw * sweeps / (step_mean / 1e3) / 1e9  # = bytes per launch / launch time
    tr = load_traffic(args.config, args.ordering, kname)
    traffic = None
    if tr is not None and tr.get("sweeps"):
        traffic = tr["dram_bytes"] / tr["sweeps"] * per_launch_sweeps
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "peak_source": peak_src, "kernel": kname,
            "bytes_per_launch": bsw * per_launch_sweeps, "launch_ms": launch_ms, "launches_per_step": n_launch,
            "b_sweep": bsw, "frac_of_8TBs_nominal": achieved / 8000.0,
            "traffic_source": tr.get("source") if tr else None}

    # ---------------- e2e: whole path from pinned host buffers, every step
    # (the device-timed mesh is released first: a user's job starts from host
    # buffers, without another resident mesh fragmenting the allocator pool)
    gm.close()
    del coords_d, elems_d
    torch.cuda.synchronize()
    e2e = None
    if not args.no_e2e:
        hc = [torch.from_numpy(c).pin_memory() for c in m["coords"]]
        he = torch.from_numpy(m["elems"]).pin_memory()
        hout = [torch.empty(V, dtype=torch.float64).pin_memory() for _ in range(dim)]
        h2d = sum(t.numel() * t.element_size() for t in hc) + he.numel() * he.element_size()
        d2h = sum(t.numel() * t.element_size() for t in hout)

        # lms_build_csr_host: elements up on the stream, coordinates on the
        # library's side stream under the CSR build and colouring
        def e2e_step():
            g = lms.Mesh.build_csr_host(hc, he)
            p = g.order(args.ordering, meshgen.RANDOM_ORDER_SEED if args.ordering == "random" else 0)
            g.permute(p)
            g.set_schedule(args.schedule, args.tile, args.lag)
            g.smooth(sweeps)
            out = g.coords()
            for o, h in zip(out, hout):
                h.copy_(o, non_blocking=True)
            torch.cuda.synchronize()
            g.close()
        for _ in range(2):  # first calls (module loading, pool growth)
            e2e_step()
        # phase breakdown of one e2e step (CUDA events; informational).  It runs
        # before the last warm steps: its smooth(1) + smooth(n - 1) split
        # allocates differently, and the plain steps after it settle the scratch
        # cache for the timed ones
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
        evs[0].record(stream)
        evs[1].record(stream)
        g = lms.Mesh.build_csr_host(hc, he)
        evs[2].record(stream)
        p = g.order(args.ordering, meshgen.RANDOM_ORDER_SEED if args.ordering == "random" else 0)
        g.permute(p)
        evs[3].record(stream)
        g.set_schedule(args.schedule, args.tile, args.lag)
        g.smooth(1)
        evs[4].record(stream)
        g.smooth(sweeps - 1)
        evs[5].record(stream)
        out = g.coords()
        for o, h in zip(out, hout):
            h.copy_(o, non_blocking=True)
        evs[6].record(stream)
        torch.cuda.synchronize()
        g.close()
        names = ["h2d", "h2d+build_csr+colour", "order+permute", "schedule+1sweep", "sweeps", "d2h"]
        e2e_phases = {nm: evs[i].elapsed_time(evs[i + 1]) for i, nm in enumerate(names) if i > 0}
        for _ in range(3):  # warm steps: the library's scratch cache settles into the steady pattern
            e2e_step()
        n_e2e = max(3, min(args.steps, 5))
        torch.cuda.synchronize()
        sev = [torch.cuda.Event(enable_timing=True) for _ in range(n_e2e + 1)]
        sev[0].record(stream)
        for k in range(n_e2e):
            e2e_step()
            sev[k + 1].record(stream)
        torch.cuda.synchronize()
        lat_ms = sev[0].elapsed_time(sev[-1]) / n_e2e
        step_ms = [round(sev[k].elapsed_time(sev[k + 1]), 2) for k in range(n_e2e)]
        # throughput with N jobs in flight (a serving loop, N = 4 by default):
        # job k runs on stream k % N, so one job's H2D / D2H copies (PCIe) and
        # its host round trips overlap the other jobs' kernels; the kernels
        # themselves still share the SMs.  Every job copies its whole input
        # from pinned host memory and its result back.  (Measured on one box:
        # N = 2 35.0-36.2 ms per job, N = 3 34.0-34.3, N = 4 33.5-34.2 once
        # the library's scratch cache holds all N jobs' blocks -- with a 16 GB
        # cap N = 4 stalled 50-150 ms in some runs; profiles/round2/tile_walk/.)
        nj = max(1, args.jobs_in_flight)
        strs = [torch.cuda.Stream() for _ in range(nj)]
        houts = [hout] + [[torch.empty(V, dtype=torch.float64).pin_memory() for _ in range(dim)] for _ in range(nj - 1)]
        n_pipe = max(n_e2e, 2 * nj)

        def e2e_job(slot, keep):
            with torch.cuda.stream(strs[slot]):
                g = lms.Mesh.build_csr_host(hc, he)
                g.set_async_errors(True)  # smooth() returns once enqueued; checked after the loop
                p = g.order(args.ordering, meshgen.RANDOM_ORDER_SEED if args.ordering == "random" else 0)
                g.permute(p)
                g.set_schedule(args.schedule, args.tile, args.lag)
                g.smooth(sweeps)
                out = g.coords()
                for o, h in zip(out, houts[slot]):
                    h.copy_(o, non_blocking=True)
            keep.append((g, out, p))

        def pipelined(n):
            keep = []
            torch.cuda.synchronize()
            a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a.record(strs[0])
            for st in strs[1:]:
                st.wait_event(a)
            for k in range(n):
                e2e_job(k % nj, keep)
            for st in strs[1:]:
                ev = torch.cuda.Event()
                ev.record(st)
                strs[0].wait_event(ev)
            c.record(strs[0])
            torch.cuda.synchronize()
            for g, _, _ in keep:
                g.check()
                g.close()
            return a.elapsed_time(c) / n
        pipelined(n_pipe)  # warm: the allocator caches of every stream
        # three timed runs of n_e2e jobs, the median reported (a single run
        # occasionally carries a one-off stall of a few hundred ms)
        e_runs = [pipelined(n_pipe) for _ in range(3)]
        e_ms = statistics.median(e_runs)
        e2e = {"value": vfree * sweeps / (e_ms / 1e3) * world, "unit": "vertex-updates/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e_ms,
               "jobs_in_flight": nj, "steps": n_pipe, "runs_ms_per_step": [round(x, 2) for x in e_runs],
               "latency_ms_per_job": lat_ms, "serial_value": vfree * sweeps / (lat_ms / 1e3) * world,
               "serial_step_ms": step_ms, "phases_ms": e2e_phases,
               "path": "per job: build_csr_host (H2D elems, then CSR + colouring under the H2D of coords) -> order "
                       "-> permute -> smooth(%d) -> D2H coords; %d jobs, %d in flight on %d streams (value, "
                       "ms_per_step: the median of three such runs); serial_value / latency_ms_per_job: one job at a time"
                       % (sweeps, n_pipe, nj, nj)}

    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_baseline(args, m)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "vertex-updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, cfg, sweeps, V, vfree, nnz, C, dim, world),
            "schedule": sinfo,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.record(),
            "setup_ms": setup,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_ours_dist(args, m, cfg, sweeps, world, rank, dev):
    """N > 1 (or --force-dist): the multi-GPU C ABI (include/lms.h lms_dist_*).
    Every rank builds the mesh on its GPU (lms_build_csr), relabels it, and
    calls lms_dist_create with the NCCL uid broadcast from rank 0: the
    library builds the rank's plan from its own contiguous range
    and owns the NCCL communicator.  One timed step = lms_smooth_dist(sweeps):
    per pass of P sweeps one halo exchange (ncclSend/ncclRecv over NVLink),
    then the GZ pass on the rank's local mesh.  Weak/strong: the mesh is
    fixed, so this is strong scaling; value = all ranks' updates / max time."""
    import torch
    import torch.distributed as dist

    import paper_1606_00803_b200 as lms
    stream = torch.cuda.current_stream()
    dim, V = m["dim"], m.V
    P = max(1, args.lag)
    seed = meshgen.RANDOM_ORDER_SEED if args.ordering == "random" else 0

    def uid():
        obj = [lms.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def make_dist(g):
        g.permute(g.order(args.ordering, seed))
        return lms.Dist.create(g, rank, world, uid(), sweeps_per_exchange=P, tile=args.tile)

    coords_d = [torch.from_numpy(c).to(dev) for c in m["coords"]]
    elems_d = torch.from_numpy(m["elems"]).to(dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gm = lms.Mesh.build_csr(coords_d, elems_d)
    info = gm.info()
    vfree = gm.schedule_info()["n_free"]
    d = make_dist(gm)
    gm.close()
    torch.cuda.synchronize()
    plan_s = time.perf_counter() - t0
    dinfo = d.info()
    bsw = b_sweep(dim, V, info["nnz"], vfree)
    for _ in range(args.warmup):
        d.smooth(sweeps)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = lms.kernel_launches()
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            d.smooth(sweeps)
        b.record(stream)
        torch.cuda.synchronize()
    launches = lms.kernel_launches() - launches0
    t_ms = a.elapsed_time(b)
    tt = torch.tensor([t_ms], device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms = float(tt.item())
    value = vfree * sweeps * args.steps / (t_ms / 1e3)
    # e2e: per step every rank ingests the mesh from pinned host buffers,
    # builds, orders, relabels, re-plans (lms_dist_replan: the communicator
    # is a once-per-job set-up, kept), smooths and reads its owned result back
    e2e = None
    if not args.no_e2e:
        del coords_d, elems_d
        hc = [torch.from_numpy(c).pin_memory() for c in m["coords"]]
        he = torch.from_numpy(m["elems"]).pin_memory()
        first, count = None, None

        first_, count_ = d.owned_range()
        outs = [torch.empty(count_, dtype=torch.float64).pin_memory() for _ in range(dim)]

        def e2e_step():
            g = lms.Mesh.build_csr_host(hc, he)
            g.permute(g.order(args.ordering, seed))
            d.replan(g, tile=args.tile)
            g.close()
            d.smooth(sweeps)
            f, xs = d.export_owned()
            for o, x in zip(outs, xs):
                o.copy_(x, non_blocking=True)
            torch.cuda.synchronize()
            return f, xs[0].numel()
        for _ in range(2):
            first, count = e2e_step()
        dist.barrier()
        torch.cuda.synchronize()
        n_e2e = max(2, min(args.steps, 3))
        ea = torch.cuda.Event(enable_timing=True)
        eb = torch.cuda.Event(enable_timing=True)
        ea.record(stream)
        for _ in range(n_e2e):
            e2e_step()
        eb.record(stream)
        torch.cuda.synchronize()
        e_ms = ea.elapsed_time(eb) / n_e2e
        et = torch.tensor([e_ms], device=dev)
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e_ms = float(et.item())
        h2d = sum(c.nbytes for c in m["coords"]) + m["elems"].nbytes
        e2e = {"value": vfree * sweeps / (e_ms / 1e3), "unit": "vertex-updates/s", "h2d_bytes_per_step": h2d,
               "note": "host buffers are the whole mesh on every rank (each rank builds the full mesh)",
               "d2h_bytes_per_step": 8 * dim * count, "ms_per_step": e_ms, "steps": n_e2e,
               "path": "per rank: build_csr_host (whole mesh) -> order -> permute -> lms_dist_replan (plan + NCCL "
                       "ghost lists) -> lms_smooth_dist(%d) -> lms_dist_export_owned -> D2H; max over ranks" % sweeps}
    d.close()
    peak, peak_src = peaks()
    achieved = bsw * sweeps * args.steps / (t_ms / 1e3) / 1e9 / world
    if rank == 0:
        how = (f"contiguous vertex ranges x{world} (lms_dist_*), deep halo {dinfo['depth']} hops, one NCCL "
               f"exchange per {P}-sweep pass")
        line = {
            "metric": METRIC,
            "value": value, "unit": "vertex-updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, cfg, sweeps, V, vfree, info["nnz"], info["C"], dim, world, how),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
                         "kernel": "k_sweep_gz + halo pack/unpack (per GPU)", "per_gpu": True},
            "cpu_baseline": None, "e2e": e2e, "gpu_launches": launches, "clocks": clk.record(),
            "dist": dict(dinfo, plan_s_rank0=plan_s),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
