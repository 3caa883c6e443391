#!/usr/bin/env python
"""Benchmark of the batched straightest-geodesic exponential map + EP backward (BASELINE.json).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3] [--impl ours|reference]

One "step" = one pass of the hot path over the whole query batch: forward trace of every
geodesic + the scheme's backward (EP for c2, GFD for c3). Workload at N=1 (default): config 2,
bumpy sphere (icosphere-6 displaced radially, 81 920 faces), 1 M geodesics of length
0.5 x bbox diagonal, forward + EP backward. Prints ONE JSON line.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_CROSSING = 48     # 3 vertex ids + 3 neighbour ids + one new f64 position
BYTES_PER_GEODESIC = 116    # 52 B query in + 64 B result out
EP_BYTES_PER_SAMPLE = 24 + 24 + 2 * (12 + 72)

WORKLOADS = {
    "c2": dict(name="bumpy-sphere ico-6 (81,920 faces), 1M geodesics, length 0.5 x bbox diagonal, forward + EP backward",
               scheme="ep", n=1_000_000),
    "c3": dict(name="noisy torus 1000x500 (1,000,000 faces), geodesics of length 0.5 x bbox diagonal, forward + GFD backward",
               scheme="gfd", n=1_000_000),
}


def make_workload(key, n, seed):
    from paper_2603_15780_b200 import workloads as W
    if key == "c2":
        xyz, tri = W.bumpy_sphere(6)
    else:
        xyz, tri = W.torus(1 / 3, 1 / 6, 1000, 500, noise=0.1, seed=7)
    diag = W.bbox_diagonal(xyz)
    f, b, d = W.sample_queries(xyz, tri, n, 0.5 * diag, seed=seed)
    rng = np.random.default_rng(seed + 1)
    q = rng.normal(size=(n, 3))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return xyz, tri, f, b, d, q


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML in a thread (every 2 ms plus the query time,
    so that a 20 ms region still gets samples), `nvidia-smi -lms` as the fallback when NVML cannot be loaded."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.sm, self.mx, self.seen, self.index = [], [], set(), index
        self.proc = self.nvml = self.handle = None
        self.stop = threading.Event()
        self.source = None

    def _open_nvml(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            uuid = "GPU-" + str(torch.cuda.get_device_properties(self.index).uuid)
            try:
                self.handle = pynvml.nvmlDeviceGetHandleByUUID(uuid)
            except TypeError:
                self.handle = pynvml.nvmlDeviceGetHandleByUUID(uuid.encode())
        except Exception:
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            ids = [v for v in vis.split(",") if v.strip().isdigit()]
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(int(ids[self.index]) if self.index < len(ids) else self.index)
        self.nvml = pynvml
        self.bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                     "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                     "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                     "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
        self.mx.append(float(pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)))

    def _sample_nvml(self):
        nv = self.nvml
        try:
            self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM)))
            mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
            self.seen.update(nm for nm, bit in self.bits.items() if mask & bit)
        except Exception:
            pass

    def _poll_nvml(self):
        while not self.stop.is_set():
            self._sample_nvml()
            self.stop.wait(0.002)

    def _read_smi(self):
        for line in self.proc.stdout:
            r = [c.strip() for c in line.split(",")]
            if len(r) >= 6 and r[0].replace(".", "").isdigit():
                self.sm.append(float(r[0]))
                if r[1].replace(".", "").isdigit():
                    self.mx.append(float(r[1]))
                self.seen.update(nm for k, nm in enumerate(self.NAMES) if r[2 + k] == "Active")

    def __enter__(self):
        try:
            self._open_nvml()
            self.source = "nvml"
            self.t = threading.Thread(target=self._poll_nvml, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.source = "nvidia-smi"
            self.t = threading.Thread(target=self._read_smi, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.nvml:
            self.stop.set()
            self.t.join(timeout=2)
            if not self.sm:          # a region shorter than one NVML round trip: the clock it ends on
                self._sample_nvml()
        elif self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            self.t.join(timeout=2)

    def summary(self):
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": [nm for nm in self.NAMES if nm in self.seen], "samples": len(self.sm), "source": self.source}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def gather_roofline(mesh, crossings_per_s):
    """Measured gather rates (G records/s) of scripts/micro/gather_bench.cu / gather4_bench.cu on B200 at 31 MB,
    384 MB and 1.5 GB of records, per gather; the nearest size at or above the mesh's record array is the ceiling."""
    table = {"loads": ((31e6, 67.0), (384e6, 16.5), (1.5e9, 10.3)), "coop": ((31e6, 86.6), (384e6, 65.6), (1.5e9, 40.9)),
             "tma": ((31e6, 106.0), (384e6, 65.0), (1.5e9, 40.0))}
    if not mesh.has_transport_cache:
        return None
    rec_bytes = 3 * mesh.nf * 128
    peak = next((r for size, r in table[mesh.gather] if rec_bytes <= size * 1.05), table[mesh.gather][-1][1])
    return {"gather": mesh.gather, "record_bytes": rec_bytes, "achieved_grecords_per_s": crossings_per_s / 1e9,
            "peak_grecords_per_s": peak, "frac": crossings_per_s / 1e9 / peak, "source": "scripts/micro/gather_bench.cu (profiles/tuning_r1.md)"}


def profile_traffic(workload):
    """dram bytes per launch of the trace kernel from the committed ncu capture of this workload, if any."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        return json.load(open(p)).get(workload)
    return None


# ------------------------------------------------------------------------- reference (CPU) arm

def cpu_reference(xyz, tri, f, b, d, q, scheme, budget_s=12.0, reps=3):
    """Times the UNMODIFIED reference (oracle/_ref) on a bounded prefix of the same workload with
    all host threads. Returns (crossings/s, geodesics/s, sample description, threads, ms)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import refapi
    if not refapi.available():
        raise RuntimeError("oracle/_ref/libdigeo_ref.so missing")
    rm = refapi.RefMesh.build(xyz, tri)
    # all host threads this process may run on, passed explicitly: torchrun exports OMP_NUM_THREADS=1, which the
    # reference's workers <= 0 default (tracer.cpp:547-555) would follow
    try:
        threads = len(os.sched_getaffinity(0))
    except AttributeError:
        threads = os.cpu_count() or 1
    threads = refapi.resolve_workers(threads)

    def run(k):
        t0 = time.perf_counter()
        r = rm.trace_batch(f[:k], b[:k], d[:k], workers=threads)
        if scheme == "ep":   # ep_jacobians + pullback_ambient per sample, the reference's serial loop
            rm.ep(f[:k], b[:k], d[:k], r.face, r.bary, r.dir, g=q[:k])
        else:
            rm.gfd(f[:k], b[:k], d[:k], g=q[:k], workers=threads)
        return time.perf_counter() - t0

    k = min(len(f), 2000)
    t = run(k)
    k = int(min(len(f), max(k, k * (budget_s / reps) / max(t, 1e-3))))
    times = [run(k) for _ in range(reps)]
    best = float(np.median(times))
    # crossings of the sample, counted from the reference's own polylines
    cnt = rm.trace_batch(f[:k], b[:k], d[:k], record_polyline=True, workers=threads)
    crossings = int((cnt.npoints - 2).clip(min=0).sum())
    return crossings / best, k / best, f"first {k} of {len(f)} geodesics, median of {reps}", threads, best * 1e3, crossings, k


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = WORKLOADS[args.workload]
    n = args.geodesics or wl["n"]
    xyz, tri, f, b, d, q = make_workload(args.workload, min(n, 200_000), args.seed)
    vals, ms = [], []
    threads = sample = None
    for it in range(args.warmup + args.steps):
        cps, gps, sample, threads, t_ms, _, k = cpu_reference(xyz, tri, f, b, d, q, wl["scheme"],
                                                              budget_s=max(2.0, 60.0 / (args.warmup + args.steps)), reps=1)
        if it >= args.warmup:
            vals.append(cps)
            ms.append(t_ms)
    v = float(np.median(vals))
    line = {"impl": "reference", "metric": f"face_crossings_per_s_fwd_{wl['scheme']}", "value": v,
            "unit": "face-crossings/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(np.median(ms)), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl["name"], "geodesics_per_step": k, "note": "reference CPU path (unmodified "
                       "sources compiled into oracle/_ref), OpenMP over all host threads, bounded prefix per step"},
            "cpu_baseline": {"value": v, "unit": "face-crossings/s", "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": v, "unit": "face-crossings/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line))


# ------------------------------------------------------------------------------- GPU arm

def run_ours(args):
    import torch
    import paper_2603_15780_b200 as dg

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.share_gpu:   # functional test of the N>1 path on a 1-GPU box (ranks share device 0)
        local = 0
    if dg.device_count() == 0:
        raise SystemExit("bench.py: no CUDA device (there is no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)

    wl = WORKLOADS[args.workload]
    scheme = wl["scheme"]
    n = args.geodesics or wl["n"]   # per GPU: weak scaling, the query batch is sharded, the mesh replicated
    xyz, tri, f, b, d, q = make_workload(args.workload, n, args.seed + rank)
    mesh = dg.Mesh(xyz, tri, device=local)
    eps = mesh.default_gfd_eps()

    # ---- device-resident inputs / outputs (the timed `value` region starts with these in HBM)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
    F, B, D, Q = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64), t(q, torch.float64)
    o = dict(face=torch.empty(n, dtype=torch.int32, device=dev), bary=torch.empty(n, 3, dtype=torch.float64, device=dev),
             dir=torch.empty(n, 3, dtype=torch.float64, device=dev), traced=torch.empty(n, dtype=torch.float64, device=dev),
             term=torch.empty(n, dtype=torch.uint8, device=dev), status=torch.empty(n, dtype=torch.uint8, device=dev),
             total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
    G = torch.empty(n, 3, dtype=torch.float64, device=dev)
    grad_v = torch.empty(n, 3, dtype=torch.float64, device=dev)
    grad_p = torch.empty(n, 3, dtype=torch.float64, device=dev)
    jv = torch.empty(n, 4, dtype=torch.float64, device=dev)
    jp = torch.empty(n, 4, dtype=torch.float64, device=dev)
    gathered = None
    if world > 1:
        pack = torch.empty(n, 7, dtype=torch.float64, device=dev)
        gathered = torch.empty(world * n, 7, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    G.copy_(Q)   # upstream gradient dL/dy: a fixed synthetic unit vector per sample (input of the backward)

    ev = lambda: torch.cuda.Event(enable_timing=True)
    trace_ms = []

    def step(timed):
        """forward + backward with everything resident in HBM; returns the number of our kernels launched."""
        e0, e1 = ev(), ev()
        if scheme == "ep":
            e0.record()
            mesh.trace_batch_device(F, B, D, o)
            e1.record()
            mesh.ep_backward_device(F, D, o["face"], o["dir"], G, grad_v, grad_p)
            launches = 2
        else:
            e0.record()
            mesh.trace_batch_device(F, B, D, o)
            e1.record()
            # the forward results are GFD's base traces (the `trace` argument of gfd_batched, diff.hpp:73)
            mesh.gfd_device(F, B, D, eps, eps, G, jv, jp, grad_v, grad_p, base=o)
            launches = 1 + 2 + 3  # forward walker + round 1 (job builder, payload walker on the seeds)
            #                       + round 2 (job builder, walker on the sibling groups, assemble); DESIGN.md 3.3
        if world > 1:   # results gathered over NVLink; no reduction on this path
            pack[:, 0] = o["face"].double(); pack[:, 1:4] = o["bary"]; pack[:, 4:7] = o["dir"]
            dist.all_gather_into_tensor(gathered, pack)
        if timed:
            trace_ms.append((e0, e1))
        return launches

    def sync_all():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step(False)
    sync_all()
    crossings_per_step = int(o["total_crossings"].item())

    launches = 0
    marks = []
    with ClockSampler(local) as clocks:
        sync_all()
        for _ in range(args.steps):
            flush.fill_(1)          # evict L2 between timed iterations (not timed)
            s, e = ev(), ev()
            s.record()
            launches += step(True)
            e.record()
            marks.append((s, e))
        sync_all()
    step_ms = [s.elapsed_time(e) for s, e in marks]
    total_ms = float(sum(step_ms))
    tr_ms = [s.elapsed_time(e) for s, e in trace_ms]

    # max over ranks, whole-job aggregate
    tot = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    cr = torch.tensor([float(crossings_per_step)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        dist.all_reduce(cr, op=dist.ReduceOp.SUM)
    total_ms_max = float(tot.item())
    crossings_all = float(cr.item())
    ms_per_step = total_ms_max / args.steps
    value = crossings_all / (ms_per_step * 1e-3)
    geodesics_per_s = world * n / (ms_per_step * 1e-3)

    # ---- e2e: the same step through the host-facing API with pinned HOST buffers
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    hf, hb, hd, hq = pin(f), pin(b), pin(d), pin(q)

    pinned_empty = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory().numpy()
    res = dg.TraceResult(face=pinned_empty(n, torch.int32), bary=pinned_empty((n, 3), torch.float64),
                         dir=pinned_empty((n, 3), torch.float64), traced=pinned_empty(n, torch.float64),
                         requested=pinned_empty(n, torch.float64), term=pinned_empty(n, torch.uint8),
                         status=pinned_empty(n, torch.uint8), stall=pinned_empty(n, torch.uint8),
                         npoints=pinned_empty(n, torch.int32), crossings=pinned_empty(n, torch.int32))
    hg, hgv = hq, pinned_empty((n, 3), torch.float64)   # hg: the synthetic upstream gradient

    gfd_out = dict(jv=pinned_empty((n, 4), torch.float64), jp=pinned_empty((n, 4), torch.float64),
                   degraded=pinned_empty((n, 4), torch.uint8), grad_v=hgv, grad_p=pinned_empty((n, 3), torch.float64))

    # the host-facing call of a training step: a resident batch (dg_batch_*), i.e. the forward inputs and
    # results stay on the GPU between the forward and the backward call; every step still copies its
    # inputs host -> device and every result device -> host
    batch = dg.Batch(mesh, n)
    gfd_keys = dict(jv=gfd_out["jv"], jp=gfd_out["jp"], degraded=gfd_out["degraded"], grad_v=hgv, grad_p=gfd_out["grad_p"])

    def e2e_step():
        r = batch.trace(hf, hb, hd, out=res)
        if scheme == "ep":
            out = batch.ep_backward(hg, grad_v=hgv)
        else:
            out = batch.gfd(g=hg, out=gfd_keys)
        return r, out

    e2e_reps = max(1, min(args.steps, 3))
    e2e_step()
    sync_all()
    t0 = time.perf_counter()
    for _ in range(e2e_reps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([(time.perf_counter() - t0) * 1e3 / e2e_reps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = crossings_all / (float(e2e_ms.item()) * 1e-3)
    fwd_in, fwd_out = n * (4 + 24 + 24), n * (4 + 24 + 24 + 8 + 8 + 1 + 1 + 1 + 4 + 4)
    if scheme == "ep":
        h2d, d2h = fwd_in + n * 24, fwd_out + n * 24                       # + g in, grad_v out
    else:
        h2d, d2h = fwd_in + n * 24, fwd_out + n * (32 + 32 + 4 + 24 + 24)  # + g in; jv, jp, degraded, grad_v, grad_p out

    line = None
    if rank == 0:
        peak, peak_src = measured_peak()
        t_trace = float(np.mean(tr_ms)) * 1e-3
        alg_bytes = crossings_per_step * BYTES_PER_CROSSING + n * BYTES_PER_GEODESIC
        achieved = alg_bytes / t_trace / 1e9
        traffic = profile_traffic(args.workload)
        info = dg.kernel_info(False, False, cached=mesh.has_transport_cache, tma=mesh.gather == "tma", coop=mesh.gather == "coop")
        line = {"metric": f"face_crossings_per_s_fwd_{scheme}", "value": value, "unit": "face-crossings/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": wl["name"], "geodesics_per_gpu": n, "faces": int(len(tri)),
                           "crossings_per_geodesic": crossings_per_step / n, "l2": "256 MB flush between timed steps",
                           "parallelism": f"query-sharded x{world}, mesh replicated"},
                "geodesics_per_s": geodesics_per_s,
                "forward_only": {"ms": float(np.mean(tr_ms)), "face_crossings_per_s": crossings_per_step / t_trace,
                                 "geodesics_per_s": n / t_trace},
                # rank 0's own step minus its forward trace; GFD re-traces every sample three times at full length
                # (sibling groups), so its rate counts 3 x the forward crossings
                "backward_only": {"scheme": scheme, "ms": float(np.mean(step_ms) - np.mean(tr_ms)),
                                  "retraced_face_crossings_per_s": (3 * crossings_per_step / ((np.mean(step_ms) - np.mean(tr_ms)) * 1e-3)
                                                                    if scheme == "gfd" else None)},
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                             "traffic": traffic["dram_bytes_per_launch"] if traffic else None,
                             "kernel": ("trace_fast_kernel<crossing records, TMA tile::gather4>" if mesh.gather == "tma" else
                                        "trace_fast_kernel<crossing records, cooperative 256-bit loads>" if mesh.gather == "coop" else
                                        "trace_fast_kernel<crossing records, 256-bit loads>" if mesh.has_transport_cache else
                                        "trace_fast_kernel<face records>"),
                             "peak_source": peak_src,
                             "algorithmic_bytes_per_launch": alg_bytes,
                             "note": "dependent-gather walk: bound by FP64 issue + L2 latency, not HBM bandwidth (DESIGN.md)",
                             "registers": info["registers"], "blocks_per_sm": info["blocks_per_sm"],
                             # the access pattern's own ceiling: random 128-byte records, one per lane per round, dependent
                             # next index, measured with scripts/micro/gather_bench.cu at this record-array size with the
                             # gather this mesh uses (profiles/tuning_r1.md); one record = one face crossing
                             "gather": gather_roofline(mesh, crossings_per_step / t_trace)},
                "e2e": {"value": e2e_value, "unit": "face-crossings/s", "h2d_bytes_per_step": int(h2d),
                        "d2h_bytes_per_step": int(d2h), "ms_per_step": float(e2e_ms.item())},
                "gpu_launches": launches, "clocks": clocks.summary()}
        if scheme == "gfd":
            # the kernel that takes most of a GFD step: round 2, three full-length re-traces per sample as sibling
            # groups (+ n eps-length jobs). Its duration is rank 0's backward time (job builders, seeds and assembly
            # are < 2 % of it, profiles/r1_launches_bench_c3_summary.txt); algorithmic bytes as for the forward walk.
            t_bwd = (float(np.mean(step_ms)) - float(np.mean(tr_ms))) * 1e-3
            alg2 = 3 * crossings_per_step * BYTES_PER_CROSSING + 4 * n * BYTES_PER_GEODESIC
            tr2 = profile_traffic(args.workload + "_gfd_round2")
            info2 = dg.kernel_info(False, False, cached=mesh.has_transport_cache, dense=True)
            line["roofline_gfd_round2"] = {"bound": "hbm", "achieved": alg2 / t_bwd / 1e9, "peak": peak, "unit": "GB/s",
                                           "frac": alg2 / t_bwd / 1e9 / peak,
                                           "traffic": tr2["dram_bytes_per_launch"] if tr2 else None,
                                           "kernel": "trace_fast_kernel<crossing records, 256-bit loads, sibling groups of 3>",
                                           "algorithmic_bytes_per_launch": alg2, "registers": info2["registers"],
                                           "blocks_per_sm": info2["blocks_per_sm"]}
        if not args.no_cpu and world == 1:
            try:
                cps, gps, sample, threads, _, _, _ = cpu_reference(xyz, tri, f, b, d, q, scheme)
                line["cpu_baseline"] = {"value": cps, "unit": "face-crossings/s", "cores": threads, "kind": "reference",
                                        "sample": sample, "geodesics_per_s": gps}
            except Exception as ex:  # the checker is optional for the GPU arm
                line["cpu_baseline"] = {"value": None, "unit": "face-crossings/s", "cores": 0, "kind": "reference",
                                        "sample": f"unavailable: {ex}"}
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--geodesics", type=int, default=0, help="geodesics per GPU (default: the workload's)")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--dist-backend", default="nccl", help="torch.distributed backend for N>1 (nccl on the GPU box)")
    ap.add_argument("--share-gpu", action="store_true", help="testing only: all ranks use cuda:0 (with --dist-backend gloo)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
