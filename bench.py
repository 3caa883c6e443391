#!/usr/bin/env python
"""Benchmark of the batched straightest-geodesic exponential map and its EP / GFD backward (BASELINE.json).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c2|c3|c4|c5]
                  [--blocks c3,c4,c5|none]

One "step" = one pass of the hot path over the whole query batch: forward trace of every geodesic + the
scheme's backward (EP for config 2, GFD for config 3, none for configs 4 and 5). The HEADLINE workload is
config 2 (bumpy sphere, icosphere-6 displaced radially, 81 920 faces; 1 M geodesics per GPU of length
0.5 x bbox diagonal; forward + EP). The same JSON line carries one block per further configuration of
BASELINE.json under "blocks" -- c3 (1 M-face noisy torus, 10 M geodesics in all, forward + GFD, the SAME batch
sharded over the N GPUs: strong scaling), c4 (64 concatenated meshes, 65 536 queries each, mixed lengths) and
c5 (1 M-face torus, length 5 x diameter, half vertex-to-vertex walks, 2.5 M geodesics per GPU) -- each with its
own value, roofline, e2e and cpu_baseline. With --gpus N > 1 and no torchrun environment the script starts
its N ranks itself (torch.distributed.run, one process per GPU). Prints ONE JSON line.
"""
import argparse
import importlib.util
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_CROSSING = 48     # 3 vertex ids + 3 neighbour ids + one new f64 position
BYTES_PER_GEODESIC = 116    # 52 B query in + 64 B result out

WORKLOADS = {
    "c2": dict(name="bumpy-sphere ico-6 (81,920 faces), 1M geodesics, length 0.5 x bbox diagonal, forward + EP backward",
               scheme="ep", n=1_000_000, scaling="weak", max_steps=0),
    "c3": dict(name="noisy torus 1000x500 (1,000,000 faces), 10M geodesics of length 0.5 x bbox diagonal, forward + GFD backward",
               scheme="gfd", n=10_000_000, scaling="strong", max_steps=0),
    "c4": dict(name="64 meshes of 10k-200k faces concatenated (6.8M faces), 65,536 queries per mesh, lengths log-uniform in "
                    "[0.01, 2] x bbox diagonal, forward", scheme="fwd", n=64 * 65536, scaling="strong", max_steps=0),
    # (config 5 is 100 M queries on 8 GPUs = 12.5 M per GPU; a bench step runs a fifth of one GPU's share -- 2.5 M
    # geodesics, 1.5e10 face crossings, two seconds of walker -- so that the default run stays within minutes)
    "c5": dict(name="torus 1000x500 (1,000,000 faces), 2.5M geodesics per GPU of length 5 x outer diameter, half exactly at "
                    "vertices along a meridian edge (vertex-to-vertex walks), max_steps 200000, forward",
               scheme="fwd", n=2_500_000, scaling="weak", max_steps=200_000),
}


def workloads_module():
    """paper_2603_15780_b200/workloads.py loaded BY PATH: pure numpy generators, usable by the reference arm
    without importing the package (whose __init__ maps libdigeo_b200.so)."""
    spec = importlib.util.spec_from_file_location("dg_workloads", os.path.join(ROOT, "paper_2603_15780_b200", "workloads.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def shard_bounds(weights, world):
    spec = importlib.util.spec_from_file_location("dg_sharding", os.path.join(ROOT, "paper_2603_15780_b200", "sharding.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.shard_bounds(weights, world)


def make_workload(key, n, seed):
    """The synthetic mesh and n queries of configuration `key`. Returns xyz, tri, face, bary, dir, q
    (q: unit vectors, the targets of the loss whose gradient is the backward's upstream input)."""
    W = workloads_module()
    if key == "c2":
        xyz, tri = W.bumpy_sphere(6)
    elif key in ("c3",):
        xyz, tri = W.torus(1 / 3, 1 / 6, 1000, 500, noise=0.1, seed=7)
    if key in ("c2", "c3"):
        f, b, d = W.sample_queries(xyz, tri, n, 0.5 * W.bbox_diagonal(xyz), seed=seed)
    elif key == "c4":
        xyz, tri, f, b, d, _ = W.config4(queries_per_mesh=max(1, n // 64), seed=4)
    elif key == "c5":
        xyz, tri, f, b, d = W.config5(n, seed=seed)
    else:
        raise KeyError(key)
    rng = np.random.default_rng(seed + 1)
    q = rng.normal(size=(len(f), 3))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return xyz, tri, f, b, d, q


def config_of(key, n_per_step, faces, world):
    wl = WORKLOADS[key]
    return {"workload": wl["name"], "geodesics_per_step": int(n_per_step), "faces": int(faces),
            "l2": "256 MB flush between timed steps", "parallelism": f"query-sharded x{world}, mesh replicated",
            "max_steps": wl["max_steps"] or "default 10*sqrt(F)+100"}


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


def gather_peak(mesh, device_index):
    """The access pattern's own ceiling, MEASURED IN THIS RUN (outside the timed region): scripts/micro/gather_bench --
    random 128-byte records, one per lane per round, dependent next index -- at this mesh's record-array size, the
    best of the three gathers the walker has (per-lane 256-bit loads, TMA, cooperative loads). G records/s; one
    record = one face crossing. Returns (peak, {variant: rate})."""
    exe = os.path.join(ROOT, "scripts", "micro", "gather_bench")
    if not mesh.has_transport_cache or not os.path.exists(exe):
        return None, None
    env = dict(os.environ)
    vis = [v for v in env.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
    env["CUDA_VISIBLE_DEVICES"] = vis[device_index] if device_index < len(vis) else str(device_index)
    rates = {}
    for name, variant in (("loads", 0), ("tma", 1), ("coop", 2)):
        try:
            out = subprocess.run([exe, str(3 * mesh.nf), "1000", str(variant)], env=env, capture_output=True, text=True, timeout=120)
            rates[name] = float(json.loads(out.stdout.strip().splitlines()[-1])["grecords_per_s"])
        except Exception:
            pass
    return (max(rates.values()), rates) if rates else (None, None)


def profile_traffic(key, n):
    """dram bytes per launch of the trace kernel, FROM THE COMMITTED ncu CAPTURE of this workload at this batch size
    (profiles/traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        t = json.load(open(p)).get(key)
        if t and int(t.get("geodesics", -1)) == int(n):
            return t
    return None


# ------------------------------------------------------------------------- reference (CPU) arm

def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


class CpuReference:
    """The UNMODIFIED reference (oracle/_ref) on the box's host cores, all threads: trace_batch, then the scheme's
    backward (the serial ep_jacobians + pullback_ambient loop of gradcheck.cpp:76-89, or gfd_batched_many)."""

    def __init__(self, xyz, tri, scheme, max_steps):
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import refapi
        if not refapi.available():
            raise RuntimeError("oracle/_ref/libdigeo_ref.so missing")
        self.rm = refapi.RefMesh.build(xyz, tri)
        # passed explicitly: torchrun exports OMP_NUM_THREADS=1, which the reference's workers <= 0 default
        # (tracer.cpp:547-555) would follow
        self.threads = refapi.resolve_workers(host_threads())
        self.scheme, self.max_steps = scheme, max_steps

    def run(self, f, b, d, q):
        t0 = time.perf_counter()
        r = self.rm.trace_batch(f, b, d, workers=self.threads, max_steps=self.max_steps)
        if self.scheme == "ep":
            self.rm.ep(f, b, d, r.face, r.bary, r.dir, g=q)
        elif self.scheme == "gfd":
            self.rm.gfd(f, b, d, g=q, workers=self.threads)
        return time.perf_counter() - t0

    def crossings(self, f, b, d):
        """face crossings of these queries counted from the reference's own polylines: one point per
        advance + the start point (exact on traces without vertex points)."""
        cnt = self.rm.trace_batch(f, b, d, record_polyline=True, workers=self.threads, max_steps=self.max_steps)
        return int((cnt.npoints - 2).clip(min=0).sum())


def cpu_baseline(xyz, tri, f, b, d, q, scheme, max_steps, budget_s, reps, counts=None):
    """Bounded prefix of the workload sized to ~budget_s of host time. counts: per-geodesic crossing counts of the
    same queries from the GPU run (the unit both sides are quoted in); else counted from the reference's polylines."""
    ref = CpuReference(xyz, tri, scheme, max_steps)
    k = min(len(f), 2000 if scheme != "fwd" or max_steps == 0 else 200)
    t = ref.run(f[:k], b[:k], d[:k], q[:k])
    k = int(min(len(f), max(k, k * (budget_s / reps) / max(t, 1e-3))))
    times = [ref.run(f[:k], b[:k], d[:k], q[:k]) for _ in range(reps)]
    best = float(np.median(times))
    crossings = int(np.asarray(counts[:k], dtype=np.int64).sum()) if counts is not None else ref.crossings(f[:k], b[:k], d[:k])
    return {"value": crossings / best, "unit": "face-crossings/s", "cores": ref.threads, "kind": "reference",
            "sample": f"first {k} of {len(f)} geodesics, median of {reps}", "geodesics_per_s": k / best,
            "ms": best * 1e3, "geodesics": k}


def run_reference_arm(args):
    """bench.py --impl reference: the reference's own CPU implementation of the path, all host threads, on the
    headline workload. Imports nothing from the product package."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    key = args.workload
    wl = WORKLOADS[key]
    n = args.geodesics or wl["n"]
    xyz, tri, f, b, d, q = make_workload(key, n, args.seed)
    ref = CpuReference(xyz, tri, wl["scheme"], wl["max_steps"])
    # every step runs the same bounded prefix: the whole batch when (K + W) steps of it fit ~150 s of host time
    probe = min(len(f), 2000)
    t = ref.run(f[:probe], b[:probe], d[:probe], q[:probe])
    per_step = 150.0 / (args.warmup + args.steps)
    k = int(min(len(f), max(probe, probe * per_step / max(t, 1e-3))))
    ms = []
    for it in range(args.warmup + args.steps):
        t = ref.run(f[:k], b[:k], d[:k], q[:k])
        if it >= args.warmup:
            ms.append(t * 1e3)
    crossings = ref.crossings(f[:k], b[:k], d[:k])
    t_ms = float(np.median(ms))
    v = crossings / (t_ms * 1e-3)
    cfg = config_of(key, n, len(tri), 1)
    line = {"impl": "reference", "metric": f"face_crossings_per_s_fwd_{wl['scheme']}", "value": v,
            "unit": "face-crossings/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_ms, "higher_is_better": True, "scaling": wl["scaling"], "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": cfg, "geodesics_per_s": k / (t_ms * 1e-3),
            "crossings_per_geodesic": crossings / k, "reference_sample": f"first {k} of {n} geodesics per step",
            "cpu_baseline": {"value": v, "unit": "face-crossings/s", "cores": ref.threads, "kind": "reference",
                             "sample": f"first {k} of {n} geodesics, median of {args.steps} steps",
                             "note": "unmodified reference sources compiled into oracle/_ref, OpenMP over all host threads"},
            "e2e": {"value": v, "unit": "face-crossings/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line))


# ------------------------------------------------------------------------------- GPU arm

class ResultBlock:
    """The SoA result columns of this rank's shard inside ONE contiguous device block: the kernels write straight
    into the columns, so gathering the results of all ranks is one all_gather of the block (no packing kernels).
    Layout of the gathered buffer: rank-major, each rank's block = its columns back to back, rows padded to the
    largest shard (a multiple of 8)."""

    def __init__(self, rows, rows_pad, cols, dev):
        import torch
        cols = sorted(cols, key=lambda c: -torch.empty(0, dtype=c[1]).element_size())
        self.nbytes = sum(rows_pad * w * torch.empty(0, dtype=dt).element_size() for _, dt, w in cols)
        self.buf = torch.zeros(self.nbytes, dtype=torch.uint8, device=dev)
        self.col, off = {}, 0
        for name, dt, w in cols:
            nb = rows_pad * w * torch.empty(0, dtype=dt).element_size()
            v = self.buf[off:off + nb].view(dt)[:rows * w]
            self.col[name] = v.view(rows, w) if w > 1 else v
            off += nb


def measure(key, args, ctx, headline):
    """Runs configuration `key` on this rank's shard; rank 0 returns the result dict (others None)."""
    import torch
    import paper_2603_15780_b200 as dg
    from paper_2603_15780_b200 import sharding

    rank, world, local, dev, dist = ctx["rank"], ctx["world"], ctx["local"], ctx["dev"], ctx["dist"]
    wl = WORKLOADS[key]
    scheme, max_steps = wl["scheme"], wl["max_steps"]
    base_n = (args.geodesics if (headline and args.geodesics) else wl["n"])
    if args.block_geodesics and not headline:
        base_n = min(base_n, args.block_geodesics)
    steps = args.steps if headline else max(1, min(args.steps, 3))
    warmup = args.warmup if headline else max(3, min(args.warmup, 3))

    # ---- the global batch and this rank's shard (cut by expected work: sharding.shard_bounds)
    if wl["scaling"] == "strong" or key == "c2":
        n_global = base_n if wl["scaling"] == "strong" else base_n * world
        xyz, tri, f, b, d, q = make_workload(key, n_global, args.seed)
        n_global = len(f)
        bounds = sharding.shard_bounds(np.linalg.norm(d, axis=1), world)
        sl = slice(int(bounds[rank]), int(bounds[rank + 1]))
        f, b, d, q = f[sl], b[sl], d[sl], q[sl]
    else:   # weak, per-rank query streams (config 5: 100 M queries on 8 GPUs are never materialised in one place)
        xyz, tri, f, b, d, q = make_workload(key, base_n, args.seed + 1000 * rank)
        n_global = base_n * world
        bounds = np.arange(world + 1, dtype=np.int64) * base_n
    n = len(f)
    rows_pad = int((np.diff(bounds).max() + 7) // 8 * 8)
    mesh = dg.Mesh(xyz, tri, device=local)
    eps = mesh.default_gfd_eps()

    # ---- device-resident inputs / outputs (the timed `value` region starts with these in HBM)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
    F, B, D, G = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64), t(q, torch.float64)
    f64, cols = torch.float64, [("face", torch.int32, 1), ("bary", torch.float64, 3), ("dir", torch.float64, 3),
                                ("traced", torch.float64, 1), ("term", torch.uint8, 1), ("status", torch.uint8, 1)]
    if scheme == "ep":
        cols += [("grad_v", f64, 3), ("grad_p", f64, 3)]
    elif scheme == "gfd":
        cols += [("grad_v", f64, 3), ("grad_p", f64, 3), ("jv", f64, 4), ("jp", f64, 4)]
    blk = ResultBlock(n, rows_pad, cols, dev)
    o = {k: blk.col[k] for k in ("face", "bary", "dir", "traced", "term", "status")}
    o["total_crossings"] = torch.zeros(1, dtype=torch.int64, device=dev)
    o["crossings"] = torch.empty(n, dtype=torch.int32, device=dev)
    gathered = torch.empty(world * blk.nbytes, dtype=torch.uint8, device=dev) if world > 1 else None
    flush = ctx["flush"]

    ev = lambda: torch.cuda.Event(enable_timing=True)
    trace_ms = []

    def step(timed, fused=True):
        """forward + backward with everything resident in HBM; returns the number of our kernels launched."""
        e0, e1 = ev(), ev()
        if scheme == "gfd" and fused:
            # the forward of a GFD step IS GFD's base trace (diff.cpp:288-294): it rides in round 2 as the fourth
            # sibling of the sample's re-traces (dg_trace_gfd); the backward is the pull-back of g (dg_gfd_pullback)
            e0.record()
            mesh.trace_gfd_device(F, B, D, o, eps, eps, blk.col["jv"], blk.col["jp"])
            e1.record()
            mesh.gfd_pullback_device(F, D, o["face"], blk.col["jv"], blk.col["jp"], G, blk.col["grad_v"], blk.col["grad_p"])
            launches = 2 + 2 + 3 + 1   # round 1 (job builder, seeds walker), round 2 (job builder, 4-sibling walker),
            #                            par jobs (builder, walker), assemble; pull-back
            if face_order:
                launches += 1          # the key pass of the sample order (the radix sort itself is cub's)
            if world > 1:
                gather()
            if timed:
                trace_ms.append((e0, e1))
            return launches
        e0.record()
        mesh.trace_batch_device(F, B, D, o, max_steps=max_steps)
        e1.record()
        launches = 1
        if face_order:                 # the key pass of the start-face order (the radix sort itself is cub's) and, on a
            launches += 2 if mesh.gather == "coop" else 1   # mesh beyond 250 MB, the second launch of the gated pair
        if scheme == "ep":
            mesh.ep_backward_device(F, D, o["face"], o["dir"], G, blk.col["grad_v"], blk.col["grad_p"])
            launches += 1
        elif scheme == "gfd":
            # the forward results are GFD's base traces (the `trace` argument of gfd_batched, diff.hpp:73)
            mesh.gfd_device(F, B, D, eps, eps, G, blk.col["jv"], blk.col["jp"], blk.col["grad_v"], blk.col["grad_p"], base=o)
            launches += 2 + 3   # round 1 (job builder, payload walker on the seeds) + round 2 (job builder, walker on
            #                     the sibling groups, assemble); DESIGN.md 3.3
        if world > 1:
            gather()
        if timed:
            trace_ms.append((e0, e1))
        return launches

    def gather():   # results of all shards gathered over NVLink: one collective of the SoA block, no reduction
        if ctx["backend"] == "nccl":
            dist.all_gather_into_tensor(gathered, blk.buf)
        else:       # functional test of the N>1 path on CPU-side collectives (gloo)
            parts = [torch.empty(blk.nbytes, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(parts, blk.buf.cpu())
            gathered.copy_(torch.cat(parts))

    def sync_all():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    face_order, gather_kind = mesh.trace_plan(n)   # how this launch is scheduled and how it fetches its records
    peak_g, gather_rates = gather_peak(mesh, local) if rank == 0 else (None, None)   # micro-benchmark, before the timed region
    for _ in range(warmup):
        step(False)
    sync_all()
    crossings_local = int(o["total_crossings"].item())

    launches, marks = 0, []
    with ClockSampler(local) as clocks:
        sync_all()
        for _ in range(steps):
            flush.fill_(1)          # evict L2 between timed iterations (not timed)
            s, e = ev(), ev()
            s.record()
            launches += step(True)
            e.record()
            marks.append((s, e))
        sync_all()
    step_ms = [s.elapsed_time(e) for s, e in marks]
    tr_ms = [s.elapsed_time(e) for s, e in trace_ms]
    def timed_device(fn, reps):
        fn()
        sync_all()
        ms = []
        for _ in range(reps):
            flush.fill_(1)
            s, e = ev(), ev()
            s.record(); fn(); e.record()
            ms.append((s, e))
        sync_all()
        return float(np.mean([s.elapsed_time(e) for s, e in ms]))

    # the opt-in tolerance lane (DG_LANE_FAST) on the same step: reported beside the exact lane, never instead of it
    lane_fast = None
    if mesh.has_transport_cache:
        lf_fwd = timed_device(lambda: mesh.trace_batch_device(F, B, D, o, max_steps=max_steps, lane="fast"), steps)
        lf_step = lf_fwd
        if scheme == "ep":
            lf_step = timed_device(lambda: (mesh.trace_batch_device(F, B, D, o, max_steps=max_steps, lane="fast"),
                                            mesh.ep_backward_device(F, D, o["face"], o["dir"], G, blk.col["grad_v"], blk.col["grad_p"])), steps)
        elif scheme == "gfd":
            lf_step = timed_device(lambda: (mesh.trace_gfd_device(F, B, D, o, eps, eps, blk.col["jv"], blk.col["jp"], lane="fast"),
                                            mesh.gfd_pullback_device(F, D, o["face"], blk.col["jv"], blk.col["jp"], G, blk.col["grad_v"],
                                                                     blk.col["grad_p"])), steps)
        lane_fast = {"forward_ms": lf_fwd, "step_ms": lf_step}
    separate = None
    if scheme == "gfd":
        # for comparison: the same step as two separate calls -- a lone forward launch, then GFD with the forward
        # results as known base (three sibling re-traces per sample)
        trace_ms.clear()
        sep_marks = []
        step(False, fused=False)
        sync_all()
        for _ in range(steps):
            flush.fill_(1)
            s, e = ev(), ev()
            s.record()
            step(True, fused=False)
            e.record()
            sep_marks.append((s, e))
        sync_all()
        separate = {"ms_per_step": float(np.mean([s.elapsed_time(e) for s, e in sep_marks])),
                    "forward_ms": float(np.mean([s.elapsed_time(e) for s, e in trace_ms]))}

    def over_ranks(x, op):
        v = torch.tensor([float(x)], dtype=torch.float64, device=dev)
        if world > 1:
            if ctx["backend"] == "nccl":
                dist.all_reduce(v, op=op)
            else:
                c = v.cpu(); dist.all_reduce(c, op=op); v = c
        return float(v.item())

    RO = torch.distributed.ReduceOp
    ms_per_step = over_ranks(sum(step_ms), RO.MAX) / steps           # max over ranks
    crossings_all = over_ranks(crossings_local, RO.SUM)              # whole-job aggregate
    value = crossings_all / (ms_per_step * 1e-3)

    # ---- e2e: the same step through the host-facing API with pinned HOST buffers (every step copies its inputs
    # host -> device and every result device -> host inside the timed region)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    pe = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory().numpy()
    hf, hb, hd, hg = pin(f), pin(b), pin(d), pin(q)
    res = dg.TraceResult(face=pe(n, torch.int32), bary=pe((n, 3), f64), dir=pe((n, 3), f64), traced=pe(n, f64),
                         requested=pe(n, f64), term=pe(n, torch.uint8), status=pe(n, torch.uint8), stall=pe(n, torch.uint8),
                         npoints=pe(n, torch.int32), crossings=pe(n, torch.int32))
    hgv = pe((n, 3), f64) if scheme != "fwd" else None
    gfd_keys = dict(jv=pe((n, 4), f64), jp=pe((n, 4), f64), degraded=pe((n, 4), torch.uint8), grad_v=hgv,
                    grad_p=pe((n, 3), f64)) if scheme == "gfd" else None
    batch = dg.Batch(mesh, n)

    def e2e_step():
        batch.trace(hf, hb, hd, out=res, max_steps=max_steps, gfd=(scheme == "gfd"))
        if scheme == "ep":
            batch.ep_backward(hg, grad_v=hgv)
        elif scheme == "gfd":
            batch.gfd(g=hg, out=gfd_keys)

    def timed_host(fn, reps):
        fn()
        sync_all()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return over_ranks((time.perf_counter() - t0) * 1e3 / reps, RO.MAX)

    e2e_ms = timed_host(e2e_step, max(1, min(steps, 3)))
    fwd_in, fwd_out = n * (4 + 24 + 24), n * (4 + 24 + 24 + 8 + 8 + 1 + 1 + 1 + 4 + 4)
    bwd_in = n * 24 if scheme != "fwd" else 0
    bwd_out = {"fwd": 0, "ep": n * 24, "gfd": n * (32 + 32 + 4 + 24 + 24)}[scheme]
    # the columns a training step consumes (end point, direction, length, termination, status + the gradient
    # w.r.t. v); requested / stall / npoints / crossings and, for GFD, the Jacobians stay on the device
    lean = dg.TraceResult(face=res.face, bary=res.bary, dir=res.dir, traced=res.traced, requested=None, term=res.term,
                          status=res.status, stall=None, npoints=None, crossings=None)

    def e2e_lean():
        batch.trace(hf, hb, hd, out=lean, max_steps=max_steps, gfd=(scheme == "gfd"))
        if scheme == "ep":
            batch.ep_backward(hg, grad_v=hgv)
        elif scheme == "gfd":
            batch.gfd(g=hg, out=dict(grad_v=hgv, grad_p=gfd_keys["grad_p"]))

    lean_ms = timed_host(e2e_lean, max(1, min(steps, 3)))
    lean_out = n * (4 + 24 + 24 + 8 + 1 + 1) + {"fwd": 0, "ep": n * 24, "gfd": n * 48}[scheme]
    counts = o["crossings"].cpu().numpy() if rank == 0 else None
    batch.close()

    if rank != 0:
        return None
    peak, peak_src = measured_peak()
    t_trace = float(np.mean(tr_ms)) * 1e-3
    if scheme == "gfd":   # the lone forward launch, timed in the separate-call runs above
        t_trace = separate["forward_ms"] * 1e-3
        tr_ms = [separate["forward_ms"]]
    alg_bytes = crossings_local * BYTES_PER_CROSSING + n * BYTES_PER_GEODESIC
    achieved = alg_bytes / t_trace / 1e9
    traffic = profile_traffic(key, n)
    info = dg.kernel_info(False, False, cached=mesh.has_transport_cache, tma=gather_kind == "tma", coop=gather_kind == "coop")
    cps_fwd = crossings_local / t_trace
    gather = None
    if peak_g:
        if face_order and mesh.gather == "coop":
            # on meshes beyond 250 MB of records a batch in start-face order is queued on both gathers and the mean
            # requested length, summed on the device, decides which one runs
            gather_kind = "loads while the wavefront stays near the L2 (expected crossings x sqrt(F) < 1e6), else coop: decided on the device"
        gather = {"gather": gather_kind, "start_face_order": face_order, "record_bytes": 3 * mesh.nf * 128, "achieved_grecords_per_s": cps_fwd / 1e9,
                  "peak_grecords_per_s": peak_g, "frac": cps_fwd / 1e9 / peak_g, "random_gather_grecords_per_s": gather_rates,
                  "source": "scripts/micro/gather_bench run inside this bench before the timed region; peak = the best of its "
                            "three gathers on RANDOM records of this array size (a launch scheduled in start-face order gets "
                            "L2 hits between neighbouring traces that random records do not)"}
    bwd_ms = float(np.mean(step_ms) - np.mean(tr_ms)) if scheme != "gfd" else separate["ms_per_step"] - separate["forward_ms"]
    line = {"metric": f"face_crossings_per_s_fwd_{scheme}" if scheme != "fwd" else "face_crossings_per_s_fwd",
            "value": value, "unit": "face-crossings/s", "n_gpus": world, "steps": steps, "warmup": warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": wl["scaling"], "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": config_of(key, n_global, len(tri), world),
            "geodesics_per_s": n_global / (ms_per_step * 1e-3), "crossings_per_geodesic": crossings_all / n_global,
            "shard_geodesics_rank0": n,
            "forward_only": {"ms": float(np.mean(tr_ms)), "face_crossings_per_s": cps_fwd, "geodesics_per_s": n / t_trace},
            # rank 0's own step minus its forward trace; GFD re-traces every sample three times at full length
            # (sibling groups), so its rate counts 3 x the forward crossings
            "backward_only": {"scheme": scheme, "ms": bwd_ms,
                              "retraced_face_crossings_per_s": 3 * crossings_local / (bwd_ms * 1e-3) if scheme == "gfd" else None},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic["dram_bytes_per_launch"] if traffic else None,
                         "traffic_source": (traffic["source"] + " -- a committed ncu capture, not measured in this run") if traffic else None,
                         "kernel": ("trace_fast_kernel<crossing records, TMA tile::gather4>" if gather_kind == "tma" else
                                    "trace_fast_kernel<crossing records, cooperative 256-bit loads>" if gather_kind == "coop" else
                                    "trace_fast_kernel<crossing records, 256-bit loads>" if mesh.has_transport_cache else
                                    "trace_fast_kernel<face records>"),
                         "peak_source": peak_src, "algorithmic_bytes_per_launch": alg_bytes,
                         "note": "dependent-gather walk: bound by FP64 issue + L2 latency, not HBM bandwidth (DESIGN.md)",
                         "registers": info["registers"], "blocks_per_sm": info["blocks_per_sm"], "gather": gather},
            "e2e": {"value": crossings_all / (e2e_ms * 1e-3), "unit": "face-crossings/s",
                    "h2d_bytes_per_step": int(fwd_in + bwd_in), "d2h_bytes_per_step": int(fwd_out + bwd_out), "ms_per_step": e2e_ms,
                    "training_columns_only": {"value": crossings_all / (lean_ms * 1e-3), "ms_per_step": lean_ms,
                                              "d2h_bytes_per_step": int(lean_out),
                                              "note": "same call, NULL for the outputs a training step does not read"}},
            "gpu_launches": launches, "clocks": clocks.summary()}
    if scheme == "gfd":
        # the kernel that IS the fused step: round 2 with the forward traces as fourth sibling of every sample's three
        # re-traces (4n full-length jobs); timed as the whole dg_trace_gfd call (job builders, eps-length seeds / par
        # jobs and the assembly ride along: < 3 % of it), so the fraction is a lower bound for the kernel's own
        t_fused = float(np.mean(step_ms)) * 1e-3
        alg4 = 4 * crossings_local * BYTES_PER_CROSSING + 4 * n * BYTES_PER_GEODESIC
        info4 = dg.kernel_info(False, False, cached=mesh.has_transport_cache, dense=True)
        tr4 = profile_traffic(key + "_gfd_fused", n)
        line["fused_forward_gfd"] = {"ms": float(np.mean(step_ms)), "note": "dg_trace_gfd + dg_gfd_pullback: the step `value` is quoted on",
                                     "roofline": {"bound": "hbm", "achieved": alg4 / t_fused / 1e9, "peak": peak, "unit": "GB/s",
                                                  "frac": alg4 / t_fused / 1e9 / peak,
                                                  "traffic": tr4["dram_bytes_per_launch"] if tr4 else None,
                                                  "kernel": "trace_fast_kernel<crossing records, 256-bit loads, sibling groups of 4>",
                                                  "algorithmic_bytes_per_launch": alg4, "registers": info4["registers"],
                                                  "blocks_per_sm": info4["blocks_per_sm"]}}
        line["separate_calls"] = {"ms_per_step": separate["ms_per_step"], "forward_ms": separate["forward_ms"],
                                  "value": crossings_local / (separate["ms_per_step"] * 1e-3),
                                  "note": "rank 0, lone forward launch + GFD with the forward results as known base"}
    if scheme == "gfd":
        # the kernel that takes most of a GFD step: round 2, three full-length re-traces per sample as sibling groups
        # (+ n eps-length jobs). Its duration is rank 0's backward time (job builders, seeds and assembly are < 2 % of
        # it, profiles/); algorithmic bytes as for the forward walk.
        alg2 = 3 * crossings_local * BYTES_PER_CROSSING + 4 * n * BYTES_PER_GEODESIC
        tr2 = profile_traffic(key + "_gfd_round2", n)
        info2 = dg.kernel_info(False, False, cached=mesh.has_transport_cache, dense=True)
        line["roofline_gfd_round2"] = {"bound": "hbm", "achieved": alg2 / (bwd_ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                                       "frac": alg2 / (bwd_ms * 1e-3) / 1e9 / peak,
                                       "traffic": tr2["dram_bytes_per_launch"] if tr2 else None,
                                       "kernel": "trace_fast_kernel<crossing records, 256-bit loads, sibling groups of 3>",
                                       "algorithmic_bytes_per_launch": alg2, "registers": info2["registers"],
                                       "blocks_per_sm": info2["blocks_per_sm"]}
    if lane_fast:
        line["tolerance_lane"] = {"lane": "DG_LANE_FAST (opt-in): identical face sequences on non-degenerate queries, end points within "
                                          "1e-9 x bbox diagonal (tests/test_gpu_fast_walker.py::test_tolerance_lane_parity_gate); rank 0's shard",
                                  "forward_ms": lane_fast["forward_ms"], "forward_face_crossings_per_s": crossings_local / (lane_fast["forward_ms"] * 1e-3),
                                  "step_ms": lane_fast["step_ms"], "value": crossings_local / (lane_fast["step_ms"] * 1e-3)}
    if not args.no_cpu and world == 1:
        try:
            line["cpu_baseline"] = cpu_baseline(xyz, tri, f, b, d, q, scheme, max_steps, budget_s=12.0 if headline else 4.0,
                                                reps=3 if headline else 1, counts=counts)
        except Exception as ex:  # the checker is optional for the GPU arm
            line["cpu_baseline"] = {"value": None, "unit": "face-crossings/s", "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {ex}"}
    return line


def run_ours(args):
    import torch
    import paper_2603_15780_b200 as dg

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
                         f"(python bench.py --gpus N starts them itself)")
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
    ctx = dict(rank=rank, world=world, local=local, dev=dev, dist=dist, backend=args.dist_backend,
               flush=torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev))  # > 126 MB L2
    line = measure(args.workload, args, ctx, headline=True)
    blocks = [k for k in args.blocks.split(",") if k and k != "none" and k != args.workload]
    out = {}
    for key in blocks:
        torch.cuda.empty_cache()
        out[key] = measure(key, args, ctx, headline=False)
    if rank == 0:
        if out:
            line["blocks"] = out
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def spawn_ranks(args):
    """python bench.py --gpus N without a torchrun environment: start the N ranks (one process per GPU)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS), help="the headline workload")
    ap.add_argument("--blocks", default="c3,c4,c5", help="further configurations reported under \"blocks\" (or none)")
    ap.add_argument("--geodesics", type=int, default=0, help="geodesics of the headline workload (default: the workload's)")
    ap.add_argument("--block-geodesics", type=int, default=0, help="cap on the geodesics of each block (testing)")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--dist-backend", default="nccl", help="torch.distributed backend for N>1 (nccl on the GPU box)")
    ap.add_argument("--share-gpu", action="store_true", help="testing only: all ranks use cuda:0 (with --dist-backend gloo)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
