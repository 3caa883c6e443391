"""Forward-only timing sweep of the trace kernel (device-resident inputs, CUDA events).
usage: DG_B200_LIB=build/variants/x.so python scripts/tune_trace.py c2|c3 [n]"""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15780_b200 as dg
from bench import make_workload

key = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
xyz, tri, f, b, d, q = make_workload(key, n, 42)
cache = {"on": True, "off": False}.get(os.environ.get("TC", "auto"), "auto")
mesh = dg.Mesh(xyz, tri, device=0, transport_cache=cache)
print("transport cache:", mesh.has_transport_cache, "device MB:", mesh.device_bytes / 1e6)
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
F, B, D = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64)
o = dict(face=torch.empty(n, dtype=torch.int32, device=dev), bary=torch.empty(n, 3, dtype=torch.float64, device=dev),
         dir=torch.empty(n, 3, dtype=torch.float64, device=dev), traced=torch.empty(n, dtype=torch.float64, device=dev),
         term=torch.empty(n, dtype=torch.uint8, device=dev), status=torch.empty(n, dtype=torch.uint8, device=dev),
         total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
info = dg.kernel_info(False, False)
tag = os.path.basename(os.environ.get("DG_B200_LIB", "default"))
def run(**kw):
    for _ in range(2): mesh.trace_batch_device(F, B, D, o, **kw)
    torch.cuda.synchronize()
    ts = []
    for _ in range(4):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); mesh.trace_batch_device(F, B, D, o, **kw); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    cr = int(o["total_crossings"].item())
    print(f"{tag:14s} {key} regs={info['registers']} bps={info['blocks_per_sm']} {str(kw):48s} {min(ts):8.3f} ms  {cr/min(ts)/1e6:7.2f} Gcross/s", flush=True)
run()
for rm in (2, 4, 8, 16): run(refill_min=rm)
for bps in (1, 2, 3, 4, 5, 6, 8):
    if bps <= max(info["blocks_per_sm"], 1): run(blocks_per_sm=bps)
run(sort_by_face=True)
