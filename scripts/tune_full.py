"""Timing of the full tracer variant (payload + transport matrix) on device-resident inputs."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15780_b200 as dg
from bench import make_workload
n = 400000
key = sys.argv[1] if len(sys.argv) > 1 else "c2"
cache = {"on": True, "off": False}.get(os.environ.get("TC", "auto"), "auto")
xyz, tri, f, b, d, q = make_workload(key, n, 42)
mesh = dg.Mesh(xyz, tri, device=0, transport_cache=cache)
print(key, "crossing records:", mesh.has_transport_cache)
dev = torch.device("cuda", 0)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
F, B, D, P = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64), t(q, torch.float64)
o = dict(face=torch.empty(n, dtype=torch.int32, device=dev), bary=torch.empty(n, 3, dtype=torch.float64, device=dev),
         dir=torch.empty(n, 3, dtype=torch.float64, device=dev), payload=torch.empty(n, 3, dtype=torch.float64, device=dev),
         transport=torch.empty(n, 9, dtype=torch.float64, device=dev), total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
for name, kw in (("payload+Q", dict(payload=P, want_q=True)), ("payload", dict(payload=P)), ("Q", dict(want_q=True))):
    oo = dict(o)
    if "payload" not in kw: oo.pop("payload")
    if not kw.get("want_q"): oo.pop("transport")
    ts = []
    for _ in range(4):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); mesh.trace_batch_device(F, B, D, oo, **kw); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    cr = int(o["total_crossings"].item())
    print(f"{os.path.basename(os.environ.get('DG_B200_LIB','default')):12s} full kernel {name:10s} {min(ts):8.3f} ms {cr/min(ts)/1e6:6.2f} Gcross/s regs={dg.kernel_info(False, True, True)}", flush=True)
