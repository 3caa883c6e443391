"""c2 / c3 forward with an FMA-contracted build of the library (DG_B200_LIB=build/variants/fma.so) against the
exact one: time, and how many results differ (diagnostic for the contraction lane)."""
import os, sys, subprocess, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    import paper_2603_15780_b200 as dg
    from bench import make_workload
    key, n = sys.argv[2], int(sys.argv[3])
    xyz, tri, f, b, d, q = make_workload(key, n, 42)
    mesh = dg.Mesh(xyz, tri, device=0)
    dev = torch.device("cuda", 0)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
    F, B, D = t(f, torch.int32), t(b, torch.float64), t(d, torch.float64)
    o = dict(face=torch.empty(n, dtype=torch.int32, device=dev), bary=torch.empty(n, 3, dtype=torch.float64, device=dev),
             dir=torch.empty(n, 3, dtype=torch.float64, device=dev), crossings=torch.empty(n, dtype=torch.int32, device=dev),
             total_crossings=torch.zeros(1, dtype=torch.int64, device=dev))
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); mesh.trace_batch_device(F, B, D, o); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    np.savez(sys.argv[4], face=o["face"].cpu().numpy(), bary=o["bary"].cpu().numpy(), dir=o["dir"].cpu().numpy(),
             crossings=o["crossings"].cpu().numpy(), ms=min(ts), pos=mesh.embed(o["face"].cpu().numpy(), o["bary"].cpu().numpy()))
    sys.exit(0)
for key, n in (("c2", 1_000_000), ("c3", 1_000_000)):
    res = {}
    for tag, lib in (("exact", None), ("fma", os.path.join(ROOT, "build/variants/fma.so"))):
        env = dict(os.environ)
        if lib: env["DG_B200_LIB"] = lib
        out = f"/tmp/fma_{key}_{tag}.npz"
        subprocess.check_call([sys.executable, __file__, "child", key, str(n), out], env=env)
        res[tag] = np.load(out)
    a, b = res["exact"], res["fma"]
    print(key, "exact %.3f ms, fma %.3f ms" % (a["ms"], b["ms"]), "| end faces differ:", int((a["face"] != b["face"]).sum()),
          "crossing counts differ:", int((a["crossings"] != b["crossings"]).sum()),
          "max |dpos| %.3g" % np.abs(a["pos"] - b["pos"])[a["face"] == b["face"]].max(), "max |ddir| %.3g" % np.abs(a["dir"] - b["dir"])[a["face"] == b["face"]].max(), flush=True)
