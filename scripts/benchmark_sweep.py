"""The reference's `digeo benchmark` protocol (proj/tools/digeo_main.cpp:232-286, the paper's
Fig. 2): batch sweep on icosphere-4 and face sweep at batch 2000, 5 repetitions, median / p25 /
p75, CSV `section,mesh,faces,batch,backend,median_ms,p25_ms,p75_ms,per_trace_us` -- with `gpu`
backend columns (host-facing call, copies included) next to the reference's serial / parallel.
The default record_polyline=True of the reference CLI is kept on all backends (gpu = the one-call
dg_trace_polylines; gpu_two_call = count call + host scan + fill call; gpu_nopolyline for scale).
usage: python scripts/benchmark_sweep.py [out.csv]"""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))


def run(rm, name, batch, section, rows, reps=5, backends=None):
    import paper_2603_15780_b200 as dg
    a = rm.arrays()
    m = dg.Mesh(a["xyz"], a["tri"])
    f, b, d = rm.sample_queries(42, batch, 0.1, np.pi / 2)
    fns = {"serial": lambda: rm.trace_batch(f, b, d, record_polyline=True, workers=-1),
           "parallel": lambda: rm.trace_batch(f, b, d, record_polyline=True, workers=0),
           "gpu": lambda: m.trace_batch(f, b, d, record_polyline=True, poly_views=True),   # one call, dg_trace_polylines
           "gpu_two_call": lambda: m.trace_batch(f, b, d, record_polyline=True, two_call_polylines=True),
           "gpu_nopolyline": lambda: m.trace_batch(f, b, d)}
    for backend in (backends or fns):
        fn = fns[backend]
        fn()
        t = []
        for _ in range(reps):
            t0 = time.perf_counter(); fn(); t.append((time.perf_counter() - t0) * 1e3)
        med, p25, p75 = np.percentile(t, [50, 25, 75])
        rows.append((section, name, rm.nf, batch, backend, med, p25, p75, med * 1000.0 / max(1, batch)))


def sweep(batches=(100, 1000, 10000, 100000), subdivs=(3, 4, 5, 6), reps=5, backends=None):
    import refapi
    rows = []
    m4 = refapi.RefMesh.icosphere(4)
    for batch in batches:
        run(m4, "icosphere4", batch, "batch_sweep", rows, reps, backends)
    for s in subdivs:
        run(refapi.RefMesh.icosphere(s), f"icosphere{s}", 2000, "face_sweep", rows, reps, backends)
    return rows


def write_csv(rows, out):
    with open(out, "w") as fh:
        fh.write("section,mesh,faces,batch,backend,median_ms,p25_ms,p75_ms,per_trace_us\n")
        for r in rows:
            fh.write(",".join(str(x) if not isinstance(x, float) else f"{x:.6g}" for x in r) + "\n")


if __name__ == "__main__":
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/benchmark_sweep.csv"
    write_csv(sweep(), out)
    print(open(out).read())
