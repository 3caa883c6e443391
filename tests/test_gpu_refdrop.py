"""The drop-in boundary, proven the hard way: the reference's OWN acceptance suite (proj/tests/acceptance.cpp,
stand-alone main, 10 criteria = SPEC.md:571-580) together with its gradcheck.cpp, oracles.cpp, io.cpp and opt.cpp,
all UNMODIFIED, compiled against include/digeo/{geometry,mesh,tracer,diff}.hpp and linked with libdigeo_host.so +
libdigeo_b200.so in place of the reference's mesh.cpp / tracer.cpp / diff.cpp (tests/refdrop/Makefile; the binary
is built where /root/reference exists and travels to the GPU box in tests/_build/).

Criteria 1-4 and 6 are the numeric ones of SURVEY 8(f1): sphere and torus end-point accuracy against the closed
forms, GFD and EP gradient medians of run_gradcheck, bitwise determinism over 5 fixtures x 2 000 traces with
polylines. They must print [PASS]. 8 (Projection-Integration parity), 9 (L-BFGS vs Lloyd through the
transport-matrix consumer, opt.cpp:298-323) and 10 (property bundle) exercise the same GPU path and must pass too.
Criteria 5 and 7 are wall-clock SHAPES of the CPU implementation -- 5: (forward + 10 000 per-sample ep_jacobians
calls) against one gfd_batched_many call, in [2, 6]; 7: run time linear in the face count, R^2 >= 0.9 -- which a
GPU path does not have by construction (a per-sample EP call is a kernel launch; run time is flat in F). They are
reported, not asserted; the cost ratio is pinned in crossings instead (test_gpu_acceptance.py)."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "_build", "ref_acceptance")


def test_reference_acceptance_suite_unmodified_on_the_gpu_path(gpu):
    if not os.path.exists(EXE):
        pytest.fail("tests/_build/ref_acceptance missing: build() compiles it where /root/reference exists")
    p = subprocess.run([EXE], capture_output=True, text=True, timeout=900)
    print(p.stdout)
    print(p.stderr[-2000:])
    got = {int(m.group(2)): m.group(1) for m in re.finditer(r"\[(PASS|FAIL)\] criterion\s+(\d+):", p.stdout)}
    assert sorted(got) == list(range(1, 11)), f"criteria reported: {sorted(got)}\n{p.stdout}\n{p.stderr[-2000:]}"
    must = (1, 2, 3, 4, 6, 8, 9, 10)
    failed = [c for c in must if got[c] != "PASS"]
    assert not failed, f"criteria {failed} failed:\n{p.stdout}"
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        open(os.path.join(out, "ref_acceptance.log"), "w").write(p.stdout)
