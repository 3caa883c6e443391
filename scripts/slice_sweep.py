import os, sys, time, subprocess
shapes = [("4", "1,2,3,2"), ("5", "1,3,3,3,1"), ("5", "1,2,3,3,2"), ("4", "1,2,4,3"), ("5", "1,3,4,3,1"), ("4", "1,3,3,2"), ("5", "1,2,3,2,1"), ("5", "2,3,4,3,2"), ("4", "2,4,5,3"), ("5", "1,3,4,4,2")]
for S, shape in shapes:
    env = dict(os.environ, DG_BATCH_SLICES=S)
    if shape: env["DG_BATCH_SLICE_SHAPE"] = shape
    out = subprocess.run([sys.executable, "scripts/e2e_one.py"], env=env, capture_output=True, text=True).stdout.strip().splitlines()[-1]
    print(S, shape or "equal", out, flush=True)
