"""Long randomised parity campaign (dev tool): runs tests/test_gpu_parity_fuzz.py's whole-path
comparison for seeds [lo, hi) and lists failures.  Usage: python tools/fuzz_campaign.py lo hi"""
import sys, os, traceback, time
ROOT = os.environ.get("GRAFT_REPO_ROOT", "/root/repo")
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_gpu_parity_fuzz as F
from oracle import ref
lo, hi = int(sys.argv[1]), int(sys.argv[2])
fails = 0
t0 = time.time()
for s in range(lo, hi):
    try:
        F.test_fuzz_whole_path(ref, s)
    except Exception as e:
        fails += 1
        print("FAIL", s, F._draw(s), repr(e)[:300], flush=True)
print(f"done {hi-lo} seeds, {fails} failures, {time.time()-t0:.0f}s", flush=True)
