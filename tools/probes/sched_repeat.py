"""Repeat the native-scheduler policy test (tests/test_gpu_sched.py) N times against the Python
scheduler and report every reply that differs and whether it equals some other reply (stale /
misrouted). args: [iters] [policy]. Found the default-stream wait bug (sched.stream_handle)."""
import sys, torch
sys.path.insert(0, ".")
from tests import test_gpu_sched as T
rows_of = lambda c: 8 + 5 * c
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
policy = sys.argv[2] if len(sys.argv) > 2 else "nolockstep"
ref = T._executor("python", "nolockstep")
with ref:
    want = T._run_all(ref, rows_of)
want2 = None
bad = 0
for it in range(iters):
    ex = T._executor("native", policy, wait_per_token=0.001, wait_cap=0.01)
    try:
        with ex:
            got = T._run_all(ex, rows_of)
    finally:
        ex.close()
    for c in range(T.N_CLIENTS):
        for i, (x, y) in enumerate(zip(want[c], got[c])):
            if not torch.equal(x, y):
                bad += 1
                # which other reply does it equal?
                hits = [(cc, j) for cc in range(T.N_CLIENTS) for j, z in enumerate(want[cc]) if z.shape == y.shape and torch.equal(z, y)]
                print(f"iter {it} client {c} reply {i} shape {tuple(y.shape)} mismatch; equals want {hits}; maxdiff {(x.float()-y.float()).abs().max().item():.3g}", flush=True)
print("iters", iters, "mismatches", bad)
# python executor repeatability
ref2 = T._executor("python", "nolockstep")
with ref2:
    w2 = T._run_all(ref2, rows_of)
ref2.close()
pb = sum(1 for c in range(T.N_CLIENTS) for x, y in zip(want[c], w2[c]) if not torch.equal(x, y))
print("python rerun mismatches", pb)
