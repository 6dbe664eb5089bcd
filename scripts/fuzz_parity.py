"""Dev: parity fuzzing -- the seeded random-shape GPU tests re-run with other seeds (signature fwd/bwd
with stream and basepoints, logsignature in the three bases, the saved-chunk pair).  Prints every
failure; exit code = number of failures."""
import sys
import traceback

sys.path.insert(0, ".")
import tests.test_gpu_random_shapes as rs  # noqa: E402
import tests.test_gpu_saved as sv  # noqa: E402

seeds = [int(a) for a in sys.argv[1:]] or [1, 2, 3]
fails = 0
for seed in seeds:
    jobs = [(rs.test_random_shape_parity, c) for c in rs._cases(24, seed)]
    jobs += [(rs.test_random_shape_logsignature, c) for c in rs._log_cases(18, seed + 1000)]
    jobs += [(sv.test_saved_random_shapes, c) for c in sv._random_saved_cases(8, seed + 2000)]
    for fn, args in jobs:
        try:
            fn(*args)
        except Exception:
            fails += 1
            print(f"FAIL seed={seed} {fn.__name__}{args}")
            traceback.print_exc(limit=2)
print(f"fuzz: {fails} failures over seeds {seeds}")
sys.exit(fails)
