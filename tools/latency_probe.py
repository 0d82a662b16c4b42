"""Device time of small (latency-bound) calls: config 2 T60 points and config 3 at M = 1 / 16 (A/B helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sweep as S  # noqa: E402
import workloads as W  # noqa: E402

for name, sc in [("cfg2 T60=0.2", W.cfg2(0.2)), ("cfg2 T60=0.7", W.cfg2(0.7)), ("cfg2 T60=2.0", W.cfg2(2.0)),
                 ("cfg3 diffuse M=1", W.cfg3(1, "diffuse")), ("cfg3 diffuse M=16", W.cfg3(16, "diffuse")),
                 ("cfg1", W.cfg1())]:
    fn, _ = S.scene_call(sc)
    print(f"{name:20s} {S.time_call(fn, reps=20, warm=5) * 1e3:8.1f} us")
