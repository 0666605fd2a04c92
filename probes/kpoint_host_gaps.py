"""Host-side phases of the k-point lanes: time spent in _build_host before the
native call, inside it, and after it, per lane; then per-k-point throughput at
several pipeline depths.

    python probes/kpoint_host_gaps.py [C3] [n] [depths...]
"""
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1611_00606_b200 import CONFIGS, ProblemSpec, generate, iter_hs_kpoints, pin_instance  # noqa: E402
from paper_1611_00606_b200 import pipeline  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
depths = [int(x) for x in sys.argv[3:]] or [2, 3]
p = pin_instance(generate(ProblemSpec(CONFIGS[cfg], seed=0)))

log = []
_orig_call, _orig_host = pipeline._call_build, pipeline._build_host


def call(*a, **k):
    t0 = time.perf_counter()
    r = _orig_call(*a, **k)
    log.append((threading.get_ident(), "call", t0, time.perf_counter()))
    return r


def host(*a, **k):
    t0 = time.perf_counter()
    r = _orig_host(*a, **k)
    log.append((threading.get_ident(), "host", t0, time.perf_counter()))
    return r


pipeline._call_build, pipeline._build_host = call, host
pieces = {}


def timed(name, fn):
    def w(*a, **k):
        t0 = time.perf_counter()
        r = fn(*a, **k)
        pieces.setdefault(name, []).append(time.perf_counter() - t0)
        return r
    return w


for name in ("validate_instance", "_host_problem", "_host_matrix", "_policy"):
    setattr(pipeline, name, timed(name, getattr(pipeline, name)))
for depth in depths:
    for o in iter_hs_kpoints([p] * (depth + 2), depth=depth):  # warm contexts
        del o
    log.clear()
    pieces.clear()
    t0 = time.perf_counter()
    for o in iter_hs_kpoints([p] * n, depth=depth):
        del o
    t = (time.perf_counter() - t0) / n
    calls = [e for e in log if e[1] == "call"]
    hosts = [e for e in log if e[1] == "host"]
    pre = post = 0.0
    for c in calls:
        h = min((h for h in hosts if h[0] == c[0] and h[2] <= c[2] and h[3] >= c[3]), key=lambda h: h[3] - h[2])
        pre += c[2] - h[2]
        post += h[3] - c[3]
    gaps = []
    by_lane = {}
    for h in sorted(hosts, key=lambda h: h[2]):
        if h[0] in by_lane:
            gaps.append(h[2] - by_lane[h[0]])
        by_lane[h[0]] = h[3]
    print(f"depth {depth}: {t*1e3:.1f} ms/k-point; per call: pre {pre/len(calls)*1e3:.2f} ms, "
          f"native {sum(c[3]-c[2] for c in calls)/len(calls)*1e3:.1f} ms, post {post/len(calls)*1e3:.2f} ms; "
          f"lane idle between calls {sum(gaps)/max(1,len(gaps))*1e3:.2f} ms")
    print("   pre-call pieces (mean / max ms):",
          {k: (round(sum(v) / len(v) * 1e3, 2), round(max(v) * 1e3, 2)) for k, v in pieces.items()})
