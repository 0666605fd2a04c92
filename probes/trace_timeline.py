"""Print the absolute GPU timeline of build_hs calls from an HSB_TRACE log.

    HSB_TRACE=1 python probes/kpoint_pipeline.py C3 8 2 2> trace.log
    python probes/trace_timeline.py trace.log

Each build_hs call prints "[hsb trace] <ctx> <tag> <ms>" lines (ms since a
process-wide base event); calls are split at their "start" tag.  For every
call the script lists the upload / section / download completion times and
the PCIe throughput implied by the download stamps.
"""
import sys
from collections import defaultdict

calls = []
cur = {}
for line in open(sys.argv[1]):
    if not line.startswith("[hsb trace]"):
        continue
    _, _, ctx, *tag, ms = line.split()
    tag = " ".join(tag)
    if tag == "start":
        cur[ctx] = {"ctx": ctx, "marks": []}
        calls.append(cur[ctx])
    cur[ctx]["marks"].append((tag, float(ms)))

ctx_ids = {c: i for i, c in enumerate(dict.fromkeys(c["ctx"] for c in calls))}
calls.sort(key=lambda c: c["marks"][0][1])
prev_end = None
for c in calls:
    m = c["marks"]
    t0 = m[0][1]
    d = defaultdict(list)
    for tag, t in m:
        d[tag.split()[0]].append(t)
    last_d2h = max(d.get("d2h_h", [t0]) + d.get("d2h_s", [t0]))
    line = f"lane {ctx_ids[c['ctx']]} start {t0:9.2f}"
    for key in ("h2d_b", "h2d_a", "s_done", "loop2_done", "h_done"):
        if key in d:
            line += f"  {key} +{d[key][0] - t0:6.2f}"
    if d.get("d2h_s"):
        line += f"  S-d2h +{min(d['d2h_s']) - t0:6.2f}..+{max(d['d2h_s']) - t0:6.2f}"
    if d.get("d2h_h"):
        line += f"  H-d2h ..+{max(d['d2h_h']) - t0:6.2f}"
    line += f"  end +{last_d2h - t0:6.2f}"
    if prev_end is not None:
        line += f"  (since prev call end {last_d2h - prev_end:6.2f})"
    prev_end = last_d2h
    print(line)
