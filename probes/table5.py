"""The paper's Table 5 case (NaCl, K_max 4.0: 512 atoms, N_L 49, N_G 9273) on
one B200 through the drop-in build_hs, reported next to the recorded 2xK20x
breakdown (report.TABLE5)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1611_00606_b200 import GpuPolicy, ProblemSpec, build_hs, generate, pin_instance  # noqa: E402
from paper_1611_00606_b200.report import compare_with_table5, format_table, nacl_table5_dims, summarize  # noqa: E402

fused = "--unfused" not in sys.argv
engine = "dmma" if "--dmma" in sys.argv else "int8"
t0 = time.perf_counter()
p = pin_instance(generate(ProblemSpec(nacl_table5_dims(), seed=0)))
print(f"generated NaCl 4.0 instance in {time.perf_counter() - t0:.1f} s")
for i in range(3):
    t0 = time.perf_counter()
    out = build_hs(p, GpuPolicy(fused=fused, engine=engine))
    wall = time.perf_counter() - t0
print(f"build_hs wall ({engine} engine, host numpy in/out, {'fused' if fused else 'one launch per section'}): "
      f"{wall:.3f} s; "
      f"paper: 46.97 s on 2xK20x + 16 cores (PAPER.md:547), 26.575 s on 4xK40 + 24 cores (PAPER.md:597)")
rep = summarize(out.ledger)
print(format_table(rep))
print()
print(compare_with_table5(rep))
print({k: round(v * 1e3, 2) for k, v in out.timings.items() if isinstance(v, float)})
