import sys
sys.path.insert(0, "/root/repo")
from paper_1611_00606_b200 import Dims, ProblemSpec, generate, build_hs, GpuPolicy, rel_frob_error
from oracle import brute
na, nl, ng = (int(x) for x in sys.argv[1:4])
p = generate(ProblemSpec(Dims(na, nl, ng), seed=3))
out = build_hs(p, GpuPolicy(engine="int8"))
ref = build_hs(p, GpuPolicy(engine="dmma"))
print(na, nl, ng, "H err", rel_frob_error(out.h.matrix, ref.h.matrix), "S err", rel_frob_error(out.s.matrix, ref.s.matrix))
