"""Write tests/golden/hsm_tiny/ with the REFERENCE's own storage code
(hsgen.storage.save_instance / write_matrix, /root/reference/pkg/src/hsgen/
storage.py) and the reference build_hs outputs as H.hsm / S.hsm, so the
HSM1 reader/writer (paper_1611_00606_b200/storage.py) and the GPU-backed
``run_instance_dir`` are checked against files the reference produced.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_hsm_golden.py
"""
import shutil
from pathlib import Path

from hsgen.builder import build_hs
from hsgen.matcore import Dims
from hsgen.probgen import ProblemSpec, generate
from hsgen.storage import save_instance, write_matrix

out = Path(__file__).resolve().parent / "hsm_tiny"
if out.exists():
    shutil.rmtree(out)
p = generate(ProblemSpec(Dims(2, 4, 6), seed=21, nonhpd_fraction=0.5))
save_instance(p, out, seed=21, nonhpd_fraction=0.5)
res = build_hs(p)
ref = out / "reference_outputs"
ref.mkdir()
write_matrix(ref / "H.hsm", res.h.matrix)
write_matrix(ref / "S.hsm", res.s.matrix)
print("wrote", out)
