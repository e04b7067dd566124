"""Writes tests/golden/ref_inputs.csat with the REFERENCE's own CSAT writer
(tensor_io.cpp write_inputs_file via oracle/_ref). Run here after
`make -C oracle ref`:  python tests/golden/make_csat.py
The inputs are the reference generator's (synth.cpp) B=2, S=16, m=4, H=3,
D=5, seed 77, so the fixture also pins the generator."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Reference  # noqa: E402

ref = Reference()
q, kc, w = ref.generate(2, 16, 4, 3, 5, 4, 77)
rc, n = ref.write_inputs_file(os.path.join(HERE, "ref_inputs.csat"), q, kc, w, 4, 4)
assert rc == 0 and n == os.path.getsize(os.path.join(HERE, "ref_inputs.csat")), (rc, n)
print("wrote", n, "bytes")
