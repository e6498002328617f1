"""The reference's own emitted C (oracle/_ref, built by oracle/build_ref.py)
agrees bit for bit with the golden vectors — so it is a valid CPU baseline
for bench.py — and the slab-threaded driver does not change a bit."""

import pytest

from helpers import golden_io, manifest, same_bits
from oracle import refc

PROGRAM_CASES = {"c1_dtg": "c1_dtg", "c2_maxwell": "c2_maxwell",
                 "c3_christoffel": "c3_christoffel", "p2": "c4_p2", "p3": "c4_p3"}


@pytest.mark.parametrize("prog_name,case", sorted(PROGRAM_CASES.items()))
@pytest.mark.parametrize("threads", [1, 3])
def test_reference_c_matches_golden(prog_name, case, threads):
    if not refc.available(prog_name):
        pytest.skip("oracle/_ref not built (python oracle/build_ref.py)")
    spec = manifest()["cases"][case]
    env, want = golden_io(case)
    refc.RefProgram(prog_name).run(env, spec["N"], threads=threads, min_slab=8)
    for t in spec["targets"]:
        # the reference C starts sums from 0 (codegen_c.py:206); equal bits
        # for these inputs (checked), tolerance would be 1e-13 otherwise
        assert same_bits(env[t], want[t]), t
