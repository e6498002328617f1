"""Differential fuzzing of the front end against the reference package
(build container only — skipped where /root/reference is absent): random
token soups and random well-formed programs must yield the same
diagnostics, the same trees (via render), the same validation verdicts,
signatures and counts."""

import random

import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

ref_parser = pytest.importorskip("tlang.parser")
ref_ir = pytest.importorskip("tlang.ir")

from paper_1804_10120_b200 import ir as my_ir  # noqa: E402
from paper_1804_10120_b200 import parser as my_parser  # noqa: E402

TOKENS = ["tensor", "field", "const", "index", "dim", "rank", "sym", "inner", "Sum", "sqrt",
          "A", "B", "g", "w", "i", "j", "k", "a", "0", "1", "2", "3", "2.5", "1e3", ".5",
          "(", ")", "<", ">", ",", ";", ":", "+", "-", "*", "/", "=", "+=", "-=", "*=", "/=",
          "&&", "#c\n", "\n", " ", "$", "x"]


def _compare(text):
    mine = my_parser.parse_program(text)
    ref = ref_parser.parse_program(text)
    assert [(d.line, d.col, d.message) for d in mine.diagnostics] == \
        [(d.line, d.col, d.message) for d in ref.diagnostics]
    if not ref.diagnostics:
        assert my_parser.render(mine.program) == ref_parser.render(ref.program)
        for sm, sr in zip(mine.program.statements, ref.program.statements):
            try:
                vr = ref_ir.validate_statement(sr, ref.program.decls)
            except ref_ir.ValidationError as exc:
                with pytest.raises(my_ir.ValidationError) as got:
                    my_ir.validate_statement(sm, mine.program.decls)
                assert got.value.code == exc.code
                continue
            vm = my_ir.validate_statement(sm, mine.program.decls)
            assert my_ir.signature(vm) == ref_ir.signature(vr)
            assert my_ir.count_data(vm) == ref_ir.count_data(vr)


@settings(max_examples=300, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(st.lists(st.sampled_from(TOKENS), max_size=40))
def test_token_soup_matches_reference(tokens):
    _compare(" ".join(tokens))


from helpers import FUZZ_DECLS as DECLS, fuzz_statement as _random_statement  # noqa: E402


@pytest.mark.parametrize("seed", range(400))
def test_random_statements_match_reference(seed):
    rng = random.Random(seed)
    _compare(DECLS + "".join(_random_statement(rng) for _ in range(3)))
