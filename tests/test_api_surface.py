"""The package exports every public name of the reference package
(pkg/src/tlang/__init__.py:3-28), plus the evaluate entry points of
pkg/src/tlang/evaluator.py:204-257 and the multi-domain/program extensions."""

import paper_1804_10120_b200 as tl

# pkg/src/tlang/__init__.py:9-28
REFERENCE_ALL = [
    "Declarations", "IndexVar", "Registry", "ScalarConst", "ScalarField", "Statement",
    "SymmetrySpec", "TensorField", "TensorShape", "ValidatedStatement", "canonical_index",
    "component_count", "count_data", "iter_canonical", "parse_program", "render", "signature",
    "slot_index", "validate_statement",
]


def test_reference_public_names_exported():
    missing = [n for n in REFERENCE_ALL if not hasattr(tl, n)]
    assert not missing, missing
    assert set(REFERENCE_ALL) <= set(tl.__all__)


def test_evaluate_entry_points_and_extensions():
    for name in ("eval_statement", "eval_statement_per_component", "eval_program", "eval_batch",
                 "capture_graph", "EvalError", "ValidationError"):
        assert callable(getattr(tl, name)) or isinstance(getattr(tl, name), type), name


def test_module_level_helpers():
    from paper_1804_10120_b200 import bench, evaluator, symmetry

    # symmetry.py:169 alias_table, evaluator.py:204/239, bench.py:252-271
    assert callable(symmetry.alias_table)
    assert callable(evaluator.eval_statement) and callable(evaluator.eval_statement_per_component)
    assert callable(bench.time_statement) and callable(bench.make_env) and callable(bench.bw_eff)
