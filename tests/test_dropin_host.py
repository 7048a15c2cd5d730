"""Host-side logic of the drop-in names added for the reference's public API
(no GPU): argument validation that precedes any device work, and the Foata class
structure an ExecutionTrace reports, pinned to the reference's own traces
(tests/golden/within_element.npz, tools/gen_golden.py section 13)."""

import numpy as np
import pytest

import paper_2207_00280_b200 as P
from paper_2207_00280_b200.runtime import _foata_task_count, foata_class_sizes
from tests.conftest import load_golden


@pytest.mark.parametrize("key,p", [("K2_p0_w1", 0), ("K2_p1_w3", 1), ("K3_p2_w2", 2)])
def test_foata_classes_match_reference_trace(key, p):
    g = load_golden("within_element")
    P3 = (p + 1) ** 3
    n = int(g[f"{key}_ntasks"])
    assert _foata_task_count(p, P3) == n
    sizes = foata_class_sizes(p, P3)
    assert len(sizes) == p + 7 and int(g[f"{key}_barriers"]) == p + 6
    assert int(g[f"{key}_syncs"]) == 0
    # the reference's completion order (any worker count) visits the classes in order --
    # the class of each completed task is the barrier-phase sequence the device reports --
    # and every task completes once
    cls = g[f"{key}_class_of_order"]
    assert np.array_equal(cls, np.repeat(np.arange(p + 7), sizes))
    assert np.array_equal(g[f"{key}_order_sorted"], np.arange(n))
    if f"{key}_order" in g.files:  # workers=1: the raw order is class-by-class id order
        assert np.array_equal(g[f"{key}_order"], np.arange(n))


def test_eval_basis_validation_precedes_device():
    kv = P.make_knot_vector(3, 2)
    with pytest.raises(ValueError):
        P.eval_basis(kv, 0, 3, 0.5)   # order above the degree (splines.py:100-101)
    with pytest.raises(IndexError):
        P.eval_basis(kv, 10, 2, 0.5)  # splines.py:103-104
    with pytest.raises(IndexError):
        P.eval_basis(kv, -1, 1, 0.5)
    with pytest.raises(IndexError):
        P.eval_basis_order0(kv, 7, 0.5)  # len(t) - 2 = 6 is the last span (splines.py:85-86)


def test_run_within_element_validation():
    kv = P.make_knot_vector(3, 1)
    with pytest.raises(ValueError):
        P.run_within_element((0, 0, 0), kv, "magic", 2)
    with pytest.raises(ValueError):
        P.run_within_element((0, 0, 0), kv, "classical", 2, trace=P.ExecutionTrace())
    t = P.ExecutionTrace()
    assert t.graph is None and t.completion_order == [] and t.barriers == 0
