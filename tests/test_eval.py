"""Host evaluation helpers (measurement only, no GPU): distance_threshold_recall
evalio.cpp:199-215."""
import numpy as np
import pytest


def test_distance_threshold_recall_worked_example():
    import paper_2605_27691_b200 as K
    t = np.array([[0.1, 0.2, 0.5], [0.3, 0.3, 0.9]], np.float32)
    g = np.array([[0.1, 0.3, 0.4], [0.2, 0.25, 0.3]], np.float32)
    # k=2: row 0 threshold 0.3 -> 2 of 2; row 1 threshold 0.25 -> 0 of 2
    assert K.distance_threshold_recall(t, g, 2) == 0.5
    # k=3: both rows 2 of 3 (the count stops at the first entry above, :209)
    assert K.distance_threshold_recall(t, g, 3) == (2 / 3 + 2 / 3) / 2
    # identical graphs -> 1.0 (a graph is its own distance-threshold match)
    assert K.distance_threshold_recall(g, g, 3) == 1.0
    with pytest.raises(K.InvalidArgument):
        K.distance_threshold_recall(t, g, 0)
    with pytest.raises(K.InvalidArgument):
        K.distance_threshold_recall(t, g, 4)
    with pytest.raises(K.InvalidArgument):
        K.distance_threshold_recall(t[:1], g, 2)


def test_distance_threshold_recall_ties_count():
    import paper_2605_27691_b200 as K
    # a tie with the threshold counts (<=), entries past k_eval are capped
    t = np.array([[1.0, 1.0, 1.0, 1.0]], np.float32)
    g = np.array([[0.5, 1.0, 2.0, 3.0]], np.float32)
    assert K.distance_threshold_recall(t, g, 2) == 1.0
    assert K.distance_threshold_recall(t, g, 1) == 0.0
