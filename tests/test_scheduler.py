"""The native row scheduler, restating proj/tests/test_scheduler.cpp on the product API and
checking it against the oracle / reference on random sequences."""
import numpy as np
import pytest

import paper_2311_02542_b200 as L


def test_exact_proportional_split():
    prev = L.equal_assignment(400, 3)
    nxt = L.assign_rows(400, [2e5, 1e5, 1e5], prev, 1.0)
    assert [r.count() for r in nxt.ranges] == [200, 100, 100] and nxt.valid()


def test_equal_throughputs_fixed_point():
    for d in (0.1, 0.5, 1.0):
        nxt = L.assign_rows(300, [7.0] * 3, L.equal_assignment(300, 3), d)
        assert [r.count() for r in nxt.ranges] == [100, 100, 100]


def test_dampened_largest_remainder():
    prev = L.WorkerAssignment([L.RowRange(0, 134), L.RowRange(134, 267), L.RowRange(267, 400)],
                              [134 / 400, 133 / 400, 133 / 400], 400)
    nxt = L.assign_rows(400, [2.0, 1.0, 1.0], prev, 0.5)
    assert [r.count() for r in nxt.ranges] == [167, 117, 116]


def test_errors_and_min_one_row():
    prev = L.equal_assignment(4, 4)
    with pytest.raises(L.Error):
        L.equal_assignment(3, 4)
    with pytest.raises(L.Error):
        L.assign_rows(4, [1.0] * 5, prev, 0.5)
    nxt = L.assign_rows(4, [1e9, 1, 1, 1], prev, 1.0)
    assert all(r.count() >= 1 for r in nxt.ranges) and nxt.valid()


def test_convergence_2_1_1_within_10_frames():
    height, width, cost = 400, 100, [0.5, 1.0, 1.0]
    cur = L.equal_assignment(height, 3)
    for _ in range(10):
        sim = [cur.ranges[w].count() * cost[w] for w in range(3)]
        st = L.run_frame(cur, width, lambda w, r: None, sim)
        cur = L.next_assignment(cur, st, 0.5)
    assert [abs(a - b) <= 1 for a, b in zip([r.count() for r in cur.ranges], [200, 100, 100])]


def test_dynamic_beats_static_on_row_cost_ramp():
    height, width = 300, 64
    cost = lambda y: 0.05 + 1.5 * y / 300.0  # noqa: E731

    def frame_time(a):
        return max(sum(cost(y) for y in range(r.begin, r.end)) for r in a.ranges)

    static = frame_time(L.equal_assignment(height, 3))
    cur = L.equal_assignment(height, 3)
    for _ in range(30):
        sim = [sum(cost(y) for y in range(r.begin, r.end)) for r in cur.ranges]
        cur = L.next_assignment(cur, L.run_frame(cur, width, lambda w, r: None, sim), 0.5)
    assert frame_time(cur) <= static


def test_aggregate_stats():
    frames = [L.FrameStats(wall_ms=10.0) for _ in range(100)]
    s = L.aggregate_stats(frames)
    assert s.mean_fps == pytest.approx(100) and s.p99_fps == pytest.approx(100)
    frames[99].wall_ms = 100.0
    s = L.aggregate_stats(frames)
    assert s.p99_fps < s.mean_fps and s.p99_fps < 100
    with pytest.raises(L.Error):
        L.aggregate_stats([])


def test_run_frame_disjoint_and_failure():
    cur = L.equal_assignment(64, 4)
    touched = np.zeros(64, int)

    def work(w, r):
        touched[r.begin:r.end] += 1

    L.run_frame(cur, 8, work)
    assert (touched == 1).all()

    def bad(w, r):
        if w == 2:
            raise RuntimeError("boom")

    with pytest.raises(L.Error, match="worker 2 failed: boom"):
        L.run_frame(cur, 8, bad)


def test_random_sequences_match_oracle(oracle):
    rng = np.random.default_rng(81)
    for _ in range(40):
        workers = int(rng.integers(2, 8))
        height = workers + int(rng.integers(0, 500))
        cur = L.equal_assignment(height, workers)
        ro, so = oracle.equal_assignment(height, workers)
        assert list(cur.rows()) == list(ro)
        for _ in range(10):
            tp = rng.uniform(0.1, 10.0, workers)
            d = float(rng.uniform(0.1, 1.0))
            cur = L.assign_rows(height, tp, cur, d)
            ro, so = oracle.assign_rows(height, tp, so, ro, d)
            assert list(cur.rows()) == list(ro) and np.array_equal(cur.shares, so)
            assert all(r.count() >= 1 for r in cur.ranges)
