"""Host logic of the Z trace's arrival model (bench.py: poisson_arrivals, VirtualQueue), pinned
to queueing theory: an M/D/1 queue's mean wait is rho*s / (2(1 - rho)) (Pollaczek-Khinchine)."""
import numpy as np
import pytest

import bench


def test_saturated_queue_window_is_next_w():
    q = bench.VirtualQueue(np.zeros(10), window=4)
    ttft = []
    for i in range(10):
        assert q.start(i) == list(range(i + 1, min(10, i + 5)))
        ttft.append(q.finish(i, 2.0))
    assert ttft == [2.0 * (i + 1) for i in range(10)]


def test_sparse_arrivals_never_queue():
    a = np.arange(20) * 10.0
    q = bench.VirtualQueue(a, window=4)
    for i in range(20):
        assert q.start(i) == []          # nobody else has arrived yet
        assert q.finish(i, 3.0) == pytest.approx(3.0)


def test_window_holds_only_arrived_requests():
    a = np.array([0.0, 1.0, 2.0, 50.0, 51.0])
    q = bench.VirtualQueue(a, window=3)
    assert q.start(0) == []              # t = 0: request 1 arrives at 1
    q.finish(0, 5.0)                     # t = 5: requests 1, 2 waiting, 3 not yet
    assert q.start(1) == [2]
    q.finish(1, 5.0)
    assert q.start(2) == []              # t = 10
    q.finish(2, 5.0)
    assert q.start(3) == []              # idle until 50
    assert q.t == 50.0


@pytest.mark.parametrize("rho", [0.5, 0.8])
def test_md1_mean_wait(rho):
    s, n = 1.0, 200_000
    a = bench.poisson_arrivals(n, rho, s, seed=7)
    assert np.mean(np.diff(a)) == pytest.approx(s / rho, rel=0.01)
    q = bench.VirtualQueue(a, window=0)
    wait = np.empty(n)
    for i in range(n):
        q.start(i)
        wait[i] = q.finish(i, s) - s
    assert wait.mean() == pytest.approx(rho * s / (2 * (1 - rho)), rel=0.05)
