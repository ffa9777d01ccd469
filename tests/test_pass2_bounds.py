"""Host-side bound the many-jobs pass 2 relies on (agg_jobs lists the jobs whose Q range is
not inside one pixel; the job-list agg_reduce is launched with min(jobs, 2 W) warps): with
the integer thresholds T(x) = ceil(x Qtot / W) and T'(x) = floor(x Qtot / W) (O13), at most
2 (W - 1) of any partition of [0, Qtot) into consecutive jobs straddle a pixel -- each such
job holds T(xb + 1) in (start, end] or T'(xb + 1) in [start, end), and the jobs' ranges are
disjoint.  Brute force over random partitions, including empty jobs and tiny Qtot."""
import numpy as np
import pytest


def ceil_div(a, b):
    return -(-a // b)


def straddling(cuts, Qtot, W):
    n = 0
    for start, end in zip(cuts[:-1], cuts[1:]):
        # b1raw(start) = max{x in [0, W] : T(x) <= start}
        xb = max(x for x in range(W + 1) if ceil_div(x * Qtot, W) <= start)
        if xb >= W - 1:
            continue
        nc = ceil_div((xb + 1) * Qtot, W)
        nf = (xb + 1) * Qtot // W
        if not (end < nc and end <= nf):
            n += 1
    return n


@pytest.mark.parametrize("seed", range(12))
def test_straddling_jobs_at_most_two_per_threshold(seed):
    rng = np.random.default_rng(seed)
    W = int(rng.integers(2, 40))
    Qtot = int(rng.choice([1, 2, W - 1, W, W + 1, int(rng.integers(1, 10 ** 6))]))
    Qtot = max(Qtot, 1)
    jobs = int(rng.integers(1, 400))
    cuts = np.sort(rng.integers(0, Qtot + 1, jobs - 1)).tolist()
    cuts = [0] + cuts + [Qtot]
    assert straddling(cuts, Qtot, W) <= 2 * (W - 1)


def test_bound_is_reached_order_of_magnitude():
    """Jobs of one Q unit each over Qtot = 3 W: every threshold sits in its own job."""
    W, Qtot = 16, 48
    cuts = list(range(Qtot + 1))
    n = straddling(cuts, Qtot, W)
    assert W - 1 <= n <= 2 * (W - 1)
