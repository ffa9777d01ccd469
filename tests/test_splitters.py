"""The sample sort's splitter rule (dvl_select_splitters, host code of the library; SURVEY
8(e) "Build" step 3), on CPU: exact quantiles when every cell is a sample, empty and uneven
ranks, the regular-sampling bound, and the failure when no valid choice exists."""
import numpy as np
import pytest

import paper_2306_11612_b200 as dvl


def _samples(runs, S):
    G = len(runs)
    out = np.full((G, S), np.iinfo(np.uint64).max, np.uint64)
    for p, run in enumerate(runs):
        s = min(S, len(run))
        if s:
            out[p, :s] = run[(np.arange(s, dtype=np.int64) * len(run)) // s]
    return out


@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_exact_quantiles_when_all_cells_are_samples(G):
    rng = np.random.default_rng(G)
    keys = rng.choice(1 << 40, size=100 * G, replace=False).astype(np.uint64)
    runs = [np.sort(keys[p::G]) for p in range(G)]
    spl = dvl.select_splitters(_samples(runs, 1024), [len(r) for r in runs], 1024)
    allk = np.sort(keys)
    n = len(allk)
    assert spl.tolist() == [int(allk[(k * n) // G]) for k in range(1, G)]


@pytest.mark.parametrize("counts", [[0, 500, 500], [0, 0, 900, 100], [1000, 0], [3, 2000, 40, 7]])
def test_empty_and_uneven_ranks(counts):
    rng = np.random.default_rng(sum(counts))
    G = len(counts)
    keys = rng.choice(1 << 36, size=sum(counts), replace=False).astype(np.uint64)
    cuts = np.cumsum([0] + counts)
    runs = [np.sort(keys[cuts[p]:cuts[p + 1]]) for p in range(G)]
    spl = dvl.select_splitters(_samples(runs, 64), counts, 64)
    assert np.all(np.diff(spl.astype(np.float64)) > 0)
    share = np.bincount(np.searchsorted(spl, keys, side="right"), minlength=G)
    n = sum(counts)
    assert share.min() > 0
    assert share.max() <= n / G + 2 * n / 64 + G   # regular sampling: n/G + O(n/S) per rank


def test_regular_sampling_bound_large():
    rng = np.random.default_rng(7)
    G, S = 8, 1024
    keys = rng.choice(1 << 45, size=200_000, replace=False).astype(np.uint64)
    # ranks hold random slices of very different sizes
    cuts = np.sort(rng.choice(np.arange(1, len(keys)), G - 1, replace=False))
    parts = np.split(rng.permutation(keys), cuts)
    runs = [np.sort(p) for p in parts]
    spl = dvl.select_splitters(_samples(runs, S), [len(r) for r in runs], S)
    share = np.bincount(np.searchsorted(spl, keys, side="right"), minlength=G)
    assert share.max() <= len(keys) / G + G * len(keys) / S


def test_too_few_cells_fails():
    runs = [np.array([5], np.uint64), np.array([], np.uint64), np.array([], np.uint64)]
    with pytest.raises(dvl.DvlError):
        dvl.select_splitters(_samples(runs, 4), [1, 0, 0], 4)
