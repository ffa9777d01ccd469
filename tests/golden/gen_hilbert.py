"""Regenerates the Hilbert vectors of tests/golden/spec_examples.json without the oracle's
encoder (reading A1/O3: Skilling 2004, "Programming the Hilbert curve", AIP Conf. Proc. 707).

Independent route: only Skilling's *decoder* (TransposetoAxes, restated here in Python on
big ints) is used, and the encoder is obtained by inverting it with a top-down search over
the 8 octant digits of each level.  That search relies only on the curve property that
every block of 8^k consecutive codes fills one aligned 2^k cube (pinned separately by
tests/test_oracle_hilbert.py's dyadic-block contiguity test).  No oracle/ code is imported.

Run: python tests/golden/gen_hilbert.py  (prints the JSON list; tests/test_golden.py checks
that the committed vectors equal this script's output).
"""
import json
import sys


def transpose_to_axes(X, b):
    """Skilling's TransposetoAxes for n = 3 axes (Gray decode, then undo excess work)."""
    X = list(X)
    N = 2 << (b - 1)
    t = X[2] >> 1
    for i in (2, 1):
        X[i] ^= X[i - 1]
    X[0] ^= t
    Q = 2
    while Q != N:
        P = Q - 1
        for i in (2, 1, 0):
            if X[i] & Q:
                X[0] ^= P
            else:
                t = (X[0] ^ X[i]) & P
                X[0] ^= t
                X[i] ^= t
        Q <<= 1
    return X


def decode(h, b):
    """Code -> (x, y, z): the 3b-bit code read MSB first as X[0], X[1], X[2] bits per level."""
    X = [0, 0, 0]
    for j in range(b - 1, -1, -1):
        d = (h >> (3 * j)) & 7
        X[0] |= ((d >> 2) & 1) << j
        X[1] |= ((d >> 1) & 1) << j
        X[2] |= (d & 1) << j
    return tuple(transpose_to_axes(X, b))


def encode_by_search(p, b):
    """(x, y, z) -> code by descending the octree: at level k the code block
    [prefix*8 + d] * 8^k .. + 8^k - 1 covers one aligned 2^k cube; take the digit whose
    cube contains p (exactly one does)."""
    prefix = 0
    for k in range(b - 1, -1, -1):
        hits = []
        for d in range(8):
            c = ((prefix << 3) | d) << (3 * k)
            q = decode(c, b)
            if all((q[a] >> k) == (p[a] >> k) for a in range(3)):
                hits.append(d)
        assert len(hits) == 1, (p, b, k, hits)
        prefix = (prefix << 3) | hits[0]
    assert decode(prefix, b) == tuple(p)
    return prefix


VECTORS = [("S:45", (0, 0, 0), 5),
           ("SURVEY 8(c) A1 vector", (1, 1, 1), 2),
           ("SURVEY 8(c) A1 vector", (3, 5, 7), 3),
           ("SURVEY 8(c) A1 vector", (1000, 2000, 3000), 12),
           ("SURVEY 8(c) A1 vector", ((1 << 20) - 1, 0, 0), 20),
           ("SURVEY 8(c) A1 vector", ((1 << 21) - 1, (1 << 21) - 1, (1 << 21) - 1), 21),
           ("gen_hilbert.py", (123456, 654321, 1048575), 21),
           ("gen_hilbert.py", (5, 9, 2), 4),
           ("gen_hilbert.py", (77, 1, 100), 7),
           ("gen_hilbert.py", (4095, 0, 4095), 12)]


def generate():
    return [{"cite": c, "xyz": list(p), "b": b, "h": encode_by_search(p, b)} for c, p, b in VECTORS]


if __name__ == "__main__":
    json.dump(generate(), sys.stdout, indent=1)
    print()
