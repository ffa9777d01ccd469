"""Independent pure-Python brute force for tiny inputs (exact rationals, big ints).

Used only by the tests to pin the oracle (and, transitively, the CUDA path).  Nothing here
is imported by oracle/ or by the product package.  Each routine restates the paper's
definition in the most literal form available:

* bins_rational: P:196-197 (xf1 = F(h-1)/F_max * W, xf2 = F(h)/F_max * W) and P:226-229
  (project onto integer coordinates in [0, W-1], increase every overlapped bin), read as
  half-open overlap with the W-1 clamp for zero-width trailing cells (reading A14/A19).
* reduce_rational: P:229-233 (bin value += cell value, counter += 1, divide by counter).
"""
from fractions import Fraction
import math


def bins_rational(q, W):
    """Per cell: the set of bins it overlaps, from exact rational x positions."""
    Qtot = sum(q)
    out = []
    acc = 0
    for qi in q:
        x1 = Fraction(acc * W, Qtot)
        acc += qi
        x2 = Fraction(acc * W, Qtot)
        if x2 > x1:
            bins = [x for x in range(W) if min(x2, x + 1) - max(x1, x) > 0]
        else:  # zero-width cell: the pixel that contains its position (clamped to W-1)
            bins = [min(W - 1, math.floor(x1))]
        out.append((bins[0], bins[-1]))
        assert bins == list(range(bins[0], bins[-1] + 1))
    return out


def reduce_rational(t_cols, spans, W):
    """t_cols: list over members of per-cell fp32 t values (python floats).
    Returns per member per bin (count, min, max, exact mean Fraction)."""
    res = []
    for col in t_cols:
        per = []
        for x in range(W):
            cells = [h for h, (a, b) in enumerate(spans) if a <= x <= b]
            if not cells:
                per.append((0, None, None, None))
                continue
            vals = [col[h] for h in cells]
            mean = sum(Fraction(v) for v in vals) / len(vals)
            per.append((len(cells), min(vals), max(vals), mean))
        res.append(per)
    return res
