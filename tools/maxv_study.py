"""The paper's max(V_h) accuracy experiment: over 107
random TF configurations (every member's TF drawn from the S:535 distribution), the
approximate normalisers -- R2 "conservative" (range of alpha over the members' value windows,
the default) and R1 "per entry" -- against the exact max over all cells of V_h, and what the
approximation does to the polylines (vertex counts, bin ranges and heights compared with the
exact-normaliser run).  Runs through the library on the GPU.

The paper's own numbers for this study are not recoverable from PAPER.md (the
study is unpinned), so this prints the measured distribution; it is not a parity test.

usage: python tools/maxv_study.py [config] [n_configs] > profiles/maxv_study.md
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_11612_b200 as dvl  # noqa: E402
import synth  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C1"
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 107
    cfg = synth.make_config(name)
    M, W = cfg["M"], cfg["W"]
    dvl.load()
    ctxs = {}
    for mode in ("exact", "conservative", "per_entry"):
        c = dvl.Context(device=0)
        c.build(cfg["lower"], cfg["level"], cfg["scal"])
        if cfg["domain"] is not None:
            for m in range(M):
                c.set_domain(m, float(cfg["domain"][m, 0]), float(cfg["domain"][m, 1]))
        c.set_params(1.0, 0.025, mode)
        ctxs[mode] = c
    rows = []
    for k in range(K):
        tfs = [synth.random_tf(50000 + 97 * k + m, 256, member=m) for m in range(M)]
        out = {}
        for mode, c in ctxs.items():
            for m in range(M):
                c.update_tf(m, tfs[m])
            out[mode] = (c.info()["maxV"], c.get_polylines(W), c.get_bin_ranges(W))
        ex_v, ex_p, ex_r = out["exact"]
        row = [ex_v]
        for mode in ("conservative", "per_entry"):
            v, pl, rg = out[mode]
            same_bins = bool(np.array_equal(rg[0], ex_r[0]) and np.array_equal(rg[1], ex_r[1]))
            dy = float(np.max(np.abs(pl["y"].astype(np.float64) - ex_p["y"]))) if ex_v > 0 else 0.0
            row += [v / ex_v if ex_v > 0 else float("nan"), same_bins,
                    int(np.sum(pl["count"] != ex_p["count"])), dy]
        rows.append(row)
    r = np.array(rows, dtype=object)
    print(f"# max(V_h) study: {K} random TF configurations, {name} (n = {len(cfg['level'])}, M = {M}, W = {W})\n")
    print("Normaliser ratio approx / exact (R2 must be >= 1 up to rounding: it bounds V_h),")
    print("and the effect on the polylines relative to the exact normaliser.\n")
    print("| normaliser | ratio min | ratio median | ratio max | configs with identical bins | "
          "mean #vertices with another count | max abs diff of the height y |")
    print("|---|---|---|---|---|---|---|")
    for j, mode in enumerate(("conservative (R2)", "per entry (R1)")):
        ratio = np.array([x for x in r[:, 1 + 4 * j] if x == x], dtype=float)
        same = np.array(r[:, 2 + 4 * j], dtype=bool)
        cnt = np.array(r[:, 3 + 4 * j], dtype=float)
        dy = np.array(r[:, 4 + 4 * j], dtype=float)
        print(f"| {mode} | {ratio.min():.4f} | {np.median(ratio):.4f} | {ratio.max():.4f} | "
              f"{int(same.sum())} / {K} | {cnt.mean():.1f} | {dy.max():.3g} |")
    print("\nThe height y is the TF alpha at the bin mean (the normaliser changes only the bins, "
          "through the weights), so y differences come from bins that moved.")
    for c in ctxs.values():
        c.close()


if __name__ == "__main__":
    main()
