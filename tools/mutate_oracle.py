"""Mutation check of the oracle's pins: applies one plausible mistake at a time to
oracle/dvl_oracle.c (a dropped term, a wrong sign / index / operand order), recompiles,
runs the CPU pin suite (-m "not gpu", oracle + golden tests) and records whether some pin
fails.  The source is restored afterwards.  Results: profiles/oracle_mutations.md.

Run: python tools/mutate_oracle.py
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "dvl_oracle.c")

MUTATIONS = [
    ("maxV ignores the data index range [i, j] (P:272-278)",
     "    if (i > j) return 0.0f;\n    if (mode == 0) {",
     "    i = 0; j = N - 1;\n    if (i > j) return 0.0f;\n    if (mode == 0) {"),
    ("maxV: [i, j] from the first member only",
     "        if (r[0] < i) i = r[0];\n        if (r[1] > j) j = r[1];",
     "        if (m == 0) { i = r[0]; j = r[1]; }"),
    ("index range: j = floor instead of ceil",
     "int j = (int)ceilf(th * (float)(N - 1));", "int j = (int)floorf(th * (float)(N - 1));"),
    ("R1 instead of R2 as mode 0", "    if (mode == 0) {", "    if (mode == 7) {"),
    ("epilogue: g and b channels swapped",
     "v.g = rgbay[1]; v.b = rgbay[2];", "v.g = rgbay[2]; v.b = rgbay[1];"),
    ("epilogue: y from the red channel", "v.y = rgbay[3];", "v.y = rgbay[0];"),
    ("Eq. 1: V = max only (min dropped)", "    return amax - amin;\n}\n\n/* exact",
     "    return amax;\n}\n\n/* exact"),
    ("Eq. 3: level scale dropped", "    float g = r * pow2f(L);", "    float g = r;"),
    ("Eq. 3: min importance applied after the level scale",
     "    r = r > eps ? r : eps;\n    r = r < 1.0f ? r : 1.0f;\n    float g = r * pow2f(L);",
     "    r = r < 1.0f ? r : 1.0f;\n    float g = r * pow2f(L);\n    g = g > eps ? g : eps;"),
    ("Eq. 4: exclusive prefix instead of inclusive", "        acc += q[h];\n        Q[h] = acc;",
     "        Q[h] = acc;\n        acc += q[h];"),
    ("bins: b2 without the -1", "/ Qtot) - 1;   /* ceil", "/ Qtot);   /* ceil"),
    ("bins: no W-1 clamp of b1", "x1 > (unsigned __int128)(W - 1) ? (W - 1) : x1",
     "x1"),
    ("shift: ceil(Lmax P) dropped", "    return 61 - cl - cp;", "    return 61 - cl;"),
    ("centroid: lower corner instead of centroid", "    uint32_t half = (1u << L) >> 1;",
     "    uint32_t half = 0;"),
    ("Hilbert: interleave y-major", "((uint64_t)((X[0] >> j) & 1u) << 2) | ((uint64_t)((X[1] >> j) & 1u) << 1)",
     "((uint64_t)((X[1] >> j) & 1u) << 2) | ((uint64_t)((X[0] >> j) & 1u) << 1)"),
    ("Hilbert: Gray-encode loop skipped", "    for (i = 1; i < 3; i++) X[i] ^= X[i - 1];", ""),
    ("overlap check: block length 8^L -> 4^L", "lena = 1ull << (3 * La)", "lena = 1ull << (2 * La)"),
    ("reduce: min/max over t of the next member", "float t = or_normalize(scal_s[(int64_t)m * n + h], lo[m], inv[m]);\n                int64_t k",
     "float t = or_normalize(scal_s[(int64_t)((m + 1) % M) * n + h], lo[m], inv[m]);\n                int64_t k"),
    ("sample: fraction from the upper knot", "return fmaf(fr, A[i0 + 1] - A[i0], A[i0]);",
     "return fmaf(fr, A[i0 + 1] - A[i0], A[i0 + 1]);"),
    ("normalize: NaN -> 1", "return x > 0.0f ? (x < 1.0f ? x : 1.0f) : 0.0f;",
     "return x <= 0.0f ? 0.0f : (x < 1.0f ? x : 1.0f);"),
]


def run(py=sys.executable):
    tests = ["tests/test_oracle_hilbert.py", "tests/test_oracle_build.py", "tests/test_oracle_update.py",
             "tests/test_oracle_volume.py", "tests/test_oracle_locate.py", "tests/test_golden.py"]
    r = subprocess.run([py, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", "-m", "not gpu"] + tests,
                       cwd=ROOT, capture_output=True, text=True)
    last = [l for l in r.stdout.splitlines() if l.strip()][-1]
    failed = [l.split(" ")[1] for l in r.stdout.splitlines() if l.startswith("FAILED")]
    return r.returncode, last, failed[:1]


def main():
    backup = SRC + ".orig"
    shutil.copyfile(SRC, backup)
    rows = []
    try:
        for name, a, b in MUTATIONS:
            s = open(backup).read()
            assert s.count(a) == 1, name
            open(SRC, "w").write(s.replace(a, b))
            sys.path.insert(0, ROOT)
            from oracle.oracle import compile_oracle
            compile_oracle(force=True)
            rc, last, failed = run()
            killed = rc != 0
            rows.append((name, killed, failed[0] if failed else last))
            print(("KILLED  " if killed else "SURVIVED") + "  " + name + "  " + (failed[0] if failed else last),
                  flush=True)
    finally:
        shutil.copyfile(backup, SRC)
        os.remove(backup)
        from oracle.oracle import compile_oracle
        compile_oracle(force=True)
    rc, last, _ = run()
    print("unmutated:", last)
    out = os.path.join(ROOT, "profiles", "oracle_mutations.md")
    with open(out, "w") as f:
        f.write("# Oracle mutation check (`python tools/mutate_oracle.py`)\n\n")
        f.write("Each row applies one plausible mistake to `oracle/dvl_oracle.c`, recompiles and runs the "
                "CPU pin suite (oracle + golden tests).  KILLED = some pin fails.\n\n")
        f.write("| Mutation | Result | First failing pin |\n|---|---|---|\n")
        for name, killed, why in rows:
            f.write(f"| {name} | {'KILLED' if killed else 'SURVIVED'} | `{why}` |\n")
        f.write(f"\nUnmutated suite: {last}\n")
    return 0 if all(k for _, k, _ in rows) else 1


if __name__ == "__main__":
    sys.exit(main())
