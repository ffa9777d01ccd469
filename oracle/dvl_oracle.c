/*
 * dvl_oracle.c -- plain, slow, single-threaded CPU ORACLE for the dynamic-volume-lines
 * (DVL / "interactive volume lines") hot path of arXiv 2306.11612.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load or call this file.  It shares no code,
 * header, table or constant generator with the CUDA library under
 * paper_2306_11612_b200/csrc/, and it never includes include/dvl.h.
 *
 * Citation convention: "P:n" is line n of the paper text; "S:n" is a line of
 * SPEC.md; "O#"/"A#" are the readings listed in DESIGN.md section 3 (taken from SURVEY.md
 * section 8(c)).  Every function below says which passage it restates.
 *
 * Compile: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared (no -ffast-math; x86-64 SSE
 * default rounding, no FTZ/DAZ) -- see oracle/oracle.py.
 *
 * Pins: every function here is pinned by tests/test_oracle_*.py against brute force,
 * closed forms or special cases.  "parity unpinned" items:
 * the bit pattern of detpow() for non-integer P (only the shared written recipe fixes it).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* status codes (the oracle's own numbering; tests map them by name) */
enum { OR_OK = 0, OR_E_INVAL = 1, OR_E_STATE = 2, OR_E_RANGE = 3, OR_E_OVERLAP = 4,
       OR_E_DEGENERATE = 5 };

/* ------------------------------------------------------------------------------------
 * Hilbert curve (reading A1/O3): Skilling (2004) "Programming the
 * Hilbert curve", AxestoTranspose / TransposetoAxes on n = 3 axes X = (x, y, z) with b
 * bits, restated loop for loop.  The index is the "transpose" read MSB-first,
 * X[0] bit, X[1] bit, X[2] bit per level (x most significant in each 3-bit digit).
 * ---------------------------------------------------------------------------------- */
static void axes_to_transpose(uint32_t X[3], int b)
{
    uint32_t M = 1u << (b - 1), P, Q, t;
    int i;
    /* inverse undo */
    for (Q = M; Q > 1; Q >>= 1) {
        P = Q - 1;
        for (i = 0; i < 3; i++) {
            if (X[i] & Q) {
                X[0] ^= P;                       /* invert */
            } else {
                t = (X[0] ^ X[i]) & P;           /* exchange */
                X[0] ^= t;
                X[i] ^= t;
            }
        }
    }
    /* Gray encode */
    for (i = 1; i < 3; i++) X[i] ^= X[i - 1];
    t = 0;
    for (Q = M; Q > 1; Q >>= 1)
        if (X[2] & Q) t ^= Q - 1;
    for (i = 0; i < 3; i++) X[i] ^= t;
}

static void transpose_to_axes(uint32_t X[3], int b)
{
    uint32_t N = 2u << (b - 1), P, Q, t;
    int i;
    /* Gray decode by H ^ (H/2) */
    t = X[2] >> 1;
    for (i = 2; i > 0; i--) X[i] ^= X[i - 1];
    X[0] ^= t;
    /* undo excess work */
    for (Q = 2; Q != N; Q <<= 1) {
        P = Q - 1;
        for (i = 2; i >= 0; i--) {
            if (X[i] & Q) {
                X[0] ^= P;
            } else {
                t = (X[0] ^ X[i]) & P;
                X[0] ^= t;
                X[i] ^= t;
            }
        }
    }
}

uint64_t or_hilbert_encode(uint32_t x, uint32_t y, uint32_t z, int b)
{
    uint32_t X[3] = {x, y, z};
    uint64_t h = 0;
    int j;
    axes_to_transpose(X, b);
    for (j = b - 1; j >= 0; j--) {
        h = (h << 3) | ((uint64_t)((X[0] >> j) & 1u) << 2) | ((uint64_t)((X[1] >> j) & 1u) << 1)
            | (uint64_t)((X[2] >> j) & 1u);
    }
    return h;
}

void or_hilbert_decode(uint64_t h, int b, uint32_t out[3])
{
    uint32_t X[3] = {0, 0, 0};
    int j;
    for (j = b - 1; j >= 0; j--) {
        uint32_t d = (uint32_t)((h >> (3 * j)) & 7u);
        X[0] |= ((d >> 2) & 1u) << j;
        X[1] |= ((d >> 1) & 1u) << j;
        X[2] |= (d & 1u) << j;
    }
    transpose_to_axes(X, b);
    out[0] = X[0]; out[1] = X[1]; out[2] = X[2];
}

void or_hilbert_encode_many(int64_t n, const uint32_t *xyz, int b, uint64_t *out)
{
    for (int64_t i = 0; i < n; i++)
        out[i] = or_hilbert_encode(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], b);
}

void or_hilbert_decode_many(int64_t n, const uint64_t *h, int b, uint32_t *xyz)
{
    for (int64_t i = 0; i < n; i++) or_hilbert_decode(h[i], b, xyz + 3 * i);
}

/* ------------------------------------------------------------------------------------
 * Build (P:76-82 logical grid, C_w = 2^L; P:107-111 centroid quantisation; P:309-311
 * fixed Hilbert order).  Readings O1-O5 / A2-A4 / A22.
 * ---------------------------------------------------------------------------------- */
typedef struct { uint64_t code; uint64_t id; } or_pair;

static int cmp_pair(const void *a, const void *b)
{
    const or_pair *p = (const or_pair *)a, *q = (const or_pair *)b;
    if (p->code != q->code) return p->code < q->code ? -1 : 1;
    if (p->id != q->id) return p->id < q->id ? -1 : 1;
    return 0;
}

/* O1: extent, bits, Lmax; validation of the logical-grid model. */
int or_extent(int64_t n, const uint32_t *lower, const uint8_t *level,
              uint32_t *E_out, int *b_out, int *Lmax_out)
{
    uint64_t E = 0;
    int Lmax = 0;
    if (n <= 0) return OR_E_INVAL;
    for (int64_t h = 0; h < n; h++) {
        int L = level[h];
        if (L > 20) return OR_E_INVAL;
        uint64_t w = 1ull << L;
        for (int k = 0; k < 3; k++) {
            uint64_t c = lower[3 * h + k];
            if (c % w != 0) return OR_E_INVAL;
            if (c + w > E) E = c + w;
        }
        if (L > Lmax) Lmax = L;
    }
    if (E > (1ull << 21)) return OR_E_RANGE;
    int b = 0;
    while ((1ull << b) < E) b++;           /* b = ceil(log2 E) */
    if (b < 1) b = 1;
    *E_out = (uint32_t)E;
    *b_out = b;
    *Lmax_out = Lmax;
    return OR_OK;
}

/* O2 + O3: centroid code of one cell: c = lower + (2^L >> 1) (floor of the centroid). */
uint64_t or_centroid_code(const uint32_t lower[3], int L, int b)
{
    uint32_t half = (1u << L) >> 1;
    return or_hilbert_encode(lower[0] + half, lower[1] + half, lower[2] + half, b);
}

/* O1-O5.  Outputs: codes[n] and perm[n] in curve order, level_s[n], scal_s[M*n]
 * (member-major), vmin/vmax[M] over finite values (all non-finite -> [0,0]),
 * info[3] = {E, b, Lmax}. */
int or_build(int64_t n, const uint32_t *lower, const uint8_t *level, int M,
             const float *scal /* M*n, member-major, input order */,
             uint64_t *codes, uint64_t *perm, uint8_t *level_s, float *scal_s,
             float *vmin, float *vmax, int32_t *info)
{
    uint32_t E;
    int b, Lmax;
    if (M < 1 || M > 64) return OR_E_INVAL;
    int st = or_extent(n, lower, level, &E, &b, &Lmax);
    if (st != OR_OK) return st;
    or_pair *pr = (or_pair *)malloc(sizeof(or_pair) * (size_t)n);
    if (!pr) return OR_E_INVAL;
    for (int64_t h = 0; h < n; h++) {
        pr[h].code = or_centroid_code(lower + 3 * h, level[h], b);
        pr[h].id = (uint64_t)h;
    }
    qsort(pr, (size_t)n, sizeof(or_pair), cmp_pair);
    /* O4: strictly increasing codes; consecutive dyadic code blocks disjoint. */
    for (int64_t k = 0; k + 1 < n; k++) {
        if (pr[k].code >= pr[k + 1].code) { free(pr); return OR_E_OVERLAP; }
        int La = level[pr[k].id], Lb = level[pr[k + 1].id];
        uint64_t lena = 1ull << (3 * La), lenb = 1ull << (3 * Lb);
        uint64_t sa = pr[k].code & ~(lena - 1), sb = pr[k + 1].code & ~(lenb - 1);
        if (sa + lena > sb) { free(pr); return OR_E_OVERLAP; }
    }
    for (int64_t k = 0; k < n; k++) {
        codes[k] = pr[k].code;
        perm[k] = pr[k].id;
        level_s[k] = level[pr[k].id];
    }
    for (int m = 0; m < M; m++) {
        float lo = 0.0f, hi = 0.0f;
        int any = 0;
        for (int64_t k = 0; k < n; k++) {
            float v = scal[(int64_t)m * n + (int64_t)pr[k].id];
            scal_s[(int64_t)m * n + k] = v;
            if (isfinite(v)) {
                if (!any) { lo = v; hi = v; any = 1; }
                else { if (v < lo) lo = v; if (v > hi) hi = v; }
            }
        }
        vmin[m] = lo;
        vmax[m] = hi;
    }
    info[0] = (int32_t)E; info[1] = b; info[2] = Lmax;
    free(pr);
    return OR_OK;
}

/* ------------------------------------------------------------------------------------
 * Transfer functions ("normalize the input (field) intensity and compute RGBa";
 * readings O6-O8 / A5-A7, A15).
 * ---------------------------------------------------------------------------------- */

/* O6: inverse width of a member's normalisation domain (fp32). */
float or_domain_inv(float lo, float hi)
{
    return hi > lo ? 1.0f / (hi - lo) : 0.0f;
}

/* O7: t = clamp((v - lo) * inv, 0, 1); NaN -> 0, +Inf -> 1 (two fp32 ops then clamps). */
float or_normalize(float v, float lo, float inv)
{
    float x = (v - lo) * inv;
    return x > 0.0f ? (x < 1.0f ? x : 1.0f) : 0.0f;
}

/* O8: piecewise-linear lookup of a table of N >= 2 entries at t in [0,1]. */
float or_sample(const float *A, int N, float t)
{
    float pos = t * (float)(N - 1);
    if (pos >= (float)(N - 1)) return A[N - 1];
    int i0 = (int)pos;
    float fr = pos - (float)i0;
    return fmaf(fr, A[i0 + 1] - A[i0], A[i0]);
}

/* data index range of one member: i = floor(t(vmin)(N-1)),
 * j = min(N-1, ceil(t(vmax)(N-1))). */
void or_index_range(float vmin, float vmax, float lo, float inv, int N, int32_t out[2])
{
    float tl = or_normalize(vmin, lo, inv), th = or_normalize(vmax, lo, inv);
    int i = (int)floorf(tl * (float)(N - 1));
    int j = (int)ceilf(th * (float)(N - 1));
    if (j > N - 1) j = N - 1;
    out[0] = i;
    out[1] = j;
}

/* O9: max(V_h) approximation from TFs and data ranges (eq:va).
 * mode 0 = R2 (global bound, default), mode 1 = R1 (per-entry).  alpha is M*N. */
float or_maxv_approx(int mode, int M, int N, const float *alpha, const float *vmin,
                     const float *vmax, const float *lo, const float *inv)
{
    int i = N - 1, j = 0;
    for (int m = 0; m < M; m++) {
        int32_t r[2];
        or_index_range(vmin[m], vmax[m], lo[m], inv[m], N, r);
        if (r[0] < i) i = r[0];
        if (r[1] > j) j = r[1];
    }
    if (i > j) return 0.0f;
    if (mode == 0) {
        float amax = alpha[i], amin = alpha[i];
        for (int m = 0; m < M; m++)
            for (int a = i; a <= j; a++) {
                float v = alpha[(int64_t)m * N + a];
                if (v > amax) amax = v;
                if (v < amin) amin = v;
            }
        return amax - amin;
    }
    float best = 0.0f;
    for (int a = i; a <= j; a++) {
        float amax = alpha[a], amin = alpha[a];
        for (int m = 1; m < M; m++) {
            float v = alpha[(int64_t)m * N + a];
            if (v > amax) amax = v;
            if (v < amin) amin = v;
        }
        if (amax - amin > best) best = amax - amin;
    }
    return best;
}

/* ------------------------------------------------------------------------------------
 * Importance (Eq. 1; Eq. 3; minimum importance P:138-139).
 * Readings O10 / A9-A11 / A29.
 * ---------------------------------------------------------------------------------- */

/* Eq. 1: V_h = max_m I(m,h) - min_m I(m,h), I = alpha of member m's TF at t_m (A5). */
float or_variation(int64_t h, int64_t n, int M, int N, const float *scal_s,
                   const float *alpha, const float *lo, const float *inv)
{
    float amax = 0.0f, amin = 0.0f;
    for (int m = 0; m < M; m++) {
        float t = or_normalize(scal_s[(int64_t)m * n + h], lo[m], inv[m]);
        float a = or_sample(alpha + (int64_t)m * N, N, t);
        if (m == 0) { amax = a; amin = a; }
        else { if (a > amax) amax = a; if (a < amin) amin = a; }
    }
    return amax - amin;
}

/* exact max_h V_h (mode 2). */
float or_maxv_exact(int64_t n, int M, int N, const float *scal_s, const float *alpha,
                    const float *lo, const float *inv)
{
    float best = 0.0f;
    for (int64_t h = 0; h < n; h++) {
        float v = or_variation(h, n, M, N, scal_s, alpha, lo, inv);
        if (v > best) best = v;
    }
    return best;
}

/* 2^k as an fp32 (exact for -149 <= k <= 127). */
static float pow2f(int k)
{
    union { uint32_t u; float f; } c;
    if (k >= -126) c.u = (uint32_t)(k + 127) << 23;
    else c.u = 1u << (k + 149);
    return c.f;
}

/* detpow(g, P) for non-integer P (O10 recipe, docs in DESIGN.md section 3): a fixed,
 * deterministic op sequence; accuracy is not the goal.  parity unpinned (bit pattern). */
static float log2_det(float g)
{
    int e;
    float m = frexpf(g, &e);
    if (m < 0x1.6a09e6p-1f) { m = m * 2.0f; e = e - 1; }
    float u = (m - 1.0f) / (m + 1.0f);
    float z = u * u;
    float p = 0x1.c71c72p-4f;              /* 1/9 */
    p = fmaf(p, z, 0x1.24924ap-3f);        /* 1/7 */
    p = fmaf(p, z, 0x1.99999ap-3f);        /* 1/5 */
    p = fmaf(p, z, 0x1.555556p-2f);        /* 1/3 */
    p = fmaf(p, z, 1.0f);                  /* 1/1 */
    float t1 = u * p;
    float t2 = t1 * 0x1.715476p+1f;        /* 2/ln 2 */
    return (float)e + t2;
}

static float exp2_det(float y)
{
    float k = floorf(y);
    float fr = y - k;
    float w = fr * 0x1.62e430p-1f;         /* ln 2 */
    float p = 0x1.a01a02p-16f;             /* 1/8! */
    p = fmaf(p, w, 0x1.a01a02p-13f);       /* 1/7! */
    p = fmaf(p, w, 0x1.6c16c2p-10f);       /* 1/6! */
    p = fmaf(p, w, 0x1.111112p-7f);        /* 1/5! */
    p = fmaf(p, w, 0x1.555556p-5f);        /* 1/4! */
    p = fmaf(p, w, 0x1.555556p-3f);        /* 1/3! */
    p = fmaf(p, w, 0.5f);                  /* 1/2! */
    p = fmaf(p, w, 1.0f);                  /* 1/1! */
    p = fmaf(p, w, 1.0f);                  /* 1/0! */
    if (k < -149.0f) return 0.0f;
    if (k > 127.0f) return INFINITY;
    return p * pow2f((int)k);
}

float or_detpow(float g, float P)
{
    if (g == 0.0f) return 0.0f;
    float y = P * log2_det(g);
    return exp2_det(y);
}

/* g^P: P = 0 -> 1; P = 1 -> g; integer P in [2,8] -> left-to-right repeated product;
 * otherwise detpow (O10). */
float or_powP(float g, float P)
{
    if (P == 0.0f) return 1.0f;
    if (P == 1.0f) return g;
    if (P == floorf(P) && P >= 2.0f && P <= 8.0f) {
        int ip = (int)P;
        float f = g;
        for (int k = 1; k < ip; k++) f = f * g;
        return f;
    }
    return or_detpow(g, P);
}

/* Eq. 3 with the minimum importance (A9: clamp the ratio before 2^L and ^P):
 * r = maxV > 0 ? V/maxV : 0; r = min(max(r, eps), 1); f = (r * 2^L)^P. */
float or_importance(float V, float maxV, int L, float P, float eps)
{
    float r = maxV > 0.0f ? V / maxV : 0.0f;
    r = r > eps ? r : eps;
    r = r < 1.0f ? r : 1.0f;
    float g = r * pow2f(L);
    return or_powP(g, P);
}

/* O11: fixed-point shift s = 61 - ceil(log2 n) - ceil(Lmax * P). */
int or_shift(int64_t n_global, int Lmax, float P)
{
    int cl = 0;
    while (cl < 63 && (1ll << cl) < n_global) cl++;
    int cp = (int)ceil((double)Lmax * (double)P);
    return 61 - cl - cp;
}

/* O11: q = trunc(f * 2^s) as u64. */
uint64_t or_fixed(float f, int s)
{
    float x = f * pow2f(s);
    return (uint64_t)x;
}

/* weights of every sorted cell: f[n] (fp32) and q[n] (u64). */
void or_weights(int64_t n, int M, int N, const uint8_t *level_s, const float *scal_s,
                const float *alpha, const float *lo, const float *inv, float maxV,
                float P, float eps, int s, float *f_out, uint64_t *q_out)
{
    for (int64_t h = 0; h < n; h++) {
        float V = or_variation(h, n, M, N, scal_s, alpha, lo, inv);
        float f = or_importance(V, maxV, level_s[h], P, eps);
        if (f_out) f_out[h] = f;
        q_out[h] = or_fixed(f, s);
    }
}

/* Eq. 4: inclusive prefix sum Q(h) = sum_{i<=h} q(i) in u64 (O12, A12-A13). */
uint64_t or_prefix(int64_t n, const uint64_t *q, uint64_t *Q)
{
    uint64_t acc = 0;
    for (int64_t h = 0; h < n; h++) {
        acc += q[h];
        Q[h] = acc;
    }
    return acc;
}

/* O13 (A14): projection of (xf1, xf2) = (E W/Qtot, Q W/Qtot) onto bins:
 * b1 = min(W-1, floor(E W / Qtot)); b2 = min(W-1, max(b1, ceil(Q W / Qtot) - 1)). */
void or_bins_ext(int64_t n, const uint64_t *Q, uint64_t E0, uint64_t Qtot, uint32_t W,
                 int32_t *b1, int32_t *b2);

void or_bins(int64_t n, const uint64_t *Q, uint32_t W, int32_t *b1, int32_t *b2)
{
    or_bins_ext(n, Q, 0, Q[n - 1], W, b1, b2);
}

/* the same for a contiguous piece of the cells: E of its first cell is E0, the total of
 * all cells Qtot (a shard of the curve order). */
void or_bins_ext(int64_t n, const uint64_t *Q, uint64_t E0, uint64_t Qtot, uint32_t W,
                 int32_t *b1, int32_t *b2)
{
    for (int64_t h = 0; h < n; h++) {
        unsigned __int128 E = h ? Q[h - 1] : E0;
        unsigned __int128 q = Q[h];
        unsigned __int128 x1 = (E * W) / Qtot;
        int64_t a = (int64_t)(x1 > (unsigned __int128)(W - 1) ? (W - 1) : x1);
        unsigned __int128 num = q * W;
        int64_t c = (int64_t)((num + Qtot - 1) / Qtot) - 1;   /* ceil(Q W/Qtot) - 1 */
        int64_t bb = c > a ? c : a;
        if (bb > (int64_t)W - 1) bb = (int64_t)W - 1;
        b1[h] = (int32_t)a;
        b2[h] = (int32_t)bb;
    }
}

/* vertex record (the oracle's own definition; same field order as the ABI's dvl_vertex
 * by specification, written independently). */
typedef struct { float t_min, t_max, t_mean, y, r, g, b; uint32_t count; } or_vertex;

/* O14-O15 (P:226-233 box basis, counters, divide by the counter; P:250-256 TF applied
 * per bin after the division; A15-A18): for every cell h and every bin x in
 * [b1(h), b2(h)], add t_m(h) to bin x of member m and increment its counter; then
 * mean = sum / count (double), y = alpha_m(mean), rgb = RGB_m(mean).
 * rgba is M*N*4 (member-major, entry-major, channel-minor).  out is M*W (member-major).
 * lo_out/hi_out (optional, W entries): first and last cell index of each bin. */
void or_reduce(int64_t n, int M, int N, const float *scal_s, const float *rgba,
               const float *lo, const float *inv, uint32_t W, const int32_t *b1,
               const int32_t *b2, or_vertex *out, uint64_t *lo_out, uint64_t *hi_out)
{
    double *sum = (double *)calloc((size_t)M * W, sizeof(double));
    float *mn = (float *)malloc(sizeof(float) * (size_t)M * W);
    float *mx = (float *)malloc(sizeof(float) * (size_t)M * W);
    uint32_t *cnt = (uint32_t *)calloc(W, sizeof(uint32_t));
    int64_t *first = (int64_t *)malloc(sizeof(int64_t) * W);
    int64_t *last = (int64_t *)malloc(sizeof(int64_t) * W);
    float *A = (float *)malloc(sizeof(float) * (size_t)N);
    for (uint32_t x = 0; x < W; x++) { first[x] = -1; last[x] = -1; }
    for (int64_t h = 0; h < n; h++) {
        for (int32_t x = b1[h]; x <= b2[h]; x++) {
            for (int m = 0; m < M; m++) {
                float t = or_normalize(scal_s[(int64_t)m * n + h], lo[m], inv[m]);
                int64_t k = (int64_t)m * W + x;
                if (cnt[x] == 0) { mn[k] = t; mx[k] = t; }
                else { if (t < mn[k]) mn[k] = t; if (t > mx[k]) mx[k] = t; }
                sum[k] += (double)t;
            }
            if (first[x] < 0) first[x] = h;
            last[x] = h;
            cnt[x] += 1;
        }
    }
    for (int m = 0; m < M; m++) {
        const float *tf = rgba + (int64_t)m * N * 4;
        for (uint32_t x = 0; x < W; x++) {
            int64_t k = (int64_t)m * W + x;
            or_vertex v;
            memset(&v, 0, sizeof v);
            v.count = cnt[x];
            if (cnt[x] > 0) {
                float mean = (float)(sum[k] / (double)cnt[x]);
                v.t_min = mn[k];
                v.t_max = mx[k];
                v.t_mean = mean;
                float rgbay[4];
                for (int c = 0; c < 4; c++) {
                    for (int a = 0; a < N; a++) A[a] = tf[a * 4 + c];
                    rgbay[c] = or_sample(A, N, mean);
                }
                v.r = rgbay[0]; v.g = rgbay[1]; v.b = rgbay[2]; v.y = rgbay[3];
            }
            out[k] = v;
        }
    }
    if (lo_out)
        for (uint32_t x = 0; x < W; x++) lo_out[x] = (uint64_t)first[x];
    if (hi_out)
        for (uint32_t x = 0; x < W; x++) hi_out[x] = (uint64_t)last[x];
    free(sum); free(mn); free(mx); free(cnt); free(first); free(last); free(A);
}
