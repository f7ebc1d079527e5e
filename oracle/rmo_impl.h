/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path
 * (p-FHT-FSCL-L-M, arXiv 2108.12550) used as the parity checker and as the
 * "port" CPU baseline.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product path
 * (paper_2108_12550_b200) never calls into this file.
 *
 * This header is the body; rmfht_oracle.c includes it twice, with
 * REAL=double (SFX=_f64: bit-exact restatement of the float64 reference) and
 * REAL=float (SFX=_f32: the same operation order in float32, which is the
 * arithmetic of the GPU's fp32 kernel).
 *
 * Every function cites the reference line it restates; paths are relative to
 * /root/reference/pkg/src/rmworkbench/.
 */

#define CAT_(a, b) a##b
#define CAT(a, b) CAT_(a, b)
#define FN(name) CAT(name, SFX)

typedef struct {
    int r, m, N, L, perms, tie_fix;
    int v2;  /* RMO_ORDER_V2: the float32 throughput kernel's summation orders */
    const rmo_map *maps; /* this attempt's maps, in consumption order */
    int nmaps, next_map;
    int perm_active;        /* top_decoders.py:62,77-78 */
    rmo_arena *ar;
    double margin;          /* instrumentation: min relative selection gap */
    const REAL *root_llr;   /* channel LLRs (for the root tie-fix key) */
    const rmo_map *init[RMO_MAXL]; /* root maps per root lineage */
} FN(rmo_ctx);

/* numpy pairwise summation order (numpy/_core/src/umath/loops_utils.h.src,
 * pairwise_sum), which is what np.sum(x, axis=1) uses for the contiguous
 * rows at fht_decode.py:114 and automorphism.py:233.  Verified bit-exact
 * against numpy 2.3.5 by tests/test_oracle_pins.py. */
static REAL FN(pw_sum)(const REAL *a, long n)
{
    if (n < 8) {
        REAL res = 0;
        for (long i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        REAL r[8];
        long i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        REAL res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        long n2 = n / 2;
        n2 -= n2 % 8;
        return FN(pw_sum)(a, n2) + FN(pw_sum)(a + n2, n - n2);
    }
}

static inline void FN(note)(FN(rmo_ctx) *cx, double a, double b)
{
    double g = rmo_rel_gap(a, b);
    if (g < cx->margin) cx->margin = g;
}

/* RMO_ORDER_V2 sum of |x| over a node of size n held by a lane group of lpp
 * lanes (element e = k*lpp + u): per-lane partials in slot order, then the
 * group tree with offsets 1, 2, 4, ... (rmfht_fast.cuh, fht_node). */
static REAL FN(v2_group_sum)(const REAL *a, int n, int lpp)
{
    REAL q[32];
    int act = n >= lpp ? lpp : n, V = n >= lpp ? n / lpp : 1;
    for (int u = 0; u < act; u++) {
        q[u] = a[u];
        for (int k = 1; k < V; k++) q[u] += a[k * lpp + u];
    }
    for (int off = 1; off < act; off <<= 1) {
        REAL t[32];
        for (int u = 0; u < act; u++) t[u] = q[u] + q[u ^ off];
        for (int u = 0; u < act; u++) q[u] = t[u];
    }
    return q[0];
}

/* RMO_ORDER_V2 32-lane tree (offsets 16, 8, 4, 2, 1), rmfht_fast.cuh multi_tree */
static REAL FN(v2_lane_tree)(REAL *v)
{
    for (int off = 16; off >= 1; off >>= 1) {
        REAL t[32];
        for (int l = 0; l < 32; l++) t[l] = v[l] + v[l ^ off];
        for (int l = 0; l < 32; l++) v[l] = t[l];
    }
    return v[0];
}

/* RMO_ORDER_V2 LM at the root: pairs (i, i^d) of channel indices, lane l
 * owning i = l + 32 s (rmfht_fast.cuh, lm_partial_root). */
static REAL FN(v2_lm_root)(const REAL *alpha, int N, unsigned d)
{
    REAL v[32];
    int NS = N / 32;
    unsigned c = d >> 5, delta = d & 31;
    for (int l = 0; l < 32; l++) {
        REAL acc = 0;
        int first = 1;
        if (c != 0) {
            int hb = rmo_hibit(c);
            for (int s = 0; s < NS; s++) {
                if (s >> hb & 1) continue;
                unsigned i = (unsigned)(l + 32 * s);
                REAL x = alpha[i] < 0 ? -alpha[i] : alpha[i], y = alpha[i ^ d] < 0 ? -alpha[i ^ d] : alpha[i ^ d];
                REAL mn = y < x ? y : x;
                acc = first ? mn : acc + mn;
                first = 0;
            }
        } else {
            int h = rmo_hibit(delta);
            if (!((l >> h) & 1))
                for (int s = 0; s < NS; s++) {
                    unsigned i = (unsigned)(l + 32 * s);
                    REAL x = alpha[i] < 0 ? -alpha[i] : alpha[i], y = alpha[i ^ d] < 0 ? -alpha[i ^ d] : alpha[i ^ d];
                    REAL mn = y < x ? y : x;
                    acc = first ? mn : acc + mn;
                    first = 0;
                }
        }
        v[l] = acc;
    }
    return FN(v2_lane_tree)(v);
}

/* RMO_ORDER_V2 LM at an inner permutation node: canonical pairs q = l + 32 r,
 * i = q with a zero inserted at the top bit of d (perm_ext_inner2). */
static REAL FN(v2_lm_inner)(const REAL *x, int n, unsigned d)
{
    REAL v[32];
    int H = n / 2, h = rmo_hibit(d);
    for (int l = 0; l < 32; l++) {
        REAL acc = 0;
        int r = 0;
        for (int q = l; q < H; q += 32, r++) {
            int i = ((q >> h) << (h + 1)) | (q & ((1 << h) - 1));
            REAL a = x[i] < 0 ? -x[i] : x[i], b = x[i ^ (int)d] < 0 ? -x[i ^ (int)d] : x[i ^ (int)d];
            REAL mn = b < a ? b : a;
            acc = r == 0 ? mn : acc + mn;
        }
        v[l] = acc;
    }
    return FN(v2_lane_tree)(v);
}

/* f_op, list_engine.py:15-20: min(|a|,|b|) * sgn(a) * sgn(b), sgn(0)=+1 */
static inline REAL FN(f_op)(REAL a, REAL b)
{
    REAL x = a < 0 ? -a : a, y = b < 0 ? -b : b;
    REAL mn = y < x ? y : x;
    return ((a < 0) != (b < 0)) ? -mn : mn;
}

/* g_op, list_engine.py:23-27: b + (1-2c)*a; (1-2c)*a is exactly +-a */
static inline REAL FN(g_op)(REAL a, REAL b, int c) { return c ? b - a : b + a; }

/* fht_transform, fht_decode.py:28-48: stage t has half = 2^(s-t-1);
 * lo' = hi - lo, hi' = hi + lo. */
static void FN(fht)(REAL *w, int n)
{
    for (int half = n >> 1; half >= 1; half >>= 1)
        for (int blk = 0; blk < n; blk += 2 * half)
            for (int x = 0; x < half; x++) {
                REAL lo = w[blk + x], hi = w[blk + half + x];
                w[blk + x] = hi - lo;
                w[blk + half + x] = hi + lo;
            }
}

/* fhtl, fht_decode.py:101-126.  Returns the surviving path count. */
static int FN(fhtl)(FN(rmo_ctx) *cx, const REAL *alphas, int p, int n, REAL *pms,
                    uint8_t *beta, int *lin)
{
    int L = cx->L, k = n < L ? n : L;
    size_t mark = cx->ar->top;
    REAL *w = (REAL *)rmo_alloc(cx->ar, sizeof(REAL) * (size_t)p * n);
    REAL *absw = (REAL *)rmo_alloc(cx->ar, sizeof(REAL) * (size_t)p * n);
    REAL *tmp = (REAL *)rmo_alloc(cx->ar, sizeof(REAL) * (size_t)n);
    int *bins = (int *)rmo_alloc(cx->ar, sizeof(int) * (size_t)p * k);
    REAL *pool_pm = (REAL *)rmo_alloc(cx->ar, sizeof(REAL) * (size_t)p * k);
    int *order = (int *)rmo_alloc(cx->ar, sizeof(int) * (size_t)p * k);
    uint8_t *taken = (uint8_t *)rmo_alloc(cx->ar, (size_t)n);
    for (int row = 0; row < p; row++) {
        const REAL *a = alphas + (size_t)row * n;
        REAL *wr = w + (size_t)row * n, *ar = absw + (size_t)row * n;
        for (int j = 0; j < n; j++) { wr[j] = a[j]; tmp[j] = a[j] < 0 ? -a[j] : a[j]; }
        REAL llr_abs = cx->v2 ? FN(v2_group_sum)(tmp, n, 32 / L) : FN(pw_sum)(tmp, n); /* :114 */
        FN(fht)(wr, n);                                     /* :112 */
        for (int j = 0; j < n; j++) ar[j] = wr[j] < 0 ? -wr[j] : wr[j];
        /* stable argsort of -|w| → |w| descending, ties to the lower bin (:116) */
        memset(taken, 0, (size_t)n);
        for (int i = 0; i < k; i++) {
            int best = -1;
            for (int j = 0; j < n; j++)
                if (!taken[j] && (best < 0 || ar[j] > ar[best])) best = j;
            taken[best] = 1;
            bins[row * k + i] = best;
            /* :119 pm_pool = pms[rows] + 0.5 * (llr_abs[rows] - absw[rows, bins]) */
            pool_pm[row * k + i] = pms[row] + (REAL)0.5 * (llr_abs - ar[best]);
        }
        if (k < n) { /* instrumentation: the per-path top-k cut */
            int nxt = -1;
            for (int j = 0; j < n; j++)
                if (!taken[j] && (nxt < 0 || ar[j] > ar[nxt])) nxt = j;
            FN(note)(cx, ar[bins[row * k + k - 1]], ar[nxt]);
        }
    }
    /* :120 lexsort((bins, rows, pm_pool)) — pm, then source row, then bin */
    int P = p * k;
    for (int e = 0; e < P; e++) order[e] = e;
    for (int i = 1; i < P; i++) { /* insertion sort on the composite key */
        int e = order[i], j = i - 1;
        while (j >= 0) {
            int o = order[j];
            int before = pool_pm[e] < pool_pm[o] ||
                         (pool_pm[e] == pool_pm[o] &&
                          (e / k < o / k || (e / k == o / k && bins[e] < bins[o])));
            if (!before) break;
            order[j + 1] = o;
            j--;
        }
        order[j + 1] = e;
    }
    int q = P < L ? P : L;
    if (P > L) FN(note)(cx, pool_pm[order[L - 1]], pool_pm[order[L]]);
    REAL newpm[RMO_MAXL];
    for (int o = 0; o < q; o++) {
        int e = order[o], src = e / k, b = bins[e];
        int sign = w[(size_t)src * n + b] < 0;              /* :123 */
        uint8_t *out = beta + (size_t)o * n;
        for (int j = 0; j < n; j++)                         /* _bin_codewords :58-62 */
            out[j] = (uint8_t)(rmo_parity((unsigned)(~(b | j)) & (unsigned)(n - 1)) ^ sign);
        newpm[o] = pool_pm[e];
        lin[o] = src;
    }
    for (int o = 0; o < q; o++) pms[o] = newpm[o];
    cx->ar->top = mark;
    return q;
}

/* spc_decode_list, list_engine.py:68-119. */
static int FN(spc)(FN(rmo_ctx) *cx, const REAL *alphas, int p, int n, REAL *pms,
                   uint8_t *beta, int *lin)
{
    int L = cx->L;
    size_t mark = cx->ar->top;
    REAL *mag = (REAL *)rmo_alloc(cx->ar, sizeof(REAL) * (size_t)p * n);
    int *ord = (int *)rmo_alloc(cx->ar, sizeof(int) * (size_t)p * n);
    uint8_t *sgn = (uint8_t *)rmo_alloc(cx->ar, (size_t)p * n);
    uint8_t *flips = (uint8_t *)rmo_alloc(cx->ar, (size_t)L * n);
    uint8_t *flips2 = (uint8_t *)rmo_alloc(cx->ar, (size_t)L * n);
    int parity[RMO_MAXL];
    REAL pm[2 * RMO_MAXL], par[2 * RMO_MAXL];
    int parent[2 * RMO_MAXL];
    for (int row = 0; row < p; row++) {
        const REAL *a = alphas + (size_t)row * n;
        REAL *mg = mag + (size_t)row * n;
        int *od = ord + (size_t)row * n, pr = 0;
        REAL amax = 0;
        for (int j = 0; j < n; j++) {
            mg[j] = a[j] < 0 ? -a[j] : a[j];
            sgn[(size_t)row * n + j] = a[j] < 0;           /* hard_decision :39-40 */
            pr ^= a[j] < 0;
            if (mg[j] > amax) amax = mg[j];
        }
        /* :83 stable argsort of |alpha| ascending (insertion sort is stable) */
        for (int j = 0; j < n; j++) {
            int i = j - 1;
            while (i >= 0 && mg[od[i]] > mg[j]) { od[i + 1] = od[i]; i--; }
            od[i + 1] = j;
        }
        parity[row] = pr;
        /* :88 pms + where(parity == 1, a_min, 0.0) */
        pm[row] = pms[row] + (pr ? mg[od[0]] : (REAL)0);
        par[row] = (REAL)pr;
        parent[row] = row;
        /* instrumentation: the sorted prefix that drives the splits and the
         * sign decision of the least reliable position */
        int tau0 = n < L ? n : L;
        if (tau0 > n - 1) tau0 = n - 1;
        for (int j = 0; j < tau0 + 1 && j + 1 < n; j++) FN(note)(cx, mg[od[j]], mg[od[j + 1]]);
        if (amax > 0) {
            double g = (double)mg[od[0]] / (double)amax;
            if (g < cx->margin) cx->margin = g;
        }
    }
    memset(flips, 0, (size_t)L * n);
    int tau = n < L ? n : L;
    if (tau > n - 1) tau = n - 1;                          /* :91-92 */
    int P = p;
    for (int j = 1; j <= tau; j++) {                       /* :97-112 */
        REAL cand[2 * RMO_MAXL];
        for (int i = 0; i < P; i++) {
            const REAL *mg = mag + (size_t)parent[i] * n;
            const int *od = ord + (size_t)parent[i] * n;
            REAL a_j = mg[od[j]], a_m = mg[od[0]];
            cand[2 * i] = pm[i];
            /* pms + a_j + (1 - 2 par) * a_m; the product is exactly +-a_m */
            REAL t = pm[i] + a_j;
            cand[2 * i + 1] = par[i] != 0 ? t - a_m : t + a_m;
        }
        int C = 2 * P, sel[2 * RMO_MAXL];
        for (int c = 0; c < C; c++) sel[c] = c;
        for (int i = 1; i < C; i++) { /* stable argsort */
            int e = sel[i], t = i - 1;
            while (t >= 0 && cand[sel[t]] > cand[e]) { sel[t + 1] = sel[t]; t--; }
            sel[t + 1] = e;
        }
        int K = C < L ? C : L;
        if (C > L) FN(note)(cx, cand[sel[L - 1]], cand[sel[L]]);
        REAL npm[2 * RMO_MAXL], npar[2 * RMO_MAXL];
        int npar_ent[2 * RMO_MAXL];
        for (int o = 0; o < K; o++) {
            int which = sel[o] % 2, src = sel[o] / 2;
            npm[o] = cand[sel[o]];
            memcpy(flips2 + (size_t)o * n, flips + (size_t)src * n, (size_t)n);
            if (which) flips2[(size_t)o * n + ord[(size_t)parent[src] * n + j]] ^= 1;
            npar[o] = which ? (REAL)1 - par[src] : par[src];
            npar_ent[o] = parent[src];
        }
        memcpy(flips, flips2, (size_t)K * n);
        for (int o = 0; o < K; o++) { pm[o] = npm[o]; par[o] = npar[o]; parent[o] = npar_ent[o]; }
        P = K;
    }
    for (int o = 0; o < P; o++) {                          /* :114-118 */
        uint8_t *out = beta + (size_t)o * n;
        int tot = 0;
        for (int j = 0; j < n; j++) {
            out[j] = sgn[(size_t)parent[o] * n + j] ^ flips[(size_t)o * n + j];
            tot ^= out[j];
        }
        out[ord[(size_t)parent[o] * n]] ^= (uint8_t)tot;
        pms[o] = pm[o];
        lin[o] = parent[o];
    }
    (void)parity;
    cx->ar->top = mark;
    return P;
}

/* permutation_extend, automorphism.py:207-237 (Alg. 2 lines 6-12). */
static int FN(perm_extend)(FN(rmo_ctx) *cx, const REAL *alphas, int p, int n, int is_root,
                           REAL *pms, REAL *out, int *parent, const rmo_map **chosen)
{
    int L = cx->L, trials = 2 * p, half = n >> 1;
    if (cx->next_map + trials > cx->nmaps) return -1;
    const rmo_map *mp = cx->maps + cx->next_map;
    cx->next_map += trials;
    size_t mark = cx->ar->top;
    REAL *perm = (REAL *)rmo_alloc(cx->ar, sizeof(REAL) * (size_t)trials * n);
    REAL *mins = (REAL *)rmo_alloc(cx->ar, sizeof(REAL) * (size_t)half);
    REAL lm[2 * RMO_MAXL];
    unsigned key[2 * RMO_MAXL];
    for (int t = 0; t < trials; t++) {
        int src = t % p;                                   /* :229 */
        const REAL *a = alphas + (size_t)src * n;
        REAL *v = perm + (size_t)t * n;
        for (int j = 0; j < n; j++) v[j] = a[rmo_inv(&mp[t], (unsigned)j)]; /* :230-231 */
        for (int j = 0; j < half; j++) {                   /* :232-233 */
            REAL x = v[j] < 0 ? -v[j] : v[j], y = v[j + half] < 0 ? -v[j + half] : v[j + half];
            mins[j] = y < x ? y : x;
        }
        lm[t] = FN(pw_sum)(mins, half);
        /* tie-fix key: the pairing direction d = A^-1 e_{m-1}.  At the root it is
         * taken through the path's init map (composite), elsewhere per source
         * path.  Trials with equal keys pair the same entries. */
        unsigned d = mp[t].icol[mp[t].m - 1];
        if (is_root) key[t] = rmo_lin_inv(cx->init[src], d);
        else key[t] = (unsigned)src << 16 | d;
        if (cx->v2) /* same multiset of pair minima, canonical order */
            lm[t] = is_root ? FN(v2_lm_root)(cx->root_llr, cx->N, key[t]) : FN(v2_lm_inner)(a, n, d);
    }
    if (cx->tie_fix)
        for (int t = 1; t < trials; t++)
            for (int s = 0; s < t; s++)
                if (key[s] == key[t]) { lm[t] = lm[s]; break; }
    /* :234 lexsort((arange, -lm)) → lm descending, ties to the lower trial */
    int ord[2 * RMO_MAXL];
    for (int t = 0; t < trials; t++) ord[t] = t;
    for (int i = 1; i < trials; i++) {
        int e = ord[i], j = i - 1;
        while (j >= 0 && lm[ord[j]] < lm[e]) { ord[j + 1] = ord[j]; j--; }
        ord[j + 1] = e;
    }
    int K = trials < L ? trials : L;
    if (trials > L) FN(note)(cx, lm[ord[K - 1]], lm[ord[K]]);
    REAL npm[RMO_MAXL];
    for (int o = 0; o < K; o++) {                          /* :235-237 */
        int t = ord[o];
        memcpy(out + (size_t)o * n, perm + (size_t)t * n, sizeof(REAL) * (size_t)n);
        parent[o] = t % p;
        npm[o] = pms[t % p];
        chosen[o] = &mp[t];
    }
    for (int o = 0; o < K; o++) pms[o] = npm[o];
    cx->ar->top = mark;
    return K;
}

/* _decode_node, top_decoders.py:72-113 (FHT and SPC nodes on, leaves never
 * reached: r == 1 is caught before r == 0, r == m-1 before m == 0). */
static int FN(node)(FN(rmo_ctx) *cx, int r, int mn, const REAL *alphas, int p, REAL *pms,
                    uint8_t *beta, int *lin)
{
    int n = 1 << mn;
    if (r == 1) {                                          /* :76-81 */
        cx->perm_active = 0;
        return FN(fhtl)(cx, alphas, p, n, pms, beta, lin);
    }
    if (mn >= 1 && r == mn - 1)                            /* :82-84 */
        return FN(spc)(cx, alphas, p, n, pms, beta, lin);
    if (mn == 0) return -2;                                /* leaves: not on this path */
    size_t mark = cx->ar->top;
    int L = cx->L, half = n >> 1;
    const REAL *a = alphas;
    int q = p, lineage0[RMO_MAXL];
    const rmo_map *here[RMO_MAXL];
    int have_perm = 0;
    for (int i = 0; i < p; i++) lineage0[i] = i;
    if (cx->perms && cx->perm_active && 1 < r && r < mn - 1) {   /* :93-96 */
        REAL *pa = (REAL *)rmo_alloc(cx->ar, sizeof(REAL) * (size_t)L * n);
        q = FN(perm_extend)(cx, alphas, p, n, mn == cx->m, pms, pa, lineage0, here);
        if (q < 0) return -1;
        a = pa;
        have_perm = 1;
    }
    REAL *left = (REAL *)rmo_alloc(cx->ar, sizeof(REAL) * (size_t)q * half);
    for (int row = 0; row < q; row++)                      /* :100 */
        for (int j = 0; j < half; j++)
            left[(size_t)row * half + j] = FN(f_op)(a[(size_t)row * n + j], a[(size_t)row * n + half + j]);
    uint8_t *bl = (uint8_t *)rmo_alloc(cx->ar, (size_t)L * half);
    int lin1[RMO_MAXL];
    int q1 = FN(node)(cx, r - 1, mn - 1, left, q, pms, bl, lin1);   /* :101 */
    if (q1 < 0) return q1;
    REAL *right = (REAL *)rmo_alloc(cx->ar, sizeof(REAL) * (size_t)q1 * half);
    for (int row = 0; row < q1; row++) {                   /* :102-104 */
        const REAL *ar = a + (size_t)lin1[row] * n;
        for (int j = 0; j < half; j++)
            right[(size_t)row * half + j] = FN(g_op)(ar[j], ar[half + j], bl[(size_t)row * half + j]);
    }
    uint8_t *br = (uint8_t *)rmo_alloc(cx->ar, (size_t)L * half);
    uint8_t *tmp = (uint8_t *)rmo_alloc(cx->ar, (size_t)n);
    int lin2[RMO_MAXL];
    int q2 = FN(node)(cx, r, mn - 1, right, q1, pms, br, lin2);      /* :105 */
    if (q2 < 0) return q2;
    for (int row = 0; row < q2; row++) {
        const uint8_t *l = bl + (size_t)lin2[row] * half, *rr = br + (size_t)row * half;
        for (int j = 0; j < half; j++) { tmp[j] = l[j] ^ rr[j]; tmp[half + j] = rr[j]; } /* :106-107 */
        int chain = lin1[lin2[row]];                       /* :109 */
        uint8_t *out = beta + (size_t)row * n;
        if (have_perm) {                                   /* :110-112 out[i] = beta[sigma(i)] */
            for (int i = 0; i < n; i++) out[i] = tmp[rmo_fwd(here[chain], (unsigned)i)];
        } else {
            memcpy(out, tmp, (size_t)n);
        }
        lin[row] = lineage0[chain];                        /* :113 */
    }
    cx->ar->top = mark;
    return q2;
}

/* The pm the float32 GPU kernels report (rmfht_kernels.cuh, CorrPm): the
 * decided codeword's metric recomputed from the channel LLRs by the PM
 * identity 1/2 sum(|a| - (1-2c) a) = sum of |a_i| where (a_i < 0) != c_i,
 * summed in double in the GPU's order (lane l = i mod 32 adds its positions
 * in ascending i, then the xor tree 16, 8, 4, 2, 1) and rounded once.  The
 * float64 mode reports the accumulated metric, as the reference does. */
static REAL FN(corr_pm)(const REAL *llr, const uint8_t *cw, int N)
{
    double q[32], t[32];
    for (int l = 0; l < 32; l++) {
        q[l] = 0.0;
        for (int i = l; i < N; i += 32)
            if ((llr[i] < 0) != (cw[i] != 0)) q[l] += fabs((double)llr[i]);
    }
    for (int off = 16; off >= 1; off >>= 1) {
        for (int l = 0; l < 32; l++) t[l] = q[l] + q[l ^ off];
        memcpy(q, t, sizeof q);
    }
    return (REAL)q[0];
}

/* _run_engine, top_decoders.py:116-153 (one attempt). */
static int FN(attempt)(FN(rmo_ctx) *cx, const REAL *llr, uint8_t *cw, REAL *pm_out, int *path_out)
{
    int N = cx->N, L = cx->L, p;
    size_t mark = cx->ar->top;
    REAL *alphas;
    REAL pms[RMO_MAXL];
    const rmo_map *root[RMO_MAXL];
    cx->perm_active = cx->perms;
    cx->next_map = 0;
    cx->root_llr = llr;
    if (cx->perms) {
        if (cx->nmaps < L) return -1;
        alphas = (REAL *)rmo_alloc(cx->ar, sizeof(REAL) * (size_t)L * N);
        for (int l = 0; l < L; l++) {                      /* :129-139 apply_perm = v[inv] */
            root[l] = &cx->maps[l];
            cx->init[l] = root[l];
            for (int j = 0; j < N; j++) alphas[(size_t)l * N + j] = llr[rmo_inv(root[l], (unsigned)j)];
            pms[l] = 0;
        }
        cx->next_map = L;
        p = L;
    } else {
        alphas = (REAL *)rmo_alloc(cx->ar, sizeof(REAL) * (size_t)N);
        memcpy(alphas, llr, sizeof(REAL) * (size_t)N);
        pms[0] = 0;
        p = 1;
    }
    uint8_t *beta = (uint8_t *)rmo_alloc(cx->ar, (size_t)L * N);
    int lin[RMO_MAXL];
    int q = FN(node)(cx, cx->r, cx->m, alphas, p, pms, beta, lin);
    if (q < 0) return q;
    if (cx->perms && cx->next_map != cx->nmaps) return -1;
    int best = 0;                                          /* :152 first minimum */
    for (int i = 1; i < q; i++)
        if (pms[i] < pms[best]) best = i;
    uint8_t *bb = beta + (size_t)best * N;
    for (int i = 0; i < N; i++)                            /* :147-150 unpermute by init map */
        cw[i] = cx->perms ? bb[rmo_fwd(root[lin[best]], (unsigned)i)] : bb[i];
    /* instrumentation: a competitor row with a different codeword */
    for (int i = 0; i < q; i++) {
        if (i == best) continue;
        uint8_t *bi = beta + (size_t)i * N;
        int differ = 0;
        for (int j = 0; j < N && !differ; j++) {
            uint8_t v = cx->perms ? bi[rmo_fwd(root[lin[i]], (unsigned)j)] : bi[j];
            differ = v != cw[j];
        }
        if (differ) FN(note)(cx, pms[best], pms[i]);
    }
    *pm_out = pms[best];
    *path_out = best;
    cx->ar->top = mark;
    return 0;
}

/* ensemble_decode, top_decoders.py:190-202, over a batch of frames.  With
 * perms == 0 this is fht_fscl_decode / fht_fsc_decode (one attempt, M = 1). */
int FN(rmo_decode)(int r, int m, int L, int M, int perms, int flags, const REAL *llr, long B,
                   const uint16_t *raw_maps, int nthreads, uint8_t *cw_out, REAL *pm_out,
                   int32_t *attempt_out, int32_t *path_out, REAL *att_pm, uint8_t *att_cw,
                   double *margin_out)
{
    if (m < 2 || m > RMO_MAXM || r < 1 || r > m - 1 || L < 1 || L > RMO_MAXL || M < 1) return -3;
    if (!perms) M = 1;
    int N = 1 << m;
    int S = perms ? rmo_maps_per_attempt(r, m, L, 1, NULL) : 0;
    int sizes[RMO_MAXS];
    if (perms) rmo_maps_per_attempt(r, m, L, 1, sizes);
    int err = 0;
#ifdef _OPENMP
#pragma omp parallel num_threads(nthreads > 0 ? nthreads : 1) reduction(min : err)
#endif
    {
        rmo_arena ar;
        rmo_arena_init(&ar, (size_t)(64 + 24 * L) * N * sizeof(REAL) + (1u << 20));
        rmo_map *maps = (rmo_map *)malloc(sizeof(rmo_map) * (size_t)(S > 0 ? S : 1));
        uint8_t *cw = (uint8_t *)malloc((size_t)N);
        FN(rmo_ctx) cx;
        memset(&cx, 0, sizeof cx);
        cx.r = r; cx.m = m; cx.N = N; cx.L = L; cx.perms = perms;
        cx.tie_fix = flags & RMO_TIE_FIX ? 1 : 0;
        cx.v2 = flags & RMO_ORDER_V2 ? 1 : 0;
        cx.maps = maps; cx.nmaps = S; cx.ar = &ar;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 4)
#endif
        for (long f = 0; f < B; f++) {
            REAL best_pm = 0, best_rep = 0;
            int best_a = -1, best_path = 0;
            double margin = 1e300;
            uint8_t *bcw = cw_out + (size_t)f * N;
            for (int a = 0; a < M; a++) {
                for (int s = 0; s < S; s++) {
                    const uint16_t *raw = raw_maps + (((size_t)f * M + a) * S + s) * (size_t)(m + 1);
                    if (rmo_expand(raw, sizes[s], m, &maps[s]) != 0) err = -4;
                }
                cx.margin = 1e300;
                REAL pm;
                int path;
                int rc = FN(attempt)(&cx, llr + (size_t)f * N, cw, &pm, &path);
                if (rc != 0) { err = rc; continue; }
                if (cx.margin < margin) margin = cx.margin;
                /* reported pm: accumulated (float64 = the reference) or the
                 * float32 kernels' recomputed metric; selection stays on pm */
                const REAL rep = sizeof(REAL) == 4 ? FN(corr_pm)(llr + (size_t)f * N, cw, N) : pm;
                if (att_pm) att_pm[(size_t)f * M + a] = rep;
                if (att_cw) memcpy(att_cw + ((size_t)f * M + a) * N, cw, (size_t)N);
                if (best_a >= 0) {
                    int differ = memcmp(bcw, cw, (size_t)N) != 0;
                    if (differ) {
                        double g = rmo_rel_gap((double)pm, (double)best_pm);
                        if (g < margin) margin = g;
                    }
                }
                if (best_a < 0 || pm < best_pm) {          /* :200 strict < */
                    best_pm = pm; best_rep = rep; best_a = a; best_path = path;
                    memcpy(bcw, cw, (size_t)N);
                }
            }
            pm_out[f] = best_rep;
            if (attempt_out) attempt_out[f] = best_a;
            if (path_out) path_out[f] = best_path;
            if (margin_out) margin_out[f] = margin;
        }
        free(cw);
        free(maps);
        rmo_arena_free(&ar);
    }
    return err;
}

/* ---------------------------------------------------------- Aut-SSC ----
 * ssc_decode, top_decoders.py:205-230: simplified SC with rate-0 (r < 0),
 * rate-1 (r == m), repetition (r == 0: all ones iff np.sum(a) < 0, numpy
 * pairwise order) and SPC (r == m-1: hard decisions, and on odd parity the
 * first minimum of |a| flipped) leaves; f, g and propagate_hard otherwise.
 * `out` receives the node's n bits; `scratch` holds >= n reals. */
static void FN(ssc)(int r, int m, const REAL *a, uint8_t *out, REAL *scratch)
{
    const int n = 1 << m;
    if (r < 0) { memset(out, 0, (size_t)n); return; }
    if (r == m) { for (int i = 0; i < n; i++) out[i] = a[i] < 0; return; }
    if (r == 0) { memset(out, FN(pw_sum)(a, n) < 0 ? 1 : 0, (size_t)n); return; }
    if (r == m - 1) {
        int par = 0, amin = 0;
        REAL best = 0;
        for (int i = 0; i < n; i++) {
            out[i] = a[i] < 0;
            par ^= out[i];
            REAL v = a[i] < 0 ? -a[i] : a[i];
            if (i == 0 || v < best) { best = v; amin = i; }   /* np.argmin: first minimum */
        }
        if (par) out[amin] ^= 1;
        return;
    }
    const int h = n >> 1;
    REAL *x = scratch;
    for (int i = 0; i < h; i++) x[i] = FN(f_op)(a[i], a[h + i]);
    FN(ssc)(r - 1, m - 1, x, out, scratch + h);
    for (int i = 0; i < h; i++) x[i] = FN(g_op)(a[i], a[h + i], out[i]);
    FN(ssc)(r, m - 1, x, out + h, scratch + h);
    for (int i = 0; i < h; i++) out[i] ^= out[h + i];       /* propagate_hard, list_engine.py:30-36 */
}

/* aut_ssc, top_decoders.py:235-249, over a batch: P SSC decodes of the
 * permuted frame (apply_perm: x[sigma(i)] = alpha[i]), each un-permuted
 * (cand[i] = c[sigma(i)]) and scored by correlation (:231, np.sum of
 * (1-2 cand) alpha in numpy pairwise order); the first strictly largest
 * score wins.  raw_maps [B, P, m+1]; outputs cw [B, N], score [B], winner [B]. */
int FN(rmo_aut_ssc)(int r, int m, int P, const REAL *llr, long B, const uint16_t *raw_maps, int nthreads,
                    uint8_t *cw_out, REAL *score_out, int32_t *winner_out)
{
    if (m < 2 || m > RMO_MAXM || r < 1 || r > m - 1 || P < 1) return -3;
    const int N = 1 << m;
    int err = 0;
#ifdef _OPENMP
#pragma omp parallel num_threads(nthreads > 0 ? nthreads : 1) reduction(min : err)
#endif
    {
        REAL *x = (REAL *)malloc(sizeof(REAL) * (size_t)N * 3);
        REAL *scr = x + N, *sv = x + 2 * N;
        uint8_t *c = (uint8_t *)malloc((size_t)N * 2), *cand = c + N;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 2)
#endif
        for (long f = 0; f < B; f++) {
            const REAL *al = llr + (size_t)f * N;
            REAL best = 0;
            int win = -1;
            for (int p = 0; p < P; p++) {
                rmo_map mp;
                if (rmo_expand(raw_maps + ((size_t)f * P + p) * (size_t)(m + 1), m, m, &mp) != 0) { err = -4; continue; }
                for (int i = 0; i < N; i++) x[rmo_fwd(&mp, (unsigned)i)] = al[i];
                FN(ssc)(r, m, x, c, scr);
                for (int i = 0; i < N; i++) cand[i] = c[rmo_fwd(&mp, (unsigned)i)];
                for (int i = 0; i < N; i++) sv[i] = cand[i] ? -al[i] : al[i];
                const REAL sc = FN(pw_sum)(sv, N);
                if (win < 0 || sc > best) {              /* score > best_score, best starts at -inf */
                    best = sc;
                    win = p;
                    memcpy(cw_out + (size_t)f * N, cand, (size_t)N);
                }
            }
            score_out[f] = best;
            if (winner_out) winner_out[f] = win;
        }
        free(c);
        free(x);
    }
    return err;
}

#undef FN
