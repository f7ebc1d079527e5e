// B200 (sm_100a) batched p-FHT-FSCL-L-M decoder for Reed-Muller codes.
//
// One warp decodes one (frame, attempt): L list paths spread over the 32
// lanes (32/L lanes per path).  One CTA owns one frame at a time (grid-stride
// over frames); its warps take the frame's M attempts round-robin and meet
// in a per-frame argmin.  The decoding tree is the reference's recursion
// (top_decoders.py:72-113) unrolled at compile time on (r, m, L): there is no
// HBM traffic between tree nodes — node vectors live in shared memory, FHT
// butterflies in registers and warp shuffles.
//
// Arithmetic follows the reference operation by operation (fht_decode.py,
// list_engine.py, automorphism.py) so that T=double is bit-exact with the
// float64 reference and T=float is bit-exact with the float32 restatement
// of the oracle.  Reference paths are relative to
// /root/reference/pkg/src/rmworkbench/.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rmfht {

constexpr int kMaxM = 10;          // N <= 1024 on the GPU path
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// ---------------------------------------------------------------- maps ----
// One affine map sigma(i) = A bits(i) xor b (automorphism.py:74-108), stored
// by columns for both directions so that any index costs m conditional XORs.
struct MapS {
    uint32_t icol[kMaxM];  // sigma^-1(j) = c  xor  xor_k bit_k(j) icol[k]
    uint32_t c;
    uint32_t col[kMaxM];   // sigma(i)    = b  xor  xor_k bit_k(i) col[k]
    uint32_t b;
};

template <int MN>
__device__ __forceinline__ uint32_t lin_apply(const uint32_t* cols, uint32_t x) {
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < MN; k++) v ^= (x >> k & 1u) ? cols[k] : 0u;
    return v;
}
template <int MN>
__device__ __forceinline__ uint32_t map_inv(const MapS& mp, uint32_t j) { return mp.c ^ lin_apply<MN>(mp.icol, j); }
template <int MN>
__device__ __forceinline__ uint32_t map_fwd(const MapS& mp, uint32_t i) { return mp.b ^ lin_apply<MN>(mp.col, i); }

// composite "apply first, then t" (AffinePermutation.compose, automorphism.py:114-116)
template <int MN>
__device__ void compose(MapS& out, const MapS& t, const MapS& first) {
#pragma unroll
    for (int k = 0; k < MN; k++) {
        out.icol[k] = lin_apply<MN>(first.icol, t.icol[k]);
        out.col[k] = lin_apply<MN>(t.col, first.col[k]);
    }
    out.c = lin_apply<MN>(first.icol, t.c) ^ first.c;
    out.b = lin_apply<MN>(t.col, first.b) ^ t.b;
}

// device record: (2*mg+2) uint16 = col[0..mg), b, icol[0..mg), c
__device__ __forceinline__ void load_map(MapS& out, const uint16_t* rec, int mg, int mn) {
    for (int k = 0; k < kMaxM; k++) {
        out.col[k] = k < mn ? rec[k] : 0u;
        out.icol[k] = k < mn ? rec[mg + 1 + k] : 0u;
    }
    out.b = rec[mg];
    out.c = rec[2 * mg + 1];
}

// ------------------------------------------------------------ schedule ----
__host__ __device__ constexpr int maps_per_attempt(int r, int m, int L) {
    return L + ((m - r >= 2) ? (r - 1) * 2 * L : 0);
}
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }

template <typename T>
__device__ __forceinline__ T tabs(T x) { return x < T(0) ? -x : x; }

// Reported path metric of the float32 kernels: the metric of the decided
// codeword recomputed from the channel LLRs by the PM identity (SURVEY
// §8(a): PM = 1/2 sum(|a| - (1-2c) a) = the sum of |a_i| over the positions
// whose hard decision disagrees with c) — the "ML-in-list by correlation" of
// the north star.  The accumulated float32 metric (fht_decode.py:119, ...)
// selects paths and attempts as the reference does; but its node increments
// 1/2 (llr_abs - |w|) cancel catastrophically in float32, so it is only
// reported to ~1e-4 absolute.  This sum has no cancellation: each lane adds
// its positions i = 32 t + lane in ascending t in double, then a xor tree
// (16, 8, 4, 2, 1); rounded once.  The oracle's float32 mode restates it
// (rmo_impl.h, corr_pm).
struct CorrPm {
    double acc = 0.0;
    __device__ __forceinline__ void add(float a, int bit) {
        if ((a < 0.f) != (bit != 0)) acc += fabs((double)a);
    }
    __device__ __forceinline__ float total() {
        double v = acc;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) v = v + __shfl_xor_sync(kFull, v, off);
        return (float)v;
    }
};

// offsets of level s in the per-level buffers
template <typename T, int R, int MM, int L>
__device__ __forceinline__ int lvl_off(int s) { return L * ((1 << s) - 1); }
template <int L>
__device__ __forceinline__ int b_off(int s) { return L * ((1 << (s - 1)) - 1); }

// ----------------------------------------------------------- workspace ----
template <typename T, int R, int MM, int L>
struct alignas(16) WarpWS {
    static constexpr int N = 1 << MM;
    static constexpr int S = maps_per_attempt(R, MM, L);
    static constexpr int SPCN = 1 << cmin(R + 1, MM);
    T lvl[L * N];                    // node inputs, level s at L*(2^s-1), row stride 2^s
    T permb[R >= 3 ? L * N : 1];     // winners of inner permutation nodes, per level like lvl
    T pms[L];
    T llrabs[L];
    T lm[2 * L];
    T cpm[L * L], cabs[L * L], cw[L * L];
    T best_pm;
    T best_rep;  // reported pm of the best attempt (CorrPm for float32)
    MapS maps[S > 0 ? S : 1];
    MapS comp[L];                    // root paths: composite of init and root trial maps
    MapS tcomp[2 * L];
    uint32_t best_cw[N / 32 > 0 ? N / 32 : 1];
    int cbin[L * L];
    int sel[L * L];
    int best_att, best_path, next_map, spc_cnt;
    int8_t rmB[MM + 1][L], l0[MM + 1][L], l1[MM + 1][L], l2[MM + 1][L];
    int16_t nmap[MM + 1][L];
    int8_t ident[L], rootlin[L], rootchain[L];
    uint16_t spc_ord[L * SPCN];
    uint8_t spc_sign[L * SPCN];
    uint8_t bl[L * N], br[L * N], rootout[L * N];
};

template <typename T>
struct Params {
    const T* llr;          // [B, N]
    const uint16_t* maps;  // [B, M, S, 2m+2] device map records
    long long B;
    int M, perms, tie_fix;
    uint32_t* cw;          // [B, N/32] bit-packed codewords (bit i%32 of word i/32)
    T* pm;                 // [B]
    int32_t* attempt;      // [B]
    int32_t* path;         // [B]
    T* att_pm;             // optional [B, M]
    uint32_t* att_cw;      // optional [B, M, N/32]
};

template <typename T, int R, int MM, int L>
struct Ctx {
    using WS = WarpWS<T, R, MM, L>;
    WS& ws;
    const T* alpha;  // frame LLRs in shared memory
    int perms, tie_fix;
};

// node inputs: a level buffer row (via a row map) or the root gather
template <typename T>
struct InBuf {
    const T* base;
    int stride;
    const int8_t* rm;
    __device__ __forceinline__ T get(int p, int j) const { return base[rm[p] * stride + j]; }
};
template <typename T, int MM>
struct InRoot {
    const T* alpha;
    const MapS* comp;
    const int8_t* rm;
    __device__ __forceinline__ T get(int p, int j) const { return alpha[map_inv<MM>(comp[rm[p]], (uint32_t)j)]; }
};

// -------------------------------------------------- pairwise summation ----
// numpy's pairwise order for a contiguous row of NV values (np.sum at
// fht_decode.py:114, automorphism.py:233): C = 1 chain when NV < 8, else 8
// chains per 128-block (chain q of block b sums b*128+q, +8, +16, ...
// sequentially), combined by a balanced binary tree in chain order.
// Sums NG groups; group g's result lands in out[g].
template <typename T, int NV, int NG, typename F>
__device__ __forceinline__ void pairwise_groups(F value, T* out) {
    constexpr int C = NV < 8 ? 1 : 8 * (NV > 128 ? NV / 128 : 1);
    constexpr int LEN = NV / C;
    constexpr int TASKS = NG * C;
    constexpr int G = TASKS >= 32 ? TASKS / 32 : 1;
    const int lane = lane_id();
    T acc[G];
#pragma unroll
    for (int g = 0; g < G; g++) {
        const int task = lane * G + g;
        const int grp = task / C, ch = task % C;
        T s = T(0);
        if (task < TASKS) {
            const int base = (C == 1) ? 0 : (ch / 8) * 128 + (ch % 8);
            const int step = (C == 1) ? 1 : 8;
            s = value(grp, base);
#pragma unroll 4
            for (int i = 1; i < LEN; i++) s += value(grp, base + i * step);
        }
        acc[g] = s;
    }
    if constexpr (G >= C) {
        // every lane holds G/C whole groups
#pragma unroll
        for (int w = 1; w < C; w *= 2)
#pragma unroll
            for (int g = 0; g < G; g += 2 * w) acc[g] = acc[g] + acc[g + w];
#pragma unroll
        for (int g = 0; g < G; g += C) {
            const int grp = (lane * G + g) / C;
            if (lane * G + g < TASKS) out[grp] = acc[g];
        }
    } else {
#pragma unroll
        for (int w = 1; w < G; w *= 2)
#pragma unroll
            for (int g = 0; g < G; g += 2 * w) acc[g] = acc[g] + acc[g + w];
        T v = acc[0];
#pragma unroll
        for (int off = 1; off < C / G; off *= 2) v = v + __shfl_xor_sync(kFull, v, off);
        const int task = lane * G;
        if (task < TASKS && (task % C) == 0) out[task / C] = v;
    }
}

// ------------------------------------------------------------- f and g ----
// f_op (list_engine.py:15-20): min(|a|,|b|) sgn(a) sgn(b), sgn(0) = +1
template <typename T>
__device__ __forceinline__ T f_op(T a, T b) {
    T x = tabs(a), y = tabs(b);
    T mn = y < x ? y : x;
    return ((a < T(0)) != (b < T(0))) ? -mn : mn;
}
// g_op (list_engine.py:23-27): b + (1-2c) a, the product being exactly +-a
template <typename T>
__device__ __forceinline__ T g_op(T a, T b, int c) { return c ? b - a : b + a; }

// --------------------------------------------------------------- FHTL ----
// fhtl (fht_decode.py:101-126) on P paths of size n = 2^SS.
template <typename T, int R, int MM, int L, int SS, class In>
__device__ int fhtl(Ctx<T, R, MM, L>& cx, const In& in, int P, uint8_t* out, int8_t* lin) {
    auto& ws = cx.ws;
    constexpr int n = 1 << SS, LPP = 32 / L, VPL = (n >= LPP) ? n / LPP : 1, K = cmin(L, n);
    const int lane = lane_id(), p = lane / LPP, u = lane % LPP;
    const bool act = (p < P) && (n >= LPP || u < n);
    T w[VPL];
#pragma unroll
    for (int i = 0; i < VPL; i++) {
        const int e = (n >= LPP) ? i * LPP + u : u;
        w[i] = act ? in.get(p, e) : T(0);
    }
    // llr_abs = sum |alpha| per path (:114)
    pairwise_groups<T, n, L>([&](int g, int j) { return g < P ? tabs(in.get(g, j)) : T(0); }, ws.llrabs);
    // fht_transform (:28-48): largest stride first, lo' = hi - lo, hi' = hi + lo
#pragma unroll
    for (int half = n / 2; half >= 1; half >>= 1) {
        if (half >= LPP) {
            const int hr = half / LPP;
#pragma unroll
            for (int i = 0; i < VPL; i++)
                if (!(i & hr)) {
                    T lo = w[i], hi = w[i + hr];
                    w[i] = hi - lo;
                    w[i + hr] = hi + lo;
                }
        } else {
#pragma unroll
            for (int i = 0; i < VPL; i++) {
                T o = __shfl_xor_sync(kFull, w[i], half);
                w[i] = (u & half) ? (w[i] + o) : (o - w[i]);
            }
        }
    }
    // per-path top-K by |w| descending, ties to the lower bin (:116)
    unsigned long long taken = 0ull;
#pragma unroll 1
    for (int rr = 0; rr < K; rr++) {
        T bv = T(-1), bw = T(0);
        int bb = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < VPL; i++) {
            const int e = (n >= LPP) ? i * LPP + u : u;
            const T a = tabs(w[i]);
            if (act && !((taken >> i) & 1ull) && (a > bv || (a == bv && e < bb))) { bv = a; bb = e; bw = w[i]; }
        }
#pragma unroll
        for (int off = 1; off < LPP; off <<= 1) {
            T ov = __shfl_xor_sync(kFull, bv, off), ow = __shfl_xor_sync(kFull, bw, off);
            int ob = __shfl_xor_sync(kFull, bb, off);
            if (ov > bv || (ov == bv && ob < bb)) { bv = ov; bb = ob; bw = ow; }
        }
        if (act) {
            const bool mine = (n >= LPP) ? ((bb % LPP) == u) : (bb == u);
            if (mine) taken |= 1ull << ((n >= LPP) ? bb / LPP : 0);
        }
        if (u == 0 && p < P) {
            ws.cabs[p * K + rr] = bv;
            ws.cbin[p * K + rr] = bb;
            ws.cw[p * K + rr] = bw;
        }
    }
    __syncwarp();
    // pool (:119-120): pm = pm_in + 0.5 (llr_abs - |w_b|); lexsort (pm, source, bin)
    const int PK = P * K, KEEP = cmin(L, PK);
    for (int c = lane; c < PK; c += 32) ws.cpm[c] = ws.pms[c / K] + T(0.5) * (ws.llrabs[c / K] - ws.cabs[c]);
    __syncwarp();
    for (int c = lane; c < PK; c += 32) {
        const T pc = ws.cpm[c];
        const int sc = c / K, bc = ws.cbin[c];
        int rank = 0;
        for (int d = 0; d < PK; d++) {
            const T pd = ws.cpm[d];
            const int sd = d / K;
            rank += (pd < pc) || (pd == pc && (sd < sc || (sd == sc && ws.cbin[d] < bc)));
        }
        if (rank < KEEP) ws.sel[rank] = c;
    }
    __syncwarp();
    T newpm = T(0);
    if (lane < KEEP) {
        newpm = ws.cpm[ws.sel[lane]];
        lin[lane] = (int8_t)(ws.sel[lane] / K);
    }
    // winning codewords: bit j = parity(~b & ~j & (n-1)) xor [w_b < 0] (:58-62, :123-125)
    for (int idx = lane; idx < KEEP * n; idx += 32) {
        const int o = idx / n, j = idx % n, c = ws.sel[o];
        const int b = ws.cbin[c];
        out[o * n + j] = (uint8_t)((__popc((unsigned)(~(b | j)) & (unsigned)(n - 1)) & 1) ^ (ws.cw[c] < T(0)));
    }
    __syncwarp();
    if (lane < KEEP) ws.pms[lane] = newpm;
    __syncwarp();
    return KEEP;
}

// ---------------------------------------------------------------- SPC ----
// spc_decode_list (list_engine.py:68-119) on P paths of size n = 2^SS.
template <typename T, int R, int MM, int L, int SS, class In>
__device__ int spc(Ctx<T, R, MM, L>& cx, const In& in, int P, uint8_t* out, int8_t* lin) {
    auto& ws = cx.ws;
    constexpr int n = 1 << SS;
    constexpr int TAU = cmin(cmin(L, n), n - 1);
    const int lane = lane_id();
    uint16_t* ord = ws.spc_ord;
    uint8_t* sg = ws.spc_sign;
    // per path: stable argsort of |alpha| ascending (:83), signs, parity, metric (:84-88)
    if (lane < P) {
        int par = 0;
        for (int j = 0; j < n; j++) {
            const T a = in.get(lane, j);
            sg[lane * n + j] = a < T(0);
            par ^= a < T(0);
            const T mj = tabs(a);
            int i = j - 1;
            while (i >= 0 && tabs(in.get(lane, ord[lane * n + i])) > mj) {
                ord[lane * n + i + 1] = ord[lane * n + i];
                i--;
            }
            ord[lane * n + i + 1] = (uint16_t)j;
        }
        const T amin = tabs(in.get(lane, ord[lane * n]));
        ws.cpm[lane] = ws.pms[lane] + (par ? amin : T(0));
        ws.cabs[lane] = T(par);
    }
    __syncwarp();
    // the tau splits (:97-112) — a short sequential merge; one lane runs it
    if (lane == 0) {
        T pm[2 * L], pr[2 * L];
        int parent[2 * L];
        uint32_t fl[2 * L];
        for (int i = 0; i < P; i++) { pm[i] = ws.cpm[i]; pr[i] = ws.cabs[i]; parent[i] = i; fl[i] = 0; }
        int cnt = P;
        for (int j = 1; j <= TAU; j++) {
            T cand[4 * L];
            int sel[4 * L];
            for (int i = 0; i < cnt; i++) {
                const T aj = tabs(in.get(parent[i], ord[parent[i] * n + j]));
                const T am = tabs(in.get(parent[i], ord[parent[i] * n]));
                cand[2 * i] = pm[i];
                const T t = pm[i] + aj;  // pms + a_j + (1 - 2 par) a_m
                cand[2 * i + 1] = pr[i] != T(0) ? t - am : t + am;
            }
            const int C = 2 * cnt;
            for (int c = 0; c < C; c++) {  // stable argsort
                int t = c - 1;
                while (t >= 0 && cand[sel[t]] > cand[c]) { sel[t + 1] = sel[t]; t--; }
                sel[t + 1] = c;
            }
            const int Kp = cmin(L, C);
            T npm[2 * L], npr[2 * L];
            int npa[2 * L];
            uint32_t nfl[2 * L];
            for (int o = 0; o < Kp; o++) {
                const int which = sel[o] & 1, src = sel[o] >> 1;
                npm[o] = cand[sel[o]];
                nfl[o] = fl[src] | (which ? (1u << j) : 0u);
                npr[o] = which ? T(1) - pr[src] : pr[src];
                npa[o] = parent[src];
            }
            for (int o = 0; o < Kp; o++) { pm[o] = npm[o]; pr[o] = npr[o]; parent[o] = npa[o]; fl[o] = nfl[o]; }
            cnt = Kp;
        }
        for (int o = 0; o < cnt; o++) { ws.cpm[o] = pm[o]; ws.sel[o] = parent[o]; ws.cbin[o] = (int)fl[o]; }
        ws.spc_cnt = cnt;
    }
    __syncwarp();
    const int cnt = ws.spc_cnt;
    // beta = sign xor flips; least reliable bit fixes even parity (:114-118)
    if (lane < cnt) {
        const int par = ws.sel[lane];
        const uint32_t fl = (uint32_t)ws.cbin[lane];
        int tot = 0;
        for (int j = 0; j < n; j++) {
            int b = sg[par * n + j];
            out[lane * n + j] = (uint8_t)b;
            tot ^= b;
        }
        for (int j = 1; j <= TAU; j++)
            if (fl >> j & 1u) {
                out[lane * n + ord[par * n + j]] ^= 1;
                tot ^= 1;
            }
        out[lane * n + ord[par * n]] ^= (uint8_t)tot;
        lin[lane] = (int8_t)par;
    }
    __syncwarp();
    if (lane < cnt) ws.pms[lane] = ws.cpm[lane];
    __syncwarp();
    return cnt;
}

// ------------------------------------------------ permutation extension ----
// permutation_extend (automorphism.py:207-237): 2P trials, LM = sum of
// min(|lo|,|hi|) in numpy's pairwise order, keep min(L, 2P) by LM
// descending, ties to the lower trial.  Returns the kept count; writes the
// kept order into ws.sel[0..K).
template <typename T, int R, int MM, int L>
__device__ int select_trials(Ctx<T, R, MM, L>& cx, int trials, const uint32_t* key) {
    auto& ws = cx.ws;
    const int lane = lane_id();
    if (cx.tie_fix && lane == 0) {
        // equal pairing directions pair the same entries: keep their LM equal
        for (int t = 1; t < trials; t++)
            for (int s = 0; s < t; s++)
                if (key[s] == key[t]) { ws.lm[t] = ws.lm[s]; break; }
    }
    __syncwarp();
    const int K = cmin(L, trials);
    if (lane < trials) {
        const T v = ws.lm[lane];
        int rank = 0;
        for (int s = 0; s < trials; s++) rank += (ws.lm[s] > v) || (ws.lm[s] == v && s < lane);
        if (rank < K) ws.sel[rank] = lane;
    }
    __syncwarp();
    return K;
}

template <typename T, int R, int MM, int L>
__device__ int perm_ext_root(Ctx<T, R, MM, L>& cx, int P) {
    auto& ws = cx.ws;
    constexpr int N = 1 << MM, H = N / 2;
    const int lane = lane_id(), trials = 2 * P, base = ws.next_map;
    if (lane < trials) compose<MM>(ws.tcomp[lane], ws.maps[base + lane], ws.comp[lane % P]);
    __syncwarp();
    const T* alpha = cx.alpha;
    pairwise_groups<T, H, 2 * L>(
        [&](int t, int j) {
            if (t >= trials) return T(0);
            const MapS& mp = ws.tcomp[t];
            const T x = tabs(alpha[map_inv<MM>(mp, (uint32_t)j)]), y = tabs(alpha[map_inv<MM>(mp, (uint32_t)(j + H))]);
            return y < x ? y : x;
        },
        ws.lm);
    __syncwarp();
    uint32_t key[2 * L];
#pragma unroll
    for (int t = 0; t < 2 * L; t++) key[t] = t < trials ? ws.tcomp[t].icol[MM - 1] : 0u;  // composite d
    const int K = select_trials(cx, trials, key);
    T npm = T(0);
    if (lane < K) {
        const int t = ws.sel[lane];
        ws.comp[lane] = ws.tcomp[t];
        npm = ws.pms[t % P];
        ws.l0[MM][lane] = (int8_t)(t % P);
    }
    __syncwarp();
    if (lane < K) ws.pms[lane] = npm;
    ws.next_map = base + trials;
    __syncwarp();
    return K;
}

template <typename T, int R, int MM, int L, int SS>
__device__ int perm_ext_inner(Ctx<T, R, MM, L>& cx, const InBuf<T>& in, int P) {
    auto& ws = cx.ws;
    constexpr int n = 1 << SS, H = n / 2;
    const int lane = lane_id(), trials = 2 * P, base = ws.next_map;
    pairwise_groups<T, H, 2 * L>(
        [&](int t, int j) {
            if (t >= trials) return T(0);
            const MapS& mp = ws.maps[base + t];
            const int src = t % P;
            const T x = tabs(in.get(src, map_inv<SS>(mp, (uint32_t)j))),
                    y = tabs(in.get(src, map_inv<SS>(mp, (uint32_t)(j + H))));
            return y < x ? y : x;
        },
        ws.lm);
    __syncwarp();
    uint32_t key[2 * L];
#pragma unroll
    for (int t = 0; t < 2 * L; t++)
        key[t] = t < trials ? (((uint32_t)(t % P) << 16) | ws.maps[base + t].icol[SS - 1]) : 0u;
    const int K = select_trials(cx, trials, key);
    for (int idx = lane; idx < K * n; idx += 32) {
        const int o = idx / n, j = idx % n, t = ws.sel[o];
        ws.permb[lvl_off<T, R, MM, L>(SS) + o * n + j] = in.get(t % P, map_inv<SS>(ws.maps[base + t], (uint32_t)j));
    }
    T npm = T(0);
    if (lane < K) {
        const int t = ws.sel[lane];
        npm = ws.pms[t % P];
        ws.l0[SS][lane] = (int8_t)(t % P);
        ws.nmap[SS][lane] = (int16_t)(base + t);
    }
    __syncwarp();
    if (lane < K) ws.pms[lane] = npm;
    ws.next_map = base + trials;
    __syncwarp();
    return K;
}

// ------------------------------------------------------- tree recursion ----

template <typename T, int R, int MM, int L, int RR, int SS, bool SPINE, class In>
__device__ int node(Ctx<T, R, MM, L>& cx, const In& in, int P, uint8_t* out, int8_t* lin) {
    auto& ws = cx.ws;
    if constexpr (RR == 1) {
        return fhtl<T, R, MM, L, SS>(cx, in, P, out, lin);                    // :76-81
    } else if constexpr (RR == SS - 1) {
        return spc<T, R, MM, L, SS>(cx, in, P, out, lin);                     // :82-84
    } else {
        constexpr int n = 1 << SS, h = n / 2;
        constexpr bool PERMNODE = SPINE && RR >= 2 && SS - RR >= 2;          // :93
        const int lane = lane_id();
        int8_t* l0 = ws.l0[SS];
        int8_t* l1 = ws.l1[SS];
        int8_t* l2 = ws.l2[SS];
        if (lane < L) l0[lane] = (int8_t)lane;
        __syncwarp();
        In a = in;
        bool inner_perm = false;
        if constexpr (PERMNODE) {
            if (cx.perms) {
                if constexpr (SS == MM) {
                    P = perm_ext_root(cx, P);                                  // root: maps composed
                } else {
                    P = perm_ext_inner<T, R, MM, L, SS>(cx, in, P);
                    a.base = ws.permb + lvl_off<T, R, MM, L>(SS);
                    a.stride = n;
                    a.rm = ws.ident;
                    inner_perm = true;
                }
            }
        }
        // f (:100) → left child input at level SS-1
        T* child = ws.lvl + lvl_off<T, R, MM, L>(SS - 1);
        for (int idx = lane; idx < P * h; idx += 32) {
            const int p = idx / h, j = idx % h;
            child[idx] = f_op(a.get(p, j), a.get(p, j + h));
        }
        __syncwarp();
        uint8_t* bl = ws.bl + b_off<L>(SS);
        uint8_t* br = ws.br + b_off<L>(SS);
        const InBuf<T> left{child, h, ws.ident};
        const int P1 = node<T, R, MM, L, RR - 1, SS - 1, SPINE>(cx, left, P, bl, l1);   // :101
        // alphas = alphas[lin1] (:102) as a row-map composition
        if (lane < P1) ws.rmB[SS][lane] = a.rm[l1[lane]];
        __syncwarp();
        In a2 = a;
        a2.rm = ws.rmB[SS];
        for (int idx = lane; idx < P1 * h; idx += 32) {                        // g (:104)
            const int p = idx / h, j = idx % h;
            child[idx] = g_op(a2.get(p, j), a2.get(p, j + h), (int)bl[idx]);
        }
        __syncwarp();
        const InBuf<T> right{child, h, ws.ident};
        const int P2 = node<T, R, MM, L, RR, SS - 1, false>(cx, right, P1, br, l2);      // :105
        // combine (:106-107), un-permute (:109-112), lineage (:113)
        uint8_t* dst = inner_perm ? ws.rootout : out;
        for (int idx = lane; idx < P2 * h; idx += 32) {
            const int p = idx / h, j = idx % h;
            const uint8_t r = br[idx];
            dst[p * n + j] = bl[l2[p] * h + j] ^ r;
            dst[p * n + h + j] = r;
        }
        __syncwarp();
        if (inner_perm) {
            for (int idx = lane; idx < P2 * n; idx += 32) {
                const int p = idx / n, i = idx % n;
                const MapS& mp = ws.maps[ws.nmap[SS][l1[l2[p]]]];
                out[idx] = dst[p * n + map_fwd<SS>(mp, (uint32_t)i)];
            }
            __syncwarp();
        }
        if (lane < P2) {
            const int chain = l1[l2[lane]];
            lin[lane] = l0[chain];
            if (SS == MM) ws.rootchain[lane] = (int8_t)chain;
        }
        __syncwarp();
        return P2;
    }
}

// ------------------------------------------------------------- kernel ----
template <typename T, int R, int MM, int L>
__global__ void __launch_bounds__(256) decode_kernel(Params<T> prm) {
    using WS = WarpWS<T, R, MM, L>;
    constexpr int N = 1 << MM, S = WS::S, NW = N / 32 > 0 ? N / 32 : 1;
    constexpr int REC = 2 * MM + 2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* alpha = reinterpret_cast<T*>(smem_raw);
    WS* wsarr = reinterpret_cast<WS*>(smem_raw + ((N * sizeof(T) + 15) / 16) * 16);
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), nwarps = blockDim.x >> 5, lane = lane_id();  // provably warp-uniform
    WS& ws = wsarr[warp];
    Ctx<T, R, MM, L> cx{ws, alpha, prm.perms, prm.tie_fix};
    const int Meff = prm.perms ? prm.M : 1;
    if (lane < L) ws.ident[lane] = (int8_t)lane;

    for (long long f = blockIdx.x; f < prm.B; f += gridDim.x) {
        for (int i = threadIdx.x; i < N; i += blockDim.x) alpha[i] = prm.llr[f * N + i];
        __syncthreads();
        bool have = false;
        for (int a = warp; a < Meff; a += nwarps) {
            // this attempt's map records
            if (prm.perms) {
                const uint16_t* recs = prm.maps + ((size_t)f * prm.M + a) * S * REC;
                for (int s = lane; s < S; s += 32) {
                    const int mn = s < L ? MM : MM - (s - L) / (2 * L);
                    load_map(ws.maps[s], recs + (size_t)s * REC, MM, mn);
                }
            }
            int P;
            if (prm.perms) {  // L root maps (:129-140)
                if (lane < L) ws.comp[lane] = ws.maps[lane];
                if (lane < L) ws.pms[lane] = T(0);
                ws.next_map = L;
                P = L;
            } else {
                if (lane == 0) {
                    ws.pms[0] = T(0);
                    for (int k = 0; k < kMaxM; k++) { ws.comp[0].icol[k] = 1u << k; ws.comp[0].col[k] = 1u << k; }
                    ws.comp[0].b = 0;
                    ws.comp[0].c = 0;
                }
                ws.next_map = 0;
                P = 1;
            }
            __syncwarp();
            const InRoot<T, MM> root{alpha, ws.comp, ws.ident};
            P = node<T, R, MM, L, R, MM, true>(cx, root, P, ws.rootout, ws.rootlin);
            // best path: first minimum (:152)
            int best = 0;
            for (int i = 1; i < P; i++)
                if (ws.pms[i] < ws.pms[best]) best = i;
            const T pm = ws.pms[best];
            // un-permute by the root composite (:147-150)
            constexpr bool ROOT_INTERNAL = !(R == 1 || R == MM - 1);
            const int mi = ROOT_INTERNAL ? ws.rootchain[best] : ws.rootlin[best];
            const MapS& mp = ws.comp[mi];
            uint32_t myword = 0;
            CorrPm corr;
#pragma unroll
            for (int t = 0; t < NW; t++) {
                const int i = t * 32 + lane;
                int bit = 0;
                if (i < N) {
                    const uint32_t src = prm.perms ? map_fwd<MM>(mp, (uint32_t)i) : (uint32_t)i;
                    bit = ws.rootout[best * N + src];
                    if constexpr (sizeof(T) == 4) corr.add((float)alpha[i], bit);
                }
                const uint32_t word = __ballot_sync(kFull, bit);
                if (lane == t) myword = word;
            }
            T rep = pm;
            if constexpr (sizeof(T) == 4) rep = (T)corr.total();
            if (prm.att_pm && lane == 0) prm.att_pm[(size_t)f * prm.M + a] = rep;
            if (prm.att_cw && lane < NW) prm.att_cw[((size_t)f * prm.M + a) * NW + lane] = myword;
            if (!have || pm < ws.best_pm) {  // strict <, earlier attempt keeps ties (:200)
                if (lane < NW) ws.best_cw[lane] = myword;
                if (lane == 0) { ws.best_pm = pm; ws.best_rep = rep; ws.best_att = a; ws.best_path = best; }
                have = true;
            }
            __syncwarp();
        }
        if (!have && lane == 0) ws.best_att = -1;
        __syncthreads();
        if (warp == 0) {
            int bw = -1;
            if (lane == 0) {
                for (int w = 0; w < nwarps; w++) {
                    const WS& o = wsarr[w];
                    if (o.best_att < 0) continue;
                    if (bw < 0 || o.best_pm < wsarr[bw].best_pm ||
                        (o.best_pm == wsarr[bw].best_pm && o.best_att < wsarr[bw].best_att))
                        bw = w;
                }
            }
            bw = __shfl_sync(kFull, bw, 0);
            const WS& o = wsarr[bw];
            if (lane < NW) prm.cw[f * NW + lane] = o.best_cw[lane];
            if (lane == 0) {
                prm.pm[f] = o.best_rep;
                prm.attempt[f] = o.best_att;
                prm.path[f] = o.best_path;
            }
        }
        __syncthreads();
    }
}

template <typename T, int R, int MM, int L>
constexpr size_t smem_bytes(int nwarps) {
    return ((size_t(1 << MM) * sizeof(T) + 15) / 16) * 16 + sizeof(WarpWS<T, R, MM, L>) * size_t(nwarps);
}

}  // namespace rmfht
