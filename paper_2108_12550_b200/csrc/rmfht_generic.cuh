// Generic (runtime-shaped) decoder: any RM(r, m) with N <= 1024 and any L
// the shared memory can hold, for shapes without a compile-time
// specialisation.  Same arithmetic and operation order as the
// reference-order kernel (rmfht_kernels.cuh) — bit-exact with the float64
// reference for T = double — but the decoding tree (top_decoders.py:72-113)
// is walked with an explicit stack and every node vector lives in shared
// memory.  One warp per (frame, attempt); one CTA per frame.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "rmfht_kernels.cuh"

namespace rmfht_gen {

using rmfht::kFull;
using rmfht::lane_id;
using rmfht::MapS;

constexpr int kMaxL = 16;
constexpr int kMaxDepth = 12;

struct Shape {
    int r, m, L, N, S;  // S maps per attempt
};

// small per-warp state inside Layout::small
template <typename T>
struct Small {
    T pms[kMaxL], llrabs[kMaxL], lm[2 * kMaxL], pmtmp[2 * kMaxL];
    T cpm[kMaxL * kMaxL], cabs[kMaxL * kMaxL], cw[kMaxL * kMaxL];
    int cbin[kMaxL * kMaxL], sel[kMaxL * kMaxL];
    int8_t rm[kMaxDepth][kMaxL], l0[kMaxDepth][kMaxL], l1[kMaxDepth][kMaxL], l2[kMaxDepth][kMaxL];
    int16_t nmap[kMaxDepth][kMaxL];
    int8_t ident[kMaxL], rootlin[kMaxL], rootchain[kMaxL];
    T best_pm;
    T best_rep;  // reported pm of the best attempt (rmfht::CorrPm for float32)
    int best_att, best_path, next_map, spc_cnt;
    uint32_t best_cw[32];
};

// byte offsets of the per-warp workspace (host computes, device reads)
struct Layout {
    int lvl, perm, bl, br, rootout, maps, comp, small, spc_ord, spc_sgn, pool, total;
};

template <typename T>
__host__ __device__ inline Layout layout(const Shape& sh) {
    Layout o{};
    int off = 0;
    auto take = [&](int bytes) {
        const int at = off;
        off += (bytes + 15) & ~15;
        return at;
    };
    o.lvl = take(sh.L * sh.N * (int)sizeof(T));       // level s rows at L*(2^s-1)
    o.perm = take(sh.L * sh.N * (int)sizeof(T));      // inner permutation winners, per level
    o.bl = take(sh.L * sh.N);
    o.br = take(sh.L * sh.N);
    o.rootout = take(sh.L * sh.N);
    o.maps = take((sh.S > 0 ? sh.S : 1) * (int)sizeof(MapS));
    o.comp = take(4 * sh.L * (int)sizeof(MapS));      // root paths, 2L trial composites, staging
    o.small = take((int)sizeof(Small<T>));
    o.spc_ord = take(sh.L * sh.N * 2);
    o.spc_sgn = take(sh.L * sh.N);
    o.pool = 0;
    o.total = off;
    return o;
}

template <typename T>
struct W {
    T* lvl;
    T* perm;
    uint8_t *bl, *br, *rootout;
    MapS* maps;
    MapS* comp;
    Small<T>* sm;
    uint16_t* spc_ord;
    uint8_t* spc_sgn;
    const T* alpha;
    Shape sh;
    int perms, tie_fix;
};

__device__ __forceinline__ uint32_t lin_rt(const uint32_t* cols, int mn, uint32_t x) {
    uint32_t v = 0;
    for (int k = 0; k < mn; k++) v ^= (x >> k & 1u) ? cols[k] : 0u;
    return v;
}
__device__ __forceinline__ uint32_t inv_rt(const MapS& mp, int mn, uint32_t j) { return mp.c ^ lin_rt(mp.icol, mn, j); }
__device__ __forceinline__ uint32_t fwd_rt(const MapS& mp, int mn, uint32_t i) { return mp.b ^ lin_rt(mp.col, mn, i); }

// node input: a buffer row via a row map, or the root gather
template <typename T>
struct In {
    const T* base;  // null: root gather
    int stride;
    const int8_t* rm;
    const T* alpha;
    const MapS* comp;
    int mm;
    __device__ __forceinline__ T get(int p, int j) const {
        if (base) return base[rm[p] * stride + j];
        return alpha[inv_rt(comp[rm[p]], mm, (uint32_t)j)];
    }
};

// numpy pairwise order (see rmfht_kernels.cuh): sum of |value(g, j)| style
// functor over n values for group g, computed by the whole warp; returns the
// total to every lane.
template <typename T, typename F>
__device__ T pairwise_rt(int n, F value) {
    const int lane = lane_id();
    const int C = n < 8 ? 1 : 8 * (n > 128 ? n / 128 : 1);
    const int len = n / C;
    // chains, then a balanced tree in chain order (C <= 64 for n <= 1024)
    T part = T(0);
    if (lane < C) {
        const int base = (C == 1) ? 0 : (lane / 8) * 128 + (lane % 8);
        const int step = (C == 1) ? 1 : 8;
        part = value(base);
        for (int i = 1; i < len; i++) part += value(base + i * step);
    }
    T hi = T(0);
    if (C > 32 && lane + 32 < C) {
        const int c = lane + 32;
        const int base = (c / 8) * 128 + (c % 8);
        hi = value(base);
        for (int i = 1; i < len; i++) hi += value(base + i * 8);
    }
    // balanced tree over chains 0..C-1: lanes hold chains lane and lane+32
    for (int w = 1; w < C && w < 32; w *= 2) {
        const T o = __shfl_xor_sync(kFull, part, w);
        const T o2 = __shfl_xor_sync(kFull, hi, w);
        part = part + o;
        hi = hi + o2;
    }
    if (C > 32) part = part + hi;  // the top level of the tree: (chains 0..31) + (chains 32..63)
    return __shfl_sync(kFull, part, 0);
}

template <typename T>
__device__ __forceinline__ T tabs(T x) {
    return x < T(0) ? -x : x;
}

// ------------------------------------------------------------------- FHTL
template <typename T>
__device__ int fhtl_rt(W<T>& w, const In<T>& in, int P, int n, T* scratch, uint8_t* out, int8_t* lin) {
    auto& sm = *w.sm;
    const int lane = lane_id(), L = w.sh.L, K = n < L ? n : L;
    for (int p = 0; p < P; p++) {
        // copy, FHT in place (stage order of fht_decode.py:41-47)
        T* v = scratch + p * n;
        for (int j = lane; j < n; j += 32) v[j] = in.get(p, j);
        __syncwarp();
        const T la = pairwise_rt<T>(n, [&](int j) { return tabs(v[j]); });
        if (lane == 0) sm.llrabs[p] = la;
        for (int half = n >> 1; half >= 1; half >>= 1) {
            for (int q = lane; q < n / 2; q += 32) {
                const int blk = (q / half) * 2 * half, x = q % half;
                const T lo = v[blk + x], hi = v[blk + half + x];
                v[blk + x] = hi - lo;
                v[blk + half + x] = hi + lo;
            }
            __syncwarp();
        }
        // per-path top-K by |w| desc, ties to the lower bin (:116)
        for (int rr = 0; rr < K; rr++) {
            T bv = T(-1), bw = T(0);
            int bb = 0x7fffffff;
            for (int j = lane; j < n; j += 32) {
                bool taken = false;
                for (int t = 0; t < rr; t++) taken |= sm.cbin[p * K + t] == j;
                const T a = tabs(v[j]);
                if (!taken && (a > bv || (a == bv && j < bb))) { bv = a; bb = j; bw = v[j]; }
            }
            for (int off = 16; off >= 1; off >>= 1) {
                const T ov = __shfl_xor_sync(kFull, bv, off), ow = __shfl_xor_sync(kFull, bw, off);
                const int ob = __shfl_xor_sync(kFull, bb, off);
                if (ov > bv || (ov == bv && ob < bb)) { bv = ov; bb = ob; bw = ow; }
            }
            if (lane == 0) {
                sm.cabs[p * K + rr] = bv;
                sm.cbin[p * K + rr] = bb;
                sm.cw[p * K + rr] = bw;
            }
            __syncwarp();
        }
    }
    // pool (:119-120)
    const int PK = P * K, KEEP = PK < L ? PK : L;
    for (int c = lane; c < PK; c += 32) sm.cpm[c] = sm.pms[c / K] + T(0.5) * (sm.llrabs[c / K] - sm.cabs[c]);
    __syncwarp();
    for (int c = lane; c < PK; c += 32) {
        const T pc = sm.cpm[c];
        const int sc = c / K, bc = sm.cbin[c];
        int rank = 0;
        for (int d = 0; d < PK; d++) {
            const T pd = sm.cpm[d];
            const int sd = d / K;
            rank += (pd < pc) || (pd == pc && (sd < sc || (sd == sc && sm.cbin[d] < bc)));
        }
        if (rank < KEEP) sm.sel[rank] = c;
    }
    __syncwarp();
    T newpm = T(0);
    int newlin = 0;
    if (lane < KEEP) {
        newpm = sm.cpm[sm.sel[lane]];
        newlin = sm.sel[lane] / K;
    }
    for (int idx = lane; idx < KEEP * n; idx += 32) {
        const int o = idx / n, j = idx % n, c = sm.sel[o];
        const int b = sm.cbin[c];
        out[o * n + j] = (uint8_t)((__popc((unsigned)(~(b | j)) & (unsigned)(n - 1)) & 1) ^ (sm.cw[c] < T(0)));
    }
    __syncwarp();
    for (int o = lane; o < KEEP; o += 32) {
        sm.pms[o] = newpm;
        lin[o] = (int8_t)newlin;
    }
    __syncwarp();
    return KEEP;
}

// -------------------------------------------------------------------- SPC
template <typename T>
__device__ int spc_rt(W<T>& w, const In<T>& in, int P, int n, uint8_t* out, int8_t* lin) {
    auto& sm = *w.sm;
    const int lane = lane_id(), L = w.sh.L;
    int tau = n < L ? n : L;
    if (tau > n - 1) tau = n - 1;
    uint16_t* ord = w.spc_ord;
    uint8_t* sg = w.spc_sgn;
    for (int p = lane; p < P; p += 32) {  // one lane per path: stable argsort (:83), parity (:84-88)
        int par = 0;
        for (int j = 0; j < n; j++) {
            const T a = in.get(p, j);
            sg[p * n + j] = a < T(0);
            par ^= a < T(0);
            const T mj = tabs(a);
            int i = j - 1;
            while (i >= 0 && tabs(in.get(p, ord[p * n + i])) > mj) {
                ord[p * n + i + 1] = ord[p * n + i];
                i--;
            }
            ord[p * n + i + 1] = (uint16_t)j;
        }
        const T amin = tabs(in.get(p, ord[p * n]));
        sm.pmtmp[p] = sm.pms[p] + (par ? amin : T(0));
        sm.cabs[p] = T(par);
    }
    __syncwarp();
    if (lane == 0) {  // the tau splits (:97-112)
        T pm[2 * kMaxL], pr[2 * kMaxL];
        int parent[2 * kMaxL];
        uint32_t fl[2 * kMaxL];
        for (int i = 0; i < P; i++) {
            pm[i] = sm.pmtmp[i];
            pr[i] = sm.cabs[i];
            parent[i] = i;
            fl[i] = 0;
        }
        int cnt = P;
        for (int j = 1; j <= tau; j++) {
            T cand[4 * kMaxL];
            int sel[4 * kMaxL];
            for (int i = 0; i < cnt; i++) {
                const T aj = tabs(in.get(parent[i], ord[parent[i] * n + j]));
                const T am = tabs(in.get(parent[i], ord[parent[i] * n]));
                cand[2 * i] = pm[i];
                const T t = pm[i] + aj;
                cand[2 * i + 1] = pr[i] != T(0) ? t - am : t + am;
            }
            const int C2 = 2 * cnt;
            for (int c = 0; c < C2; c++) {
                int t = c - 1;
                while (t >= 0 && cand[sel[t]] > cand[c]) {
                    sel[t + 1] = sel[t];
                    t--;
                }
                sel[t + 1] = c;
            }
            const int Kp = C2 < L ? C2 : L;
            T npm[2 * kMaxL], npr[2 * kMaxL];
            int npa[2 * kMaxL];
            uint32_t nfl[2 * kMaxL];
            for (int o = 0; o < Kp; o++) {
                const int which = sel[o] & 1, src = sel[o] >> 1;
                npm[o] = cand[sel[o]];
                nfl[o] = fl[src] | (which ? (1u << j) : 0u);
                npr[o] = which ? T(1) - pr[src] : pr[src];
                npa[o] = parent[src];
            }
            for (int o = 0; o < Kp; o++) {
                pm[o] = npm[o];
                pr[o] = npr[o];
                parent[o] = npa[o];
                fl[o] = nfl[o];
            }
            cnt = Kp;
        }
        for (int o = 0; o < cnt; o++) {
            sm.pmtmp[o] = pm[o];
            sm.sel[o] = parent[o];
            sm.cbin[o] = (int)fl[o];
        }
        sm.spc_cnt = cnt;
    }
    __syncwarp();
    const int cnt = sm.spc_cnt;
    for (int o = lane; o < cnt; o += 32) {  // (:114-118)
        const int par = sm.sel[o];
        const uint32_t fl = (uint32_t)sm.cbin[o];
        int tot = 0;
        for (int j = 0; j < n; j++) {
            const int b = sg[par * n + j];
            out[o * n + j] = (uint8_t)b;
            tot ^= b;
        }
        for (int j = 1; j <= tau; j++)
            if (fl >> j & 1u) {
                out[o * n + ord[par * n + j]] ^= 1;
                tot ^= 1;
            }
        out[o * n + ord[par * n]] ^= (uint8_t)tot;
        lin[o] = (int8_t)par;
        sm.pms[o] = sm.pmtmp[o];
    }
    __syncwarp();
    return cnt;
}

// -------------------------------------------------- permutation extension
template <typename T>
__device__ int perm_ext_rt(W<T>& w, const In<T>& in, int P, int n, bool is_root, int level) {
    auto& sm = *w.sm;
    const int lane = lane_id(), L = w.sh.L, trials = 2 * P, H = n / 2, mn = 31 - __clz(n);
    const int base = sm.next_map;
    MapS* tcomp = w.comp + L;  // trial composites at the root (after the L root paths)
    if (is_root)
        for (int t = lane; t < trials; t += 32) {
            const MapS& tm = w.maps[base + t];
            const MapS& im = w.comp[t % P];
            MapS& o = tcomp[t];
            for (int k = 0; k < mn; k++) {
                o.icol[k] = lin_rt(im.icol, mn, tm.icol[k]);
                o.col[k] = lin_rt(tm.col, mn, im.col[k]);
            }
            o.c = lin_rt(im.icol, mn, tm.c) ^ im.c;
            o.b = lin_rt(tm.col, mn, im.b) ^ tm.b;
        }
    __syncwarp();
    for (int t = 0; t < trials; t++) {  // LM (:232-233), numpy pairwise order
        const int src = t % P;
        const MapS& mp = is_root ? tcomp[t] : w.maps[base + t];
        const T lmv = pairwise_rt<T>(H, [&](int j) {
            T x, y;
            if (is_root) {
                x = tabs(w.alpha[inv_rt(mp, mn, (uint32_t)j)]);
                y = tabs(w.alpha[inv_rt(mp, mn, (uint32_t)(j + H))]);
            } else {
                x = tabs(in.get(src, inv_rt(mp, mn, (uint32_t)j)));
                y = tabs(in.get(src, inv_rt(mp, mn, (uint32_t)(j + H))));
            }
            return y < x ? y : x;
        });
        if (lane == 0) sm.lm[t] = lmv;
    }
    __syncwarp();
    if (w.tie_fix && lane == 0)  // equal pairing directions pair the same entries
        for (int t = 1; t < trials; t++)
            for (int s2 = 0; s2 < t; s2++) {
                const uint32_t kt = is_root ? tcomp[t].icol[mn - 1] : (((uint32_t)(t % P) << 16) | w.maps[base + t].icol[mn - 1]);
                const uint32_t ks = is_root ? tcomp[s2].icol[mn - 1] : (((uint32_t)(s2 % P) << 16) | w.maps[base + s2].icol[mn - 1]);
                if (kt == ks) {
                    sm.lm[t] = sm.lm[s2];
                    break;
                }
            }
    __syncwarp();
    const int K = trials < L ? trials : L;
    for (int t = lane; t < trials; t += 32) {  // (:234)
        const T v = sm.lm[t];
        int rank = 0;
        for (int s2 = 0; s2 < trials; s2++) rank += (sm.lm[s2] > v) || (sm.lm[s2] == v && s2 < t);
        if (rank < K) sm.sel[rank] = t;
    }
    __syncwarp();
    if (is_root) {
        for (int o = lane; o < K; o += 32) w.comp[3 * L + o] = tcomp[sm.sel[o]];  // stage
        __syncwarp();
        for (int o = lane; o < K; o += 32) w.comp[o] = w.comp[3 * L + o];
    } else {
        T* dst = w.perm + w.sh.L * ((1 << level) - 1);
        for (int idx = lane; idx < K * n; idx += 32) {
            const int o = idx / n, j = idx % n, t = sm.sel[o];
            dst[o * n + j] = in.get(t % P, inv_rt(w.maps[base + t], mn, (uint32_t)j));
        }
    }
    T npm = T(0);
    if (lane < K) npm = sm.pms[sm.sel[lane] % P];
    __syncwarp();
    for (int o = lane; o < K; o += 32) {
        sm.pms[o] = npm;
        sm.l0[level][o] = (int8_t)(sm.sel[o] % P);
        sm.nmap[level][o] = (int16_t)(base + sm.sel[o]);
    }
    sm.next_map = base + trials;
    __syncwarp();
    return K;
}

// ------------------------------------------------------ explicit-stack walk
struct Frame {
    int8_t r, s, phase, perm;  // perm: 0 none, 1 root (composites), 2 inner (buffer)
    int16_t P, P1;
};

template <typename T>
__device__ int walk(W<T>& w, int P0) {
    auto& sm = *w.sm;
    const int lane = lane_id(), L = w.sh.L, MM = w.sh.m;
    Frame st[kMaxDepth];
    int sp = 0;
    st[0] = Frame{(int8_t)w.sh.r, (int8_t)MM, 0, 0, (int16_t)P0, 0};
    int ret_P = P0;
    while (sp >= 0) {
        Frame& fr = st[sp];
        const int s = fr.s, r = fr.r, n = 1 << s;
        // where this node's output goes: the parent's left/right buffer, or the root output
        uint8_t* out = sp == 0 ? w.rootout : (st[sp - 1].phase == 1 ? w.bl : w.br) + L * ((1 << (s)) - 1);
        int8_t* lin = sp == 0 ? sm.rootlin : (st[sp - 1].phase == 1 ? sm.l1[s + 1] : sm.l2[s + 1]);
        // this node's input
        In<T> in;
        if (sp == 0) {
            in = In<T>{nullptr, 0, sm.ident, w.alpha, w.comp, MM};
        } else {
            in = In<T>{w.lvl + L * ((1 << s) - 1), n, sm.ident, w.alpha, w.comp, MM};
        }
        if (r == 1 || (s >= 1 && r == s - 1)) {
            int P2;
            if (r == 1) {
                // the transform runs in place on its own (then dead) input rows; at
                // the root (r = 1: no permutation nodes) the permutation area is free
                T* scr = sp == 0 ? w.perm : w.lvl + L * ((1 << s) - 1);
                P2 = fhtl_rt(w, in, fr.P, n, scr, out, lin);
            } else {
                P2 = spc_rt(w, in, fr.P, n, out, lin);
            }
            ret_P = P2;
            sp--;
            continue;
        }
        const int h = n / 2;
        T* child = w.lvl + L * ((1 << (s - 1)) - 1);
        if (fr.phase == 0) {
            for (int i = lane; i < L; i += 32) sm.l0[s][i] = (int8_t)i;
            __syncwarp();
            int P = fr.P;
            In<T> a = in;
            const bool spine = (MM - s) == (w.sh.r - r);  // left spine of the root
            if (w.perms && spine && r >= 2 && s - r >= 2 && sm.next_map < w.sh.S) {
                const bool is_root = sp == 0;
                P = perm_ext_rt(w, in, P, n, is_root, s);
                if (!is_root) {
                    a = In<T>{w.perm + L * ((1 << s) - 1), n, sm.ident, w.alpha, w.comp, MM};
                    fr.perm = 2;
                } else {
                    fr.perm = 1;
                }
            }
            fr.P = (int16_t)P;
            for (int idx = lane; idx < P * h; idx += 32) {  // f (:100)
                const int p = idx / h, j = idx % h;
                child[idx] = rmfht::f_op(a.get(p, j), a.get(p, j + h));
            }
            __syncwarp();
            fr.phase = 1;
            st[++sp] = Frame{(int8_t)(r - 1), (int8_t)(s - 1), 0, 0, (int16_t)P, 0};
            continue;
        }
        if (fr.phase == 1) {
            const int P1 = ret_P;
            fr.P1 = (int16_t)P1;
            In<T> a = (fr.perm == 2) ? In<T>{w.perm + L * ((1 << s) - 1), n, sm.ident, w.alpha, w.comp, MM} : in;
            const int8_t* l1 = sm.l1[s];
            const uint8_t* bl = w.bl + L * ((1 << (s - 1)) - 1);
            for (int idx = lane; idx < P1 * h; idx += 32) {  // alphas[lin1] (:102), g (:104)
                const int p = idx / h, j = idx % h;
                const int rp = l1[p];
                const T x = (a.base ? a.base[rp * n + j] : w.alpha[inv_rt(w.comp[rp], MM, (uint32_t)j)]);
                const T y = (a.base ? a.base[rp * n + j + h] : w.alpha[inv_rt(w.comp[rp], MM, (uint32_t)(j + h))]);
                child[idx] = rmfht::g_op(x, y, (int)bl[idx]);
            }
            __syncwarp();
            fr.phase = 2;
            st[++sp] = Frame{(int8_t)r, (int8_t)(s - 1), 0, 0, (int16_t)P1, 0};
            continue;
        }
        // phase 2: combine (:106-107), un-permute (:109-112), lineage (:113)
        const int P2 = ret_P;
        const int8_t* l0 = sm.l0[s];
        const int8_t* l1 = sm.l1[s];
        const int8_t* l2 = sm.l2[s];
        const uint8_t* bl = w.bl + L * ((1 << (s - 1)) - 1);
        const uint8_t* br = w.br + L * ((1 << (s - 1)) - 1);
        uint8_t* dst = (fr.perm == 2) ? w.rootout : out;  // inner perm: stage, then gather
        for (int idx = lane; idx < P2 * h; idx += 32) {
            const int p = idx / h, j = idx % h;
            const uint8_t rb = br[idx];
            dst[p * n + j] = bl[l2[p] * h + j] ^ rb;
            dst[p * n + h + j] = rb;
        }
        __syncwarp();
        if (fr.perm == 2) {
            for (int idx = lane; idx < P2 * n; idx += 32) {
                const int p = idx / n, i = idx % n;
                const MapS& mp = w.maps[sm.nmap[s][l1[l2[p]]]];
                out[idx] = dst[p * n + fwd_rt(mp, s, (uint32_t)i)];
            }
            __syncwarp();
        }
        for (int p = lane; p < P2; p += 32) {
            const int ch = l1[l2[p]];
            lin[p] = l0[ch];
            if (sp == 0) sm.rootchain[p] = (int8_t)ch;
        }
        __syncwarp();
        ret_P = P2;
        sp--;
    }
    return ret_P;
}

template <typename T>
__global__ void __launch_bounds__(128) decode_kernel_generic(rmfht::Params<T> prm, Shape sh, Layout lay) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = sh.N, L = sh.L, MM = sh.m, NW = N / 32 > 0 ? N / 32 : 1, REC = 2 * MM + 2;
    T* alpha = reinterpret_cast<T*>(smem_raw);
    unsigned char* wbase = smem_raw + ((N * sizeof(T) + 15) / 16) * 16;
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), nwarps = blockDim.x >> 5, lane = lane_id();  // provably warp-uniform
    unsigned char* mine = wbase + (size_t)warp * lay.total;
    W<T> w;
    w.lvl = reinterpret_cast<T*>(mine + lay.lvl);
    w.perm = reinterpret_cast<T*>(mine + lay.perm);
    w.bl = mine + lay.bl;
    w.br = mine + lay.br;
    w.rootout = mine + lay.rootout;
    w.maps = reinterpret_cast<MapS*>(mine + lay.maps);
    w.comp = reinterpret_cast<MapS*>(mine + lay.comp);
    w.sm = reinterpret_cast<Small<T>*>(mine + lay.small);
    w.spc_ord = reinterpret_cast<uint16_t*>(mine + lay.spc_ord);
    w.spc_sgn = mine + lay.spc_sgn;
    w.alpha = alpha;
    w.sh = sh;
    w.perms = prm.perms;
    w.tie_fix = prm.tie_fix;
    auto& sm = *w.sm;
    for (int i = lane; i < kMaxL; i += 32) sm.ident[i] = (int8_t)i;
    const int Meff = prm.perms ? prm.M : 1;
    for (long long f = blockIdx.x; f < prm.B; f += gridDim.x) {
        for (int i = threadIdx.x; i < N; i += blockDim.x) alpha[i] = prm.llr[f * N + i];
        __syncthreads();
        bool have = false;
        for (int a = warp; a < Meff; a += nwarps) {
            int P;
            if (prm.perms) {
                const uint16_t* recs = prm.maps + ((size_t)f * prm.M + a) * sh.S * REC;
                for (int s = lane; s < sh.S; s += 32) {
                    const int mn = s < L ? MM : MM - (s - L) / (2 * L);
                    rmfht::load_map(w.maps[s], recs + (size_t)s * REC, MM, mn);
                }
                __syncwarp();
                for (int l = lane; l < L; l += 32) {
                    w.comp[l] = w.maps[l];
                    sm.pms[l] = T(0);
                }
                sm.next_map = L;
                P = L;
            } else {
                if (lane == 0) {
                    sm.pms[0] = T(0);
                    for (int k = 0; k < rmfht::kMaxM; k++) {
                        w.comp[0].icol[k] = 1u << k;
                        w.comp[0].col[k] = 1u << k;
                    }
                    w.comp[0].b = 0;
                    w.comp[0].c = 0;
                }
                sm.next_map = 0;
                P = 1;
            }
            __syncwarp();
            P = walk(w, P);
            int best = 0;
            for (int i = 1; i < P; i++)
                if (sm.pms[i] < sm.pms[best]) best = i;
            const T pm = sm.pms[best];
            const bool root_internal = !(sh.r == 1 || sh.r == MM - 1);
            const int mi = (root_internal && prm.perms) ? sm.rootchain[best] : sm.rootlin[best];
            const MapS& mp = w.comp[mi];
            uint32_t myword = 0;
            rmfht::CorrPm corr;
            for (int t = 0; t < NW; t++) {
                const int i = t * 32 + lane;
                int bit = 0;
                if (i < N) {
                    const uint32_t src = prm.perms ? fwd_rt(mp, MM, (uint32_t)i) : (uint32_t)i;
                    bit = w.rootout[best * N + src];
                    if constexpr (sizeof(T) == 4) corr.add((float)alpha[i], bit);
                }
                const uint32_t word = __ballot_sync(kFull, bit);
                if (lane == t) myword = word;
            }
            T rep = pm;
            if constexpr (sizeof(T) == 4) rep = (T)corr.total();
            if (prm.att_pm && lane == 0) prm.att_pm[(size_t)f * prm.M + a] = rep;
            if (prm.att_cw && lane < NW) prm.att_cw[((size_t)f * prm.M + a) * NW + lane] = myword;
            if (!have || pm < sm.best_pm) {
                if (lane < NW) sm.best_cw[lane] = myword;
                if (lane == 0) {
                    sm.best_pm = pm;
                    sm.best_rep = rep;
                    sm.best_att = a;
                    sm.best_path = best;
                }
                have = true;
            }
            __syncwarp();
        }
        if (!have && lane == 0) sm.best_att = -1;
        __syncthreads();
        if (warp == 0) {
            int bw = -1;
            if (lane == 0)
                for (int q = 0; q < nwarps; q++) {
                    const Small<T>& o = *reinterpret_cast<Small<T>*>(wbase + (size_t)q * lay.total + lay.small);
                    if (o.best_att < 0) continue;
                    const Small<T>& cur = *reinterpret_cast<Small<T>*>(wbase + (size_t)(bw < 0 ? 0 : bw) * lay.total + lay.small);
                    if (bw < 0 || o.best_pm < cur.best_pm || (o.best_pm == cur.best_pm && o.best_att < cur.best_att)) bw = q;
                }
            bw = __shfl_sync(kFull, bw, 0);
            const Small<T>& o = *reinterpret_cast<Small<T>*>(wbase + (size_t)bw * lay.total + lay.small);
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

}  // namespace rmfht_gen
