/*
 * rmfht.h — C ABI of the B200 batched p-FHT-FSCL-L-M decoder
 * (librmfht.so, paper_2108_12550_b200/csrc).
 *
 * The reference (arXiv 2108.12550 workbench, pkg/src/rmworkbench) is a pure
 * Python package with no FFI; its boundary for this path is the Python
 * function family in top_decoders.py, which this ABI replaces:
 *
 *   decode(spec, alpha, cfg, rng)                  top_decoders.py:252-271
 *   ensemble_decode(spec, alpha, L, M, rng, sampler)  top_decoders.py:190-202
 *   p_fht_fscl(spec, alpha, L, rng, sampler)       top_decoders.py:178-187
 *   fht_fscl_decode / fht_fsc_decode               top_decoders.py:170-175
 *   sampler: () -> AffinePermutation  (plugin hook, automorphism.py:225-226,
 *                                      top_decoders.py:129-130)
 *
 * The Python mirror (paper_2108_12550_b200/top_decoders.py) binds these
 * entry points with ctypes; INTEGRATION.md shows the binding.
 *
 * Conventions: all device pointers are caller-owned, including the launch
 * workspace (rmfht_workspace_bytes); launches are ordered on the given
 * cudaStream_t (passed as void*) with no host synchronisation and no device
 * allocation; plans hold no device memory and no mutable state after their
 * one-time kernel setup, so one plan may be launched from several threads
 * and streams at once (each launch with its own workspace).  Like the
 * reference functions (pure, top_decoders.py:252-282) a launch reads its
 * inputs and writes only its outputs and its workspace.
 * Every function returns 0 on success and a negative code on error, with a
 * one-line message from rmfht_last_error() (thread-local).
 */
#ifndef RMFHT_H
#define RMFHT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rmfht_plan rmfht_plan;

/* dtype: arithmetic of the decoder.  F32 is the throughput path; F64
 * reproduces the float64 reference bit-for-bit. */
enum { RMFHT_F32 = 0, RMFHT_F64 = 1 };

/* flags */
enum {
    RMFHT_PERMUTATIONS = 1,   /* p-FHT-FSCL (else FHT-FSCL / FHT-FSC, M forced to 1) */
    RMFHT_TIE_FIX = 2,        /* equal pairing directions keep equal LM (default for F32) */
    RMFHT_NO_TIE_FIX = 4,     /* force it off (default for F64) */
    RMFHT_REFERENCE_ORDER = 8, /* F32: use the reference-operation-order kernel instead of the
                                  throughput kernel (whose LM / llr_abs summation orders differ) */
    RMFHT_NO_LOCKSTEP = 16,    /* throughput kernel: no barrier between rounds of work items */
    RMFHT_LOCKSTEP_4 = 32,     /* ... barrier per group of 4 warps instead of the whole CTA */
    RMFHT_LOCKSTEP_8 = 64,     /* ... per group of 8 warps */
    RMFHT_GENERIC = 128,       /* use the generic runtime-shaped kernel even if a specialisation exists */
    RMFHT_AUT_SSC = 256        /* Aut-SSC (aut_ssc, top_decoders.py:235-249): with RMFHT_PERMUTATIONS
                                  and L = 1, M = P SSC decodes per frame, one map of m variables each
                                  (S = 1); d_pm receives the winning correlation, d_attempt the
                                  winning decode (first strictly largest score), d_path 0; the diag
                                  outputs hold every decode's score and codeword.  m <= 10. */
};

enum {
    RMFHT_OK = 0,
    RMFHT_ECONFIG = -1,       /* ConfigurationError (rm_core.py:72-77, top_decoders.py:38-42) */
    RMFHT_EVALUE = -2,        /* ValueError: bad sizes / singular map (top_decoders.py:120-121) */
    RMFHT_EUNSUPPORTED = -3,  /* valid configuration with no compiled kernel */
    RMFHT_ECUDA = -4          /* CUDA runtime error */
};

/* Validate (r, m, L, M) like build_code + DecoderConfig and bind the kernel
 * specialised on the static node schedule (accounting.plan_visits,
 * accounting.py:96-123). */
int rmfht_plan_create(int r, int m, int L, int M, int flags, int dtype, rmfht_plan **out);
void rmfht_plan_destroy(rmfht_plan *plan);

/* Permutation-table layout: S maps per attempt, in the reference's
 * consumption order (L root maps, top_decoders.py:129-132; then 2L maps per
 * permutation node, automorphism.py:224-228).  sizes[s] = variables of map s. */
int rmfht_plan_maps_per_attempt(const rmfht_plan *plan);
int rmfht_plan_map_sizes(const rmfht_plan *plan, int *sizes);
int rmfht_plan_record_u16(const rmfht_plan *plan); /* 2m+2 */

/* Host: convert `count` raw maps (m+1 uint16 each: row masks of A, bit j of
 * row r = A[r, j] (automorphism.py:122-124), then b at index m) laid out as
 * [.., S, m+1] into device records [.., S, 2m+2] (columns of A, b, columns
 * of A^-1, A^-1 b).  Fails with RMFHT_EVALUE on a singular A. */
int rmfht_expand_maps(const rmfht_plan *plan, const uint16_t *raw, uint16_t *rec, long long count);

/* Host: sample the permutation table of frames frame0 .. frame0+B-1 —
 * uniform (A, b) in GL(m_node, 2) x F_2^m_node per slot (the reference
 * sampler's distribution, automorphism.py:127-161; A drawn column by column,
 * each uniform outside the span of the previous ones), from a
 * counter-based stream keyed by (seed, frame, attempt, slot), so a frame's
 * maps do not depend on the batch it is drawn in.  identity_root != 0 makes
 * attempt 0's L root maps the identity ("decoder 0 = identity").  Writes raw
 * maps [B, M, S, m+1] and/or device records [B, M, S, 2m+2] (either may be
 * NULL).  Multithreaded (OpenMP). */
int rmfht_sample_maps(const rmfht_plan *plan, uint64_t seed, long long frame0, long long B,
                      int identity_root, uint16_t *raw, uint16_t *rec);

/* Device: the same table as rmfht_sample_maps (bit-identical), written as
 * device records straight to d_rec [B, M, S, 2m+2]; stream-ordered. */
int rmfht_sample_maps_device(const rmfht_plan *plan, uint64_t seed, long long frame0, long long B,
                             int identity_root, uint16_t *d_rec, void *stream);

/* Bytes of device workspace a launch of B frames needs: the throughput
 * kernel's per-(frame, attempt) records and, with sampled != 0
 * (rmfht_decode_launch_sampled), the drawn permutation table.  0 when the
 * plan's kernel needs none.  Negative on error. */
long long rmfht_workspace_bytes(const rmfht_plan *plan, long long B, int sampled);

/* Decode B frames whose permutations are drawn on the device from
 * (seed, frame0 + frame index) — no host table ("NULL for
 * on-device sampling with (seed, frame_offset)").  The table lives in the
 * caller's workspace d_work (rmfht_workspace_bytes(plan, B, 1) bytes,
 * 256-byte aligned); RMFHT_EVALUE if it is missing or too small. */
int rmfht_decode_launch_sampled(const rmfht_plan *plan, const void *d_llr, uint64_t seed, long long frame0,
                                int identity_root, uint32_t *d_cw, void *d_pm, int32_t *d_attempt,
                                int32_t *d_path, long long B, void *d_work, long long work_bytes, void *stream);

/* Decode B frames.  d_llr [B, 2^m] float or double (per dtype); d_maps
 * [B, M, S, 2m+2] records (ignored without RMFHT_PERMUTATIONS); outputs
 * d_cw [B, max(1, 2^m/32)] bit-packed codewords (bit i%32 of word i/32),
 * d_pm [B] (dtype), d_attempt [B] selected attempt (first strict minimum,
 * top_decoders.py:200), d_path [B] selected path within it (:152).
 * d_work: rmfht_workspace_bytes(plan, B, 0) bytes (may be NULL when that is 0). */
int rmfht_decode_launch(const rmfht_plan *plan, const void *d_llr, const uint16_t *d_maps,
                        uint32_t *d_cw, void *d_pm, int32_t *d_attempt, int32_t *d_path,
                        long long B, void *d_work, long long work_bytes, void *stream);

/* As above, also writing every attempt's (pm, codeword): d_att_pm [B, M],
 * d_att_cw [B, M, max(1, 2^m/32)] (either may be NULL). */
int rmfht_decode_launch_diag(const rmfht_plan *plan, const void *d_llr, const uint16_t *d_maps,
                             uint32_t *d_cw, void *d_pm, int32_t *d_attempt, int32_t *d_path,
                             void *d_att_pm, uint32_t *d_att_cw, long long B, void *d_work,
                             long long work_bytes, void *stream);

/* On-device frames: B frames frame0 .. frame0+B-1 of SNR
 * point `point` — uniform info bits of RM(r, m) (rm_core.py:182-186), polar
 * transform (rm_core.py:102-118), BPSK + AWGN with standard deviation sigma
 * by the inverse-CDF method, LLR = 2y/sigma^2 (channel_model.py:41-61; the
 * per-frame pipeline of harness.py:103-107).  Counter-based streams keyed by
 * (seed, point, frame).  Writes d_llr [B, 2^m] float32 and the transmitted
 * codewords d_tx [B, max(1, 2^m/32)] bit-packed like d_cw. */
int rmfht_gen_frames(int r, int m, uint64_t seed, long long point, long long frame0, long long B, double sigma,
                     int zero_noise, float *d_llr, uint32_t *d_tx, void *stream);

/* Error counting (harness.py:79-84,109-112): for each of B frames, if d_cw
 * differs from d_tx, d_counts[0] += 1, and if also corr(cw) >= corr(tx),
 * corr(c) = sum (1-2c) llr (top_decoders.py:231), d_counts[1] += 1
 * (maximum-likelihood lower bound).  d_counts: 2 x uint64, accumulated. */
int rmfht_count_errors(int m, const float *d_llr, const uint32_t *d_tx, const uint32_t *d_cw, long long B,
                       unsigned long long *d_counts, void *stream);

/* Kernel launches per rmfht_decode_launch call (for the bench's launch count). */
int rmfht_plan_launches_per_call(const rmfht_plan *plan);

/* Which kernel the plan runs: 1 = reference-order (rmfht_kernels.cuh),
 * 2 = float32 throughput kernel (rmfht_fast.cuh), 3 = generic runtime-shaped
 * kernel (rmfht_generic.cuh, reference order), 4 = Aut-SSC (rmfht_ssc.cu),
 * 5 = lane-per-frame FHT-FSC kernel for N <= 64 (rmfht_lane.cuh),
 * 6 = pair kernel, r = 2, L = 2, N <= 128 (rmfht_pair.cuh),
 * 7 = lane-group kernel, r = 2, L = 1, m = 8 or 9, M a multiple of 4
 * (rmfht_grp.cuh); 0 for a NULL plan. */
int rmfht_plan_kernel(const rmfht_plan *plan);

const char *rmfht_last_error(void);
int rmfht_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RMFHT_H */
