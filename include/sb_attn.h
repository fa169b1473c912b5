/* sb_attn.h — C ABI of the B200-native stick-breaking attention hot path.
 *
 * Drop-in boundary for the reference's tiled operator.
 * Plain C types only; every call is stream-ordered, never synchronises the
 * host, keeps no mutable global state (beyond one-time kernel attributes) and
 * is bit-deterministic (no atomics on the data path).  The caller allocates
 * every buffer, matching the reference's caller-owns-outputs convention
 * (blocked.py:160-163, :250, :286-287).
 *
 * Reference interfaces each entry point replaces (paths under
 * /root/reference/pkg/src/sbattn/):
 *   sb_fwd       blocked.py:129  blocked_forward(q, k, v, layout, skip, skip_eps,
 *                                two_phase)      -> (o, RowLogAccumulator, TileStats)
 *                blocked.py:218  sb_forward_blocked(q, k, v, layout, **kw)
 *   sb_bwd       blocked.py:299  blocked_backward_twophase(cache, d_o, layout,
 *                                row_offset)     -> (d_q, d_k, d_v, n_stored)
 *                (phases = 1 / 2: its two sweeps, blocked.py:337-357 / :367-386)
 *   sb_state_elems          the BlockedCache (blocked.py:90-98) the backward needs
 *                           beyond q, k, v and first_kb: O(L) per head here
 *   sb_bwd_workspace_bytes  the M / N snapshot dicts (RowLogAccumulator.m_blocks,
 *                           blocked.py:70-80, :353) + the dZ tile store, all
 *                           transient inside one backward call
 *   sb_snapshot_elems / sb_varlen_elems  blocked.py:58-60 BlockLayout.n_tiles x
 *                           d_block (one snapshot array), first_kb sizes for varlen
 *   sb_status_string        the ValueError messages of blocked.py:115-119,
 *                           :155-156, :246-247, :315-316, :398-399
 *
 * Intermediates (BASELINE north_star: "cut the O(L^2/d_block) M/N intermediates"):
 * the reference keeps one `a` snapshot per row per visited tile from the forward
 * to the backward (M, blocked.py:188-189) and one `b` snapshot per row per tile
 * between its two backward sweeps (N, :353).  Here the forward keeps only the
 * final `a` per row (float64, the `state` array: O(L)); phase 1 of the backward
 * rolls the per-tile snapshots back from it (M(kb) = a_final + the row totals of
 * -lt of tiles <= kb, recomputed from the same tile math) and hands them to
 * phase 2 inside the caller's workspace.  The store-mode backward has no N at
 * all (phase 2 reads phase 1's dZ tiles).
 */
#ifndef SB_ATTN_H
#define SB_ATTN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (0 = ok); non-zero mirror the reference's ValueError cases */
enum {
  SB_OK = 0,
  SB_ERR_SHAPE = 1,        /* q/k/v/d_o shape or stride mismatch (blocked.py:116-119, :246) */
  SB_ERR_SKIP_EPS = 2,     /* skip_eps outside (0, 1) (blocked.py:155-156) */
  SB_ERR_BLOCK = 3,        /* d_block != 64 or seq_len < 1 (blocked.py:64-65) */
  SB_ERR_UNSUPPORTED = 4,  /* head_dim not in {64, 128}, non-16B-aligned strides */
  SB_ERR_NULL = 5,         /* required pointer is NULL (e.g. missing state, blocked.py:315-316) */
  SB_ERR_DEVICE = 6,       /* no sm_100 device / driver entry point unavailable */
  SB_ERR_LAUNCH = 7        /* CUDA launch or tensor-map encoding failed */
};

/* Problem description.  q, k, v, o, d_o, dq, dk, dv are bf16 with the element
 * strides below and a contiguous last (head_dim) dimension, e.g. (B, H, L, d)
 * contiguous: stride_b = H*L*d, stride_h = L*d, stride_l = d; or (B, L, H, d):
 * stride_b = L*H*d, stride_l = H*d, stride_h = d.
 *
 * Packed variable-length batches (cu_seqlens != NULL): the tensors are
 * (total_tokens, H, d) with token stride stride_l and head stride stride_h
 * (stride_b unused); sequence b is tokens cu_seqlens[b] .. cu_seqlens[b+1]-1
 * (cu_seqlens: DEVICE int32 [batch+1], cu_seqlens[0] = 0); seqlen must be at least
 * the longest sequence (work items are counted from it: sb_bwd checks it against the
 * host offsets, sb_fwd cannot).  Every sequence is an independent problem
 * whose 64-blocks start at its first token.  Per-row outputs (log_rem,
 * row_offset) are then (total_tokens, H); first_kb and M/N are packed sequence
 * by sequence, head-major (sizes: sb_varlen_elems). */
typedef struct sb_params {
  int32_t batch, heads, seqlen, head_dim;
  int64_t stride_b, stride_h, stride_l;
  const int32_t* cu_seqlens; /* NULL: uniform batch; else packed varlen (device pointer) */
  float scale;               /* logit scale; 0 selects 1/sqrt(head_dim) (blocked.py:159) */
  int32_t block;             /* skip / snapshot granularity; must be 64 (blocked.py:41) */
  int32_t skip;              /* enable block skipping (blocked.py:175-176) */
  float skip_eps;            /* in (0, 1); 0 selects 1e-6 (blocked.py:43) */
  int32_t total_tokens;      /* varlen only: rows of the packed tensors */
} sb_params_t;

/* Float elements of ONE snapshot array (M or N) of a uniform batch: 64 (header)
 * + batch * heads * n_tiles * 64 with n_tiles = nb*(nb+1)/2, nb = ceil(L/64);
 * 0 for varlen batches (use sb_varlen_elems). */
size_t sb_snapshot_elems(const sb_params_t* p);

/* Float elements of the forward's state array (the only O(L)-sized thing the
 * backward needs from the forward besides first_kb): 64 + 2 * rows (the final
 * a of every row as float64), rows = batch*heads*seqlen, or total_tokens*heads
 * for varlen.  16-byte aligned. */
size_t sb_state_elems(const sb_params_t* p);

/* Varlen sizes from a HOST copy of cu_seqlens ([batch+1]): *snapshot = floats of
 * one snapshot array (64 + heads * sum_b n_tiles(L_b) * 64), *first_kb = int32
 * elements of first_kb (heads * sum_b nb(L_b)).  Returns SB_OK or SB_ERR_SHAPE
 * (decreasing offsets). */
int sb_varlen_elems(const sb_params_t* p, const int32_t* cu_seqlens_host, size_t* snapshot,
                    size_t* first_kb);

/* Forward.  Outputs: o (bf16, q's layout), log_rem [B,H,L] float (natural log of
 * the remaining stick mass, RowLogAccumulator.a), first_kb [B,H,nb] int32
 * (TileStats.first_kb), state (sb_state_elems floats, opaque; required by sb_bwd),
 * tile_counters (nullable) += {visited} (TileStats.visited).  stream is a
 * cudaStream_t (NULL = legacy default stream).
 * state may be NULL: a forward for inference, the reference's
 * blocked_forward(two_phase=False) (blocked.py:136, :163, :188); o, log_rem and
 * first_kb are identical, only sb_bwd cannot follow it.  No call writes anything
 * O(L^2/64) sized. */
int sb_fwd(const sb_params_t* p, const void* q, const void* k, const void* v, void* o,
           float* log_rem, int32_t* first_kb, float* state, unsigned long long* tile_counters,
           void* stream);

/* Bytes of the backward's workspace: the M snapshots (+ header), then either
 * (store != 0) the dZ tiles phase 1 writes for phase 2 (bf16, 16 KB per 128-row x
 * 64-key tile, n_qt*(n_qt+1) per (b,h) unit, n_qt = ceil(L/128)) or (store == 0,
 * recompute mode: phase 2 recomputes dO.V^T and dZ) the N snapshots.  Same
 * results bit for bit either way.  cu_seqlens_host: host offsets for varlen
 * batches (else NULL).  0 if the sizes cannot be computed. */
size_t sb_bwd_workspace_bytes(const sb_params_t* p, const int32_t* cu_seqlens_host, int store);

/* Two-phase backward.  row_offset (nullable) [B,H,L] float is the per-row offset
 * subtracted from dO.V^T (blocked.py:241-242, :274-276); state and first_kb come
 * from sb_fwd on the same inputs (sb_bwd reads only the per-row part past the
 * 64-float header).  workspace: device, 128-byte aligned, at least
 * sb_bwd_workspace_bytes(p, cu_seqlens_host, store) bytes (checked: SB_ERR_SHAPE;
 * varlen batches must pass cu_seqlens_host).  phases = 3 runs both sweeps; 1 runs
 * phase 1 (dq, the M snapshots and the dZ tiles or N, blocked.py:337-357); 2 runs
 * phase 2 (dk, dv, blocked.py:367-386) and must follow phase 1 on the stream with
 * the same workspace.  Writes dq, dk, dv (bf16, q's layout). */
int sb_bwd(const sb_params_t* p, const void* q, const void* k, const void* v, const void* d_o,
           const float* row_offset, const float* state, const int32_t* first_kb, void* dq,
           void* dk, void* dv, void* workspace, size_t workspace_bytes,
           const int32_t* cu_seqlens_host, int store, int phases, void* stream);

const char* sb_status_string(int status);
int sb_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SB_ATTN_H */
