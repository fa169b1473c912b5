// C-ABI entry points (include/sb_attn.h): validation mirroring the reference's
// ValueErrors, TMA tensor-map encoding and kernel dispatch.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "../../include/sb_attn.h"
#include "sb_args.cuh"

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  // function-local static: initialised once, thread-safe (C++11)
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
  }();
  return fn;
}

// The tensor-map encoder is a driver call and needs a current context on the calling
// thread.  A thread that has only run cached-allocator work (torch's autograd worker
// calling the backward) may have the right current device but no context bound yet:
// cudaSetDevice on the current device binds its primary context without changing it.
int ensure_context() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaSetDevice(dev) != cudaSuccess)
    return SB_ERR_DEVICE;
  return SB_OK;
}

// 4-D map over (d, L, H, B) of a bf16 tensor; box = 64 columns x rows.
int make_map(CUtensorMap* m, const void* ptr, const sb_params_t* p, int rows) {
  auto fn = encode_fn();
  if (!fn) return SB_ERR_DEVICE;
  // varlen: one (total_tokens, H) "batch"; kernels add the sequence's first row
  const bool vl = p->cu_seqlens != nullptr;
  const cuuint64_t dims[4] = {(cuuint64_t)p->head_dim,
                              (cuuint64_t)(vl ? p->total_tokens : p->seqlen),
                              (cuuint64_t)p->heads, (cuuint64_t)(vl ? 1 : p->batch)};
  // strides of singleton dimensions are never dereferenced; keep them legal
  auto legal = [](int64_t s_el, int n, int64_t fallback) -> cuuint64_t {
    int64_t s = s_el * 2;
    if (n == 1 && (s <= 0 || s % 16)) s = fallback;
    return (cuuint64_t)s;
  };
  const int64_t fb = (int64_t)p->head_dim * 2 * 16;
  const cuuint64_t strides[3] = {
      legal(p->stride_l, (int)dims[1], fb), legal(p->stride_h, p->heads, fb),
      legal(vl ? 0 : p->stride_b, (int)dims[3], fb)};
  const cuuint32_t box[4] = {64, (cuuint32_t)rows, 1, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS && std::getenv("SB_DEBUG"))
    std::fprintf(stderr, "make_map: %d ptr %p dims %llu %llu %llu %llu strides %llu %llu %llu rows %d\n",
                 (int)r, ptr, (unsigned long long)dims[0], (unsigned long long)dims[1],
                 (unsigned long long)dims[2], (unsigned long long)dims[3],
                 (unsigned long long)strides[0], (unsigned long long)strides[1],
                 (unsigned long long)strides[2], rows);
  return r == CUDA_SUCCESS ? SB_OK : SB_ERR_LAUNCH;
}

// 3-D map over the dZ tile workspace: 64 bf16 columns x 128 rows x n_tiles, the
// 128B-swizzled smem image of a tile (store mode of the backward).
int make_tile_map(CUtensorMap* m, void* ptr, size_t bytes) {
  auto fn = encode_fn();
  if (!fn) return SB_ERR_DEVICE;
  const cuuint64_t dims[3] = {64, 128, (cuuint64_t)(bytes / sb::kZTileBytes)};
  const cuuint64_t strides[2] = {128, (cuuint64_t)sb::kZTileBytes};
  const cuuint32_t box[3] = {64, 128, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, ptr, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS && std::getenv("SB_DEBUG"))
    std::fprintf(stderr, "make_tile_map: %d ptr %p bytes %zu\n", (int)r, ptr, bytes);
  return r == CUDA_SUCCESS ? SB_OK : SB_ERR_LAUNCH;
}

int validate(const sb_params_t* p) {
  if (!p) return SB_ERR_NULL;
  if (p->cu_seqlens && p->total_tokens < 1) return SB_ERR_SHAPE;
  if (p->block != 64) return SB_ERR_BLOCK;
  if (p->seqlen < 1 || p->batch < 1 || p->heads < 1) return SB_ERR_BLOCK;
  if (p->head_dim != 64 && p->head_dim != 128) return SB_ERR_UNSUPPORTED;
  if (p->skip && !(p->skip_eps == 0.0f || (p->skip_eps > 0.0f && p->skip_eps < 1.0f)))
    return SB_ERR_SKIP_EPS;
  // the skip-on forward packs a warpgroup's stop tile into 13 bits (sb_fwd_pp.cu)
  if (p->skip && (p->seqlen + 63) / 64 >= 8192) return SB_ERR_UNSUPPORTED;
  for (int64_t s : {p->stride_l, p->stride_h, p->stride_b})
    if (s < 0) return SB_ERR_SHAPE;
  if ((p->stride_l * 2) % 16 || (p->heads > 1 && (p->stride_h * 2) % 16) ||
      (!p->cu_seqlens && p->batch > 1 && (p->stride_b * 2) % 16))
    return SB_ERR_UNSUPPORTED;
  return SB_OK;
}

sb::Geom geom(const sb_params_t* p) {
  sb::Geom g;
  g.B = p->batch;
  g.H = p->heads;
  g.L = p->seqlen;
  g.nb = (p->seqlen + 63) / 64;
  g.n_qt = (p->seqlen + 127) / 128;
  g.n_tiles = (int64_t)g.nb * (g.nb + 1) / 2;
  const float scale = p->scale != 0.0f ? p->scale : (float)(1.0 / std::sqrt((double)p->head_dim));
  g.scale_log2 = scale * sb::kLog2e;
  g.sb = p->stride_b;
  g.sh = p->stride_h;
  g.sl = p->stride_l;
  g.cu = p->cu_seqlens;
  // grouped_order: units per group such that the group's K and V (bf16) fit a
  // 16 MiB slice of the 126 MB L2 (at least 8 units; measured best for phase 2 at
  // C2).  A small problem (fewer than ~4 forward items per SM: strong-scaling
  // shares, short varlen batches) is one group in global longest-first order
  // instead, so its heaviest items all start first.
  // (varlen: the mean sequence length, so a group holds about as many tokens)
  const int64_t len = (p->cu_seqlens && p->batch > 0) ? p->total_tokens / p->batch : p->seqlen;
  const int64_t unit_bytes = 4 * std::max<int64_t>(1, len) * p->head_dim;
  const int64_t bh = (int64_t)p->batch * p->heads;
  const int64_t fwd_items = (int64_t)((g.n_qt + 1) / 2) * bh;
  int64_t ug = std::max<int64_t>(8, (16ll << 20) / unit_bytes);
  if (fwd_items < 4 * 148) ug = bh;
  g.ugroup = (int)std::max<int64_t>(1, std::min<int64_t>(bh, ug));
  return g;
}

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; }

uint32_t* g_trace = nullptr;  // SB_TRACE builds: set by sb_debug_set_trace

// Snapshot floats (header + one float per row per tile) of a uniform batch or, with
// host offsets, of a packed varlen batch; -1 on bad offsets.
int64_t snapshot_floats(const sb_params_t* p, const int32_t* cu_host) {
  if (!p->cu_seqlens) {
    const int64_t nb = (p->seqlen + 63) / 64;
    return sb::kSchedHeader + (int64_t)p->batch * p->heads * (nb * (nb + 1) / 2) * 64;
  }
  if (!cu_host) return -1;
  int64_t tiles = 0;
  for (int b = 0; b < p->batch; ++b) {
    const int64_t L = cu_host[b + 1] - cu_host[b];
    if (L < 0) return -1;
    const int64_t nb = (L + 63) / 64;
    tiles += nb * (nb + 1) / 2;
  }
  return sb::kSchedHeader + (int64_t)p->heads * tiles * 64;
}

// dZ tiles (store mode) of a uniform or (host offsets) varlen batch; -1 on bad offsets.
int64_t ztile_count(const sb_params_t* p, const int32_t* cu_host) {
  if (!p->cu_seqlens) {
    const int64_t nq = (p->seqlen + 127) / 128;
    return (int64_t)p->batch * p->heads * nq * (nq + 1);
  }
  if (!cu_host) return -1;
  int64_t tiles = 0;
  for (int b = 0; b < p->batch; ++b) {
    const int64_t nq = (cu_host[b + 1] - cu_host[b] + 127) / 128;
    tiles += (int64_t)p->heads * nq * (nq + 1);
  }
  return tiles;
}

constexpr int64_t kWsAlign = 1024;
int64_t round_up(int64_t x) { return (x + kWsAlign - 1) / kWsAlign * kWsAlign; }

}  // namespace

extern "C" {

size_t sb_snapshot_elems(const sb_params_t* p) {
  if (!p || p->seqlen < 1 || p->cu_seqlens) return 0;
  return (size_t)snapshot_floats(p, nullptr);
}

size_t sb_state_elems(const sb_params_t* p) {
  if (!p || p->seqlen < 1) return 0;
  const int64_t rows = p->cu_seqlens ? (int64_t)p->total_tokens * p->heads
                                     : (int64_t)p->batch * p->heads * p->seqlen;
  return (size_t)(sb::kSchedHeader + 2 * rows);
}

int sb_varlen_elems(const sb_params_t* p, const int32_t* cu, size_t* snapshot,
                    size_t* first_kb) {
  if (!p || !cu || !snapshot || !first_kb) return SB_ERR_NULL;
  size_t nbs = 0;
  for (int b = 0; b < p->batch; ++b) {
    const int L = cu[b + 1] - cu[b];
    if (L < 0) return SB_ERR_SHAPE;
    nbs += (size_t)(L + 63) / 64;
  }
  sb_params_t q = *p;
  q.cu_seqlens = cu;  // any non-NULL: varlen sizing from the host offsets
  *snapshot = (size_t)snapshot_floats(&q, cu);
  *first_kb = (size_t)p->heads * nbs;
  return SB_OK;
}

int sb_fwd(const sb_params_t* p, const void* q, const void* k, const void* v, void* o,
           float* log_rem, int32_t* first_kb, float* state, unsigned long long* tile_counters,
           void* stream) {
  int st = validate(p);
  if (st) return st;
  // state == NULL: forward for inference (blocked_forward(two_phase=False),
  // blocked.py:136, :163, :188); the backward then cannot run on this forward
  if (!q || !k || !v || !o || !log_rem || !first_kb) return SB_ERR_NULL;
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o)) return SB_ERR_UNSUPPORTED;
  if (state && !aligned16(state)) return SB_ERR_UNSUPPORTED;
  CUtensorMap tq, tk, tv;
  if ((st = ensure_context()) || (st = make_map(&tq, q, p, 128)) || (st = make_map(&tk, k, p, 64)) ||
      (st = make_map(&tv, v, p, 64)))
    return st;
  sb::FwdArgs a;
  a.g = geom(p);
  a.o = reinterpret_cast<__nv_bfloat16*>(o);
  a.log_rem = log_rem;
  a.first_kb = first_kb;
  a.state = state ? reinterpret_cast<double*>(state + sb::kSchedHeader) : nullptr;
  a.counters = tile_counters;
  const double eps = p->skip_eps != 0.0f ? (double)p->skip_eps : 1e-6;
  const double le2 = std::log(eps) / std::log(2.0);
  a.log_eps2_hi = (float)le2;
  a.log_eps2_lo = (float)(le2 - (double)a.log_eps2_hi);
  a.trace = g_trace;
  a.sched = reinterpret_cast<unsigned*>(state);  // NULL: items dealt statically
  int rc = sb::fwd_pp_dispatch(p->head_dim, p->skip != 0, tq, tk, tv, a,
                               reinterpret_cast<cudaStream_t>(stream));
  return rc ? SB_ERR_LAUNCH : SB_OK;
}

size_t sb_bwd_workspace_bytes(const sb_params_t* p, const int32_t* cu_host, int store) {
  if (!p || p->seqlen < 1) return 0;
  const int64_t m = snapshot_floats(p, cu_host), z = ztile_count(p, cu_host);
  if (m < 0 || z < 0) return 0;
  const int64_t mb = round_up(m * 4);
  return (size_t)(store ? mb + z * sb::kZTileBytes : mb + m * 4);
}

int sb_bwd(const sb_params_t* p, const void* q, const void* k, const void* v, const void* d_o,
           const float* row_offset, const float* state, const int32_t* first_kb, void* dq,
           void* dk, void* dv, void* workspace, size_t workspace_bytes,
           const int32_t* cu_seqlens_host, int store, int phases, void* stream) {
  if (phases < 1 || phases > 3) return SB_ERR_SHAPE;
  int st = validate(p);
  if (st) return st;
  if (!q || !k || !v || !d_o || !first_kb || !dq || !dk || !dv || !workspace) return SB_ERR_NULL;
  if (!state) return SB_ERR_NULL;  // blocked.py:315-316: the forward's state is missing
  if (p->cu_seqlens && !cu_seqlens_host) return SB_ERR_NULL;  // varlen sizes need the offsets
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(d_o) || !aligned16(dq) ||
      !aligned16(dk) || !aligned16(dv) || !aligned16(state) ||
      (reinterpret_cast<uintptr_t>(workspace) & 127))
    return SB_ERR_UNSUPPORTED;
  if (p->cu_seqlens) {
    // the host offsets must describe the batch the kernels see: every sequence within
    // seqlen (item counts come from it) and the last offset at total_tokens
    if (cu_seqlens_host[0] != 0 || cu_seqlens_host[p->batch] != p->total_tokens)
      return SB_ERR_SHAPE;
    for (int b = 0; b < p->batch; ++b)
      if (cu_seqlens_host[b + 1] - cu_seqlens_host[b] > p->seqlen) return SB_ERR_SHAPE;
  }
  const size_t need = sb_bwd_workspace_bytes(p, cu_seqlens_host, store);
  if (need == 0 || workspace_bytes < need) return SB_ERR_SHAPE;
  const int64_t m = snapshot_floats(p, cu_seqlens_host), mb = round_up(m * 4);
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  CUtensorMap tq, tdo, tk, tv, tz;
  if ((st = ensure_context()) || (st = make_map(&tq, q, p, 128)) || (st = make_map(&tdo, d_o, p, 128)) ||
      (st = make_map(&tk, k, p, 64)) || (st = make_map(&tv, v, p, 64)))
    return st;
  std::memset(&tz, 0, sizeof(tz));
  if (store && (st = make_tile_map(&tz, ws + mb, (size_t)ztile_count(p, cu_seqlens_host) *
                                                   sb::kZTileBytes)))
    return st;
  sb::BwdArgs a;
  a.g = geom(p);
  a.dq = reinterpret_cast<__nv_bfloat16*>(dq);
  a.dk = reinterpret_cast<__nv_bfloat16*>(dk);
  a.dv = reinterpret_cast<__nv_bfloat16*>(dv);
  a.row_offset = row_offset;
  a.first_kb = first_kb;
  a.state = reinterpret_cast<const double*>(state + sb::kSchedHeader);
  // workspace: M snapshots (written by phase 1; their header holds the work-queue
  // counters), then the dZ tiles (store mode) or the N snapshots (recompute mode)
  a.M = reinterpret_cast<float*>(ws);
  a.N = store ? nullptr : reinterpret_cast<float*>(ws + mb);
  a.q = reinterpret_cast<const __nv_bfloat16*>(q);
  a.k = reinterpret_cast<const __nv_bfloat16*>(k);
  a.trace = g_trace;
  a.sched = reinterpret_cast<unsigned*>(ws);
  int rc = sb::bwd_dispatch(p->head_dim, tq, tdo, tk, tv, tz, a, phases, store != 0,
                            reinterpret_cast<cudaStream_t>(stream));
  if (rc && std::getenv("SB_DEBUG"))
    std::fprintf(stderr, "sb_bwd: dispatch error %d (%s)\n", rc, cudaGetErrorString((cudaError_t)rc));
  return rc ? SB_ERR_LAUNCH : SB_OK;
}

const char* sb_status_string(int s) {
  switch (s) {
    case SB_OK: return "ok";
    case SB_ERR_SHAPE: return "q, k, v (and d_o) must share one layout and shape";
    case SB_ERR_SKIP_EPS: return "skip_eps must be in (0, 1)";
    case SB_ERR_BLOCK: return "seq_len, batch, heads must be >= 1 and d_block must be 64";
    case SB_ERR_UNSUPPORTED: return "unsupported configuration (head_dim must be 64 or 128, "
                                    "16-byte aligned rows and strides)";
    case SB_ERR_NULL: return "required pointer is NULL (the two-phase backward needs the forward's "
                             "state; varlen needs host cu_seqlens)";
    case SB_ERR_DEVICE: return "CUDA driver entry point unavailable (no sm_100 device?)";
    case SB_ERR_LAUNCH: return "CUDA launch failed";
    default: return "unknown status";
  }
}

int sb_version(void) { return 5; }  // 2: packed varlen; 3: dZ tile workspace (sb_bwd_ws);
                                    // 4: M-free inference forward, N-free store mode;
                                    // 5: O(L) forward state, M rolled back in phase 1,
                                    //    one sb_bwd with a caller-sized workspace

#ifdef SB_TRACE
// debug builds only: device buffer of kTraceCtas*4*64*16 uint32 clock stamps
void sb_debug_set_trace(void* buf) { g_trace = reinterpret_cast<uint32_t*>(buf); }
#endif

}  // extern "C"
