// Kernel argument blocks shared by the launchers (sb_fwd_pp.cu, sb_bwd.cu) and the C ABI.
#pragma once
#include "sb_common.cuh"

namespace sb {

struct FwdArgs {
  Geom g;
  __nv_bfloat16* o;
  float* log_rem;        // [B,H,L] natural log of remaining stick mass
  int32_t* first_kb;     // [B,H,nb]
  double* state;         // [B,H,L] final a per row (log2 units, float64): the O(L) state
                         // the backward rolls the M snapshots back from; nullable
  unsigned long long* counters;  // [2]: visited tiles, total tiles (nullable)
  float log_eps2_hi;     // log2(skip_eps) as a float pair (hi + lo)
  float log_eps2_lo;
  uint32_t* trace;       // SB_TRACE builds only (libsbattn_trace.so); null otherwise
  unsigned* sched;       // work-queue counter (state header), zeroed before the launch
};

struct BwdArgs {
  Geom g;
  __nv_bfloat16* dq;
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  const float* row_offset;  // [B,H,L] or null
  const int32_t* first_kb;  // [B,H,nb] from the forward
  const double* state;      // [B,H,L] the forward's final a per row (log2 units)
  float* M;                 // a-snapshots (log2 units): phase 1 writes, phase 2 reads
  float* N;                 // phase-1 b snapshots, read by the recompute-mode phase 2
  const __nv_bfloat16* q;   // raw q / k rows: phase 1's rare exact lt path (a logit with
  const __nv_bfloat16* k;   // 2^z = inf needs z itself)
  uint32_t* trace;          // SB_TRACE builds only (libsbattn_trace.so); null otherwise
  unsigned* sched;          // work-queue counters [2] (M header), zeroed before the launch
};

// Event timeline for kernel tuning (tools/trace_kernels.py).  Compiled only with
// -DSB_TRACE: slot = (CTA < kTraceCtas, role < 4, tile < 64, event < 16) -> SM clock.
constexpr int kTraceCtas = 4;
#ifdef SB_TRACE
#define SB_TR(args, role, j, ev)                                                          \
  do {                                                                                    \
    if ((args).trace && blockIdx.x < kTraceCtas && (j) < 64)                              \
      (args).trace[((blockIdx.x * 4 + (role)) * 64 + (j)) * 16 + (ev)] = (uint32_t)clock(); \
  } while (0)
#else
#define SB_TR(args, role, j, ev) do { } while (0)
#endif

// store = dZ tile workspace mode (tz maps it; phase 1 writes, phase 2 reads)
int bwd_dispatch(int D, const CUtensorMap& tq, const CUtensorMap& tdo, const CUtensorMap& tk,
                 const CUtensorMap& tv, const CUtensorMap& tz, const BwdArgs& a, int phases,
                 bool store, cudaStream_t stream);
int fwd_pp_dispatch(int D, bool skip, const CUtensorMap& tq, const CUtensorMap& tk,
                    const CUtensorMap& tv, const FwdArgs& a, cudaStream_t stream);

}  // namespace sb
