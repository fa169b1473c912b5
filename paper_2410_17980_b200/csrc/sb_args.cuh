// Kernel argument blocks shared by the launchers (sb_fwd.cu, sb_bwd.cu) and the C ABI.
#pragma once
#include "sb_common.cuh"

namespace sb {

struct FwdArgs {
  Geom g;
  __nv_bfloat16* o;
  float* log_rem;        // [B,H,L] natural log of remaining stick mass
  int32_t* first_kb;     // [B,H,nb]
  float* M;              // [B,H,n_tiles,64] a-snapshots (log2 units), nullable
  unsigned long long* counters;  // [2]: visited tiles, total tiles (nullable)
  double log_eps;        // log(skip_eps)
};

int fwd_dispatch(int D, bool skip, const CUtensorMap& tq, const CUtensorMap& tk,
                 const CUtensorMap& tv, const FwdArgs& a, cudaStream_t stream);

}  // namespace sb
