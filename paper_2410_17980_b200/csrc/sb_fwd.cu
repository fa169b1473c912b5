// Stick-breaking attention forward (K1 of SURVEY.md §2.2) for sm_100a.
//
// Restates blocked_forward (reference blocked.py:129-206, two_phase=True):
// per query block, key blocks right to left,
//     z = q k^T * scale,  lt = -softplus(z) (0 where masked),
//     A = exp(z + suffix_cumsum(lt) + a),  O += A V,  a += rowsum(lt)
// with the optional skip check `max_rows(a) < log(eps)` before every key
// block left of the diagonal (blocked.py:175-176), M snapshots (a in effect per
// tile, blocked.py:188-189) and first_kb (blocked.py:192, :202).
//
// One CTA = one (b, h, 128-row query tile) = two reference query blocks
// (64-row skip groups). Warp roles:
//   warps 0-3  "stick" warps: thread r owns query row r. tcgen05.ld the S tile
//              row from TMEM, run the sequential right-to-left suffix scan in
//              registers (same order as np.cumsum), write A (bf16) into a
//              128B-swizzled smem tile for the A*V MMA; epilogue O, a.
//   warp 4     TMEM allocator + TMA producer (lane 0): Q once, K/V ring.
//   warp 5     MMA issuer (lane 0): S = Q K^T (TMEM, double buffered),
//              O += A V (TMEM accumulator, no rescaling — stick-breaking
//              weights are absolute).
#include "sb_args.cuh"

namespace sb {


template <int D>
struct FwdCfg {
  static constexpr int kStages = D == 128 ? 3 : 4;
  static constexpr int kQBytes = kTileM * D * 2;      // 128 x D bf16
  static constexpr int kKVBytes = kBlock * D * 2;     // 64 x D bf16
  static constexpr int kPBytes = kTileM * kBlock * 2; // 128 x 64 bf16
  static constexpr int kOffQ = 0;
  static constexpr int kOffK = kOffQ + kQBytes;
  static constexpr int kOffV = kOffK + kStages * kKVBytes;
  static constexpr int kOffP = kOffV + kStages * kKVBytes;
  static constexpr int kOffBar = kOffP + 2 * kPBytes;
  static constexpr int kNumBars = 1 + 3 * kStages + 2 + 2 + 2 + 2 + 1;
  static constexpr int kOffMisc = kOffBar + kNumBars * 8;
  static constexpr int kSmem = kOffMisc + 128 + 1024;  // + alignment slack
  static constexpr uint32_t kTmemCols = 256;           // S[2] (2x64) + O (D <= 128)
  static constexpr uint32_t kColS = 0, kColO = 128;
};

template <int D, bool kSkip>
__global__ void __launch_bounds__(192, 1)
    sb_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const FwdArgs args) {
  using C = FwdCfg<D>;
  constexpr int ST = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const Geom& g = args.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // heavy-first schedule: the last query tiles have the longest key sweeps
  const int BH = g.B * g.H;
  const int qt = g.n_qt - 1 - (int)(blockIdx.x / BH);
  const int bh = (int)(blockIdx.x % BH);
  const int b = bh / g.H, h = bh % g.H;
  const int qb0 = 2 * qt;
  const int kb_hi = min(qb0 + 1, g.nb - 1);  // diagonal block of the upper (or only) half
  const int n_kv = kb_hi + 1;                // tiles without skipping (kb = kb_hi .. 0)

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* bar_q = bars;
  uint64_t* bar_kfull = bars + 1;
  uint64_t* bar_vfull = bar_kfull + ST;
  uint64_t* bar_kvempty = bar_vfull + ST;
  uint64_t* bar_sfull = bar_kvempty + ST;
  uint64_t* bar_sempty = bar_sfull + 2;
  uint64_t* bar_pfull = bar_sempty + 2;
  uint64_t* bar_pempty = bar_pfull + 2;
  uint64_t* bar_ofull = bar_pempty + 2;
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);
  uint32_t* tmem_slot = misc;                        // TMEM base address
  volatile int* n_eff = reinterpret_cast<volatile int*>(misc + 1);  // tiles to run
  double* red = reinterpret_cast<double*>(misc + 2); // [2][4] per-warp max(a) (skip)

  if (threadIdx.x == 0) {
    mbar_init(bar_q, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(bar_kfull + s, 1);
      mbar_init(bar_vfull + s, 1);
      mbar_init(bar_kvempty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar_sfull + s, 1);
      mbar_init(bar_sempty + s, 128);
      mbar_init(bar_pfull + s, 128);
      mbar_init(bar_pempty + s, 1);
    }
    mbar_init(bar_ofull, 1);
    *n_eff = n_kv;
    fence_mbar_init();
  }
  if (warp == 4) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
      const int row0 = qt * kTileM;
      mbar_expect_tx(bar_q, C::kQBytes);
      for (int c = 0; c < D / 64; ++c)
        tma_load_4d(&tm_q, bar_q, smem + C::kOffQ + c * (kTileM * 128), c * 64, row0, h, b);
      int issued = 0;
      for (int j = 0; j < n_kv; ++j) {
        const int s = j % ST;
        if (j >= ST) {
          const uint32_t par = ((j / ST) - 1) & 1;
          bool stop = false;
          while (!mbar_try_wait(bar_kvempty + s, par)) {
            if (kSkip && *n_eff <= j) { stop = true; break; }
          }
          if (stop) break;
        }
        if (kSkip && *n_eff <= j) break;
        const int kb = kb_hi - j;
        mbar_expect_tx(bar_kfull + s, C::kKVBytes);
        for (int c = 0; c < D / 64; ++c)
          tma_load_4d(&tm_k, bar_kfull + s, smem + C::kOffK + s * C::kKVBytes + c * (kBlock * 128),
                      c * 64, kb * kBlock, h, b);
        mbar_expect_tx(bar_vfull + s, C::kKVBytes);
        for (int c = 0; c < D / 64; ++c)
          tma_load_4d(&tm_v, bar_vfull + s, smem + C::kOffV + s * C::kKVBytes + c * (kBlock * 128),
                      c * 64, kb * kBlock, h, b);
        ++issued;
      }
      // never leave the CTA with bulk copies in flight (early exit under skip)
      for (int j = max(0, issued - ST); j < issued; ++j) {
        mbar_wait(bar_kfull + (j % ST), (j / ST) & 1);
        mbar_wait(bar_vfull + (j % ST), (j / ST) & 1);
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16(128, 64, 0, 0);  // Q K^T: both K-major
      constexpr uint32_t idesc_o = idesc_bf16(128, D, 0, 1);   // A V: V is MN-major
      const uint32_t q_addr = smem_u32(smem + C::kOffQ);
      const uint32_t k_addr = smem_u32(smem + C::kOffK);
      const uint32_t v_addr = smem_u32(smem + C::kOffV);
      const uint32_t p_addr = smem_u32(smem + C::kOffP);
      mbar_wait(bar_q, 0);
      auto issue_pv = [&](int i) -> bool {
        mbar_wait(bar_pfull + (i & 1), (i >> 1) & 1);
        const bool last = (*n_eff <= i + 1);
        const int s = i % ST;
        mbar_wait(bar_vfull + s, (i / ST) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < kBlock / 16; ++k) {
          const uint64_t ad = sdesc_sw128(p_addr + (i & 1) * C::kPBytes + k * 32, 16, 1024);
          const uint64_t bd = sdesc_sw128(v_addr + s * C::kKVBytes + k * 2048, kBlock * 128, 1024);
          umma_ss(tbase + C::kColO, ad, bd, idesc_o, (i > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(bar_pempty + (i & 1));
        umma_commit(bar_kvempty + s);
        return last;
      };
      bool done = false;
      for (int j = 0; j < n_kv; ++j) {
        const int s = j % ST;
        // K_j, unless the stick warps have already ended the sweep before tile j
        bool have_k = true;
        while (!mbar_try_wait(bar_kfull + s, (j / ST) & 1)) {
          if (kSkip && *n_eff <= j) { have_k = false; break; }
        }
        if (have_k) {
          if (j >= 2) mbar_wait(bar_sempty + (j & 1), ((j >> 1) + 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off = (k >> 2) * (kTileM * 128) + (k & 3) * 32;
            const uint32_t offk = (k >> 2) * (kBlock * 128) + (k & 3) * 32;
            const uint64_t ad = sdesc_sw128(q_addr + off, 16, 1024);
            const uint64_t bd = sdesc_sw128(k_addr + s * C::kKVBytes + offk, 16, 1024);
            umma_ss(tbase + C::kColS + (j & 1) * 64, ad, bd, idesc_s, k > 0 ? 1u : 0u);
          }
          umma_commit(bar_sfull + (j & 1));
        }
        if (j >= 1) {
          done = issue_pv(j - 1);
          if (done) break;
        }
      }
      if (!done) issue_pv(n_kv - 1);
      umma_commit(bar_ofull);
    }
  } else {
    // ------------------------------------------------------------ stick warps
    const int r = threadIdx.x;  // 0..127 == TMEM lane == query row in the tile
    const int half = r >> 6;
    const int my_qb = qb0 + half;
    const int row = qt * kTileM + r;
    const bool row_valid = row < g.L;
    const bool half_exists = my_qb < g.nb;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const int64_t unit = (int64_t)b * g.H + h;
    float* Mrow = args.M ? args.M + unit * g.n_tiles * kBlock + (r & 63) : nullptr;
    uint8_t* pbuf = smem + C::kOffP;
    const uint32_t p_row = smem_u32(pbuf) + r * 128;

    double a_d = 0.0;      // running log remaining mass (natural log), f64
    float a2 = 0.0f;       // same in log2 units, f32, feeds the exponent
    bool act[2] = {qb0 < g.nb, qb0 + 1 < g.nb};  // halves still sweeping (skip)
    bool active = half_exists;  // this row's half has not hit the skip criterion
    int lowest = my_qb;         // leftmost processed key block (first_kb)
    int visited = 0;
    int j = 0;
    for (; j < n_kv; ++j) {
      const int kb = kb_hi - j;
      mbar_wait(bar_sfull + (j & 1), (j >> 1) & 1);
      tc_fence_after();
      float s[64];
      tmem_ld32(tbase + lane_base + C::kColS + (j & 1) * 64, s);
      tmem_ld32(tbase + lane_base + C::kColS + (j & 1) * 64 + 32, s + 32);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(bar_sempty + (j & 1));

      const bool live = active && kb <= my_qb;  // tile belongs to this row's sweep
      uint32_t pk[32];
      if (live) {
        const int lim = (kb == my_qb) ? (r & 63) : kBlock;  // strict causality on the diagonal
        float cum = 0.0f;
#pragma unroll
        for (int c = kBlock - 1; c >= 0; --c) {
          const float Z = s[c] * g.scale_log2;
          const float t = ex2(Z);
          const float lt = (c < lim) ? -softplus2(Z, t) : 0.0f;
          cum += lt;
          s[c] = (c < lim) ? ex2(Z + cum + a2) : 0.0f;
        }
#pragma unroll
        for (int c = 0; c < 32; ++c) pk[c] = pack_bf16(s[2 * c], s[2 * c + 1]);
        if (Mrow && row_valid) Mrow[tile_index(my_qb, kb) * kBlock] = a2;
        a_d += (double)cum * (double)kLn2;
        a2 = (float)(a_d * 1.4426950408889634);
        lowest = kb;
        ++visited;
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) pk[c] = 0u;
      }
      if (j >= 2) mbar_wait(bar_pempty + (j & 1), ((j >> 1) + 1) & 1);
      const uint32_t pb = p_row + (j & 1) * C::kPBytes;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        st_shared_v4(pb + ((c ^ (r & 7)) << 4), pk[4 * c], pk[4 * c + 1], pk[4 * c + 2],
                     pk[4 * c + 3]);
      fence_proxy_async_smem();

      bool stop = false;
      if (kSkip) {
        // decision for the next key block kb-1 (blocked.py:175-176), per 64-row
        // half: max over its rows of a < log(eps), checked only left of the
        // half's diagonal. Every stick thread derives both halves' state from
        // the same per-warp maxima, so the decision is CTA-uniform.
        double m = row_valid ? a_d : -INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) red[(j & 1) * 4 + warp] = m;
        named_bar_sync(1, 128);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const double mh = fmax(red[(j & 1) * 4 + 2 * hh], red[(j & 1) * 4 + 2 * hh + 1]);
          if (act[hh] && (kb - 1) < qb0 + hh && mh < args.log_eps) act[hh] = false;
        }
        active = act[half];
        stop = !act[0] && !act[1];
        if (stop && r == 0) *n_eff = j + 1;
      }
      mbar_arrive(bar_pfull + (j & 1));
      if (stop) break;
    }

    // ------------------------------------------------------------ epilogue
    mbar_wait(bar_ofull, 0);
    tc_fence_after();
    __nv_bfloat16* orow = args.o + (int64_t)b * g.sb + (int64_t)h * g.sh + (int64_t)row * g.sl;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      float ov[32];
      tmem_ld32(tbase + lane_base + C::kColO + c * 32, ov);
      tmem_wait_ld();
      if (row_valid) {
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
          dst[q4] = make_uint4(pack_bf16(ov[8 * q4], ov[8 * q4 + 1]),
                               pack_bf16(ov[8 * q4 + 2], ov[8 * q4 + 3]),
                               pack_bf16(ov[8 * q4 + 4], ov[8 * q4 + 5]),
                               pack_bf16(ov[8 * q4 + 6], ov[8 * q4 + 7]));
      }
    }
    if (row_valid) args.log_rem[unit * g.L + row] = (float)a_d;
    if (half_exists && (r & 63) == 0) {
      args.first_kb[unit * g.nb + my_qb] = lowest;
      if (args.counters) atomicAdd(args.counters, (unsigned long long)visited);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) tmem_dealloc<C::kTmemCols>(tbase);
}

template <int D, bool kSkip>
static int launch_fwd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                      const FwdArgs& a, cudaStream_t stream) {
  using C = FwdCfg<D>;
  auto kern = sb_fwd_kernel<D, kSkip>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
  if (e != cudaSuccess) return (int)e;
  const unsigned grid = (unsigned)(a.g.n_qt * a.g.B * a.g.H);
  kern<<<grid, 192, C::kSmem, stream>>>(tq, tk, tv, a);
  return (int)cudaGetLastError();
}

int fwd_dispatch(int D, bool skip, const CUtensorMap& tq, const CUtensorMap& tk,
                 const CUtensorMap& tv, const FwdArgs& a, cudaStream_t stream) {
  if (D == 128) return skip ? launch_fwd<128, true>(tq, tk, tv, a, stream)
                            : launch_fwd<128, false>(tq, tk, tv, a, stream);
  if (D == 64) return skip ? launch_fwd<64, true>(tq, tk, tv, a, stream)
                           : launch_fwd<64, false>(tq, tk, tv, a, stream);
  return -1;
}

}  // namespace sb
