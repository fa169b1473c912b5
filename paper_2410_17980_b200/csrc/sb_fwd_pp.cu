// Stick-breaking attention forward, persistent ping-pong kernel (skip off and,
// with kSkip, skip on), sm_100a.
//
// Restates blocked_forward (reference blocked.py:129-206), organised for
// throughput: a work item is TWO 128-row query tiles of the same
// (b, h) (tiles 2p and 2p+1, i.e. four reference query blocks) whose shared K/V
// blocks stream right to left once; persistent CTAs walk the items. Each query tile has its own stick
// warpgroup (WG0 / WG1, thread r <-> TMEM lane r <-> query row), its own
// MMA-issuer thread and its own S/P buffers, so the two warpgroups interleave
// on every SMSP without any cross-warpgroup synchronisation; each thread scans
// all 64 key columns of its row in registers.
//
// Per element (product form, sb_common.cuh): t = 2^Z, r = 1/(1+t), sigma = t*r,
// A = sigma * (e^a * prod of r to the right), with one rcp per 16 columns
// (batched_row).  The row total of lt for `a` is -lg2 of the tile's product of
// (1+t); rows outside the batched range retry a wider range, then take the
// per-element path (sb_common.cuh).  kSkip computes exact lt sums for the skip
// decisions (see the kernel's comment).
// No M snapshots (blocked.py:188-189): the running `a` is accumulated in float64
// and only its final value per row is kept (`state`, O(L)); the backward's phase 1
// rolls the per-tile a back from it, tile by tile, left to right (sb_bwd.cu).
//
// Warps: 0-3 WG0, 4-7 WG1, 8 TMA producer (+TMEM allocator), 9 MMA for WG0,
// 10 MMA for WG1.
#include "sb_args.cuh"

namespace sb {

template <int D>
struct FwdPPCfg {
  // K/V ring: 3 stages at both head dims (d=64: 4 stages measured 0.671 vs 0.610 ms on
  // the C2 shape, C4 1.82 vs 1.74 ms; 2 and 6 stages slower too; d=128: 4 stages 0.72 vs
  // 0.61 ms)
  static constexpr int kStages = 3;
  static constexpr int kThreads = 11 * 32;
  static constexpr int kQBytes = kTileM * D * 2;
  static constexpr int kKVBytes = kBlock * D * 2;
  static constexpr int kPBytes = kTileM * kBlock * 2;
  static constexpr int kOffQ = 0;                                // Q[2]
  static constexpr int kOffK = kOffQ + 2 * kQBytes;
  static constexpr int kOffV = kOffK + kStages * kKVBytes;
  static constexpr int kOffP = kOffV + kStages * kKVBytes;       // P[wg][buf]
  static constexpr int kOffBar = kOffP + 4 * kPBytes;
  static constexpr int kNumBars = 2 + 3 * kStages + 2 * 8 + 2 + 2 + 1 + 8 + 2 + 2;
  static constexpr int kOffMisc = kOffBar + kNumBars * 8;
  // misc: TMEM slot, work-queue ring, skip flags (+64), skip max exchange (+128)
  static constexpr int kSmem = kOffMisc + 256 + 1024;
  // per WG w: S at w*128 (single-buffered), Q (MMA A operand) at w*128 + 64,
  // O at 256 + w*128
  static constexpr uint32_t kTmemCols = 512;
};

// Work item: (unit, query-tile pair p); all roles derive the same list.
struct FwdItem {
  Unit u;
  int b, h, p, kbhi0, kbhi1, n_s;
  bool has1, valid;
};
__device__ __forceinline__ FwdItem fwd_item(const Geom& g, int idx) {
  FwdItem it;
  int item, bh;
  grouped_order(idx, (g.n_qt + 1) / 2, g.B * g.H, g.ugroup, item, bh);
  it.b = bh / g.H;
  it.h = bh % g.H;
  it.u = make_unit(g, it.b, it.h);
  const int n_pairs = (it.u.n_qt + 1) / 2;
  it.valid = item < n_pairs;  // varlen: shorter sequences have fewer pairs
  it.p = n_pairs - 1 - item;  // heaviest pairs first (longest-processing-time order)
  it.has1 = 2 * it.p + 1 < it.u.n_qt;
  it.kbhi0 = min(4 * it.p + 1, it.u.nb - 1);
  it.kbhi1 = it.has1 ? min(4 * it.p + 3, it.u.nb - 1) : it.kbhi0;
  it.n_s = it.kbhi1 + 1;  // stream tiles, kb = kbhi1 .. 0
  return it;
}

// Persistent: one CTA per SM takes items from a global work queue (heaviest
// first: grouped_order's LPT order, handed out dynamically).  The
// K/V ring and each warpgroup's S/P buffers run on counters that continue
// across items; Q of the next item loads once the last S of the current item
// was issued (q_free), and the next item's first A.V waits until the
// warpgroup has read O out of TMEM (ofree).
// kSkip: block skipping (blocked.py:175-176) with the exact-path kernel's
// decision arithmetic (f64 running `a` from f32 exact lt sums, max over each
// 64-row query block before every tile), so first_kb is bit-exact against the
// oracle.  Per element one more MUFU (lg2 of the exact softplus) than skip off.
// A warpgroup whose two query blocks are both done publishes its stop (stream
// tile count) before releasing S, so its issuer never issues the next S; the
// producer stops loading once both warpgroups stopped and publishes how many
// tiles it loaded (bar_nload), so each issuer can release the tail of the ring.
template <int D, bool kSkip>
__global__ void __launch_bounds__(FwdPPCfg<D>::kThreads, 1)
    sb_fwd_pp_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const FwdArgs args) {
  using C = FwdPPCfg<D>;
  constexpr int ST = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const Geom& g = args.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = ((g.n_qt + 1) / 2) * g.B * g.H;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  // Q landed, one barrier per warpgroup: each completes once per item that has a
  // tile for that warpgroup, so a warpgroup that sits out items (no second tile:
  // odd tile counts, short varlen sequences) can never wait on a phase two ahead
  // of the barrier (a parity wait cannot tell those apart: that race read a stale
  // Q tile whenever WG1 skipped two items in a row)
  uint64_t* bar_q = bars;  // [2]
  uint64_t* bar_kfull = bars + 2;
  uint64_t* bar_vfull = bar_kfull + ST;
  uint64_t* bar_kvempty = bar_vfull + ST;
  uint64_t* wgbars = bar_kvempty + ST;  // per wg: sfull[2], sempty[2], pfull[2], pempty[2]
  uint64_t* bar_ofull = wgbars + 16;    // [2]
  uint64_t* bar_ofree = bar_ofull + 2;  // [2]
  uint64_t* bar_qfree = bar_ofree + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);
  const SchedRing sq{reinterpret_cast<int*>(smem + C::kOffMisc + 16), bar_qfree + 1, bar_qfree + 5};
  uint64_t* bar_qtm = bar_qfree + 9;  // [2] the warpgroup copied its Q tile into TMEM
  uint64_t* bar_nload = bar_qtm + 2;  // [2] (skip) the producer's tile count of an item
  // skip: per warpgroup (seq << 13) | stop of its current item (-1: none yet), and
  // per item parity the number of stream tiles the producer loaded
  // (polled flags: shared-memory atomics, see sched_consume)
  int* wg_done = reinterpret_cast<int*>(smem + C::kOffMisc + 64);
  int* nload_v = wg_done + 2;
  // skip votes [wg][round parity][quarter]: (round << 1) | vote, polled like the flags
  int* votes = reinterpret_cast<int*>(smem + C::kOffMisc + 128);
  // one read per warp (lane 0, broadcast): every lane must take the same branch
  auto flag_read = [](int* f) -> int {
    int v = 0;
    if ((threadIdx.x & 31) == 0) v = atomicAdd(f, 0);
    return __shfl_sync(0xffffffffu, v, 0);
  };
  auto stop_of = [&](int w, int seq) -> int {
    const int v = flag_read(wg_done + w);
    return (v >> 13) == seq ? (v & 8191) : 0x7fffffff;
  };

  if (threadIdx.x == 0) {
    mbar_init(bar_q, 1);
    mbar_init(bar_q + 1, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(bar_kfull + s, 1);
      mbar_init(bar_vfull + s, 1);
      mbar_init(bar_kvempty + s, 2);  // one arrival per warpgroup issuer
    }
    for (int w = 0; w < 2; ++w)
      for (int s = 0; s < 2; ++s) {
        mbar_init(wgbars + w * 8 + 0 + s, 1);    // sfull
        mbar_init(wgbars + w * 8 + 2 + s, 128);  // sempty
        mbar_init(wgbars + w * 8 + 4 + s, 128);  // pfull
        mbar_init(wgbars + w * 8 + 6 + s, 1);    // pempty
      }
    for (int w = 0; w < 2; ++w) {
      mbar_init(bar_ofull + w, 1);
      mbar_init(bar_ofree + w, 128);
    }
    mbar_init(bar_qfree, 2);
    mbar_init(bar_qtm, 128);
    mbar_init(bar_qtm + 1, 128);
    mbar_init(bar_nload, 1);
    mbar_init(bar_nload + 1, 1);
    for (int i = 0; i < 16; ++i) votes[i] = -2;  // round -1: none yet
    wg_done[0] = wg_done[1] = -1;
    sched_init(sq, 10);  // consumers: stick warps 0-7, issuer warps 9-10
    fence_mbar_init();
  }
  if (warp == 8) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 8) {
    // ------------------------------------------------------------ TMA producer
    const bool leader = elect_one();
    if (leader) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
    }
    int jg = 0, ni = 0;
    for (int k = 0;; ++k) {
      const int idx = sched_produce(sq, k, args.sched, n_items);
      if (idx < 0) break;
      const FwdItem it = fwd_item(g, idx);
      if (!it.valid) continue;
      const Unit& u = it.u;
      if (ni >= 1) mbar_wait_warp(bar_qfree, (ni - 1) & 1);
      if (leader) {
        for (int w = 0; w < (it.has1 ? 2 : 1); ++w) {
          mbar_expect_tx(bar_q + w, C::kQBytes);
          for (int c = 0; c < D / 64; ++c)
            tma_load_4d(&tm_q, bar_q + w, smem + C::kOffQ + w * C::kQBytes + c * (kTileM * 128),
                        c * 64, u.trow0 + (2 * it.p + w) * kTileM, it.h, u.tb);
        }
      }
      __syncwarp();
      int n_load = it.n_s;
      for (int j = 0; j < it.n_s; ++j, ++jg) {
        const int s = jg % ST;
        // wait for the slot: it is always freed, also after both warpgroups stopped
        // (their issuers release every loaded tile they no longer read as it lands)
        if (jg >= ST) mbar_wait_warp(bar_kvempty + s, ((jg / ST) - 1) & 1);
        // skip: stop once both warpgroups are done (their stops are published before
        // they release S; one look per tile, the ring slack absorbs the lag)
        if (kSkip && j > 0 && stop_of(0, ni) <= j && (!it.has1 || stop_of(1, ni) <= j)) {
          n_load = j;
          break;
        }
        const int kb = it.kbhi1 - j;
        if (leader) {
          mbar_expect_tx(bar_kfull + s, C::kKVBytes);
          for (int c = 0; c < D / 64; ++c)
            tma_load_4d(&tm_k, bar_kfull + s, smem + C::kOffK + s * C::kKVBytes + c * (kBlock * 128),
                        c * 64, u.trow0 + kb * kBlock, it.h, u.tb);
          mbar_expect_tx(bar_vfull + s, C::kKVBytes);
          for (int c = 0; c < D / 64; ++c)
            tma_load_4d(&tm_v, bar_vfull + s, smem + C::kOffV + s * C::kKVBytes + c * (kBlock * 128),
                        c * 64, u.trow0 + kb * kBlock, it.h, u.tb);
        }
        __syncwarp();
      }
      if constexpr (kSkip) {
        if (leader) {
          atomicExch(nload_v + (ni & 1), n_load);
          mbar_arrive(bar_nload + (ni & 1));
        }
        __syncwarp();
      }
      ++ni;
    }
  } else if (warp == 9 || warp == 10) {
    // ------------------------------------------------------------ MMA issuer of one WG
    // The whole warp runs the (uniform) control flow and computes descriptors in
    // uniform registers; one elected lane issues the MMAs and their commits.
    const int w = warp - 9;
    uint64_t* sfull = wgbars + w * 8;
    uint64_t* sempty = sfull + 2;
    uint64_t* pfull = sfull + 4;
    uint64_t* pempty = sfull + 6;
    constexpr uint32_t idesc_s = idesc_bf16(128, 64, 0, 0);  // Q K^T: both K-major
    constexpr uint32_t idesc_o = idesc_bf16(128, D, 0, 1);   // A V: V is MN-major
    const uint64_t dk = sdesc_sw128(smem_u32(smem + C::kOffK), 16, 1024);
    const uint64_t dv = sdesc_sw128(smem_u32(smem + C::kOffV), kBlock * 128, 1024);
    const uint64_t dp = sdesc_sw128(smem_u32(smem + C::kOffP + w * 2 * C::kPBytes), 16, 1024);
    const uint32_t tS = tbase + w * 128, tQ = tS + 64, tO = tbase + 256 + w * 128;
    const bool leader = elect_one();
    int jg = 0, ni = 0, ig = 0, nwi = 0;
    // skip: release stream tiles j_from.. of item ni (this warpgroup no longer reads
    // them) as they land, until the producer has published how many it loaded; the
    // producer may need those slots back before it knows (the other warpgroup can
    // still be sweeping).  Returns that count.
    auto release_tail = [&](int j_from) -> int {
      uint64_t* nb_bar = bar_nload + (ni & 1);
      const uint32_t nb_par = (ni >> 1) & 1;
      for (int j = j_from;; ++j) {
        const int js = jg + j, s = js % ST;
        const uint32_t par = (js / ST) & 1;
        const long long t0 = clock64();
        for (;;) {
          // landed-test first, count second: if the count is not out yet, a landed
          // tile cannot be the next item's (the producer publishes before loading it)
          // warp-uniform decisions (a lane breaking out alone could let the ring slot
          // complete its next phase before the others poll: see mbar_wait_warp)
          const bool kv = __any_sync(
              0xffffffffu, mbar_test(bar_kfull + s, par) && mbar_test(bar_vfull + s, par));
          if (__any_sync(0xffffffffu, mbar_test(nb_bar, nb_par))) {
            const int n = flag_read(nload_v + (ni & 1));
            if (j >= n) return n;
          }
          if (kv) break;
          if (watchdog_expired(t0)) __trap();  // deadlock: fail loudly (sm100.cuh)
          __nanosleep(64);  // back off (the issuer warps share SMSPs with stick warps)
        }
        if (leader) mbar_arrive(bar_kvempty + s);
        __syncwarp();
      }
    };
    for (int k = 0;; ++k) {
      const int idx = sched_consume(sq, k);
      if (idx < 0) break;
      const FwdItem it = fwd_item(g, idx);
      if (!it.valid) continue;
      if (w == 1 && !it.has1) {  // no tile for this warpgroup: release the stream
        int n_rel = it.n_s;
        if constexpr (kSkip) {
          n_rel = release_tail(0);
        } else {
          for (int j = 0; j < n_rel; ++j) {
            const int js = jg + j;
            mbar_wait_warp(bar_vfull + js % ST, (js / ST) & 1);
            if (leader) mbar_arrive(bar_kvempty + js % ST);
            __syncwarp();
          }
        }
        // (after a V of this item landed: the producer is past the previous
        // item's q_free phase, so this arrival counts for this item's phase)
        if (leader) mbar_arrive(bar_qfree);
        __syncwarp();
        jg += n_rel;
        ++ni;
        continue;
      }
      const int j0 = it.kbhi1 - (w ? it.kbhi1 : it.kbhi0);  // first stream tile of this WG
      const int n_w = it.n_s - j0;
      // S = Q K^T reads Q from TMEM (copied there by the warpgroup); the smem Q
      // buffer of this warpgroup is free for the next item from then on
      mbar_wait_warp(bar_qtm + w, nwi & 1);
      if (leader) mbar_arrive(bar_qfree);
      __syncwarp();
      auto issue_pv = [&](int i) {  // local tile i == stream tile j0 + i
        const int js = jg + j0 + i, s = js % ST, gi = ig + i;
        mbar_wait_warp(pfull + (gi & 1), (gi >> 1) & 1);
        SB_TR(args, 2 + w, gi, 9);
        mbar_wait_warp(bar_vfull + s, (js / ST) & 1);
        // O of the previous item must be out of TMEM before it is overwritten
        if (i == 0 && nwi >= 1) mbar_wait_warp(bar_ofree + w, (nwi - 1) & 1);
        tc_fence_after();
        if (leader) {
#pragma unroll
          for (int k = 0; k < kBlock / 16; ++k)
            umma_ss_at(tO, dp, (gi & 1) * C::kPBytes + k * 32, dv, s * C::kKVBytes + k * 2048,
                       idesc_o, (i > 0 || k > 0) ? 1u : 0u);
          umma_commit(pempty + (gi & 1));
          umma_commit(bar_kvempty + s);
        }
        __syncwarp();
        SB_TR(args, 2 + w, gi, 11);
      };
      for (int j = 0; j < j0; ++j) {  // stream tiles right of this WG's diagonal
        const int js = jg + j;
        mbar_wait_warp(bar_vfull + js % ST, (js / ST) & 1);
        if (leader) mbar_arrive(bar_kvempty + js % ST);
        __syncwarp();
      }
      int n_proc = n_w;  // tiles this warpgroup processes (skip: up to its stop)
      for (int i = 0; i < n_w; ++i) {
        const int js = jg + j0 + i, s = js % ST, gi = ig + i;
        if (gi >= 1) mbar_wait_warp(sempty, (gi - 1) & 1);  // S is single-buffered
        // skip: the warpgroup published its stop before releasing S of tile i-1
        if (kSkip && i > 0 && stop_of(w, ni) <= j0 + i) {
          n_proc = i;
          break;
        }
        mbar_wait_warp(bar_kfull + s, (js / ST) & 1);
        SB_TR(args, 2 + w, gi, 8);
        tc_fence_after();
        if (leader) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t offk = (k >> 2) * (kBlock * 128) + (k & 3) * 32;
            umma_ts_at(tS, tQ + k * 8, dk, s * C::kKVBytes + offk, idesc_s, k > 0);
          }
          umma_commit(sfull);
        }
        __syncwarp();
        SB_TR(args, 2 + w, gi, 10);
        if (i >= 1) issue_pv(i - 1);
      }
      issue_pv(n_proc - 1);
      if (leader) umma_commit(bar_ofull + w);
      __syncwarp();
      if constexpr (kSkip) {
        // release the loaded stream tiles this warpgroup no longer reads
        jg += release_tail(j0 + n_proc);
      } else {
        jg += it.n_s;
      }
      ig += n_proc;
      ++ni;
      ++nwi;
    }
  } else {
    // ------------------------------------------------------------ stick warpgroups
    const int w = warp >> 2;
    uint64_t* sfull = wgbars + w * 8;
    uint64_t* sempty = sfull + 2;
    uint64_t* pfull = sfull + 4;
    uint64_t* pempty = sfull + 6;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t tS = tbase + w * 128 + lane_base, tQ = tS + 64,
                   tO = tbase + 256 + w * 128 + lane_base;
    const uint32_t p_row = smem_u32(smem + C::kOffP + w * 2 * C::kPBytes) + r * 128;
    const float sl2 = g.scale_log2;
    const bool tr = quarter == 0 && lane == 0;
    if (tr) SB_TR(args, w, 0, 14);
    int ig = 0, nwi = 0, ni = 0, nv = 0;  // nv: skip-vote rounds of this warpgroup
    for (int k = 0;; ++k) {
      const int idx = sched_consume(sq, k);
      if (idx < 0) break;
      const FwdItem it = fwd_item(g, idx);
      if (!it.valid) continue;
      ++ni;
      if (w == 1 && !it.has1) continue;
      const Unit& u = it.u;
      {
        // copy this thread's Q row (TMA-swizzled smem) into TMEM lane r: the A
        // operand of S = Q K^T, two bf16 of d per 32-bit column
        mbar_wait(bar_q + w, nwi & 1);  // this warpgroup's nwi-th tile
        const uint32_t qrow = smem_u32(smem + C::kOffQ + w * C::kQBytes) + r * 128;
        uint32_t qv[D / 2];
#pragma unroll
        for (int c = 0; c < D / 8; ++c) {
          const uint4 x = ld_shared_v4(qrow + (c >> 3) * (kTileM * 128) + (((c & 7) ^ (r & 7)) << 4));
          qv[4 * c] = x.x;
          qv[4 * c + 1] = x.y;
          qv[4 * c + 2] = x.z;
          qv[4 * c + 3] = x.w;
        }
        if constexpr (D == 128) tmem_st64(tQ, qv);
        else tmem_st32(tQ, qv);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(bar_qtm + w);
      }
      const int qt = 2 * it.p + w;
      const int my_qb = 2 * qt + (r >> 6);
      const int row = qt * kTileM + r;
      const bool row_valid = row < u.L;
      const int kbhi = w ? it.kbhi1 : it.kbhi0;
      const int n_w = kbhi + 1;
      // running remaining mass a (log2 units): a2 float32 (the tile math) with a2_lo
      // its compensation; a2 + a2_lo is the backward's state and, skip on, what the
      // skip decisions compare
      float a2 = 0.0f, a2_lo = 0.0f;
      // skip: the two query blocks' sweep state, and (thread (r & 63) == 0) the
      // block's leftmost visited tile and count
      const int qb0 = 2 * qt, half = r >> 6;
      bool act[2] = {qb0 < u.nb, qb0 + 1 < u.nb};
      int lowest = my_qb, visited = 0, n_proc = n_w;
      bool my_vote = false;  // skip: this warp's latest vote (all its rows below log eps)
      const int j0 = it.kbhi1 - kbhi;  // stream index of this warpgroup's first tile
      // d = 64, skip off: P(i)'s fence and `pfull` move into tile i+1, behind its S load
      // (C4 forward 1.770 -> 1.733 ms).  Not at d = 128: there the issuer then queues the
      // longer P.V(i) right before S(i+1) (C2 forward 0.617 -> 0.690 ms); not skip on,
      // whose tiles can end an item early.
      constexpr bool kDeferP = !kSkip && D == 64;
      for (int i = 0; i < n_w; ++i) {
        const int kb = kbhi - i, gi = ig + i;
        if (tr) SB_TR(args, w, gi, 0);
        mbar_wait(sfull, gi & 1);
        tc_fence_after();
        float s[64];
        tmem_ld32(tS, s);
        tmem_ld32(tS + 32, s + 32);
        if (kDeferP && i > 0) {
          // the previous tile's P: its proxy fence waits for the shared stores while
          // this tile's S is in flight from TMEM
          fence_proxy_async_smem();
          mbar_arrive(pfull + ((gi - 1) & 1));
        }
        tmem_wait_ld();
        if (tr) SB_TR(args, w, gi, 1);
        uint32_t pk[32];
        bool slow = false;
        const bool diag = kb == my_qb;
        const int lim = diag ? (r & 63) : kBlock;
        bool done = false;
        if (kSkip && i > 0 && my_vote) {
          // skip check for this tile (blocked.py:175-176) on a after the previous one:
          // every valid row of a query block below log eps <=> the block's max is.
          // The four warps voted at the end of tile i-1 (one __all_sync each, vote
          // round rv = nv-1), each into its slot of the round's parity as one word
          // (rv << 1) | vote; a slot cannot move on to round rv+2 before this warp
          // released S(i).  a only decreases, so votes are monotone: a warp whose
          // own vote is false knows its block goes on and need not look (nor can the
          // warpgroup be done); the others wait for the four round-rv words (the
          // other block's state only matters for `done`, its latest round tells it).
          // A warpgroup whose blocks both stopped runs this tile as a no-op (S(i) is
          // already issued) and publishes its stop before releasing S, so S(i+1) is
          // never issued.
          const int rv = nv - 1;
          int vbits = 0;
          if (lane == 0) {
            int* slot = votes + (w * 2 + (rv & 1)) * 4;
            const long long t0 = clock64();
            for (int q = 0; q < 4; ++q) {
              int v;
              while (((v = atomicAdd(slot + q, 0)) >> 1) != rv)
                if (watchdog_expired(t0)) __trap();  // deadlock: fail loudly (sm100.cuh)
              vbits |= (v & 1) << q;
            }
          }
          vbits = __shfl_sync(0xffffffffu, vbits, 0);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh)
            if (act[hh] && kb < qb0 + hh && ((vbits >> (2 * hh)) & 3) == 3) act[hh] = false;
          done = !act[0] && !act[1];
          if (done) {
            n_proc = i + 1;
            if (r == 0) atomicExch(wg_done + w, ((ni - 1) << 13) | (j0 + i + 1));
          }
        }
        // warp-uniform: a warp's rows share one 64-row half
        const bool math = (!kSkip || act[half]) && kb <= my_qb;
        float2 Em[2];  // skip on: per group prod (1+t) - 1 (batched_row)
        if (math) {
          // batched reciprocal (sb_common.cuh): one rcp per 16 columns (leaves t in s[])
          float Q = ex2(a2), Dhi = 1.0f, Dlo = 1.0f;
          slow = diag ? !batched_row<true, kSkip>(s, pk, sl2, lim, Q, Dhi, Dlo, Em)
                      : !batched_row<false, kSkip>(s, pk, sl2, kBlock, Q, Dhi, Dlo, Em);
          // skip off: the tile's row total of lt (phase 1 recomputes it with the same
          // operations), accumulated compensated: a2 + a2_lo.  Skip on: the accurate
          // total for the decisions, after S is released (below)
          if (!kSkip && !slow) two_sum_acc(a2, a2_lo, -(lg2(Dhi) + lg2(Dlo)));
          if (kSkip) {
            lowest = kb;
            ++visited;
          }
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c) pk[c] = 0u;
        }
        const bool batched_ok = math && !slow;  // a not yet updated for slow rows
        if (__any_sync(0xffffffffu, slow)) {
          // a group product of (1+t) reached 2^64: per-element path for those rows
          // (S is still in TMEM: s_empty not yet signalled)
          tmem_ld32(tS, s);
          tmem_ld32(tS + 32, s + 32);
          tmem_wait_ld();
          if (slow) {  // the wider batched range (sb_common.cuh) first
            float lsum = 0.0f;
            const bool okw = diag ? batched_row_wide<true>(s, pk, sl2, lim, ex2(a2), lsum)
                                  : batched_row_wide<false>(s, pk, sl2, kBlock, ex2(a2), lsum);
            if (okw) {
              two_sum_acc(a2, a2_lo, -lsum);
              slow = false;
            }
          }
          if (__any_sync(0xffffffffu, slow)) {  // s[] holds t now: raw S again (warp-collective)
            tmem_ld32(tS, s);
            tmem_ld32(tS + 32, s + 32);
            tmem_wait_ld();
          }
          if (slow) {
            // per-element product form for A; the row's lt from each 16-column
            // group's product of r (one lg2 per group), or the exact softplus sum
            // for a group whose product leaves the normal range or holds a logit
            // beyond the clamp (2 MUFU per element instead of 3)
            float Ql = ex2(a2), lt = 0.0f;
#pragma unroll
            for (int g = kBlock / 16 - 1; g >= 0; --g) {
              float pr = 1.0f;
              bool big = false;
#pragma unroll
              for (int c = 16 * g + 15; c >= 16 * g; c -= 2) {
                float A[2];
#pragma unroll
                for (int uu = 0; uu < 2; ++uu) {
                  const int cc = c - uu;
                  const float Zr = s[cc] * sl2;
                  big = big || (Zr > 126.0f && cc < lim);
                  const float t = ex2(fminf(Zr, 126.0f));  // t finite: sigma = t*r <= 1
                  float rr = rcp(1.0f + t), sg = t * rr;
                  if (cc >= lim) { rr = 1.0f; sg = 0.0f; }
                  A[uu] = sg * Ql;
                  Ql *= rr;
                  pr *= rr;
                }
                pk[(c - 1) >> 1] = pack_bf16(A[1], A[0]);
              }
              if (!big && pr >= kProdFloor) {
                lt += lg2(pr);
              } else {
#pragma unroll
                for (int cc = 16 * g; cc < 16 * g + 16; ++cc) {
                  const float Zr = s[cc] * sl2;
                  lt -= (cc < lim) ? softplus2(Zr, ex2(fminf(Zr, 126.0f))) : 0.0f;
                }
              }
            }
            two_sum_acc(a2, a2_lo, lt);
          }
        }
        tc_fence_before();
        mbar_arrive(sempty);  // S(i+1) may overwrite the buffer now
        if (tr) SB_TR(args, w, gi, 2);
        if (gi >= 2) mbar_wait(pempty + (gi & 1), ((gi >> 1) + 1) & 1);
        if (tr) SB_TR(args, w, gi, 3);
        const uint32_t pb = p_row + (gi & 1) * C::kPBytes;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          st_shared_v4(pb + ((c ^ (r & 7)) << 4), pk[4 * c], pk[4 * c + 1], pk[4 * c + 2],
                       pk[4 * c + 3]);
        if (!kDeferP) {
          fence_proxy_async_smem();
          mbar_arrive(pfull + (gi & 1));
        }
        if (tr) SB_TR(args, w, gi, 4);
        if (kSkip && !done) {
          // the row total of lt for the skip decisions (blocked.py:175-176), after the
          // tile's S and P turnaround (fast rows; the slow ones updated a already)
          if (batched_ok) two_sum_acc(a2, a2_lo, -lt_row_from_em(Em));
          // this warp's vote for the next tile's check: all its valid rows' a below log
          // eps (a - log eps from the compensated pairs: exact near a tie, where a2 and
          // the threshold's high part are within a factor 2).  Vote round nv of this
          // warpgroup: slot nv & 1
          if (i + 1 < n_w) {
            const bool below =
                !row_valid || (a2 - args.log_eps2_hi) + (a2_lo - args.log_eps2_lo) < 0.0f;
            my_vote = __all_sync(0xffffffffu, below);
            if (lane == 0) atomicExch(votes + (w * 2 + (nv & 1)) * 4 + quarter, (nv << 1) | my_vote);
            ++nv;
          }
        }
        if (done) break;
      }
      if (kDeferP) {  // the item's last P
        fence_proxy_async_smem();
        mbar_arrive(pfull + ((ig + n_w - 1) & 1));
      }
      // epilogue: O rows leave in 64-column halves through this warp's 4 KB slice
      // of the (now idle: ofull) P buffers as coalesced row segments
      mbar_wait(bar_ofull + w, nwi & 1);
      tc_fence_after();
      const int row0 = qt * kTileM + quarter * 32;
      const int nvalid = max(0, min(32, u.L - row0));
      const uint32_t stage = smem_u32(smem + C::kOffP + w * 2 * C::kPBytes) + quarter * 4096;
#pragma unroll 1
      for (int c = 0; c < D / 64; ++c) {
        float ov[64];
        tmem_ld32(tO + c * 64, ov);
        tmem_ld32(tO + c * 64 + 32, ov + 32);
        tmem_wait_ld();
        if (c + 1 == D / 64) {
          tc_fence_before();
          mbar_arrive(bar_ofree + w);  // the next item's A.V may overwrite O
        }
        warp_store_rows<8>(ov, 1.0f, stage, args.o + u.out_off + (int64_t)row0 * g.sl + c * 64,
                           g.sl, nvalid);
      }
      if (row_valid) {
        const int64_t ri = u.rem_off + row * u.rem_stride;
        const double a_d = (double)a2 + (double)a2_lo;
        args.log_rem[ri] = (float)(a_d * (double)kLn2);
        // the backward's state: final a in log2 units, float64
        if (args.state) args.state[ri] = a_d;
      }
      if (my_qb < u.nb && (r & 63) == 0) {
        args.first_kb[u.fkb_off + my_qb] = kSkip ? lowest : 0;
        if (args.counters)
          atomicAdd(args.counters, (unsigned long long)(kSkip ? visited : my_qb + 1));
      }
      ig += n_proc;
      ++nwi;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) tmem_dealloc<C::kTmemCols>(tbase);
}

template <int D, bool kSkip>
static int launch_fwd_pp(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                         const FwdArgs& a, cudaStream_t stream) {
  using C = FwdPPCfg<D>;
  auto kern = sb_fwd_pp_kernel<D, kSkip>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
  if (e != cudaSuccess) return (int)e;
  if (a.sched && (e = cudaMemsetAsync(a.sched, 0, sizeof(unsigned), stream)) != cudaSuccess)
    return (int)e;
  // persistent: one CTA per SM (fewer if there are fewer work items)
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned items = (unsigned)(((a.g.n_qt + 1) / 2) * a.g.B * a.g.H);
  kern<<<items < (unsigned)sms ? items : (unsigned)sms, C::kThreads, C::kSmem, stream>>>(tq, tk, tv,
                                                                                         a);
  return (int)cudaGetLastError();
}

int fwd_pp_dispatch(int D, bool skip, const CUtensorMap& tq, const CUtensorMap& tk,
                    const CUtensorMap& tv, const FwdArgs& a, cudaStream_t stream) {
  if (D == 128) return skip ? launch_fwd_pp<128, true>(tq, tk, tv, a, stream)
                            : launch_fwd_pp<128, false>(tq, tk, tv, a, stream);
  if (D == 64) return skip ? launch_fwd_pp<64, true>(tq, tk, tv, a, stream)
                           : launch_fwd_pp<64, false>(tq, tk, tv, a, stream);
  return -1;
}

}  // namespace sb
