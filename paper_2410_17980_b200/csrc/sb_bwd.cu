// Stick-breaking attention two-phase backward (K2 + K3 of SURVEY.md §2.2), sm_100a.
//
// Restates blocked_backward_twophase (reference blocked.py:299-392):
//   recompute_tile (:325-335): z, lt, A = exp(z + suffix_cumsum(lt) + M)
//   dW = dO V^T - row_offset; dAt = A*dW; sigma = 1 - exp(lt);
//   dZ = dAt - sigma*(prefix_cumsum(dAt) + b)
// Phase 1 (:337-357): per query tile, key blocks left to right from first_kb,
//   b carried in registers, N snapshot = b in effect per tile, dQ += dZ K.
// Phase 2 (:367-386): per 64-key block, query tiles top to bottom over visited
//   tiles, b = N snapshot, dK += dZ^T Q, dV += A^T dO — owned rows, no atomics,
//   deterministic.  dK and dV are accumulated in TMEM with M = 128 keys (A^T /
//   dZ^T reach the tensor core through MN-major smem descriptors).
// Store mode (default when the workspace fits): phase 1 also TMA-stores every dZ
//   tile; phase 2 (sb_bwd_kvs_kernel) loads it instead of recomputing dO V^T and
//   dZ, and recomputes only A (same results bit for bit: the stored tiles are the
//   values the recompute-mode phase 2, sb_bwd_kv_kernel, would compute).
//
// Both phases use the ping-pong layout of sb_fwd_pp.cu: two stick warpgroups
// per CTA (thread r <-> TMEM lane r <-> query row, all 64 key columns of a tile
// in registers), each with its own MMA-issuer thread and TMEM/smem buffers.
//   phase 1: WG w owns query tile 2p+w; both share one K/V stream.
//   phase 2: WG w owns key block 2p+w; both share one Q/dO stream.
// Tile math is the product form (sb_common.cuh): A_c = sigma_c * e^M *
// prod_{c'>c} r_c', sigma = t/(1+t), r = 1/(1+t), with one rcp per 16 columns
// (batched reciprocal, recompute_row).
// Warps: 0-3 WG0, 4-7 WG1, 8 TMA producer (+TMEM allocator), 9/10 MMA for WG0/WG1,
// 11 phase 1's V producer / phase 2's dO producer (store mode: 10 loads dZ, 9 is
// the single issuer); warpgroup 2 hands its registers to the stick warpgroups
// (setmaxnreg).
#include "sb_args.cuh"

namespace sb {

constexpr int kBwdThreads = 12 * 32;  // WG0, WG1 stick; WG2 = producer, MMA0, MMA1, idle
constexpr bool kPingPongQ = true;  // phase 1: the warpgroups take turns at the recompute
// setmaxnreg only redistributes the CTA's launch allocation (384 threads x 168
// registers): 128 x low + 256 x high <= 384 x 168, otherwise .inc blocks forever.
constexpr int kRegsLaunch = 168;
constexpr int kRegsLowQ = 72, kRegsHighQ = 216;    // phase 1
constexpr int kRegsLowKV = 88, kRegsHighKV = 208;  // phase 2 (issuer holds more descriptors)
static_assert(128 * kRegsLowKV + 256 * kRegsHighKV <= kBwdThreads * kRegsLaunch, "register budget");
static_assert(128 * kRegsLowQ + 256 * kRegsHighQ <= kBwdThreads * kRegsLaunch, "register budget");

// Recompute of one row of a tile: on entry s[] = raw q.k dot products, on exit
// s[c] = A_c and sg[c] = -sigma_c (both 0 where masked; negated for dz_row).  E = e^M (the M
// snapshot in linear space).
// Batched reciprocal per group of 16 columns (see batched_row in sb_common.cuh):
// with P_i = prod_{k<=i} (1+t_k) (within the group), u_i = t_i P_{i-1} and one
// rcp of the group total P_15,
//   A_i = u_i * (Q_g/P_15),   sigma_i = u_i / P_i,
// where Q_g = E * prod of r over the groups to the right.  Pass 1 (left to
// right) keeps t in s[] and P in sg[]; pass 2 walks each group right to left
// with the running 1/P_i (one FFMA per element).  The four groups are
// independent chains in both passes (only the scalar Q_g links them), so the
// scheduler can interleave them: 6 FP32 ops + 1 ex2 per element.  A row whose
// group product reaches 2^64 (large logits; t = inf included) falls back to one
// rcp per element.
// Split in two so phase 1 can derive E from the group totals in between
// (row_pass1 -> tot[], then row_pass2 with E).
// kSigma = false (store-mode phase 2): A only; sg[] is scratch.
template <bool kDiag>
__device__ __forceinline__ void row_pass1(float* s, float* sg, float scale_log2, int lim,
                                          float* tot) {
#ifdef SB_NOMATH  // tuning ablation: pipeline without the stick math
  tot[0] = tot[1] = tot[2] = tot[3] = 1.0f;
  return;
#endif
  // The multiplies run as packed f32x2 (FMUL2 / FFMA2, sb_common.cuh batched_row):
  // the scale on adjacent column pairs, everything else on the group pairs
  // (0,1) and (2,3), i.e. columns (c, c+16); bit-identical to the scalar form.
  const float2 sl2 = make_float2(scale_log2, scale_log2);
  float2 tp[2] = {make_float2(1.0f, 1.0f), make_float2(1.0f, 1.0f)};
#pragma unroll
  for (int c = 0; c < kBlock; c += 2) {
    const float2 z = mul2(make_float2(s[c], s[c + 1]), sl2);
    float t0 = ex2(z.x), t1 = ex2(z.y);
    if (kDiag) {
      t0 = c < lim ? t0 : 0.0f;
      t1 = c + 1 < lim ? t1 : 0.0f;
    }
    s[c] = t0;
    s[c + 1] = t1;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = 32 * h + i;
      tp[h] = fma2(tp[h], make_float2(s[c], s[c + 16]), tp[h]);
      sg[c] = tp[h].x;
      sg[c + 16] = tp[h].y;
    }
  tot[0] = tp[0].x;
  tot[1] = tp[0].y;
  tot[2] = tp[1].x;
  tot[3] = tp[1].y;
}

template <bool kSigma = true>
__device__ __forceinline__ void row_pass2(float* s, float* sg, float E, const float* tot) {
#ifdef SB_NOMATH
#pragma unroll
  for (int c = 0; c < kBlock; ++c) { s[c] *= E; sg[c] = E; }
  return;
#endif
  constexpr int NG = kBlock / 16;
  bool ok = true;
#pragma unroll
  for (int g = 0; g < NG; ++g) ok = ok && (tot[g] < kBatchedMax);
  auto fast = [&]() {
    // ninv = -1/P_i (running): sg leaves as -sigma for dz_row's FFMA2
    float2 inv[2], K[2];
    inv[1].y = rcp(tot[3]);
    inv[1].x = rcp(tot[2]);
    inv[0].y = rcp(tot[1]);
    inv[0].x = rcp(tot[0]);
#pragma unroll
    for (int h = 0; h < 2; ++h) inv[h] = make_float2(-inv[h].x, -inv[h].y);
    // first u = t_i P_{i-1} (into s[]) and sigma, which need no E; then A = u K with
    // the E-dependent group seeds K, so E (phase 1 derives it from this tile's group
    // totals) has the whole first loop to arrive
#pragma unroll
    for (int i = 15; i >= 0; --i)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 32 * h + i;
        const float2 t = make_float2(s[c], s[c + 16]);
        const float2 u = i ? mul2(t, make_float2(sg[c - 1], sg[c + 15])) : t;
        if (kSigma) {
          const float2 sgm = mul2(u, inv[h]);
          sg[c] = sgm.x;
          sg[c + 16] = sgm.y;
          inv[h] = fma2(inv[h], t, inv[h]);
        }
        s[c] = u.x;
        s[c + 16] = u.y;
      }
    const float Q = E;
    K[1].y = Q * rcp(tot[3]);
    K[1].x = K[1].y * rcp(tot[2]);
    K[0].y = K[1].x * rcp(tot[1]);
    K[0].x = K[0].y * rcp(tot[0]);
#pragma unroll
    for (int i = 15; i >= 0; --i)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = 32 * h + i;
        const float2 a = mul2(make_float2(s[c], s[c + 16]), K[h]);
        s[c] = a.x;
        s[c + 16] = a.y;
      }
  };
  if (ok) {
    fast();
  } else {
    // the wider range (sb_common.cuh), with the fast path's seed arithmetic
    bool wide = true;
    float k0 = E;
#pragma unroll
    for (int g = NG - 1; g >= 0; --g) {
      wide = wide && (tot[g] < kBatchedWide);
      k0 = k0 * rcp(tot[g]);
    }
    if (wide && batched_seed_ok(k0, E)) {
      fast();
    } else {
      float Q = E;
#pragma unroll
      for (int c = kBlock - 1; c >= 0; --c) {
        const float t = s[c];
        const float r = rcp(1.0f + t);
        const float sgm = fminf(t * r, 1.0f);  // t = inf: NaN -> 1
        s[c] = sgm * Q;
        sg[c] = -sgm;
        Q *= r;
      }
    }
  }
}

template <bool kDiag, bool kSigma = true>
__device__ __forceinline__ void recompute_row(float* s, float* sg, float scale_log2, float E,
                                              int lim) {
  float tot[4];
  row_pass1<kDiag>(s, sg, scale_log2, lim, tot);
  row_pass2<kSigma>(s, sg, E, tot);
}

// Row total of lt over one tile in log2 units, L = log2 prod (1+t) >= 0, for a row
// outside the 2^64 range (rare: large logits): t[] = the row's t values (masked
// columns 0), tot[] the group products of (1+t).  lg2 per group below 2^126 (as the
// forward's wider range), past that the exact softplus of every element of the
// group (softplus2 of Z = lg2 t; where t = inf, z itself from the q row and the key
// rows in global memory).  Out of line with t[] in local memory, so the hot
// path's code and registers stay as they were.
__device__ __noinline__ float row_lt_total_slow(const float* t, float4 tot4,
                                                const __nv_bfloat16* qrow,
                                                const __nv_bfloat16* krow0, int64_t ld, int d,
                                                float scale_log2) {
  const float tot[4] = {tot4.x, tot4.y, tot4.z, tot4.w};
  float lg[4];
  for (int g = 0; g < 4; ++g) {
    if (tot[g] < kBatchedWide) {
      lg[g] = lg2(tot[g]);
      continue;
    }
    float sum = 0.0f;
    for (int c = 16 * g; c < 16 * g + 16; ++c) {
      const float tc = t[c];
      if (!(tc > 0.0f)) continue;  // masked, or softplus below the float range
      float Z;
      if (tc < INFINITY) {
        Z = lg2(tc);
      } else {
        float z = 0.0f;
        const __nv_bfloat16* kr = krow0 + c * ld;
        for (int i = 0; i < d; ++i) z = fmaf(__bfloat162float(qrow[i]), __bfloat162float(kr[i]), z);
        Z = z * scale_log2;
      }
      sum += softplus2(Z, tc);
    }
    lg[g] = sum;
  }
  return (lg[3] + lg[2]) + (lg[1] + lg[0]);
}

// dAt = A * (dW - off) with dW streamed from TMEM in 16-column chunks (warp-collective).
template <bool kOff>
__device__ __forceinline__ void load_dat(float* s, uint32_t taddr, float off) {
#pragma unroll
  for (int ch = 0; ch < 2; ++ch) {
    float w[32];
    tmem_ld32(taddr + ch * 32, w);
    tmem_wait_ld();
#pragma unroll
    for (int c = 0; c < 32; ++c) s[ch * 32 + c] *= kOff ? (w[c] - off) : w[c];
  }
}

// dZ = dAt - sigma*(prefix(dAt) + b), packed to bf16; returns b + rowsum(dAt).
// nsg[] = -sigma (recompute_row's output).  Four prefix chains of 16 columns run
// as two f32x2 pairs, chains (0,1) and (2,3) = columns (c, c+16): a first pass
// sums each chain, the second runs every chain from its exact offset
// (b + the sums to its left) with one FADD2 and one FFMA2 per column pair.
__device__ __forceinline__ float dz_row(const float* dat, const float* nsg, float b, uint32_t* pk) {
  float2 sa = make_float2(0.0f, 0.0f), sb2 = sa;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    sa = add2(sa, make_float2(dat[c], dat[c + 16]));
    sb2 = add2(sb2, make_float2(dat[c + 32], dat[c + 48]));
  }
  const float o1 = b + sa.x, o2 = o1 + sa.y, o3 = o2 + sb2.x;
  float2 xa = make_float2(b, o1), xb = make_float2(o2, o3);
  float2 za0 = xa, zb0 = xb;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const float2 da = make_float2(dat[c], dat[c + 16]);
    const float2 db = make_float2(dat[c + 32], dat[c + 48]);
    xa = add2(xa, da);
    xb = add2(xb, db);
    const float2 za = fma2(make_float2(nsg[c], nsg[c + 16]), xa, da);
    const float2 zb = fma2(make_float2(nsg[c + 32], nsg[c + 48]), xb, db);
    if (c & 1) {
      pk[c >> 1] = pack_bf16(za0.x, za.x);
      pk[(c + 16) >> 1] = pack_bf16(za0.y, za.y);
      pk[(c + 32) >> 1] = pack_bf16(zb0.x, zb.x);
      pk[(c + 48) >> 1] = pack_bf16(zb0.y, zb.y);
    } else {
      za0 = za;
      zb0 = zb;
    }
  }
  return o3 + sb2.y;
}

__device__ __forceinline__ void store_row_sw128(uint32_t row_addr, int r, const uint32_t* pk) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
    st_shared_v4(row_addr + ((c ^ (r & 7)) << 4), pk[4 * c], pk[4 * c + 1], pk[4 * c + 2],
                 pk[4 * c + 3]);
}

// ============================================================================
// Phase 1: dQ and N.  CTA = (b, h, query tiles 2p and 2p+1).
template <int D>
struct BwdQCfg {
  // K ring (S(j) and dQ(j) read K(j): released at the end of tile j); V ring (only
  // dW(j) reads V(j): released early in tile j).
  // Q only stages the copy into TMEM at the item start: d = 128 keeps ONE Q buffer that
  // the two warpgroups' tiles take in turn, which makes room for a second V stage and a
  // fourth K stage (C2 phase 1 0.909 -> 0.896 ms with dW(j+1) issued ahead of dQ(j);
  // V ring 2 alone 0.902); d = 64 has room for a Q buffer per warpgroup, a K ring of 6
  // and a V ring of 3 (C4 phase 1: K 3 / V 1 2.33 -> K 4 / V 2 2.31 (round 1) ->
  // K 6 / V 3 2.353 -> 2.311 ms in one A/B; K 8 did not help)
#ifndef SB_P1_KST128
#define SB_P1_KST128 4
#endif
#ifndef SB_P1_VST128
#define SB_P1_VST128 2
#endif
#ifndef SB_P1_KST64
#define SB_P1_KST64 6
#endif
#ifndef SB_P1_VST64
#define SB_P1_VST64 3
#endif
  static constexpr int kStages = D == 64 ? SB_P1_KST64 : SB_P1_KST128;   // K ring
  static constexpr int kVStages = D == 64 ? SB_P1_VST64 : SB_P1_VST128;  // V ring (own producer)
  static constexpr int kQBufs = D == 64 ? 2 : (SB_P1_VST128 > 1 ? 1 : 2);
  static constexpr int kQBytes = kTileM * D * 2;
  static constexpr int kKVBytes = kBlock * D * 2;
  static constexpr int kZBytes = kTileM * kBlock * 2;
  static constexpr int kOffQ = 0;                          // Q[kQBufs]
  static constexpr int kOffDO = kOffQ + kQBufs * kQBytes;  // dO[2]
  static constexpr int kOffK = kOffDO + 2 * kQBytes;    // K ring
  static constexpr int kOffV = kOffK + kStages * kKVBytes;
  static constexpr int kOffZ = kOffV + kVStages * kKVBytes;  // Z[2] (one per WG)
  static constexpr int kOffBar = kOffZ + 2 * kZBytes;
  static constexpr int kNumBars = 2 + 2 * kStages + 2 * kVStages + 2 * 8 + 1 + 8 + 2 + 2;
  static constexpr int kOffMisc = kOffBar + kNumBars * 8;
  static constexpr int kSmem = kOffMisc + 64 + 1024;
  static_assert(kSmem <= 232448, "exceeds the 227 KB opt-in shared memory per block");
  __host__ __device__ static constexpr int q_off(int w) { return kOffQ + (kQBufs == 2 ? w : 0) * kQBytes; }
  static constexpr uint32_t kTmemCols = 512;  // per WG w at w*256: S +0, dW +64, dQ +128
};

// Work item of phase 1: (unit, query-tile pair p); all roles derive the same list.
struct QItem {
  Unit u;
  int b, h, p, kbhi0, kbhi1, kb_lo, n_s;
  bool has1, valid;
};
__device__ __forceinline__ QItem q_item(const Geom& g, const int* first_kb, int idx,
                                        bool even_lo = false) {
  QItem it;
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
  it.kb_lo = it.kbhi1;
  if (it.valid) {
    const int* fkb = first_kb + it.u.fkb_off;
    for (int qb = 4 * it.p; qb <= it.kbhi1; ++qb) it.kb_lo = min(it.kb_lo, fkb[qb]);
    // store mode: start at an even key block so every key pair phase 2 loads has
    // both of its tiles written (the extra tile is all dead rows: dZ = 0)
    if (even_lo) it.kb_lo &= ~1;
  }
  it.n_s = it.kbhi1 - it.kb_lo + 1;  // stream tiles, kb = kb_lo .. kbhi1
  return it;
}

// Persistent: one CTA per SM takes (unit, query pair) items from a global work
// queue.  The K ring / V buffer and each warpgroup's S, dW, dZ barriers run on
// counters that continue across items; the next item's Q[w] loads once warpgroup w
// copied the current Q tile into TMEM (bar_qtm), its dO once both warpgroups issued
// their last dW of the current item (qdo_free), and its
// first dQ MMA waits until the warpgroup read dQ out of TMEM (dq_free).
// kStoreZ (store mode): each dZ tile also goes to the tile workspace (TMA store
// from the swizzled smem buffer, issued with the dQ MMA) for phase 2 to reuse.
template <int D, bool kStoreZ>
__global__ void __launch_bounds__(kBwdThreads, 1)
    sb_bwd_q_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                    const __grid_constant__ CUtensorMap tm_z, const BwdArgs args) {
  using C = BwdQCfg<D>;
  constexpr int ST = C::kStages, VST = C::kVStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const Geom& g = args.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = ((g.n_qt + 1) / 2) * g.B * g.H;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  // Q/dO landed, one barrier per warpgroup (completes once per item with a tile for
  // it; see the forward's bar_q: a shared one let WG1's issuer, skipping items
  // without a second tile, alias a phase two ahead)
  uint64_t* bar_qdo = bars;  // [2]
  uint64_t* bar_kfull = bars + 2;
  uint64_t* bar_kempty = bar_kfull + ST;
  uint64_t* bar_vfull = bar_kempty + ST;
  uint64_t* bar_vempty = bar_vfull + VST;
  uint64_t* wgbars = bar_vempty + VST;  // per wg: sfull, sempty, wfull, wempty, zfull, zempty, done, dq_free
  uint64_t* bar_qdofree = wgbars + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);
  const SchedRing sq{reinterpret_cast<int*>(smem + C::kOffMisc + 16), bar_qdofree + 1,
                     bar_qdofree + 5};
  uint64_t* bar_qtm = bar_qdofree + 9;  // [2] the warpgroup copied its Q tile into TMEM
  // Q and dO land on separate barriers (bar_qdo: Q only), Q first: the Q copy into TMEM
  // and the item's first S do not wait for dO
  uint64_t* bar_do = bar_qdofree + 11;  // [2]

  if (threadIdx.x == 0) {
    mbar_init(bar_qdo, 1);
    mbar_init(bar_qdo + 1, 1);
    mbar_init(bar_qtm, 128);
    mbar_init(bar_qtm + 1, 128);
    mbar_init(bar_do, 1);
    mbar_init(bar_do + 1, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(bar_kfull + s, 1);
      mbar_init(bar_kempty + s, 2);  // one arrival per warpgroup issuer (dQ read K)
    }
    for (int s = 0; s < VST; ++s) {
      mbar_init(bar_vfull + s, 1);
      mbar_init(bar_vempty + s, 2);  // one arrival per warpgroup issuer (dW read V)
    }
    for (int w = 0; w < 2; ++w) {
      mbar_init(wgbars + w * 8 + 0, 1);    // sfull: S = Q K^T landed in TMEM
      mbar_init(wgbars + w * 8 + 1, 128);  // sempty: S read into registers
      mbar_init(wgbars + w * 8 + 2, 1);    // wfull: dW = dO V^T landed
      mbar_init(wgbars + w * 8 + 3, 128);  // wempty: dW read
      mbar_init(wgbars + w * 8 + 4, 128);  // zfull: dZ in smem
      mbar_init(wgbars + w * 8 + 5, kStoreZ ? 2 : 1);  // zempty: dQ MMA (+ tile store) read dZ
      mbar_init(wgbars + w * 8 + 6, 1);    // done: the item's last dQ MMA completed
      mbar_init(wgbars + w * 8 + 7, 128);  // dq_free: dQ read out of TMEM
    }
    mbar_init(bar_qdofree, 2);
    sched_init(sq, 11);  // consumers: stick warps 0-7, issuer warps 9-10, V producer 11
    fence_mbar_init();
  }
  if (warp == 8) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp >= 8) {
    reg_dealloc<kRegsLowQ>();
    if (warp == 8) {
      // ---------------------------------------------------------- TMA producer
      const bool leader = elect_one();
      if (leader) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_do);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
      }
      int jg = 0, ni = 0, nq[2] = {0, 0}, qlast = -1;
      for (int kq = 0;; ++kq) {
        const int idx = sched_produce(sq, kq, args.sched, n_items);
        if (idx < 0) break;
        const QItem it = q_item(g, args.first_kb, idx, kStoreZ);
        if (!it.valid) continue;
        const Unit& u = it.u;
        const int nw = it.has1 ? 2 : 1;
        // A Q buffer is free as soon as the warpgroup whose tile it held copied it into
        // TMEM (early in that item): the next Q loads while the current item still
        // streams.  One shared buffer (d = 128): WG1's tile first (WG1 takes the first
        // turn of every round), WG0's after WG1 copied it (L2-prefetched meanwhile).
        for (int i = 0; i < nw; ++i) {
          const int w = C::kQBufs == 2 ? i : nw - 1 - i;
          const int prev = C::kQBufs == 2 ? w : qlast;
          if (prev >= 0 && nq[prev] >= 1) mbar_wait_warp(bar_qtm + prev, (nq[prev] - 1) & 1);
          if (leader) {
            mbar_expect_tx(bar_qdo + w, C::kQBytes);
            for (int c = 0; c < D / 64; ++c)
              tma_load_4d(&tm_q, bar_qdo + w, smem + C::q_off(w) + c * (kTileM * 128), c * 64,
                          u.trow0 + (2 * it.p + w) * kTileM, it.h, u.tb);
            if (C::kQBufs == 1 && i == 0 && nw == 2)
              for (int c = 0; c < D / 64; ++c)
                tma_prefetch_4d(&tm_q, c * 64, u.trow0 + 2 * it.p * kTileM, it.h, u.tb);
          }
          __syncwarp();
          ++nq[w];
          qlast = w;
        }
        // dO: once both warpgroups issued the previous item's last dW
        if (ni >= 1) mbar_wait_warp(bar_qdofree, (ni - 1) & 1);
        SB_TR(args, 0, ni, 12);
        if (leader) {
          for (int w = 0; w < nw; ++w) {
            mbar_expect_tx(bar_do + w, C::kQBytes);
            for (int c = 0; c < D / 64; ++c)
              tma_load_4d(&tm_do, bar_do + w,
                          smem + C::kOffDO + w * C::kQBytes + c * (kTileM * 128), c * 64,
                          u.trow0 + (2 * it.p + w) * kTileM, it.h, u.tb);
          }
        }
        __syncwarp();
        for (int j = 0; j < it.n_s; ++j, ++jg) {
          const int s = jg % ST;
          if (jg >= ST) mbar_wait_warp(bar_kempty + s, ((jg / ST) - 1) & 1);
          SB_TR(args, 2, jg, 12);
          const int kb = it.kb_lo + j;
          if (leader) {
            mbar_expect_tx(bar_kfull + s, C::kKVBytes);
            for (int c = 0; c < D / 64; ++c)
              tma_load_4d(&tm_k, bar_kfull + s,
                          smem + C::kOffK + s * C::kKVBytes + c * (kBlock * 128), c * 64,
                          u.trow0 + kb * kBlock, it.h, u.tb);
          }
          __syncwarp();
        }
        ++ni;
      }
    } else if (warp == 11) {
      // ---------------------------------------------------------- V producer: its ring
      // is released early (dW reads V), so it runs ahead of the K ring's producer
      const bool leader = elect_one();
      int jg = 0;
      for (int kq = 0;; ++kq) {
        const int idx = sched_consume(sq, kq);
        if (idx < 0) break;
        const QItem it = q_item(g, args.first_kb, idx, kStoreZ);
        if (!it.valid) continue;
        const Unit& u = it.u;
        for (int j = 0; j < it.n_s; ++j, ++jg) {
          const int s = jg % VST;
          if (jg >= VST) mbar_wait_warp(bar_vempty + s, ((jg / VST) - 1) & 1);
          if (leader) {
            mbar_expect_tx(bar_vfull + s, C::kKVBytes);
            for (int c = 0; c < D / 64; ++c)
              tma_load_4d(&tm_v, bar_vfull + s, smem + C::kOffV + s * C::kKVBytes + c * (kBlock * 128),
                          c * 64, u.trow0 + (it.kb_lo + j) * kBlock, it.h, u.tb);
          }
          __syncwarp();
        }
      }
    } else if (warp == 9 || warp == 10) {
      // ---------------------------------------------------------- MMA issuer of one WG
      // whole warp: uniform control flow and descriptors; one elected lane issues
      const int w = warp - 9;
      uint64_t *sfull = wgbars + w * 8, *sempty = sfull + 1, *wfull = sfull + 2,
               *wempty = sfull + 3, *zfull = sfull + 4, *zempty = sfull + 5, *done = sfull + 6,
               *dq_free = sfull + 7;
      constexpr uint32_t idesc_s = idesc_bf16(128, 64, 0, 0);  // Q K^T, dO V^T
      constexpr uint32_t idesc_q = idesc_bf16(128, D, 0, 1);   // dZ K: K is MN-major
      const uint64_t ddo = sdesc_sw128(smem_u32(smem + C::kOffDO + w * C::kQBytes), 16, 1024);
      const uint64_t dk = sdesc_sw128(smem_u32(smem + C::kOffK), 16, 1024);
      const uint64_t dkmn = sdesc_sw128(smem_u32(smem + C::kOffK), kBlock * 128, 1024);
      const uint64_t dv = sdesc_sw128(smem_u32(smem + C::kOffV), 16, 1024);
      const uint64_t dz = sdesc_sw128(smem_u32(smem + C::kOffZ + w * C::kZBytes), 16, 1024);
      // per warpgroup: dQ accumulator (128 columns), one buffer for S and then dW (64),
      // Q (the TS MMA's A operand, 64)
      const uint32_t tQ = tbase + w * 256, tS = tQ + 128, tW = tS, tQtm = tQ + 192;
      const bool leader = elect_one();
      int jg = 0, ni = 0, ig = 0, nwi = 0;
      for (int kq = 0;; ++kq) {
        const int idx = sched_consume(sq, kq);
        if (idx < 0) break;
        const QItem it = q_item(g, args.first_kb, idx, kStoreZ);
        if (!it.valid) continue;
        if (w == 1 && !it.has1) {  // no tile for this warpgroup: release the stream
          for (int j = 0; j < it.n_s; ++j) {
            const int js = jg + j;
            mbar_wait_warp(bar_kfull + js % ST, (js / ST) & 1);
            if (leader) mbar_arrive(bar_kempty + js % ST);
            mbar_wait_warp(bar_vfull + js % VST, (js / VST) & 1);
            if (leader) mbar_arrive(bar_vempty + js % VST);
            __syncwarp();
          }
          // (after a K of this item landed: the producer is past the previous
          // item's qdo_free phase, so this arrival counts for this item's phase)
          if (leader) mbar_arrive(bar_qdofree);
          __syncwarp();
          jg += it.n_s;
          ++ni;
          continue;
        }
        const int n_w = (w ? it.kbhi1 : it.kbhi0) - it.kb_lo + 1;
        // Static issue order: S(j+1) once S(j) was read (it runs while the
        // warpgroup still works on tile j), dW(j+1) once dW(j) was read and V(j+1)
        // landed, dQ(j) once dZ(j) is in smem.
        auto issue_s = [&](int j) {
          const int js = jg + j, s = js % ST, gi = ig + j;
          mbar_wait_warp(bar_kfull + s, (js / ST) & 1);
          SB_TR(args, 2 + w, gi, 13);
          // the shared S/dW buffer is free once dW(j-1) was read; the item's first S
          // needs this item's Q in TMEM
          if (gi >= 1) mbar_wait_warp(wempty, (gi - 1) & 1);
          if (j == 0) mbar_wait_warp(bar_qtm + w, nwi & 1);
          SB_TR(args, 2 + w, gi, 8);
          tc_fence_after();
          if (leader) {
#pragma unroll
            for (int k = 0; k < D / 16; ++k) {
              const uint32_t offk = (k >> 2) * (kBlock * 128) + (k & 3) * 32;
              umma_ts_at(tS, tQtm + k * 8, dk, s * C::kKVBytes + offk, idesc_s, k > 0);
            }
            umma_commit(sfull);
          }
          __syncwarp();
        };
        auto issue_w = [&](int j) {
          const int js = jg + j, gi = ig + j, sv = js % VST;
          if (j == 0) mbar_wait_warp(bar_do + w, nwi & 1);  // this warpgroup's nwi-th dO tile
          mbar_wait_warp(bar_vfull + sv, (js / VST) & 1);
          mbar_wait_warp(sempty, gi & 1);  // S(j) was read out of the shared buffer
          SB_TR(args, 2 + w, gi, 10);
          tc_fence_after();
          if (leader) {
#pragma unroll
            for (int k = 0; k < D / 16; ++k) {
              const uint32_t off = (k >> 2) * (kTileM * 128) + (k & 3) * 32;
              const uint32_t offk = (k >> 2) * (kBlock * 128) + (k & 3) * 32;
              umma_ss_at(tW, ddo, off, dv, sv * C::kKVBytes + offk, idesc_s, k > 0);
            }
            umma_commit(wfull);
            umma_commit(bar_vempty + sv);
            if (j + 1 == n_w) umma_commit(bar_qdofree);  // Q and dO read for the last time
          }
          __syncwarp();
        };
        issue_s(0);
        issue_w(0);
        for (int j = 0; j < n_w; ++j) {
          if (j + 1 < n_w) issue_s(j + 1);
          // dW(j+1) ahead of dQ(j), as soon as dW(j) was read (C4 phase 1 2.32 -> 2.30 ms;
          // C2 0.902 -> 0.896; with d=128's former single V buffer the early order was
          // slower, 0.915 -> 0.956 ms: dW(j+1) then waited for V behind dQ(j))
#ifndef SB_P1_EARLYW128
#define SB_P1_EARLYW128 1
#endif
          constexpr bool kEarlyW = D == 64 || SB_P1_EARLYW128;
          if (kEarlyW && j + 1 < n_w) issue_w(j + 1);
          const int js = jg + j, s = js % ST, gi = ig + j;
          mbar_wait_warp(zfull, gi & 1);
          SB_TR(args, 2 + w, gi, 11);
          // the previous item's dQ must be out of TMEM before it is overwritten
          if (j == 0 && nwi >= 1) mbar_wait_warp(dq_free, (nwi - 1) & 1);
          tc_fence_after();
          if (leader) {
#pragma unroll
            for (int k = 0; k < kBlock / 16; ++k)
              umma_ss_at(tQ, dz, k * 32, dkmn, s * C::kKVBytes + k * 2048, idesc_q,
                         (j > 0 || k > 0) ? 1u : 0u);
            umma_commit(zempty);
            umma_commit(bar_kempty + s);
            if (j + 1 == n_w) umma_commit(done);
            if (kStoreZ) {  // dZ(j) -> tile workspace
              tma_store_3d(&tm_z, smem + C::kOffZ + w * C::kZBytes, 0, 0,
                           (int)(it.u.z_off + ztile(2 * it.p + w, it.kb_lo + j)));
              bulk_commit();
            }
          }
          __syncwarp();
          if (!kEarlyW && j + 1 < n_w) issue_w(j + 1);
          if (kStoreZ) {  // the store has read the buffer: second arrival on zempty
            if (leader) {
              bulk_wait_read0();
              mbar_arrive(zempty);
            }
            __syncwarp();
          }
        }
        for (int j = n_w; j < it.n_s; ++j) {  // stream tiles right of this WG's diagonal
          // release each buffer in its own phase: wait until tile j occupies it
          const int js = jg + j;
          mbar_wait_warp(bar_kfull + js % ST, (js / ST) & 1);
          if (leader) mbar_arrive(bar_kempty + js % ST);
          mbar_wait_warp(bar_vfull + js % VST, (js / VST) & 1);
          if (leader) mbar_arrive(bar_vempty + js % VST);
          __syncwarp();
        }
        jg += it.n_s;
        ig += n_w;
        ++ni;
        ++nwi;
      }
      // the dZ tile stores must have reached global memory before the CTA exits
      if (kStoreZ && leader) bulk_wait0();
      __syncwarp();
    }
  } else {
    reg_alloc<kRegsHighQ>();
    // ------------------------------------------------------------ stick warpgroups
    const int w = warp >> 2;
    uint64_t *sfull = wgbars + w * 8, *sempty = sfull + 1, *wfull = sfull + 2,
             *wempty = sfull + 3, *zfull = sfull + 4, *zempty = sfull + 5, *done = sfull + 6,
             *dq_free = sfull + 7;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t tQ = tbase + w * 256 + lane_base, tS = tQ + 128, tW = tS, tQtm = tQ + 192;
    const uint32_t z_row = smem_u32(smem + C::kOffZ + w * C::kZBytes) + r * 128;
    const float scale = g.scale_log2 * kLn2;
    const bool tr = quarter == 0 && lane == 0;
    if (tr) SB_TR(args, w, 0, 14);
    // Ping-pong of the MUFU-heavy recompute: the two warpgroups take turns (named
    // barriers 1 and 2, FA3-style), so one's recompute overlaps the other's dW
    // wait, dZ math and stores instead of both contending for the MUFU at once.
    // Round k of an item: WG1 (the query tile with the longer key stream) waits
    // bar 2, recomputes, arrives on bar 1; then WG0 waits bar 1, recomputes,
    // arrives on bar 2.  Both run max(n0, n1) rounds per item (a warpgroup without
    // a tile in a round passes straight through).  (WG1 first: 0.94-0.95 ms vs
    // 0.96-0.97 with WG0 first; letting WG0 skip its trailing rounds and go on to
    // its epilogue: 1.14 ms, the turn order then drifts.)
    const uint32_t bar_mine = 1 + w, bar_other = 2 - w;
    auto pp_round_pass = [&]() {
      named_bar_sync(bar_mine, 256);
      named_bar_arrive(bar_other, 256);
    };
    if (kPingPongQ && w == 0) named_bar_arrive(2, 256);  // WG1 (the longer tile stream) goes first
    int ig = 0, nwi = 0;
    for (int kq = 0;; ++kq) {
      const int idx = sched_consume(sq, kq);
      if (idx < 0) break;
      const QItem it = q_item(g, args.first_kb, idx, kStoreZ);
      if (!it.valid) continue;
      const int n0 = it.kbhi0 - it.kb_lo + 1, n1 = it.has1 ? it.kbhi1 - it.kb_lo + 1 : 0;
      const int n_rounds = max(n0, n1);
      if (w == 1 && !it.has1) {
        if (kPingPongQ)
          for (int j = 0; j < n_rounds; ++j) pp_round_pass();
        continue;
      }
      const Unit& u = it.u;
      const int qt = 2 * it.p + w;
      const int my_qb = 2 * qt + (r >> 6);
      const int row = qt * kTileM + r;
      const bool row_valid = row < u.L;
      const bool half_exists = my_qb < u.nb;
      const int my_first = half_exists ? args.first_kb[u.fkb_off + my_qb] : u.nb;
      const float off =
          (args.row_offset && row_valid) ? args.row_offset[u.rem_off + row * u.rem_stride] : 0.0f;
      // M snapshots (a in effect per tile, blocked.py:188-189) are rolled back from the
      // forward's final a, left to right: M(kb) = a_final + sum_{kb' <= kb} L(kb'), L =
      // the tile's row total of -lt (float64 running sum); phase 2 reads what this
      // writes.  store mode: no N (phase 2 takes dZ from the tile workspace)
      float* Mrow = args.M + u.m_off + (r & 63);
      float* Nrow = kStoreZ ? nullptr : args.N + u.m_off + (r & 63);
      const int n_w = (w ? it.kbhi1 : it.kbhi0) - it.kb_lo + 1;
      // the rolled-back a as a compensated float pair (float64 adds cost 6% in the forward)
      float m_hi, m_lo;
      {
        const double a0 = row_valid ? args.state[u.rem_off + row * u.rem_stride] : 0.0;
        m_hi = (float)a0;
        m_lo = (float)(a0 - (double)m_hi);
      }
      float bsum = 0.0f;  // running b (blocked.py:342, :354)
      {
        // copy this thread's Q row (TMA-swizzled smem) into TMEM lane r: the A operand of
        // the TS MMA S = Q K^T (as the forward does)
        mbar_wait(bar_qdo + w, nwi & 1);
        const uint32_t qrow = smem_u32(smem + C::q_off(w)) + r * 128;
        uint32_t qv[D / 2];
#pragma unroll
        for (int c = 0; c < D / 8; ++c) {
          const uint4 x = ld_shared_v4(qrow + (c >> 3) * (kTileM * 128) + (((c & 7) ^ (r & 7)) << 4));
          qv[4 * c] = x.x;
          qv[4 * c + 1] = x.y;
          qv[4 * c + 2] = x.z;
          qv[4 * c + 3] = x.w;
        }
        if constexpr (D == 128) tmem_st64(tQtm, qv);
        else tmem_st32(tQtm, qv);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(bar_qtm + w);
      }
      if (tr) SB_TR(args, w, nwi, 11);
      for (int j = 0; j < n_w; ++j) {
        const int kb = it.kb_lo + j, gi = ig + j;
        const bool live = row_valid && kb >= my_first && kb <= my_qb;
        const int64_t t = tile_index(my_qb, kb) * kBlock;
        if (tr) SB_TR(args, w, gi, 0);
        mbar_wait(sfull, gi & 1);
        tc_fence_after();
        float s[64], sg[64];
        tmem_ld32(tS, s);
        tmem_ld32(tS + 32, s + 32);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(sempty);  // S(j+1) may overwrite the buffer now
        if (tr) SB_TR(args, w, gi, 1);
        const bool diag = kb == my_qb;  // warp-uniform
        if (kPingPongQ) named_bar_sync(bar_mine, 256);
        if (tr) SB_TR(args, w, gi, 7);
        // dead rows/tiles run the same code with e^M = 0 and b = 0: A = 0, dZ = 0
        float tot[4], Mk;
        if (diag) row_pass1<true>(s, sg, g.scale_log2, r & 63, tot);
        else row_pass1<false>(s, sg, g.scale_log2, kBlock, tot);
        if (tr) SB_TR(args, w, gi, 8);
        // the turn ends with the ex2 pass (the MUFU-heavy part): L, E and the
        // FMA-pipe pass 2 overlap the other warpgroup's ex2 pass (0.6% faster than
        // holding the turn to the end of pass 2)
        if (kPingPongQ) named_bar_arrive(bar_other, 256);
        {
          float L;
          if (tot[0] < kBatchedMax && tot[1] < kBatchedMax && tot[2] < kBatchedMax &&
              tot[3] < kBatchedMax) {
            L = lg2(tot[3] * tot[2]) + lg2(tot[1] * tot[0]);  // the forward's fast path
          } else {
            float tl[kBlock];  // local-memory copy for the out-of-line rare path
#pragma unroll
            for (int c = 0; c < kBlock; ++c) tl[c] = s[c];
            L = row_lt_total_slow(tl, make_float4(tot[0], tot[1], tot[2], tot[3]),
                                  args.q + u.out_off + (int64_t)row * g.sl,
                                  args.k + u.out_off + (int64_t)kb * kBlock * g.sl, g.sl, D,
                                  g.scale_log2);
          }
          // M = (hi + L) + lo: two FADDs after L, exact where M is small (where e^M matters)
          Mk = (m_hi + L) + m_lo;
          if (live) two_sum_acc(m_hi, m_lo, L);
        }
        const float E = live ? ex2(Mk) : 0.0f;

        row_pass2(s, sg, E, tot);
        if (tr) SB_TR(args, w, gi, 2);
        mbar_wait(wfull, gi & 1);
        tc_fence_after();
        if (args.row_offset) load_dat<true>(s, tW, off);
        else load_dat<false>(s, tW, off);
        tc_fence_before();
        mbar_arrive(wempty);
        if (tr) SB_TR(args, w, gi, 3);
        uint32_t pk[32];
        if (!kStoreZ && live) Nrow[t] = bsum;  // b in effect for this tile (blocked.py:353)
        const float bnext = dz_row(s, sg, live ? bsum : 0.0f, pk);
        bsum = live ? bnext : bsum;
        if (tr) SB_TR(args, w, gi, 4);
        if (gi >= 1) mbar_wait(zempty, (gi - 1) & 1);
        if (tr) SB_TR(args, w, gi, 5);
        store_row_sw128(z_row, r, pk);
        fence_proxy_async_smem();
        mbar_arrive(zfull);
        if (tr) SB_TR(args, w, gi, 6);
        // this tile's M snapshot for phase 2 (blocked.py:188-189), written late so the
        // store never waits on the L -> M chain
        if (live) Mrow[t] = Mk;
      }
      if (kPingPongQ)
        for (int j = n_w; j < n_rounds; ++j) pp_round_pass();
      mbar_wait(done, nwi & 1);
      // store mode: the last tile's TMA store must have read the buffer too
      if (kStoreZ) mbar_wait(zempty, (ig + n_w - 1) & 1);
      if (tr) SB_TR(args, w, 0, 15);
      if (tr) SB_TR(args, w, nwi, 9);
      tc_fence_after();
      // dQ rows leave in 64-column halves through this warp's 4 KB slice of the
      // (now idle: `done`) dZ buffer as coalesced row segments
      const int row0 = qt * kTileM + quarter * 32;
      const int nvalid = max(0, min(32, u.L - row0));
      const uint32_t stage = smem_u32(smem + C::kOffZ + w * C::kZBytes) + quarter * 4096;
#pragma unroll 1
      for (int c = 0; c < D / 64; ++c) {
        float v[64];
        tmem_ld32(tQ + c * 64, v);
        tmem_ld32(tQ + c * 64 + 32, v + 32);
        tmem_wait_ld();
        if (c + 1 == D / 64) {
          tc_fence_before();
          mbar_arrive(dq_free);  // the next item's dQ may overwrite TMEM
        }
        warp_store_rows<8>(v, scale, stage, args.dq + u.out_off + (int64_t)row0 * g.sl + c * 64,
                           g.sl, nvalid);
      }
      if (tr) SB_TR(args, w, nwi, 10);
      ig += n_w;
      ++nwi;
    }
  }
  // ping-pong: WG0's last arrival on bar 2 still waits for WG1
  if (kPingPongQ && warp >= 4 && warp < 8) named_bar_sync(2, 256);
  tc_fence_before();
  __syncthreads();
  if (warp == 8) tmem_dealloc<C::kTmemCols>(tbase);
}

// ============================================================================
// Phase 2: dK and dV.  CTA = (b, h, key blocks 2p and 2p+1 = one 128-key pair);
// query tiles stream top to bottom.  Warpgroup w owns key block 2p+w for the
// stick math (thread r <-> query row r of the tile) and head-dim half w of the
// dK/dV epilogue (thread r <-> key r of the pair).  Every MMA spans BOTH key blocks (N = 128 keys): the
// tensor core's shared-memory operand traffic per FLOP is 2/3 of two N = 64 MMAs
// (measured: 128x64x16 SS-MMAs are smem-bound at 48 clk, 128x128x16 run at the
// full 64 clk), and one elected thread issues everything in a fixed order.
//   S   = Q  [K0;K1]^T    (M=128 rows, N=128 keys)       TMEM cols   0..127
//   dW  = dO [V0;V1]^T                                    TMEM cols 128..255
//   dV += [A0 A1]^T dO    (M=128 keys, N=D, K=128 rows)   cols 256..256+D
//   dK += [dZ0 dZ1]^T Q                                   cols 384..384+D
// dV/dK come out key-major (lane = key), so the epilogue writes whole key rows.
template <int D>
struct BwdKVCfg {
  static constexpr int kStages = D == 128 ? 2 : 3;
  static constexpr int kQBytes = kTileM * D * 2;
  static constexpr int kPairBytes = 2 * kBlock * D * 2;  // K (or V) of both key blocks
  static constexpr int kPBytes = kTileM * kBlock * 2;    // A / dZ of one warpgroup
  static constexpr int kOffK = 0;                        // chunk c: rows 0..127 = K0;K1
  static constexpr int kOffV = kOffK + kPairBytes;
  static constexpr int kOffQ = kOffV + kPairBytes;         // Q ring (kStages)
  static constexpr int kOffDO = kOffQ + kStages * kQBytes;  // dO: one buffer (free after dV)
  static constexpr int kOffA = kOffDO + kQBytes;            // A: WG0 then WG1 (contiguous)
  static constexpr int kOffZ = kOffA + 2 * kPBytes;         // dZ: WG0 then WG1
  static constexpr int kOffBar = kOffZ + 2 * kPBytes;
  static constexpr int kNumBars = 1 + 2 * kStages + 2 + 11 + 8;
  static constexpr int kOffMisc = kOffBar + kNumBars * 8;
  static constexpr int kSmem = kOffMisc + 64 + 1024;
  static_assert(kSmem <= 232448, "exceeds the 227 KB opt-in shared memory per block");
  static constexpr uint32_t kTmemCols = 512;
};

// a tile (qb, kb) is live when the forward visited it: first_kb[qb] <= kb <= qb
// (blocked.py:372-373)
__device__ __forceinline__ bool tile_live(const int* fkb, int nb, int qb, int kb) {
  return qb < nb && kb < nb && qb >= kb && fkb[qb] <= kb;
}

// Warp-cooperative iterator over the query tiles holding a live tile for key
// block kb0 or kb0+1: 32 tiles are tested at once (one per lane) and kept as a
// ballot mask, so the per-tile cost is a find-first-set.  `mine` holds, for the
// same window, whether tile (2 qt + half, kb) is live for the calling warp's own
// 64-row half and key block (stick warps), so no per-tile first_kb loads remain.
// Call convergently.
struct LiveQt {
  const int* fkb;
  int nb, n_qt, kb0, half, kb, base;
  uint32_t mask, mine;
  __device__ __forceinline__ void fill(int from) {
    base = from;
    const int qt = from + (int)(threadIdx.x & 31);
    const bool l = qt < n_qt && (tile_live(fkb, nb, 2 * qt, kb0) || tile_live(fkb, nb, 2 * qt + 1, kb0) ||
                                 tile_live(fkb, nb, 2 * qt, kb0 + 1) ||
                                 tile_live(fkb, nb, 2 * qt + 1, kb0 + 1));
    mask = __ballot_sync(0xffffffffu, l);
    mine = __ballot_sync(0xffffffffu, qt < n_qt && tile_live(fkb, nb, 2 * qt + half, kb));
  }
  __device__ __forceinline__ int next() {
    while (mask == 0) {
      if (base + 32 >= n_qt) return n_qt;
      fill(base + 32);
    }
    const int bit = __ffs(mask) - 1;
    mask &= mask - 1;
    return base + bit;
  }
  // liveness of the tile just returned by next() for this warp's half / key block
  __device__ __forceinline__ bool mine_live(int qt) const {
    return qt < n_qt && ((mine >> (qt - base)) & 1u);
  }
};

// Phase 2 work distribution: dynamic queue (SchedRing) or static "snake"
// striding (round k: CTA c takes item k*G + c, or k*G + G-1-c on odd rounds, so
// heavy-first rounds alternate direction: max/mean CTA load 1.05 vs 1.07).
constexpr bool kDynamicKV = false;  // recompute-mode phase 2: dynamic measured slower (1.44 vs 1.34 ms)
constexpr bool kDynamicKVS = true;  // store-mode phase 2: dynamic 0.85 vs static snake 0.95 ms
__device__ __forceinline__ int snake_item(int k) {
  return k * (int)gridDim.x + ((k & 1) ? (int)gridDim.x - 1 - (int)blockIdx.x : (int)blockIdx.x);
}

// Work item of phase 2: (unit, key pair p).  Every role derives the same item
// list, so they agree on which items carry work without communicating.
struct KVItem {
  Unit u;
  int b, h, kb0;
  bool valid;  // the key pair exists (varlen: shorter sequences have fewer)
};
__device__ __forceinline__ KVItem kv_item(const Geom& g, int idx) {
  KVItem it;
  int p, bh;
  grouped_order(idx, (g.nb + 1) / 2, g.B * g.H, g.ugroup, p, bh);
  it.b = bh / g.H;
  it.h = bh % g.H;
  it.u = make_unit(g, it.b, it.h);
  it.kb0 = 2 * p;
  it.valid = it.kb0 < it.u.nb;
  return it;
}

// Persistent: one CTA per SM takes items from a global work queue (LPT order
// within groups of 8 units, handed out dynamically).  The Q/dO ring and every per-tile
// barrier run on a CTA-wide tile counter across items, so the producer fetches
// the next item's K/V and first Q/dO tiles while the warpgroups finish the
// current item and write its dK/dV.  Per item: bar_kv (K/V landed), kv_free
// (last S/dW of the item read K/V), done (last dK^T issued), acc_free (the
// warpgroups read dV/dK out of TMEM).
template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1)
    sb_bwd_kv_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                     const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                     const BwdArgs args) {
  using C = BwdKVCfg<D>;
  constexpr int ST = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const Geom& g = args.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = ((g.nb + 1) / 2) * g.B * g.H;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* bar_kv = bars;
  uint64_t* bar_qfull = bars + 1;
  uint64_t* bar_qempty = bar_qfull + ST;
  uint64_t* bar_dofull = bar_qempty + ST;  // dO of the current tile landed
  uint64_t* bar_doempty = bar_dofull + 1;  // dV (its last reader) completed
  uint64_t* sfull = bar_doempty + 1;  // S = Q K^T landed in TMEM
  uint64_t* sempty = sfull + 1;       // S read by both warpgroups
  uint64_t* wfull = sfull + 2;        // dW = dO V^T landed
  uint64_t* wempty = sfull + 3;       // dW read
  uint64_t* afull = sfull + 4;        // A of both warpgroups in smem
  uint64_t* aused = sfull + 5;        // dV MMA read A
  uint64_t* zfull = sfull + 6;        // dZ in smem
  uint64_t* zused = sfull + 7;        // dK^T MMA read dZ
  uint64_t* done = sfull + 8;         // item's last dK^T complete
  uint64_t* kv_free = sfull + 9;      // item's last S / dW read K/V
  uint64_t* acc_free = sfull + 10;    // dV/dK read out of TMEM
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);
  const SchedRing sq{reinterpret_cast<int*>(smem + C::kOffMisc + 16), sfull + 11, sfull + 15};

  if (threadIdx.x == 0) {
    mbar_init(bar_kv, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(bar_qfull + s, 1);
      mbar_init(bar_qempty + s, 1);
    }
    mbar_init(bar_dofull, 1);
    mbar_init(bar_doempty, 1);
    mbar_init(sfull, 1);
    mbar_init(sempty, 256);
    mbar_init(wfull, 1);
    mbar_init(wempty, 256);
    mbar_init(afull, 256);
    mbar_init(aused, 1);
    mbar_init(zfull, 256);
    mbar_init(zused, 1);
    mbar_init(done, 1);
    mbar_init(kv_free, 1);
    mbar_init(acc_free, 256);
    sched_init(sq, 9);  // consumers: stick warps 0-7, issuer warp 9
    fence_mbar_init();
  }
  if (warp == 8) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t tS = tbase, tW = tbase + 128, tV = tbase + 256, tK = tbase + 384;

  if (warp >= 8) {
    reg_dealloc<kRegsLowKV>();
    if (warp == 8) {
      // ---------------------------------------------------------- TMA producer
      const bool leader = elect_one();
      if (leader) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_do);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
      }
      int jg = 0, ni = 0;  // tiles and work items so far
      for (int kq = 0;; ++kq) {
        const int idx = kDynamicKV ? sched_produce(sq, kq, args.sched + 1, n_items)
                                   : snake_item(kq);
        if (idx < 0 || idx >= n_items) break;
        const KVItem wi = kv_item(g, idx);
        if (!wi.valid) continue;
        const Unit& u = wi.u;
        LiveQt it{args.first_kb + u.fkb_off, u.nb, u.n_qt, wi.kb0, 0, wi.kb0, 0, 0u, 0u};
        it.fill(wi.kb0 / 2);
        int qt = it.next();
        if (qt >= u.n_qt) continue;  // nothing visited: the warpgroups write zeros
        if (ni >= 1) mbar_wait_warp(kv_free, (ni - 1) & 1);
        if (leader) {
          // both key blocks; rows past L (odd nb) are zero-filled by the TMA
          mbar_expect_tx(bar_kv, 2 * C::kPairBytes);
          for (int w = 0; w < 2; ++w)  // the K/V tensor maps have 64-row boxes
            for (int c = 0; c < D / 64; ++c) {
              const int off = c * (2 * kBlock * 128) + w * (kBlock * 128);
              tma_load_4d(&tm_k, bar_kv, smem + C::kOffK + off, c * 64,
                          u.trow0 + (wi.kb0 + w) * kBlock, wi.h, u.tb);
              tma_load_4d(&tm_v, bar_kv, smem + C::kOffV + off, c * 64,
                          u.trow0 + (wi.kb0 + w) * kBlock, wi.h, u.tb);
            }
        }
        __syncwarp();
        for (; qt < u.n_qt; qt = it.next(), ++jg) {
          const int s = jg % ST;
          if (jg >= ST) mbar_wait_warp(bar_qempty + s, ((jg / ST) - 1) & 1);
          SB_TR(args, 2, jg, 12);
          if (leader) {
            uint8_t* qdst = smem + C::kOffQ + s * C::kQBytes;
            mbar_expect_tx(bar_qfull + s, C::kQBytes);
            for (int c = 0; c < D / 64; ++c)
              tma_load_4d(&tm_q, bar_qfull + s, qdst + c * (kTileM * 128), c * 64,
                          u.trow0 + qt * kTileM, wi.h, u.tb);
          }
          __syncwarp();
          if (jg >= 1) mbar_wait_warp(bar_doempty, (jg - 1) & 1);  // dV(jg-1) read dO
          if (leader) {
            mbar_expect_tx(bar_dofull, C::kQBytes);
            for (int c = 0; c < D / 64; ++c)
              tma_load_4d(&tm_do, bar_dofull, smem + C::kOffDO + c * (kTileM * 128), c * 64,
                          u.trow0 + qt * kTileM, wi.h, u.tb);
          }
          __syncwarp();
        }
        ++ni;
      }
    } else if (warp == 9) {
      // ---------------------------------------------------------- MMA issuer
      // whole warp: uniform control flow and descriptors; one elected lane issues.
      constexpr uint32_t idesc_s = idesc_bf16(128, 128, 0, 0);  // Q K^T, dO V^T (N = 2 blocks)
      // dV = A^T dO, dK = dZ^T Q: M = 128 keys, N = D; A^T / dZ^T and dO / Q are read
      // straight from their row-major tiles as MN-major operands
      constexpr uint32_t idesc_t = idesc_bf16(128, D, 1, 1);
      const uint64_t dk = sdesc_sw128(smem_u32(smem + C::kOffK), 16, 1024);
      const uint64_t dv = sdesc_sw128(smem_u32(smem + C::kOffV), 16, 1024);
      const uint64_t dq = sdesc_sw128(smem_u32(smem + C::kOffQ), 16, 1024);
      const uint64_t dqmn = sdesc_sw128(smem_u32(smem + C::kOffQ), kTileM * 128, 1024);
      const uint64_t ddo = sdesc_sw128(smem_u32(smem + C::kOffDO), 16, 1024);
      const uint64_t ddomn = sdesc_sw128(smem_u32(smem + C::kOffDO), kTileM * 128, 1024);
      const uint64_t da = sdesc_sw128(smem_u32(smem + C::kOffA), C::kPBytes, 1024);
      const uint64_t dz = sdesc_sw128(smem_u32(smem + C::kOffZ), C::kPBytes, 1024);
      const bool leader = elect_one();
      // Fixed issue order matching the warpgroups' event order:
      // dV(j) [A(j) in smem], S(j+1) [S(j) read, Q(j+1) landed], dW(j+1)
      // [dW(j) read], dK(j) [dZ(j) in smem].
      auto issue_s = [&](int jg) {
        const uint32_t qo = (jg % ST) * C::kQBytes;
        mbar_wait_warp(bar_qfull + jg % ST, (jg / ST) & 1);
        SB_TR(args, 2, jg, 13);
        if (jg >= 1) mbar_wait_warp(sempty, (jg - 1) & 1);
        SB_TR(args, 2, jg, 8);
        tc_fence_after();
        if (leader) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off = (k >> 2) * (kTileM * 128) + (k & 3) * 32;
            const uint32_t offk = (k >> 2) * (2 * kBlock * 128) + (k & 3) * 32;
            umma_ss_at(tS, dq, qo + off, dk, offk, idesc_s, k > 0);
          }
          umma_commit(sfull);
        }
        __syncwarp();
      };
      auto issue_w = [&](int jg, bool last) {
        mbar_wait_warp(bar_dofull, jg & 1);
        if (jg >= 1) mbar_wait_warp(wempty, (jg - 1) & 1);
        SB_TR(args, 2, jg, 10);
        tc_fence_after();
        if (leader) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off = (k >> 2) * (kTileM * 128) + (k & 3) * 32;
            const uint32_t offk = (k >> 2) * (2 * kBlock * 128) + (k & 3) * 32;
            umma_ss_at(tW, ddo, off, dv, offk, idesc_s, k > 0);
          }
          umma_commit(wfull);
          if (last) umma_commit(kv_free);  // the item's K/V pair may be replaced
        }
        __syncwarp();
      };
      int jg = 0, ni = 0;
      for (int kq = 0;; ++kq) {
        const int idx = kDynamicKV ? sched_consume(sq, kq) : snake_item(kq);
        if (idx < 0 || idx >= n_items) break;
        const KVItem wi = kv_item(g, idx);
        if (!wi.valid) continue;
        const Unit& u = wi.u;
        LiveQt it{args.first_kb + u.fkb_off, u.nb, u.n_qt, wi.kb0, 0, wi.kb0, 0, 0u, 0u};
        it.fill(wi.kb0 / 2);
        int n = 0;
        for (int qt = it.next(); qt < u.n_qt; qt = it.next()) ++n;
        if (n == 0) continue;
        mbar_wait_warp(bar_kv, ni & 1);
        issue_s(jg);
        issue_w(jg, n == 1);
        // Fixed issue order: dV(j) [A(j) in smem], S(j+1) [S(j) read, Q(j+1)
        // landed], dK(j) [dZ(j) in smem], dW(j+1) [dW(j) read, dO(j+1) landed:
        // dO is single-buffered, reloaded once dV(j) has read it].
        for (int j = 0; j < n; ++j, ++jg) {
          const int s = jg % ST;
          const uint32_t qo = s * C::kQBytes;
          mbar_wait_warp(afull, jg & 1);
          // the previous item's dV/dK must be out of TMEM before overwriting
          if (j == 0 && ni >= 1) mbar_wait_warp(acc_free, (ni - 1) & 1);
          SB_TR(args, 2, jg, 9);
          tc_fence_after();
          if (leader) {
#pragma unroll
            for (int k = 0; k < kTileM / 16; ++k)  // dV += A^T dO  (K = query rows)
              umma_ss_at(tV, da, k * 2048, ddomn, k * 2048, idesc_t,
                      (j > 0 || k > 0) ? 1u : 0u);
            umma_commit(aused);
            umma_commit(bar_doempty);
          }
          __syncwarp();
          if (j + 1 < n) issue_s(jg + 1);
          mbar_wait_warp(zfull, jg & 1);
          SB_TR(args, 2, jg, 11);
          tc_fence_after();
          if (leader) {
#pragma unroll
            for (int k = 0; k < kTileM / 16; ++k)  // dK += dZ^T Q
              umma_ss_at(tK, dz, k * 2048, dqmn, qo + k * 2048, idesc_t,
                      (j > 0 || k > 0) ? 1u : 0u);
            umma_commit(zused);
            umma_commit(bar_qempty + s);
            if (j + 1 == n) umma_commit(done);
          }
          __syncwarp();
          if (j + 1 < n) issue_w(jg + 1, j + 2 == n);
        }
        ++ni;
      }
    }
  } else {
    reg_alloc<kRegsHighKV>();
    // ------------------------------------------------------------ stick warpgroups
    const int w = warp >> 2;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t tSw = tS + lane_base + w * 64, tWw = tW + lane_base + w * 64;
    const uint32_t a_row = smem_u32(smem + C::kOffA + w * C::kPBytes) + r * 128;
    const uint32_t z_row = smem_u32(smem + C::kOffZ + w * C::kPBytes) + r * 128;
    const float scale = g.scale_log2 * kLn2;
    const bool tr = quarter == 0 && lane == 0;
    int jg = 0, ni = 0;
    for (int kq = 0;; ++kq) {
      const int idx = kDynamicKV ? sched_consume(sq, kq) : snake_item(kq);
      if (idx < 0 || idx >= n_items) break;
      const KVItem wi = kv_item(g, idx);
      if (!wi.valid) continue;
      const Unit& u = wi.u;
      const int kb = wi.kb0 + w;
      // half = which 64-row half of the query tile this warp's rows are in
      LiveQt it{args.first_kb + u.fkb_off, u.nb, u.n_qt, wi.kb0, quarter >> 1, kb, 0, 0u, 0u};
      it.fill(wi.kb0 / 2);  // query tile kb0/2 holds the diagonal of key block kb0
      int qt = it.next();
      const bool any = qt < u.n_qt;
      const float* Mbase = args.M + u.m_off + (r & 63);
      const float* Nbase = args.N + u.m_off + (r & 63);
      // Per-tile operands: M (needed first) and the liveness of the next tile are
      // obtained half a tile ahead; N and the row offset at the top of their own
      // tile (consumed after the recompute).  Indices are clamped so every load is
      // in bounds whether or not the tile is live.
      auto tix = [&](int qt) -> int64_t {
        const int qb = min(2 * qt + (r >> 6), u.nb - 1);
        return tile_index(qb, min(kb, qb)) * kBlock;
      };
      auto is_live = [&](int qt) -> bool { return it.mine_live(qt) && qt * kTileM + r < u.L; };
      if (tr && ni == 0) SB_TR(args, w, 0, 14);
      if (tr && jg >= 1) SB_TR(args, w, jg - 1, 11);
      bool live = is_live(qt);
      float Ma = Mbase[tix(qt)];
      for (; qt < u.n_qt; ++jg) {
        const int my_qb = 2 * qt + (r >> 6);
        const float Nb = Nbase[tix(qt)];
        const float off =
            args.row_offset
                ? args.row_offset[u.rem_off + min(qt * kTileM + r, u.L - 1) * u.rem_stride]
                : 0.0f;
        const float E = live ? ex2(Ma) : 0.0f;  // dead rows/tiles: A = 0, dZ = 0
        if (tr) SB_TR(args, w, jg, 0);
        mbar_wait(sfull, jg & 1);
        tc_fence_after();
        float s[64], sg[64];
        tmem_ld32(tSw, s);
        tmem_ld32(tSw + 32, s + 32);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(sempty);  // S(j+1) may overwrite the buffer now
        if (tr) SB_TR(args, w, jg, 1);
        const bool diag = kb == my_qb;  // warp-uniform
        if (diag) recompute_row<true>(s, sg, g.scale_log2, E, r & 63);
        else recompute_row<false>(s, sg, g.scale_log2, E, kBlock);
        if (tr) SB_TR(args, w, jg, 2);
        const int qt_next = it.next();  // warp-collective
        const bool live_next = is_live(qt_next);
        const float Ma_next = Mbase[tix(qt_next)];
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) pk[c] = pack_bf16(s[2 * c], s[2 * c + 1]);
        if (jg >= 1) mbar_wait(aused, (jg - 1) & 1);  // dV of the previous tile read A
        if (tr) SB_TR(args, w, jg, 8);
        store_row_sw128(a_row, r, pk);
        fence_proxy_async_smem();
        mbar_arrive(afull);
        if (tr) SB_TR(args, w, jg, 3);
        mbar_wait(wfull, jg & 1);
        tc_fence_after();
        if (args.row_offset) load_dat<true>(s, tWw, off);  // warp-collective
        else load_dat<false>(s, tWw, off);
        tc_fence_before();
        mbar_arrive(wempty);
        if (tr) SB_TR(args, w, jg, 4);
        dz_row(s, sg, live ? Nb : 0.0f, pk);
        if (tr) SB_TR(args, w, jg, 5);
        if (jg >= 1) mbar_wait(zused, (jg - 1) & 1);  // dK of the previous tile read dZ
        if (tr) SB_TR(args, w, jg, 6);
        store_row_sw128(z_row, r, pk);
        fence_proxy_async_smem();
        mbar_arrive(zfull);
        if (tr) SB_TR(args, w, jg, 7);
        qt = qt_next;
        live = live_next;
        Ma = Ma_next;
      }

      // epilogue: dV / dK in TMEM (lane = key of the pair, columns = head dim).
      // Warp (w, quarter) owns keys 32*quarter .. +31 of the pair (lane = key) and
      // head-dim columns w*D/2 .. +D/2; rows leave through this warp's 4 KB slice
      // of the A buffers (free: every MMA of the item completed, `done`) as
      // coalesced row segments.
      if (any) {
        mbar_wait(done, ni & 1);
        tc_fence_after();
      }
      if (tr && jg >= 1) SB_TR(args, w, jg - 1, 9);
      {
        constexpr int HD = D / 2;
        const int key0 = wi.kb0 * kBlock + quarter * 32;
        const int nvalid = max(0, min(32, u.L - key0));
        // the warp's OWN 32 A rows (4 KB at w * kPBytes + quarter * 4 KB): the other
        // warpgroup may already be writing A rows of its next item (at D = 64 a
        // packed 2 KB-per-warp staging overlapped them: racecheck, many items per CTA)
        static_assert(32 * HD * 2 <= 32 * 128, "staging fits the warp's own A rows");
        const uint32_t stage = smem_u32(smem + C::kOffA) + (warp & 7) * (32 * 128);
#pragma unroll 1
        for (int t = 0; t < 2; ++t) {
          float a[HD];
          if (any) {
            const uint32_t tacc = (t ? tK : tV) + lane_base + w * HD;
#pragma unroll
            for (int c = 0; c < HD; c += 32) tmem_ld32(tacc + c, a + c);
            tmem_wait_ld();
          } else {
#pragma unroll
            for (int c = 0; c < HD; ++c) a[c] = 0.0f;
          }
          if (tr && jg >= 1) SB_TR(args, w, jg - 1, 12 + t);
          if (t == 1 && any) {
            tc_fence_before();
            mbar_arrive(acc_free);  // the next item's dV/dK may start
          }
          __nv_bfloat16* dst = (t ? args.dk : args.dv) + u.out_off + (int64_t)key0 * g.sl + w * HD;
          warp_store_rows<HD / 8>(a, t ? scale : 1.0f, stage, dst, g.sl, nvalid);
        }
      }
      if (tr && jg >= 1) SB_TR(args, w, jg - 1, 10);
      if (any) ++ni;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) tmem_dealloc<C::kTmemCols>(tbase);
}

// A only (store-mode phase 2), software-pipelined across the four 16-column
// groups, right to left: group g's ex2 pass (MUFU) is interleaved with group
// g+1's product pass (FMA pipe), so one warp keeps both pipes busy instead of
// running 64 ex2 back to back and then 128 multiplies.  Per element the
// arithmetic is exactly recompute_row<kDiag, false>'s fast path (same
// operations, same order: bit-identical A).  On exit pk[] holds A as bf16x2
// and s[] the masked t values; returns false if a group product reached 2^64
// (the caller redoes that row with the per-element path).
template <bool kDiag>
__device__ __forceinline__ bool recompute_a_pipe(float* s, uint32_t* pk, float scale_log2, float E,
                                                 int lim) {
#ifdef SB_NOMATH  // tuning ablation: pipeline without the stick math
#pragma unroll
  for (int c = 0; c < kBlock; c += 2) pk[c >> 1] = pack_bf16(s[c] * E, s[c + 1] * E);
  return true;
#endif
  // packed f32x2 multiplies on adjacent column pairs (FMUL2; the product chain
  // stays scalar): same operations per element, bit-identical
  const float2 sl2 = make_float2(scale_log2, scale_log2);
  float P[64];
  float tot = 1.0f;
#pragma unroll
  for (int i = 0; i < 16; i += 2) {  // prologue: pass 1 of group 3
    const int c = 48 + i;
    const float2 z = mul2(make_float2(s[c], s[c + 1]), sl2);
    float t0 = ex2(z.x), t1 = ex2(z.y);
    if (kDiag) {
      t0 = c < lim ? t0 : 0.0f;
      t1 = c + 1 < lim ? t1 : 0.0f;
    }
    s[c] = t0;
    s[c + 1] = t1;
    tot = fmaf(tot, t0, tot);
    P[c] = tot;
    tot = fmaf(tot, t1, tot);
    P[c + 1] = tot;
  }
  bool ok = tot < kBatchedMax;
  float Kn = E * rcp(tot);  // K of the group whose product pass runs next
  float Q = Kn;
#pragma unroll
  for (int g = 2; g >= 0; --g) {
    tot = 1.0f;
    const float2 K2 = make_float2(Kn, Kn);
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      const int c = 16 * g + i;  // pass 1, group g (two columns)
      const float2 z = mul2(make_float2(s[c], s[c + 1]), sl2);
      float t0 = ex2(z.x), t1 = ex2(z.y);
      if (kDiag) {
        t0 = c < lim ? t0 : 0.0f;
        t1 = c + 1 < lim ? t1 : 0.0f;
      }
      s[c] = t0;
      s[c + 1] = t1;
      tot = fmaf(tot, t0, tot);
      P[c] = tot;
      tot = fmaf(tot, t1, tot);
      P[c + 1] = tot;
      const int c2 = c + 16;  // pass 2, group g + 1 (two columns)
      const float2 t2 = make_float2(s[c2], s[c2 + 1]);
      const float2 u = i ? mul2(t2, make_float2(P[c2 - 1], P[c2])) : make_float2(t2.x, t2.y * P[c2]);
      const float2 a = mul2(u, K2);
      pk[c2 >> 1] = pack_bf16(a.x, a.y);
    }
    ok = ok && (tot < kBatchedMax);
    Kn = Q * rcp(tot);
    Q = Kn;
  }
  const float2 K2 = make_float2(Kn, Kn);
#pragma unroll
  for (int i = 0; i < 16; i += 2) {  // epilogue: pass 2 of group 0
    const float2 t2 = make_float2(s[i], s[i + 1]);
    const float2 u = i ? mul2(t2, make_float2(P[i - 1], P[i])) : make_float2(t2.x, t2.y * P[i]);
    const float2 a = mul2(u, K2);
    pk[i >> 1] = pack_bf16(a.x, a.y);
  }
  return ok;
}

// ============================================================================
// Phase 2, store mode: dZ tiles come from the workspace phase 1 wrote, so a
// key pair's tile needs only S = Q [K0;K1]^T and A (no dO V^T, no dZ math):
//   dV += [A0 A1]^T dO, dK += [dZ0 dZ1]^T Q  (dZ TMA-loaded).
// Tensor-pipe order per tile j: dK(j) (needs only loaded data), S(j+1)
// (double-buffered in TMEM, runs while the warpgroups compute A(j)), dV(j).
// Issuing dK first frees Q(j) and dZ(j) early, so Q and dZ rings of 2 stages
// have a whole tile of slack for their refills; dO (single) is refilled while
// dK(j+1) and S(j+2) run.  Three producer warps (K+Q, dZ, dO) refill each
// buffer the moment the MMA reading it completes, prefetching into L2 ahead.
// Producer look-ahead: walks the CTA's (item, query tile) sequence kPrefetch
// tiles ahead of the loads and prefetches those tiles into L2, so a buffer's
// refill (issued when the MMA reading it completes) hits L2 instead of HBM.
constexpr int kPrefetch = 4;
struct KVCursor {
  const Geom* g;
  const int* first_kb;
  int n_items, kq, qt;
  KVItem wi;
  LiveQt it;
  __device__ __forceinline__ bool open_next_item() {
    for (;;) {
      const int idx = snake_item(++kq);
      if (idx >= n_items) return false;
      wi = kv_item(*g, idx);
      if (!wi.valid) continue;
      it = LiveQt{first_kb + wi.u.fkb_off, wi.u.nb, wi.u.n_qt, wi.kb0, 0, wi.kb0, 0, 0u, 0u};
      it.fill(wi.kb0 / 2);
      qt = it.next();
      if (qt < wi.u.n_qt) return true;
    }
  }
  // next tile; false at the end of the CTA's work (warp-collective)
  __device__ __forceinline__ bool advance() {
    qt = it.next();
    return qt < wi.u.n_qt || open_next_item();
  }
};

template <int D>
struct BwdKVSCfg {
  // Q ring: 2 stages fill the 227 KB at d = 128; d = 64 has room for 4 (C4 phase 2
  // 2.071 -> 2.045 ms; 3 stages 2.058)
#ifndef SB_P2_QST64
#define SB_P2_QST64 4
#endif
  static constexpr int kStages = D == 64 ? SB_P2_QST64 : 2;
  static constexpr int kQBytes = kTileM * D * 2;
  static constexpr int kPairBytes = 2 * kBlock * D * 2;  // K of both key blocks
  static constexpr int kPBytes = kTileM * kBlock * 2;    // A / dZ of one key block
  static constexpr int kOffK = 0;
  static constexpr int kOffQ = kOffK + kPairBytes;
  static constexpr int kOffDO = kOffQ + kStages * kQBytes;  // single buffer (free after dV)
  static constexpr int kOffA = kOffDO + kQBytes;            // key block 0 then 1
  static constexpr int kOffZ = kOffA + 2 * kPBytes;         // dZ ring: 2 x (block 0, block 1)
  static constexpr int kOffBar = kOffZ + 2 * 2 * kPBytes;
  static constexpr int kNumBars = 1 + 2 * kStages + 2 + 4 + 9 + 8;  // + work-queue ring
  static constexpr int kOffMisc = kOffBar + kNumBars * 8;
  static constexpr int kSmem = kOffMisc + 64 + 1024;
  static_assert(kSmem <= 232448, "exceeds the 227 KB opt-in shared memory per block");
  static constexpr uint32_t kTmemCols = 512;
};

template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1)
    sb_bwd_kvs_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                      const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_z,
                      const BwdArgs args) {
  using C = BwdKVSCfg<D>;
  constexpr int ST = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const Geom& g = args.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = ((g.nb + 1) / 2) * g.B * g.H;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* bar_kv = bars;
  uint64_t* bar_qfull = bars + 1;
  uint64_t* bar_qempty = bar_qfull + ST;
  uint64_t* bar_dofull = bar_qempty + ST;
  uint64_t* bar_doempty = bar_dofull + 1;
  uint64_t* bar_zfull = bar_doempty + 1;  // [2] dZ pair landed
  uint64_t* bar_zempty = bar_zfull + 2;   // [2] dK read it
  uint64_t* sfull = bar_zempty + 2;  // [2] S double-buffered in TMEM (cols 0 / 128)
  uint64_t* sempty = sfull + 2;      // [2]
  uint64_t* afull = sfull + 4;
  uint64_t* aused = sfull + 5;
  uint64_t* done = sfull + 6;
  uint64_t* kv_free = sfull + 7;
  uint64_t* acc_free = sfull + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffMisc);
  // dynamic work queue (kDynamicKVS): warp 8 takes items from a global counter (the
  // N header's second word) and hands them to every other role through this ring
  const SchedRing sq{reinterpret_cast<int*>(smem + C::kOffMisc + 16), acc_free + 1, acc_free + 5};
  auto next_item = [&](int kq) -> int {
    if (!kDynamicKVS) {
      const int idx = snake_item(kq);
      return idx < n_items ? idx : -1;
    }
    return warp == 8 ? sched_produce(sq, kq, args.sched + 1, n_items) : sched_consume(sq, kq);
  };

  if (threadIdx.x == 0) {
    if (kDynamicKVS) sched_init(sq, 11);  // consumers: sticks 0-7, warps 9, 10, 11
    mbar_init(bar_kv, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(bar_qfull + s, 1);
      mbar_init(bar_qempty + s, 1);
    }
    mbar_init(bar_dofull, 1);
    mbar_init(bar_doempty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar_zfull + s, 1);
      mbar_init(bar_zempty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(sfull + s, 1);
      mbar_init(sempty + s, 256);
    }
    mbar_init(afull, 256);
    mbar_init(aused, 1);
    mbar_init(done, 1);
    mbar_init(kv_free, 1);
    mbar_init(acc_free, 256);
    fence_mbar_init();
  }
  if (warp == 8) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t tS = tbase, tV = tbase + 256, tK = tbase + 384;

  if (warp >= 8) {
    reg_dealloc<kRegsLowKV>();
    if (warp == 8 || warp >= 10) {
      // ---------------------------------------------------------- TMA producers
      // warp 8: K pair + Q ring; warp 10: dZ pair; warp 11: dO
      const bool leader = elect_one();
      if (leader) {
        if (warp == 8) {
          tma_prefetch(&tm_q);
          tma_prefetch(&tm_k);
        } else {
          tma_prefetch(warp == 10 ? &tm_z : &tm_do);
        }
      }
      // L2 look-ahead (see KVCursor): this warp's stream only
      KVCursor ahead{&g, args.first_kb, n_items, -1, 0};
      bool more = !kDynamicKVS && ahead.open_next_item();  // look-ahead needs a static order
      auto prefetch_one = [&]() {
        if (!more) return;
        if (leader) {
          const Unit& v = ahead.wi.u;
          if (warp == 10) {
            for (int w = 0; w < 2; ++w)
              tma_prefetch_3d(&tm_z, 0, 0, (int)(v.z_off + ztile(ahead.qt, ahead.wi.kb0 + w)));
          } else {
            for (int c = 0; c < D / 64; ++c)
              tma_prefetch_4d(warp == 8 ? &tm_q : &tm_do, c * 64, v.trow0 + ahead.qt * kTileM,
                              ahead.wi.h, v.tb);
          }
        }
        __syncwarp();
        more = ahead.advance();
      };
      for (int i = 0; i < kPrefetch; ++i) prefetch_one();
      int jg = 0, ni = 0;
      for (int kq = 0;; ++kq) {
        const int idx = next_item(kq);
        if (idx < 0) break;
        const KVItem wi = kv_item(g, idx);
        if (!wi.valid) continue;
        const Unit& u = wi.u;
        LiveQt it{args.first_kb + u.fkb_off, u.nb, u.n_qt, wi.kb0, 0, wi.kb0, 0, 0u, 0u};
        it.fill(wi.kb0 / 2);
        int qt = it.next();
        if (qt >= u.n_qt) continue;  // nothing visited: the warpgroups write zeros
        if (warp == 8) {
          if (ni >= 1) mbar_wait_warp(kv_free, (ni - 1) & 1);
          if (leader) {
            mbar_expect_tx(bar_kv, C::kPairBytes);
            for (int w = 0; w < 2; ++w)  // the K tensor map has 64-row boxes
              for (int c = 0; c < D / 64; ++c)
                tma_load_4d(&tm_k, bar_kv,
                            smem + C::kOffK + c * (2 * kBlock * 128) + w * (kBlock * 128), c * 64,
                            u.trow0 + (wi.kb0 + w) * kBlock, wi.h, u.tb);
          }
          __syncwarp();
        }
        for (; qt < u.n_qt; qt = it.next(), ++jg) {
          prefetch_one();
          if (warp == 8) {
            const int s = jg % ST;
            if (jg >= ST) mbar_wait_warp(bar_qempty + s, ((jg / ST) - 1) & 1);
            SB_TR(args, 3, jg, 0);
            if (leader) {
              mbar_expect_tx(bar_qfull + s, C::kQBytes);
              for (int c = 0; c < D / 64; ++c)
                tma_load_4d(&tm_q, bar_qfull + s,
                            smem + C::kOffQ + s * C::kQBytes + c * (kTileM * 128), c * 64,
                            u.trow0 + qt * kTileM, wi.h, u.tb);
            }
          } else if (warp == 10) {
            const int z = jg & 1;
            if (jg >= 2) mbar_wait_warp(bar_zempty + z, ((jg >> 1) - 1) & 1);  // dK(jg-2) read dZ
            SB_TR(args, 3, jg, 2);
            if (leader) {
#ifdef SB_NOZ  // tuning ablation: no dZ traffic (dK reads whatever is in the buffer)
              mbar_arrive(bar_zfull + z);
#else
              mbar_expect_tx(bar_zfull + z, 2 * kZTileBytes);
              for (int w = 0; w < 2; ++w)
                tma_load_3d(&tm_z, bar_zfull + z, smem + C::kOffZ + (2 * z + w) * C::kPBytes, 0, 0,
                            (int)(u.z_off + ztile(qt, wi.kb0 + w)));
#endif
            }
          } else {
            if (jg >= 1) mbar_wait_warp(bar_doempty, (jg - 1) & 1);  // dV(jg-1) read dO
            SB_TR(args, 3, jg, 4);
            if (leader) {
              mbar_expect_tx(bar_dofull, C::kQBytes);
              for (int c = 0; c < D / 64; ++c)
                tma_load_4d(&tm_do, bar_dofull, smem + C::kOffDO + c * (kTileM * 128), c * 64,
                            u.trow0 + qt * kTileM, wi.h, u.tb);
            }
          }
          __syncwarp();
        }
        ++ni;
      }
    } else if (warp == 9) {
      // ---------------------------------------------------------- MMA issuer
      constexpr uint32_t idesc_s = idesc_bf16(128, 128, 0, 0);  // Q K^T (N = 2 blocks)
      constexpr uint32_t idesc_t = idesc_bf16(128, D, 1, 1);    // A^T dO, dZ^T Q: MN-major
      const uint64_t dk = sdesc_sw128(smem_u32(smem + C::kOffK), 16, 1024);
      const uint64_t dq = sdesc_sw128(smem_u32(smem + C::kOffQ), 16, 1024);
      const uint64_t dqmn = sdesc_sw128(smem_u32(smem + C::kOffQ), kTileM * 128, 1024);
      const uint64_t ddomn = sdesc_sw128(smem_u32(smem + C::kOffDO), kTileM * 128, 1024);
      const uint64_t da = sdesc_sw128(smem_u32(smem + C::kOffA), C::kPBytes, 1024);
      const uint64_t dz = sdesc_sw128(smem_u32(smem + C::kOffZ), C::kPBytes, 1024);
      const bool leader = elect_one();
      auto issue_s = [&](int jg, bool last) {
        const uint32_t qo = (jg % ST) * C::kQBytes;
        const int b = jg & 1;
        SB_TR(args, 2, jg, 0);
        mbar_wait_warp(bar_qfull + jg % ST, (jg / ST) & 1);
        SB_TR(args, 2, jg, 1);
        if (jg >= 2) mbar_wait_warp(sempty + b, ((jg >> 1) - 1) & 1);
        SB_TR(args, 2, jg, 2);
        tc_fence_after();
        if (leader) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off = (k >> 2) * (kTileM * 128) + (k & 3) * 32;
            const uint32_t offk = (k >> 2) * (2 * kBlock * 128) + (k & 3) * 32;
            umma_ss_at(tS + b * 128, dq, qo + off, dk, offk, idesc_s, k > 0);
          }
          umma_commit(sfull + b);
          if (last) umma_commit(kv_free);  // the item's K pair may be replaced
        }
        __syncwarp();
      };
      int jg = 0, ni = 0;
      for (int kq = 0;; ++kq) {
        const int idx = next_item(kq);
        if (idx < 0) break;
        const KVItem wi = kv_item(g, idx);
        if (!wi.valid) continue;
        const Unit& u = wi.u;
        LiveQt it{args.first_kb + u.fkb_off, u.nb, u.n_qt, wi.kb0, 0, wi.kb0, 0, 0u, 0u};
        it.fill(wi.kb0 / 2);
        int n = 0;
        for (int qt = it.next(); qt < u.n_qt; qt = it.next()) ++n;
        if (n == 0) continue;
        mbar_wait_warp(bar_kv, ni & 1);
        issue_s(jg, n == 1);
        for (int j = 0; j < n; ++j, ++jg) {
          const int s = jg % ST, z = jg & 1;
          mbar_wait_warp(bar_zfull + z, (jg >> 1) & 1);
          SB_TR(args, 2, jg, 7);
          if (j == 0 && ni >= 1) mbar_wait_warp(acc_free, (ni - 1) & 1);  // epilogue read dK/dV
          tc_fence_after();
          if (leader) {
#pragma unroll
            for (int k = 0; k < kTileM / 16; ++k)  // dK += dZ^T Q
              umma_ss_at(tK, dz, 2 * z * C::kPBytes + k * 2048, dqmn, s * C::kQBytes + k * 2048,
                         idesc_t, (j > 0 || k > 0) ? 1u : 0u);
            umma_commit(bar_zempty + z);
            umma_commit(bar_qempty + s);  // S(j) and dK(j) read Q(j)
          }
          __syncwarp();
          // S(j+1) into the other TMEM buffer: it runs while the warpgroups
          // compute A(j)
          if (j + 1 < n) issue_s(jg + 1, j + 2 == n);
          mbar_wait_warp(afull, jg & 1);
          SB_TR(args, 2, jg, 4);
          mbar_wait_warp(bar_dofull, jg & 1);
          SB_TR(args, 2, jg, 5);
          tc_fence_after();
          if (leader) {
#pragma unroll
            for (int k = 0; k < kTileM / 16; ++k)  // dV += A^T dO  (K = query rows)
              umma_ss_at(tV, da, k * 2048, ddomn, k * 2048, idesc_t, (j > 0 || k > 0) ? 1u : 0u);
            umma_commit(aused);
            umma_commit(bar_doempty);
            if (j + 1 == n) umma_commit(done);
          }
          __syncwarp();
        }
        ++ni;
      }
    }
  } else {
    reg_alloc<kRegsHighKV>();
    // ------------------------------------------------------------ stick warpgroups
    // warpgroup w: A of key block kb0 + w for the tile's 128 query rows
    const int w = warp >> 2;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t tSw0 = tS + lane_base + w * 64;
    const uint32_t a_row = smem_u32(smem + C::kOffA + w * C::kPBytes) + r * 128;
    const float scale = g.scale_log2 * kLn2;
    const bool tr = quarter == 0 && lane == 0;
    if (tr) SB_TR(args, w, 0, 14);
    int jg = 0, ni = 0;
    for (int kq = 0;; ++kq) {
      const int idx = next_item(kq);
      if (idx < 0) break;
      const KVItem wi = kv_item(g, idx);
      if (!wi.valid) continue;
      const Unit& u = wi.u;
      const int kb = wi.kb0 + w;
      LiveQt it{args.first_kb + u.fkb_off, u.nb, u.n_qt, wi.kb0, quarter >> 1, kb, 0, 0u, 0u};
      it.fill(wi.kb0 / 2);
      int qt = it.next();
      const bool any = qt < u.n_qt;
      const float* Mbase = args.M + u.m_off + (r & 63);
      auto tix = [&](int qt) -> int64_t {
        const int qb = min(2 * qt + (r >> 6), u.nb - 1);
        return tile_index(qb, min(kb, qb)) * kBlock;
      };
      auto is_live = [&](int qt) -> bool { return it.mine_live(qt) && qt * kTileM + r < u.L; };
      bool live = is_live(qt);
      // M snapshots: prefetched into L1 two tiles ahead, loaded one tile ahead (a global
      // load's latency under this kernel's traffic exceeds one tile)
      float Ma = Mbase[tix(qt)];
      {  // L1 prefetch of the next tile's M; its load, one tile later, then hits L1
        LiveQt peek = it;
        prefetch_l1(Mbase + tix(peek.next()));
      }
      if (tr) SB_TR(args, w, ni, 12);
      for (; qt < u.n_qt; ++jg) {
        const int my_qb = 2 * qt + (r >> 6);
        const uint32_t tSw = tSw0 + (jg & 1) * 128;
        if (tr) SB_TR(args, w, jg, 0);
        mbar_wait(sfull + (jg & 1), (jg >> 1) & 1);
        if (tr) SB_TR(args, w, jg, 1);
        tc_fence_after();
        const float E = live ? ex2(Ma) : 0.0f;  // dead rows/tiles: A = 0 (M load hidden by the wait)
        float sv[64];
        tmem_ld32(tSw, sv);
        tmem_ld32(tSw + 32, sv + 32);
        tmem_wait_ld();
        const bool diag = kb == my_qb;  // warp-uniform
        // the recompute-mode kernel's A arithmetic exactly (bit-identical results)
        uint32_t pk[32];
        const bool ok = diag ? recompute_a_pipe<true>(sv, pk, g.scale_log2, E, r & 63)
                             : recompute_a_pipe<false>(sv, pk, g.scale_log2, E, kBlock);
        if (__any_sync(0xffffffffu, !ok)) {
          // outside the 2^64 range: recompute_row (wider-range retry, else one rcp
          // per element) on S reloaded for those rows, as the recompute-mode kernel
          tmem_ld32(tSw, sv);
          tmem_ld32(tSw + 32, sv + 32);
          tmem_wait_ld();
          if (!ok) {
            float sg[64];
            if (diag) recompute_row<true, false>(sv, sg, g.scale_log2, E, r & 63);
            else recompute_row<false, false>(sv, sg, g.scale_log2, E, kBlock);
#pragma unroll
            for (int i = 0; i < 32; ++i) pk[i] = pack_bf16(sv[2 * i], sv[2 * i + 1]);
          }
        }
        tc_fence_before();
        if (tr) SB_TR(args, w, jg, 2);
        mbar_arrive(sempty + (jg & 1));  // S(j+2) may overwrite the buffer now
        const int qt_next = it.next();  // warp-collective
        const bool live_next = is_live(qt_next);
        // (a register loaded two tiles ahead and rotated stalled on its MOV every tile:
        // the compiler materialises the rotation right after the load; 0.848 -> 0.828 ms)
        const float Ma_next = Mbase[tix(qt_next)];
        {
          LiveQt peek = it;
          prefetch_l1(Mbase + tix(peek.next()));
        }
        if (jg >= 1) mbar_wait(aused, (jg - 1) & 1);  // dV of the previous tile read A
        if (tr) SB_TR(args, w, jg, 3);
        store_row_sw128(a_row, r, pk);
        fence_proxy_async_smem();
        mbar_arrive(afull);
        if (tr) SB_TR(args, w, jg, 4);
        qt = qt_next;
        live = live_next;
        Ma = Ma_next;
      }

      // epilogue (as the recompute-mode kernel): lane = key, warp (w, quarter)
      // owns keys 32*quarter.. and head-dim columns w*D/2..; rows leave through
      // this warp's slice of the A buffers (free: `done`)
      if (any) {
        mbar_wait(done, ni & 1);
        if (tr && ni == 0) SB_TR(args, w, 0, 15);
        if (tr) SB_TR(args, w, ni, 9);
        tc_fence_after();
      }
      {
        constexpr int HD = D / 2;
        const int key0 = wi.kb0 * kBlock + quarter * 32;
        const int nvalid = max(0, min(32, u.L - key0));
        // the warp's OWN 32 A rows (4 KB at w * kPBytes + quarter * 4 KB): the other
        // warpgroup may already be writing A rows of its next item (at D = 64 a
        // packed 2 KB-per-warp staging overlapped them: racecheck, many items per CTA)
        static_assert(32 * HD * 2 <= 32 * 128, "staging fits the warp's own A rows");
        const uint32_t stage = smem_u32(smem + C::kOffA) + (warp & 7) * (32 * 128);
#pragma unroll 1
        for (int t = 0; t < 2; ++t) {
          float a[HD];
          if (any) {
            const uint32_t tacc = (t ? tK : tV) + lane_base + w * HD;
#pragma unroll
            for (int c = 0; c < HD; c += 32) tmem_ld32(tacc + c, a + c);
            tmem_wait_ld();
          } else {
#pragma unroll
            for (int c = 0; c < HD; ++c) a[c] = 0.0f;
          }
          if (tr && t == 0) SB_TR(args, w, ni, 13);
          if (t == 1 && any) {
            tc_fence_before();
            mbar_arrive(acc_free);  // the next item's dV/dK may start
          }
          __nv_bfloat16* dst = (t ? args.dk : args.dv) + u.out_off + (int64_t)key0 * g.sl + w * HD;
          warp_store_rows<HD / 8>(a, t ? scale : 1.0f, stage, dst, g.sl, nvalid);
          if (tr) SB_TR(args, w, ni, 10 + t);
        }
      }
      if (any) ++ni;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) tmem_dealloc<C::kTmemCols>(tbase);
}

template <int D>
static int launch_bwd(const CUtensorMap& tq, const CUtensorMap& tdo, const CUtensorMap& tk,
                      const CUtensorMap& tv, const CUtensorMap& tz, const BwdArgs& a, int phases,
                      bool store, cudaStream_t stream) {
  const unsigned BH = (unsigned)(a.g.B * a.g.H);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (phases & 1) {
    using C = BwdQCfg<D>;
    auto kern = store ? sb_bwd_q_kernel<D, true> : sb_bwd_q_kernel<D, false>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return (int)e;
    if ((e = cudaMemsetAsync(a.sched, 0, sizeof(unsigned), stream)) != cudaSuccess) return (int)e;
    // persistent: one CTA per SM (fewer if there are fewer work items)
    const unsigned items = (unsigned)((a.g.n_qt + 1) / 2) * BH;
    kern<<<items < (unsigned)sms ? items : (unsigned)sms, kBwdThreads, C::kSmem, stream>>>(
        tq, tdo, tk, tv, tz, a);
    if ((e = cudaGetLastError()) != cudaSuccess) return (int)e;
  }
  if (phases & 2) {
    const unsigned items = (unsigned)((a.g.nb + 1) / 2) * BH;
    const unsigned grid = items < (unsigned)sms ? items : (unsigned)sms;
    cudaError_t e;
    if (store) {
      using C = BwdKVSCfg<D>;
      auto kern = sb_bwd_kvs_kernel<D>;
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
      if (e != cudaSuccess) return (int)e;
      if (kDynamicKVS && (e = cudaMemsetAsync(a.sched + 1, 0, sizeof(unsigned), stream)) != cudaSuccess)
        return (int)e;
      kern<<<grid, kBwdThreads, C::kSmem, stream>>>(tq, tdo, tk, tz, a);
    } else {
      using C = BwdKVCfg<D>;
      auto kern = sb_bwd_kv_kernel<D>;
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
      if (e != cudaSuccess) return (int)e;
      if ((e = cudaMemsetAsync(a.sched + 1, 0, sizeof(unsigned), stream)) != cudaSuccess)
        return (int)e;
      kern<<<grid, kBwdThreads, C::kSmem, stream>>>(tq, tdo, tk, tv, a);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return (int)e;
  }
  return 0;
}

int bwd_dispatch(int D, const CUtensorMap& tq, const CUtensorMap& tdo, const CUtensorMap& tk,
                 const CUtensorMap& tv, const CUtensorMap& tz, const BwdArgs& a, int phases,
                 bool store, cudaStream_t stream) {
  if (D == 128) return launch_bwd<128>(tq, tdo, tk, tv, tz, a, phases, store, stream);
  if (D == 64) return launch_bwd<64>(tq, tdo, tk, tv, tz, a, phases, store, stream);
  return -1;
}

}  // namespace sb

#ifdef SB_WATCHDOG_PRINT
extern "C" int sb_debug_set_wd_bwd(void* p) {
  return (int)cudaMemcpyToSymbol(sb::g_sb_wd, &p, sizeof(p));
}
#endif
