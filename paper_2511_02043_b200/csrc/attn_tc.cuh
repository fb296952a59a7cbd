// attn_tc.cu -- bf16 fused attention forward on the 5th-generation tensor cores
// (sm_100a): TMA -> mbarrier ring -> tcgen05.mma (accumulators in TMEM) ->
// tcgen05.ld -> online softmax in registers -> P back into TMEM -> tcgen05.mma.
//
// This is the single monolithic kernel Flashlight's compiler emits per
// attention program: "each thread block computes tiles of the
// dot-product S = QK^T/sqrt(d), applies the online softmax to each tile via a
// fused max-reduction and rescaled accumulation, and multiplies the resulting
// softmax output with the corresponding tiles of V".  Re-designed for B200:
//
//  * CTA = 384 threads, one CTA per SM (TMEM: all 512 columns).
//      warps 0-3  softmax WG0: query tile 0 (thread = row = TMEM lane)
//      warps 4-7  softmax WG1: query tile 1 (differential attention: map 1)
//      warp  8    TMA producer (one elected lane)
//      warp  9    MMA issuer (one elected lane) + TMEM allocator
//  * TMEM columns: S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [256+D,256+2D);
//    P_i (bf16, 64 columns) aliases the upper half of S_i (the
//    whole D_v lives in one accumulator -- "tiling-aware dimension elimination").
//  * MMA issue order S0(0) S1(0) | PV0(j) S0(j+1) PV1(j) S1(j+1) | ... so the two
//    softmax warpgroups ping-pong against the tensor pipe; tcgen05 ops issued by
//    one thread execute in order, so S_i(j+1) may overwrite P_i(j) after PV_i(j).
//  * Online softmax (Alg.2, semantic fusion P:L685-697) in the log2
//    domain with CONDITIONAL rescaling: the running reference m_ref only moves
//    when the row max grows by more than TAU = 8 (p <= 2^8 stays exact in fp32
//    and representable in bf16).  Licensed by the closed form of do[j]
//     whose proof never uses m[j] = max.
//  * Masks are per-row key intervals (masks.cuh): KV tiles outside the union
//    are never loaded, tiles inside every row's interval run mask-free, only
//    boundary tiles pay two compares per element.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "masks.cuh"
#include "params.h"
#include "ptx.cuh"

namespace fl {

#ifdef FL_TIMING
// Diagnostic build only (-DFL_TIMING): cycle counters of thread 0 of each softmax
// warpgroup and of the MMA issuer, summed over CTAs; read with fl_debug_timing().
static __device__ unsigned long long g_fl_timing[3][16];   // per translation unit
#define FL_T(slot)                                    \
  do {                                                \
    const long long t_now_ = clock64();               \
    t_acc[slot] += t_now_ - t_prev;                   \
    t_prev = t_now_;                                  \
  } while (0)
#else
#define FL_T(slot) \
  do {             \
  } while (0)
#endif

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
#ifndef FL_TAU
#define FL_TAU 8.0f
#endif
constexpr float kTau = FL_TAU;
constexpr int kThreadsTc = 384;
// Register split via setmaxnreg: the CTA launches with 168 regs/thread (launch
// bounds 384 x 1); the control warpgroup gives registers back and the two softmax
// warpgroups take them.  inc blocks until the CTA's pool can pay, so the split
// must fit in what the CTA owns or the second softmax WG deadlocks.
// Measured (profiles/r01b_ab_knobs.txt): differential attention and ALiBi gain from 216 softmax registers
// (diff 699 -> 727, ALiBi 1022 -> 1040 TF/s), softcap / sliding / document lose 2-4 % and the small
// heads 6 %, plain causal is neutral -> 216 only for DIFF and ALiBi.
#ifndef FL_REGS_CTL
#define FL_REGS_CTL(W) ((W) ? 72 : 88)
#define FL_REGS_SOFTMAX(W) ((W) ? 216 : 208)
#endif
constexpr uint32_t kRegsLaunch = 168;
template <bool WIDE>
struct RegCfg {
  static constexpr uint32_t CTL = FL_REGS_CTL(WIDE), SOFTMAX = FL_REGS_SOFTMAX(WIDE);
  static_assert(2 * 128 * SOFTMAX + 128 * CTL <= kThreadsTc * kRegsLaunch, "setmaxnreg split exceeds CTA pool");
};
// FL_MASK_BLOCKLIST: at most this many listed KV blocks per query block on the bf16 path.
constexpr int kMaxSelTc = 256;

// LIST (RSA block lists): both warpgroups work on the SAME 128-row query block and split its
// listed KV blocks (WG0 entries 0, 2, 4, ..., WG1 entries 1, 3, 5, ...), each with its own
// (m, l, O) partial; WG0 merges the two partials in the epilogue (the online-softmax closed
// form, applied across the two halves of the list).  One Q tile, and step j of the
// schedule carries two different KV tiles, so the ring holds 4 entries per step.
// BIG: small heads (D = 32) without staged bias tiles (no bias, or the pair bias resident in TMEM) spend
// the shared memory the bias tiles would take on a second Q buffer (the next unit's Q loads while this
// unit's S MMAs still read the current one) and a 16-entry K/V ring (more than one unit of look-ahead).
template <int D, bool DIFF, bool LIST = false, bool BIG = false>
struct TcCfg {
  static constexpr int BM = 128;                     // query rows per tile (= TMEM lanes)
  static constexpr int BN = 128;                     // keys per KV tile
  static constexpr int CH = D >= 64 ? 64 : 32;       // elements per swizzle row
  static constexpr int SWB = CH * 2;                 // swizzle bytes: 128 or 64
  static constexpr int NCH = D / CH;                 // swizzle chunks per row
  static constexpr int CHUNK_BYTES = BM * SWB;
  static constexpr int TILE_BYTES = BM * D * 2;
  static constexpr int NQ = LIST ? 1 : 2;            // Q tiles resident per unit
#ifndef FL_NSLOT64
#define FL_NSLOT64 6
#endif
#ifndef FL_BIG_NSLOT
#define FL_BIG_NSLOT 8
#endif
  static constexpr int NSLOT = LIST ? (D == 128 ? 5 : 8) : (D == 128 ? 4 : (D == 64 ? FL_NSLOT64 : (BIG ? FL_BIG_NSLOT : 8)));
  static constexpr int NQBUF = BIG ? 2 : 1;          // Q buffers (units it, it + 1)
  static constexpr uint32_t LAYOUT = SWB == 128 ? kLayoutSW128 : kLayoutSW64;
  static constexpr int SBO = 8 * SWB;                // 8-row (K-major) / 8-key (MN-major) group stride
  static constexpr uint32_t COL_S0 = 0, COL_S1 = 128, COL_O0 = 256, COL_O1 = 256 + D;
  static constexpr uint32_t P_OFF = 64;              // P_i at S_i + 64
  static constexpr int SMEM_Q = 0;
  static constexpr int SMEM_RING = NQBUF * NQ * TILE_BYTES;
  // Small heads (D = 32, Evoformer) have shared memory to spare: the additive (pair) bias tiles come
  // through TMA into a per-warpgroup double buffer (2 slabs of 128 rows x 64 keys, 128-B swizzle).
  static constexpr bool BIAS_TMA_OK = D == 32;
  static constexpr int BIAS_TILE = 128 * 128 * 2;
  static constexpr int SMEM_BIAS = SMEM_RING + NSLOT * TILE_BYTES;
  static constexpr bool BIAS_AREA = BIAS_TMA_OK && !BIG;   // bias tiles, else (unused) the small-head gate rows
  static constexpr int SMEM_BAR = SMEM_BIAS + (BIAS_AREA ? 4 * BIAS_TILE : 0);
  // q_full[NQBUF] q_empty[NQBUF] | full[NSLOT] empty[NSLOT] | s_full[2] p_full[2] o_full[2] | unit_full[2] unit_empty[2]
  // | bias_full[4] bias_empty[4]
  static constexpr int NBAR = 2 * NQBUF + 2 * NSLOT + 6 + 4 + 8;
  static constexpr int SMEM_SCHED = SMEM_BAR + NBAR * 8 + 16;       // blocklist schedule (RSA), 2 slots
  static constexpr int SCHED_WORDS = 2 * kMaxSelTc + 24;  // schedule, count, the decoded Work (WORK_OFF), unit id
  static constexpr int WORK_OFF = 2 * kMaxSelTc + 4;
  static constexpr int KBITS_WORDS = 64;             // small heads: key-mask bits (S_k <= 2048) in the unit slot
  static constexpr int SMEM_ML = SMEM_SCHED + 2 * SCHED_WORDS * 4;      // LIST: WG1's (m, l) per row
  // ALiBi on the tensor core (kAlibiMma): the constant A tile of ones and two per-unit B tiles of slope*c
  // (K = 16, 32-B rows, SW32 atoms), 1024-B aligned
  static constexpr int SMEM_AUG = (SMEM_ML + (LIST ? 2 * 128 * 4 : 0) + 1023) / 1024 * 1024;
  static constexpr int AUG_TILE = 128 * 32;
  static constexpr int SMEM_TOTAL = SMEM_ML + (LIST ? 2 * 128 * 4 : 0) + 1024;  // + alignment slack
  static constexpr int SMEM_TOTAL_AUG = SMEM_AUG + 3 * AUG_TILE + 1024;
  static constexpr uint32_t IDESC_S = idesc_bf16_f32(128, BN, 0);   // Q (K-major) x K (K-major)
  static constexpr uint32_t IDESC_O = idesc_bf16_f32(128, D, 1);    // P (TMEM) x V (MN-major)
  // Small heads with a TMA'd pair bias: the tensor core adds it, S += (c I) . Bias with c = 1/scale
  // split into two bf16 terms (c_hi + c_lo, relative error ~2e-7); the scaled identities live in TMEM
  // (A operand, 64 columns each, after O1) and the bias tile is the MN-major B operand (like V).
  static constexpr uint32_t COL_ID = 256 + 2 * D;
  // Resident pair bias (unit_order 1, S_k <= 384): row r's bias for keys [0, S_k) as bf16 pairs in the
  // 192 columns after O1 (D = 32: [320, 512)), key k at column COL_BR + k / 2 -- replaces the identity MMAs
  static constexpr uint32_t COL_BR = 256 + 2 * D;
  static constexpr int BR_KEYS = 2 * (512 - (256 + 2 * D));
  static constexpr uint32_t IDESC_B = idesc_bf16_f32(128, 128, 1);
  static constexpr int ENTRIES_PER_TILE = DIFF ? 3 : 2;              // K0 [K1] V
};

// Softcap (no bias): tanh is monotone, so the row max of cap*tanh(a s) is cap*tanh(a max s) -- the max is
// taken on the raw scores (one tanh per row), and the per-score tanh moves off the critical max -> exp
// chain into the exp loop.  There it runs on the FMA pipe (kSoftcapPoly): tanh(a s) = a s P((a s)^2), P the
// odd minimax fit of degree 9 on |a s| <= 1.5 (|error| < 8.2e-5 in fp32, below tanh.approx.f32's 2^-11
// relative error), prescaled by a = scale / cap per call, whenever every |a s| of a warp's tile is <= 1.5
// (one warp vote on the raw max / min; with |Q|, |K| <= 1 and cap = 20 that is every tile at D <= 512),
// else on the MUFU.  The MUFU then carries one op per score (ex2) instead of two.
#ifndef FL_SOFTCAP_MUFU
constexpr bool kSoftcapPoly = true;
#else
constexpr bool kSoftcapPoly = false;
#endif
// groups of 4 scores (index (c/4) % 8) whose softcap tanh stays on the MUFU in the poly path (balances the
// FMA and MUFU pipes); A/B'd in profiles/r02_ab.md
#ifndef FL_TANH_MUFU_MASK
#define FL_TANH_MUFU_MASK 0u
#endif
constexpr uint32_t kTanhMufuMask = FL_TANH_MUFU_MASK;
constexpr float kTanhX0 = 1.5f;
constexpr float kTanhC0 = 0.9993646741f, kTanhC1 = -0.3268460035f, kTanhC2 = 0.1141102985f,
                kTanhC3 = -0.02846436948f, kTanhC4 = 0.003358259564f;
// Which groups of 4 scores (index (c/4) % 8) take the FMA-pipe exp2 (ex2_emu2) instead of
// the MUFU.  On paper a 3/8 fraction balances the pipes (MUFU 1/16 clk/SM per score vs FMA
// ~(2 + 6 f)/128), but measured on B200 (profiles/r01_ab_*.txt) the softmax warpgroups are
// latency/issue-bound, not MUFU-bound, and the extra ~5 instructions per emulated score cost
// more than they save (causal 1071 -> 982 TF/s with 3/8), so the default is 0 (all MUFU).
template <int D, int MOD>
struct EmuCfg {
#ifdef FL_EMU_MASK
  static constexpr uint32_t MASK = FL_EMU_MASK;
#else
  // measured (profiles/r01_ab_pingpong_emu.txt): softcap (tanh + ex2 on the MUFU) +2 % with 3/8,
  // D = 64 (diff, 2x MUFU per flop) +1.6 % with 2/8, D = 128 plain exp: no gain -> all MUFU
  static constexpr uint32_t MASK = MOD == MOD_SOFTCAP ? (kSoftcapPoly ? 0u : 0x4Au) : (D <= 64 ? 0x11u : 0u);
#endif
};

// ALiBi on the tensor core: s + (slope / scale) * c for the key index c within the tile is a rank-1 term,
// so S_i gets it from one extra K = 16 MMA: A = ones (columns 0-2), B row c = slope*c/scale split into
// three bf16 terms (hi + mid + lo, residual ~ |slope c / scale| 2^-24).  The per-tile remainder
// slope * (k0 - q_abs) stays in the exp FFMA's offset (delta), so the softmax loop runs ALiBi at the
// cost of plain attention (one FFMA per score less); 1/8 more tensor work on the S MMA.
#ifndef FL_ALIBI_FFMA
constexpr bool kAlibiMma = true;
#else
constexpr bool kAlibiMma = false;
#endif

// Ping-pong of the two softmax warpgroups' exp loops on named barriers (FA3-style).  Measured
// slower with the persistent kernel (causal 982 vs 1071 TF/s, diff 624 vs 681): the alternation
// serialises the exp loops while neither the MUFU nor the issue slots are saturated.  Opt-in.
#ifdef FL_PINGPONG
constexpr bool kPingPong = true;
#else
constexpr bool kPingPong = false;
#endif

// The KV tiles a CTA walks form a "schedule" indexed by step j; warpgroup i works on
// steps [lo[i], hi[i]).  For every interval mask (masks.cuh) step j IS KV tile j.  For
// the RSA block list (FL_MASK_BLOCKLIST) the unit is ONE query block whose cleaned,
// ascending list sits in shared memory: step j gives KV tile sched[2j] to WG0 and
// sched[2j+1] to WG1.
struct Work {
  int b, g, h;
  int g1;               // G index of warpgroup 1 (PAIR: g + 1, else g)
  int q0[2];            // first query row of each warpgroup's tile
  int lo[2], hi[2];     // schedule range [lo, hi) each warpgroup needs
  int lo_cta, hi_cta;
  const uint32_t* sched;  // blocklist schedule (nullptr for interval masks)
};

// Work unit u (persistent CTAs walk u = blockIdx.x, blockIdx.x + gridDim.x, ...).
// (b,h)-major so the ~148 co-resident CTAs share a few heads' K/V in L2; inside a
// head the heaviest (latest, for causal) query blocks go first, and the stride of
// gridDim.x cycles every CTA through light and heavy blocks (static balance).
// PAIR (small heads whose S_q leaves half of a 256-row unit empty, e.g. Evoformer rows at
// N_res = 384): the two warpgroups take the same 128-row query block of two neighbouring G
// entries (MSA rows s, s+1), each with its own Q, K, V and output, so no warpgroup idles.
template <int D, bool DIFF, bool LIST, bool PAIR>
__device__ __forceinline__ Work decode_work(const AttnParams& p, int u) {
  Work w;
  const int rows_per_unit = (DIFF || LIST || PAIR) ? 128 : 256;
  const int nqb = (p.Sq + rows_per_unit - 1) / rows_per_unit;
  const int bgh = u / nqb;
  const int qb = nqb - 1 - u % nqb;
  w.h = bgh % p.Hq;
  if (PAIR && p.unit_order == 1) {
    // resident pair bias: segment (b, h, q-block) major, G pairs minor -- a CTA's consecutive units share
    // the bias rows it holds in TMEM; q-blocks of one head run in lockstep on sibling CTAs (K/V via L2)
    const int ngp = (p.G + 1) >> 1;
    const int nqb128 = (p.Sq + 127) / 128;
    int seg = u / ngp;
    w.g = (u % ngp) * 2;
    w.g1 = w.g + 1;
    const int qb128 = seg % nqb128;
    seg /= nqb128;
    w.h = seg % p.Hq;
    w.b = seg / p.Hq;
    w.q0[0] = w.q0[1] = qb128 * 128;
  } else if (PAIR) {
    const int ngp = (p.G + 1) >> 1;
    w.g = ((bgh / p.Hq) % ngp) * 2;
    w.g1 = w.g + 1;
    w.b = bgh / (p.Hq * ngp);
  } else {
    w.g = (bgh / p.Hq) % p.G;
    w.g1 = w.g;
    w.b = bgh / (p.Hq * p.G);
  }
  w.lo_cta = 1 << 30;
  w.hi_cta = 0;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    if (!(PAIR && p.unit_order == 1)) w.q0[i] = (DIFF || LIST || PAIR) ? qb * 128 : qb * 256 + i * 128;
    w.lo[i] = w.hi[i] = 0;
    if (!LIST && w.q0[i] < p.Sq && !(PAIR && i == 1 && w.g1 >= p.G)) {
      const int q_last = min(p.Sq, w.q0[i] + 128) - 1;
      Interval iv = rows_union(p, w.b, w.q0[i], q_last);
      if (iv.hi > iv.lo) {
        w.lo[i] = iv.lo / 128;
        w.hi[i] = (iv.hi + 127) / 128;
      }
    }
    if (w.hi[i] > w.lo[i]) {
      w.lo_cta = min(w.lo_cta, w.lo[i]);
      w.hi_cta = max(w.hi_cta, w.hi[i]);
    }
  }
  if (w.hi_cta <= w.lo_cta) w.lo_cta = w.hi_cta = 0;
  w.sched = nullptr;
  return w;
}

// Blocklist mode: one thread copies the unit's list into `sched`, dropping entries
// outside [0, nkb) and repeats (the list is ascending, fl_attn.h), and stores the
// entry count n after it.  WG0 takes entries 0, 2, ... (ceil(n/2) steps), WG1 entries
// 1, 3, ... (floor(n/2) steps).
__device__ __forceinline__ void build_sched(const AttnParams& p, const Work& w, uint32_t* sched) {
  const int nkb = (p.Sk + 127) / 128;
  const int64_t bgh = ((int64_t)w.b * p.G + w.g) * p.Hq + w.h;
  const int64_t row = bgh * p.n_qblk + w.q0[0] / 128;
  const int32_t* li = p.blk_idx + row * p.max_sel;
  const int cnt = min(p.blk_cnt[row], p.max_sel);
  int n = 0, last = -1;
  for (int a = 0; a < cnt && n < kMaxSelTc; ++a) {
    const int j = li[a];
    if (j < 0 || j >= nkb || j <= last) continue;
    sched[n++] = (uint32_t)j;
    last = j;
  }
  reinterpret_cast<int*>(sched + 2 * kMaxSelTc)[0] = n;
}

__device__ __forceinline__ void load_sched(Work& w, const uint32_t* sched) {
  const int n = reinterpret_cast<const int*>(sched + 2 * kMaxSelTc)[0];
  w.sched = sched;
  w.lo[0] = w.lo[1] = 0;
  w.hi[0] = (n + 1) >> 1;
  w.hi[1] = n >> 1;
  w.lo_cta = 0;
  w.hi_cta = w.hi[0];
}

__device__ __forceinline__ bool needs(const Work& w, int i, int j) {
  // select, not w.lo[i]: a runtime index would force Work into local memory
  const int lo = i ? w.lo[1] : w.lo[0], hi = i ? w.hi[1] : w.hi[0];
  return j >= lo && j < hi;
}
// KV tile of warpgroup i at step j
template <bool LIST>
__device__ __forceinline__ int kv_tile(const Work& w, int i, int j) {
  if constexpr (LIST) return (int)w.sched[2 * j + i];
  return j;
}
__device__ __forceinline__ int next_tile(const Work& w, int j) {
  for (++j; j < w.hi_cta; ++j)
    if (needs(w, 0, j) || needs(w, 1, j)) return j;
  return -1;
}

// PAIR: 0 none, 1 paired G entries, 2 paired with the pair bias resident in TMEM (unit_order 1)
template <int D, bool DIFF, int MOD, bool BIAS, bool LIST, int PAIR = 0>
__global__ void __launch_bounds__(kThreadsTc, 1)
    attn_tc_kernel(const __grid_constant__ AttnParams p, const __grid_constant__ TmaMaps maps, int n_units) {
#ifdef FL_BIG   // measured slower (evo_row 0.405 -> 0.423 ms, evo_col unchanged: profiles/r02_ab.md): opt-in
  using C = TcCfg<D, DIFF, LIST, (D == 32 && !DIFF && !LIST && (!BIAS || PAIR == 2))>;
#else
  using C = TcCfg<D, DIFF, LIST>;
#endif
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned (SW128 atoms); offset arithmetic on smem_raw keeps the shared address space visible
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem + C::SMEM_Q;
  uint8_t* sRing = smem + C::SMEM_RING;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::SMEM_BAR);
  uint64_t* q_full = bars;                           // [NQBUF]
  uint64_t* q_empty = bars + C::NQBUF;               // [NQBUF]
  uint64_t* full = bars + 2 * C::NQBUF;
  uint64_t* empty = full + C::NSLOT;
  uint64_t* s_full = empty + C::NSLOT;
  uint64_t* p_full = s_full + 2;
  uint64_t* o_full = p_full + 2;
  uint64_t* unit_full = o_full + 2;                  // work-unit broadcast (producer -> MMA, softmax), 2 slots
  uint64_t* unit_empty = unit_full + 2;
  uint64_t* bias_full = unit_empty + 2;              // [wg * 2 + stage]
  uint64_t* bias_empty = bias_full + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bias_empty + 4);
  uint8_t* sBias = smem + C::SMEM_BIAS;
  // resident pair bias (Evoformer rows, unit_order 1): the softmax warpgroups add it from TMEM
  constexpr bool bias_res = C::BIAS_TMA_OK && BIAS && PAIR == 2;
  const bool bias_tma = C::BIAS_TMA_OK && BIAS && maps.bias_tma && !bias_res;
#ifdef FL_NO_BIAS_MMA
  const bool bias_mma = false;
#else
  const bool bias_mma = bias_tma && MOD == MOD_NONE;  // raw-score domain: S += bias / scale on the tensor core
#endif
  uint32_t* sched_base = reinterpret_cast<uint32_t*>(smem + C::SMEM_SCHED);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 8 && lane == 0) {
    for (int b = 0; b < C::NQBUF; ++b) {
      mbar_init(&q_full[b], 1);
      mbar_init(&q_empty[b], DIFF ? 1 + 128 : 1);    // last S MMA of a unit (+ diff: WG0 done with xbuf)
    }
    for (int s = 0; s < C::NSLOT; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&o_full[i], 1);
      mbar_init(&unit_full[i], 1);
      mbar_init(&unit_empty[i], 1 + 256);            // MMA lane + both softmax warpgroups
      for (int st = 0; st < 2; ++st) {
        mbar_init(&bias_full[i * 2 + st], 1);
        // the warpgroup's threads after reading their rows, or the MMA commit when the tensor core adds it
        mbar_init(&bias_empty[i * 2 + st], bias_mma ? 1 : 128);
      }
    }
    fence_mbar_init();
  }
  constexpr bool kAug = kAlibiMma && MOD == MOD_ALIBI;
  uint8_t* sAug = smem + C::SMEM_AUG;               // [ones A | B unit parity 0 | B unit parity 1]
  if constexpr (kAug) {
    // A: every row [1 1 1 0 0 0 0 0 | 1 1 1 0 0 0 0 0] -- ones in BOTH 16-B chunks of the 32-B row, so A
    // reads the same whatever the 32-B swizzle does; B (written per unit by the producer) holds its three
    // terms in one chunk and zeros in the other, so each term is counted exactly once either way
    for (int i = threadIdx.x; i < 3 * C::AUG_TILE / 16; i += kThreadsTc) {
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (i < C::AUG_TILE / 16) v = make_uint4(0x3F803F80u, 0x3F80u, 0u, 0u);
      reinterpret_cast<uint4*>(sAug)[i] = v;
    }
    fence_proxy_async_smem();
  }
  if (warp == 9) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (bias_mma) {
    // scaled identities c_hi I, c_lo I (bf16 pairs per 32-bit column: row r's entry at column r / 2)
    if (warp < 4) {
      const int r = threadIdx.x;
      const float cf = 1.f / p.scale;
      const float c_hi = __bfloat162float(__float2bfloat16_rn(cf));
      const float c_lo = cf - c_hi;
      const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
#pragma unroll
      for (int t2 = 0; t2 < 2; ++t2) {
        const float cv = t2 ? c_lo : c_hi;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t v[32];
#pragma unroll
          for (int w2 = 0; w2 < 32; ++w2) {
            const int word = half * 32 + w2;
            v[w2] = word == (r >> 1) ? pack_bf16((r & 1) ? 0.f : cv, (r & 1) ? cv : 0.f) : 0u;
          }
          tmem_st32(tmem + lane_base + C::COL_ID + t2 * 64 + half * 32, v);
        }
      }
      tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }

  // Dynamic persistent scheduling: the producer claims units (first blockIdx.x, then
  // gridDim.x + atomicAdd(tile_ctr)) in the (b,h)-major, heaviest-first order of
  // decode_work, so SMs that finish early take the next unit (greedy LPT within a head)
  // and publishes the id (and, for block lists, the merged schedule) in slot it & 1.
  auto get_unit = [&](int it) -> int {
    mbar_wait(&unit_full[it & 1], (it >> 1) & 1);
    return static_cast<int>(sched_base[(it & 1) * C::SCHED_WORDS + C::SCHED_WORDS - 1]);
  };
  // Work of the unit published in slot it & 1 (by value: keeps it in registers)
  // the producer publishes the decoded unit in the slot, so the MMA issuer and the softmax warpgroups do
  // not redo decode_work's integer divisions on their critical path at every unit start
  // (small heads only: their units are a few tiles long; at D >= 64 the registers the loaded fields occupy
  // cost more in spills than the recomputation, which the compiler can rematerialise from the parameters)
  auto unit_work_pub = [&](int it) -> Work {
    const uint32_t* sc = sched_base + (it & 1) * C::SCHED_WORDS;
    const int* f = reinterpret_cast<const int*>(sc + C::WORK_OFF);
    Work w;
    w.b = f[0]; w.g = f[1]; w.g1 = f[2]; w.h = f[3];
    w.q0[0] = f[4]; w.q0[1] = f[5];
    w.lo[0] = f[6]; w.hi[0] = f[7]; w.lo[1] = f[8]; w.hi[1] = f[9];
    w.lo_cta = f[10]; w.hi_cta = f[11];
    w.sched = LIST ? sc : nullptr;
    return w;
  };
  auto unit_work = [&](int u, int it) -> Work {
    if constexpr (D > 32) {
      Work w = decode_work<D, DIFF, LIST, (PAIR != 0)>(p, u);
      if constexpr (LIST) load_sched(w, sched_base + (it & 1) * C::SCHED_WORDS);
      return w;
    }
    const uint32_t* sc = sched_base + (it & 1) * C::SCHED_WORDS;
    const int* f = reinterpret_cast<const int*>(sc + C::WORK_OFF);
    Work w;
    w.b = f[0]; w.g = f[1]; w.g1 = f[2]; w.h = f[3];
    w.q0[0] = f[4]; w.q0[1] = f[5];
    w.lo[0] = f[6]; w.hi[0] = f[7]; w.lo[1] = f[8]; w.hi[1] = f[9];
    w.lo_cta = f[10]; w.hi_cta = f[11];
    w.sched = LIST ? sc : nullptr;
    return w;
  };
  auto unit_seg = [&](int it) { return reinterpret_cast<const int*>(sched_base + (it & 1) * C::SCHED_WORDS + C::WORK_OFF)[12]; };
  auto release_unit = [&](int it) { mbar_arrive(&unit_empty[it & 1]); };

  if (warp >= 8) {
   regs_dec<RegCfg<(DIFF || MOD == MOD_ALIBI)>::CTL>();
   if (warp == 8) {
    // ============================== TMA producer ==============================
    if (lane == 0) {
      tma_prefetch_desc(&maps.q);
      tma_prefetch_desc(&maps.k);
      tma_prefetch_desc(&maps.v);
      int e = 0, it = 0;
      int u = blockIdx.x, u_end = n_units;
      if (PAIR != 0 && p.unit_order == 1) {
        // static contiguous chunks: with grid = n_seg * cps every segment gets cps CTAs at the same offsets
        const int ngp = (p.G + 1) >> 1, n_seg = n_units / ngp, grid = (int)gridDim.x, c = (int)blockIdx.x;
        if (grid >= n_seg && grid % n_seg == 0) {
          const int cps = grid / n_seg, seg = c / cps, part = c % cps;
          u = seg * ngp + (int)((long long)part * ngp / cps);
          u_end = seg * ngp + (int)((long long)(part + 1) * ngp / cps);
        } else {
          u = (int)((long long)c * n_units / grid);
          u_end = (int)((long long)(c + 1) * n_units / grid);
        }
        if (u >= u_end) u = n_units;
      }
      int bcnt[2] = {0, 0};                            // bias tiles issued per warpgroup (stage = bcnt & 1)
      if (bias_tma) tma_prefetch_desc(&maps.bias);
      for (;; ++it) {
        uint32_t* sc = sched_base + (it & 1) * C::SCHED_WORDS;
        if (it >= 2) mbar_wait(&unit_empty[it & 1], ((it >> 1) - 1) & 1);
        sc[C::SCHED_WORDS - 1] = static_cast<uint32_t>(u);
        if (u >= n_units) {
          mbar_arrive(&unit_full[it & 1]);             // end marker
          break;
        }
        Work w = decode_work<D, DIFF, LIST, (PAIR != 0)>(p, u);
        if constexpr (LIST) {
          build_sched(p, w, sc);
          load_sched(w, sc);
        } else if (C::BIAS_TMA_OK && p.keybits && p.keybits_words <= (PAIR ? C::KBITS_WORDS / 2 : C::KBITS_WORDS)) {
          // small heads: the unit's key-mask bits (Evoformer MSA mask, <= 64 words) ride in the unit
          // slot, so the softmax warpgroups never wait on a global load for them (PAIR: both G entries)
          for (int pi = 0; pi < (PAIR ? 2 : 1); ++pi) {
            const int gg = pi ? min(w.g1, p.G - 1) : w.g;
            const uint32_t* kb = p.keybits + ((int64_t)w.b * p.G + gg) * p.keybits_words;
            uint32_t* dst = sc + pi * (C::KBITS_WORDS / 2);
            for (int i0 = 0; i0 < p.keybits_words; i0 += 16) {   // 16 loads in flight per batch
              uint32_t tmp[16];
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (i0 + i < p.keybits_words) tmp[i] = __ldg(kb + i0 + i);
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (i0 + i < p.keybits_words) dst[i0 + i] = tmp[i];
            }
          }
        }
        {
          int* f = reinterpret_cast<int*>(sc + C::WORK_OFF);
          f[0] = w.b; f[1] = w.g; f[2] = w.g1; f[3] = w.h;
          f[4] = w.q0[0]; f[5] = w.q0[1];
          f[6] = w.lo[0]; f[7] = w.hi[0]; f[8] = w.lo[1]; f[9] = w.hi[1];
          f[10] = w.lo_cta; f[11] = w.hi_cta;
          f[12] = (PAIR != 0 && p.unit_order == 1) ? u / ((p.G + 1) >> 1) : 0;   // resident-bias segment
        }
        mbar_arrive(&unit_full[it & 1]);               // release: id / schedule / Work visible to the waiters
        const int u_next = (PAIR != 0 && p.unit_order == 1) ? (u + 1 < u_end ? u + 1 : n_units)
                                                       : (int)gridDim.x + atomicAdd(p.tile_ctr, 1);   // latency hidden behind this unit
        const int hkv = w.h / p.grp;
        const int g1c = min(w.g1, p.G - 1);               // PAIR with odd G: WG1 of the last pair idles
        const int gq = maps.q_bcast_g ? 0 : w.g, bq = maps.q_bcast_b ? 0 : w.b;
        const int gk = maps.k_bcast_g ? 0 : w.g, bk = maps.k_bcast_b ? 0 : w.b;
        const int gv = maps.v_bcast_g ? 0 : w.g, bv = maps.v_bcast_b ? 0 : w.b;
        const int gq1 = maps.q_bcast_g ? 0 : g1c, gk1 = maps.k_bcast_g ? 0 : g1c, gv1 = maps.v_bcast_g ? 0 : g1c;
        const int qbuf = it % C::NQBUF, quse = it / C::NQBUF;
        // the S MMAs (and diff xbuf reads) of the unit that last used this Q buffer are done
        if (it >= C::NQBUF) mbar_wait(&q_empty[qbuf], (quse - 1) & 1);
        if constexpr (kAug) {
          // this unit's B tile (buffer it & 1; the S MMAs of unit it - 2 that read it are done): key c ->
          // slope*c/scale as hi + mid + lo bf16 terms in the 16-B chunk the SW32 swizzle maps chunk 0 to
          const float sl = (p.alibi ? p.alibi[w.h] : exp2f(-8.f * (float)(w.h + 1) / (float)p.Hq)) / p.scale;
          uint8_t* bt = sAug + (1 + (it & 1)) * C::AUG_TILE;
          for (int c = 0; c < 128; ++c) {
            const float a = sl * (float)c;
            const float hi = __bfloat162float(__float2bfloat16_rn(a));
            const float mid = __bfloat162float(__float2bfloat16_rn(a - hi));
            const float lo = a - hi - mid;
            const int ch = (c >> 2) & 1;
            *reinterpret_cast<uint2*>(bt + c * 32 + ch * 16) = make_uint2(pack_bf16(hi, mid), pack_bf16(lo, 0.f));
            *reinterpret_cast<uint2*>(bt + c * 32 + (ch ^ 1) * 16) = make_uint2(0u, 0u);
          }
          fence_proxy_async_smem();                    // generic-proxy stores -> the tensor core (via q_full)
        }
        mbar_arrive_expect_tx(&q_full[qbuf], C::NQ * C::TILE_BYTES);
        for (int i = 0; i < C::NQ; ++i) {
          const int qh = DIFF ? w.h + i * p.Hq : w.h;
          for (int c = 0; c < C::NCH; ++c)
            tma_load_5d(sQ + (qbuf * C::NQ + i) * C::TILE_BYTES + c * C::CHUNK_BYTES, &maps.q, &q_full[qbuf], c * C::CH, w.q0[i], qh,
                        i ? gq1 : gq, bq);
        }
        auto load_entry = [&](const CUtensorMap* m, int tile, int head, int gg, int bb) {
          const int slot = e % C::NSLOT;
          int row, bc;
          kv_tile_coords(p, w.b, tile, bb, row, bc);    // paged KV: the tile's page of the pool
          if (e >= C::NSLOT) mbar_wait(&empty[slot], ((e / C::NSLOT) - 1) & 1);
          mbar_arrive_expect_tx(&full[slot], C::TILE_BYTES);
          uint8_t* dst = sRing + slot * C::TILE_BYTES;
          for (int c = 0; c < C::NCH; ++c)
            tma_load_5d(dst + c * C::CHUNK_BYTES, m, &full[slot], c * C::CH, row, head, gg, bc);
          ++e;
        };
        for (int j = next_tile(w, w.lo_cta - 1); j >= 0; j = next_tile(w, j)) {
          if constexpr (LIST) {
            // step j: K(WG0) [K(WG1)] V(WG0) [V(WG1)] -- the order the MMA issuer acquires them
            const bool n1 = needs(w, 1, j);
            load_entry(&maps.k, kv_tile<LIST>(w, 0, j), hkv, gk, bk);
            if (n1) load_entry(&maps.k, kv_tile<LIST>(w, 1, j), hkv, gk, bk);
            load_entry(&maps.v, kv_tile<LIST>(w, 0, j), hkv, gv, bv);
            if (n1) load_entry(&maps.v, kv_tile<LIST>(w, 1, j), hkv, gv, bv);
          } else if constexpr (PAIR != 0) {
            // step j: K(g) [K(g+1)] V(g) [V(g+1)] -- the same KV tile of two G entries
            const bool n1 = needs(w, 1, j);
            load_entry(&maps.k, j, hkv, gk, bk);
            if (n1) load_entry(&maps.k, j, hkv, gk1, bk);
            load_entry(&maps.v, j, hkv, gv, bv);
            if (n1) load_entry(&maps.v, j, hkv, gv1, bv);
          } else {
            for (int t = 0; t < C::ENTRIES_PER_TILE; ++t) {
              const bool is_v = t == C::ENTRIES_PER_TILE - 1;
              load_entry(is_v ? &maps.v : &maps.k, j, is_v ? hkv : hkv + t * p.Hkv, is_v ? gv : gk, is_v ? bv : bk);
            }
          }
          if (bias_tma) {
            const int bb2 = maps.bias_bcast_b ? 0 : w.b;
            for (int i = 0; i < 2; ++i) {
              if (!needs(w, i, j)) continue;
              const int gb = maps.bias_bcast_g ? 0 : (i ? g1c : w.g);
              const int st = bcnt[i] & 1;
              if (bcnt[i] >= 2) mbar_wait(&bias_empty[i * 2 + st], ((bcnt[i] >> 1) - 1) & 1);
              mbar_arrive_expect_tx(&bias_full[i * 2 + st], C::BIAS_TILE);
              uint8_t* dst = sBias + (i * 2 + st) * C::BIAS_TILE;
              for (int c = 0; c < 2; ++c)
                tma_load_5d(dst + c * (C::BIAS_TILE / 2), &maps.bias, &bias_full[i * 2 + st],
                            kv_tile<LIST>(w, i, j) * C::BN + c * 64, w.q0[i], w.h, gb, bb2);
              ++bcnt[i];
            }
          }
        }
        u = u_next;
      }
    }
  } else if (warp == 9) {
    // ============================== MMA issuer ==============================
    if (lane == 0) {
      const uint32_t ring_addr = smem_u32(sRing);
      uint32_t sq_addr = smem_u32(sQ);                 // this unit's Q buffer
      int e = 0;
      auto acquire = [&]() -> int {
        const int slot = e % C::NSLOT;
        mbar_wait(&full[slot], (e / C::NSLOT) & 1);
        ++e;
        return slot;
      };
      int bcnt_m[2] = {0, 0};                          // bias tiles consumed per warpgroup (bias_mma)
      const uint32_t saug_addr = smem_u32(sAug);
      int it_mma = 0;                                  // unit counter (ALiBi B tile parity)
      const uint32_t sbias_addr = smem_u32(sBias);
      auto issue_s = [&](int i, int kslot) {
        const uint32_t qa = sq_addr + (LIST ? 0 : i) * C::TILE_BYTES, ka = ring_addr + kslot * C::TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk * 16 / C::CH) * C::CHUNK_BYTES + (kk * 16 % C::CH) * 2;
          umma_ss(tmem + (i ? C::COL_S1 : C::COL_S0), smem_desc(qa + off, 16, C::SBO, C::LAYOUT),
                  smem_desc(ka + off, 16, C::SBO, C::LAYOUT), C::IDESC_S, kk > 0);
        }
        if constexpr (kAug)                            // S_i += ones . (slope c / scale)^T (ALiBi, rank 1)
          umma_ss(tmem + (i ? C::COL_S1 : C::COL_S0), smem_desc(saug_addr, 16, 256, kLayoutSW32),
                  smem_desc(saug_addr + (1 + (it_mma & 1)) * C::AUG_TILE, 16, 256, kLayoutSW32), C::IDESC_S, 1u);
        if (bias_mma) {                                // S_i += (c_hi I + c_lo I) . Bias tile
          const int st = bcnt_m[i] & 1;
          mbar_wait(&bias_full[i * 2 + st], (bcnt_m[i] >> 1) & 1);
          tc_fence_after();
          const uint32_t ba = sbias_addr + (i * 2 + st) * C::BIAS_TILE;
#pragma unroll
          for (int t2 = 0; t2 < 2; ++t2)
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              umma_ts(tmem + (i ? C::COL_S1 : C::COL_S0), tmem + C::COL_ID + t2 * 64 + kk * 8,
                      smem_desc(ba + kk * 16 * 128, C::BIAS_TILE / 2, 1024, kLayoutSW128), C::IDESC_B, 1u);
          umma_commit(&bias_empty[i * 2 + st]);
          ++bcnt_m[i];
        }
        umma_commit(&s_full[i]);
      };
      int pv_cnt[2] = {0, 0};                          // cumulative: p_full parity
      bool first_pv[2];                                // per unit: first PV overwrites O
      auto issue_pv = [&](int i, int vslot) {
        mbar_wait(&p_full[i], pv_cnt[i] & 1);
        tc_fence_after();
        const uint32_t va = ring_addr + vslot * C::TILE_BYTES;
        const uint32_t pcol = (i ? C::COL_S1 : C::COL_S0) + C::P_OFF;
#pragma unroll
        for (int kk = 0; kk < C::BN / 16; ++kk) {
          umma_ts(tmem + (i ? C::COL_O1 : C::COL_O0), tmem + pcol + kk * 8,
                  smem_desc(va + kk * 16 * C::SWB, C::CHUNK_BYTES, C::SBO, C::LAYOUT), C::IDESC_O,
                  (!first_pv[i] || kk > 0) ? 1u : 0u);
        }
        first_pv[i] = false;
        ++pv_cnt[i];
      };
      int it = 0;
      for (;; ++it) {
        const int u = get_unit(it);
        if (u >= n_units) break;
        const Work w = unit_work_pub(it);           // published by the producer: no decode on the MMA's path
        it_mma = it;
        first_pv[0] = first_pv[1] = true;
        int j = next_tile(w, w.lo_cta - 1);
        const int qbuf = it % C::NQBUF;
        uint64_t* q_empty_u = &q_empty[qbuf];
        sq_addr = smem_u32(sQ) + qbuf * C::NQ * C::TILE_BYTES;
        mbar_wait(&q_full[qbuf], (it / C::NQBUF) & 1);  // always: Q of this unit has landed
        tc_fence_after();
        if (j >= 0) {
          // K of warpgroup 1 is a separate ring entry for diff (map 1) and block lists (its own tile);
          // V is separate for block lists only.  Entries a warpgroup does not need are not loaded.
          constexpr bool kSepK = DIFF || LIST || PAIR != 0;
          constexpr bool kSepV = LIST || PAIR != 0;
          int ks0 = acquire();
          int ks1 = kSepK ? ((!kSepV || needs(w, 1, j)) ? acquire() : -1) : ks0;
          if (needs(w, 0, j)) issue_s(0, ks0);
          if (needs(w, 1, j)) issue_s(1, ks1);
          umma_commit(&empty[ks0]);
          if (kSepK && ks1 >= 0) umma_commit(&empty[ks1]);
          if (next_tile(w, j) < 0) umma_commit(q_empty_u);   // Q is free once the last S MMA is done
          while (j >= 0) {
            const int va = acquire();
            const int vb = kSepV ? (needs(w, 1, j) ? acquire() : -1) : va;
            const int jn = next_tile(w, j);
            int kn0 = -1, kn1 = -1;
            if (jn >= 0) {
              kn0 = acquire();
              kn1 = kSepK ? ((!kSepV || needs(w, 1, jn)) ? acquire() : -1) : kn0;
            }
            if (needs(w, 0, j)) {
              issue_pv(0, va);
              if (j == w.hi[0] - 1) umma_commit(&o_full[0]);
            }
            if (jn >= 0 && needs(w, 0, jn)) issue_s(0, kn0);
            if (needs(w, 1, j)) {
              issue_pv(1, vb);
              if (j == w.hi[1] - 1) umma_commit(&o_full[1]);
            }
            umma_commit(&empty[va]);
            if (kSepV && vb >= 0) umma_commit(&empty[vb]);
            if (jn >= 0) {
              if (needs(w, 1, jn)) issue_s(1, kn1);
              umma_commit(&empty[kn0]);
              if (kSepK && kn1 >= 0) umma_commit(&empty[kn1]);
              if (next_tile(w, jn) < 0) umma_commit(q_empty_u);
            }
            j = jn;
          }
        } else {
          umma_commit(q_empty_u);
        }
        release_unit(it);
      }
    }
   }
  } else {
    regs_inc<RegCfg<(DIFF || MOD == MOD_ALIBI)>::SOFTMAX>();
#ifdef FL_TIMING
    long long t_acc[16] = {0};
    long long t_prev = clock64();
#endif
    // ============================== softmax warpgroups ==============================
    const int wg = warp >> 2;
    const int r = threadIdx.x & 127;                 // row within the tile == TMEM lane
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t col_s = wg ? C::COL_S1 : C::COL_S0;
    // small heads without TMA'd bias tiles: the bias-tile area holds each thread's 64-B gate row
    const bool gate_async = D <= 32 && C::BIAS_AREA && !bias_tma && p.gate_mode != GATE_NONE && !(DIFF && wg == 1);
    uint8_t* sGateRow = sBias + (wg * 128 + r) * 64;
    const uint32_t col_o = wg ? C::COL_O1 : C::COL_O0;
    const float sc_l2 = p.scale * kLog2e;
    const float cap_in = MOD == MOD_SOFTCAP ? p.scale / p.softcap : 0.f;   // s*scale/cap
    const float cap_out = MOD == MOD_SOFTCAP ? p.softcap * kLog2e : 0.f;
    // softcap tanh polynomial prescaled by a = cap_in: tanh(a s) = s * sum_i (kTanhC_i a^(2i+1)) (s^2)^i
    constexpr bool kCapFirst = MOD == MOD_SOFTCAP && !BIAS;   // max on raw scores, tanh in the exp loop
    float tc0 = 0.f, tc1 = 0.f, tc2 = 0.f, tc3 = 0.f, tc4 = 0.f;
    if (kCapFirst && kSoftcapPoly) {
      const float a2 = cap_in * cap_in;
      tc0 = kTanhC0 * cap_in;
      tc1 = kTanhC1 * cap_in * a2;
      tc2 = kTanhC2 * cap_in * a2 * a2;
      tc3 = kTanhC3 * cap_in * a2 * a2 * a2;
      tc4 = kTanhC4 * cap_in * a2 * a2 * a2 * a2;
    }
    const float s_poly_max = MOD == MOD_SOFTCAP ? kTanhX0 / cap_in : 0.f;   // |s| bound of the polynomial
    int s_cnt = 0, o_cnt = 0;                        // cumulative s_full / o_full phases of this WG
    int b_cnt = 0;                                   // bias tiles consumed (TMA path)
    bool pp_started = false;                         // ping-pong: first common tile of the CTA's life seen
    bool o_lent = false;                             // LIST, WG1: O1 / (m, l) still being read by WG0
    int res_seg = -1;                                // bias_res: segment whose bias rows TMEM holds
    int it = 0;
    for (;; ++it) {
    const int u = get_unit(it);
    if (u >= n_units) break;
    FL_T(11);                                        // 11: waiting for the next unit id
    const Work w = unit_work(u, it);
    const int gw = wg ? w.g1 : w.g;                  // this warpgroup's G entry
    const int q = (wg ? w.q0[1] : w.q0[0]) + r;
    const bool row_valid = q < p.Sq && (!PAIR || gw < p.G);
    const int q_abs = q + p.q_off;
    const Interval iv = row_interval(p, w.b, q);
    float slope_l2 = 0.f;
    if (MOD == MOD_ALIBI)
      slope_l2 = kLog2e * (p.alibi ? p.alibi[w.h] : exp2f(-8.f * (float)(w.h + 1) / (float)p.Hq));
    const uint32_t* kbits =
        p.keybits ? p.keybits + ((int64_t)w.b * p.G + min(gw, p.G - 1)) * p.keybits_words : nullptr;
    // The unit's key-mask bits (Evoformer MSA mask: <= 16 words) are staged once per unit in shared
    // memory, so no tile waits on a global load for them.
    // small heads: staged in the unit slot by the producer (read before release_unit)
    const uint32_t* kb_smem = sched_base + (it & 1) * C::SCHED_WORDS + (PAIR && wg ? C::KBITS_WORDS / 2 : 0);
    const bool kb_staged =
        !LIST && C::BIAS_TMA_OK && kbits && p.keybits_words <= (PAIR ? C::KBITS_WORDS / 2 : C::KBITS_WORDS);
    FL_T(12);                                        // 12: unit setup (work decode, key-mask staging)
    // small heads: the gate row (64 B at c = 32) is copied by cp.async into this thread's slot of the
    // (otherwise unused) bias-tile area now, tiles before the epilogue reads it (an L1 prefetch here, or
    // loads issued in the epilogue, left the first use of the gate stalled: 5 % of the ncu samples)
    if (gate_async && row_valid) {
      const uint4* gsrc = reinterpret_cast<const uint4*>(static_cast<const unsigned short*>(p.gate) + w.b * p.gs.b +
                                                         gw * p.gs.g + (int64_t)w.h * p.gs.h + (int64_t)q * p.gs.s);
#pragma unroll
      for (int t8 = 0; t8 < 4; ++t8) cp_async_16(sGateRow + ((t8 ^ (r & 3)) << 4), gsrc + t8);
      cp_async_commit();
    }
    if constexpr (bias_res) {
      // resident pair bias: on a new (b, h, q-block) segment both warpgroups refill the row's bias in TMEM
      // (WG0 keys [0, BR_KEYS/2), WG1 the rest), between two barriers so no tile reads a half-written row
      const int seg = unit_seg(it);
      if (seg != res_seg) {
        if (res_seg >= 0) named_bar_sync(6, 256);   // both warpgroups are done with the old rows
        const unsigned short* brow = static_cast<const unsigned short*>(p.bias) + w.b * p.bs.b +
                                     (int64_t)w.h * p.bs.h + (int64_t)(q < p.Sq ? q : 0) * p.bs.s;
#pragma unroll 1
        for (int ch = 0; ch < C::BR_KEYS / 2 / 64; ++ch) {
          const int kb0 = wg * (C::BR_KEYS / 2) + ch * 64;
          uint32_t bv[32];
#pragma unroll
          for (int t8 = 0; t8 < 8; ++t8) {
            const int k8 = kb0 + t8 * 8;
            uint4 v4 = make_uint4(0u, 0u, 0u, 0u);
            if (q < p.Sq) {
              if (k8 + 8 <= p.Sk) {
                v4 = __ldg(reinterpret_cast<const uint4*>(brow + k8));
              } else {
                uint32_t e2[4];
#pragma unroll
                for (int t = 0; t < 4; ++t)
                  e2[t] = (k8 + 2 * t < p.Sk ? (uint32_t)brow[k8 + 2 * t] : 0u) |
                          ((k8 + 2 * t + 1 < p.Sk ? (uint32_t)brow[k8 + 2 * t + 1] : 0u) << 16);
                v4 = make_uint4(e2[0], e2[1], e2[2], e2[3]);
              }
            }
            bv[4 * t8] = v4.x;
            bv[4 * t8 + 1] = v4.y;
            bv[4 * t8 + 2] = v4.z;
            bv[4 * t8 + 3] = v4.w;
          }
          tmem_st32(tmem + lane_base + C::COL_BR + (kb0 >> 1), bv);
        }
        tmem_wait_st();
        tc_fence_before();
        named_bar_sync(6, 256);
        tc_fence_after();
        res_seg = seg;
      }
    }
    const unsigned char* bias_row = nullptr;
    if (BIAS)
      bias_row = static_cast<const unsigned char*>(p.bias) +
                 (w.b * p.bs.b + min(gw, p.G - 1) * p.bs.g + (int64_t)w.h * p.bs.h + (int64_t)(row_valid ? q : 0) * p.bs.s) *
                     (p.bias_dtype == 1 ? 4 : 2);

    float m_ref = -INFINITY, l = 0.f;
    int n_done = 0;
    for (int j = next_tile(w, w.lo_cta - 1); j >= 0; j = next_tile(w, j)) {
      if (!needs(w, wg, j)) continue;
      const int k0 = kv_tile<LIST>(w, wg, j) * 128;
      uint32_t kw[4];                                  // key-mask bits of this tile, loaded before the S wait
      if (kb_staged) {
#pragma unroll
        for (int t = 0; t < 4; ++t) kw[t] = kb_smem[(k0 >> 5) + t];
      } else if (kbits) {
#pragma unroll
        for (int t = 0; t < 4; ++t) kw[t] = __ldg(kbits + (k0 >> 5) + t);
      }
      FL_T(0);                                         // 0: tile bookkeeping / previous epilogue
      mbar_wait(&s_full[wg], s_cnt & 1);
      FL_T(1);                                         // 1: waiting for S
      ++s_cnt;
      tc_fence_after();
      uint32_t s[128];
      tmem_ld32(tmem + lane_base + col_s + 0, &s[0]);
      tmem_ld32(tmem + lane_base + col_s + 32, &s[32]);
      tmem_ld32(tmem + lane_base + col_s + 64, &s[64]);
      tmem_ld32(tmem + lane_base + col_s + 96, &s[96]);
      tmem_wait_ld();
      FL_T(2);                                         // 2: tcgen05.ld of S
      // ---- score modification (Eq.4) in the log2 domain: x = log2(e) * mod(scale * s)
      float x[128];
      // The log2-domain score is x * xscale + delta, with the per-element work kept minimal:
      //  * kRaw (none / ALiBi): x = s + bias / scale + (slope / scale) * c, xscale = scale * log2(e),
      //    delta = slope * log2(e) * (k0 - q_abs) (per row and tile) -- one FFMA per element for ALiBi;
      //  * softcap without bias: x = tanh(s * scale / cap), xscale = cap * log2(e), delta = 0;
      //  * softcap with bias: x in log2 units (G16 order: bias before the cap), xscale = 1.
      // xscale and delta fold into the row max (a scalar op) and into the exp FFMA.
      constexpr bool kRaw = MOD == MOD_NONE || MOD == MOD_ALIBI;
      const float bias_k = kRaw ? 1.f / p.scale : kLog2e;
      const float delta = MOD == MOD_ALIBI ? slope_l2 * (float)(k0 - q_abs) : 0.f;
      const float slope_r = MOD == MOD_ALIBI ? slope_l2 / sc_l2 : 0.f;
      bool poly = false;                               // kCapFirst: this warp's tile takes the FMA-pipe tanh
      if (kCapFirst && kSoftcapPoly) {
        float am0 = 0.f, am1 = 0.f;
#pragma unroll
        for (int c = 0; c < 128; c += 4) {
          am0 = fmax3(am0, fabsf(__uint_as_float(s[c])), fabsf(__uint_as_float(s[c + 1])));
          am1 = fmax3(am1, fabsf(__uint_as_float(s[c + 2])), fabsf(__uint_as_float(s[c + 3])));
        }
        poly = __all_sync(0xffffffffu, fmaxf(am0, am1) <= s_poly_max);
      }
#pragma unroll
      for (int c = 0; c < 128; ++c) {
        float v = __uint_as_float(s[c]);
        if (kCapFirst) {
          // raw score: tanh after the row max (exp loop)
        } else if (MOD == MOD_ALIBI && !kAug) {
          v = fmaf(slope_r, (float)c, v);
        } else if (!kRaw) {
          v *= sc_l2;
        }
        x[c] = v;
      }
      if (BIAS && !bias_mma) {  // additive bias (Evoformer pair bias), then softcap if any (order G16)
        if constexpr (bias_res) {
          // this row's bias for the tile's keys: 64 TMEM columns of bf16 pairs
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            uint32_t bw[32];
            tmem_ld32(tmem + lane_base + C::COL_BR + (k0 >> 1) + h2 * 32, bw);
            tmem_wait_ld();
#pragma unroll
            for (int t = 0; t < 32; ++t)
              ffma2(x[h2 * 64 + 2 * t], x[h2 * 64 + 2 * t + 1], bf16_lo(bw[t]), bf16_hi(bw[t]), bias_k, bias_k,
                    x[h2 * 64 + 2 * t], x[h2 * 64 + 2 * t + 1]);
          }
        } else {
        if (bias_tma) {
          // this row of the bias tile from shared memory: slab c holds keys [64c, 64c+64), 16-byte
          // chunk k of row r at (k ^ (r & 7)) -- the TMA 128-B swizzle, so 8 consecutive rows hit
          // 8 different bank groups
          const int st = b_cnt & 1;
          FL_T(3);
          mbar_wait(&bias_full[wg * 2 + st], (b_cnt >> 1) & 1);
          FL_T(9);                                     // 9: waiting for the pair-bias tile
          const uint8_t* bt = sBias + (wg * 2 + st) * C::BIAS_TILE + r * 128;
#pragma unroll
#ifdef FL_ABL_BIAS
          if (false)
#endif
          for (int b4 = 0; b4 < 4; ++b4) {             // 4 batches of 4 x 16 B: no spills in the score loop
            uint4 u4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int c8 = b4 * 4 + e;
              u4[e] = *reinterpret_cast<const uint4*>(bt + (c8 >> 3) * (C::BIAS_TILE / 2) + (((c8 & 7) ^ (r & 7)) << 4));
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int c8 = b4 * 4 + e;
              const uint32_t ww[4] = {u4[e].x, u4[e].y, u4[e].z, u4[e].w};
#pragma unroll
              for (int t = 0; t < 4; ++t)
                ffma2(x[c8 * 8 + 2 * t], x[c8 * 8 + 2 * t + 1], bf16_lo(ww[t]), bf16_hi(ww[t]), bias_k, bias_k,
                      x[c8 * 8 + 2 * t], x[c8 * 8 + 2 * t + 1]);
            }
          }
          mbar_arrive(&bias_empty[wg * 2 + st]);
          ++b_cnt;
        } else if (p.bias_vec && k0 + 128 <= p.Sk) {
          // full tile: issue 8 independent 16-byte loads before the first use (one L2 round trip
          // per half row instead of one per load)
          const uint4* br = reinterpret_cast<const uint4*>(bias_row + (int64_t)k0 * 2);
#pragma unroll
          for (int h8 = 0; h8 < 2; ++h8) {
            uint4 u4[8];
#pragma unroll
            for (int c8 = 0; c8 < 8; ++c8) u4[c8] = __ldg(br + h8 * 8 + c8);
#pragma unroll
            for (int c8 = 0; c8 < 8; ++c8) {
              const uint32_t ww[4] = {u4[c8].x, u4[c8].y, u4[c8].z, u4[c8].w};
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const int c = (h8 * 8 + c8) * 8 + 2 * t;
                x[c] = fmaf(bf16_lo(ww[t]), bias_k, x[c]);
                x[c + 1] = fmaf(bf16_hi(ww[t]), bias_k, x[c + 1]);
              }
            }
          }
        } else if (p.bias_vec) {  // ragged last tile: element loads, predicated, batched the same way
          const unsigned short* bs16 = reinterpret_cast<const unsigned short*>(bias_row);
#pragma unroll
          for (int h8 = 0; h8 < 4; ++h8) {
            unsigned short us[32];
#pragma unroll
            for (int t = 0; t < 32; ++t) {
              const int k = k0 + h8 * 32 + t;
              us[t] = k < p.Sk ? bs16[k] : (unsigned short)0;
            }
#pragma unroll
            for (int t = 0; t < 32; ++t)
              x[h8 * 32 + t] = fmaf(__uint_as_float((uint32_t)us[t] << 16), bias_k, x[h8 * 32 + t]);
          }
        } else {
#pragma unroll
          for (int c = 0; c < 128; ++c) {
            const int k = min(k0 + c, p.Sk - 1);
            const float bv =
                p.bias_dtype == 1
                    ? reinterpret_cast<const float*>(bias_row)[(int64_t)k * p.bs.d]
                    : __uint_as_float((uint32_t)reinterpret_cast<const unsigned short*>(bias_row)[(int64_t)k * p.bs.d]
                                      << 16);
            x[c] = fmaf(bv, bias_k, x[c]);
          }
        }
        }
        if (MOD == MOD_SOFTCAP) {
#pragma unroll
          for (int c = 0; c < 128; ++c) x[c] = cap_out * tanh_approx(x[c] * (kLn2 / p.softcap));
        }
      }
      // ---- masking: only tiles that are not inside every row's interval
      const bool full_tile = tile_inside(iv, k0, p.Sk);
      if (__any_sync(0xffffffffu, !full_tile)) {
#pragma unroll
        for (int c = 0; c < 128; ++c) {
          const int k = k0 + c;
          x[c] = (k >= iv.lo && k < iv.hi) ? x[c] : -INFINITY;
        }
      }
      // key mask: the words are the same for every row (warp-uniform), so fully kept tiles skip it
      if (kbits && (kw[0] & kw[1] & kw[2] & kw[3]) != 0xFFFFFFFFu) {
#pragma unroll
        for (int c = 0; c < 128; ++c) x[c] = ((kw[c >> 5] >> (c & 31)) & 1u) ? x[c] : -INFINITY;
      }
      // ---- online softmax with conditional rescale (threshold kTau, log2 units)
      float mt0 = -INFINITY, mt1 = -INFINITY, mt2 = -INFINITY, mt3 = -INFINITY;
#pragma unroll
      for (int c = 0; c < 128; c += 8) {
        mt0 = fmax3(mt0, x[c], x[c + 1]);
        mt1 = fmax3(mt1, x[c + 2], x[c + 3]);
        mt2 = fmax3(mt2, x[c + 4], x[c + 5]);
        mt3 = fmax3(mt3, x[c + 6], x[c + 7]);
      }
      const float xscale = kRaw ? sc_l2 : (MOD == MOD_SOFTCAP && !BIAS ? cap_out : 1.f);
      float mt;
      if (kCapFirst) {                                 // max of cap tanh(a s) = cap tanh(a max s): one tanh per row
        const float smax = fmaxf(fmaxf(mt0, mt1), fmaxf(mt2, mt3));
        mt = smax == -INFINITY ? -INFINITY : cap_out * tanh_approx(smax * cap_in);
      } else {
        mt = fmaf(fmaxf(fmaxf(mt0, mt1), fmaxf(mt2, mt3)), xscale, delta);   // -inf stays -inf
      }
      FL_T(3);                                         // 3: score mod + mask + row max
      const bool rescale = mt > m_ref + kTau;          // also true for the first finite tile (m_ref = -inf)
      const float factor = rescale ? ex2(m_ref - mt) : 1.f;
      if (n_done > 0 && __any_sync(0xffffffffu, rescale)) {
        // O_i is quiescent: PV_i(j-1) completed before S_i(j)'s commit arrived.
#pragma unroll
        for (int c = 0; c < D; c += 32) {
          uint32_t o[32];
          tmem_ld32(tmem + lane_base + col_o + c, o);
          tmem_wait_ld();
#pragma unroll
          for (int t = 0; t < 32; ++t) o[t] = __float_as_uint(__uint_as_float(o[t]) * factor);
          tmem_st32(tmem + lane_base + col_o + c, o);
        }
      }
      if (rescale) {
        l *= factor;
        m_ref = mt;
      }
      const float neg_m = (m_ref == -INFINITY ? 0.f : -m_ref) + delta;   // exp2(x * xscale + delta - m_ref)
      // Ping-pong: the two warpgroups take turns on the MUFU (exp) pipe for the
      // tiles both need, so each exp loop runs at full rate while the tensor
      // pipe works for the other warpgroup (CTA-local named barriers 2 and 3).
      // The alternation runs across units: WG0 waits for WG1's previous common
      // tile except at the CTA's first one (and once more after its last unit);
      // WG1 signals after every common tile.
      const bool common = kPingPong && needs(w, 0, j) && needs(w, 1, j);
      FL_T(4);                                         // 4: O rescale
      if (common) {
        if (wg == 0 && pp_started) named_bar_sync(2, 256);
        if (wg == 1) named_bar_sync(3, 256);
        pp_started = true;
      }
      FL_T(5);                                         // 5: ping-pong wait
      float ls0 = 0.f, ls1 = 0.f, ls2 = 0.f, ls3 = 0.f;
      uint32_t pk[64];
      // P for scores c..c+3 given their (modified) log2-domain values: exp FFMA, ex2 (MUFU or FMA-pipe
      // emulation), row-sum, bf16 pack
      auto exp4 = [&](const int c, float v0, float v1, float v2, float v3) {
        float a0, a1, a2, a3;
        ffma2(a0, a1, v0, v1, xscale, xscale, neg_m, neg_m);
        ffma2(a2, a3, v2, v3, xscale, xscale, neg_m, neg_m);
        if ((EmuCfg<D, MOD>::MASK >> ((c >> 2) & 7)) & 1u) {
          ex2_emu2(a0, a1);
          ex2_emu2(a2, a3);
        } else {
          a0 = ex2(a0);
          a1 = ex2(a1);
          a2 = ex2(a2);
          a3 = ex2(a3);
        }
        fadd2(ls0, ls1, ls0, ls1, a0, a1);
        fadd2(ls2, ls3, ls2, ls3, a2, a3);
        pk[c >> 1] = pack_bf16(a0, a1);
        pk[(c >> 1) + 1] = pack_bf16(a2, a3);
      };
      // tanh(a s) of a pair on the FMA pipe; -inf: u = +inf, P = +inf (tc4 > 0), result -inf
      auto tanh_poly2 = [&](float& v0, float& v1) {
        float u0, u1, p0, p1;
        fmul2(u0, u1, v0, v1, v0, v1);
        ffma2(p0, p1, u0, u1, tc4, tc4, tc3, tc3);
        ffma2(p0, p1, p0, p1, u0, u1, tc2, tc2);
        ffma2(p0, p1, p0, p1, u0, u1, tc1, tc1);
        ffma2(p0, p1, p0, p1, u0, u1, tc0, tc0);
        fmul2(v0, v1, p0, p1, v0, v1);
      };
      if (kCapFirst && kSoftcapPoly && poly) {
        // software-pipelined: the FMA-pipe tanh of scores c+4..c+7 is issued before the MUFU ex2 of
        // c..c+3, so the polynomial runs under the exp loop instead of as a pass before it
        float t0 = x[0], t1 = x[1], t2 = x[2], t3 = x[3];
        tanh_poly2(t0, t1);
        tanh_poly2(t2, t3);
#pragma unroll
        for (int c = 0; c < 128; c += 4) {
          float n0 = 0.f, n1 = 0.f, n2 = 0.f, n3 = 0.f;
          if (c + 4 < 128) {
            n0 = x[c + 4];
            n1 = x[c + 5];
            n2 = x[c + 6];
            n3 = x[c + 7];
            if ((kTanhMufuMask >> (((c + 4) >> 2) & 7)) & 1u) {   // this group's tanh on the MUFU
              n0 = n0 == -INFINITY ? -INFINITY : tanh_approx(n0 * cap_in);
              n1 = n1 == -INFINITY ? -INFINITY : tanh_approx(n1 * cap_in);
              n2 = n2 == -INFINITY ? -INFINITY : tanh_approx(n2 * cap_in);
              n3 = n3 == -INFINITY ? -INFINITY : tanh_approx(n3 * cap_in);
            } else {
              tanh_poly2(n0, n1);
              tanh_poly2(n2, n3);
            }
          }
          exp4(c, t0, t1, t2, t3);
          t0 = n0;
          t1 = n1;
          t2 = n2;
          t3 = n3;
        }
      } else {
        if (kCapFirst) {                               // x = tanh(a s) on the MUFU; -inf stays -inf
#pragma unroll
          for (int c = 0; c < 128; ++c) x[c] = x[c] == -INFINITY ? -INFINITY : tanh_approx(x[c] * cap_in);
        }
#pragma unroll
        for (int c = 0; c < 128; c += 4) exp4(c, x[c], x[c + 1], x[c + 2], x[c + 3]);
      }
      FL_T(6);                                         // 6: exp loop
      if (common) {
        if (wg == 0) named_bar_arrive(3, 256);
        if (wg == 1) named_bar_arrive(2, 256);
      }
      l += (ls0 + ls1) + (ls2 + ls3);
      tmem_st32(tmem + lane_base + col_s + C::P_OFF, &pk[0]);
      tmem_st32(tmem + lane_base + col_s + C::P_OFF + 32, &pk[32]);
      tmem_wait_st();
      tc_fence_before();
      if (LIST && o_lent) {                            // PV1 of this tile overwrites O1: WG0 must have read it
        named_bar_sync(5, 256);
        o_lent = false;
      }
      mbar_arrive(&p_full[wg]);
      ++n_done;
      FL_T(7);                                         // 7: P store + arrive
    }
    release_unit(it);

    // ============================== epilogue ==============================
    // O_i of the next unit is first written by PV_i(next, first), which waits for this
    // warpgroup's p_full of that tile -- i.e. after this epilogue has read O_i.
#ifndef FL_ABL_GATE
    const bool gated = p.gate_mode != GATE_NONE && row_valid && !(DIFF && wg == 1);
#else
    const bool gated = false;
#endif
    const uint4* gp = reinterpret_cast<const uint4*>(static_cast<const unsigned short*>(p.gate) + w.b * p.gs.b +
                                                     gw * p.gs.g + (int64_t)w.h * p.gs.h + (int64_t)q * p.gs.s);
    if (n_done > 0) {
      mbar_wait(&o_full[wg], o_cnt & 1);
      ++o_cnt;
      tc_fence_after();
    }
    bool empty_row = m_ref == -INFINITY || !(l > 0.f);   // G7 (emulated exps of -inf are ~2^-126, not 0)
    float inv_l = empty_row ? 0.f : 1.f / l;
    float* ml = reinterpret_cast<float*>(smem + C::SMEM_ML);   // LIST: WG1's (m, l) per row
    float c1 = 0.f;                                  // LIST: weight of WG1's partial O1
    if (LIST && wg == 1) {
      if (o_lent) named_bar_sync(5, 256);            // WG0 is done with the previous unit's (m, l)
      ml[r] = m_ref;
      ml[128 + r] = l;
      named_bar_arrive(4, 256);
      o_lent = true;
      continue;                                      // WG0 writes the merged rows
    }
    if (LIST) {
      // merge the two halves of the list: O = (O0 2^(m0-m) + O1 2^(m1-m)) / (l0 2^(m0-m) + l1 2^(m1-m))
      named_bar_sync(4, 256);
      tc_fence_after();
      const float m1 = ml[r], l1 = ml[128 + r];
      const float mm = fmaxf(m_ref, m1);
      const float a0 = m_ref == -INFINITY ? 0.f : ex2(m_ref - mm), a1 = m1 == -INFINITY ? 0.f : ex2(m1 - mm);
      const float lt = l * a0 + l1 * a1;
      empty_row = mm == -INFINITY || !(lt > 0.f);
      inv_l = empty_row ? 0.f : a0 / lt;
      c1 = empty_row ? 0.f : a1 / lt;
      m_ref = mm;
      l = lt;
    }
    const float lam = DIFF ? diff_lambda(p, w.h) : 0.f;
    float* xbuf = reinterpret_cast<float*>(sQ);      // diff: map-1 rows handed to WG0 (Q is dead now)
    if (DIFF && wg == 1) {
      if (n_done == 0) mbar_wait(q_full, it & 1);    // never overwrite Q while its TMA may be in flight
#pragma unroll
      for (int c = 0; c < D; c += 32) {
        uint32_t o[32];
        if (n_done > 0) {
          tmem_ld32(tmem + lane_base + col_o + c, o);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int t = 0; t < 32; ++t) o[t] = 0u;
        }
#pragma unroll
        for (int t4 = 0; t4 < 8; ++t4) {
          const int chunk = (c >> 2) + t4;           // 16-byte chunk index within the row
          float4 v = make_float4(__uint_as_float(o[4 * t4]) * inv_l, __uint_as_float(o[4 * t4 + 1]) * inv_l,
                                 __uint_as_float(o[4 * t4 + 2]) * inv_l, __uint_as_float(o[4 * t4 + 3]) * inv_l);
          reinterpret_cast<float4*>(xbuf + r * D)[chunk ^ (r & 7)] = v;
        }
      }
      named_bar_sync(1, 256);
    } else {
      if (DIFF) named_bar_sync(1, 256);
      const int64_t obase = w.b * p.os.b + gw * p.os.g + (int64_t)w.h * p.os.h + (int64_t)q * p.os.s;
      // DIFF-Transformer epilogue (NEXT-2): the row's A_0 - lambda A_1 in registers, then per-head RMSNorm
      // over D_v and the (1 - lambda_init) scale before the store
      float norm_k = 1.f;
      float drow[DIFF ? D : 1];
      if (DIFF && p.diff_norm) {
        float ss0 = 0.f, ss1 = 0.f;
#pragma unroll
        for (int c = 0; c < D; c += 32) {
          uint32_t o[32];
          if (n_done > 0) {
            tmem_ld32(tmem + lane_base + col_o + c, o);
            tmem_wait_ld();
          } else {
#pragma unroll
            for (int t = 0; t < 32; ++t) o[t] = 0u;
          }
#pragma unroll
          for (int t4 = 0; t4 < 8; ++t4) {
            const float4 v = reinterpret_cast<const float4*>(xbuf + r * D)[((c >> 2) + t4) ^ (r & 7)];
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float f = fmaf(-lam, vv[e], __uint_as_float(o[4 * t4 + e]) * inv_l);
              drow[c + 4 * t4 + e] = f;
              if (e & 1) ss1 = fmaf(f, f, ss1); else ss0 = fmaf(f, f, ss0);
            }
          }
        }
        norm_k = rsqrtf((ss0 + ss1) / (float)D + p.diff_norm_eps) * (1.f - p.lambda_init);
      }
#pragma unroll
      for (int c = 0; c < D; c += 32) {
        float f[32];
        if (DIFF && p.diff_norm) {
#pragma unroll
          for (int t = 0; t < 32; ++t)
            f[t] = drow[c + t] * norm_k * (p.diff_norm_w ? __ldg(p.diff_norm_w + c + t) : 1.f);
        } else {
        uint32_t o[32];
        if (n_done > 0) {
          tmem_ld32(tmem + lane_base + col_o + c, o);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int t = 0; t < 32; ++t) o[t] = 0u;
        }
#pragma unroll
        for (int t = 0; t < 32; ++t) f[t] = __uint_as_float(o[t]) * inv_l;
        if (LIST && w.hi[1] > 0) {                     // WG1's partial, read from its TMEM columns (same lanes)
          tmem_ld32(tmem + lane_base + C::COL_O1 + c, o);
          tmem_wait_ld();
#pragma unroll
          for (int t = 0; t < 32; ++t) f[t] = fmaf(__uint_as_float(o[t]), c1, f[t]);
        }
        if (DIFF) {
#pragma unroll
          for (int t4 = 0; t4 < 8; ++t4) {
            const float4 v = reinterpret_cast<const float4*>(xbuf + r * D)[((c >> 2) + t4) ^ (r & 7)];
            f[4 * t4] -= lam * v.x;
            f[4 * t4 + 1] -= lam * v.y;
            f[4 * t4 + 2] -= lam * v.z;
            f[4 * t4 + 3] -= lam * v.w;
          }
        }
        }
        if (gated) {
          uint4 g4[4];
          if (gate_async) {                            // staged by cp.async at the unit's start
            cp_async_wait_all();
#pragma unroll
            for (int t8 = 0; t8 < 4; ++t8) g4[t8] = reinterpret_cast<const uint4*>(sGateRow)[t8 ^ (r & 3)];
          } else {
#pragma unroll
            for (int t8 = 0; t8 < 4; ++t8) g4[t8] = __ldg(gp + (c >> 3) + t8);
          }
#pragma unroll
          for (int t8 = 0; t8 < 4; ++t8) {
            const uint4 u4 = g4[t8];
            const uint32_t ww[4] = {u4.x, u4.y, u4.z, u4.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              float g0 = bf16_lo(ww[t]), g1 = bf16_hi(ww[t]);
              if (p.gate_mode == GATE_SIGMOID) {           // sigma(g) = (1 + tanh(g/2)) / 2: one MUFU op
                g0 = fmaf(0.5f, tanh_approx(0.5f * g0), 0.5f);
                g1 = fmaf(0.5f, tanh_approx(0.5f * g1), 0.5f);
              }
              f[t8 * 8 + 2 * t] *= g0;
              f[t8 * 8 + 2 * t + 1] *= g1;
            }
          }
        }
        if (row_valid) {
          uint4* op = reinterpret_cast<uint4*>(static_cast<unsigned short*>(p.o) + obase + c);
#pragma unroll
          for (int t8 = 0; t8 < 4; ++t8)
            op[t8] = make_uint4(pack_bf16(f[t8 * 8 + 0], f[t8 * 8 + 1]), pack_bf16(f[t8 * 8 + 2], f[t8 * 8 + 3]),
                                pack_bf16(f[t8 * 8 + 4], f[t8 * 8 + 5]), pack_bf16(f[t8 * 8 + 6], f[t8 * 8 + 7]));
        }
      }
      if (p.lse && row_valid)
        p.lse[w.b * p.lses.b + gw * p.lses.g + (int64_t)w.h * p.lses.h + (int64_t)q * p.lses.s] =
            empty_row ? -INFINITY : (m_ref + __log2f(l)) * kLn2;
      if (DIFF) mbar_arrive(q_empty);                 // WG0 is done reading xbuf (sQ)
      if (LIST) named_bar_arrive(5, 256);             // WG0 is done reading O1 and (m, l)
    }
    FL_T(10);                                        // 10: epilogue
    }  // unit loop
    if (LIST && o_lent) named_bar_sync(5, 256);
    if (wg == 0 && pp_started) named_bar_sync(2, 256);   // matches WG1's arrive after its last common tile
#ifdef FL_TIMING
    FL_T(8);
    if (r == 0) {
      for (int i = 0; i < 13; ++i) atomicAdd(&g_fl_timing[wg][i], (unsigned long long)t_acc[i]);
      atomicAdd(&g_fl_timing[wg][15], (unsigned long long)s_cnt);
    }
#endif
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 9) tmem_dealloc<512>(tmem);
}

// Schedule / tile-classifier dump (fl_debug_schedule): for every (unit, warpgroup) the
// work decode_work gives it and, per KV tile, whether the softmax warpgroup runs it (needs) and which of
// its four warps apply the element-wise mask (tile_inside false for some row) -- the same functions the
// kernel calls.  Record: [u, wg, b, g, h, q0, lo, hi] + max_tiles codes (-1 = not run, else warp bits).
template <bool DIFF, bool PAIR>
__global__ void sched_dump_kernel(const __grid_constant__ AttnParams p, int n_units, int max_tiles, int32_t* out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_units * 2) return;
  const int u = t >> 1, wg = t & 1;
  const Work w = decode_work<128, DIFF, false, PAIR>(p, u);
  int32_t* rec = out + (int64_t)t * (8 + max_tiles);
  const int q0 = wg ? w.q0[1] : w.q0[0];
  rec[0] = u;
  rec[1] = wg;
  rec[2] = w.b;
  rec[3] = wg ? w.g1 : w.g;
  rec[4] = w.h;
  rec[5] = q0;
  rec[6] = wg ? w.lo[1] : w.lo[0];
  rec[7] = wg ? w.hi[1] : w.hi[0];
  for (int j = 0; j < max_tiles; ++j) {
    int code = -1;
    if (j >= w.lo_cta && j < w.hi_cta && needs(w, wg, j)) {
      code = 0;
      for (int r = 0; r < 128; ++r)
        if (!tile_inside(row_interval(p, w.b, q0 + r), j * 128, p.Sk)) code |= 1 << (r >> 5);
    }
    rec[8 + j] = code;
  }
}

// Small-head pairing (Evoformer rows: S_q leaves half of a 256-row unit empty) and the resident pair bias
// (bf16, key-contiguous, broadcast over G, S_k within the free TMEM columns, raw-score domain).
static inline bool small_head_pair(const AttnParams& p) {
  return p.Dqk == 32 && p.maps == 1 && p.mask != MASK_BLOCKLIST && p.G >= 2 && p.Sq % 256 != 0 && p.Sq % 256 <= 128;
}
static inline bool bias_resident(const AttnParams& p) {
  return p.bias && p.bias_vec && p.bs.g == 0 && p.Sk <= TcCfg<32, false>::BR_KEYS && p.mod == MOD_NONE;
}

static inline int num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

template <int D, bool DIFF, int MOD>
static cudaError_t launch_one(const AttnParams& p, const TmaMaps& maps, cudaStream_t stream) {
  // RSA block lists (FL_MASK_BLOCKLIST) get their own instantiation (no bias, no diff: host.cu) so the
  // interval-mask kernels keep the schedule arithmetic out of their softmax loop.
  auto kern = p.mask == MASK_BLOCKLIST ? attn_tc_kernel<D, false, MOD, false, true>
              : p.bias                 ? attn_tc_kernel<D, DIFF, MOD, true, false>
                                       : attn_tc_kernel<D, DIFF, MOD, false, false>;
  const bool list = p.mask == MASK_BLOCKLIST;
  // small heads whose S_q leaves half of the last 256-row unit empty (Evoformer rows): pair G entries
  bool pair = false;
  AttnParams pp = p;
  if constexpr (D == 32 && !DIFF) {
    if (small_head_pair(p)) {
      pair = true;
      kern = p.bias ? attn_tc_kernel<D, false, MOD, true, false, 1> : attn_tc_kernel<D, false, MOD, false, false, 1>;
      if constexpr (MOD == MOD_NONE) {
        if (bias_resident(p)) {
          pp.unit_order = 1;
          kern = attn_tc_kernel<D, false, MOD, true, false, 2>;
        }
      }
    }
  }
  const int smem_bytes = (kAlibiMma && MOD == MOD_ALIBI) ? (list ? TcCfg<D, false, true>::SMEM_TOTAL_AUG
                                                                  : TcCfg<D, DIFF>::SMEM_TOTAL_AUG)
                       : list ? TcCfg<D, false, true>::SMEM_TOTAL
#ifdef FL_BIG
                       : D == 32 ? std::max(TcCfg<D, DIFF>::SMEM_TOTAL, TcCfg<D, DIFF, false, true>::SMEM_TOTAL)
#endif
                                 : TcCfg<D, DIFF>::SMEM_TOTAL;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  if (e != cudaSuccess) return e;
  const int rows_per_unit = (DIFF || list || pair) ? 128 : 256;
  const long long units = (long long)p.B * (pair ? (p.G + 1) / 2 : p.G) * p.Hq * ((p.Sq + rows_per_unit - 1) / rows_per_unit);
  if (units >= (1ll << 31)) return cudaErrorInvalidValue;
  // persistent: one CTA per SM (TMEM and shared memory admit one), each walks units with stride grid
  int grid = (int)std::min<long long>(units, num_sms());
  if (pp.unit_order == 1) {                          // static chunks: cps CTAs per (b, h, q-block) segment
    const int n_seg = (int)(units / ((p.G + 1) / 2));
    grid = n_seg <= num_sms() ? n_seg * (num_sms() / n_seg) : num_sms();
  }
  kern<<<grid, kThreadsTc, smem_bytes, stream>>>(pp, maps, (int)units);
  return cudaGetLastError();
}

template <int D, bool DIFF>
static cudaError_t launch_mod(const AttnParams& p, const TmaMaps& maps, cudaStream_t stream) {
  switch (p.mod) {
    case MOD_ALIBI: return launch_one<D, DIFF, MOD_ALIBI>(p, maps, stream);
    case MOD_SOFTCAP: return launch_one<D, DIFF, MOD_SOFTCAP>(p, maps, stream);
    default: return launch_one<D, DIFF, MOD_NONE>(p, maps, stream);
  }
}

// debug_timing of the FL_TIMING build: the counters of the translation unit that instantiates it
template <int Dummy>
static cudaError_t debug_timing_tu(unsigned long long* out, int reset) {
#ifdef FL_TIMING
  cudaError_t e = cudaMemcpyFromSymbol(out, g_fl_timing, sizeof(g_fl_timing));
  if (e == cudaSuccess && reset) {
    unsigned long long z[3][16] = {};
    e = cudaMemcpyToSymbol(g_fl_timing, z, sizeof(z));
  }
  return e;
#else
  (void)out;
  (void)reset;
  return cudaErrorNotSupported;
#endif
}

}  // namespace fl
