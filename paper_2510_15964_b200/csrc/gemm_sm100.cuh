// Persistent grouped gather-GEMM on sm_100a: TMA -> smem (SWIZZLE_128B) ->
// tcgen05.mma (fp32 accumulators in TMEM, double-buffered) -> fused epilogue.
//
//   C[rows of item b, :] = A[rows of item b, :K_b] * B_b^T
//
// B operand modes (the neuron-sparse MLP of sf/neuron_ops.py:75-95):
//   kDense   : B is K-major [N, K] (row n contiguous along K).
//   kDenseMN : B is MN-major [K, N] (the torch.addmm weight layout), loaded as 64-column atoms.
//   kNGather : B is K-major [d_ff, K]; the item's packed N columns are its
//              active neuron blocks (ids[b][*]), each a contiguous run of `blk`
//              rows of W1^T (fc1) or W2 (fc2 input-grad). One TMA box per block.
//   kKGather : B is MN-major [d_ff, N]; the item's packed K rows are its active
//              neuron blocks, each `blk` contiguous rows of W2 (fc2) or W1^T
//              (fc1 input-grad). A is the packed hidden [M, ld] (K = count*blk).
//
// Warp roles: w0 = TMA producer, w1 = MMA issuer (lane 0), w2..w9 = epilogue
// (one accumulator row per thread, half of the tile's columns per warp). Grid = #SMs; tiles strided over CTAs, with
// the M tile fastest so co-resident CTAs share the same weight (B) tile in L2.
//
// CTAS = 2 (dense and item-packed modes): a cluster pair owns a 256 x BN tile and issues
// tcgen05.mma.cta_group::2 (M = 256) from the even CTA. Each CTA loads its 128 rows of A and its
// half of B (BN/2 rows, or BN/2 columns for the MN-major K-side), so a stage is 32 KB instead of
// 48 KB (6 stages) and L2 -> SM traffic per FLOP drops by 1.5x. Both CTAs' TMA count bytes on the
// leader's full barrier; the MMA commits multicast to both CTAs' empty / accumulator barriers;
// both CTAs' epilogue warps release the leader's accumulator barrier. Each CTA's TMEM holds its
// 128 rows x BN columns, so the epilogue is the 1-CTA one.
//
// Wide pairs (CTAS = 2, BN = 512): a 256 x w tile (w <= 512) as two cta_group::2 MMAs per K step into one
// 512-column accumulator. Per SM and K stage: 48 KB in, 8.4 MFLOP, which keeps the mainloop at the tcgen05
// floor (~1040 cycles per 64-deep stage measured, tools/dense_trace.py) where the 128 x 256 single-CTA tile
// (48 KB per 4.2 MFLOP) and the 256 x 256 pair run at ~70% of it. The epilogue is not overlapped (no second
// accumulator), so it is kept to convert + store when there is no bias / LoRA term.
// CL = 2 (two pairs per cluster sharing the B tile, multicast): measured no faster than pairs and the
// 4-CTA clusters only fit 132 SMs; kept for tests / experiments (lx_gemm_set_cta_pair(4)).
#pragma once
#include "ptx.cuh"

namespace lx {

// kPackedN / kPackedK: the same two gathers, but over an item-packed copy of the active rows
// ([n_items, packed_stride, K|N], built once per layer by lx_pack_active_rows): one 256-row box
// (N side) or four 64x64 boxes (K side) per stage instead of one 2 KB box per neuron block.
// kDenseDual: K-major B holding a bf16 hi/lo pair [W_hi | W_lo] (the lo half at K offset args.dual_k): each stage
// loads A once and B's hi and lo boxes, and issues two MMAs into one accumulator (A W_hi + A W_lo), so the
// float32-faithful predictor GEMMs read A once instead of once per term. CTA pairs, N tile = BN / 2.
enum BMode : int { kDense = 0, kNGather = 1, kKGather = 2, kPackedN = 3, kPackedK = 4, kDenseMN = 5, kDenseDual = 6 };
template <int BMODE>
LX_DEV constexpr bool is_ng() { return BMODE == kNGather || BMODE == kPackedN; }
template <int BMODE>
LX_DEV constexpr bool is_kg() { return BMODE == kKGather || BMODE == kPackedK; }
template <int BMODE>
LX_DEV constexpr bool is_dense() { return BMODE == kDense || BMODE == kDenseMN || BMODE == kDenseDual; }  // no counts
template <int BMODE>
LX_DEV constexpr bool b_mn() { return is_kg<BMODE>() || BMODE == kDenseMN; }  // B is MN-major [K, N] (64-col atoms)
enum EpiKind : int {
  kEpiStoreF32 = 0,   // C (fp32)
  kEpiStoreBF16 = 1,  // C (bf16)
  kEpiFc1 = 2,        // relu(acc + b1[c] + s*ax1[row]·B1[:,c])  -> bf16 packed hidden
  kEpiFc2 = 3,        // acc + b2[c] + s*ax2[row]·B2[:,c]        -> bf16
  kEpiDa = 4,         // (acc + dax2[row]·A2[c,:]) * (a[row,j] > 0) -> bf16 packed dz
  kEpiDx = 5,         // acc + dax1[row]·A1[c,:]                  -> bf16
  kEpiMask = 6,       // OR_rows(acc > thr) per column -> bitmask words (+ optional fp32 dump)
  kEpiFc1Raw = 7,     // acc + b1[c] + s*ax1[row]·B1[:,c] (no ReLU)  -> bf16 packed (neuron_matmul_fwd1 API)
  kEpiCe = 8,         // LM-head logits l: per (row, BN/2-column segment) m = max l and z = sum exp(l - m) -> ce_stats,
                      // bf16 exp(l - m) -> out, the target's fp32 logit -> ce_tl (no fp32 logits are stored)
};

// Debug-only phase trace (lx_debug_set_gemm_trace): per CTA 32 clock64 stamps, NULL in production.
__device__ unsigned long long* g_gemm_trace = nullptr;
LX_DEV void gemm_stamp(int slot) {
  unsigned long long* t = g_gemm_trace;
  if (t != nullptr) {
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    t[blockIdx.x * 32 + slot] = c;
  }
}

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 bf16 = 128 B = one SWIZZLE_128B row
// epilogue: 8 warps = the 4 TMEM lane groups twice; warps 2..5 take columns [0, BN/2) of their rows,
// warps 6..9 columns [BN/2, BN) (two warps per SM sub-partition hide each other's latency)
constexpr int kEpiWarps = 8;
constexpr int kGemmThreads = 64 + 32 * kEpiWarps;
constexpr int kMaxR = 16;
constexpr int kMaxItems = 512;

struct GemmArgs {
  // problem
  int n_items;        // groups (sequences)
  int rows_per_item;  // tokens per item
  int n_dense;        // N for kDense / kKGather
  int k_dense;        // K for kDense / kNGather
  const int* counts;  // [n_items] active blocks per item (gather modes)
  const int* ids;     // [n_items, ids_stride] ascending active block ids
  int ids_stride;
  int blk;            // neuron block size (multiple of 16)
  // epilogue
  void* out;
  int ldo;
  const float* bias;      // indexed by original column
  const float* lora_x;    // [M, r] fp32 (row factor)
  const float* lora_w;    // column factor: w(r, c) = lora_w[r*w_sr + c*w_sc]
  long long w_sr, w_sc;
  int lora_r;
  float lora_scale;
  const __nv_bfloat16* act;  // kEpiDa: packed relu output a (same layout as out)
  int ld_act;
  float thr;            // kEpiMask
  uint32_t* bits;       // kEpiMask: [n_items, bits_slots, bits_stride] words: slot t = rows [32t, 32t + 32) of the item
  int bits_stride;
  int bits_slots;       // ceil(rows_per_item / 32); every (slot, word) is stored exactly once (no atomics, no memset)
  const int64_t* ce_tgt;  // kEpiCe: target id per row
  float2* ce_stats;       // kEpiCe: [rows, ce_nseg] (segment max, sum of exp(l - max)), segments of BN/2 columns
  float* ce_tl;           // kEpiCe: [rows] fp32 logit of the target
  int ce_nseg;
  int out_f32;          // store fp32 instead of bf16 (any epilogue except kEpiMask)
  const float* resid;   // fp32 [rows, ldo]: out = resid + value (fused residual add; requires out_f32)
  int packed_stride;    // kPacked*: rows per item in the packed weight copy
  int spin;             // producer / MMA issuer poll (test_wait) instead of try_wait (set by the launcher)
  int a_k_split;        // kDense: A's K coordinate is k - a_k_split for k >= a_k_split (0: off). With B =
                        // [W_hi | W_lo] (segments a_k_split wide) one GEMM computes A W_hi + A W_lo.
  int dual_k;           // kDenseDual: K coordinate of W_lo in B (k_dense = the K extent of A and of each half)
  uint16_t* relu_bits;  // kEpiFc1 writes / kEpiDa reads relu'(z) = (bf16 a > 0) as bits: row-major [rows][ld_bits]
  int ld_bits;          // uint16 words per row (16 columns each; tiles start at multiples of 16 columns)
};

constexpr int kStgPitch = 80;  // bytes per staged row: 64 B of bf16 + 16 B pad (conflict-free 16 B writes)

// LEAN (the dual predictor GEMMs: no bias / LoRA columns to stage): one more pipeline stage in place of the
// LoRA column-factor area, i.e. more bytes in flight per SM for the HBM-streamed weights
template <int BN, int CTAS = 1, bool LEAN = false>
struct GemmSmem {
  static constexpr int kStages = (CTAS == 2 ? (BN > 256 ? 3 : BN >= 256 ? 5 : 7) : (BN >= 256 ? 3 : 5)) + (LEAN ? 1 : 0);
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = (BN / CTAS) * kBK * 2;  // this CTA's share of the B tile
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kBarOff = kStages * kStageBytes;
  // wide pair tiles re-cut the same ring into more, smaller stages when the launch's tile width is below BN
  static constexpr int kMaxStg = (CTAS == 2 && BN > 256) ? 8 : kStages;
  static constexpr int kMiscOff = kBarOff + (2 * kMaxStg + 4) * 8;
  static constexpr int kEpiOff = (kMiscOff + 16 + 4 * (kMaxItems + 2) + 127) / 128 * 128;  // + prefix, tile width
  static constexpr int kEpiBytes = BN * 4 + (LEAN ? 0 : BN * kMaxR * 4);
  static constexpr int kStgOff = kEpiOff + kEpiBytes;  // per epilogue warp: 32 rows x kStgPitch
  static constexpr int kTotal = kStgOff + kEpiWarps * 32 * kStgPitch + 1024;  // + alignment slack
};

template <int BMODE, int BN, int CTAS>
using GemmSmemFor = GemmSmem<BN, CTAS, BMODE == kDenseDual>;

struct TileInfo {
  int item, mt, nt;
  int n0;        // first packed/dense column of this tile
  int n_cols;    // valid packed/dense columns in this tile
  int k_stages;  // K pipeline stages
  int k_total;   // K extent (elements)
};

// Wide pair tiles (CTAS = 2, BN = 512, N-side gathers): one accumulator of up to 512 columns per CTA, tile width
// w (a multiple of 64, chosen per launch on the device from the counts: the narrowest w whose tiles fit in one
// round of CTA pairs), computed as two cta_group::2 MMAs (N = min(w, 256), then the rest).
template <int BMODE, int BN>
LX_DEV int item_n_tiles(const GemmArgs& a, int cnt, int wsel = 0) {
  if (is_ng<BMODE>()) {
    const int w = wsel ? wsel : BN;
    return (cnt * a.blk + w - 1) / w;
  }
  const int w = wsel ? wsel : (BMODE == kDenseDual ? BN / 2 : BN);
  return (a.n_dense + w - 1) / w;
}

template <int BMODE, int BN>
LX_DEV TileInfo decode_tile(const GemmArgs& a, const int* prefix, const int* cnts, int m_tiles, int t, int wsel = 0) {
  // m_tiles counts tiles of kBM * CTAS rows (the caller's choice)
  int lo = 0, hi = a.n_items;  // largest item with prefix[item] <= t
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (prefix[mid] <= t) lo = mid; else hi = mid;
  }
  TileInfo ti;
  ti.item = lo;
  int local = t - prefix[lo];
  ti.mt = local % m_tiles;
  ti.nt = local / m_tiles;
  int cnt = is_dense<BMODE>() ? 0 : __ldg(cnts + lo);
  int n_total = is_ng<BMODE>() ? cnt * a.blk : a.n_dense;
  // an item's active columns are split into equal-width tiles (multiples of 16, <= BN): no short last
  // tile whose CTA idles while the full ones finish
  int w = BMODE == kDenseDual ? BN / 2 : BN;
  if (wsel) {
    w = wsel;  // wide pair tiles: uniform width chosen for the launch
  } else if (is_ng<BMODE>()) {
    const int nt_item = (n_total + BN - 1) / BN;
    const int q = a.blk > 16 ? a.blk : 16;  // whole neuron blocks (gather boxes are per block)
    if (nt_item > 0) w = min(BN, ((n_total + nt_item - 1) / nt_item + q - 1) / q * q);
  }
  ti.n0 = ti.nt * w;
  ti.n_cols = min(w, n_total - ti.n0);
  ti.k_total = is_kg<BMODE>() ? cnt * a.blk : a.k_dense;
  ti.k_stages = (ti.k_total + kBK - 1) / kBK;
  return ti;
}

template <int BMODE, int EPI, int BN, int CTAS = 1, int CL = 1>
__global__ void __launch_bounds__(kGemmThreads, 1)
gemm_sm100_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b, GemmArgs args) {
  static_assert(CTAS == 1 || (is_dense<BMODE>() || BMODE == kPackedN || BMODE == kPackedK), "CTA pairs: dense / packed B only");
  static_assert(BMODE != kDenseMN || CTAS == 1 || BN > 256, "MN-major dense B: single CTA or wide pairs");
  using L = GemmSmemFor<BMODE, BN, CTAS>;
  constexpr bool kWide = BN > 256;  // wide pair tiles (CTAS == 2, N-side gathers)
  static_assert(!kWide || (CTAS == 2 && (is_dense<BMODE>() || BMODE == kPackedN || BMODE == kPackedK)),
                "wide tiles: CTA pairs, dense / packed B only");
  // wide-tile width granularity: whole 32-row boxes per CTA half (N side), whole 64-column atoms (K side)
  constexpr int kWq = b_mn<BMODE>() ? 128 : 64;
  constexpr int kAccBufs = 2 * BN <= 512 ? 2 : 1;  // TMEM accumulators (double-buffered when two fit)
  static_assert(CL == 1 || (CTAS == 2 && !kWide), "pair clusters: CTA pairs, 256-column tiles");
  constexpr int TM = kBM * CTAS;  // rows per (pair) tile
  // CL = 2: a cluster of two CTA pairs takes two adjacent row tiles of the same B tile; each CTA loads half of
  // its B half and multicasts it to the matching CTA of the other pair (half the L2 -> SM bytes for B)
  constexpr int TMc = TM * CL;  // rows per cluster tile
  constexpr int kCluster = CTAS * CL;
  const bool kSpin = args.spin != 0;  // producer / MMA issuer poll their barriers instead of try_wait
  constexpr int BNC = BN / CTAS;  // this CTA's share of the N tile
  constexpr int S0 = L::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* empty = full + L::kMaxStg;
  uint64_t* tfull = empty + L::kMaxStg;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kMiscOff);
  int* prefix = reinterpret_cast<int*>(smem + L::kMiscOff + 16);
  int* wsel_s = prefix + kMaxItems + 1;
  float* s_bias = reinterpret_cast<float*>(smem + L::kEpiOff);
  float* s_w = s_bias + BN;

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = CTAS == 2 ? cluster_ctarank() : 0;  // rank * kBM: this CTA's rows in the cluster tile
  const uint32_t prank = rank & 1, pidx = rank >> 1;       // rank in the pair, pair in the cluster
  const bool leader = prank == 0;
  const int m_tiles = (args.rows_per_item + TMc - 1) / TMc;
  const int t0 = blockIdx.x / kCluster, t_step = gridDim.x / kCluster;

  if (warp == 0 && lane == 0) {
    gemm_stamp(0);
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    for (int i = 0; i < L::kMaxStg; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, CL); }
    for (int i = 0; i < 2; ++i) { mbar_init(tfull + i, 1); mbar_init(tempty + i, kEpiWarps * CTAS); }
    fence_mbar_init();
  }
  if (warp == 2) {
    if (CTAS == 2) tmem_alloc_cg2<512>(tmem_slot);
    else tmem_alloc<512>(tmem_slot);
  }
  // pairs: arrive on the cluster barrier now (barrier inits released), wait once the tile table is built, so
  // the peer handshake overlaps the PDL wait and the prologue instead of following it
  if (CTAS == 2) cluster_arrive();
  // prologue above overlaps the predecessor kernel's tail (programmatic dependent launch)
  pdl_wait_trigger();
  if (threadIdx.x == 0) gemm_stamp(14);
  // ---- tile table: prefix[b] = first tile index of item b (counts are device-resident)
  // counts -> shared memory in one parallel round trip (the epilogue's staging area is free until the first tile)
  int* s_cnt = reinterpret_cast<int*>(smem + L::kEpiOff);
  if (!is_dense<BMODE>())
    for (int b = threadIdx.x; b < args.n_items; b += blockDim.x) s_cnt[b] = __ldg(args.counts + b);
  __syncthreads();
  if (threadIdx.x == 0) gemm_stamp(15);
  if (warp == 0) {
    // warp-parallel: lane L tests the width (L + 1) * kWq, then a warp scan builds the item prefix
    int wsel = (kWide && EPI == kEpiCe) ? BN : 0;  // CE segments are BN / 2 columns: full-width tiles
    if (kWide && EPI != kEpiCe) {  // narrowest multiple-of-64 width whose tiles fit in one round of pairs (else the widest)
      const int pairs = gridDim.x / kCluster;
      const int w_l = ((int)lane + 1) * kWq;
      bool fits = false;
      if (w_l < BN) {
        int tot = 0;
        for (int b = 0; b < args.n_items; ++b) tot += m_tiles * item_n_tiles<BMODE, BN>(args, s_cnt[b], w_l);
        fits = tot <= pairs;
      }
      const uint32_t fit_mask = __ballot_sync(0xffffffffu, fits);
      wsel = fit_mask ? (__ffs(fit_mask)) * kWq : BN;
    }
    if (lane == 0) *wsel_s = wsel;
    int carry = 0;
    for (int b0 = 0; b0 < args.n_items; b0 += 32) {
      const int b = b0 + (int)lane;
      const int cnt = (b < args.n_items && !is_dense<BMODE>()) ? s_cnt[b] : 0;
      const int nt = b < args.n_items ? m_tiles * item_n_tiles<BMODE, BN>(args, cnt, wsel) : 0;
      int inc = nt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if ((int)lane >= o) inc += t;
      }
      if (b < args.n_items) prefix[b] = carry + inc - nt;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) prefix[args.n_items] = carry;
  }
  if (threadIdx.x == 0) gemm_stamp(16);
  tc_fence_before();
  __syncthreads();
  if (CTAS == 2) cluster_wait();  // both CTAs' barriers initialised before any cross-CTA signal
  tc_fence_after();
  if (threadIdx.x == 0) gemm_stamp(17);
  const uint32_t tmem_base = *tmem_slot;
  const int n_tiles_total = prefix[args.n_items];
  const int wsel = *wsel_s;
  // pipeline ring: wide pairs hold A (16 KB) + this CTA's half of a wsel-wide B tile (64 B per column) per stage,
  // so a narrower launch width gives more stages in flight over the same shared memory (latency-bound mainloop)
  const int stage_bytes = (kWide && wsel) ? L::kABytes + 64 * wsel : L::kStageBytes;
  const int S = kWide ? min(L::kMaxStg, (S0 * L::kStageBytes) / stage_bytes) : S0;

  // counts are needed by every role to decode tiles; read through L1 per decode.
  const int* cnts = args.counts;

  if (warp == 0) {
    // ================= TMA producer (whole warp: gather boxes are issued one per lane, in parallel;
    // each lane holds its neuron-block id in a register for the whole tile / stage)
    const uint64_t pol_w = policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    for (int t = t0; t < n_tiles_total; t += t_step) {
      TileInfo ti = decode_tile<BMODE, BN>(args, prefix, cnts, m_tiles, t, wsel);
      const int row0 = ti.item * args.rows_per_item + ti.mt * TMc + rank * kBM;
      const int* ids = args.ids + (size_t)ti.item * args.ids_stride;
      int my_row = 0;  // kNGather: this lane's gathered W row (block id * blk), lane < nb
      int nb_n = 0;
      if (BMODE == kNGather) {
        nb_n = (ti.n_cols + args.blk - 1) / args.blk;
        if ((int)lane < nb_n) my_row = __ldg(ids + ti.n0 / args.blk + lane) * args.blk;
      }
      for (int ks = 0; ks < ti.k_stages; ++ks) {
        uint8_t* sa = smem + stage * stage_bytes;
        uint8_t* sb = sa + L::kABytes;
        int nb_k = 0, my_k_row = 0;
        if (BMODE == kKGather) {
          const int kb0 = ks * kBK / args.blk;
          nb_k = min(kBK / args.blk, ti.k_total / args.blk - kb0);
          const int j = lane / (BN / 64);
          if (j < nb_k) my_k_row = __ldg(ids + kb0 + j) * args.blk;
        }
        if (kSpin) mbar_spin(empty + stage, phase ^ 1);
        else mbar_wait(empty + stage, phase ^ 1);
        if (CTAS == 2) {
          // pair: this CTA's A rows and half of B; bytes of both halves counted on the leader's barrier
          if (kWide) {
            // N split as two cta_group::2 MMAs: n1 = min(w, 256) columns, then n2; each CTA holds n1/2 + n2/2
            // rows of B (rows n0 + rank n1/2 .., then n0 + n1 + rank n2/2 ..), loaded as 32-row boxes
            const int nm = (ti.n_cols + kWq - 1) / kWq * kWq, n1 = nm < 256 ? nm : 256, n2 = nm - n1;
            if (lane == 0) {
              if (leader) mbar_arrive_expect_tx(full + stage, 2 * (L::kABytes + (n1 / 2 + n2 / 2) * 128));
              const int ak =
                  (is_dense<BMODE>() && args.a_k_split && ks * kBK >= args.a_k_split) ? ks * kBK - args.a_k_split : ks * kBK;
              tma_load_2d_cg2(sa, &tmap_a, full + stage, ak, row0, pol_w);
              if (!b_mn<BMODE>()) {  // K-major B (dense, packed N side): 32-row boxes
                const int b0 = ti.item * args.packed_stride + ti.n0;
                for (int r0 = 0; r0 < n1 / 2; r0 += 32)
                  tma_load_2d_cg2(sb + r0 * 128, &tmap_b, full + stage, ks * kBK, b0 + prank * (n1 / 2) + r0, pol_w);
                for (int r0 = 0; r0 < n2 / 2; r0 += 32)
                  tma_load_2d_cg2(sb + 128 * 128 + r0 * 128, &tmap_b, full + stage, ks * kBK, b0 + n1 + prank * (n2 / 2) + r0,
                                  pol_w);
              } else {  // MN-major B ([64 K rows] x 64-column atoms of 8 KB)
                const int k0 = ti.item * args.packed_stride + ks * kBK;
                for (int c0 = 0; c0 < n1 / 2; c0 += 64)
                  tma_load_2d_cg2(sb + c0 / 64 * (kBK * 128), &tmap_b, full + stage, ti.n0 + prank * (n1 / 2) + c0, k0, pol_w);
                for (int c0 = 0; c0 < n2 / 2; c0 += 64)
                  tma_load_2d_cg2(sb + 128 * 128 + c0 / 64 * (kBK * 128), &tmap_b, full + stage, ti.n0 + n1 + prank * (n2 / 2) + c0,
                                  k0, pol_w);
              }
            }
            __syncwarp();
            if (++stage == S) { stage = 0; phase ^= 1; }
            continue;
          }
          if (lane == 0) {
            if (leader) mbar_arrive_expect_tx(full + stage, 2 * (L::kABytes + L::kBBytes));
            const int ak =
                (is_dense<BMODE>() && args.a_k_split && ks * kBK >= args.a_k_split) ? ks * kBK - args.a_k_split : ks * kBK;
            tma_load_2d_cg2(sa, &tmap_a, full + stage, ak, row0, pol_w);
            if (CL == 1) {
              if (BMODE == kDense) tma_load_2d_cg2(sb, &tmap_b, full + stage, ks * kBK, ti.n0 + prank * BNC, pol_w);
              if (BMODE == kDenseDual) {  // this CTA's BNC/2 rows of the N tile, hi then lo
                tma_load_2d_cg2(sb, &tmap_b, full + stage, ks * kBK, ti.n0 + prank * (BNC / 2), pol_w);
                tma_load_2d_cg2(sb + (BNC / 2) * 128, &tmap_b, full + stage, args.dual_k + ks * kBK, ti.n0 + prank * (BNC / 2),
                                pol_w);
              }
              if (BMODE == kPackedN)
                tma_load_2d_cg2(sb, &tmap_b, full + stage, ks * kBK, ti.item * args.packed_stride + ti.n0 + prank * BNC,
                                pol_w);
              if (BMODE == kPackedK)
                for (int a = 0; a < BNC / 64; ++a)
                  tma_load_2d_cg2(sb + a * (kBK * 128), &tmap_b, full + stage, ti.n0 + prank * BNC + a * 64,
                                  ti.item * args.packed_stride + ks * kBK, pol_w);
            } else {
              // quarter of the B tile: rows (K-major) / 64-column atoms (MN-major) [pidx * BNC/2, +BNC/2) of this
              // CTA's half, to this CTA and its counterpart in the other pair
              const uint16_t mc = (uint16_t)((1u << prank) | (1u << (prank + 2)));
              const int nq = ti.n0 + prank * BNC + pidx * (BNC / 2);
              if (BMODE == kDense)
                tma_load_2d_cg2_mc(sb + pidx * (BNC / 2) * 128, &tmap_b, full + stage, ks * kBK, nq, mc, pol_w);
              if (BMODE == kPackedN)
                tma_load_2d_cg2_mc(sb + pidx * (BNC / 2) * 128, &tmap_b, full + stage, ks * kBK,
                                   ti.item * args.packed_stride + nq, mc, pol_w);
              if (BMODE == kPackedK)
                for (int a = 0; a < BNC / 128; ++a)
                  tma_load_2d_cg2_mc(sb + (pidx * (BNC / 128) + a) * (kBK * 128), &tmap_b, full + stage, nq + a * 64,
                                     ti.item * args.packed_stride + ks * kBK, mc, pol_w);
            }
          }
          __syncwarp();
          if (++stage == S) { stage = 0; phase ^= 1; }
          continue;
        }
        if (lane == 0) {
          uint32_t bytes = L::kABytes;
          if (is_dense<BMODE>() || BMODE == kPackedN || BMODE == kPackedK) bytes += BN * kBK * 2;
          else if (BMODE == kNGather) bytes += nb_n * args.blk * kBK * 2;
          else bytes += nb_k * (BN / 64) * args.blk * 128;
          mbar_arrive_expect_tx(full + stage, bytes);
          const int ak = (is_dense<BMODE>() && args.a_k_split && ks * kBK >= args.a_k_split) ? ks * kBK - args.a_k_split : ks * kBK;
          tma_load_2d(sa, &tmap_a, full + stage, ak, row0);
          if (BMODE == kDense) tma_load_2d_hint(sb, &tmap_b, full + stage, ks * kBK, ti.n0, pol_w);
          if (BMODE == kPackedN)  // rows [nt*BN, nt*BN+BN) of this item's packed copy, one box
            tma_load_2d_hint(sb, &tmap_b, full + stage, ks * kBK, ti.item * args.packed_stride + ti.n0, pol_w);
          if (BMODE == kDenseMN)  // 64 K-rows x BN columns: one box per 64-column atom
            for (int a = 0; a < BN / 64; ++a)
              tma_load_2d_hint(sb + a * (kBK * 128), &tmap_b, full + stage, ti.n0 + a * 64, ks * kBK, pol_w);
          if (BMODE == kPackedK)  // 64 packed K-rows x BN columns: one box per 64-column atom
            for (int a = 0; a < BN / 64; ++a)
              tma_load_2d_hint(sb + a * (kBK * 128), &tmap_b, full + stage, ti.n0 + a * 64,
                               ti.item * args.packed_stride + ks * kBK, pol_w);
        }
        if (BMODE == kNGather) {
          if ((int)lane < nb_n)
            tma_load_2d_hint(sb + lane * args.blk * 128, &tmap_b, full + stage, ks * kBK, my_row, pol_w);
        } else if (BMODE == kKGather) {
          const int j = lane / (BN / 64), a = lane % (BN / 64);
          if (j < nb_k)
            tma_load_2d_hint(sb + a * (kBK * 128) + j * args.blk * 128, &tmap_b, full + stage, ti.n0 + a * 64,
                             my_k_row, pol_w);
        }
        __syncwarp();
        if (++stage == S) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer
    if (lane == 0 && leader) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = t0; t < n_tiles_total; t += t_step, ++it) {
        TileInfo ti = decode_tile<BMODE, BN>(args, prefix, cnts, m_tiles, t, wsel);
        const int buf = kAccBufs == 2 ? (it & 1) : 0;
        const uint32_t use_phase = kAccBufs == 2 ? ((it >> 1) & 1) : (it & 1);
        mbar_wait(tempty + buf, use_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * BN;
        // pairs always run the full N (each CTA holds BN/2 of B; columns past n_cols are discarded)
        int n_mma = (is_ng<BMODE>() && CTAS == 1) ? ((ti.n_cols + 15) / 16) * 16 : (BMODE == kDenseDual ? BN / 2 : BN);
        const int nm_w = (ti.n_cols + kWq - 1) / kWq * kWq, n1_w = nm_w < 256 ? nm_w : 256, n2_w = nm_w - n1_w;
        if (kWide) n_mma = n1_w;
        const uint32_t idesc = make_idesc_bf16(TM, n_mma, false, b_mn<BMODE>());
        const uint32_t idesc2 = make_idesc_bf16(TM, n2_w > 0 ? n2_w : 16, false, b_mn<BMODE>());
        for (int ks = 0; ks < ti.k_stages; ++ks) {
          if (kSpin) mbar_spin(full + stage, phase);
          else mbar_wait(full + stage, phase);
          if (ks == 0 && it < 3) gemm_stamp(2 + 4 * it);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * stage_bytes);
          const uint32_t sb = sa + L::kABytes;
          int kk_n = min(kBK, ti.k_total - ks * kBK);
          kk_n = (kk_n + 15) / 16;
          for (int kk = 0; kk < kk_n; ++kk) {
            uint64_t da = make_sdesc(sa + kk * 32, 16, 1024);
            uint64_t db = b_mn<BMODE>() ? make_sdesc(sb + kk * 2048, kBK * 128, 1024) : make_sdesc(sb + kk * 32, 16, 1024);
            if (CTAS == 2) mma_bf16_ss_cg2(d_tmem, da, db, idesc, (ks | kk) != 0);
            else mma_bf16_ss(d_tmem, da, db, idesc, (ks | kk) != 0);
            if (BMODE == kDenseDual)  // + A W_lo: the lo rows follow the hi rows in this CTA's B half
              mma_bf16_ss_cg2(d_tmem, da, make_sdesc(sb + (BNC / 2) * 128 + kk * 32, 16, 1024), idesc, 1);
            if (kWide && n2_w > 0)  // second N part: this CTA's B half at +16 KB of the stage, accumulator columns 256..
              mma_bf16_ss_cg2(d_tmem + 256, da,
                              b_mn<BMODE>() ? make_sdesc(sb + 128 * 128 + kk * 2048, kBK * 128, 1024)
                                             : make_sdesc(sb + 128 * 128 + kk * 32, 16, 1024),
                              idesc2, (ks | kk) != 0);
          }
          if (CTAS == 2) mma_commit_cg2(empty + stage, CL == 2 ? 0xF : 0x3);  // frees the stage in both pairs
          else mma_commit(empty + stage);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        if (it < 3) gemm_stamp(3 + 4 * it);
        if (CTAS == 2) mma_commit_cg2(tfull + buf, (uint16_t)(3u << (2 * pidx)));  // this pair (also with no MMA)
        else if (ti.k_stages > 0) mma_commit(tfull + buf);
        else mbar_arrive(tfull + buf);
      }
    }
  } else {
    // ================= epilogue (warps 2..9): thread <-> accumulator row, half of the columns
    const int quad = warp & 3;
    const int r_in_tile = quad * 32 + lane;
    const int ep_tid = threadIdx.x - 64;
    const int col_half = (warp - 2) / 4;
    uint8_t* stg = smem + L::kStgOff + (warp - 2) * 32 * kStgPitch;
    int it = 0;
    for (int t = t0; t < n_tiles_total; t += t_step, ++it) {
      TileInfo ti = decode_tile<BMODE, BN>(args, prefix, cnts, m_tiles, t, wsel);
      const int buf = kAccBufs == 2 ? (it & 1) : 0;
      const int* ids = args.ids + (size_t)ti.item * args.ids_stride;
      const int local_row = ti.mt * TMc + rank * kBM + r_in_tile;
      const bool row_ok = local_row < args.rows_per_item;
      const size_t grow = (size_t)ti.item * args.rows_per_item + local_row;
      const int r = args.lora_r;
      constexpr bool kLora = EPI == kEpiFc1 || EPI == kEpiFc1Raw || EPI == kEpiFc2 || EPI == kEpiDa || EPI == kEpiDx;

      // stage per-column bias / LoRA column factors for this tile (skipped when there are none: the plain
      // product's epilogue is then convert + store only)
      const int r_even = (r + 1) & ~1;  // the paired FMA below reads factor pairs (q, q + 1)
      const bool cols = kLora && (args.bias != nullptr || (r > 0 && args.lora_w != nullptr));
      if (cols) {
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
        for (int c = ep_tid; c < BN; c += 32 * kEpiWarps) {
          int j = ti.n0 + c;
          int oc = j;
          if (is_ng<BMODE>()) oc = (c < ti.n_cols) ? __ldg(ids + j / args.blk) * args.blk + j % args.blk : 0;
          bool ok = c < ti.n_cols;
          s_bias[c] = (ok && args.bias) ? __ldg(args.bias + oc) : 0.f;
          for (int q = 0; q < r_even; ++q)  // column pairs interleaved: [c/2][q][c&1] for the paired FMA below
            s_w[(c >> 1) * 2 * kMaxR + 2 * q + (c & 1)] =
                (ok && q < r && args.lora_w) ? __ldg(args.lora_w + q * args.w_sr + (long long)oc * args.w_sc) : 0.f;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
      }
      // staged bf16 stores: lane l writes rows 8p + l/4 (p = 0..3) of this warp's 32, 16 B at column 8(l%4)
      __nv_bfloat16* st_row[4];
#pragma unroll
      for (int pss = 0; pss < 4; ++pss) {
        const int lrow = ti.mt * TMc + rank * kBM + quad * 32 + pss * 8 + (lane >> 2);
        st_row[pss] = lrow < args.rows_per_item ? reinterpret_cast<__nv_bfloat16*>(args.out) +
                                                      ((size_t)ti.item * args.rows_per_item + lrow) * args.ldo + 8 * (lane & 3)
                                                : nullptr;
      }
      float xr[kMaxR];
#pragma unroll
      for (int q = 0; q < kMaxR; ++q) xr[q] = 0.f;
      if (kLora && args.lora_x && row_ok) {
#pragma unroll
        for (int q = 0; q < kMaxR; ++q)
          if (q < r) xr[q] = __ldg(args.lora_x + grow * r + q) * args.lora_scale;
      }

      const int n_chunks = (ti.n_cols + 31) / 32;
      constexpr int kHalf = (BMODE == kDenseDual ? BN / 2 : BN) / 64;  // 32-column chunks per column half
      const int ch_lo = col_half * kHalf, ch_hi = min(n_chunks, (col_half + 1) * kHalf);
      // kEpiDa with relu bits: this row's relu'(z) words for every chunk of its column half (2 B per 16 columns),
      // loaded before the accumulator wait, so their latency hides under the tile's mainloop; rb[0] is the
      // current chunk's word (the array shifts down one per chunk)
      constexpr int kRb = EPI == kEpiDa ? kHalf : 1;
      uint32_t rb[kRb];
      const bool use_bits = EPI == kEpiDa && args.relu_bits != nullptr;
#pragma unroll
      for (int k = 0; k < kRb; ++k) {
        rb[k] = 0u;
        const int ch = ch_lo + k;
        if (use_bits && row_ok && ch < ch_hi) {
          const uint16_t* bp = args.relu_bits + grow * args.ld_bits + (ti.n0 + ch * 32) / 16;
          rb[k] = (uint32_t)__ldg(bp) | ((ch * 32 + 16 < ti.n_cols) ? (uint32_t)__ldg(bp + 1) << 16 : 0u);
        }
      }

      // kEpiFc1 relu bits: a full column half of 8 full chunks at a 256-column boundary is collected in registers
      // and written as two 16-byte stores (per-chunk 2-byte stores cost a partial-sector write each)
      constexpr int kBw = (EPI == kEpiFc1 && kHalf == 8) ? 8 : 1;
      uint32_t bw[kBw];
      const bool bits_vec = kBw == 8 && args.relu_bits != nullptr && row_ok && (args.ld_bits % 8) == 0 &&
                            ((ti.n0 + ch_lo * 32) % 256) == 0 && ch_hi - ch_lo == 8 && ch_hi * 32 <= ti.n_cols;

      mbar_wait(tfull + buf, kAccBufs == 2 ? ((it >> 1) & 1) : (it & 1));
      if (ep_tid == 0 && it < 3) gemm_stamp(4 + 4 * it);
      tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(quad * 32) << 16) + buf * BN;
      // software-pipelined: chunk ch + 1's TMEM load is in flight while chunk ch is processed
      uint32_t raw[32];
      // kEpiCe: max of this row's logits over the column half (its segment); exp / sum / store in the chunk loop
      float ce_m = -INFINITY, ce_z = 0.f, ce_tlv = 0.f;
      bool ce_has_t = false;
      long long ce_tcol = -1;
      if (EPI == kEpiCe) {
        if (row_ok) ce_tcol = args.ce_tgt[grow] - ti.n0;
        for (int ch = ch_lo; ch < ch_hi; ++ch) {
          tmem_ld_32x32b_x32(t_row + ch * 32, raw);
          tmem_ld_wait_regs(raw);
          const int nvm = min(32, ti.n_cols - ch * 32);
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i < nvm) ce_m = fmaxf(ce_m, __uint_as_float(raw[i]));
        }
      }
      if (ti.k_stages > 0 && ch_lo < ch_hi) tmem_ld_32x32b_x32(t_row + ch_lo * 32, raw);
      for (int ch = ch_lo; ch < ch_hi; ++ch) {
        float v[32];
        if (ti.k_stages > 0) {
          tmem_ld_wait_regs(raw);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(raw[i]);
          if (ch + 1 < ch_hi) tmem_ld_32x32b_x32(t_row + (ch + 1) * 32, raw);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
        const int c0 = ch * 32;
        const int nv = min(32, ti.n_cols - c0);
        const int j0 = ti.n0 + c0;  // packed / dense column of v[0]
        if (EPI == kEpiCe) {
          const float ml = ce_m * 1.4426950408889634f;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            if (c0 + i == ce_tcol) {
              ce_tlv = v[i];
              ce_has_t = true;
            }
            const float e = i < nv ? ex2(fmaf(v[i], 1.4426950408889634f, -ml)) : 0.f;
            ce_z += e;
            v[i] = e;
          }
        }

        if (EPI == kEpiMask) {
          uint32_t word = 0;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            bool act = row_ok && i < nv && v[i] > args.thr;
            uint32_t bal = __ballot_sync(0xffffffffu, act);
            if (bal) word |= 1u << i;
          }
          // this warp's 32 rows are one slot: a plain store of the word (the compaction ORs the slots)
          const int slot = (ti.mt * TMc + rank * kBM + quad * 32) / 32;
          if (lane == 0 && slot < args.bits_slots)
            args.bits[((size_t)ti.item * args.bits_slots + slot) * args.bits_stride + j0 / 32] = word;
          if (args.out && row_ok) {
            float* o = reinterpret_cast<float*>(args.out) + grow * args.ldo + j0;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i < nv) o[i] = v[i];
          }
          continue;
        }
        if (kLora && cols && r == 0) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += s_bias[c0 + i];
        } else if (kLora && cols) {
          // two columns per fma.rn.f32x2 (FFMA2): same per-column operation order as scalar fmaf, half the issue
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float* w = s_w + (c0 + i) * kMaxR;  // pair (c0+i, c0+i+1), c0 + i even
            float a0 = v[i] + s_bias[c0 + i], a1 = v[i + 1] + s_bias[c0 + i + 1];
#pragma unroll
            for (int q = 0; q < kMaxR; q += 2) {
              if (q < r) {
                float4 wq = *reinterpret_cast<const float4*>(w + 2 * q);  // (q,c) (q,c+1) (q+1,c) (q+1,c+1)
                ffma2(a0, a1, xr[q], xr[q], wq.x, wq.y);
                ffma2(a0, a1, xr[q + 1], xr[q + 1], wq.z, wq.w);
              }
            }
            v[i] = a0;
            v[i + 1] = a1;
          }
        }
        if (EPI == kEpiFc1) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
        }
        // kEpiFc1 relu bits from the packed bf16 words pk[16] of this chunk (see relu_bits in GemmArgs)
        auto relu_bits_store = [&](const uint32_t* pk) {
          if (!(EPI == kEpiFc1 && args.relu_bits != nullptr && row_ok)) return;
          // per bf16 half: a > 0 by one bf16x2 compare (1.0 / 0.0 per half: bit 7 of each half), two bits per pair
          uint32_t m2[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const __nv_bfloat162 gt = __hgt2(*reinterpret_cast<const __nv_bfloat162*>(&pk[i]), __float2bfloat162_rn(0.f));
            const uint32_t g = *reinterpret_cast<const uint32_t*>(&gt);
            m2[i] = ((g >> 7) & 1u) | ((g >> 22) & 2u);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) m2[i] = m2[2 * i] | (m2[2 * i + 1] << 2);
#pragma unroll
          for (int i = 0; i < 4; ++i) m2[i] = m2[2 * i] | (m2[2 * i + 1] << 4);
#pragma unroll
          for (int i = 0; i < 2; ++i) m2[i] = m2[2 * i] | (m2[2 * i + 1] << 8);
          uint32_t word = m2[0] | (m2[1] << 16);
          if (nv < 32) word &= (1u << nv) - 1u;
          if (bits_vec) {  // collected, stored as 32 contiguous bytes after the last chunk
#pragma unroll
            for (int k = 0; k + 1 < kBw; ++k) bw[k] = bw[k + 1];
            bw[kBw - 1] = word;
          } else {
            uint16_t* bp = args.relu_bits + grow * args.ld_bits + j0 / 16;
            bp[0] = (uint16_t)(word & 0xffffu);
            if (nv > 16) bp[1] = (uint16_t)(word >> 16);
          }
        };
        if (EPI == kEpiDa && use_bits) {
          const uint32_t word = rb[0];
#pragma unroll
          for (int k = 0; k + 1 < kRb; ++k) rb[k] = rb[k + 1];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = ((word >> i) & 1u) ? v[i] : 0.f;
        } else if (EPI == kEpiDa) {
          if (row_ok) {
            const __nv_bfloat16* ap = args.act + grow * args.ld_act + j0;
            uint32_t aw[16];
            if (nv == 32) {  // 64 contiguous bytes of this row: four 16B loads
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                uint4 p = *reinterpret_cast<const uint4*>(ap + 8 * i);
                aw[4 * i] = p.x; aw[4 * i + 1] = p.y; aw[4 * i + 2] = p.z; aw[4 * i + 3] = p.w;
              }
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const uint32_t lo = (2 * i < nv) ? __bfloat16_as_ushort(ap[2 * i]) : 0u;
                const uint32_t hi = (2 * i + 1 < nv) ? __bfloat16_as_ushort(ap[2 * i + 1]) : 0u;
                aw[i] = lo | (hi << 16);
              }
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              // relu'(z) = (a > 0): sign bit clear and nonzero magnitude of the bf16 activation
              const uint32_t h = (aw[i >> 1] >> ((i & 1) * 16)) & 0xffffu;
              v[i] = (h != 0u && (h & 0x8000u) == 0u) ? v[i] : 0.f;
            }
          }
        }
        // bf16 full chunks go through the warp's staging rows (all lanes take part); else per-row stores
        const bool stg_ok = !(EPI == kEpiStoreF32 || args.out_f32) && nv == 32 && (args.ldo % 8) == 0 &&
                            (reinterpret_cast<uintptr_t>(args.out) & 15) == 0;
        if (!row_ok && !stg_ok) continue;
        if (EPI == kEpiStoreF32 || args.out_f32) {
          float* o = reinterpret_cast<float*>(args.out) + grow * args.ldo + j0;
          if (args.resid) {
            const float* rp = args.resid + grow * args.ldo + j0;
            if (nv == 32) {
#pragma unroll
              for (int i = 0; i < 32; i += 4) {
                float4 rv = *reinterpret_cast<const float4*>(rp + i);
                v[i] += rv.x; v[i + 1] += rv.y; v[i + 2] += rv.z; v[i + 3] += rv.w;
              }
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (i < nv) v[i] += rp[i];
            }
          }
          if (nv == 32 && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(o + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i < nv) o[i] = v[i];
          }
        } else if (stg_ok) {
          // bf16 chunk through shared memory: this thread's 64 B row segment in, then lane l stores
          // row 8p + l/4, bytes 16(l%4).. : each warp store covers 8 rows x 64 B instead of 32 x 16 B
          uint32_t p[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) p[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
          relu_bits_store(p);
          uint8_t* mine = stg + lane * kStgPitch;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            *reinterpret_cast<uint4*>(mine + 16 * i) = make_uint4(p[4 * i], p[4 * i + 1], p[4 * i + 2], p[4 * i + 3]);
          __syncwarp();
#pragma unroll
          for (int pss = 0; pss < 4; ++pss) {
            if (st_row[pss]) {
              const uint4 val =
                  *reinterpret_cast<const uint4*>(stg + (pss * 8 + (lane >> 2)) * kStgPitch + 16 * (lane & 3));
              *reinterpret_cast<uint4*>(st_row[pss] + j0) = val;
            }
          }
          __syncwarp();
        } else {
          __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(args.out) + grow * args.ldo + j0;
          if (nv == 32 && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
            uint32_t p[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) p[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
            relu_bits_store(p);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              *reinterpret_cast<uint4*>(o + 8 * i) = make_uint4(p[4 * i], p[4 * i + 1], p[4 * i + 2], p[4 * i + 3]);
          } else {
            uint32_t p[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) p[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
            relu_bits_store(p);
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i < nv) o[i] = __float2bfloat16_rn(v[i]);
          }
        }
      }
      if constexpr (kBw == 8) {
        if (bits_vec) {
          uint4* bp = reinterpret_cast<uint4*>(args.relu_bits + grow * args.ld_bits + (ti.n0 + ch_lo * 32) / 16);
          bp[0] = make_uint4(bw[0], bw[1], bw[2], bw[3]);
          bp[1] = make_uint4(bw[4], bw[5], bw[6], bw[7]);
        }
      }
      if (EPI == kEpiCe && row_ok) {
        args.ce_stats[grow * args.ce_nseg + (ti.n0 + col_half * (BN / 2)) / (BN / 2)] = make_float2(ce_m, ce_z);
        if (ce_has_t) args.ce_tl[grow] = ce_tlv;
      }
      // release the accumulator buffer to the MMA warp
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CTAS == 2) mbar_arrive_leader(tempty + buf);
        else mbar_arrive(tempty + buf);
      }
      if (ep_tid == 0 && it < 3) gemm_stamp(5 + 4 * it);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CTAS == 2) cluster_sync();  // the peer's TMEM / barriers stay valid until the leader is done
  if (threadIdx.x == 0) gemm_stamp(1);
  if (warp == 2) {
    tc_fence_after();
    if (CTAS == 2) tmem_dealloc_cg2<512>(tmem_base);
    else tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace lx
