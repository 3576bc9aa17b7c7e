// K3 on tcgen05 — block-sparse flash attention forward for sm_100a
// (sf/block_sparse.py:47-126 fused: SDD -> sparse softmax -> DSD, sf/model.py:343-353).
//
// Forward: one CTA per (128-query tile, head, item) walking the CSR list of its pool pattern
// over 128x128 tiles (64-bit masks of active 16x16 cells); backward: dK/dV per 128-key tile over
// the CSC list, dQ per 128-query tile over the CSR list. Warp roles in every kernel:
//   warp 0      TMA producer (Q/K/V/dO tiles straight from the fused projection output)
//   warp 1      MMA issuer (lane 0)
//   warps 2..5  softmax: thread <-> tile row (TMEM lane); no shuffles, a thread owns its row
// P and dS never touch shared memory: they are written as bf16 into TMEM and consumed as the
// A operand of the next MMA (TS form). Q/K are K-major operands (rows of hd); V, dO, Q, K also
// serve as MN-major B operands (K = rows) of P.V, P^T.dO, dS^T.Q and dS.K from the same tiles.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"

namespace lx {

constexpr int kAT = 128;  // query / key tile edge

// Debug-only phase trace (lx_debug_set_attn_trace): per CTA 32 clock64 stamps, NULL in production.
__device__ unsigned long long* g_attn_trace = nullptr;
LX_DEV void trace_stamp(int slot) {
  unsigned long long* t = g_attn_trace;
  if (t != nullptr) {
    const size_t cta = blockIdx.x + (size_t)gridDim.x * (blockIdx.y + (size_t)gridDim.y * blockIdx.z);
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    t[cta * 32 + slot] = c;
    if (slot == 0) {
      unsigned smid;
      asm("mov.u32 %0, %%smid;" : "=r"(smid));
      t[cta * 32 + 31] = smid;
    }
  }
}

LX_DEV void trace_put(int slot, unsigned long long v) {
  unsigned long long* t = g_attn_trace;
  if (t != nullptr) t[(blockIdx.x + (size_t)gridDim.x * (blockIdx.y + (size_t)gridDim.y * blockIdx.z)) * 32 + slot] = v;
}

// Gathered 128-tile tables (patterns.tables128_from_grids): header [nt, P, s, attn_blk, gu, nsub, per, 0];
// per pattern row_ptr[nt+1] col_ptr[nt+1] csr[nt*nt][10] csc[nt*nt][10]. A CSR entry of query tile i is one
// gathered key tile: nsub = 128 / gu units of gu consecutive keys (entry[2 + k] = unit id of slot k, padding
// repeats the first unit), entry[0..1] the 64-bit mask of active 16x16 cells (bit a*8 + b, a = query cell
// of the tile, b = key cell of the gathered tile). CSC entries gather query units for a key tile the same
// way (a = gathered query cell, b = key cell). Work per tile list is ceil(active units / nsub) MMA tiles.
constexpr int kEntryInts = 10;
struct Tab128 {
  const int32_t *row_ptr, *col_ptr, *csr, *csc;
};
LX_DEV Tab128 tab128(const int32_t* t, int p) {
  const int nt = t[0], per = t[6];
  const int32_t* b = t + 8 + (size_t)p * per;
  Tab128 v;
  v.row_ptr = b;
  v.col_ptr = b + nt + 1;
  v.csr = v.col_ptr + nt + 1;
  v.csc = v.csr + kEntryInts * nt * nt;
  return v;
}
LX_DEV uint64_t ent_mask(const int32_t* e) {
  return ((uint64_t)(uint32_t)__ldg(e + 1) << 32) | (uint32_t)__ldg(e);
}
// one gathered 128-row tile of one 64-column atom: nsub TMA boxes of gu rows (tm's box height is gu)
LX_DEV void tma_load_gather(uint8_t* dst, const CUtensorMap* tm, uint64_t* bar, int col, int row_base, const int32_t* ent,
                            int gu, int nsub) {
  for (int k = 0; k < nsub; ++k) tma_load_2d(dst + k * gu * 128, tm, bar, col, row_base + __ldg(ent + 2 + k) * gu);
}
// token row of row r of a gathered tile
LX_DEV int gathered_row(const int32_t* ent, int r, int gu) { return __ldg(ent + 2 + r / gu) * gu + r % gu; }

LX_DEV void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
LX_DEV void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
LX_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Smem tiles are 128 rows x HD bf16 as [HD/64 atoms][128 rows][128B] (SWIZZLE_128B), used as a
// K-major operand (rows = M/N, K = hd) or as an MN-major B operand (K = rows, N = hd).
LX_DEV uint64_t desc_kmajor(uint32_t base, int kk) {  // K = hd step kk (16 elements)
  return make_sdesc(base + (kk >> 2) * (kAT * 128) + (kk & 3) * 32, 16, 1024);
}
LX_DEV uint64_t desc_mnmajor(uint32_t base, int kk) {  // K = rows step kk (16 rows), N = hd atoms at 16KB
  return make_sdesc(base + kk * 16 * 128, kAT * 128, 1024);
}
__host__ __device__ constexpr int tmem_cols_pow2(int c) { return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512; }

// ============================================================================ forward
// Persistent: grid = min(#units, kCtas x #SMs); CTA c walks units u = c, c + G, ... with
// u = (item * H + h) * nqt + qt, so the CTAs resident at a time cover consecutive (item, head)s
// and share their K/V tiles in L2. TMEM per CTA: S [0,128) | P [128,192) (bf16 pairs) | O.
// Q is double-buffered across units and K/V stream through a 2-stage ring indexed by a running
// entry counter g, so the next unit's Q and first K/V load under the current unit's tail.
// Per entry g (key tile j of the unit's CSR list):
//   MMA      S(g) = Q K_j^T as soon as the softmax has pulled S(g-1) into registers (s_free),
//            then O += P(g-1) V_{j'} once P(g-1) is in TMEM (p_full)
//   softmax  S(g) -> registers, release S; row max; lazy rescale (the running max only moves
//            when it grows by > 2^8, FA4-style, so O is rarely touched); P(g) = 2^(S c - m) as bf16
//            into the P region after PV(g-1) completed (pv_done)
// so S(g+1) runs on the tensor core while the softmax of g runs. A unit's epilogue reads O
// after its last PV and releases it (o_free) before the next unit's first PV overwrites it.
template <int HD>
struct AttnFwdSmem {
  static constexpr int kAtoms = HD / 64;
  static constexpr int kT = kAtoms * kAT * 128;  // one 128 x HD tile
  static constexpr int kOffQ = 0;                // Q[2]
  static constexpr int kOffK = 2 * kT;           // K[2]
  static constexpr int kOffV = 4 * kT;           // V[2]
  static constexpr int kOffRed = 6 * kT;        // softmax pair exchange [2][2][128] max + [2][128] sum
  static constexpr int kOffBar = kOffRed + 768 * 4;
  static constexpr int kTotal = kOffBar + 256 + 1024;
  static constexpr int kCtas = HD == 64 ? 2 : 1;
  static constexpr int kTmem = tmem_cols_pow2(kAT + 64 + HD);
  static constexpr int kThreads = 320;  // TMA warp, MMA warp, 8 softmax warps
};

LX_DEV void decode_unit(int u, int nqt, int H, int& qt, int& h, int& item) {
  qt = u % nqt;
  const int r = u / nqt;
  h = r % H;
  item = r / H;
}

template <int HD>
__global__ void __launch_bounds__(AttnFwdSmem<HD>::kThreads, AttnFwdSmem<HD>::kCtas)
bsattn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_g, int gu, int s,
                     int H, int d_model,
                     const int32_t* __restrict__ pidx, int item_stride, const int32_t* __restrict__ tables,
                     float scale_log2, __nv_bfloat16* __restrict__ o, int ldo, float* __restrict__ lse, int n_units) {
  pdl_wait_trigger();
  using L = AttnFwdSmem<HD>;
  constexpr int A = L::kAtoms;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = align_smem_1024(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::kOffBar);
  uint64_t* q_full = bars + 0;    // [2]
  uint64_t* q_empty = bars + 2;   // [2]
  uint64_t* k_full = bars + 4;    // [2]  K and V have separate barriers: K(g)'s stage is refilled as
  uint64_t* k_empty = bars + 6;   // [2]  soon as S(g) completes, V(g)'s once PV(g) completes
  uint64_t* v_full = bars + 8;    // [2]
  uint64_t* v_empty = bars + 10;  // [2]
  uint64_t* s_full = bars + 12;
  uint64_t* s_free = bars + 13;
  uint64_t* p_full = bars + 14;
  uint64_t* pv_done = bars + 15;
  uint64_t* o_free = bars + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int nqt = (s + kAT - 1) / kAT;

  if (warp == 0 && lane == 0) {
    trace_stamp(0);
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_g);
    for (int i = 0; i < 2; ++i) {
      mbar_init(q_full + i, 1);
      mbar_init(q_empty + i, 1);
      mbar_init(k_full + i, 1);
      mbar_init(k_empty + i, 1);
      mbar_init(v_full + i, 1);
      mbar_init(v_empty + i, 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 8);
    mbar_init(p_full, 8);
    mbar_init(pv_done, 1);
    mbar_init(o_free, 8);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<L::kTmem>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_s = tmem, t_p = tmem + kAT, t_o = tmem + kAT + 64;

  if (warp == 0) {
    if (lane == 0) {
      const int nsub = kAT / gu;
      int g = 0, ul = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        int qt, h, item;
        decode_unit(u, nqt, H, qt, h, item);
        const Tab128 tv = tab128(tables, __ldg(pidx + item * item_stride + h));
        const int e0 = __ldg(tv.row_ptr + qt), n = __ldg(tv.row_ptr + qt + 1) - e0;
        if (n == 0) continue;
        const int row_base = item * s;
        const int qcol = h * HD, kcol = d_model + h * HD, vcol = 2 * d_model + h * HD;
        const int qb = ul & 1;
        mbar_wait(q_empty + qb, ((ul >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(q_full + qb, L::kT);
        for (int a = 0; a < A; ++a)
          tma_load_2d(sm + L::kOffQ + qb * L::kT + a * kAT * 128, &tm_qkv, q_full + qb, qcol + a * 64, row_base + qt * kAT);
        for (int e = 0; e < n; ++e, ++g) {
          const int st = g & 1;
          const int32_t* ent = tv.csr + (size_t)(e0 + e) * kEntryInts;
          uint8_t* sk = sm + L::kOffK + st * L::kT;
          uint8_t* sv = sm + L::kOffV + st * L::kT;
          mbar_wait(k_empty + st, ((g >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(k_full + st, L::kT);
          for (int a = 0; a < A; ++a) tma_load_gather(sk + a * kAT * 128, &tm_g, k_full + st, kcol + a * 64, row_base, ent, gu, nsub);
          mbar_wait(v_empty + st, ((g >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(v_full + st, L::kT);
          for (int a = 0; a < A; ++a) tma_load_gather(sv + a * kAT * 128, &tm_g, v_full + st, vcol + a * 64, row_base, ent, gu, nsub);
        }
        ++ul;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc_s = make_idesc_bf16(kAT, kAT, false, false);  // S = Q K^T
      const uint32_t idesc_o = make_idesc_bf16(kAT, HD, false, true);    // O += P V (V MN-major)
      // deferred PV of the previous entry: (entry index, kv stage, first entry of its unit, unit ordinal)
      int pv_g = -1, pv_st = 0, pv_first = 0, pv_ul = 0;
      auto issue_pv = [&]() {
        if (pv_first && pv_ul >= 1) mbar_wait(o_free, (pv_ul - 1) & 1);  // previous unit's O read out
        mbar_wait(v_full + pv_st, (pv_g >> 1) & 1);
        mbar_wait(p_full, pv_g & 1);
        tc_fence_after();
        const uint32_t sv = smem_u32(sm + L::kOffV + pv_st * L::kT);
        for (int kk = 0; kk < kAT / 16; ++kk)
          mma_bf16_ts(t_o, t_p + kk * 8, desc_mnmajor(sv, kk), idesc_o, !(pv_first && kk == 0));
        mma_commit(pv_done);
        mma_commit(v_empty + pv_st);
      };
      int g = 0, ul = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        int qt, h, item;
        decode_unit(u, nqt, H, qt, h, item);
        const Tab128 tv = tab128(tables, __ldg(pidx + item * item_stride + h));
        const int n = __ldg(tv.row_ptr + qt + 1) - __ldg(tv.row_ptr + qt);
        if (n == 0) continue;
        const int qb = ul & 1;
        const uint32_t sq = smem_u32(sm + L::kOffQ + qb * L::kT);
        mbar_wait(q_full + qb, (ul >> 1) & 1);
        for (int e = 0; e < n; ++e, ++g) {
          const int st = g & 1;
          mbar_wait(k_full + st, (g >> 1) & 1);
          if (g >= 1) mbar_wait(s_free, (g - 1) & 1);  // S(g-1) is in the softmax registers
          tc_fence_after();
          const uint32_t sk = smem_u32(sm + L::kOffK + st * L::kT);
          for (int kk = 0; kk < HD / 16; ++kk) mma_bf16_ss(t_s, desc_kmajor(sq, kk), desc_kmajor(sk, kk), idesc_s, kk != 0);
          mma_commit(s_full);
          mma_commit(k_empty + st);
          if (e == n - 1) mma_commit(q_empty + qb);
          if (pv_g >= 0) issue_pv();
          pv_g = g;
          pv_st = st;
          pv_first = e == 0;
          pv_ul = ul;
        }
        ++ul;
      }
      if (pv_g >= 0) issue_pv();
    }
  } else {
    // 8 softmax warps: warp w owns TMEM lanes 32*(w%4).. (query rows) and S columns [64*half, +64),
    // half = (w-2)/4; the two warps of a row exchange their partial row max through shared memory
    // (pair barrier 1 + quad) so both apply the same max; row sums stay partial until the epilogue.
    const int quad = warp & 3, half = (warp - 2) >> 2;
    const int r = quad * 32 + lane;  // query row within the tile
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    float* red = reinterpret_cast<float*>(sm + L::kOffRed);  // [2 parity][2 half][128]
    const uint32_t bar_id = 1 + quad;
    int g = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      int qt, h, item;
      decode_unit(u, nqt, H, qt, h, item);
      const Tab128 tv = tab128(tables, __ldg(pidx + item * item_stride + h));
      const int e0 = __ldg(tv.row_ptr + qt), n = __ldg(tv.row_ptr + qt + 1) - e0;
      const int row = qt * kAT + r;
      const int row_base = item * s;
      float m = -INFINITY, l = 0.f;  // running max (log2 domain, scaled) and this half's row sum
      for (int e = 0; e < n; ++e, ++g) {
        const int32_t* ent = tv.csr + (size_t)(e0 + e) * kEntryInts;
        const uint32_t lo = (uint32_t)__ldg(ent), hi = (uint32_t)__ldg(ent + 1);
        // 16-key groups 4*half .. 4*half+3 of this row's 16-row group
        const uint32_t mrow = (uint32_t)((((uint64_t)hi << 32) | lo) >> ((r >> 4) * 8 + 4 * half)) & 0xfu;
        const bool full = __all_sync(0xffffffffu, mrow == 0xfu);
        mbar_wait(s_full, g & 1);
        tc_fence_after();
        uint32_t sv[2][32];
        tmem_ld_32x32b_x32(t_s + lane_base + half * 64, sv[0]);
        tmem_ld_32x32b_x32(t_s + lane_base + half * 64 + 32, sv[1]);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_free);
        float mx = -INFINITY;
        if (full) {
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int i = 0; i < 32; ++i) mx = fmaxf(mx, __uint_as_float(sv[c][i]));
        } else {
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if ((mrow >> (c * 2 + (i >> 4))) & 1u) mx = fmaxf(mx, __uint_as_float(sv[c][i]));
        }
        float* rp = red + (g & 1) * 256;
        rp[half * 128 + r] = mx;
        asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
        mx = fmaxf(mx, rp[(half ^ 1) * 128 + r]);
        const float mxs = mx * scale_log2;
        const float m_new = mxs > m + 8.f ? mxs : m;  // lazy: keep the stale max while P <= 2^8
        const float alpha = m_new == m ? 1.f : ex2(m - m_new);
        const float use = m_new == -INFINITY ? 0.f : m_new;
        m = m_new;
        // P region free and O stable: PV(g-1) completed (by now, usually)
        if (g >= 1) mbar_wait(pv_done, (g - 1) & 1);
        tc_fence_after();
        float rs = 0.f;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float p0 = ex2(fmaf(__uint_as_float(sv[c][2 * i]), scale_log2, -use));
            float p1 = ex2(fmaf(__uint_as_float(sv[c][2 * i + 1]), scale_log2, -use));
            if (!full && !((mrow >> (c * 2 + (i >> 3))) & 1u)) p0 = p1 = 0.f;
            rs += p0 + p1;
            pk[i] = pack_bf16x2(p0, p1);
          }
          tmem_st_32x32b_x16(t_p + lane_base + half * 32 + c * 16, pk);
        }
        // O rescale (this warp's half of the O columns), rare with the lazy max
        if (e >= 1 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
          for (int c = 0; c < HD / 64; ++c) {
            uint32_t ov[32];
            const uint32_t ta = t_o + lane_base + half * (HD / 2) + c * 32;
            tmem_ld_32x32b_x32(ta, ov);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
            tmem_st_32x32b_x32(ta, ov);
          }
        }
        l = l * alpha + rs;
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
      }
      if (n == 0) {  // no key tile for this query tile: zero output (never for pool patterns)
        if (row < s) {
          __nv_bfloat16* op = o + ((size_t)row_base + row) * ldo + h * HD + half * (HD / 2);
          for (int c = 0; c < HD / 2; c += 8) *reinterpret_cast<uint4*>(op + c) = make_uint4(0u, 0u, 0u, 0u);
          if (half == 0) lse[((size_t)item * H + h) * s + row] = -INFINITY;
        }
        continue;
      }
      mbar_wait(pv_done, (g - 1) & 1);  // the unit's last PV
      tc_fence_after();
      uint32_t ov[HD / 64][32];
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) tmem_ld_32x32b_x32(t_o + lane_base + half * (HD / 2) + c * 32, ov[c]);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_free);
      // total row sum = both halves' partial sums (same max, same alpha history)
      float* rl = red + 512;
      rl[half * 128 + r] = l;
      asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
      l += rl[(half ^ 1) * 128 + r];
      asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");  // rl reusable by the next unit
      const float inv = l > 0.f ? 1.f / l : 0.f;
      if (row < s) {
        __nv_bfloat16* op = o + ((size_t)row_base + row) * ldo + h * HD + half * (HD / 2);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float f[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) f[k] = __uint_as_float(ov[c][8 * i + k]) * inv;
            *reinterpret_cast<uint4*>(op + c * 32 + 8 * i) = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]),
                                                                        pack_bf16x2(f[4], f[5]), pack_bf16x2(f[6], f[7]));
          }
        }
        if (half == 0) lse[((size_t)item * H + h) * s + row] = (m + __log2f(l)) * 0.6931471805599453f;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<L::kTmem>(tmem);
  }
}

template <int HD>
static int launch_fwd_tc(const uint16_t* qkv, int ld, int n_items, int s, int H, const int32_t* pidx, int item_stride,
                         const int32_t* tables128, int gu, float scale, uint16_t* o, int ldo, float* lse, cudaStream_t st) {
  CUtensorMap tm, tm_g;
  int rc = make_tmap_bf16_2d(&tm, qkv, ld, (uint64_t)n_items * s, ld, 64, kAT);
  if (rc) return rc;
  if ((rc = make_tmap_bf16_2d(&tm_g, qkv, ld, (uint64_t)n_items * s, ld, 64, gu))) return rc;
  constexpr int smem = AttnFwdSmem<HD>::kTotal;
  static cudaError_t attr = cudaFuncSetAttribute(bsattn_fwd_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  LX_CHECK_CUDA(attr);
  const int n_units = ((s + kAT - 1) / kAT) * H * n_items;
  const int grid = n_units < AttnFwdSmem<HD>::kCtas * num_sms() ? n_units : AttnFwdSmem<HD>::kCtas * num_sms();
  launch_k(bsattn_fwd_tc_kernel<HD>, grid, AttnFwdSmem<HD>::kThreads, smem, st, tm, tm_g, gu, s, H, H * HD, pidx, item_stride, tables128,
                                                    scale * 1.4426950408889634f, reinterpret_cast<__nv_bfloat16*>(o), ldo,
                                                    lse, n_units);
  return launch_check("bsattn_fwd_tc");
}

// ============================================================================ backward
// Both kernels keep one 128-column TMEM region R that is reused, in MMA issue order, for
// S (S^T), dP (dP^T) and -- as bf16 A operands in its first 64 columns -- P (P^T) and dS (dS^T).
// P stays in registers (bf16) between the two softmax phases of an entry.
template <int HD>
struct AttnBwdSmem {
  static constexpr int kT = (HD / 64) * kAT * 128;  // 128 rows x HD
  static constexpr int kSt = 2;                     // Q/dO (dkdv) or K/V (dq) ring stages
  // [fixed pair (K|V) or (Q|dO)] [kSt x ring pair] [lse2 [kSt][128]] [delta [kSt][128]] [bars]
  static constexpr int kOffRing = 2 * kT;
  static constexpr int kOffL = kOffRing + 2 * kSt * kT;
  static constexpr int kOffBar = kOffL + 2 * kSt * kAT * 4;
  static constexpr int kTotal = kOffBar + 256 + 1024;
  static constexpr int kCtas = HD == 64 ? 2 : 1;
};

template <int HD>
__global__ void __launch_bounds__(192, AttnBwdSmem<HD>::kCtas)
bsattn_dkdv_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                      const __grid_constant__ CUtensorMap tm_g, const __grid_constant__ CUtensorMap tm_do_g, int gu, int s, int H,
                      int d_model, const int32_t* __restrict__ pidx, int item_stride, const int32_t* __restrict__ tables,
                      float scale, float scale_log2, const float* __restrict__ lse, const float* __restrict__ delta,
                      __nv_bfloat16* __restrict__ dkv, int ld_dkv) {
  pdl_wait_trigger();
  if (threadIdx.x == 0) trace_stamp(0);
  using L = AttnBwdSmem<HD>;
  constexpr int A = HD / 64;
  constexpr int kTmem = tmem_cols_pow2(kAT + 2 * HD);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = align_smem_1024(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::kOffBar);
  uint64_t* kv_full = bars + 0;
  uint64_t* qd_full = bars + 1;   // [2]: TMA (1 arrive + tx) + 32 producer lanes (lse/delta)
  uint64_t* qd_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;
  uint64_t* p_ready = bars + 6;
  uint64_t* dp_full = bars + 7;
  uint64_t* ds_ready = bars + 8;
  uint64_t* done = bars + 9;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);
  float* sL = reinterpret_cast<float*>(sm + L::kOffL);  // [kSt][128] lse * log2(e) (+inf past s)
  float* sD = sL + L::kSt * kAT;                        // [kSt][128] delta

  const int kt = blockIdx.x, h = blockIdx.y, item = blockIdx.z;
  const uint32_t warp = warp_id(), lane = lane_id();
  const Tab128 tv = tab128(tables, __ldg(pidx + item * item_stride + h));
  const int e0 = __ldg(tv.col_ptr + kt), n = __ldg(tv.col_ptr + kt + 1) - e0;
  const int row_base = item * s;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_g);
    tma_prefetch_desc(&tm_do_g);
    mbar_init(kv_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(qd_full + i, 33);
      mbar_init(qd_empty + i, 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_ready, 4);
    mbar_init(dp_full, 1);
    mbar_init(ds_ready, 4);
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<kTmem>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_r = tmem, t_dv = tmem + kAT, t_dk = tmem + kAT + HD;

  if (warp == 0) {
    const float* lse_b = lse + ((size_t)item * H + h) * s;
    const float* del_b = delta + ((size_t)item * H + h) * s;
    const int qcol = h * HD, kcol = d_model + h * HD, vcol = 2 * d_model + h * HD;
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * L::kT);
      for (int a = 0; a < A; ++a) {
        tma_load_2d(sm + a * kAT * 128, &tm_qkv, kv_full, kcol + a * 64, row_base + kt * kAT);
        tma_load_2d(sm + L::kT + a * kAT * 128, &tm_qkv, kv_full, vcol + a * 64, row_base + kt * kAT);
      }
    }
    const int nsub = kAT / gu;
    for (int e = 0; e < n; ++e) {
      const int st = e % L::kSt;
      mbar_wait(qd_empty + st, ((e / L::kSt) & 1) ^ 1);
      const int32_t* ent = tv.csc + (size_t)(e0 + e) * kEntryInts;
      if (lane == 0) {
        uint8_t* sq = sm + L::kOffRing + st * 2 * L::kT;
        mbar_arrive_expect_tx(qd_full + st, 2 * L::kT);
        for (int a = 0; a < A; ++a) {
          tma_load_gather(sq + a * kAT * 128, &tm_g, qd_full + st, qcol + a * 64, row_base, ent, gu, nsub);
          tma_load_gather(sq + L::kT + a * kAT * 128, &tm_do_g, qd_full + st, h * HD + a * 64, row_base, ent, gu, nsub);
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int qi = lane * 4 + k, q = gathered_row(ent, qi, gu);  // gathered query units lie inside the item
        sL[st * kAT + qi] = __ldg(lse_b + q) * 1.4426950408889634f;
        sD[st * kAT + qi] = __ldg(del_b + q);
      }
      mbar_arrive(qd_full + st);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_s = make_idesc_bf16(kAT, kAT, false, false);  // S^T, dP^T: B K-major
      const uint32_t id_g = make_idesc_bf16(kAT, HD, false, true);    // dV, dK: B MN-major
      const uint32_t sk = smem_u32(sm), sv = sk + L::kT;
      mbar_wait(kv_full, 0);
      trace_stamp(1);
      for (int e = 0; e < n; ++e) {
        const int st = e % L::kSt;
        const uint32_t sq = smem_u32(sm + L::kOffRing + st * 2 * L::kT), sdo = sq + L::kT;
        mbar_wait(qd_full + st, (e / L::kSt) & 1);
        if (e < 4) trace_stamp(2 + 6 * e);  // q/dO tile landed, S MMA issued next
        tc_fence_after();
        for (int kk = 0; kk < HD / 16; ++kk) mma_bf16_ss(t_r, desc_kmajor(sk, kk), desc_kmajor(sq, kk), id_s, kk != 0);
        mma_commit(s_full);
        mbar_wait(p_ready, e & 1);
        tc_fence_after();
        for (int kk = 0; kk < kAT / 16; ++kk) mma_bf16_ts(t_dv, t_r + kk * 8, desc_mnmajor(sdo, kk), id_g, (e | kk) != 0);
        for (int kk = 0; kk < HD / 16; ++kk) mma_bf16_ss(t_r, desc_kmajor(sv, kk), desc_kmajor(sdo, kk), id_s, kk != 0);
        mma_commit(dp_full);
        mbar_wait(ds_ready, e & 1);
        tc_fence_after();
        for (int kk = 0; kk < kAT / 16; ++kk) mma_bf16_ts(t_dk, t_r + kk * 8, desc_mnmajor(sq, kk), id_g, (e | kk) != 0);
        mma_commit(qd_empty + st);
      }
      mma_commit(done);
    }
  } else {
    const int quad = warp & 3;
    const int kr = quad * 32 + lane;  // key row within the tile
    const int ep_tid = threadIdx.x - 64;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const int cj = kr >> 4;
    for (int e = 0; e < n; ++e) {
      const int st = e % L::kSt;
      const int32_t* ent = tv.csc + (size_t)(e0 + e) * kEntryInts;
        const uint32_t lo = (uint32_t)__ldg(ent), hi = (uint32_t)__ldg(ent + 1);
      const uint64_t mask = ((uint64_t)hi << 32) | lo;
      const float* l2 = sL + st * kAT;
      const float* dl = sD + st * kAT;
      mbar_wait(qd_full + st, (e / L::kSt) & 1);  // lse / delta staged with the tiles
      mbar_wait(s_full, e & 1);
      if (e < 4 && ep_tid == 0) trace_stamp(3 + 6 * e);  // S in TMEM
      tc_fence_after();
      uint32_t pp[4][16];  // P^T (bf16 pairs) for the whole row, reused by dS^T
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        uint32_t sv_[2][32];
        tmem_ld_32x32b_x32(t_r + lane_base + h2 * 64, sv_[0]);
        tmem_ld_32x32b_x32(t_r + lane_base + h2 * 64 + 32, sv_[1]);
        tmem_ld_wait();
#pragma unroll
        for (int c2 = 0; c2 < 2; ++c2) {
          const int c = h2 * 2 + c2;
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int qi = c * 32 + 2 * u;
            const bool on = (mask >> ((qi >> 4) * 8 + cj)) & 1ull;
            const float p0 = on ? ex2(fmaf(__uint_as_float(sv_[c2][2 * u]), scale_log2, -l2[qi])) : 0.f;
            const float p1 = on ? ex2(fmaf(__uint_as_float(sv_[c2][2 * u + 1]), scale_log2, -l2[qi + 1])) : 0.f;
            pp[c][u] = pack_bf16x2(p0, p1);
          }
          tmem_st_32x32b_x16(t_r + lane_base + c * 16, pp[c]);  // S^T chunk c/2 already consumed
        }
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_ready);
      if (e < 4 && ep_tid == 0) trace_stamp(4 + 6 * e);  // P stored
      mbar_wait(dp_full, e & 1);
      if (e < 4 && ep_tid == 0) trace_stamp(5 + 6 * e);  // dP in TMEM
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t dv_[32], dd[16];
        tmem_ld_32x32b_x32(t_r + lane_base + c * 32, dv_);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int qi = c * 32 + 2 * u;
          const __nv_bfloat162 pb = *reinterpret_cast<const __nv_bfloat162*>(&pp[c][u]);
          dd[u] = pack_bf16x2(__low2float(pb) * (__uint_as_float(dv_[2 * u]) - dl[qi]),
                              __high2float(pb) * (__uint_as_float(dv_[2 * u + 1]) - dl[qi + 1]));
        }
        tmem_st_32x32b_x16(t_r + lane_base + c * 16, dd);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_ready);
      if (e < 4 && ep_tid == 0) trace_stamp(6 + 6 * e);  // dS stored
    }
    mbar_wait(done, 0);
    if (ep_tid == 0) trace_stamp(26);
    tc_fence_after();
    const int key = kt * kAT + kr;
#pragma unroll
    for (int which = 0; which < 2; ++which) {  // 0: dK (scaled), 1: dV
      const uint32_t tcol = which == 0 ? t_dk : t_dv;
      const float mul = which == 0 ? scale : 1.f;
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t ov[32];
        tmem_ld_32x32b_x32(tcol + lane_base + c * 32, ov);
        tmem_ld_wait();
        if (key < s) {  // n == 0: no query tile attends to this key tile -> zero gradient
          __nv_bfloat16* op = dkv + ((size_t)row_base + key) * ld_dkv + (which + 1) * d_model + h * HD + c * 32;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float f[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) f[k] = n > 0 ? __uint_as_float(ov[8 * i + k]) * mul : 0.f;
            *reinterpret_cast<uint4*>(op + 8 * i) = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]),
                                                               pack_bf16x2(f[4], f[5]), pack_bf16x2(f[6], f[7]));
          }
        }
      }
    }
  }
  if (threadIdx.x == 64) trace_stamp(27);
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmem>(tmem);
  }
}

template <int HD>
__global__ void __launch_bounds__(192, AttnBwdSmem<HD>::kCtas)
bsattn_dq_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_g, int gu, int s, int H,
                    int d_model, const int32_t* __restrict__ pidx, int item_stride, const int32_t* __restrict__ tables,
                    float scale, float scale_log2, const float* __restrict__ lse, const float* __restrict__ delta,
                    __nv_bfloat16* __restrict__ dq, int ld_dq, const float* __restrict__ kbar_g) {
  pdl_wait_trigger();
  using L = AttnBwdSmem<HD>;  // [Q | dO] [kSt x (K | V)] [kbar]
  constexpr int A = HD / 64;
  constexpr int kTmem = tmem_cols_pow2(kAT + HD);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = align_smem_1024(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::kOffBar);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;
  uint64_t* p_done = bars + 6;
  uint64_t* dp_full = bars + 7;
  uint64_t* ds_ready = bars + 8;
  uint64_t* done = bars + 9;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);
  float* kbar = reinterpret_cast<float*>(sm + L::kOffL);

  const int qt = blockIdx.x, h = blockIdx.y, item = blockIdx.z;
  const uint32_t warp = warp_id(), lane = lane_id();
  const Tab128 tv = tab128(tables, __ldg(pidx + item * item_stride + h));
  const int e0 = __ldg(tv.row_ptr + qt), n = __ldg(tv.row_ptr + qt + 1) - e0;
  const int row_base = item * s;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_g);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(kv_full + i, 1);
      mbar_init(kv_empty + i, 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_done, 4);
    mbar_init(dp_full, 1);
    mbar_init(ds_ready, 4);
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<kTmem>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_r = tmem, t_dq = tmem + kAT;

  if (warp == 0) {
    if (lane == 0) {
      const int qcol = h * HD, kcol = d_model + h * HD, vcol = 2 * d_model + h * HD;
      mbar_arrive_expect_tx(q_full, 2 * L::kT);
      for (int a = 0; a < A; ++a) {
        tma_load_2d(sm + a * kAT * 128, &tm_qkv, q_full, qcol + a * 64, row_base + qt * kAT);
        tma_load_2d(sm + L::kT + a * kAT * 128, &tm_do, q_full, h * HD + a * 64, row_base + qt * kAT);
      }
      const int nsub = kAT / gu;
      for (int e = 0; e < n; ++e) {
        const int st = e % L::kSt;
        mbar_wait(kv_empty + st, ((e / L::kSt) & 1) ^ 1);
        const int32_t* ent = tv.csr + (size_t)(e0 + e) * kEntryInts;
        uint8_t* skv = sm + L::kOffRing + st * 2 * L::kT;
        mbar_arrive_expect_tx(kv_full + st, 2 * L::kT);
        for (int a = 0; a < A; ++a) {
          tma_load_gather(skv + a * kAT * 128, &tm_g, kv_full + st, kcol + a * 64, row_base, ent, gu, nsub);
          tma_load_gather(skv + L::kT + a * kAT * 128, &tm_g, kv_full + st, vcol + a * 64, row_base, ent, gu, nsub);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_s = make_idesc_bf16(kAT, kAT, false, false);
      const uint32_t id_g = make_idesc_bf16(kAT, HD, false, true);
      const uint32_t sq = smem_u32(sm), sdo = sq + L::kT;
      mbar_wait(q_full, 0);
      for (int e = 0; e < n; ++e) {
        const int st = e % L::kSt;
        const uint32_t sk = smem_u32(sm + L::kOffRing + st * 2 * L::kT), sv = sk + L::kT;
        mbar_wait(kv_full + st, (e / L::kSt) & 1);
        tc_fence_after();
        for (int kk = 0; kk < HD / 16; ++kk) mma_bf16_ss(t_r, desc_kmajor(sq, kk), desc_kmajor(sk, kk), id_s, kk != 0);
        mma_commit(s_full);
        mbar_wait(p_done, e & 1);
        tc_fence_after();
        for (int kk = 0; kk < HD / 16; ++kk) mma_bf16_ss(t_r, desc_kmajor(sdo, kk), desc_kmajor(sv, kk), id_s, kk != 0);
        mma_commit(dp_full);
        mbar_wait(ds_ready, e & 1);
        tc_fence_after();
        for (int kk = 0; kk < kAT / 16; ++kk) mma_bf16_ts(t_dq, t_r + kk * 8, desc_mnmajor(sk, kk), id_g, (e | kk) != 0);
        mma_commit(kv_empty + st);
      }
      mma_commit(done);
    }
  } else {
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const int row = qt * kAT + r;
    const size_t lrow = ((size_t)item * H + h) * s + (row < s ? row : 0);
    const float l2 = __ldg(lse + lrow) * 1.4426950408889634f, dl = __ldg(delta + lrow);
    const int ci = r >> 4;
    // eps = row sum of the bf16 dS fed to the MMA. Exactly, sum_j dS_ij = 0 (softmax Jacobian), so
    // dq_i = sum_j dS_ij (k_j - kbar) for any kbar; rounding leaves eps != 0, whose product with
    // the keys' common mode kbar is removed in the epilogue.
    float eps = 0.f;
    for (int e = 0; e < n; ++e) {
      const int32_t* ent = tv.csr + (size_t)(e0 + e) * kEntryInts;
        const uint32_t lo = (uint32_t)__ldg(ent), hi = (uint32_t)__ldg(ent + 1);
      const uint32_t mrow = (uint32_t)((((uint64_t)hi << 32) | lo) >> (ci * 8)) & 0xffu;
      mbar_wait(s_full, e & 1);
      tc_fence_after();
      uint32_t pp[4][16];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t sv_[32];
        tmem_ld_32x32b_x32(t_r + lane_base + c * 32, sv_);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const bool on = (mrow >> (c * 2 + (u >> 3))) & 1u;
          const float p0 = on ? ex2(fmaf(__uint_as_float(sv_[2 * u]), scale_log2, -l2)) : 0.f;
          const float p1 = on ? ex2(fmaf(__uint_as_float(sv_[2 * u + 1]), scale_log2, -l2)) : 0.f;
          pp[c][u] = pack_bf16x2(p0, p1);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_done);
      mbar_wait(dp_full, e & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t dv_[32], dd[16];
        tmem_ld_32x32b_x32(t_r + lane_base + c * 32, dv_);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const __nv_bfloat162 pb = *reinterpret_cast<const __nv_bfloat162*>(&pp[c][u]);
          dd[u] = pack_bf16x2(__low2float(pb) * (__uint_as_float(dv_[2 * u]) - dl),
                              __high2float(pb) * (__uint_as_float(dv_[2 * u + 1]) - dl));
          const __nv_bfloat162 rb = *reinterpret_cast<const __nv_bfloat162*>(&dd[u]);
          eps += __low2float(rb) + __high2float(rb);
        }
        tmem_st_32x32b_x16(t_r + lane_base + c * 16, dd);  // dP chunk c/2 already consumed
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_ready);
    }
    // kbar = mean over the item's keys (bsattn_prep_kernel)
    if (r < HD) kbar[r] = __ldg(kbar_g + ((size_t)item * H + h) * HD + r);
    asm volatile("bar.sync 1, 128;" ::: "memory");
    mbar_wait(done, 0);
    tc_fence_after();
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t ov[32];
      tmem_ld_32x32b_x32(t_dq + lane_base + c * 32, ov);
      tmem_ld_wait();
      if (row < s) {
        float f[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) f[i] = n > 0 ? (__uint_as_float(ov[i]) - eps * kbar[c * 32 + i]) * scale : 0.f;
        __nv_bfloat16* op = dq + ((size_t)row_base + row) * ld_dq + h * HD + c * 32;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          *reinterpret_cast<uint4*>(op + 8 * i) =
              make_uint4(pack_bf16x2(f[8 * i], f[8 * i + 1]), pack_bf16x2(f[8 * i + 2], f[8 * i + 3]),
                         pack_bf16x2(f[8 * i + 4], f[8 * i + 5]), pack_bf16x2(f[8 * i + 6], f[8 * i + 7]));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmem>(tmem);
  }
}

// Backward prologue, one launch (three block ranges):
//  [0, nb_delta)            delta[item, h, row] = sum_c dO[row, c] * O[row, c] (== rowsum(dP * P),
//                           sf/block_sparse.py:102-113): one warp per token row, lane l reads 16 B chunks
//                           l, l+32, ... of O and dO (all in flight), a group of HD/8 lanes holds one head;
//  [nb_delta, +n_items*H)   kbar[item, h, :] = mean of K over the item's first min(s, 128) keys (the dQ
//                           kernels' common-mode vector, fixed-order tree);
//  [.., +nb_desc)           per-unit work descriptors {e0, n, pattern} of the dK/dV walk (CSC of each key
//                           tile) and the dQ walk (CSR of each query tile), so the persistent kernels read one
//                           int4 per unit (prefetched a unit ahead) instead of a pidx -> table -> pointer chain.
template <int HD>
__global__ void __launch_bounds__(256) bsattn_prep_kernel(const __nv_bfloat16* __restrict__ o,
                                                          const __nv_bfloat16* __restrict__ d_o, int ld, int n_rows_total,
                                                          int s, int H, float* __restrict__ delta,
                                                          const __nv_bfloat16* __restrict__ qkv, int ldq,
                                                          float* __restrict__ kbar, const int32_t* __restrict__ pidx,
                                                          int item_stride, const int32_t* __restrict__ tables,
                                                          int4* __restrict__ desc_kv, int4* __restrict__ desc_q, int n_units,
                                                          int nb_delta, int nb_kbar) {
  pdl_wait_trigger();
  const int d = H * HD;
  // block roles: [descriptors | kbar | delta]; the short latency-bound roles are scheduled first, under the
  // bandwidth-bound delta blocks
  const int nb_desc = (int)gridDim.x - nb_delta - nb_kbar;
  if ((int)blockIdx.x >= nb_desc + nb_kbar) {
    const int bdx = blockIdx.x - nb_desc - nb_kbar;
    constexpr int G = HD / 8;  // lanes per head
    constexpr int kIt = 8;     // 16 B chunks per lane per pass (2048 columns)
    const int row = (bdx * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= n_rows_total) return;
    const int n_it = (d + 255) / 256;
    const uint4* a = reinterpret_cast<const uint4*>(o + (size_t)row * ld);
    const uint4* b = reinterpret_cast<const uint4*>(d_o + (size_t)row * ld);
    const size_t out_row = (size_t)(row / s) * H * s + row % s;
    for (int base = 0; base < n_it; base += kIt) {
      uint4 va[kIt], vb[kIt];
#pragma unroll
      for (int i = 0; i < kIt; ++i) {
        const int c = (base + i) * 32 + lane;
        const bool ok = base + i < n_it && c * 8 < d;
        va[i] = ok ? __ldg(a + c) : make_uint4(0u, 0u, 0u, 0u);
        vb[i] = ok ? __ldg(b + c) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int i = 0; i < kIt; ++i) {
        const int it = base + i;
        if (it >= n_it) break;
        const uint32_t xa[4] = {va[i].x, va[i].y, va[i].z, va[i].w}, xb[4] = {vb[i].x, vb[i].y, vb[i].z, vb[i].w};
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const __nv_bfloat162 p = *reinterpret_cast<const __nv_bfloat162*>(&xa[k]);
          const __nv_bfloat162 q = *reinterpret_cast<const __nv_bfloat162*>(&xb[k]);
          acc = fmaf(__low2float(p), __low2float(q), acc);
          acc = fmaf(__high2float(p), __high2float(q), acc);
        }
#pragma unroll
        for (int off = 1; off < G; off <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        const int h = (it * 32 + lane) * 8 / HD;
        if ((lane % G) == 0 && h < H) delta[out_row + (size_t)h * s] = acc;
      }
    }
    return;
  }
  if ((int)blockIdx.x >= nb_desc) {
    // kbar of (item, h) over the item's first min(s, 128) keys: any fixed vector is exact for the dQ
    // identity sum_j dS_ij (k_j - kbar) = sum_j dS_ij k_j; the first tile's mean estimates the common mode.
    // 16-byte loads: thread t reads chunk t % (HD / 8) of rows t / (HD / 8), + 256 / (HD / 8), ...
    __shared__ float part[256 / (HD / 8)][HD];
    constexpr int CH = HD / 8, RS = 256 / CH;
    const int ih = blockIdx.x - nb_desc, item = ih / H, h = ih % H;
    const int ch = threadIdx.x % CH, r0 = threadIdx.x / CH;
    const int nr = s < kAT ? s : kAT;
    const __nv_bfloat16* kp = qkv + (size_t)item * s * ldq + d + h * HD + ch * 8;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    constexpr int kLd = (kAT + RS - 1) / RS;  // rows per thread: all loads issued before the sums
    uint4 v[kLd];
#pragma unroll
    for (int i = 0; i < kLd; ++i) {
      const int r = r0 + i * RS;
      v[i] = r < nr ? __ldg(reinterpret_cast<const uint4*>(kp + (size_t)r * ldq)) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int i = 0; i < kLd; ++i) {
      const uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const __nv_bfloat162 p2 = *reinterpret_cast<const __nv_bfloat162*>(&w[q]);
        acc[2 * q] += __low2float(p2);
        acc[2 * q + 1] += __high2float(p2);
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) part[r0][ch * 8 + q] = acc[q];
    __syncthreads();
    if ((int)threadIdx.x < HD) {
      float t = 0.f;
      for (int g2 = 0; g2 < RS; ++g2) t += part[g2][threadIdx.x];
      kbar[(size_t)ih * HD + threadIdx.x] = t / (float)nr;
    }
    return;
  }
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n_units) return;
  const int nt = __ldg(tables), per = __ldg(tables + 6);
  const int t = u % nt, h = (u / nt) % H, item = u / (nt * H);
  const int p = __ldg(pidx + item * item_stride + h);
  const int32_t* b = tables + 8 + (size_t)p * per;
  const int r0 = __ldg(b + t), r1 = __ldg(b + t + 1);
  const int c0 = __ldg(b + nt + 1 + t), c1 = __ldg(b + nt + 2 + t);
  desc_q[u] = make_int4(r0, r1 - r0, p, 0);
  desc_kv[u] = make_int4(c0, c1 - c0, p, 0);
}

// the pattern's CSR (csc = false) or CSC entry array, from a unit descriptor
LX_DEV const int32_t* desc_entries(const int32_t* tables, int nt, int per, int p, bool csc) {
  return tables + 8 + (size_t)p * per + 2 * (nt + 1) + (csc ? kEntryInts * nt * nt : 0);
}

// ============================================================================ backward dK/dV, ping-pong
// Persistent: grid = #SMs, one CTA per SM (512 TMEM columns); CTA c walks units u = c, c + G, ... with
// u = (item * H + h) * nkt + kt (a key tile of one head). Two epilogue warpgroups alternate over the
// unit's CSC list of query tiles (WG w takes entries e = w, w + 2, ...) with one S/dP TMEM buffer each,
// so the tensor core computes S(e+1) / dV(e) / dP(e) for one warpgroup while the other runs its exp or
// dS math — the two dependency chains interleave inside the CTA instead of stalling it:
//   MMA:  S(0) S(1) | per e: [p_ready] dV += P^T dO, dP^T = V dO^T -> dp_full | [ds_ready] dK += dS^T Q,
//         release the Q/dO stage, S(e+2) into the freed buffer
//   WG w: [s_full] P = exp2(S c - lse) as bf16 into its buffer -> p_ready | [dp_full] dS = P (dP - delta)
//         -> ds_ready
// K/V are double-buffered across units (HD 64) and Q/dO stream through a kSt-stage ring, so the next
// unit's loads overlap this unit's tail; the unit epilogue (dK by WG0, dV by WG1, key column sums for
// the dQ kernel's common-mode correction) overlaps the next unit's first S MMAs.
constexpr int kBwdThreads = 64 + 32 * 8;  // producer, MMA issuer, two 4-warp epilogue groups

template <int HD>
struct AttnDkdvPP {
  static constexpr int kT = (HD / 64) * kAT * 128;  // one 128 x HD bf16 tile
#ifndef LX_DKDV_KV
#define LX_DKDV_KV 2
#define LX_DKDV_ST 3
#endif
  static constexpr int kKV = HD == 64 ? LX_DKDV_KV : 1;  // K/V buffers
  static constexpr int kSt = HD == 64 ? LX_DKDV_ST : 2;  // Q/dO ring stages
  static constexpr int kOffRing = kKV * 2 * kT;
  static constexpr int kOffL = kOffRing + kSt * 2 * kT;          // lse [kSt][128], delta [kSt][128]
  static constexpr int kStgPitch = 144;                          // staging row: 128 B of bf16 + 16 B pad
  // HD 128 stages 16 rows per warp at a time (two rounds), so the kernel fits in 227 KB of shared memory
  static constexpr int kStgRows = HD == 64 ? 32 : 16;
  static constexpr int kOffStg = kOffL + 2 * kSt * kAT * 4;      // [8 warps][kStgRows rows][kStgPitch]
  static constexpr int kOffBar = kOffStg + 8 * kStgRows * kStgPitch;
  static constexpr int kTotal = kOffBar + 512 + 1024;
};

template <int HD>
__global__ void __launch_bounds__(kBwdThreads, 1)
bsattn_dkdv_pp_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                      const __grid_constant__ CUtensorMap tm_g, const __grid_constant__ CUtensorMap tm_do_g, int gu, int s, int H,
                      int n_units, const int32_t* __restrict__ pidx, int item_stride, const int32_t* __restrict__ tables,
                      float scale, float scale_log2, const float* __restrict__ lse, const float* __restrict__ delta,
                      __nv_bfloat16* __restrict__ dkv, int ld_dkv, const int4* __restrict__ desc) {
  using L = AttnDkdvPP<HD>;
  constexpr int A = HD / 64;
  const int d_model = H * HD;
  const int nkt = (s + kAT - 1) / kAT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = align_smem_1024(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::kOffBar);
  uint64_t* kv_full = bars;                // [kKV]
  uint64_t* kv_empty = bars + 2;           // [kKV]
  uint64_t* qd_full = bars + 4;            // [kSt] TMA + bulk copies (1 arrive + tx)
  uint64_t* qd_empty = bars + 8;           // [kSt]
  uint64_t* s_full = bars + 12;            // [2]
  uint64_t* p_ready = bars + 14;           // [2] 4 warps
  uint64_t* dp_full = bars + 16;           // [2]
  uint64_t* ds_ready = bars + 18;          // [2] 4 warps
  uint64_t* acc_full = bars + 20;
  uint64_t* acc_empty = bars + 21;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 22);
  uint64_t* sMask = bars + 32;                          // [kSt] cell mask of the staged entry
  float* sL = reinterpret_cast<float*>(sm + L::kOffL);  // [kSt][128] lse (natural log) of the gathered rows
  float* sD = sL + L::kSt * kAT;                        // [kSt][128] delta

  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_g);
    tma_prefetch_desc(&tm_do_g);
    for (int i = 0; i < L::kKV; ++i) {
      mbar_init(kv_full + i, 1);
      mbar_init(kv_empty + i, 1);
    }
    for (int i = 0; i < L::kSt; ++i) {
      mbar_init(qd_full + i, 1);
      mbar_init(qd_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(p_ready + i, 4);
      mbar_init(dp_full + i, 1);
      mbar_init(ds_ready + i, 4);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait_trigger();
  if (threadIdx.x == 0) trace_stamp(0);
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_dv = tmem + 2 * kAT, t_dk = tmem + 2 * kAT + HD;

  // unit -> (item, h, kt) and its CSC range from the prep kernel's descriptors, read one unit ahead
  const int tab_nt = __ldg(tables), tab_per = __ldg(tables + 6);
  auto dload = [&](int u) { return u < n_units ? __ldg(desc + u) : make_int4(0, 0, 0, 0); };
  auto unit_of = [&](int u, int4& dnext, int& item, int& h, int& kt, const int32_t*& ents, int& e0, int& n) {
    const int4 dd = dnext;
    dnext = dload(u + gridDim.x);
    kt = u % nkt;
    h = (u / nkt) % H;
    item = u / (nkt * H);
    e0 = dd.x;
    n = dd.y;
    ents = desc_entries(tables, tab_nt, tab_per, dd.z, true);
  };

  if (warp == 0) {
    // ================= producer: K/V per unit, then the unit's Q/dO tiles (+ lse / delta rows)
    int kvi = 0, g = 0;
    int4 dnext = dload(blockIdx.x);
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++kvi) {
      int item, h, kt, e0, n;
      const int32_t* ents;
      unit_of(u, dnext, item, h, kt, ents, e0, n);
      const int row_base = item * s;
      const int kvb = kvi % L::kKV;
      mbar_wait(kv_empty + kvb, ((kvi / L::kKV) & 1) ^ 1);
      if (lane == 0) {
        uint8_t* skv = sm + kvb * 2 * L::kT;
        mbar_arrive_expect_tx(kv_full + kvb, 2 * L::kT);
        for (int a = 0; a < A; ++a) {
          tma_load_2d(skv + a * kAT * 128, &tm_qkv, kv_full + kvb, d_model + h * HD + a * 64, row_base + kt * kAT);
          tma_load_2d(skv + L::kT + a * kAT * 128, &tm_qkv, kv_full + kvb, 2 * d_model + h * HD + a * 64,
                      row_base + kt * kAT);
        }
      }
      const float* lse_b = lse + ((size_t)item * H + h) * s;
      const float* del_b = delta + ((size_t)item * H + h) * s;
      const int nsub = kAT / gu;
      for (int e = 0; e < n; ++e, ++g) {
        const int st = g % L::kSt;
        mbar_wait(qd_empty + st, ((g / L::kSt) & 1) ^ 1);
        const int32_t* ent = ents + (size_t)(e0 + e) * kEntryInts;
        if (lane == 0) {
          // entry mask, Q / dO tiles and the gathered rows' lse / delta, all landing on qd_full[st]
          sMask[st] = ent_mask(ent);
          uint8_t* sq = sm + L::kOffRing + st * 2 * L::kT;
          mbar_arrive_expect_tx(qd_full + st, 2 * L::kT + 2 * kAT * 4);
          for (int a = 0; a < A; ++a) {
            tma_load_gather(sq + a * kAT * 128, &tm_g, qd_full + st, h * HD + a * 64, row_base, ent, gu, nsub);
            tma_load_gather(sq + L::kT + a * kAT * 128, &tm_do_g, qd_full + st, h * HD + a * 64, row_base, ent, gu, nsub);
          }
          for (int k = 0; k < nsub; ++k) {  // gathered query units lie inside the item
            const int q0 = __ldg(ent + 2 + k) * gu;
            bulk_load_1d(sL + st * kAT + k * gu, lse_b + q0, gu * 4, qd_full + st);
            bulk_load_1d(sD + st * kAT + k * gu, del_b + q0, gu * 4, qd_full + st);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer
    if (lane == 0) {
      const uint32_t id_s = make_idesc_bf16(kAT, kAT, false, false);  // S^T, dP^T: B K-major
      const uint32_t id_g = make_idesc_bf16(kAT, HD, false, true);    // dV, dK: B MN-major
      int kvi = 0, g = 0, acc_i = 0;
      int use[2] = {0, 0};
      int4 dnext = dload(blockIdx.x);
      for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++kvi, ++acc_i) {
        int item, h, kt, e0, n;
        const int32_t* ents;
        unit_of(u, dnext, item, h, kt, ents, e0, n);
        const int kvb = kvi % L::kKV;
        mbar_wait(kv_full + kvb, (kvi / L::kKV) & 1);
        if (kvi < 5) trace_stamp(2 + 5 * kvi);  // debug timeline: K/V landed (MMA view)
        const uint32_t sk = smem_u32(sm + kvb * 2 * L::kT), sv = sk + L::kT;
        auto issue_s = [&](int e) {  // S^T(e) = K Q(e)^T into buffer e & 1
          const int gg = g + e, st = gg % L::kSt;
          mbar_wait(qd_full + st, (gg / L::kSt) & 1);
          tc_fence_after();
          const uint32_t sq = smem_u32(sm + L::kOffRing + st * 2 * L::kT);
          const uint32_t tb = tmem + (e & 1) * kAT;
          for (int kk = 0; kk < HD / 16; ++kk) mma_bf16_ss(tb, desc_kmajor(sk, kk), desc_kmajor(sq, kk), id_s, kk != 0);
          mma_commit(s_full + (e & 1));
        };
        if (n > 0) issue_s(0);
        if (n > 1) issue_s(1);
        mbar_wait(acc_empty, (acc_i & 1) ^ 1);  // the previous unit's dK / dV have been drained
        tc_fence_after();
        // fixed two-deep schedule (deterministic accumulation order dV(0), dV(1), ..., dK(0), dK(1), ...):
        // per pair (e, e+1): dV/dP of both, then dK of both, each dK followed by the S two entries ahead
        auto issue_vp = [&](int e) {
          const int b = e & 1, gg = g + e, st = gg % L::kSt;
          const uint32_t sq = smem_u32(sm + L::kOffRing + st * 2 * L::kT), sdo = sq + L::kT;
          const uint32_t tb = tmem + b * kAT;
          mbar_wait(p_ready + b, use[b] & 1);
          tc_fence_after();
          for (int kk = 0; kk < kAT / 16; ++kk) mma_bf16_ts(t_dv, tb + kk * 8, desc_mnmajor(sdo, kk), id_g, (e | kk) != 0);
          for (int kk = 0; kk < HD / 16; ++kk) mma_bf16_ss(tb, desc_kmajor(sv, kk), desc_kmajor(sdo, kk), id_s, kk != 0);
          mma_commit(dp_full + b);
        };
        auto issue_k = [&](int e) {
          const int b = e & 1, gg = g + e, st = gg % L::kSt;
          const uint32_t sq = smem_u32(sm + L::kOffRing + st * 2 * L::kT);
          const uint32_t tb = tmem + b * kAT;
          mbar_wait(ds_ready + b, use[b] & 1);
          tc_fence_after();
          for (int kk = 0; kk < kAT / 16; ++kk) mma_bf16_ts(t_dk, tb + kk * 8, desc_mnmajor(sq, kk), id_g, (e | kk) != 0);
          mma_commit(qd_empty + st);
          ++use[b];
          if (e + 2 < n) issue_s(e + 2);
        };
        for (int e = 0; e < n; e += 2) {
          issue_vp(e);
          if (e + 1 < n) issue_vp(e + 1);
          issue_k(e);
          if (e + 1 < n) issue_k(e + 1);
        }
        if (n > 0) {
          mma_commit(acc_full);
          mma_commit(kv_empty + kvb);
        } else {
          mbar_arrive(acc_full);
          mbar_arrive(kv_empty + kvb);
        }
        g += n;
      }
    }
  } else {
    // ================= epilogue warpgroups: wg = (warp - 2) / 4 owns TMEM buffer wg; thread = key row
    const int wg = (warp - 2) >> 2, quad = warp & 3;
    const int kr = quad * 32 + lane;
    const int ep_tid = threadIdx.x - 64;  // 0..255
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const uint32_t tb = tmem + wg * kAT + lane_base;
    const int cj = kr >> 4;
    int kvi = 0, g = 0, acc_i = 0, use = 0;
    int4 dnext = dload(blockIdx.x);
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++kvi, ++acc_i) {
      int item, h, kt, e0, n;
      const int32_t* ents;
      unit_of(u, dnext, item, h, kt, ents, e0, n);
      const int row_base = item * s;
      for (int e = wg; e < n; e += 2, ++use) {
        const int gg = g + e, st = gg % L::kSt;
        const float* l2 = sL + st * kAT;
        const float* dl = sD + st * kAT;
        mbar_wait(qd_full + st, (gg / L::kSt) & 1);  // mask, lse / delta staged with the tiles
        const uint64_t mask = sMask[st];
        const bool full = mask == ~0ull;
        mbar_wait(s_full + wg, use & 1);
        const bool tr = kvi < 5 && e == 0 && ep_tid == 0;
        if (tr) trace_stamp(3 + 5 * kvi);  // first entry's S ready
        tc_fence_after();
        uint32_t pp[4][16];  // P^T (bf16 pairs) for the whole row, reused by dS^T
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          uint32_t sv_[2][32];
          tmem_ld_32x32b_x32(tb + h2 * 64, sv_[0]);
          tmem_ld_32x32b_x32(tb + h2 * 64 + 32, sv_[1]);
          tmem_ld_wait();
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) {
            const int c = h2 * 2 + c2;
#pragma unroll
            for (int u2 = 0; u2 < 16; ++u2) {
              const int qi = c * 32 + 2 * u2;
              const float p0 = ex2(fmaf(__uint_as_float(sv_[c2][2 * u2]), scale_log2, -l2[qi] * 1.4426950408889634f));
              const float p1 = ex2(fmaf(__uint_as_float(sv_[c2][2 * u2 + 1]), scale_log2, -l2[qi + 1] * 1.4426950408889634f));
              const bool on = full || ((mask >> ((qi >> 4) * 8 + cj)) & 1ull);
              pp[c][u2] = on ? pack_bf16x2(p0, p1) : 0u;
            }
            tmem_st_32x32b_x16(tb + c * 16, pp[c]);  // S^T chunk c/2 already consumed
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_ready + wg);
        mbar_wait(dp_full + wg, use & 1);
        tc_fence_after();
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          uint32_t dv_[2][32];
          tmem_ld_32x32b_x32(tb + h2 * 64, dv_[0]);
          tmem_ld_32x32b_x32(tb + h2 * 64 + 32, dv_[1]);
          tmem_ld_wait();
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) {
            const int c = h2 * 2 + c2;
            uint32_t dd[16];
#pragma unroll
            for (int u2 = 0; u2 < 16; ++u2) {
              const int qi = c * 32 + 2 * u2;
              const __nv_bfloat162 pb = *reinterpret_cast<const __nv_bfloat162*>(&pp[c][u2]);
              dd[u2] = pack_bf16x2(__low2float(pb) * (__uint_as_float(dv_[c2][2 * u2]) - dl[qi]),
                                   __high2float(pb) * (__uint_as_float(dv_[c2][2 * u2 + 1]) - dl[qi + 1]));
            }
            tmem_st_32x32b_x16(tb + c * 16, dd);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(ds_ready + wg);
        if (tr) trace_stamp(4 + 5 * kvi);  // first entry's dS stored
      }
      // ---- unit epilogue: WG0 stores dK (scaled), WG1 dV; then the key tile's column sums
      mbar_wait(acc_full, acc_i & 1);
      if (kvi < 5 && (ep_tid & 127) == 0) trace_stamp(5 + 5 * kvi);  // dK/dV accumulated (draining WG view)
      tc_fence_after();
      // dK / dV rows -> bf16 through a per-warp staging tile, stored as full 128-byte row segments
      const uint32_t tcol = (wg == 0 ? t_dk : t_dv) + lane_base;
      const float mul = wg == 0 ? scale : 1.f;
      uint8_t* stg = sm + L::kOffStg + (warp - 2) * L::kStgRows * L::kStgPitch;
      constexpr int kRounds = 32 / L::kStgRows;
#pragma unroll
      for (int cp = 0; cp < HD / 64; ++cp) {
        uint4 pk[8];  // this lane's row: 64 columns as bf16
#pragma unroll
        for (int c2 = 0; c2 < 2; ++c2) {
          uint32_t ov[32];
          tmem_ld_32x32b_x32(tcol + cp * 64 + c2 * 32, ov);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float f[8];
#pragma unroll
            for (int k2 = 0; k2 < 8; ++k2) f[k2] = n > 0 ? __uint_as_float(ov[8 * i + k2]) * mul : 0.f;
            pk[4 * c2 + i] = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                                        pack_bf16x2(f[6], f[7]));
          }
        }
#pragma unroll
        for (int rd = 0; rd < kRounds; ++rd) {
          if ((int)lane / L::kStgRows == rd) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              *reinterpret_cast<uint4*>(stg + (lane % L::kStgRows) * L::kStgPitch + 16 * i) = pk[i];
          }
          __syncwarp();
#pragma unroll
          for (int pass = 0; pass < L::kStgRows / 4; ++pass) {  // lane -> row pass*4 + lane/8, 16-byte piece lane%8
            const int rr = pass * 4 + (lane >> 3), piece = lane & 7;
            const int key = kt * kAT + quad * 32 + rd * L::kStgRows + rr;
            if (key < s) {
              const uint4 v = *reinterpret_cast<const uint4*>(stg + rr * L::kStgPitch + piece * 16);
              *reinterpret_cast<uint4*>(dkv + ((size_t)row_base + key) * ld_dkv + (wg + 1) * d_model + h * HD + cp * 64 +
                                        piece * 8) = v;
            }
          }
          __syncwarp();
        }
      }
      tc_fence_before();
      asm volatile("bar.sync 1, 256;" ::: "memory");  // every epilogue thread has drained TMEM
      if (ep_tid == 0) {
        if (kvi < 5) trace_stamp(6 + 5 * kvi);  // drained
        mbar_arrive(acc_empty);
      }
      g += n;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ============================================================================ backward dK/dV, two unit streams
// At sparse layouts most units (key tile, head, item) hold one or two query tiles, so the ping-pong kernel above
// runs one serial chain per unit (K/V -> S -> P -> dV, dP -> dS -> dK -> drain) with one of its warpgroups idle.
// Here a CTA runs two INDEPENDENT unit streams, each a full pipeline of its own: producer warp, MMA-issuer warp, a
// 4-warp epilogue group, its own K/V buffer, Q/dO ring, S/dP TMEM buffer and dK/dV accumulators (HD 64: TMEM
// S/dP at 128 w, dV / dK at 256 + 128 w). The two chains meet only at the tensor core and the MUFU, which
// interleave them. The CTA's units are ordered by entry count (largest first) and dealt greedily to the stream
// with the smaller load (entries + 1 per unit), so the streams finish together; each unit's dK/dV sums run in
// entry order (deterministic). An empty unit is written as zeros by its epilogue group alone.
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kDsThreads = 384;  // warps 0/1 stream-0 producer/MMA, 2-5 and 6-9 epilogue groups, 10/11 stream-1
constexpr int kDsSortMax = 64;   // units per CTA dealt by entry count; beyond, units alternate between streams
template <int HD>
struct AttnDkdvDs {
  static constexpr int kT = kAT * 128;                       // one 128 x 64 bf16 tile
  static constexpr int kSt = 2;                              // Q/dO ring stages per stream
  static constexpr int kStgRows = 16;                        // drain staging rows per warp (two rounds)
  static constexpr int kStgPitch = 144;
  static constexpr int kOffRing = 2 * kT;                    // per stream: [K|V] [ring] [lse|delta] [staging]
  static constexpr int kOffL = kOffRing + kSt * 2 * kT;
  static constexpr int kOffStg = kOffL + 2 * kSt * kAT * 4;
  static constexpr int kStream = kOffStg + 4 * kStgRows * kStgPitch;  // 107 KB, a multiple of 1024
  static constexpr int kOffBar = 2 * kStream;
  static constexpr int kTotal = kOffBar + 512 + 1024;
  static_assert(kStream % 1024 == 0, "stream 1's tiles must stay 1024-aligned for SWIZZLE_128B");
};

template <int HD>
__global__ void __launch_bounds__(kDsThreads, 1)
bsattn_dkdv_ds_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                      const __grid_constant__ CUtensorMap tm_g, const __grid_constant__ CUtensorMap tm_do_g, int gu, int s, int H,
                      int n_units, const int32_t* __restrict__ pidx, int item_stride, const int32_t* __restrict__ tables,
                      float scale, float scale_log2, const float* __restrict__ lse, const float* __restrict__ delta,
                      __nv_bfloat16* __restrict__ dkv, int ld_dkv, const int4* __restrict__ desc, int deal) {
  static_assert(HD == 64, "two streams' S/dP buffers and dK/dV accumulators fill TMEM at HD 64");
  using L = AttnDkdvDs<HD>;
  const int d_model = H * HD;
  const int nkt = (s + kAT - 1) / kAT;
  extern __shared__ uint8_t smem_raw[];
  __shared__ int s_list[2][kDsSortMax];
  __shared__ int s_cnt[2];
  __shared__ int s_n[kDsSortMax], s_ord[kDsSortMax];  // entry counts of this CTA's units, their sorted order
  uint8_t* sm = align_smem_1024(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::kOffBar);
  // per stream w, at bars + 16 w: kv_full, kv_empty, qd_full[2], qd_empty[2], s_full, p_ready (4 warps), dp_full,
  // ds_ready (4 warps), acc_full, acc_empty (1 arrival after the group's drain barrier)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 32);
  uint64_t* sMaskAll = bars + 40;  // [2][kSt]

  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_g);
    tma_prefetch_desc(&tm_do_g);
    for (int w = 0; w < 2; ++w) {
      uint64_t* b = bars + 16 * w;
      for (int i = 0; i < 6; ++i) mbar_init(b + i, 1);
      mbar_init(b + 6, 1);
      mbar_init(b + 7, 4);
      mbar_init(b + 8, 1);
      mbar_init(b + 9, 4);
      mbar_init(b + 10, 1);
      mbar_init(b + 11, 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  pdl_wait_trigger();
  if (threadIdx.x == 0) trace_stamp(6);
  const int G = gridDim.x;
  const int n_mine = n_units > (int)blockIdx.x ? (n_units - (int)blockIdx.x + G - 1) / G : 0;
  const bool dealt = deal && n_mine <= kDsSortMax;
  if (dealt) {
    // the CTA's units by entry count, descending (ties by index): each thread ranks one unit, then thread 0 deals
    // them in that order to the stream with the smaller load (entries + 1 per unit; stream 0 on ties)
    const int k = threadIdx.x;
    const int nk = k < n_mine ? __ldg(desc + blockIdx.x + k * G).y : 0;
    if (k < n_mine) s_n[k] = nk;
    __syncthreads();
    if (k < n_mine) {
      int rank = 0;
      for (int j = 0; j < n_mine; ++j) {
        const int nj = s_n[j];
        rank += (nj > nk) | (nj == nk && j < k);
      }
      s_ord[rank] = k;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int load0 = 0, load1 = 0, c0 = 0, c1 = 0;
      for (int i = 0; i < n_mine; ++i) {
        const int kk = s_ord[i];
        if (load0 <= load1) {
          s_list[0][c0++] = blockIdx.x + kk * G;
          load0 += s_n[kk] + 1;
        } else {
          s_list[1][c1++] = blockIdx.x + kk * G;
          load1 += s_n[kk] + 1;
        }
      }
      s_cnt[0] = c0;
      s_cnt[1] = c1;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) trace_stamp(0);

  const int tab_nt = __ldg(tables), tab_per = __ldg(tables + 6);
  // stream w's i-th unit and its count
  auto n_stream = [&](int w) { return dealt ? s_cnt[w] : (n_mine + 1 - w) / 2; };
  auto unit = [&](int w, int i, int& item, int& h, int& kt, const int32_t*& ents, int& e0, int& n) {
    const int u = dealt ? s_list[w][i] : (int)blockIdx.x + (2 * i + w) * G;
    const int4 dd = __ldg(desc + u);
    kt = u % nkt;
    h = (u / nkt) % H;
    item = u / (nkt * H);
    e0 = dd.x;
    n = dd.y;
    ents = desc_entries(tables, tab_nt, tab_per, dd.z, true);
  };

  if (warp < 2 || warp >= 10) {
    const int w = warp >= 10 ? 1 : 0;
    uint64_t* b = bars + 16 * w;
    uint64_t *kv_full = b, *kv_empty = b + 1, *qd_full = b + 2, *qd_empty = b + 4, *s_full = b + 6, *p_ready = b + 7,
             *dp_full = b + 8, *ds_ready = b + 9, *acc_full = b + 10, *acc_empty = b + 11;
    uint8_t* smw = sm + w * L::kStream;
    uint64_t* sMask = sMaskAll + w * L::kSt;
    float* sL = reinterpret_cast<float*>(smw + L::kOffL);
    float* sD = sL + L::kSt * kAT;
    const int nu = n_stream(w);
    if ((warp & 1) == 0) {
      // ================= producer of stream w: K/V per non-empty unit, then its Q/dO tiles (+ lse / delta rows)
      int g = 0, kvn = 0;
      for (int i = 0; i < nu; ++i) {
        int item, h, kt, e0, n;
        const int32_t* ents;
        unit(w, i, item, h, kt, ents, e0, n);
        if (n == 0) continue;
        const int row_base = item * s;
        mbar_wait(kv_empty, (kvn & 1) ^ 1);
        ++kvn;
        if (lane == 0) {
          mbar_arrive_expect_tx(kv_full, 2 * L::kT);
          tma_load_2d(smw, &tm_qkv, kv_full, d_model + h * HD, row_base + kt * kAT);
          tma_load_2d(smw + L::kT, &tm_qkv, kv_full, 2 * d_model + h * HD, row_base + kt * kAT);
        }
        const float* lse_b = lse + ((size_t)item * H + h) * s;
        const float* del_b = delta + ((size_t)item * H + h) * s;
        const int nsub = kAT / gu;
        for (int e = 0; e < n; ++e, ++g) {
          const int st = g % L::kSt;
          mbar_wait(qd_empty + st, ((g / L::kSt) & 1) ^ 1);
          const int32_t* ent = ents + (size_t)(e0 + e) * kEntryInts;
          if (lane == 0) {
            sMask[st] = ent_mask(ent);
            uint8_t* sq = smw + L::kOffRing + st * 2 * L::kT;
            mbar_arrive_expect_tx(qd_full + st, 2 * L::kT + 2 * kAT * 4);
            tma_load_gather(sq, &tm_g, qd_full + st, h * HD, row_base, ent, gu, nsub);
            tma_load_gather(sq + L::kT, &tm_do_g, qd_full + st, h * HD, row_base, ent, gu, nsub);
            for (int k = 0; k < nsub; ++k) {
              const int q0 = __ldg(ent + 2 + k) * gu;
              bulk_load_1d(sL + st * kAT + k * gu, lse_b + q0, gu * 4, qd_full + st);
              bulk_load_1d(sD + st * kAT + k * gu, del_b + q0, gu * 4, qd_full + st);
            }
          }
          __syncwarp();
        }
      }
    } else if (lane == 0) {
      // ================= MMA issuer of stream w: per entry S^T = K Q^T | [p_ready] dV += P^T dO, dP^T = V dO^T |
      // [ds_ready] dK += dS^T Q, then the next entry's S into the freed buffer
      const uint32_t id_s = make_idesc_bf16(kAT, kAT, false, false);
      const uint32_t id_g = make_idesc_bf16(kAT, HD, false, true);
      const uint32_t tb = tmem + w * kAT, t_dv = tmem + 2 * kAT + w * 2 * HD, t_dk = t_dv + HD;
      const uint32_t sk = smem_u32(smw), sv = sk + L::kT;
      int g = 0, kvn = 0, accn = 0;
      for (int i = 0; i < nu; ++i) {
        int item, h, kt, e0, n;
        const int32_t* ents;
        unit(w, i, item, h, kt, ents, e0, n);
        if (n == 0) continue;
        mbar_wait(kv_full, kvn & 1);
        ++kvn;
        for (int j = 0; j < n; ++j) {
          const int gg = g + j, st = gg % L::kSt;
          const uint32_t sq = smem_u32(smw + L::kOffRing + st * 2 * L::kT), sdo = sq + L::kT;
          mbar_wait(qd_full + st, (gg / L::kSt) & 1);
          tc_fence_after();
          for (int kk = 0; kk < HD / 16; ++kk) mma_bf16_ss(tb, desc_kmajor(sk, kk), desc_kmajor(sq, kk), id_s, kk != 0);
          mma_commit(s_full);
          if (j == 0) {
            mbar_wait(acc_empty, (accn & 1) ^ 1);  // this stream's previous unit has been drained
            tc_fence_after();
          }
          mbar_wait(p_ready, gg & 1);
          tc_fence_after();
          for (int kk = 0; kk < kAT / 16; ++kk) mma_bf16_ts(t_dv, tb + kk * 8, desc_mnmajor(sdo, kk), id_g, (j | kk) != 0);
          for (int kk = 0; kk < HD / 16; ++kk) mma_bf16_ss(tb, desc_kmajor(sv, kk), desc_kmajor(sdo, kk), id_s, kk != 0);
          mma_commit(dp_full);
          if (j + 1 == n) mma_commit(kv_empty);  // K and V are read by S and dP only
          mbar_wait(ds_ready, gg & 1);
          tc_fence_after();
          for (int kk = 0; kk < kAT / 16; ++kk) mma_bf16_ts(t_dk, tb + kk * 8, desc_mnmajor(sq, kk), id_g, (j | kk) != 0);
          mma_commit(qd_empty + st);
        }
        mma_commit(acc_full);
        ++accn;
        g += n;
      }
    }
  } else {
    // ================= epilogue group wg = stream wg; thread = key row
    const int wg = (warp - 2) >> 2, quad = warp & 3;
    uint64_t* b = bars + 16 * wg;
    uint64_t *qd_full = b + 2, *s_full = b + 6, *p_ready = b + 7, *dp_full = b + 8, *ds_ready = b + 9,
             *acc_full = b + 10, *acc_empty = b + 11;
    uint8_t* smw = sm + wg * L::kStream;
    const uint64_t* sMask = sMaskAll + wg * L::kSt;
    const float* sL = reinterpret_cast<const float*>(smw + L::kOffL);
    const float* sD = sL + L::kSt * kAT;
    const int kr = quad * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const uint32_t tb = tmem + wg * kAT + lane_base;
    const int cj = kr >> 4;
    const int nu = n_stream(wg);
    int g = 0, accn = 0;
    for (int i = 0; i < nu; ++i) {
      int item, h, kt, e0, n;
      const int32_t* ents;
      unit(wg, i, item, h, kt, ents, e0, n);
      for (int j = 0; j < n; ++j) {
        const int gg = g + j, st = gg % L::kSt;
        const float* l2 = sL + st * kAT;
        const float* dl = sD + st * kAT;
        mbar_wait(qd_full + st, (gg / L::kSt) & 1);
        const uint64_t mask = sMask[st];
        uint32_t mrow = 0;  // bit q16: cell (query group q16, this thread's key group) is active
#pragma unroll
        for (int q16 = 0; q16 < 8; ++q16) mrow |= (uint32_t)((mask >> (q16 * 8 + cj)) & 1ull) << q16;
        mbar_wait(s_full, gg & 1);
        tc_fence_after();
        uint32_t pp[4][16];
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          uint32_t sv_[2][32];
          tmem_ld_32x32b_x32(tb + h2 * 64, sv_[0]);
          tmem_ld_32x32b_x32(tb + h2 * 64 + 32, sv_[1]);
          tmem_ld_wait();
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) {
            const int c = h2 * 2 + c2;
#pragma unroll
            for (int u2 = 0; u2 < 16; ++u2) {
              const int qi = c * 32 + 2 * u2;
              const float2 nl = mul2(*reinterpret_cast<const float2*>(l2 + qi), make_float2(-kLog2e, -kLog2e));
              const float2 x = fma2(make_float2(__uint_as_float(sv_[c2][2 * u2]), __uint_as_float(sv_[c2][2 * u2 + 1])),
                                    make_float2(scale_log2, scale_log2), nl);
              const uint32_t pk = pack_bf16x2(ex2(x.x), ex2(x.y));
              pp[c][u2] = (mrow >> (c * 2 + (u2 >> 3))) & 1u ? pk : 0u;
            }
            tmem_st_32x32b_x16(tb + c * 16, pp[c]);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_ready);
        mbar_wait(dp_full, gg & 1);
        tc_fence_after();
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          uint32_t dv_[2][32];
          tmem_ld_32x32b_x32(tb + h2 * 64, dv_[0]);
          tmem_ld_32x32b_x32(tb + h2 * 64 + 32, dv_[1]);
          tmem_ld_wait();
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) {
            const int c = h2 * 2 + c2;
            uint32_t dd[16];
#pragma unroll
            for (int u2 = 0; u2 < 16; ++u2) {
              const int qi = c * 32 + 2 * u2;
              const float2 pf = bf16x2_unpack(pp[c][u2]);
              const float2 t = sub2(make_float2(__uint_as_float(dv_[c2][2 * u2]), __uint_as_float(dv_[c2][2 * u2 + 1])),
                                    *reinterpret_cast<const float2*>(dl + qi));
              const float2 r2 = mul2(pf, t);
              dd[u2] = pack_bf16x2(r2.x, r2.y);
            }
            tmem_st_32x32b_x16(tb + c * 16, dd);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(ds_ready);
      }
      g += n;
      // ---- unit drain: dK (scaled) into column block 1, dV into block 2, through 16-row staging
      if (n > 0) {
        mbar_wait(acc_full, accn & 1);
        tc_fence_after();
      }
      const int row_base = item * s;
      uint8_t* stg = smw + L::kOffStg + quad * L::kStgRows * L::kStgPitch;
#pragma unroll
      for (int which = 0; which < 2; ++which) {
        const uint32_t tcol = tmem + 2 * kAT + wg * 2 * HD + (which == 0 ? HD : 0) + lane_base;
        const float mul = which == 0 ? scale : 1.f;
        uint4 pk[8];
        if (n > 0) {
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) {
            uint32_t ov[32];
            tmem_ld_32x32b_x32(tcol + c2 * 32, ov);
            tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float f[8];
#pragma unroll
              for (int k2 = 0; k2 < 8; ++k2) f[k2] = __uint_as_float(ov[8 * q + k2]) * mul;
              pk[4 * c2 + q] = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                                          pack_bf16x2(f[6], f[7]));
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) pk[q] = make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int rd = 0; rd < 32 / L::kStgRows; ++rd) {
          if ((int)lane / L::kStgRows == rd) {
#pragma unroll
            for (int q = 0; q < 8; ++q)
              *reinterpret_cast<uint4*>(stg + (lane % L::kStgRows) * L::kStgPitch + 16 * q) = pk[q];
          }
          __syncwarp();
#pragma unroll
          for (int pass = 0; pass < L::kStgRows / 4; ++pass) {
            const int rr = pass * 4 + (lane >> 3), piece = lane & 7;
            const int key = kt * kAT + quad * 32 + rd * L::kStgRows + rr;
            if (key < s) {
              const uint4 v = *reinterpret_cast<const uint4*>(stg + rr * L::kStgPitch + piece * 16);
              *reinterpret_cast<uint4*>(dkv + ((size_t)row_base + key) * ld_dkv + (which + 1) * d_model + h * HD +
                                        piece * 8) = v;
            }
          }
          __syncwarp();
        }
      }
      if (n > 0) {
        tc_fence_before();
        asm volatile("bar.sync %0, 128;" ::"r"(1 + wg) : "memory");  // the group has drained its accumulators
        if ((threadIdx.x & 127) == 0) mbar_arrive(acc_empty);
        ++accn;
      }
    }
    if ((threadIdx.x & 127) == 0) {
      trace_stamp(0 + 1 + wg);
      trace_put(0 + 3 + wg, ((unsigned long long)nu << 32) | (unsigned)g);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ============================================================================ backward dQ, ping-pong
// Same structure as the dK/dV kernel over query-tile units (CSR walk over key tiles): WG w takes the
// unit's entries e = w, w + 2, ... with its own S/dP TMEM buffer; per entry the MMA issuer computes
// S = Q K^T, dP = dO V^T (after the WG pulled P into registers) and dQ += dS K (after the WG wrote the
// bf16 dS back over its dP), in the fixed order dP(e) dP(e+1) dQ(e) dQ(e+1) (deterministic sums).
// The bf16 row-sum residual eps of dS (see bsattn_dq_tc_kernel) is summed per WG and combined in a
// fixed order at the unit end before the common-mode correction.
template <int HD>
struct AttnDqPP {
  static constexpr int kT = (HD / 64) * kAT * 128;
  static constexpr int kQB = HD == 64 ? 2 : 1;  // Q/dO buffers (next unit prefetched)
  static constexpr int kSt = HD == 64 ? 3 : 2;  // K/V ring stages
  static constexpr int kOffRing = kQB * 2 * kT;
  static constexpr int kOffMisc = kOffRing + kSt * 2 * kT;  // kbar [128] + eps [2][128]
  static constexpr int kStgPitch = 80;                      // staging row: 64 B of bf16 + 16 B pad
  static constexpr int kOffStg = kOffMisc + 384 * 4;        // [8 warps][32 rows][kStgPitch]
  static constexpr int kOffBar = kOffStg + 8 * 32 * kStgPitch;
  static constexpr int kTotal = kOffBar + 512 + 1024;
};

template <int HD>
__global__ void __launch_bounds__(kBwdThreads, 1)
bsattn_dq_pp_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_g, int gu, int s, int H,
                    int n_units, const int32_t* __restrict__ pidx, int item_stride, const int32_t* __restrict__ tables,
                    float scale, float scale_log2, const float* __restrict__ lse, const float* __restrict__ delta,
                    __nv_bfloat16* __restrict__ dq, int ld_dq, const float* __restrict__ kbar_g, const int4* __restrict__ desc) {
  using L = AttnDqPP<HD>;
  constexpr int A = HD / 64;
  const int d_model = H * HD;
  const int nqt = (s + kAT - 1) / kAT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = align_smem_1024(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::kOffBar);
  uint64_t* q_full = bars;        // [kQB]
  uint64_t* q_empty = bars + 2;   // [kQB]
  uint64_t* kv_full = bars + 4;   // [kSt]
  uint64_t* kv_empty = bars + 8;  // [kSt]
  uint64_t* s_full = bars + 12;   // [2]
  uint64_t* p_done = bars + 14;   // [2] 4 warps
  uint64_t* dp_full = bars + 16;  // [2]
  uint64_t* ds_ready = bars + 18; // [2] 4 warps
  uint64_t* acc_full = bars + 20;
  uint64_t* acc_empty = bars + 21;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 22);
  uint64_t* sMask = bars + 32;    // [kSt] cell mask of the staged K/V entry
  float* kbar = reinterpret_cast<float*>(sm + L::kOffMisc);
  float* eps_x = kbar + 128;  // [2][128]

  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_g);
    for (int i = 0; i < L::kQB; ++i) {
      mbar_init(q_full + i, 1);
      mbar_init(q_empty + i, 1);
    }
    for (int i = 0; i < L::kSt; ++i) {
      mbar_init(kv_full + i, 1);
      mbar_init(kv_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(p_done + i, 4);
      mbar_init(dp_full + i, 1);
      mbar_init(ds_ready + i, 4);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait_trigger();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_dq = tmem + 2 * kAT;

  // unit -> (item, h, qt) and its CSR range from the prep kernel's descriptors, read one unit ahead
  const int tab_nt = __ldg(tables), tab_per = __ldg(tables + 6);
  auto dload = [&](int u) { return u < n_units ? __ldg(desc + u) : make_int4(0, 0, 0, 0); };
  auto unit_of = [&](int u, int4& dnext, int& item, int& h, int& qt, const int32_t*& ents, int& e0, int& n) {
    const int4 dd = dnext;
    dnext = dload(u + gridDim.x);
    qt = u % nqt;
    h = (u / nqt) % H;
    item = u / (nqt * H);
    e0 = dd.x;
    n = dd.y;
    ents = desc_entries(tables, tab_nt, tab_per, dd.z, false);
  };

  if (warp == 0) {
    // ================= producer: Q/dO per unit, then the unit's K/V tiles
    if (lane == 0) {
      int qi_ = 0, g = 0;
      int4 dnext = dload(blockIdx.x);
      for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++qi_) {
        int item, h, qt, e0, n;
        const int32_t* ents;
        unit_of(u, dnext, item, h, qt, ents, e0, n);
        const int row_base = item * s;
        const int qb = qi_ % L::kQB;
        mbar_wait(q_empty + qb, ((qi_ / L::kQB) & 1) ^ 1);
        uint8_t* sq = sm + qb * 2 * L::kT;
        mbar_arrive_expect_tx(q_full + qb, 2 * L::kT);
        for (int a = 0; a < A; ++a) {
          tma_load_2d(sq + a * kAT * 128, &tm_qkv, q_full + qb, h * HD + a * 64, row_base + qt * kAT);
          tma_load_2d(sq + L::kT + a * kAT * 128, &tm_do, q_full + qb, h * HD + a * 64, row_base + qt * kAT);
        }
        for (int e = 0; e < n; ++e, ++g) {
          const int st = g % L::kSt;
          mbar_wait(kv_empty + st, ((g / L::kSt) & 1) ^ 1);
          const int32_t* ent = ents + (size_t)(e0 + e) * kEntryInts;
          uint8_t* skv = sm + L::kOffRing + st * 2 * L::kT;
          sMask[st] = ent_mask(ent);  // released to the epilogue by the arrive below
          mbar_arrive_expect_tx(kv_full + st, 2 * L::kT);
          for (int a = 0; a < A; ++a) {
            tma_load_gather(skv + a * kAT * 128, &tm_g, kv_full + st, d_model + h * HD + a * 64, row_base, ent, gu, kAT / gu);
            tma_load_gather(skv + L::kT + a * kAT * 128, &tm_g, kv_full + st, 2 * d_model + h * HD + a * 64, row_base, ent,
                            gu, kAT / gu);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer
    if (lane == 0) {
      const uint32_t id_s = make_idesc_bf16(kAT, kAT, false, false);
      const uint32_t id_g = make_idesc_bf16(kAT, HD, false, true);
      int qi_ = 0, g = 0, acc_i = 0;
      int use[2] = {0, 0};
      int4 dnext = dload(blockIdx.x);
      for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++qi_, ++acc_i) {
        int item, h, qt, e0, n;
        const int32_t* ents;
        unit_of(u, dnext, item, h, qt, ents, e0, n);
        const int qb = qi_ % L::kQB;
        mbar_wait(q_full + qb, (qi_ / L::kQB) & 1);
        const uint32_t sq = smem_u32(sm + qb * 2 * L::kT), sdo = sq + L::kT;
        auto issue_s = [&](int e) {  // S(e) = Q K(e)^T into buffer e & 1
          const int gg = g + e, st = gg % L::kSt;
          mbar_wait(kv_full + st, (gg / L::kSt) & 1);
          tc_fence_after();
          const uint32_t sk = smem_u32(sm + L::kOffRing + st * 2 * L::kT);
          const uint32_t tb = tmem + (e & 1) * kAT;
          for (int kk = 0; kk < HD / 16; ++kk) mma_bf16_ss(tb, desc_kmajor(sq, kk), desc_kmajor(sk, kk), id_s, kk != 0);
          mma_commit(s_full + (e & 1));
        };
        auto issue_p = [&](int e) {  // dP(e) = dO V(e)^T once the WG pulled P(e) into registers
          const int b = e & 1, gg = g + e, st = gg % L::kSt;
          const uint32_t sv = smem_u32(sm + L::kOffRing + st * 2 * L::kT) + L::kT;
          const uint32_t tb = tmem + b * kAT;
          mbar_wait(p_done + b, use[b] & 1);
          tc_fence_after();
          for (int kk = 0; kk < HD / 16; ++kk) mma_bf16_ss(tb, desc_kmajor(sdo, kk), desc_kmajor(sv, kk), id_s, kk != 0);
          mma_commit(dp_full + b);
        };
        auto issue_q = [&](int e) {  // dQ += dS(e) K(e)
          const int b = e & 1, gg = g + e, st = gg % L::kSt;
          const uint32_t sk = smem_u32(sm + L::kOffRing + st * 2 * L::kT);
          const uint32_t tb = tmem + b * kAT;
          mbar_wait(ds_ready + b, use[b] & 1);
          tc_fence_after();
          for (int kk = 0; kk < kAT / 16; ++kk) mma_bf16_ts(t_dq, tb + kk * 8, desc_mnmajor(sk, kk), id_g, (e | kk) != 0);
          mma_commit(kv_empty + st);
          ++use[b];
          if (e + 2 < n) issue_s(e + 2);
        };
        if (n > 0) issue_s(0);
        if (n > 1) issue_s(1);
        mbar_wait(acc_empty, (acc_i & 1) ^ 1);  // the previous unit's dQ has been drained
        tc_fence_after();
        for (int e = 0; e < n; e += 2) {
          issue_p(e);
          if (e + 1 < n) issue_p(e + 1);
          issue_q(e);
          if (e + 1 < n) issue_q(e + 1);
        }
        if (n > 0) {
          mma_commit(acc_full);
          mma_commit(q_empty + qb);
        } else {
          mbar_arrive(acc_full);
          mbar_arrive(q_empty + qb);
        }
        g += n;
      }
    }
  } else {
    // ================= epilogue warpgroups: wg owns TMEM buffer wg; thread = query row
    const int wg = (warp - 2) >> 2, quad = warp & 3;
    const int r = quad * 32 + lane;
    const int ep_tid = threadIdx.x - 64;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const uint32_t tb = tmem + wg * kAT + lane_base;
    const int ci = r >> 4;
    uint8_t* stg = sm + L::kOffStg + (warp - 2) * 32 * L::kStgPitch;
    int acc_i = 0, use = 0, g = 0;
    int4 dnext = dload(blockIdx.x);
    // this thread's row terms (lse, delta) and kbar component of a unit: loaded one unit ahead
    float l2n = 0.f, dln = 0.f, kbn = 0.f;
    auto row_terms = [&](int u) {
      if (u >= n_units) return;
      const int qt_ = u % nqt, h_ = (u / nqt) % H, it_ = u / (nqt * H), row_ = qt_ * kAT + r;
      const size_t lr = ((size_t)it_ * H + h_) * s + (row_ < s ? row_ : 0);
      l2n = __ldg(lse + lr);
      dln = __ldg(delta + lr);
      if (r < HD) kbn = __ldg(kbar_g + ((size_t)it_ * H + h_) * HD + r);
    };
    row_terms(blockIdx.x);
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++acc_i) {
      int item, h, qt, e0, n;
      const int32_t* ents;
      unit_of(u, dnext, item, h, qt, ents, e0, n);
      const int row_base = item * s;
      const float l2 = l2n * 1.4426950408889634f, dl = dln, kb = kbn;
      row_terms(u + gridDim.x);
      float eps = 0.f;
      for (int e = wg; e < n; e += 2, ++use) {
        const int gg = g + e, st = gg % L::kSt;
        mbar_wait(kv_full + st, (gg / L::kSt) & 1);  // the entry's mask was staged with its K/V tiles
        const uint32_t mrow = (uint32_t)(sMask[st] >> (ci * 8)) & 0xffu;
        mbar_wait(s_full + wg, use & 1);
        tc_fence_after();
        uint32_t pp[4][16];
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          uint32_t sv_[2][32];
          tmem_ld_32x32b_x32(tb + h2 * 64, sv_[0]);
          tmem_ld_32x32b_x32(tb + h2 * 64 + 32, sv_[1]);
          tmem_ld_wait();
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) {
            const int c = h2 * 2 + c2;
#pragma unroll
            for (int u2 = 0; u2 < 16; ++u2) {
              const bool on = (mrow >> (c * 2 + (u2 >> 3))) & 1u;
              const float p0 = ex2(fmaf(__uint_as_float(sv_[c2][2 * u2]), scale_log2, -l2));
              const float p1 = ex2(fmaf(__uint_as_float(sv_[c2][2 * u2 + 1]), scale_log2, -l2));
              pp[c][u2] = on ? pack_bf16x2(p0, p1) : 0u;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_done + wg);
        mbar_wait(dp_full + wg, use & 1);
        tc_fence_after();
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          uint32_t dv_[2][32];
          tmem_ld_32x32b_x32(tb + h2 * 64, dv_[0]);
          tmem_ld_32x32b_x32(tb + h2 * 64 + 32, dv_[1]);
          tmem_ld_wait();
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) {
            const int c = h2 * 2 + c2;
            uint32_t dd[16];
#pragma unroll
            for (int u2 = 0; u2 < 16; ++u2) {
              const __nv_bfloat162 pb = *reinterpret_cast<const __nv_bfloat162*>(&pp[c][u2]);
              dd[u2] = pack_bf16x2(__low2float(pb) * (__uint_as_float(dv_[c2][2 * u2]) - dl),
                                   __high2float(pb) * (__uint_as_float(dv_[c2][2 * u2 + 1]) - dl));
              const __nv_bfloat162 rb = *reinterpret_cast<const __nv_bfloat162*>(&dd[u2]);
              eps += __low2float(rb) + __high2float(rb);
            }
            tmem_st_32x32b_x16(tb + c * 16, dd);  // dP chunk c/2 already consumed
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(ds_ready + wg);
      }
      // ---- unit epilogue: eps of both warpgroups (fixed order), key mean kbar, dQ rows (WG w: columns
      // [w HD/2, (w+1) HD/2)) through the staging tile as 64-byte row segments
      eps_x[wg * 128 + r] = eps;
      if (wg == 0 && r < HD) kbar[r] = kb;  // mean key of (item, h), bsattn_prep_kernel
      mbar_wait(acc_full, acc_i & 1);
      asm volatile("bar.sync 1, 256;" ::: "memory");
      tc_fence_after();
      const float eps_row = eps_x[r] + eps_x[128 + r];
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) {
        const int col0 = wg * (HD / 2) + c * 32;
        uint32_t ov[32];
        tmem_ld_32x32b_x32(t_dq + lane_base + col0, ov);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float f[8];
#pragma unroll
          for (int k2 = 0; k2 < 8; ++k2)
            f[k2] = n > 0 ? (__uint_as_float(ov[8 * i + k2]) - eps_row * kbar[col0 + 8 * i + k2]) * scale : 0.f;
          *reinterpret_cast<uint4*>(stg + lane * L::kStgPitch + 16 * i) =
              make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]), pack_bf16x2(f[6], f[7]));
        }
        __syncwarp();
#pragma unroll
        for (int pass = 0; pass < 4; ++pass) {  // lane -> row pass*8 + lane/4, 16-byte piece lane%4
          const int rr = pass * 8 + (lane >> 2), piece = lane & 3;
          const int qrow = qt * kAT + quad * 32 + rr;
          if (qrow < s)
            *reinterpret_cast<uint4*>(dq + ((size_t)row_base + qrow) * ld_dq + h * HD + col0 + piece * 8) =
                *reinterpret_cast<const uint4*>(stg + rr * L::kStgPitch + piece * 16);
        }
        __syncwarp();
      }
      tc_fence_before();
      asm volatile("bar.sync 1, 256;" ::: "memory");  // TMEM drained, eps_x / kbar reusable
      if (ep_tid == 0) mbar_arrive(acc_empty);
      g += n;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ============================================================================ backward dQ, two unit streams
// The dQ counterpart of bsattn_dkdv_ds_kernel: two independent pipelines per CTA over query-tile units (producer,
// MMA issuer and 4-warp epilogue group each; TMEM S/dP at 128 w, dQ at 256 + 64 w), units dealt by entry count.
// Per entry: S = Q K^T | [p_done] dP = dO V^T over S | [ds_ready] dQ += dS K (dS as bf16 over dP). A stream's
// group owns whole units, so the bf16 row-sum residual eps of dS (see bsattn_dq_tc_kernel) is a per-thread sum.
template <int HD>
struct AttnDqDs {
  static constexpr int kT = kAT * 128;
  static constexpr int kSt = 2;                                // K/V ring stages per stream
  static constexpr int kStgPitch = 80;                         // staging row: 64 B of bf16 + 16 B pad
  static constexpr int kOffRing = 2 * kT;                      // per stream: [Q|dO] [ring] [kbar] [staging]
  static constexpr int kOffKbar = kOffRing + kSt * 2 * kT;
  static constexpr int kOffStg = kOffKbar + 64 * 4;
  static constexpr int kStream = (kOffStg + 4 * 32 * kStgPitch + 1023) / 1024 * 1024;
  static constexpr int kOffBar = 2 * kStream;
  static constexpr int kTotal = kOffBar + 512 + 1024;
};

template <int HD>
__global__ void __launch_bounds__(kDsThreads, 1)
bsattn_dq_ds_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_g, int gu, int s, int H,
                    int n_units, const int32_t* __restrict__ pidx, int item_stride, const int32_t* __restrict__ tables,
                    float scale, float scale_log2, const float* __restrict__ lse, const float* __restrict__ delta,
                    __nv_bfloat16* __restrict__ dq, int ld_dq, const float* __restrict__ kbar_g, const int4* __restrict__ desc, int deal) {
  static_assert(HD == 64, "two streams' S/dP buffers and dQ accumulators fit TMEM at HD 64");
  using L = AttnDqDs<HD>;
  const int d_model = H * HD;
  const int nqt = (s + kAT - 1) / kAT;
  extern __shared__ uint8_t smem_raw[];
  __shared__ int s_list[2][kDsSortMax];
  __shared__ int s_cnt[2];
  __shared__ int s_n[kDsSortMax], s_ord[kDsSortMax];  // entry counts of this CTA's units, their sorted order
  uint8_t* sm = align_smem_1024(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::kOffBar);
  // per stream w, at bars + 16 w: q_full, q_empty, kv_full[2], kv_empty[2], s_full, p_done (4 warps), dp_full,
  // ds_ready (4 warps), acc_full, acc_empty
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 32);
  uint64_t* sMaskAll = bars + 40;  // [2][kSt]

  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_g);
    for (int w = 0; w < 2; ++w) {
      uint64_t* b = bars + 16 * w;
      for (int i = 0; i < 6; ++i) mbar_init(b + i, 1);
      mbar_init(b + 6, 1);
      mbar_init(b + 7, 4);
      mbar_init(b + 8, 1);
      mbar_init(b + 9, 4);
      mbar_init(b + 10, 1);
      mbar_init(b + 11, 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  pdl_wait_trigger();
  if (threadIdx.x == 0) trace_stamp(7);
  const int G = gridDim.x;
  const int n_mine = n_units > (int)blockIdx.x ? (n_units - (int)blockIdx.x + G - 1) / G : 0;
  const bool dealt = deal && n_mine <= kDsSortMax;
  if (dealt) {
    // the CTA's units by entry count, descending (ties by index): each thread ranks one unit, then thread 0 deals
    // them in that order to the stream with the smaller load (entries + 1 per unit; stream 0 on ties)
    const int k = threadIdx.x;
    const int nk = k < n_mine ? __ldg(desc + blockIdx.x + k * G).y : 0;
    if (k < n_mine) s_n[k] = nk;
    __syncthreads();
    if (k < n_mine) {
      int rank = 0;
      for (int j = 0; j < n_mine; ++j) {
        const int nj = s_n[j];
        rank += (nj > nk) | (nj == nk && j < k);
      }
      s_ord[rank] = k;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int load0 = 0, load1 = 0, c0 = 0, c1 = 0;
      for (int i = 0; i < n_mine; ++i) {
        const int kk = s_ord[i];
        if (load0 <= load1) {
          s_list[0][c0++] = blockIdx.x + kk * G;
          load0 += s_n[kk] + 1;
        } else {
          s_list[1][c1++] = blockIdx.x + kk * G;
          load1 += s_n[kk] + 1;
        }
      }
      s_cnt[0] = c0;
      s_cnt[1] = c1;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) trace_stamp(8);

  const int tab_nt = __ldg(tables), tab_per = __ldg(tables + 6);
  auto n_stream = [&](int w) { return dealt ? s_cnt[w] : (n_mine + 1 - w) / 2; };
  auto unit_id = [&](int w, int i) { return dealt ? s_list[w][i] : (int)blockIdx.x + (2 * i + w) * G; };
  auto unit = [&](int w, int i, int& item, int& h, int& qt, const int32_t*& ents, int& e0, int& n) {
    const int u = unit_id(w, i);
    const int4 dd = __ldg(desc + u);
    qt = u % nqt;
    h = (u / nqt) % H;
    item = u / (nqt * H);
    e0 = dd.x;
    n = dd.y;
    ents = desc_entries(tables, tab_nt, tab_per, dd.z, false);
  };

  if (warp < 2 || warp >= 10) {
    const int w = warp >= 10 ? 1 : 0;
    uint64_t* b = bars + 16 * w;
    uint64_t *q_full = b, *q_empty = b + 1, *kv_full = b + 2, *kv_empty = b + 4, *s_full = b + 6, *p_done = b + 7,
             *dp_full = b + 8, *ds_ready = b + 9, *acc_full = b + 10, *acc_empty = b + 11;
    uint8_t* smw = sm + w * L::kStream;
    uint64_t* sMask = sMaskAll + w * L::kSt;
    const int nu = n_stream(w);
    if ((warp & 1) == 0) {
      // ================= producer of stream w: Q/dO per non-empty unit, then its K/V tiles
      if (lane == 0) {
        int g = 0, qn = 0;
        for (int i = 0; i < nu; ++i) {
          int item, h, qt, e0, n;
          const int32_t* ents;
          unit(w, i, item, h, qt, ents, e0, n);
          if (n == 0) continue;
          const int row_base = item * s;
          mbar_wait(q_empty, (qn & 1) ^ 1);
          ++qn;
          mbar_arrive_expect_tx(q_full, 2 * L::kT);
          tma_load_2d(smw, &tm_qkv, q_full, h * HD, row_base + qt * kAT);
          tma_load_2d(smw + L::kT, &tm_do, q_full, h * HD, row_base + qt * kAT);
          for (int e = 0; e < n; ++e, ++g) {
            const int st = g % L::kSt;
            mbar_wait(kv_empty + st, ((g / L::kSt) & 1) ^ 1);
            const int32_t* ent = ents + (size_t)(e0 + e) * kEntryInts;
            uint8_t* skv = smw + L::kOffRing + st * 2 * L::kT;
            sMask[st] = ent_mask(ent);
            mbar_arrive_expect_tx(kv_full + st, 2 * L::kT);
            tma_load_gather(skv, &tm_g, kv_full + st, d_model + h * HD, row_base, ent, gu, kAT / gu);
            tma_load_gather(skv + L::kT, &tm_g, kv_full + st, 2 * d_model + h * HD, row_base, ent, gu, kAT / gu);
          }
        }
      }
    } else if (lane == 0) {
      // ================= MMA issuer of stream w
      const uint32_t id_s = make_idesc_bf16(kAT, kAT, false, false);
      const uint32_t id_g = make_idesc_bf16(kAT, HD, false, true);
      const uint32_t tb = tmem + w * kAT, t_dq = tmem + 2 * kAT + w * HD;
      const uint32_t sq = smem_u32(smw), sdo = sq + L::kT;
      int g = 0, qn = 0, accn = 0;
      for (int i = 0; i < nu; ++i) {
        int item, h, qt, e0, n;
        const int32_t* ents;
        unit(w, i, item, h, qt, ents, e0, n);
        if (n == 0) continue;
        mbar_wait(q_full, qn & 1);
        ++qn;
        for (int j = 0; j < n; ++j) {
          const int gg = g + j, st = gg % L::kSt;
          const uint32_t sk = smem_u32(smw + L::kOffRing + st * 2 * L::kT), sv = sk + L::kT;
          mbar_wait(kv_full + st, (gg / L::kSt) & 1);
          tc_fence_after();
          for (int kk = 0; kk < HD / 16; ++kk) mma_bf16_ss(tb, desc_kmajor(sq, kk), desc_kmajor(sk, kk), id_s, kk != 0);
          mma_commit(s_full);
          if (j == 0) {
            mbar_wait(acc_empty, (accn & 1) ^ 1);  // this stream's previous dQ has been drained
            tc_fence_after();
          }
          mbar_wait(p_done, gg & 1);
          tc_fence_after();
          for (int kk = 0; kk < HD / 16; ++kk) mma_bf16_ss(tb, desc_kmajor(sdo, kk), desc_kmajor(sv, kk), id_s, kk != 0);
          mma_commit(dp_full);
          if (j + 1 == n) mma_commit(q_empty);  // Q and dO are read by S and dP only
          mbar_wait(ds_ready, gg & 1);
          tc_fence_after();
          for (int kk = 0; kk < kAT / 16; ++kk) mma_bf16_ts(t_dq, tb + kk * 8, desc_mnmajor(sk, kk), id_g, (j | kk) != 0);
          mma_commit(kv_empty + st);
        }
        mma_commit(acc_full);
        ++accn;
        g += n;
      }
    }
  } else {
    // ================= epilogue group wg = stream wg; thread = query row
    const int wg = (warp - 2) >> 2, quad = warp & 3;
    uint64_t* b = bars + 16 * wg;
    uint64_t *kv_full = b + 2, *s_full = b + 6, *p_done = b + 7, *dp_full = b + 8, *ds_ready = b + 9, *acc_full = b + 10,
             *acc_empty = b + 11;
    uint8_t* smw = sm + wg * L::kStream;
    const uint64_t* sMask = sMaskAll + wg * L::kSt;
    float* kbar = reinterpret_cast<float*>(smw + L::kOffKbar);
    uint8_t* stg = smw + L::kOffStg + quad * 32 * L::kStgPitch;
    const int r = quad * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const uint32_t tb = tmem + wg * kAT + lane_base;
    const uint32_t t_dq = tmem + 2 * kAT + wg * HD + lane_base;
    const int ci = r >> 4;
    const int nu = n_stream(wg);
    // this thread's row terms (lse, delta) and kbar component of the stream's next unit, loaded one unit ahead
    float l2n = 0.f, dln = 0.f, kbn = 0.f;
    auto row_terms = [&](int i) {
      if (i >= nu) return;
      const int u = unit_id(wg, i);
      const int qt_ = u % nqt, h_ = (u / nqt) % H, it_ = u / (nqt * H), row_ = qt_ * kAT + r;
      const size_t lr = ((size_t)it_ * H + h_) * s + (row_ < s ? row_ : 0);
      l2n = __ldg(lse + lr);
      dln = __ldg(delta + lr);
      if (r < HD) kbn = __ldg(kbar_g + ((size_t)it_ * H + h_) * HD + r);
    };
    row_terms(0);
    int g = 0, accn = 0;
    for (int i = 0; i < nu; ++i) {
      int item, h, qt, e0, n;
      const int32_t* ents;
      unit(wg, i, item, h, qt, ents, e0, n);
      const float l2 = l2n * 1.4426950408889634f, dl = dln, kb = kbn;
      row_terms(i + 1);
      float2 eps2 = make_float2(0.f, 0.f);  // bf16 dS row sum, even / odd columns
      for (int j = 0; j < n; ++j) {
        const int gg = g + j, st = gg % L::kSt;
        mbar_wait(kv_full + st, (gg / L::kSt) & 1);
        const uint32_t mrow = (uint32_t)(sMask[st] >> (ci * 8)) & 0xffu;
        mbar_wait(s_full, gg & 1);
        tc_fence_after();
        uint32_t pp[4][16];
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          uint32_t sv_[2][32];
          tmem_ld_32x32b_x32(tb + h2 * 64, sv_[0]);
          tmem_ld_32x32b_x32(tb + h2 * 64 + 32, sv_[1]);
          tmem_ld_wait();
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) {
            const int c = h2 * 2 + c2;
#pragma unroll
            for (int u2 = 0; u2 < 16; ++u2) {
              const float2 x = fma2(make_float2(__uint_as_float(sv_[c2][2 * u2]), __uint_as_float(sv_[c2][2 * u2 + 1])),
                                    make_float2(scale_log2, scale_log2), make_float2(-l2, -l2));
              const uint32_t pk = pack_bf16x2(ex2(x.x), ex2(x.y));
              pp[c][u2] = (mrow >> (c * 2 + (u2 >> 3))) & 1u ? pk : 0u;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_done);
        mbar_wait(dp_full, gg & 1);
        tc_fence_after();
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          uint32_t dv_[2][32];
          tmem_ld_32x32b_x32(tb + h2 * 64, dv_[0]);
          tmem_ld_32x32b_x32(tb + h2 * 64 + 32, dv_[1]);
          tmem_ld_wait();
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) {
            const int c = h2 * 2 + c2;
            uint32_t dd[16];
#pragma unroll
            for (int u2 = 0; u2 < 16; ++u2) {
              const float2 pf = bf16x2_unpack(pp[c][u2]);
              const float2 t = sub2(make_float2(__uint_as_float(dv_[c2][2 * u2]), __uint_as_float(dv_[c2][2 * u2 + 1])),
                                    make_float2(dl, dl));
              const float2 r2 = mul2(pf, t);
              dd[u2] = pack_bf16x2(r2.x, r2.y);
              eps2 = add2(eps2, bf16x2_unpack(dd[u2]));
            }
            tmem_st_32x32b_x16(tb + c * 16, dd);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(ds_ready);
      }
      g += n;
      // ---- unit drain: dQ rows with the common-mode correction, through the staging tile (64-byte row segments)
      const int row_base = item * s;
      const float eps = eps2.x + eps2.y;
      if (n > 0) {
        if (r < HD) kbar[r] = kb;  // mean key of (item, h), bsattn_prep_kernel
        mbar_wait(acc_full, accn & 1);
        asm volatile("bar.sync %0, 128;" ::"r"(1 + wg) : "memory");
        tc_fence_after();
      }
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        const int col0 = c * 32;
        uint32_t ov[32];
        if (n > 0) {
          tmem_ld_32x32b_x32(t_dq + col0, ov);
          tmem_ld_wait();
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float f[8];
#pragma unroll
          for (int k2 = 0; k2 < 8; ++k2)
            f[k2] = n > 0 ? (__uint_as_float(ov[8 * q + k2]) - eps * kbar[col0 + 8 * q + k2]) * scale : 0.f;
          *reinterpret_cast<uint4*>(stg + lane * L::kStgPitch + 16 * q) =
              make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]), pack_bf16x2(f[6], f[7]));
        }
        __syncwarp();
#pragma unroll
        for (int pass = 0; pass < 4; ++pass) {
          const int rr = pass * 8 + (lane >> 2), piece = lane & 3;
          const int qrow = qt * kAT + quad * 32 + rr;
          if (qrow < s)
            *reinterpret_cast<uint4*>(dq + ((size_t)row_base + qrow) * ld_dq + h * HD + col0 + piece * 8) =
                *reinterpret_cast<const uint4*>(stg + rr * L::kStgPitch + piece * 16);
        }
        __syncwarp();
      }
      if (n > 0) {
        tc_fence_before();
        asm volatile("bar.sync %0, 128;" ::"r"(1 + wg) : "memory");  // TMEM drained, kbar reusable
        if ((threadIdx.x & 127) == 0) mbar_arrive(acc_empty);
        ++accn;
      }
    }
    if ((threadIdx.x & 127) == 0) {
      trace_stamp(8 + 1 + wg);
      trace_put(8 + 3 + wg, ((unsigned long long)nu << 32) | (unsigned)g);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// LX_ATTN_DKDV_DS=0: the entry-alternating dK/dV ping-pong kernel at HD 64 instead of the two-stream one
static bool dkdv_ds() {
  static const bool on = [] { const char* e = getenv("LX_ATTN_DKDV_DS"); return !(e && e[0] == '0'); }();
  return on;
}

// LX_ATTN_DS_DEAL=0: the two-stream kernels alternate a CTA's units between the streams instead of dealing them
static int ds_deal() {
  static const int on = [] { const char* e = getenv("LX_ATTN_DS_DEAL"); return !(e && e[0] == '0'); }();
  return on;
}

// LX_ATTN_DQ_DS=0: the entry-alternating dQ ping-pong kernel at HD 64 instead of the two-stream one
static bool dq_ds() {
  static const bool on = [] { const char* e = getenv("LX_ATTN_DQ_DS"); return !(e && e[0] == '0'); }();
  return on;
}

template <int HD>
static int launch_bwd_tc(const uint16_t* qkv, int ld, int ld_d, const uint16_t* o, const uint16_t* d_o, int ld_o, int n_items, int s,
                         int H, const int32_t* pidx, int item_stride, const int32_t* tables128, int gu, float scale,
                         const float* lse, float* delta, float* ws, uint16_t* dqkv, cudaStream_t st) {
  const int rows = n_items * s;
  LX_REQUIRE(ld_o % 8 == 0, LX_ERR_SHAPE, "attention bwd: O / dO row stride must be a multiple of 8");
  const int nt = (s + kAT - 1) / kAT;
  const int n_units = nt * H * n_items;
  // ws: kbar [n_items * H * HD] floats, then the dK/dV and dQ unit descriptors (int4 [n_units] each)
  float* kbar = ws;
  int4* desc_kv = reinterpret_cast<int4*>(ws + (size_t)n_items * H * HD);
  int4* desc_q = desc_kv + n_units;
  const int nb_delta = (rows * 32 + 255) / 256, nb_kbar = n_items * H, nb_desc = (n_units + 255) / 256;
  launch_k(bsattn_prep_kernel<HD>, nb_delta + nb_kbar + nb_desc, 256, 0, st, reinterpret_cast<const __nv_bfloat16*>(o),
           reinterpret_cast<const __nv_bfloat16*>(d_o), ld_o, rows, s, H, delta, reinterpret_cast<const __nv_bfloat16*>(qkv), ld,
           kbar, pidx, item_stride, tables128, desc_kv, desc_q, n_units, nb_delta, nb_kbar);
  int rc = launch_check("bsattn_prep");
  if (rc) return rc;
  CUtensorMap tm_qkv, tm_do, tm_g, tm_do_g;
  if ((rc = make_tmap_bf16_2d(&tm_qkv, qkv, ld, (uint64_t)rows, ld, 64, kAT))) return rc;
  if ((rc = make_tmap_bf16_2d(&tm_do, d_o, ld_o, (uint64_t)rows, ld_o, 64, kAT))) return rc;
  if ((rc = make_tmap_bf16_2d(&tm_g, qkv, ld, (uint64_t)rows, ld, 64, gu))) return rc;
  if ((rc = make_tmap_bf16_2d(&tm_do_g, d_o, ld_o, (uint64_t)rows, ld_o, 64, gu))) return rc;
  constexpr int smem = AttnBwdSmem<HD>::kTotal;
  static cudaError_t a1 = cudaFuncSetAttribute(bsattn_dkdv_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  static cudaError_t a2 = cudaFuncSetAttribute(bsattn_dq_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  LX_CHECK_CUDA(a1);
  LX_CHECK_CUDA(a2);
  dim3 grid(nt, H, n_items);
  const float sl2 = scale * 1.4426950408889634f;
  // the dK/dV ping-pong kernel's rings + staging fit in shared memory for HD 64; HD 128 keeps the 2-CTA kernel
  static const bool old_bwd = getenv("LX_ATTN_BWD_OLD") != nullptr || AttnDkdvPP<HD>::kTotal > 227 * 1024;
  if (old_bwd) {
    launch_k(bsattn_dkdv_tc_kernel<HD>, grid, 192, smem, st, tm_qkv, tm_do, tm_g, tm_do_g, gu, s, H, H * HD, pidx, item_stride,
             tables128, scale, sl2, lse, delta, reinterpret_cast<__nv_bfloat16*>(dqkv), ld_d);
  } else if (HD == 64 && dkdv_ds()) {
    constexpr int smem_ds = AttnDkdvDs<64>::kTotal;
    static cudaError_t a5 = cudaFuncSetAttribute(bsattn_dkdv_ds_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_ds);
    LX_CHECK_CUDA(a5);
    launch_k(bsattn_dkdv_ds_kernel<64>, std::min(n_units, num_sms()), kDsThreads, smem_ds, st, tm_qkv, tm_do, tm_g, tm_do_g,
             gu, s, H, n_units, pidx, item_stride, tables128, scale, sl2, lse, delta,
             reinterpret_cast<__nv_bfloat16*>(dqkv), ld_d, (const int4*)desc_kv, ds_deal());
  } else {
    constexpr int smem_pp = AttnDkdvPP<HD>::kTotal;
    static cudaError_t a3 = cudaFuncSetAttribute(bsattn_dkdv_pp_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_pp);
    LX_CHECK_CUDA(a3);
    launch_k(bsattn_dkdv_pp_kernel<HD>, std::min(n_units, num_sms()), kBwdThreads, smem_pp, st, tm_qkv, tm_do, tm_g, tm_do_g,
             gu, s, H, n_units, pidx, item_stride, tables128, scale, sl2, lse, delta,
             reinterpret_cast<__nv_bfloat16*>(dqkv), ld_d, (const int4*)desc_kv);
  }
  if ((rc = launch_check("bsattn_dkdv_tc"))) return rc;
  // the dQ ping-pong kernel fits at HD 128 too (1 Q/dO buffer, 2-stage K/V ring: 215 KB), whichever dK/dV ran
  static const bool old_dq = getenv("LX_ATTN_BWD_OLD") != nullptr || AttnDqPP<HD>::kTotal > 227 * 1024;
  if (HD == 64 && !old_dq && dq_ds()) {
    constexpr int smem_dq = AttnDqDs<64>::kTotal;
    static cudaError_t a6 = cudaFuncSetAttribute(bsattn_dq_ds_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_dq);
    LX_CHECK_CUDA(a6);
    launch_k(bsattn_dq_ds_kernel<64>, std::min(n_units, num_sms()), kDsThreads, smem_dq, st, tm_qkv, tm_do, tm_g, gu, s, H,
             n_units, pidx, item_stride, tables128, scale, sl2, lse, delta, reinterpret_cast<__nv_bfloat16*>(dqkv), ld_d,
             (const float*)kbar, (const int4*)desc_q, ds_deal());
  } else if (old_dq) {
    launch_k(bsattn_dq_tc_kernel<HD>, grid, 192, smem, st, tm_qkv, tm_do, tm_g, gu, s, H, H * HD, pidx, item_stride, tables128,
             scale, sl2, lse, delta, reinterpret_cast<__nv_bfloat16*>(dqkv), ld_d, (const float*)kbar);
  } else {
    constexpr int smem_dq = AttnDqPP<HD>::kTotal;
    static cudaError_t a4 = cudaFuncSetAttribute(bsattn_dq_pp_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_dq);
    LX_CHECK_CUDA(a4);
    launch_k(bsattn_dq_pp_kernel<HD>, std::min(n_units, num_sms()), kBwdThreads, smem_dq, st, tm_qkv, tm_do, tm_g, gu, s, H,
             n_units, pidx, item_stride, tables128, scale, sl2, lse, delta, reinterpret_cast<__nv_bfloat16*>(dqkv), ld_d,
             (const float*)kbar, (const int4*)desc_q);
  }
  return launch_check("bsattn_dq_tc");
}

}  // namespace lx

using namespace lx;

extern "C" {

// Debug: route the tcgen05 attention kernels' per-CTA phase stamps to a device buffer of
// [n_ctas][32] uint64 (NULL disables). Not part of the production path.
int lx_debug_set_attn_trace(unsigned long long* buf) {
  LX_CHECK_CUDA(cudaMemcpyToSymbol(g_attn_trace, &buf, sizeof(buf)));
  return 0;
}

int lx_bsattn_bwd_tc(const uint16_t* qkv, int ld, int ld_d, const uint16_t* o, const uint16_t* d_o, int ld_o, int n_items,
                     int s, int H, int hd, const int32_t* pattern_idx, int item_stride, const int32_t* tables128,
                     int gather_rows, float scale, const float* lse, float* delta_ws, float* ws, uint16_t* dqkv,
                     lx_stream_t stream) {
  LX_REQUIRE(gather_rows >= 16 && gather_rows <= 128 && (gather_rows & (gather_rows - 1)) == 0, LX_ERR_LAYOUT,
             "attention bwd: gather_rows %d must be a power of two in [16, 128]", gather_rows);
  LX_REQUIRE(ld >= 3 * H * hd && ld_d >= 3 * H * hd && ld % 8 == 0 && ld_d % 8 == 0 && ld_o % 8 == 0, LX_ERR_SHAPE,
             "attention bwd (tcgen05): qkv / dqkv must be fused [M, >= 3*H*hd] with 16B-aligned rows");
  switch (hd) {
    case 64: return launch_bwd_tc<64>(qkv, ld, ld_d, o, d_o, ld_o, n_items, s, H, pattern_idx, item_stride, tables128, gather_rows, scale, lse, delta_ws, ws, dqkv, stream);
    case 128: return launch_bwd_tc<128>(qkv, ld, ld_d, o, d_o, ld_o, n_items, s, H, pattern_idx, item_stride, tables128, gather_rows, scale, lse, delta_ws, ws, dqkv, stream);
    default: LX_REQUIRE(false, LX_ERR_UNSUPPORTED, "tcgen05 attention: head_dim %d unsupported (64, 128)", hd);
  }
}

int lx_bsattn_fwd_tc(const uint16_t* qkv, int ld, int n_items, int s, int H, int hd, const int32_t* pattern_idx,
                     int item_stride, const int32_t* tables128, int gather_rows, float scale, uint16_t* o, int ldo,
                     float* lse, lx_stream_t stream) {
  LX_REQUIRE(gather_rows >= 16 && gather_rows <= 128 && (gather_rows & (gather_rows - 1)) == 0, LX_ERR_LAYOUT,
             "attention: gather_rows %d must be a power of two in [16, 128]", gather_rows);
  LX_REQUIRE(ld % 8 == 0 && ldo % 8 == 0 && ld >= 3 * H * hd, LX_ERR_SHAPE,
             "attention (tcgen05): qkv must be the fused [M, >= 3*H*hd] projection output (16B-aligned rows)");
  LX_REQUIRE(n_items >= 1 && n_items < 65536 && H >= 1 && H < 65536, LX_ERR_SHAPE, "attention: bad grid");
  switch (hd) {
    case 64: return launch_fwd_tc<64>(qkv, ld, n_items, s, H, pattern_idx, item_stride, tables128, gather_rows, scale, o, ldo, lse, stream);
    case 128: return launch_fwd_tc<128>(qkv, ld, n_items, s, H, pattern_idx, item_stride, tables128, gather_rows, scale, o, ldo, lse, stream);
    default: LX_REQUIRE(false, LX_ERR_UNSUPPORTED, "tcgen05 attention: head_dim %d unsupported (64, 128)", hd);
  }
}

}  // extern "C"
