// K3 on tcgen05 — block-sparse flash attention forward for sm_100a
// (sf/block_sparse.py:47-126 fused: SDD -> sparse softmax -> DSD, sf/model.py:343-353).
//
// One CTA per (128-query tile, head, item), walking the CSR list of its pool
// pattern over 128x128 tiles (64-bit masks of active 16x16 cells):
//   warp 0      TMA producer: Q once, then K_j / V_j tiles into a 2-stage ring
//   warp 1      MMA issuer (lane 0): S_j = Q K_j^T into TMEM (double-buffered),
//               then O += P_{j-1} V_{j-1} (software-pipelined one tile behind)
//   warps 2..5  softmax: thread <-> query row; tcgen05.ld of the S row, -inf on
//               inactive cells, online max/sum (no shuffles: a thread owns its row),
//               O rescale in TMEM, P (bf16) into shared memory in the UMMA K-major
//               SWIZZLE_128B layout, then O / l and the row LSE at the end.
// Q/K are K-major operands (rows of hd), V is the MN-major B operand of P.V
// (rows of hd, K = keys) — all three straight from the projection output by TMA.
#include "common.cuh"
#include "ptx.cuh"

namespace lx {

constexpr int kAT = 128;  // query / key tile edge

// 128x128 tile tables (built by patterns.tables_from_grids(tile=128)): per pattern
// row_ptr[nt+1] csr_col[nt2] csr_lo[nt2] csr_hi[nt2] col_ptr[nt+1] csc_row[nt2] csc_lo[nt2] csc_hi[nt2]
struct Tab128 {
  const int32_t *row_ptr, *csr_col, *csr_lo, *csr_hi, *col_ptr, *csc_row, *csc_lo, *csc_hi;
};
LX_DEV Tab128 tab128(const int32_t* t, int p) {
  const int nt = t[0];
  const int per = 2 * (nt + 1) + 6 * nt * nt;
  const int32_t* b = t + 4 + (size_t)p * per;
  Tab128 v;
  v.row_ptr = b;
  v.csr_col = b + nt + 1;
  v.csr_lo = v.csr_col + nt * nt;
  v.csr_hi = v.csr_lo + nt * nt;
  v.col_ptr = v.csr_hi + nt * nt;
  v.csc_row = v.col_ptr + nt + 1;
  v.csc_lo = v.csc_row + nt * nt;
  v.csc_hi = v.csc_lo + nt * nt;
  return v;
}

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
LX_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

template <int HD>
struct AttnFwdSmem {
  static constexpr int kAtoms = HD / 64;
  static constexpr int kQ = kAtoms * kAT * 128;   // [atoms][128 rows][128B]
  static constexpr int kKV = kAtoms * kAT * 128;  // one K or V tile
  static constexpr int kP = 2 * kAT * 128;        // [2 key atoms][128 rows][128B]
  static constexpr int kOffK = kQ;
  static constexpr int kOffV = kOffK + 2 * kKV;
  static constexpr int kOffP = kOffV + 2 * kKV;
  static constexpr int kOffBar = kOffP + kP;
  static constexpr int kTotal = kOffBar + 256 + 1024;
};

template <int HD>
__global__ void __launch_bounds__(192, 1)
bsattn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, int s, int H, int d_model,
                     const int32_t* __restrict__ pidx, int item_stride, const int32_t* __restrict__ tables,
                     float scale_log2, __nv_bfloat16* __restrict__ o, int ldo, float* __restrict__ lse) {
  using L = AttnFwdSmem<HD>;
  constexpr int A = L::kAtoms;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::kOffBar);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;    // [2]
  uint64_t* s_free = bars + 7;    // [2]
  uint64_t* p_full = bars + 9;
  uint64_t* o_done = bars + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int qt = blockIdx.x, h = blockIdx.y, item = blockIdx.z;
  const uint32_t warp = warp_id(), lane = lane_id();
  const Tab128 tv = tab128(tables, __ldg(pidx + item * item_stride + h));
  const int e0 = __ldg(tv.row_ptr + qt), e1 = __ldg(tv.row_ptr + qt + 1);
  const int n = e1 - e0;
  const int row_base = item * s;  // first token row of this item in qkv

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(kv_full + i, 1);
      mbar_init(kv_empty + i, 1);
      mbar_init(s_full + i, 1);
      mbar_init(s_free + i, 4);
    }
    mbar_init(p_full, 4);
    mbar_init(o_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_o = tmem + 2 * kAT;  // O accumulator columns [256, 256+HD)

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      const int qcol = h * HD, kcol = d_model + h * HD, vcol = 2 * d_model + h * HD;
      mbar_arrive_expect_tx(q_full, L::kQ);
      for (int a = 0; a < A; ++a) tma_load_2d(sm + a * kAT * 128, &tm_qkv, q_full, qcol + a * 64, row_base + qt * kAT);
      for (int e = 0; e < n; ++e) {
        const int st = e & 1;
        mbar_wait(kv_empty + st, ((e >> 1) & 1) ^ 1);
        const int j = __ldg(tv.csr_col + e0 + e);
        mbar_arrive_expect_tx(kv_full + st, 2 * L::kKV);
        uint8_t* sk = sm + L::kOffK + st * L::kKV;
        uint8_t* sv = sm + L::kOffV + st * L::kKV;
        for (int a = 0; a < A; ++a) {
          tma_load_2d(sk + a * kAT * 128, &tm_qkv, kv_full + st, kcol + a * 64, row_base + j * kAT);
          tma_load_2d(sv + a * kAT * 128, &tm_qkv, kv_full + st, vcol + a * 64, row_base + j * kAT);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc_s = make_idesc_bf16(kAT, kAT, false, false);  // S = Q K^T: both K-major
      const uint32_t idesc_o = make_idesc_bf16(kAT, HD, false, true);    // O += P V: V is MN-major
      const uint32_t sq = smem_u32(sm), sp = smem_u32(sm + L::kOffP);
      mbar_wait(q_full, 0);
      auto issue_pv = [&](int e) {  // O += P_e V_e
        const int st = e & 1;
        mbar_wait(p_full, e & 1);
        tc_fence_after();
        const uint32_t sv = smem_u32(sm + L::kOffV + st * L::kKV);
        for (int kk = 0; kk < kAT / 16; ++kk) {
          const uint64_t da = make_sdesc(sp + (kk >> 2) * (kAT * 128) + (kk & 3) * 32, 16, 1024);
          const uint64_t db = make_sdesc(sv + kk * 16 * 128, kAT * 128, 1024);
          mma_bf16_ss(t_o, da, db, idesc_o, (e | kk) != 0);
        }
        mma_commit(o_done);
        mma_commit(kv_empty + st);
      };
      for (int e = 0; e < n; ++e) {
        const int st = e & 1;
        mbar_wait(kv_full + st, (e >> 1) & 1);
        mbar_wait(s_free + st, ((e >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t sk = smem_u32(sm + L::kOffK + st * L::kKV);
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * (kAT * 128) + (kk & 3) * 32;
          mma_bf16_ss(tmem + st * kAT, make_sdesc(sq + off, 16, 1024), make_sdesc(sk + off, 16, 1024), idesc_s, kk != 0);
        }
        mma_commit(s_full + st);
        if (e >= 1) issue_pv(e - 1);
      }
      if (n >= 1) issue_pv(n - 1);
    }
  } else {
    // ---------------------------------------------------------------- softmax warps
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // query row within the tile
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    float m = -INFINITY, l = 0.f;
    uint8_t* prow = sm + L::kOffP + r * 128;
    for (int e = 0; e < n; ++e) {
      const int st = e & 1;
      const uint32_t lo = (uint32_t)__ldg(tv.csr_lo + e0 + e), hi = (uint32_t)__ldg(tv.csr_hi + e0 + e);
      const uint64_t mask = ((uint64_t)hi << 32) | lo;
      const uint32_t mrow = (uint32_t)(mask >> ((r >> 4) * 8)) & 0xffu;  // active 16-key groups of this row
      mbar_wait(s_full + st, (e >> 1) & 1);
      tc_fence_after();
      uint32_t sr[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(tmem + lane_base + st * kAT + c * 32, sr[c]);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_free + st);
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const bool on = (mrow >> (c * 2 + (i >> 4))) & 1u;
          float v = on ? __uint_as_float(sr[c][i]) * scale_log2 : -INFINITY;
          sr[c][i] = __float_as_uint(v);
          mx = fmaxf(mx, v);
        }
      const float m_new = fmaxf(m, mx);
      const float use = m_new == -INFINITY ? 0.f : m_new;
      const float alpha = exp2f(m - use);
      m = m_new;
      float rs = 0.f;
      uint32_t pk[4][16];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float p0 = exp2f(__uint_as_float(sr[c][2 * i]) - use);
          const float p1 = exp2f(__uint_as_float(sr[c][2 * i + 1]) - use);
          rs += p0 + p1;
          pk[c][i] = pack_bf16x2(p0, p1);
        }
      l = l * alpha + rs;
      // P_{e-1} V_{e-1} must be complete before P is overwritten and O rescaled
      if (e >= 1) {
        mbar_wait(o_done, (e - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
          for (int c = 0; c < HD / 32; ++c) {
            uint32_t ov[32];
            tmem_ld_32x32b_x32(t_o + lane_base + c * 32, ov);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
            tmem_st_32x32b_x32(t_o + lane_base + c * 32, ov);
          }
          tmem_st_wait();
        }
      }
      // P row -> shared memory, K-major SWIZZLE_128B: 16B chunk cc of row r at (cc ^ (r & 7))
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int chunk = c * 4 + q;  // 16B chunk over the 128 keys (8 keys each)
          const int atom = chunk >> 3, cc = chunk & 7;
          *reinterpret_cast<uint4*>(prow + atom * (kAT * 128) + ((cc ^ (r & 7)) << 4)) =
              make_uint4(pk[c][4 * q], pk[c][4 * q + 1], pk[c][4 * q + 2], pk[c][4 * q + 3]);
        }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    // epilogue: O / l -> bf16 rows, LSE
    if (n >= 1) {
      mbar_wait(o_done, (n - 1) & 1);
      tc_fence_after();
    }
    const int row = qt * kAT + r;
    const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t ov[32];
      tmem_ld_32x32b_x32(t_o + lane_base + c * 32, ov);
      tmem_ld_wait();
      if (row < s) {
        __nv_bfloat16* op = o + ((size_t)row_base + row) * ldo + h * HD + c * 32;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          *reinterpret_cast<uint4*>(op + 8 * i) = make_uint4(
              pack_bf16x2(__uint_as_float(ov[8 * i]) * inv, __uint_as_float(ov[8 * i + 1]) * inv),
              pack_bf16x2(__uint_as_float(ov[8 * i + 2]) * inv, __uint_as_float(ov[8 * i + 3]) * inv),
              pack_bf16x2(__uint_as_float(ov[8 * i + 4]) * inv, __uint_as_float(ov[8 * i + 5]) * inv),
              pack_bf16x2(__uint_as_float(ov[8 * i + 6]) * inv, __uint_as_float(ov[8 * i + 7]) * inv));
      }
    }
    if (row < s) lse[((size_t)item * H + h) * s + row] = (m + log2f(l)) * 0.6931471805599453f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int HD>
static int launch_fwd_tc(const uint16_t* qkv, int ld, int n_items, int s, int H, const int32_t* pidx, int item_stride,
                         const int32_t* tables128, float scale, uint16_t* o, int ldo, float* lse, cudaStream_t st) {
  CUtensorMap tm;
  int rc = make_tmap_bf16_2d(&tm, qkv, ld, (uint64_t)n_items * s, ld, 64, kAT);
  if (rc) return rc;
  constexpr int smem = AttnFwdSmem<HD>::kTotal;
  static cudaError_t attr = cudaFuncSetAttribute(bsattn_fwd_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  LX_CHECK_CUDA(attr);
  dim3 grid((s + kAT - 1) / kAT, H, n_items);
  bsattn_fwd_tc_kernel<HD><<<grid, 192, smem, st>>>(tm, s, H, ld / 3, pidx, item_stride, tables128, scale * 1.4426950408889634f,
                                                    reinterpret_cast<__nv_bfloat16*>(o), ldo, lse);
  return launch_check("bsattn_fwd_tc");
}

// ============================================================================ backward
// Shared pieces: smem tiles of 128 rows x HD (A atoms of [128 rows x 128B]), used either as a
// K-major operand (rows = M/N, K = hd) or as an MN-major B operand (K = rows, N = hd).
LX_DEV uint64_t desc_kmajor(uint32_t base, int kk) {  // K = hd step kk (16 elements)
  return make_sdesc(base + (kk >> 2) * (kAT * 128) + (kk & 3) * 32, 16, 1024);
}
LX_DEV uint64_t desc_mnmajor(uint32_t base, int kk) {  // K = rows step kk (16 rows), N = hd atoms at 16KB
  return make_sdesc(base + kk * 16 * 128, kAT * 128, 1024);
}
// bf16x8 chunk (16B) of a 128-wide K-major SWIZZLE_128B row written by the thread owning row r
LX_DEV void st_swz_chunk(uint8_t* tile, int r, int chunk, uint4 v) {
  const int atom = chunk >> 3, cc = chunk & 7;
  *reinterpret_cast<uint4*>(tile + atom * (kAT * 128) + r * 128 + ((cc ^ (r & 7)) << 4)) = v;
}

template <int HD>
struct AttnBwdSmem {
  static constexpr int kTile = (HD / 64) * kAT * 128;  // 128 rows x HD
  static constexpr int kPS = 2 * kAT * 128;            // 128 x 128 bf16 operand
  // dkdv: [K | V | 2 x (Q | dO) | P^T | dS^T | lse2[2][128] | delta[2][128]]
  static constexpr int kSt = HD == 128 ? 1 : 2;  // Q/dO (dkdv) or K/V (dq) ring stages
  static constexpr int kOffQ = 2 * kTile;
  static constexpr int kOffP = kOffQ + 2 * kSt * kTile;
  static constexpr int kOffDS = kOffP + kPS;
  static constexpr int kOffL = kOffDS + kPS;
  static constexpr int kOffBar = kOffL + 4 * kAT * 4;
  static constexpr int kTotal = kOffBar + 256 + 1024;
};

template <int HD>
__global__ void __launch_bounds__(192, 1)
bsattn_dkdv_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do, int s, int H,
                      int d_model, const int32_t* __restrict__ pidx, int item_stride, const int32_t* __restrict__ tables,
                      float scale, float scale_log2, const float* __restrict__ lse, const float* __restrict__ delta,
                      __nv_bfloat16* __restrict__ dkv, int ld_dkv, float* __restrict__ ksum) {
  using L = AttnBwdSmem<HD>;
  constexpr int A = HD / 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::kOffBar);
  uint64_t* kv_full = bars + 0;
  uint64_t* qd_full = bars + 1;   // [2]
  uint64_t* qd_empty = bars + 3;  // [2]
  uint64_t* st_full = bars + 5;
  uint64_t* p_ready = bars + 6;
  uint64_t* done = bars + 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);
  float* sL = reinterpret_cast<float*>(sm + L::kOffL);  // [2][128] lse * log2(e)
  float* sD = sL + 2 * kAT;                             // [2][128] delta

  const int kt = blockIdx.x, h = blockIdx.y, item = blockIdx.z;
  const uint32_t warp = warp_id(), lane = lane_id();
  const Tab128 tv = tab128(tables, __ldg(pidx + item * item_stride + h));
  const int e0 = __ldg(tv.col_ptr + kt), n = __ldg(tv.col_ptr + kt + 1) - e0;
  const int row_base = item * s;
  const float* lse_b = lse + ((size_t)item * H + h) * s;
  const float* del_b = delta + ((size_t)item * H + h) * s;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
    mbar_init(kv_full, 1);
    for (int i = 0; i < 2; ++i) { mbar_init(qd_full + i, 1); mbar_init(qd_empty + i, 1); }
    mbar_init(st_full, 1);
    mbar_init(p_ready, 4);
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_s = tmem, t_dp = tmem + kAT, t_dv = tmem + 2 * kAT, t_dk = tmem + 2 * kAT + HD;

  if (warp == 0) {
    if (lane == 0) {
      const int qcol = h * HD, kcol = d_model + h * HD, vcol = 2 * d_model + h * HD;
      mbar_arrive_expect_tx(kv_full, 2 * L::kTile);
      for (int a = 0; a < A; ++a) {
        tma_load_2d(sm + a * kAT * 128, &tm_qkv, kv_full, kcol + a * 64, row_base + kt * kAT);
        tma_load_2d(sm + L::kTile + a * kAT * 128, &tm_qkv, kv_full, vcol + a * 64, row_base + kt * kAT);
      }
      for (int e = 0; e < n; ++e) {
        const int st = e % L::kSt;
        mbar_wait(qd_empty + st, ((e / L::kSt) & 1) ^ 1);
        const int i = __ldg(tv.csc_row + e0 + e);
        uint8_t* sq = sm + L::kOffQ + st * 2 * L::kTile;
        mbar_arrive_expect_tx(qd_full + st, 2 * L::kTile);
        for (int a = 0; a < A; ++a) {
          tma_load_2d(sq + a * kAT * 128, &tm_qkv, qd_full + st, qcol + a * 64, row_base + i * kAT);
          tma_load_2d(sq + L::kTile + a * kAT * 128, &tm_do, qd_full + st, h * HD + a * 64, row_base + i * kAT);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_s = make_idesc_bf16(kAT, kAT, false, false);  // S^T, dP^T: B K-major
      const uint32_t id_g = make_idesc_bf16(kAT, HD, false, true);    // dV, dK: B MN-major
      const uint32_t sk = smem_u32(sm), sv = sk + L::kTile;
      const uint32_t sp = smem_u32(sm + L::kOffP), sds = smem_u32(sm + L::kOffDS);
      mbar_wait(kv_full, 0);
      for (int e = 0; e < n; ++e) {
        const int st = e % L::kSt;
        const uint32_t sq = smem_u32(sm + L::kOffQ + st * 2 * L::kTile), sdo = sq + L::kTile;
        mbar_wait(qd_full + st, (e / L::kSt) & 1);
        tc_fence_after();
        for (int kk = 0; kk < HD / 16; ++kk) mma_bf16_ss(t_s, desc_kmajor(sk, kk), desc_kmajor(sq, kk), id_s, kk != 0);
        for (int kk = 0; kk < HD / 16; ++kk) mma_bf16_ss(t_dp, desc_kmajor(sv, kk), desc_kmajor(sdo, kk), id_s, kk != 0);
        mma_commit(st_full);
        mbar_wait(p_ready, e & 1);
        tc_fence_after();
        for (int kk = 0; kk < kAT / 16; ++kk) {
          const uint32_t off = (kk >> 2) * (kAT * 128) + (kk & 3) * 32;
          mma_bf16_ss(t_dv, make_sdesc(sp + off, 16, 1024), desc_mnmajor(sdo, kk), id_g, (e | kk) != 0);
          mma_bf16_ss(t_dk, make_sdesc(sds + off, 16, 1024), desc_mnmajor(sq, kk), id_g, (e | kk) != 0);
        }
        mma_commit(qd_empty + st);
      }
      mma_commit(done);
    }
  } else {
    const int quad = warp & 3;
    const int kr = quad * 32 + lane;  // key row within the tile
    const int ep_tid = threadIdx.x - 64;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    uint8_t* tP = sm + L::kOffP;
    uint8_t* tDS = sm + L::kOffDS;
    for (int e = 0; e < n; ++e) {
      const int st = e & 1;  // lse/delta slot: entries e and e+2 are separated by the named barrier of e+1
      const int i = __ldg(tv.csc_row + e0 + e);
      {
        const int q = i * kAT + ep_tid;
        sL[st * kAT + ep_tid] = q < s ? __ldg(lse_b + q) * 1.4426950408889634f : INFINITY;
        sD[st * kAT + ep_tid] = q < s ? __ldg(del_b + q) : 0.f;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const uint32_t lo = (uint32_t)__ldg(tv.csc_lo + e0 + e), hi = (uint32_t)__ldg(tv.csc_hi + e0 + e);
      const uint64_t mask = ((uint64_t)hi << 32) | lo;
      const int cj = kr >> 4;
      mbar_wait(st_full, e & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t sv_[32], dv_[32];
        tmem_ld_32x32b_x32(t_s + lane_base + c * 32, sv_);
        tmem_ld_32x32b_x32(t_dp + lane_base + c * 32, dv_);
        tmem_ld_wait();
        uint32_t pp[16], dd[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          float p2[2], d2[2];
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            const int qi = c * 32 + 2 * u + w;
            const bool on = (mask >> ((qi >> 4) * 8 + cj)) & 1ull;
            const float p = on ? exp2f(__uint_as_float(sv_[2 * u + w]) * scale_log2 - sL[st * kAT + qi]) : 0.f;
            p2[w] = p;
            d2[w] = p * (__uint_as_float(dv_[2 * u + w]) - sD[st * kAT + qi]);
          }
          pp[u] = pack_bf16x2(p2[0], p2[1]);
          dd[u] = pack_bf16x2(d2[0], d2[1]);
        }
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          st_swz_chunk(tP, kr, c * 4 + q4, make_uint4(pp[4 * q4], pp[4 * q4 + 1], pp[4 * q4 + 2], pp[4 * q4 + 3]));
          st_swz_chunk(tDS, kr, c * 4 + q4, make_uint4(dd[4 * q4], dd[4 * q4 + 1], dd[4 * q4 + 2], dd[4 * q4 + 3]));
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_ready);
    }
    mbar_wait(done, 0);
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
        if (key < s && n > 0) {
          __nv_bfloat16* op = dkv + ((size_t)row_base + key) * ld_dkv + (which + 1) * d_model + h * HD + c * 32;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            *reinterpret_cast<uint4*>(op + 8 * i) = make_uint4(
                pack_bf16x2(__uint_as_float(ov[8 * i]) * mul, __uint_as_float(ov[8 * i + 1]) * mul),
                pack_bf16x2(__uint_as_float(ov[8 * i + 2]) * mul, __uint_as_float(ov[8 * i + 3]) * mul),
                pack_bf16x2(__uint_as_float(ov[8 * i + 4]) * mul, __uint_as_float(ov[8 * i + 5]) * mul),
                pack_bf16x2(__uint_as_float(ov[8 * i + 6]) * mul, __uint_as_float(ov[8 * i + 7]) * mul));
        } else if (key < s) {  // no query tile attends to this key tile: zero gradient
          __nv_bfloat16* op = dkv + ((size_t)row_base + key) * ld_dkv + (which + 1) * d_model + h * HD + c * 32;
#pragma unroll
          for (int i = 0; i < 4; ++i) *reinterpret_cast<uint4*>(op + 8 * i) = make_uint4(0u, 0u, 0u, 0u);
        }
      }
    }
    // column sums of this key tile (keys < s) -> ksum[item, h, kt, :], the common mode the dQ
    // kernel removes (see bsattn_dq_tc_kernel)
    {
      constexpr int G = 128 / HD;  // row groups
      const int col = ep_tid % HD, grp = ep_tid / HD, rows = kAT / G;
      const uint8_t* katom = sm + (col >> 6) * (kAT * 128);
      float acc = 0.f;
      for (int rr = 0; rr < rows; ++rr) {
        const int r = grp * rows + rr;
        if (kt * kAT + r < s) {
          const __nv_bfloat16 kv =
              *reinterpret_cast<const __nv_bfloat16*>(katom + r * 128 + ((((col & 63) >> 3) ^ (r & 7)) << 4) + (col & 7) * 2);
          acc += __bfloat162float(kv);
        }
      }
      sL[ep_tid] = acc;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (grp == 0) {
        for (int g2 = 1; g2 < G; ++g2) acc += sL[g2 * HD + col];
        ksum[(((size_t)item * H + h) * gridDim.x + kt) * HD + col] = acc;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int HD>
__global__ void __launch_bounds__(192, 1)
bsattn_dq_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do, int s, int H,
                    int d_model, const int32_t* __restrict__ pidx, int item_stride, const int32_t* __restrict__ tables,
                    float scale, float scale_log2, const float* __restrict__ lse, const float* __restrict__ delta,
                    __nv_bfloat16* __restrict__ dq, int ld_dq, const float* __restrict__ ksum) {
  using L = AttnBwdSmem<HD>;  // [Q | dO | 2 x (K | V) | - | dS]
  constexpr int A = HD / 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::kOffBar);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* st_full = bars + 5;
  uint64_t* p_ready = bars + 6;
  uint64_t* done = bars + 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

  const int qt = blockIdx.x, h = blockIdx.y, item = blockIdx.z;
  const uint32_t warp = warp_id(), lane = lane_id();
  const Tab128 tv = tab128(tables, __ldg(pidx + item * item_stride + h));
  const int e0 = __ldg(tv.row_ptr + qt), n = __ldg(tv.row_ptr + qt + 1) - e0;
  const int row_base = item * s;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) { mbar_init(kv_full + i, 1); mbar_init(kv_empty + i, 1); }
    mbar_init(st_full, 1);
    mbar_init(p_ready, 4);
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_s = tmem, t_dp = tmem + kAT, t_dq = tmem + 2 * kAT;

  if (warp == 0) {
    if (lane == 0) {
      const int qcol = h * HD, kcol = d_model + h * HD, vcol = 2 * d_model + h * HD;
      mbar_arrive_expect_tx(q_full, 2 * L::kTile);
      for (int a = 0; a < A; ++a) {
        tma_load_2d(sm + a * kAT * 128, &tm_qkv, q_full, qcol + a * 64, row_base + qt * kAT);
        tma_load_2d(sm + L::kTile + a * kAT * 128, &tm_do, q_full, h * HD + a * 64, row_base + qt * kAT);
      }
      for (int e = 0; e < n; ++e) {
        const int st = e % L::kSt;
        mbar_wait(kv_empty + st, ((e / L::kSt) & 1) ^ 1);
        const int j = __ldg(tv.csr_col + e0 + e);
        uint8_t* skv = sm + L::kOffQ + st * 2 * L::kTile;
        mbar_arrive_expect_tx(kv_full + st, 2 * L::kTile);
        for (int a = 0; a < A; ++a) {
          tma_load_2d(skv + a * kAT * 128, &tm_qkv, kv_full + st, kcol + a * 64, row_base + j * kAT);
          tma_load_2d(skv + L::kTile + a * kAT * 128, &tm_qkv, kv_full + st, vcol + a * 64, row_base + j * kAT);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_s = make_idesc_bf16(kAT, kAT, false, false);
      const uint32_t id_g = make_idesc_bf16(kAT, HD, false, true);
      const uint32_t sq = smem_u32(sm), sdo = sq + L::kTile, sds = smem_u32(sm + L::kOffDS);
      mbar_wait(q_full, 0);
      for (int e = 0; e < n; ++e) {
        const int st = e % L::kSt;
        const uint32_t sk = smem_u32(sm + L::kOffQ + st * 2 * L::kTile), sv = sk + L::kTile;
        mbar_wait(kv_full + st, (e / L::kSt) & 1);
        tc_fence_after();
        for (int kk = 0; kk < HD / 16; ++kk) mma_bf16_ss(t_s, desc_kmajor(sq, kk), desc_kmajor(sk, kk), id_s, kk != 0);
        for (int kk = 0; kk < HD / 16; ++kk) mma_bf16_ss(t_dp, desc_kmajor(sdo, kk), desc_kmajor(sv, kk), id_s, kk != 0);
        mma_commit(st_full);
        mbar_wait(p_ready, e & 1);
        tc_fence_after();
        for (int kk = 0; kk < kAT / 16; ++kk) {
          const uint32_t off = (kk >> 2) * (kAT * 128) + (kk & 3) * 32;
          mma_bf16_ss(t_dq, make_sdesc(sds + off, 16, 1024), desc_mnmajor(sk, kk), id_g, (e | kk) != 0);
        }
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
    uint8_t* tDS = sm + L::kOffDS;
    const int ci = r >> 4;
    // eps = row sum of the bf16 dS fed to the MMA. Exactly, sum_j dS_ij = 0 (softmax Jacobian), so
    // dq_i = sum_j dS_ij (k_j - kbar) for any kbar; rounding leaves eps != 0, whose product with
    // the keys' common mode kbar is removed in the epilogue.
    float eps = 0.f;
    for (int e = 0; e < n; ++e) {
      const uint32_t lo = (uint32_t)__ldg(tv.csr_lo + e0 + e), hi = (uint32_t)__ldg(tv.csr_hi + e0 + e);
      const uint32_t mrow = (uint32_t)((((uint64_t)hi << 32) | lo) >> (ci * 8)) & 0xffu;
      mbar_wait(st_full, e & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t sv_[32], dv_[32];
        tmem_ld_32x32b_x32(t_s + lane_base + c * 32, sv_);
        tmem_ld_32x32b_x32(t_dp + lane_base + c * 32, dv_);
        tmem_ld_wait();
        uint32_t dd[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          float d2[2];
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            const int ki = c * 32 + 2 * u + w;
            const bool on = (mrow >> (ki >> 4)) & 1u;
            const float p = on ? exp2f(__uint_as_float(sv_[2 * u + w]) * scale_log2 - l2) : 0.f;
            d2[w] = p * (__uint_as_float(dv_[2 * u + w]) - dl);
          }
          dd[u] = pack_bf16x2(d2[0], d2[1]);
          const __nv_bfloat162 rb = *reinterpret_cast<const __nv_bfloat162*>(&dd[u]);
          eps += __low2float(rb) + __high2float(rb);
        }
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
          st_swz_chunk(tDS, r, c * 4 + q4, make_uint4(dd[4 * q4], dd[4 * q4 + 1], dd[4 * q4 + 2], dd[4 * q4 + 3]));
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_ready);
    }
    // kbar = mean over the item's keys (column sums from the dK/dV kernel)
    float* kbar = reinterpret_cast<float*>(sm + L::kOffP);
    if (r < HD) {
      const float* ks = ksum + ((size_t)item * H + h) * gridDim.x * HD + r;
      float acc = 0.f;
      for (int t = 0; t < (int)gridDim.x; ++t) acc += __ldg(ks + t * HD);
      kbar[r] = acc / (float)s;
    }
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
        for (int i = 0; i < 32; ++i) f[i] = (__uint_as_float(ov[i]) - eps * kbar[c * 32 + i]) * scale;
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
    tmem_dealloc<512>(tmem);
  }
}

// delta[item, h, row] = sum_c dO[row, c] * O[row, c]  (== rowsum(dP * P), sf/block_sparse.py:102-113)
__global__ void bsattn_delta_tc_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ d_o, int ld,
                                       int n_rows_total, int s, int H, int hd, float* __restrict__ delta) {
  const int warp_g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp_g >= n_rows_total * H) return;
  const int row = warp_g / H, h = warp_g % H;
  const __nv_bfloat16* a = o + (size_t)row * ld + h * hd;
  const __nv_bfloat16* b = d_o + (size_t)row * ld + h * hd;
  float acc = 0.f;
  for (int c = lane * 2; c < hd; c += 64) {
    __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162*>(a + c);
    __nv_bfloat162 y = *reinterpret_cast<const __nv_bfloat162*>(b + c);
    acc += __bfloat162float(x.x) * __bfloat162float(y.x) + __bfloat162float(x.y) * __bfloat162float(y.y);
  }
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) delta[((size_t)(row / s) * H + h) * s + row % s] = acc;
}

template <int HD>
static int launch_bwd_tc(const uint16_t* qkv, int ld, const uint16_t* o, const uint16_t* d_o, int ld_o, int n_items, int s,
                         int H, const int32_t* pidx, int item_stride, const int32_t* tables128, float scale,
                         const float* lse, float* delta, float* ksum, uint16_t* dqkv, cudaStream_t st) {
  const int rows = n_items * s;
  bsattn_delta_tc_kernel<<<(rows * H * 32 + 255) / 256, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(o),
                                                                        reinterpret_cast<const __nv_bfloat16*>(d_o), ld_o,
                                                                        rows, s, H, HD, delta);
  int rc = launch_check("bsattn_delta_tc");
  if (rc) return rc;
  CUtensorMap tm_qkv, tm_do;
  if ((rc = make_tmap_bf16_2d(&tm_qkv, qkv, ld, (uint64_t)rows, ld, 64, kAT))) return rc;
  if ((rc = make_tmap_bf16_2d(&tm_do, d_o, ld_o, (uint64_t)rows, ld_o, 64, kAT))) return rc;
  constexpr int smem = AttnBwdSmem<HD>::kTotal;
  static cudaError_t a1 = cudaFuncSetAttribute(bsattn_dkdv_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  static cudaError_t a2 = cudaFuncSetAttribute(bsattn_dq_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  LX_CHECK_CUDA(a1);
  LX_CHECK_CUDA(a2);
  dim3 grid((s + kAT - 1) / kAT, H, n_items);
  const float sl2 = scale * 1.4426950408889634f;
  bsattn_dkdv_tc_kernel<HD><<<grid, 192, smem, st>>>(tm_qkv, tm_do, s, H, ld / 3, pidx, item_stride, tables128, scale, sl2,
                                                     lse, delta, reinterpret_cast<__nv_bfloat16*>(dqkv), ld, ksum);
  if ((rc = launch_check("bsattn_dkdv_tc"))) return rc;
  bsattn_dq_tc_kernel<HD><<<grid, 192, smem, st>>>(tm_qkv, tm_do, s, H, ld / 3, pidx, item_stride, tables128, scale, sl2,
                                                   lse, delta, reinterpret_cast<__nv_bfloat16*>(dqkv), ld, ksum);
  return launch_check("bsattn_dq_tc");
}

}  // namespace lx

using namespace lx;

extern "C" {

int lx_bsattn_bwd_tc(const uint16_t* qkv, int ld, const uint16_t* o, const uint16_t* d_o, int ld_o, int n_items, int s,
                     int H, int hd, const int32_t* pattern_idx, int item_stride, const int32_t* tables128, float scale,
                     const float* lse, float* delta_ws, float* ksum_ws, uint16_t* dqkv, lx_stream_t stream) {
  LX_REQUIRE(ld == 3 * H * hd && ld % 8 == 0 && ld_o % 8 == 0, LX_ERR_SHAPE,
             "attention bwd (tcgen05): qkv / dqkv must be fused [M, 3*H*hd]");
  switch (hd) {
    case 64: return launch_bwd_tc<64>(qkv, ld, o, d_o, ld_o, n_items, s, H, pattern_idx, item_stride, tables128, scale, lse, delta_ws, ksum_ws, dqkv, stream);
    case 128: return launch_bwd_tc<128>(qkv, ld, o, d_o, ld_o, n_items, s, H, pattern_idx, item_stride, tables128, scale, lse, delta_ws, ksum_ws, dqkv, stream);
    default: LX_REQUIRE(false, LX_ERR_UNSUPPORTED, "tcgen05 attention: head_dim %d unsupported (64, 128)", hd);
  }
}

int lx_bsattn_fwd_tc(const uint16_t* qkv, int ld, int n_items, int s, int H, int hd, const int32_t* pattern_idx,
                     int item_stride, const int32_t* tables128, float scale, uint16_t* o, int ldo, float* lse,
                     lx_stream_t stream) {
  LX_REQUIRE(ld % 8 == 0 && ldo % 8 == 0 && ld == 3 * H * hd, LX_ERR_SHAPE,
             "attention (tcgen05): qkv must be the fused [M, 3*H*hd] projection output");
  LX_REQUIRE(n_items >= 1 && n_items < 65536 && H >= 1 && H < 65536, LX_ERR_SHAPE, "attention: bad grid");
  switch (hd) {
    case 64: return launch_fwd_tc<64>(qkv, ld, n_items, s, H, pattern_idx, item_stride, tables128, scale, o, ldo, lse, stream);
    case 128: return launch_fwd_tc<128>(qkv, ld, n_items, s, H, pattern_idx, item_stride, tables128, scale, o, ldo, lse, stream);
    default: LX_REQUIRE(false, LX_ERR_UNSUPPORTED, "tcgen05 attention: head_dim %d unsupported (64, 128)", hd);
  }
}

}  // extern "C"
