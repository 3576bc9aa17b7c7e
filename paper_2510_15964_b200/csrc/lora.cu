// Skinny rank-r LoRA kernels of the neuron-sparse MLP and the attention
// projections (sf/model.py:292-304,380-395, sf/autograd.py:48-58,97-123).
// All are single HBM passes over one bf16 activation tensor, optionally
// restricted to an item's packed active columns.
//
//   rowproj : Y[M, r]   = scale * X[M, K] W           (x A1, a A2[cols], dO B2^T, dz B1[:,cols]^T)
//   colgrad : G[q, c]   = scale * sum_rows P[row, q] X[row, c]   (dB1[:,cols], dA2[cols], dB2, dA1)
//   colsum  : g[c]      = sum_rows X[row, c]                     (BitFit db1[cols], db2)
//
// rowproj: a CTA owns 32 rows of one item and streams K in 512-wide chunks;
// the chunk of W (gathered through the item's block ids) is staged once in
// shared memory with coalesced loads and reused by all 32 rows; each lane
// consumes 16 contiguous bf16 per row per chunk (two 16B loads).
// colgrad: a CTA owns 256 columns x 256 rows; a lane owns 8 adjacent
// columns (one 16B load per row), warps split the rows and reduce through
// shared memory; one partial per (item, 256-row split) is written and a fixed-
// order final pass sums partials over splits and items (deterministic).
#include "common.cuh"
#include "ptx.cuh"

namespace lx {

constexpr int kRpRows = 32;     // rows per CTA
constexpr int kRpChunk = 512;   // K per staged chunk
constexpr int kRpMaxR = 16;

template <int R>
__global__ void __launch_bounds__(256) rowproj_kernel(const __nv_bfloat16* __restrict__ x, int ldx, int s, int K,
                                                      const float* __restrict__ w, long long w_sk, long long w_sq, int r,
                                                      float scale, const int32_t* __restrict__ counts,
                                                      const int32_t* __restrict__ ids, int ids_stride, int blk,
                                                      float* __restrict__ y, int ldy) {
  // staged W chunk [kRpChunk][RS]: RS = R + 4 so the 8 lanes of a quarter-warp, reading 8 consecutive
  // k-rows with float4 loads, hit 8 distinct 4-bank groups (conflict-free)
  constexpr int RS = R + 4;
  __shared__ __align__(16) float s_w[kRpChunk * RS];
  const int item = blockIdx.y;
  const int row_base = blockIdx.x * kRpRows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k_item = counts ? __ldg(counts + item) * blk : K;
  const int32_t* my_ids = ids ? ids + (size_t)item * ids_stride : nullptr;
  constexpr int kRowsPerWarp = kRpRows / 8;
  float acc[kRowsPerWarp][R];
#pragma unroll
  for (int a = 0; a < kRowsPerWarp; ++a)
#pragma unroll
    for (int q = 0; q < R; ++q) acc[a][q] = 0.f;
  const bool k_fast = (w_sk == 1);  // pick the staging order that is coalesced in global memory
  for (int k0 = 0; k0 < k_item; k0 += kRpChunk) {
    __syncthreads();
    for (int e = threadIdx.x; e < kRpChunk * R; e += 256) {
      int kk, q;
      if (k_fast) { q = e / kRpChunk; kk = e % kRpChunk; } else { kk = e / R; q = e % R; }
      const int k = k0 + kk;
      float val = 0.f;
      if (k < k_item && q < r) {
        long long ko = my_ids ? (long long)__ldg(my_ids + k / blk) * blk + k % blk : k;
        val = __ldg(w + ko * w_sk + q * w_sq);
      }
      s_w[kk * RS + q] = val;
    }
    __syncthreads();
    // lane l takes k = k0 + e*32 + l (e = 0..15): coalesced 64B x loads per warp step, and the
    // W rows read by a quarter-warp are 8 consecutive rows at stride RS (conflict-free)
    const int kmax = min(kRpChunk, k_item - k0);
#pragma unroll
    for (int a = 0; a < kRowsPerWarp; ++a) {
      const int lr = row_base + warp * kRowsPerWarp + a;
      if (lr >= s) continue;
      const unsigned short* xr =
          reinterpret_cast<const unsigned short*>(x + ((size_t)item * s + lr) * ldx + k0) + lane;
      unsigned short xb[kRpChunk / 32];
#pragma unroll
      for (int e = 0; e < kRpChunk / 32; ++e) xb[e] = (e * 32 + (int)lane < kmax) ? xr[e * 32] : (unsigned short)0;
#pragma unroll
      for (int e = 0; e < kRpChunk / 32; ++e) {
        const float xv = bf16_bits_to_float(xb[e]);
        const float4* wr = reinterpret_cast<const float4*>(s_w + (e * 32 + lane) * RS);
#pragma unroll
        for (int q4 = 0; q4 < R / 4; ++q4) {
          float4 ww = wr[q4];
          acc[a][q4 * 4 + 0] = fmaf(xv, ww.x, acc[a][q4 * 4 + 0]);
          acc[a][q4 * 4 + 1] = fmaf(xv, ww.y, acc[a][q4 * 4 + 1]);
          acc[a][q4 * 4 + 2] = fmaf(xv, ww.z, acc[a][q4 * 4 + 2]);
          acc[a][q4 * 4 + 3] = fmaf(xv, ww.w, acc[a][q4 * 4 + 3]);
        }
      }
    }
  }
#pragma unroll
  for (int a = 0; a < kRowsPerWarp; ++a) {
    const int lr = row_base + warp * kRowsPerWarp + a;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      float v = acc[a][q];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      acc[a][q] = v;
    }
    if (lr < s && lane < r) {
      float v = 0.f;
#pragma unroll
      for (int q = 0; q < R; ++q)
        if (q == lane) v = acc[a][q];
      y[((size_t)item * s + lr) * ldy + lane] = v * scale;
    }
  }
}

// ---------------------------------------------------------------- rowproj on tensor cores
// Y[M, R] = X[M, K] W[K, R] with mma.sync m16n8k16 (bf16 in, fp32 accumulate): a warp owns
// 16 rows and walks K in steps of 16; A fragments come straight from global (X rows are
// contiguous along K), B fragments from the W chunk staged in shared memory as bf16 [n][k].
// The CUDA-core form is shared-memory-bandwidth bound (R*4 bytes of W per X element).
LX_DEV void mma16816_rp(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}


// W packed once per call: wp[item][hl][q][k] bf16 (hl = 0: hi, 1: lo), k over the item's packed K
// (gathered through ids), rows q >= r and columns k >= k_item zero. Kp = K rounded up to 16.
__global__ void rowproj_wpack_kernel(const float* __restrict__ w, long long w_sk, long long w_sq, int r, int RP, int K,
                                     int Kp, const int32_t* __restrict__ counts, const int32_t* __restrict__ ids,
                                     int ids_stride, int blk, __nv_bfloat16* __restrict__ wp) {
  const int item = blockIdx.y;
  const int k_item = counts ? __ldg(counts + item) * blk : K;
  const int32_t* my_ids = ids ? ids + (size_t)item * ids_stride : nullptr;
  __nv_bfloat16* out = wp + (size_t)item * 2 * RP * Kp;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < RP * Kp; e += gridDim.x * blockDim.x) {
    const int q = e / Kp, k = e % Kp;
    float val = 0.f;
    if (k < k_item && q < r) {
      const long long ko = my_ids ? (long long)__ldg(my_ids + k / blk) * blk + k % blk : k;
      val = __ldg(w + ko * w_sk + q * w_sq);
    }
    const __nv_bfloat16 hi = __float2bfloat16_rn(val);
    out[e] = hi;
    out[(size_t)RP * Kp + e] = __float2bfloat16_rn(val - __bfloat162float(hi));
  }
}

// Y[M, R] = X W on tensor cores, A and B fragments straight from global (L2-resident W pack);
// a CTA owns 16 rows, its kRpWarps warps interleave k-steps (kRpU in flight each: ~64 KB of X
// in flight per SM, enough to stream at HBM rate) and reduce through shared memory.
// Y[M, R] = X W on tensor cores (mma.sync m16n8k16), streaming X once at HBM rate.
// K is summed over, so the MMA's k-slots may be mapped to any permutation of the physical k applied
// to both X and W: within each 32-wide k block, lane t (= lane % 4) owns physical k [8t, 8t+8) and
// feeds MMA step j (0, 1) with k 8t+4j+{0,1} (slots 2t, 2t+1) and 8t+4j+{2,3} (slots 2t+8, 2t+9).
// One 16B load per row (g, g+8) then serves two MMA steps, and the packed W ([q][k], hi/lo bf16)
// is read the same way. A CTA owns 16 rows; kRpWarps warps take interleaved 32-k blocks (kRpU in
// flight each) and reduce through shared memory.
constexpr int kRpWarps = 8, kRpU = 8;

template <int NT>
__global__ void __launch_bounds__(32 * kRpWarps) rowproj_mma2_kernel(const __nv_bfloat16* __restrict__ x, int ldx, int s, int K,
                                                           int Kp, int r, float scale, const int32_t* __restrict__ counts,
                                                           int blk, const __nv_bfloat16* __restrict__ wp,
                                                           float* __restrict__ y, int ldy) {
  constexpr int RP = 8 * NT;
  __shared__ float s_red[kRpWarps][16][RP + 1];
  const int item = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int row0 = blockIdx.x * 16;
  const int k_item = counts ? __ldg(counts + item) * blk : K;
  const int ra = row0 + g, rb = ra + 8;
  const __nv_bfloat16* xa = x + ((size_t)item * s + min(ra, s - 1)) * ldx + 8 * t;
  const __nv_bfloat16* xb = x + ((size_t)item * s + min(rb, s - 1)) * ldx + 8 * t;
  const __nv_bfloat16* wh = wp + (size_t)item * 2 * RP * Kp + (size_t)g * Kp + 8 * t;  // row q = g (+8 per n-tile)
  const __nv_bfloat16* wl = wh + (size_t)RP * Kp;
  float acc[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
  for (int kb = warp * 32; kb < k_item; kb += 32 * kRpWarps * kRpU) {
    uint4 va[kRpU], vb[kRpU], vh[kRpU][NT], vl[kRpU][NT];
    // all loads of the round issued before any MMA (unconditional, clamped addresses; out-of-range
    // lanes are zeroed afterwards): kRpU x 1 KB of X per warp in flight
    uint32_t okm = 0;
#pragma unroll
    for (int u = 0; u < kRpU; ++u) {
      const int k0 = kb + u * 32 * kRpWarps;
      const bool ok = k0 + 8 * t < k_item;  // k_item is a multiple of 16: a lane's 8 k are all in or all out
      okm |= ok ? 1u << u : 0u;
      const int kl = ok ? k0 : 0;
      va[u] = __ldg(reinterpret_cast<const uint4*>(xa + kl));
      vb[u] = __ldg(reinterpret_cast<const uint4*>(xb + kl));
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        vh[u][n] = __ldg(reinterpret_cast<const uint4*>(wh + (size_t)n * 8 * Kp + kl));
        vl[u][n] = __ldg(reinterpret_cast<const uint4*>(wl + (size_t)n * 8 * Kp + kl));
      }
    }
    asm volatile("" ::: "memory");
#pragma unroll
    for (int u = 0; u < kRpU; ++u) {
      if (!((okm >> u) & 1u)) {
        va[u] = vb[u] = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int n = 0; n < NT; ++n) vh[u][n] = vl[u][n] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
#pragma unroll
    for (int u = 0; u < kRpU; ++u) {
      const uint32_t a0[4] = {va[u].x, vb[u].x, va[u].y, vb[u].y};  // step 0
      const uint32_t a1[4] = {va[u].z, vb[u].z, va[u].w, vb[u].w};  // step 1
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        mma16816_rp(acc[n], a0, vh[u][n].x, vh[u][n].y);
        mma16816_rp(acc[n], a0, vl[u][n].x, vl[u][n].y);
        mma16816_rp(acc[n], a1, vh[u][n].z, vh[u][n].w);
        mma16816_rp(acc[n], a1, vl[u][n].z, vl[u][n].w);
      }
    }
  }
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    const int q = n * 8 + t * 2;
    s_red[warp][g][q] = acc[n][0];
    s_red[warp][g][q + 1] = acc[n][1];
    s_red[warp][g + 8][q] = acc[n][2];
    s_red[warp][g + 8][q + 1] = acc[n][3];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 16 * RP; e += 32 * kRpWarps) {
    const int rr = e / RP, q = e % RP, row = row0 + rr;
    if (q < r && row < s) {
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < kRpWarps; ++w) v += s_red[w][rr][q];
      y[((size_t)item * s + row) * ldy + q] = v * scale;
    }
  }
}

constexpr int kCgCols = 128;  // columns per CTA: 8 consumer warps x 16 columns
constexpr int kCgRows = 256;  // rows per CTA (one split): 2 CTAs per SM keep ~128 KB of X in flight

// partial[item][split][q][col] = sum over the split's rows of P[row, q] X[row, col] over the item's
// packed columns, on tensor cores: it is the GEMM D[col][q] = X^T[col][row] P[row][q] with
// m = column, n = q, k = row (mma.sync m16n8k16, bf16 in, fp32 accumulate). Warp 8 streams
// [32 rows x 128 cols] X tiles (two SWIZZLE_128B boxes of 64 columns) through a kCgSt-stage TMA
// ring (the whole 256-row split in flight); consumer warp w owns columns 16w..16w+15 and takes its
// A fragments with ldmatrix.trans straight from the swizzled tile. P is staged once per split as
// bf16 hi + lo ([q][row], padded rows: conflict-free B fragment loads), so X (P_hi + P_lo) keeps
// ~16 mantissa bits of P. No cross-warp reduction: every warp owns distinct output columns.
// The CUDA-core form of this kernel was FMA-bound (R FMAs per X element).
constexpr int kCgSt = 8, kCgTile = 32 * kCgCols * 2;  // bytes per stage (2 atoms of [32][128B])
constexpr int kCgPStride = kCgRows + 8;               // bf16 elements per staged P row

// Debug-only phase trace (lx_debug_set_colgrad_trace): per CTA 8 clock64 stamps, NULL in production.
__device__ unsigned long long* g_cg_trace = nullptr;
LX_DEV void cg_stamp(int slot) {
  unsigned long long* t = g_cg_trace;
  if (t != nullptr) {
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    const size_t cta = blockIdx.x + (size_t)gridDim.x * (blockIdx.y + (size_t)gridDim.y * blockIdx.z);
    t[cta * 8 + slot] = c;
  }
}

template <int RN>
struct CgSmem {
  static constexpr int kOffP = kCgSt * kCgTile;  // s_pt [2][RN][kCgPStride] bf16
  static constexpr int kOffBar = kOffP + 2 * RN * kCgPStride * 2;
  static constexpr int kTotal = kOffBar + 2 * kCgSt * 8 + 1024;
};

LX_DEV void ldsm_x4_trans(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

template <int RN>
__global__ void __launch_bounds__(288, 2) colgrad_partial_kernel(const __grid_constant__ CUtensorMap tm_x, const float* __restrict__ p,
                                                              int ldp, int s, int ncols, int r,
                                                              const int32_t* __restrict__ counts, int blk,
                                                              float* __restrict__ ws) {
  constexpr int NT = RN / 8;
  extern __shared__ uint8_t cg_raw[];
  uint8_t* sm = align_smem_1024(cg_raw);
  __nv_bfloat16* s_pt = reinterpret_cast<__nv_bfloat16*>(sm + CgSmem<RN>::kOffP);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + CgSmem<RN>::kOffBar);
  uint64_t* empty = full + kCgSt;
  const int item = blockIdx.z, split = blockIdx.y;
  const int n_splits = gridDim.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_item = counts ? __ldg(counts + item) * blk : ncols;
  if (blockIdx.x * kCgCols >= n_item) return;  // beyond the item's packed width: never read
  const int r0 = split * kCgRows;
  const int nrows = min(kCgRows, s - r0);
  const int n_tiles = (nrows + 31) / 32;
  if (threadIdx.x == 0) {
    cg_stamp(0);
    for (int i = 0; i < kCgSt; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, 8);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 8) {
    if (lane == 0) {
      tma_prefetch_desc(&tm_x);
      for (int t = 0; t < n_tiles; ++t) {
        const int st = t % kCgSt;
        mbar_wait(empty + st, ((t / kCgSt) & 1) ^ 1);
        mbar_arrive_expect_tx(full + st, kCgTile);
        uint8_t* dst = sm + st * kCgTile;
        const int row = item * s + r0 + t * 32;
        tma_load_2d(dst, &tm_x, full + st, blockIdx.x * kCgCols, row);
        tma_load_2d(dst + kCgTile / 2, &tm_x, full + st, blockIdx.x * kCgCols + 64, row);
      }
    }
    return;
  }
  // P rows of this split -> smem as bf16 hi/lo, transposed (p == NULL: column sums, P[:, 0] = 1);
  // rows past nrows and columns q >= r are zero
  for (int e = threadIdx.x; e < kCgRows * RN; e += 256) {
    const int i = e / RN, q = e % RN;
    float v = 0.f;
    if (i < nrows && q < r) v = p ? __ldg(p + ((size_t)item * s + r0 + i) * ldp + q) : 1.f;
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    s_pt[q * kCgPStride + i] = hi;
    s_pt[(RN + q) * kCgPStride + i] = __float2bfloat16_rn(v - __bfloat162float(hi));
  }
  asm volatile("bar.sync 1, 256;" ::: "memory");
  if (threadIdx.x == 0) cg_stamp(1);
  float acc[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
  const int g = lane >> 2, t4 = lane & 3;
  // ldmatrix.trans: lane L addresses row (L & 7) of matrix L >> 3; matrices (rows k0.., cols 16w..),
  // (k0.., 16w+8..), (k0+8.., 16w..), (k0+8.., 16w+8..) = the A fragment a0..a3 of m16 x k16
  const int mi = lane >> 3, ri = lane & 7;
  const int ld_row = ri + ((mi >> 1) << 3);
  const int ld_chunk = 2 * (warp & 3) + (mi & 1);
  const uint32_t sm_base = smem_u32(sm) + (warp >> 2) * (kCgTile / 2);
  const uint32_t pt_base = smem_u32(s_pt) + (g * kCgPStride + 2 * t4) * 2;
  for (int t = 0; t < n_tiles; ++t) {
    const int st = t % kCgSt;
    mbar_wait(full + st, (t / kCgSt) & 1);
    if (threadIdx.x == 0 && t == 0) cg_stamp(2);
#pragma unroll
    for (int k0 = 0; k0 < 32; k0 += 16) {
      const int row = k0 + ld_row;
      uint32_t a[4];
      ldsm_x4_trans(sm_base + st * kCgTile + row * 128 + ((ld_chunk ^ (row & 7)) << 4), a);
      const int kk = t * 32 + k0;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
#pragma unroll
        for (int hl = 0; hl < 2; ++hl) {
          const uint32_t pb = pt_base + ((hl * RN + 8 * n) * kCgPStride + kk) * 2;
          uint32_t b0, b1;
          asm volatile("ld.shared.b32 %0, [%1];" : "=r"(b0) : "r"(pb));
          asm volatile("ld.shared.b32 %0, [%1];" : "=r"(b1) : "r"(pb + 16));
          mma16816_rp(acc[n], a, b0, b1);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);
  }
  if (threadIdx.x == 0) cg_stamp(3);
  // D[m = column][n = q]: d0 (col g, q 2t), d1 (g, 2t+1), d2 (g+8, 2t), d3 (g+8, 2t+1)
  float* out = ws + ((size_t)item * n_splits + split) * r * (size_t)ncols;
  const int c = blockIdx.x * kCgCols + warp * 16 + g;
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    const int q = 8 * n + 2 * t4;
    if (q < r) {
      if (c < ncols) out[(size_t)q * ncols + c] = acc[n][0];
      if (c + 8 < ncols) out[(size_t)q * ncols + c + 8] = acc[n][2];
    }
    if (q + 1 < r) {
      if (c < ncols) out[(size_t)(q + 1) * ncols + c] = acc[n][1];
      if (c + 8 < ncols) out[(size_t)(q + 1) * ncols + c + 8] = acc[n][3];
    }
  }
  if (threadIdx.x == 0) cg_stamp(4);
}

// G(q, c_orig) = scale * sum_items sum_splits partial[item][split][q][pos_item(c_orig)]
__global__ void colgrad_final_kernel(const float* __restrict__ ws, int n_items, int n_splits, int ncols, int r,
                                     const int32_t* __restrict__ pos, int blk, float scale, float* __restrict__ g,
                                     long long g_sq, long long g_sc) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int q = blockIdx.y;
  if (c >= ncols || q >= r) return;
  float acc = 0.f;
  // items in groups of 8: all position lookups, then all partial loads, are independent (in flight together);
  // the summation order stays fixed (item-major, split-minor) -> deterministic
  for (int b0 = 0; b0 < n_items; b0 += 8) {
    int pcs[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int b = b0 + u;
      pcs[u] = -1;
      if (b < n_items) {
        if (pos) {
          const int pb = __ldg(pos + (size_t)b * (ncols / blk) + c / blk);
          pcs[u] = pb < 0 ? -1 : pb * blk + c % blk;
        } else {
          pcs[u] = c;
        }
      }
    }
    for (int sp0 = 0; sp0 < n_splits; sp0 += 4) {
      float vals[8][4];
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int t = 0; t < 4; ++t)
          vals[u][t] = (pcs[u] >= 0 && sp0 + t < n_splits)
                           ? __ldg(ws + (((size_t)(b0 + u) * n_splits + sp0 + t) * r + q) * ncols + pcs[u])
                           : 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int t = 0; t < 4; ++t) acc += vals[u][t];
    }
  }
  g[(long long)q * g_sq + (long long)c * g_sc] = acc * scale;
}

template <int RN>
static int colgrad_impl(const float* p, int ldp, const uint16_t* x, int ldx, int n_items, int s, int ncols, int r,
                        float scale, const int32_t* counts, const int32_t* pos, int blk, float* g, long long g_sq,
                        long long g_sc, float* ws, cudaStream_t stream) {
  // shared columns (no counts): every item reads the same columns -> one item of n_items * s rows
  const int items = counts ? n_items : 1, rows = counts ? s : n_items * s;
  const int splits = (rows + kCgRows - 1) / kCgRows;
  dim3 g1((ncols + kCgCols - 1) / kCgCols, splits, items);
  constexpr int smem = CgSmem<RN>::kTotal;
  static cudaError_t attr = cudaFuncSetAttribute(colgrad_partial_kernel<RN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  LX_CHECK_CUDA(attr);
  // X as [n_items*s, ldx]: boxes of 64 columns x 32 rows (columns past ncols / the item's width are
  // never combined; rows past an item's split are weighted by P = 0)
  CUtensorMap tm;
  int rc0 = make_tmap_bf16_2d(&tm, x, (uint64_t)ldx, (uint64_t)n_items * s, (uint64_t)ldx, 64, 32);
  if (rc0) return rc0;
  colgrad_partial_kernel<RN><<<g1, 288, smem, stream>>>(tm, p, ldp, rows, ncols, r, counts, counts ? blk : 1, ws);
  int rc = launch_check("colgrad_partial");
  if (rc) return rc;
  dim3 g2((ncols + 255) / 256, r);
  colgrad_final_kernel<<<g2, 256, 0, stream>>>(ws, items, splits, ncols, r, counts ? pos : nullptr,
                                                  counts ? blk : 1, scale, g, g_sq, g_sc);
  return launch_check("colgrad_final");
}

}  // namespace lx

using namespace lx;

extern "C" {

long long lx_rowproj_ws_bytes(int n_items, int K, int r, int gathered) {
  const int RP = r <= 8 ? 8 : 16;
  return (long long)(gathered ? n_items : 1) * 2 * RP * K * 2;
}

int lx_rowproj(const uint16_t* x, int ldx, int n_items, int s, int K, const float* w, long long w_sk, long long w_sq,
               int r, float scale, const int32_t* counts, const int32_t* ids, int blk, float* y, int ldy, void* wpack_ws,
               lx_stream_t stream) {
  LX_REQUIRE(ldy >= r, LX_ERR_SHAPE, "rowproj: ldy < r");
  LX_REQUIRE(r >= 1 && r <= kRpMaxR, LX_ERR_UNSUPPORTED, "rowproj: rank %d outside [1, %d]", r, kRpMaxR);
  LX_REQUIRE(ldx % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0, LX_ERR_SHAPE,
             "rowproj: 16B-aligned rows required (row stride multiple of 8)");
  LX_REQUIRE(!counts || K % blk == 0, LX_ERR_MASK, "rowproj: K not a multiple of blk");
  LX_REQUIRE(ldx >= ((K + 15) / 16) * 16, LX_ERR_SHAPE, "rowproj: row stride must cover K rounded up to 16");
  const auto* xb = reinterpret_cast<const __nv_bfloat16*>(x);
  const int ids_stride = counts ? K / blk : 0, b = counts ? blk : 1;
  if (K % 16 == 0 && wpack_ws) {  // tensor-core path (K and every item's packed K are multiples of 16)
    const int NT = r <= 8 ? 1 : 2, RP = 8 * NT;
    const int items_w = counts ? n_items : 1;
    const int Kp = K;
    dim3 gp((RP * Kp + 255) / 256 < 64 ? (RP * Kp + 255) / 256 : 64, items_w);
    rowproj_wpack_kernel<<<gp, 256, 0, stream>>>(w, w_sk, w_sq, r, RP, K, Kp, counts, ids, ids_stride, b,
                                                 reinterpret_cast<__nv_bfloat16*>(wpack_ws));
    int rc = launch_check("rowproj_wpack");
    if (rc) return rc;
    dim3 grid((s + 15) / 16, n_items);
    const auto* wpb = reinterpret_cast<const __nv_bfloat16*>(wpack_ws);
    if (!counts && n_items > 1) {
      // dense W is shared by all items: index it as item 0 by treating the batch as one item
      grid = dim3((n_items * s + 15) / 16, 1);
      if (NT == 1)
        rowproj_mma2_kernel<1><<<grid, 32 * kRpWarps, 0, stream>>>(xb, ldx, n_items * s, K, Kp, r, scale, nullptr, b, wpb, y, ldy);
      else
        rowproj_mma2_kernel<2><<<grid, 32 * kRpWarps, 0, stream>>>(xb, ldx, n_items * s, K, Kp, r, scale, nullptr, b, wpb, y, ldy);
    } else if (NT == 1) {
      rowproj_mma2_kernel<1><<<grid, 32 * kRpWarps, 0, stream>>>(xb, ldx, s, K, Kp, r, scale, counts, b, wpb, y, ldy);
    } else {
      rowproj_mma2_kernel<2><<<grid, 32 * kRpWarps, 0, stream>>>(xb, ldx, s, K, Kp, r, scale, counts, b, wpb, y, ldy);
    }
    return launch_check("rowproj_mma");
  }
  dim3 grid((s + kRpRows - 1) / kRpRows, n_items);
  if (r <= 8)
    rowproj_kernel<8><<<grid, 256, 0, stream>>>(xb, ldx, s, K, w, w_sk, w_sq, r, scale, counts, ids, ids_stride, b, y, ldy);
  else
    rowproj_kernel<16><<<grid, 256, 0, stream>>>(xb, ldx, s, K, w, w_sk, w_sq, r, scale, counts, ids, ids_stride, b, y, ldy);
  return launch_check("rowproj");
}

int lx_debug_set_colgrad_trace(unsigned long long* buf) {
  LX_CHECK_CUDA(cudaMemcpyToSymbol(g_cg_trace, &buf, sizeof(buf)));
  return 0;
}

long long lx_colgrad_ws_floats(int n_items, int s, int ncols, int r) {
  // bound for both layouts: per item (gathered) or one item of n_items * s rows (shared columns)
  long long splits = (s + kCgRows - 1) / kCgRows;
  return (long long)n_items * splits * r * ncols;
}

int lx_colgrad(const float* p, int ldp, const uint16_t* x, int ldx, int n_items, int s, int ncols, int r, float scale,
               const int32_t* counts, const int32_t* pos, int blk, float* g, long long g_sq, long long g_sc, float* ws,
               lx_stream_t stream) {
  LX_REQUIRE(r >= 1 && r <= 16, LX_ERR_UNSUPPORTED, "colgrad: rank %d outside [1, 16]", r);
  LX_REQUIRE(!p || ldp >= r, LX_ERR_SHAPE, "colgrad: ldp < r");
  LX_REQUIRE(ncols % 4 == 0, LX_ERR_SHAPE, "colgrad: ncols must be a multiple of 4");
  LX_REQUIRE(!counts || (pos && ncols % blk == 0), LX_ERR_MASK, "colgrad: gathered columns need pos and ncols %% blk == 0");
  LX_REQUIRE(ldx % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0, LX_ERR_SHAPE, "colgrad: 16B-aligned rows required");
  if (r > 8) return colgrad_impl<16>(p, ldp, x, ldx, n_items, s, ncols, r, scale, counts, pos, blk, g, g_sq, g_sc, ws, stream);
  return colgrad_impl<8>(p, ldp, x, ldx, n_items, s, ncols, r, scale, counts, pos, blk, g, g_sq, g_sc, ws, stream);
}

int lx_colsum(const uint16_t* x, int ldx, int n_items, int s, int ncols, const int32_t* counts, const int32_t* pos,
              int blk, float* out, float* ws, lx_stream_t stream) {
  return lx_colgrad(nullptr, 1, x, ldx, n_items, s, ncols, 1, 1.f, counts, pos, blk, out, 0, 1, ws, stream);
}

}  // extern "C"
