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

constexpr int kCgCols = 256;  // 32 lanes x 8 columns
constexpr int kCgRows = 256;  // rows per split (8 warps x 32 rows)

// partial[item][split][q][col] over the item's packed columns (dynamic smem: s_p | s_red)
template <int R>
__global__ void __launch_bounds__(256) colgrad_partial_kernel(const float* __restrict__ p, int ldp,
                                                              const __nv_bfloat16* __restrict__ x, int ldx, int s, int ncols,
                                                              int r, const int32_t* __restrict__ counts, int blk,
                                                              float* __restrict__ ws) {
  extern __shared__ float cg_smem[];
  float* s_p = cg_smem;                          // [kCgRows][R]
  float* s_red = cg_smem + kCgRows * R;          // [8][R][kCgCols + 4]
  constexpr int kRedStride = kCgCols + 4;
  const int item = blockIdx.z, split = blockIdx.y;
  const int n_splits = gridDim.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_item = counts ? __ldg(counts + item) * blk : ncols;
  const int c0 = blockIdx.x * kCgCols + lane * 8;
  const int r0 = split * kCgRows;
  if (blockIdx.x * kCgCols >= n_item) return;  // beyond the item's packed width: never read
  for (int e = threadIdx.x; e < kCgRows * R; e += 256) {
    const int lr = r0 + e / R, q = e % R;
    s_p[e] = (lr < s && q < r) ? (p ? __ldg(p + ((size_t)item * s + lr) * ldp + q) : 1.f) : 0.f;
  }
  __syncthreads();
  float acc[8][R];
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int q = 0; q < R; ++q) acc[j][q] = 0.f;
  const int nrows = min(kCgRows, s - r0);
  if (c0 < n_item) {
    // warp w owns rows w, w+8, ...; 4 rows in flight per lane
    for (int i0 = warp; i0 < nrows; i0 += 32) {
      uint4 pk[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * 8;
        pk[u] = i < nrows ? *reinterpret_cast<const uint4*>(x + ((size_t)item * s + r0 + i) * ldx + c0)
                          : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * 8;
        if (i >= nrows) break;
        const uint32_t pw[4] = {pk[u].x, pk[u].y, pk[u].z, pk[u].w};
        const float* pp = s_p + i * R;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float xv = bf16_bits_to_float((pw[j >> 1] >> ((j & 1) * 16)) & 0xffff);
#pragma unroll
          for (int q = 0; q < R; ++q) acc[j][q] = fmaf(pp[q], xv, acc[j][q]);
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < R; ++q)
#pragma unroll
    for (int j = 0; j < 8; ++j) s_red[(warp * R + q) * kRedStride + lane * 8 + j] = acc[j][q];
  __syncthreads();
  float* out = ws + (((size_t)item * n_splits + split) * R) * ncols;
  for (int e = threadIdx.x; e < R * kCgCols; e += 256) {
    const int q = e / kCgCols, cc = e % kCgCols, c = blockIdx.x * kCgCols + cc;
    if (q >= r || c >= ncols) continue;
    float v = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < 8; ++w2) v += s_red[(w2 * R + q) * kRedStride + cc];
    out[(size_t)q * ncols + c] = v;
  }
}

// G(q, c_orig) = scale * sum_items sum_splits partial[item][split][q][pos_item(c_orig)]
template <int R>
__global__ void colgrad_final_kernel(const float* __restrict__ ws, int n_items, int n_splits, int ncols, int r,
                                     const int32_t* __restrict__ pos, int blk, float scale, float* __restrict__ g,
                                     long long g_sq, long long g_sc) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int q = blockIdx.y;
  if (c >= ncols || q >= r) return;
  float acc = 0.f;
  for (int b = 0; b < n_items; ++b) {
    int pc = c;
    if (pos) {
      int pb = __ldg(pos + (size_t)b * (ncols / blk) + c / blk);
      if (pb < 0) continue;
      pc = pb * blk + c % blk;
    }
    for (int sp = 0; sp < n_splits; ++sp) acc += ws[(((size_t)b * n_splits + sp) * R + q) * ncols + pc];
  }
  g[(long long)q * g_sq + (long long)c * g_sc] = acc * scale;
}

template <int R>
static int colgrad_impl(const float* p, int ldp, const uint16_t* x, int ldx, int n_items, int s, int ncols, int r,
                        float scale, const int32_t* counts, const int32_t* pos, int blk, float* g, long long g_sq,
                        long long g_sc, float* ws, cudaStream_t stream) {
  const int splits = (s + kCgRows - 1) / kCgRows;
  dim3 g1((ncols + kCgCols - 1) / kCgCols, splits, n_items);
  const int smem = (kCgRows * R + 8 * R * (kCgCols + 4)) * 4;
  static cudaError_t attr = cudaFuncSetAttribute(colgrad_partial_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  LX_CHECK_CUDA(attr);
  colgrad_partial_kernel<R><<<g1, 256, smem, stream>>>(p, ldp, reinterpret_cast<const __nv_bfloat16*>(x), ldx, s, ncols, r,
                                                    counts, counts ? blk : 1, ws);
  int rc = launch_check("colgrad_partial");
  if (rc) return rc;
  dim3 g2((ncols + 255) / 256, r);
  colgrad_final_kernel<R><<<g2, 256, 0, stream>>>(ws, n_items, splits, ncols, r, counts ? pos : nullptr,
                                                  counts ? blk : 1, scale, g, g_sq, g_sc);
  return launch_check("colgrad_final");
}

}  // namespace lx

using namespace lx;

extern "C" {

int lx_rowproj(const uint16_t* x, int ldx, int n_items, int s, int K, const float* w, long long w_sk, long long w_sq,
               int r, float scale, const int32_t* counts, const int32_t* ids, int blk, float* y, int ldy,
               lx_stream_t stream) {
  LX_REQUIRE(ldy >= r, LX_ERR_SHAPE, "rowproj: ldy < r");
  LX_REQUIRE(r >= 1 && r <= kRpMaxR, LX_ERR_UNSUPPORTED, "rowproj: rank %d outside [1, %d]", r, kRpMaxR);
  LX_REQUIRE(ldx % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0, LX_ERR_SHAPE,
             "rowproj: 16B-aligned rows required (row stride multiple of 8)");
  LX_REQUIRE(!counts || K % blk == 0, LX_ERR_MASK, "rowproj: K not a multiple of blk");
  LX_REQUIRE(ldx >= ((K + 15) / 16) * 16, LX_ERR_SHAPE, "rowproj: row stride must cover K rounded up to 16");
  dim3 grid((s + kRpRows - 1) / kRpRows, n_items);
  const auto* xb = reinterpret_cast<const __nv_bfloat16*>(x);
  const int ids_stride = counts ? K / blk : 0, b = counts ? blk : 1;
  if (r <= 8)
    rowproj_kernel<8><<<grid, 256, 0, stream>>>(xb, ldx, s, K, w, w_sk, w_sq, r, scale, counts, ids, ids_stride, b, y, ldy);
  else
    rowproj_kernel<16><<<grid, 256, 0, stream>>>(xb, ldx, s, K, w, w_sk, w_sq, r, scale, counts, ids, ids_stride, b, y, ldy);
  return launch_check("rowproj");
}

long long lx_colgrad_ws_floats(int n_items, int s, int ncols, int r) {
  long long splits = (s + kCgRows - 1) / kCgRows;
  int rr = r <= 1 ? 1 : (r <= 8 ? 8 : 16);
  return (long long)n_items * splits * rr * ncols;
}

int lx_colgrad(const float* p, int ldp, const uint16_t* x, int ldx, int n_items, int s, int ncols, int r, float scale,
               const int32_t* counts, const int32_t* pos, int blk, float* g, long long g_sq, long long g_sc, float* ws,
               lx_stream_t stream) {
  LX_REQUIRE(r >= 1 && r <= 16, LX_ERR_UNSUPPORTED, "colgrad: rank %d outside [1, 16]", r);
  LX_REQUIRE(!p || ldp >= r, LX_ERR_SHAPE, "colgrad: ldp < r");
  LX_REQUIRE(!counts || (pos && ncols % blk == 0), LX_ERR_MASK, "colgrad: gathered columns need pos and ncols %% blk == 0");
  LX_REQUIRE(ldx % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0, LX_ERR_SHAPE, "colgrad: 16B-aligned rows required");
  if (r == 1) return colgrad_impl<1>(p, ldp, x, ldx, n_items, s, ncols, r, scale, counts, pos, blk, g, g_sq, g_sc, ws, stream);
  if (r <= 8) return colgrad_impl<8>(p, ldp, x, ldx, n_items, s, ncols, r, scale, counts, pos, blk, g, g_sq, g_sc, ws, stream);
  return colgrad_impl<16>(p, ldp, x, ldx, n_items, s, ncols, r, scale, counts, pos, blk, g, g_sq, g_sc, ws, stream);
}

int lx_colsum(const uint16_t* x, int ldx, int n_items, int s, int ncols, const int32_t* counts, const int32_t* pos,
              int blk, float* out, float* ws, lx_stream_t stream) {
  return lx_colgrad(nullptr, 1, x, ldx, n_items, s, ncols, 1, 1.f, counts, pos, blk, out, 0, 1, ws, stream);
}

}  // extern "C"
