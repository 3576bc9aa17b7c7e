// Skinny rank-r LoRA kernels of the neuron-sparse MLP (sf/model.py:380-395,
// sf/autograd.py:97-123). All are HBM-bound single passes over one bf16
// activation tensor, optionally restricted to an item's packed active columns.
//
//   rowproj : Y[M, r]   = scale * X[M, K] W           (x A1, a A2[cols], dO B2^T, dz B1[:,cols]^T)
//   colgrad : G[q, c]   = scale * sum_rows P[row, q] X[row, c]   (dB1[:,cols], dA2[cols], dB2, dA1)
//   colsum  : g[c]      = sum_rows X[row, c]                     (BitFit db1[cols], db2)
//
// colgrad/colsum are deterministic: per-(item, row-split) partials in a
// workspace, then a fixed-order reduction per original column.
#include "common.cuh"
#include "ptx.cuh"

namespace lx {

constexpr int kRpRows = 16;    // rows per CTA (8 warps x 2 rows)
constexpr int kRpChunk = 256;  // K chunk staged in smem
constexpr int kRpMaxR = 16;

__global__ void __launch_bounds__(256) rowproj_kernel(const __nv_bfloat16* __restrict__ x, int ldx, int s, int K,
                                                      const float* __restrict__ w, long long w_sk, long long w_sq, int r,
                                                      float scale, const int32_t* __restrict__ counts,
                                                      const int32_t* __restrict__ ids, int ids_stride, int blk,
                                                      float* __restrict__ y) {
  __shared__ __align__(16) float s_w[kRpChunk * kRpMaxR];
  const int item = blockIdx.y;
  const int row_base = blockIdx.x * kRpRows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k_item = counts ? __ldg(counts + item) * blk : K;
  const int32_t* my_ids = ids ? ids + (size_t)item * ids_stride : nullptr;
  float acc[2][kRpMaxR];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int q = 0; q < kRpMaxR; ++q) acc[a][q] = 0.f;
  for (int k0 = 0; k0 < k_item; k0 += kRpChunk) {
    __syncthreads();
    for (int e = threadIdx.x; e < kRpChunk * kRpMaxR; e += blockDim.x) {
      int kk = e / kRpMaxR, q = e % kRpMaxR, k = k0 + kk;
      float val = 0.f;
      if (k < k_item && q < r) {
        long long ko = my_ids ? (long long)__ldg(my_ids + k / blk) * blk + k % blk : k;
        val = __ldg(w + ko * w_sk + q * w_sq);
      }
      s_w[e] = val;
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      int lr = row_base + warp * 2 + a;
      if (lr >= s) continue;
      const __nv_bfloat16* xr = x + ((size_t)item * s + lr) * ldx + k0;
      // lane covers 8 consecutive k per step
      for (int kk = lane * 8; kk < kRpChunk && k0 + kk < k_item; kk += 256) {
        uint4 p = *reinterpret_cast<const uint4*>(xr + kk);
        uint32_t pw[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (k0 + kk + e >= k_item) break;
          float xv = bf16_bits_to_float((pw[e >> 1] >> ((e & 1) * 16)) & 0xffff);
          const float4* wr = reinterpret_cast<const float4*>(s_w + (kk + e) * kRpMaxR);
#pragma unroll
          for (int q4 = 0; q4 < kRpMaxR / 4; ++q4) {
            if (q4 * 4 < r) {
              float4 ww = wr[q4];
              acc[a][q4 * 4 + 0] = fmaf(xv, ww.x, acc[a][q4 * 4 + 0]);
              acc[a][q4 * 4 + 1] = fmaf(xv, ww.y, acc[a][q4 * 4 + 1]);
              acc[a][q4 * 4 + 2] = fmaf(xv, ww.z, acc[a][q4 * 4 + 2]);
              acc[a][q4 * 4 + 3] = fmaf(xv, ww.w, acc[a][q4 * 4 + 3]);
            }
          }
        }
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    int lr = row_base + warp * 2 + a;
#pragma unroll
    for (int q = 0; q < kRpMaxR; ++q) {
      float v = acc[a][q];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && q < r && lr < s) y[((size_t)item * s + lr) * r + q] = v * scale;
    }
  }
}

constexpr int kCgCols = 256;  // columns per CTA (one per thread)
constexpr int kCgRows = 64;   // rows per split

// partial[item][split][q][col] over the item's packed columns
__global__ void __launch_bounds__(256) colgrad_partial_kernel(const float* __restrict__ p, const __nv_bfloat16* __restrict__ x,
                                                              int ldx, int s, int ncols, int r,
                                                              const int32_t* __restrict__ counts, int blk,
                                                              float* __restrict__ ws) {
  __shared__ float s_p[kCgRows * kRpMaxR];
  const int item = blockIdx.z, split = blockIdx.y;
  const int n_splits = gridDim.y;
  const int c = blockIdx.x * kCgCols + threadIdx.x;
  const int n_item = counts ? __ldg(counts + item) * blk : ncols;
  const int r0 = split * kCgRows;
  const int rr = max(r, 1);
  for (int e = threadIdx.x; e < kCgRows * rr; e += blockDim.x) {
    int lr = r0 + e / rr;
    s_p[e] = (lr < s) ? (p ? __ldg(p + ((size_t)item * s + lr) * r + e % rr) : 1.f) : 0.f;
  }
  __syncthreads();
  if (blockIdx.x * kCgCols >= n_item) {
    // columns beyond this item's packed width: nothing to write (never read)
    return;
  }
  float acc[kRpMaxR];
#pragma unroll
  for (int q = 0; q < kRpMaxR; ++q) acc[q] = 0.f;
  if (c < n_item) {
    const int nrows = min(kCgRows, s - r0);
    for (int i = 0; i < nrows; ++i) {
      float xv = __bfloat162float(x[((size_t)item * s + r0 + i) * ldx + c]);
#pragma unroll
      for (int q = 0; q < kRpMaxR; ++q)
        if (q < rr) acc[q] = fmaf(s_p[i * rr + q], xv, acc[q]);
    }
  }
  float* out = ws + (((size_t)item * n_splits + split) * rr) * ncols;
#pragma unroll
  for (int q = 0; q < kRpMaxR; ++q)
    if (q < rr && c < ncols) out[(size_t)q * ncols + c] = acc[q];
}

// G(q, c_orig) = scale * sum_items sum_splits partial[item][split][q][pos_item(c_orig)]
__global__ void colgrad_final_kernel(const float* __restrict__ ws, int n_items, int n_splits, int ncols, int r,
                                     const int32_t* __restrict__ pos, int blk, float scale, float* __restrict__ g,
                                     long long g_sq, long long g_sc) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int q = blockIdx.y;
  if (c >= ncols) return;
  const int rr = max(r, 1);
  float acc = 0.f;
  for (int b = 0; b < n_items; ++b) {
    int pc = c;
    if (pos) {
      int pb = __ldg(pos + (size_t)b * (ncols / blk) + c / blk);
      if (pb < 0) continue;
      pc = pb * blk + c % blk;
    }
    for (int sp = 0; sp < n_splits; ++sp) acc += ws[(((size_t)b * n_splits + sp) * rr + q) * ncols + pc];
  }
  g[(long long)q * g_sq + (long long)c * g_sc] = acc * scale;
}

}  // namespace lx

using namespace lx;

extern "C" {

int lx_rowproj(const uint16_t* x, int ldx, int n_items, int s, int K, const float* w, long long w_sk, long long w_sq,
               int r, float scale, const int32_t* counts, const int32_t* ids, int blk, float* y, lx_stream_t stream) {
  LX_REQUIRE(r >= 1 && r <= kRpMaxR, LX_ERR_UNSUPPORTED, "rowproj: rank %d outside [1, %d]", r, kRpMaxR);
  LX_REQUIRE(ldx % 8 == 0, LX_ERR_SHAPE, "rowproj: row stride must be a multiple of 8");
  LX_REQUIRE(!counts || K % blk == 0, LX_ERR_MASK, "rowproj: K not a multiple of blk");
  dim3 grid((s + kRpRows - 1) / kRpRows, n_items);
  rowproj_kernel<<<grid, 256, 0, stream>>>(reinterpret_cast<const __nv_bfloat16*>(x), ldx, s, K, w, w_sk, w_sq, r, scale,
                                           counts, ids, counts ? K / blk : 0, counts ? blk : 1, y);
  return launch_check("rowproj");
}

long long lx_colgrad_ws_floats(int n_items, int s, int ncols, int r) {
  long long splits = (s + kCgRows - 1) / kCgRows;
  return (long long)n_items * splits * (r > 0 ? r : 1) * ncols;
}

int lx_colgrad(const float* p, const uint16_t* x, int ldx, int n_items, int s, int ncols, int r, float scale,
               const int32_t* counts, const int32_t* pos, int blk, float* g, long long g_sq, long long g_sc, float* ws,
               lx_stream_t stream) {
  LX_REQUIRE(r >= 1 && r <= kRpMaxR, LX_ERR_UNSUPPORTED, "colgrad: rank %d outside [1, %d]", r, kRpMaxR);
  LX_REQUIRE(!counts || (pos && ncols % blk == 0), LX_ERR_MASK, "colgrad: gathered columns need pos and ncols %% blk == 0");
  const int splits = (s + kCgRows - 1) / kCgRows;
  dim3 g1((ncols + kCgCols - 1) / kCgCols, splits, n_items);
  colgrad_partial_kernel<<<g1, kCgCols, 0, stream>>>(p, reinterpret_cast<const __nv_bfloat16*>(x), ldx, s, ncols, r, counts,
                                                     counts ? blk : 1, ws);
  int rc = launch_check("colgrad_partial");
  if (rc) return rc;
  dim3 g2((ncols + 255) / 256, r);
  colgrad_final_kernel<<<g2, 256, 0, stream>>>(ws, n_items, splits, ncols, r, counts ? pos : nullptr, counts ? blk : 1,
                                               scale, g, g_sq, g_sc);
  return launch_check("colgrad_final");
}

int lx_colsum(const uint16_t* x, int ldx, int n_items, int s, int ncols, const int32_t* counts, const int32_t* pos,
              int blk, float* out, float* ws, lx_stream_t stream) {
  return lx_colgrad(nullptr, x, ldx, n_items, s, ncols, 1, 1.f, counts, pos, blk, out, 0, 1, ws, stream);
}

}  // extern "C"
