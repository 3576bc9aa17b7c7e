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

constexpr int kRmRows = 16;    // rows per CTA; its 4 warps split K and reduce through shared memory
constexpr int kRmChunk = 256;  // K per staged W chunk
constexpr int kRmStride = kRmChunk + 8;  // bf16 elements per n-row in smem (conflict-free 32-bit reads)

template <int NT>  // NT n8-tiles: R <= 8*NT
__global__ void __launch_bounds__(128) rowproj_mma_kernel(const __nv_bfloat16* __restrict__ x, int ldx, int s, int K,
                                                          const float* __restrict__ w, long long w_sk, long long w_sq,
                                                          int r, float scale, const int32_t* __restrict__ counts,
                                                          const int32_t* __restrict__ ids, int ids_stride, int blk,
                                                          float* __restrict__ y, int ldy) {
  // W chunk as a bf16 (hi, lo) pair: W ~= hi + lo to ~2^-17 relative, so X (exact bf16) . W keeps
  // fp32-level accuracy with two MMAs per step
  __shared__ __align__(16) __nv_bfloat16 s_hi[8 * NT * kRmStride];
  __shared__ __align__(16) __nv_bfloat16 s_lo[8 * NT * kRmStride];
  __shared__ float s_red[4][16][8 * NT + 1];
  const int item = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = blockIdx.x * kRmRows;
  const int k_item = counts ? __ldg(counts + item) * blk : K;
  const int32_t* my_ids = ids ? ids + (size_t)item * ids_stride : nullptr;
  const int ra = row0 + (lane >> 2), rb = ra + 8;
  const uint32_t* xa = reinterpret_cast<const uint32_t*>(x + ((size_t)item * s + min(ra, s - 1)) * ldx) + (lane & 3);
  const uint32_t* xb = reinterpret_cast<const uint32_t*>(x + ((size_t)item * s + min(rb, s - 1)) * ldx) + (lane & 3);
  float acc[NT][4];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
  const bool k_fast = (w_sk == 1);
  for (int k0 = 0; k0 < k_item; k0 += kRmChunk) {
    __syncthreads();
    for (int e = threadIdx.x; e < 8 * NT * kRmChunk; e += 128) {
      int kk, q;
      if (k_fast) { q = e / kRmChunk; kk = e % kRmChunk; } else { kk = e / (8 * NT); q = e % (8 * NT); }
      const int k = k0 + kk;
      float val = 0.f;
      if (k < k_item && q < r) {
        long long ko = my_ids ? (long long)__ldg(my_ids + k / blk) * blk + k % blk : k;
        val = __ldg(w + ko * w_sk + q * w_sq);
      }
      const __nv_bfloat16 hi = __float2bfloat16_rn(val);
      s_hi[q * kRmStride + kk] = hi;
      s_lo[q * kRmStride + kk] = __float2bfloat16_rn(val - __bfloat162float(hi));
    }
    __syncthreads();
    const int kn = min(kRmChunk, k_item - k0);  // multiple of 16
    // warp w takes k-steps w, w+4, ...: all four A-fragment loads of two steps are in flight together
    for (int ks = warp * 16; ks < kn; ks += 128) {
      const int kw = (k0 + ks) >> 1;
      const bool two = ks + 64 < kn;
      uint32_t a[4] = {__ldg(xa + kw), __ldg(xb + kw), __ldg(xa + kw + 4), __ldg(xb + kw + 4)};
      uint32_t a2[4] = {0u, 0u, 0u, 0u};
      if (two) {
        a2[0] = __ldg(xa + kw + 32); a2[1] = __ldg(xb + kw + 32); a2[2] = __ldg(xa + kw + 36); a2[3] = __ldg(xb + kw + 36);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 1 && !two) break;
        const int kk = ks + h * 64;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int off = (t * 8 + (lane >> 2)) * kRmStride + kk + (lane & 3) * 2;
          const uint32_t h0 = *reinterpret_cast<const uint32_t*>(s_hi + off);
          const uint32_t h1 = *reinterpret_cast<const uint32_t*>(s_hi + off + 8);
          const uint32_t l0 = *reinterpret_cast<const uint32_t*>(s_lo + off);
          const uint32_t l1 = *reinterpret_cast<const uint32_t*>(s_lo + off + 8);
          mma16816_rp(acc[t], h ? a2 : a, h0, h1);
          mma16816_rp(acc[t], h ? a2 : a, l0, l1);
        }
      }
    }
  }
  // reduce the four warps' partial sums
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const int q = t * 8 + (lane & 3) * 2;
    s_red[warp][lane >> 2][q] = acc[t][0];
    s_red[warp][lane >> 2][q + 1] = acc[t][1];
    s_red[warp][(lane >> 2) + 8][q] = acc[t][2];
    s_red[warp][(lane >> 2) + 8][q + 1] = acc[t][3];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 16 * 8 * NT; e += 128) {
    const int rr = e / (8 * NT), q = e % (8 * NT), row = row0 + rr;
    if (q < r && row < s)
      y[((size_t)item * s + row) * ldy + q] = (s_red[0][rr][q] + s_red[1][rr][q] + s_red[2][rr][q] + s_red[3][rr][q]) * scale;
  }
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
// a CTA owns 16 rows, its 4 warps interleave k-steps and reduce through shared memory.
template <int NT>
__global__ void __launch_bounds__(128) rowproj_mma2_kernel(const __nv_bfloat16* __restrict__ x, int ldx, int s, int K,
                                                           int Kp, int r, float scale, const int32_t* __restrict__ counts,
                                                           int blk, const __nv_bfloat16* __restrict__ wp,
                                                           float* __restrict__ y, int ldy) {
  constexpr int RP = 8 * NT;
  __shared__ float s_red[4][16][RP + 1];
  const int item = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = blockIdx.x * 16;
  const int k_item = counts ? __ldg(counts + item) * blk : K;
  const int ra = row0 + (lane >> 2), rb = ra + 8;
  const uint32_t* xa = reinterpret_cast<const uint32_t*>(x + ((size_t)item * s + min(ra, s - 1)) * ldx) + (lane & 3);
  const uint32_t* xb = reinterpret_cast<const uint32_t*>(x + ((size_t)item * s + min(rb, s - 1)) * ldx) + (lane & 3);
  const uint32_t* wh = reinterpret_cast<const uint32_t*>(wp + (size_t)item * 2 * RP * Kp + (lane >> 2) * Kp) + (lane & 3);
  const uint32_t* wl = wh + (size_t)RP * Kp / 2;
  float acc[NT][4];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
  constexpr int U = 4;  // k-steps in flight per warp
  for (int kb = warp * 16; kb < k_item; kb += 64 * U) {
    uint32_t a[U][4], bh[U][NT][2], bl[U][NT][2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int ks = kb + u * 64;
      const bool ok = ks < k_item;
      const int kw = ks >> 1;
      a[u][0] = ok ? __ldg(xa + kw) : 0u;
      a[u][1] = ok ? __ldg(xb + kw) : 0u;
      a[u][2] = ok ? __ldg(xa + kw + 4) : 0u;
      a[u][3] = ok ? __ldg(xb + kw + 4) : 0u;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const size_t o = (size_t)t * 8 * Kp / 2 + kw;
        bh[u][t][0] = ok ? __ldg(wh + o) : 0u;
        bh[u][t][1] = ok ? __ldg(wh + o + 4) : 0u;
        bl[u][t][0] = ok ? __ldg(wl + o) : 0u;
        bl[u][t][1] = ok ? __ldg(wl + o + 4) : 0u;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        mma16816_rp(acc[t], a[u], bh[u][t][0], bh[u][t][1]);
        mma16816_rp(acc[t], a[u], bl[u][t][0], bl[u][t][1]);
      }
  }
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const int q = t * 8 + (lane & 3) * 2;
    s_red[warp][lane >> 2][q] = acc[t][0];
    s_red[warp][lane >> 2][q + 1] = acc[t][1];
    s_red[warp][(lane >> 2) + 8][q] = acc[t][2];
    s_red[warp][(lane >> 2) + 8][q + 1] = acc[t][3];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 16 * RP; e += 128) {
    const int rr = e / RP, q = e % RP, row = row0 + rr;
    if (q < r && row < s)
      y[((size_t)item * s + row) * ldy + q] = (s_red[0][rr][q] + s_red[1][rr][q] + s_red[2][rr][q] + s_red[3][rr][q]) * scale;
  }
}

constexpr int kCgCols = 256;  // 32 lanes x 8 columns
constexpr int kCgRows = 128;  // rows per split (8 warps x 16 rows)

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
    // warp w owns rows w, w+8, ...; 8 rows in flight per lane
    for (int i0 = warp; i0 < nrows; i0 += 64) {
      uint4 pk[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * 8;
        pk[u] = i < nrows ? *reinterpret_cast<const uint4*>(x + ((size_t)item * s + r0 + i) * ldx + c0)
                          : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
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
    for (int sp = 0; sp < n_splits; ++sp) {
      float vals[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        vals[u] = pcs[u] >= 0 ? ws[(((size_t)(b0 + u) * n_splits + sp) * R + q) * ncols + pcs[u]] : 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += vals[u];
    }
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
        rowproj_mma2_kernel<1><<<grid, 128, 0, stream>>>(xb, ldx, n_items * s, K, Kp, r, scale, nullptr, b, wpb, y, ldy);
      else
        rowproj_mma2_kernel<2><<<grid, 128, 0, stream>>>(xb, ldx, n_items * s, K, Kp, r, scale, nullptr, b, wpb, y, ldy);
    } else if (NT == 1) {
      rowproj_mma2_kernel<1><<<grid, 128, 0, stream>>>(xb, ldx, s, K, Kp, r, scale, counts, b, wpb, y, ldy);
    } else {
      rowproj_mma2_kernel<2><<<grid, 128, 0, stream>>>(xb, ldx, s, K, Kp, r, scale, counts, b, wpb, y, ldy);
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
