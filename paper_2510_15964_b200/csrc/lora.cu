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
// colgrad: one grouped launch per sublayer backward over 64-column chunks x
// row splits on mma.sync (see colgrad_group_kernel below).
#include <algorithm>

#include <cstdlib>

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
  pdl_wait_trigger();
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
  pdl_wait_trigger();
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
constexpr int kRpWarps = 8, kRpU = 4;  // 2 CTAs per SM: the 16-row CTAs of M = 4096 fit in one wave

// W pack: wp + item * w_item_stride holds [2][RP][Kp] (hi, lo); with `ids` the pack is the FULL W
// (shared by the items, w_item_stride 0) and packed k maps to ids[item][k / blk] * blk + k % blk.
// yb (optional): bf16 copy of Y (the LoRA rows of a K-extended projection GEMM operand).
template <int NT>
__global__ void __launch_bounds__(32 * kRpWarps, 2) rowproj_mma2_kernel(const __nv_bfloat16* __restrict__ x, int ldx, int s, int K,
                                                           int Kp, int r, float scale, const int32_t* __restrict__ counts,
                                                           int blk, const __nv_bfloat16* __restrict__ wp,
                                                           long long w_item_stride, const int32_t* __restrict__ ids,
                                                           int ids_stride, float* __restrict__ y, int ldy,
                                                           __nv_bfloat16* __restrict__ yb, int ldyb) {
  pdl_wait_trigger();
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
  const __nv_bfloat16* wh = wp + (size_t)item * w_item_stride + (size_t)g * Kp;  // row q = g (+8 per n-tile)
  const __nv_bfloat16* wl = wh + (size_t)RP * Kp;
  const int32_t* my_ids = ids ? ids + (size_t)item * ids_stride : nullptr;
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
      int kw = kl + 8 * t;  // this lane's first k (8 consecutive k stay inside one neuron block)
      if (my_ids) kw = ok ? __ldg(my_ids + kw / blk) * blk + kw % blk : 0;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        vh[u][n] = __ldg(reinterpret_cast<const uint4*>(wh + (size_t)n * 8 * Kp + kw));
        vl[u][n] = __ldg(reinterpret_cast<const uint4*>(wl + (size_t)n * 8 * Kp + kw));
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
      if (yb) yb[((size_t)item * s + row) * ldyb + q] = __float2bfloat16_rn(v * scale);
    }
  }
}

// Dense-K variant for K <= kRpsMaxK (the projections' LoRA down-products, K = d): the CTA's 16 rows of X are
// fetched with one 1-D bulk copy per row into shared memory (rows padded to K + 32 elements: the lanes' 16-byte
// fragment reads of rows g, g + 8 fall in distinct bank groups), so all of the CTA's X is in flight at once
// instead of kRpU 32-k blocks per warp round trip; the MMAs then read A fragments from shared memory and the
// hi/lo W pack from L1/L2 as above. Same k-slot mapping, same fixed-order warp reduction (identical results).
constexpr int kRpsMaxK = 4096;
// RG row groups of 16 per CTA share every W fragment load (RG = 2 halves the W pack re-reads from L2, which at
// 16 rows per CTA were as many bytes as X itself); X smem is 16 * RG rows of K + 32 elements.
template <int NT, int RG>
__global__ void __launch_bounds__(32 * kRpWarps, 2) rowproj_smem_kernel(const __nv_bfloat16* __restrict__ x, int ldx, int rows,
                                                           int K, int Kp, int r, float scale,
                                                           const __nv_bfloat16* __restrict__ wp, float* __restrict__ y,
                                                           int ldy, __nv_bfloat16* __restrict__ yb, int ldyb,
                                                           long long seg_x, long long seg_w, int seg_y, int seg_yb) {
  // blockIdx.y = segment: independent problems at fixed element offsets (lx_rowproj_packed_seg)
  x += blockIdx.y * seg_x;
  wp += blockIdx.y * seg_w;
  y += blockIdx.y * seg_y;
  if (yb) yb += blockIdx.y * seg_yb;
  constexpr int RP = 8 * NT;
  constexpr int TR = 16 * RG;  // rows per CTA
  extern __shared__ __align__(128) uint8_t rps_smem[];
  __shared__ float s_red[kRpWarps][TR][RP + 1];
  __shared__ __align__(8) uint64_t bar;
  const int pitch = K + 32;  // elements
  __nv_bfloat16* sx = reinterpret_cast<__nv_bfloat16*>(rps_smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int row0 = blockIdx.x * TR;
  const int nr = min(TR, rows - row0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait_trigger();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, (uint32_t)nr * K * 2);
    for (int i = 0; i < nr; ++i) bulk_load_1d(sx + (size_t)i * pitch, x + (size_t)(row0 + i) * ldx, K * 2, &bar);
  }
  // rows past the end (last CTA): zero in shared memory, never read from global
  for (int i = nr + warp; i < TR; i += kRpWarps)
    for (int c = lane * 8; c < K; c += 256) *reinterpret_cast<uint4*>(sx + (size_t)i * pitch + c) = make_uint4(0u, 0u, 0u, 0u);
  const __nv_bfloat16* wh = wp + (size_t)g * Kp;
  const __nv_bfloat16* wl = wh + (size_t)RP * Kp;
  float acc[RG][NT][4];
#pragma unroll
  for (int q = 0; q < RG; ++q)
#pragma unroll
    for (int n = 0; n < NT; ++n) acc[q][n][0] = acc[q][n][1] = acc[q][n][2] = acc[q][n][3] = 0.f;
  __syncthreads();
  mbar_wait(&bar, 0);
  for (int k0 = warp * 32; k0 < K; k0 += 32 * kRpWarps) {
    uint32_t a0[RG][4], a1[RG][4];
#pragma unroll
    for (int q = 0; q < RG; ++q) {
      const __nv_bfloat16* xa = sx + (size_t)(16 * q + g) * pitch + 8 * t;
      const uint4 va = *reinterpret_cast<const uint4*>(xa + k0);
      const uint4 vb = *reinterpret_cast<const uint4*>(xa + (size_t)8 * pitch + k0);
      a0[q][0] = va.x; a0[q][1] = vb.x; a0[q][2] = va.y; a0[q][3] = vb.y;
      a1[q][0] = va.z; a1[q][1] = vb.z; a1[q][2] = va.w; a1[q][3] = vb.w;
    }
    const int kw = k0 + 8 * t;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const uint4 vh = __ldg(reinterpret_cast<const uint4*>(wh + (size_t)n * 8 * Kp + kw));
      const uint4 vl = __ldg(reinterpret_cast<const uint4*>(wl + (size_t)n * 8 * Kp + kw));
#pragma unroll
      for (int q = 0; q < RG; ++q) {
        mma16816_rp(acc[q][n], a0[q], vh.x, vh.y);
        mma16816_rp(acc[q][n], a0[q], vl.x, vl.y);
        mma16816_rp(acc[q][n], a1[q], vh.z, vh.w);
        mma16816_rp(acc[q][n], a1[q], vl.z, vl.w);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < RG; ++q)
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int c = n * 8 + t * 2;
      s_red[warp][16 * q + g][c] = acc[q][n][0];
      s_red[warp][16 * q + g][c + 1] = acc[q][n][1];
      s_red[warp][16 * q + g + 8][c] = acc[q][n][2];
      s_red[warp][16 * q + g + 8][c + 1] = acc[q][n][3];
    }
  __syncthreads();
  for (int e = threadIdx.x; e < TR * RP; e += 32 * kRpWarps) {
    const int rr = e / RP, q = e % RP, row = row0 + rr;
    if (q < r && row < rows) {
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < kRpWarps; ++w) v += s_red[w][rr][q];
      y[(size_t)row * ldy + q] = v * scale;
      if (yb) yb[(size_t)row * ldyb + q] = __float2bfloat16_rn(v * scale);
    }
  }
}

// ---------------------------------------------------------------- parameter packing
// dst[i*dst_sr + j*dst_sc] = bf16(scale * src[i*src_sr + j*src_sc]) over a segment table (device memory);
// lo_off != 0 also writes the bf16 residual (hi/lo split) at dst + lo_off. One launch refreshes every
// LoRA factor's rowproj pack and K-extended projection rows after the optimizer step.
__global__ void pack_params_kernel(const lx_pack_segment* __restrict__ segs) {
  pdl_wait_trigger();
  const lx_pack_segment sg = segs[blockIdx.y];
  const long long n = (long long)sg.rows * sg.cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / sg.cols, j = e % sg.cols;
    const float v = sg.scale * __ldg(sg.src + i * sg.src_sr + j * sg.src_sc);
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(sg.dst) + i * sg.dst_sr + j * sg.dst_sc;
    *d = hi;
    if (sg.lo_off) d[sg.lo_off] = __float2bfloat16_rn(v - __bfloat162float(hi));
  }
}

// ---------------------------------------------------------------- colgrad (grouped)
// G_i(q, c) = scale_i * sum_rows P_i[row, q] X_i[row, c] for up to kCgMaxProbs problems per launch (all
// LoRA / BitFit column reductions of one sublayer's backward). It is the GEMM D[q][c] = P^T X with
// m = q, n = column, k = row, on mma.sync m16n8k16 (bf16 in, fp32 accumulate): the 16 m-rows of one
// MMA carry P_hi (rows 0..7) and P_lo (rows 8..15) of 8 ranks, so X (P_hi + P_lo) keeps ~16 mantissa
// bits of P at no extra MMA cost. A prep launch writes each P once in fragment order: per 128-row block
// and lane, the lane's A fragments of the block's 8 k-steps as 8*MT contiguous 16-byte chunks (rotated
// by lane: conflict-free LDS.128), fetched per stage with one 1-D bulk copy. Column sums (P == NULL)
// use an all-ones P. Rows past a unit (ragged items) carry P = 0, so no masking is needed.
//
// HBM-bound streaming: persistent CTAs (2 per SM); one producer thread walks the CTA's units and
// TMA-loads [128 rows x 64 columns] X stages (16 KB) plus the matching Pt tile through a
// 4-5 stage mbarrier ring that crosses unit boundaries; consumer warp w owns columns 8w..8w+7
// of the chunk (ldmatrix.trans B fragments, no cross-warp reduction), so the steady state has no
// CTA-wide barrier and ~6 stages x 16 KB per SM in flight.
//
// Unit = (problem, 64-column chunk, row split). Dense problems (pos == NULL) treat the batch as one item
// of n_items*s rows; gathered problems (per-item packed columns, pos[b][block] >= 0 when active) take the
// chunk in ORIGINAL columns, loop over the items whose blocks in the chunk are active (one TMA box per
// active 16-column sub-block, addressed through pos), so the partials of every item line up and inactive
// columns come out exactly 0. A unit writes its partial [r][64] (or G itself when it is the only split);
// a final launch sums the splits in order: deterministic, no float atomics.
constexpr int kCgMaxProbs = 16;  // two layers of LoRA factors (q/v/fc1/fc2 A and B) per launch
constexpr int kCgChunk = 64;
constexpr int kCgConsumers = 8;
constexpr int kCgThreads = 32 * (kCgConsumers + 1);
constexpr int kCgRows = 128;  // rows per stage = rows per split of a gathered problem
constexpr int kCgMaxSlots = 32;  // units per CTA
constexpr int kCgMaxItems = 16;  // items of a gathered problem
constexpr int kCgRowsDense = 256;
constexpr int kCgXBytes = kCgRows * 128;
enum : int { kCgLast = 1, kCgEmpty = 2, kCgGath = 4 };

struct CgProb {
  const float* p;
  uint32_t* pt;       // fragment blocks [nblocks][32 lanes][8*MT chunks][4 words]
  const int32_t* pos;
  float* g;
  float* ws;  // partials [chunks][splits][r][64] (splits > 1)
  long long g_sq, g_sc;
  int ldp, ncols, r, blk, chunks, splits, rows_per_split, rows_eff, unit0;
  int nblocks;  // 128-row fragment blocks (gathered: per item ceil(s/128), item-major)
  float scale;
};
struct CgGroup {
  CUtensorMap tx[kCgMaxProbs];  // X: dense box 64 x 128 (SWIZZLE_128B); gathered box 16 x 128 (SWIZZLE_32B)
  CgProb pr[kCgMaxProbs];
  int n_probs, n_items, s, n_units, mt;
};

struct CgSlot {
  int prob, chunk, split, items;  // items: bitmask of the items with work (bit 0 for dense problems)
};

template <int MT>
struct CgSmemL {
  static constexpr int kStages = MT == 1 ? 5 : 4;
  static constexpr int kStageBytes = kCgXBytes + 32 * 8 * MT * 16;  // X tile + fragment block (32 lanes x 8*MT x 16 B)
  static constexpr int kRing = kStages * kStageBytes;
  static constexpr int kBar = kRing;                                // full[S], empty[S]
  static constexpr int kMeta = kBar + 2 * kStages * 8;              // int4 per stage
  static constexpr int kSlots = kMeta + kStages * 16;               // (kCgMaxSlots + 1) slots (+ sentinel)
  static constexpr int kPos = kSlots + (kCgMaxSlots + 1) * 16;      // [slot][item][4] packed column starts
  static constexpr int kTotal = kPos + kCgMaxSlots * kCgMaxItems * 4 * 4 + 1024;
};

LX_DEV void ldsm_x4_trans(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
LX_DEV void bulk_load(void* smem_dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int MT>
__global__ void __launch_bounds__(kCgThreads, 2) colgrad_group_kernel(const __grid_constant__ CgGroup grp) {
  pdl_wait_trigger();
  using L = CgSmemL<MT>;
  constexpr int kCgStages = L::kStages, kCgStageBytes = L::kStageBytes;
  extern __shared__ uint8_t cg_raw[];
  uint8_t* sm = align_smem_1024(cg_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + L::kBar);
  uint64_t* empty = full + kCgStages;
  int4* meta = reinterpret_cast<int4*>(sm + L::kMeta);
  CgSlot* slots = reinterpret_cast<CgSlot*>(sm + L::kSlots);
  int* postab = reinterpret_cast<int*>(sm + L::kPos);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- this CTA's units (round robin) and, for gathered problems, each (unit, item)'s packed column
  // starts of the chunk's four 16-column sub-blocks (-1 inactive): one parallel lookup round
  const int n_slots = (grp.n_units - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  if (tid <= n_slots) {
    CgSlot sl = {0, 0, 0, 0};
    if (tid < n_slots) {
      const int u = blockIdx.x + tid * gridDim.x;
      int pi = 0;
      while (pi + 1 < grp.n_probs && u >= grp.pr[pi + 1].unit0) ++pi;
      const CgProb& P = grp.pr[pi];
      const int local = u - P.unit0;
      sl.prob = pi;
      sl.chunk = local / P.splits;
      sl.split = local % P.splits;
      sl.items = P.pos ? 0 : 1;
    }
    slots[tid] = sl;
  }
  if (tid == 0) {
    for (int i = 0; i < kCgStages; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, kCgConsumers);
    }
    fence_mbar_init();
  }
  __syncthreads();
  for (int e = tid; e < n_slots * kCgMaxItems * 4; e += kCgThreads) {
    const int k = e / (kCgMaxItems * 4), item = (e / 4) % kCgMaxItems, sb = e % 4;
    const CgSlot sl = slots[k];
    const CgProb& P = grp.pr[sl.prob];
    int v = -1;
    if (P.pos && item < grp.n_items) {
      const int oc = sl.chunk * kCgChunk + sb * 16;
      if (oc < P.ncols) {
        const int pb = __ldg(P.pos + (size_t)item * (P.ncols / P.blk) + oc / P.blk);
        if (pb >= 0) v = pb * P.blk + oc % P.blk;
      }
    }
    postab[e] = v;
    if (v >= 0) atomicOr(&slots[k].items, 1 << item);
  }
  __syncthreads();

  if (warp == kCgConsumers) {
    // ================= producer (one thread)
    if (lane == 0 && n_slots > 0) {
      for (int i = 0; i < grp.n_probs; ++i) {
        tma_prefetch_desc(&grp.tx[i]);
      }
      int stage = 0;
      uint32_t phase = 0;
      auto emit = [&](int slot, int prob, int chunk, int row0, int nvalid, int flags, int subs, int item) {
        mbar_wait(empty + stage, phase ^ 1);
        meta[stage] = make_int4(slot, nvalid, flags | (subs << 4), item);
        uint8_t* xs = sm + stage * kCgStageBytes;
        if (flags & kCgEmpty) {
          mbar_arrive(full + stage);
        } else {
          const CgProb& P = grp.pr[prob];
          const int pbytes = 32 * 8 * grp.mt * 16;
          if (flags & kCgGath) {
            mbar_arrive_expect_tx(full + stage, __popc(subs) * (kCgXBytes / 4) + pbytes);
            for (int sb = 0; sb < 4; ++sb)
              if ((subs >> sb) & 1)
                tma_load_2d(xs + sb * (kCgXBytes / 4), &grp.tx[prob], full + stage,
                            postab[(slot * kCgMaxItems + item) * 4 + sb], row0);
          } else {
            mbar_arrive_expect_tx(full + stage, kCgXBytes + pbytes);
            tma_load_2d(xs, &grp.tx[prob], full + stage, chunk * kCgChunk, row0);
          }
          const int blk_i = (flags & kCgGath) ? item * ((grp.s + kCgRows - 1) / kCgRows) + (row0 - item * grp.s) / kCgRows
                                              : row0 / kCgRows;
          bulk_load(xs + kCgXBytes, P.pt + (size_t)blk_i * 32 * 8 * grp.mt * 4, pbytes, full + stage);
        }
        if (++stage == kCgStages) { stage = 0; phase ^= 1; }
      };
      for (int k = 0; k < n_slots; ++k) {
        const CgSlot sl = slots[k];
        const CgProb& P = grp.pr[sl.prob];
        const int nr = min(P.rows_per_split, P.rows_eff - sl.split * P.rows_per_split);
        if (P.pos == nullptr) {
          const int nst = (nr + kCgRows - 1) / kCgRows;
          for (int st = 0; st < nst; ++st)
            emit(k, sl.prob, sl.chunk, sl.split * P.rows_per_split + st * kCgRows, min(kCgRows, nr - st * kCgRows),
                 st == nst - 1 ? kCgLast : 0, 0xF, 0);
        } else if (sl.items == 0) {
          emit(k, sl.prob, sl.chunk, 0, 0, kCgLast | kCgEmpty, 0, 0);
        } else {
          for (int m = sl.items; m; m &= m - 1) {
            const int item = __ffs(m) - 1;
            int subs = 0;
            for (int sb = 0; sb < 4; ++sb) subs |= (postab[(k * kCgMaxItems + item) * 4 + sb] >= 0) << sb;
            emit(k, sl.prob, sl.chunk, item * grp.s + sl.split * P.rows_per_split, nr,
                 kCgGath | ((m & (m - 1)) == 0 ? kCgLast : 0), subs, item);
          }
        }
      }
    }
    return;
  }

  // ================= consumers: warp w owns columns 8w .. 8w+7 of the chunk
  const int g = lane >> 2, t = lane & 3;
  const int lm_row = (lane >> 3) * 8 + (lane & 7);  // ldmatrix.trans: matrix lane/8 = k rows 8*(lane/8)..
  float acc[MT][4];
#pragma unroll
  for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.f;
  int stage = 0;
  uint32_t phase = 0;
#pragma unroll 1
  for (int k = 0; k < n_slots;) {
    mbar_wait(full + stage, phase);
    const int4 mt4 = meta[stage];
    const int flags = mt4.z & 0xF, subs = mt4.z >> 4;
    const CgSlot sl = slots[mt4.x];
    const CgProb& P = grp.pr[sl.prob];
    const uint32_t xs = smem_u32(sm + stage * kCgStageBytes);
    const bool active = !(flags & kCgEmpty) &&
                        ((flags & kCgGath) ? ((subs >> (warp >> 1)) & 1) : (sl.chunk * kCgChunk + 8 * warp < P.ncols));
    if (active) {
      // this lane's A fragments of the block: chunk j at rotated position (j + lane) % (8*MT)
      const uint32_t pa = xs + kCgXBytes + lane * (8 * MT * 16);
#pragma unroll
      for (int h = 0; h < 4; ++h) {  // 32-row quarters: one ldmatrix.x4.trans = B of two k-steps
        const int row = h * 32 + lm_row;
        uint32_t b[4];
        const uint32_t xa = (flags & kCgGath)
                                ? xs + (warp >> 1) * (kCgXBytes / 4) + row * 32 + (((warp & 1) ^ ((row >> 2) & 1)) << 4)
                                : xs + row * 128 + ((warp ^ (row & 7)) << 4);
        ldsm_x4_trans(xa, b);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
          for (int m = 0; m < MT; ++m) {
            const int j = (h * 2 + kk) * MT + m;
            uint32_t a[4];
            asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3])
                         : "r"(pa + (((j + lane) & (8 * MT - 1)) << 4)));
            mma16816_rp(acc[m], a, b[2 * kk], b[2 * kk + 1]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + stage);
    if (++stage == kCgStages) { stage = 0; phase ^= 1; }
    if (flags & kCgLast) {
      // unit done: rows g (hi) and g+8 (lo) of m-tile m are rank q = g + 8m; columns 8w + 2t, +1
      const int col = sl.chunk * kCgChunk + 8 * warp + 2 * t;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const int q = g + 8 * m;
        const float v0 = acc[m][0] + acc[m][2], v1 = acc[m][1] + acc[m][3];
        acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.f;
        if (q >= P.r || col >= P.ncols) continue;
        if (P.splits == 1) {
          P.g[(long long)q * P.g_sq + (long long)col * P.g_sc] = v0 * P.scale;
          P.g[(long long)q * P.g_sq + (long long)(col + 1) * P.g_sc] = v1 * P.scale;
        } else {
          float* part = P.ws + (((size_t)sl.chunk * P.splits + sl.split) * P.r + q) * kCgChunk + 8 * warp + 2 * t;
          *reinterpret_cast<float2*>(part) = make_float2(v0, v1);
        }
      }
      ++k;
    }
  }
}

// fragment blocks: block bi, lane (g, t), chunk j = k-step * MT + m holds the m16n8k16 A fragment of
// k-step rows 16*ks + {2t, 2t+1, 2t+8, 2t+9}: regs (hi, lo, hi, lo) of rank q = 8m + g
__global__ void colgrad_prep_kernel(const __grid_constant__ CgGroup grp) {
  pdl_wait_trigger();
  const CgProb& P = grp.pr[blockIdx.y];
  const int MT = grp.mt, nw = 32 * 8 * MT * 4;  // words per block
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= P.nblocks * nw) return;
  const int bi = e / nw, w = e % nw;
  const int lane = w / (8 * MT * 4), pos = (w / 4) % (8 * MT), reg = w % 4;
  const int j = (pos - lane) & (8 * MT - 1);  // logical chunk stored at rotated position pos
  const int ks = j / MT, m = j % MT, g = lane >> 2, t = lane & 3;
  const int q = 8 * m + g;
  // block rows -> activation rows
  int row_base, nvalid;
  if (P.pos) {
    const int nsb = (grp.s + kCgRows - 1) / kCgRows;
    const int item = bi / nsb, sb = bi % nsb;
    row_base = item * grp.s + sb * kCgRows;
    nvalid = min(kCgRows, grp.s - sb * kCgRows);
  } else {
    row_base = bi * kCgRows;
    nvalid = min(kCgRows, grp.n_items * grp.s - row_base);
  }
  const int k0 = ks * 16 + 2 * t + (reg >= 2 ? 8 : 0);
  uint32_t word = 0;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int k = k0 + half;
    float v = 0.f;
    if (k < nvalid && q < P.r) v = P.p ? __ldg(P.p + (size_t)(row_base + k) * P.ldp + q) : 1.f;
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    const __nv_bfloat16 out = (reg & 1) ? __float2bfloat16_rn(v - __bfloat162float(hi)) : hi;
    word |= (uint32_t)__bfloat16_as_ushort(out) << (16 * half);
  }
  P.pt[e] = word;
}

// G(q, c) = scale * sum over splits (in order) of the partials, for the problems with splits > 1
__global__ void colgrad_final_kernel(const __grid_constant__ CgGroup grp) {
  pdl_wait_trigger();
  const CgProb& P = grp.pr[blockIdx.y];
  if (P.splits == 1) return;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= P.chunks * P.r * kCgChunk) return;
  const int chunk = e / (P.r * kCgChunk), q = (e / kCgChunk) % P.r, c = e % kCgChunk;
  const int col = chunk * kCgChunk + c;
  if (col >= P.ncols) return;
  const float* src = P.ws + ((size_t)chunk * P.splits * P.r + q) * kCgChunk + c;
  float v = 0.f;
#pragma unroll 4
  for (int sp = 0; sp < P.splits; ++sp) v += src[(size_t)sp * P.r * kCgChunk];
  P.g[(long long)q * P.g_sq + (long long)col * P.g_sc] = v * P.scale;
}

// host-side layout of one problem (shared by the workspace query and the launch)
static void cg_layout(const lx_colgrad_problem& q, int n_items, int s, CgProb& o) {
  o.chunks = (q.ncols + kCgChunk - 1) / kCgChunk;
  const bool gathered = q.pos != nullptr;
  o.rows_eff = gathered ? s : n_items * s;
  o.rows_per_split = gathered ? kCgRows : kCgRowsDense;
  o.splits = (o.rows_eff + o.rows_per_split - 1) / o.rows_per_split;
  o.nblocks = gathered ? n_items * ((s + kCgRows - 1) / kCgRows) : (n_items * s + kCgRows - 1) / kCgRows;
}

static int cg_mt(const lx_colgrad_problem* probs, int n) {
  int mr = 0;
  for (int i = 0; i < n; ++i) mr = probs[i].r > mr ? probs[i].r : mr;
  return mr > 8 ? 2 : 1;
}

// floats: fragment blocks (32 * 8 * MT * 4 words per block) + partials, each rounded to 64 floats (256 B)
static long long cg_ws_floats(const lx_colgrad_problem& q, int n_items, int s, int mt, long long* pt_floats) {
  CgProb o;
  cg_layout(q, n_items, s, o);
  const long long pt = (long long)o.nblocks * 32 * 8 * mt * 4;
  const long long part = o.splits > 1 ? ((long long)o.chunks * o.splits * q.r * kCgChunk + 63) / 64 * 64 : 0;
  if (pt_floats) *pt_floats = pt;
  return pt + part;
}

}  // namespace lx

using namespace lx;

// the dynamic shared-memory opt-in of rowproj_smem_kernel is per instantiation: set once for all four
static cudaError_t rowproj_smem_attr() {
  static const cudaError_t attr = [] {
    cudaError_t e = cudaFuncSetAttribute(rowproj_smem_kernel<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(rowproj_smem_kernel<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(rowproj_smem_kernel<2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(rowproj_smem_kernel<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    return e;
  }();
  return attr;
}

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
    launch_k(rowproj_wpack_kernel, gp, 256, 0, stream, w, w_sk, w_sq, r, RP, K, Kp, counts, ids, ids_stride, b,
                                                 reinterpret_cast<__nv_bfloat16*>(wpack_ws));
    int rc = launch_check("rowproj_wpack");
    if (rc) return rc;
    dim3 grid((s + 15) / 16, n_items);
    const auto* wpb = reinterpret_cast<const __nv_bfloat16*>(wpack_ws);
    if (!counts && n_items > 1) {
      // dense W is shared by all items: index it as item 0 by treating the batch as one item
      grid = dim3((n_items * s + 15) / 16, 1);
      if (NT == 1)
        launch_k(rowproj_mma2_kernel<1>, grid, 32 * kRpWarps, 0, stream, xb, ldx, n_items * s, K, Kp, r, scale, nullptr, b, wpb,
                                                                   2LL * 8 * Kp, nullptr, 0, y, ldy, nullptr, 0);
      else
        launch_k(rowproj_mma2_kernel<2>, grid, 32 * kRpWarps, 0, stream, xb, ldx, n_items * s, K, Kp, r, scale, nullptr, b, wpb,
                                                                   2LL * 16 * Kp, nullptr, 0, y, ldy, nullptr, 0);
    } else if (NT == 1) {
      launch_k(rowproj_mma2_kernel<1>, grid, 32 * kRpWarps, 0, stream, xb, ldx, s, K, Kp, r, scale, counts, b, wpb, 2LL * 8 * Kp,
                                                                 nullptr, 0, y, ldy, nullptr, 0);
    } else {
      launch_k(rowproj_mma2_kernel<2>, grid, 32 * kRpWarps, 0, stream, xb, ldx, s, K, Kp, r, scale, counts, b, wpb, 2LL * 16 * Kp,
                                                                 nullptr, 0, y, ldy, nullptr, 0);
    }
    return launch_check("rowproj_mma");
  }
  dim3 grid((s + kRpRows - 1) / kRpRows, n_items);
  if (r <= 8)
    launch_k(rowproj_kernel<8>, grid, 256, 0, stream, xb, ldx, s, K, w, w_sk, w_sq, r, scale, counts, ids, ids_stride, b, y, ldy);
  else
    launch_k(rowproj_kernel<16>, grid, 256, 0, stream, xb, ldx, s, K, w, w_sk, w_sq, r, scale, counts, ids, ids_stride, b, y, ldy);
  return launch_check("rowproj");
}

int lx_rowproj_packed(const uint16_t* x, int ldx, int n_items, int s, int K, const uint16_t* wpack, int K_full, int RP,
                      int r, float scale, const int32_t* counts, const int32_t* ids, int blk, float* y, int ldy,
                      uint16_t* yb, int ldyb, lx_stream_t stream) {
  LX_REQUIRE(RP == 8 || RP == 16, LX_ERR_UNSUPPORTED, "rowproj_packed: RP must be 8 or 16");
  LX_REQUIRE(r >= 1 && r <= RP, LX_ERR_UNSUPPORTED, "rowproj_packed: rank %d outside [1, RP]", r);
  LX_REQUIRE(ldy >= r && (!yb || ldyb >= r), LX_ERR_SHAPE, "rowproj_packed: output stride < r");
  LX_REQUIRE(K % 16 == 0 && K_full % 8 == 0 && ldx % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                 (reinterpret_cast<uintptr_t>(wpack) & 15) == 0,
             LX_ERR_SHAPE, "rowproj_packed: K % 16, 16B-aligned rows and pack required");
  LX_REQUIRE(!counts || (ids && blk % 8 == 0 && K % blk == 0), LX_ERR_MASK, "rowproj_packed: gathered K needs ids, blk % 8");
  LX_REQUIRE(counts || K <= K_full, LX_ERR_SHAPE, "rowproj_packed: K exceeds the pack");
  const auto* xb = reinterpret_cast<const __nv_bfloat16*>(x);
  const auto* wp = reinterpret_cast<const __nv_bfloat16*>(wpack);
  auto* ybf = reinterpret_cast<__nv_bfloat16*>(yb);
  const int items = counts ? n_items : 1, rows = counts ? s : n_items * s;
  dim3 grid((rows + 15) / 16, items);
  static const bool use_smem = [] { const char* e = getenv("LX_ROWPROJ_SMEM"); return !(e && e[0] == '0'); }();
  if (!counts && use_smem && K <= kRpsMaxK && K % 8 == 0 && ldx % 8 == 0) {
    // dense K: X rows staged in shared memory by bulk copies (rowproj_smem_kernel), 32 rows per CTA when they fit
    const bool two = (size_t)32 * (K + 32) * 2 <= 160 * 1024;
    const dim3 g2((rows + (two ? 31 : 15)) / (two ? 32 : 16));
    const size_t smem = (size_t)(two ? 32 : 16) * (K + 32) * 2;
    const cudaError_t attr = rowproj_smem_attr();
    LX_CHECK_CUDA(attr);
    auto kern = RP == 8 ? (two ? rowproj_smem_kernel<1, 2> : rowproj_smem_kernel<1, 1>)
                        : (two ? rowproj_smem_kernel<2, 2> : rowproj_smem_kernel<2, 1>);
    launch_k(kern, g2, 32 * kRpWarps, smem, stream, xb, ldx, rows, K, K_full, r, scale, wp, y, ldy, ybf, ldyb, 0LL, 0LL, 0, 0);
    return launch_check("rowproj_smem");
  }

  if (RP == 8)
    launch_k(rowproj_mma2_kernel<1>, grid, 32 * kRpWarps, 0, stream, xb, ldx, rows, K, K_full, r, scale, counts, counts ? blk : 1, wp,
                                                               0, counts ? ids : nullptr, counts ? K / blk : 0, y, ldy, ybf, ldyb);
  else
    launch_k(rowproj_mma2_kernel<2>, grid, 32 * kRpWarps, 0, stream, xb, ldx, rows, K, K_full, r, scale, counts, counts ? blk : 1, wp,
                                                               0, counts ? ids : nullptr, counts ? K / blk : 0, y, ldy, ybf, ldyb);
  return launch_check("rowproj_packed");
}

int lx_rowproj_packed_seg(const uint16_t* x, int ldx, long long x_seg, int n_rows, int K, const uint16_t* wpack,
                          long long w_seg, int K_full, int RP, int r, float scale, float* y, int ldy, int y_seg, uint16_t* yb,
                          int ldyb, int yb_seg, int n_seg, lx_stream_t stream) {
  LX_REQUIRE(RP == 8 || RP == 16, LX_ERR_UNSUPPORTED, "rowproj_packed_seg: RP must be 8 or 16");
  LX_REQUIRE(r >= 1 && r <= RP && n_seg >= 1 && n_seg <= 65535 && n_rows >= 1, LX_ERR_SHAPE,
             "rowproj_packed_seg: rank %d / segments %d / rows %d", r, n_seg, n_rows);
  LX_REQUIRE(ldy >= r && (!yb || ldyb >= r), LX_ERR_SHAPE, "rowproj_packed_seg: output stride < r");
  LX_REQUIRE(K % 16 == 0 && K <= K_full && K <= kRpsMaxK && ldx % 8 == 0 && x_seg % 8 == 0 && w_seg % 8 == 0 &&
                 (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(wpack) & 15) == 0,
             LX_ERR_SHAPE, "rowproj_packed_seg: dense K (%% 16, <= %d) with 16-byte aligned rows, segments and pack", kRpsMaxK);
  LX_CHECK_CUDA(rowproj_smem_attr());
  const bool two = (size_t)32 * (K + 32) * 2 <= 160 * 1024;
  const dim3 g2((n_rows + (two ? 31 : 15)) / (two ? 32 : 16), n_seg);
  const size_t smem = (size_t)(two ? 32 : 16) * (K + 32) * 2;
  auto kern = RP == 8 ? (two ? rowproj_smem_kernel<1, 2> : rowproj_smem_kernel<1, 1>)
                      : (two ? rowproj_smem_kernel<2, 2> : rowproj_smem_kernel<2, 1>);
  launch_k(kern, g2, 32 * kRpWarps, smem, stream, reinterpret_cast<const __nv_bfloat16*>(x), ldx, n_rows, K, K_full, r, scale,
           reinterpret_cast<const __nv_bfloat16*>(wpack), y, ldy, reinterpret_cast<__nv_bfloat16*>(yb), ldyb, x_seg, w_seg,
           y_seg, yb_seg);
  return launch_check("rowproj_packed_seg");
}

int lx_pack_params(const lx_pack_segment* segs, int n_segs, lx_stream_t stream) {
  LX_REQUIRE(n_segs >= 0, LX_ERR_SHAPE, "pack_params: negative segment count");
  if (n_segs == 0) return LX_OK;
  launch_k(pack_params_kernel, dim3(64, n_segs), 256, 0, stream, segs);
  return launch_check("pack_params");
}

long long lx_colgrad_group_ws_floats(const lx_colgrad_problem* probs, int n_probs, int n_items, int s) {
  const int mt = cg_mt(probs, n_probs);
  long long tot = 0;
  for (int i = 0; i < n_probs; ++i) tot += cg_ws_floats(probs[i], n_items, s, mt, nullptr);
  return tot;
}

int lx_colgrad_group(const lx_colgrad_problem* probs, int n_probs, int n_items, int s, float* ws, lx_stream_t stream) {
  LX_REQUIRE(n_probs >= 1 && n_probs <= kCgMaxProbs, LX_ERR_UNSUPPORTED, "colgrad_group: 1..%d problems", kCgMaxProbs);
  LX_REQUIRE(n_items >= 1 && s >= 1, LX_ERR_SHAPE, "colgrad_group: empty batch");
  LX_REQUIRE(ws != nullptr && (reinterpret_cast<uintptr_t>(ws) & 255) == 0, LX_ERR_SHAPE,
             "colgrad_group: 256B-aligned workspace required");
  CgGroup grp;
  memset(&grp, 0, sizeof(grp));
  grp.n_probs = n_probs;
  grp.n_items = n_items;
  grp.s = s;
  grp.mt = cg_mt(probs, n_probs);
  const int M = n_items * s;
  int units = 0, max_final = 0, max_blk_words = 0;
  long long ws_off = 0;
  for (int i = 0; i < n_probs; ++i) {
    const lx_colgrad_problem& q = probs[i];
    LX_REQUIRE(q.r >= 1 && q.r <= 16, LX_ERR_UNSUPPORTED, "colgrad: rank %d outside [1, 16]", q.r);
    LX_REQUIRE(!q.p || q.ldp >= q.r, LX_ERR_SHAPE, "colgrad: ldp < r");
    LX_REQUIRE(q.ncols % 8 == 0, LX_ERR_SHAPE, "colgrad: ncols must be a multiple of 8");
    LX_REQUIRE(!q.pos || (q.blk % 16 == 0 && q.ncols % q.blk == 0), LX_ERR_MASK,
               "colgrad: gathered columns need blk %% 16 == 0 and ncols %% blk == 0");
    LX_REQUIRE(!q.pos || n_items <= kCgMaxItems, LX_ERR_UNSUPPORTED, "colgrad: gathered problems take <= %d items",
               kCgMaxItems);
    LX_REQUIRE(q.ldx % 8 == 0 && (reinterpret_cast<uintptr_t>(q.x) & 15) == 0, LX_ERR_SHAPE,
               "colgrad: 16B-aligned rows required");
    CgProb& o = grp.pr[i];
    cg_layout(q, n_items, s, o);
    long long pt_floats = 0;
    const long long need = cg_ws_floats(q, n_items, s, grp.mt, &pt_floats);
    o.p = q.p;
    o.pt = reinterpret_cast<uint32_t*>(ws + ws_off);
    o.ws = ws + ws_off + pt_floats;
    ws_off += need;
    o.pos = q.pos;
    o.g = q.g;
    o.g_sq = q.g_sq;
    o.g_sc = q.g_sc;
    o.ldp = q.ldp;
    o.ncols = q.ncols;
    o.r = q.r;
    o.blk = q.pos ? q.blk : 1;
    o.scale = q.scale;
    o.unit0 = units;
    units += o.chunks * o.splits;
    if (o.splits > 1) max_final = std::max(max_final, o.chunks * q.r * kCgChunk);
    max_blk_words = std::max(max_blk_words, o.nblocks * 32 * 8 * grp.mt * 4);
    int rc = q.pos ? make_tmap_bf16_2d_sw(&grp.tx[i], q.x, (uint64_t)q.ldx, (uint64_t)M, (uint64_t)q.ldx, 16, kCgRows,
                                          CU_TENSOR_MAP_SWIZZLE_32B)
                   : make_tmap_bf16_2d_sw(&grp.tx[i], q.x, (uint64_t)q.ncols, (uint64_t)M, (uint64_t)q.ldx, 64, kCgRows,
                                          CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
  }
  grp.n_units = units;
  const int grid = std::max(std::min(units, 2 * num_sms()), (units + kCgMaxSlots - 1) / kCgMaxSlots);
  LX_REQUIRE((units + grid - 1) / grid <= kCgMaxSlots, LX_ERR_UNSUPPORTED, "colgrad_group: too many units");
  launch_k(colgrad_prep_kernel, dim3((max_blk_words + 255) / 256, n_probs), 256, 0, stream, grp);
  int rc = launch_check("colgrad_prep");
  if (rc) return rc;
  if (grp.mt == 2) {
    constexpr int smem = CgSmemL<2>::kTotal;
    static cudaError_t attr = cudaFuncSetAttribute(colgrad_group_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    LX_CHECK_CUDA(attr);
    launch_k(colgrad_group_kernel<2>, grid, kCgThreads, smem, stream, grp);
  } else {
    constexpr int smem = CgSmemL<1>::kTotal;
    static cudaError_t attr = cudaFuncSetAttribute(colgrad_group_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    LX_CHECK_CUDA(attr);
    launch_k(colgrad_group_kernel<1>, grid, kCgThreads, smem, stream, grp);
  }
  rc = launch_check("colgrad_group");
  if (rc || max_final == 0) return rc;
  launch_k(colgrad_final_kernel, dim3((max_final + 255) / 256, n_probs), 256, 0, stream, grp);
  return launch_check("colgrad_final");
}

}  // extern "C"
