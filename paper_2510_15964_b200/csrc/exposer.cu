// Exposer oracle mode on the GPU — the dense ground truth the predictors are trained against
// and checked by (sf/exposer.py:47-111, used by OracleProvider / ShadowyProvider,
// sf/harness.py:157-190). Verification mode: it pays the dense cost the hot path avoids.
//
// Attention (exact_attention + block_mass, sf/exposer.py:47-68): one CTA per (query block, head,
//   item). Sub-tiles of 16 query rows: raw dot products in fp32 FFMA (the reference's float32
//   matmul), staged as one [16 x s] row strip in shared memory; then per row, in float64 like the
//   reference (the np.float64 scale promotes raw scores to float64): scale, max, exp, sum, divide;
//   the probabilities are summed into the n_b key blocks with fixed-order warp reductions, so the
//   [n_b x n_b] block-mass grid is deterministic.
// Pattern choice (select_pattern_by_coverage, sf/exposer.py:71-85): one thread per (item, head)
//   (or per item, heads summed in head order, for the shadowy provider sf/harness.py:183-187):
//   total = numpy's pairwise float64 sum of the grid, each pattern's mass a sequential float64 sum
//   over its row-major cells, mass/total >= tau - 1e-9, fewest blocks then pool order, else dense.
//   Given the same grid the index is bit-identical to the reference.
// MLP (block_importance + filter_neuron_blocks, sf/exposer.py:94-111): max of relu(z) per
//   (item, neuron block) — a max is order-free, so integer atomicMax on the non-negative float bits
//   is deterministic — then peak-relative float64 filtering into the bitmask the compaction kernel
//   (mask_build.cu) lowers to NeuronMasks.
#include <algorithm>

#include "common.cuh"
#include "ptx.cuh"

namespace lx {

constexpr int kExRows = 16;    // query rows per sub-tile
constexpr int kExKeys = 128;   // keys per staged K tile
constexpr int kExThreads = 256;
constexpr int kExMaxNb = 64;
constexpr int kExMaxPool = 16;

__device__ __forceinline__ bool ex_pool_member(int kind, int p, int i, int j) {  // sf/patterns.py:63-85
  const int dd = i - j;
  switch (kind) {
    case 0: return dd == 0;
    case 1: return dd <= p && dd >= -p;
    case 2: return dd >= 0 && dd <= p;
    case 3: return i < p || j < p || dd == 0;
    case 4: return ((dd % p) + p) % p == 0;
    default: return true;
  }
}

// grid (n_b, H, n_items); q and k fp32 rows [n_items * s, ld] (own base pointers), head h at columns h*hd
__global__ void __launch_bounds__(kExThreads) exact_mass_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                                                int ld, int s, int H, int hd, int n_b, double scale,
                                                                double* __restrict__ mass) {
  pdl_wait_trigger();  // launched with PDL (launch_k): see the predecessor's writes first
  extern __shared__ float ex_smem[];
  const int br = blockIdx.x, h = blockIdx.y, item = blockIdx.z;
  const int blk = s / n_b;
  const int ks = hd | 1;  // odd K row stride: lane-distinct key rows hit distinct banks
  float* Qs = ex_smem;                   // [16][hd]
  float* Ks = Qs + kExRows * hd;         // [128][ks]
  float* Ss = Ks + kExKeys * ks;         // [16][s]
  __shared__ double part[kExThreads / 32][kExMaxNb];
  __shared__ double acc[kExMaxNb];
  __shared__ double rowe[kExThreads / 32][kExMaxNb];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = threadIdx.x; c < n_b; c += blockDim.x) acc[c] = 0.0;
  const float* qh = q + (size_t)item * s * ld + h * hd;
  const float* kh = k + (size_t)item * s * ld + h * hd;
  // 16-byte rows: every head's row start is float4-aligned
  const bool vec = (hd & 3) == 0 && (ld & 3) == 0 && ((reinterpret_cast<uintptr_t>(kh) & 15) == 0);
  for (int r0 = 0; r0 < blk; r0 += kExRows) {
    const int nr = min(kExRows, blk - r0);
    __syncthreads();
    for (int e = threadIdx.x; e < kExRows * hd; e += blockDim.x) {
      const int r = e / hd, c = e % hd;
      Qs[e] = r < nr ? qh[(size_t)(br * blk + r0 + r) * ld + c] : 0.f;
    }
    // raw dot products: warp w owns rows 2w, 2w+1; lane owns keys lane + 32u of each 128-key tile
    for (int j0 = 0; j0 < s; j0 += kExKeys) {
      const int nk = min(kExKeys, s - j0);
      __syncthreads();
      if (vec) {
        // float4 loads issued in batches of 8 before any shared store: one memory round trip per batch
        const int hd4 = hd >> 2, n4 = kExKeys * hd4;
        for (int e0 = threadIdx.x; e0 < n4; e0 += 8 * kExThreads) {
          float4 v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * kExThreads, j = e / hd4;
            v[u] = (e < n4 && j < nk) ? __ldg(reinterpret_cast<const float4*>(kh + (size_t)(j0 + j) * ld) + e % hd4)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * kExThreads;
            if (e < n4) {
              float* dst = Ks + (e / hd4) * ks + 4 * (e % hd4);
              dst[0] = v[u].x, dst[1] = v[u].y, dst[2] = v[u].z, dst[3] = v[u].w;
            }
          }
        }
      } else {
        for (int e = threadIdx.x; e < kExKeys * hd; e += blockDim.x) {
          const int j = e / hd, c = e % hd;
          Ks[j * ks + c] = j < nk ? kh[(size_t)(j0 + j) * ld + c] : 0.f;
        }
      }
      __syncthreads();
      float a[2][4];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int u = 0; u < 4; ++u) a[i][u] = 0.f;
      const float* q0 = Qs + (2 * warp) * hd;
      const float* q1 = q0 + hd;
      for (int c = 0; c < hd; ++c) {
        const float x0 = q0[c], x1 = q1[c];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float kv = Ks[(lane + 32 * u) * ks + c];
          a[0][u] = fmaf(x0, kv, a[0][u]);
          a[1][u] = fmaf(x1, kv, a[1][u]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = lane + 32 * u;
        if (j < nk) {
          Ss[(2 * warp) * s + j0 + j] = a[0][u];
          Ss[(2 * warp + 1) * s + j0 + j] = a[1][u];
        }
      }
    }
    __syncthreads();
    // float64 softmax per row and block sums (sf/tensor_core.py:85-91, sf/exposer.py:62-68)
    for (int c = threadIdx.x; c < (kExThreads / 32) * n_b; c += blockDim.x) part[c / n_b][c % n_b] = 0.0;
    __syncthreads();
    for (int rr = 0; rr < 2; ++rr) {
      const int r = 2 * warp + rr;
      if (r >= nr) continue;
      const float* row = Ss + r * s;
      double mx = -INFINITY;
      for (int j = lane; j < s; j += 32) mx = fmax(mx, (double)row[j] * scale);
      for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      // one exp per element: block sums of e = exp(raw - max) first, the row sum is their fixed-order
      // total, and each block's probability mass is its e-sum / row sum (= the sum of e / row sum up
      // to float64 rounding)
      for (int bc = 0; bc < n_b; ++bc) {
        double ps = 0.0;
        for (int j = bc * blk + lane; j < (bc + 1) * blk; j += 32) ps += exp((double)row[j] * scale - mx);
        for (int o = 16; o; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
        if (lane == 0) rowe[warp][bc] = ps;
      }
      __syncwarp();
      if (lane == 0) {
        double sum = 0.0;
        for (int bc = 0; bc < n_b; ++bc) sum += rowe[warp][bc];
        for (int bc = 0; bc < n_b; ++bc) part[warp][bc] += rowe[warp][bc] / sum;  // rows 2w then 2w+1
      }
      __syncwarp();
    }
    __syncthreads();
    for (int bc = threadIdx.x; bc < n_b; bc += blockDim.x) {
      double t = acc[bc];
      for (int w = 0; w < kExThreads / 32; ++w) t += part[w][bc];
      acc[bc] = t;
    }
  }
  __syncthreads();
  for (int bc = threadIdx.x; bc < n_b; bc += blockDim.x)
    mass[(((size_t)item * H + h) * n_b + br) * n_b + bc] = acc[bc];
}

// numpy's pairwise float64 sum (numpy/_core/src/umath/loops_utils.h.src, PW_BLOCKSIZE 128) over a
// contiguous run: < 8 sequential, <= 128 eight strided accumulators, else split at an 8-aligned half
__device__ double np_pairwise_sum(const double* a, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

// one warp per (item, head) grid — or per item with the heads summed (shadowy). Lanes own pool
// patterns (each pattern's mass is the reference's sequential sum over its row-major cells); lane 0
// takes numpy's pairwise total and the fewest-blocks / pool-order choice.
__global__ void coverage_select_kernel(const double* __restrict__ mass, int n_items, int H, int n_b,
                                       const int32_t* __restrict__ pool_kind, const int32_t* __restrict__ pool_param,
                                       int n_pool, double tau, int head_sum, int32_t* __restrict__ pattern_idx) {
  pdl_wait_trigger();  // launched with PDL (launch_k): see the predecessor's writes first
  const int n_sel = head_sum ? n_items : n_items * H;
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= n_sel) return;
  const int cells = n_b * n_b;
  extern __shared__ double sel_smem[];
  double* g = sel_smem + (size_t)(threadIdx.x >> 5) * cells;  // this warp's grid, staged once
  if (head_sum) {  // sum(block_mass(p) for p in probs): elementwise, head order
    const double* base = mass + (size_t)t * H * cells;
    for (int e = lane; e < cells; e += 32) {
      double v = base[e];
      for (int hh = 1; hh < H; ++hh) v += base[(size_t)hh * cells + e];
      g[e] = v;
    }
  } else {
    const double* src = mass + (size_t)t * cells;
    for (int e = lane; e < cells; e += 32) g[e] = src[e];
  }
  __syncwarp();
  double m = 0.0;
  int nnz = 0;
  if (lane < n_pool) {
    const int kind = pool_kind[lane], prm = pool_param[lane];
    for (int i = 0; i < n_b; ++i)
      for (int j = 0; j < n_b; ++j)
        if (ex_pool_member(kind, prm, i, j)) {
          m += g[i * n_b + j];
          ++nnz;
        }
  }
  const double total = lane == 0 ? np_pairwise_sum(g, cells) : 0.0;
  __shared__ double s_m[8][kExMaxPool];
  __shared__ int s_n[8][kExMaxPool];
  const int wl = threadIdx.x >> 5;
  if (lane < n_pool) s_m[wl][lane] = m, s_n[wl][lane] = nnz;
  __syncwarp();
  if (lane == 0) {
    int best = -1, best_n = 0;
    if (total > 0) {
      const double thr = tau - 1e-9;
      for (int p = 0; p < n_pool; ++p)
        if (s_m[wl][p] / total >= thr && (best < 0 || s_n[wl][p] < best_n)) best = p, best_n = s_n[wl][p];
    }
    const int pick = best < 0 ? n_pool - 1 : best;  // dense is the pool's last entry
    if (head_sum) {
      for (int hh = 0; hh < H; ++hh) pattern_idx[(size_t)t * H + hh] = pick;
    } else {
      pattern_idx[t] = pick;
    }
  }
}

// grid (ceil(n_cols / 256), row chunks, n_items): thread = one column, max over its rows, then the
// block max through the non-negative float bits (atomicMax on int is exact and order-free)
__global__ void block_importance_kernel(const float* __restrict__ z, int ldz, int s, int n_cols, int blk,
                                        int rows_per_cta, int n_blk, int* __restrict__ imp_bits) {
  pdl_wait_trigger();  // launched with PDL (launch_k): see the predecessor's writes first
  const int item = blockIdx.z;
  const int r0 = blockIdx.y * rows_per_cta, r1 = min(s, r0 + rows_per_cta);
  const bool vec = (n_cols & 3) == 0 && (ldz & 3) == 0 && (blk & 3) == 0;
  const int col = (blockIdx.x * blockDim.x + threadIdx.x) * (vec ? 4 : 1);  // first of this thread's columns
  float m = 0.f;  // relu: max(z, 0) >= 0, and |relu| = relu
  if (col < n_cols) {
    const float* zc = z + (size_t)item * s * ldz + col;
    if (vec) {  // four columns of one block per thread, 512 B per warp per row
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int r = r0; r < r1; ++r) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(zc + (size_t)r * ldz));
        a.x = fmaxf(a.x, v.x), a.y = fmaxf(a.y, v.y), a.z = fmaxf(a.z, v.z), a.w = fmaxf(a.w, v.w);
      }
      m = fmaxf(fmaxf(a.x, a.y), fmaxf(a.z, a.w));
    } else {
      for (int r = r0; r < r1; ++r) m = fmaxf(m, zc[(size_t)r * ldz]);
    }
  }
  if (col < n_cols && m > 0.f) atomicMax(imp_bits + (size_t)item * n_blk + col / blk, __float_as_int(m));
}

// one warp per item: peak, then active iff (double)imp > theta * peak (strict), all-zero -> none
__global__ void filter_blocks_kernel(const float* __restrict__ imp, int n_items, int n_blk, double theta,
                                     uint32_t* __restrict__ bits) {
  pdl_wait_trigger();  // launched with PDL (launch_k): see the predecessor's writes first
  const int item = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (item >= n_items) return;
  const float* v = imp + (size_t)item * n_blk;
  float pk = 0.f;
  for (int b = lane; b < n_blk; b += 32) pk = fmaxf(pk, v[b]);
  for (int o = 16; o; o >>= 1) pk = fmaxf(pk, __shfl_xor_sync(0xffffffffu, pk, o));
  const double cut = theta * (double)pk;
  const int words = (n_blk + 31) / 32;
  for (int w0 = 0; w0 < words; ++w0) {
    const int b = w0 * 32 + lane;
    const bool on = pk > 0.f && b < n_blk && (double)v[b] > cut;
    const uint32_t word = __ballot_sync(0xffffffffu, on);
    if (lane == 0) bits[(size_t)item * words + w0] = word;
  }
}

}  // namespace lx

using namespace lx;

extern "C" {

size_t lx_exact_mass_smem(int s, int hd) {
  return sizeof(float) * ((size_t)kExRows * hd + (size_t)kExKeys * (hd | 1) + (size_t)kExRows * s);
}

int lx_exact_block_mass(const float* q, const float* k, int ld, int n_items, int s, int H, int hd, int n_b,
                        double* mass, lx_stream_t stream) {
  LX_REQUIRE(n_items >= 1 && s >= 1 && H >= 1 && hd >= 1 && n_b >= 1, LX_ERR_SHAPE, "exact_block_mass: empty shape");
  LX_REQUIRE(s % n_b == 0, LX_ERR_LAYOUT, "matrix side %d not divisible by grid side %d", s, n_b);
  LX_REQUIRE(n_b <= kExMaxNb, LX_ERR_UNSUPPORTED, "grid side %d > %d", n_b, kExMaxNb);
  LX_REQUIRE(ld >= H * hd, LX_ERR_SHAPE, "row stride %d < H*hd", ld);
  const size_t smem = lx_exact_mass_smem(s, hd);
  LX_REQUIRE(smem <= 212 * 1024, LX_ERR_UNSUPPORTED, "exact attention strip (s=%d, hd=%d) exceeds shared memory", s, hd);
  static cudaError_t attr =
      cudaFuncSetAttribute(exact_mass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 212 * 1024);
  LX_CHECK_CUDA(attr);
  const double scale = 1.0 / sqrt((double)hd);  // sf/exposer.py:52
  launch_k(exact_mass_kernel, dim3(n_b, H, n_items), kExThreads, smem, stream, q, k, ld, s, H, hd, n_b, scale, mass);
  return launch_check("exact_block_mass");
}

int lx_select_by_coverage(const double* mass, int n_items, int H, int n_b, const int32_t* pool_kind,
                          const int32_t* pool_param, int n_pool, double tau, int head_sum, int32_t* pattern_idx,
                          lx_stream_t stream) {
  LX_REQUIRE(n_items >= 1 && H >= 1 && n_b >= 1, LX_ERR_SHAPE, "select_by_coverage: empty shape");
  LX_REQUIRE(n_pool >= 1 && n_pool <= kExMaxPool, LX_ERR_PATTERN, "pool size %d outside [1, %d]", n_pool, kExMaxPool);
  LX_REQUIRE(tau > 0 && tau <= 1, LX_ERR_SHAPE, "coverage tau must be in (0, 1], got %g", tau);
  const int n_sel = head_sum ? n_items : n_items * H;
  const size_t per_warp = sizeof(double) * n_b * n_b;
  const int wpb = (int)std::max<size_t>(1, std::min<size_t>(8, (200u * 1024u) / per_warp));
  static cudaError_t attr =
      cudaFuncSetAttribute(coverage_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  LX_CHECK_CUDA(attr);
  launch_k(coverage_select_kernel, (n_sel + wpb - 1) / wpb, 32 * wpb, per_warp * wpb, stream, mass, n_items, H, n_b, pool_kind, pool_param,
           n_pool, tau, head_sum, pattern_idx);
  return launch_check("select_by_coverage");
}

int lx_block_importance(const float* z, int ldz, int n_items, int s, int n_cols, int blk, float* imp,
                        lx_stream_t stream) {
  LX_REQUIRE(n_items >= 1 && n_cols >= 1 && blk >= 1 && s >= 0, LX_ERR_SHAPE, "block_importance: empty shape");
  LX_REQUIRE(ldz >= n_cols, LX_ERR_SHAPE, "row stride %d < columns %d", ldz, n_cols);
  const int n_blk = (n_cols + blk - 1) / blk;
  LX_CHECK_CUDA(cudaMemsetAsync(imp, 0, sizeof(float) * n_items * n_blk, stream));
  if (s == 0) return 0;
  // enough CTAs to fill the SMs several times over; each column strip reads rows_per_cta rows
  const bool vec = (n_cols % 4) == 0 && (ldz % 4) == 0 && (blk % 4) == 0;
  const int col_ctas = (n_cols / (vec ? 4 : 1) + 255) / 256;
  int row_ctas = max(1, (4 * num_sms()) / max(1, col_ctas * n_items));
  row_ctas = min(row_ctas, (s + 31) / 32);
  const int rpc = (s + row_ctas - 1) / row_ctas;
  launch_k(block_importance_kernel, dim3(col_ctas, (s + rpc - 1) / rpc, n_items), 256, 0, stream, z, ldz, s, n_cols,
           blk, rpc, n_blk, reinterpret_cast<int*>(imp));
  return launch_check("block_importance");
}

int lx_filter_neuron_blocks(const float* imp, int n_items, int n_blk, double theta, uint32_t* bits,
                            lx_stream_t stream) {
  LX_REQUIRE(n_items >= 1 && n_blk >= 1, LX_ERR_SHAPE, "filter_neuron_blocks: empty shape");
  LX_REQUIRE(theta >= 0 && theta <= 1, LX_ERR_SHAPE, "theta must be in [0, 1], got %g", theta);
  launch_k(filter_blocks_kernel, (n_items + 3) / 4, 128, 0, stream, imp, n_items, n_blk, theta, bits);
  return launch_check("filter_neuron_blocks");
}

}  // extern "C"
