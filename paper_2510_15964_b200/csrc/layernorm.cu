// LayerNorm forward/backward (sf/model.py:307-312, sf/autograd.py:61-66).
// Forward reads the fp32 residual row once into registers, writes bf16 for the
// GEMMs, and — fused — the predictor's sqrt(s)-downsampled rows
// (sf/predictor.py:62-71), so the attention predictor never re-reads h1.
#include "common.cuh"
#include "ptx.cuh"

namespace lx {

constexpr int kLnThreads = 256;
constexpr int kLnMaxVec = 8;  // float4 per thread -> d <= 256*4*8 = 8192

__device__ __forceinline__ float block_sum(float v, float* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float t = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
  return t;
}

// VEC = float4 per thread, ceil(d / 4 / 256): registers (and so resident CTAs) sized to the row, not to the max d
template <int VEC>
__global__ void __launch_bounds__(kLnThreads) ln_fwd_kernel(const float* __restrict__ x, int d, const float* __restrict__ g,
                                                             const float* __restrict__ b, float eps,
                                                             __nv_bfloat16* __restrict__ y, int ldy, float* __restrict__ mean_out,
                                                             float* __restrict__ istd_out, int s, int m_small,
                                                             __nv_bfloat16* __restrict__ x_small,
                                                             const __nv_bfloat16* __restrict__ delta,
                                                             float* __restrict__ resid_out) {
  pdl_wait_trigger();
  __shared__ float red[32];
  const size_t row = blockIdx.x;
  const float4* xr = reinterpret_cast<const float4*>(x + row * d);
  const int nv = d / 4;
  float4 v[VEC];
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    int c = threadIdx.x + i * kLnThreads;
    v[i] = c < nv ? xr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    if (delta && c < nv) {  // fused residual add: y = x + delta (sf/model.py:420, 427), y kept in fp32
      const uint2 p = reinterpret_cast<const uint2*>(delta + row * d)[c];
      v[i].x += bf16_bits_to_float(p.x & 0xffff);
      v[i].y += bf16_bits_to_float(p.x >> 16);
      v[i].z += bf16_bits_to_float(p.y & 0xffff);
      v[i].w += bf16_bits_to_float(p.y >> 16);
      reinterpret_cast<float4*>(resid_out + row * d)[c] = v[i];
    }
    sum += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  }
  const float mu = block_sum(sum, red) / d;
  float sq = 0.f;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    int c = threadIdx.x + i * kLnThreads;
    if (c < nv) {
      float a = v[i].x - mu, bb = v[i].y - mu, cc = v[i].z - mu, dd = v[i].w - mu;
      sq += (a * a + bb * bb) + (cc * cc + dd * dd);
    }
  }
  const float var = block_sum(sq, red) / d;
  const float istd = 1.0f / sqrtf(var + eps);
  if (threadIdx.x == 0) {
    mean_out[row] = mu;
    istd_out[row] = istd;
  }
  // fused downsample: token t of its sequence is sampled iff t == (i*s)//m for some i
  __nv_bfloat16* xs_row = nullptr;
  if (x_small) {
    int t = row % s, item = row / s;
    int i = (int)(((long long)t * m_small + s - 1) / s);
    if (i < m_small && (int)(((long long)i * s) / m_small) == t) xs_row = x_small + ((size_t)item * m_small + i) * d;
  }
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const float4* b4 = reinterpret_cast<const float4*>(b);
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    int c = threadIdx.x + i * kLnThreads;
    if (c < nv) {
      float4 gg = g4[c], bb = b4[c];
      float o0 = (v[i].x - mu) * istd * gg.x + bb.x;
      float o1 = (v[i].y - mu) * istd * gg.y + bb.y;
      float o2 = (v[i].z - mu) * istd * gg.z + bb.z;
      float o3 = (v[i].w - mu) * istd * gg.w + bb.w;
      uint2 pk = make_uint2(pack_bf16x2(o0, o1), pack_bf16x2(o2, o3));
      *reinterpret_cast<uint2*>(y + row * ldy + 4 * c) = pk;
      if (xs_row) *reinterpret_cast<uint2*>(xs_row + 4 * c) = pk;
    }
  }
}

template <bool kF32, int VEC>
__global__ void __launch_bounds__(kLnThreads) ln_bwd_kernel(const void* __restrict__ dy_, const float* __restrict__ x,
                                                             const float* __restrict__ g, const float* __restrict__ mean,
                                                             const float* __restrict__ istd, int d,
                                                             float* __restrict__ dx, __nv_bfloat16* __restrict__ dx_bf16) {
  pdl_wait_trigger();
  __shared__ float red[32];
  const size_t row = blockIdx.x;
  const float mu = mean[row], is = istd[row];
  const int nv = d / 4;
  float4 gv[VEC], xh[VEC], cur[VEC];
  float4* o = reinterpret_cast<float4*>(dx + row * d);
  // the accumulator row is loaded with the inputs (one DRAM round trip per row, not two around the block sums)
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = threadIdx.x + i * kLnThreads;
    cur[i] = c < nv ? o[c] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    int c = threadIdx.x + i * kLnThreads;
    gv[i] = xh[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c < nv) {
      float4 dy;
      if (kF32) {
        dy = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(dy_) + row * d)[c];
      } else {
        uint2 p = reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(dy_) + row * d)[c];
        dy.x = bf16_bits_to_float(p.x & 0xffff);
        dy.y = bf16_bits_to_float(p.x >> 16);
        dy.z = bf16_bits_to_float(p.y & 0xffff);
        dy.w = bf16_bits_to_float(p.y >> 16);
      }
      float4 xx = reinterpret_cast<const float4*>(x + row * d)[c];
      float4 gg = reinterpret_cast<const float4*>(g)[c];
      gv[i] = make_float4(dy.x * gg.x, dy.y * gg.y, dy.z * gg.z, dy.w * gg.w);
      xh[i] = make_float4((xx.x - mu) * is, (xx.y - mu) * is, (xx.z - mu) * is, (xx.w - mu) * is);
      s1 += (gv[i].x + gv[i].y) + (gv[i].z + gv[i].w);
      s2 += (gv[i].x * xh[i].x + gv[i].y * xh[i].y) + (gv[i].z * xh[i].z + gv[i].w * xh[i].w);
    }
  }
  const float mg = block_sum(s1, red) / d;
  const float mgx = block_sum(s2, red) / d;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    int c = threadIdx.x + i * kLnThreads;
    if (c < nv) {
      cur[i].x += is * (gv[i].x - mg - xh[i].x * mgx);
      cur[i].y += is * (gv[i].y - mg - xh[i].y * mgx);
      cur[i].z += is * (gv[i].z - mg - xh[i].z * mgx);
      cur[i].w += is * (gv[i].w - mg - xh[i].w * mgx);
      o[c] = cur[i];
      if (dx_bf16)  // bf16 copy of the updated residual gradient: the next GEMMs' operand
        *reinterpret_cast<uint2*>(dx_bf16 + row * d + 4 * c) =
            make_uint2(pack_bf16x2(cur[i].x, cur[i].y), pack_bf16x2(cur[i].z, cur[i].w));
    }
  }
}

// ---------------------------------------------------------------- warp-per-row variants (d <= 2048)
// One warp owns a row: lane l holds float4 chunks l, l+32, ... (VEC of them) in registers, both
// reductions are warp shuffles (no block barriers), and 8 rows per CTA keep ~64-160 KB in flight per SM.
LX_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Row sum over the TPR threads that own a row. TPR 64 (d = 2048: 8 float4 per lane instead of 16, so ~60 instead of
// ~120 registers and twice the rows in flight per SM): the two warps' partial sums meet in shared memory behind a
// 64-thread named barrier (id 1 + row slot), added in warp order (deterministic). k selects the slot pair of the
// first / second reduction of a row, so a partner still reading slot k of this row never races the next write.
template <int TPR>
LX_DEV float row_sum(float v, float* red, int k) {
  v = warp_sum(v);
  if (TPR == 32) return v;
  constexpr int W = TPR / 32;  // warps per row
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[k * 8 + warp] = v;
  asm volatile("bar.sync %0, %1;" ::"r"(1 + warp / W), "n"(TPR) : "memory");
  const int w0 = warp & ~(W - 1);
  float t = red[k * 8 + w0];
#pragma unroll
  for (int j = 1; j < W; ++j) t += red[k * 8 + w0 + j];
  return t;
}

template <int VEC, int TPR>
__global__ void __launch_bounds__(256) ln_fwd_warp_kernel(const float* __restrict__ x, int M, int d,
                                                          const float* __restrict__ g, const float* __restrict__ b,
                                                          float eps, __nv_bfloat16* __restrict__ y, int ldy,
                                                          float* __restrict__ mean_out, float* __restrict__ istd_out, int s,
                                                          int m_small, __nv_bfloat16* __restrict__ x_small,
                                                          const __nv_bfloat16* __restrict__ delta,
                                                          float* __restrict__ resid_out) {
  pdl_wait_trigger();
  constexpr int RPC = 256 / TPR;  // rows per CTA pass
  __shared__ float red[16];
  const int lane = threadIdx.x % TPR;
  const int nv = d / 4;
#pragma unroll 1
  for (int row = blockIdx.x * RPC + (int)threadIdx.x / TPR; row < M; row += gridDim.x * RPC) {
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)row * d);
  const uint2* dr = delta ? reinterpret_cast<const uint2*>(delta + (size_t)row * d) : nullptr;
  float4 v[VEC];
  uint2 dv[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = lane + TPR * i;
    v[i] = c < nv ? __ldg(xr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    dv[i] = (dr && c < nv) ? __ldg(dr + c) : make_uint2(0u, 0u);
  }
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = lane + TPR * i;
    if (dr && c < nv) {  // fused residual add: y = x + delta (sf/model.py:420, 427), y kept in fp32
      v[i].x += bf16_bits_to_float(dv[i].x & 0xffff);
      v[i].y += bf16_bits_to_float(dv[i].x >> 16);
      v[i].z += bf16_bits_to_float(dv[i].y & 0xffff);
      v[i].w += bf16_bits_to_float(dv[i].y >> 16);
      reinterpret_cast<float4*>(resid_out + (size_t)row * d)[c] = v[i];
    }
    sum += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  }
  const float mu = row_sum<TPR>(sum, red, 0) / d;
  float sq = 0.f;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = lane + TPR * i;
    if (c < nv) {
      const float a = v[i].x - mu, bb = v[i].y - mu, cc = v[i].z - mu, dd = v[i].w - mu;
      sq += (a * a + bb * bb) + (cc * cc + dd * dd);
    }
  }
  const float istd = 1.0f / sqrtf(row_sum<TPR>(sq, red, 1) / d + eps);
  if (lane == 0) {
    mean_out[row] = mu;
    istd_out[row] = istd;
  }
  __nv_bfloat16* xs_row = nullptr;  // fused downsample: token t is sampled iff t == (i*s)//m for some i
  if (x_small) {
    const int t = row % s, item = row / s;
    const int i = (int)(((long long)t * m_small + s - 1) / s);
    if (i < m_small && (int)(((long long)i * s) / m_small) == t) xs_row = x_small + ((size_t)item * m_small + i) * d;
  }
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const float4* b4 = reinterpret_cast<const float4*>(b);
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = lane + TPR * i;
    if (c < nv) {
      const float4 gg = __ldg(g4 + c), bb = __ldg(b4 + c);
      const uint2 pk = make_uint2(pack_bf16x2((v[i].x - mu) * istd * gg.x + bb.x, (v[i].y - mu) * istd * gg.y + bb.y),
                                  pack_bf16x2((v[i].z - mu) * istd * gg.z + bb.z, (v[i].w - mu) * istd * gg.w + bb.w));
      *reinterpret_cast<uint2*>(y + (size_t)row * ldy + 4 * c) = pk;
      if (xs_row) *reinterpret_cast<uint2*>(xs_row + 4 * c) = pk;
    }
  }
  }
}

template <bool kF32, int VEC, int TPR>
__global__ void __launch_bounds__(256) ln_bwd_warp_kernel(const void* __restrict__ dy_, const float* __restrict__ x,
                                                          const float* __restrict__ g, const float* __restrict__ mean,
                                                          const float* __restrict__ istd, int M, int d,
                                                          float* __restrict__ dx, __nv_bfloat16* __restrict__ dx_bf16) {
  pdl_wait_trigger();
  constexpr int RPC = 256 / TPR;
  __shared__ float red[16];
  const int lane = threadIdx.x % TPR;
  const int nv = d / 4;
#pragma unroll 1
  for (int row = blockIdx.x * RPC + (int)threadIdx.x / TPR; row < M; row += gridDim.x * RPC) {
  const float mu = __ldg(mean + row), is = __ldg(istd + row);
  float4* o = reinterpret_cast<float4*>(dx + (size_t)row * d);
  float4 cur[VEC];  // the accumulator row is loaded with the inputs: one round trip per row
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = lane + TPR * i;
    cur[i] = c < nv ? o[c] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float4 gv[VEC], xh[VEC];
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = lane + TPR * i;
    float4 dy = make_float4(0.f, 0.f, 0.f, 0.f), xx = dy, gg = dy;
    if (c < nv) {
      if (kF32) {
        dy = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(dy_) + (size_t)row * d) + c);
      } else {
        const uint2 p = __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(dy_) + (size_t)row * d) + c);
        dy = make_float4(bf16_bits_to_float(p.x & 0xffff), bf16_bits_to_float(p.x >> 16), bf16_bits_to_float(p.y & 0xffff),
                         bf16_bits_to_float(p.y >> 16));
      }
      xx = __ldg(reinterpret_cast<const float4*>(x + (size_t)row * d) + c);
      gg = __ldg(reinterpret_cast<const float4*>(g) + c);
    }
    gv[i] = make_float4(dy.x * gg.x, dy.y * gg.y, dy.z * gg.z, dy.w * gg.w);
    xh[i] = c < nv ? make_float4((xx.x - mu) * is, (xx.y - mu) * is, (xx.z - mu) * is, (xx.w - mu) * is)
                   : make_float4(0.f, 0.f, 0.f, 0.f);
    s1 += (gv[i].x + gv[i].y) + (gv[i].z + gv[i].w);
    s2 += (gv[i].x * xh[i].x + gv[i].y * xh[i].y) + (gv[i].z * xh[i].z + gv[i].w * xh[i].w);
  }
  const float mg = row_sum<TPR>(s1, red, 0) / d, mgx = row_sum<TPR>(s2, red, 1) / d;
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const int c = lane + TPR * i;
    if (c < nv) {
      cur[i].x += is * (gv[i].x - mg - xh[i].x * mgx);
      cur[i].y += is * (gv[i].y - mg - xh[i].y * mgx);
      cur[i].z += is * (gv[i].z - mg - xh[i].z * mgx);
      cur[i].w += is * (gv[i].w - mg - xh[i].w * mgx);
      o[c] = cur[i];
      if (dx_bf16)  // bf16 copy of the updated residual gradient: the next GEMMs' operand
        *reinterpret_cast<uint2*>(dx_bf16 + (size_t)row * d + 4 * c) =
            make_uint2(pack_bf16x2(cur[i].x, cur[i].y), pack_bf16x2(cur[i].z, cur[i].w));
    }
  }
  }
}

// persistent grid for the warp-per-row kernels: as many 8-row CTAs as fit at once (no partial last wave)
template <typename K>
static int ln_grid(K kern, int M, int rows_per_cta = 8) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0) != cudaSuccess || per_sm < 1) per_sm = 1;
  const int ctas = (M + rows_per_cta - 1) / rows_per_cta;
  return ctas < per_sm * num_sms() ? ctas : per_sm * num_sms();
}

// threads per row at d = 2048 (LX_LN_TPR = 64 / 128 / 256 for measurements; default 128: four warps per row,
// 4 float4 per lane; measured per launch: fwd 21.9 / 18.5 / 16.7 us and bwd 24.1 / 20.8 / 18.8 us at 32 / 64 / 128)
static int ln_tpr() {
  static const int t = [] { const char* e = getenv("LX_LN_TPR"); return e ? atoi(e) : 128; }();
  return t;
}

// LX_LN_BLOCK=1: the one-CTA-per-row block kernels for 2048 < d <= 4096 as well (measurements)
static bool ln_block() {
  static const bool b = [] { const char* e = getenv("LX_LN_BLOCK"); return e && e[0] == '1'; }();
  return b;
}

template <int VEC, int TPR = 32>
static void ln_fwd_warp(const float* x, const uint16_t* delta, float* resid_out, int M, int d, const float* gamma,
                        const float* beta, float eps, uint16_t* y, int ldy, float* mean, float* inv_std, int s, int m_small,
                        uint16_t* x_small, cudaStream_t st) {
  auto kern = ln_fwd_warp_kernel<VEC, TPR>;
  launch_k(kern, ln_grid(kern, M, 256 / TPR), 256, 0, st, x, M, d, gamma, beta, eps, reinterpret_cast<__nv_bfloat16*>(y), ldy, mean,
                                                       inv_std, s > 0 ? s : 1, m_small,
                                                       reinterpret_cast<__nv_bfloat16*>(x_small),
                                                       reinterpret_cast<const __nv_bfloat16*>(delta), resid_out);
}

template <int VEC, int TPR = 32>
static void ln_bwd_warp(const void* dy, int dy_is_f32, const float* x, const float* gamma, const float* mean,
                        const float* inv_std, int M, int d, float* dx, __nv_bfloat16* ob, cudaStream_t st) {
  auto kern = dy_is_f32 ? ln_bwd_warp_kernel<true, VEC, TPR> : ln_bwd_warp_kernel<false, VEC, TPR>;
  launch_k(kern, ln_grid(kern, M, 256 / TPR), 256, 0, st, dy, x, gamma, mean, inv_std, M, d, dx, ob);
}

}  // namespace lx

using namespace lx;

extern "C" {

int lx_layernorm_fwd(const float* x, const uint16_t* delta, float* resid_out, int M, int d, const float* gamma,
                     const float* beta, float eps, uint16_t* y, int ldy, float* mean, float* inv_std, int s, int m_small,
                     uint16_t* x_small, lx_stream_t stream) {
  LX_REQUIRE(d % 4 == 0 && d <= kLnThreads * 4 * kLnMaxVec, LX_ERR_UNSUPPORTED, "layernorm: d=%d unsupported", d);
  LX_REQUIRE(M >= 1, LX_ERR_SHAPE, "layernorm: empty input");
  LX_REQUIRE(!delta || resid_out, LX_ERR_SHAPE, "layernorm: residual add needs resid_out");
  if (x_small) LX_REQUIRE(s >= 1 && m_small >= 1 && M % s == 0, LX_ERR_SHAPE, "layernorm: bad downsample shape");
  LX_REQUIRE(ldy >= d && ldy % 4 == 0, LX_ERR_SHAPE, "layernorm: output row stride %d < d or not a multiple of 4", ldy);
  const int per_lane = (d / 4 + 31) / 32;  // float4 chunks per lane in the warp-per-row kernel
  if (per_lane <= 16) {
    if (per_lane <= 4) ln_fwd_warp<4>(x, delta, resid_out, M, d, gamma, beta, eps, y, ldy, mean, inv_std, s, m_small, x_small, stream);
    else if (per_lane <= 8) ln_fwd_warp<8>(x, delta, resid_out, M, d, gamma, beta, eps, y, ldy, mean, inv_std, s, m_small, x_small, stream);
    else if (ln_tpr() == 64) ln_fwd_warp<8, 64>(x, delta, resid_out, M, d, gamma, beta, eps, y, ldy, mean, inv_std, s, m_small, x_small, stream);
    else if (ln_tpr() == 256) ln_fwd_warp<2, 256>(x, delta, resid_out, M, d, gamma, beta, eps, y, ldy, mean, inv_std, s, m_small, x_small, stream);
    else ln_fwd_warp<4, 128>(x, delta, resid_out, M, d, gamma, beta, eps, y, ldy, mean, inv_std, s, m_small, x_small, stream);
    return launch_check("layernorm_fwd");
  }
  if (d <= 4096 && !ln_block()) {  // cfg4: four warps per row, 8 float4 per lane
    ln_fwd_warp<8, 128>(x, delta, resid_out, M, d, gamma, beta, eps, y, ldy, mean, inv_std, s, m_small, x_small, stream);
    return launch_check("layernorm_fwd");
  }
  const int vec = (d / 4 + kLnThreads - 1) / kLnThreads;  // block kernel: float4 per thread
  auto kf = vec <= 4 ? ln_fwd_kernel<4> : vec <= 6 ? ln_fwd_kernel<6> : ln_fwd_kernel<8>;
  launch_k(kf, M, kLnThreads, 0, stream, x, d, gamma, beta, eps, reinterpret_cast<__nv_bfloat16*>(y), ldy, mean, inv_std,
           s > 0 ? s : 1, m_small, reinterpret_cast<__nv_bfloat16*>(x_small), reinterpret_cast<const __nv_bfloat16*>(delta),
           resid_out);
  return launch_check("layernorm_fwd");
}

int lx_layernorm_bwd(const void* dy, int dy_is_f32, const float* x, const float* gamma, const float* mean,
                     const float* inv_std, int M, int d, float* dx_accum, uint16_t* dx_bf16, lx_stream_t stream) {
  LX_REQUIRE(d % 4 == 0 && d <= kLnThreads * 4 * kLnMaxVec, LX_ERR_UNSUPPORTED, "layernorm: d=%d unsupported", d);
  auto* ob = reinterpret_cast<__nv_bfloat16*>(dx_bf16);
  const int per_lane = (d / 4 + 31) / 32;
  if (per_lane <= 16) {
    if (per_lane <= 4) ln_bwd_warp<4>(dy, dy_is_f32, x, gamma, mean, inv_std, M, d, dx_accum, ob, stream);
    else if (per_lane <= 8) ln_bwd_warp<8>(dy, dy_is_f32, x, gamma, mean, inv_std, M, d, dx_accum, ob, stream);
    else if (ln_tpr() == 64) ln_bwd_warp<8, 64>(dy, dy_is_f32, x, gamma, mean, inv_std, M, d, dx_accum, ob, stream);
    else if (ln_tpr() == 256) ln_bwd_warp<2, 256>(dy, dy_is_f32, x, gamma, mean, inv_std, M, d, dx_accum, ob, stream);
    else ln_bwd_warp<4, 128>(dy, dy_is_f32, x, gamma, mean, inv_std, M, d, dx_accum, ob, stream);
    return launch_check("layernorm_bwd");
  }
  if (d <= 4096 && !ln_block()) {
    ln_bwd_warp<8, 128>(dy, dy_is_f32, x, gamma, mean, inv_std, M, d, dx_accum, ob, stream);
    return launch_check("layernorm_bwd");
  }
  const int vec = (d / 4 + kLnThreads - 1) / kLnThreads;
  auto kb = dy_is_f32 ? (vec <= 4 ? ln_bwd_kernel<true, 4> : vec <= 6 ? ln_bwd_kernel<true, 6> : ln_bwd_kernel<true, 8>)
                      : (vec <= 4 ? ln_bwd_kernel<false, 4> : vec <= 6 ? ln_bwd_kernel<false, 6> : ln_bwd_kernel<false, 8>);
  launch_k(kb, M, kLnThreads, 0, stream, dy, x, gamma, mean, inv_std, d, dx_accum, ob);
  return launch_check("layernorm_bwd");
}

}  // extern "C"
