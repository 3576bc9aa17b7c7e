// C-ABI: generic tcgen05 GEMM and the neuron-sparse MLP GEMMs (K2).
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "gemm_sm100.cuh"

namespace lx {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("LX_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int make_tmap_bf16_2d(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_stride_elems,
                      uint32_t box_inner, uint32_t box_outer) {
  return make_tmap_bf16_2d_sw(map, ptr, inner, outer, row_stride_elems, box_inner, box_outer, CU_TENSOR_MAP_SWIZZLE_128B);
}

int make_tmap_bf16_2d_sw(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_stride_elems,
                         uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz) {
  auto enc = get_encode();
  LX_REQUIRE(enc != nullptr, LX_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  LX_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0, LX_ERR_SHAPE, "TMA base pointer must be 16B aligned");
  LX_REQUIRE((row_stride_elems * 2) % 16 == 0, LX_ERR_SHAPE, "row stride must be a multiple of 8 bf16 elements");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  LX_REQUIRE(r == CUDA_SUCCESS, LX_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d): inner=%llu outer=%llu box=%u,%u", (int)r,
             (unsigned long long)inner, (unsigned long long)outer, box_inner, box_outer);
  return LX_OK;
}

// CTA pairs (cta_group::2) for the dense / item-packed modes, selectable with lx_gemm_set_cta_pair.
// Default single-CTA: at the MLP shapes (about one tile per CTA) the pair's cluster launch delays the
// first stage by ~1.4k cycles and costs more than its halved B traffic saves (tools/gemm_trace.py).
static int g_cta_pair = 0;

template <int BMODE, int EPI, int BN, int CTAS = 1, int CL = 1>
static int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& args_in, cudaStream_t st) {
  static const int spin = [] { const char* e = getenv("LX_GEMM_SPIN"); return e ? atoi(e) : 0; }();
  GemmArgs args = args_in;
  args.spin = spin;
  auto kern = gemm_sm100_kernel<BMODE, EPI, BN, CTAS, CL>;
  constexpr int smem = GemmSmemFor<BMODE, BN, CTAS>::kTotal;
  constexpr int kCl = CTAS * CL;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  static int grid = 0;  // persistent grid: every CTA (cluster) resident at once
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    grid = num_sms() / kCl * kCl;
    if (attr_err == cudaSuccess && kCl > 2) {
      // clusters of 4 must fit inside a GPC: size the grid by how many the device can hold at once
      cfg.gridDim = dim3(grid);
      int n = 0;
      attr_err = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
      if (attr_err == cudaSuccess && n > 0) grid = std::min(grid, n * kCl);
    }
  });
  LX_CHECK_CUDA(attr_err);
  LX_REQUIRE(args.n_items >= 1 && args.n_items <= kMaxItems, LX_ERR_UNSUPPORTED, "n_items must be in [1, %d]", kMaxItems);
  LX_REQUIRE(args.lora_r >= 0 && args.lora_r <= kMaxR, LX_ERR_UNSUPPORTED, "LoRA rank must be <= %d", kMaxR);
  if (CTAS == 1) {
    launch_k(kern, num_sms(), kGemmThreads, smem, st, ta, tb, args);
    return launch_check("gemm_sm100");
  }
  cfg.gridDim = dim3(grid);
  LX_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, args));
  return launch_check("gemm_sm100 (cta pair)");
}

// N-side packed gathers (fc1, fc2 input-grad): wide CTA-pair tiles (256 rows x up to 512 columns, the width chosen on
// the device so the tiles fit in one round of pairs) unless LX_GEMM_WIDE=0 or a pair mode is forced. Halves the
// L2 -> SM bytes per FLOP of the 128 x 256 single-CTA tile and avoids a second, mostly empty round of tiles.
static bool wide_pairs() {
  static const bool on = [] { const char* e = getenv("LX_GEMM_WIDE"); return !(e && e[0] == '0'); }();
  return on && g_cta_pair == 0;
}
// dense / packed B: pick the CTA-pair engine when enabled (B boxes are then BN/2 rows on the N side)
// tb1: B boxes for 1-CTA 256-wide tiles; tb2: 128-row boxes (pair, BN 256); tb4: 64-row boxes (pair, BN 128)
template <int BMODE, int EPI>
static int launch_gemm_auto(const CUtensorMap& ta, const CUtensorMap& tb1, const CUtensorMap& tb2, const CUtensorMap& tb4,
                            const GemmArgs& args, cudaStream_t st) {
  if (g_cta_pair == 2) return launch_gemm<BMODE, EPI, 128, 2>(ta, tb4, args, st);
  if (g_cta_pair == 1) return launch_gemm<BMODE, EPI, 256, 2>(ta, tb2, args, st);
  if (g_cta_pair == 3) return launch_gemm<BMODE, EPI, 128, 1>(ta, tb2, args, st);  // single CTA, 128 x 128 tiles
  if (g_cta_pair == 4) return launch_gemm<BMODE, EPI, 256, 2, 2>(ta, tb4, args, st);  // two pairs, B multicast
  return launch_gemm<BMODE, EPI, 256, 1>(ta, tb1, args, st);
}

template <int EPI>
static int launch_packed_n(const CUtensorMap& ta, const uint16_t* wp, int n_items, int d, int d_ff, const CUtensorMap& tb,
                           const CUtensorMap& tb2, const CUtensorMap& tb4, const GemmArgs& args, cudaStream_t st) {
  if (wide_pairs()) {
    CUtensorMap tb32;
    int rc = make_tmap_bf16_2d(&tb32, wp, d, (uint64_t)n_items * d_ff, d, kBK, 32);
    if (rc) return rc;
    return launch_gemm<kPackedN, EPI, 512, 2>(ta, tb32, args, st);
  }
  return launch_gemm_auto<kPackedN, EPI>(ta, tb, tb2, tb4, args, st);
}


// float32-faithful predictor GEMMs (hi/lo weight pair, one A read per K stage): 256 x 128 CTA-pair tiles
int gemm_dual_launch(bool mask_epi, const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& args, cudaStream_t st) {
  return mask_epi ? launch_gemm<kDenseDual, kEpiMask, 256, 2>(ta, tb, args, st)
                  : launch_gemm<kDenseDual, kEpiStoreF32, 256, 2>(ta, tb, args, st);
}

// ---- LM head + cross-entropy without fp32 logits (sf/model.py:449-472)
// combine: per row, lse = M + log sum_t z_t 2^((m_t - M) log2 e) over the logits GEMM's segment stats (fixed order:
// lane-strided partial sums, then a butterfly), loss = lse - l_target, and per segment the factor
// c_t = exp(m_t - lse) * inv_s that turns the stored bf16 exp(l - m_t) into the softmax / s. One warp per row.
__global__ void __launch_bounds__(256) ce_combine_kernel(const float2* __restrict__ stats, int nseg, const float* __restrict__ tl,
                                                         int rows, float inv_s, float* __restrict__ row_loss,
                                                         float* __restrict__ coef) {
  pdl_wait_trigger();
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float2* st = stats + (size_t)row * nseg;
  float mx = -INFINITY;
  for (int k = lane; k < nseg; k += 32) mx = fmaxf(mx, st[k].x);
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float z = 0.f;
  for (int k = lane; k < nseg; k += 32) {
    const float2 p = st[k];
    if (p.y > 0.f) z += p.y * __expf(p.x - mx);
  }
  for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  const float lse = mx + __logf(z);
  for (int k = lane; k < nseg; k += 32) {
    const float2 p = st[k];
    coef[(size_t)row * nseg + k] = p.y > 0.f ? __expf(p.x - lse) * inv_s : 0.f;
  }
  if (lane == 0) row_loss[row] = lse - tl[row];
}

// rescale in place: g[r, j] = bf16(float(g[r, j]) * c[r, j / seg] - (j == target[r]) * inv_s), 8 columns per thread
__global__ void __launch_bounds__(256) ce_rescale_kernel(__nv_bfloat16* __restrict__ g, int ldg, int rows, int V,
                                                         const float* __restrict__ coef, int nseg, int seg,
                                                         const int64_t* __restrict__ tgt, float inv_s) {
  pdl_wait_trigger();
  const int v8 = (V + 7) / 8;
  const long long n = (long long)rows * v8;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(e / v8), j0 = (int)(e % v8) * 8;
    const float c = __ldg(coef + (size_t)row * nseg + j0 / seg);
    const long long t = __ldg(tgt + row);
    __nv_bfloat16* p = g + (size_t)row * ldg + j0;
    if (j0 + 8 <= V) {
      uint4 w = *reinterpret_cast<const uint4*>(p);
      uint32_t* u = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float a = __bfloat162float(__ushort_as_bfloat16((unsigned short)(u[k] & 0xffffu))) * c;
        float b = __bfloat162float(__ushort_as_bfloat16((unsigned short)(u[k] >> 16))) * c;
        if (j0 + 2 * k == t) a -= inv_s;
        if (j0 + 2 * k + 1 == t) b -= inv_s;
        u[k] = pack_bf16x2(a, b);
      }
      *reinterpret_cast<uint4*>(p) = w;
    } else {
      for (int k = 0; j0 + k < V; ++k) {
        float a = __bfloat162float(p[k]) * c;
        if (j0 + k == t) a -= inv_s;
        p[k] = __float2bfloat16_rn(a);
      }
    }
  }
}

static GemmArgs base_args(int n_items, int rows, int n_dense, int k_dense) {
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.n_items = n_items;
  a.rows_per_item = rows;
  a.n_dense = n_dense;
  a.k_dense = k_dense;
  a.blk = 16;
  a.lora_scale = 1.f;
  return a;
}

// copy item b's active neuron-block rows (ascending) of one or two [d_ff, d] weights (W1^T and W2 share the ids)
// into packed[b][0 : count*blk]. Persistent: warps walk the flat list of ACTIVE rows (item prefix of the counts in
// shared memory), one warp per packed row, 16-byte loads/stores with four in flight per lane -- no CTA per inactive
// row (at 85% sparsity the old row grid launched ~7x more CTAs than rows to copy).
constexpr int kPackCtasPerSm = 4;
__global__ void __launch_bounds__(256) pack_rows_kernel(const uint4* __restrict__ wa, const uint4* __restrict__ wb, int d16,
                                                        int d_ff, int blk, int n_items, const int32_t* __restrict__ counts,
                                                        const int32_t* __restrict__ ids, uint4* __restrict__ pa,
                                                        uint4* __restrict__ pb) {
  __shared__ int pre[kMaxItems + 1];
  pdl_wait_trigger();
  if (threadIdx.x < 32) {  // warp scan of the active row counts
    int carry = 0;
    for (int b0 = 0; b0 < n_items; b0 += 32) {
      const int b = b0 + (int)threadIdx.x;
      const int v = b < n_items ? __ldg(counts + b) * blk : 0;
      int inc = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if ((int)threadIdx.x >= o) inc += t;
      }
      if (b < n_items) pre[b] = carry + inc - v;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (threadIdx.x == 0) pre[n_items] = carry;
  }
  __syncthreads();
  const int total = pre[n_items], n_w = wb ? 2 : 1;
  const int lane = threadIdx.x & 31;
  for (int f = blockIdx.x * 8 + (threadIdx.x >> 5); f < n_w * total; f += gridDim.x * 8) {
    const int which = f >= total, fr = f - which * total;
    int lo = 0, hi = n_items;  // largest item with pre[item] <= fr
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (pre[mid] <= fr) lo = mid; else hi = mid;
    }
    const int prow = fr - pre[lo];
    const int src = __ldg(ids + (size_t)lo * (d_ff / blk) + prow / blk) * blk + prow % blk;
    const uint4* sp = (which ? wb : wa) + (size_t)src * d16;
    uint4* dp = (which ? pb : pa) + ((size_t)lo * d_ff + prow) * d16;
    for (int i0 = lane; i0 < d16; i0 += 128) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + 32 * u < d16) v[u] = __ldg(sp + i0 + 32 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + 32 * u < d16) dp[i0 + 32 * u] = v[u];
    }
  }
}

static int check_blk(int blk) {
  LX_REQUIRE(blk == 16 || blk == 32 || blk == 64, LX_ERR_UNSUPPORTED,
             "neuron block size %d unsupported on the sm_100a path (16, 32 or 64)", blk);
  return LX_OK;
}

}  // namespace lx

using namespace lx;

extern "C" {

const char* lx_last_error(void) { return g_err; }
int lx_abi_version(void) { return 1; }
int lx_device_sm_count(void) { return num_sms(); }
int lx_debug_set_gemm_trace(unsigned long long* buf) {
  LX_CHECK_CUDA(cudaMemcpyToSymbol(g_gemm_trace, &buf, sizeof(buf)));
  return 0;
}

int lx_gemm_set_cta_pair(int mode) {
  const int prev = g_cta_pair;
  g_cta_pair = (mode >= 1 && mode <= 5) ? mode : 0;
  return prev;
}

int lx_gemm_bf16_tn(const uint16_t* a, int lda, const uint16_t* b, int ldb, void* c, int ldc, int c_is_f32, int M, int N,
                    int K, int a_k_split, lx_stream_t stream) {
  LX_REQUIRE(M > 0 && N > 0 && K > 0, LX_ERR_SHAPE, "gemm: empty shape");
  LX_REQUIRE(a_k_split >= 0 && a_k_split % kBK == 0 && a_k_split < K, LX_ERR_SHAPE,
             "gemm: a_k_split %d must be a multiple of %d below K", a_k_split, kBK);
  CUtensorMap ta, tb;
  int rc;
  // with a K split, A spans K - a_k_split columns (its tail reads zero-filled past them)
  if ((rc = make_tmap_bf16_2d(&ta, a, a_k_split ? K - a_k_split : K, M, lda, kBK, kBM))) return rc;
  CUtensorMap tb2, tb4;
  if ((rc = make_tmap_bf16_2d(&tb, b, K, N, ldb, kBK, 256))) return rc;
  if ((rc = make_tmap_bf16_2d(&tb2, b, K, N, ldb, kBK, 128))) return rc;
  if ((rc = make_tmap_bf16_2d(&tb4, b, K, N, ldb, kBK, 64))) return rc;
  GemmArgs args = base_args(1, M, N, K);
  args.out = c;
  args.ldo = ldc;
  args.a_k_split = a_k_split;
  // under-filled single-CTA problems (e.g. the predictor projection, M = B*m = 184): 128-wide tiles
  const long long tiles256 = (long long)((M + kBM - 1) / kBM) * ((N + 255) / 256);
  if (g_cta_pair == 0 && tiles256 < num_sms())
    return c_is_f32 ? launch_gemm<kDense, kEpiStoreF32, 128, 1>(ta, tb2, args, stream)
                    : launch_gemm<kDense, kEpiStoreBF16, 128, 1>(ta, tb2, args, stream);
  return c_is_f32 ? launch_gemm_auto<kDense, kEpiStoreF32>(ta, tb, tb2, tb4, args, stream)
                  : launch_gemm_auto<kDense, kEpiStoreBF16>(ta, tb, tb2, tb4, args, stream);
}

static int linear_impl(const uint16_t* a, int lda, const uint16_t* b, int ldb, bool b_kn, int M, int N, int K, void* out,
                       int ldo, int out_f32, const float* resid, const float* bias, const float* lora_x,
                       const float* lora_w, long long w_sr, long long w_sc, int r, float scaling, cudaStream_t stream) {
  LX_REQUIRE(M > 0 && N > 0 && K > 0, LX_ERR_SHAPE, "linear: empty shape");
  LX_REQUIRE(!resid || out_f32, LX_ERR_SHAPE, "linear: residual add needs fp32 output");
  CUtensorMap ta, tb;
  int rc;
  if ((rc = make_tmap_bf16_2d(&ta, a, K, M, lda, kBK, kBM))) return rc;
  GemmArgs args = base_args(1, M, N, K);
  args.out = out;
  args.ldo = ldo;
  args.out_f32 = out_f32;
  args.resid = resid;
  args.bias = bias;
  args.lora_x = lora_x;
  args.lora_w = lora_w;
  args.w_sr = w_sr;
  args.w_sc = w_sc;
  args.lora_r = (lora_x && lora_w) ? r : 0;
  args.lora_scale = scaling;
  // engine: wide CTA pairs (256 x 512 tiles, tcgen05 floor in the mainloop) when they fill at least half of the
  // pairs, else single-CTA 128 x 256 tiles (small M: more, shorter tiles); lx_gemm_set_cta_pair forces a variant
  const long long wide_tiles = (long long)((M + 255) / 256) * ((N + 511) / 512);
  const bool wide = g_cta_pair == 5 || (g_cta_pair == 0 && wide_tiles * 4 >= num_sms());
  if (b_kn) {  // B [K, N] row-major: MN-major 64 x 64 atoms
    if ((rc = make_tmap_bf16_2d(&tb, b, N, K, ldb, kBK, 64))) return rc;
    return wide ? launch_gemm<kDenseMN, kEpiFc2, 512, 2>(ta, tb, args, stream)
                : launch_gemm<kDenseMN, kEpiFc2, 256>(ta, tb, args, stream);
  }
  if (wide) {  // 32-row B boxes
    if ((rc = make_tmap_bf16_2d(&tb, b, K, N, ldb, kBK, 32))) return rc;
    return launch_gemm<kDense, kEpiFc2, 512, 2>(ta, tb, args, stream);
  }
  if (g_cta_pair == 1 || g_cta_pair == 4) {  // CTA pairs (B half = 128-row boxes), or two pairs multicasting B
    if ((rc = make_tmap_bf16_2d(&tb, b, K, N, ldb, kBK, g_cta_pair == 4 ? 64 : 128))) return rc;
    return g_cta_pair == 4 ? launch_gemm<kDense, kEpiFc2, 256, 2, 2>(ta, tb, args, stream)
                           : launch_gemm<kDense, kEpiFc2, 256, 2>(ta, tb, args, stream);
  }
  static int forced_bn = [] { const char* e = getenv("LX_LINEAR_BN"); return e ? atoi(e) : 0; }();
  const int bn = forced_bn == 128 ? 128 : 256;
  if ((rc = make_tmap_bf16_2d(&tb, b, K, N, ldb, kBK, bn))) return rc;
  return bn == 128 ? launch_gemm<kDense, kEpiFc2, 128>(ta, tb, args, stream)
                   : launch_gemm<kDense, kEpiFc2, 256>(ta, tb, args, stream);
}

int lx_linear(const uint16_t* a, int lda, const uint16_t* b_t, int ldb, int M, int N, int K, void* out, int ldo,
              int out_f32, const float* resid, const float* bias, const float* lora_x, const float* lora_w,
              long long w_sr, long long w_sc, int r, float scaling, lx_stream_t stream) {
  return linear_impl(a, lda, b_t, ldb, false, M, N, K, out, ldo, out_f32, resid, bias, lora_x, lora_w, w_sr, w_sc, r,
                     scaling, stream);
}

int lx_linear_kn(const uint16_t* a, int lda, const uint16_t* b, int ldb, int M, int N, int K, void* out, int ldo,
                 int out_f32, const float* resid, const float* bias, const float* lora_x, const float* lora_w,
                 long long w_sr, long long w_sc, int r, float scaling, lx_stream_t stream) {
  return linear_impl(a, lda, b, ldb, true, M, N, K, out, ldo, out_f32, resid, bias, lora_x, lora_w, w_sr, w_sc, r,
                     scaling, stream);
}

// B-operand tensor map of an MLP GEMM: gathered blocks of the full weight, or the item-packed copy.
// N side: K-major boxes [64 K x blk rows] (gather) / [64 K x 256 rows] (packed).
// K side: MN-major boxes [64 N x blk rows] (gather) / [64 N x 64 rows] (packed).
static int mlp_tmap_b(CUtensorMap* tb, const uint16_t* w, const uint16_t* wp, int n_items, int d, int d_ff, int blk,
                      bool n_side, int n_rows = 256) {
  if (wp) return make_tmap_bf16_2d(tb, wp, d, (uint64_t)n_items * d_ff, d, kBK, n_side ? n_rows : 64);
  return make_tmap_bf16_2d(tb, w, d, d_ff, d, kBK, blk);
}

int lx_neuron_fc1(const uint16_t* x, int n_items, int s, int d, int d_ff, int blk, const uint16_t* w1_t,
                  const int32_t* counts, const int32_t* ids, const float* b1, const float* ax1, const float* b1_lora,
                  int r, float scaling, int apply_relu, uint16_t* a_out, int ld_h, const uint16_t* w1_packed,
                  uint16_t* relu_bits, lx_stream_t stream) {
  int rc;
  if ((rc = check_blk(blk))) return rc;
  LX_REQUIRE(d_ff % blk == 0, LX_ERR_MASK, "d_ff %d not a multiple of blk %d on the device path", d_ff, blk);
  CUtensorMap ta, tb;
  if ((rc = make_tmap_bf16_2d(&ta, x, d, (uint64_t)n_items * s, d, kBK, kBM))) return rc;
  if ((rc = mlp_tmap_b(&tb, w1_t, w1_packed, n_items, d, d_ff, blk, true))) return rc;
  GemmArgs args = base_args(n_items, s, 0, d);
  LX_REQUIRE(!relu_bits || (apply_relu && ld_h % 16 == 0), LX_ERR_SHAPE,
             "neuron_fc1: relu bits need apply_relu and ld_h %% 16 == 0");
  args.relu_bits = relu_bits;
  args.ld_bits = ld_h / 16;
  args.counts = counts;
  args.ids = ids;
  args.ids_stride = d_ff / blk;
  args.blk = blk;
  args.packed_stride = d_ff;
  args.out = a_out;
  args.ldo = ld_h;
  args.bias = b1;
  args.lora_x = ax1;
  args.lora_w = b1_lora;
  args.w_sr = d_ff;
  args.w_sc = 1;
  args.lora_r = (ax1 && b1_lora) ? r : 0;
  args.lora_scale = scaling;
  if (w1_packed) {
    CUtensorMap tb2, tb4;
    if ((rc = mlp_tmap_b(&tb2, w1_t, w1_packed, n_items, d, d_ff, blk, true, 128))) return rc;
    if ((rc = mlp_tmap_b(&tb4, w1_t, w1_packed, n_items, d, d_ff, blk, true, 64))) return rc;
    return apply_relu ? launch_packed_n<kEpiFc1>(ta, w1_packed, n_items, d, d_ff, tb, tb2, tb4, args, stream)
                      : launch_packed_n<kEpiFc1Raw>(ta, w1_packed, n_items, d, d_ff, tb, tb2, tb4, args, stream);
  }
  return apply_relu ? launch_gemm<kNGather, kEpiFc1, 256>(ta, tb, args, stream)
                    : launch_gemm<kNGather, kEpiFc1Raw, 256>(ta, tb, args, stream);
}

int lx_neuron_fc2(const uint16_t* a, int ld_h, int n_items, int s, int d, int d_ff, int blk, const uint16_t* w2,
                  const int32_t* counts, const int32_t* ids, const float* b2, const float* ax2, const float* b2_lora,
                  int r, float scaling, void* out, int out_f32, const float* resid, const uint16_t* w2_packed,
                  lx_stream_t stream) {
  int rc;
  if ((rc = check_blk(blk))) return rc;
  LX_REQUIRE(d_ff % blk == 0, LX_ERR_MASK, "d_ff %d not a multiple of blk %d on the device path", d_ff, blk);
  LX_REQUIRE(!resid || out_f32, LX_ERR_SHAPE, "fc2: residual add needs fp32 output");
  CUtensorMap ta, tb;
  if ((rc = make_tmap_bf16_2d(&ta, a, d_ff, (uint64_t)n_items * s, ld_h, kBK, kBM))) return rc;
  if ((rc = mlp_tmap_b(&tb, w2, w2_packed, n_items, d, d_ff, blk, false))) return rc;
  GemmArgs args = base_args(n_items, s, d, 0);
  args.counts = counts;
  args.ids = ids;
  args.ids_stride = d_ff / blk;
  args.blk = blk;
  args.packed_stride = d_ff;
  args.out = out;
  args.ldo = d;
  args.bias = b2;
  args.lora_x = ax2;
  args.lora_w = b2_lora;
  args.w_sr = d;
  args.w_sc = 1;
  args.lora_r = (ax2 && b2_lora) ? r : 0;
  args.lora_scale = scaling;
  args.out_f32 = out_f32;
  args.resid = resid;
  if (w2_packed) {
    return launch_gemm_auto<kPackedK, kEpiFc2>(ta, tb, tb, tb, args, stream);
  }
  return launch_gemm<kKGather, kEpiFc2, 256>(ta, tb, args, stream);
}

int lx_neuron_fc2_dgrad(const uint16_t* d_out, int n_items, int s, int d, int d_ff, int blk, const uint16_t* w2,
                        const int32_t* counts, const int32_t* ids, const float* dax2, const float* a2_lora, int r,
                        const uint16_t* a, uint16_t* dz, int ld_h, const uint16_t* w2_packed, const uint16_t* relu_bits,
                        lx_stream_t stream) {
  int rc;
  if ((rc = check_blk(blk))) return rc;
  CUtensorMap ta, tb;
  if ((rc = make_tmap_bf16_2d(&ta, d_out, d, (uint64_t)n_items * s, d, kBK, kBM))) return rc;
  if ((rc = mlp_tmap_b(&tb, w2, w2_packed, n_items, d, d_ff, blk, true))) return rc;
  GemmArgs args = base_args(n_items, s, 0, d);
  args.counts = counts;
  args.ids = ids;
  args.ids_stride = d_ff / blk;
  args.blk = blk;
  args.packed_stride = d_ff;
  args.out = dz;
  args.ldo = ld_h;
  args.lora_x = dax2;
  args.lora_w = a2_lora;
  args.w_sr = 1;
  args.w_sc = r;
  args.lora_r = (dax2 && a2_lora) ? r : 0;
  args.act = reinterpret_cast<const __nv_bfloat16*>(a);
  args.ld_act = ld_h;
  LX_REQUIRE(!relu_bits || ld_h % 16 == 0, LX_ERR_SHAPE, "neuron_fc2_dgrad: relu bits need ld_h %% 16 == 0");
  args.relu_bits = const_cast<uint16_t*>(relu_bits);
  args.ld_bits = ld_h / 16;
  if (w2_packed) {
    CUtensorMap tb2, tb4;
    if ((rc = mlp_tmap_b(&tb2, w2, w2_packed, n_items, d, d_ff, blk, true, 128))) return rc;
    if ((rc = mlp_tmap_b(&tb4, w2, w2_packed, n_items, d, d_ff, blk, true, 64))) return rc;
    return launch_packed_n<kEpiDa>(ta, w2_packed, n_items, d, d_ff, tb, tb2, tb4, args, stream);
  }
  return launch_gemm<kNGather, kEpiDa, 256>(ta, tb, args, stream);
}

int lx_neuron_fc1_dgrad(const uint16_t* dz, int ld_h, int n_items, int s, int d, int d_ff, int blk,
                        const uint16_t* w1_t, const int32_t* counts, const int32_t* ids, const float* dax1,
                        const float* a1_lora, int r, void* dx, int out_f32, const uint16_t* w1_packed,
                        lx_stream_t stream) {
  int rc;
  if ((rc = check_blk(blk))) return rc;
  CUtensorMap ta, tb;
  if ((rc = make_tmap_bf16_2d(&ta, dz, d_ff, (uint64_t)n_items * s, ld_h, kBK, kBM))) return rc;
  if ((rc = mlp_tmap_b(&tb, w1_t, w1_packed, n_items, d, d_ff, blk, false))) return rc;
  GemmArgs args = base_args(n_items, s, d, 0);
  args.counts = counts;
  args.ids = ids;
  args.ids_stride = d_ff / blk;
  args.blk = blk;
  args.packed_stride = d_ff;
  args.out = dx;
  args.ldo = d;
  args.lora_x = dax1;
  args.lora_w = a1_lora;
  args.w_sr = 1;
  args.w_sc = r;
  args.lora_r = (dax1 && a1_lora) ? r : 0;
  args.out_f32 = out_f32;
  if (w1_packed) {
    return launch_gemm_auto<kPackedK, kEpiDx>(ta, tb, tb, tb, args, stream);
  }
  return launch_gemm<kKGather, kEpiDx, 256>(ta, tb, args, stream);
}

int lx_pack_active_rows(const uint16_t* w, int d_ff, int d, int blk, int n_items, const int32_t* counts,
                        const int32_t* ids, uint16_t* packed, lx_stream_t stream) {
  return lx_pack_active_rows2(w, nullptr, d_ff, d, blk, n_items, counts, ids, packed, nullptr, stream);
}

int lx_lm_head_ce_nseg(int V) { return 2 * ((V + 511) / 512); }  // two 256-column halves per 512-wide tile

int lx_lm_head_ce(const uint16_t* hf, int ld_hf, int rows, int d, const uint16_t* emb, int V, const int64_t* targets,
                  float inv_s, uint16_t* g, int ldg, float* stats_ws, float* coef_ws, float* tl_ws, float* row_loss,
                  lx_stream_t stream) {
  LX_REQUIRE(rows >= 1 && d >= 1 && V >= 1, LX_ERR_SHAPE, "lm_head_ce: empty shape");
  LX_REQUIRE(ldg >= V && ldg % 8 == 0 && (reinterpret_cast<uintptr_t>(g) & 15) == 0, LX_ERR_SHAPE,
             "lm_head_ce: gradient rows need ldg >= V, a multiple of 8, 16-byte aligned");
  CUtensorMap ta, tb;
  int rc;
  if ((rc = make_tmap_bf16_2d(&ta, hf, d, rows, ld_hf, kBK, kBM))) return rc;
  if ((rc = make_tmap_bf16_2d(&tb, emb, d, V, d, kBK, 32))) return rc;  // wide pair tiles: 32-row B boxes
  const int nseg = lx_lm_head_ce_nseg(V);
  GemmArgs args = base_args(1, rows, V, d);
  args.out = g;
  args.ldo = ldg;
  args.ce_tgt = targets;
  args.ce_stats = reinterpret_cast<float2*>(stats_ws);
  args.ce_tl = tl_ws;
  args.ce_nseg = nseg;
  if ((rc = launch_gemm<kDense, kEpiCe, 512, 2>(ta, tb, args, stream))) return rc;
  launch_k(ce_combine_kernel, (rows + 7) / 8, 256, 0, stream, reinterpret_cast<const float2*>(stats_ws), nseg,
           (const float*)tl_ws, rows, inv_s, row_loss, coef_ws);
  if ((rc = launch_check("ce_combine"))) return rc;
  launch_k(ce_rescale_kernel, 8 * num_sms(), 256, 0, stream, reinterpret_cast<__nv_bfloat16*>(g), ldg, rows, V,
           (const float*)coef_ws, nseg, 256, targets, inv_s);
  return launch_check("ce_rescale");
}

int lx_pack_active_rows2(const uint16_t* w_a, const uint16_t* w_b, int d_ff, int d, int blk, int n_items,
                         const int32_t* counts, const int32_t* ids, uint16_t* packed_a, uint16_t* packed_b,
                         lx_stream_t stream) {
  LX_REQUIRE(d % 8 == 0 && d_ff % blk == 0, LX_ERR_SHAPE, "pack_active_rows: d %% 8 and d_ff %% blk required");
  LX_REQUIRE(n_items >= 1 && n_items <= kMaxItems, LX_ERR_UNSUPPORTED, "pack_active_rows: n_items must be in [1, %d]",
             kMaxItems);
  LX_REQUIRE(!w_b == !packed_b, LX_ERR_SHAPE, "pack_active_rows: second weight and its pack go together");
  const int rows_max = n_items * d_ff * (w_b ? 2 : 1);
  const int grid = std::min((rows_max + 7) / 8, kPackCtasPerSm * num_sms());
  launch_k(pack_rows_kernel, grid, 256, 0, stream, reinterpret_cast<const uint4*>(w_a), reinterpret_cast<const uint4*>(w_b),
           d / 8, d_ff, blk, n_items, counts, ids, reinterpret_cast<uint4*>(packed_a), reinterpret_cast<uint4*>(packed_b));
  return launch_check("pack_active_rows");
}

}  // extern "C"
