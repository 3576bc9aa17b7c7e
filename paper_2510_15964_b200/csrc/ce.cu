// Tied-unembedding cross-entropy forward + backward in one pass pair per row
// (sf/model.py:454-472): loss_row = logsumexp(l) - l[target];
// grad = (softmax(l) - onehot(target)) * inv_s, written bf16 for the d_hf GEMM.
// A CTA per row at a time: an online (max, sum-exp) sweep, then a write sweep.
#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"

namespace lx {

__device__ __forceinline__ void online_merge(float& m, float& sum, float m2, float s2) {
  const float mn = fmaxf(m, m2);
  sum = (m == -INFINITY ? 0.f : sum * __expf(m - mn)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mn));
  m = mn;
}

// Persistent rows: up to kCeCtasPerSm CTAs per SM loop over the rows. Both sweeps issue kCeU float4
// loads per thread before using them (the write sweep was L2-latency bound with one load in flight),
// merged in the same order as a one-at-a-time loop, so the per-thread (max, sum) sequence is unchanged.
// Measured (tools/ce_probe.py, 1024 x 50272 logits): 2 CTAs/SM 105 us, 4 89 us, 8 85 us. Fewer live
// rows (L2-resident second sweep) lose to fewer loads in flight, so the default keeps one row per CTA
// for a 1024-row chunk.
constexpr int kCeThreads = 256, kCeU = 8, kCeCtasPerSm = 8;

__global__ void __launch_bounds__(kCeThreads) ce_kernel(const float* __restrict__ logits, int rows, int V,
                                                        const int64_t* __restrict__ tgt, float inv_s,
                                                        float* __restrict__ row_loss, __nv_bfloat16* __restrict__ grad) {
  pdl_wait_trigger();
  __shared__ float sm[kCeThreads / 32], ss[kCeThreads / 32], s_lse;
  const int nv = V / 4;
#pragma unroll 1
  for (int row_i = blockIdx.x; row_i < rows; row_i += gridDim.x) {
    const size_t row = row_i;
    const float4* l4 = reinterpret_cast<const float4*>(logits + row * V);
    float m = -INFINITY, sum = 0.f;
#pragma unroll 1
    for (int i0 = threadIdx.x; i0 < nv; i0 += kCeThreads * kCeU) {
      float4 x[kCeU];
#pragma unroll
      for (int u = 0; u < kCeU; ++u) {
        const int i = i0 + u * kCeThreads;
        x[u] = i < nv ? __ldcg(l4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kCeU; ++u) {
        if (i0 + u * kCeThreads < nv) {
          const float mx = fmaxf(fmaxf(x[u].x, x[u].y), fmaxf(x[u].z, x[u].w));
          const float s2 = __expf(x[u].x - mx) + __expf(x[u].y - mx) + __expf(x[u].z - mx) + __expf(x[u].w - mx);
          online_merge(m, sum, mx, s2);
        }
      }
    }
    for (int i = nv * 4 + threadIdx.x; i < V; i += kCeThreads) online_merge(m, sum, logits[row * V + i], 1.f);
    for (int o = 16; o; o >>= 1) {
      float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, sum, o);
      online_merge(m, sum, m2, s2);
    }
    if ((threadIdx.x & 31) == 0) { sm[threadIdx.x >> 5] = m; ss[threadIdx.x >> 5] = sum; }
    __syncthreads();
    if (threadIdx.x == 0) {
      float M = sm[0], S = ss[0];
      for (int w = 1; w < kCeThreads / 32; ++w) online_merge(M, S, sm[w], ss[w]);
      s_lse = M + logf(S);
      row_loss[row] = s_lse - logits[row * V + tgt[row]];
    }
    __syncthreads();
    const float lse = s_lse;
    const int64_t t = tgt[row];
    __nv_bfloat16* g = grad + row * V;
#pragma unroll 1
    for (int i0 = threadIdx.x; i0 < nv; i0 += kCeThreads * kCeU) {
      float4 x[kCeU];  // all loads of the round in flight before any store (L2 round trips overlap)
#pragma unroll
      for (int u = 0; u < kCeU; ++u) {
        const int i = i0 + u * kCeThreads;
        x[u] = i < nv ? __ldcs(l4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);  // last use of the logits: evict-first
      }
#pragma unroll
      for (int u = 0; u < kCeU; ++u) {
        const int i = i0 + u * kCeThreads;
        if (i < nv) {
          float p0 = __expf(x[u].x - lse), p1 = __expf(x[u].y - lse), p2 = __expf(x[u].z - lse), p3 = __expf(x[u].w - lse);
          const int64_t c = 4 * (int64_t)i;
          if (c == t) p0 -= 1.f;
          if (c + 1 == t) p1 -= 1.f;
          if (c + 2 == t) p2 -= 1.f;
          if (c + 3 == t) p3 -= 1.f;
          *reinterpret_cast<uint2*>(g + c) =
              make_uint2(pack_bf16x2(p0 * inv_s, p1 * inv_s), pack_bf16x2(p2 * inv_s, p3 * inv_s));
        }
      }
    }
    for (int i = nv * 4 + threadIdx.x; i < V; i += kCeThreads) {
      float p = __expf(logits[row * V + i] - lse) - (i == t ? 1.f : 0.f);
      g[i] = __float2bfloat16_rn(p * inv_s);
    }
    __syncthreads();  // s_lse / sm / ss are rewritten by the next row
  }
}

}  // namespace lx

using namespace lx;

extern "C" {

int lx_cross_entropy(const float* logits, int rows, int V, const int64_t* targets, float inv_s, float* row_loss,
                     uint16_t* grad_bf16, lx_stream_t stream) {
  LX_REQUIRE(rows >= 1 && V >= 1, LX_ERR_SHAPE, "cross_entropy: empty shape");
  LX_REQUIRE(V % 4 == 0, LX_ERR_UNSUPPORTED, "cross_entropy: vocab must be a multiple of 4");
  static const int per_sm = getenv("LX_CE_CTAS_PER_SM") ? atoi(getenv("LX_CE_CTAS_PER_SM")) : kCeCtasPerSm;  // experiment knob
  const int cap = (per_sm > 0 ? per_sm : kCeCtasPerSm) * num_sms();
  const int grid = rows < cap ? rows : cap;
  launch_k(ce_kernel, grid, kCeThreads, 0, stream, logits, rows, V, targets, inv_s, row_loss,
           reinterpret_cast<__nv_bfloat16*>(grad_bf16));
  return launch_check("cross_entropy");
}

}  // extern "C"
