// Tied-unembedding cross-entropy forward + backward in one pass pair per row
// (sf/model.py:454-472): loss_row = logsumexp(l) - l[target];
// grad = (softmax(l) - onehot(target)) * inv_s, written bf16 for the d_hf GEMM.
// One CTA per row: an online (max, sum-exp) sweep, then a write sweep.
#include "common.cuh"
#include "ptx.cuh"

namespace lx {

__device__ __forceinline__ void online_merge(float& m, float& sum, float m2, float s2) {
  const float mn = fmaxf(m, m2);
  sum = (m == -INFINITY ? 0.f : sum * __expf(m - mn)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mn));
  m = mn;
}

__global__ void __launch_bounds__(256) ce_kernel(const float* __restrict__ logits, int V, const int64_t* __restrict__ tgt,
                                                 float inv_s, float* __restrict__ row_loss, __nv_bfloat16* __restrict__ grad) {
  pdl_wait_trigger();
  const size_t row = blockIdx.x;
  const float4* l4 = reinterpret_cast<const float4*>(logits + row * V);
  const int nv = V / 4;
  float m = -INFINITY, sum = 0.f;
  for (int i = threadIdx.x; i < nv; i += 256) {
    float4 x = l4[i];
    float mx = fmaxf(fmaxf(x.x, x.y), fmaxf(x.z, x.w));
    float s2 = __expf(x.x - mx) + __expf(x.y - mx) + __expf(x.z - mx) + __expf(x.w - mx);
    online_merge(m, sum, mx, s2);
  }
  for (int i = nv * 4 + threadIdx.x; i < V; i += 256) online_merge(m, sum, logits[row * V + i], 1.f);
  for (int o = 16; o; o >>= 1) {
    float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, sum, o);
    online_merge(m, sum, m2, s2);
  }
  __shared__ float sm[8], ss[8], s_lse;
  if ((threadIdx.x & 31) == 0) { sm[threadIdx.x >> 5] = m; ss[threadIdx.x >> 5] = sum; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = sm[0], S = ss[0];
    for (int w = 1; w < 8; ++w) online_merge(M, S, sm[w], ss[w]);
    s_lse = M + logf(S);
    const int64_t t = tgt[row];
    row_loss[row] = s_lse - logits[row * V + t];
  }
  __syncthreads();
  const float lse = s_lse;
  const int64_t t = tgt[row];
  __nv_bfloat16* g = grad + row * V;
  for (int i = threadIdx.x; i < nv; i += 256) {
    float4 x = l4[i];
    float p0 = __expf(x.x - lse), p1 = __expf(x.y - lse), p2 = __expf(x.z - lse), p3 = __expf(x.w - lse);
    const int64_t c = 4 * (int64_t)i;
    if (c == t) p0 -= 1.f;
    if (c + 1 == t) p1 -= 1.f;
    if (c + 2 == t) p2 -= 1.f;
    if (c + 3 == t) p3 -= 1.f;
    *reinterpret_cast<uint2*>(g + c) = make_uint2(pack_bf16x2(p0 * inv_s, p1 * inv_s), pack_bf16x2(p2 * inv_s, p3 * inv_s));
  }
  for (int i = nv * 4 + threadIdx.x; i < V; i += 256) {
    float p = __expf(logits[row * V + i] - lse) - (i == t ? 1.f : 0.f);
    g[i] = __float2bfloat16_rn(p * inv_s);
  }
}

}  // namespace lx

using namespace lx;

extern "C" {

int lx_cross_entropy(const float* logits, int rows, int V, const int64_t* targets, float inv_s, float* row_loss,
                     uint16_t* grad_bf16, lx_stream_t stream) {
  LX_REQUIRE(rows >= 1 && V >= 1, LX_ERR_SHAPE, "cross_entropy: empty shape");
  LX_REQUIRE(V % 4 == 0, LX_ERR_UNSUPPORTED, "cross_entropy: vocab must be a multiple of 4");
  launch_k(ce_kernel, rows, 256, 0, stream, logits, V, targets, inv_s, row_loss, reinterpret_cast<__nv_bfloat16*>(grad_bf16));
  return launch_check("cross_entropy");
}

}  // extern "C"
