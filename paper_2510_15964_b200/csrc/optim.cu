// Adam over the flat trainable buffer (sf/autograd.py:203-225): float64 moments, fp32 parameters,
// one pass (the fp32 mean gradient is widened in registers). Same operation order as the reference:
//   m = b1 m + (1 - b1) g;  v = b2 v + (1 - b2) g g;  p -= fp32(lr * (m / c1) / (sqrt(v / c2) + eps))
// with c1 = 1 - b1^t, c2 = 1 - b2^t.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "ptx.cuh"

namespace lx {

__global__ void __launch_bounds__(256) adam_kernel(float* __restrict__ p, const float* __restrict__ g, double* __restrict__ m,
                                                   double* __restrict__ v, long long n, double lr, double b1, double b2,
                                                   double eps, double c1, double c2) {
  pdl_wait_trigger();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    const double gi = (double)g[i];
    const double mi = b1 * m[i] + (1.0 - b1) * gi;
    const double vi = b2 * v[i] + (1.0 - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    const double mh = mi / c1, vh = vi / c2;
    p[i] -= (float)(lr * mh / (sqrt(vh) + eps));
  }
}

}  // namespace lx

using namespace lx;

extern "C" {

int lx_adam_step(float* params, const float* grads, double* m, double* v, long long n, double lr, double b1, double b2,
                 double eps, int t, lx_stream_t stream) {
  LX_REQUIRE(n >= 0 && t >= 1, LX_ERR_SHAPE, "adam: n >= 0 and step t >= 1 required");
  if (n == 0) return LX_OK;
  const double c1 = 1.0 - pow(b1, (double)t), c2 = 1.0 - pow(b2, (double)t);
  const long long blocks = std::min<long long>((n + 255) / 256, 8LL * num_sms());
  launch_k(adam_kernel, (unsigned)blocks, 256, 0, stream, params, grads, m, v, n, lr, b1, b2, eps, c1, c2);
  return launch_check("adam");
}

}  // extern "C"
