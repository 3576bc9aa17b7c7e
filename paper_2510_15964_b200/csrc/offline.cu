// Offline predictor pipeline on the GPU (sf/harness.py:251-371, sf/predictor.py:171-298):
// the two non-GEMM pieces of MLP-predictor training. The GEMMs (logits = X Wa, grad = X^T dL)
// are plain fp32 library GEMMs; Adam is lx_adam_step (optim.cu).
//
// lx_block_activity — mlp_truth_labels (sf/predictor.py:251-259): bit b of row t set iff any
//   neuron of block b has z > 0 for token t. One CTA per row: coalesced column sweep, warp
//   ballots, shared-memory OR words (OR is idempotent, so the bits are deterministic).
// lx_weighted_bce — the loss and logit gradient of train_mlp_predictor (sf/predictor.py:281-289):
//   per element, with y the truth bit and w = recall_weight,
//     loss = -(w y log sigmoid(l) + (1 - y) log(1 - sigmoid(l)))   (stable log-sum-exp forms)
//     dL/dl = (w y (sigmoid(l) - 1) + (1 - y) sigmoid(l)) / (rows * n_blk)
//   row_loss[t] = sum over the row in float64, fixed order (the caller sums rows in order).
#include "common.cuh"
#include "ptx.cuh"

namespace lx {

__global__ void block_activity_kernel(const float* __restrict__ z, int ldz, int n_cols, int blk, int words,
                                      uint32_t* __restrict__ bits) {
  pdl_wait_trigger();  // launched with PDL (launch_k): see the predecessor's writes first
  extern __shared__ uint32_t act[];
  const int row = blockIdx.x;
  for (int w = threadIdx.x; w < words; w += blockDim.x) act[w] = 0u;
  __syncthreads();
  const float* zr = z + (size_t)row * ldz;
  for (int c0 = 0; c0 < n_cols; c0 += blockDim.x) {
    const int c = c0 + threadIdx.x;
    const bool on = c < n_cols && zr[c] > 0.f;
    const uint32_t lanes = __ballot_sync(0xffffffffu, on);
    // the warp's lanes of one block are contiguous, [lo, hi]; its lowest lane publishes the block
    const int lane = threadIdx.x & 31, base = c - lane, b = c / blk;
    const int lo = max(0, b * blk - base), hi = min(31, (b + 1) * blk - 1 - base);
    if (c < n_cols && lane == lo) {
      const uint32_t span = (hi - lo == 31) ? 0xffffffffu : (((1u << (hi - lo + 1)) - 1u) << lo);
      if (lanes & span) atomicOr(&act[b >> 5], 1u << (b & 31));
    }
  }
  __syncthreads();
  for (int w = threadIdx.x; w < words; w += blockDim.x) bits[(size_t)row * words + w] = act[w];
}

__device__ __forceinline__ float log_sigmoid(float x) {  // -logaddexp(0, -x)
  return -(fmaxf(-x, 0.f) + log1pf(expf(-fabsf(x))));
}

// one warp per row
__global__ void weighted_bce_kernel(const float* __restrict__ logits, int ld, int rows, int n_blk,
                                    const uint32_t* __restrict__ labels, int words, float pos_w, double inv_size,
                                    float* __restrict__ d_logits, int ldd, double* __restrict__ row_loss) {
  pdl_wait_trigger();  // launched with PDL (launch_k): see the predecessor's writes first
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* lr = logits + (size_t)row * ld;
  const uint32_t* yr = labels + (size_t)row * words;
  double acc = 0.0;
  for (int b = lane; b < n_blk; b += 32) {
    const float l = lr[b];
    const bool y = (yr[b >> 5] >> (b & 31)) & 1u;
    const float ls = log_sigmoid(l), l1m = log_sigmoid(-l);  // log(1 - sigmoid(l)) = log sigmoid(-l)
    acc += y ? -(double)pos_w * ls : -(double)l1m;
    const float sg = 1.f / (1.f + expf(-l));
    const double g = y ? (double)pos_w * (sg - 1.f) : (double)sg;
    d_logits[(size_t)row * ldd + b] = (float)(g * inv_size);
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) row_loss[row] = acc;
}

}  // namespace lx

using namespace lx;

extern "C" {

int lx_block_activity(const float* z, int ldz, int rows, int n_cols, int blk, uint32_t* bits, lx_stream_t stream) {
  LX_REQUIRE(rows >= 1 && n_cols >= 1 && blk >= 1, LX_ERR_SHAPE, "block_activity: empty shape");
  LX_REQUIRE(ldz >= n_cols, LX_ERR_SHAPE, "row stride %d < columns %d", ldz, n_cols);
  const int n_blk = (n_cols + blk - 1) / blk, words = (n_blk + 31) / 32;
  launch_k(block_activity_kernel, rows, 256, sizeof(uint32_t) * words, stream, z, ldz, n_cols, blk, words, bits);
  return launch_check("block_activity");
}

int lx_weighted_bce(const float* logits, int ld, int rows, int n_blk, const uint32_t* labels, float pos_w,
                    float* d_logits, int ldd, double* row_loss, lx_stream_t stream) {
  LX_REQUIRE(rows >= 1 && n_blk >= 1, LX_ERR_SHAPE, "weighted_bce: empty shape");
  LX_REQUIRE(pos_w >= 1.f, LX_ERR_SHAPE, "recall_weight must be >= 1");
  const int words = (n_blk + 31) / 32;
  const double inv_size = 1.0 / ((double)rows * (double)n_blk);
  launch_k(weighted_bce_kernel, (rows + 7) / 8, 256, 0, stream, logits, ld, rows, n_blk, labels, words, pos_w, inv_size,
           d_logits, ldd, row_loss);
  return launch_check("weighted_bce");
}

}  // extern "C"
