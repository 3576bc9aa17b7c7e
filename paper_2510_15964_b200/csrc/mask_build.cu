// K1 — predictor scoring + prolonged-range aggregation -> compacted index lists.
//
// MLP (sf/predictor.py:121-139, sf/neuron_ops.py:67-72):
//   S = h * Wa_hat on tcgen05 (gemm_sm100, kEpiMask epilogue): each epilogue warp ORs
//   (S > thr) over its 32 rows with ballots and stores one 32-bit word per
//   (item, 32-row group, 32 blocks) -- every word stored exactly once, so no memset and
//   no atomics. The compaction kernel ORs an item's groups and turns the bitmask into
//   ascending active-block ids, counts and the inverse map pos[item][blk] (packed
//   position or -1): two launches per call.
// Attention (sf/predictor.py:62-118, sf/exposer.py:71-85):
//   [Q_hat | K_hat] = X_small * [Wq_hat | Wk_hat] for every head at once (one
//   tcgen05 GEMM), then one CTA per (item, head): S_hat = Q_hat K_hat^T (fp32),
//   per-matrix max, fp32 threshold frac*peak (NEP-50 rounding), strict '>',
//   OR over items (batch scope), nearest-cell upsample, integer coverage counts
//   per pool pattern and the fp64 (mass/total >= tau - 1e-9) selection with the
//   fewest-blocks / pool-order tie-break.
#include <cstdlib>
#include "common.cuh"
#include "gemm_sm100.cuh"

namespace lx {

int gemm_dual_launch(bool mask_epi, const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& args, cudaStream_t st);
// LX_PRED_DUAL=0: the k_terms 2 scoring GEMMs as one K-extended GEMM (A re-read per term) instead of the dual
// hi/lo CTA-pair engine (measurements)
static bool pred_dual() {
  static const bool on = [] { const char* e = getenv("LX_PRED_DUAL"); return !(e && e[0] == '0'); }();
  return on;
}

constexpr int kCompactMaxWords = 512;  // n_blk <= 16384 neuron blocks

// bits -> ascending active ids, counts and the inverse map, one CTA per item, fully parallel:
// per-word popcounts, one warp's exclusive scan over the words, then one thread per block writes
// its id at (word prefix + popc of the lower bits of its word). No serial per-bit loop.
// bits [n_items, n_slots, words]: an item's mask is the OR of its slots (the scoring GEMM's 32-row groups)
__global__ void mask_compact_kernel(const uint32_t* __restrict__ bits, int n_items, int n_blk, int scope_batch,
                                    int n_slots, int32_t* __restrict__ counts, int32_t* __restrict__ ids,
                                    int32_t* __restrict__ pos) {
  pdl_wait_trigger();
  const int item = blockIdx.x;
  const int words = (n_blk + 31) / 32;
  __shared__ uint32_t s_v[kCompactMaxWords];
  __shared__ int s_pre[kCompactMaxWords];
  __shared__ int s_total;
  for (int w = threadIdx.x; w < words; w += blockDim.x) {
    uint32_t v = 0;
    const int b0 = scope_batch ? 0 : item, b1 = scope_batch ? n_items : item + 1;
    for (int b = b0; b < b1; ++b)
      for (int t = 0; t < n_slots; ++t) v |= bits[((size_t)b * n_slots + t) * words + w];
    if (w == words - 1 && (n_blk & 31)) v &= (1u << (n_blk & 31)) - 1u;
    s_v[w] = v;
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan of the word popcounts: lane owns a contiguous run of words
    const int lane = threadIdx.x, per = (words + 31) / 32, w0 = lane * per, w1 = min(words, w0 + per);
    int local = 0;
    for (int w = w0; w < w1; ++w) local += __popc(s_v[w]);
    int inc = local;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    int run = inc - local;
    for (int w = w0; w < w1; ++w) {
      s_pre[w] = run;
      run += __popc(s_v[w]);
    }
    if (lane == 31) s_total = inc;
  }
  __syncthreads();
  int32_t* my_ids = ids + (size_t)item * n_blk;
  int32_t* my_pos = pos ? pos + (size_t)item * n_blk : nullptr;
  for (int b = threadIdx.x; b < n_blk; b += blockDim.x) {
    const uint32_t v = s_v[b >> 5];
    const int l = b & 31;
    const bool on = (v >> l) & 1u;
    const int r = s_pre[b >> 5] + __popc(v & ((1u << l) - 1u));
    if (on) my_ids[r] = b;
    if (my_pos) my_pos[b] = on ? r : -1;
  }
  const int total = s_total;
  if (threadIdx.x == 0) counts[item] = total;
  for (int j = total + threadIdx.x; j < n_blk; j += blockDim.x) my_ids[j] = 0;  // defined tail (no fill launch)
}

// membership of block (i, j) in pool pattern (kind, p) — sf/patterns.py:63-85
__device__ __forceinline__ bool pool_member(int kind, int p, int i, int j) {
  int dd = i - j;
  switch (kind) {
    case 0: return dd == 0;                                  // blockdiag
    case 1: return dd <= p && dd >= -p;                      // band{p}
    case 2: return dd >= 0 && dd <= p;                       // causal{p}
    case 3: return i < p || j < p || dd == 0;                // global{p}
    case 4: return ((dd % p) + p) % p == 0;                  // strided{p}
    default: return true;                                    // dense
  }
}

constexpr int kMaxPool = 16;
constexpr int kMaxM = 64;

// two blocks per SM (register cap, full shared-memory carveout): the (item, head) blocks are latency chains, and
// one resident block per SM ran the 256 blocks at cfg3 in two waves
__global__ void __launch_bounds__(256, 2) attn_pattern_kernel(const float* __restrict__ proj, int n_items, int m, int H, int r, float frac,
                                    double tau, int n_b, const int32_t* __restrict__ pool_kind,
                                    const int32_t* __restrict__ pool_param, int n_pool, int scope_batch,
                                    int32_t* __restrict__ pattern_idx, float* __restrict__ dump) {
  pdl_wait_trigger();
  const int h = blockIdx.x;
  const int item0 = scope_batch ? 0 : blockIdx.y;
  const int item1 = scope_batch ? n_items : blockIdx.y + 1;
  const int ldp = 2 * H * r;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, n_warps = blockDim.x >> 5;
  __shared__ float s_hat[kMaxM * kMaxM];
  __shared__ unsigned char cell[kMaxM * kMaxM];
  __shared__ float s_red[32];
  __shared__ int s_cnt[kMaxPool + 1][2];  // [pattern][0] = mass, [1] = active blocks; [kMaxPool][0] = total
  __shared__ int s_pool[2][kMaxPool];     // pool kinds / parameters (loaded once, off the coverage loop)
  extern __shared__ float s_qk[];          // [2][m][rs]: this (item, head)'s Q_hat and K_hat rows
  const int mm = m * m;
  const bool vec = (r & 3) == 0;
  const int rs = vec ? r + 4 : r + 1;      // 16B-aligned rows (float4 path) / odd stride (scalar path)
  for (int e = threadIdx.x; e < mm; e += blockDim.x) cell[e] = 0;
  if (threadIdx.x < (kMaxPool + 1) * 2) (&s_cnt[0][0])[threadIdx.x] = 0;
  if (threadIdx.x < n_pool) {
    s_pool[0][threadIdx.x] = __ldg(pool_kind + threadIdx.x);
    s_pool[1][threadIdx.x] = __ldg(pool_param + threadIdx.x);
  }
  for (int item = item0; item < item1; ++item) {
    __syncthreads();
    if (vec && blockDim.x % (r / 4) == 0) {
      // thread -> (row, float4 column): no index division in the loop; batches of 8 loads before any store
      const int r4 = r / 4, rp = blockDim.x / r4, t4 = threadIdx.x % r4, nrow = 2 * m;
      for (int base = threadIdx.x / r4; base < nrow; base += 8 * rp) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int row = base + u * rp;
          if (row < nrow) {
            const int which = row >= m, i = which ? row - m : row;
            v[u] = __ldg(reinterpret_cast<const float4*>(proj + (size_t)(item * m + i) * ldp + (which ? H + h : h) * r) + t4);
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int row = base + u * rp;
          if (row < nrow) reinterpret_cast<float4*>(s_qk + row * rs)[t4] = v[u];
        }
      }
    } else if (vec) {
      // float4 loads, issued in batches of 8 before any store (one round trip per batch)
      const int r4 = r / 4, nq = 2 * m * r4;
      for (int e0 = threadIdx.x; e0 < nq; e0 += 8 * blockDim.x) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * blockDim.x;
          if (e < nq) {
            const int which = e / (m * r4), rem = e % (m * r4), i = rem / r4, t4 = rem % r4;
            v[u] = __ldg(reinterpret_cast<const float4*>(proj + (size_t)(item * m + i) * ldp + (which ? H + h : h) * r) + t4);
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * blockDim.x;
          if (e < nq) {
            const int which = e / (m * r4), rem = e % (m * r4), i = rem / r4, t4 = rem % r4;
            reinterpret_cast<float4*>(s_qk + (which * m + i) * rs)[t4] = v[u];
          }
        }
      }
    } else {
      for (int e = threadIdx.x; e < 2 * m * r; e += blockDim.x) {  // coalesced: consecutive threads, consecutive t
        const int which = e / (m * r), rem = e % (m * r), i = rem / r, t = rem % r;
        s_qk[(which * m + i) * rs + t] = proj[(size_t)(item * m + i) * ldp + (which ? H + h : h) * r + t];
      }
    }
    __syncthreads();
    // S_hat = (X Wq)(X Wk)^T  (sf/predictor.py:74-76): warp w takes rows i = w, w + n_warps, ..., lane j a
    // column; q_i is a warp broadcast, k_j rows are conflict-free (row stride rs = r + 4 / r + 1). Four
    // partial sums over t mod 4 combined in a fixed order: deterministic.
    if (vec) {
      // two rows per pass (i, i + n_warps): each k_j float4 feeds both, twice the independent FMA chains; per
      // (i, j) the same four partial sums in the same order as the one-row loop below
      for (int i = warp; i < m; i += 2 * n_warps) {
        const int i2 = i + n_warps < m ? i + n_warps : i;
        const float* qr = s_qk + i * rs;
        const float* qr2 = s_qk + i2 * rs;
        for (int j = lane; j < m; j += 32) {
          const float* kr = s_qk + (m + j) * rs;
          float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f, b0 = 0.f, b1 = 0.f, b2 = 0.f, b3 = 0.f;
#pragma unroll 8
          for (int t = 0; t < r; t += 4) {
            const float4 k4 = *reinterpret_cast<const float4*>(kr + t);
            const float4 q4 = *reinterpret_cast<const float4*>(qr + t), p4 = *reinterpret_cast<const float4*>(qr2 + t);
            a0 = fmaf(q4.x, k4.x, a0);
            a1 = fmaf(q4.y, k4.y, a1);
            a2 = fmaf(q4.z, k4.z, a2);
            a3 = fmaf(q4.w, k4.w, a3);
            b0 = fmaf(p4.x, k4.x, b0);
            b1 = fmaf(p4.y, k4.y, b1);
            b2 = fmaf(p4.z, k4.z, b2);
            b3 = fmaf(p4.w, k4.w, b3);
          }
          const float acc = (a0 + a1) + (a2 + a3), acc2 = (b0 + b1) + (b2 + b3);
          s_hat[i * m + j] = acc;
          if (dump) dump[((size_t)item * H + h) * mm + i * m + j] = acc;
          if (i2 != i) {
            s_hat[i2 * m + j] = acc2;
            if (dump) dump[((size_t)item * H + h) * mm + i2 * m + j] = acc2;
          }
        }
      }
    } else
    for (int i = warp; i < m; i += n_warps) {
      const float* qr = s_qk + i * rs;
      for (int j = lane; j < m; j += 32) {
        const float* kr = s_qk + (m + j) * rs;
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
        if (vec) {
#pragma unroll 8
          for (int t = 0; t < r; t += 4) {
            const float4 q4 = *reinterpret_cast<const float4*>(qr + t), k4 = *reinterpret_cast<const float4*>(kr + t);
            a0 = fmaf(q4.x, k4.x, a0);
            a1 = fmaf(q4.y, k4.y, a1);
            a2 = fmaf(q4.z, k4.z, a2);
            a3 = fmaf(q4.w, k4.w, a3);
          }
        } else {
          int t = 0;
          for (; t + 4 <= r; t += 4) {
            a0 = fmaf(qr[t], kr[t], a0);
            a1 = fmaf(qr[t + 1], kr[t + 1], a1);
            a2 = fmaf(qr[t + 2], kr[t + 2], a2);
            a3 = fmaf(qr[t + 3], kr[t + 3], a3);
          }
          for (; t < r; ++t) a0 = fmaf(qr[t], kr[t], a0);
        }
        const float acc = (a0 + a1) + (a2 + a3);
        s_hat[i * m + j] = acc;
        if (dump) dump[((size_t)item * H + h) * mm + i * m + j] = acc;
      }
    }
    __syncthreads();
    // per-matrix max (sf/predictor.py:89)
    float mx = -INFINITY;
    for (int e = threadIdx.x; e < mm; e += blockDim.x) mx = fmaxf(mx, s_hat[e]);
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) s_red[warp] = mx;
    __syncthreads();
    if (threadIdx.x < 32) {
      float v = threadIdx.x < n_warps ? s_red[threadIdx.x] : -INFINITY;
      for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (threadIdx.x == 0) s_red[0] = v;
    }
    __syncthreads();
    // threshold = fp32(frac) * peak rounded to fp32; strict '>' (sf/predictor.py:90, NEP 50)
    const float thr = __fmul_rn(frac, s_red[0]);
    for (int e = threadIdx.x; e < mm; e += blockDim.x) cell[e] |= (s_hat[e] > thr) ? 1 : 0;  // OR over batch
  }
  __syncthreads();
  // upsample (sf/predictor.py:79-84) + integer coverage counts per pattern (sf/exposer.py:71-85): warp w
  // owns patterns w, w + 8 (no per-thread loop over the pool), lanes sweep the grid cells, integer warp
  // sums (order-free); warp 0 also counts the active cells
  const int cells = n_b * n_b;
  for (int p = warp; p < n_pool; p += n_warps) {
    const int kind = s_pool[0][p], prm = s_pool[1][p];
    int mass = 0, nnz = 0, tot = 0;
    for (int e = lane; e < cells; e += 32) {
      const int i = e / n_b, j = e - (e / n_b) * n_b;
      const int si = min((i * m) / n_b, m - 1), sj = min((j * m) / n_b, m - 1);
      const bool on = cell[si * m + sj] != 0;
      const bool in = pool_member(kind, prm, i, j);
      nnz += in;
      mass += in && on;
      tot += on;
    }
    mass = __reduce_add_sync(0xffffffffu, mass);
    nnz = __reduce_add_sync(0xffffffffu, nnz);
    tot = __reduce_add_sync(0xffffffffu, tot);
    if (lane == 0) {
      s_cnt[p][0] = mass;
      s_cnt[p][1] = nnz;
      if (p == 0) s_cnt[kMaxPool][0] = tot;
    }
  }
  __syncthreads();
  if (warp == 0) {
    // lane p: fp64 coverage mass/total >= tau - 1e-9 (the reference's float64 division, one per lane);
    // the winner is the fewest active blocks, then the lowest pool index: min over (nnz, p)
    const int total = s_cnt[kMaxPool][0];
    int key = 0x7fffffff;
    if (total > 0 && lane < n_pool) {
      const double frac_cov = (double)s_cnt[lane][0] / (double)total;
      if (frac_cov >= tau - 1e-9) key = (s_cnt[lane][1] << 5) | lane;
    }
    key = __reduce_min_sync(0xffffffffu, key);
    if (lane == 0)
      pattern_idx[(size_t)(scope_batch ? 0 : blockIdx.y) * H + h] = key == 0x7fffffff ? n_pool - 1 : (key & 31);
  }
}

}  // namespace lx

using namespace lx;

extern "C" {

int lx_mask_compact(const uint32_t* bits, int n_items, int n_blk, int scope_batch, int32_t* counts, int32_t* ids,
                    int32_t* pos, lx_stream_t stream) {
  LX_REQUIRE(n_items >= 1 && n_blk >= 1, LX_ERR_SHAPE, "mask_compact: empty shape");
  LX_REQUIRE(n_blk <= 32 * kCompactMaxWords, LX_ERR_UNSUPPORTED, "mask_compact: n_blk %d > %d", n_blk, 32 * kCompactMaxWords);
  launch_k(mask_compact_kernel, n_items, 512, 0, stream, bits, n_items, n_blk, scope_batch, 1, counts, ids, pos);
  return launch_check("mask_compact");
}

static int mask_compact_slots(const uint32_t* bits, int n_items, int n_blk, int scope_batch, int n_slots, int32_t* counts,
                              int32_t* ids, int32_t* pos, cudaStream_t stream) {
  launch_k(mask_compact_kernel, n_items, 512, 0, stream, bits, n_items, n_blk, scope_batch, n_slots, counts, ids, pos);
  return launch_check("mask_compact");
}

int lx_predict_mlp_mask(const uint16_t* h, int n_items, int s, int d, const uint16_t* wa_t, int n_blk, int k_terms,
                        float threshold, int scope_batch, uint32_t* bits_ws, int32_t* counts, int32_t* ids, int32_t* pos,
                        float* scores_dump, lx_stream_t stream) {
  LX_REQUIRE(n_items >= 1 && s >= 1 && d >= 1 && n_blk >= 1, LX_ERR_SHAPE, "predict_mlp_mask: empty shape");
  LX_REQUIRE(k_terms >= 1 && k_terms <= 3 && (k_terms == 1 || d % kBK == 0), LX_ERR_SHAPE,
             "predict_mlp_mask: k_terms %d (1..3; split terms need d %% %d == 0)", k_terms, kBK);
  LX_REQUIRE(n_items <= kMaxItems, LX_ERR_UNSUPPORTED, "too many items");
  const int words = (n_blk + 31) / 32;
  const int slots = (s + 31) / 32;  // bits_ws: [n_items, slots, words], every word stored by the GEMM (no memset)
  // 128-wide tiles when 256-wide ones would leave SMs idle (n_blk = 512: 64 tiles at B = 8 x 512 tokens)
  const long long tiles256 = (long long)n_items * ((s + kBM - 1) / kBM) * ((n_blk + 255) / 256);
  const int bn = tiles256 < num_sms() ? 128 : 256;
  CUtensorMap ta, tb;
  int rc;
  if (k_terms == 2 && pred_dual()) {
    // h [M, d] read once per K stage against W_hi and W_lo (two MMAs into one accumulator), 256 x 128 pair tiles
    if ((rc = make_tmap_bf16_2d(&ta, h, d, (uint64_t)n_items * s, d, kBK, kBM))) return rc;
    if ((rc = make_tmap_bf16_2d(&tb, wa_t, 2 * d, n_blk, 2 * d, kBK, 64))) return rc;
    GemmArgs args;
    memset(&args, 0, sizeof(args));
    args.n_items = n_items;
    args.rows_per_item = s;
    args.n_dense = n_blk;
    args.k_dense = d;
    args.dual_k = d;
    args.blk = 16;
    args.out = scores_dump;
    args.ldo = n_blk;
    args.thr = threshold;
    args.bits = bits_ws;
    args.bits_stride = words;
    args.bits_slots = slots;
    args.lora_scale = 1.f;
    if ((rc = gemm_dual_launch(true, ta, tb, args, stream))) return rc;
    return mask_compact_slots(bits_ws, n_items, n_blk, scope_batch, slots, counts, ids, pos, stream);
  }
  // k_terms 2: h [M, d] x [W_hi | W_lo]; 3: [x_hi | x_lo] [M, 2d] x [W_hi | W_lo | W_hi] (A's K wraps at d)
  const int a_cols = k_terms == 3 ? 2 * d : d, kt = k_terms * d;
  if ((rc = make_tmap_bf16_2d(&ta, h, a_cols, (uint64_t)n_items * s, a_cols, kBK, kBM))) return rc;
  if ((rc = make_tmap_bf16_2d(&tb, wa_t, kt, n_blk, kt, kBK, bn))) return rc;
  GemmArgs args;
  memset(&args, 0, sizeof(args));
  args.n_items = n_items;
  args.rows_per_item = s;
  args.n_dense = n_blk;
  args.k_dense = kt;
  args.a_k_split = k_terms > 1 ? d : 0;
  args.blk = 16;
  args.out = scores_dump;
  args.ldo = n_blk;
  args.thr = threshold;
  args.bits = bits_ws;
  args.bits_stride = words;
  args.bits_slots = slots;
  args.lora_scale = 1.f;
  if (bn == 128) {
    auto kern = gemm_sm100_kernel<kDense, kEpiMask, 128>;
    constexpr int smem = GemmSmem<128>::kTotal;
    static cudaError_t attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    LX_CHECK_CUDA(attr);
    launch_k(kern, num_sms(), kGemmThreads, smem, stream, ta, tb, args);
  } else {
    auto kern = gemm_sm100_kernel<kDense, kEpiMask, 256>;
    constexpr int smem = GemmSmem<256>::kTotal;
    static cudaError_t attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    LX_CHECK_CUDA(attr);
    launch_k(kern, num_sms(), kGemmThreads, smem, stream, ta, tb, args);
  }
  if ((rc = launch_check("mlp mask gemm"))) return rc;
  return mask_compact_slots(bits_ws, n_items, n_blk, scope_batch, slots, counts, ids, pos, stream);
}

int lx_predict_attention_patterns(const uint16_t* x_small, int n_items, int m, int d, const uint16_t* wqk_t, int H,
                                  int r, int k_terms, float threshold_frac, double tau, int n_b, const int32_t* pool_kind,
                                  const int32_t* pool_param, int n_pool, int scope_batch, float* proj_ws,
                                  int32_t* pattern_idx, float* scores_dump, lx_stream_t stream) {
  LX_REQUIRE(m >= 1 && m <= kMaxM, LX_ERR_UNSUPPORTED, "downsampled length m=%d outside [1, %d] (s <= 4096)", m, kMaxM);
  LX_REQUIRE(n_pool >= 1 && n_pool <= kMaxPool, LX_ERR_PATTERN, "pool size %d outside [1, %d]", n_pool, kMaxPool);
  LX_REQUIRE(tau > 0 && tau <= 1, LX_ERR_SHAPE, "coverage tau must be in (0, 1]");
  LX_REQUIRE(k_terms >= 1 && k_terms <= 3 && (k_terms == 1 || d % 64 == 0), LX_ERR_SHAPE,
             "predict_attention_patterns: k_terms %d (1..3; split terms need d %% 64 == 0)", k_terms);
  int rc;
  if (k_terms == 2 && pred_dual()) {
    // x_small [B*m, d] read once per K stage against W_hi and W_lo: B*m <= 256 rows fit one pair tile, so every
    // weight row is streamed from HBM once
    CUtensorMap ta, tb;
    if ((rc = make_tmap_bf16_2d(&ta, x_small, d, (uint64_t)n_items * m, d, kBK, kBM))) return rc;
    if ((rc = make_tmap_bf16_2d(&tb, wqk_t, 2 * d, 2 * H * r, 2 * d, kBK, 64))) return rc;
    GemmArgs args;
    memset(&args, 0, sizeof(args));
    args.n_items = 1;
    args.rows_per_item = n_items * m;
    args.n_dense = 2 * H * r;
    args.k_dense = d;
    args.dual_k = d;
    args.blk = 16;
    args.out = proj_ws;
    args.ldo = 2 * H * r;
    args.out_f32 = 1;
    args.lora_scale = 1.f;
    rc = gemm_dual_launch(false, ta, tb, args, stream);
  } else {
  // k_terms 2: x_small [M, d] x [W_hi | W_lo]; 3: [x_hi | x_lo] [M, 2d] x [W_hi | W_lo | W_hi]
  rc = lx_gemm_bf16_tn(x_small, k_terms == 3 ? 2 * d : d, wqk_t, k_terms * d, proj_ws, 2 * H * r, 1, n_items * m,
                           2 * H * r, k_terms * d, k_terms > 1 ? d : 0, stream);
  }
  if (rc) return rc;
  dim3 grid(H, scope_batch ? 1 : n_items);
  const size_t smem = sizeof(float) * 2 * m * (r + 4);
  LX_REQUIRE(smem <= 200 * 1024, LX_ERR_UNSUPPORTED, "predictor rank %d x m %d exceeds shared memory", r, m);
  static cudaError_t attr = [] {
    cudaError_t e = cudaFuncSetAttribute(attn_pattern_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(attn_pattern_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
    return e;
  }();
  LX_CHECK_CUDA(attr);
  launch_k(attn_pattern_kernel, grid, 256, smem, stream, proj_ws, n_items, m, H, r, threshold_frac, tau, n_b, pool_kind,
                                                     pool_param, n_pool, scope_batch, pattern_idx, scores_dump);
  return launch_check("attn_pattern");
}

}  // extern "C"
