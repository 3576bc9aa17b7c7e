// Bottleneck adapter on the device (sf/model.py:76-83,315-319; sf/autograd.py:69-75), fp32 like the reference:
//   forward   out = x + relu(x Wd + bd) Wu + bu            (x fp32 [M, d], Wd [d, r], Wu [r, d], r <= 16)
//   backward  dh = (dy Wu^T) * (z > 0);  dx = dy + dh Wd^T
//             gWu = relu(z)^T dy, gbu = sum dy, gWd = x^T dh, gbd = sum dh      (summed over rows)
// HBM-bound row work: CTAs own 16-row tiles and stream Wd / Wu through shared memory in 32 KB column chunks;
// two rows per warp, the r dot products reduced with butterfly shuffles. The column
// reductions for the gradients run as (column block x row chunk) CTAs writing partial sums, finished by a
// fixed-order sum over the chunks: deterministic, no atomics.
#include <algorithm>

#include "common.cuh"
#include "ptx.cuh"

namespace lx {

constexpr int kAdChunks = 16;  // row chunks of the gradient column reductions

template <int R>
LX_DEV void warp_allreduce(float (&a)[R]) {
#pragma unroll
  for (int j = 0; j < R; ++j)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a[j] += __shfl_xor_sync(0xffffffffu, a[j], o);
}

// Row kernels: a CTA owns a tile of kAdRows rows (2 per warp) and streams the weights through shared memory in
// column chunks of 8192 / R columns (so any d fits): pass 1 accumulates the R dot products of its rows chunk by chunk,
// pass 2 writes the rows chunk by chunk. The tile's x / dy rows are re-read in pass 2 from L2. Rows move as float4
// with kAdU loads per row in flight per lane (the scalar one-load-per-iteration form was latency-bound at ~4 B/clk
// per SM); a chunk sits in shared memory as [j][c] (padded rows), read as float4 over c: conflict-free.
constexpr int kAdRows = 16;
constexpr int kAdU = 4;

template <int R, bool BWD>
__global__ void __launch_bounds__(256) adapter_rows_kernel(const float* __restrict__ x, int ldx, int M, int d,
                                                           const float* __restrict__ w_in,   // fwd Wd [d][R]; bwd Wu [R][d]
                                                           const float* __restrict__ b_in,   // fwd bd [R]; bwd unused
                                                           const float* __restrict__ w_out,  // fwd Wu [R][d]; bwd Wd [d][R]
                                                           const float* __restrict__ b_out,  // fwd bu [d]; bwd unused
                                                           float* __restrict__ zr,           // fwd: z out; bwd: z in
                                                           float* __restrict__ dh,           // bwd: dh out
                                                           float* __restrict__ out, int ldo,
                                                           const float* __restrict__ resid, int ldr) {  // fwd: out += resid
  constexpr int kAdCh = 8192 / R;  // 32 KB of weights per chunk
  constexpr int kP = kAdCh + 4;    // padded [j] row (float4-aligned)
  __shared__ __align__(16) float sw[R * kP];
  pdl_wait_trigger();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int n_tiles = (M + kAdRows - 1) / kAdRows;
  // stage columns [c0, c0 + nc) of a weight as [j][c]; `rc`: the source is [d][R] (row c holds the R values)
  // (8 loads per thread in flight per round: a one-load-per-iteration loop is 32 dependent L2 round trips per chunk)
  auto stage = [&](const float* w, bool rc, int c0, int nc) {
    __syncthreads();
    constexpr int kSU = 8;
    for (int i0 = threadIdx.x; i0 < nc * R; i0 += kSU * 256) {
      float v[kSU];
#pragma unroll
      for (int u = 0; u < kSU; ++u) {
        const int i = i0 + u * 256;
        if (i < nc * R) v[u] = rc ? __ldg(w + (size_t)(c0 + i / R) * R + i % R) : __ldg(w + (size_t)(i / nc) * d + c0 + i % nc);
      }
#pragma unroll
      for (int u = 0; u < kSU; ++u) {
        const int i = i0 + u * 256;
        if (i < nc * R) {
          if (rc) sw[(i % R) * kP + i / R] = v[u];
          else sw[(i / nc) * kP + i % nc] = v[u];
        }
      }
    }
    __syncthreads();
  };
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int row0 = tile * kAdRows + wid * 2;
    float acc[2][R];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int j = 0; j < R; ++j) acc[q][j] = 0.f;
    // pass 1: t_j = sum_c x[c] W_in(c, j)
    for (int c0 = 0; c0 < d; c0 += kAdCh) {
      const int nc4 = min(kAdCh, d - c0) / 4;
      stage(w_in, !BWD, c0, nc4 * 4);
      for (int cb = lane; cb < nc4; cb += 32 * kAdU) {
        float4 xv[2][kAdU];
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int u = 0; u < kAdU; ++u) {
            const int c4 = cb + 32 * u;
            xv[q][u] = (row0 + q < M && c4 < nc4)
                           ? __ldg(reinterpret_cast<const float4*>(x + (size_t)(row0 + q) * ldx + c0) + c4)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
        for (int u = 0; u < kAdU; ++u) {
          const int c4 = cb + 32 * u;
          if (c4 < nc4) {
#pragma unroll
            for (int j = 0; j < R; ++j) {
              const float4 w = *reinterpret_cast<const float4*>(sw + j * kP + 4 * c4);
#pragma unroll
              for (int q = 0; q < 2; ++q) {
                acc[q][j] = fmaf(xv[q][u].x, w.x, acc[q][j]);
                acc[q][j] = fmaf(xv[q][u].y, w.y, acc[q][j]);
                acc[q][j] = fmaf(xv[q][u].z, w.z, acc[q][j]);
                acc[q][j] = fmaf(xv[q][u].w, w.w, acc[q][j]);
              }
            }
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      warp_allreduce<R>(acc[q]);
      const int row = row0 + q;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        if (BWD) {
          const bool on = row < M && zr[(size_t)row * R + j] > 0.f;
          acc[q][j] = on ? acc[q][j] : 0.f;  // dh = (dy Wu^T) * relu'(z)
          if (row < M && lane == j) dh[(size_t)row * R + j] = acc[q][j];
        } else {
          const float zj = acc[q][j] + b_in[j];
          if (row < M && lane == j) zr[(size_t)row * R + j] = zj;
          acc[q][j] = fmaxf(zj, 0.f);  // h
        }
      }
    }
    // pass 2: out[c] = x[c] (+ bu[c]) + sum_j a_j W_out(j, c)
    for (int c0 = 0; c0 < d; c0 += kAdCh) {
      const int nc4 = min(kAdCh, d - c0) / 4;
      stage(w_out, BWD, c0, nc4 * 4);
      for (int cb = lane; cb < nc4; cb += 32 * kAdU) {
        // every global load of the iteration (rows, bias, residual rows) issued before any use
        float4 xv[2][kAdU], rv[2][kAdU], bv[kAdU];
        const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < kAdU; ++u) {
          const int c4 = cb + 32 * u;
          bv[u] = (!BWD && c4 < nc4) ? __ldg(reinterpret_cast<const float4*>(b_out + c0) + c4) : z4;
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const bool ok = row0 + q < M && c4 < nc4;
            xv[q][u] = ok ? __ldg(reinterpret_cast<const float4*>(x + (size_t)(row0 + q) * ldx + c0) + c4) : z4;
            rv[q][u] = (!BWD && resid && ok) ? __ldg(reinterpret_cast<const float4*>(resid + (size_t)(row0 + q) * ldr + c0) + c4)
                                             : z4;
          }
        }
#pragma unroll
        for (int u = 0; u < kAdU; ++u) {
          const int c4 = cb + 32 * u;
          if (c4 >= nc4) continue;
          const float4 bc = bv[u];
          float4 v[2];
#pragma unroll
          for (int q = 0; q < 2; ++q)
            v[q] = make_float4(xv[q][u].x + bc.x, xv[q][u].y + bc.y, xv[q][u].z + bc.z, xv[q][u].w + bc.w);
#pragma unroll
          for (int j = 0; j < R; ++j) {
            const float4 w = *reinterpret_cast<const float4*>(sw + j * kP + 4 * c4);
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              v[q].x = fmaf(acc[q][j], w.x, v[q].x);
              v[q].y = fmaf(acc[q][j], w.y, v[q].y);
              v[q].z = fmaf(acc[q][j], w.z, v[q].z);
              v[q].w = fmaf(acc[q][j], w.w, v[q].w);
            }
          }
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (row0 + q >= M) continue;
            if (!BWD && resid)  // the block's residual add, after the adapter's own (same order as resid + out)
              v[q] = make_float4(rv[q][u].x + v[q].x, rv[q][u].y + v[q].y, rv[q][u].z + v[q].z, rv[q][u].w + v[q].w);
            reinterpret_cast<float4*>(out + (size_t)(row0 + q) * ldo + c0)[c4] = v[q];
          }
        }
      }
    }
  }
}

// column pass: CTA (column block of 32, row chunk) -> partials of gWu [R][32], gbu [32], gWd [32][R]; the chunk-0
// column block also sums dh for gbd. 8 warps stride the chunk's rows; lane = column; fixed-order warp merge.
template <int R>
__global__ void __launch_bounds__(256) adapter_bwd_cols_kernel(const float* __restrict__ dy, int ldy,
                                                               const float* __restrict__ x, int ldx, int M, int d,
                                                               const float* __restrict__ z, const float* __restrict__ dh,
                                                               float* __restrict__ part) {
  __shared__ float red[8][2 * R + 2][32];
  pdl_wait_trigger();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane, chunk = blockIdx.y;
  const int r0 = (int)(((long long)M * chunk) / kAdChunks), r1 = (int)(((long long)M * (chunk + 1)) / kAdChunks);
  float gwu[R], gwd[R], gbu = 0.f, gbd = 0.f;
#pragma unroll
  for (int j = 0; j < R; ++j) gwu[j] = gwd[j] = 0.f;
  const bool col_ok = c < d;
  // rows wid, wid + 8, ... in order (the accumulation order of a one-row loop), four rows' loads in flight
  constexpr int kRU = 4;
  for (int row = r0 + wid; row < r1; row += 8 * kRU) {
    float g[kRU], xv[kRU], gd[kRU];
    float4 zz[kRU][R / 4], dd[kRU][R / 4];
#pragma unroll
    for (int u = 0; u < kRU; ++u) {
      const int rr = row + 8 * u;
      const bool ok = rr < r1;
      g[u] = (ok && col_ok) ? dy[(size_t)rr * ldy + c] : 0.f;
      xv[u] = (ok && col_ok) ? x[(size_t)rr * ldx + c] : 0.f;
      gd[u] = (ok && blockIdx.x == 0 && lane < R) ? dh[(size_t)rr * R + lane] : 0.f;
#pragma unroll
      for (int t = 0; t < R / 4; ++t) {
        zz[u][t] = ok ? __ldg(reinterpret_cast<const float4*>(z + (size_t)rr * R) + t) : make_float4(0.f, 0.f, 0.f, 0.f);
        dd[u][t] = ok ? __ldg(reinterpret_cast<const float4*>(dh + (size_t)rr * R) + t) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int u = 0; u < kRU; ++u) {
      if (row + 8 * u >= r1) break;
      gbu += g[u];
#pragma unroll
      for (int t = 0; t < R / 4; ++t) {
        const float zj[4] = {zz[u][t].x, zz[u][t].y, zz[u][t].z, zz[u][t].w};
        const float dj[4] = {dd[u][t].x, dd[u][t].y, dd[u][t].z, dd[u][t].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          gwu[4 * t + e] = fmaf(fmaxf(zj[e], 0.f), g[u], gwu[4 * t + e]);
          gwd[4 * t + e] = fmaf(xv[u], dj[e], gwd[4 * t + e]);
        }
      }
      if (blockIdx.x == 0 && lane < R) gbd += gd[u];
    }
  }
#pragma unroll
  for (int j = 0; j < R; ++j) {
    red[wid][j][lane] = gwu[j];
    red[wid][R + j][lane] = gwd[j];
  }
  red[wid][2 * R][lane] = gbu;
  red[wid][2 * R + 1][lane] = gbd;
  __syncthreads();
  // partial layout per chunk: [gWu R*d][gbu d][gWd d*R][gbd R]
  float* pc = part + (size_t)chunk * ((size_t)2 * R * d + d + R);
  for (int q = threadIdx.x; q < (2 * R + 2) * 32; q += blockDim.x) {
    const int k = q / 32, l = q % 32, cc = blockIdx.x * 32 + l;
    float t = 0.f;
    for (int w = 0; w < 8; ++w) t += red[w][k][l];
    if (k < R) {
      if (cc < d) pc[(size_t)k * d + cc] = t;
    } else if (k < 2 * R) {
      if (cc < d) pc[(size_t)R * d + d + (size_t)cc * R + (k - R)] = t;
    } else if (k == 2 * R) {
      if (cc < d) pc[(size_t)R * d + cc] = t;
    } else if (blockIdx.x == 0 && l < R) {
      pc[(size_t)2 * R * d + d + l] = t;
    }
  }
}

// gradients = sum of the chunks' partials in chunk order, scaled (the engine's 1/B batch mean), written to the
// four destinations
__global__ void __launch_bounds__(256) adapter_bwd_final_kernel(const float* __restrict__ part, int n, float scale,
                                                                float* __restrict__ g_wu, float* __restrict__ g_bu,
                                                                float* __restrict__ g_wd, float* __restrict__ g_bd, int R,
                                                                int d) {
  pdl_wait_trigger();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float t = 0.f;
    for (int ch = 0; ch < kAdChunks; ++ch) t += part[(size_t)ch * n + i];
    t *= scale;
    if (i < R * d) g_wu[i] = t;
    else if (i < R * d + d) g_bu[i - R * d] = t;
    else if (i < 2 * R * d + d) g_wd[i - R * d - d] = t;
    else g_bd[i - 2 * R * d - d] = t;
  }
}

template <int R>
static int adapter_fwd_t(const float* x, int ldx, int M, int d, const float* wd, const float* bd, const float* wu,
                         const float* bu, float* z, float* out, int ldo, const float* resid, int ldr, cudaStream_t st) {
  const int tiles = (M + kAdRows - 1) / kAdRows;
  launch_k(adapter_rows_kernel<R, false>, std::min(tiles, 4 * num_sms()), 256, 0, st, x, ldx, M, d, wd, bd, wu, bu, z,
           (float*)nullptr, out, ldo, resid, ldr);
  return launch_check("adapter_fwd");
}

template <int R>
static int adapter_bwd_t(const float* dy, int ldy, const float* x, int ldx, int M, int d, const float* z, const float* wd,
                         const float* wu, float* dh, float* dx, int lddx, float* part, float scale, float* g_wd, float* g_bd,
                         float* g_wu, float* g_bu, cudaStream_t st) {
  const int tiles = (M + kAdRows - 1) / kAdRows;
  launch_k(adapter_rows_kernel<R, true>, std::min(tiles, 4 * num_sms()), 256, 0, st, dy, ldy, M, d, wu, (const float*)nullptr,
           wd, (const float*)nullptr, (float*)z, dh, dx, lddx, (const float*)nullptr, 0);
  int rc = launch_check("adapter_bwd_rows");
  if (rc) return rc;
  launch_k(adapter_bwd_cols_kernel<R>, dim3((d + 31) / 32, kAdChunks), 256, 0, st, dy, ldy, x, ldx, M, d, z,
           (const float*)dh, part);
  if ((rc = launch_check("adapter_bwd_cols"))) return rc;
  const int n = 2 * R * d + d + R;
  launch_k(adapter_bwd_final_kernel, std::min((n + 255) / 256, 4 * num_sms()), 256, 0, st, (const float*)part, n, scale,
           g_wu, g_bu, g_wd, g_bd, R, d);
  return launch_check("adapter_bwd_final");
}

}  // namespace lx

using namespace lx;

extern "C" {

long long lx_adapter_ws_floats(int d, int r) { return (long long)kAdChunks * (2LL * r * d + d + r); }

int lx_adapter_fwd(const float* x, int ldx, int M, int d, int r, const float* w_down, const float* b_down, const float* w_up,
                   const float* b_up, float* z, float* out, int ldo, const float* resid, int ldr, lx_stream_t stream) {
  LX_REQUIRE(M >= 1 && d >= 1 && (r == 8 || r == 16), LX_ERR_UNSUPPORTED, "adapter: rank %d (8 or 16 supported)", r);
  LX_REQUIRE(d % 4 == 0 && ldx % 4 == 0 && ldo % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                 (reinterpret_cast<uintptr_t>(out) & 15) == 0,
             LX_ERR_UNSUPPORTED, "adapter: d and row strides must be multiples of 4 floats, rows 16-byte aligned");
  LX_REQUIRE(!resid || (ldr % 4 == 0 && (reinterpret_cast<uintptr_t>(resid) & 15) == 0), LX_ERR_UNSUPPORTED,
             "adapter: residual row stride must be a multiple of 4 floats, rows 16-byte aligned");
  if (r == 8) return adapter_fwd_t<8>(x, ldx, M, d, w_down, b_down, w_up, b_up, z, out, ldo, resid, ldr, stream);
  return adapter_fwd_t<16>(x, ldx, M, d, w_down, b_down, w_up, b_up, z, out, ldo, resid, ldr, stream);
}

int lx_adapter_bwd(const float* dy, int ldy, const float* x, int ldx, int M, int d, int r, const float* z,
                   const float* w_down, const float* w_up, float* dh, float* dx, int lddx, float* ws, float scale,
                   float* g_w_down, float* g_b_down, float* g_w_up, float* g_b_up, lx_stream_t stream) {
  LX_REQUIRE(M >= 1 && d >= 1 && (r == 8 || r == 16), LX_ERR_UNSUPPORTED, "adapter: rank %d (8 or 16 supported)", r);
  LX_REQUIRE(d % 4 == 0 && ldy % 4 == 0 && lddx % 4 == 0 && (reinterpret_cast<uintptr_t>(dy) & 15) == 0 &&
                 (reinterpret_cast<uintptr_t>(dx) & 15) == 0,
             LX_ERR_UNSUPPORTED, "adapter: d and row strides must be multiples of 4 floats, rows 16-byte aligned");
  if (r == 8)
    return adapter_bwd_t<8>(dy, ldy, x, ldx, M, d, z, w_down, w_up, dh, dx, lddx, ws, scale, g_w_down, g_b_down, g_w_up,
                            g_b_up, stream);
  return adapter_bwd_t<16>(dy, ldy, x, ldx, M, d, z, w_down, w_up, dh, dx, lddx, ws, scale, g_w_down, g_b_down, g_w_up,
                           g_b_up, stream);
}

}  // extern "C"
