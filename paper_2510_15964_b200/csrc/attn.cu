// K3 — block-sparse attention walking the predicted per-(item, head) pool
// pattern (sf/block_sparse.py:47-137, sf/model.py:322-360, sf/autograd.py:127-162).
//
// Layout: q, k, v, o are the projection outputs [n_items*s, ld] (bf16), head h
// at columns [h*hd, (h+1)*hd). The pool pattern of (item, head) selects a
// precomputed tile table (the paper's offline pool, built once per (s,
// attn_blk)): CSR over 64-row query tiles and CSC over 64-key tiles, each
// entry carrying a 16-bit mask of its active 16x16 cells. Inactive tiles are
// never touched; inactive cells inside a touched tile are -inf (zero
// probability, zero gradient) exactly as the reference's -inf semantics.
//
// Forward: online softmax (flash style), saves lse (natural log) per row.
// Backward (deterministic, no float atomics): delta = rowsum(dO*O) (equal to
// the reference's rowsum(dP*P), sf/block_sparse.py:102-113); dK/dV per key
// tile over the CSC list; dQ per query tile over the CSR list.
//
// Math: warp-level bf16 mma.sync m16n8k16 with fp32 accumulation.
#include <vector>

#include "common.cuh"
#include "ptx.cuh"

namespace lx {

constexpr int kT = 64;  // tile edge (rows and keys)
constexpr float kLog2e = 1.4426950408889634f;

// ------------------------------------------------------------ warp MMA helpers
LX_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
LX_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
LX_DEV void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
LX_DEV void cp_async16(uint32_t saddr, const void* g, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(valid ? 16 : 0) : "memory");
}
LX_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
LX_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// tile [64 x HD] bf16 in smem with padded rows (HD + 8) -> conflict-free ldmatrix
template <int HD>
struct TileSmem {
  static constexpr int kStride = HD + 8;
  static constexpr int kElems = kT * kStride;
};

// async load of a 64-row tile (rows >= s zero-filled) by all 128 threads
template <int HD>
LX_DEV void load_tile(__nv_bfloat16* dst, const __nv_bfloat16* src, int ld, int row0, int s) {
  constexpr int kChunks = HD / 8;  // 16B chunks per row
  const uint32_t base = smem_u32(dst);
  for (int e = threadIdx.x; e < kT * kChunks; e += 128) {
    int r = e / kChunks, c = e % kChunks;
    bool ok = row0 + r < s;
    const __nv_bfloat16* g = src + (size_t)(ok ? row0 + r : 0) * ld + c * 8;
    cp_async16(base + (r * TileSmem<HD>::kStride + c * 8) * 2, g, ok);
  }
}

// A fragments (16 rows x HD) of rows [r0, r0+16) from a padded tile
template <int HD>
LX_DEV void load_a_frags(const __nv_bfloat16* tile, int r0, uint32_t (&f)[HD / 16][4]) {
  const int lane = threadIdx.x & 31;
  const uint32_t base = smem_u32(tile);
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk) {
    int row = r0 + (lane & 7) + ((lane >> 3) & 1) * 8;
    int col = kk * 16 + (lane >> 4) * 8;
    ldsm_x4(base + (row * TileSmem<HD>::kStride + col) * 2, f[kk][0], f[kk][1], f[kk][2], f[kk][3]);
  }
}

// acc[16 x 64] += A(16 x HD) * T^T where T is a [64 x HD] tile (B = N x K row-major)
template <int HD>
LX_DEV void mma_a_bt(float (&acc)[8][4], const uint32_t (&a)[HD / 16][4], const __nv_bfloat16* tile) {
  const int lane = threadIdx.x & 31;
  const uint32_t base = smem_u32(tile);
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
    for (int np = 0; np < 4; ++np) {
      int row = np * 16 + (lane & 7) + (lane >> 4) * 8;
      int col = kk * 16 + ((lane >> 3) & 1) * 8;
      uint32_t b0, b1, b2, b3;
      ldsm_x4(base + (row * TileSmem<HD>::kStride + col) * 2, b0, b1, b2, b3);
      mma16816(acc[2 * np], a[kk], b0, b1);
      mma16816(acc[2 * np + 1], a[kk], b2, b3);
    }
  }
}

// acc[16 x HD] += P(16 x 64, C-fragment registers) * T where T is [64 x HD] (K x N row-major)
template <int HD>
LX_DEV void mma_p_t(float (&acc)[HD / 8][4], const float (&p)[8][4], const __nv_bfloat16* tile) {
  const int lane = threadIdx.x & 31;
  const uint32_t base = smem_u32(tile);
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    uint32_t a[4] = {pack_bf16x2(p[2 * kk][0], p[2 * kk][1]), pack_bf16x2(p[2 * kk][2], p[2 * kk][3]),
                     pack_bf16x2(p[2 * kk + 1][0], p[2 * kk + 1][1]), pack_bf16x2(p[2 * kk + 1][2], p[2 * kk + 1][3])};
#pragma unroll
    for (int np = 0; np < HD / 16; ++np) {
      int row = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
      int col = np * 16 + (lane >> 4) * 8;
      uint32_t b0, b1, b2, b3;
      ldsm_x4_t(base + (row * TileSmem<HD>::kStride + col) * 2, b0, b1, b2, b3);
      mma16816(acc[2 * np], a, b0, b1);
      mma16816(acc[2 * np + 1], a, b2, b3);
    }
  }
}

// ------------------------------------------------------------ tile tables
// int32 layout: [0]=nt, [1]=n_pool, then per pattern p at base = 4 + p*per:
//   row_ptr[nt+1], csr_col[nt*nt], csr_mask[nt*nt], col_ptr[nt+1], csc_row[nt*nt], csc_mask[nt*nt]
__host__ __device__ __forceinline__ int table_per_pattern(int nt) { return 2 * (nt + 1) + 4 * nt * nt; }

struct TableView {
  const int32_t *row_ptr, *csr_col, *csr_mask, *col_ptr, *csc_row, *csc_mask;
};
LX_DEV TableView table_view(const int32_t* t, int p) {
  const int nt = t[0];
  const int32_t* b = t + 4 + (size_t)p * table_per_pattern(nt);
  TableView v;
  v.row_ptr = b;
  v.csr_col = b + nt + 1;
  v.csr_mask = v.csr_col + nt * nt;
  v.col_ptr = v.csr_mask + nt * nt;
  v.csc_row = v.col_ptr + nt + 1;
  v.csc_mask = v.csc_row + nt * nt;
  return v;
}

// ------------------------------------------------------------ forward
template <int HD>
__global__ void __launch_bounds__(128) bsattn_fwd_kernel(const __nv_bfloat16* __restrict__ q,
                                                         const __nv_bfloat16* __restrict__ k,
                                                         const __nv_bfloat16* __restrict__ v, int ld, int s, int H,
                                                         const int32_t* __restrict__ pidx, int item_stride,
                                                         const int32_t* __restrict__ tables, float scale_log2,
                                                         __nv_bfloat16* __restrict__ o, int ldo, float* __restrict__ lse) {
  extern __shared__ __align__(16) uint8_t sm[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(sm);
  __nv_bfloat16* sK = sQ + TileSmem<HD>::kElems;  // 2 buffers
  __nv_bfloat16* sV = sK + 2 * TileSmem<HD>::kElems;
  const int qt = blockIdx.x, h = blockIdx.y, item = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TableView tv = table_view(tables, __ldg(pidx + item * item_stride + h));
  const int e0 = tv.row_ptr[qt], e1 = tv.row_ptr[qt + 1];
  const size_t item_row = (size_t)item * s;
  const __nv_bfloat16* qb = q + item_row * ld + h * HD;
  const __nv_bfloat16* kb = k + item_row * ld + h * HD;
  const __nv_bfloat16* vb = v + item_row * ld + h * HD;

  load_tile<HD>(sQ, qb, ld, qt * kT, s);
  if (e0 < e1) {
    int j = tv.csr_col[e0];
    load_tile<HD>(sK, kb, ld, j * kT, s);
    load_tile<HD>(sV, vb, ld, j * kT, s);
  }
  cp_async_commit();

  uint32_t qf[HD / 16][4];
  float oacc[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};

  for (int e = e0; e < e1; ++e) {
    const int buf = (e - e0) & 1;
    if (e + 1 < e1) {
      int jn = tv.csr_col[e + 1];
      load_tile<HD>(sK + (buf ^ 1) * TileSmem<HD>::kElems, kb, ld, jn * kT, s);
      load_tile<HD>(sV + (buf ^ 1) * TileSmem<HD>::kElems, vb, ld, jn * kT, s);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (e == e0) load_a_frags<HD>(sQ, warp * 16, qf);
    const uint32_t mask = (uint32_t)tv.csr_mask[e];
    float sacc[8][4];
#pragma unroll
    for (int t = 0; t < 8; ++t) sacc[t][0] = sacc[t][1] = sacc[t][2] = sacc[t][3] = 0.f;
    mma_a_bt<HD>(sacc, qf, sK + buf * TileSmem<HD>::kElems);
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const bool on = (mask >> (warp * 4 + (t >> 1))) & 1u;
#pragma unroll
      for (int i = 0; i < 4; ++i) sacc[t][i] = on ? sacc[t][i] * scale_log2 : -INFINITY;
      mx[0] = fmaxf(mx[0], fmaxf(sacc[t][0], sacc[t][1]));
      mx[1] = fmaxf(mx[1], fmaxf(sacc[t][2], sacc[t][3]));
    }
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      mx[rr] = fmaxf(mx[rr], __shfl_xor_sync(0xffffffffu, mx[rr], 1));
      mx[rr] = fmaxf(mx[rr], __shfl_xor_sync(0xffffffffu, mx[rr], 2));
    }
    float alpha[2], use[2], rsum[2] = {0.f, 0.f};
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      float mn = fmaxf(m_r[rr], mx[rr]);
      use[rr] = mn == -INFINITY ? 0.f : mn;
      alpha[rr] = exp2f(m_r[rr] - use[rr]);
      m_r[rr] = mn;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      sacc[t][0] = exp2f(sacc[t][0] - use[0]);
      sacc[t][1] = exp2f(sacc[t][1] - use[0]);
      sacc[t][2] = exp2f(sacc[t][2] - use[1]);
      sacc[t][3] = exp2f(sacc[t][3] - use[1]);
      rsum[0] += sacc[t][0] + sacc[t][1];
      rsum[1] += sacc[t][2] + sacc[t][3];
    }
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      rsum[rr] += __shfl_xor_sync(0xffffffffu, rsum[rr], 1);
      rsum[rr] += __shfl_xor_sync(0xffffffffu, rsum[rr], 2);
      l_r[rr] = l_r[rr] * alpha[rr] + rsum[rr];
    }
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      oacc[i][0] *= alpha[0];
      oacc[i][1] *= alpha[0];
      oacc[i][2] *= alpha[1];
      oacc[i][3] *= alpha[1];
    }
    mma_p_t<HD>(oacc, sacc, sV + buf * TileSmem<HD>::kElems);
    __syncthreads();
  }
  cp_async_wait<0>();
  // epilogue
  const int r_lo = qt * kT + warp * 16 + (lane >> 2);
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int row = r_lo + rr * 8;
    if (row >= s) continue;
    const float inv = l_r[rr] > 0.f ? 1.f / l_r[rr] : 0.f;
    __nv_bfloat16* orow = o + (item_row + row) * ldo + h * HD;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      int col = i * 8 + (lane & 3) * 2;
      *reinterpret_cast<uint32_t*>(orow + col) = pack_bf16x2(oacc[i][2 * rr] * inv, oacc[i][2 * rr + 1] * inv);
    }
    if ((lane & 3) == 0)
      lse[((size_t)item * H + h) * s + row] = (m_r[rr] + log2f(l_r[rr])) * 0.6931471805599453f;
  }
}

// ------------------------------------------------------------ backward
// delta[item, h, row] = sum_c dO[row, c] * O[row, c]
__global__ void bsattn_delta_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ d_o, int ld,
                                    int n_rows_total, int s, int H, int hd, float* __restrict__ delta) {
  const int warp_g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp_g >= n_rows_total * H) return;
  const int row = warp_g / H, h = warp_g % H;
  const __nv_bfloat16* a = o + (size_t)row * ld + h * hd;
  const __nv_bfloat16* b = d_o + (size_t)row * ld + h * hd;
  float acc = 0.f;
  for (int c = lane * 2; c < hd; c += 64) {
    __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162*>(a + c);
    __nv_bfloat162 y = *reinterpret_cast<const __nv_bfloat162*>(b + c);
    acc += __bfloat162float(x.x) * __bfloat162float(y.x) + __bfloat162float(x.y) * __bfloat162float(y.y);
  }
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) {
    int item = row / s, t = row % s;
    delta[((size_t)item * H + h) * s + t] = acc;
  }
}

// dK, dV for one 64-key tile, walking the CSC list (query tiles that attend to it)
template <int HD>
__global__ void __launch_bounds__(128) bsattn_dkdv_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v,
    const __nv_bfloat16* __restrict__ d_o, int ld, int ld_o, int s, int H, const int32_t* __restrict__ pidx, int item_stride,
    const int32_t* __restrict__ tables, float scale, float scale_log2, const float* __restrict__ lse,
    const float* __restrict__ delta, __nv_bfloat16* __restrict__ dk, __nv_bfloat16* __restrict__ dv) {
  extern __shared__ __align__(16) uint8_t sm[];
  constexpr int E = TileSmem<HD>::kElems;
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(sm);
  __nv_bfloat16* sV = sK + E;
  __nv_bfloat16* sQ = sV + E;       // 2 buffers
  __nv_bfloat16* sdO = sQ + 2 * E;  // 2 buffers
  float* sL = reinterpret_cast<float*>(sdO + 2 * E);  // 2 x 64 lse*log2e
  float* sD = sL + 2 * kT;                             // 2 x 64 delta
  const int kt = blockIdx.x, h = blockIdx.y, item = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TableView tv = table_view(tables, __ldg(pidx + item * item_stride + h));
  const int e0 = tv.col_ptr[kt], e1 = tv.col_ptr[kt + 1];
  const size_t item_row = (size_t)item * s;
  const size_t off = item_row * ld + h * HD;
  const float* lse_b = lse + ((size_t)item * H + h) * s;
  const float* del_b = delta + ((size_t)item * H + h) * s;

  load_tile<HD>(sK, k + off, ld, kt * kT, s);
  load_tile<HD>(sV, v + off, ld, kt * kT, s);
  auto load_q = [&](int e, int buf) {
    int i = tv.csc_row[e];
    load_tile<HD>(sQ + buf * E, q + off, ld, i * kT, s);
    load_tile<HD>(sdO + buf * E, d_o + item_row * ld_o + h * HD, ld_o, i * kT, s);
    if (threadIdx.x < kT) {
      int row = i * kT + threadIdx.x;
      sL[buf * kT + threadIdx.x] = row < s ? lse_b[row] * kLog2e : 0.f;
      sD[buf * kT + threadIdx.x] = row < s ? del_b[row] : 0.f;
    }
  };
  if (e0 < e1) load_q(e0, 0);
  cp_async_commit();

  uint32_t kf[HD / 16][4], vf[HD / 16][4];
  float dkacc[HD / 8][4], dvacc[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) dkacc[i][c] = dvacc[i][c] = 0.f;

  for (int e = e0; e < e1; ++e) {
    const int buf = (e - e0) & 1;
    if (e + 1 < e1) load_q(e + 1, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (e == e0) {
      load_a_frags<HD>(sK, warp * 16, kf);
      load_a_frags<HD>(sV, warp * 16, vf);
    }
    const uint32_t mask = (uint32_t)tv.csc_mask[e];
    const __nv_bfloat16* Qt = sQ + buf * E;
    const __nv_bfloat16* dOt = sdO + buf * E;
    float st[8][4], dpt[8][4];
#pragma unroll
    for (int t = 0; t < 8; ++t)
#pragma unroll
      for (int c = 0; c < 4; ++c) st[t][c] = dpt[t][c] = 0.f;
    mma_a_bt<HD>(st, kf, Qt);    // S^T[key, q]
    mma_a_bt<HD>(dpt, vf, dOt);  // dP^T[key, q]
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const bool on = (mask >> ((t >> 1) * 4 + warp)) & 1u;
      const int qc = t * 8 + (lane & 3) * 2;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int qi = qc + (c & 1);
        float p = on ? exp2f(st[t][c] * scale_log2 - sL[buf * kT + qi]) : 0.f;
        st[t][c] = p;                                    // P^T
        dpt[t][c] = p * (dpt[t][c] - sD[buf * kT + qi]);  // dS^T
      }
    }
    mma_p_t<HD>(dvacc, st, dOt);
    mma_p_t<HD>(dkacc, dpt, Qt);
    __syncthreads();
  }
  cp_async_wait<0>();
  const int r_lo = kt * kT + warp * 16 + (lane >> 2);
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int row = r_lo + rr * 8;
    if (row >= s) continue;
    __nv_bfloat16* dkr = dk + (item_row + row) * ld + h * HD;
    __nv_bfloat16* dvr = dv + (item_row + row) * ld + h * HD;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      int col = i * 8 + (lane & 3) * 2;
      *reinterpret_cast<uint32_t*>(dkr + col) = pack_bf16x2(dkacc[i][2 * rr] * scale, dkacc[i][2 * rr + 1] * scale);
      *reinterpret_cast<uint32_t*>(dvr + col) = pack_bf16x2(dvacc[i][2 * rr], dvacc[i][2 * rr + 1]);
    }
  }
}

// dQ for one 64-row query tile, walking the CSR list
template <int HD>
__global__ void __launch_bounds__(128) bsattn_dq_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v,
    const __nv_bfloat16* __restrict__ d_o, int ld, int ld_o, int s, int H, const int32_t* __restrict__ pidx, int item_stride,
    const int32_t* __restrict__ tables, float scale, float scale_log2, const float* __restrict__ lse,
    const float* __restrict__ delta, __nv_bfloat16* __restrict__ dq) {
  extern __shared__ __align__(16) uint8_t sm[];
  constexpr int E = TileSmem<HD>::kElems;
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(sm);
  __nv_bfloat16* sdO = sQ + E;
  __nv_bfloat16* sK = sdO + E;      // 2 buffers
  __nv_bfloat16* sV = sK + 2 * E;   // 2 buffers
  const int qt = blockIdx.x, h = blockIdx.y, item = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TableView tv = table_view(tables, __ldg(pidx + item * item_stride + h));
  const int e0 = tv.row_ptr[qt], e1 = tv.row_ptr[qt + 1];
  const size_t item_row = (size_t)item * s;
  const size_t off = item_row * ld + h * HD;
  const float* lse_b = lse + ((size_t)item * H + h) * s;
  const float* del_b = delta + ((size_t)item * H + h) * s;

  load_tile<HD>(sQ, q + off, ld, qt * kT, s);
  load_tile<HD>(sdO, d_o + item_row * ld_o + h * HD, ld_o, qt * kT, s);
  if (e0 < e1) {
    int j = tv.csr_col[e0];
    load_tile<HD>(sK, k + off, ld, j * kT, s);
    load_tile<HD>(sV, v + off, ld, j * kT, s);
  }
  cp_async_commit();
  const int r_lo = qt * kT + warp * 16 + (lane >> 2);
  float lrow[2], drow[2];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    int row = r_lo + rr * 8;
    lrow[rr] = row < s ? lse_b[row] * kLog2e : 0.f;
    drow[rr] = row < s ? del_b[row] : 0.f;
  }
  uint32_t qf[HD / 16][4], dof[HD / 16][4];
  float dqacc[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) dqacc[i][0] = dqacc[i][1] = dqacc[i][2] = dqacc[i][3] = 0.f;

  for (int e = e0; e < e1; ++e) {
    const int buf = (e - e0) & 1;
    if (e + 1 < e1) {
      int jn = tv.csr_col[e + 1];
      load_tile<HD>(sK + (buf ^ 1) * E, k + off, ld, jn * kT, s);
      load_tile<HD>(sV + (buf ^ 1) * E, v + off, ld, jn * kT, s);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (e == e0) {
      load_a_frags<HD>(sQ, warp * 16, qf);
      load_a_frags<HD>(sdO, warp * 16, dof);
    }
    const uint32_t mask = (uint32_t)tv.csr_mask[e];
    float sc[8][4], dp[8][4];
#pragma unroll
    for (int t = 0; t < 8; ++t)
#pragma unroll
      for (int c = 0; c < 4; ++c) sc[t][c] = dp[t][c] = 0.f;
    mma_a_bt<HD>(sc, qf, sK + buf * E);
    mma_a_bt<HD>(dp, dof, sV + buf * E);
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const bool on = (mask >> (warp * 4 + (t >> 1))) & 1u;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int rr = c >> 1;
        float p = on ? exp2f(sc[t][c] * scale_log2 - lrow[rr]) : 0.f;
        sc[t][c] = p * (dp[t][c] - drow[rr]);  // dS
      }
    }
    mma_p_t<HD>(dqacc, sc, sK + buf * E);
    __syncthreads();
  }
  cp_async_wait<0>();
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int row = r_lo + rr * 8;
    if (row >= s) continue;
    __nv_bfloat16* dqr = dq + (item_row + row) * ld + h * HD;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      int col = i * 8 + (lane & 3) * 2;
      *reinterpret_cast<uint32_t*>(dqr + col) = pack_bf16x2(dqacc[i][2 * rr] * scale, dqacc[i][2 * rr + 1] * scale);
    }
  }
}

// host-side pool membership (sf/patterns.py:63-85), kinds as in mask_build.cu
static bool host_member(int kind, int p, int i, int j) {
  int dd = i - j;
  switch (kind) {
    case 0: return dd == 0;
    case 1: return dd <= p && dd >= -p;
    case 2: return dd >= 0 && dd <= p;
    case 3: return i < p || j < p || dd == 0;
    case 4: return ((dd % p) + p) % p == 0;
    default: return true;
  }
}

template <int HD>
static int launch_fwd(const uint16_t* q, const uint16_t* k, const uint16_t* v, int ld, int n_items, int s, int H,
                      const int32_t* pidx, int item_stride, const int32_t* tables, float scale, uint16_t* o, int ldo,
                      float* lse, cudaStream_t st) {
  const int smem = 5 * TileSmem<HD>::kElems * 2;
  auto kern = bsattn_fwd_kernel<HD>;
  static cudaError_t attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  LX_CHECK_CUDA(attr);
  dim3 grid((s + kT - 1) / kT, H, n_items);
  kern<<<grid, 128, smem, st>>>(reinterpret_cast<const __nv_bfloat16*>(q), reinterpret_cast<const __nv_bfloat16*>(k),
                                reinterpret_cast<const __nv_bfloat16*>(v), ld, s, H, pidx, item_stride, tables,
                                scale * kLog2e, reinterpret_cast<__nv_bfloat16*>(o), ldo, lse);
  return launch_check("bsattn_fwd");
}

template <int HD>
static int launch_bwd(const uint16_t* q, const uint16_t* k, const uint16_t* v, const uint16_t* o, const uint16_t* d_o,
                      int ld, int ld_o, int n_items, int s, int H, const int32_t* pidx, int item_stride, const int32_t* tables,
                      float scale, const float* lse, float* delta, uint16_t* dq, uint16_t* dk, uint16_t* dv,
                      cudaStream_t st) {
  using bf = const __nv_bfloat16*;
  const int rows = n_items * s;
  bsattn_delta_kernel<<<(rows * H * 32 + 255) / 256, 256, 0, st>>>(reinterpret_cast<bf>(o), reinterpret_cast<bf>(d_o),
                                                                  ld_o, rows, s, H, HD, delta);
  int rc = launch_check("bsattn_delta");
  if (rc) return rc;
  constexpr int E = TileSmem<HD>::kElems;
  const int smem_kv = 6 * E * 2 + 4 * kT * 4;
  const int smem_q = 6 * E * 2;
  static cudaError_t a1 = cudaFuncSetAttribute(bsattn_dkdv_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv);
  static cudaError_t a2 = cudaFuncSetAttribute(bsattn_dq_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_q);
  LX_CHECK_CUDA(a1);
  LX_CHECK_CUDA(a2);
  dim3 grid((s + kT - 1) / kT, H, n_items);
  bsattn_dkdv_kernel<HD><<<grid, 128, smem_kv, st>>>(reinterpret_cast<bf>(q), reinterpret_cast<bf>(k),
                                                     reinterpret_cast<bf>(v), reinterpret_cast<bf>(d_o), ld, ld_o, s, H, pidx,
                                                     item_stride, tables, scale, scale * kLog2e, lse, delta,
                                                     reinterpret_cast<__nv_bfloat16*>(dk),
                                                     reinterpret_cast<__nv_bfloat16*>(dv));
  if ((rc = launch_check("bsattn_dkdv"))) return rc;
  bsattn_dq_kernel<HD><<<grid, 128, smem_q, st>>>(reinterpret_cast<bf>(q), reinterpret_cast<bf>(k),
                                                  reinterpret_cast<bf>(v), reinterpret_cast<bf>(d_o), ld, ld_o, s, H, pidx,
                                                  item_stride, tables, scale, scale * kLog2e, lse, delta,
                                                  reinterpret_cast<__nv_bfloat16*>(dq));
  return launch_check("bsattn_dq");
}

}  // namespace lx

using namespace lx;

extern "C" {

int lx_attn_tables_size(int n_pool, int s, int attn_blk, int* n_ints) {
  const int nt = (s + kT - 1) / kT;
  *n_ints = 4 + n_pool * table_per_pattern(nt);
  return 0;
}

int lx_attn_tables(const int32_t* pool_kind, const int32_t* pool_param, int n_pool, int s, int attn_blk, int32_t* out,
                   int out_ints) {
  LX_REQUIRE(attn_blk >= 16 && attn_blk % 16 == 0, LX_ERR_UNSUPPORTED,
             "attn_blk %d unsupported on the sm_100a path (multiple of 16)", attn_blk);
  LX_REQUIRE(s % attn_blk == 0, LX_ERR_LAYOUT, "sequence length %d != n_b*blk", s);
  const int nt = (s + kT - 1) / kT;
  int need = 0;
  lx_attn_tables_size(n_pool, s, attn_blk, &need);
  LX_REQUIRE(out_ints >= need, LX_ERR_SHAPE, "attn tables: buffer too small");
  memset(out, 0, sizeof(int32_t) * need);
  out[0] = nt;
  out[1] = n_pool;
  out[2] = s;
  out[3] = attn_blk;
  const int ncell = s / 16;
  std::vector<int> tmask(nt * nt);
  for (int p = 0; p < n_pool; ++p) {
    std::fill(tmask.begin(), tmask.end(), 0);
    for (int ci = 0; ci < ncell; ++ci)
      for (int cj = 0; cj < ncell; ++cj)
        if (host_member(pool_kind[p], pool_param[p], ci * 16 / attn_blk, cj * 16 / attn_blk))
          tmask[(ci / 4) * nt + cj / 4] |= 1 << ((ci % 4) * 4 + cj % 4);
    int32_t* b = out + 4 + (size_t)p * table_per_pattern(nt);
    int32_t *row_ptr = b, *csr_col = b + nt + 1, *csr_mask = csr_col + nt * nt;
    int32_t *col_ptr = csr_mask + nt * nt, *csc_row = col_ptr + nt + 1, *csc_mask = csc_row + nt * nt;
    int n = 0;
    for (int i = 0; i < nt; ++i) {
      row_ptr[i] = n;
      for (int j = 0; j < nt; ++j)
        if (tmask[i * nt + j]) { csr_col[n] = j; csr_mask[n] = tmask[i * nt + j]; ++n; }
    }
    row_ptr[nt] = n;
    n = 0;
    for (int j = 0; j < nt; ++j) {
      col_ptr[j] = n;
      for (int i = 0; i < nt; ++i)
        if (tmask[i * nt + j]) { csc_row[n] = i; csc_mask[n] = tmask[i * nt + j]; ++n; }
    }
    col_ptr[nt] = n;
    // every block-row must be covered (sf/block_sparse.py:91-92): pool patterns keep the diagonal
    for (int i = 0; i < nt; ++i)
      LX_REQUIRE(row_ptr[i + 1] > row_ptr[i], LX_ERR_LAYOUT, "pattern %d leaves query tile %d uncovered", p, i);
  }
  return LX_OK;
}

int lx_bsattn_fwd(const uint16_t* q, const uint16_t* k, const uint16_t* v, int ld, int n_items, int s, int H, int hd,
                  const int32_t* pattern_idx, int item_stride, const int32_t* tables, int n_pool, float scale,
                  uint16_t* o, int ldo, float* lse, lx_stream_t stream) {
  LX_REQUIRE(ld % 8 == 0 && ldo % 8 == 0, LX_ERR_SHAPE, "attention: row strides must be multiples of 8");
  LX_REQUIRE(n_items >= 1 && n_items < 65536 && H >= 1 && H < 65536, LX_ERR_SHAPE, "attention: bad grid");
  switch (hd) {
    case 32: return launch_fwd<32>(q, k, v, ld, n_items, s, H, pattern_idx, item_stride, tables, scale, o, ldo, lse, stream);
    case 64: return launch_fwd<64>(q, k, v, ld, n_items, s, H, pattern_idx, item_stride, tables, scale, o, ldo, lse, stream);
    case 128: return launch_fwd<128>(q, k, v, ld, n_items, s, H, pattern_idx, item_stride, tables, scale, o, ldo, lse, stream);
    default: LX_REQUIRE(false, LX_ERR_UNSUPPORTED, "head_dim %d unsupported (32, 64, 128)", hd);
  }
}

int lx_bsattn_bwd(const uint16_t* q, const uint16_t* k, const uint16_t* v, const uint16_t* o, const uint16_t* d_o, int ld,
                  int ld_o, int n_items, int s, int H, int hd, const int32_t* pattern_idx, int item_stride, const int32_t* tables,
                  int n_pool, float scale, const float* lse, float* delta_ws, uint16_t* dq, uint16_t* dk, uint16_t* dv,
                  lx_stream_t stream) {
  LX_REQUIRE(ld % 8 == 0 && ld_o % 8 == 0, LX_ERR_SHAPE, "attention: row strides must be multiples of 8");
  switch (hd) {
    case 32: return launch_bwd<32>(q, k, v, o, d_o, ld, ld_o, n_items, s, H, pattern_idx, item_stride, tables, scale, lse, delta_ws, dq, dk, dv, stream);
    case 64: return launch_bwd<64>(q, k, v, o, d_o, ld, ld_o, n_items, s, H, pattern_idx, item_stride, tables, scale, lse, delta_ws, dq, dk, dv, stream);
    case 128: return launch_bwd<128>(q, k, v, o, d_o, ld, ld_o, n_items, s, H, pattern_idx, item_stride, tables, scale, lse, delta_ws, dq, dk, dv, stream);
    default: LX_REQUIRE(false, LX_ERR_UNSUPPORTED, "head_dim %d unsupported (32, 64, 128)", hd);
  }
}

}  // extern "C"
