// Batch-norm / ReLU / residual-add / pooling kernels of the conv-net training
// step, NHWC activations (bf16, or fp32 in the fp32
// parity mode) viewed as [rows, C].
//
// Memory-bound: every thread moves 8 channels (16 B of bf16) per access with
// coalesced row-major access, grid-stride loops over grids sized in multiples
// of the 148 SMs, and 32-bit index math with multiply-shift division.
// Per-channel reductions are deterministic two-level reductions (fixed row
// chunks -> fp32 partials -> fixed-order double finalize, one warp per
// channel) so a step is bitwise reproducible whatever the swap schedule.
//
// Contract (oracle/numerics.py): x̂ = (y−μ)·rstd with batch statistics and
// biased variance, eps = 1e-5; out = rnd(relu(γx̂ + β + res)); backward
// dz = g·[out>0], dβ = Σdz, dγ = Σdz·x̂, dy = γ·rstd·(dz − dβ/n − x̂·dγ/n).
// Algorithmic bytes per launch = one read of every input + one write of every
// output (roofline: HBM).
#include "common.cuh"

namespace oc {

namespace {

constexpr float kEps = 1e-5f;
constexpr int kStatBlocks = 148 * 4;  // row chunks of the two-level reductions

inline int stat_blocks(int64_t rows) { return (int)std::min<int64_t>(kStatBlocks, std::max<int64_t>(1, rows / 64)); }

// ---------------------------------------------------------------- statistics
// Partial Σy, Σy² over a contiguous row chunk per block.  Thread t covers the
// 8 channels starting at (t % (C/8))·8 of every (256/(C/8))-th row.
template <typename T>
__global__ void __launch_bounds__(256) stats_partial(int64_t rows, int C, const T* __restrict__ y,
                                                     float* __restrict__ part) {
  const int g = C / 8;
  const int tpr = 256 / g;
  const int t = threadIdx.x;
  const int cg = t % g, rr = t / g;
  const int64_t chunk = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * chunk, r1 = min(rows, r0 + chunk);
  float s[8] = {}, q[8] = {};
  if (rr < tpr)
#pragma unroll 2
    for (int64_t r = r0 + rr; r < r1; r += tpr) {
      V8 x = ld8(y + r * C + cg * 8);
#pragma unroll
      for (int i = 0; i < 8; ++i) { s[i] += x.v[i]; q[i] = fmaf(x.v[i], x.v[i], q[i]); }
    }
  extern __shared__ float sm[];        // [256][16]
#pragma unroll
  for (int i = 0; i < 8; ++i) { sm[t * 16 + i] = s[i]; sm[t * 16 + 8 + i] = q[i]; }
  __syncthreads();
  for (int c = t; c < C; c += 256) {   // fixed-order combine of the threads sharing a channel group
    const int grp = c / 8, lane = c % 8;
    float as = 0.f, aq = 0.f;
    for (int k = 0; k < tpr; ++k) {
      as += sm[(k * g + grp) * 16 + lane];
      aq += sm[(k * g + grp) * 16 + 8 + lane];
    }
    part[(int64_t)blockIdx.x * 2 * C + c] = as;
    part[(int64_t)blockIdx.x * 2 * C + C + c] = aq;
  }
}

// one warp per channel: lane-strided partial sums in double, then a fixed xor tree
__device__ __forceinline__ void chunk_sums(int nblk, int C, int c, const float* __restrict__ part, double& s,
                                           double& q) {
  const int lane = threadIdx.x & 31;
  s = 0;
  q = 0;
  for (int b = lane; b < nblk; b += 32) {
    s += part[(int64_t)b * 2 * C + c];
    q += part[(int64_t)b * 2 * C + C + c];
  }
  s = warp_sum(s);
  q = warp_sum(q);
}

// stat[0][c] = μ, stat[1][c] = rstd
__global__ void stats_finalize(int nblk, int64_t rows, int C, const float* __restrict__ part, float* __restrict__ stat) {
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= C) return;
  double s, q;
  chunk_sums(nblk, C, c, part, s, q);
  if ((threadIdx.x & 31) != 0) return;
  const double mu = s / rows;
  double var = q / rows - mu * mu;
  if (var < 0) var = 0;
  stat[c] = (float)mu;
  stat[C + c] = (float)(1.0 / sqrt(var + (double)kEps));
}

template <typename T>
Status batch_stats(OpArgs& a, int64_t rows, int C, const T* y, float* stat) {
  if (C % 8 || C > 2048) return Status::make(OC_E_UNSUPPORTED, "bn: C must be a multiple of 8 and <= 2048");
  const int nblk = stat_blocks(rows);
  if (a.ws_bytes < (size_t)nblk * 2 * C * 4) return Status::make(OC_E_INVARIANT, "bn: workspace too small");
  stats_partial<T><<<nblk, 256, 256 * 16 * 4, a.stream>>>(rows, C, y, (float*)a.ws);
  OC_LAUNCH_CHECK(a);
  stats_finalize<<<(C + 7) / 8, 256, 0, a.stream>>>(nblk, rows, C, (const float*)a.ws, stat);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

size_t bn_ws(const JVal& at) {
  const int64_t rows = at.geti("rows") ? at.geti("rows") : at.geti("N") * at.geti("H") * at.geti("W");
  return (size_t)stat_blocks(rows) * 2 * at.geti("C") * 4;
}

// ---------------------------------------------------------------- forward
// Elementwise kernels map thread t of a block to channel group t % (C/8) of
// row t / (C/8), blocks to consecutive row groups: a block touches one
// contiguous span, and each thread's 8 channels — hence its per-channel
// parameters, held in registers — never change.
inline int rowgroup_blocks(int64_t rows, int C) {
  const int tpr = 256 / (C / 8);
  return (int)std::max<int64_t>(1, std::min<int64_t>((rows + tpr - 1) / tpr, 148 * 16));
}

template <typename T>
__global__ void __launch_bounds__(256) bn_apply_fwd(int64_t rows, int C, const T* __restrict__ y,
                                                    const float* __restrict__ stat, const float* __restrict__ gamma,
                                                    const float* __restrict__ beta, const T* __restrict__ res,
                                                    T* __restrict__ out, int relu) {
  const int gC = C / 8, tpr = 256 / gC;
  const int cg = threadIdx.x % gC, rr = threadIdx.x / gC;
  if (rr >= tpr) return;
  float mu[8], rs[8], gm[8], bt[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = cg * 8 + k;
    mu[k] = stat[c];
    rs[k] = stat[C + c];
    gm[k] = gamma[c];
    bt[k] = beta[c];
  }
  const int64_t stride = (int64_t)gridDim.x * tpr;
#pragma unroll 2
  for (int64_t r = (int64_t)blockIdx.x * tpr + rr; r < rows; r += stride) {
    const int64_t o = r * C + cg * 8;
    V8 x = ld8(y + o);
    V8 rv;
    if (res) rv = ld8(res + o);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float z = fmaf(gm[k], (x.v[k] - mu[k]) * rs[k], bt[k]);
      if (res) z += rv.v[k];
      if (relu) z = fmaxf(z, 0.f);
      x.v[k] = z;
    }
    st8(out + o, x);
  }
}

enum { BF_Y, BF_STAT, BF_GAMMA, BF_BETA, BF_RES, BF_OUT };
template <typename T>
Status bn_fwd_t(OpArgs& a) {
  const int64_t rows = A(a, "rows");
  const int C = (int)A(a, "C");
  auto y = (const T*)a.p(BF_Y);
  // attrs.stat_in: the producing conv already wrote μ, rstd (fused statistics epilogue)
  if (!Ab(a, "stat_in")) OC_TRY(batch_stats<T>(a, rows, C, y, (float*)a.p(BF_STAT)));
  bn_apply_fwd<T><<<rowgroup_blocks(rows, C), 256, 0, a.stream>>>(rows, C, y, (const float*)a.p(BF_STAT),
                                                                  (const float*)a.p(BF_GAMMA),
                                                                  (const float*)a.p(BF_BETA), (const T*)a.p(BF_RES),
                                                                  (T*)a.p(BF_OUT), Ab(a, "relu") ? 1 : 0);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

// ---------------------------------------------------------------- backward
// ReLU mask of the BN output: from the stored output when there is one
// (residual blocks), else recomputed from y: relu'(γx̂ + β) (the BN-ReLU output
// is then not needed by the backward, shrinking its working set)
// MASK: 0 none, 1 from the stored output, 2 recomputed from y (as bnb_apply)
template <typename T, int MASK>
__global__ void __launch_bounds__(256) bnb_partial(int64_t rows, int C, const T* __restrict__ g,
                                                   const T* __restrict__ out, const T* __restrict__ y,
                                                   const float* __restrict__ stat, const float* __restrict__ gamma,
                                                   const float* __restrict__ beta, float* __restrict__ part) {
  const int gC = C / 8, tpr = 256 / gC;
  const int t = threadIdx.x, cg = t % gC, rr = t / gC;
  const int64_t chunk = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * chunk, r1 = min(rows, r0 + chunk);
  float s[8] = {}, q[8] = {};
  float mu[8], rs[8], gm[8], bt[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    mu[i] = stat[cg * 8 + i];
    rs[i] = stat[C + cg * 8 + i];
    gm[i] = gamma[cg * 8 + i];
    bt[i] = MASK == 2 ? beta[cg * 8 + i] : 0.f;
  }
  if (rr < tpr)
#pragma unroll 2
    for (int64_t r = r0 + rr; r < r1; r += tpr) {
      const int64_t o = r * C + cg * 8;
      V8 gv = ld8(g + o), yv = ld8(y + o);
      V8 ov;
      if (MASK == 1) ov = ld8(out + o);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float xh = (yv.v[i] - mu[i]) * rs[i];
        const bool on = MASK == 0 || (MASK == 1 ? ov.v[i] > 0.f : fmaf(gm[i], xh, bt[i]) > 0.f);
        const float dz = on ? gv.v[i] : 0.f;
        s[i] += dz;
        q[i] = fmaf(dz, xh, q[i]);
      }
    }
  extern __shared__ float sm[];
#pragma unroll
  for (int i = 0; i < 8; ++i) { sm[t * 16 + i] = s[i]; sm[t * 16 + 8 + i] = q[i]; }
  __syncthreads();
  for (int c = t; c < C; c += 256) {
    const int grp = c / 8, lane = c % 8;
    float as = 0.f, aq = 0.f;
    for (int k = 0; k < tpr; ++k) {
      as += sm[(k * gC + grp) * 16 + lane];
      aq += sm[(k * gC + grp) * 16 + 8 + lane];
    }
    part[(int64_t)blockIdx.x * 2 * C + c] = as;
    part[(int64_t)blockIdx.x * 2 * C + C + c] = aq;
  }
}

// dβ = Σdz, dγ = Σdz·x̂
__global__ void bnb_finalize(int nblk, int C, const float* __restrict__ part, float* __restrict__ dgamma,
                             float* __restrict__ dbeta) {
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= C) return;
  double s, q;
  chunk_sums(nblk, C, c, part, s, q);
  if ((threadIdx.x & 31) != 0) return;
  dbeta[c] = (float)s;
  dgamma[c] = (float)q;
}

enum { BB_G, BB_OUT, BB_Y, BB_STAT, BB_GAMMA, BB_DGAMMA, BB_DBETA, BB_ACC, BB_BETA };
template <typename T>
Status bn_bwd_reduce_t(OpArgs& a) {
  const int64_t rows = A(a, "rows");
  const int C = (int)A(a, "C");
  const int nblk = stat_blocks(rows);
  if (a.ws_bytes < (size_t)nblk * 2 * C * 4) return Status::make(OC_E_INVARIANT, "bn_bwd: workspace too small");
  if (Ab(a, "relu") && !a.p(BB_OUT) && !a.p(BB_BETA))
    return Status::make(OC_E_INVALID, "bn_bwd: ReLU mask needs the output or beta");
  const int mask = !Ab(a, "relu") ? 0 : (a.p(BB_OUT) ? 1 : 2);
  auto kp = mask == 0 ? bnb_partial<T, 0> : (mask == 1 ? bnb_partial<T, 1> : bnb_partial<T, 2>);
  kp<<<nblk, 256, 256 * 16 * 4, a.stream>>>(rows, C, (const T*)a.p(BB_G), (const T*)a.p(BB_OUT), (const T*)a.p(BB_Y),
                                            (const float*)a.p(BB_STAT), (const float*)a.p(BB_GAMMA),
                                            (const float*)a.p(BB_BETA), (float*)a.ws);
  OC_LAUNCH_CHECK(a);
  bnb_finalize<<<(C + 7) / 8, 256, 0, a.stream>>>(nblk, C, (const float*)a.ws, (float*)a.p(BB_DGAMMA),
                                                  (float*)a.p(BB_DBETA));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

// dy = γ·rstd·(dz − dβ/n − x̂·dγ/n), written over y — or, when the BN input
// already holds a gradient contribution (acc), accumulated into it as
// rnd(G + dy); dz written over g (residual branch)
// Variants by (mask source, residual dz output, accumulation) so each keeps
// only the per-channel parameters it reads live in registers.
// MASK: 0 none, 1 from the stored output, 2 recomputed from y (γx̂ + β > 0)
template <typename T, int MASK, bool DZ, bool ACC>
__global__ void __launch_bounds__(256) bnb_apply(int64_t rows, int C, float inv_n, T* g, const T* __restrict__ out,
                                                 T* y, const float* __restrict__ stat, const float* __restrict__ gamma,
                                                 const float* __restrict__ beta, const float* __restrict__ dgamma,
                                                 const float* __restrict__ dbeta, T* acc) {
  const int gC = C / 8, tpr = 256 / gC;
  const int cg = threadIdx.x % gC, rr = threadIdx.x / gC;
  if (rr >= tpr) return;
  float mu[8], rs[8], gm[8], bt[8], a1[8], c1[8], c2[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = cg * 8 + k;
    mu[k] = stat[c];
    rs[k] = stat[C + c];
    gm[k] = gamma[c];
    bt[k] = MASK == 2 ? beta[c] : 0.f;
    a1[k] = gm[k] * rs[k];
    c1[k] = dbeta[c] * inv_n;
    c2[k] = dgamma[c] * inv_n;
  }
  const int64_t stride = (int64_t)gridDim.x * tpr;
#pragma unroll 2
  for (int64_t r = (int64_t)blockIdx.x * tpr + rr; r < rows; r += stride) {
    const int64_t o = r * C + cg * 8;
    V8 gv = ld8(g + o), yv = ld8(y + o);
    V8 ov;
    if (MASK == 1) ov = ld8(out + o);
    V8 dz, dy;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float xh = (yv.v[k] - mu[k]) * rs[k];
      const bool on = MASK == 0 || (MASK == 1 ? ov.v[k] > 0.f : fmaf(gm[k], xh, bt[k]) > 0.f);
      const float z = on ? gv.v[k] : 0.f;
      dz.v[k] = z;
      dy.v[k] = a1[k] * (z - c1[k] - xh * c2[k]);
    }
    if (ACC) {
      V8 old = ld8(acc + o);
#pragma unroll
      for (int k = 0; k < 8; ++k) dy.v[k] += old.v[k];
      st8(acc + o, dy);
    } else {
      st8(y + o, dy);
    }
    if (DZ) st8(g + o, dz);
  }
}

template <typename T, int MASK>
Status bnb_apply_launch(OpArgs& a, int64_t rows, int C, bool dz, bool acc, T* accp) {
  auto k = dz ? (acc ? bnb_apply<T, MASK, true, true> : bnb_apply<T, MASK, true, false>)
              : (acc ? bnb_apply<T, MASK, false, true> : bnb_apply<T, MASK, false, false>);
  k<<<rowgroup_blocks(rows, C), 256, 0, a.stream>>>(
      rows, C, 1.f / (float)rows, (T*)a.p(BB_G), (const T*)a.p(BB_OUT), (T*)a.p(BB_Y), (const float*)a.p(BB_STAT),
      (const float*)a.p(BB_GAMMA), (const float*)a.p(BB_BETA), (const float*)a.p(BB_DGAMMA),
      (const float*)a.p(BB_DBETA), accp);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

template <typename T>
Status bn_bwd_apply_t(OpArgs& a) {
  const int64_t rows = A(a, "rows");
  const int C = (int)A(a, "C");
  if (C % 8 || C > 2048) return Status::make(OC_E_UNSUPPORTED, "bn: C must be a multiple of 8 and <= 2048");
  const bool relu = Ab(a, "relu"), dz = Ab(a, "has_res"), acc = Ab(a, "accumulate");
  T* accp = acc ? (T*)a.p(BB_ACC) : nullptr;
  if (!relu) return bnb_apply_launch<T, 0>(a, rows, C, dz, acc, accp);
  if (a.p(BB_OUT)) return bnb_apply_launch<T, 1>(a, rows, C, dz, acc, accp);
  return bnb_apply_launch<T, 2>(a, rows, C, dz, acc, accp);
}

// ---------------------------------------------------------------- stem: BN-ReLU-maxpool
struct PoolGeom {
  int N, H, W, C, r, st, pad, P, Q;
  FastDivU fc8, fQ, fP, fW, fH;
};

PoolGeom geom(const OpArgs& a) {
  PoolGeom g{(int)A(a, "N"), (int)A(a, "H"), (int)A(a, "W"), (int)A(a, "C"), (int)A(a, "r"),
             (int)A(a, "stride"), (int)A(a, "pad"), (int)A(a, "P"), (int)A(a, "Q")};
  g.fc8.init(g.C / 8);
  g.fQ.init(g.Q);
  g.fP.init(g.P);
  g.fW.init(g.W);
  g.fH.init(g.H);
  return g;
}

// out[n,p,q,c] = max over the r×r window of rnd(relu(bn(y))) (first max,
// row-major taps, padding excluded); idx = tap of the max (u8)
template <typename T>
__global__ void bn_relu_pool(PoolGeom g, const T* __restrict__ y, const float* __restrict__ stat,
                             const float* __restrict__ gamma, const float* __restrict__ beta, T* __restrict__ out,
                             uint8_t* __restrict__ idx) {
  const int C = g.C;
  const uint32_t total = (uint32_t)g.N * g.P * g.Q * (C / 8);
  // the grid stride is a multiple of C/8 when 256 is (C a power of two up to
  // 2048): a thread's channel group never changes, its BN parameters stay in registers
  const bool fixed_cg = 256 % (C / 8) == 0;
  float gm[8], bt[8], mu[8], rs[8];
  int cg_loaded = -1;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t t0 = g.fc8.div(i);
    const int cg = (int)(i - t0 * (C / 8));
    const uint32_t t1 = g.fQ.div(t0);
    const int q = (int)(t0 - t1 * g.Q);
    const uint32_t n = g.fP.div(t1);
    const int p = (int)(t1 - n * g.P);
    float best[8];
    uint8_t bi[8];
    if (gamma && (!fixed_cg || cg_loaded < 0)) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int c = cg * 8 + k;
        gm[k] = gamma[c]; bt[k] = beta[c]; mu[k] = stat[c]; rs[k] = stat[C + c];
      }
      cg_loaded = cg;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      best[k] = -INFINITY;
      bi[k] = 0;
    }
    for (int u = 0; u < g.r; ++u) {
      const int h = p * g.st - g.pad + u;
      if (h < 0 || h >= g.H) continue;
      for (int v = 0; v < g.r; ++v) {
        const int w = q * g.st - g.pad + v;
        if (w < 0 || w >= g.W) continue;
        V8 x = ld8(y + (((int64_t)n * g.H + h) * g.W + w) * C + cg * 8);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          // plain max-pool (gamma == nullptr) pools the stored values themselves
          const float z = gamma ? rnd<T>(fmaxf(fmaf(gm[k], (x.v[k] - mu[k]) * rs[k], bt[k]), 0.f)) : x.v[k];
          if (z > best[k]) { best[k] = z; bi[k] = (uint8_t)(u * g.r + v); }
        }
      }
    }
    V8 o;
#pragma unroll
    for (int k = 0; k < 8; ++k) o.v[k] = best[k];
    const int64_t oo = (int64_t)i * 8;
    st8(out + oo, o);
    uint2 packed;
    packed.x = bi[0] | (bi[1] << 8) | (bi[2] << 16) | ((uint32_t)bi[3] << 24);
    packed.y = bi[4] | (bi[5] << 8) | (bi[6] << 16) | ((uint32_t)bi[7] << 24);
    *reinterpret_cast<uint2*>(idx + oo) = packed;
  }
}

// The stem geometry (3×3, stride 2, pad 1, bf16, C = 64) tiled: a block takes
// 4 × 16 output pixels, stages their 9 × 33 input pixels in shared memory with
// BN-ReLU applied and rounded once per element (padding as −inf, which never
// wins the first-max rule), then each thread pools from shared memory — y is
// read about once instead of 9 BN evaluations per output.
constexpr int PT_P = 4, PT_Q = 16, PT_R = 2 * PT_P + 1, PT_C = 2 * PT_Q + 1;
__global__ void __launch_bounds__(256) bn_relu_pool_tiled(PoolGeom g, const __nv_bfloat16* __restrict__ y,
                                                          const float* __restrict__ stat,
                                                          const float* __restrict__ gamma,
                                                          const float* __restrict__ beta,
                                                          __nv_bfloat16* __restrict__ out, uint8_t* __restrict__ idx) {
  __shared__ uint4 tile[PT_R * PT_C * 8];
  __shared__ float prm[4][64];
  const int tq = (g.Q + PT_Q - 1) / PT_Q, tp = (g.P + PT_P - 1) / PT_P;
  const int b = blockIdx.x;
  const int n = b / (tp * tq), r0 = b % (tp * tq);
  const int p0 = (r0 / tq) * PT_P, q0 = (r0 % tq) * PT_Q;
  if (threadIdx.x < 64) {
    prm[0][threadIdx.x] = gamma[threadIdx.x];
    prm[1][threadIdx.x] = beta[threadIdx.x];
    prm[2][threadIdx.x] = stat[threadIdx.x];
    prm[3][threadIdx.x] = stat[64 + threadIdx.x];
  }
  __syncthreads();
  const int h0 = 2 * p0 - 1, w0 = 2 * q0 - 1;
  for (int e = threadIdx.x; e < PT_R * PT_C * 8; e += 256) {
    const int cg = e & 7, pix = e >> 3;
    const int h = h0 + pix / PT_C, w = w0 + pix % PT_C;
    __nv_bfloat162 z2[4];
    if (h >= 0 && h < g.H && w >= 0 && w < g.W) {
      const V8 x = ld8(y + (((int64_t)n * g.H + h) * g.W + w) * 64 + cg * 8);
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        const int c = cg * 8 + k;
        const float a0 = fmaxf(fmaf(prm[0][c], (x.v[k] - prm[2][c]) * prm[3][c], prm[1][c]), 0.f);
        const float a1 = fmaxf(fmaf(prm[0][c + 1], (x.v[k + 1] - prm[2][c + 1]) * prm[3][c + 1], prm[1][c + 1]), 0.f);
        z2[k / 2] = __floats2bfloat162_rn(a0, a1);
      }
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) z2[k] = __floats2bfloat162_rn(-INFINITY, -INFINITY);
    }
    tile[e] = *reinterpret_cast<uint4*>(z2);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < PT_P * PT_Q * 8; e += 256) {
    const int cg = e & 7, o = e >> 3;
    const int p = p0 + o / PT_Q, q = q0 + o % PT_Q;
    if (p >= g.P || q >= g.Q) continue;
    float best[8];
    uint8_t bi[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { best[k] = -INFINITY; bi[k] = 0; }
#pragma unroll
    for (int u = 0; u < 3; ++u)
#pragma unroll
      for (int v = 0; v < 3; ++v) {
        const uint4 c4 = tile[((2 * (o / PT_Q) + u) * PT_C + 2 * (o % PT_Q) + v) * 8 + cg];
        const __nv_bfloat162* z2 = reinterpret_cast<const __nv_bfloat162*>(&c4);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __bfloat1622float2(z2[k]);
          if (f.x > best[2 * k]) { best[2 * k] = f.x; bi[2 * k] = (uint8_t)(u * 3 + v); }
          if (f.y > best[2 * k + 1]) { best[2 * k + 1] = f.y; bi[2 * k + 1] = (uint8_t)(u * 3 + v); }
        }
      }
    V8 ov;
#pragma unroll
    for (int k = 0; k < 8; ++k) ov.v[k] = best[k];
    const int64_t oo = (((int64_t)n * g.P + p) * g.Q + q) * 64 + cg * 8;
    st8(out + oo, ov);
    uint2 packed;
    packed.x = bi[0] | (bi[1] << 8) | (bi[2] << 16) | ((uint32_t)bi[3] << 24);
    packed.y = bi[4] | (bi[5] << 8) | (bi[6] << 16) | ((uint32_t)bi[7] << 24);
    *reinterpret_cast<uint2*>(idx + oo) = packed;
  }
}

enum { RP_Y, RP_STAT, RP_GAMMA, RP_BETA, RP_OUT, RP_IDX };
template <typename T>
Status bn_relu_pool_fwd_t(OpArgs& a) {
  PoolGeom g = geom(a);
  auto y = (const T*)a.p(RP_Y);
  if (!Ab(a, "stat_in")) OC_TRY(batch_stats<T>(a, (int64_t)g.N * g.H * g.W, g.C, y, (float*)a.p(RP_STAT)));
  const int64_t total = (int64_t)g.N * g.P * g.Q * (g.C / 8);
  const char* et = std::getenv("OC_POOL_TILED");
  if (sizeof(T) == 2 && g.C == 64 && g.r == 3 && g.st == 2 && g.pad == 1 && !(et && et[0] == '0')) {
    const int64_t blocks = (int64_t)g.N * ((g.P + PT_P - 1) / PT_P) * ((g.Q + PT_Q - 1) / PT_Q);
    bn_relu_pool_tiled<<<(unsigned)blocks, 256, 0, a.stream>>>(
        g, (const __nv_bfloat16*)y, (const float*)a.p(RP_STAT), (const float*)a.p(RP_GAMMA),
        (const float*)a.p(RP_BETA), (__nv_bfloat16*)a.p(RP_OUT), (uint8_t*)a.p(RP_IDX));
    OC_LAUNCH_CHECK(a);
    return Status::ok();
  }
  bn_relu_pool<T><<<grid_for(total, 256, 2), 256, 0, a.stream>>>(g, y, (const float*)a.p(RP_STAT),
                                                                 (const float*)a.p(RP_GAMMA),
                                                                 (const float*)a.p(RP_BETA), (T*)a.p(RP_OUT),
                                                                 (uint8_t*)a.p(RP_IDX));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

// gradient reaching pool-input position (n,h,w,c) through the max pool:
// Σ over windows whose argmax is this position of their output gradient,
// rounded to T unless the caller accumulates it first
template <typename T, bool ROUND = true>
__device__ __forceinline__ void pooled_grad8(const PoolGeom& g, int n, int h, int w, int cg, const T* __restrict__ gp,
                                             const uint8_t* __restrict__ idx, float ga[8]) {
  const int r = g.r, st = g.st;
#pragma unroll
  for (int k = 0; k < 8; ++k) ga[k] = 0.f;
  // windows p with p·st − pad <= h <= p·st − pad + r − 1
  const int p_lo = max(0, (h + g.pad - r + st) / st), p_hi = min(g.P - 1, (h + g.pad) / st);
  const int q_lo = max(0, (w + g.pad - r + st) / st), q_hi = min(g.Q - 1, (w + g.pad) / st);
  for (int p = p_lo; p <= p_hi; ++p) {
    const int u = h - (p * st - g.pad);
    if (u < 0 || u >= r) continue;
    for (int q = q_lo; q <= q_hi; ++q) {
      const int v = w - (q * st - g.pad);
      if (v < 0 || v >= r) continue;
      const uint8_t tap = (uint8_t)(u * r + v);
      const int64_t oo = (((int64_t)n * g.P + p) * g.Q + q) * g.C + cg * 8;
      uint2 packed = *reinterpret_cast<const uint2*>(idx + oo);
      V8 gv = ld8(gp + oo);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t word = k < 4 ? packed.x : packed.y;
        const uint8_t b = (word >> (8 * (k & 3))) & 0xff;
        if (b == tap) ga[k] += gv.v[k];
      }
    }
  }
  if (ROUND) {
#pragma unroll
    for (int k = 0; k < 8; ++k) ga[k] = rnd<T>(ga[k]);
  }
}

// plain max-pool backward: dx = rnd(Σ routed) or, accumulating, rnd(dx + Σ routed)
template <typename T>
__global__ void mp_bwd(PoolGeom g, const T* __restrict__ gp, const uint8_t* __restrict__ idx, T* dx, int accumulate) {
  const int C = g.C;
  const uint32_t total = (uint32_t)g.N * g.H * g.W * (C / 8);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t r = g.fc8.div(i);
    const int cg = (int)(i - r * (C / 8));
    const uint32_t t1 = g.fW.div(r);
    const int w = (int)(r - t1 * g.W);
    const uint32_t n = g.fH.div(t1);
    const int h = (int)(t1 - n * g.H);
    float ga[8];
    pooled_grad8<T, false>(g, (int)n, h, w, cg, gp, idx, ga);
    V8 o;
    if (accumulate) o = ld8(dx + (int64_t)i * 8);
#pragma unroll
    for (int k = 0; k < 8; ++k) o.v[k] = accumulate ? o.v[k] + ga[k] : ga[k];
    st8(dx + (int64_t)i * 8, o);
  }
}

enum { MP_X, MP_OUT, MP_IDX };
template <typename T>
Status maxpool_fwd_t(OpArgs& a) {
  PoolGeom g = geom(a);
  const int64_t total = (int64_t)g.N * g.P * g.Q * (g.C / 8);
  bn_relu_pool<T><<<grid_for(total, 256, 2), 256, 0, a.stream>>>(g, (const T*)a.p(MP_X), nullptr, nullptr, nullptr,
                                                                 (T*)a.p(MP_OUT), (uint8_t*)a.p(MP_IDX));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
enum { MB_G, MB_IDX, MB_DX };
template <typename T>
Status maxpool_bwd_t(OpArgs& a) {
  PoolGeom g = geom(a);
  const int64_t total = (int64_t)g.N * g.H * g.W * (g.C / 8);
  mp_bwd<T><<<grid_for(total, 256, 2), 256, 0, a.stream>>>(g, (const T*)a.p(MB_G), (const uint8_t*)a.p(MB_IDX),
                                                           (T*)a.p(MB_DX), Ab(a, "accumulate") ? 1 : 0);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

// ---------------------------------------------------------------- per-pixel softmax CE
// rows = pixels, K classes (logits and dlogits in the act dtype); loss = mean
// over rows, reduced in fixed order (per-block partials, then one warp)
template <typename T>
__global__ void ce_pix_rows(int64_t rows, int K, const T* __restrict__ z, const int* __restrict__ lab,
                            T* __restrict__ dz, float inv_rows, float* __restrict__ part) {
  float acc = 0.f;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const T* zr = z + r * K;
    float mx = -INFINITY;
    for (int k = 0; k < K; ++k) mx = fmaxf(mx, ld_f(zr + k));
    float s = 0.f;
    for (int k = 0; k < K; ++k) s += expf(ld_f(zr + k) - mx);
    const int y = lab[r];
    acc += (logf(s) + mx) - ld_f(zr + y);
    const float inv_s = 1.f / s;
    for (int k = 0; k < K; ++k)
      st_f(dz + r * K + k, (expf(ld_f(zr + k) - mx) * inv_s - (k == y ? 1.f : 0.f)) * inv_rows);
  }
  acc = warp_sum(acc);
  __shared__ float red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}
__global__ void ce_pix_final(int nblk, const float* __restrict__ part, float inv_rows, float* __restrict__ loss) {
  double s = 0;
  for (int b = threadIdx.x; b < nblk; b += 32) s += part[b];
  s = warp_sum(s);
  if (threadIdx.x == 0) loss[0] = (float)(s * inv_rows);
}
enum { CP_Z, CP_LAB, CP_LOSS, CP_DZ };
template <typename T>
Status softmax_ce_pix_t(OpArgs& a) {
  const int64_t rows = A(a, "rows");
  const int K = (int)A(a, "K");
  const int nblk = grid_for(rows, 256, 4);
  if (a.ws_bytes < (size_t)nblk * 4) return Status::make(OC_E_INVARIANT, "ce_pix: workspace too small");
  ce_pix_rows<T><<<nblk, 256, 0, a.stream>>>(rows, K, (const T*)a.p(CP_Z), (const int*)a.p(CP_LAB), (T*)a.p(CP_DZ),
                                             1.f / (float)rows, (float*)a.ws);
  OC_LAUNCH_CHECK(a);
  ce_pix_final<<<1, 32, 0, a.stream>>>(nblk, (const float*)a.ws, 1.f / (float)rows, (float*)a.p(CP_LOSS));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
size_t ce_pix_ws(const JVal& at) { return (size_t)grid_for(at.geti("rows"), 256, 4) * 4; }

template <typename T>
__global__ void __launch_bounds__(256) pbn_partial(PoolGeom g, const T* __restrict__ gp,
                                                   const uint8_t* __restrict__ idx, const T* __restrict__ y,
                                                   const float* __restrict__ stat, const float* __restrict__ gamma,
                                                   const float* __restrict__ beta, float* __restrict__ part) {
  const int C = g.C, gC = C / 8, tpr = 256 / gC;
  const int t = threadIdx.x, cg = t % gC, rr = t / gC;
  const int64_t rows = (int64_t)g.N * g.H * g.W;
  const int64_t chunk = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * chunk, r1 = min(rows, r0 + chunk);
  float s[8] = {}, q[8] = {};
  float mu[8], rs[8], gm[8], bt[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = (cg * 8 + k) % C;
    mu[k] = stat[c];
    rs[k] = stat[C + c];
    gm[k] = gamma[c];
    bt[k] = beta[c];
  }
  if (rr < tpr)
    for (int64_t r = r0 + rr; r < r1; r += tpr) {
      const uint32_t t1 = g.fW.div((uint32_t)r);
      const int w = (int)((uint32_t)r - t1 * g.W);
      const uint32_t n = g.fH.div(t1);
      const int h = (int)(t1 - n * g.H);
      float ga[8];
      pooled_grad8<T>(g, (int)n, h, w, cg, gp, idx, ga);
      V8 yv = ld8(y + r * C + cg * 8);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float xh = (yv.v[k] - mu[k]) * rs[k];
        const float z = fmaf(gm[k], xh, bt[k]);
        const float dz = z > 0.f ? ga[k] : 0.f;
        s[k] += dz;
        q[k] = fmaf(dz, xh, q[k]);
      }
    }
  extern __shared__ float sm[];
#pragma unroll
  for (int i = 0; i < 8; ++i) { sm[t * 16 + i] = s[i]; sm[t * 16 + 8 + i] = q[i]; }
  __syncthreads();
  for (int c = t; c < C; c += 256) {
    const int grp = c / 8, lane = c % 8;
    float as = 0.f, aq = 0.f;
    for (int k = 0; k < tpr; ++k) {
      as += sm[(k * gC + grp) * 16 + lane];
      aq += sm[(k * gC + grp) * 16 + 8 + lane];
    }
    part[(int64_t)blockIdx.x * 2 * C + c] = as;
    part[(int64_t)blockIdx.x * 2 * C + C + c] = aq;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) pbn_apply(PoolGeom g, const T* __restrict__ gp, const uint8_t* __restrict__ idx,
                                                 T* y, const float* __restrict__ stat, const float* __restrict__ gamma,
                                                 const float* __restrict__ beta, const float* __restrict__ dgamma,
                                                 const float* __restrict__ dbeta, float inv_n) {
  const int C = g.C, gC = C / 8, tpr = 256 / gC;
  const int cg = threadIdx.x % gC, rr = threadIdx.x / gC;
  if (rr >= tpr) return;
  float mu[8], rs[8], gm[8], bt[8], dg[8], db[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = cg * 8 + k;
    mu[k] = stat[c];
    rs[k] = stat[C + c];
    gm[k] = gamma[c];
    bt[k] = beta[c];
    dg[k] = dgamma[c];
    db[k] = dbeta[c];
  }
  const int64_t rows = (int64_t)g.N * g.H * g.W;
  const int64_t stride = (int64_t)gridDim.x * tpr;
  for (int64_t r = (int64_t)blockIdx.x * tpr + rr; r < rows; r += stride) {
    const uint32_t t1 = g.fW.div((uint32_t)r);
    const int w = (int)((uint32_t)r - t1 * g.W);
    const uint32_t n = g.fH.div(t1);
    const int h = (int)(t1 - n * g.H);
    float ga[8];
    pooled_grad8<T>(g, (int)n, h, w, cg, gp, idx, ga);
    const int64_t o = r * C + cg * 8;
    V8 yv = ld8(y + o);
    V8 dy;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float xh = (yv.v[k] - mu[k]) * rs[k];
      const float z = fmaf(gm[k], xh, bt[k]);
      const float dz = z > 0.f ? ga[k] : 0.f;
      dy.v[k] = gm[k] * rs[k] * (dz - db[k] * inv_n - xh * dg[k] * inv_n);
    }
    st8(y + o, dy);   // in place: each thread reads only its own y
  }
}

// 3×3 / stride-2 / pad-1 pool over an even H × W map (the stem): a thread
// owns the 2×2 input block (2i..2i+1, 2j..2j+1) × 8 channels, which only the
// windows (i|i+1, j|j+1) reach; each window's argmax tap lands in at most one
// of the four pixels.  Windows are visited in (p, q) ascending order, the order
// pooled_grad8 sums them in, so the routed gradients are bitwise the same.
template <typename T>
__device__ __forceinline__ void pool_block_grad(const PoolGeom& g, int n, int i, int j, int cg, const T* __restrict__ gp,
                                                const uint8_t* __restrict__ idx, float ga[4][8]) {
#pragma unroll
  for (int px = 0; px < 4; ++px)
#pragma unroll
    for (int k = 0; k < 8; ++k) ga[px][k] = 0.f;
#pragma unroll
  for (int wi = 0; wi < 2; ++wi) {
    const int p = i + wi;
    if (p >= g.P) continue;
#pragma unroll
    for (int wj = 0; wj < 2; ++wj) {
      const int q = j + wj;
      if (q >= g.Q) continue;
      const int64_t oo = (((int64_t)n * g.P + p) * g.Q + q) * g.C + cg * 8;
      const uint2 packed = *reinterpret_cast<const uint2*>(idx + oo);
      const V8 gv = ld8(gp + oo);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t tap = ((k < 4 ? packed.x : packed.y) >> (8 * (k & 3))) & 0xff;
        const int u = (int)((tap * 11) >> 5), v = (int)tap - 3 * u;   // tap / 3, tap % 3 for tap < 9
        const int dr = 2 * wi - 1 + u, dc = 2 * wj - 1 + v;           // row / col inside the 2×2 block
#pragma unroll
        for (int px = 0; px < 4; ++px)
          if (dr == (px >> 1) && dc == (px & 1)) ga[px][k] += gv.v[k];
      }
    }
  }
#pragma unroll
  for (int px = 0; px < 4; ++px)
#pragma unroll
    for (int k = 0; k < 8; ++k) ga[px][k] = rnd<T>(ga[px][k]);
}

inline bool stem_pool(const PoolGeom& g) {
  return g.r == 3 && g.st == 2 && g.pad == 1 && g.H % 2 == 0 && g.W % 2 == 0 && g.P == g.H / 2 && g.Q == g.W / 2;
}

template <typename T>
__global__ void __launch_bounds__(256) pbn_partial_blk(PoolGeom g, const T* __restrict__ gp,
                                                       const uint8_t* __restrict__ idx, const T* __restrict__ y,
                                                       const float* __restrict__ stat,
                                                       const float* __restrict__ gamma,
                                                       const float* __restrict__ beta, float* __restrict__ part) {
  const int C = g.C, gC = C / 8, tpr = 256 / gC;
  const int t = threadIdx.x, cg = t % gC, rr = t / gC;
  const int64_t units = (int64_t)g.N * g.P * g.Q;           // 2×2 input blocks
  const int64_t chunk = (units + gridDim.x - 1) / gridDim.x;
  const int64_t u0 = blockIdx.x * chunk, u1 = min(units, u0 + chunk);
  float s[8] = {}, q[8] = {};
  float mu[8], rs[8], gm[8], bt[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = (cg * 8 + k) % C;
    mu[k] = stat[c];
    rs[k] = stat[C + c];
    gm[k] = gamma[c];
    bt[k] = beta[c];
  }
  if (rr < tpr)
    for (int64_t u = u0 + rr; u < u1; u += tpr) {
      const uint32_t t1 = g.fQ.div((uint32_t)u);
      const int j = (int)((uint32_t)u - t1 * g.Q);
      const uint32_t n = g.fP.div(t1);
      const int i = (int)(t1 - n * g.P);
      float ga[4][8];
      pool_block_grad<T>(g, (int)n, i, j, cg, gp, idx, ga);
#pragma unroll
      for (int px = 0; px < 4; ++px) {
        const int64_t o = (((int64_t)n * g.H + 2 * i + (px >> 1)) * g.W + 2 * j + (px & 1)) * C + cg * 8;
        const V8 yv = ld8(y + o);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float xh = (yv.v[k] - mu[k]) * rs[k];
          const float z = fmaf(gm[k], xh, bt[k]);
          const float dz = z > 0.f ? ga[px][k] : 0.f;
          s[k] += dz;
          q[k] = fmaf(dz, xh, q[k]);
        }
      }
    }
  extern __shared__ float sm[];
#pragma unroll
  for (int k = 0; k < 8; ++k) { sm[t * 16 + k] = s[k]; sm[t * 16 + 8 + k] = q[k]; }
  __syncthreads();
  for (int c = t; c < C; c += 256) {
    const int grp = c / 8, lane = c % 8;
    float as = 0.f, aq = 0.f;
    for (int k = 0; k < tpr; ++k) {
      as += sm[(k * gC + grp) * 16 + lane];
      aq += sm[(k * gC + grp) * 16 + 8 + lane];
    }
    part[(int64_t)blockIdx.x * 2 * C + c] = as;
    part[(int64_t)blockIdx.x * 2 * C + C + c] = aq;
  }
}

// (256, 3): 80 registers instead of 121 — three blocks per SM; measured 8 % faster
// despite a small stack spill (the same bound made pbn_partial_blk 27 % slower)
template <typename T>
__global__ void __launch_bounds__(256, 3) pbn_apply_blk(PoolGeom g, const T* __restrict__ gp,
                                                     const uint8_t* __restrict__ idx, T* y,
                                                     const float* __restrict__ stat, const float* __restrict__ gamma,
                                                     const float* __restrict__ beta, const float* __restrict__ dgamma,
                                                     const float* __restrict__ dbeta, float inv_n) {
  const int C = g.C, gC = C / 8, tpr = 256 / gC;
  const int cg = threadIdx.x % gC, rr = threadIdx.x / gC;
  if (rr >= tpr) return;
  float mu[8], rs[8], gm[8], bt[8], dg[8], db[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = cg * 8 + k;
    mu[k] = stat[c];
    rs[k] = stat[C + c];
    gm[k] = gamma[c];
    bt[k] = beta[c];
    dg[k] = dgamma[c];
    db[k] = dbeta[c];
  }
  const int64_t units = (int64_t)g.N * g.P * g.Q;
  const int64_t stride = (int64_t)gridDim.x * tpr;
  for (int64_t u = (int64_t)blockIdx.x * tpr + rr; u < units; u += stride) {
    const uint32_t t1 = g.fQ.div((uint32_t)u);
    const int j = (int)((uint32_t)u - t1 * g.Q);
    const uint32_t n = g.fP.div(t1);
    const int i = (int)(t1 - n * g.P);
    float ga[4][8];
    pool_block_grad<T>(g, (int)n, i, j, cg, gp, idx, ga);
#pragma unroll
    for (int px = 0; px < 4; ++px) {
      const int64_t o = (((int64_t)n * g.H + 2 * i + (px >> 1)) * g.W + 2 * j + (px & 1)) * C + cg * 8;
      const V8 yv = ld8(y + o);
      V8 dy;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float xh = (yv.v[k] - mu[k]) * rs[k];
        const float z = fmaf(gm[k], xh, bt[k]);
        const float dz = z > 0.f ? ga[px][k] : 0.f;
        dy.v[k] = gm[k] * rs[k] * (dz - db[k] * inv_n - xh * dg[k] * inv_n);
      }
      st8(y + o, dy);   // in place: each thread reads only its own four pixels of y
    }
  }
}

enum { PB_G, PB_IDX, PB_Y, PB_STAT, PB_GAMMA, PB_BETA, PB_DGAMMA, PB_DBETA };
template <typename T>
Status pool_bn_bwd_reduce_t(OpArgs& a) {
  PoolGeom g = geom(a);
  const int64_t rows = (int64_t)g.N * g.H * g.W;
  const int nblk = stat_blocks(rows);
  if (a.ws_bytes < (size_t)nblk * 2 * g.C * 4) return Status::make(OC_E_INVARIANT, "pool_bn_bwd: workspace too small");
  if (stem_pool(g))
    pbn_partial_blk<T><<<nblk, 256, 256 * 16 * 4, a.stream>>>(
        g, (const T*)a.p(PB_G), (const uint8_t*)a.p(PB_IDX), (const T*)a.p(PB_Y), (const float*)a.p(PB_STAT),
        (const float*)a.p(PB_GAMMA), (const float*)a.p(PB_BETA), (float*)a.ws);
  else
    pbn_partial<T><<<nblk, 256, 256 * 16 * 4, a.stream>>>(
        g, (const T*)a.p(PB_G), (const uint8_t*)a.p(PB_IDX), (const T*)a.p(PB_Y), (const float*)a.p(PB_STAT),
        (const float*)a.p(PB_GAMMA), (const float*)a.p(PB_BETA), (float*)a.ws);
  OC_LAUNCH_CHECK(a);
  bnb_finalize<<<(g.C + 7) / 8, 256, 0, a.stream>>>(nblk, g.C, (const float*)a.ws, (float*)a.p(PB_DGAMMA),
                                                    (float*)a.p(PB_DBETA));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
template <typename T>
Status pool_bn_bwd_apply_t(OpArgs& a) {
  PoolGeom g = geom(a);
  const int64_t rows = (int64_t)g.N * g.H * g.W;
  if (g.C % 8 || g.C > 2048) return Status::make(OC_E_UNSUPPORTED, "pool_bn: C must be a multiple of 8 and <= 2048");
  if (stem_pool(g))
    pbn_apply_blk<T><<<rowgroup_blocks(rows / 4, g.C), 256, 0, a.stream>>>(
        g, (const T*)a.p(PB_G), (const uint8_t*)a.p(PB_IDX), (T*)a.p(PB_Y), (const float*)a.p(PB_STAT),
        (const float*)a.p(PB_GAMMA), (const float*)a.p(PB_BETA), (const float*)a.p(PB_DGAMMA),
        (const float*)a.p(PB_DBETA), 1.f / (float)rows);
  else
    pbn_apply<T><<<rowgroup_blocks(rows, g.C), 256, 0, a.stream>>>(
        g, (const T*)a.p(PB_G), (const uint8_t*)a.p(PB_IDX), (T*)a.p(PB_Y), (const float*)a.p(PB_STAT),
        (const float*)a.p(PB_GAMMA), (const float*)a.p(PB_BETA), (const float*)a.p(PB_DGAMMA),
        (const float*)a.p(PB_DBETA), 1.f / (float)rows);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

// ---------------------------------------------------------------- global average pool
template <typename T>
__global__ void gap_fwd_k(int N, int HW, int C, const T* __restrict__ x, T* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N * C) return;
  const int n = i / C, c = i % C;
  float s = 0.f;
  for (int k = 0; k < HW; ++k) s += ld_f(x + ((int64_t)n * HW + k) * C + c);
  st_f(out + i, s / (float)HW);
}
template <typename T>
__global__ void gap_bwd_k(int N, int HW, int C, const T* __restrict__ g, T* __restrict__ dx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)N * HW * C) return;
  const int c = (int)(i % C);
  const int n = (int)(i / ((int64_t)HW * C));
  st_f(dx + i, ld_f(g + (int64_t)n * C + c) / (float)HW);
}
template <typename T>
Status gap_fwd_t(OpArgs& a) {
  const int N = (int)A(a, "N"), HW = (int)A(a, "HW"), C = (int)A(a, "C");
  gap_fwd_k<T><<<(N * C + 255) / 256, 256, 0, a.stream>>>(N, HW, C, (const T*)a.p(0), (T*)a.p(1));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
template <typename T>
Status gap_bwd_t(OpArgs& a) {
  const int N = (int)A(a, "N"), HW = (int)A(a, "HW"), C = (int)A(a, "C");
  const int64_t tot = (int64_t)N * HW * C;
  gap_bwd_k<T><<<(int)((tot + 255) / 256), 256, 0, a.stream>>>(N, HW, C, (const T*)a.p(0), (T*)a.p(1));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

// ---------------------------------------------------------------- residual add
// out = rnd(a + b) (pre-activation blocks); 16-byte vectors
template <typename T>
__global__ void add_k(uint32_t n8, const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += gridDim.x * blockDim.x) {
    V8 x = ld8(a + (int64_t)i * 8), y = ld8(b + (int64_t)i * 8);
#pragma unroll
    for (int k = 0; k < 8; ++k) x.v[k] += y.v[k];
    st8(out + (int64_t)i * 8, x);
  }
}
template <typename T>
Status add_fwd_t(OpArgs& a) {
  const int64_t n = A(a, "n");
  if (n % 8) return Status::make(OC_E_UNSUPPORTED, "add: element count must be a multiple of 8");
  const uint32_t n8 = (uint32_t)(n / 8);
  add_k<T><<<grid_for(n8, 256, 4), 256, 0, a.stream>>>(n8, (const T*)a.p(0), (const T*)a.p(1), (T*)a.p(2));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

// dtype dispatch: attrs.dtype = "bf16" (default) | "f32"
#define OC_DT_DISPATCH(name)                                                  \
  Status name(OpArgs& a) {                                                    \
    return As(a, "dtype", "bf16") == "f32" ? name##_t<float>(a) : name##_t<__nv_bfloat16>(a); \
  }
OC_DT_DISPATCH(bn_fwd)
OC_DT_DISPATCH(bn_bwd_reduce)
OC_DT_DISPATCH(bn_bwd_apply)
OC_DT_DISPATCH(bn_relu_pool_fwd)
OC_DT_DISPATCH(pool_bn_bwd_reduce)
OC_DT_DISPATCH(pool_bn_bwd_apply)
OC_DT_DISPATCH(gap_fwd)
OC_DT_DISPATCH(gap_bwd)
OC_DT_DISPATCH(add_fwd)
OC_DT_DISPATCH(maxpool_fwd)
OC_DT_DISPATCH(maxpool_bwd)
OC_DT_DISPATCH(softmax_ce_pix)

}  // namespace

// BN batch statistics for a producer op (conv_fwd with attrs.bn_stat): from the
// partial sums its epilogue wrote (part[slot][2][C], Σy and Σy² of the stored
// bf16 values), or — when the conv ran on a path without that epilogue — the
// usual two-level reduction over y
Status bn_stats_from_parts(OpArgs& a, int nslots, int64_t rows, int C, const float* part, float* stat) {
  stats_finalize<<<(C + 7) / 8, 256, 0, a.stream>>>(nslots, rows, C, part, stat);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
Status bn_stats_of(OpArgs& a, int64_t rows, int C, const void* y, bool f32, float* stat) {
  return f32 ? batch_stats<float>(a, rows, C, (const float*)y, stat)
             : batch_stats<__nv_bfloat16>(a, rows, C, (const __nv_bfloat16*)y, stat);
}

extern const OpDesc kAddFwd{"add_fwd", {"a", "b", "out"}, add_fwd, nullptr};
extern const OpDesc kMaxpoolFwd{"maxpool_fwd", {"x", "out", "idx"}, maxpool_fwd, nullptr};
extern const OpDesc kMaxpoolBwd{"maxpool_bwd", {"g", "idx", "dx"}, maxpool_bwd, nullptr};
extern const OpDesc kSoftmaxCEPix{"softmax_ce_pix", {"logits", "labels", "loss", "dlogits"}, softmax_ce_pix,
                                  ce_pix_ws};

extern const OpDesc kBnFwd{"bn_fwd", {"y", "stat", "gamma", "beta", "res", "out"}, bn_fwd, bn_ws};
extern const OpDesc kBnBwdReduce{"bn_bwd_reduce",
                                 {"g", "out", "y", "stat", "gamma", "dgamma", "dbeta", "acc", "beta"}, bn_bwd_reduce,
                                 bn_ws};
extern const OpDesc kBnBwdApply{"bn_bwd_apply", {"g", "out", "y", "stat", "gamma", "dgamma", "dbeta", "acc", "beta"},
                                bn_bwd_apply, nullptr};
extern const OpDesc kBnReluPoolFwd{"bn_relu_pool_fwd", {"y", "stat", "gamma", "beta", "out", "idx"}, bn_relu_pool_fwd,
                                   bn_ws};
extern const OpDesc kPoolBnBwdReduce{"pool_bn_bwd_reduce",
                                     {"g", "idx", "y", "stat", "gamma", "beta", "dgamma", "dbeta"},
                                     pool_bn_bwd_reduce, bn_ws};
extern const OpDesc kPoolBnBwdApply{"pool_bn_bwd_apply", {"g", "idx", "y", "stat", "gamma", "beta", "dgamma", "dbeta"},
                                    pool_bn_bwd_apply, nullptr};
extern const OpDesc kGapFwd{"gap_fwd", {"x", "out"}, gap_fwd, nullptr};
extern const OpDesc kGapBwd{"gap_bwd", {"g", "dx"}, gap_bwd, nullptr};

}  // namespace oc
