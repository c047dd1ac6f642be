// Batch-norm / ReLU / residual-add / pooling kernels of the conv-net training
// step, NHWC bf16 activations viewed as [rows, C].
//
// Memory-bound: every kernel moves 16-byte vectors (8 bf16 channels) per
// thread with coalesced row-major access and grids sized in multiples of the
// 148 SMs.  Per-channel reductions are deterministic two-level reductions
// (fixed row chunks -> fp32 partials -> fixed-order double finalize) so the
// step is bitwise reproducible whatever the swap schedule.
//
// Contract (oracle/numerics.py): x̂ = (y−μ)·rstd with batch statistics and
// biased variance, eps = 1e-5; out = rnd(relu(γx̂ + β + res)); backward
// dz = g·[out>0], dβ = Σdz, dγ = Σdz·x̂, dy = γ·rstd·(dz − dβ/n − x̂·dγ/n).
#include "common.cuh"

namespace oc {

namespace {

constexpr float kEps = 1e-5f;
constexpr int kStatBlocks = 148 * 4;  // row chunks of the two-level reductions

struct V8 {
  float v[8];
};

__device__ __forceinline__ V8 ld8(const __nv_bfloat16* p) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
  V8 r;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    r.v[2 * i] = f.x;
    r.v[2 * i + 1] = f.y;
  }
  return r;
}

__device__ __forceinline__ void st8(__nv_bfloat16* p, const V8& x) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(x.v[2 * i], x.v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}

// ---------------------------------------------------------------- statistics
// Partial Σy, Σy² over a contiguous row chunk per block.  Thread t covers the
// 8 channels starting at (t % (C/8))·8 of every (256/(C/8))-th row.
__global__ void __launch_bounds__(256) stats_partial(int64_t rows, int C, const __nv_bfloat16* __restrict__ y,
                                                     float* __restrict__ part) {
  const int g = C / 8;                 // threads per row
  const int tpr = 256 / g;             // rows per block iteration (C <= 2048)
  const int t = threadIdx.x;
  const int cg = t % g, rr = t / g;
  const int64_t chunk = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * chunk, r1 = min(rows, r0 + chunk);
  float s[8] = {}, q[8] = {};
  if (rr < tpr)
    for (int64_t r = r0 + rr; r < r1; r += tpr) {
      V8 x = ld8(y + r * C + cg * 8);
#pragma unroll
      for (int i = 0; i < 8; ++i) { s[i] += x.v[i]; q[i] = fmaf(x.v[i], x.v[i], q[i]); }
    }
  extern __shared__ float sm[];        // [256][16]
#pragma unroll
  for (int i = 0; i < 8; ++i) { sm[t * 16 + i] = s[i]; sm[t * 16 + 8 + i] = q[i]; }
  __syncthreads();
  // fixed-order combine of the tpr threads sharing a channel group
  for (int c = t; c < C; c += 256) {
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

// stat[0][c] = μ, stat[1][c] = rstd  (fixed-order double sum over chunks)
// one warp per channel: lane-strided partial sums, then a fixed xor tree
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

__global__ void stats_finalize(int nblk, int64_t rows, int C, const float* __restrict__ part, float* __restrict__ stat) {
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= C) return;
  double s, q;
  chunk_sums(nblk, C, c, part, s, q);
  if ((threadIdx.x & 31) != 0) return;
  double mu = s / rows;
  double var = q / rows - mu * mu;
  if (var < 0) var = 0;
  stat[c] = (float)mu;
  stat[C + c] = (float)(1.0 / sqrt(var + (double)kEps));
}

Status batch_stats(OpArgs& a, int64_t rows, int C, const __nv_bfloat16* y, float* stat) {
  if (C % 8 || C > 2048) return Status::make(OC_E_UNSUPPORTED, "bn: C must be a multiple of 8 and <= 2048");
  const int nblk = (int)std::min<int64_t>(kStatBlocks, std::max<int64_t>(1, rows / 64));
  if (a.ws_bytes < (size_t)nblk * 2 * C * 4) return Status::make(OC_E_INVARIANT, "bn: workspace too small");
  stats_partial<<<nblk, 256, 256 * 16 * 4, a.stream>>>(rows, C, y, (float*)a.ws);
  OC_LAUNCH_CHECK(a);
  stats_finalize<<<(C + 7) / 8, 256, 0, a.stream>>>(nblk, rows, C, (const float*)a.ws, stat);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

// ---------------------------------------------------------------- forward
__global__ void bn_apply_fwd(int64_t n8, int C, const __nv_bfloat16* __restrict__ y, const float* __restrict__ stat,
                             const float* __restrict__ gamma, const float* __restrict__ beta,
                             const __nv_bfloat16* __restrict__ res, __nv_bfloat16* __restrict__ out, int relu) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int c0 = (int)((i * 8) % C);
    V8 x = ld8(y + i * 8);
    V8 r;
    if (res) r = ld8(res + i * 8);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int c = c0 + k;
      float z = fmaf(gamma[c], (x.v[k] - stat[c]) * stat[C + c], beta[c]);
      if (res) z += r.v[k];
      if (relu) z = fmaxf(z, 0.f);
      x.v[k] = z;
    }
    st8(out + i * 8, x);
  }
}

enum { BF_Y, BF_STAT, BF_GAMMA, BF_BETA, BF_RES, BF_OUT };
Status bn_fwd(OpArgs& a) {
  const int64_t rows = A(a, "rows");
  const int C = (int)A(a, "C");
  auto y = (const __nv_bfloat16*)a.p(BF_Y);
  OC_TRY(batch_stats(a, rows, C, y, (float*)a.p(BF_STAT)));
  const int64_t n8 = rows * C / 8;
  bn_apply_fwd<<<grid_for(n8, 256, 4), 256, 0, a.stream>>>(n8, C, y, (const float*)a.p(BF_STAT),
                                                           (const float*)a.p(BF_GAMMA), (const float*)a.p(BF_BETA),
                                                           (const __nv_bfloat16*)a.p(BF_RES),
                                                           (__nv_bfloat16*)a.p(BF_OUT), Ab(a, "relu") ? 1 : 0);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
size_t bn_ws(const JVal& at) {
  int64_t rows = at.geti("rows"), C = at.geti("C");
  int64_t nblk = std::min<int64_t>(kStatBlocks, std::max<int64_t>(1, rows / 64));
  return (size_t)(nblk * 2 * C * 4);
}

// ---------------------------------------------------------------- backward
// partial Σdz, Σdz·x̂ per channel
__global__ void __launch_bounds__(256) bnb_partial(int64_t rows, int C, const __nv_bfloat16* __restrict__ g,
                                                   const __nv_bfloat16* __restrict__ out,
                                                   const __nv_bfloat16* __restrict__ y,
                                                   const float* __restrict__ stat, int relu, float* __restrict__ part) {
  const int gC = C / 8, tpr = 256 / gC;
  const int t = threadIdx.x, cg = t % gC, rr = t / gC;
  const int64_t chunk = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * chunk, r1 = min(rows, r0 + chunk);
  float s[8] = {}, q[8] = {};
  float mu[8], rs[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { mu[i] = stat[cg * 8 + i]; rs[i] = stat[C + cg * 8 + i]; }
  if (rr < tpr)
    for (int64_t r = r0 + rr; r < r1; r += tpr) {
      const int64_t o = r * C + cg * 8;
      V8 gv = ld8(g + o), yv = ld8(y + o);
      V8 ov;
      if (relu) ov = ld8(out + o);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float dz = (!relu || ov.v[i] > 0.f) ? gv.v[i] : 0.f;
        s[i] += dz;
        q[i] = fmaf(dz, (yv.v[i] - mu[i]) * rs[i], q[i]);
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

enum { BB_G, BB_OUT, BB_Y, BB_STAT, BB_GAMMA, BB_DGAMMA, BB_DBETA };
Status bn_bwd_reduce(OpArgs& a) {
  const int64_t rows = A(a, "rows");
  const int C = (int)A(a, "C");
  const int nblk = (int)std::min<int64_t>(kStatBlocks, std::max<int64_t>(1, rows / 64));
  if (a.ws_bytes < (size_t)nblk * 2 * C * 4) return Status::make(OC_E_INVARIANT, "bn_bwd: workspace too small");
  bnb_partial<<<nblk, 256, 256 * 16 * 4, a.stream>>>(rows, C, (const __nv_bfloat16*)a.p(BB_G),
                                                     (const __nv_bfloat16*)a.p(BB_OUT),
                                                     (const __nv_bfloat16*)a.p(BB_Y), (const float*)a.p(BB_STAT),
                                                     Ab(a, "relu") ? 1 : 0, (float*)a.ws);
  OC_LAUNCH_CHECK(a);
  bnb_finalize<<<(C + 7) / 8, 256, 0, a.stream>>>(nblk, C, (const float*)a.ws, (float*)a.p(BB_DGAMMA),
                                                      (float*)a.p(BB_DBETA));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

// dy = γ·rstd·(dz − dβ/n − x̂·dγ/n), written over y; dz written over g (residual branch)
__global__ void bnb_apply(int64_t n8, int C, float inv_n, __nv_bfloat16* g, const __nv_bfloat16* __restrict__ out,
                          __nv_bfloat16* y, const float* __restrict__ stat, const float* __restrict__ gamma,
                          const float* __restrict__ dgamma, const float* __restrict__ dbeta, int relu, int write_dz) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int c0 = (int)((i * 8) % C);
    V8 gv = ld8(g + i * 8), yv = ld8(y + i * 8);
    V8 ov;
    if (relu) ov = ld8(out + i * 8);
    V8 dz, dy;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int c = c0 + k;
      const float z = (!relu || ov.v[k] > 0.f) ? gv.v[k] : 0.f;
      const float xh = (yv.v[k] - stat[c]) * stat[C + c];
      dz.v[k] = z;
      dy.v[k] = gamma[c] * stat[C + c] * (z - dbeta[c] * inv_n - xh * dgamma[c] * inv_n);
    }
    st8(y + i * 8, dy);
    if (write_dz) st8(g + i * 8, dz);
  }
}

enum { BA_G, BA_OUT, BA_Y, BA_STAT, BA_GAMMA, BA_DGAMMA, BA_DBETA };
Status bn_bwd_apply(OpArgs& a) {
  const int64_t rows = A(a, "rows");
  const int C = (int)A(a, "C");
  const int64_t n8 = rows * C / 8;
  bnb_apply<<<grid_for(n8, 256, 4), 256, 0, a.stream>>>(
      n8, C, 1.f / (float)rows, (__nv_bfloat16*)a.p(BA_G), (const __nv_bfloat16*)a.p(BA_OUT),
      (__nv_bfloat16*)a.p(BA_Y), (const float*)a.p(BA_STAT), (const float*)a.p(BA_GAMMA),
      (const float*)a.p(BA_DGAMMA), (const float*)a.p(BA_DBETA), Ab(a, "relu") ? 1 : 0,
      Ab(a, "has_res") ? 1 : 0);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

// ---------------------------------------------------------------- stem: BN-ReLU-maxpool
// out[n,p,q,c] = max over the r×r window of rnd(relu(bn(y))) (first max,
// row-major taps, padding excluded); idx = tap of the max (u8)
__global__ void bn_relu_pool(int N, int H, int W, int C, int r, int st, int pad, int P, int Q,
                             const __nv_bfloat16* __restrict__ y, const float* __restrict__ stat,
                             const float* __restrict__ gamma, const float* __restrict__ beta,
                             __nv_bfloat16* __restrict__ out, uint8_t* __restrict__ idx) {
  const int64_t total = (int64_t)N * P * Q * (C / 8);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int cg = (int)(i % (C / 8));
    int64_t t = i / (C / 8);
    const int q = (int)(t % Q); t /= Q;
    const int p = (int)(t % P);
    const int n = (int)(t / P);
    float best[8];
    uint8_t bi[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { best[k] = -INFINITY; bi[k] = 0; }
    for (int u = 0; u < r; ++u) {
      const int h = p * st - pad + u;
      if (h < 0 || h >= H) continue;
      for (int v = 0; v < r; ++v) {
        const int w = q * st - pad + v;
        if (w < 0 || w >= W) continue;
        V8 x = ld8(y + (((int64_t)n * H + h) * W + w) * C + cg * 8);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int c = cg * 8 + k;
          float z = fmaxf(fmaf(gamma[c], (x.v[k] - stat[c]) * stat[C + c], beta[c]), 0.f);
          z = rnd<__nv_bfloat16>(z);
          if (z > best[k]) { best[k] = z; bi[k] = (uint8_t)(u * r + v); }
        }
      }
    }
    V8 o;
#pragma unroll
    for (int k = 0; k < 8; ++k) o.v[k] = best[k];
    const int64_t oo = (((int64_t)n * P + p) * Q + q) * C + cg * 8;
    st8(out + oo, o);
    uint2 packed;
    packed.x = bi[0] | (bi[1] << 8) | (bi[2] << 16) | ((uint32_t)bi[3] << 24);
    packed.y = bi[4] | (bi[5] << 8) | (bi[6] << 16) | ((uint32_t)bi[7] << 24);
    *reinterpret_cast<uint2*>(idx + oo) = packed;
  }
}

enum { RP_Y, RP_STAT, RP_GAMMA, RP_BETA, RP_OUT, RP_IDX };
Status bn_relu_pool_fwd(OpArgs& a) {
  const int N = (int)A(a, "N"), H = (int)A(a, "H"), W = (int)A(a, "W"), C = (int)A(a, "C");
  const int r = (int)A(a, "r"), st = (int)A(a, "stride"), pad = (int)A(a, "pad");
  const int P = (int)A(a, "P"), Q = (int)A(a, "Q");
  auto y = (const __nv_bfloat16*)a.p(RP_Y);
  OC_TRY(batch_stats(a, (int64_t)N * H * W, C, y, (float*)a.p(RP_STAT)));
  const int64_t total = (int64_t)N * P * Q * (C / 8);
  bn_relu_pool<<<grid_for(total, 256, 2), 256, 0, a.stream>>>(N, H, W, C, r, st, pad, P, Q, y,
                                                              (const float*)a.p(RP_STAT), (const float*)a.p(RP_GAMMA),
                                                              (const float*)a.p(RP_BETA),
                                                              (__nv_bfloat16*)a.p(RP_OUT), (uint8_t*)a.p(RP_IDX));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
size_t rp_ws(const JVal& at) {
  int64_t rows = at.geti("N") * at.geti("H") * at.geti("W"), C = at.geti("C");
  int64_t nblk = std::min<int64_t>(kStatBlocks, std::max<int64_t>(1, rows / 64));
  return (size_t)(nblk * 2 * C * 4);
}

// gradient reaching bn-output position (n,h,w,c) through the max pool:
// rnd(Σ over windows whose argmax is this position of their output gradient)
struct PoolGeom { int N, H, W, C, r, st, pad, P, Q; };

__device__ __forceinline__ void pooled_grad8(const PoolGeom& g, int n, int h, int w, int cg,
                                             const __nv_bfloat16* __restrict__ gp, const uint8_t* __restrict__ idx,
                                             float ga[8]) {
#pragma unroll
  for (int k = 0; k < 8; ++k) ga[k] = 0.f;
  const int p_lo = max(0, (h + g.pad - g.r + g.st) / g.st), p_hi = min(g.P - 1, (h + g.pad) / g.st);
  const int q_lo = max(0, (w + g.pad - g.r + g.st) / g.st), q_hi = min(g.Q - 1, (w + g.pad) / g.st);
  for (int p = p_lo; p <= p_hi; ++p) {
    const int u = h - (p * g.st - g.pad);
    if (u < 0 || u >= g.r) continue;
    for (int q = q_lo; q <= q_hi; ++q) {
      const int v = w - (q * g.st - g.pad);
      if (v < 0 || v >= g.r) continue;
      const uint8_t tap = (uint8_t)(u * g.r + v);
      const int64_t oo = (((int64_t)n * g.P + p) * g.Q + q) * g.C + cg * 8;
      uint2 packed = *reinterpret_cast<const uint2*>(idx + oo);
      V8 gv = ld8(gp + oo);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        uint32_t word = k < 4 ? packed.x : packed.y;
        uint8_t b = (word >> (8 * (k & 3))) & 0xff;
        if (b == tap) ga[k] += gv.v[k];
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) ga[k] = rnd<__nv_bfloat16>(ga[k]);
}

__global__ void __launch_bounds__(256) pbn_partial(PoolGeom g, const __nv_bfloat16* __restrict__ gp,
                                                   const uint8_t* __restrict__ idx, const __nv_bfloat16* __restrict__ y,
                                                   const float* __restrict__ stat, const float* __restrict__ gamma,
                                                   const float* __restrict__ beta, float* __restrict__ part) {
  const int C = g.C, gC = C / 8, tpr = 256 / gC;
  const int t = threadIdx.x, cg = t % gC, rr = t / gC;
  const int64_t rows = (int64_t)g.N * g.H * g.W;
  const int64_t chunk = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * chunk, r1 = min(rows, r0 + chunk);
  float s[8] = {}, q[8] = {};
  if (rr < tpr)
    for (int64_t r = r0 + rr; r < r1; r += tpr) {
      const int w = (int)(r % g.W);
      const int h = (int)((r / g.W) % g.H);
      const int n = (int)(r / ((int64_t)g.W * g.H));
      float ga[8];
      pooled_grad8(g, n, h, w, cg, gp, idx, ga);
      V8 yv = ld8(y + r * C + cg * 8);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int c = cg * 8 + k;
        const float xh = (yv.v[k] - stat[c]) * stat[C + c];
        const float z = fmaf(gamma[c], xh, beta[c]);
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

__global__ void pbn_apply(PoolGeom g, const __nv_bfloat16* __restrict__ gp, const uint8_t* __restrict__ idx,
                          __nv_bfloat16* y, const float* __restrict__ stat, const float* __restrict__ gamma,
                          const float* __restrict__ beta, const float* __restrict__ dgamma,
                          const float* __restrict__ dbeta, float inv_n) {
  const int C = g.C, gC = C / 8;
  const int64_t total = (int64_t)g.N * g.H * g.W * gC;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int cg = (int)(i % gC);
    const int64_t r = i / gC;
    const int w = (int)(r % g.W);
    const int h = (int)((r / g.W) % g.H);
    const int n = (int)(r / ((int64_t)g.W * g.H));
    float ga[8];
    pooled_grad8(g, n, h, w, cg, gp, idx, ga);
    V8 yv = ld8(y + r * C + cg * 8);
    V8 dy;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int c = cg * 8 + k;
      const float xh = (yv.v[k] - stat[c]) * stat[C + c];
      const float z = fmaf(gamma[c], xh, beta[c]);
      const float dz = z > 0.f ? ga[k] : 0.f;
      dy.v[k] = gamma[c] * stat[C + c] * (dz - dbeta[c] * inv_n - xh * dgamma[c] * inv_n);
    }
    st8(y + r * C + cg * 8, dy);   // in place: each thread reads only its own y
  }
}

enum { PB_G, PB_IDX, PB_Y, PB_STAT, PB_GAMMA, PB_BETA, PB_DGAMMA, PB_DBETA };
PoolGeom geom(const OpArgs& a) {
  return PoolGeom{(int)A(a, "N"), (int)A(a, "H"), (int)A(a, "W"), (int)A(a, "C"), (int)A(a, "r"),
                  (int)A(a, "stride"), (int)A(a, "pad"), (int)A(a, "P"), (int)A(a, "Q")};
}
Status pool_bn_bwd_reduce(OpArgs& a) {
  PoolGeom g = geom(a);
  const int64_t rows = (int64_t)g.N * g.H * g.W;
  const int nblk = (int)std::min<int64_t>(kStatBlocks, std::max<int64_t>(1, rows / 64));
  pbn_partial<<<nblk, 256, 256 * 16 * 4, a.stream>>>(g, (const __nv_bfloat16*)a.p(PB_G), (const uint8_t*)a.p(PB_IDX),
                                                     (const __nv_bfloat16*)a.p(PB_Y), (const float*)a.p(PB_STAT),
                                                     (const float*)a.p(PB_GAMMA), (const float*)a.p(PB_BETA),
                                                     (float*)a.ws);
  OC_LAUNCH_CHECK(a);
  bnb_finalize<<<(g.C + 7) / 8, 256, 0, a.stream>>>(nblk, g.C, (const float*)a.ws, (float*)a.p(PB_DGAMMA),
                                                        (float*)a.p(PB_DBETA));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
Status pool_bn_bwd_apply(OpArgs& a) {
  PoolGeom g = geom(a);
  const int64_t rows = (int64_t)g.N * g.H * g.W;
  const int64_t total = rows * (g.C / 8);
  pbn_apply<<<grid_for(total, 256, 2), 256, 0, a.stream>>>(
      g, (const __nv_bfloat16*)a.p(PB_G), (const uint8_t*)a.p(PB_IDX), (__nv_bfloat16*)a.p(PB_Y),
      (const float*)a.p(PB_STAT), (const float*)a.p(PB_GAMMA), (const float*)a.p(PB_BETA),
      (const float*)a.p(PB_DGAMMA), (const float*)a.p(PB_DBETA), 1.f / (float)rows);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

// ---------------------------------------------------------------- global average pool
__global__ void gap_fwd_k(int N, int HW, int C, const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N * C) return;
  const int n = i / C, c = i % C;
  float s = 0.f;
  for (int k = 0; k < HW; ++k) s += __bfloat162float(x[((int64_t)n * HW + k) * C + c]);
  out[i] = __float2bfloat16_rn(s / (float)HW);
}
__global__ void gap_bwd_k(int N, int HW, int C, const __nv_bfloat16* __restrict__ g, __nv_bfloat16* __restrict__ dx) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)N * HW * C) return;
  const int c = (int)(i % C);
  const int n = (int)(i / ((int64_t)HW * C));
  dx[i] = __float2bfloat16_rn(__bfloat162float(g[(int64_t)n * C + c]) / (float)HW);
}
Status gap_fwd(OpArgs& a) {
  const int N = (int)A(a, "N"), HW = (int)A(a, "HW"), C = (int)A(a, "C");
  gap_fwd_k<<<(N * C + 255) / 256, 256, 0, a.stream>>>(N, HW, C, (const __nv_bfloat16*)a.p(0), (__nv_bfloat16*)a.p(1));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
Status gap_bwd(OpArgs& a) {
  const int N = (int)A(a, "N"), HW = (int)A(a, "HW"), C = (int)A(a, "C");
  const int64_t tot = (int64_t)N * HW * C;
  gap_bwd_k<<<(int)((tot + 255) / 256), 256, 0, a.stream>>>(N, HW, C, (const __nv_bfloat16*)a.p(0),
                                                            (__nv_bfloat16*)a.p(1));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

}  // namespace

extern const OpDesc kBnFwd{"bn_fwd", {"y", "stat", "gamma", "beta", "res", "out"}, bn_fwd, bn_ws};
extern const OpDesc kBnBwdReduce{"bn_bwd_reduce", {"g", "out", "y", "stat", "gamma", "dgamma", "dbeta"},
                                 bn_bwd_reduce, bn_ws};
extern const OpDesc kBnBwdApply{"bn_bwd_apply", {"g", "out", "y", "stat", "gamma", "dgamma", "dbeta"}, bn_bwd_apply,
                                nullptr};
extern const OpDesc kBnReluPoolFwd{"bn_relu_pool_fwd", {"y", "stat", "gamma", "beta", "out", "idx"}, bn_relu_pool_fwd,
                                   rp_ws};
extern const OpDesc kPoolBnBwdReduce{"pool_bn_bwd_reduce",
                                     {"g", "idx", "y", "stat", "gamma", "beta", "dgamma", "dbeta"},
                                     pool_bn_bwd_reduce, rp_ws};
extern const OpDesc kPoolBnBwdApply{"pool_bn_bwd_apply", {"g", "idx", "y", "stat", "gamma", "beta", "dgamma", "dbeta"},
                                    pool_bn_bwd_apply, nullptr};
extern const OpDesc kGapFwd{"gap_fwd", {"x", "out"}, gap_fwd, nullptr};
extern const OpDesc kGapBwd{"gap_bwd", {"g", "dx"}, gap_bwd, nullptr};

}  // namespace oc
