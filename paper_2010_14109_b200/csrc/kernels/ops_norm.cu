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
#include "tc_util.cuh"

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

// ---- stem geometry (3×3 / stride 2 / pad 1 over an even H × W map, P = H/2,
// Q = W/2) staged by whole image rows: NHWC makes an image row one contiguous
// W·C·sizeof(T) run, so a block's operands arrive as a few 1-D bulk copies
// (cp.async.bulk, completion on one mbarrier) — every byte in flight at once
// without registers, which the per-thread 16-byte loads of the round-1
// kernels (0.26-0.39 of HBM) did not reach.
inline bool stem_pool(const PoolGeom& g) {
  return g.r == 3 && g.st == 2 && g.pad == 1 && g.H % 2 == 0 && g.W % 2 == 0 && g.P == g.H / 2 && g.Q == g.W / 2;
}
constexpr int kRowSmemMax = 200 * 1024;
template <typename T>
inline bool rows_fit(const PoolGeom& g, int bytes) {
  return stem_pool(g) && g.C % 8 == 0 && 256 % (g.C / 8) == 0 && ((size_t)g.Q * g.C) % 16 == 0 &&
         ((size_t)g.W * g.C * sizeof(T)) % 16 == 0 && bytes <= kRowSmemMax;
}
template <typename T>
inline int fwd_rows_smem(const PoolGeom& g) { return 3 * g.W * g.C * (int)sizeof(T) + 16; }
// one stage of the backward: y rows 2i, 2i+1; gp and idx rows i, i+1
template <typename T>
__host__ __device__ inline int bwd_stage_bytes(const PoolGeom& g) {
  return 2 * g.W * g.C * (int)sizeof(T) + 2 * g.Q * g.C * (int)sizeof(T) + 2 * g.Q * g.C;
}

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(tcu::smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bar_init_one(uint64_t* bar) {
  tcu::mbar_init(bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// out[n,p,q,c] = max over the 3×3 window of rnd(relu(bn(y))) (first max, row-major
// taps, padding excluded); block = one output row p: input rows 2p−1..2p+1 are
// bulk-loaded, BN-ReLU-rounded once per element in place (the missing row −1 as
// −inf, which never wins the first-max rule), then pooled from shared memory
template <typename T>
__global__ void __launch_bounds__(256) bn_relu_pool_rows(PoolGeom g, const T* __restrict__ y,
                                                         const float* __restrict__ stat,
                                                         const float* __restrict__ gamma,
                                                         const float* __restrict__ beta, T* __restrict__ out,
                                                         uint8_t* __restrict__ idx) {
  extern __shared__ __align__(128) uint8_t rsm[];
  T* rows = reinterpret_cast<T*>(rsm);
  const int C = g.C, gC = C / 8, W = g.W;
  const int rowe = W * C;
  uint64_t* bar = reinterpret_cast<uint64_t*>(rsm + 3 * rowe * sizeof(T));
  const int n = blockIdx.x / g.P, p = blockIdx.x % g.P, h0 = 2 * p - 1;
  if (threadIdx.x == 0) bar_init_one(bar);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t rb = (uint32_t)(rowe * sizeof(T));
    tcu::mbar_expect_tx(bar, (h0 < 0 ? 2u : 3u) * rb);
    for (int r = h0 < 0 ? 1 : 0; r < 3; ++r)
      bulk_load(tcu::smem_u32(rows) + r * rb, y + ((int64_t)n * g.H + h0 + r) * rowe, rb, bar);
  }
  const int cg = threadIdx.x % gC;   // fixed: 256 is a multiple of C/8
  float gm[8], bt[8], mu[8], rs[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = cg * 8 + k;
    gm[k] = gamma[c]; bt[k] = beta[c]; mu[k] = stat[c]; rs[k] = stat[C + c];
  }
  tcu::mbar_wait(bar, 0);
  for (int e = threadIdx.x; e < 3 * W * gC; e += 256) {
    T* at = rows + (int64_t)e * 8;
    V8 z;
    if (h0 + e / (W * gC) >= 0) {
      const V8 x = ld8(at);
#pragma unroll
      for (int k = 0; k < 8; ++k) z.v[k] = fmaxf(fmaf(gm[k], (x.v[k] - mu[k]) * rs[k], bt[k]), 0.f);
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) z.v[k] = -INFINITY;
    }
    st8(at, z);   // rounded to T once per element
  }
  __syncthreads();
  for (int e = threadIdx.x; e < g.Q * gC; e += 256) {
    const int q = e / gC;
    const int64_t oo = (((int64_t)n * g.P + p) * g.Q + q) * C + cg * 8;
    if constexpr (sizeof(T) == 2) {
      // bf16 pairs: z > best as a 16-bit lane mask, max, and the tap index
      // selected per lane (exact: comparisons of stored bf16 values), about a
      // third of the instructions of the per-channel fp32 loop (the kernel is
      // issue-bound, ncu: SM throughput 80 % at 0.35 of HBM)
      __nv_bfloat162 best[4];
      uint32_t bi[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) { best[k] = __floats2bfloat162_rn(-INFINITY, -INFINITY); bi[k] = 0; }
#pragma unroll
      for (int u = 0; u < 3; ++u)
#pragma unroll
        for (int v = 0; v < 3; ++v) {
          const int w = 2 * q - 1 + v;
          if (w < 0) continue;
          const uint4 c4 = *reinterpret_cast<const uint4*>(rows + ((int64_t)u * W + w) * C + cg * 8);
          const __nv_bfloat162* z2 = reinterpret_cast<const __nv_bfloat162*>(&c4);
          const uint32_t tap2 = (uint32_t)(u * 3 + v) * 0x00010001u;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t m = __hgt2_mask(z2[k], best[k]);
            best[k] = __hmax2(z2[k], best[k]);
            bi[k] = (m & tap2) | (~m & bi[k]);
          }
        }
      *reinterpret_cast<uint4*>(out + oo) = *reinterpret_cast<const uint4*>(best);
      uint2 packed;
      packed.x = __byte_perm(bi[0], bi[1], 0x6420);
      packed.y = __byte_perm(bi[2], bi[3], 0x6420);
      *reinterpret_cast<uint2*>(idx + oo) = packed;
      continue;
    }
    float best[8];
    uint8_t bi[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { best[k] = -INFINITY; bi[k] = 0; }
#pragma unroll
    for (int u = 0; u < 3; ++u)
#pragma unroll
      for (int v = 0; v < 3; ++v) {
        const int w = 2 * q - 1 + v;
        if (w < 0) continue;
        const V8 z = ld8(rows + ((int64_t)u * W + w) * C + cg * 8);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (z.v[k] > best[k]) { best[k] = z.v[k]; bi[k] = (uint8_t)(u * 3 + v); }
      }
    V8 o;
#pragma unroll
    for (int k = 0; k < 8; ++k) o.v[k] = best[k];
    st8(out + oo, o);
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
  if (rows_fit<T>(g, fwd_rows_smem<T>(g))) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(bn_relu_pool_rows<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRowSmemMax);
      attr = true;
    }
    bn_relu_pool_rows<T><<<(unsigned)(g.N * g.P), 256, fwd_rows_smem<T>(g), a.stream>>>(
        g, y, (const float*)a.p(RP_STAT), (const float*)a.p(RP_GAMMA), (const float*)a.p(RP_BETA), (T*)a.p(RP_OUT),
        (uint8_t*)a.p(RP_IDX));
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

// Backward of the stem's BN-ReLU-maxpool, staged by image row pairs: unit
// (n, i) = input rows 2i, 2i+1, which only the windows of pooled rows i and
// i+1 reach.  A stage holds the two y rows, and gp / idx rows i, i+1 (row i+1
// absent for the last pair).  Thread item (j, cg) owns the 2×2 input block
// (2i..2i+1, 2j..2j+1) × 8 channels; windows are visited in (p, q) ascending
// order — the order pooled_grad8 sums them in, so the routed gradients are
// bitwise those of the generic kernels.
template <typename T>
struct RowStage {
  T* y;          // [2][W][C]
  T* gp;         // [2][Q][C]
  uint8_t* ix;   // [2][Q][C]
  __device__ RowStage(uint8_t* base, const PoolGeom& g) {
    y = reinterpret_cast<T*>(base);
    gp = y + 2 * g.W * g.C;
    ix = reinterpret_cast<uint8_t*>(gp + 2 * g.Q * g.C);
  }
};
// thread 0: bulk loads of unit u = n·P + i into the stage, completion on bar
template <typename T>
__device__ __forceinline__ void issue_rows(const PoolGeom& g, int64_t u, const RowStage<T>& s, uint64_t* bar,
                                           const T* __restrict__ y, const T* __restrict__ gp,
                                           const uint8_t* __restrict__ idx) {
  const int i = (int)(u % g.P);
  const int two = i + 1 < g.P ? 2 : 1;
  const uint32_t yb = 2u * g.W * g.C * sizeof(T), gb = (uint32_t)(g.Q * g.C * sizeof(T)), ib = (uint32_t)(g.Q * g.C);
  tcu::mbar_expect_tx(bar, yb + two * (gb + ib));
  bulk_load(tcu::smem_u32(s.y), y + u * 2 * g.W * g.C, yb, bar);   // rows 2i, 2i+1 of image n = rows 2u, 2u+1
  bulk_load(tcu::smem_u32(s.gp), gp + u * g.Q * g.C, two * gb, bar);
  bulk_load(tcu::smem_u32(s.ix), idx + u * g.Q * g.C, two * ib, bar);
}
// routed gradient of the 2×2 block (2i.., 2j..) from the staged windows (rows
// i, i+1), pixel by pixel: with stride 2 and pad 1 each block pixel is reached
// by fixed (window, tap) pairs — (0,0) ← (i,j) tap 4; (0,1) ← (i,j) 5,
// (i,j+1) 3; (1,0) ← (i,j) 7, (i+1,j) 1; (1,1) ← (i,j) 8, (i,j+1) 6, (i+1,j) 2,
// (i+1,j+1) 0 — summed in that (p, q) ascending order, the order pooled_grad8
// uses; 9 compare-adds per channel instead of decoding every window's taps
template <typename T>
__device__ __forceinline__ void block_grad_smem(const PoolGeom& g, bool last_row, int j, int cg,
                                                const RowStage<T>& s, float ga[4][8]) {
  const bool has_r = !last_row, has_c = j + 1 < g.Q;
  const int o00 = j * g.C + cg * 8, o01 = o00 + g.C, o10 = o00 + g.Q * g.C, o11 = o10 + g.C;
  const uint2 i00 = *reinterpret_cast<const uint2*>(s.ix + o00);
  const uint2 i01 = has_c ? *reinterpret_cast<const uint2*>(s.ix + o01) : make_uint2(~0u, ~0u);
  const uint2 i10 = has_r ? *reinterpret_cast<const uint2*>(s.ix + o10) : make_uint2(~0u, ~0u);
  const uint2 i11 = has_r && has_c ? *reinterpret_cast<const uint2*>(s.ix + o11) : make_uint2(~0u, ~0u);
  const V8 g00 = ld8(s.gp + o00);
  V8 g01, g10, g11;
#pragma unroll
  for (int k = 0; k < 8; ++k) g01.v[k] = g10.v[k] = g11.v[k] = 0.f;
  if (has_c) g01 = ld8(s.gp + o01);
  if (has_r) g10 = ld8(s.gp + o10);
  if (has_r && has_c) g11 = ld8(s.gp + o11);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int sh = 8 * (k & 3);
    const uint32_t t00 = ((k < 4 ? i00.x : i00.y) >> sh) & 0xff, t01 = ((k < 4 ? i01.x : i01.y) >> sh) & 0xff;
    const uint32_t t10 = ((k < 4 ? i10.x : i10.y) >> sh) & 0xff, t11 = ((k < 4 ? i11.x : i11.y) >> sh) & 0xff;
    float a = 0.f;
    if (t00 == 4) a += g00.v[k];
    ga[0][k] = a;
    a = 0.f;
    if (t00 == 5) a += g00.v[k];
    if (t01 == 3) a += g01.v[k];
    ga[1][k] = a;
    a = 0.f;
    if (t00 == 7) a += g00.v[k];
    if (t10 == 1) a += g10.v[k];
    ga[2][k] = a;
    a = 0.f;
    if (t00 == 8) a += g00.v[k];
    if (t01 == 6) a += g01.v[k];
    if (t10 == 2) a += g10.v[k];
    if (t11 == 0) a += g11.v[k];
    ga[3][k] = a;
  }
#pragma unroll
  for (int px = 0; px < 4; ++px)
#pragma unroll
    for (int k = 0; k < 8; ++k) ga[px][k] = rnd<T>(ga[px][k]);
}

// dγ, dβ partials: grid = stat_blocks(rows) persistent blocks, each over a
// contiguous chunk of row pairs through a two-stage ring (the next pair's
// copies in flight while this one is reduced); fixed chunking and fixed-order
// block sums keep the result bitwise reproducible
template <typename T>
__global__ void __launch_bounds__(256, 2) pbn_partial_rows(PoolGeom g, const T* __restrict__ gp,
                                                        const uint8_t* __restrict__ idx, const T* __restrict__ y,
                                                        const float* __restrict__ stat,
                                                        const float* __restrict__ gamma,
                                                        const float* __restrict__ beta, float* __restrict__ part) {
  extern __shared__ __align__(128) uint8_t rsm[];
  const int C = g.C, gC = C / 8, tpr = 256 / gC;
  const int t = threadIdx.x, cg = t % gC;
  const int sb = bwd_stage_bytes<T>(g);
  uint64_t* bar = reinterpret_cast<uint64_t*>(rsm + 2 * sb);
  const int64_t units = (int64_t)g.N * g.P;
  const int64_t chunk = (units + gridDim.x - 1) / gridDim.x;
  const int64_t u0 = blockIdx.x * chunk, u1 = min(units, u0 + chunk);
  if (t == 0) { bar_init_one(&bar[0]); bar_init_one(&bar[1]); }
  __syncthreads();
  if (t == 0)
    for (int k = 0; k < 2; ++k)
      if (u0 + k < u1) issue_rows<T>(g, u0 + k, RowStage<T>(rsm + k * sb, g), &bar[k], y, gp, idx);
  float s[8] = {}, q[8] = {};
  float mu[8], rs[8], gm[8], bt[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = cg * 8 + k;
    mu[k] = stat[c]; rs[k] = stat[C + c]; gm[k] = gamma[c]; bt[k] = beta[c];
  }
  for (int64_t u = u0; u < u1; ++u) {
    const int k2 = (int)((u - u0) & 1);
    tcu::mbar_wait(&bar[k2], (uint32_t)(((u - u0) >> 1) & 1));
    const RowStage<T> S(rsm + k2 * sb, g);
    const bool last_row = (int)(u % g.P) + 1 >= g.P;
    for (int e = t; e < g.Q * gC; e += 256) {
      const int j = e / gC;
      float ga[4][8];
      block_grad_smem<T>(g, last_row, j, cg, S, ga);
#pragma unroll
      for (int px = 0; px < 4; ++px) {
        const V8 yv = ld8(S.y + ((px >> 1) * g.W + 2 * j + (px & 1)) * C + cg * 8);
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
    __syncthreads();   // stage k2 fully read
    if (t == 0 && u + 2 < u1) {
      tcu::fence_async_smem();
      issue_rows<T>(g, u + 2, S, &bar[k2], y, gp, idx);
    }
  }
  float* sm = reinterpret_cast<float*>(rsm);   // the stages are idle now
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

// dy = γ·rstd·(dz − dβ/n − x̂·dγ/n) written over y: persistent blocks over
// contiguous chunks of row pairs through the same two-stage ring; a block
// reads only its own staged copy of its rows of y, so the in-place global
// write never races a reader
template <typename T>
__global__ void __launch_bounds__(256, 2) pbn_apply_rows(PoolGeom g, const T* __restrict__ gp,
                                                         const uint8_t* __restrict__ idx, T* y,
                                                         const float* __restrict__ stat,
                                                         const float* __restrict__ gamma,
                                                         const float* __restrict__ beta,
                                                         const float* __restrict__ dgamma,
                                                         const float* __restrict__ dbeta, float inv_n) {
  extern __shared__ __align__(128) uint8_t rsm[];
  const int C = g.C, gC = C / 8;
  const int t = threadIdx.x, cg = t % gC;
  const int sb = bwd_stage_bytes<T>(g);
  uint64_t* bar = reinterpret_cast<uint64_t*>(rsm + 2 * sb);
  const int64_t units = (int64_t)g.N * g.P;
  const int64_t chunk = (units + gridDim.x - 1) / gridDim.x;
  const int64_t u0 = blockIdx.x * chunk, u1 = min(units, u0 + chunk);
  if (t == 0) { bar_init_one(&bar[0]); bar_init_one(&bar[1]); }
  __syncthreads();
  if (t == 0)
    for (int k = 0; k < 2; ++k)
      if (u0 + k < u1) issue_rows<T>(g, u0 + k, RowStage<T>(rsm + k * sb, g), &bar[k], y, gp, idx);
  float mu[8], rs[8], gm[8], bt[8], dg[8], db[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = cg * 8 + k;
    mu[k] = stat[c]; rs[k] = stat[C + c]; gm[k] = gamma[c]; bt[k] = beta[c]; dg[k] = dgamma[c]; db[k] = dbeta[c];
  }
  for (int64_t u = u0; u < u1; ++u) {
    const int k2 = (int)((u - u0) & 1);
    tcu::mbar_wait(&bar[k2], (uint32_t)(((u - u0) >> 1) & 1));
    const RowStage<T> S(rsm + k2 * sb, g);
    const bool last_row = (int)(u % g.P) + 1 >= g.P;
    T* yo = y + u * 2 * g.W * C;
    for (int e = t; e < g.Q * gC; e += 256) {
      const int j = e / gC;
      float ga[4][8];
      block_grad_smem<T>(g, last_row, j, cg, S, ga);
#pragma unroll
      for (int px = 0; px < 4; ++px) {
        const int o = ((px >> 1) * g.W + 2 * j + (px & 1)) * C + cg * 8;
        const V8 yv = ld8(S.y + o);
        V8 dy;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float xh = (yv.v[k] - mu[k]) * rs[k];
          const float z = fmaf(gm[k], xh, bt[k]);
          const float dz = z > 0.f ? ga[px][k] : 0.f;
          dy.v[k] = gm[k] * rs[k] * (dz - db[k] * inv_n - xh * dg[k] * inv_n);
        }
        st8(yo + o, dy);
      }
    }
    __syncthreads();   // stage k2 fully read
    if (t == 0 && u + 2 < u1) {
      tcu::fence_async_smem();
      issue_rows<T>(g, u + 2, S, &bar[k2], y, gp, idx);
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
  const int sb2 = 2 * bwd_stage_bytes<T>(g) + 16;
  if (rows_fit<T>(g, sb2) && 256 * 16 * 4 <= sb2) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(pbn_partial_rows<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRowSmemMax);
      attr = true;
    }
    pbn_partial_rows<T><<<nblk, 256, sb2, a.stream>>>(
        g, (const T*)a.p(PB_G), (const uint8_t*)a.p(PB_IDX), (const T*)a.p(PB_Y), (const float*)a.p(PB_STAT),
        (const float*)a.p(PB_GAMMA), (const float*)a.p(PB_BETA), (float*)a.ws);
  }
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
  const int sb1 = 2 * bwd_stage_bytes<T>(g) + 16;
  if (rows_fit<T>(g, sb1)) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(pbn_apply_rows<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRowSmemMax);
      attr = true;
    }
    const int64_t units = (int64_t)g.N * g.P;
    pbn_apply_rows<T><<<(unsigned)std::min<int64_t>(units, 2 * 148), 256, sb1, a.stream>>>(
        g, (const T*)a.p(PB_G), (const uint8_t*)a.p(PB_IDX), (T*)a.p(PB_Y), (const float*)a.p(PB_STAT),
        (const float*)a.p(PB_GAMMA), (const float*)a.p(PB_BETA), (const float*)a.p(PB_DGAMMA),
        (const float*)a.p(PB_DBETA), 1.f / (float)rows);
  }
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
