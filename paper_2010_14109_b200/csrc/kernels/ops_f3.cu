// Layer kernels of the paper's other two families (PAPER.md
// Pix2PixHD 512×1024, DeepLabv3+ 513×513): bilinear upsampling
// (DeepLabv3+ decoder, ASPP image pooling), instance normalisation and
// reflection padding (Pix2PixHD's generator) and the L1 loss of the
// synthetic Pix2PixHD step.  NHWC activations, bf16 (or fp32 in the parity
// mode); memory-bound — roofline: HBM, algorithmic bytes = one read of every
// input + one write of every output.  Every reduction runs in a fixed order
// (fixed row chunks → fp32 partials → fixed-order double finalize; gathers
// instead of scatters in the backward passes), so a step is bitwise
// reproducible whatever the swap schedule.  Definitions: oracle/numerics.py
// (upsample_bilinear, instance_norm, reflect_pad, l1_loss) and
// oracle/layerwise.py.
#include "common.cuh"

namespace oc {

namespace {

constexpr float kEps = 1e-5f;

// ---------------------------------------------------------------- bilinear
// 1-D weights, half-pixel centres (align_corners = false): output i samples
// src = max((i + 0.5)·n_in/n_out − 0.5, 0), i0 = floor(src), i1 = min(i0+1, n_in−1),
// λ = src − i0 (coordinates in double, as the oracle's definition)
__device__ __forceinline__ void bl_coeff(int i, int n_in, int n_out, int& i0, int& i1, float& lam) {
  double src = ((double)i + 0.5) * ((double)n_in / (double)n_out) - 0.5;
  if (src < 0) src = 0;
  int f = (int)floor(src);
  if (f > n_in - 1) f = n_in - 1;
  i0 = f;
  i1 = f + 1 < n_in ? f + 1 : n_in - 1;
  lam = (float)(src - (double)f);
}

template <typename T>
__global__ void __launch_bounds__(256) bl_fwd(int N, int H, int W, int C, int Ho, int Wo, const T* __restrict__ x,
                                              T* __restrict__ y) {
  const int64_t total = (int64_t)N * Ho * Wo * C;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    int64_t t = i / C;
    const int wo = (int)(t % Wo);
    t /= Wo;
    const int ho = (int)(t % Ho), n = (int)(t / Ho);
    int r0, r1, c0, c1;
    float a, b;
    bl_coeff(ho, H, Ho, r0, r1, a);
    bl_coeff(wo, W, Wo, c0, c1, b);
    const T* xn = x + (int64_t)n * H * W * C + c;
    const float v00 = ld_f(xn + ((int64_t)r0 * W + c0) * C), v01 = ld_f(xn + ((int64_t)r0 * W + c1) * C);
    const float v10 = ld_f(xn + ((int64_t)r1 * W + c0) * C), v11 = ld_f(xn + ((int64_t)r1 * W + c1) * C);
    // rows first, then columns (the oracle's separable order)
    const float top = v00 * (1.f - a) + v10 * a, bot = v01 * (1.f - a) + v11 * a;
    st_f(y + i, top * (1.f - b) + bot * b);
  }
}

// weight of output index o on input index j along one axis (0 if o does not read j)
__device__ __forceinline__ float bl_w(int o, int j, int n_in, int n_out) {
  int i0, i1;
  float lam;
  bl_coeff(o, n_in, n_out, i0, i1, lam);
  float w = 0.f;
  if (i0 == j) w += 1.f - lam;
  if (i1 == j) w += lam;
  return w;
}

// the output indices that can read input index j: o with src(o) in (j − 1, j + 1]
__device__ __forceinline__ void bl_range(int j, int n_in, int n_out, int& lo, int& hi) {
  const double s = (double)n_out / (double)n_in;
  lo = (int)floor(((double)j - 1.0 + 0.5) * s - 0.5) - 1;
  hi = (int)ceil(((double)j + 1.0 + 0.5) * s - 0.5) + 1;
  if (lo < 0) lo = 0;
  if (hi > n_out - 1) hi = n_out - 1;
}

// dx[n,h,w,c] = Σ_{ho,wo} wr(ho,h)·wc(wo,w)·g[n,ho,wo,c] — a gather in fixed
// (ho, wo) order per input pixel: deterministic
template <typename T>
__global__ void __launch_bounds__(256) bl_bwd(int N, int H, int W, int C, int Ho, int Wo, const T* __restrict__ g,
                                              T* dx, int acc) {
  const int64_t total = (int64_t)N * H * W * C;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    int64_t t = i / C;
    const int w = (int)(t % W);
    t /= W;
    const int h = (int)(t % H), n = (int)(t / H);
    int hl, hh, wl, wh;
    bl_range(h, H, Ho, hl, hh);
    bl_range(w, W, Wo, wl, wh);
    const T* gn = g + (int64_t)n * Ho * Wo * C + c;
    float s = 0.f;
    for (int ho = hl; ho <= hh; ++ho) {
      const float wr = bl_w(ho, h, H, Ho);
      if (wr == 0.f) continue;
      float row = 0.f;
      for (int wo = wl; wo <= wh; ++wo) {
        const float wc = bl_w(wo, w, W, Wo);
        if (wc != 0.f) row += wc * ld_f(gn + ((int64_t)ho * Wo + wo) * C);
      }
      s += wr * row;
    }
    if (acc) s += ld_f(dx + i);
    st_f(dx + i, s);
  }
}

template <typename T>
Status upsample_bilinear_fwd_t(OpArgs& a) {
  const int N = (int)A(a, "N"), H = (int)A(a, "H"), W = (int)A(a, "W"), C = (int)A(a, "C");
  const int Ho = (int)A(a, "Ho"), Wo = (int)A(a, "Wo");
  bl_fwd<T><<<grid_for((int64_t)N * Ho * Wo * C, 256, 4), 256, 0, a.stream>>>(N, H, W, C, Ho, Wo, (const T*)a.p(0),
                                                                               (T*)a.p(1));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
template <typename T>
Status upsample_bilinear_bwd_t(OpArgs& a) {
  const int N = (int)A(a, "N"), H = (int)A(a, "H"), W = (int)A(a, "W"), C = (int)A(a, "C");
  const int Ho = (int)A(a, "Ho"), Wo = (int)A(a, "Wo");
  bl_bwd<T><<<grid_for((int64_t)N * H * W * C, 256, 2), 256, 0, a.stream>>>(N, H, W, C, Ho, Wo, (const T*)a.p(0),
                                                                             (T*)a.p(1), Ab(a, "accumulate") ? 1 : 0);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

// ---------------------------------------------------------------- instance norm
// Statistics per (sample, channel) over the H·W positions.  Blocks own
// (sample, row chunk) pairs; thread t covers 8 channels of every
// (256/(C/8))-th row; partials [n][chunk][2][C] fp32, finalised in double in
// chunk order.  C % 8 == 0, C <= 2048.
constexpr int kInChunks = 128;  // row chunks per sample (fills the SMs at batch 1-2)

template <typename T, int MODE>   // MODE 0: Σx, Σx²   1: Σdz, Σdz·x̂ (mask x̂ > 0 if relu)
__global__ void __launch_bounds__(256) in_partial(int HW, int C, const T* __restrict__ x, const T* __restrict__ g,
                                                  const float* __restrict__ stat, int relu, float* __restrict__ part) {
  const int n = blockIdx.y, ch = blockIdx.x;
  const int gC = C / 8, tpr = 256 / gC;
  const int t = threadIdx.x, cg = t % gC, rr = t / gC;
  const int64_t chunk = (HW + kInChunks - 1) / kInChunks;
  const int64_t r0 = ch * chunk, r1 = min((int64_t)HW, r0 + chunk);
  float s[8] = {}, q[8] = {};
  float mu[8], rs[8];
  if (MODE == 1) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      mu[k] = stat[((int64_t)n * 2) * C + cg * 8 + k];
      rs[k] = stat[((int64_t)n * 2 + 1) * C + cg * 8 + k];
    }
  }
  const T* xn = x + (int64_t)n * HW * C;
  const T* gn = MODE == 1 ? g + (int64_t)n * HW * C : nullptr;
  if (rr < tpr)
    for (int64_t r = r0 + rr; r < r1; r += tpr) {
      const V8 xv = ld8(xn + r * C + cg * 8);
      if (MODE == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          s[k] += xv.v[k];
          q[k] = fmaf(xv.v[k], xv.v[k], q[k]);
        }
      } else {
        const V8 gv = ld8(gn + r * C + cg * 8);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float xh = (xv.v[k] - mu[k]) * rs[k];
          const float dz = (!relu || xh > 0.f) ? gv.v[k] : 0.f;
          s[k] += dz;
          q[k] = fmaf(dz, xh, q[k]);
        }
      }
    }
  extern __shared__ float sm[];
#pragma unroll
  for (int k = 0; k < 8; ++k) { sm[t * 16 + k] = s[k]; sm[t * 16 + 8 + k] = q[k]; }
  __syncthreads();
  float* pp = part + ((int64_t)n * kInChunks + ch) * 2 * C;
  for (int c = t; c < C; c += 256) {
    const int grp = c / 8, lane = c % 8;
    float as = 0.f, aq = 0.f;
    for (int k = 0; k < tpr; ++k) {
      as += sm[(k * gC + grp) * 16 + lane];
      aq += sm[(k * gC + grp) * 16 + 8 + lane];
    }
    pp[c] = as;
    pp[C + c] = aq;
  }
}

// MODE 0: stat[n] = [μ; rstd]; MODE 1: sums[n] = [Σdz; Σdz·x̂] (double, chunk order)
template <int MODE>
__global__ void in_finalize(int N, int HW, int C, const float* __restrict__ part, float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)N * C) return;
  const int n = (int)(i / C), c = (int)(i % C);
  double s = 0, q = 0;
  for (int ch = 0; ch < kInChunks; ++ch) {
    const float* pp = part + ((int64_t)n * kInChunks + ch) * 2 * C;
    s += pp[c];
    q += pp[C + c];
  }
  if (MODE == 0) {
    const double mu = s / HW, var = q / HW - mu * mu;
    out[((int64_t)n * 2) * C + c] = (float)mu;
    out[((int64_t)n * 2 + 1) * C + c] = (float)(1.0 / sqrt((var > 0 ? var : 0) + (double)kEps));
  } else {
    out[((int64_t)n * 2) * C + c] = (float)s;
    out[((int64_t)n * 2 + 1) * C + c] = (float)q;
  }
}

// MODE 0 (forward): out = rnd(relu?(x̂));  MODE 1 (backward):
// dx = rnd(rstd·(dz − Σdz/HW − x̂·Σdz·x̂/HW))  (+ dx when accumulating)
template <typename T, int MODE>
__global__ void __launch_bounds__(256) in_apply(int N, int HW, int C, const T* __restrict__ x, const T* __restrict__ g,
                                                const float* __restrict__ stat, const float* __restrict__ sums,
                                                int relu, T* out, int acc) {
  const int64_t n8 = (int64_t)N * HW * C / 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * 8;
    const int c0 = (int)(e % C);
    const int n = (int)(e / ((int64_t)HW * C));
    const V8 xv = ld8(x + e);
    V8 o;
    if (MODE == 0) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float xh = (xv.v[k] - stat[((int64_t)n * 2) * C + c0 + k]) * stat[((int64_t)n * 2 + 1) * C + c0 + k];
        o.v[k] = relu ? fmaxf(xh, 0.f) : xh;
      }
    } else {
      const V8 gv = ld8(g + e);
      const float inv = 1.f / (float)HW;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float mu = stat[((int64_t)n * 2) * C + c0 + k], rs = stat[((int64_t)n * 2 + 1) * C + c0 + k];
        const float xh = (xv.v[k] - mu) * rs;
        const float dz = (!relu || xh > 0.f) ? gv.v[k] : 0.f;
        const float sdz = sums[((int64_t)n * 2) * C + c0 + k], sdx = sums[((int64_t)n * 2 + 1) * C + c0 + k];
        o.v[k] = rs * (dz - sdz * inv - xh * (sdx * inv));
      }
      if (acc) {
        const V8 old = ld8(out + e);
#pragma unroll
        for (int k = 0; k < 8; ++k) o.v[k] += old.v[k];
      }
    }
    st8(out + e, o);
  }
}

size_t in_ws(const JVal& at) {
  return (size_t)at.geti("N") * kInChunks * 2 * at.geti("C") * 4 + (size_t)at.geti("N") * 2 * at.geti("C") * 4;
}

// roles: x, out, stat
template <typename T>
Status instnorm_fwd_t(OpArgs& a) {
  const int N = (int)A(a, "N"), HW = (int)A(a, "HW"), C = (int)A(a, "C");
  if (C % 8 || C > 2048) return Status::make(OC_E_UNSUPPORTED, "instance norm: C % 8 == 0, C <= 2048");
  if (a.ws_bytes < in_ws(*a.attrs)) return Status::make(OC_E_INVARIANT, "instance norm: workspace too small");
  float* part = (float*)a.ws;
  float* stat = (float*)a.p(2);
  in_partial<T, 0><<<dim3(kInChunks, N), 256, 256 * 16 * 4, a.stream>>>(HW, C, (const T*)a.p(0), nullptr, nullptr, 0,
                                                                         part);
  OC_LAUNCH_CHECK(a);
  in_finalize<0><<<(N * C + 255) / 256, 256, 0, a.stream>>>(N, HW, C, part, stat);
  OC_LAUNCH_CHECK(a);
  in_apply<T, 0><<<grid_for((int64_t)N * HW * C / 8, 256, 2), 256, 0, a.stream>>>(
      N, HW, C, (const T*)a.p(0), nullptr, stat, nullptr, Ab(a, "relu") ? 1 : 0, (T*)a.p(1), 0);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
// roles: g, x, stat, dx
template <typename T>
Status instnorm_bwd_t(OpArgs& a) {
  const int N = (int)A(a, "N"), HW = (int)A(a, "HW"), C = (int)A(a, "C");
  if (C % 8 || C > 2048) return Status::make(OC_E_UNSUPPORTED, "instance norm: C % 8 == 0, C <= 2048");
  if (a.ws_bytes < in_ws(*a.attrs)) return Status::make(OC_E_INVARIANT, "instance norm: workspace too small");
  float* part = (float*)a.ws;
  float* sums = part + (size_t)N * kInChunks * 2 * C;
  const int relu = Ab(a, "relu") ? 1 : 0;
  in_partial<T, 1><<<dim3(kInChunks, N), 256, 256 * 16 * 4, a.stream>>>(HW, C, (const T*)a.p(1), (const T*)a.p(0),
                                                                         (const float*)a.p(2), relu, part);
  OC_LAUNCH_CHECK(a);
  in_finalize<1><<<(N * C + 255) / 256, 256, 0, a.stream>>>(N, HW, C, part, sums);
  OC_LAUNCH_CHECK(a);
  in_apply<T, 1><<<grid_for((int64_t)N * HW * C / 8, 256, 2), 256, 0, a.stream>>>(
      N, HW, C, (const T*)a.p(1), (const T*)a.p(0), (const float*)a.p(2), sums, relu, (T*)a.p(3),
      Ab(a, "accumulate") ? 1 : 0);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

// ---------------------------------------------------------------- reflection padding
__device__ __forceinline__ int refl(int k, int n) {
  k = k < 0 ? -k : k;
  return k >= n ? 2 * (n - 1) - k : k;
}

template <typename T>
__global__ void __launch_bounds__(256) rp_fwd(int N, int H, int W, int C, int p, const T* __restrict__ x,
                                              T* __restrict__ y) {
  const int Hp = H + 2 * p, Wp = W + 2 * p, C8 = C / 8;
  const int64_t total = (int64_t)N * Hp * Wp * C8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(i % C8);
    int64_t t = i / C8;
    const int j = (int)(t % Wp);
    t /= Wp;
    const int r = (int)(t % Hp), n = (int)(t / Hp);
    const int h = refl(r - p, H), w = refl(j - p, W);
    *reinterpret_cast<uint4*>((char*)y + i * 8 * sizeof(T)) =
        *reinterpret_cast<const uint4*>((const char*)x + ((((int64_t)n * H + h) * W + w) * C + c8 * 8) * sizeof(T));
    if (sizeof(T) == 4)
      *reinterpret_cast<uint4*>((char*)y + i * 8 * sizeof(T) + 16) = *reinterpret_cast<const uint4*>(
          (const char*)x + ((((int64_t)n * H + h) * W + w) * C + c8 * 8) * sizeof(T) + 16);
  }
}

// padded positions of one axis that read input index h (in increasing order):
// h + p always; p − h (top reflection) for 1 <= h <= p; 2(n−1) − h + p (bottom)
// for n−1−p <= h <= n−2
__device__ __forceinline__ int rp_srcs(int h, int n, int p, int* out) {
  int k = 0;
  if (h >= 1 && h <= p) out[k++] = p - h;
  out[k++] = h + p;
  if (h >= n - 1 - p && h <= n - 2) out[k++] = 2 * (n - 1) - h + p;
  return k;
}

template <typename T>
__global__ void __launch_bounds__(256) rp_bwd(int N, int H, int W, int C, int p, const T* __restrict__ g, T* dx,
                                              int acc) {
  const int Hp = H + 2 * p, Wp = W + 2 * p, C8 = C / 8;
  const int64_t total = (int64_t)N * H * W * C8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(i % C8);
    int64_t t = i / C8;
    const int w = (int)(t % W);
    t /= W;
    const int h = (int)(t % H), n = (int)(t / H);
    int rs[3], cs[3];
    const int nr = rp_srcs(h, H, p, rs), nc = rp_srcs(w, W, p, cs);
    float s[8] = {};
    for (int a = 0; a < nr; ++a)
      for (int b = 0; b < nc; ++b) {
        const V8 v = ld8(g + (((int64_t)n * Hp + rs[a]) * Wp + cs[b]) * C + c8 * 8);
#pragma unroll
        for (int k = 0; k < 8; ++k) s[k] += v.v[k];
      }
    V8 o;
    const int64_t e = (((int64_t)n * H + h) * W + w) * C + c8 * 8;
    if (acc) {
      const V8 old = ld8(dx + e);
#pragma unroll
      for (int k = 0; k < 8; ++k) o.v[k] = s[k] + old.v[k];
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) o.v[k] = s[k];
    }
    st8(dx + e, o);
  }
}

// narrow tensors (C % 8 != 0: the 3-channel image): one element per thread
template <typename T>
__global__ void __launch_bounds__(256) rp_fwd1(int N, int H, int W, int C, int p, const T* __restrict__ x,
                                               T* __restrict__ y) {
  const int Hp = H + 2 * p, Wp = W + 2 * p;
  const int64_t total = (int64_t)N * Hp * Wp * C;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    int64_t t = i / C;
    const int j = (int)(t % Wp);
    t /= Wp;
    const int r = (int)(t % Hp), n = (int)(t / Hp);
    y[i] = x[(((int64_t)n * H + refl(r - p, H)) * W + refl(j - p, W)) * C + c];
  }
}
template <typename T>
__global__ void __launch_bounds__(256) rp_bwd1(int N, int H, int W, int C, int p, const T* __restrict__ g, T* dx,
                                               int acc) {
  const int Hp = H + 2 * p, Wp = W + 2 * p;
  const int64_t total = (int64_t)N * H * W * C;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    int64_t t = i / C;
    const int w = (int)(t % W);
    t /= W;
    const int h = (int)(t % H), n = (int)(t / H);
    int rs[3], cs[3];
    const int nr = rp_srcs(h, H, p, rs), nc = rp_srcs(w, W, p, cs);
    float s = 0.f;
    for (int a = 0; a < nr; ++a)
      for (int b = 0; b < nc; ++b) s += ld_f(g + (((int64_t)n * Hp + rs[a]) * Wp + cs[b]) * C + c);
    if (acc) s += ld_f(dx + i);
    st_f(dx + i, s);
  }
}

template <typename T>
Status reflect_pad_fwd_t(OpArgs& a) {
  const int N = (int)A(a, "N"), H = (int)A(a, "H"), W = (int)A(a, "W"), C = (int)A(a, "C"), p = (int)A(a, "pad");
  if (p >= H || p >= W) return Status::make(OC_E_UNSUPPORTED, "reflect pad: pad < H, W");
  if (C % 8) {
    rp_fwd1<T><<<grid_for((int64_t)N * (H + 2 * p) * (W + 2 * p) * C, 256, 4), 256, 0, a.stream>>>(
        N, H, W, C, p, (const T*)a.p(0), (T*)a.p(1));
  } else {
    const int64_t n = (int64_t)N * (H + 2 * p) * (W + 2 * p) * (C / 8);
    rp_fwd<T><<<grid_for(n, 256, 4), 256, 0, a.stream>>>(N, H, W, C, p, (const T*)a.p(0), (T*)a.p(1));
  }
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
template <typename T>
Status reflect_pad_bwd_t(OpArgs& a) {
  const int N = (int)A(a, "N"), H = (int)A(a, "H"), W = (int)A(a, "W"), C = (int)A(a, "C"), p = (int)A(a, "pad");
  if (p >= H || p >= W) return Status::make(OC_E_UNSUPPORTED, "reflect pad: pad < H, W");
  const int acc = Ab(a, "accumulate") ? 1 : 0;
  if (C % 8)
    rp_bwd1<T><<<grid_for((int64_t)N * H * W * C, 256, 2), 256, 0, a.stream>>>(N, H, W, C, p, (const T*)a.p(0),
                                                                               (T*)a.p(1), acc);
  else
    rp_bwd<T><<<grid_for((int64_t)N * H * W * (C / 8), 256, 2), 256, 0, a.stream>>>(N, H, W, C, p, (const T*)a.p(0),
                                                                                     (T*)a.p(1), acc);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

// ---------------------------------------------------------------- L1 loss
// loss = mean |y − t| (per-block partial sums, then a fixed-order double sum),
// dy = rnd(sign(y − t)/count)
constexpr int kL1Blocks = 148 * 4;
template <typename T>
__global__ void __launch_bounds__(256) l1_k(int64_t n, const T* __restrict__ y, const T* __restrict__ t, T* dy,
                                            float inv, float* __restrict__ part) {
  float s = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float d = ld_f(y + i) - ld_f(t + i);
    s += fabsf(d);
    st_f(dy + i, d > 0.f ? inv : (d < 0.f ? -inv : 0.f));
  }
  __shared__ float red[8];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float b = 0.f;
    for (int k = 0; k < 8; ++k) b += red[k];
    part[blockIdx.x] = b;
  }
}
__global__ void l1_final(int nblk, const float* __restrict__ part, double inv, float* loss) {
  double s = 0;
  for (int k = 0; k < nblk; ++k) s += part[k];
  loss[0] = (float)(s * inv);
}
// roles: y, target, loss, dy
template <typename T>
Status l1_loss_t(OpArgs& a) {
  const int64_t n = A(a, "n");
  if (a.ws_bytes < (size_t)kL1Blocks * 4) return Status::make(OC_E_INVARIANT, "l1: workspace too small");
  l1_k<T><<<kL1Blocks, 256, 0, a.stream>>>(n, (const T*)a.p(0), (const T*)a.p(1), (T*)a.p(3), 1.f / (float)n,
                                           (float*)a.ws);
  OC_LAUNCH_CHECK(a);
  l1_final<<<1, 1, 0, a.stream>>>(kL1Blocks, (const float*)a.ws, 1.0 / (double)n, (float*)a.p(2));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
size_t l1_ws(const JVal&) { return (size_t)kL1Blocks * 4; }

#define OC_F3_DISPATCH(name)                                                                      \
  Status name(OpArgs& a) {                                                                        \
    return As(a, "dtype", "bf16") == "f32" ? name##_t<float>(a) : name##_t<__nv_bfloat16>(a);    \
  }
OC_F3_DISPATCH(upsample_bilinear_fwd)
OC_F3_DISPATCH(upsample_bilinear_bwd)
OC_F3_DISPATCH(instnorm_fwd)
OC_F3_DISPATCH(instnorm_bwd)
OC_F3_DISPATCH(reflect_pad_fwd)
OC_F3_DISPATCH(reflect_pad_bwd)
OC_F3_DISPATCH(l1_loss)

}  // namespace

extern const OpDesc kUpsampleBilinearFwd{"upsample_bilinear_fwd", {"x", "y"}, upsample_bilinear_fwd, nullptr};
extern const OpDesc kUpsampleBilinearBwd{"upsample_bilinear_bwd", {"g", "dx"}, upsample_bilinear_bwd, nullptr};
extern const OpDesc kInstnormFwd{"instnorm_fwd", {"x", "out", "stat"}, instnorm_fwd, in_ws};
extern const OpDesc kInstnormBwd{"instnorm_bwd", {"g", "x", "stat", "dx"}, instnorm_bwd, in_ws};
extern const OpDesc kReflectPadFwd{"reflect_pad_fwd", {"x", "y"}, reflect_pad_fwd, nullptr};
extern const OpDesc kReflectPadBwd{"reflect_pad_bwd", {"g", "dx"}, reflect_pad_bwd, nullptr};
extern const OpDesc kL1Loss{"l1_loss", {"y", "target", "loss", "dy"}, l1_loss, l1_ws};

}  // namespace oc
