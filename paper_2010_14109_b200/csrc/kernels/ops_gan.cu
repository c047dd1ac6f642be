// Kernels of the BigGAN-style GAN step (configs[4]): nearest
// ×2 upsampling, 2×2 average pooling, ReLU, tanh, batch concatenation, the
// learned-gain residual of self-attention, SAGAN attention and the hinge
// losses.  Activations bf16 (or fp32 in the parity mode), NHWC; the numerics
// contract is oracle/numerics.py (GAN layers): a tensor with several gradient
// contributions accumulates G = rnd(c_first), then G = rnd(G + c).
//
// Attention (per sample, L = H·W positions): S = q kᵀ (fp32, workspace),
// P = rnd(softmax_rows(S)) stored as an activation (the L×L map the config
// is meant to swap), o = rnd(P v); backward dv = rnd(Pᵀ do), dP = do vᵀ
// (fp32), dS = P ⊙ (dP − rowsum), rowsum_i = do_i·o_i, dq = rnd(dS k),
// dk = rnd(dSᵀ q).  bf16: the products run on the tensor cores (gemm_tc.cuh;
// dS as an exact bf16 hi + lo pair); fp32 parity mode: the batched SIMT GEMM
// (gemm_simt.cuh, exact FFMA).  Samples go through the fp32 L×L workspace a
// few at a time.
#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "gemm_simt.cuh"
#include "gemm_tc.cuh"

namespace oc {

namespace {

using simt::gemm;

// ---------------------------------------------------------------- upsample ×2 (nearest)
template <typename T>
__global__ void up2_fwd_k(int64_t n8, int H, int W, int C8, const T* __restrict__ x, T* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(i % C8);
    int64_t t = i / C8;
    const int ow = (int)(t % (2 * W));
    t /= 2 * W;
    const int oh = (int)(t % (2 * H));
    const int64_t n = t / (2 * H);
    st8(y + i * 8, ld8(x + (((n * H + oh / 2) * W + ow / 2) * C8 + c8) * 8));
  }
}
// dx = ((g00 + g01) + g10) + g11, rounded; accumulating: rnd(dx + Σ)
template <typename T>
__global__ void up2_bwd_k(int64_t n8, int H, int W, int C8, const T* __restrict__ g, T* dx, int acc) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(i % C8);
    int64_t t = i / C8;
    const int w = (int)(t % W);
    t /= W;
    const int h = (int)(t % H);
    const int64_t n = t / H;
    auto at = [&](int a, int b) { return ld8(g + (((n * 2 * H + 2 * h + a) * 2 * W + 2 * w + b) * C8 + c8) * 8); };
    const V8 g00 = at(0, 0), g01 = at(0, 1), g10 = at(1, 0), g11 = at(1, 1);
    V8 s;
#pragma unroll
    for (int k = 0; k < 8; ++k) s.v[k] = ((g00.v[k] + g01.v[k]) + g10.v[k]) + g11.v[k];
    if (acc) {
      const V8 o = ld8(dx + i * 8);
#pragma unroll
      for (int k = 0; k < 8; ++k) s.v[k] += o.v[k];
    }
    st8(dx + i * 8, s);
  }
}

// ---------------------------------------------------------------- 2×2 average pool
template <typename T>
__global__ void ap2_fwd_k(int64_t n8, int H, int W, int C8, const T* __restrict__ x, T* __restrict__ y) {
  const int P = H / 2, Q = W / 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(i % C8);
    int64_t t = i / C8;
    const int q = (int)(t % Q);
    t /= Q;
    const int p = (int)(t % P);
    const int64_t n = t / P;
    auto at = [&](int a, int b) { return ld8(x + (((n * H + 2 * p + a) * W + 2 * q + b) * C8 + c8) * 8); };
    const V8 x00 = at(0, 0), x01 = at(0, 1), x10 = at(1, 0), x11 = at(1, 1);
    V8 s;
#pragma unroll
    for (int k = 0; k < 8; ++k) s.v[k] = 0.25f * (((x00.v[k] + x01.v[k]) + x10.v[k]) + x11.v[k]);
    st8(y + i * 8, s);
  }
}
// dx[2p+a, 2q+b] = ¼ g[p, q] (accumulating: rnd(dx + ¼ g))
template <typename T>
__global__ void ap2_bwd_k(int64_t n8, int H, int W, int C8, const T* __restrict__ g, T* dx, int acc) {
  const int P = H / 2, Q = W / 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(i % C8);
    int64_t t = i / C8;
    const int w = (int)(t % W);
    t /= W;
    const int h = (int)(t % H);
    const int64_t n = t / H;
    V8 s = ld8(g + (((n * P + h / 2) * Q + w / 2) * C8 + c8) * 8);
#pragma unroll
    for (int k = 0; k < 8; ++k) s.v[k] *= 0.25f;
    if (acc) {
      const V8 o = ld8(dx + i * 8);
#pragma unroll
      for (int k = 0; k < 8; ++k) s.v[k] += o.v[k];
    }
    st8(dx + i * 8, s);
  }
}

// ---------------------------------------------------------------- ReLU, tanh
template <typename T>
__global__ void relu_fwd_k(int64_t n8, const T* __restrict__ x, T* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    V8 v = ld8(x + i * 8);
#pragma unroll
    for (int k = 0; k < 8; ++k) v.v[k] = fmaxf(v.v[k], 0.f);
    st8(y + i * 8, v);
  }
}
// c = g·[x > 0] (ReLU'(0) = 0), stored or accumulated
template <typename T>
__global__ void relu_bwd_k(int64_t n8, const T* __restrict__ g, const T* __restrict__ x, T* dx, int acc) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const V8 gv = ld8(g + i * 8), xv = ld8(x + i * 8);
    V8 s;
#pragma unroll
    for (int k = 0; k < 8; ++k) s.v[k] = xv.v[k] > 0.f ? gv.v[k] : 0.f;
    if (acc) {
      const V8 o = ld8(dx + i * 8);
#pragma unroll
      for (int k = 0; k < 8; ++k) s.v[k] += o.v[k];
    }
    st8(dx + i * 8, s);
  }
}
template <typename T>
__global__ void tanh_fwd_k(int64_t n8, const T* __restrict__ x, T* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    V8 v = ld8(x + i * 8);
#pragma unroll
    for (int k = 0; k < 8; ++k) v.v[k] = tanhf(v.v[k]);
    st8(y + i * 8, v);
  }
}
// c = g·(1 − y²)
template <typename T>
__global__ void tanh_bwd_k(int64_t n8, const T* __restrict__ g, const T* __restrict__ y, T* dx, int acc) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const V8 gv = ld8(g + i * 8), yv = ld8(y + i * 8);
    V8 s;
#pragma unroll
    for (int k = 0; k < 8; ++k) s.v[k] = gv.v[k] * (1.f - yv.v[k] * yv.v[k]);
    if (acc) {
      const V8 o = ld8(dx + i * 8);
#pragma unroll
      for (int k = 0; k < 8; ++k) s.v[k] += o.v[k];
    }
    st8(dx + i * 8, s);
  }
}

// ---------------------------------------------------------------- batch concatenation
template <typename T>
__global__ void concat_k(int64_t na8, int64_t nb8, const T* __restrict__ a, const T* __restrict__ b,
                         T* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na8 + nb8;
       i += (int64_t)gridDim.x * blockDim.x)
    st8(out + i * 8, i < na8 ? ld8(a + i * 8) : ld8(b + (i - na8) * 8));
}

// ---------------------------------------------------------------- channel concatenation (DenseNet)
template <typename T>
__global__ void concat_ch_k(int64_t rows, int Ca8, int Cb8, const T* __restrict__ a, const T* __restrict__ b,
                            T* __restrict__ out) {
  const int C8 = Ca8 + Cb8;
  const int64_t n = rows * C8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / C8;
    const int c8 = (int)(i - r * C8);
    st8(out + i * 8, c8 < Ca8 ? ld8(a + (r * Ca8 + c8) * 8) : ld8(b + (r * Cb8 + c8 - Ca8) * 8));
  }
}
// da, db = the channel slices of g (each stored, or accumulated rnd(d + slice); null = not wanted)
template <typename T>
__global__ void concat_ch_bwd_k(int64_t rows, int Ca8, int Cb8, const T* __restrict__ g, T* da, T* db, int acc_a,
                                int acc_b) {
  const int C8 = Ca8 + Cb8;
  const int64_t n = rows * C8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / C8;
    const int c8 = (int)(i - r * C8);
    T* d = c8 < Ca8 ? (da ? da + (r * Ca8 + c8) * 8 : nullptr) : (db ? db + (r * Cb8 + c8 - Ca8) * 8 : nullptr);
    if (!d) continue;
    V8 v = ld8(g + i * 8);
    if (c8 < Ca8 ? acc_a : acc_b) {
      const V8 o = ld8(d);
#pragma unroll
      for (int k = 0; k < 8; ++k) v.v[k] += o.v[k];
    }
    st8(d, v);
  }
}

// ---------------------------------------------------------------- y = x + γ·a
template <typename T>
__global__ void scale_add_k(int64_t n8, const T* __restrict__ x, const T* __restrict__ a,
                            const float* __restrict__ gain, T* __restrict__ y) {
  const float gm = gain[0];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    V8 xv = ld8(x + i * 8);
    const V8 av = ld8(a + i * 8);
#pragma unroll
    for (int k = 0; k < 8; ++k) xv.v[k] += gm * av.v[k];
    st8(y + i * 8, xv);
  }
}
// da = rnd(γ·g); per-block partial Σ g·a over fixed chunks (deterministic)
template <typename T>
__global__ void __launch_bounds__(256) scale_add_bwd_k(int64_t n8, const T* __restrict__ g, const T* __restrict__ a,
                                                       const float* __restrict__ gain, T* __restrict__ da,
                                                       float* __restrict__ part) {
  const float gm = gain[0];
  const int64_t chunk = (n8 + gridDim.x - 1) / gridDim.x;
  const int64_t i0 = blockIdx.x * chunk, i1 = min(n8, i0 + chunk);
  float s = 0.f;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const V8 gv = ld8(g + i * 8), av = ld8(a + i * 8);
    V8 d;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      s = fmaf(gv.v[k], av.v[k], s);
      d.v[k] = gm * gv.v[k];
    }
    st8(da + i * 8, d);
  }
  s = warp_sum(s);
  __shared__ float red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}
__global__ void sum_parts_k(int n, const float* __restrict__ part, float* __restrict__ out) {
  double s = 0;
  for (int i = threadIdx.x; i < n; i += 32) s += part[i];
  s = warp_sum(s);
  if (threadIdx.x == 0) out[0] = (float)s;
}

// ---------------------------------------------------------------- attention helpers
// P[row] = rnd(softmax(S[row])), one warp per row (fixed-order reductions)
template <typename T>
__global__ void softmax_rows_k(int64_t rows, int L, const float* __restrict__ S, T* __restrict__ P) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int lane = threadIdx.x & 31;
  const float* s = S + r * L;
  float mx = -INFINITY;
  for (int j = lane; j < L; j += 32) mx = fmaxf(mx, s[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float sum = 0.f;
  for (int j = lane; j < L; j += 32) sum += expf(s[j] - mx);
  sum = warp_sum(sum);
  const float inv = 1.f / sum;
  for (int j = lane; j < L; j += 32) st_f(P + r * L + j, expf(s[j] - mx) * inv);
}
// the same, one pass: a row of L = 128·NCH values held in registers (float4
// per lane per chunk), so S is read once
template <typename T, int NCH>
__global__ void softmax_rows_reg_k(int64_t rows, const float* __restrict__ S, T* __restrict__ P) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int lane = threadIdx.x & 31;
  constexpr int L = 128 * NCH;
  const float4* s = reinterpret_cast<const float4*>(S + r * L);
  float4 v[NCH];
  float mx = -INFINITY;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    v[c] = __ldcs(s + c * 32 + lane);
    mx = fmaxf(mx, fmaxf(fmaxf(v[c].x, v[c].y), fmaxf(v[c].z, v[c].w)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float sum = 0.f;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    v[c] = make_float4(expf(v[c].x - mx), expf(v[c].y - mx), expf(v[c].z - mx), expf(v[c].w - mx));
    sum += (v[c].x + v[c].y) + (v[c].z + v[c].w);
  }
  sum = warp_sum(sum);
  const float inv = 1.f / sum;
  T* p = P + r * L;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int j = (c * 32 + lane) * 4;
    st_f(p + j, v[c].x * inv);
    st_f(p + j + 1, v[c].y * inv);
    st_f(p + j + 2, v[c].z * inv);
    st_f(p + j + 3, v[c].w * inv);
  }
}
template <typename T>
void softmax_rows(OpArgs& a, int64_t rows, int L, const float* S, T* P) {
  // 4-warp blocks: the 4096-wide rows hold ~170 registers per thread, so
  // small blocks let three of them share an SM
  const int g = (int)((rows + 3) / 4);
  switch (L) {
    case 4096: softmax_rows_reg_k<T, 32><<<g, 128, 0, a.stream>>>(rows, S, P); return;
    case 2048: softmax_rows_reg_k<T, 16><<<g, 128, 0, a.stream>>>(rows, S, P); return;
    case 1024: softmax_rows_reg_k<T, 8><<<g, 128, 0, a.stream>>>(rows, S, P); return;
    case 512: softmax_rows_reg_k<T, 4><<<g, 128, 0, a.stream>>>(rows, S, P); return;
    case 256: softmax_rows_reg_k<T, 2><<<g, 128, 0, a.stream>>>(rows, S, P); return;
    case 128: softmax_rows_reg_k<T, 1><<<g, 128, 0, a.stream>>>(rows, S, P); return;
    default: softmax_rows_k<T><<<(int)((rows + 7) / 8), 256, 0, a.stream>>>(rows, L, S, P);
  }
}
// rs[row] = do[row] · o[row] (= rowsum(dP ⊙ P))
template <typename T>
__global__ void rowdot_k(int64_t rows, int d, const T* __restrict__ a, const T* __restrict__ b, float* __restrict__ out) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int lane = threadIdx.x & 31;
  float s = 0.f;
  for (int j = lane; j < d; j += 32) s = fmaf(ld_f(a + r * d + j), ld_f(b + r * d + j), s);
  s = warp_sum(s);
  if (lane == 0) out[r] = s;
}
// dS = P ⊙ (dP − rs_row), in place over dP
template <typename T>
__global__ void dsoftmax_k(int64_t n, int L, const T* __restrict__ P, const float* __restrict__ rs, float* dP) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dP[i] = ld_f(P + i) * (dP[i] - rs[i / L]);
}

int64_t attn_chunk(int64_t N, int64_t L) {
  const int64_t per = L * L * 4 + L * 4;
  int64_t c = (256ll << 20) / per;
  return std::max<int64_t>(1, std::min<int64_t>(N, c));
}
// tensor-core split-K partials of the products that reduce over L
size_t attn_split_ws(int64_t N, int64_t L, int dq, int dv) {
  const int64_t cn = attn_chunk(N, L);
  tcg::Gemm pv{(int)L, dv, (int)L, (int)cn, nullptr, L, 1, L * L, false, nullptr, dv, 1, L * dv, nullptr, dv, L * dv,
               false};
  tcg::Gemm dvg{(int)L, dv, (int)L, (int)N, nullptr, 1, L, L * L, false, nullptr, dv, 1, L * dv, nullptr, dv, L * dv,
                false};
  tcg::Gemm dqg{(int)L, dq, (int)L, (int)cn, nullptr, L, 1, L * L, true, nullptr, dq, 1, L * dq, nullptr, dq, L * dq,
                false};
  return std::max({tcg::ws_bytes(pv), tcg::ws_bytes(dvg), tcg::ws_bytes(dqg)});
}

// ---------------------------------------------------------------- ops
#define OC_GAN_DISPATCH(name)                                                               \
  Status name(OpArgs& a) {                                                                  \
    return As(a, "dtype", "bf16") == "f32" ? name##_t<float>(a) : name##_t<__nv_bfloat16>(a); \
  }

template <typename T>
Status upsample2_fwd_t(OpArgs& a) {
  const int N = (int)A(a, "N"), H = (int)A(a, "H"), W = (int)A(a, "W"), C = (int)A(a, "C");
  if (C % 8) return Status::make(OC_E_UNSUPPORTED, "upsample2: C % 8");
  const int64_t n8 = (int64_t)N * 4 * H * W * C / 8;
  up2_fwd_k<T><<<grid_for(n8, 256, 4), 256, 0, a.stream>>>(n8, H, W, C / 8, (const T*)a.p(0), (T*)a.p(1));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
template <typename T>
Status upsample2_bwd_t(OpArgs& a) {
  const int N = (int)A(a, "N"), H = (int)A(a, "H"), W = (int)A(a, "W"), C = (int)A(a, "C");
  const int64_t n8 = (int64_t)N * H * W * C / 8;
  up2_bwd_k<T><<<grid_for(n8, 256, 4), 256, 0, a.stream>>>(n8, H, W, C / 8, (const T*)a.p(0), (T*)a.p(1),
                                                           Ab(a, "accumulate") ? 1 : 0);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
template <typename T>
Status avgpool2_fwd_t(OpArgs& a) {
  const int N = (int)A(a, "N"), H = (int)A(a, "H"), W = (int)A(a, "W"), C = (int)A(a, "C");
  if (C % 8 || H % 2 || W % 2) return Status::make(OC_E_UNSUPPORTED, "avgpool2: C % 8, odd H/W");
  const int64_t n8 = (int64_t)N * (H / 2) * (W / 2) * C / 8;
  ap2_fwd_k<T><<<grid_for(n8, 256, 4), 256, 0, a.stream>>>(n8, H, W, C / 8, (const T*)a.p(0), (T*)a.p(1));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
template <typename T>
Status avgpool2_bwd_t(OpArgs& a) {
  const int N = (int)A(a, "N"), H = (int)A(a, "H"), W = (int)A(a, "W"), C = (int)A(a, "C");
  const int64_t n8 = (int64_t)N * H * W * C / 8;
  ap2_bwd_k<T><<<grid_for(n8, 256, 4), 256, 0, a.stream>>>(n8, H, W, C / 8, (const T*)a.p(0), (T*)a.p(1),
                                                           Ab(a, "accumulate") ? 1 : 0);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
template <typename T>
Status relu_fwd_t(OpArgs& a) {
  const int64_t n = A(a, "n");
  if (n % 8) return Status::make(OC_E_UNSUPPORTED, "relu: n % 8");
  relu_fwd_k<T><<<grid_for(n / 8, 256, 4), 256, 0, a.stream>>>(n / 8, (const T*)a.p(0), (T*)a.p(1));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
template <typename T>
Status relu_bwd_t(OpArgs& a) {
  const int64_t n = A(a, "n");
  relu_bwd_k<T><<<grid_for(n / 8, 256, 4), 256, 0, a.stream>>>(n / 8, (const T*)a.p(0), (const T*)a.p(1),
                                                               (T*)a.p(2), Ab(a, "accumulate") ? 1 : 0);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
template <typename T>
Status tanh_fwd_t(OpArgs& a) {
  const int64_t n = A(a, "n");
  if (n % 8) return Status::make(OC_E_UNSUPPORTED, "tanh: n % 8");
  tanh_fwd_k<T><<<grid_for(n / 8, 256, 4), 256, 0, a.stream>>>(n / 8, (const T*)a.p(0), (T*)a.p(1));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
template <typename T>
Status tanh_bwd_t(OpArgs& a) {
  const int64_t n = A(a, "n");
  tanh_bwd_k<T><<<grid_for(n / 8, 256, 4), 256, 0, a.stream>>>(n / 8, (const T*)a.p(0), (const T*)a.p(1),
                                                               (T*)a.p(2), Ab(a, "accumulate") ? 1 : 0);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
template <typename T>
Status concat_batch_t(OpArgs& a) {
  const int64_t na = A(a, "na"), nb = A(a, "nb");
  if (na % 8 || nb % 8) return Status::make(OC_E_UNSUPPORTED, "concat: sizes % 8");
  concat_k<T><<<grid_for((na + nb) / 8, 256, 4), 256, 0, a.stream>>>(na / 8, nb / 8, (const T*)a.p(0),
                                                                     (const T*)a.p(1), (T*)a.p(2));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
template <typename T>
Status concat_ch_fwd_t(OpArgs& a) {
  const int64_t rows = A(a, "rows");
  const int Ca = (int)A(a, "Ca"), Cb = (int)A(a, "Cb");
  if (Ca % 8 || Cb % 8) return Status::make(OC_E_UNSUPPORTED, "concat: channels % 8");
  concat_ch_k<T><<<grid_for(rows * (Ca + Cb) / 8, 256, 4), 256, 0, a.stream>>>(rows, Ca / 8, Cb / 8, (const T*)a.p(0),
                                                                               (const T*)a.p(1), (T*)a.p(2));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
template <typename T>
Status concat_ch_bwd_t(OpArgs& a) {
  const int64_t rows = A(a, "rows");
  const int Ca = (int)A(a, "Ca"), Cb = (int)A(a, "Cb");
  if (Ca % 8 || Cb % 8) return Status::make(OC_E_UNSUPPORTED, "concat: channels % 8");
  concat_ch_bwd_k<T><<<grid_for(rows * (Ca + Cb) / 8, 256, 4), 256, 0, a.stream>>>(
      rows, Ca / 8, Cb / 8, (const T*)a.p(0), (T*)a.p(1), (T*)a.p(2), Ab(a, "acc_a") ? 1 : 0, Ab(a, "acc_b") ? 1 : 0);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
enum { SA_X, SA_A, SA_GAIN, SA_Y };
template <typename T>
Status scale_add_fwd_t(OpArgs& a) {
  const int64_t n = A(a, "n");
  if (n % 8) return Status::make(OC_E_UNSUPPORTED, "scale_add: n % 8");
  scale_add_k<T><<<grid_for(n / 8, 256, 4), 256, 0, a.stream>>>(n / 8, (const T*)a.p(SA_X), (const T*)a.p(SA_A),
                                                                (const float*)a.p(SA_GAIN), (T*)a.p(SA_Y));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
enum { SB_G, SB_A, SB_GAIN, SB_DGAIN, SB_DA };
constexpr int kSumBlocks = 148 * 2;
template <typename T>
Status scale_add_bwd_t(OpArgs& a) {
  const int64_t n = A(a, "n");
  if (a.ws_bytes < kSumBlocks * 4) return Status::make(OC_E_INVARIANT, "scale_add_bwd: workspace");
  scale_add_bwd_k<T><<<kSumBlocks, 256, 0, a.stream>>>(n / 8, (const T*)a.p(SB_G), (const T*)a.p(SB_A),
                                                       (const float*)a.p(SB_GAIN), (T*)a.p(SB_DA), (float*)a.ws);
  OC_LAUNCH_CHECK(a);
  sum_parts_k<<<1, 32, 0, a.stream>>>(kSumBlocks, (const float*)a.ws, (float*)a.p(SB_DGAIN));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
size_t scale_add_ws(const JVal&) { return kSumBlocks * 4; }

enum { AT_Q, AT_K, AT_V, AT_P, AT_O };
// samples [n0, n0 + nb) of the batch; p holds just those samples' maps
template <typename T>
Status attn_fwd_t(OpArgs& a) {
  const int64_t L = A(a, "L"), s0 = A(a, "n0"), N = A(a, "nb", A(a, "N"));
  const int dq = (int)A(a, "dq"), dv = (int)A(a, "dv");
  const T *q = (const T*)a.p(AT_Q) + s0 * L * dq, *k = (const T*)a.p(AT_K) + s0 * L * dq;
  const T* v = (const T*)a.p(AT_V) + s0 * L * dv;
  T *P = (T*)a.p(AT_P), *O = (T*)a.p(AT_O) + s0 * L * dv;
  const int64_t cn = attn_chunk(N, L);
  constexpr bool TC = std::is_same<T, __nv_bfloat16>::value;
  const size_t sws = TC ? attn_split_ws(N, L, dq, dv) : 0;
  if (a.ws_bytes < (size_t)(cn * L * L * 4 + cn * L * 4) + sws) return Status::make(OC_E_INVARIANT, "attn: workspace");
  float* S = (float*)a.ws;
  void* part = (char*)a.ws + cn * L * L * 4 + cn * L * 4;
  for (int64_t n0 = 0; n0 < N; n0 += cn) {
    const int b = (int)std::min<int64_t>(cn, N - n0);
    if (TC) {
      if (dq <= 64) {
        // P straight from q, k: the scores are recomputed on the tensor cores, never stored
        OC_TRY(tcg::attn_softmax(a, (const __nv_bfloat16*)(q + n0 * L * dq), (const __nv_bfloat16*)(k + n0 * L * dq),
                                 (__nv_bfloat16*)(P + n0 * L * L), b, (int)L, dq, S, (size_t)(cn * L * L * 4)));
      } else {
        // S = q kᵀ: A = q (K-major), B(k, n) = k[n][k] (K-major); fp32 out
        OC_TRY(tcg::gemm(a, {(int)L, (int)L, dq, b, q + n0 * L * dq, dq, 1, L * dq, false, k + n0 * L * dq, 1, dq,
                             L * dq, S, L, L * L, true}));
        softmax_rows<T>(a, b * L, (int)L, S, P + n0 * L * L);
        OC_LAUNCH_CHECK(a);
      }
      // o = P v: B(k, n) = v[k][n] (MN-major)
      OC_TRY(tcg::gemm(a, {(int)L, dv, (int)L, b, P + n0 * L * L, L, 1, L * L, false, v + n0 * L * dv, dv, 1,
                           L * dv, O + n0 * L * dv, dv, L * dv, false}, part, sws));
      continue;
    }
    // S = q kᵀ (fp32)
    OC_TRY((gemm<T, T, float, false>(a, (int)L, (int)L, dq, q + n0 * L * dq, dq, 1, nullptr, k + n0 * L * dq, 1, dq,
                                     S, L, 1, nullptr, false, false, b, L * dq, L * dq, L * L)));
    softmax_rows_k<T><<<(int)((b * L + 7) / 8), 256, 0, a.stream>>>(b * L, (int)L, S, P + n0 * L * L);
    OC_LAUNCH_CHECK(a);
    // o = P v
    OC_TRY((gemm<T, T, T, false>(a, (int)L, dv, (int)L, P + n0 * L * L, L, 1, nullptr, v + n0 * L * dv, dv, 1,
                                 O + n0 * L * dv, dv, 1, nullptr, false, false, b, L * L, L * dv, L * dv)));
  }
  return Status::ok();
}
enum { AB_Q, AB_K, AB_V, AB_P, AB_O, AB_DO, AB_DQ, AB_DK, AB_DV };
template <typename T>
Status attn_bwd_t(OpArgs& a) {
  const int64_t L = A(a, "L"), s0 = A(a, "n0"), N = A(a, "nb", A(a, "N"));
  const int dq = (int)A(a, "dq"), dv = (int)A(a, "dv");
  const int64_t oq = s0 * L * dq, ov = s0 * L * dv;
  const T *q = (const T*)a.p(AB_Q) + oq, *k = (const T*)a.p(AB_K) + oq, *v = (const T*)a.p(AB_V) + ov;
  const T *P = (const T*)a.p(AB_P), *O = (const T*)a.p(AB_O) + ov, *dO = (const T*)a.p(AB_DO) + ov;
  T *dQ = (T*)a.p(AB_DQ) + oq, *dK = (T*)a.p(AB_DK) + oq, *dV = (T*)a.p(AB_DV) + ov;
  const int64_t cn = attn_chunk(N, L);
  constexpr bool TC = std::is_same<T, __nv_bfloat16>::value;
  const size_t sws = TC ? attn_split_ws(N, L, dq, dv) : 0;
  if (a.ws_bytes < (size_t)(cn * L * L * 4 + cn * L * 4) + sws) return Status::make(OC_E_INVARIANT, "attn: workspace");
  float* dS = (float*)a.ws;
  float* rs = dS + cn * L * L;
  void* part = (char*)a.ws + cn * L * L * 4 + cn * L * 4;
  // dv = Pᵀ do (all samples in one batched launch)
  if (TC)   // A(m = j, k = i) = P[i][j] (MN-major), B(k = i, n) = do[i][n] (MN-major)
    OC_TRY(tcg::gemm(a, {(int)L, dv, (int)L, (int)N, P, 1, L, L * L, false, dO, dv, 1, L * dv, dV, dv, L * dv, false},
                     part, sws));
  else
    OC_TRY((gemm<T, T, T, false>(a, (int)L, dv, (int)L, P, 1, L, nullptr, dO, dv, 1, dV, dv, 1, nullptr, false, false,
                                 (int)N, L * L, L * dv, L * dv)));
  for (int64_t n0 = 0; n0 < N; n0 += cn) {
    const int b = (int)std::min<int64_t>(cn, N - n0);
    if (TC) {
      rowdot_k<T><<<(int)((b * L + 7) / 8), 256, 0, a.stream>>>(b * L, dv, dO + n0 * L * dv, O + n0 * L * dv, rs);
      OC_LAUNCH_CHECK(a);
      // dS = P ⊙ (do vᵀ − rs) straight from the product's epilogue:
      // A = do (K-major), B(k, n) = v[n][k] (K-major)
      tcg::Gemm g{(int)L, (int)L, dv, b, dO + n0 * L * dv, dv, 1, L * dv, false, v + n0 * L * dv, 1, dv, L * dv,
                  dS, L, L * L, true};
      g.ep_p = (const __nv_bfloat16*)(P + n0 * L * L);
      g.ldp = L;
      g.p_b = L * L;
      g.ep_rs = rs;
      g.rs_b = L;
      OC_TRY(tcg::gemm(a, g));
      // dq = dS k: A = dS (K-major fp32), B(k, n) = k[k][n] (MN-major)
      OC_TRY(tcg::gemm(a, {(int)L, dq, (int)L, b, dS, L, 1, L * L, true, k + n0 * L * dq, dq, 1, L * dq,
                           dQ + n0 * L * dq, dq, L * dq, false}, part, sws));
      // dk = dSᵀ q: A(m = j, k = i) = dS[i][j] (MN-major fp32), B(k = i, n) = q[i][n]
      OC_TRY(tcg::gemm(a, {(int)L, dq, (int)L, b, dS, 1, L, L * L, true, q + n0 * L * dq, dq, 1, L * dq,
                           dK + n0 * L * dq, dq, L * dq, false}, part, sws));
      continue;
    }
    // dP = do vᵀ (fp32), rowsum, dS = P ⊙ (dP − rs)
    OC_TRY((gemm<T, T, float, false>(a, (int)L, (int)L, dv, dO + n0 * L * dv, dv, 1, nullptr, v + n0 * L * dv, 1,
                                     dv, dS, L, 1, nullptr, false, false, b, L * dv, L * dv, L * L)));
    rowdot_k<T><<<(int)((b * L + 7) / 8), 256, 0, a.stream>>>(b * L, dv, dO + n0 * L * dv, O + n0 * L * dv, rs);
    OC_LAUNCH_CHECK(a);
    dsoftmax_k<T><<<grid_for(b * L * L, 256, 4), 256, 0, a.stream>>>(b * L * L, (int)L, P + n0 * L * L, rs, dS);
    OC_LAUNCH_CHECK(a);
    // dq = dS k, dk = dSᵀ q
    OC_TRY((gemm<float, T, T, false>(a, (int)L, dq, (int)L, dS, L, 1, nullptr, k + n0 * L * dq, dq, 1,
                                     dQ + n0 * L * dq, dq, 1, nullptr, false, false, b, L * L, L * dq, L * dq)));
    OC_TRY((gemm<float, T, T, false>(a, (int)L, dq, (int)L, dS, 1, L, nullptr, q + n0 * L * dq, dq, 1,
                                     dK + n0 * L * dq, dq, 1, nullptr, false, false, b, L * L, L * dq, L * dq)));
  }
  return Status::ok();
}
size_t attn_ws(const JVal& at) {
  const int64_t N = at.geti("nb", at.geti("N")), L = at.geti("L");
  const int64_t cn = attn_chunk(N, L);
  const bool tc = at.gets("dtype", "bf16") != "f32";
  return (size_t)(cn * L * L * 4 + cn * L * 4) +
         (tc ? attn_split_ws(N, L, (int)at.geti("dq"), (int)at.geti("dv")) : 0);
}

OC_GAN_DISPATCH(upsample2_fwd)
OC_GAN_DISPATCH(upsample2_bwd)
OC_GAN_DISPATCH(avgpool2_fwd)
OC_GAN_DISPATCH(avgpool2_bwd)
OC_GAN_DISPATCH(relu_fwd)
OC_GAN_DISPATCH(relu_bwd)
OC_GAN_DISPATCH(tanh_fwd)
OC_GAN_DISPATCH(tanh_bwd)
OC_GAN_DISPATCH(concat_batch)
OC_GAN_DISPATCH(concat_ch_fwd)
OC_GAN_DISPATCH(concat_ch_bwd)
OC_GAN_DISPATCH(scale_add_fwd)
OC_GAN_DISPATCH(scale_add_bwd)
OC_GAN_DISPATCH(attn_fwd)
OC_GAN_DISPATCH(attn_bwd)

// ---------------------------------------------------------------- hinge losses (fp32 scores)
// D: L = mean(relu(1 − s_real)) + mean(relu(1 + s_fake)); ds as in the oracle
__global__ void hinge_d_k(int nr, int nf, const float* __restrict__ s, float* __restrict__ loss,
                          float* __restrict__ ds) {
  if (threadIdx.x != 0) return;
  double lr = 0, lf = 0;
  for (int i = 0; i < nr; ++i) {
    lr += fmax(0.0, 1.0 - (double)s[i]);
    ds[i] = s[i] < 1.f ? -1.f / (float)nr : 0.f;
  }
  for (int i = 0; i < nf; ++i) {
    lf += fmax(0.0, 1.0 + (double)s[nr + i]);
    ds[nr + i] = s[nr + i] > -1.f ? 1.f / (float)nf : 0.f;
  }
  loss[0] = (float)(lr / nr + lf / nf);
}
// G: L = −mean(s), ds = −1/n
__global__ void hinge_g_k(int n, const float* __restrict__ s, float* __restrict__ loss, float* __restrict__ ds) {
  if (threadIdx.x != 0) return;
  double t = 0;
  for (int i = 0; i < n; ++i) {
    t += s[i];
    ds[i] = -1.f / (float)n;
  }
  loss[0] = (float)(-t / n);
}
Status hinge_d(OpArgs& a) {
  hinge_d_k<<<1, 32, 0, a.stream>>>((int)A(a, "n_real"), (int)A(a, "n_fake"), (const float*)a.p(0),
                                    (float*)a.p(1), (float*)a.p(2));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}
Status hinge_g(OpArgs& a) {
  hinge_g_k<<<1, 32, 0, a.stream>>>((int)A(a, "n"), (const float*)a.p(0), (float*)a.p(1), (float*)a.p(2));
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

}  // namespace

extern const OpDesc kUpsample2Fwd{"upsample2_fwd", {"x", "y"}, upsample2_fwd, nullptr};
extern const OpDesc kUpsample2Bwd{"upsample2_bwd", {"g", "dx"}, upsample2_bwd, nullptr};
extern const OpDesc kAvgpool2Fwd{"avgpool2_fwd", {"x", "y"}, avgpool2_fwd, nullptr};
extern const OpDesc kAvgpool2Bwd{"avgpool2_bwd", {"g", "dx"}, avgpool2_bwd, nullptr};
extern const OpDesc kReluFwd{"relu_fwd", {"x", "y"}, relu_fwd, nullptr};
extern const OpDesc kReluBwd{"relu_bwd", {"g", "x", "dx"}, relu_bwd, nullptr};
extern const OpDesc kTanhFwd{"tanh_fwd", {"x", "y"}, tanh_fwd, nullptr};
extern const OpDesc kTanhBwd{"tanh_bwd", {"g", "y", "dx"}, tanh_bwd, nullptr};
extern const OpDesc kConcatBatch{"concat_batch", {"a", "b", "out"}, concat_batch, nullptr};
extern const OpDesc kConcatChFwd{"concat_ch_fwd", {"a", "b", "out"}, concat_ch_fwd, nullptr};
extern const OpDesc kConcatChBwd{"concat_ch_bwd", {"g", "da", "db"}, concat_ch_bwd, nullptr};
extern const OpDesc kScaleAddFwd{"scale_add_fwd", {"x", "a", "gain", "y"}, scale_add_fwd, nullptr};
extern const OpDesc kScaleAddBwd{"scale_add_bwd", {"g", "a", "gain", "dgain", "da"}, scale_add_bwd, scale_add_ws};
extern const OpDesc kAttnFwd{"attn_fwd", {"q", "k", "v", "p", "o"}, attn_fwd, attn_ws};
extern const OpDesc kAttnBwd{"attn_bwd", {"q", "k", "v", "p", "o", "do", "dq", "dk", "dv"}, attn_bwd, attn_ws};
extern const OpDesc kHingeD{"hinge_d", {"score", "loss", "dscore"}, hinge_d, nullptr};
extern const OpDesc kHingeG{"hinge_g", {"score", "loss", "dscore"}, hinge_g, nullptr};

}  // namespace oc
