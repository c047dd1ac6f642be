// Convolution as implicit GEMM on CUDA cores (FFMA, fp32 accumulation) —
// the fp32 parity mode's convolution (no TF32) and the fallback for
// shapes outside the tcgen05 tiling; also the cross-check of conv_tc.cu.
// NHWC activations of type T (bf16 or fp32), KRSC fp32 weight masters rounded
// to T on load (the act-dtype weight copy of the numerics contract).
//   fprop  y[m=(n,p,q), k]   = Σ_{(r,s,c)} x[n, p·st−pad+d·r, q·st−pad+d·s, c] · W[k,r,s,c]
//   dgrad  dx[m=(n,h,w), c]  = Σ_{(r,s,k)} dy[n, (h+pad−d·r)/st, (w+pad−d·s)/st, k] · W[k,r,s,c]
//                              (terms with a non-integer or out-of-range index vanish)
//   wgrad  dW[k, (r,s,c)]    = Σ_{m=(n,p,q)} dy[m,k] · x[n, p·st−pad+d·r, q·st−pad+d·s, c]
//   (d = dilation, 1 unless the atrous convs of DeepLabv3+)
//          deterministic split-K over m: fixed partial slices, fixed-order sum
#include "conv.cuh"

namespace oc {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4;

template <int MODE, typename T>
__global__ void __launch_bounds__(256) conv_simt(ConvGeom g, const T* __restrict__ a_src, const float* __restrict__ w,
                                                 const T* __restrict__ b_src, void* out, int accumulate,
                                                 int64_t k_step) {
  int64_t M, N, Kg;
  if (MODE == 0) { M = (int64_t)g.N * g.P * g.Q; N = g.K; Kg = (int64_t)g.R * g.S * g.C; }
  else if (MODE == 1) { M = (int64_t)g.N * g.H * g.W; N = g.C; Kg = (int64_t)g.R * g.S * g.K; }
  else { M = g.K; N = (int64_t)g.R * g.S * g.C; Kg = (int64_t)g.N * g.P * g.Q; }
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  // M tiles on grid.x (up to 2^31 - 1), N tiles on grid.y
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  int64_t kb = 0, ke = Kg;
  if (MODE == 2) {  // split-K slice z
    kb = (int64_t)blockIdx.z * k_step;
    ke = (kb + k_step < Kg) ? kb + k_step : Kg;
  }
  float acc[TM][TN] = {};
  for (int64_t k0 = kb; k0 < ke; k0 += BK) {
#pragma unroll
    for (int rep = 0; rep < 4; ++rep) {
      const int e = tid + rep * 256;
      {  // A tile: As[kk][mm]
        const int mm = e % BM, kk = e / BM;
        const int64_t gm = m0 + mm, gk = k0 + kk;
        float v = 0.f;
        if (gm < M && gk < ke) {
          if (MODE == 0) {
            const int c = (int)(gk % g.C);
            const int64_t rs = gk / g.C;
            const int s = (int)(rs % g.S), r = (int)(rs / g.S);
            const int q = (int)(gm % g.Q);
            const int64_t t = gm / g.Q;
            const int p = (int)(t % g.P), n = (int)(t / g.P);
            const int h = p * g.st - g.pad + dil_of(g) * r, ww = q * g.st - g.pad + dil_of(g) * s;
            if (h >= 0 && h < g.H && ww >= 0 && ww < g.W) v = ld_f(a_src + (((int64_t)n * g.H + h) * g.W + ww) * g.C + c);
          } else if (MODE == 1) {
            const int k = (int)(gk % g.K);
            const int64_t rs = gk / g.K;
            const int s = (int)(rs % g.S), r = (int)(rs / g.S);
            const int ww = (int)(gm % g.W);
            const int64_t t = gm / g.W;
            const int h = (int)(t % g.H), n = (int)(t / g.H);
            const int pn = h + g.pad - dil_of(g) * r, qn = ww + g.pad - dil_of(g) * s;
            if (pn >= 0 && qn >= 0 && pn % g.st == 0 && qn % g.st == 0) {
              const int p = pn / g.st, q = qn / g.st;
              if (p < g.P && q < g.Q) v = ld_f(a_src + (((int64_t)n * g.P + p) * g.Q + q) * g.K + k);
            }
          } else {
            v = ld_f(a_src + gk * g.K + gm);  // dy[m][k], GEMM row = k
          }
        }
        As[kk][mm] = v;
      }
      {  // B tile: Bs[kk][nn]
        const int nn = e % BN, kk = e / BN;
        const int64_t gn = n0 + nn, gk = k0 + kk;
        float v = 0.f;
        if (gn < N && gk < ke) {
          if (MODE == 0) {
            v = rnd<T>(w[gn * Kg + gk]);
          } else if (MODE == 1) {
            const int k = (int)(gk % g.K);
            const int64_t rs = gk / g.K;
            v = rnd<T>(w[((int64_t)k * g.R * g.S + rs) * g.C + gn]);
          } else {
            const int c = (int)(gn % g.C);
            const int64_t rs = gn / g.C;
            const int s = (int)(rs % g.S), r = (int)(rs / g.S);
            const int q = (int)(gk % g.Q);
            const int64_t t = gk / g.Q;
            const int p = (int)(t % g.P), n = (int)(t / g.P);
            const int h = p * g.st - g.pad + dil_of(g) * r, ww = q * g.st - g.pad + dil_of(g) * s;
            if (h >= 0 && h < g.H && ww >= 0 && ww < g.W) v = ld_f(b_src + (((int64_t)n * g.H + h) * g.W + ww) * g.C + c);
          }
        }
        Bs[kk][nn] = v;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t gm = m0 + ty * TM + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t gn = n0 + tx * TN + j;
      if (gn >= N) continue;
      if (MODE == 2) {
        ((float*)out)[((int64_t)blockIdx.z * M + gm) * N + gn] = acc[i][j];
      } else {
        T* o = (T*)out + gm * N + gn;
        float v = acc[i][j];
        if (accumulate) v += ld_f(o);
        st_f(o, v);
      }
    }
  }
}

__global__ void splitk_reduce(int splits, int64_t n, const float* __restrict__ part, float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += part[(int64_t)z * n + i];
    out[i] = s;
  }
}

}  // namespace

// split count the workspace is sized for (two CTAs per SM, at most 64)
int wgrad_splits_simt(const ConvGeom& g) {
  const int64_t tiles = ((g.K + BM - 1) / BM) * (((int64_t)g.R * g.S * g.C + BN - 1) / BN);
  return (int)std::max<int64_t>(1, std::min<int64_t>(64, 296 / std::max<int64_t>(1, tiles)));
}
// split count a launch uses: about four CTAs per SM, each split at least 8
// K-blocks deep, as many as the workspace it was given holds (a weight
// gradient with few (k, r, s, c) outputs — the 3-channel first conv of
// ResNet-1001, one tile — ran 64 splits on 64 SMs for 1 ms)
int wgrad_splits_run(const ConvGeom& g, size_t ws_bytes) {
  const int64_t tiles = ((g.K + BM - 1) / BM) * (((int64_t)g.R * g.S * g.C + BN - 1) / BN);
  const int64_t depth = std::max<int64_t>(1, (int64_t)g.N * g.P * g.Q / (8 * BK));
  const int64_t fit = (int64_t)(ws_bytes / ((size_t)g.K * g.R * g.S * g.C * 4));
  const int64_t want = std::min<int64_t>(std::min<int64_t>(1024, depth), 4 * 148 / std::max<int64_t>(1, tiles));
  return (int)std::max<int64_t>(std::min<int64_t>(wgrad_splits_simt(g), fit), std::min(want, fit));
}

template <typename T>
Status conv_fprop_simt(OpArgs& a, const ConvGeom& g, const T* x, const float* w, T* y, bool accumulate) {
  dim3 grid((unsigned)(((int64_t)g.N * g.P * g.Q + BM - 1) / BM), (g.K + BN - 1) / BN);
  if (a.ktimer) a.ktimer->begin(a.stream);
  conv_simt<0, T><<<grid, 256, 0, a.stream>>>(g, x, w, nullptr, y, accumulate ? 1 : 0, 0);
  if (a.ktimer) a.ktimer->end(a.stream);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

template <typename T>
Status conv_dgrad_simt(OpArgs& a, const ConvGeom& g, const T* dy, const float* w, T* dx, bool accumulate) {
  dim3 grid((unsigned)(((int64_t)g.N * g.H * g.W + BM - 1) / BM), (g.C + BN - 1) / BN);
  if (a.ktimer) a.ktimer->begin(a.stream);
  conv_simt<1, T><<<grid, 256, 0, a.stream>>>(g, dy, w, nullptr, dx, accumulate ? 1 : 0, 0);
  if (a.ktimer) a.ktimer->end(a.stream);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

template <typename T>
Status conv_wgrad_simt(OpArgs& a, const ConvGeom& g, const T* dy, const T* x, float* dw) {
  const int splits = std::max(1, wgrad_splits_run(g, a.ws_bytes));
  const int64_t Kg = (int64_t)g.N * g.P * g.Q;
  int64_t step = (Kg + splits - 1) / splits;
  step = (step + BK - 1) / BK * BK;
  const int64_t n = (int64_t)g.K * g.R * g.S * g.C;
  if (a.ws_bytes < (size_t)(splits * n * 4)) return Status::make(OC_E_INVARIANT, "wgrad: workspace too small");
  dim3 grid((g.K + BM - 1) / BM, (unsigned)(((int64_t)g.R * g.S * g.C + BN - 1) / BN), splits);
  if (a.ktimer) a.ktimer->begin(a.stream);
  conv_simt<2, T><<<grid, 256, 0, a.stream>>>(g, dy, nullptr, x, a.ws, 0, step);
  if (a.ktimer) a.ktimer->end(a.stream);
  OC_LAUNCH_CHECK(a);
  splitk_reduce<<<grid_for(n, 256, 4), 256, 0, a.stream>>>(splits, n, (const float*)a.ws, dw);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

template Status conv_fprop_simt<__nv_bfloat16>(OpArgs&, const ConvGeom&, const __nv_bfloat16*, const float*,
                                                __nv_bfloat16*, bool);
template Status conv_fprop_simt<float>(OpArgs&, const ConvGeom&, const float*, const float*, float*, bool);
template Status conv_dgrad_simt<__nv_bfloat16>(OpArgs&, const ConvGeom&, const __nv_bfloat16*, const float*,
                                                __nv_bfloat16*, bool);
template Status conv_dgrad_simt<float>(OpArgs&, const ConvGeom&, const float*, const float*, float*, bool);
template Status conv_wgrad_simt<__nv_bfloat16>(OpArgs&, const ConvGeom&, const __nv_bfloat16*, const __nv_bfloat16*,
                                                float*);
template Status conv_wgrad_simt<float>(OpArgs&, const ConvGeom&, const float*, const float*, float*);

size_t conv_wgrad_ws_simt(const ConvGeom& g) {
  return (size_t)wgrad_splits_simt(g) * g.K * g.R * g.S * g.C * 4;
}

}  // namespace oc
