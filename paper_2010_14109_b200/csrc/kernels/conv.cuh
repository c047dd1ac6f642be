// Convolution entry points (implicit GEMM, NHWC / KRSC).
#pragma once
#include "common.cuh"

namespace oc {

struct ConvGeom {
  int N, H, W, C, K, R, S, st, pad, P, Q;
  int Cw;   // channels of the weight tensor W[K][R][S][Cw], Cw <= C: activation
            // channels past Cw are zero padding (a narrow stem input stored in
            // 16-byte pixels, attrs "Cw"); default Cw = C
  int pad_slice;  // narrow inputs: images per zero-padding slice (attrs
                  // "pad_slice"; 0 = as many as fit 32 MiB)
  int nopadh;     // kernel geometry of the folded stem: no vertical padding
                  // (the vertical taps live in the channels), pad is horizontal only
  int dil;        // dilation (atrous conv, DeepLabv3+): tap (r, s) reads input pixel
                  // (p·st − pad + dil·r, q·st − pad + dil·s); 0 or 1 = none (attrs "dil")
};
__host__ __device__ inline int dil_of(const ConvGeom& g) { return g.dil > 1 ? g.dil : 1; }

inline ConvGeom conv_geom(const OpArgs& a) {
  ConvGeom g{(int)A(a, "N"), (int)A(a, "H"), (int)A(a, "W"), (int)A(a, "C"), (int)A(a, "K"), (int)A(a, "R"),
             (int)A(a, "S"), (int)A(a, "stride"), (int)A(a, "pad"), (int)A(a, "P"), (int)A(a, "Q"),
             (int)A(a, "Cw", A(a, "C")), (int)A(a, "pad_slice", 0)};
  g.nopadh = 0;
  g.dil = (int)A(a, "dil", 1);
  return g;
}
inline ConvGeom conv_geom(const JVal& j) {
  ConvGeom g{(int)j.geti("N"), (int)j.geti("H"), (int)j.geti("W"), (int)j.geti("C"), (int)j.geti("K"),
             (int)j.geti("R"), (int)j.geti("S"), (int)j.geti("stride"), (int)j.geti("pad"), (int)j.geti("P"),
             (int)j.geti("Q"), (int)j.geti("Cw", j.geti("C")), (int)j.geti("pad_slice", 0)};
  g.nopadh = 0;
  g.dil = (int)j.geti("dil", 1);
  return g;
}

// CUDA-core implicit GEMM (conv_simt.cu); T = __nv_bfloat16 or float
template <typename T>
Status conv_fprop_simt(OpArgs& a, const ConvGeom& g, const T* x, const float* w, T* y, bool accumulate = false);
template <typename T>
Status conv_dgrad_simt(OpArgs& a, const ConvGeom& g, const T* dy, const float* w, T* dx, bool accumulate);
template <typename T>
Status conv_wgrad_simt(OpArgs& a, const ConvGeom& g, const T* dy, const T* x, float* dw);
size_t conv_wgrad_ws_simt(const ConvGeom& g);

}  // namespace oc
