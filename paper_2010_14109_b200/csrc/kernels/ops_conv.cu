// Convolution ops of the training step: forward, data gradient, weight
// gradient, and the 2×2 stride-2 transposed convolution
// of the U-Net decoder expressed through the same kernels (a transposed conv
// is the data gradient of the strided conv it inverts).  bf16 activations
// dispatch to the tcgen05 tensor-core implicit GEMM (conv_tc.cu) when the
// shape fits its tiling (channels in multiples of 64, or of 8 with one tap
// per 16-byte chunk — the stem input zero-padded to 8 channels, attrs Cw = 3;
// other narrow inputs gather into registers), else to the CUDA-core implicit GEMM
// (conv_simt.cu).  fp32 activations (attrs.dtype = "f32", the 1e-5 parity
// mode) always run on CUDA cores — no TF32.  attrs.impl = "simt" or
// OC_CONV_IMPL=simt force CUDA cores.
#include <cstdlib>
#include <cstring>

#include "conv.cuh"

namespace oc {

bool conv_tc_ok(const ConvGeom& g, int mode);
size_t conv_tc_ws(const ConvGeom& g, int mode);
Status conv_fprop_tc(OpArgs& a, const ConvGeom& g, const __nv_bfloat16* x, const float* w, __nv_bfloat16* y,
                     bool accumulate, float* stat = nullptr, bool* stat_done = nullptr);
size_t conv_tc_stat_ws(const ConvGeom& g);
Status bn_stats_of(OpArgs& a, int64_t rows, int C, const void* y, bool f32, float* stat);
Status conv_dgrad_tc(OpArgs& a, const ConvGeom& g, const __nv_bfloat16* dy, const float* w, __nv_bfloat16* dx,
                     bool accumulate);
Status conv_wgrad_tc(OpArgs& a, const ConvGeom& g, const __nv_bfloat16* dy, const __nv_bfloat16* x, float* dw);

namespace {

bool force_simt(const OpArgs* a) {
  static int env = -1;
  if (env < 0) {
    const char* e = std::getenv("OC_CONV_IMPL");
    env = (e && std::strcmp(e, "simt") == 0) ? 1 : 0;
  }
  return env == 1 || (a && As(*a, "impl") == "simt");
}
bool f32(const OpArgs& a) { return As(a, "dtype", "bf16") == "f32"; }

Status padded_unsupported() {
  return Status::make(OC_E_UNSUPPORTED, "conv: zero-padded input channels (Cw < C) need the tensor-core path");
}

// y = conv(x, w) (+ y when accumulating)
Status fprop(OpArgs& a, const ConvGeom& g, const void* x, const float* w, void* y, bool acc) {
  if (f32(a) && g.Cw != g.C) return padded_unsupported();
  if (f32(a)) return conv_fprop_simt<float>(a, g, (const float*)x, w, (float*)y, acc);
  if (!force_simt(&a) && conv_tc_ok(g, 0))
    return conv_fprop_tc(a, g, (const __nv_bfloat16*)x, w, (__nv_bfloat16*)y, acc);
  if (g.Cw != g.C) return padded_unsupported();
  return conv_fprop_simt<__nv_bfloat16>(a, g, (const __nv_bfloat16*)x, w, (__nv_bfloat16*)y, acc);
}
Status dgrad(OpArgs& a, const ConvGeom& g, const void* dy, const float* w, void* dx, bool acc) {
  if (f32(a) && g.Cw != g.C) return padded_unsupported();
  if (f32(a)) return conv_dgrad_simt<float>(a, g, (const float*)dy, w, (float*)dx, acc);
  if (!force_simt(&a) && conv_tc_ok(g, 1))
    return conv_dgrad_tc(a, g, (const __nv_bfloat16*)dy, w, (__nv_bfloat16*)dx, acc);
  if (g.Cw != g.C) return padded_unsupported();
  return conv_dgrad_simt<__nv_bfloat16>(a, g, (const __nv_bfloat16*)dy, w, (__nv_bfloat16*)dx, acc);
}
Status wgrad(OpArgs& a, const ConvGeom& g, const void* dy, const void* x, float* dw) {
  if (f32(a) && g.Cw != g.C) return padded_unsupported();
  if (f32(a)) return conv_wgrad_simt<float>(a, g, (const float*)dy, (const float*)x, dw);
  if (!force_simt(&a) && conv_tc_ok(g, 2))
    return conv_wgrad_tc(a, g, (const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, dw);
  if (g.Cw != g.C) return padded_unsupported();
  return conv_wgrad_simt<__nv_bfloat16>(a, g, (const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, dw);
}

enum { CF_X, CF_W, CF_Y, CF_STAT };
// attrs.bn_stat (role "stat"): also produce the batch statistics [μ; rstd] of y
// for the BN that consumes it — from the tensor-core epilogue's per-channel
// partial sums when that path ran (no extra pass over y), else by the BN
// reduction over y
Status conv_fwd(OpArgs& a) {
  const ConvGeom g = conv_geom(a);
  const bool acc = Ab(a, "accumulate");
  float* stat = (float*)a.p(CF_STAT);
  if (!stat) return fprop(a, g, a.p(CF_X), (const float*)a.p(CF_W), a.p(CF_Y), acc);
  bool done = false;
  if (!f32(a) && !force_simt(&a) && conv_tc_ok(g, 0) && !acc) {
    OC_TRY(conv_fprop_tc(a, g, (const __nv_bfloat16*)a.p(CF_X), (const float*)a.p(CF_W), (__nv_bfloat16*)a.p(CF_Y),
                         false, stat, &done));
  } else {
    OC_TRY(fprop(a, g, a.p(CF_X), (const float*)a.p(CF_W), a.p(CF_Y), acc));
  }
  if (!done) OC_TRY(bn_stats_of(a, (int64_t)g.N * g.P * g.Q, g.K, a.p(CF_Y), f32(a), stat));
  return Status::ok();
}
enum { CD_DY, CD_W, CD_DX };
Status conv_dgrad(OpArgs& a) {
  return dgrad(a, conv_geom(a), a.p(CD_DY), (const float*)a.p(CD_W), a.p(CD_DX), Ab(a, "accumulate"));
}
enum { CW_DY, CW_X, CW_DW };
Status conv_wgrad(OpArgs& a) { return wgrad(a, conv_geom(a), a.p(CW_DY), a.p(CW_X), (float*)a.p(CW_DW)); }

// Transposed conv (2×2, stride 2): attrs describe the strided conv g it
// inverts — g's input is the big map (C = K_out), its output the small map
// (K = C_in), its weight [C_in][2][2][K_out] is the transposed conv's weight.
//   y_big   = dgrad_g(dy = x_small)                     (convT forward)
//   dx_small = fprop_g(x = dy_big)                      (convT data gradient)
//   dW      = wgrad_g(dy = x_small, x = dy_big)         (convT weight gradient)
Status convT_fwd(OpArgs& a) {
  return dgrad(a, conv_geom(a), a.p(CF_X), (const float*)a.p(CF_W), a.p(CF_Y), false);
}
Status convT_dgrad(OpArgs& a) {
  return fprop(a, conv_geom(a), a.p(CD_DY), (const float*)a.p(CD_W), a.p(CD_DX), Ab(a, "accumulate"));
}
Status convT_wgrad(OpArgs& a) { return wgrad(a, conv_geom(a), a.p(CW_X), a.p(CW_DY), (float*)a.p(CW_DW)); }

size_t ws_fwd(const JVal& at) {
  const ConvGeom g = conv_geom(at);
  return conv_tc_ws(g, 0) + (at.getb("bn_stat") ? conv_tc_stat_ws(g) : 0);
}
size_t ws_dgrad(const JVal& at) { return conv_tc_ws(conv_geom(at), 1); }
size_t ws_wgrad(const JVal& at) {
  ConvGeom g = conv_geom(at);
  return std::max(conv_wgrad_ws_simt(g), conv_tc_ws(g, 2));
}

}  // namespace

extern const OpDesc kConvFwd{"conv_fwd", {"x", "w", "y", "stat"}, conv_fwd, ws_fwd};
extern const OpDesc kConvDgrad{"conv_dgrad", {"dy", "w", "dx"}, conv_dgrad, ws_dgrad};
extern const OpDesc kConvWgrad{"conv_wgrad", {"dy", "x", "dw"}, conv_wgrad, ws_wgrad};
extern const OpDesc kConvTFwd{"convT_fwd", {"x", "w", "y"}, convT_fwd, ws_dgrad};
extern const OpDesc kConvTDgrad{"convT_dgrad", {"dy", "w", "dx"}, convT_dgrad, ws_fwd};
extern const OpDesc kConvTWgrad{"convT_wgrad", {"dy", "x", "dw"}, convT_wgrad, ws_wgrad};

}  // namespace oc
