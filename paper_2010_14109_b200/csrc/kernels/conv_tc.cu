// Convolution on the 5th-generation tensor cores — the host side of every
// bf16 tensor-core conv (weight transforms, narrow-input re-layouts,
// channel padding, split-K reduction, dispatch) and the cp.async-gathered
// implicit-GEMM kernel used where the TMA kernel (conv_tma.cu) does not
// apply (narrow-channel weight gradients such as the space-to-depth stem).
//
//   fprop  D[m=(n,p,q)][k]        = Σ_{(r,s,c)} X[n,p·st−pad+r,q·st−pad+s,c] · W[k,r,s,c]
//          A = im2col(X) (K-major rows), B = W_bf16 [K][RSC] (K-major)
//   dgrad  D[m=(n,h,w)][c]        = Σ_{(r,s,k)} dY[n,(h+pad−r)/st,(w+pad−s)/st,k] · W[k,r,s,c]
//          one launch per output phase (h mod st, w mod st) over that phase's
//          valid taps only, so a stride-2 dgrad does no wasted MMA work;
//          A = gathered dY (K-major), B = Wt_bf16 [C][R][S][K] (K-major)
//   wgrad  D[(r,s,c)][k]          = Σ_{m=(n,p,q)} X[n,p·st−pad+r,q·st−pad+s,c] · dY[m,k]
//          both operands MN-major (contiguous along channels), deterministic
//          split-K over m (fixed slices, fixed-order sum), then dW[k][(r,s,c)]
//   narrow inputs (C % 8 != 0, the 3-channel image): re-laid out slice by
//          slice in the workspace — space-to-depth for a stride-2 stem, else
//          8-channel 16-byte pixels (weight channels Cw = 3)
//   channel counts the 64-wide tiles do not divide: operands zero-padded to
//          multiples of 64 in workspace copies, real channels stored
//
// cp.async kernel: UMMA M = 128, N = BN (64 or 128), K-block 64 (one
// 128-byte swizzle row of bf16).  CTA: warps 0-3 gather and run the epilogue,
// warp 4 issues the MMAs from one lane.  96 KB of stages (4 at BN=64, 3 at
// BN=128), each filled by cp.async with completion tracked by the stage's
// mbarrier (cp.async.mbarrier.arrive.noinc), so two CTAs share an SM and one's
// epilogue overlaps the other's main loop.  Producer address arithmetic is
// hoisted out of the K loop and uses 32-bit multiply-shift division.
#include "tc_util.cuh"

namespace oc {

namespace tc {

using namespace tcu;

constexpr int BM = 128, BKE = 64, NPROD = 128, NTHREADS = 160;
// pipeline depth: 96 KB of stages either way, so two CTAs share an SM
__host__ __device__ constexpr int stages_for(int bn) { return bn == 64 ? 4 : 3; }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}



struct Params {
  ConvGeom g;
  const __nv_bfloat16* act;    // fprop: X; dgrad: dY; wgrad: X
  const __nv_bfloat16* wgt;    // fprop: W_bf16 [K][kpad]; dgrad: Wt_bf16 [C][RS][K]; wgrad: dY
  void* out;                   // fprop/dgrad: bf16 NHWC; wgrad: fp32 partials [z][RSC][K]
  int accumulate;              // dgrad: out = rnd(acc + out)
  int M, N;                    // GEMM sizes (M < 2^31)
  int nkb;                     // K-blocks (per split for wgrad)
  int kb_per_split;            // wgrad
  int gemm_k;                  // wgrad: N·P·Q
  int ph, pw, Hp, Wp;          // dgrad phase: output sub-grid h = h'·st + ph
  int r0, s0, nr, ns;          // dgrad taps: r = r0 + st·i (i < nr), s = s0 + st·j (j < ns)
  int kpad;                    // fprop: padded RSC (row pitch of W_bf16)
  int kch;                     // fprop: C; dgrad: K (channels reduced per tap)
  int narrow;                  // fprop, C % 64 != 0 (C % 8 == 0): each 16-byte chunk of a
                               // K-block is its own (tap, c0); chunks past R·S·C are zero
  FastDiv fQ, fP, fWp, fHp, fC, fS, fKch, fns;
};

template <int MODE, int BN>
__global__ void __launch_bounds__(NTHREADS, 1) conv_tc_kernel(const Params P) {
  constexpr int NST = stages_for(BN);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  constexpr int A_BYTES = BM * BKE * 2;    // 16 KB
  constexpr int B_BYTES = BN * BKE * 2;
  constexpr int STAGE = A_BYTES + B_BYTES;
  uint64_t* full = (uint64_t*)(smem + NST * STAGE);
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;
  uint32_t* tmem_slot = (uint32_t*)(tfull + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const ConvGeom& g = P.g;
  const int m0 = blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  const int z = blockIdx.z;
  int kb_begin = 0, nkb = P.nkb;
  if (MODE == WGRAD) {
    kb_begin = z * P.kb_per_split;
    const int total = (P.gemm_k + BKE - 1) / BKE;
    nkb = total - kb_begin < P.kb_per_split ? total - kb_begin : P.kb_per_split;
    if (nkb < 0) nkb = 0;
  }

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) { mbar_init(&full[s], NPROD); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (tid < NPROD) {
    // ------------------------------------------------------------ producers
    const int ch = tid & 7;
    // per-thread row state, fixed for the whole tile
    int rh[8], rw[8];            // fprop: h0, w0 of the output pixel; dgrad: pbase, qbase
    int64_t rbase[8];            // element offset of the row's (n, h0, w0) / (n, pbase, qbase)
    bool rok[8];
    int w_r = 0, w_s = 0, w_c = 0;   // WGRAD: fixed (r,s,c) of this thread's 8 MN elements
    bool w_ok = false;
    if (MODE == FPROP || MODE == DGRAD) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int m = m0 + (tid >> 3) + 16 * i;
        rok[i] = m < P.M;
        const int mm = rok[i] ? m : 0;
        if (MODE == FPROP) {
          const uint32_t t = P.fQ.div(mm);
          const int q = mm - (int)t * g.Q;
          const uint32_t n = P.fP.div(t);
          const int p = (int)t - (int)n * g.P;
          rh[i] = p * g.st - g.pad;
          rw[i] = q * g.st - g.pad;
          rbase[i] = (int64_t)n * g.H * g.W * g.C;
        } else {
          const uint32_t t = P.fWp.div(mm);
          const int wq = mm - (int)t * P.Wp;
          const uint32_t n = P.fHp.div(t);
          const int hq = (int)t - (int)n * P.Hp;
          const int h = hq * g.st + P.ph, w = wq * g.st + P.pw;
          rh[i] = (h + g.pad - P.r0) / g.st;     // p for the first valid tap row; exact division
          rw[i] = (w + g.pad - P.s0) / g.st;
          rbase[i] = (int64_t)n * g.P * g.Q * g.K;
        }
      }
    }
    if (MODE == WGRAD) {
      const int rsc = m0 + (tid & 15) * 8;
      w_ok = rsc < P.M;
      const int rs = (int)P.fC.div(w_ok ? rsc : 0);
      w_c = (w_ok ? rsc : 0) - rs * g.C;
      w_r = (int)P.fS.div(rs);
      w_s = rs - w_r * g.S;
    }

    for (int it = 0; it < nkb; ++it) {
      const int s = it % NST;
      if (it >= NST) mbar_wait(&empty[s], (uint32_t)((it / NST - 1) & 1));
      const uint32_t a_base = smem_u32(smem + s * STAGE);
      const uint32_t b_base = a_base + A_BYTES;
      const int kb = kb_begin + it;
      if (MODE == FPROP || MODE == DGRAD) {
        // K-block kb covers one tap and 64 consecutive reduced channels (kch % 64 == 0),
        // or, narrow, 8 chunks each of its own tap
        const int kk0 = kb * BKE;
        const int kt = P.narrow ? kk0 + ch * 8 : kk0;
        const bool kok = !P.narrow || kt < g.R * g.S * g.C;
        const int tap = (int)P.fKch.div(kt), c0 = kt - tap * P.kch + (P.narrow ? 0 : ch * 8);
        int dr, ds;   // fprop: r, s; dgrad: tap indices i, j
        if (MODE == FPROP) { dr = (int)P.fS.div(tap); ds = tap - dr * g.S; }
        else { dr = (int)P.fns.div(tap); ds = tap - dr * P.ns; }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int row = (tid >> 3) + 16 * i;
          bool ok;
          const __nv_bfloat16* src;
          if (MODE == FPROP) {
            const int h = rh[i] + dr, w = rw[i] + ds;
            ok = kok && rok[i] && (unsigned)h < (unsigned)g.H && (unsigned)w < (unsigned)g.W;
            src = P.act + rbase[i] + ((int64_t)h * g.W + w) * g.C + c0;
          } else {
            const int p = rh[i] - dr, q = rw[i] - ds;
            ok = rok[i] && (unsigned)p < (unsigned)g.P && (unsigned)q < (unsigned)g.Q;
            src = P.act + rbase[i] + ((int64_t)p * g.Q + q) * g.K + c0;
          }
          cp_async16(a_base + row * 128 + ((ch ^ (row & 7)) << 4), ok ? src : P.act, ok);
        }
        int r, sx;
        if (MODE == FPROP) { r = dr; sx = ds; }
        else { r = P.r0 + g.st * dr; sx = P.s0 + g.st * ds; }
#pragma unroll
        for (int i = 0; i < BN / 16; ++i) {
          const int row = (tid >> 3) + 16 * i;
          const int nn = n0 + row;
          const bool ok = nn < P.N;
          const __nv_bfloat16* src;
          if (MODE == FPROP) src = P.wgt + (int64_t)nn * P.kpad + kk0 + ch * 8;
          else src = P.wgt + ((int64_t)nn * g.R * g.S + r * g.S + sx) * g.K + c0;
          cp_async16(b_base + row * 128 + ((ch ^ (row & 7)) << 4), ok ? src : P.wgt, ok);
        }
      } else {
        // WGRAD, MN-major tiles: K-row kr (an output pixel m) holds 128 (r,s,c) of X for A
        // and BN output channels of dY for B.  Atom (8 K-rows × 64 MN) = 1 KB;
        // A: [atom_k 8][atom_mn 2][8][128 B]  (LBO 1 KB, SBO 2 KB)
        // B: [atom_k 8][atom_mn BN/64][8][128 B] (LBO 1 KB, SBO BN/64 KB)
        const int mbase = kb * BKE;
        const int j = tid & 15;
#pragma unroll 4
        for (int i = 0; i < 8; ++i) {
          const int kr = (tid >> 4) + 8 * i;
          const int mm = mbase + kr;
          const bool mok = mm < P.gemm_k;
          const uint32_t t = P.fQ.div(mok ? mm : 0);
          const int q = (mok ? mm : 0) - (int)t * g.Q;
          const uint32_t n = P.fP.div(t);
          const int p = (int)t - (int)n * g.P;
          const int h0 = p * g.st - g.pad, w0 = q * g.st - g.pad;
          const int row = kr & 7;
          const uint32_t dst = a_base + (kr >> 3) * 2048 + (j >> 3) * 1024 + row * 128 + (((j & 7) ^ row) << 4);
          const int h = h0 + w_r, w = w0 + w_s;
          const bool ok = mok && w_ok && (unsigned)h < (unsigned)g.H && (unsigned)w < (unsigned)g.W;
          const __nv_bfloat16* src = P.act + (((int64_t)n * g.H + h) * g.W + w) * g.C + w_c;
          cp_async16(dst, ok ? src : P.act, ok);
        }
        constexpr int BCH = BN / 8;
#pragma unroll
        for (int i = 0; i < (64 * BCH) / NPROD; ++i) {
          const int e = tid + NPROD * i;
          const int kr = e / BCH, jj = e % BCH;
          const int mm = mbase + kr;
          const int kk = n0 + jj * 8;
          const bool ok = mm < P.gemm_k && kk < P.N;
          const __nv_bfloat16* src = P.wgt + (int64_t)mm * g.K + kk;
          const int row = kr & 7;
          const uint32_t dst = b_base + (kr >> 3) * (BN / 64) * 1024 + (jj >> 3) * 1024 + row * 128 +
                               (((jj & 7) ^ row) << 4);
          cp_async16(dst, ok ? src : P.wgt, ok);
        }
      }
      // the stage's full barrier receives this thread's arrival when its copies
      // land (no wait here: the producer runs ahead by up to NST stages)
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[s])) : "memory");
    }
  } else if (warp == 4) {
    // ------------------------------------------------------------ MMA issuer (one elected lane)
    constexpr uint32_t ID = idesc(BN, MODE == WGRAD, MODE == WGRAD);
    for (int it = 0; it < nkb; ++it) {
      const int s = it % NST;
      mbar_wait(&full[s], (uint32_t)((it / NST) & 1));
      fence_async_smem();   // cp.async (generic proxy) writes -> tcgen05 operand reads
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) {
        const uint32_t a_base = smem_u32(smem + s * STAGE);
        const uint32_t b_base = a_base + A_BYTES;
#pragma unroll
        for (int k = 0; k < BKE / 16; ++k) {
          uint64_t da, db;
          if (MODE == WGRAD) {
            da = sdesc(a_base + k * 2 * 2048, 1024, 2048);
            db = sdesc(b_base + k * 2 * (BN / 64) * 1024, 1024, (BN / 64) * 1024);
          } else {
            da = sdesc(a_base + k * 32, 16, 1024);
            db = sdesc(b_base + k * 32, 16, 1024);
          }
          mma_bf16(tmem, da, db, ID, (it > 0 || k > 0) ? 1u : 0u);
        }
        mma_commit(&empty[s]);
      }
      __syncwarp();
    }
    if (nkb > 0 && lane == 0) mma_commit(tfull);
    __syncwarp();
  }

  // ------------------------------------------------------------ epilogue (warps 0-3)
  if (tid < NPROD) {
    const int row = warp * 32 + lane;
    const int m = m0 + row;
    if (nkb > 0) {
      mbar_wait(tfull, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    int64_t orow = m;
    if (MODE == DGRAD && m < P.M) {
      const uint32_t t = P.fWp.div(m);
      const int wq = m - (int)t * P.Wp;
      const uint32_t n = P.fHp.div(t);
      const int hq = (int)t - (int)n * P.Hp;
      orow = ((int64_t)n * g.H + hq * g.st + P.ph) * g.W + wq * g.st + P.pw;
    }
#pragma unroll
    for (int j0 = 0; j0 < BN; j0 += 32) {
      uint32_t v[32];
      if (nkb > 0) {
        TMEM_LD32(tmem + ((uint32_t)(warp * 32) << 16) + j0, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0u;
      }
      if (m >= P.M) continue;
      if (MODE == WGRAD) {
        float* o = (float*)P.out + ((int64_t)z * P.M + m) * P.N + n0 + j0;
        if (n0 + j0 + 32 <= P.N) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            float4 f = make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]),
                                   __uint_as_float(v[i + 3]));
            if (P.accumulate) {   // later image slice: partial += (fixed slice order)
              const float4 old = *reinterpret_cast<const float4*>(o + i);
              f.x += old.x; f.y += old.y; f.z += old.z; f.w += old.w;
            }
            *reinterpret_cast<float4*>(o + i) = f;
          }
        } else {
          for (int i = 0; i < 32 && n0 + j0 + i < P.N; ++i)
            o[i] = P.accumulate ? o[i] + __uint_as_float(v[i]) : __uint_as_float(v[i]);
        }
      } else {
        __nv_bfloat16* o = (__nv_bfloat16*)P.out + orow * P.N + n0 + j0;
        if (n0 + j0 + 32 <= P.N) {
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            float f[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) f[u] = __uint_as_float(v[i + u]);
            if (P.accumulate) {
              uint4 old = *reinterpret_cast<const uint4*>(o + i);
              const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&old);
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                float2 ff = __bfloat1622float2(h2[u]);
                f[2 * u] += ff.x;
                f[2 * u + 1] += ff.y;
              }
            }
            uint4 pk;
            __nv_bfloat162* p2 = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
            for (int u = 0; u < 4; ++u) p2[u] = __floats2bfloat162_rn(f[2 * u], f[2 * u + 1]);
            *reinterpret_cast<uint4*>(o + i) = pk;
          }
        } else {
          for (int i = 0; i < 32 && n0 + j0 + i < P.N; ++i) {
            float f = __uint_as_float(v[i]);
            if (P.accumulate) f += __bfloat162float(o[i]);
            o[i] = __float2bfloat16_rn(f);
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)BN));
  }
}

// fp32 KRSC master -> bf16 [K][kpad] (fprop; (r,s,c) over the activation's C
// channels, zero past Cw and past RSC) or [C][R][S][K] (dgrad, Cw = C)
// 32-bit indices (weights hold < 2^31 elements); the transposed copy walks
// the output so its 2-byte stores coalesce (the fp32 reads go through L2)
__global__ void weight_bf16(const float* __restrict__ w, __nv_bfloat16* __restrict__ out, int K, int RS, int C,
                            int transpose, int kpad, int Cw, int Kw = 1 << 30) {
  const int n = transpose ? K * RS * C : K * kpad;
  const int rsc = RS * C;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (transpose) {
      const int k = i % K, t = i / K;   // out[(c·RS + rs)·K + k]
      const int rs = t % RS, c = t / RS;
      out[i] = __float2bfloat16_rn(w[(k * RS + rs) * C + c]);
    } else {
      const int k = i / kpad, j = i - k * kpad;
      const int rs = j / C, c = j - rs * C;
      out[i] = (j < rsc && c < Cw && k < Kw) ? __float2bfloat16_rn(w[(k * RS + rs) * Cw + c])
                                             : __float2bfloat16_rn(0.f);
    }
  }
}

// dW[k][(r,s,c)] = Σ_z part[z][(r,s,c)][k] in split order; partial rows of the
// padding channels c >= Cw are dropped.  32×32 tiles through shared memory so
// both the partial reads (along k) and the dW writes (along rsc) coalesce.
__global__ void __launch_bounds__(1024) wgrad_reduce(int splits, int RSC, int K, int C, int Cw,
                                                     const float* __restrict__ part, float* __restrict__ dw,
                                                     int Kw = 1 << 30) {
  __shared__ float tile[32][33];
  const int64_t n = (int64_t)RSC * K;
  const int k0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 × 32, one output each
  {
    const int rsc = r0 + ty, k = k0 + tx;
    float s = 0.f;
    if (rsc < RSC && k < K) {
      const int64_t i = (int64_t)rsc * K + k;
#pragma unroll 8
      for (int zz = 0; zz < splits; ++zz) s += part[(int64_t)zz * n + i];   // loads independent, sum in order
    }
    tile[ty][tx] = s;
  }
  __syncthreads();
  const int k = k0 + ty, rsc = r0 + tx;
  if (rsc >= RSC || k >= K || k >= Kw) return;
  const int rs = rsc / C, c = rsc - rs * C;
  if (c >= Cw) return;
  dw[(int64_t)k * (RSC / C) * Cw + rs * Cw + c] = tile[tx][ty];
}

template <int MODE, int BN>
Status launch(OpArgs& a, const Params& P, dim3 grid) {
  constexpr int smem = stages_for(BN) * (BM * BKE * 2 + BN * BKE * 2) + 1024 + 256;
  auto kern = conv_tc_kernel<MODE, BN>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  if (a.ktimer) a.ktimer->begin(a.stream);
  kern<<<grid, NTHREADS, smem, a.stream>>>(P);
  if (a.ktimer) a.ktimer->end(a.stream);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

int wgrad_splits(const ConvGeom& g, int BN) {
  const int64_t tiles = ((int64_t)g.R * g.S * g.C + BM - 1) / BM * ((g.K + BN - 1) / BN);
  const int64_t kbs = ((int64_t)g.N * g.P * g.Q + BKE - 1) / BKE;
  int64_t s = (2 * 148 + tiles - 1) / tiles;
  if (s > kbs) s = kbs;
  if (s > 128) s = 128;
  return (int)(s < 1 ? 1 : s);
}

void fill_divs(Params& P) {
  const ConvGeom& g = P.g;
  P.fQ.init(g.Q);
  P.fP.init(g.P);
  P.fWp.init(P.Wp > 0 ? P.Wp : 1);
  P.fHp.init(P.Hp > 0 ? P.Hp : 1);
  P.fC.init(g.C);
  P.fS.init(g.S);
  P.fKch.init(P.kch > 0 ? P.kch : 1);
  P.fns.init(P.ns > 0 ? P.ns : 1);
}

}  // namespace tc

using namespace tc;

bool conv_tma_ok(const ConvGeom& g, int mode);
// cmem (optional): channels per pixel of the gathered tensor in memory (x for
// fprop / wgrad, dY for dgrad) when it is narrower than the kernel's padded
// channel count — the tensor map's channel extent, so the channels past it
// arrive as the TMA engine's zero fill instead of through a padded copy
Status conv_fprop_tma(OpArgs& a, const ConvGeom& g, const __nv_bfloat16* x, const __nv_bfloat16* wb, int kpad,
                      __nv_bfloat16* y, bool accumulate, int nst = 0, float* stat_part = nullptr,
                      int* stat_slots = nullptr, int cmem = 0);
namespace tma {
int stat_slots_max();   // epilogue statistics slots per launch (CTA × epilogue warp)
int sm_count();
int grid_cap(int ctas);   // OC_CONV_MAX_CTAS (tests)
}  // namespace tma
Status bn_stats_from_parts(OpArgs& a, int nslots, int64_t rows, int C, const float* part, float* stat);
Status conv_dgrad_tma(OpArgs& a, const ConvGeom& g, const __nv_bfloat16* dy, const __nv_bfloat16* wt,
                      __nv_bfloat16* dx, bool accumulate, int nst = 0, int cmem = 0);
// cmem: channels per pixel of x in memory; kmem: of dY (0 = the geometry's own)
Status conv_wgrad_tma(OpArgs& a, const ConvGeom& g, const __nv_bfloat16* x, const __nv_bfloat16* dy, float* part,
                      int splits, int kb_per_split, bool accumulate, int cmem = 0, int kmem = 0);


// channel counts the 64-wide tiles do not divide (e.g. ResNet-1001's 16/32,
// BigGAN's 96, attention's 12-48): zero-padded to multiples of 64 in
// workspace copies (operands) and zero-padded weights, only the real
// channels stored (TMA kernels)
bool pad_path(const ConvGeom& g, int mode) {
  // output channels the 8-wide rows do not divide (the 3-channel image a
  // generator emits, a 21-class segmentation head) run through a padded
  // output buffer (fprop) or a padded dY copy (dgrad / wgrad)
  if (g.Cw != g.C) return false;
  if (g.C % 8) {
    // a narrow input (an image): fprop gathers it natively (Narrow); its data
    // gradient (a discriminator's image input in a generator step) is computed
    // into a 64-channel padded workspace output and the real channels copied
    // (or added) out; its weight gradient, when K needs padding too, reads a
    // 16-channel padded copy of X (the native 16-channel wgrad gather)
    if (dil_of(g) != 1) return false;
    if (mode == DGRAD) return g.st == 1 || g.st == 2;
    if (mode == WGRAD) return g.K % 64 != 0 && g.C < 16;
    return false;
  }
  if (g.K % 8) return dil_of(g) == 1;
  // 8/16-channel pixels are gathered natively by the fprop kernel, 16-channel ones by wgrad
  const bool nch = (mode == FPROP && (g.C == 8 || g.C == 16)) || (mode == WGRAD && g.C == 16);
  if (mode == DGRAD) return g.C % 64 != 0 || g.K % 64 != 0;
  return g.K % 64 != 0 || (g.C % 64 != 0 && !nch);
}

bool conv_tc_ok(const ConvGeom& g, int mode);

namespace {

int kpad_of(const ConvGeom& g) { return (g.R * g.S * g.C + BKE - 1) / BKE * BKE; }
size_t align256(size_t b) { return (b + 255) / 256 * 256; }

// Narrow input (C % 8 != 0, the 3-channel network input): the kernels see a
// re-laid-out copy, written into the workspace one slice of images at a time
// so it stays small and is never part of the budgeted memory:
//   stride 2, C <= 4, even H, W: space-to-depth.  X'[n][u][v][(a·2+b)·C + c] =
//     X[n][2u+a][2v+b][c] in 16-channel (32-byte) pixels, and the stride-2 R×S
//     conv becomes a stride-1 R'×S' conv over X' with pad' = ⌈pad/2⌉ and
//     W'[k][i][j][(a,b,c)] = W[k][2(i−pad')+a+pad][2(j−pad')+b+pad][c] (zero
//     outside the filter): the same products, 4× fewer gathered boxes
//   otherwise: 8-channel (16-byte) pixels, zero past C
struct Narrow {
  bool on, s2d;
  ConvGeom g0;        // the op's geometry
  ConvGeom gk;        // the geometry the kernels run
  int64_t slice;      // images per slice
  size_t slice_bytes;
};
Narrow narrow_of(const ConvGeom& g) {
  Narrow n{g.C % 8 != 0, false, g, g, g.N, 0};
  if (!n.on) return n;
  if (g.st == 2 && g.C <= 4 && g.H % 2 == 0 && g.W % 2 == 0 && g.R == g.S) {
    n.s2d = true;
    const int c = (g.pad + 1) / 2;
    int R2 = 1;
    while (2 * (R2 - 1 - c) + 1 + g.pad < g.R - 1) ++R2;
    n.gk.H = g.H / 2;
    n.gk.W = g.W / 2;
    n.gk.C = 16;
    n.gk.Cw = 16;
    n.gk.R = n.gk.S = R2;
    n.gk.st = 1;
    n.gk.pad = c;
  } else {
    n.gk.C = (g.C + 7) / 8 * 8;
    n.gk.Cw = g.C;
  }
  const int64_t per = (int64_t)n.gk.H * n.gk.W * n.gk.C * 2;
  n.slice = g.pad_slice > 0 ? g.pad_slice : (32ll << 20) / per;
  if (n.slice < 1) n.slice = 1;
  if (n.slice > g.N) n.slice = g.N;
  n.slice_bytes = align256((size_t)(n.slice * per));
  return n;
}

// forward conv of a narrow input whose output width K is a multiple of 8 but
// not of 64 (a discriminator's 3 -> 96 input conv): the kernels run Kp =
// up64(K) weight rows (zero past K) and store the first K columns (nst); 0 = n/a
int narrow_fprop_kp(const Narrow& nw, const ConvGeom& g0) {
  if (!nw.on || nw.s2d || g0.K % 64 == 0 || g0.K % 8 != 0) return 0;
  return (g0.K + 63) / 64 * 64;
}

}  // namespace

bool conv_tc_ok(const ConvGeom& g, int mode) {
  // 32-bit element indices: the TMA kernels address rows (output pixels) with
  // 32-bit indices and let the tensor maps form the byte offsets, so they need
  // only M = images · P · Q < 2^31 per launch (narrow inputs run one
  // re-laid-out slice of images per launch); the cp.async kernels also form
  // 32-bit element offsets of whole activation tensors
  const Narrow nw = narrow_of(g);
  const int64_t nimg = nw.on ? nw.slice : g.N;
  ConvGeom gk = nw.gk;
  const int kp = mode == FPROP ? narrow_fprop_kp(nw, g) : 0;
  if (kp) gk.K = kp;
  const bool tma = conv_tma_ok(gk, mode) || pad_path(g, mode);
  if (tma) {
    if (nimg * g.P * g.Q >= (1ll << 31) || (int64_t)g.N * g.H * g.W >= (1ll << 31)) return false;
  } else if ((int64_t)g.N * g.H * g.W * ((g.C + 63) / 64 * 64) >= (1ll << 31) ||
             (int64_t)g.N * g.P * g.Q * ((g.K + 63) / 64 * 64) >= (1ll << 31)) {
    return false;
  }
  if (dil_of(g) > 1)   // atrous convs: the TMA kernels with dilated im2col offsets, 64-channel operands
    return g.C % 64 == 0 && g.K % 64 == 0 && g.Cw == g.C && (mode != DGRAD || g.st == 1);
  if (pad_path(g, mode)) return true;
  // zero-padded activation channels (Cw < C) only on the 16-byte-chunk paths
  if (g.Cw != g.C && (g.C % 8 != 0 || g.Cw > g.C || mode == DGRAD)) return false;
  if (mode == DGRAD) return g.K % 64 == 0 && g.C % 64 == 0 && (g.st == 1 || g.st == 2);
  if (kp) return tma;
  return g.K % 64 == 0;
}

namespace {

__global__ void pad_pixels(int64_t rows, int C, int C8, const __nv_bfloat16* __restrict__ x,
                           __nv_bfloat16* __restrict__ out) {
  const unsigned short* xs = reinterpret_cast<const unsigned short*>(x);
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    for (int c0 = 0; c0 < C8; c0 += 8) {
      uint32_t v[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (c0 + e < C) v[e >> 1] |= (uint32_t)xs[r * C + c0 + e] << (16 * (e & 1));
      *reinterpret_cast<uint4*>(out + r * C8 + c0) = make_uint4(v[0], v[1], v[2], v[3]);
    }
  }
}

// X [n][H][W][C] -> X' [n][H/2][W/2][16]
// grid: x over v, y over (n, u) — no 64-bit index division
__global__ void s2d_pixels(int rows, int H2, int W2, int C, const __nv_bfloat16* __restrict__ x,
                           __nv_bfloat16* __restrict__ out) {
  const unsigned short* xs = reinterpret_cast<const unsigned short*>(x);
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  for (int y = blockIdx.y; v < W2 && y < rows; y += gridDim.y) {
    const int u = y % H2;
    const int64_t n = y / H2;
    const int64_t i = (int64_t)y * W2 + v;
    uint4* o = reinterpret_cast<uint4*>(out + i * 16);
    if (C == 3) {
      // the 2 × 2 block is two contiguous, 4-byte aligned 12-byte runs ((a, b, c) order = memory order)
      const uint32_t* r0 = reinterpret_cast<const uint32_t*>(x + ((n * 2 * H2 + 2 * u) * 2 * W2 + 2 * v) * 3);
      const uint32_t* r1 = r0 + 3 * W2;
      o[0] = make_uint4(__ldg(r0), __ldg(r0 + 1), __ldg(r0 + 2), __ldg(r1));
      o[1] = make_uint4(__ldg(r1 + 1), __ldg(r1 + 2), 0u, 0u);
      continue;
    }
    uint32_t w[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    for (int ab = 0; ab < 4; ++ab) {
      const int64_t src = ((n * 2 * H2 + 2 * u + (ab >> 1)) * 2 * W2 + 2 * v + (ab & 1)) * C;
      for (int c = 0; c < C; ++c) {
        const int e = ab * C + c;
        w[e >> 1] |= (uint32_t)xs[src + c] << (16 * (e & 1));
      }
    }
    o[0] = make_uint4(w[0], w[1], w[2], w[3]);
    o[1] = make_uint4(w[4], w[5], w[6], w[7]);
  }
}


Status pad_slice(OpArgs& a, const Narrow& nw, int64_t n0, int64_t nn, const __nv_bfloat16* x,
                 __nv_bfloat16* buf) {
  const ConvGeom& g0 = nw.g0;
  const __nv_bfloat16* xs = x + n0 * g0.H * g0.W * g0.C;
  if (nw.s2d) {
    const int rows = (int)(nn * nw.gk.H);
    const dim3 grid((nw.gk.W + 127) / 128, (unsigned)std::min(rows, 65535));
    s2d_pixels<<<grid, 128, 0, a.stream>>>(rows, nw.gk.H, nw.gk.W, g0.C, xs, buf);
  } else {
    const int64_t rows = nn * g0.H * g0.W;
    pad_pixels<<<grid_for(rows, 256, 2), 256, 0, a.stream>>>(rows, g0.C, nw.gk.C, xs, buf);
  }
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

// W'[k][(i,j,(a,b,c))] (bf16, row pitch kpad) from W[k][R][S][C] for the space-to-depth conv
__global__ void weight_bf16_s2d(const float* __restrict__ w, __nv_bfloat16* __restrict__ out, int K, int R, int S,
                                int C, int R2, int S2, int c2, int pad, int kpad) {
  const int64_t n = (int64_t)K * kpad;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(e / kpad), jj = (int)(e % kpad);
    const int tap = jj / 16, ch = jj % 16;
    float v = 0.f;
    if (tap < R2 * S2 && ch < 4 * C) {
      const int i = tap / S2, j = tap % S2, ab = ch / C, c = ch % C;
      const int r = 2 * (i - c2) + (ab >> 1) + pad, s = 2 * (j - c2) + (ab & 1) + pad;
      if (r >= 0 && r < R && s >= 0 && s < S) v = w[(((int64_t)k * R + r) * S + s) * C + c];
    }
    out[e] = __float2bfloat16_rn(v);
  }
}

// dW[k][r][s][c] = Σ_z part[z][(i,j,(a,b,c))][k], the (i,j,a,b) holding filter tap (r,s).
// A block = 32 consecutive elements (k fastest: the partials are read
// coalesced) × 8 split groups; group g sums the splits z ≡ g (mod 8) in order,
// then the 8 group sums are added in order (fixed: bitwise reproducible)
__global__ void __launch_bounds__(256) wgrad_reduce_s2d(int splits, int RSC2, int K, const float* __restrict__ part,
                                                        float* __restrict__ dw, int R, int S, int C, int S2, int c2,
                                                        int pad) {
  __shared__ float sm[8][33];
  const int n = K * R * S * C;
  const int l = threadIdx.x & 31, gz = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + l;
  int row = 0, k = 0, r = 0, s = 0, c = 0;
  float acc = 0.f;
  if (e < n) {
    k = e % K;
    int t = e / K;
    c = t % C;
    t /= C;
    s = t % S;
    r = t / S;
    const int tr = r + 2 * c2 - pad, ts = s + 2 * c2 - pad;
    row = ((tr >> 1) * S2 + (ts >> 1)) * 16 + ((tr & 1) * 2 + (ts & 1)) * C + c;
#pragma unroll 4
    for (int z = gz; z < splits; z += 8) acc += part[((int64_t)z * RSC2 + row) * K + k];
  }
  sm[gz][l] = acc;
  __syncthreads();
  if (gz == 0 && e < n) {
    float tot = 0.f;
#pragma unroll
    for (int g2 = 0; g2 < 8; ++g2) tot += sm[g2][l];
    dw[(((int64_t)k * R + r) * S + s) * C + c] = tot;
  }
}

int wgrad_bn(const ConvGeom& g) { return g.K % 128 == 0 ? 128 : 64; }

}  // namespace

namespace {

int up64(int c) { return (c + 63) / 64 * 64; }

// the padded problem: C -> Cp, K -> Kp; operand copies in image slices
struct PadPlan {
  ConvGeom gk;             // padded geometry (full batch)
  bool pad_x, pad_y;       // X (C channels) / dY (K channels) need a padded copy
  bool pad_out;            // dgrad of a narrow input: dX computed Cp wide in the workspace, real channels copied out
  int64_t slice;
  size_t xbytes, ybytes, obytes;   // per-slice copy / padded-output bytes
};
PadPlan pad_plan(const ConvGeom& g, int mode) {
  PadPlan p{g, false, false, false, g.N, 0, 0, 0};
  const bool nch = (mode == FPROP && (g.C == 8 || g.C == 16)) || (mode == WGRAD && g.C == 16);
  const bool narrow_w = mode == WGRAD && g.C % 8 != 0 && g.C < 16;   // X padded to the 16-channel gather
  const int Cp = (g.C % 64 == 0 || nch) ? g.C : (narrow_w ? 16 : up64(g.C)), Kp = up64(g.K);
  p.gk.C = p.gk.Cw = Cp;
  p.gk.K = Kp;
  // an operand of >= 64 channels whose pixels are 16-byte rows is read in
  // place (the tensor map's channel extent is its own, the TMA engine zero-fills
  // the padding channels); narrower ones get a padded copy
  const bool x_direct = g.C % 8 == 0 && g.C >= 16, y_direct = g.K % 8 == 0 && g.K >= 16;
  p.pad_x = Cp != g.C && mode != DGRAD && !x_direct;
  // dY copy for dgrad / wgrad; for fprop with K % 8 != 0 the same buffer holds the padded output
  p.pad_y = Kp != g.K && (mode == FPROP ? g.K % 8 != 0 : !y_direct);
  p.pad_out = mode == DGRAD && g.C % 8 != 0;
  const int64_t px = p.pad_x ? (int64_t)g.H * g.W * Cp * 2 : 0, py = p.pad_y ? (int64_t)g.P * g.Q * Kp * 2 : 0;
  const int64_t po = p.pad_out ? (int64_t)g.H * g.W * Cp * 2 : 0;
  if (px + py + po > 0) p.slice = std::max<int64_t>(1, std::min<int64_t>(g.N, (64ll << 20) / (px + py + po)));
  p.xbytes = align256((size_t)(p.slice * px));
  p.ybytes = align256((size_t)(p.slice * py));
  p.obytes = align256((size_t)(p.slice * po));
  return p;
}
int tma_wgrad_splits(const ConvGeom& gk, int64_t slice) {
  const int BN = gk.K % 128 == 0 ? 128 : 64;
  const int64_t tiles = ((int64_t)gk.R * gk.S * gk.C + BM - 1) / BM * (gk.K / BN);
  const int64_t kbs = (slice * gk.P * gk.Q + 127) / 128;
  int64_t s2 = (2 * 148) / tiles;
  return (int)(s2 < 1 ? 1 : (s2 > kbs ? kbs : s2));
}
size_t pad_ws(const ConvGeom& g, int mode) {
  const PadPlan p = pad_plan(g, mode);
  const ConvGeom& k = p.gk;
  if (mode == FPROP) return align256((size_t)k.K * kpad_of(k) * 2) + p.xbytes + p.ybytes;
  if (mode == DGRAD) return align256((size_t)k.C * k.R * k.S * k.K * 2) + p.ybytes + p.obytes;
  return align256((size_t)tma_wgrad_splits(k, p.slice) * k.R * k.S * k.C * k.K * 4) + p.xbytes + p.ybytes;
}

// Wt[c][rs][k] for c < Cp, k < Kp: W[k][rs][c] inside the real channels, else 0
__global__ void weight_bf16_tpad(const float* __restrict__ w, __nv_bfloat16* __restrict__ out, int K, int RS, int C,
                                 int Kp, int Cp) {
  const int64_t n = (int64_t)Cp * RS * Kp;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % Kp);
    const int64_t t = i / Kp;
    const int rs = (int)(t % RS), c = (int)(t / RS);
    out[i] = (c < C && k < K) ? __float2bfloat16_rn(w[((int64_t)k * RS + rs) * C + c]) : __float2bfloat16_rn(0.f);
  }
}

// y[r][k] = yp[r][k] for k < K (or rnd(y + yp) when accumulating): the real
// channels of a padded-output conv
__global__ void unpad_pixels(int64_t rows, int K, int Kp, const __nv_bfloat16* __restrict__ yp,
                             __nv_bfloat16* __restrict__ y, int acc) {
  const int64_t n = rows * K;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / K;
    const int k = (int)(i - r * K);
    float v = __bfloat162float(yp[r * Kp + k]);
    if (acc) v += __bfloat162float(y[i]);
    y[i] = __float2bfloat16_rn(v);
  }
}

Status pad_copy(OpArgs& a, int64_t rows, int C, int Cp, const __nv_bfloat16* src, __nv_bfloat16* dst) {
  pad_pixels<<<grid_for(rows, 256, 2), 256, 0, a.stream>>>(rows, C, Cp, src, dst);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

Status conv_fprop_pad(OpArgs& a, const ConvGeom& g, const __nv_bfloat16* x, const float* w, __nv_bfloat16* y,
                      bool accumulate) {
  const PadPlan pp = pad_plan(g, FPROP);
  const ConvGeom& k = pp.gk;
  const int kpad = kpad_of(k);
  __nv_bfloat16* wb = (__nv_bfloat16*)a.ws;
  __nv_bfloat16* xbuf = (__nv_bfloat16*)((char*)a.ws + align256((size_t)k.K * kpad * 2));
  weight_bf16<<<grid_for((int64_t)k.K * kpad, 256, 1), 256, 0, a.stream>>>(w, wb, k.K, k.R * k.S, k.C, 0, kpad, g.C,
                                                                            g.K);
  OC_LAUNCH_CHECK(a);
  for (int64_t n0 = 0; n0 < g.N; n0 += pp.slice) {
    const int64_t nn = std::min<int64_t>(pp.slice, g.N - n0);
    ConvGeom gs = k;
    gs.N = (int)nn;
    const __nv_bfloat16* act = x + n0 * g.H * g.W * g.C;
    int cmem = g.C;
    if (pp.pad_x) {
      OC_TRY(pad_copy(a, nn * g.H * g.W, g.C, k.C, act, xbuf));
      act = xbuf;
      cmem = k.C;
    }
    if (pp.pad_y) {   // K % 8 != 0: all Kp channels into the workspace, then the real ones out
      __nv_bfloat16* ybuf = (__nv_bfloat16*)((char*)xbuf + pp.xbytes);
      OC_TRY(conv_fprop_tma(a, gs, act, wb, kpad, ybuf, false, 0, nullptr, nullptr, cmem));
      const int64_t rows = nn * g.P * g.Q;
      unpad_pixels<<<grid_for(rows * g.K, 256, 4), 256, 0, a.stream>>>(rows, g.K, k.K, ybuf,
                                                                       y + n0 * g.P * g.Q * g.K, accumulate ? 1 : 0);
      OC_LAUNCH_CHECK(a);
      continue;
    }
    OC_TRY(conv_fprop_tma(a, gs, act, wb, kpad, y + n0 * g.P * g.Q * g.K, accumulate, g.K, nullptr, nullptr, cmem));
  }
  return Status::ok();
}

Status conv_dgrad_pad(OpArgs& a, const ConvGeom& g, const __nv_bfloat16* dy, const float* w, __nv_bfloat16* dx,
                      bool accumulate) {
  const PadPlan pp = pad_plan(g, DGRAD);
  const ConvGeom& k = pp.gk;
  __nv_bfloat16* wt = (__nv_bfloat16*)a.ws;
  __nv_bfloat16* ybuf = (__nv_bfloat16*)((char*)a.ws + align256((size_t)k.C * k.R * k.S * k.K * 2));
  weight_bf16_tpad<<<grid_for((int64_t)k.C * k.R * k.S * k.K, 256, 4), 256, 0, a.stream>>>(w, wt, g.K, g.R * g.S,
                                                                                            g.C, k.K, k.C);
  OC_LAUNCH_CHECK(a);
  for (int64_t n0 = 0; n0 < g.N; n0 += pp.slice) {
    const int64_t nn = std::min<int64_t>(pp.slice, g.N - n0);
    ConvGeom gs = k;
    gs.N = (int)nn;
    const __nv_bfloat16* act = dy + n0 * g.P * g.Q * g.K;
    int kmem = g.K;
    if (pp.pad_y) {
      OC_TRY(pad_copy(a, nn * g.P * g.Q, g.K, k.K, act, ybuf));
      act = ybuf;
      kmem = k.K;
    }
    if (pp.pad_out) {
      // narrow dX: all Cp channels into the workspace, then the real ones out;
      // accumulating, the old dX is padded into the workspace first and the
      // kernel's epilogue adds to it (one rounding of old + dgrad, as the
      // direct path; adding a rounded dgrad afterwards would round twice)
      __nv_bfloat16* obuf = (__nv_bfloat16*)((char*)ybuf + pp.ybytes);
      __nv_bfloat16* dxs = dx + n0 * g.H * g.W * g.C;
      const int64_t rows = nn * g.H * g.W;
      if (accumulate) OC_TRY(pad_copy(a, rows, g.C, k.C, dxs, obuf));
      OC_TRY(conv_dgrad_tma(a, gs, act, wt, obuf, accumulate, k.C, kmem));
      unpad_pixels<<<grid_for(rows * g.C, 256, 4), 256, 0, a.stream>>>(rows, g.C, k.C, obuf, dxs, 0);
      OC_LAUNCH_CHECK(a);
      continue;
    }
    OC_TRY(conv_dgrad_tma(a, gs, act, wt, dx + n0 * g.H * g.W * g.C, accumulate, g.C, kmem));
  }
  return Status::ok();
}

Status conv_wgrad_pad(OpArgs& a, const ConvGeom& g, const __nv_bfloat16* dy, const __nv_bfloat16* x, float* dw) {
  const PadPlan pp = pad_plan(g, WGRAD);
  const ConvGeom& k = pp.gk;
  const int splits = tma_wgrad_splits(k, pp.slice);
  const int RSCp = k.R * k.S * k.C;
  float* part = (float*)a.ws;
  __nv_bfloat16* xbuf = (__nv_bfloat16*)((char*)a.ws + align256((size_t)splits * RSCp * k.K * 4));
  __nv_bfloat16* ybuf = (__nv_bfloat16*)((char*)xbuf + pp.xbytes);
  for (int64_t n0 = 0, sl = 0; n0 < g.N; n0 += pp.slice, ++sl) {
    const int64_t nn = std::min<int64_t>(pp.slice, g.N - n0);
    ConvGeom gs = k;
    gs.N = (int)nn;
    const __nv_bfloat16* xa = x + n0 * g.H * g.W * g.C;
    const __nv_bfloat16* ya = dy + n0 * g.P * g.Q * g.K;
    int cmem = g.C, kmem = g.K;
    if (pp.pad_x) {
      OC_TRY(pad_copy(a, nn * g.H * g.W, g.C, k.C, xa, xbuf));
      xa = xbuf;
      cmem = k.C;
    }
    if (pp.pad_y) {
      OC_TRY(pad_copy(a, nn * g.P * g.Q, g.K, k.K, ya, ybuf));
      ya = ybuf;
      kmem = k.K;
    }
    OC_TRY(conv_wgrad_tma(a, gs, xa, ya, part, splits, 0, sl > 0, cmem, kmem));
  }
  wgrad_reduce<<<dim3((k.K + 31) / 32, (RSCp + 31) / 32), 1024, 0, a.stream>>>(splits, RSCp, k.K, k.C, g.C, part, dw,
                                                                              g.K);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

}  // namespace

size_t conv_tc_ws(const ConvGeom& g0, int mode) {
  if (pad_path(g0, mode)) return pad_ws(g0, mode);
  const Narrow nw = narrow_of(g0);
  const ConvGeom& g = nw.gk;
  if (mode == WGRAD) {
    ConvGeom gs = g;
    gs.N = (int)nw.slice;
    const int64_t nsl = (g.N + nw.slice - 1) / nw.slice;
    return align256((size_t)wgrad_splits(gs, wgrad_bn(g)) * g.R * g.S * g.C * g.K * 4) + nw.slice_bytes;
  }
  const int kp = mode == FPROP ? narrow_fprop_kp(nw, g0) : 0;
  return align256((size_t)(kp ? kp : g.K) * kpad_of(g) * 2) + nw.slice_bytes;
}

// partial-sum region of the fused BN statistics: one set of slots per image slice
size_t conv_tc_stat_ws(const ConvGeom& g0) {
  const Narrow nw = narrow_of(g0);
  const int64_t nsl = (g0.N + nw.slice - 1) / nw.slice;
  return align256((size_t)nsl * tma::stat_slots_max() * 2 * g0.K * 4);
}

Status conv_fprop_tc(OpArgs& a, const ConvGeom& g0, const __nv_bfloat16* x, const float* w, __nv_bfloat16* y,
                     bool accumulate, float* stat, bool* stat_done) {
  if (stat_done) *stat_done = false;
  if (pad_path(g0, FPROP)) return conv_fprop_pad(a, g0, x, w, y, accumulate);
  const Narrow nw = narrow_of(g0);
  const int kp = narrow_fprop_kp(nw, g0);
  ConvGeom g = nw.gk;
  if (kp) g.K = kp;   // weight rows past the real K are zero; only the first K columns are stored
  __nv_bfloat16* wb = (__nv_bfloat16*)a.ws;
  const int kpad = kpad_of(g);
  __nv_bfloat16* xbuf = (__nv_bfloat16*)((char*)a.ws + align256((size_t)g.K * kpad * 2));
  // fused statistics: slices append their epilogue slots (part[slot][2][K]) after the conv workspace
  float* part = stat ? (float*)((char*)a.ws + conv_tc_ws(g0, FPROP)) : nullptr;
  int nslots = 0;
  bool fused = stat != nullptr && !kp;   // stored columns ≠ computed ones: statistics in a separate pass
  if (nw.s2d)
    weight_bf16_s2d<<<grid_for((int64_t)g.K * kpad, 256, 4), 256, 0, a.stream>>>(
        w, wb, g.K, g0.R, g0.S, g0.C, g.R, g.S, g.pad, g0.pad, kpad);
  else
    weight_bf16<<<grid_for((int64_t)g.K * kpad, 256, 1), 256, 0, a.stream>>>(w, wb, g.K, g.R * g.S, g.C, 0, kpad,
                                                                              g.Cw, g0.K);
  OC_LAUNCH_CHECK(a);
  for (int64_t n0 = 0; n0 < g.N; n0 += nw.slice) {
    const int64_t nn = g.N - n0 < nw.slice ? g.N - n0 : nw.slice;
    Params P{};
    P.g = g;
    P.g.N = (int)nn;
    P.act = x;
    if (nw.on) {
      Status st = pad_slice(a, nw, n0, nn, x, xbuf);
      if (!st.good()) return st;
      P.act = xbuf;
    }
    P.wgt = wb;
    P.out = y + n0 * g.P * g.Q * g0.K;
    P.M = (int)(nn * g.P * g.Q);
    P.N = g.K;
    P.kpad = kpad;
    P.kch = g.C;
    P.narrow = g.C % 64 != 0 ? 1 : 0;
    P.nkb = kpad / BKE;
    P.accumulate = accumulate ? 1 : 0;
    if (conv_tma_ok(P.g, FPROP)) {
      int sl = 0;
      Status st = conv_fprop_tma(a, P.g, P.act, wb, kpad, (__nv_bfloat16*)P.out, accumulate, kp ? g0.K : 0,
                                 fused ? part + (size_t)nslots * 2 * g.K : nullptr, fused ? &sl : nullptr);
      if (!st.good()) return st;
      if (sl == 0) fused = false;
      nslots += sl;
      continue;
    }
    if (kp) return Status::make(OC_E_INVARIANT, "conv: padded-K narrow fprop needs the TMA kernels");
    fused = false;
    fill_divs(P);
    const dim3 grid((P.M + BM - 1) / BM, g.K / (g.K % 128 == 0 ? 128 : 64), 1);
    Status st = g.K % 128 == 0 ? launch<FPROP, 128>(a, P, grid) : launch<FPROP, 64>(a, P, grid);
    if (!st.good()) return st;
  }
  if (fused) {
    OC_TRY(bn_stats_from_parts(a, nslots, (int64_t)g.N * g.P * g.Q, g.K, part, stat));
    if (stat_done) *stat_done = true;
  }
  return Status::ok();
}

Status conv_dgrad_tc(OpArgs& a, const ConvGeom& g, const __nv_bfloat16* dy, const float* w, __nv_bfloat16* dx,
                     bool accumulate) {
  if (pad_path(g, DGRAD)) return conv_dgrad_pad(a, g, dy, w, dx, accumulate);
  __nv_bfloat16* wt = (__nv_bfloat16*)a.ws;
  const int64_t nw = (int64_t)g.K * g.R * g.S * g.C;
  weight_bf16<<<grid_for(nw, 256, 1), 256, 0, a.stream>>>(w, wt, g.K, g.R * g.S, g.C, 1, 0, g.C);
  OC_LAUNCH_CHECK(a);
  if (conv_tma_ok(g, DGRAD)) return conv_dgrad_tma(a, g, dy, wt, dx, accumulate);
  for (int ph = 0; ph < g.st; ++ph)
    for (int pw = 0; pw < g.st; ++pw) {
      Params P{};
      P.g = g;
      P.act = dy;
      P.wgt = wt;
      P.out = dx;
      P.accumulate = accumulate ? 1 : 0;
      P.ph = ph;
      P.pw = pw;
      P.Hp = (g.H - ph + g.st - 1) / g.st;
      P.Wp = (g.W - pw + g.st - 1) / g.st;
      // taps with (h + pad − r) divisible by st for h ≡ ph (mod st)
      P.r0 = (ph + g.pad) % g.st;
      P.s0 = (pw + g.pad) % g.st;
      P.nr = P.r0 < g.R ? (g.R - P.r0 + g.st - 1) / g.st : 0;
      P.ns = P.s0 < g.S ? (g.S - P.s0 + g.st - 1) / g.st : 0;
      P.M = g.N * P.Hp * P.Wp;
      P.N = g.C;
      P.kch = g.K;
      P.nkb = P.nr * P.ns * g.K / BKE;
      if (P.M == 0) continue;
      if (P.nkb == 0 && accumulate) continue;  // no taps reach this phase: G stays as is
      fill_divs(P);
      const dim3 grid((P.M + BM - 1) / BM, g.C / (g.C % 128 == 0 ? 128 : 64), 1);
      Status st = g.C % 128 == 0 ? launch<DGRAD, 128>(a, P, grid) : launch<DGRAD, 64>(a, P, grid);
      if (!st.good()) return st;
    }
  return Status::ok();
}

Status conv_wgrad_tc(OpArgs& a, const ConvGeom& g0, const __nv_bfloat16* dy, const __nv_bfloat16* x, float* dw) {
  if (pad_path(g0, WGRAD)) return conv_wgrad_pad(a, g0, dy, x, dw);
  const Narrow nw = narrow_of(g0);
  const ConvGeom& g = nw.gk;
  const int BN = wgrad_bn(g);
  ConvGeom gs = g;
  gs.N = (int)nw.slice;
  int splits = wgrad_splits(gs, BN);
  if (conv_tma_ok(g, WGRAD)) {
    // persistent kernel: at most two units per SM, balanced (floor, not ceil)
    const int64_t tiles = ((int64_t)g.R * g.S * g.C + BM - 1) / BM * (g.K / BN);
    const int64_t kbs = ((int64_t)gs.N * g.P * g.Q + BKE - 1) / BKE;
    int64_t s2 = (2 * (int64_t)tma::grid_cap(tma::sm_count())) / tiles;
    s2 = s2 < 1 ? 1 : (s2 > kbs ? kbs : s2);
    splits = (int)(s2 < splits ? s2 : splits);
  }
  const int64_t nsl = (g.N + nw.slice - 1) / nw.slice;
  const int RSC = g.R * g.S * g.C;
  // one set of split partials; image slices after the first accumulate into it
  float* part = (float*)a.ws;
  __nv_bfloat16* xbuf = (__nv_bfloat16*)((char*)a.ws + align256((size_t)splits * RSC * g.K * 4));
  for (int64_t sl = 0; sl < nsl; ++sl) {
    const int64_t n0 = sl * nw.slice;
    const int64_t nn = g.N - n0 < nw.slice ? g.N - n0 : nw.slice;
    Params P{};
    P.g = g;
    P.g.N = (int)nn;
    P.act = x;
    if (nw.on) {
      Status st = pad_slice(a, nw, n0, nn, x, xbuf);
      if (!st.good()) return st;
      P.act = xbuf;
    }
    P.wgt = dy + n0 * g.P * g.Q * g.K;
    P.out = part;
    P.accumulate = sl > 0 ? 1 : 0;
    P.M = RSC;
    P.N = g.K;
    P.gemm_k = (int)(nn * g.P * g.Q);
    const int kbs = (P.gemm_k + BKE - 1) / BKE;
    P.kb_per_split = (kbs + splits - 1) / splits;
    P.nkb = P.kb_per_split;
    if (conv_tma_ok(P.g, WGRAD)) {
      Status st = conv_wgrad_tma(a, P.g, P.act, P.wgt, (float*)P.out, splits, P.kb_per_split, sl > 0);
      if (!st.good()) return st;
      continue;
    }
    fill_divs(P);
    dim3 grid((P.M + BM - 1) / BM, g.K / BN, splits);
    Status st = BN == 128 ? launch<WGRAD, 128>(a, P, grid) : launch<WGRAD, 64>(a, P, grid);
    if (!st.good()) return st;
  }
  if (nw.s2d)
    wgrad_reduce_s2d<<<(unsigned)((g0.K * g0.R * g0.S * g0.C + 31) / 32), 256, 0, a.stream>>>(
        splits, RSC, g.K, part, dw, g0.R, g0.S, g0.C, g.S, g.pad, g0.pad);
  else
    wgrad_reduce<<<dim3((g.K + 31) / 32, (RSC + 31) / 32), 1024, 0, a.stream>>>(splits, RSC, g.K, g.C, g.Cw, part,
                                                                               dw);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

}  // namespace oc
