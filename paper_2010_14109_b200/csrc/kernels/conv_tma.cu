// Convolution on the 5th-generation tensor cores with TMA-fed operands: a
// persistent, warp-specialised implicit GEMM.
//
//   warp 0      one elected thread issues the TMA loads of a K-block into a
//               ring of shared-memory stages (mbarrier full/empty pipeline);
//               the activation operand is gathered by the TMA engine in
//               im2col mode (a box of output pixels × 64 channels at one
//               filter tap, zero fill outside the image), the weight / dY
//               operand with tiled 2-D loads, both in the UMMA SWIZZLE_128B
//               canonical layouts
//   warp 1      one elected thread issues tcgen05.mma (bf16 × bf16 -> fp32)
//               into one of two TMEM accumulators, so the epilogue of tile t
//               overlaps the main loop of tile t+1
//   warps 2-5   epilogue: tcgen05.ld TMEM -> registers -> bf16 / fp32 rows;
//               fprop / stride-1 dgrad stage 32 × 64 bf16 boxes in shared
//               memory (SWIZZLE_128B) and store them with TMA, optionally
//               summing Σy, Σy² per channel for the BN that follows
//
// One CTA per SM loops over tiles (tile u, u + gridDim.x, ...).  CG = 2 runs
// CTA pairs (cta_group::2, a 2-CTA cluster on one TPC): 256-row MMAs issued by
// the leader, each CTA staging its own A rows and half of the B columns (the
// operand traffic per FLOP that bounds the single-CTA kernel).
//   fprop   D[(n,p,q)][k] = Σ_{r,s,c} X[n, p·st−pad+r, q·st−pad+s, c] · W[k,r,s,c]
//   dgrad   per output phase (h mod st, w mod st), a stride-1 gather over dY
//           at the phase's taps only, W's taps reversed so the im2col offsets
//           run forward: stride 1 gives D[(n,h,w)][c] = Σ_{r',s',k}
//           dY[n, h−pad'+r', w−pad'+s', k] · W[k, R−1−r', S−1−s', c], pad' = R−1−pad
//   wgrad   D[(r,s,c)][k] = Σ_{(n,p,q)} X[n, p·st−pad+r, q·st−pad+s, c] · dY[(n,p,q), k]:
//           A = two im2col boxes of 64 pixels × 64 channels (MN-major),
//           B = dY rows (MN-major), deterministic split-K over pixel blocks
//   narrow  fprop over 8- or 16-channel (16 / 32-byte) pixels: 8 or 4 im2col
//           boxes of 128 pixels per K-block, one filter tap each, in the
//           no-swizzle core-matrix layout (LBO = 2 KB between taps) or the
//           SWIZZLE_32B layout (one tap per K-step)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "tc_util.cuh"

namespace oc {
namespace tma {

using namespace tcu;

constexpr int BM = 128, BK = 64, NTHREADS = 192;
constexpr int WKB = 128;   // wgrad K-block: 128 pixels (one 16 KB MN-major atom column per 64 channels)
__host__ __device__ constexpr int kblock(int mode) { return mode == 2 ? WKB : BK; }
// stages: as many as fit 192 KB (at most 8); fprop / dgrad add 32 KB of
// epilogue staging (two 32-row × 64-column bf16 boxes per epilogue warp)
constexpr int STG_BYTES = 8 * 4096;
// accumulating epilogue: the old output boxes stream through two more 4 KB
// buffers per epilogue warp, loaded two boxes ahead (the ring gives up 32 KB)
constexpr int OLD_BYTES = 8 * 4096;
__host__ __device__ constexpr int tma_stage_bytes(int bn, int mt, int kb) { return mt * BM * kb * 2 + bn * kb * 2; }
__host__ __device__ constexpr int tma_stages(int bn, int mt, int kb, bool acc = false) {
  return (192 * 1024 - (acc ? OLD_BYTES : 0)) / tma_stage_bytes(bn, mt, kb) < 8
             ? (192 * 1024 - (acc ? OLD_BYTES : 0)) / tma_stage_bytes(bn, mt, kb)
             : 8;
}
__host__ __device__ constexpr int tma_smem(int bn, int mt, int kb, bool acc = false) {
  return tma_stages(bn, mt, kb, acc) * tma_stage_bytes(bn, mt, kb) + (kb == WKB ? 0 : STG_BYTES) +
         (acc ? OLD_BYTES : 0) + 1024 + 256;
}

struct Params {
  CUtensorMap ta;          // im2col map of the gathered activation (X or dY)
  CUtensorMap tb;          // tiled map of the other operand (W_bf16, Wt_bf16 or dY)
  CUtensorMap tc;          // tstore: tiled map of the bf16 output rows (boxes of 32 rows × 64 columns, SWIZZLE_128B)
  int tstore;              // 1: the epilogue stores through shared memory with TMA (row-contiguous output)
  float* stat_part;        // tstore + fused BN statistics: part[slot][2][N] (Σy, Σy² of the stored bf16 values)
  void* out;               // bf16 [M][N] rows, or fp32 wgrad partials [z][M][N]
  int nst;                 // fprop/dgrad: stored columns (row stride) when N is zero-padded; 0 = N
  int accumulate;          // out = rnd(acc + out)
  int M, N;                // GEMM rows / columns
  int num_m, num_n, splits;
  int nkb;                 // fprop/dgrad: K-blocks per tile; wgrad: pixel blocks in all
  int kb_per_split;        // wgrad
  int Pd, Qd, st, padh, padw;  // im2col base of output pixel (n,p,q): (w, h) = (q·st − padw, p·st − padh)
  int R, S, Cr;            // im2col tap grid (dgrad: the phase's nr × ns); channels reduced per tap
  // dgrad phase (ph, pw) of stride dst: im2col tap (i', j') is filter tap
  // (r0 + dst·(R−1−i'), s0 + dst·(S−1−j')) of W (width Sw), and GEMM row
  // (n, h', w') is dx pixel (n, h'·dst + ph, w'·dst + pw) of an Ho × Wo map
  int Sw, r0, s0, dst, ph, pw, Ho, Wo;
  FastDiv fQ, fP, fCb, fS;
  unsigned long long* probe;   // launch probe (timeline mode), or null
  int dil;                     // im2col tap offsets × dil (atrous convs); 0/1 = none
};

__device__ __forceinline__ void base_of(const Params& P, int pix, int& w, int& h, int& n) {
  const uint32_t t = P.fQ.div((uint32_t)pix);
  const int q = pix - (int)t * P.Qd;
  const uint32_t nn = P.fP.div(t);
  const int p = (int)t - (int)nn * P.Pd;
  w = q * P.st - P.padw;
  h = p * P.st - P.padh;
  n = (int)nn;
}

// CG = 2: CTA pairs (cta_group::2).  A unit is MT tiles of 256 rows (CTA rank
// r holds rows 128·r .. 128·r + 127 of each) × BN columns; each CTA stages its
// own A rows and B columns [BN/2·r, BN/2·(r+1)), rank 0 issues 256 × BN MMAs.
// ACC: the TMA-store epilogue accumulates into the existing output (P.accumulate
// with P.tstore) — a separate instantiation, so the plain epilogue's code is unchanged
template <int MODE, int BN, int NCH, int MT, int CG = 1, bool ACC = false>
__global__ void __launch_bounds__(NTHREADS, 1) conv_tma_kernel(const __grid_constant__ Params P) {
  static_assert(CG == 1 || (NCH == 0 && (MODE != WGRAD || BN / CG >= 64)), "CTA pairs: 64-channel pixels; wgrad: whole 64-column B atoms per CTA");
  constexpr int KB = kblock(MODE);              // K extent of a stage (elements, or wgrad pixels)
  constexpr int ATOM = KB * 128;                 // wgrad: one 64-wide MN-major atom column
  constexpr int NST = tma_stages(BN / CG, MT, KB, ACC);
  static_assert(NST >= 2, "conv_tma: at least two ring stages");
  constexpr int A_TILE = BM * KB * 2, A_BYTES = MT * A_TILE, B_BYTES = (BN / CG) * KB * 2, STAGE = A_BYTES + B_BYTES;
  constexpr uint32_t TCOLS = 2 * MT * BN;   // two accumulator sets of MT tiles × BN columns
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* stg = smem + NST * STAGE;   // epilogue staging (fprop / dgrad)
  uint8_t* obuf = stg + STG_BYTES;     // ACC: old-output boxes (warp q, buffer b) at (2q + b) · 4 KB
  uint64_t* full = (uint64_t*)(stg + (MODE == WGRAD ? 0 : STG_BYTES) + (ACC ? OLD_BYTES : 0));
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;
  uint64_t* tempty = tfull + 2;
  uint64_t* ldbar = tempty + 2;        // accumulate epilogue: old-output box loads into obuf (warp q, buffer b) -> 2q + b
  uint32_t* tmem_slot = (uint32_t*)(ldbar + 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  KProbe kp;
  if (threadIdx.x == 0) probe_begin(kp);

  if (NCH) {
    // taps past R·S are never loaded; their (weight-zero) A columns must hold
    // finite values, so the stages start zeroed
    for (int i = threadIdx.x; i < NST * STAGE / 16; i += NTHREADS)
      asm volatile("st.shared.v4.b32 [%0], {%1,%1,%1,%1};" ::"r"(smem_u32(smem) + i * 16), "r"(0) : "memory");
    fence_async_smem();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&P.ta);
    tma_prefetch(&P.tb);
    for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4 * CG); }
    for (int b = 0; b < 8; ++b) mbar_init(&ldbar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(TCOLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(TCOLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (CG == 2) cluster_sync();   // peer barriers initialised before any remote arrive
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;
  const int u0 = blockIdx.x / CG, ustep = gridDim.x / CG;

  // a unit = MT consecutive 128-row tiles (super-tile mt) × one BN column block (× one split)
  const int units = P.num_m * P.num_n * (MODE == WGRAD ? P.splits : 1);
  auto unit_of = [&](int u, int& mt, int& nt, int& z, int& kb0, int& nk) {
    nt = u % P.num_n;
    const int t = u / P.num_n;
    mt = t % P.num_m;
    z = t / P.num_m;
    if (MODE == WGRAD) {
      kb0 = z * P.kb_per_split;
      nk = P.nkb - kb0 < P.kb_per_split ? P.nkb - kb0 : P.kb_per_split;
      if (nk < 0) nk = 0;
    } else {
      kb0 = 0;
      nk = P.nkb;
    }
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t it = 0;
      for (int u = u0; u < units; u += ustep) {
        int mt, nt, z, kb0, nk;
        unit_of(u, mt, nt, z, kb0, nk);
        int bw[MT], bh[MT], bn[MT];
#pragma unroll
        for (int t = 0; t < MT; ++t) {
          bw[t] = bh[t] = bn[t] = 0;
          if (MODE != WGRAD) base_of(P, ((mt * MT + t) * CG + (int)rank) * BM, bw[t], bh[t], bn[t]);
        }
        for (int i = 0; i < nk; ++i, ++it) {
          const int sg = (int)(it % NST);
          if (it >= (uint32_t)NST) mbar_wait(&empty[sg], ((it / NST) - 1) & 1);
          const uint32_t a = smem_u32(smem + sg * STAGE), b = a + A_BYTES;
          const int kb = kb0 + i;
          if (MODE == WGRAD && NCH == 16) {
            // 16-channel input (the space-to-depth stem): 8 taps per 128-row tile,
            // one box of KB pixels × 16 channels (SWIZZLE_32B) each
            int pw, ph, pn;
            base_of(P, kb * KB, pw, ph, pn);
            constexpr int BOX = KB * 32;
            const int t0 = mt * 8;
            int ntap = P.R * P.S - t0;
            ntap = ntap < 8 ? ntap : 8;
            mbar_expect_tx(&full[sg], B_BYTES + ntap * BOX);
            for (int j = 0; j < ntap; ++j) {
              const int r = (int)P.fS.div((uint32_t)(t0 + j)), s = t0 + j - r * P.S;
              tma_load_im2col(a + j * BOX, &P.ta, &full[sg], 0, pw, ph, pn, (uint16_t)s, (uint16_t)r);
            }
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tma_load_2d(b + j * ATOM, &P.tb, &full[sg], nt * BN + j * 64, kb * KB);
          } else if (MODE == WGRAD) {
            int pw, ph, pn;
            base_of(P, kb * KB, pw, ph, pn);
            // 64-row (tap, 64-channel) blocks of (r,s,c) inside the M range
            // (pair: this CTA's 128 rows, and half of the BN columns)
            auto nrb_of = [&](int rk) {
              const int n = (P.M + 63) / 64 - (mt * MT * CG + rk) * 2;
              return n < 0 ? 0 : (n < 2 * MT ? n : 2 * MT);
            };
            const int rb0 = (mt * MT * CG + (int)rank) * 2;
            const int nrb = nrb_of((int)rank);
            if (CG == 2) {
              const uint32_t fb = mapa(smem_u32(&full[sg]), 0);
              if (rank == 0) mbar_expect_tx(&full[sg], 2 * B_BYTES + (nrb_of(0) + nrb_of(1)) * ATOM);
              for (int j = 0; j < nrb; ++j) {
                const int blk = rb0 + j;
                const int tap = (int)P.fCb.div((uint32_t)blk), cb = blk - tap * (P.Cr / 64);
                const int dl = P.dil > 1 ? P.dil : 1;
                const int r = (int)P.fS.div((uint32_t)tap) * dl, s = (tap - (r / dl) * P.S) * dl;
                tma_load_im2col_pair(a + j * ATOM, &P.ta, fb, cb * 64, pw, ph, pn, (uint16_t)s, (uint16_t)r);
              }
#pragma unroll
              for (int j = 0; j < BN / CG / 64; ++j)
                tma_load_2d_pair(b + j * ATOM, &P.tb, fb, nt * BN + (int)rank * (BN / CG) + j * 64, kb * KB);
            } else {
              mbar_expect_tx(&full[sg], B_BYTES + nrb * ATOM);
              for (int j = 0; j < nrb; ++j) {
                const int blk = rb0 + j;
                const int tap = (int)P.fCb.div((uint32_t)blk), cb = blk - tap * (P.Cr / 64);
                const int dl = P.dil > 1 ? P.dil : 1;
                const int r = (int)P.fS.div((uint32_t)tap) * dl, s = (tap - (r / dl) * P.S) * dl;
                tma_load_im2col(a + j * ATOM, &P.ta, &full[sg], cb * 64, pw, ph, pn, (uint16_t)s, (uint16_t)r);
              }
#pragma unroll
              for (int j = 0; j < BN / 64; ++j) tma_load_2d(b + j * ATOM, &P.tb, &full[sg], nt * BN + j * 64, kb * KB);
            }
          } else if (NCH) {
            // 64 / NCH taps per K-block, one box of 128 pixels × NCH channels each
            constexpr int TPB = 64 / (NCH ? NCH : 64), BOX = BM * NCH * 2;
            const int t0 = kb * TPB;
            int ntap = P.R * P.S - t0;
            ntap = ntap < TPB ? ntap : TPB;
            mbar_expect_tx(&full[sg], B_BYTES + MT * ntap * BOX);
#pragma unroll
            for (int t = 0; t < MT; ++t)
              for (int j = 0; j < ntap; ++j) {
                const int r = (int)P.fS.div((uint32_t)(t0 + j)), s = t0 + j - r * P.S;
                tma_load_im2col(a + t * A_TILE + j * BOX, &P.ta, &full[sg], 0, bw[t], bh[t], bn[t], (uint16_t)s,
                                (uint16_t)r);
              }
            tma_load_2d(b, &P.tb, &full[sg], kb * BK, nt * BN);
          } else {
            const int tap = (int)P.fCb.div((uint32_t)kb), cb = kb - tap * (P.Cr / 64);
            const int r0_ = (int)P.fS.div((uint32_t)tap), s0_ = tap - r0_ * P.S;
            const int btap = MODE == DGRAD ? (P.r0 + P.dst * (P.R - 1 - r0_)) * P.Sw + P.s0 + P.dst * (P.S - 1 - s0_)
                                           : tap;
            const int dl = P.dil > 1 ? P.dil : 1;
            const int r = r0_ * dl, s = s0_ * dl;   // im2col offsets (dilated taps)
            if (CG == 2) {
              // both CTAs' bytes land on the leader's barrier
              const uint32_t fb = mapa(smem_u32(&full[sg]), 0);
              if (rank == 0) mbar_expect_tx(&full[sg], CG * STAGE);
#pragma unroll
              for (int t = 0; t < MT; ++t)
                tma_load_im2col_pair(a + t * A_TILE, &P.ta, fb, cb * 64, bw[t], bh[t], bn[t], (uint16_t)s,
                                     (uint16_t)r);
              tma_load_2d_pair(b, &P.tb, fb, btap * P.Cr + cb * 64, nt * BN + (int)rank * (BN / CG));
            } else {
              mbar_expect_tx(&full[sg], STAGE);
#pragma unroll
              for (int t = 0; t < MT; ++t)
                tma_load_im2col(a + t * A_TILE, &P.ta, &full[sg], cb * 64, bw[t], bh[t], bn[t], (uint16_t)s,
                                (uint16_t)r);
              tma_load_2d(b, &P.tb, &full[sg], btap * P.Cr + cb * 64, nt * BN);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (pair: the leader only)
    constexpr uint32_t ID = idesc_m(BM * CG, BN, MODE == WGRAD, MODE == WGRAD);
    uint32_t it = 0, lt = 0;
    for (int u = (CG == 2 && rank != 0) ? units : u0; u < units; u += ustep, ++lt) {
      int mt, nt, z, kb0, nk;
      unit_of(u, mt, nt, z, kb0, nk);
      const uint32_t buf = lt & 1;
      if (lt >= 2) mbar_wait(&tempty[buf], ((lt >> 1) - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t d = tmem + buf * MT * BN;
      for (int i = 0; i < nk; ++i, ++it) {
        const int sg = (int)(it % NST);
        mbar_wait(&full[sg], (it / NST) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
          const uint32_t a0 = smem_u32(smem + sg * STAGE), b = a0 + A_BYTES;
#pragma unroll
          for (int k = 0; k < KB / 16; ++k) {
            uint64_t db;
            if (MODE == WGRAD) db = sdesc(b + k * 2048, ATOM, 1024);   // MN-major: atom columns ATOM apart, K groups 1 KB
            else db = sdesc(b + k * 32, 16, 1024);                      // K-major SWIZZLE_128B
#pragma unroll
            for (int t = 0; t < MT; ++t) {
              const uint32_t a = a0 + t * A_TILE;
              uint64_t da;
              if (MODE == WGRAD && NCH == 16) da = sdesc(a + k * 512, KB * 32, 256, 6);   // MN-major SW32: taps KB·32 B apart
              else if (MODE == WGRAD) da = sdesc(a + k * 2048, ATOM, 1024);
              else if (NCH == 8) da = sdesc(a + k * 2 * 2048, 2048, 128, 0);   // no swizzle: taps 2 KB apart
              else if (NCH == 16) da = sdesc(a + k * 4096, 16, 256, 6);        // SWIZZLE_32B: one tap per K-step
              else da = sdesc(a + k * 32, 16, 1024);
              if (CG == 2) mma_bf16_pair(d + t * BN, da, db, ID, (i > 0 || k > 0) ? 1u : 0u);
              else mma_bf16(d + t * BN, da, db, ID, (i > 0 || k > 0) ? 1u : 0u);
            }
          }
          if (CG == 2) mma_commit_pair(&empty[sg]);
          else mma_commit(&empty[sg]);
        }
        __syncwarp();
      }
      if (lane == 0) {
        if (CG == 2) mma_commit_pair(&tfull[buf]);
        else mma_commit(&tfull[buf]);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2-5)
    const int q = warp & 3;            // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;
    uint32_t lt = 0, sc = 0;
    // TMA-store epilogue: the warp's 32 rows × 64 columns go to a SWIZZLE_128B
    // staging box (row r's 16-byte chunk c at r·128 + (c ^ r % 8)·16: the
    // rows' stores spread over all banks) and one lane stores the box with
    // TMA — whole 128-byte row segments instead of 32 rows × 16 bytes per
    // instruction
    if (MODE != WGRAD && P.tstore) {
      // fused BN statistics: the grid is a multiple of num_n, so a CTA's N
      // block (u mod num_n) is fixed and lane l owns columns 2l, 2l+1 of each
      // 64-column box for the whole launch (fixed order: bitwise reproducible)
      float ssum[BN / 64][2], ssq[BN / 64][2];
#pragma unroll
      for (int jb = 0; jb < BN / 64; ++jb) ssum[jb][0] = ssum[jb][1] = ssq[jb][0] = ssq[jb][1] = 0.f;
      // ACC: this warp's boxes form one stream over its tiles (box s = tile
      // lt, box b of NB, s = lt·NB + b); box s+2 is loaded into obuf buffer
      // s & 1 as soon as box s has been consumed, so each load has two boxes
      // of epilogue work (and the next tile's MMA wait) to arrive in
      constexpr int NB = MT * (BN / 64);
      auto issue_old = [&](uint32_t sidx) {
        const int uu = u0 + (int)(sidx / NB) * ustep;
        if (uu >= units) return;
        int mt_, nt_, z_, kb0_, nk_;
        unit_of(uu, mt_, nt_, z_, kb0_, nk_);
        const int bb = (int)(sidx % NB), t_ = bb / (BN / 64), j_ = (bb % (BN / 64)) * 64;
        uint64_t* lb = &ldbar[q * 2 + (sidx & 1)];
        mbar_expect_tx(lb, 4096);
        tma_load_2d(smem_u32(obuf) + (uint32_t)(q * 2 + (sidx & 1)) * 4096u, &P.tc, lb, nt_ * BN + j_,
                    ((mt_ * MT + t_) * CG + (int)rank) * BM + q * 32);
      };
      if (ACC && lane == 0) {
        issue_old(0);
        if (NB > 1 || u0 + ustep < units) issue_old(1);
      }
      for (int u = u0; u < units; u += ustep, ++lt) {
        int mt, nt, z, kb0, nk;
        unit_of(u, mt, nt, z, kb0, nk);
        const uint32_t buf = lt & 1;
        mbar_wait(&tfull[buf], (lt >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int t = 0; t < MT; ++t) {
          const int row0 = ((mt * MT + t) * CG + (int)rank) * BM + q * 32;
#pragma unroll
          for (int j0 = 0; j0 < BN; j0 += 64, ++sc) {
            uint32_t v0[32], v1[32];
            const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (buf * MT + t) * BN + j0;
            TMEM_LD32(ta, v0);
            TMEM_LD32(ta + 32, v1);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");   // this buffer's last store read
            __syncwarp();
            const uint32_t sb = smem_u32(stg) + (uint32_t)(q * 2 + (sc & 1)) * 4096u;
            if constexpr (!ACC) {
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                uint32_t w[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const uint32_t lo = c < 4 ? v0[c * 8 + 2 * e] : v1[(c - 4) * 8 + 2 * e];
                  const uint32_t hi = c < 4 ? v0[c * 8 + 2 * e + 1] : v1[(c - 4) * 8 + 2 * e + 1];
                  __nv_bfloat162 h2 =
                      __floats2bfloat162_rn(nk ? __uint_as_float(lo) : 0.f, nk ? __uint_as_float(hi) : 0.f);
                  w[e] = *reinterpret_cast<uint32_t*>(&h2);
                }
                asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(sb + lane * 128 + ((c ^ (lane & 7)) << 4)),
                             "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                             : "memory");
              }
            } else {
              // out = rnd(old + acc): the old box arrived by TMA (issued two
              // boxes earlier) in the swizzled layout the store uses (rows past M zero-filled)
              const uint32_t ob = smem_u32(obuf) + (uint32_t)(q * 2 + (sc & 1)) * 4096u;
              mbar_wait(&ldbar[q * 2 + (sc & 1)], (sc >> 1) & 1);
              uint32_t old[8][4];
#pragma unroll
              for (int c = 0; c < 8; ++c)
                asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(old[c][0]), "=r"(old[c][1]), "=r"(old[c][2]), "=r"(old[c][3])
                             : "r"(ob + lane * 128 + ((c ^ (lane & 7)) << 4))
                             : "memory");
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                uint32_t w[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const uint32_t lo = c < 4 ? v0[c * 8 + 2 * e] : v1[(c - 4) * 8 + 2 * e];
                  const uint32_t hi = c < 4 ? v0[c * 8 + 2 * e + 1] : v1[(c - 4) * 8 + 2 * e + 1];
                  const float2 o2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&old[c][e]));
                  __nv_bfloat162 h2 = __floats2bfloat162_rn((nk ? __uint_as_float(lo) : 0.f) + o2.x,
                                                            (nk ? __uint_as_float(hi) : 0.f) + o2.y);
                  w[e] = *reinterpret_cast<uint32_t*>(&h2);
                }
                asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(sb + lane * 128 + ((c ^ (lane & 7)) << 4)),
                             "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                             : "memory");
              }
            }
            fence_async_smem();
            __syncwarp();
            if (ACC && lane == 0) issue_old(sc + 2);   // obuf (sc & 1) consumed: load box sc + 2 into it
            if (P.stat_part) {
              // column sums of the 32 staged rows (conflict-free: the swizzle
              // spreads a row's eight 16-byte chunks over all banks); rows past M are zero
              // (plain loads, all issued before the sums: the row order of the sums is fixed)
              const uint8_t* sbp = stg + (q * 2 + (sc & 1)) * 4096 + (lane & 3) * 4;
              uint32_t wv[32];
#pragma unroll
              for (int r = 0; r < 32; ++r)
                wv[r] = *reinterpret_cast<const uint32_t*>(sbp + r * 128 + ((((uint32_t)lane >> 2) ^ (uint32_t)(r & 7)) << 4));
              float s0 = 0.f, s1 = 0.f, q0 = 0.f, q1 = 0.f;
#pragma unroll
              for (int r = 0; r < 32; ++r) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&wv[r]));
                s0 += f.x;
                s1 += f.y;
                q0 = fmaf(f.x, f.x, q0);
                q1 = fmaf(f.y, f.y, q1);
              }
              ssum[j0 / 64][0] += s0;
              ssum[j0 / 64][1] += s1;
              ssq[j0 / 64][0] += q0;
              ssq[j0 / 64][1] += q1;
            }
            if (lane == 0) {
              if (row0 < P.M && nt * BN + j0 < (P.nst ? P.nst : P.N))
                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&P.tc),
                             "r"(sb), "r"(nt * BN + j0), "r"(row0)
                             : "memory");
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          if (CG == 2) mbar_arrive_cluster(mapa(smem_u32(&tempty[buf]), 0));
          else mbar_arrive(&tempty[buf]);
        }
      }
      if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      __syncwarp();
      if (P.stat_part && u0 < units) {
        const int slot = (u0 / P.num_n) * (4 * CG) + (int)rank * 4 + q;
        const int nt = u0 % P.num_n;
        float* pp = P.stat_part + (int64_t)slot * 2 * P.N;
#pragma unroll
        for (int jb = 0; jb < BN / 64; ++jb) {
          const int c = nt * BN + jb * 64 + 2 * lane;
          *reinterpret_cast<float2*>(pp + c) = make_float2(ssum[jb][0], ssum[jb][1]);
          *reinterpret_cast<float2*>(pp + P.N + c) = make_float2(ssq[jb][0], ssq[jb][1]);
        }
      }
    } else
    for (int u = u0; u < units; u += ustep, ++lt) {
      int mt, nt, z, kb0, nk;
      unit_of(u, mt, nt, z, kb0, nk);
      const uint32_t buf = lt & 1;
      mbar_wait(&tfull[buf], (lt >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        const int m = ((mt * MT + t) * CG + (int)rank) * BM + row;
        int64_t orow = m;
        if (MODE == DGRAD && m < P.M) {
          int w, h, n;
          base_of(P, m, w, h, n);     // (w, h) = (w' − pad', h' − pad')
          orow = ((int64_t)n * P.Ho + (h + P.padh) * P.dst + P.ph) * P.Wo + (w + P.padw) * P.dst + P.pw;
        }
#pragma unroll
        for (int j0 = 0; j0 < BN; j0 += 32) {
          uint32_t v[32];
          TMEM_LD32(tmem + ((uint32_t)(q * 32) << 16) + (buf * MT + t) * BN + j0, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (nk == 0) {
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = 0u;
          }
          if (m >= P.M) continue;
          const int col = nt * BN + j0;
          if (MODE == WGRAD) {
            float* o = (float*)P.out + ((int64_t)z * P.M + m) * P.N + col;
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
            const int nst = P.nst ? P.nst : P.N;   // padded output channels past nst are not stored
            __nv_bfloat16* o = (__nv_bfloat16*)P.out + orow * nst + col;
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
              if (col + i >= nst) break;
              float f[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(v[i + e]);
              if (P.accumulate) {
                uint4 old = *reinterpret_cast<const uint4*>(o + i);
                const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&old);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 ff = __bfloat1622float2(h2[e]);
                  f[2 * e] += ff.x;
                  f[2 * e + 1] += ff.y;
                }
              }
              uint4 pk;
              __nv_bfloat162* p2 = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
              for (int e = 0; e < 4; ++e) p2[e] = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
              *reinterpret_cast<uint4*>(o + i) = pk;
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) mbar_arrive_cluster(mapa(smem_u32(&tempty[buf]), 0));
        else mbar_arrive(&tempty[buf]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (CG == 2) cluster_sync();   // the leader's MMAs read this CTA's stages and write its TMEM
  else __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (CG == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
  }
  if (threadIdx.x == 0) probe_end(P.probe, kp);
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// CTA pairs the device can hold at once (one 2-CTA cluster per TPC at our
// shared-memory footprint); 74 on a 148-SM B200
int max_pairs() {
  static int n = 0;
  if (!n) {
    n = sm_count() / 2;
  }
  return n;
}

// Upper bound on the persistent grid, read at every launch (OC_CONV_MAX_CTAS,
// tests only): with a few CTAs every CTA loops over many work units, so the
// parity tests reach the persistent-loop regime the full-size step runs in
// (mbarrier phase wrap, TMEM double-buffer alternation, stat slots summed
// across units) on shapes the oracle finishes in seconds.
int grid_cap(int ctas) {
  const char* e = std::getenv("OC_CONV_MAX_CTAS");
  const int cap = e ? std::atoi(e) : 0;
  return (cap > 0 && cap < ctas) ? cap : ctas;
}

// epilogue statistics slots one launch may write (CTA x epilogue warp); the
// BN-statistics workspace is sized from this (conv_tc_stat_ws)
int stat_slots_max() { return sm_count() * 4; }

Status encode_fail(CUresult r, const char* what) { return cu_status(r, what); }

// NHWC bf16 activation [N][H][W][C] gathered for an output grid Pd × Qd
Status make_im2col(CUtensorMap* m, const void* base, int N, int H, int W, int C, int ch, int pix, int Pd, int Qd,
                   int st, int padh, int padw, CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B) {
  Driver* d;
  std::string msg;
  if (!driver(d, msg)) return Status::make(OC_E_CUDA, msg);
  const cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  const cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
  // bounding box of the base pixels, {W, H}: first at −pad, last at (Q−1)·st − pad
  const int lower[2] = {-padw, -padh};
  const int upper[2] = {(Qd - 1) * st - padw - (W - 1), (Pd - 1) * st - padh - (H - 1)};
  const cuuint32_t es[4] = {1, (cuuint32_t)st, (cuuint32_t)st, 1};
  CUresult r = d->TensorMapEncodeIm2col(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
                                        lower, upper, (cuuint32_t)ch, (cuuint32_t)pix, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? Status::ok() : encode_fail(r, "cuTensorMapEncodeIm2col");
}

// row-major bf16 [rows][cols], boxes of 64 columns × box_rows rows, SWIZZLE_128B
Status make_tiled(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint32_t box_rows) {
  Driver* d;
  std::string msg;
  if (!driver(d, msg)) return Status::make(OC_E_CUDA, msg);
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = d->TensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                                       box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? Status::ok() : encode_fail(r, "cuTensorMapEncodeTiled");
}

// the TMA-store epilogue for row-contiguous bf16 outputs that are not accumulated
Status set_tstore(Params& P, void* out, int rows, int cols_stored, bool ok) {
  P.tstore = 0;
  if (!ok || cols_stored % 8) return Status::ok();
  Status st = make_tiled(&P.tc, out, (uint64_t)cols_stored, (uint64_t)rows, 32);
  if (!st.good()) return st;
  P.tstore = 1;
  return Status::ok();
}

void fill(Params& P) {
  P.fQ.init(P.Qd);
  P.fP.init(P.Pd);
  P.fCb.init(P.Cr / 64 > 0 ? P.Cr / 64 : 1);
  P.fS.init(P.S);
}

int conv_mt() { return 2; }

template <int MODE, int BN, int NCH, int MT, int CG = 1>
Status launch_mt(OpArgs& a, Params P, int* stat_slots = nullptr) {
  int smem = tma_smem(BN / CG, MT, kblock(MODE));
  auto kern = conv_tma_kernel<MODE, BN, NCH, MT, CG, false>;
  if constexpr (MODE != WGRAD && NCH == 0)
    if (P.accumulate && P.tstore) {
      kern = conv_tma_kernel<MODE, BN, NCH, MT, CG, true>;
      smem = tma_smem(BN / CG, MT, kblock(MODE), true);
    }
  static bool attr[2] = {false, false};
  const int ai = (P.accumulate && P.tstore) ? 1 : 0;
  if (!attr[ai]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (CG == 2) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
    attr[ai] = true;
  }
  P.num_m = (P.M + BM * MT * CG - 1) / (BM * MT * CG);   // super-tiles of MT × (128·CG) rows
  const int units = P.num_m * P.num_n * (MODE == WGRAD ? P.splits : 1);
  if (units == 0) return Status::ok();
  int ctas = std::min(units, CG == 1 ? sm_count() : max_pairs());   // CTAs, or pairs
  ctas = CG == 1 ? grid_cap(ctas) : std::max(1, grid_cap(2 * ctas) / 2);
  if (P.stat_part) {
    // fused statistics: whole groups of num_n CTAs (pairs), 4·CG slots per group member
    // (units = num_m · num_n >= num_n, so a capped grid rounds up to one group)
    ctas = std::max(ctas / P.num_n, 1) * P.num_n;
    if (ctas > (CG == 1 ? sm_count() : max_pairs()))
      return Status::make(OC_E_INVARIANT, "conv: statistics epilogue needs num_n CTAs");
    if (ctas / P.num_n * 4 * CG > stat_slots_max())
      return Status::make(OC_E_INVARIANT, "conv: more statistics slots than the workspace holds");
    if (stat_slots) *stat_slots = ctas / P.num_n * 4 * CG;
  }
  if (a.ktimer) {
    P.probe = a.ktimer->probe_slot(a.stream);
    a.ktimer->begin(a.stream);
  }
  if (CG == 1) {
    kern<<<ctas, NTHREADS, smem, a.stream>>>(P);
  } else {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(NTHREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = a.stream;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(2 * ctas);
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, P);
    if (e != cudaSuccess) return cuda_status(e, "conv_tma pair launch");
  }
  if (a.ktimer) a.ktimer->end(a.stream);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

// wgrad keeps single 128-row tiles: its M = R·S·C is short (e.g. 576) and
// pairs would pad it further.
template <int MODE, int BN, int NCH>
Status launch(OpArgs& a, const Params& P, int* stat_slots = nullptr) {
  return (MODE != WGRAD && conv_mt() == 2) ? launch_mt<MODE, BN, NCH, 2>(a, P, stat_slots)
                                           : launch_mt<MODE, BN, NCH, 1>(a, P, stat_slots);
}

// Tile shape of the 64-channel fprop / dgrad GEMM (M rows, N columns).
// Shared memory feeds both the TMA writes and the UMMA operand reads
// (128 B/clk per SM); per 128 × N × 16 MMA step (N/2 cycles) a single CTA
// reads A (4 KB) + B (N·32 B) and the TMA writes the next K-block.  CTA pairs
// (cta_group::2) stage half of B per CTA, which lowers that traffic:
//   pair N=256: 128 B/clk at the MMA rate (fits), pair N=128 ×2 tiles: 176,
//   single N=128 ×2 tiles: 224 (the MMA can run at most ~57 %), pair N=64: 304,
//   single N=64: 352.  The choice weighs that against wave quantisation over
//   the persistent grid (148 CTAs or max_pairs() pairs).  OC_CONV_CG=1 keeps
//   single CTAs.
struct Tile { int bn, mt, cg; };
// nkb: 64-wide K-blocks per tile.  Short reductions (1×1 convs over ≤ 512
// channels, the phases of a strided dgrad) spend most of a unit in its
// epilogue; there single CTAs (and, for ≤ 2 K-blocks, single tiles) measured
// faster than pairs: ResNet-50 1×1 64→256 fprop 0.134 → 0.101 ms, the 3×3
// stride-2 dgrad phases 0.113 → 0.097 ms.
Tile choose_tile(int M, int N, int nkb) {
  const char* e = std::getenv("OC_CONV_CG");
  const int env = (e && e[0] == '1') ? 1 : 2;
  // OC_CONV_TILE="bn,mt,cg" forces one of the shapes below (tests)
  if (const char* f = std::getenv("OC_CONV_TILE")) {
    Tile t{0, 0, 0};
    if (std::sscanf(f, "%d,%d,%d", &t.bn, &t.mt, &t.cg) == 3 && t.bn > 0 && N % t.bn == 0 &&
        ((t.bn == 256 && t.mt == 1 && t.cg == 2) || ((t.bn == 128 || t.bn == 64) && t.mt == 2) ||
         ((t.bn == 128 || t.bn == 64) && t.mt == 1 && t.cg == 1)))
      return t;
  }
  if (nkb <= 8) return Tile{N % 128 == 0 ? 128 : 64, nkb <= 2 ? 1 : conv_mt(), 1};
  const Tile cand[5] = {{256, 1, 2}, {128, 2, 2}, {128, 2, 1}, {64, 2, 2}, {64, 2, 1}};
  const double eff[5] = {0.85, 128.0 / 176, 128.0 / 224, 128.0 / 304, 128.0 / 352};
  Tile best{N % 128 == 0 ? 128 : 64, conv_mt(), 1};
  double bt = 1e300;
  for (int i = 0; i < 5; ++i) {
    const Tile& t = cand[i];
    if (N % t.bn) continue;
    if (t.cg == 2 && env == 1) continue;
    if (t.mt != conv_mt() && t.cg == 1) continue;
    const int rows = BM * t.mt * t.cg;
    const long units = (long)((M + rows - 1) / rows) * (N / t.bn);
    const int slots = t.cg == 2 ? max_pairs() : sm_count();
    const double waves = (double)((units + slots - 1) / slots);
    const double time = waves * rows * t.bn / t.cg / eff[i];   // per SM
    if (time < bt * 0.999) { bt = time; best = t; }
  }
  return best;
}

template <int MODE>
Status launch_tile(OpArgs& a, const Params& P, Tile t, int* ss = nullptr) {
  if (t.cg == 2) {
    if (t.bn == 256) return launch_mt<MODE, 256, 0, 1, 2>(a, P, ss);
    if (t.bn == 128) return launch_mt<MODE, 128, 0, 2, 2>(a, P, ss);
    return launch_mt<MODE, 64, 0, 2, 2>(a, P, ss);
  }
  if (t.mt == 1) return t.bn == 128 ? launch_mt<MODE, 128, 0, 1>(a, P, ss) : launch_mt<MODE, 64, 0, 1>(a, P, ss);
  return t.bn == 128 ? launch_mt<MODE, 128, 0, 2>(a, P, ss) : launch_mt<MODE, 64, 0, 2>(a, P, ss);
}

// ---------------------------------------------------------------- stem
// The space-to-depth stem (a 4×4 stride-1 conv over 16-channel, 32-byte
// pixels, K = 64 outputs) gathered as halo tiles instead of im2col boxes:
// the im2col kernel fetches every 32-byte pixel once per tap (16×) and is
// L2→SM bound.  Here a unit is a 16 × 8 block of output pixels of one image;
// the producer loads, per horizontal tap j, one tiled box of 19 rows × 8
// pixels (SWIZZLE_32B, zero fill outside the image) — 4 boxes, 19 KB, for
// all 16 taps — and tap (i, j)'s A operand is box j from row i on (a
// 256-byte, pattern-aligned offset).  The whole weight W' (64 × 256 bf16,
// 32 KB) stays resident in shared memory.  Epilogue as the generic kernel's
// TMA-store path (4-D boxes of 4 × 8 pixels × 64 channels) with the fused
// BN statistics.
namespace stem {

constexpr int TH = 16, TW = 8, TAP = 4, HR = TH + TAP - 1;
constexpr int COPY = HR * TW * 32;              // 4864 B = 19 SW32 pattern repeats
constexpr int ASTAGE = TAP * COPY;              // 19456 B
constexpr int NSTG = 8;
constexpr int BBYTES = 4 * 8192;                // W': 4 SWIZZLE_128B boxes of 64 K × 64 rows
constexpr int SMEM = BBYTES + NSTG * ASTAGE + STG_BYTES + 1024 + 256;

struct Params {
  CUtensorMap tx;   // X' [N][H'][W'][16] bf16, box {16, 8, 19, 1}, SWIZZLE_32B
  CUtensorMap tw;   // W' [64][256] bf16, box {64, 64}, SWIZZLE_128B
  CUtensorMap ty;   // y [N][P][Q][64] bf16, box {64, 8, 4, 1}, SWIZZLE_128B
  int tq, tpq, units, pad;
  float* stat_part;   // fused BN statistics: part[slot][2][64]
  unsigned long long* probe;
};

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, uint64_t* b, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(dst),
      "l"(map), "r"(smem_u32(b)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__global__ void __launch_bounds__(NTHREADS, 1) stem_kernel(const __grid_constant__ Params P) {
  constexpr uint32_t TCOLS = 128;   // two 64-column accumulators
  KProbe kp;
  if (threadIdx.x == 0) probe_begin(kp);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* bsm = smem;
  uint8_t* asm_ = smem + BBYTES;
  uint8_t* stg = asm_ + NSTG * ASTAGE;
  uint64_t* full = (uint64_t*)(stg + STG_BYTES);
  uint64_t* empty = full + NSTG;
  uint64_t* tfull = empty + NSTG;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint32_t* tmem_slot = (uint32_t*)(bfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&P.tx);
    tma_prefetch(&P.tw);
    for (int s = 0; s < NSTG; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
    mbar_init(bfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  auto tile_of = [&](int u, int& n, int& p0, int& q0) {
    n = u / P.tpq;
    const int r = u - n * P.tpq;
    const int tp = r / P.tq;
    p0 = tp * TH;
    q0 = (r - tp * P.tq) * TW;
  };

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(bfull, BBYTES);
      for (int k = 0; k < 4; ++k) tma_load_2d(smem_u32(bsm) + k * 8192, &P.tw, bfull, k * 64, 0);
      uint32_t it = 0;
      for (int u = blockIdx.x; u < P.units; u += gridDim.x, ++it) {
        int n, p0, q0;
        tile_of(u, n, p0, q0);
        const int sg = (int)(it % NSTG);
        if (it >= (uint32_t)NSTG) mbar_wait(&empty[sg], ((it / NSTG) - 1) & 1);
        const uint32_t a = smem_u32(asm_) + sg * ASTAGE;
        mbar_expect_tx(&full[sg], ASTAGE);
#pragma unroll
        for (int j = 0; j < TAP; ++j) tma_load_4d(a + j * COPY, &P.tx, &full[sg], 0, q0 + j - P.pad, p0 - P.pad, n);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t ID = idesc(64, false, false);
    if (lane == 0) mbar_wait(bfull, 0);
    __syncwarp();
    uint32_t it = 0, lt = 0;
    for (int u = blockIdx.x; u < P.units; u += gridDim.x, ++it, ++lt) {
      const uint32_t buf = lt & 1;
      if (lt >= 2) mbar_wait(&tempty[buf], ((lt >> 1) - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int sg = (int)(it % NSTG);
      mbar_wait(&full[sg], (it / NSTG) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) {
        const uint32_t a = smem_u32(asm_) + sg * ASTAGE, b = smem_u32(bsm);
#pragma unroll
        for (int i = 0; i < TAP; ++i)
#pragma unroll
          for (int j = 0; j < TAP; ++j) {
            const int t = i * TAP + j;   // W' column block t·16 (tap (i, j), 16 channels)
            const uint64_t da = sdesc(a + j * COPY + i * 256, 16, 256, 6);
            const uint64_t db = sdesc(b + (t >> 2) * 8192 + (t & 3) * 32, 16, 1024);
            mma_bf16(tmem + buf * 64, da, db, ID, t > 0 ? 1u : 0u);
          }
        mma_commit(&empty[sg]);
        mma_commit(&tfull[buf]);
      }
      __syncwarp();
    }
  } else {
    const int q = warp & 3;
    float s0a = 0.f, s1a = 0.f, q0a = 0.f, q1a = 0.f;
    uint32_t lt = 0, sc = 0;
    for (int u = blockIdx.x; u < P.units; u += gridDim.x, ++lt, ++sc) {
      int n, p0, q0;
      tile_of(u, n, p0, q0);
      const uint32_t buf = lt & 1;
      mbar_wait(&tfull[buf], (lt >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t v0[32], v1[32];
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + buf * 64;
      TMEM_LD32(ta, v0);
      TMEM_LD32(ta + 32, v1);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);   // accumulator drained into registers
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
      const uint32_t sb = smem_u32(stg) + (uint32_t)(q * 2 + (sc & 1)) * 4096u;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t lo = c < 4 ? v0[c * 8 + 2 * e] : v1[(c - 4) * 8 + 2 * e];
          const uint32_t hi = c < 4 ? v0[c * 8 + 2 * e + 1] : v1[(c - 4) * 8 + 2 * e + 1];
          __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(lo), __uint_as_float(hi));
          w[e] = *reinterpret_cast<uint32_t*>(&h2);
        }
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(sb + lane * 128 + ((c ^ (lane & 7)) << 4)),
                     "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                     : "memory");
      }
      fence_async_smem();
      __syncwarp();
      if (P.stat_part) {
        const uint8_t* sbp = stg + (q * 2 + (sc & 1)) * 4096 + (lane & 3) * 4;
        uint32_t wv[32];
#pragma unroll
        for (int r = 0; r < 32; ++r)
          wv[r] = *reinterpret_cast<const uint32_t*>(sbp + r * 128 + ((((uint32_t)lane >> 2) ^ (uint32_t)(r & 7)) << 4));
        float s0 = 0.f, s1 = 0.f, q0s = 0.f, q1s = 0.f;
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&wv[r]));
          s0 += f.x;
          s1 += f.y;
          q0s = fmaf(f.x, f.x, q0s);
          q1s = fmaf(f.y, f.y, q1s);
        }
        s0a += s0;
        s1a += s1;
        q0a += q0s;
        q1a += q1s;
      }
      if (lane == 0) {
        asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(&P.ty),
                     "r"(sb), "r"(0), "r"(q0), "r"(p0 + q * 4), "r"(n)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
    if (P.stat_part) {
      float* pp = P.stat_part + (int64_t)(blockIdx.x * 4 + q) * 2 * 64;
      *reinterpret_cast<float2*>(pp + 2 * lane) = make_float2(s0a, s1a);
      *reinterpret_cast<float2*>(pp + 64 + 2 * lane) = make_float2(q0a, q1a);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
  }
  if (threadIdx.x == 0) probe_end(P.probe, kp);
}

// Weight gradient of the same stem, halo-gathered: dW'[(t, c)][k] = Σ_pixels
// X'(pixel shifted by tap t = (i, j))[c] · dY[pixel][k].  Per 16 × 8 tile of
// output pixels (one 128-pixel K-block) the producer loads, per j, a box of
// 23 rows × 8 pixels of X' (SWIZZLE_32B) and the tile's dY rows (SWIZZLE_128B).
// The MN-major A operand of horizontal tap j stacks 8 vertical taps i = 0..7
// (the four real ones and four that only fill the 128-row MMA) whose 16-channel
// atoms are the same box one pixel row apart: LBO = SBO = 256 bytes.  Each CTA
// accumulates its tiles in four TMEM accumulators (one per j) and writes its
// split partial part[z = CTA][(t, c)][k] once (slices after the first add).
constexpr int WHR = TH + 7;                    // 23 rows: vertical taps 0..7 over 16 rows
constexpr int WCOPY = WHR * TW * 32;           // 5888 B
constexpr int WSTAGE = TAP * WCOPY + TH * TW * 128;   // + dY tile 16 KB = 39936 B
constexpr int WNSTG = 5;
constexpr int WSMEM = WNSTG * WSTAGE + 1024 + 256;

struct WParams {
  CUtensorMap tx;   // X' box {16, 8, 23, 1}, SWIZZLE_32B
  CUtensorMap tdy;  // dY [N][P][Q][64] box {64, 8, 16, 1}, SWIZZLE_128B
  int tq, tpq, units, pad, accumulate;
  float* part;      // [gridDim.x][256][64]
  unsigned long long* probe;
};

__global__ void __launch_bounds__(NTHREADS, 1) stem_wgrad_kernel(const __grid_constant__ WParams P) {
  constexpr uint32_t TCOLS = 256;   // four 64-column accumulators (j = 0..3)
  KProbe kp;
  if (threadIdx.x == 0) probe_begin(kp);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + WNSTG * WSTAGE);
  uint64_t* empty = full + WNSTG;
  uint64_t* tfull = empty + WNSTG;
  uint32_t* tmem_slot = (uint32_t*)(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&P.tx);
    tma_prefetch(&P.tdy);
    for (int s = 0; s < WNSTG; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  auto tile_of = [&](int u, int& n, int& p0, int& q0) {
    n = u / P.tpq;
    const int r = u - n * P.tpq;
    const int tp = r / P.tq;
    p0 = tp * TH;
    q0 = (r - tp * P.tq) * TW;
  };
  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int u = blockIdx.x; u < P.units; u += gridDim.x, ++it) {
        int n, p0, q0;
        tile_of(u, n, p0, q0);
        const int sg = (int)(it % WNSTG);
        if (it >= (uint32_t)WNSTG) mbar_wait(&empty[sg], ((it / WNSTG) - 1) & 1);
        const uint32_t a = smem_u32(smem) + sg * WSTAGE;
        mbar_expect_tx(&full[sg], WSTAGE);
#pragma unroll
        for (int j = 0; j < TAP; ++j) tma_load_4d(a + j * WCOPY, &P.tx, &full[sg], 0, q0 + j - P.pad, p0 - P.pad, n);
        tma_load_4d(a + TAP * WCOPY, &P.tdy, &full[sg], 0, q0, p0, n);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t ID = idesc(64, true, true);
    uint32_t it = 0;
    for (int u = blockIdx.x; u < P.units; u += gridDim.x, ++it) {
      const int sg = (int)(it % WNSTG);
      mbar_wait(&full[sg], (it / WNSTG) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (lane == 0) {
        const uint32_t a = smem_u32(smem) + sg * WSTAGE, b = a + TAP * WCOPY;
#pragma unroll
        for (int k = 0; k < TH * TW / 16; ++k) {   // 16 pixels (two tile rows) per MMA
          const uint64_t db = sdesc(b + k * 2048, 16384, 1024);
#pragma unroll
          for (int j = 0; j < TAP; ++j)
            mma_bf16(tmem + j * 64, sdesc(a + j * WCOPY + k * 512, 256, 256, 6), db, ID, (it > 0 || k > 0) ? 1u : 0u);
        }
        mma_commit(&empty[sg]);
      }
      __syncwarp();
    }
    if (lane == 0) mma_commit(tfull);   // arrives once all issued MMAs completed (also with no units)
    __syncwarp();
  } else {
    const int q = warp & 3;
    const int r = q * 32 + lane;        // D row = (vertical tap i, channel c)
    const int i = r >> 4, c = r & 15;
    mbar_wait(tfull, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const bool any = blockIdx.x < P.units;
#pragma unroll
    for (int j = 0; j < TAP; ++j) {
      uint32_t v0[32], v1[32];
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + j * 64;
      TMEM_LD32(ta, v0);
      TMEM_LD32(ta + 32, v1);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (i >= TAP) continue;
      float* o = P.part + ((int64_t)blockIdx.x * 256 + (i * TAP + j) * 16 + c) * 64;
#pragma unroll
      for (int e = 0; e < 64; e += 4) {
        const uint32_t* v = e < 32 ? &v0[e] : &v1[e - 32];
        float4 f = any ? make_float4(__uint_as_float(v[0]), __uint_as_float(v[1]), __uint_as_float(v[2]),
                                     __uint_as_float(v[3]))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
        if (P.accumulate) {
          const float4 old = *reinterpret_cast<const float4*>(o + e);
          f.x += old.x; f.y += old.y; f.z += old.z; f.w += old.w;
        }
        *reinterpret_cast<float4*>(o + e) = f;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
  }
  if (threadIdx.x == 0) probe_end(P.probe, kp);
}

Status encode_tiled(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                    const cuuint32_t* box, CUtensorMapSwizzle sw) {
  Driver* d;
  std::string msg;
  if (!driver(d, msg)) return Status::make(OC_E_CUDA, msg);
  const cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = d->TensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims, strides,
                                       box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? Status::ok() : encode_fail(r, "cuTensorMapEncodeTiled (stem)");
}

}  // namespace stem

}  // namespace tma

using namespace tma;

// which kernel geometries the TMA kernels take (after the narrow-input re-layout)
bool conv_tma_ok(const ConvGeom& g, int mode) {
  if (g.pad > 127 || g.R > 64 || g.S > 64 || g.st > 8 || dil_of(g) * (g.R - 1) > 127) return false;
  if (dil_of(g) > 1 && (g.C % 64 != 0 || (mode == DGRAD && g.st != 1))) return false;
  if (g.nopadh && mode == DGRAD) return false;
  if (mode == FPROP) return g.K % 64 == 0 && (g.C % 64 == 0 || g.C == 8 || g.C == 16);
  if (mode == DGRAD) return g.C % 64 == 0 && g.K % 64 == 0;
  return (g.C % 64 == 0 || g.C == 16) && g.K % 64 == 0;
}

// y[M = N·P·Q][K] = im2col(x) · W_bf16[K][kpad]ᵀ
// nst (optional): the stored output channels when g.K is a zero-padded width
bool stem_enabled() {
  const char* e = std::getenv("OC_CONV_STEM");
  return !(e && e[0] == '0');
}

// the halo-tile stem kernel (namespace stem): 4×4 stride-1 conv over 16-channel
// pixels with 64 outputs, output map tiled exactly by 16 × 8 blocks
Status conv_stem_tma(OpArgs& a, const ConvGeom& g, const __nv_bfloat16* x, const __nv_bfloat16* wb, int kpad,
                     __nv_bfloat16* y, float* stat_part, int* stat_slots) {
  using namespace stem;
  stem::Params P{};
  {
    const cuuint64_t dims[4] = {16, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.N};
    const cuuint64_t strides[3] = {32, (cuuint64_t)g.W * 32, (cuuint64_t)g.H * g.W * 32};
    const cuuint32_t box[4] = {16, TW, HR, 1};
    OC_TRY(encode_tiled(&P.tx, x, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_32B));
  }
  OC_TRY(make_tiled(&P.tw, wb, (uint64_t)kpad, 64, 64));
  {
    const cuuint64_t dims[4] = {64, (cuuint64_t)g.Q, (cuuint64_t)g.P, (cuuint64_t)g.N};
    const cuuint64_t strides[3] = {128, (cuuint64_t)g.Q * 128, (cuuint64_t)g.P * g.Q * 128};
    const cuuint32_t box[4] = {64, TW, 4, 1};
    OC_TRY(encode_tiled(&P.ty, y, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B));
  }
  P.tq = g.Q / TW;
  P.tpq = (g.P / TH) * P.tq;
  P.units = g.N * P.tpq;
  P.pad = g.pad;
  P.stat_part = stat_part;
  if (P.units == 0) return Status::ok();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(stem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    attr = true;
  }
  const int ctas = grid_cap(std::min(P.units, sm_count()));
  if (stat_part && stat_slots) *stat_slots = ctas * 4;
  if (a.ktimer) {
    P.probe = a.ktimer->probe_slot(a.stream);
    a.ktimer->begin(a.stream);
  }
  stem_kernel<<<ctas, NTHREADS, SMEM, a.stream>>>(P);
  if (a.ktimer) a.ktimer->end(a.stream);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

// stat_part (optional): fused BN statistics of y (TMA-store epilogue only); on
// return *stat_slots = the slots written (0: not fused, the caller reduces y)
Status conv_fprop_tma(OpArgs& a, const ConvGeom& g, const __nv_bfloat16* x, const __nv_bfloat16* wb, int kpad,
                      __nv_bfloat16* y, bool accumulate, int nst, float* stat_part, int* stat_slots, int cmem) {
  if (stat_slots) *stat_slots = 0;
  if (g.C == 16 && g.R == 4 && g.S == 4 && g.st == 1 && !g.nopadh && g.K == 64 && kpad == 256 && g.P % 16 == 0 &&
      g.Q % 8 == 0 && !accumulate && !nst && stem_enabled() && dil_of(g) == 1)
    return conv_stem_tma(a, g, x, wb, kpad, y, stat_part, stat_slots);
  const int nch = g.C % 64 == 0 ? 0 : g.C;     // 8 or 16: narrow pixels, one tap per box
  Params P{};
  const int padh = g.nopadh ? 0 : g.pad;
  Status st = make_im2col(&P.ta, x, g.N, g.H, g.W, cmem > 0 ? cmem : g.C, nch ? nch : 64, BM, g.P, g.Q, g.st, padh, g.pad,
                          nch == 8 ? CU_TENSOR_MAP_SWIZZLE_NONE
                                   : (nch == 16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_128B));
  if (!st.good()) return st;
  const Tile tile = nch ? Tile{g.K % 128 == 0 ? 128 : 64, conv_mt(), 1} : choose_tile(g.N * g.P * g.Q, g.K, kpad / BK);
  const int BN = tile.bn;
  st = make_tiled(&P.tb, wb, (uint64_t)kpad, (uint64_t)g.K, (uint32_t)(BN / tile.cg));
  if (!st.good()) return st;
  P.out = y;
  P.nst = nst;
  P.accumulate = accumulate ? 1 : 0;
  // (the accumulating TMA epilogue is instantiated for 64-channel pixels only)
  st = set_tstore(P, y, g.N * g.P * g.Q, nst ? nst : g.K, !(accumulate && nch));
  if (!st.good()) return st;
  P.M = g.N * g.P * g.Q;
  P.N = g.K;
  P.num_m = (P.M + BM - 1) / BM;
  P.num_n = g.K / BN;
  P.splits = 1;
  P.nkb = kpad / BK;
  P.Pd = g.P;
  P.Qd = g.Q;
  P.st = g.st;
  P.padh = padh;
  P.padw = g.pad;
  P.R = g.R;
  P.S = g.S;
  P.Cr = g.C;
  P.dil = dil_of(g);
  fill(P);
  int* ss = nullptr;
  if (stat_part && P.tstore && !nst && !accumulate) {
    P.stat_part = stat_part;
    ss = stat_slots;
  }
  if (nch == 8) return BN == 128 ? launch<FPROP, 128, 8>(a, P, ss) : launch<FPROP, 64, 8>(a, P, ss);
  if (nch == 16) return BN == 128 ? launch<FPROP, 128, 16>(a, P, ss) : launch<FPROP, 64, 16>(a, P, ss);
  return launch_tile<FPROP>(a, P, tile, ss);
}

// dgrad, one launch per output phase (h mod st, w mod st) over that phase's
// valid taps: dx[(n,h',w')][C] = im2col_{pad''}(dy) · Wt_bf16[C][(r,s,K)]ᵀ at the
// phase's filter taps; a phase no tap reaches gets zeros (or keeps dx when accumulating)
Status conv_dgrad_tma(OpArgs& a, const ConvGeom& g, const __nv_bfloat16* dy, const __nv_bfloat16* wt,
                      __nv_bfloat16* dx, bool accumulate, int nst, int cmem) {
  // phases no filter tap reaches (e.g. 3 of the 4 phases of a 1×1 stride-2 conv):
  // without accumulation their dx is zero — cleared once for the whole tensor
  bool tapless = false;
  for (int ph = 0; ph < g.st; ++ph)
    for (int pw = 0; pw < g.st; ++pw)
      tapless |= ((ph + g.pad) % g.st >= g.R) || ((pw + g.pad) % g.st >= g.S);
  if (tapless && !accumulate) {
    cudaError_t e = cudaMemsetAsync(dx, 0, (size_t)g.N * g.H * g.W * (nst ? nst : g.C) * 2, a.stream);
    if (e != cudaSuccess) return cuda_status(e, "dgrad zero fill");
  }
  for (int ph = 0; ph < g.st; ++ph)
    for (int pw = 0; pw < g.st; ++pw) {
      Params P{};
      const int Hp = (g.H - ph + g.st - 1) / g.st, Wp = (g.W - pw + g.st - 1) / g.st;
      const int r0 = (ph + g.pad) % g.st, s0 = (pw + g.pad) % g.st;
      const int nr = r0 < g.R ? (g.R - r0 + g.st - 1) / g.st : 0;
      const int ns = s0 < g.S ? (g.S - s0 + g.st - 1) / g.st : 0;
      if (Hp <= 0 || Wp <= 0) continue;
      if (nr == 0 || ns == 0) continue;   // zero (cleared above) or unchanged (accumulating)
      // dy row of (h', tap i') is h' − pad'' + i' with pad'' = nr − 1 − (ph + pad − r0)/st
      // (dilation d, stride 1 only: tap i' reads dy row h' − (d·(nr − 1) − pad) + d·i')
      const int dl = dil_of(g);
      const int dh = (ph + g.pad - r0) / g.st, dw = (pw + g.pad - s0) / g.st;
      const int padh = nr > 0 ? dl * (nr - 1) - dh : 0, padw = ns > 0 ? dl * (ns - 1) - dw : 0;
      Status st = make_im2col(&P.ta, dy, g.N, g.P, g.Q, cmem > 0 ? cmem : g.K, 64, BM, Hp, Wp, 1, padh, padw);
      if (!st.good()) return st;
      const Tile tile = choose_tile(g.N * Hp * Wp, g.C, std::max(1, nr * ns * g.K / BK));
      const int BN = tile.bn;
      st = make_tiled(&P.tb, wt, (uint64_t)g.R * g.S * g.K, (uint64_t)g.C, (uint32_t)(BN / tile.cg));
      if (!st.good()) return st;
      P.out = dx;
      P.nst = nst;
      P.accumulate = accumulate ? 1 : 0;
      st = set_tstore(P, dx, g.N * Hp * Wp, nst ? nst : g.C, g.st == 1);
      if (!st.good()) return st;
      P.M = g.N * Hp * Wp;
      P.N = g.C;
      P.num_m = (P.M + BM - 1) / BM;
      P.num_n = g.C / BN;
      P.splits = 1;
      P.nkb = nr * ns * g.K / BK;
      P.Pd = Hp;
      P.Qd = Wp;
      P.st = 1;
      P.padh = padh;
      P.padw = padw;
      P.R = nr > 0 ? nr : 1;
      P.S = ns > 0 ? ns : 1;
      P.Cr = g.K;
      P.Sw = g.S;
      P.r0 = r0;
      P.s0 = s0;
      P.dst = g.st;
      P.ph = ph;
      P.pw = pw;
      P.Ho = g.H;
      P.Wo = g.W;
      P.dil = dl;
      fill(P);
      st = launch_tile<DGRAD>(a, P, tile);
      if (!st.good()) return st;
    }
  return Status::ok();
}

// the halo-tile stem weight gradient (namespace stem): one split partial per CTA
Status conv_stem_wgrad_tma(OpArgs& a, const ConvGeom& g, const __nv_bfloat16* x, const __nv_bfloat16* dy,
                           float* part, int splits, bool accumulate) {
  using namespace stem;
  WParams P{};
  {
    const cuuint64_t dims[4] = {16, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.N};
    const cuuint64_t strides[3] = {32, (cuuint64_t)g.W * 32, (cuuint64_t)g.H * g.W * 32};
    const cuuint32_t box[4] = {16, TW, WHR, 1};
    OC_TRY(encode_tiled(&P.tx, x, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_32B));
  }
  {
    const cuuint64_t dims[4] = {64, (cuuint64_t)g.Q, (cuuint64_t)g.P, (cuuint64_t)g.N};
    const cuuint64_t strides[3] = {128, (cuuint64_t)g.Q * 128, (cuuint64_t)g.P * g.Q * 128};
    const cuuint32_t box[4] = {64, TW, TH, 1};
    OC_TRY(encode_tiled(&P.tdy, dy, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B));
  }
  P.tq = g.Q / TW;
  P.tpq = (g.P / TH) * P.tq;
  P.units = g.N * P.tpq;
  P.pad = g.pad;
  P.accumulate = accumulate ? 1 : 0;
  P.part = part;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(stem_wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, WSMEM);
    attr = true;
  }
  if (a.ktimer) {
    P.probe = a.ktimer->probe_slot(a.stream);
    a.ktimer->begin(a.stream);
  }
  stem_wgrad_kernel<<<splits, NTHREADS, WSMEM, a.stream>>>(P);   // every CTA writes its partial (zeros if idle)
  if (a.ktimer) a.ktimer->end(a.stream);
  OC_LAUNCH_CHECK(a);
  return Status::ok();
}

// wgrad partials part[z][R·S·C][K] over pixel blocks [z·kbps, (z+1)·kbps)
Status conv_wgrad_tma(OpArgs& a, const ConvGeom& g, const __nv_bfloat16* x, const __nv_bfloat16* dy, float* part,
                      int splits, int kb_per_split, bool accumulate, int cmem, int kmem) {
  if (g.C == 16 && g.R == 4 && g.S == 4 && g.st == 1 && !g.nopadh && g.K == 64 && g.P % 16 == 0 && g.Q % 8 == 0 &&
      splits >= 1 && splits <= 1024 && stem_enabled() && dil_of(g) == 1)
    return conv_stem_wgrad_tma(a, g, x, dy, part, splits, accumulate);
  Params P{};
  const int nch = g.C == 16 ? 16 : 0;
  const int padh = g.nopadh ? 0 : g.pad;
  Status st = make_im2col(&P.ta, x, g.N, g.H, g.W, cmem > 0 ? cmem : g.C, nch ? 16 : 64, WKB, g.P, g.Q, g.st, padh, g.pad,
                          nch ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_128B);
  if (!st.good()) return st;
  const int BN = g.K % 128 == 0 ? 128 : 64;
  // CTA pairs over 256 (r,s,c) rows × 256 columns (half of B per CTA) when K
  // allows: measured at ResNet-18 b=256 l3/l4 797 -> 937 / 732 -> 839 TF/s;
  // 128-column pairs were slower than single CTAs (l2: 781 -> 644), so they
  // are only forced (OC_WGRAD_CG=2, tests).  OC_WGRAD_CG=1 keeps single CTAs.
  const char* ecg = std::getenv("OC_WGRAD_CG");
  const bool force = ecg && ecg[0] == '2', off = ecg && ecg[0] == '1';
  const int pbn = (nch || off) ? 0 : (g.K % 256 == 0 ? 256 : ((force && g.K % 128 == 0) ? 128 : 0));
  st = make_tiled(&P.tb, dy, (uint64_t)(kmem > 0 ? kmem : g.K), (uint64_t)g.N * g.P * g.Q, WKB);
  if (!st.good()) return st;
  P.out = part;
  P.accumulate = accumulate ? 1 : 0;
  P.M = g.R * g.S * g.C;
  P.N = g.K;
  P.num_m = (P.M + BM - 1) / BM;
  P.num_n = g.K / BN;
  P.splits = splits;
  P.nkb = (g.N * g.P * g.Q + WKB - 1) / WKB;
  P.kb_per_split = (P.nkb + splits - 1) / splits;
  (void)kb_per_split;
  P.Pd = g.P;
  P.Qd = g.Q;
  P.st = g.st;
  P.padh = padh;
  P.padw = g.pad;
  P.R = g.R;
  P.S = g.S;
  P.Cr = g.C;
  P.dil = dil_of(g);
  fill(P);
  if (nch) return BN == 128 ? launch<WGRAD, 128, 16>(a, P) : launch<WGRAD, 64, 16>(a, P);
  if (pbn == 256) {
    P.num_n = g.K / 256;
    return launch_mt<WGRAD, 256, 0, 1, 2>(a, P);
  }
  if (pbn == 128) return launch_mt<WGRAD, 128, 0, 1, 2>(a, P);
  return BN == 128 ? launch<WGRAD, 128, 0>(a, P) : launch<WGRAD, 64, 0>(a, P);
}

}  // namespace oc
