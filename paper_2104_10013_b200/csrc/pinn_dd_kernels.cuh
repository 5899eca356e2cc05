// pinn_dd_kernels.cuh -- the fused kernels (templated on the network shape).
//
// K1  k_fused<MODE=0>: one persistent CTA per SM; for every tile of P points of
//     one subdomain: layer-by-layer forward Taylor jets (weights in SMEM,
//     pre-activation jets stashed in TMEM), pointwise operator + loss terms +
//     adjoint seeds (epilogue), reverse sweep through the jets, dW/db/da
//     partials accumulated per chunk.  Algorithm 1 red stage + J + gradient.
// K2  k_fused<MODE=1>: forward + payload epilogue at interface points
//     (Algorithm 1).
// K5  k_reduce_adam: fixed-order reduction of the chunk partials, J_q assembly
//     (Eq. 5/6) and the per-subdomain Adam step.
// K6  k_predict: value-only forward + Eq. (4) stitching.
#pragma once

#include <type_traits>

#include "pinn_dd_device.cuh"

namespace pinn {

// unroll factors of the GEMM loops (i-quads forward, 10-row blocks of the input
// adjoint, points of dW); overridable at build time for variant sweeps
#ifndef PINN_DWPRE_MAX
#define PINN_DWPRE_MAX 32
#endif
#ifndef PINN_UF_FWD
#define PINN_UF_FWD 0   // 0 = fully unrolled (gemm_fwd)
#endif
#ifndef PINN_UF_BWD
#define PINN_UF_BWD 1
#endif
#ifndef PINN_UF_DW
#define PINN_UF_DW 8
#endif
constexpr int kUfFwd = PINN_UF_FWD, kUfDw = PINN_UF_DW;

// Development build only (-DPINN_PHASE_PROF): thread 0 of every CTA charges
// the clock cycles between phase marks to the phase that just ended; CTAs
// 0..3 print their totals at exit (tools/phase_prof.sh).  Phases are CTA-
// barrier delimited, so thread 0's split is the CTA's.
#ifdef PINN_PHASE_PROF
#define PROF_MARK(k)                                  \
  do {                                                \
    if (threadIdx.x == 0) {                           \
      const long long t_ = clock64();                 \
      prof_acc[prof_cur] += t_ - prof_t0;             \
      prof_t0 = t_;                                   \
      prof_cur = (k);                                 \
    }                                                 \
  } while (0)
#else
#define PROF_MARK(k) \
  do {               \
  } while (0)
#endif
constexpr int kUfBwd = PINN_UF_BWD;
// the input-adjoint GEMM's block loop fully unrolled (0) for the uniform-
// activation width-80 instances only: C4 K1 15.06 -> 14.82 ms, while C5's
// per-region-activation instance (+4 %) and width 40 (+3.8 %) lose with it
template <int N, int ACT>
constexpr int kUfBwdOf = (N == 80 && ACT != kActMixed && kUfBwd == 1) ? 0 : kUfBwd;

// CTA barrier preceded by an explicit warp reconvergence.
__device__ __forceinline__ void cta_sync() {
  __syncwarp();
  __syncthreads();
}

__device__ __forceinline__ void rmw_store(float* p, float v, bool first) {
  *p = first ? v : (*p + v);
}

// block-wide sum of R values per thread, fixed order (shuffle tree, then warps 0..3)
template <int R, int NT, class T>
__device__ __forceinline__ void block_sum(T* v, T* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    T x = v[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    v[r] = x;
  }
  cta_sync();
  if (lane == 0) {
#pragma unroll
    for (int r = 0; r < R; ++r) red[w * R + r] = v[r];
  }
  cta_sync();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      T s = T(0);
#pragma unroll
      for (int ww = 0; ww < NT / 32; ++ww) s += red[ww * R + r];
      v[r] = s;
    }
  }
}

template <int N, int NH, int DO, int T>
__device__ __forceinline__ void load_weights(const float* __restrict__ G, float slope_n, float* sm) {
  using C = KCfg<N, NH, DO, T>;
  using LY = Lay<N, NH, DO>;
  const int tid = threadIdx.x;
  for (int e = tid; e < 3 * N; e += T) sm[C::oW1 + e] = G[LY::offW(1) + e];   // W^1 [N][2], b^1 (offB(1) = 2N)
  static_assert(LY::offB(1) == 2 * N && C::oB1 == 2 * N, "W^1/b^1 contiguous");
  // hidden W^k rows: float4 copies; row j of layer k lands at j*WS + (j/kJT)*4.
  // Every load of a layer is issued before its stores (one L2 round trip per
  // layer, not one per float4: with C5's one-tile chunks of ten regions the
  // weights are reloaded for most tiles, and the serial copy loop was 5 % of K1)
  constexpr int Q = N / 4;   // float4 per row
  constexpr int IT = (N * Q + T - 1) / T;
#pragma unroll 1
  for (int k = 2; k <= NH; ++k) {
    const float4* W = reinterpret_cast<const float4*>(G + LY::offW(k));
    float* dst = sm + C::oWh + (k - 2) * C::WROWS;
    float4 v[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int e = tid + it * T;
      if (e < N * Q) v[it] = __ldcg(W + e);
    }
    const float bk = tid < N ? G[LY::offB(k) + tid] : 0.0f;
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int e = tid + it * T;
      if (e < N * Q) {
        const int j = e / Q, q = e - (e / Q) * Q;
        *reinterpret_cast<float4*>(dst + j * C::WS + (j / kJT) * 4 + 4 * q) = v[it];
      }
    }
    static_assert(N <= T, "one bias per thread");
    if (tid < N) sm[C::oBh + (k - 2) * N + tid] = bk;
  }
  for (int e = tid; e < DO * N; e += T) {
    const int o = e / N, i = e - (e / N) * N;
    sm[C::oWo + o * C::WS + i] = G[LY::offW(NH + 1) + e];
  }
  for (int e = tid; e < DO; e += T) sm[C::oBo + e] = G[LY::offB(NH + 1) + e];
  for (int e = tid; e < NH; e += T) sm[C::oSl + e] = slope_n * G[LY::offA(e + 1)];
}

// gradient accumulator: shared memory for the whole chunk (DWS), else the
// chunk's global partial (read-modify-write per tile, `first` = first tile)
template <bool DWS>
__device__ __forceinline__ void acc_add(float* base, int off, float v, bool first) {
  if constexpr (DWS) {
    base[off] += v;
  } else {
    base[off] = first ? v : base[off] + v;
  }
}

__device__ __forceinline__ float comp(const float4& v, int m) {
  return m == 0 ? v.x : (m == 1 ? v.y : (m == 2 ? v.z : v.w));
}

// packed FP32 FMA (FFMA2, sm_100): acc.{xy,zw} += w * h.{xy,zw}.  Same
// rounding as four fmaf calls; one issue slot per two FMAs.
__device__ __forceinline__ void fma4(float4& acc, float w, const float4& h) {
  const float2 ww = make_float2(w, w);
  const float2 lo = __ffma2_rn(ww, make_float2(h.x, h.y), make_float2(acc.x, acc.y));
  const float2 hi = __ffma2_rn(ww, make_float2(h.z, h.w), make_float2(acc.z, acc.w));
  acc = make_float4(lo.x, lo.y, hi.x, hi.y);
}

// compile-time loop: f(I) for I = B, B + S, ... < E, expanded in place
template <int B, int E, int S, class F>
__device__ __forceinline__ void static_for(F& f) {
  if constexpr (B < E) {
    f(B);
    static_for<B + S, E, S>(f);
  }
}

// forward GEMM of one hidden layer for this thread's (point, neuron block):
// z[jj].c = sum_i W[j][i] Hin[i][p].c  (+ b on the value channel).
// Per i-quad all kJT jet accumulators are updated once per input component, so
// consecutive FMAs are independent.
template <int N, int NH, int DO, int T, int UF>
__device__ __forceinline__ void gemm_fwd(const float4* __restrict__ Hin, const float* __restrict__ W,
                                         const float* __restrict__ b, float4* z, int pg, int nb) {
  using C = KCfg<N, NH, DO, T>;
  const int j0 = nb * kJT;
#pragma unroll
  for (int jj = 0; jj < kJT; ++jj) z[jj] = make_float4(b[j0 + jj], 0.0f, 0.0f, 0.0f);
  const float* Wb = W + j0 * C::WS + nb * 4;
  auto quad = [&](int i) {
    float4 h[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) h[m] = Hin[C::row(i + m) + pg];
    float4 w[kJT];
#pragma unroll
    for (int jj = 0; jj < kJT; ++jj) w[jj] = *reinterpret_cast<const float4*>(Wb + jj * C::WS + i);
#pragma unroll
    for (int m = 0; m < 4; ++m) {
#pragma unroll
      for (int jj = 0; jj < kJT; ++jj) fma4(z[jj], comp(w[jj], m), h[m]);
    }
  };
  if constexpr (UF == 0) {
    // fully unrolled: the compiler unrolls width 80's 20 i-quads only 4-fold
    // whatever the pragma says, and that loop rotates the accumulator
    // registers across its back edge (46 MOVs per 320 FFMA2): C4 K1 15.44 ->
    // 15.05 ms.  The per-region-activation instance (C5) keeps the loop (the
    // larger body measured 0.3 % slower there).
    if constexpr (N == 80) {
      // software-pipelined: the operands of i-quad q + 1 are loaded before the
      // FMAs of quad q (two register sets; the fully unrolled loop's top stall
      // was the shared-load scoreboard): C4 K1 14.90 -> 14.80 ms
      float4 hA[4], wA[kJT], hB[4], wB[kJT];
      auto ld = [&](int i, float4* h, float4* w) {
#pragma unroll
        for (int m = 0; m < 4; ++m) h[m] = Hin[C::row(i + m) + pg];
#pragma unroll
        for (int jj = 0; jj < kJT; ++jj) w[jj] = *reinterpret_cast<const float4*>(Wb + jj * C::WS + i);
      };
      auto mm = [&](const float4* h, const float4* w) {
#pragma unroll
        for (int m = 0; m < 4; ++m) {
#pragma unroll
          for (int jj = 0; jj < kJT; ++jj) fma4(z[jj], comp(w[jj], m), h[m]);
        }
      };
      ld(0, hA, wA);
      auto step = [&](int i) {
        if (((i / 4) & 1) == 0) {
          if (i + 4 < N) ld(i + 4, hB, wB);
          mm(hA, wA);
        } else {
          if (i + 4 < N) ld(i + 4, hA, wA);
          mm(hB, wB);
        }
      };
      static_for<0, N, 4>(step);
    } else {
      static_for<0, N, 4>(quad);
    }
  } else {
#pragma unroll UF
    for (int i = 0; i < N; i += 4) quad(i);
  }
}

// reverse GEMM (input adjoint): hb[ii].c = sum_j Zb[j][p].c W[j][j0 + ii]
template <int N, int NH, int DO, int T, int UF>
__device__ __forceinline__ void gemm_bwd(const float4* __restrict__ Zb, const float* __restrict__ W, float4* hb,
                                         int pg, int nb) {
  using C = KCfg<N, NH, DO, T>;
  const int j0 = nb * kJT;
#pragma unroll
  for (int e = 0; e < kJT; ++e) hb[e] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  auto blk = [&](int jb) {
    // rows jb*kJT .. +kJT-1 share the block skew jb*4
    const float* Wrow = W + jb * (kJT * C::WS + 4) + j0;
    const float4* Zrow = Zb + C::row(jb * kJT) + pg;   // rows of one block share its skew
#pragma unroll
    for (int jj = 0; jj < kJT; ++jj) {
      const float4 zb = Zrow[jj * C::PSTR];
      const float* wr = Wrow + jj * C::WS;
#pragma unroll
      for (int q = 0; q < kJT / 2; ++q) {
        const float2 w = *reinterpret_cast<const float2*>(wr + 2 * q);
        fma4(hb[2 * q], w.x, zb);
        fma4(hb[2 * q + 1], w.y, zb);
      }
    }
  };
  if constexpr (UF == 0) {
    static_for<0, C::NB, 1>(blk);
  } else {
#pragma unroll UF
    for (int jb = 0; jb < C::NB; ++jb) blk(jb);
  }
}

// weight and bias gradient of one hidden layer (mapping B):
// dW[j][i] += sum_p sum_c Zb[j][p].c H[i][p].c ;  db[j] += sum_p Zb[j][p].x
// thread = (row block jb, column block ib, point split s); rows/cols interleaved.
template <int N, int NH, int DO, int T, bool DWS, int UF>
__device__ __forceinline__ void gemm_dw(const float4* __restrict__ Zb, const float4* __restrict__ H, float* accW,
                                        float* accB, bool first, float* sDw) {
  using C = KCfg<N, NH, DO, T>;
  constexpr int JB = C::JB, IB = C::IB, NJ = C::NJ, NI = C::NI, NBLK = C::NBLK, S = C::S;
  constexpr int PS = C::P / S;
  const int tid = threadIdx.x;
  if (tid < NBLK * S) {
    const int r = tid % NBLK, s = tid / NBLK;
    // a warp covers 8 row blocks x 4 column blocks: its Zb row loads are 8
    // distinct float4 (one wavefront) and its H loads 4 (broadcast).  For
    // NJ = 16 (width 80) the plain r % NJ split gave 16 x 2 per warp (two
    // wavefronts per Zb load: 15 instead of 10 per point and warp)
    const int jb = NJ == 16 ? ((r & 7) | (((r >> 5) & 1) << 3)) : r % NJ;
    const int ib = NJ == 16 ? (((r >> 3) & 3) | ((r >> 6) << 2)) : r / NJ;
    float2 acc2[JB][IB];   // (x.x + z.z, y.y + w.w) channel pairs, one FFMA2 each
#pragma unroll
    for (int jj = 0; jj < JB; ++jj) {
#pragma unroll
      for (int ii = 0; ii < IB; ++ii) acc2[jj][ii] = make_float2(0.0f, 0.0f);
    }
    auto pt = [&](int p) {
      float4 zr[JB], hr[IB];
#pragma unroll
      for (int jj = 0; jj < JB; ++jj) zr[jj] = Zb[C::row(jb + NJ * jj) + p];
#pragma unroll
      for (int ii = 0; ii < IB; ++ii) hr[ii] = H[C::row(ib + NI * ii) + p];
#pragma unroll
      for (int jj = 0; jj < JB; ++jj)
#pragma unroll
        for (int ii = 0; ii < IB; ++ii) {
          acc2[jj][ii] = __ffma2_rn(make_float2(zr[jj].x, zr[jj].y), make_float2(hr[ii].x, hr[ii].y), acc2[jj][ii]);
          acc2[jj][ii] = __ffma2_rn(make_float2(zr[jj].z, zr[jj].w), make_float2(hr[ii].z, hr[ii].w), acc2[jj][ii]);
        }
    };
    if constexpr (UF == 0) {
      auto ptS = [&](int p) { pt(s * PS + p); };
      static_for<0, PS, 1>(ptS);
    } else {
#pragma unroll UF
      for (int p = s * PS; p < (s + 1) * PS; ++p) pt(p);
    }
    float acc[JB][IB];
#pragma unroll
    for (int jj = 0; jj < JB; ++jj)
#pragma unroll
      for (int ii = 0; ii < IB; ++ii) acc[jj][ii] = acc2[jj][ii].x + acc2[jj][ii].y;
    if constexpr (S == 1 && DWS) {
      // shared chunk accumulator, entries private to this thread: loads first
      float cur[JB][IB];
#pragma unroll
      for (int jj = 0; jj < JB; ++jj) {
#pragma unroll
        for (int ii = 0; ii < IB; ++ii) cur[jj][ii] = accW[(jb + NJ * jj) * N + ib + NI * ii];
      }
#pragma unroll
      for (int jj = 0; jj < JB; ++jj) {
#pragma unroll
        for (int ii = 0; ii < IB; ++ii) accW[(jb + NJ * jj) * N + ib + NI * ii] = cur[jj][ii] + acc[jj][ii];
      }
    } else {
      // db^k is summed once per row by db_sum (the NI threads of a row block
      // used to repeat it: 5 FADDs per point, 10 % of the FMA-pipe cycles of dW)
#pragma unroll
      for (int jj = 0; jj < JB; ++jj)
#pragma unroll
        for (int ii = 0; ii < IB; ++ii) sDw[s * C::SSPL + (jb + NJ * jj) * C::SROW + ib + NI * ii] = acc[jj][ii];
    }
  }
}

// second half of gemm_dw for S > 1: sum the S point-split partials in fixed
// order into the accumulator.  Called after the CTA barrier that follows
// gemm_bwd, so it needs no barrier of its own and its shared-memory latency
// overlaps the activation-buffer stores that follow.
// Global chunk partial (!DWS) with few entries per thread: its current values
// are loaded right after gemm_dw (before gemm_bwd and the barrier), so the L2
// round trip overlaps the input-adjoint GEMM instead of following the barrier.
// db^k[j] = sum_p Zb^k[j][p].value, written to the scratch's db slot
// sDw[DBOFF + j] for gemm_dw_reduce (after the next barrier).  TPR threads per
// row (consecutive lanes), each 4 interleaved chains over every TPR-th point,
// combined in a fixed order (chains, then an xor-shuffle tree): width 20 puts
// 80 threads on 20 rows of 64 points instead of 20 threads on 64 each.
// Called after the input-adjoint GEMM and before the barrier that precedes
// the next writes of the Zb buffer.
template <int N, int NH, int DO, int T, bool DWS>
__device__ __forceinline__ void db_sum(const float4* __restrict__ Zb, float* sDw, float* accB) {
  using C = KCfg<N, NH, DO, T>;
  {
    constexpr int TPR = (N * 4 <= T && C::P % 16 == 0) ? 4 : ((N * 2 <= T && C::P % 8 == 0) ? 2 : 1);
    static_assert(C::P % (4 * TPR) == 0, "four chains per thread");
    constexpr int DBOFF = C::S * C::SSPL;
    const int tid = threadIdx.x;
    const int j = tid / TPR, sub = tid % TPR;
    float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
    if (j < N) {
      const float4* z = Zb + C::row(j);
#pragma unroll
      for (int p = sub; p < C::P; p += 4 * TPR) {
        a0 += z[p].x;
        a1 += z[p + TPR].x;
        a2 += z[p + 2 * TPR].x;
        a3 += z[p + 3 * TPR].x;
      }
    }
    float v = (a0 + a1) + (a2 + a3);
#pragma unroll
    for (int o = 1; o < TPR; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (j < N && sub == 0) {
      if constexpr (C::S == 1 && DWS)
        accB[j] += v;   // the chunk's shared accumulator (gemm_dw_reduce is empty on this path)
      else
        sDw[DBOFF + j] = v;
    }
  }
}

template <int N, int NH, int DO, int T, bool DWS>
struct DwPre {
  static constexpr int IT = (N * N + T - 1) / T;
  static constexpr bool ON = !DWS && IT <= PINN_DWPRE_MAX;
};

template <int N, int NH, int DO, int T, bool DWS>
__device__ __forceinline__ void gemm_dw_prefetch(const float* accW, const float* accB, bool first, float* pre,
                                                 float& preb) {
  if constexpr (DwPre<N, NH, DO, T, DWS>::ON) {
    constexpr int NE = N * N, IT = DwPre<N, NH, DO, T, DWS>::IT;
    const int tid = threadIdx.x;
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int e = tid + it * T;
      pre[it] = (!first && e < NE) ? __ldcg(accW + e) : 0.0f;
    }
    preb = (!first && tid < N) ? __ldcg(accB + tid) : 0.0f;
  }
}

template <int N, int NH, int DO, int T, bool DWS>
__device__ __forceinline__ void gemm_dw_reduce(float* accW, float* accB, bool first, const float* sDw,
                                               const float* pre, float preb) {
  using C = KCfg<N, NH, DO, T>;
  constexpr int S = C::S;
  constexpr bool PRE = DwPre<N, NH, DO, T, DWS>::ON;
  if constexpr (!DWS || S > 1) {
    // thread e owns dW entries e, e + T, ... in natural [j][i] order: the
    // scratch rows, the shared accumulator and the global partial are all read
    // contiguously (no bank conflicts, coalesced); every load is issued before
    // any store (the entries are distinct).  Split order s = 0 .. S-1.
    const int tid = threadIdx.x;
    constexpr int NE = N * N, IT = (NE + T - 1) / T;
    float v[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int e = tid + it * T;
      if (e < NE) {
        const int j = e / N, i = e - (e / N) * N;
        const float* src = sDw + j * C::SROW + i;
        float x = src[0];
#pragma unroll
        for (int s = 1; s < S; ++s) x += src[s * C::SSPL];
        v[it] = x;
      }
    }
    float cur[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int e = tid + it * T;
      if constexpr (PRE)
        cur[it] = pre[it];
      else if (e < NE)
        cur[it] = (DWS || !first) ? accW[e] : 0.0f;
    }
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int e = tid + it * T;
      if (e < NE) accW[e] = (DWS || !first) ? cur[it] + v[it] : v[it];
    }
    if (tid < N) {
      const float x = sDw[S * C::SSPL + tid];   // db_sum
      if constexpr (PRE)
        accB[tid] = first ? x : preb + x;
      else
        accB[tid] = (DWS || !first) ? accB[tid] + x : x;
    }
  }
}

// epilogue of one point (K2): u(x_I) and f.n (cPINN) or F (XPINN) into its
// payload row (Algorithm 1)
template <int DO>
__device__ __forceinline__ void point_payload(const KArgs& a, int64_t gp, float x, float y, const float4* U,
                                              int step = 0, int* xcount = nullptr) {
  constexpr int NF = DO + (DO == 3 ? 3 : 1);
  float r[3];
  float dr[3][DO][4];
  int ne;
  const int info = a.pinfo[gp];
  if (info & 4) {
    const float2 n = a.seg_normal[info >> 3];
    ne = pde_flux<DO>(a.pc, U, x, y, n.x, n.y, r, dr);
  } else {
    ne = pde_residual<DO>(a.pc, U, x, y, r, dr);
  }
  float* q = a.payload + size_t(gp) * NF;
#pragma unroll
  for (int o = 0; o < DO; ++o) q[o] = U[o].x;
  for (int e = 0; e < ne; ++e) q[DO + e] = r[e];
  // a point of a cut edge also goes to its neighbour's rank (Algorithm 1 lines
  // 244-252): into the send buffer (the NCCL exchange reads it after this
  // kernel), or -- peer stores, fused step -- straight into the neighbour's
  // receive slot of this step's parity, counted per peer in xcount
  const int ss = a.psend ? a.psend[gp] : -1;
  if (ss >= 0) {
    float* w;
    if (xcount) {
      int i = 0;
      while (i + 1 < a.px.n && ss >= a.px.send_off[i + 1]) ++i;
      w = a.px.dst[i] + (step & 1) * a.px.slot_stride[i] + (ss - a.px.send_off[i]) * NF;
      atomicAdd(xcount + i, 1);
    } else {
      w = a.sendbuf + size_t(ss) * NF;
    }
#pragma unroll
    for (int o = 0; o < DO; ++o) w[o] = U[o].x;
    for (int e = 0; e < ne; ++e) w[DO + e] = r[e];
  }
}

// the peer-store protocol of the fused step (PeerX): after a payload chunk,
// release this chunk's row counts to the peers' arrival counters (the CTA
// barrier orders every thread's row stores before thread 0's release)
__device__ __forceinline__ void publish_peer_rows(const KArgs& a, int* xcount) {
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int i = 0; i < a.px.n; ++i)
      if (xcount[i]) {
        red_release_sys_add(a.px.peer_flag[i], (unsigned long long)xcount[i]);
        xcount[i] = 0;
      }
  }
}
// before an interface loss chunk: every local payload chunk and every peer's
// rows of this step have arrived
// A wait that has not ended after ~20 s (a peer that never runs its step)
// traps: the launch fails with an error instead of hanging the device.
__device__ __forceinline__ void spin_guard(long long t0) {
  if (clock64() - t0 > 40000000000LL) __trap();
}
__device__ __forceinline__ void wait_payload(const KArgs& a, int n_pay, int step) {
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    while (ld_acquire_gpu(a.sched + 4) < n_pay) {
      __nanosleep(64);
      spin_guard(t0);
    }
    for (int i = 0; i < a.px.n; ++i) {
      const unsigned long long want = (unsigned long long)(step + 1) * (unsigned long long)a.px.expect[i];
      while (ld_acquire_sys_u64(a.px.my_flag + i) < want) {
        __nanosleep(64);
        spin_guard(t0);
      }
    }
  }
}

// Sticky schedule (MODE 2): thread 0 claims the next chunk of subdomain q,
// else of the next subdomains in turn (q + 1, q + 2, ...); returns the chunk
// index, or -1 when every queue is empty.  A CTA's first subdomain comes from
// its position in the cumulative tile count, so the CTAs start spread over the
// subdomains in proportion to their work.  Which CTA runs a chunk never
// changes its result (every chunk owns its partial slot).
__device__ __forceinline__ int sticky_first_sub(const KArgs& a) {
  const long long tot = a.sub_tiles[a.n_sub];
  const long long target = ((2LL * blockIdx.x + 1) * tot) / (2LL * gridDim.x);
  int q = 0;
  while (q + 1 < a.n_sub && a.sub_tiles[q + 1] <= target) ++q;
  return q;
}
// Claim from the current queue (one atomic; its chunk range is cached in
// st[4], st[5]), else scan the other queues in turn.  A queue's chunks are
// contiguous in chunk order (sub_chunk_off), already largest first with the
// interface chunks last, so the claimed place k IS chunk off + k.
__device__ __forceinline__ int sticky_claim(const KArgs& a, volatile int* st) {
  const int q = st[0];
  if (q >= 0) {
    const int k = atomicAdd(a.sub_ctr + q, 1);
    if (k < st[5]) {
      st[3] = k;
      return st[4] + k;
    }
  }
  const int q0 = q < 0 ? sticky_first_sub(a) : q + 1;
  for (int d = 0; d < a.n_sub; ++d) {
    int qq = q0 + d;
    if (qq >= a.n_sub) qq -= a.n_sub;
    if (qq == q) continue;   // just found empty
    const int off = a.sub_chunk_off[qq], n = a.sub_chunk_off[qq + 1] - off;
    if (*reinterpret_cast<volatile int*>(a.sub_ctr + qq) >= n) continue;
    const int k = atomicAdd(a.sub_ctr + qq, 1);
    if (k < n) {
      st[0] = qq;
      st[3] = k;
      st[4] = off;
      st[5] = n;
      return off + k;
    }
  }
  return -1;
}
// next work item of a persistent CTA (thread 0): payload chunks [0, n_pay)
// from the global counter first, then loss chunks n_pay + c -- chunk c
// directly when sticky, else the position in `order`
// (thread 0's state lives in shared memory: st[0] = current subdomain or -1
// before the first claim, st[1] = 1 once the global payload queue is empty,
// st[2] = a chunk claimed ahead (-1: none), st[3] = the current chunk's place
// in its queue, st[4], st[5] = the queue's first chunk and length)
__device__ __forceinline__ int next_item(const KArgs& a, int n_pay, volatile int* st) {
  if (st[2] >= 0) {
    const int c = st[2];
    st[2] = -1;
    return n_pay + c;
  }
  if (st[1] == 0) {
    const int idx = atomicAdd(a.sched, 1);
    if (a.sub_chunk_off == nullptr || idx < n_pay) return idx;
    st[1] = 1;
  }
  const int c = sticky_claim(a, st);
  return c < 0 ? a.n_chunks + n_pay : n_pay + c;
}
// Claim-ahead (thread 0, sticky phase; the TF32 kernel only -- the FP32 one
// measured 2 % slower with it): at the start of a chunk, claim the next chunk
// of the same queue so the atomic's round trip overlaps the tiles (C5 TF32 K1
// 0.265 -> 0.258 ms); only while >= kAheadMin chunks remain behind it, so the
// schedule's tail is claimed one at a time as before.
// Returns the claimed place in the queue (or -1); sticky_ahead_finish turns it
// into st[2] after the chunk.
constexpr int kAheadMin = 16;
__device__ __forceinline__ int sticky_ahead_issue(const KArgs& a, volatile int* st) {
  if (a.sub_chunk_off == nullptr || st[1] == 0 || st[0] < 0) return -1;
  if (st[3] + kAheadMin >= st[5]) return -1;
  return atomicAdd(a.sub_ctr + st[0], 1);
}
__device__ __forceinline__ void sticky_ahead_finish(const KArgs& a, volatile int* st, int k) {
  if (k < 0) return;
  if (k < st[5]) {
    st[2] = st[4] + k;
    st[3] = k;
  }
}
__device__ __forceinline__ void sticky_reset(const KArgs& a) {
  if (a.sub_chunk_off)
    for (int q = 0; q < a.n_sub; ++q) a.sub_ctr[q] = 0;
}

// epilogue of one point (K1): its loss terms (Eq. 3/5/6; lsum = MSE_u, MSE_F,
// MSE_uavg, MSE_if partials) and the adjoint seeds Ub = dJ/dU (a8)
template <int DO>
__device__ __forceinline__ void point_adjoint(const KArgs& a, int64_t gp, float x, float y, float4 lw,
                                              const float4* U, float4* Ub, float* lsum, int64_t roff = 0) {
  constexpr int NF = DO + (DO == 3 ? 3 : 1);
  const int info = a.pinfo[gp];
  const int kind = info & 3;
  const float inv = a.pinv[gp];
  float r[3];
  float dr[3][DO][4];
  if (kind == 0) {
    // residual point: W_F (1/N_F) sum_e F_e^2
    const int ne = pde_residual<DO>(a.pc, U, x, y, r, dr);
    for (int e = 0; e < ne; ++e) {
      lsum[1] += inv * r[e] * r[e];
      const float cf = 2.0f * lw.y * inv * r[e];
#pragma unroll
      for (int o = 0; o < DO; ++o) {
        Ub[o].x = fmaf(cf, dr[e][o][0], Ub[o].x);
        Ub[o].y = fmaf(cf, dr[e][o][1], Ub[o].y);
        Ub[o].z = fmaf(cf, dr[e][o][2], Ub[o].z);
        Ub[o].w = fmaf(cf, dr[e][o][3], Ub[o].w);
      }
    }
  } else if (kind == 1) {
    // training point: W_u (1/N_u) sum_o mask_o |u^(i)_o - u_o|^2
#pragma unroll
    for (int o = 0; o < DO; ++o) {
      const float m = a.mask[size_t(o) * a.n_points + gp];
      const float d = m * (U[o].x - a.target[size_t(o) * a.n_points + gp]);
      lsum[0] += inv * d * d;
      Ub[o].x += 2.0f * lw.x * inv * d;
    }
  } else {
    // interface point: neighbour payload is a constant
    int64_t tw = a.ptwin[gp];
    if (tw >= a.n_points) tw += roff;                          // received rows: this step's slot
    const float* q = a.payload + size_t(tw) * NF;   // read via L2 (__ldcg): rows written by other CTAs / GPUs
#pragma unroll
    for (int o = 0; o < DO; ++o) {
      const float d = U[o].x - __ldcg(q + o);   // u_q - {{u}} = d / 2  (Z1)
      lsum[2] += inv * 0.25f * d * d;
      Ub[o].x += 0.5f * lw.z * inv * d;
    }
    int ne;
    if (info & 4) {
      const float2 n = a.seg_normal[info >> 3];
      ne = pde_flux<DO>(a.pc, U, x, y, n.x, n.y, r, dr);
    } else {
      ne = pde_residual<DO>(a.pc, U, x, y, r, dr);
    }
    for (int e = 0; e < ne; ++e) {
      const float d = r[e] - __ldcg(q + DO + e);
      lsum[3] += inv * d * d;
      const float cf = 2.0f * lw.w * inv * d;
#pragma unroll
      for (int o = 0; o < DO; ++o) {
        Ub[o].x = fmaf(cf, dr[e][o][0], Ub[o].x);
        Ub[o].y = fmaf(cf, dr[e][o][1], Ub[o].y);
        Ub[o].z = fmaf(cf, dr[e][o][2], Ub[o].z);
        Ub[o].w = fmaf(cf, dr[e][o][3], Ub[o].w);
      }
    }
  }
}

// Runs f(integral_constant<AS>) with the chunk's activation: the compiled one,
// or -- per-subdomain (kActMixed) instances -- a branch on the runtime `act`
// (uniform per chunk) around the small activation loop only, so the GEMM code
// exists once per kernel instead of once per activation (C5's kernel was
// three copies of everything: 0.36 no-instruction stalls per issue).
template <int ACT, class F>
__device__ __forceinline__ void with_act(int act, F&& f) {
  if constexpr (ACT != kActMixed) {
    f(std::integral_constant<int, ACT>{});
  } else {
    if (act == 0)
      f(std::integral_constant<int, 0>{});
    else if (act == 1)
      f(std::integral_constant<int, 1>{});
    else
      f(std::integral_constant<int, 2>{});
  }
}

template <int N, int NH, int DO, int ACT, int MODE, int T>
__global__ void __launch_bounds__(T, 256 / T) k_fused(const KArgs a) {
  using C = KCfg<N, NH, DO, T>;
  using LY = Lay<N, NH, DO>;
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x;
  // thread -> (point group pg, neuron block nb).  With 8 neuron blocks the
  // 8-lane phases of a 128-bit shared store hold 4 blocks x 2 points (lane
  // bits 0,1,3 -> nb, bits 2,4 -> point), which makes the activation stores
  // conflict-free (8 blocks x 1 point hit 4 bank groups twice); the loads see
  // the same address sets per warp as before.
  const int lane = tid & 31;
  const int nb = C::NB == 8 ? ((lane & 3) | (((lane >> 3) & 1) << 2)) : tid % C::NB;
  const int pg = C::NB == 8 ? ((tid >> 5) * 4 + (((lane >> 2) & 1) | ((lane >> 4) << 1))) : tid / C::NB;
  const int j0 = nb * kJT;
  const float* sW1 = sm + C::oW1;
  const float* sB1 = sm + C::oB1;
  const float* sWh = sm + C::oWh;
  const float* sBh = sm + C::oBh;
  const float* sWo = sm + C::oWo;
  const float* sBo = sm + C::oBo;
  const float* sSl = sm + C::oSl;
  float4* buf0 = reinterpret_cast<float4*>(sm + C::oBuf);
  float4* buf1 = buf0 + C::BUF / 4;
  float4* sU = reinterpret_cast<float4*>(sm + C::oU);
  float* sX = sm + C::oX;
  float* sY = sX + C::P;
  float* sRed = sm + C::oRed;
  float* sDw = sm + C::oDw;
  float* sAcc = sm + C::oAcc;
  constexpr bool DSM = C::DW_SMEM;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + C::TOTAL - 8);
  const float m1 = a.m1, m2 = a.m2;

#ifdef PINN_PHASE_PROF
  long long prof_acc[20] = {};
  long long prof_t0 = clock64();
  int prof_cur = 0;
#endif
  Stash st;
  st.tid = tid;
  st.nthr = T;
  st.g = nullptr;
  st.taddr = 0;
  if constexpr (MODE != 1) {
    if (a.gstash == nullptr) {
      if (tid < 32) {
        __syncwarp();
        tmem_alloc<2 * T>(tslot);
      }
      tmem_fence_before();
      cta_sync();
      tmem_fence_after();
      const int warp = tid >> 5;
      st.taddr = *tslot + (uint32_t((warp & 3) * 32) << 16) + uint32_t((warp >> 2) * kStashCols);
    } else {
      st.g = a.gstash + size_t(blockIdx.x) * NH * kA * T;
    }
  }

  // persistent CTAs take chunks from a global counter in `order` (largest
  // chunks first, one-tile chunks last), so the tail is one tile long.  Which
  // CTA runs a chunk never changes its result: every chunk owns its partial
  // slot and K5 sums the slots in a fixed order.
  // MODE 2 (the fused single-GPU step): indices [0, n_chunks2) are the
  // payload chunks (K2's work), then the loss chunks; an interface loss chunk
  // waits until every payload chunk is done (all CTAs are resident and payload
  // chunks are handed out first, so the wait always ends).
  int& s_next = *reinterpret_cast<int*>(sm + C::TOTAL - 7);   // next chunk index (dynamic smem, after tslot)
  int* xcount = reinterpret_cast<int*>(sm + C::TOTAL - 16);    // [kMaxPeers] peer rows of a payload chunk
  int cur_sub = -1;
  const int n_pay = MODE == 2 ? a.n_chunks2 : 0;
  // peer-store exchange of the fused step: this launch's step index (receive
  // slot parity, expected arrivals) and per-peer row counts of a payload chunk
  const bool px = MODE == 2 && a.px.n > 0;
  const int xstep = px ? *reinterpret_cast<volatile int*>(a.px.step) : 0;
  const int64_t roff = px ? int64_t(xstep & 1) * a.px.n_recv : 0;
  if (tid < kMaxPeers) xcount[tid] = 0;
  volatile int* sst = reinterpret_cast<volatile int*>(sm + C::TOTAL - 6);   // sticky state [6] (next_item)
  if (tid == 0) {
    sst[0] = -1;
    sst[1] = 0;
    sst[2] = -1;
    sst[3] = 0;
  }
#pragma unroll 1
  for (;;) {
    PROF_MARK(0);
    if (tid == 0) s_next = MODE == 2 ? next_item(a, n_pay, sst) : atomicAdd(a.sched, 1);
    cta_sync();
    const int idx = s_next;
    if (idx >= a.n_chunks + n_pay) break;
    const bool pay = MODE == 1 || (MODE == 2 && idx < n_pay);   // payload chunk (forward + payload epilogue)
    const int li = idx - n_pay;
    const bool direct = MODE == 2 && a.sub_chunk_off != nullptr;   // sticky: li is the chunk index
    const int c = pay ? (MODE == 2 ? idx : (a.order ? a.order[idx] : idx)) : (direct ? li : (a.order ? a.order[li] : li));
    const Chunk ch = (MODE == 2 && pay) ? a.chunks2[c] : a.chunks[c];
    if (MODE == 2 && !pay && ch.pad) {
      // interface loss chunk: acquire the completed payload rows (local, and the peers')
      wait_payload(a, n_pay, xstep);
      cta_sync();
    }
    if (ch.sub != cur_sub) {
      cta_sync();
      PROF_MARK(1);
      load_weights<N, NH, DO, T>(a.params + size_t(ch.sub) * a.pstride, a.slope_n, sm);
      cur_sub = ch.sub;
    }
    PROF_MARK(0);
    const float4 lw = a.sub_w[ch.sub];
    const int act = ACT == kActMixed ? a.sub_act[ch.sub] : ACT;   // uniform per chunk
    float* Pc = a.partial + size_t(c) * a.pstride;
    float* A = DSM ? sAcc : Pc;   // gradient accumulator of this chunk
    if (DSM && !pay) {
      cta_sync();
      for (int e = tid; e < C::ACC; e += T) sAcc[e] = 0.0f;
    }
    const int ntiles = (ch.count + C::P - 1) / C::P;
    if (!pay) {
      if (ntiles == 0) {   // a subdomain without points: its slot holds zeros
        if (!DSM)
          for (int e = tid; e < a.pstride; e += T) Pc[e] = 0.0f;
        if (tid < 4) a.partial_loss[size_t(c) * 4 + tid] = 0.0f;
      }
    }
    // the chunk's tiles, compiled once per mode (payload / loss); a per-
    // subdomain-activation instance branches on `act` around each activation
    // loop only (with_act), never around the GEMMs
    auto chunk_body = [&](auto mode_c) {
      constexpr int MS = decltype(mode_c)::value;   // 0 loss + gradient, 1 payload
      // coordinates of the next tile are loaded into registers while the
      // current tile computes (thread p < P owns point p of a tile)
      static_assert(C::P <= T, "one staged point per thread");
      float cx = 0.0f, cy = 0.0f;
      if (tid < min(C::P, ch.count)) {
        cx = a.coords[int64_t(ch.start) + tid];
        cy = a.coords[a.n_points + int64_t(ch.start) + tid];
      }
      float lsum[4] = {0.0f, 0.0f, 0.0f, 0.0f};   // this thread's MSE_u, MSE_F, MSE_uavg, MSE_if partials (chunk)
#pragma unroll 1
      for (int t = 0; t < ntiles; ++t) {
        const int64_t p0 = int64_t(ch.start) + int64_t(t) * C::P;
        const int np = min(C::P, ch.count - t * C::P);
        const bool first = (t == 0);
        PROF_MARK(MS == 1 ? 10 : 2);
        cta_sync();
        if (tid < C::P) {
          sX[tid] = cx;
          sY[tid] = cy;
          cx = cy = 0.0f;
          if (t + 1 < ntiles && tid < min(C::P, ch.count - (t + 1) * C::P)) {
            cx = a.coords[p0 + C::P + tid];
            cy = a.coords[a.n_points + p0 + C::P + tid];
          }
        }
        cta_sync();

        PROF_MARK(MS == 1 ? 10 : 3);
        // ------------------------------------------------------------ forward
        float4 z[kJT];   // this thread's neurons' jets (value, d1, d2, Delta_S)
        {
          const float x = sX[pg], y = sY[pg];
#pragma unroll
          for (int jj = 0; jj < kJT; ++jj) {
            const int j = j0 + jj;
            const float w0 = sW1[2 * j], w1 = sW1[2 * j + 1];
            // z = W^1 x + b^1; dz/dx1 = W^1[:,0]; dz/dx2 = W^1[:,1]; Delta z = 0
            z[jj] = make_float4(fmaf(w0, x, fmaf(w1, y, sB1[j])), w0, w1, 0.0f);
          }
          const float s = sSl[0];
          with_act<ACT>(act, [&](auto act_c) {
            constexpr int AS = decltype(act_c)::value;
#pragma unroll
            for (int jj = 0; jj < kJT; ++jj) z[jj].x = stash_x<AS>(z[jj].x, s, act);
            if constexpr (MS == 0) st.store(0, reinterpret_cast<const float*>(z));
#pragma unroll
            for (int jj = 0; jj < kJT; ++jj) buf0[C::row(j0) + jj * C::PSTR + pg] = act_fwd<AS>(z[jj], s, m1, m2, act);
          });
        }
        cta_sync();
#pragma unroll 1
        for (int k = 2; k <= NH; ++k) {
          const float4* Hin = (k & 1) ? buf1 : buf0;
          float4* Hout = (k & 1) ? buf0 : buf1;
          PROF_MARK(MS == 1 ? 10 : 12);
          gemm_fwd<N, NH, DO, T, (ACT == kActMixed && kUfFwd == 0) ? 10 : kUfFwd>(Hin, sWh + (k - 2) * C::WROWS, sBh + (k - 2) * N, z, pg, nb);
          PROF_MARK(MS == 1 ? 10 : 13);
          const float s = sSl[k - 1];
          with_act<ACT>(act, [&](auto act_c) {
            constexpr int AS = decltype(act_c)::value;
#pragma unroll
            for (int jj = 0; jj < kJT; ++jj) z[jj].x = stash_x<AS>(z[jj].x, s, act);
            if constexpr (MS == 0) st.store(k - 1, reinterpret_cast<const float*>(z));
#pragma unroll
            for (int jj = 0; jj < kJT; ++jj) Hout[C::row(j0) + jj * C::PSTR + pg] = act_fwd<AS>(z[jj], s, m1, m2, act);
          });
          PROF_MARK(MS == 1 ? 10 : 14);
          cta_sync();
        }
        PROF_MARK(MS == 1 ? 10 : 4);
        const float4* HL = (NH & 1) ? buf0 : buf1;   // H^{NH}
        // output layer: 4 lanes per (point, output), each over every 4th input,
        // combined by a fixed xor-shuffle tree (short dependent chains)
        static_assert((4 * C::P * DO) % 32 == 0, "warp-uniform trip count");
        for (int t4 = tid; t4 < 4 * C::P * DO; t4 += T) {
          const int qq = t4 & 3, idx = t4 >> 2;
          const int p = idx % C::P, o = idx / C::P;
          float4 acc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
          const float* w = sWo + o * C::WS;
          // constant trip count (N / 4 for every qq): fully unrolled, so all
          // its shared loads issue up front (the 4-fold unrolled loop stalled
          // on the shared-load scoreboard)
#pragma unroll
          for (int ii = 0; ii < N / 4; ++ii) {
            const int i = qq + 4 * ii;
            fma4(acc, w[i], HL[C::row(i) + p]);
          }
#pragma unroll
          for (int off = 1; off < 4; off <<= 1) {
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
            acc.z += __shfl_xor_sync(0xffffffffu, acc.z, off);
            acc.w += __shfl_xor_sync(0xffffffffu, acc.w, off);
          }
          acc.x += sBo[o];
          if (qq == 0) sU[p * DO + o] = acc;
        }
        cta_sync();

        PROF_MARK(MS == 1 ? 11 : 5);
        // ----------------------------------------------------------- epilogue
        if constexpr (MS == 1) {
          // payload: u(x_I) and f.n (cPINN) or F (XPINN) (Algorithm 1)
          for (int p = tid; p < np; p += T) {
            float4 U[DO];
#pragma unroll
            for (int o = 0; o < DO; ++o) U[o] = sU[p * DO + o];
            point_payload<DO>(a, p0 + p, sX[p], sY[p], U, xstep, px ? xcount : nullptr);
          }
          continue;
        } else {
          for (int p = tid; p < C::P; p += T) {
            float4 U[DO], Ub[DO];
#pragma unroll
            for (int o = 0; o < DO; ++o) {
              U[o] = sU[p * DO + o];
              Ub[o] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            }
            if (p < np) point_adjoint<DO>(a, p0 + p, sX[p], sY[p], lw, U, Ub, lsum, roff);
#pragma unroll
            for (int o = 0; o < DO; ++o) sU[p * DO + o] = Ub[o];
          }
          cta_sync();

          PROF_MARK(6);
          // ------------------------------------------------------------ reverse
          // output layer: dW^L, db^L
          for (int t4 = tid; t4 < 4 * DO * N; t4 += T) {   // warp-uniform trip count
            const int qq = t4 & 3, idx = t4 >> 2;
            const int o = idx / N, i = idx % N;
            // global chunk partial: its current value is loaded before the dot product
            [[maybe_unused]] const float prev = (!DSM && qq == 0 && !first) ? __ldcg(A + LY::offW(NH + 1) + idx) : 0.0f;
            float2 a2 = make_float2(0.0f, 0.0f);   // channel pairs (x.x + z.z, y.y + w.w)
#pragma unroll
            for (int pp = 0; pp < C::P / 4; ++pp) {
              const int p = qq + 4 * pp;
              const float4 h = HL[C::row(i) + p];
              const float4 ub = sU[p * DO + o];
              a2 = __ffma2_rn(make_float2(h.x, h.y), make_float2(ub.x, ub.y), a2);
              a2 = __ffma2_rn(make_float2(h.z, h.w), make_float2(ub.z, ub.w), a2);
            }
            float acc = a2.x + a2.y;
            acc += __shfl_xor_sync(__activemask(), acc, 1);
            acc += __shfl_xor_sync(__activemask(), acc, 2);
            if (qq == 0) {
              if constexpr (DSM)
                acc_add<DSM>(A, LY::offW(NH + 1) + idx, acc, first);
              else
                A[LY::offW(NH + 1) + idx] = first ? acc : prev + acc;
            }
          }
          if (tid < DO) {
            float acc = 0.0f;
            for (int p = 0; p < C::P; ++p) acc += sU[p * DO + tid].x;
            acc_add<DSM>(A, LY::offB(NH + 1) + tid, acc, first);
          }
          float4 hb[kJT];
#pragma unroll
          for (int e = 0; e < kJT; ++e) hb[e] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
          for (int o = 0; o < DO; ++o) {
            const float4 ub = sU[pg * DO + o];
#pragma unroll
            for (int jj = 0; jj < kJT; ++jj) {
              fma4(hb[jj], sWo[o * C::WS + j0 + jj], ub);
            }
          }
          {
            st.load(NH - 1, reinterpret_cast<float*>(z));
            const float s = sSl[NH - 1];
            with_act<ACT>(act, [&](auto act_c) {
              constexpr int AS = decltype(act_c)::value;
#pragma unroll
              for (int jj = 0; jj < kJT; ++jj) hb[jj] = act_bwd<AS>(z[jj], hb[jj], s, m1, m2, act);
            });
            if (NH >= 2) {
              st.load(NH - 2, reinterpret_cast<float*>(z));   // BUF3: stays raw (layer NH - 1's jets)
              if constexpr (!C::BUF3) {
                const float s2 = sSl[NH - 2];
                with_act<ACT>(act, [&](auto act_c) {
                  constexpr int AS = decltype(act_c)::value;
#pragma unroll
                  for (int jj = 0; jj < kJT; ++jj) z[jj] = act_fwd<AS>(z[jj], s2, m1, m2, act);
                });
              }
            }
          }
          float4* bufZ = buf0;   // adjoint of the current layer's pre-activation
          float4* bufH = buf1;   // activation of the layer below
          float4* bufN = reinterpret_cast<float4*>(sm + C::oBuf3);   // BUF3: the next step's bufH
          cta_sync();
          PROF_MARK(7);
#pragma unroll
          for (int jj = 0; jj < kJT; ++jj) bufZ[C::row(j0) + jj * C::PSTR + pg] = hb[jj];
          if (NH >= 2) {
            if constexpr (C::BUF3) {
              const float s2 = sSl[NH - 2];
              with_act<ACT>(act, [&](auto act_c) {
                constexpr int AS = decltype(act_c)::value;
#pragma unroll
                for (int jj = 0; jj < kJT; ++jj)
                  bufH[C::row(j0) + jj * C::PSTR + pg] = act_fwd<AS>(z[jj], s2, m1, m2, act);
              });
            } else {
#pragma unroll
              for (int jj = 0; jj < kJT; ++jj) bufH[C::row(j0) + jj * C::PSTR + pg] = z[jj];
            }
          }
          cta_sync();
#pragma unroll 1
          for (int k = NH; k >= 2; --k) {
            // dW^k, db^k
            PROF_MARK(15);
            gemm_dw<N, NH, DO, T, DSM, kUfDw>(bufZ, bufH, A + LY::offW(k), A + LY::offB(k), first, sDw);   // partials
            float pre[DwPre<N, NH, DO, T, DSM>::IT], preb = 0.0f;
            gemm_dw_prefetch<N, NH, DO, T, DSM>(A + LY::offW(k), A + LY::offB(k), first, pre, preb);
            // adjoint of H^{k-1}, then of Z^{k-1}
            PROF_MARK(16);
            gemm_bwd<N, NH, DO, T, kUfBwdOf<N, ACT>>(bufZ, sWh + (k - 2) * C::WROWS, hb, pg, nb);
            PROF_MARK(17);
            if constexpr (!C::BUF3) st.load(k - 2, reinterpret_cast<float*>(z));   // BUF3: z holds it already
            const float s = sSl[k - 2];
            with_act<ACT>(act, [&](auto act_c) {
              constexpr int AS = decltype(act_c)::value;
#pragma unroll
              for (int jj = 0; jj < kJT; ++jj) hb[jj] = act_bwd<AS>(z[jj], hb[jj], s, m1, m2, act);
            });
            const bool more = (k - 1 >= 2);
            if (more) {
              st.load(k - 3, reinterpret_cast<float*>(z));
              const float s2 = sSl[k - 3];
              with_act<ACT>(act, [&](auto act_c) {
                constexpr int AS = decltype(act_c)::value;
                if constexpr (C::BUF3) {
                  // H^{k-2} straight into the free buffer (nobody reads it this step);
                  // z keeps layer k-2's raw jets for the next step's act_bwd
#pragma unroll
                  for (int jj = 0; jj < kJT; ++jj)
                    bufN[C::row(j0) + jj * C::PSTR + pg] = act_fwd<AS>(z[jj], s2, m1, m2, act);
                } else {
#pragma unroll
                  for (int jj = 0; jj < kJT; ++jj) z[jj] = act_fwd<AS>(z[jj], s2, m1, m2, act);
                }
              });
            }
            db_sum<N, NH, DO, T, DSM>(bufZ, sDw, A + LY::offB(k));
            PROF_MARK(18);
            cta_sync();
            PROF_MARK(19);
            gemm_dw_reduce<N, NH, DO, T, DSM>(A + LY::offW(k), A + LY::offB(k), first, sDw, pre, preb);
#pragma unroll
            for (int jj = 0; jj < kJT; ++jj) {
              bufZ[C::row(j0) + jj * C::PSTR + pg] = hb[jj];
              if (!C::BUF3 && more) bufH[C::row(j0) + jj * C::PSTR + pg] = z[jj];
            }
            if constexpr (C::BUF3) {
              float4* t = bufH;
              bufH = bufN;
              bufN = t;
            }
            cta_sync();
          }
          PROF_MARK(8);
          // layer 1: dW^1[j] = sum_p zb_v x_p + zb_{d_i}; db^1 = sum_p zb_v
          for (int t4 = tid; t4 < 4 * N; t4 += T) {
            const int qq = t4 & 3, j = t4 >> 2;
            const bool pf = !DSM && qq == 0 && !first;   // global partial: load before the sums
            [[maybe_unused]] const float p0 = pf ? __ldcg(A + LY::offW(1) + 2 * j) : 0.0f;
            [[maybe_unused]] const float p1 = pf ? __ldcg(A + LY::offW(1) + 2 * j + 1) : 0.0f;
            [[maybe_unused]] const float pb = pf ? __ldcg(A + LY::offB(1) + j) : 0.0f;
            float a0 = 0.0f, a1 = 0.0f, ab = 0.0f;
#pragma unroll
            for (int pp = 0; pp < C::P / 4; ++pp) {
              const int p = qq + 4 * pp;
              const float4 zb = bufZ[C::row(j) + p];
              a0 = fmaf(zb.x, sX[p], a0) + zb.y;
              a1 = fmaf(zb.x, sY[p], a1) + zb.z;
              ab += zb.x;
            }
            const unsigned mk = __activemask();
#pragma unroll
            for (int o = 1; o < 4; o <<= 1) {
              a0 += __shfl_xor_sync(mk, a0, o);
              a1 += __shfl_xor_sync(mk, a1, o);
              ab += __shfl_xor_sync(mk, ab, o);
            }
            if (qq == 0) {
              if constexpr (DSM) {
                acc_add<DSM>(A, LY::offW(1) + 2 * j, a0, first);
                acc_add<DSM>(A, LY::offW(1) + 2 * j + 1, a1, first);
                acc_add<DSM>(A, LY::offB(1) + j, ab, first);
              } else {
                A[LY::offW(1) + 2 * j] = first ? a0 : p0 + a0;
                A[LY::offW(1) + 2 * j + 1] = first ? a1 : p1 + a1;
                A[LY::offB(1) + j] = first ? ab : pb + ab;
              }
            }
          }
          // the slope entries of the partial stay 0 (K5 fills them)
          if (tid == 0 && first && !DSM) {
#pragma unroll
            for (int k = 1; k <= NH; ++k) Pc[LY::offA(k)] = 0.0f;
          }
        }
      }
      PROF_MARK(9);
      if constexpr (MS == 0) {
        // loss partials of the chunk: fixed-order block reduction once per chunk
        if (ntiles > 0) {
          block_sum<4, T>(lsum, sRed);
          if (tid == 0) {
#pragma unroll
            for (int r = 0; r < 4; ++r) a.partial_loss[size_t(c) * 4 + r] = lsum[r];
          }
        }
      }
    };
    if constexpr (MODE == 2) {
      if (pay)
        chunk_body(std::integral_constant<int, 1>{});
      else
        chunk_body(std::integral_constant<int, 0>{});
    } else {
      chunk_body(std::integral_constant<int, MODE>{});
    }
    if (MODE == 2 && pay) {
      // publish this payload chunk (release: all its rows are written)
      cta_sync();
      if (px) publish_peer_rows(a, xcount);
      if (tid == 0) {
        __threadfence();
        atomicAdd(a.sched + 4, 1);
      }
    }
    if (DSM && !pay) {
      // flush the chunk's gradient (slope slots stay 0; K5 fills them)
      cta_sync();
      for (int e = tid; e < C::ACC; e += T) Pc[e] = sAcc[e];
    }
    cta_sync();   // every thread has read s_next before it is overwritten
  }
#ifdef PINN_PHASE_PROF
  PROF_MARK(0);
  if (tid == 0 && blockIdx.x < 4)
    printf("PHASE N=%d NH=%d MODE=%d cta=%d: %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld "
           "%lld %lld %lld %lld %lld\n", N, NH, MODE, int(blockIdx.x), prof_acc[0], prof_acc[1], prof_acc[2],
           prof_acc[3], prof_acc[4], prof_acc[5], prof_acc[6], prof_acc[7], prof_acc[8], prof_acc[9], prof_acc[10],
           prof_acc[11], prof_acc[12], prof_acc[13], prof_acc[14], prof_acc[15], prof_acc[16], prof_acc[17],
           prof_acc[18], prof_acc[19]);
#endif
  // the last CTA to leave re-arms the counter for the next launch
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(a.sched + 1, 1) == int(gridDim.x) - 1) {
      a.sched[0] = 0;
      a.sched[1] = 0;
      if (MODE == 2) a.sched[4] = 0;
      if (MODE == 2) sticky_reset(a);
      if (px) *a.px.step = xstep + 1;
      __threadfence();
    }
  }
  if constexpr (MODE != 1) {
    if (a.gstash == nullptr) {
      tmem_fence_before();
      cta_sync();
      tmem_fence_after();
      if (tid < 32) {
        __syncwarp();
        tmem_dealloc<2 * T>(*tslot);
      }
    }
  }
}

// ----------------------------------------------------------------------------
// K5a k_reduce: gradient reduction over chunk partials (fixed order) and J_q
// assembly (Eq. 5/6).  K5b k_slope_adam: slope gradients from the exact
// homogeneity identity  a_k dJ/da_k = <W^k, dJ/dW^k> + <b^k, dJ/db^k>
// (J depends on s_k = n a_k, W^k, b^k only through s_k W^k and s_k b^k),
// evaluated as fp64 dot products, then optionally the Adam step.
// ----------------------------------------------------------------------------
constexpr int kMaxHidden = 8;
constexpr int kRB = 256;

// per-subdomain status bits (loss column 5)
constexpr int kFlagJ = 1;          // J_q non-finite
constexpr int kFlagGrad = 2;       // a W / b gradient entry non-finite
constexpr int kFlagSlopeGrad = 4;  // a slope gradient non-finite
constexpr int kFlagSlopeZero = 8;  // a^k == 0: the slope identity is undefined (gradient set to NaN)

struct RArgs {
  const float* partial;
  const float* partial_loss;
  const int32_t* sub_chunk;   // [n_sub+1]
  int pstride;
  float* grad;                // [n_sub][pstride]
  float* params;
  float* m;
  float* v;
  int32_t* tstep;             // [n_sub]
  int32_t* done;              // [n_sub] block counters
  const float4* sub_w;        // loss weights
  const float4* sub_adam;     // lr, beta1, beta2, eps
  float* loss;                // [n_sub][8]
  int32_t* sflag;             // [n_sub] status bits of the current evaluation (zeroed before K5a)
  double* slope_part;         // [n_sub][gridDim.x][kMaxHidden] per-block slope partials (K5a -> K5b)
  int mode;                   // k_slope_adam: 0 slopes only, 1 slopes + Adam, 2 Adam only
  int n_hidden;               // 0: no slope parameters
  int nb5a;                   // K5a blocks per subdomain (slope_part stride)
  int offW[kMaxHidden], nW[kMaxHidden], offB[kMaxHidden], nB[kMaxHidden], offA[kMaxHidden];
};

// K5a: gradient of subdomain q (blockIdx.y) = sum of its chunk partials,
// accumulated in FP64 (the slope identity below is a cancelling dot product of
// these sums, so their rounding matters).  A block owns kRW
// consecutive entries (a lane owns 4: one 512-B float4 row segment per chunk
// and warp); warp w sums chunks c0 + w, c0 + w + 8, ... with 8 loads in
// flight, and warp 0 adds the 8 warp sums in warp order -- a fixed order, so
// the result is bitwise reproducible, with 64 row loads in flight per entry
// instead of 8 (C3's single subdomain: 105 chunk partials of 7 blocks were a
// 20 us latency chain).  Indices that are not parameters (16-B padding, slope
// slots) are never written by K1; the partial region is zeroed once at create.
// RB threads per block: 256, or 512 for small nets (width 20: few entry
// blocks, so 16 warps per block halve each warp's chain of chunk rows; the
// choice depends only on the net, so it is the same under every placement)
constexpr int kRW = 128;   // entries per K5a block
template <int RB>
__global__ void __launch_bounds__(RB) k_reduce(const RArgs r) {
  __shared__ double red[RB / 32][kRW];
  const int q = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int i0 = blockIdx.x * kRW;
  const int i = i0 + 4 * lane;   // this lane's 4 entries (pstride is a multiple of 4)
  const int c0 = r.sub_chunk[q], c1 = r.sub_chunk[q + 1];
  const float* P = r.params + size_t(q) * r.pstride;
  {
    double g[4] = {0.0, 0.0, 0.0, 0.0};
    if (i < r.pstride) {
      constexpr int NW = RB / 32;
      const float4* src = reinterpret_cast<const float4*>(r.partial + i);
      const size_t cs = size_t(r.pstride) / 4;   // float4 per partial
      int c = c0 + w;
      for (; c + 7 * NW < c1; c += 8 * NW) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + size_t(c + u * NW) * cs);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          g[0] += double(v[u].x); g[1] += double(v[u].y); g[2] += double(v[u].z); g[3] += double(v[u].w);
        }
      }
      for (; c < c1; c += NW) {
        const float4 v = __ldcg(src + size_t(c) * cs);
        g[0] += double(v.x); g[1] += double(v.y); g[2] += double(v.z); g[3] += double(v.w);
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) red[w][4 * lane + e] = g[e];
  }
  __syncthreads();
  if (w == 0) {
    double g[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int ww = 0; ww < RB / 32; ++ww)
#pragma unroll
      for (int e = 0; e < 4; ++e) g[e] += red[ww][4 * lane + e];
    if (i < r.pstride) {
      float4 gf = make_float4(float(g[0]), float(g[1]), float(g[2]), float(g[3]));
      *reinterpret_cast<float4*>(r.grad + size_t(q) * r.pstride + i) = gf;
      if (!isfinite(gf.x) || !isfinite(gf.y) || !isfinite(gf.z) || !isfinite(gf.w)) atomicOr(r.sflag + q, kFlagGrad);
    }
    // per-block partial sums of <W^k, dJ/dW^k> + <b^k, dJ/db^k> (fp64, fixed
    // order, from the FP64 sums above) for the slope identity; K5b combines
    // them (no cross-block reads of parameters that K5b's Adam updates)
    for (int k = 0; k < r.n_hidden; ++k) {
      const int w0 = r.offW[k], w1 = w0 + r.nW[k], b0 = r.offB[k], b1 = b0 + r.nB[k];
      double* slot = r.slope_part + (size_t(q) * gridDim.x + blockIdx.x) * kMaxHidden + k;
      const bool hit = (w0 < i0 + kRW && w1 > i0) || (b0 < i0 + kRW && b1 > i0);   // warp-uniform
      if (!hit) {
        if (lane == 0) *slot = 0.0;
        continue;
      }
      double acc = 0.0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int ie = i + e;
        if ((ie >= w0 && ie < w1) || (ie >= b0 && ie < b1)) acc += double(P[ie]) * g[e];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) *slot = acc;
    }
  }
  if (blockIdx.x == 0 && w == 1) {
    // loss terms of subdomain q: lane l sums chunks c0 + l, c0 + l + 32, ...; fixed shuffle tree
    const int tid = lane;
    double l4[4] = {0.0, 0.0, 0.0, 0.0};
    for (int c = c0 + tid; c < c1; c += 32) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(r.partial_loss) + c);
      l4[0] += v.x; l4[1] += v.y; l4[2] += v.z; l4[3] += v.w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int t = 0; t < 4; ++t) l4[t] += __shfl_xor_sync(0xffffffffu, l4[t], o);
    if (tid == 0) {
      const float4 w = r.sub_w[q];
      const double J = double(w.x) * l4[0] + double(w.y) * l4[1] + double(w.z) * l4[2] + double(w.w) * l4[3];
      float* L = r.loss + size_t(q) * 8;
      L[0] = float(l4[0]); L[1] = float(l4[1]); L[2] = float(l4[2]); L[3] = float(l4[3]); L[4] = float(J);
      L[6] = 0.0f; L[7] = 0.0f;
      if (!isfinite(L[4])) atomicOr(r.sflag + q, kFlagJ);
    }
  }
}

// K5b: slope gradients, then (mode 1, 2) the Adam step; the last block of a
// subdomain publishes its status bits in loss column 5 (and advances t).
__global__ void __launch_bounds__(kRB) k_slope_adam(const RArgs r) {
  const int q = blockIdx.y;
  const int i0 = blockIdx.x * kRB;
  const int tid = threadIdx.x;
  const float* P = r.params + size_t(q) * r.pstride;
  float* G = r.grad + size_t(q) * r.pstride;
  // slope gradients: the block owning a^k combines K5a's
  // per-block partials in block order.  a^k = 0 leaves the identity
  // undefined: the gradient is set to NaN and flagged (never a silent 0).
  // Warp k handles a^k: its lanes sum K5a's block partials of the blocks that
  // overlap W^k / b^k (lane-strided, fixed order), then a fixed shuffle tree.
  const int k = tid >> 5, lane = tid & 31;
  if (r.mode != 2 && k < r.n_hidden) {
    const int oa = r.offA[k];
    if (oa >= i0 && oa < i0 + kRB) {
      const int bb0 = r.offW[k] / kRW, bb1 = (r.offB[k] + r.nB[k] - 1) / kRW + 1;
      const double* sp = r.slope_part + size_t(q) * r.nb5a * kMaxHidden + k;
      double sum = 0.0;
      for (int b = bb0 + lane; b < bb1; b += 32) sum += sp[size_t(b) * kMaxHidden];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane == 0) {
        const double a = double(P[oa]);
        float ga;
        if (a == 0.0) {
          ga = __int_as_float(0x7fc00000);
          atomicOr(r.sflag + q, kFlagSlopeZero);
        } else {
          ga = float(sum / a);
          if (!isfinite(ga)) atomicOr(r.sflag + q, kFlagSlopeGrad);
        }
        G[oa] = ga;
      }
    }
  }
  __syncthreads();
  const int t = r.tstep[q] + 1;
  if (r.mode != 0) {
    const int i = i0 + tid;
    if (i < r.pstride) {
      const float g = G[i];
      const float4 ad = r.sub_adam[q];
      const size_t k = size_t(q) * r.pstride + i;
      const float mm = ad.y * r.m[k] + (1.0f - ad.y) * g;
      const float vv = ad.z * r.v[k] + (1.0f - ad.z) * g * g;
      r.m[k] = mm;
      r.v[k] = vv;
      const float mh = mm / (1.0f - powf(ad.y, float(t)));
      const float vh = vv / (1.0f - powf(ad.z, float(t)));
      r.params[k] -= ad.x * mh / (sqrtf(vh) + ad.w);
    }
  }
  // the last block of subdomain q publishes the status bits and (Adam) advances t
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const int prev = atomicAdd(&r.done[q], 1);
    if (prev == int(gridDim.x) - 1) {
      __threadfence();
      if (r.mode != 0) r.tstep[q] = t;
      // publish this evaluation's status bits, then clear them for the next
      // one (every K5a is followed by a K5b, so no memset node is needed)
      if (r.mode != 2) r.loss[size_t(q) * 8 + 5] = float(atomicExch(r.sflag + q, 0));
      r.done[q] = 0;
      __threadfence();
    }
  }
}

__global__ void k_gather(const float* src, const int32_t* map, int n, int pstride, int sub_stride_dst,
                         float* dst, int n_sub) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int q = blockIdx.y;
  if (i < n && q < n_sub) dst[size_t(q) * sub_stride_dst + i] = src[size_t(q) * pstride + map[i]];
}
__global__ void k_scatter(const float* src, const int32_t* map, int n, int pstride, int sub_stride_src,
                          float* dst, int n_sub) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int q = blockIdx.y;
  if (i < n && q < n_sub) dst[size_t(q) * pstride + map[i]] = src[size_t(q) * sub_stride_src + i];
}

// ----------------------------------------------------------------------------
// K6: value-only forward + Eq. (4) stitching.  The owners of a
// point are the caller's list (kind 0) or classified here (kind 1 Cartesian
// cells, kind 2 nearest-seed cells inside a polygon), in FP64.
// ----------------------------------------------------------------------------
struct Geo {
  int kind;                 // 0 caller's owners, 1 boxes, 2 Voronoi
  int owner_mode;           // 0 stitched (1/S), 1 lowest-id owner only
  const int32_t* owners;    // kind 0: [n][4] local ids, -1 unused
  int n_geo;
  const float* geo;         // boxes [n_geo][4] / seeds [n_geo][2]
  const int32_t* local;     // [n_geo] local subdomain, -1 = other rank
  int n_poly;
  const float* poly;        // [n_poly][2]
  float tol;
};

// even-odd crossing test; points within 1e-9 of an edge count as inside
__device__ __forceinline__ bool in_polygon(double x, double y, const float* P, int n) {
  bool in = false;
  for (int i = 0, j = n - 1; i < n; j = i++) {
    const double xi = P[2 * i], yi = P[2 * i + 1], xj = P[2 * j], yj = P[2 * j + 1];
    const double ex = xj - xi, ey = yj - yi;
    const double l2 = ex * ex + ey * ey;
    double t = l2 > 0.0 ? ((x - xi) * ex + (y - yi) * ey) / l2 : 0.0;
    t = fmin(1.0, fmax(0.0, t));
    const double dx = x - (xi + t * ex), dy = y - (yi + t * ey);
    if (dx * dx + dy * dy <= 1e-18) return true;
    if ((yi > y) != (yj > y) && x < (xj - xi) * (y - yi) / (yj - yi) + xi) in = !in;
  }
  return in;
}

// local owners (<= 4) of point (x, y) and their weight (1/S, or 1 for the
// lowest-id owner in owner mode); returns the number of local owners
__device__ __forceinline__ int classify(const Geo& G, int64_t p, float xf, float yf, int* own, float& w) {
  int nl = 0, S = 0;
  if (G.kind == 0) {
    for (int k = 0; k < 4; ++k) {
      const int q = G.owners[p * 4 + k];
      if (q >= 0) own[nl++] = q;
    }
    S = nl;
    w = S > 0 ? 1.0f / float(S) : 0.0f;
    return nl;
  }
  const double x = xf, y = yf, tol = G.tol;
  int first = -1;
  if (G.kind == 1) {
    for (int g = 0; g < G.n_geo; ++g) {
      const float* B = G.geo + 4 * g;
      if (x >= double(B[0]) - tol && x <= double(B[2]) + tol && y >= double(B[1]) - tol && y <= double(B[3]) + tol) {
        ++S;
        if (first < 0) first = g;
        const int q = G.local[g];
        if (q >= 0 && nl < 4 && (G.owner_mode == 0 || g == first)) own[nl++] = q;
      }
    }
  } else if (in_polygon(x, y, G.poly, G.n_poly)) {
    double dmin = 1e300;
    for (int g = 0; g < G.n_geo; ++g) {
      const double dx = x - double(G.geo[2 * g]), dy = y - double(G.geo[2 * g + 1]);
      dmin = fmin(dmin, sqrt(dx * dx + dy * dy));
    }
    for (int g = 0; g < G.n_geo; ++g) {
      const double dx = x - double(G.geo[2 * g]), dy = y - double(G.geo[2 * g + 1]);
      if (sqrt(dx * dx + dy * dy) <= dmin + tol) {
        ++S;
        if (first < 0) first = g;
        const int q = G.local[g];
        if (q >= 0 && nl < 4 && (G.owner_mode == 0 || g == first)) own[nl++] = q;
      }
    }
  }
  w = G.owner_mode == 1 ? 1.0f : (S > 0 ? 1.0f / float(S) : 0.0f);
  return nl;
}

template <int N, int NH, int DO, int ACT>
__global__ void k_predict(const float* params, int pstride, float slope_n, const float* pts, const Geo G,
                          int64_t n, float* out, const int32_t* sub_act) {
  using LY = Lay<N, NH, DO>;
  const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const float x = pts[p], y = pts[n + p];
  float acc[DO];
#pragma unroll
  for (int o = 0; o < DO; ++o) acc[o] = 0.0f;
  int own[4];
  float wgt;
  const int nl = classify(G, p, x, y, own, wgt);
  for (int k = 0; k < nl; ++k) {
    const int q = own[k];
    const int act = ACT == kActMixed ? sub_act[q] : ACT;
    const float* P = params + size_t(q) * pstride;
    float h[N], g[N];
    float s = slope_n * P[LY::offA(1)];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      float s0, s1, s2, s3;
      act_derivs<ACT>(s * (P[2 * j] * x + P[2 * j + 1] * y + P[LY::offB(1) + j]), s0, s1, s2, s3, act);
      h[j] = s0;
    }
    for (int l = 2; l <= NH; ++l) {
      s = slope_n * P[LY::offA(l)];
      const float* W = P + LY::offW(l);
      const float* b = P + LY::offB(l);
      for (int j = 0; j < N; ++j) {
        float zz = b[j];
#pragma unroll
        for (int i = 0; i < N; ++i) zz = fmaf(W[j * N + i], h[i], zz);
        g[j] = zz;
      }
#pragma unroll
      for (int j = 0; j < N; ++j) {
        float s0, s1, s2, s3;
        act_derivs<ACT>(s * g[j], s0, s1, s2, s3, act);
        h[j] = s0;
      }
    }
    const float* W = P + LY::offW(NH + 1);
#pragma unroll
    for (int o = 0; o < DO; ++o) {
      float u = P[LY::offB(NH + 1) + o];
#pragma unroll
      for (int i = 0; i < N; ++i) u = fmaf(W[o * N + i], h[i], u);
      acc[o] += u;
    }
  }
#pragma unroll
  for (int o = 0; o < DO; ++o) out[size_t(o) * n + p] = acc[o] * wgt;   // indicator 1/S
}

}  // namespace pinn
