// pinn_dd_device.cuh -- device-side building blocks of the fused sm_100a
// cPINN / XPINN training step (arXiv 2104.10013).  P:n = PAPER.md line n.
//
// Forward-mode Taylor jets.  Every point carries C = 4 channels through the
// network: value, d/dx1, d/dx2 and the masked Laplacian Delta_S (S = dims whose
// pure second derivatives the operator needs; only pure seconds are needed,
// never mixed ones).  For a hidden pre-activation z with jets (z, g1, g2, L)
// and slope s = n a^k (reading Z6) the activation h = sigma(s z)
// propagates as
//   h_v = sigma(u),  h_i = sigma'(u) s g_i,  h_L = sigma''(u) s^2 Q + sigma'(u) s L,
//   u = s z,  Q = sum_{i in S} g_i^2.
// The reverse sweep (act_bwd) is the exact adjoint of that map, including the
// derivative with respect to the slope s (for da^k = n dJ/ds).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pinn {

constexpr int kThreads = 256;   // default CTA: 8 warps, 2 per scheduler; warps w, w+4 share TMEM lane quarter w%4
constexpr int kC = 4;           // jet channels
constexpr int kJT = 10;         // neurons per thread (mapping A)
constexpr int kA = kC * kJT;    // stash floats per thread per hidden layer
constexpr int kStashCols = 256; // TMEM columns per thread (a 128-thread CTA allocates 256, a 256-thread CTA 512)

__host__ __device__ constexpr int al4(int x) { return (x + 3) & ~3; }

// Internal (16-byte padded) parameter layout of one network
// [2, N x NH, DO]; the packed layout of the ABI is W1 b1 a1 W2 b2 a2 ... WL bL.
template <int N, int NH, int DO>
struct Lay {
  // Closed forms (no recursion: a recursive constexpr evaluated with a runtime
  // layer index compiles to a recursive device CALL, which clobbers the warp
  // convergence-barrier registers and leaves warps diverged at bar.sync).
  static constexpr int L = NH + 1;
  static constexpr int H1 = al4(al4(2 * N) + N) + 4;          // start of W^2
  static constexpr int SH = al4(N * N) + al4(N) + 4;          // one hidden layer block
  __host__ __device__ static constexpr int nin(int k) { return k == 1 ? 2 : N; }
  __host__ __device__ static constexpr int nout(int k) { return k == L ? DO : N; }
  __host__ __device__ static constexpr int offW(int k) { return k == 1 ? 0 : H1 + (k - 2) * SH; }
  __host__ __device__ static constexpr int offB(int k) {
    return k == 1 ? al4(2 * N) : offW(k) + al4(nout(k) * N);
  }
  __host__ __device__ static constexpr int offA(int k) { return offB(k) + al4(N); }
  __host__ __device__ static constexpr int total() { return al4(offB(L) + DO); }
};

// recursive reference definition, checked at compile time against the closed forms
template <int N, int NH, int DO>
struct LayRef {
  static constexpr int L = NH + 1;
  static constexpr int nin(int k) { return k == 1 ? 2 : N; }
  static constexpr int nout(int k) { return k == L ? DO : N; }
  static constexpr int offW(int k) { return k == 1 ? 0 : al4(offA(k - 1) + 1); }
  static constexpr int offB(int k) { return al4(offW(k) + nout(k) * nin(k)); }
  static constexpr int offA(int k) { return al4(offB(k) + nout(k)); }
};
template <int N, int NH, int DO>
constexpr bool lay_ok() {
  for (int k = 1; k <= NH + 1; ++k) {
    if (Lay<N, NH, DO>::offW(k) != LayRef<N, NH, DO>::offW(k)) return false;
    if (Lay<N, NH, DO>::offB(k) != LayRef<N, NH, DO>::offB(k)) return false;
    if (k <= NH && Lay<N, NH, DO>::offA(k) != LayRef<N, NH, DO>::offA(k)) return false;
  }
  return true;
}

// Kernel geometry for width N (mapping A: thread = (point group pg, neuron block nb)).
// T = threads per CTA: 256 (one CTA per SM) or 128 (two CTAs per SM, each
// with its own barrier domain, so one CTA's barrier / latency-bound phases
// overlap the other's GEMMs).
template <int N, int NH, int DO, int T = kThreads>
struct KCfg {
  static_assert(N % kJT == 0, "width must be a multiple of kJT");
  static_assert(lay_ok<N, NH, DO>(), "closed-form parameter layout mismatch");
  static_assert(NH * kA <= kStashCols, "reverse-mode stash exceeds the TMEM columns per thread");
  static constexpr int NB = N / kJT;           // neuron blocks
  static constexpr int P = T / NB;             // points per tile (1 point per thread)
  static constexpr int CPS = 256 / T;          // CTAs per SM
  static constexpr int PSTR = P + 1;           // float4 row stride of activation buffers (odd)
  // float4 skew per block of kJT rows: for NB = 2 (width 20) the 8 lanes of a
  // 128-bit store phase (2 neuron blocks x 4 points) then hit 8 distinct 16-B
  // bank groups instead of 2-way conflicts (C3 K1 0.284 -> 0.269 ms).  For
  // NB = 8 the analogous skew (7) slowed 5x80 down (17.97 vs 16.53 ms: it
  // moves the dW-block row reads onto shared banks), so it stays 0 there.
  static constexpr int SKW = NB == 2 ? ((4 - (kJT * PSTR) % 8) % 8 + 8) % 8 : 0;
  __host__ __device__ static constexpr int row(int j) { return j * PSTR + (j / kJT) * SKW; }
  // W^k (k = 2..NH) rows: j*WS + (j/kJT)*4 floats (block skew against bank conflicts)
  static constexpr int WS = al4(N);
  static constexpr int WROWS = N * WS + NB * 4;            // floats per hidden W in smem
  // mapping B (dW): JB x IB register block, interleaved rows, S point splits
  static constexpr int JB = 5;
  static constexpr int IB = 5;
  static constexpr int NJ = N / JB;
  static constexpr int NI = N / IB;
  static constexpr int NBLK = NJ * NI;
  static constexpr int S_MAX = T / NBLK;
  static constexpr int S = S_MAX >= 16 ? 16 : (S_MAX >= 8 ? 8 : (S_MAX >= 4 ? 4 : (S_MAX >= 2 ? 2 : 1)));
  static constexpr size_t SMEM_CAP = T == 256 ? 227 * 1024 : 113 * 1024;   // per CTA at CPS CTAs / SM
  static_assert(P % S == 0, "points per split");
  // smem carve (in floats)
  static constexpr int oW1 = 0;                            // [N][2]
  static constexpr int oB1 = oW1 + 2 * N;                  // [N]
  static constexpr int oWh = al4(oB1 + N);                 // NH-1 hidden layers
  static constexpr int oBh = oWh + (NH - 1) * WROWS;       // [NH-1][N]
  static constexpr int oWo = al4(oBh + (NH - 1) * N);      // [DO][WS]
  static constexpr int oBo = oWo + DO * WS;                // [DO]
  static constexpr int oSl = al4(oBo + DO);                // [NH] slopes s_k = n a^k
  static constexpr int oBuf = al4(oSl + NH) ;              // 2 x [N][PSTR] float4
  static constexpr int BUF = (row(N - 1) + PSTR) * 4;     // floats per activation buffer
  static constexpr int oU = oBuf + 2 * BUF;                // [P][DO] float4
  static constexpr int oX = oU + P * DO * 4;               // [2][P]
  static constexpr int oRed = al4(oX + 2 * P);             // reduction scratch [8 warps][4]
  static constexpr int oDw = oRed + 32;                    // dW/db scratch (split partials / coalescing)
  static constexpr int ACC = Lay<N, NH, DO>::total();
  // scratch: split s holds dW^k as [j][N + 1] (row padding spreads the dW-block
  // writers over the banks; readers walk rows contiguously) then db^k [N]
  // row stride of the split scratch: N + 1 spreads the 16 x 2 / 4 x 8 (width
  // 40: 8 x 4 with NJ = 8 -> stride 41) dW-block writers over the banks; for
  // width 80's 8 x 4 warp blocks, 84 (= 20 mod 32) does
  static constexpr int SROW = N == 80 ? N + 4 : N + 1;
  static constexpr int SSPL = N * SROW;                    // floats per split (W part)
  static constexpr int SCR1 = S * SSPL + S * N;
  static constexpr bool DW_SMEM = (size_t(al4(al4(oDw + (S > 1 ? SCR1 : 0)) + ACC + 4)) * 4) <= SMEM_CAP;
  // the scratch is needed for S > 1 (split partials) and, with the chunk
  // accumulator in global memory, to coalesce the per-tile read-modify-write
  static constexpr int SCR = (S > 1 || !DW_SMEM) ? SCR1 : 0;
  static constexpr int oAcc = al4(oDw + SCR);              // per-chunk gradient accumulator
  // a third activation buffer (widths <= 40, where it fits): the reverse
  // sweep then reads each stash slot from TMEM once (its raw jets stay in
  // registers for the next step's act_bwd; the recomputed activation goes
  // straight into the free buffer) instead of twice
  static constexpr int oBuf3 = al4(oAcc + (DW_SMEM ? ACC : 0));
  static constexpr bool BUF3 = N <= 40 && size_t(al4(oBuf3 + BUF + 16)) * 4 <= SMEM_CAP;
  static constexpr int TOTAL = al4(oBuf3 + (BUF3 ? BUF : 0) + 16);  // + peer row counts [8], tmem slot, s_next, sticky state [4]
  static constexpr size_t SMEM = size_t(TOTAL) * 4;
  static_assert(SMEM <= SMEM_CAP, "shared memory budget");
  static_assert(NBLK * S <= T, "dW blocks per CTA");
  static_assert(T == 256 || T == 128, "128 or 256 threads per CTA");
  static_assert(T == 256 || NH * kA <= kStashCols, "stash columns of a 128-thread CTA");

};

// ----------------------------------------------------------------------------
// activations sigma, sigma', sigma'', sigma''' (ACT: 0 tanh, 1 sin, 2 cos)
// kActMixed: the activation is the runtime argument `act`, one per subdomain
// (Table 3) -- uniform per chunk, so the branch never diverges.
// ----------------------------------------------------------------------------
constexpr int kActMixed = 3;

#ifndef PINN_MUFU_SINCOS
#define PINN_MUFU_SINCOS 1
#endif
// sin and cos of x for |x| up to ~1e4: 3-term Cody-Waite reduction by pi/2 and
// minimax polynomials on [-pi/4, pi/4] (~1e-7 relative).  Replaces sincosf,
// whose Payne-Hanek slow path bloats the unrolled jet loops (instruction-cache
// misses in the per-subdomain-activation kernel).
__device__ __forceinline__ void fast_sincos(float x, float* sn, float* cs) {
#if PINN_MUFU_SINCOS
  // 2-term Cody-Waite reduction by 2 pi to [-pi, pi], then the MUFU sin / cos
  // (|error| <= 2^-21.4 there): 6 FMA-pipe instructions + 2 on the XU pipe
  const float k = rintf(x * 0.159154943091895f);
  float r = fmaf(-k, 6.28318548202514648f, x);
  r = fmaf(-k, -1.7484555314695172e-7f, r);
  *sn = __sinf(r);
  *cs = __cosf(r);
#else
  const float k = rintf(x * 0.636619772f);
  float r = fmaf(-k, 1.5703125f, x);
  r = fmaf(-k, 4.837512969970703125e-4f, r);
  r = fmaf(-k, 7.54978995489188216e-8f, r);
  const float z = r * r;
  const float s = fmaf(r * z, fmaf(z, fmaf(z, -1.9515295891e-4f, 8.3321608736e-3f), -1.6666654611e-1f), r);
  const float co = fmaf(z * z, fmaf(z, fmaf(z, 2.443315711809948e-5f, -1.388731625493765e-3f), 4.166664568298827e-2f),
                        fmaf(-0.5f, z, 1.0f));
  const int q = int(k) & 3;
  const float a = (q & 1) ? co : s;    // sin for q = 0, 2
  const float b = (q & 1) ? s : co;    // cos for q = 0, 2
  *sn = (q & 2) ? -a : a;
  *cs = ((q + 1) & 2) ? -b : b;
#endif
}
template <int ACT>
__device__ __forceinline__ int act_sel(int act) {
  return ACT == kActMixed ? act : ACT;
}
template <int ACT>
__device__ __forceinline__ void act_derivs(float u, float& s0, float& s1, float& s2, float& s3, int act = ACT) {
  const int A = act_sel<ACT>(act);
  if (A == 0) {
    float t = tanhf(u);
    s0 = t;
    s1 = 1.0f - t * t;
    s2 = -2.0f * t * s1;
    s3 = s1 * (6.0f * t * t - 2.0f);
  } else if (A == 1) {
    float sn, cs;
    fast_sincos(u, &sn, &cs);
    s0 = sn; s1 = cs; s2 = -sn; s3 = -cs;
  } else {
    float sn, cs;
    fast_sincos(u, &sn, &cs);
    s0 = cs; s1 = -sn; s2 = -cs; s3 = sn;
  }
}

// What the reverse sweep needs of a hidden pre-activation jet (z, g1, g2, L):
// sigma^(k)(s z) for k = 0..3 and (g1, g2, L).  For tanh every sigma^(k) is a
// polynomial in t = tanh(s z), so the stash keeps (t, g1, g2, L) and the
// reverse pass evaluates no transcendental; sin / cos keep the reduced angle
// of s z (two MUFU ops per evaluation).
#if PINN_MUFU_SINCOS
// sin / cos stash the reduced angle r = s z - 2 pi k in [-pi, pi] (the first
// half of fast_sincos), so every later evaluation -- forward map, reverse
// adjoint, reverse recompute -- is the two MUFU ops alone: bitwise the values
// fast_sincos(s z) gives, without repeating the reduction
__device__ __forceinline__ float reduce_2pi(float x) {
  const float k = rintf(x * 0.159154943091895f);
  const float r = fmaf(-k, 6.28318548202514648f, x);
  return fmaf(-k, -1.7484555314695172e-7f, r);
}
#endif
template <int ACT>
__device__ __forceinline__ float stash_x(float zx, float s, int act = ACT) {
#if PINN_MUFU_SINCOS
  return act_sel<ACT>(act) == 0 ? tanhf(s * zx) : reduce_2pi(s * zx);
#else
  return act_sel<ACT>(act) == 0 ? tanhf(s * zx) : zx;
#endif
}
// Scaled derivatives of the activation at u = s z from the stash form x:
// d0 = sigma, c1 = s sigma', p2 = s^2 sigma'', r3 = s^3 sigma^(3).  For tanh
// (x = t) they are polynomials in t: sigma' = 1 - t^2 =: a, sigma'' = -2 t a,
// sigma^(3) = a (6 t^2 - 2) = a (4 - 6 a).
template <int ACT>
__device__ __forceinline__ void scaled_derivs(float x, float s, float& d0, float& c1, float& p2, float& r3,
                                              int act = ACT) {
  if (act_sel<ACT>(act) == 0) {
    const float a = fmaf(-x, x, 1.0f);
    d0 = x;
    c1 = s * a;
    p2 = (x * a) * (-2.0f * s * s);
    r3 = (a * (s * s * s)) * fmaf(-6.0f, a, 4.0f);
  } else {
    float s0, s1, s2, s3;
#if PINN_MUFU_SINCOS
    // x = r, the reduced angle (stash_x)
    const float sn = __sinf(x), cs = __cosf(x);
    if (act_sel<ACT>(act) == 1) {
      s0 = sn; s1 = cs; s2 = -sn; s3 = -cs;
    } else {
      s0 = cs; s1 = -sn; s2 = -cs; s3 = sn;
    }
#else
    act_derivs<ACT>(s * x, s0, s1, s2, s3, act);
#endif
    d0 = s0;
    c1 = s * s1;
    p2 = (s * s) * s2;
    r3 = (s * s * s) * s3;
  }
}

// forward jet map of one neuron from its stash form (x, g1, g2, L):
// h = (sigma, sigma' s g1, sigma' s g2, sigma'' s^2 Q + sigma' s L)
template <int ACT>
__device__ __forceinline__ float4 act_fwd(float4 z, float s, float m1, float m2, int act = ACT) {
  float d0, c1, p2, r3;
  scaled_derivs<ACT>(z.x, s, d0, c1, p2, r3, act);
  const float Q = fmaf(m2 * z.z, z.z, (m1 * z.y) * z.y);
  return make_float4(d0, c1 * z.y, c1 * z.z, fmaf(p2, Q, c1 * z.w));
}

// adjoint of act_fwd: given hb = dJ/dh (4 channels) and the stash form of the
// pre-activation jets, return zb = dJ/dz (4 channels).  The slope gradient is
// NOT accumulated here: J depends on (s_k, W^k, b^k) only through s_k W^k and
// s_k b^k, so a_k dJ/da_k = <W^k, dJ/dW^k> + <b^k, dJ/db^k> exactly; K5
// evaluates that identity once per step.
//   zb  = s sigma' hb_v + s^2 sigma'' (hb_1 g1 + hb_2 g2) + hb_L (s^3 sigma^(3) Q + s^2 sigma'' L)
//   g1b = s sigma' hb_1 + 2 m1 hb_L s^2 sigma'' g1   (g2b likewise),   Lb = s sigma' hb_L
template <int ACT>
__device__ __forceinline__ float4 act_bwd(float4 z, float4 hb, float s, float m1, float m2, int act = ACT) {
  float d0, c1, p2, r3;
  scaled_derivs<ACT>(z.x, s, d0, c1, p2, r3, act);
  const float Q = fmaf(m2 * z.z, z.z, (m1 * z.y) * z.y);
  const float A = hb.w * p2;
  const float zb = fmaf(c1, hb.x, fmaf(p2, fmaf(hb.z, z.z, hb.y * z.y), fmaf(A, z.w, hb.w * (r3 * Q))));
  const float g1 = fmaf(c1, hb.y, (A * (2.0f * m1)) * z.y);
  const float g2 = fmaf(c1, hb.z, (A * (2.0f * m2)) * z.z);
  return make_float4(zb, g1, g2, c1 * hb.w);
}

// ----------------------------------------------------------------------------
// TMEM stash: each thread keeps its own pre-activation jets of every hidden
// layer in its TMEM lane (warp w owns lanes 32w..32w+31; 512 columns).
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int COLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(slot)), "n"(COLS));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}
template <int COLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "n"(COLS));
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// load 8 columns and wait in the same asm block so the values are valid on exit
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// Stash policy: TMEM (default) or a per-CTA global scratch (debug fallback).
// Thread tid owns TMEM lane 32*(warp%4) + lane, columns [256*(warp/4), +256).
struct Stash {
  uint32_t taddr;     // TMEM address of this thread's column block
  float* g;           // global fallback base for this CTA (or nullptr)
  int tid;
  int nthr;           // threads per CTA (global fallback stride)
  __device__ __forceinline__ void store(int slot, const float* v) {
    if (g == nullptr) {
      __syncwarp();   // tcgen05.st is .sync.aligned: the warp must be converged
#pragma unroll
      for (int q = 0; q < kA / 8; ++q) tmem_st8(taddr + slot * kA + q * 8, v + q * 8);
      tmem_wait_st();
    } else {
#pragma unroll
      for (int a = 0; a < kA; ++a) g[(size_t(slot) * kA + a) * nthr + tid] = v[a];
    }
  }
  __device__ __forceinline__ void load(int slot, float* v) {
    if (g == nullptr) {
      __syncwarp();   // tcgen05.ld is .sync.aligned
#pragma unroll
      for (int q = 0; q < kA / 8; ++q) tmem_ld8(taddr + slot * kA + q * 8, v + q * 8);
    } else {
#pragma unroll
      for (int a = 0; a < kA; ++a) v[a] = g[(size_t(slot) * kA + a) * nthr + tid];
    }
  }
};

// ----------------------------------------------------------------------------
// pointwise operators.  U[o] = (u, d1 u, d2 u, Delta_S u) of output o.
// r[e] and dr[e][o][c] = d r_e / d U[o].c
// ----------------------------------------------------------------------------
constexpr int PDE_BURGERS = 0, PDE_POISSON = 1, PDE_HEAT = 2, PDE_NS = 3, PDE_HEAT_INV = 4;

struct PdeConst {
  int pde;
  float nu, re;
};

__device__ __forceinline__ void heat_K(float x, float y, float& K, float& Kx, float& Ky) {
  float e = __expf(0.1f * y);
  float sn, cs;
  sincosf(0.5f * x, &sn, &cs);
  K = 20.0f + e * sn;
  Kx = 0.5f * e * cs;
  Ky = 0.1f * e * sn;
}

// residual F := L_x(u) - f
template <int DO>
__device__ __forceinline__ int pde_residual(const PdeConst& pc, const float4* U, float x, float y, float* r,
                                            float (*dr)[DO][4]) {
#pragma unroll
  for (int e = 0; e < 3; ++e)
#pragma unroll
    for (int o = 0; o < DO; ++o) dr[e][o][0] = dr[e][o][1] = dr[e][o][2] = dr[e][o][3] = 0.0f;
  if (pc.pde == PDE_BURGERS) {
    // u_t + u u_x - nu u_xx; channels (u, u_x, u_t, u_xx)
    const float4 u = U[0];
    r[0] = u.z + u.x * u.y - pc.nu * u.w;
    dr[0][0][0] = u.y; dr[0][0][1] = u.x; dr[0][0][2] = 1.0f; dr[0][0][3] = -pc.nu;
    return 1;
  } else if (pc.pde == PDE_POISSON) {
    // Delta u - f, f = -2 pi^2 sin(pi x) sin(pi y) (reading Z15)
    const float4 u = U[0];
    const float PI = 3.14159265358979323846f;
    float f = -2.0f * PI * PI * sinpif(x) * sinpif(y);
    r[0] = u.w - f;
    dr[0][0][3] = 1.0f;
    return 1;
  } else if (pc.pde == PDE_HEAT) {
    // d_x(K u_x) + d_y(K u_y) - f, f = 4 exp(-0.1 y)
    const float4 u = U[0];
    float K, Kx, Ky;
    heat_K(x, y, K, Kx, Ky);
    float f = 4.0f * __expf(-0.1f * y);
    r[0] = K * u.w + Kx * u.y + Ky * u.z - f;
    dr[0][0][1] = Kx; dr[0][0][2] = Ky; dr[0][0][3] = K;
    return 1;
  } else if (pc.pde == PDE_HEAT_INV) {
    // inverse heat (K unknown): outputs (T, K) of one net,
    // F = K Delta T + K_x T_x + K_y T_y - f, f = 4 exp(-0.1 y) (reading Z17b)
    if constexpr (DO == 2) {
      const float4 T = U[0], K = U[1];
      const float f = 4.0f * __expf(-0.1f * y);
      r[0] = K.x * T.w + K.y * T.y + K.z * T.z - f;
      dr[0][0][1] = K.y; dr[0][0][2] = K.z; dr[0][0][3] = K.x;
      dr[0][1][0] = T.w; dr[0][1][1] = T.y; dr[0][1][2] = T.z;
    }
    return 1;
  } else {
    // steady incompressible NS, outputs (u, v, p)
    if constexpr (DO == 3) {
      const float4 u = U[0], v = U[1], p = U[2];
      const float ir = 1.0f / pc.re;
      r[0] = u.x * u.y + v.x * u.z + p.y - u.w * ir;
      r[1] = u.x * v.y + v.x * v.z + p.z - v.w * ir;
      r[2] = u.y + v.z;
      dr[0][0][0] = u.y; dr[0][0][1] = u.x; dr[0][0][2] = v.x; dr[0][0][3] = -ir;
      dr[0][1][0] = u.z; dr[0][2][1] = 1.0f;
      dr[1][0][0] = v.y; dr[1][1][0] = v.z; dr[1][1][1] = u.x; dr[1][1][2] = v.x; dr[1][1][3] = -ir;
      dr[1][2][2] = 1.0f;
      dr[2][0][1] = 1.0f; dr[2][1][2] = 1.0f;
    }
    return 3;
  }
}

// normal flux f(u).n of the conservation form (cPINN; Table 1)
template <int DO>
__device__ __forceinline__ int pde_flux(const PdeConst& pc, const float4* U, float x, float y, float n1, float n2,
                                        float* r, float (*dr)[DO][4]) {
#pragma unroll
  for (int e = 0; e < 3; ++e)
#pragma unroll
    for (int o = 0; o < DO; ++o) dr[e][o][0] = dr[e][o][1] = dr[e][o][2] = dr[e][o][3] = 0.0f;
  if (pc.pde == PDE_BURGERS) {
    // space-time flux (u^2/2 - nu u_x, u) . n (reading Z13)
    const float4 u = U[0];
    r[0] = (0.5f * u.x * u.x - pc.nu * u.y) * n1 + u.x * n2;
    dr[0][0][0] = u.x * n1 + n2;
    dr[0][0][1] = -pc.nu * n1;
    return 1;
  } else if (pc.pde == PDE_POISSON || pc.pde == PDE_HEAT) {
    const float4 u = U[0];
    float K = 1.0f, Kx, Ky;
    if (pc.pde == PDE_HEAT) heat_K(x, y, K, Kx, Ky);
    r[0] = K * (u.y * n1 + u.z * n2);
    dr[0][0][1] = K * n1;
    dr[0][0][2] = K * n2;
    return 1;
  } else if (pc.pde == PDE_HEAT_INV) {
    // K grad T . n with K the net's second output
    if constexpr (DO == 2) {
      const float4 T = U[0], K = U[1];
      const float gn = T.y * n1 + T.z * n2;
      r[0] = K.x * gn;
      dr[0][0][1] = K.x * n1; dr[0][0][2] = K.x * n2;
      dr[0][1][0] = gn;
    }
    return 1;
  } else {
    if constexpr (DO == 3) {
      const float4 u = U[0], v = U[1], p = U[2];
      const float ir = 1.0f / pc.re;
      r[0] = (u.x * u.x + p.x - u.y * ir) * n1 + (u.x * v.x - u.z * ir) * n2;
      r[1] = (u.x * v.x - v.y * ir) * n1 + (v.x * v.x + p.x - v.z * ir) * n2;
      r[2] = u.x * n1 + v.x * n2;
      dr[0][0][0] = 2.0f * u.x * n1 + v.x * n2; dr[0][1][0] = u.x * n2; dr[0][2][0] = n1;
      dr[0][0][1] = -ir * n1; dr[0][0][2] = -ir * n2;
      dr[1][0][0] = v.x * n1; dr[1][1][0] = u.x * n1 + 2.0f * v.x * n2; dr[1][2][0] = n2;
      dr[1][1][1] = -ir * n1; dr[1][1][2] = -ir * n2;
      dr[2][0][0] = n1; dr[2][1][0] = n2;
    }
    return 3;
  }
}

// ----------------------------------------------------------------------------
// kernel argument block
// ----------------------------------------------------------------------------
struct Chunk {
  int32_t sub;     // local subdomain
  int32_t start;   // first point
  int32_t count;   // points (<= tiles_per_chunk * P)
  int32_t pad;
};

__device__ __forceinline__ int ld_acquire_gpu(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Peer-store exchange of the fused step (PINN_DD_FLAG_PEER_STORES, Algorithm 1
// green stage inside the launch): payload chunks store the rows of
// cut edges straight into the neighbour GPU's receive slot (CUDA-IPC-mapped,
// over NVLink) and release-add the row count to its arrival counter; interface
// loss chunks acquire-wait for every peer's rows of this step.  Receive slots
// alternate by step parity (a neighbour can be one step ahead of our reads).
constexpr int kMaxPeers = 8;
struct PeerX {
  int n;                                      // peers (0: off)
  int64_t send_off[kMaxPeers + 1];            // send-slot ranges of the peers (psend indices)
  float* dst[kMaxPeers];                      // peer's receive slot 0, first row of ours
  int64_t slot_stride[kMaxPeers];             // floats from the peer's slot 0 to its slot 1
  unsigned long long* peer_flag[kMaxPeers];   // peer's arrival counter for our rows
  const unsigned long long* my_flag;          // [n] arrivals here, per peer (cumulative)
  int64_t expect[kMaxPeers];                  // rows per step from each peer
  int64_t n_recv;                             // rows of one receive slot here
  int* step;                                  // steps completed (parity, expected arrivals)
};

__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}

struct KArgs {
  const float* coords;      // [2][n_points]
  const float* target;      // [DO][n_points]
  const float* mask;        // [DO][n_points]
  const int32_t* pinfo;     // kind (bits 0-1: 0 residual, 1 data, 2 interface) | flux (bit 2) | seg << 3
  const float* pinv;        // 1 / N of the point's class (per edge for interface points)
  const int32_t* ptwin;     // payload row of the twin (interface points)
  const float2* seg_normal; // [n_seg]
  const float* params;      // internal [n_sub][PSTRIDE]
  const int32_t* sub_act;   // [n_sub] activation per subdomain (read only by kActMixed instances)
  const float4* sub_w;      // [n_sub] (w_u, w_f, w_i, w_if)
  const Chunk* chunks;
  const Chunk* chunks2;     // payload chunks (MODE 2: the fused step runs them first)
  int n_chunks2;
  const int32_t* order;     // [n_chunks] processing order (nullptr = identity)
  int32_t* sched;           // chunk counter, CTAs done (zero between launches); MODE 2: [4] payload chunks done
  // MODE 2 sticky schedule (nullptr: one global queue in `order`): per-
  // subdomain chunk queues, so that a CTA keeps its subdomain's weights in
  // shared memory until that subdomain runs out of chunks
  const int32_t* sub_chunk_off; // [n_sub + 1] each subdomain's chunks (contiguous, in claim order)
  int32_t* sub_ctr;             // [n_sub] claims (zero between launches)
  const int32_t* sub_tiles;     // [n_sub + 1] cumulative tiles (first claim of each CTA)
  int n_sub;
  int n_chunks;
  int64_t n_points;
  int pstride;              // floats per subdomain in params / partial
  float* partial;           // [n_chunks][pstride]
  float* partial_loss;      // [n_chunks][4]
  float* payload;           // [rows][NF]
  const int32_t* psend;     // [n_points] row of the point in the send buffer, -1 = not sent (nullptr: no peers)
  float* sendbuf;           // [n_send][NF] payload rows of cut edges, in the peers' receive order
  PeerX px;                 // peer-store exchange of the fused step (px.n == 0: off)
  float* gstash;            // global stash fallback (nullptr = TMEM)
  PdeConst pc;
  int method;               // 0 pinn, 1 cpinn, 2 xpinn, 3 hybrid (per-edge choice in pinfo bit 2)
  float slope_n;
  float m1, m2;             // Laplacian mask (x1 in S, x2 in S)
};

}  // namespace pinn
