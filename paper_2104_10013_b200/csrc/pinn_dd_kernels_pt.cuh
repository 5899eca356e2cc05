// pinn_dd_kernels_pt.cuh -- K1/K2 for narrow networks (width N <= 20; C1 3x20,
// C3 5x20): one thread = one collocation point with all N neurons of every
// layer in registers (jets z[c*N + j], c = value, d1, d2, Delta_S).
//
// Compared with k_fused (mapping A: a point's neurons spread over N/kJT
// threads that exchange activations through shared memory after every layer),
// here the forward pass, the output layer, the pointwise epilogue and the
// input adjoint H^{k-1}-bar = W^k^T Z^k-bar are thread-local: no shared-memory
// round trip and no CTA barrier per layer.  Only dW^k = sum_p Z^k-bar (x) H^{k-1}
// (a sum over the tile's points) goes through shared memory, with two
// alternating buffer pairs so that each layer needs a single barrier.
//
// 128 threads (4 warps), tile = 128 points; thread t owns TMEM lane t and its
// 512 columns, which hold the reverse-mode stash of all NH hidden layers
// (NH * 4N <= 512).  Same KArgs, chunk schedule, partial slots and fixed-order
// reductions as k_fused, so results do not depend on which CTA runs a chunk.
#pragma once

#include "pinn_dd_kernels.cuh"

namespace pinn {

constexpr int kPT = 128;   // threads per CTA = points per tile

template <int N, int NH, int DO>
struct PtCfg {
  static_assert(NH * 4 * N <= 512, "stash exceeds the TMEM columns of one lane");
  static_assert(N % 5 == 0 && N % 4 == 0, "width");
  static constexpr int P = kPT;
  static constexpr int PSTR = P + 1;                      // float4 row stride (odd)
  static constexpr int NN = N * N;
  static constexpr int oW1 = 0;                           // W^1 [N][2], b^1 [N]
  static constexpr int oB1 = 2 * N;
  static constexpr int oWT = al4(3 * N);                  // hidden W^T [NH-1][i][j] (forward)
  static constexpr int oW = oWT + (NH - 1) * NN;          // hidden W   [NH-1][j][i] (input adjoint)
  static constexpr int oBh = oW + (NH - 1) * NN;          // [NH-1][N]
  static constexpr int oWo = al4(oBh + (NH - 1) * N);     // [DO][N]
  static constexpr int oBo = oWo + DO * N;
  static constexpr int oSl = al4(oBo + DO);               // slopes s_k = n a^k
  static constexpr int BUF = N * PSTR * 4;                // one [N][PSTR] float4 buffer
  static constexpr int oBuf = al4(oSl + NH);              // Z-bar / H buffer pairs A, B
  static constexpr int oU = oBuf + 4 * BUF;               // [P][DO] float4 output adjoint seeds
  static constexpr int oX = oU + P * DO * 4;              // x1[P], x2[P]
  static constexpr int oRed = al4(oX + 2 * P);            // block-sum scratch [4][4]
  // dW: thread = (JB x IB block, point split); two scratch buffers (alternate layers)
  static constexpr int JB = 5, IB = 5;
  static constexpr int NJ = N / JB, NI = N / IB, NBLK = NJ * NI;
  static constexpr int S = kPT / NBLK;
  static constexpr int PS = P / S;
  static constexpr int SCR = S * NBLK * JB * IB + S * NJ * JB;
  static constexpr int oDw = oRed + 16;
  static constexpr int oAcc = al4(oDw + 2 * SCR);         // gradient accumulator of the chunk
  static constexpr int ACC = Lay<N, NH, DO>::total();
  static constexpr int TOTAL = al4(oAcc + ACC + 4);       // + TMEM address slot
  static constexpr size_t SMEM = size_t(TOTAL) * 4;
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert(NBLK * S == kPT && P % S == 0, "dW mapping");
};

template <int N, int NH, int DO>
__device__ __forceinline__ void load_weights_pt(const float* __restrict__ G, float slope_n, float* sm) {
  using C = PtCfg<N, NH, DO>;
  using LY = Lay<N, NH, DO>;
  const int tid = threadIdx.x;
  for (int e = tid; e < 3 * N; e += kPT) sm[C::oW1 + e] = G[LY::offW(1) + e];   // W^1 then b^1
#pragma unroll 1
  for (int k = 2; k <= NH; ++k) {
    const float* W = G + LY::offW(k);
    for (int e = tid; e < C::NN; e += kPT) {
      const int j = e / N, i = e - (e / N) * N;
      const float w = W[e];
      sm[C::oW + (k - 2) * C::NN + e] = w;
      sm[C::oWT + (k - 2) * C::NN + i * N + j] = w;
    }
    for (int e = tid; e < N; e += kPT) sm[C::oBh + (k - 2) * N + e] = G[LY::offB(k) + e];
  }
  for (int e = tid; e < DO * N; e += kPT) sm[C::oWo + e] = G[LY::offW(NH + 1) + e];
  for (int e = tid; e < DO; e += kPT) sm[C::oBo + e] = G[LY::offB(NH + 1) + e];
  for (int e = tid; e < NH; e += kPT) sm[C::oSl + e] = slope_n * G[LY::offA(e + 1)];
}

// block-wide sum over the 4 warps of a kPT CTA; result valid in thread 0
__device__ __forceinline__ void pt_block_sum4(float* v, float* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    float x = v[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    v[r] = x;
  }
  if (lane == 0) {
#pragma unroll
    for (int r = 0; r < 4; ++r) red[w * 4 + r] = v[r];
  }
  cta_sync();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int r = 0; r < 4; ++r) v[r] = red[r] + red[4 + r] + red[8 + r] + red[12 + r];
  }
}

// dW^k, db^k partials of one layer from the buffer pair (Zb, H) into scratch
template <int N, int NH, int DO>
__device__ __forceinline__ void pt_dw_partial(const float4* __restrict__ Zb, const float4* __restrict__ H,
                                              float* scr) {
  using C = PtCfg<N, NH, DO>;
  constexpr int JB = C::JB, IB = C::IB, NJ = C::NJ, NI = C::NI, NBLK = C::NBLK, PS = C::PS;
  constexpr int DBOFF = C::S * NBLK * JB * IB;
  const int tid = threadIdx.x;
  const int r = tid % NBLK, s = tid / NBLK;
  const int jb = r % NJ, ib = r / NJ;
  float acc[JB][IB];
  float db[JB];
#pragma unroll
  for (int jj = 0; jj < JB; ++jj) {
    db[jj] = 0.0f;
#pragma unroll
    for (int ii = 0; ii < IB; ++ii) acc[jj][ii] = 0.0f;
  }
#pragma unroll 4
  for (int p = s * PS; p < (s + 1) * PS; ++p) {
    float4 zr[JB], hr[IB];
#pragma unroll
    for (int jj = 0; jj < JB; ++jj) zr[jj] = Zb[(jb + NJ * jj) * C::PSTR + p];
#pragma unroll
    for (int ii = 0; ii < IB; ++ii) hr[ii] = H[(ib + NI * ii) * C::PSTR + p];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int jj = 0; jj < JB; ++jj)
#pragma unroll
        for (int ii = 0; ii < IB; ++ii) acc[jj][ii] = fmaf(comp(zr[jj], m), comp(hr[ii], m), acc[jj][ii]);
#pragma unroll
    for (int jj = 0; jj < JB; ++jj) db[jj] += zr[jj].x;
  }
#pragma unroll
  for (int jj = 0; jj < JB; ++jj)
#pragma unroll
    for (int ii = 0; ii < IB; ++ii) scr[(s * NBLK + r) * JB * IB + jj * IB + ii] = acc[jj][ii];
  if (ib == 0) {
#pragma unroll
    for (int jj = 0; jj < JB; ++jj) scr[DBOFF + (s * NJ + jb) * JB + jj] = db[jj];
  }
}

// fixed-order sum of the S point-split partials into the accumulator
template <int N, int NH, int DO>
__device__ __forceinline__ void pt_dw_reduce(const float* scr, float* accW, float* accB) {
  using C = PtCfg<N, NH, DO>;
  constexpr int JB = C::JB, IB = C::IB, NJ = C::NJ, NI = C::NI, NBLK = C::NBLK, S = C::S;
  constexpr int DBOFF = S * NBLK * JB * IB;
  const int tid = threadIdx.x;
  for (int e = tid; e < NBLK * JB; e += kPT) {
    const int r = e / JB, jj = e - (e / JB) * JB;
    const int jb = r % NJ, ib = r / NJ;
    const float* src = scr + r * JB * IB + jj * IB;
    float v[IB];
#pragma unroll
    for (int ii = 0; ii < IB; ++ii) v[ii] = src[ii];
#pragma unroll
    for (int s = 1; s < S; ++s)
#pragma unroll
      for (int ii = 0; ii < IB; ++ii) v[ii] += src[s * NBLK * JB * IB + ii];
#pragma unroll
    for (int ii = 0; ii < IB; ++ii) accW[(jb + NJ * jj) * N + ib + NI * ii] += v[ii];
  }
  for (int e = tid; e < NJ * JB; e += kPT) {
    const int jb = e / JB, jj = e % JB;
    float v = 0.0f;
#pragma unroll
    for (int s = 0; s < S; ++s) v += scr[DBOFF + (s * NJ + jb) * JB + jj];
    accB[jb + NJ * jj] += v;
  }
}

template <int N, int NH, int DO, int ACT, int MODE>
__global__ void __launch_bounds__(kPT, 1) k_fused_pt(const KArgs a) {
  using C = PtCfg<N, NH, DO>;
  using LY = Lay<N, NH, DO>;
  constexpr int J4 = 4 * N;   // jets of one layer per point
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x;
  const float* sW1 = sm + C::oW1;
  const float* sB1 = sm + C::oB1;
  const float* sSl = sm + C::oSl;
  float4* bufs = reinterpret_cast<float4*>(sm + C::oBuf);   // pair A: [0] Z-bar, [1] H; pair B: [2], [3]
  float4* sU = reinterpret_cast<float4*>(sm + C::oU);
  float* sX = sm + C::oX;
  float* sY = sX + C::P;
  float* sRed = sm + C::oRed;
  float* sAcc = sm + C::oAcc;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + C::TOTAL - 4);
  const float m1 = a.m1, m2 = a.m2;

  uint32_t taddr = 0;
  float* gst = nullptr;
  if constexpr (MODE == 0) {
    if (a.gstash == nullptr) {
      if (tid < 32) {
        __syncwarp();
        tmem_alloc<512>(tslot);
      }
      tmem_fence_before();
      cta_sync();
      tmem_fence_after();
      taddr = *tslot + (uint32_t((tid >> 5) * 32) << 16);
    } else {
      gst = a.gstash + size_t(blockIdx.x) * NH * J4 * kPT;
    }
  }
  // stash of hidden layer slot+1: column slot*4N + 4j + c (neuron-major, so one
  // 8-column access holds the four jets of neurons 2q and 2q+1)
  auto stash_store = [&](int slot, const float* z) {   // z in registers as z[c*N + j]
    if (gst == nullptr) __syncwarp();
#pragma unroll
    for (int q = 0; q < N / 2; ++q) {
      float v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = z[(e & 3) * N + 2 * q + (e >> 2)];
      if (gst == nullptr) {
        tmem_st8(taddr + slot * J4 + q * 8, v);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) gst[(size_t(slot) * J4 + q * 8 + e) * kPT + tid] = v[e];
      }
    }
    if (gst == nullptr) tmem_wait_st();
  };
  auto stash_load8 = [&](int slot, int q, float* v) {   // neurons 2q, 2q+1
    if (gst == nullptr) {
      tmem_ld8(taddr + slot * J4 + q * 8, v);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = gst[(size_t(slot) * J4 + q * 8 + e) * kPT + tid];
    }
  };

  __shared__ int s_next;
  int cur_sub = -1;
#pragma unroll 1
  for (;;) {
    if (tid == 0) s_next = atomicAdd(a.sched, 1);
    cta_sync();
    const int idx = s_next;
    if (idx >= a.n_chunks) break;
    const int c = a.order ? a.order[idx] : idx;
    const Chunk ch = a.chunks[c];
    if (ch.sub != cur_sub) {
      cta_sync();
      load_weights_pt<N, NH, DO>(a.params + size_t(ch.sub) * a.pstride, a.slope_n, sm);
      cur_sub = ch.sub;
    }
    const float4 lw = a.sub_w[ch.sub];
    const int act = ACT == kActMixed ? a.sub_act[ch.sub] : ACT;
    float* Pc = a.partial + size_t(c) * a.pstride;
    if constexpr (MODE == 0) {
      cta_sync();
      for (int e = tid; e < C::ACC; e += kPT) sAcc[e] = 0.0f;
    }
    const int ntiles = (ch.count + C::P - 1) / C::P;
    if constexpr (MODE == 0) {
      if (ntiles == 0 && tid < 4) a.partial_loss[size_t(c) * 4 + tid] = 0.0f;
    }
#pragma unroll 1
    for (int t = 0; t < ntiles; ++t) {
      const int64_t p0 = int64_t(ch.start) + int64_t(t) * C::P;
      const int np = min(C::P, ch.count - t * C::P);
      const bool first = (t == 0);
      const bool valid = tid < np;
      float x = 0.0f, y = 0.0f;
      if (valid) {
        x = a.coords[p0 + tid];
        y = a.coords[a.n_points + p0 + tid];
      }
      cta_sync();   // the previous tile's readers of sX / buffers are done (and weights are visible)
      sX[tid] = x;
      sY[tid] = y;

      // ------------------------------------------------ forward (thread-local)
      // this thread's activations live in column `tid` of the pair-B H buffer
      // (thread-private until the reverse pass), so the GEMM loops index them
      // at run time without spilling a register array
      float4* HF = bufs + 3 * N * C::PSTR;
      {
        float z[J4];
#pragma unroll
        for (int j = 0; j < N; ++j) {
          const float w0 = sW1[2 * j], w1 = sW1[2 * j + 1];
          z[j] = fmaf(w0, x, fmaf(w1, y, sB1[j]));   // z = W^1 x + b^1
          z[N + j] = w0;
          z[2 * N + j] = w1;
          z[3 * N + j] = 0.0f;
        }
        const float s = sSl[0];
#pragma unroll
        for (int j = 0; j < N; ++j) z[j] = stash_x<ACT>(z[j], s, act);
        if constexpr (MODE == 0) stash_store(0, z);
#pragma unroll
        for (int j = 0; j < N; ++j)
          HF[j * C::PSTR + tid] =
              act_fwd<ACT>(make_float4(z[j], z[N + j], z[2 * N + j], z[3 * N + j]), s, m1, m2, act);
      }
#pragma unroll 1
      for (int k = 2; k <= NH; ++k) {
        const float* WT = sm + C::oWT + (k - 2) * C::NN;
        const float* bk = sm + C::oBh + (k - 2) * N;
        float z[J4];
#pragma unroll
        for (int j = 0; j < N; ++j) {
          z[j] = bk[j];
          z[N + j] = 0.0f;
          z[2 * N + j] = 0.0f;
          z[3 * N + j] = 0.0f;
        }
#pragma unroll 2
        for (int i = 0; i < N; ++i) {
          float w[N];
#pragma unroll
          for (int q = 0; q < N / 4; ++q) {
            const float4 v = *reinterpret_cast<const float4*>(WT + i * N + 4 * q);
            w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
          }
          const float4 hv = HF[i * C::PSTR + tid];
#pragma unroll
          for (int j = 0; j < N; ++j) {
            z[j] = fmaf(w[j], hv.x, z[j]);
            z[N + j] = fmaf(w[j], hv.y, z[N + j]);
            z[2 * N + j] = fmaf(w[j], hv.z, z[2 * N + j]);
            z[3 * N + j] = fmaf(w[j], hv.w, z[3 * N + j]);
          }
        }
        const float s = sSl[k - 1];
#pragma unroll
        for (int j = 0; j < N; ++j) z[j] = stash_x<ACT>(z[j], s, act);
        if constexpr (MODE == 0) stash_store(k - 1, z);
#pragma unroll
        for (int j = 0; j < N; ++j)
          HF[j * C::PSTR + tid] =
              act_fwd<ACT>(make_float4(z[j], z[N + j], z[2 * N + j], z[3 * N + j]), s, m1, m2, act);
      }
      // output layer jets U[o] = W^L H + b^L
      float4 U[DO];
#pragma unroll
      for (int o = 0; o < DO; ++o) {
        const float* w = sm + C::oWo + o * N;
        float4 u = make_float4(sm[C::oBo + o], 0.0f, 0.0f, 0.0f);
#pragma unroll 4
        for (int i = 0; i < N; ++i) {
          const float wi = w[i];
          const float4 hv = HF[i * C::PSTR + tid];
          u.x = fmaf(wi, hv.x, u.x);
          u.y = fmaf(wi, hv.y, u.y);
          u.z = fmaf(wi, hv.z, u.z);
          u.w = fmaf(wi, hv.w, u.w);
        }
        U[o] = u;
      }

      if constexpr (MODE == 1) {
        if (valid) point_payload<DO>(a, p0 + tid, x, y, U);
        continue;
      } else {
        // ---------------------------------------------- epilogue (thread-local)
        float lsum[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        float4 Ub[DO];
#pragma unroll
        for (int o = 0; o < DO; ++o) Ub[o] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if (valid) point_adjoint<DO>(a, p0 + tid, x, y, lw, U, Ub, lsum);

        // ----------------------------------------------------------- reverse
        // output layer: dW^L / db^L need H^{NH} (already in HB) and Ub of all points
        float4* ZA = bufs;
        float4* HA = bufs + N * C::PSTR;
        float4* ZB = bufs + 2 * N * C::PSTR;
        float4* HB = HF;
#pragma unroll
        for (int o = 0; o < DO; ++o) sU[tid * DO + o] = Ub[o];
        // adjoint of H^{NH}: hb = W^L^T Ub, then of Z^{NH}
        float hb[J4];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
          for (int o = 0; o < DO; ++o) {
            const float w = sm[C::oWo + o * N + i];
            v.x = fmaf(Ub[o].x, w, v.x);
            v.y = fmaf(Ub[o].y, w, v.y);
            v.z = fmaf(Ub[o].z, w, v.z);
            v.w = fmaf(Ub[o].w, w, v.w);
          }
          hb[i] = v.x; hb[N + i] = v.y; hb[2 * N + i] = v.z; hb[3 * N + i] = v.w;
        }
        {
          const float s = sSl[NH - 1];
          if (gst == nullptr) __syncwarp();
#pragma unroll
          for (int q = 0; q < N / 2; ++q) {
            float v[8];
            stash_load8(NH - 1, q, v);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int j = 2 * q + u;
              const float4 o = act_bwd<ACT>(make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]),
                                            make_float4(hb[j], hb[N + j], hb[2 * N + j], hb[3 * N + j]), s, m1,
                                            m2, act);
              hb[j] = o.x; hb[N + j] = o.y; hb[2 * N + j] = o.z; hb[3 * N + j] = o.w;
            }
          }
        }
        cta_sync();   // HB (H^{NH}) and sU complete
        for (int t4 = tid; t4 < 4 * DO * N; t4 += kPT) {   // warp-uniform trip count
          const int qq = t4 & 3, id = t4 >> 2;
          const int o = id / N, i = id % N;
          float acc = 0.0f;
#pragma unroll 4
          for (int p = qq; p < C::P; p += 4) {
            const float4 hh = HB[i * C::PSTR + p];
            const float4 ub = sU[p * DO + o];
            acc = fmaf(hh.x, ub.x, fmaf(hh.y, ub.y, fmaf(hh.z, ub.z, fmaf(hh.w, ub.w, acc))));
          }
          acc += __shfl_xor_sync(__activemask(), acc, 1);
          acc += __shfl_xor_sync(__activemask(), acc, 2);
          if (qq == 0) sAcc[LY::offW(NH + 1) + id] += acc;
        }
        if (tid < DO) {
          float acc = 0.0f;
          for (int p = 0; p < C::P; ++p) acc += sU[p * DO + tid].x;
          sAcc[LY::offB(NH + 1) + tid] += acc;
        }
        // hidden layers k = NH .. 2: hb holds Z^k-bar of this point
#pragma unroll 1
        for (int k = NH; k >= 2; --k) {
          const bool pairB = ((NH - k) & 1) == 1;   // layer NH uses pair A (HB held H^{NH})
          float4* Zb = pairB ? ZB : ZA;
          float4* Hb = pairB ? HB : HA;
          float* scr = sm + C::oDw + ((NH - k) & 1) * C::SCR;
          {
            // Z^k-bar and H^{k-1} (recomputed from the stash of layer k-1, slot k-2)
            const float s1 = sSl[k - 2];
            if (gst == nullptr) __syncwarp();
#pragma unroll
            for (int q = 0; q < N / 2; ++q) {
              float v[8];
              stash_load8(k - 2, q, v);
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                const int j = 2 * q + u;
                Zb[j * C::PSTR + tid] = make_float4(hb[j], hb[N + j], hb[2 * N + j], hb[3 * N + j]);
                Hb[j * C::PSTR + tid] =
                    act_fwd<ACT>(make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]), s1, m1, m2, act);
              }
            }
          }
          cta_sync();   // this layer's pair is complete; the previous layer's dW scratch too
          if (k < NH) {
            float* prev = sm + C::oDw + ((NH - k - 1) & 1) * C::SCR;
            pt_dw_reduce<N, NH, DO>(prev, sAcc + LY::offW(k + 1), sAcc + LY::offB(k + 1));
          }
          pt_dw_partial<N, NH, DO>(Zb, Hb, scr);
          // input adjoint hb' = W^k^T Z^k-bar (thread-local), then through layer k-1
          const float* W = sm + C::oW + (k - 2) * C::NN;
          float hn[J4];
#pragma unroll
          for (int e = 0; e < J4; ++e) hn[e] = 0.0f;
#pragma unroll 2
          for (int j = 0; j < N; ++j) {
            float w[N];
#pragma unroll
            for (int q = 0; q < N / 4; ++q) {
              const float4 v = *reinterpret_cast<const float4*>(W + j * N + 4 * q);
              w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
            }
            const float4 zb = Zb[j * C::PSTR + tid];   // this thread's own Z^k-bar row
#pragma unroll
            for (int i = 0; i < N; ++i) {
              hn[i] = fmaf(w[i], zb.x, hn[i]);
              hn[N + i] = fmaf(w[i], zb.y, hn[N + i]);
              hn[2 * N + i] = fmaf(w[i], zb.z, hn[2 * N + i]);
              hn[3 * N + i] = fmaf(w[i], zb.w, hn[3 * N + i]);
            }
          }
          const float s = sSl[k - 2];
          if (gst == nullptr) __syncwarp();
#pragma unroll
          for (int q = 0; q < N / 2; ++q) {
            float v[8];
            stash_load8(k - 2, q, v);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int j = 2 * q + u;
              const float4 o = act_bwd<ACT>(make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]),
                                            make_float4(hn[j], hn[N + j], hn[2 * N + j], hn[3 * N + j]), s, m1,
                                            m2, act);
              hb[j] = o.x; hb[N + j] = o.y; hb[2 * N + j] = o.z; hb[3 * N + j] = o.w;
            }
          }
        }
        // layer 1: dW^1[j] = sum_p zb_v x_p + zb_{d_i}; db^1 = sum_p zb_v  (Z^1-bar of every point)
        float4* Z1 = ((NH - 1) & 1) == 1 ? ZB : ZA;   // the pair not used by layer 2
#pragma unroll
        for (int j = 0; j < N; ++j) Z1[j * C::PSTR + tid] = make_float4(hb[j], hb[N + j], hb[2 * N + j], hb[3 * N + j]);
        cta_sync();
        if (NH >= 2) {
          float* prev = sm + C::oDw + ((NH - 2) & 1) * C::SCR;
          pt_dw_reduce<N, NH, DO>(prev, sAcc + LY::offW(2), sAcc + LY::offB(2));
        }
        for (int t4 = tid; t4 < 4 * N; t4 += kPT) {
          const int qq = t4 & 3, j = t4 >> 2;
          float a0 = 0.0f, a1 = 0.0f, ab = 0.0f;
#pragma unroll 4
          for (int p = qq; p < C::P; p += 4) {
            const float4 zb = Z1[j * C::PSTR + p];
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
            sAcc[LY::offW(1) + 2 * j] += a0;
            sAcc[LY::offW(1) + 2 * j + 1] += a1;
            sAcc[LY::offB(1) + j] += ab;
          }
        }
        // loss partials of the tile
        pt_block_sum4(lsum, sRed);
        if (tid == 0) {
#pragma unroll
          for (int r = 0; r < 4; ++r) rmw_store(a.partial_loss + size_t(c) * 4 + r, lsum[r], first);
        }
      }
    }
    if constexpr (MODE == 0) {
      cta_sync();
      for (int e = tid; e < C::ACC; e += kPT) Pc[e] = sAcc[e];
    }
    cta_sync();   // every thread has read s_next before it is overwritten
  }
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(a.sched + 1, 1) == int(gridDim.x) - 1) {
      a.sched[0] = 0;
      a.sched[1] = 0;
      __threadfence();
    }
  }
  if constexpr (MODE == 0) {
    if (a.gstash == nullptr) {
      cta_sync();
      tmem_fence_after();
      if (tid < 32) {
        __syncwarp();
        tmem_dealloc<512>(*tslot);
      }
    }
  }
}

}  // namespace pinn
