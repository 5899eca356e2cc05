// pinn_dd_kernels_tc.cuh -- K1 / K2 for width-80 networks with the hidden-layer
// contractions on the 5th-generation tensor cores (tcgen05.mma kind::tf32,
// accumulators in TMEM): SURVEY 8(f) row f2, DESIGN.md 11.  Selected with
// PINN_DD_FLAG_TF32; the FP32 CUDA-core kernel (pinn_dd_kernels.cuh) stays the
// default.  P:n = PAPER.md line n.
//
// Tile = 32 points x 4 jet channels = 128 rows m (the MMA's M):
//   m = 32 q + 8 c + p'   (lane quarter q = point / 8, channel c, p' = point % 8)
// so that tcgen05.ld.16x256b at lane bases 0 and 16 of a quarter hands thread
// t of the quarter's warp all four channels of point 8q + t/4, for the two
// columns 2 (t % 4) + {0, 1} of every 8-column block.  Warps w
// and w + 4 share quarter w % 4 and split the 80 neurons 40 / 40, so a thread
// owns (one point, 10 neurons) exactly like the CUDA-core kernel.
//
// Per hidden layer k (Eq. 2; forward Taylor jets):
//   forward   Z^k[m][j]  = sum_i H^{k-1}[m][i] W^k[j][i] (+ b^k via a ones column)
//   adjoint   Hb^{k-1}[m][i] = sum_j Zb^k[m][j] W^k[j][i]
//   weights   dW^k[j][i] = sum_m Zb^k[m][j] H^{k-1}[m][i] (db^k = the ones column)
// Every operand lives in shared memory ONCE, in the SWIZZLE_128B_BASE32B
// arrangement (atoms of 4 rows x 32 floats, 32-B granule ^= row % 4): the same
// bytes are a K-major operand (rows = M/N, K contiguous) and an MN-major one
// (rows = K, M/N contiguous) -- measured on the B200 (tools/tc_probe3.cu,
// profiles/r02_tc_probe3.log).  H^{k-1} [m][i] and Zb^k [m][j] are written by
// the CUDA-core epilogues (activation maps, tf32-rounded); W^k [j][i] with
// b^k in column 80 is loaded once per subdomain.
//
// TMEM (512 columns): R = [0, 80) input adjoint; S_k = [80 k, 80 k + 80) the
// pre-activation jets of layer k (the forward MMA's accumulator, rewritten in
// stash form: t = tanh(s z) for tanh), k = 1..NH; the accumulator of
// dW^k^T (96 lanes x 80 columns) reuses S_k after the
// reverse sweep has read it.  dW^k is computed transposed (lanes = inputs i,
// columns = neurons j), so adding it into the chunk's gradient partial is a
// coalesced stream of fire-and-forget reductions (one per entry per tile).
//
// Precision: single-pass TF32 products (10-bit mantissa, FP32 accumulate);
// activations, loss, adjoint seeds and every reduction stay FP32.  The looser
// tolerance is stated in DESIGN.md 6 (north star: "the looser bound stated
// numerically if TF32/BF16 tensor-core layers are used").
#pragma once

#include "pinn_dd_kernels.cuh"

namespace pinn {

namespace tc {

constexpr int N = 80;        // width
constexpr int P = 32;        // points per tile
constexpr int M = 128;       // MMA rows = P x 4 channels
constexpr int T = 256;       // threads per CTA
constexpr int CP = 96;       // padded contiguous extent of an operand row (3 atoms of 32)
constexpr int NA = CP / 32;  // atoms per 4-row group
constexpr int KF = 88;       // forward K: 80 inputs + the ones (bias) column, rounded to 8
constexpr int OPER = M * CP; // floats of an activation operand buffer
constexpr int WOPER = N * CP;   // floats of one W operand
constexpr int TCOLS = 512;   // TMEM columns allocated

// float index of element (r, c) of an operand stored in SW128_32B (rows r,
// contiguous c, NA atoms per 4-row group)
__device__ __forceinline__ int sw32(int r, int c) {
  const int b = (r & 3) * 128 + (c & 31) * 4;
  return (((r >> 2) * NA + (c >> 5)) * 512 + (b ^ (((b >> 7) & 3) << 5))) >> 2;
}

// round to the nearest tf32, ties away from zero: the value cvt.rna.tf32.f32
// gives for every finite x (half a tf32 ulp added to the sign-magnitude bits,
// a mantissa carry moves into the exponent), in two integer instructions --
// sm_100 has no native cvt.rna.tf32, its emulation took four (FSETP, SEL, LOP3,
// IADD3) per operand value.  Non-finite inputs stay non-finite.
__device__ __forceinline__ float to_tf32(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}

// shared-memory matrix descriptor (layout type 1 = SWIZZLE_128B_BASE32B)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = uint64_t(1) << 61;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;
  return d;
}
// K-major view (rows = M or N, K contiguous), k-step ks of 8 elements
__device__ __forceinline__ uint64_t kmajor(uint32_t base, int ks) {
  return sdesc(base + (ks >> 2) * 512 + (ks & 3) * 32, 512, NA * 512);
}
// MN-major view (rows = K, M or N contiguous), k-step ks of 8 rows
__device__ __forceinline__ uint64_t mnmajor(uint32_t base, int ks) {
  return sdesc(base + ks * 2 * (NA * 512), 512, NA * 512);
}
// instruction descriptor: kind::tf32, FP32 accumulate
__host__ __device__ constexpr uint32_t idesc(int m, int n, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) |
         (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// tcgen05.ld / st 16x256b.x1: lanes t/4, t/4 + 8 of the addressed 16-lane
// half, columns 2 (t % 4) + {0, 1}
__device__ __forceinline__ void ld16(uint32_t a, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a)
               : "memory");
}
__device__ __forceinline__ void st16(uint32_t a, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(a), "r"(r[0]), "r"(r[1]),
               "r"(r[2]), "r"(r[3])
               : "memory");
}
__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void ld32x16(uint32_t a, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(a)
      : "memory");
}

__device__ __forceinline__ void ld32x8(uint32_t a, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(a)
               : "memory");
}
// fire-and-forget add into the chunk partial.  Each partial entry is added to
// by one thread only (fixed thread <-> entry map, tiles of a chunk in order),
// so the adds land in program order: the sum is deterministic.
__device__ __forceinline__ void red_add(float* p, float v) {
  asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// the thread's view of a tile: point pt (0..31), quarter q, half hf, lane-in-quarter rows
struct Who {
  int q, hf, a, pp, pt;
  __device__ __forceinline__ Who(int tid) {
    const int w = tid >> 5, l = tid & 31;
    q = w & 3;
    hf = w >> 2;
    a = l & 3;
    pp = l >> 2;
    pt = 8 * q + pp;
  }
  // neuron of the thread's slot jj (0..9): blocks of 8 columns, two per block
  __device__ __forceinline__ int j(int jj) const { return 40 * hf + 8 * (jj >> 1) + 2 * a + (jj & 1); }
  // operand row of channel c
  __device__ __forceinline__ int row(int c) const { return 32 * q + 8 * c + pp; }
};

// load the thread's 10 neurons x 4 channels from TMEM columns [col0, col0 + 80)
__device__ __forceinline__ void tload(uint32_t tbase, const Who& w, int col0, float4* z) {
  uint32_t r[5][2][4];
#pragma unroll
  for (int b = 0; b < 5; ++b)
#pragma unroll
    for (int h = 0; h < 2; ++h)
      ld16(tbase + (uint32_t(32 * w.q + 16 * h) << 16) + uint32_t(col0 + 40 * w.hf + 8 * b), r[b][h]);
  ld_wait();
#pragma unroll
  for (int b = 0; b < 5; ++b)
#pragma unroll
    for (int e = 0; e < 2; ++e)
      z[2 * b + e] = make_float4(__uint_as_float(r[b][0][e]), __uint_as_float(r[b][0][2 + e]),
                                 __uint_as_float(r[b][1][e]), __uint_as_float(r[b][1][2 + e]));
}
__device__ __forceinline__ void tstore(uint32_t tbase, const Who& w, int col0, const float4* z) {
#pragma unroll
  for (int b = 0; b < 5; ++b) {
    uint32_t r0[4] = {__float_as_uint(z[2 * b].x), __float_as_uint(z[2 * b + 1].x), __float_as_uint(z[2 * b].y),
                      __float_as_uint(z[2 * b + 1].y)};
    uint32_t r1[4] = {__float_as_uint(z[2 * b].z), __float_as_uint(z[2 * b + 1].z), __float_as_uint(z[2 * b].w),
                      __float_as_uint(z[2 * b + 1].w)};
    st16(tbase + (uint32_t(32 * w.q) << 16) + uint32_t(col0 + 40 * w.hf + 8 * b), r0);
    st16(tbase + (uint32_t(32 * w.q + 16) << 16) + uint32_t(col0 + 40 * w.hf + 8 * b), r1);
  }
  st_wait();
}
// write the thread's 10 neurons x 4 channels into an operand buffer (tf32-rounded)
__device__ __forceinline__ void owrite(float* buf, const Who& w, const float4* h) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int r = w.row(c);
#pragma unroll
    for (int b = 0; b < 5; ++b) {
      const float v0 = to_tf32(comp(h[2 * b], c)), v1 = to_tf32(comp(h[2 * b + 1], c));
      *reinterpret_cast<float2*>(buf + sw32(r, w.j(2 * b))) = make_float2(v0, v1);
    }
  }
}

template <int NH, int DO>
struct TcCfg {
  // shared-memory carve (floats); operands first (1024-B aligned)
  static constexpr int oW = 0;                               // (NH-1) x [80 rows j][96] W^k | b^k
  static constexpr int oH = oW + (NH - 1) * WOPER;           // [128 m][96] H^{k-1} (+ ones column 80)
  static constexpr int oZ = oH + OPER;                       // [128 m][96] Zb^k
  // while Zb^k is not live (output layer, layer 1) its buffer also holds the
  // output-layer partials [2 halves][P][DO] float4 and the per-quarter
  // reduction scratch [4][N][4]
  static constexpr int oUp = oZ;
  static constexpr int oRed = oUp + 2 * 4 * P * DO;
  static_assert(oRed + 4 * N * 4 <= oZ + OPER, "aliases inside the Zb buffer");
  static constexpr int oW1 = oZ + OPER;                      // (the MN-major dW read of Zb runs 512 B past it)
  static constexpr int oB1 = oW1 + 2 * N;
  static constexpr int oWo = oB1 + N;                        // [DO][80]
  static constexpr int oBo = oWo + DO * N;
  static constexpr int oSl = al4(oBo + DO);                  // slopes s_k = n a^k
  static constexpr int oX = al4(oSl + NH);                   // [2][P]
  static constexpr int oU = oX + 2 * P;                      // [P][DO] float4
  static constexpr int oMisc = oU + 4 * P * DO;              // loss scratch [8][4], mbarrier, tmem slot, s_next
  static constexpr int TOTAL = oMisc + 32 + 28;  // loss scratch, 2 mbarriers, tmem slot, s_next, peer counts, sticky state
  static constexpr size_t SMEM = size_t(TOTAL) * 4;
  static_assert(SMEM <= 227 * 1024, "shared memory budget of the tensor-core kernel");
  static_assert((oH * 4) % 1024 == 0 && (oZ * 4) % 1024 == 0 && (WOPER * 4) % 1024 == 0, "operand alignment");
  static_assert(80 * (NH + 1) <= TCOLS, "TMEM columns");
};

}  // namespace tc

// K1 (MODE 0), K2 (MODE 1) and the fused step (MODE 2) with tensor-core hidden
// layers; same chunk schedule, epilogues and outputs as k_fused (N = 80).
template <int NH, int DO, int ACT, int MODE>
__global__ void __launch_bounds__(tc::T, 1) k_fused_tc(const KArgs a) {
  using namespace tc;
  using C = TcCfg<NH, DO>;
  using LY = Lay<N, NH, DO>;
  extern __shared__ __align__(1024) float smt[];
  float* sm = smt;
  const int tid = threadIdx.x;
  const Who w(tid);
  if ((smem_u32(sm) & 1023u) != 0u) __trap();   // SW128_32B operands need 1024-B aligned buffers
  float* sW = sm + C::oW;
  float* sH = sm + C::oH;
  float* sZ = sm + C::oZ;
  const float* sW1 = sm + C::oW1;
  const float* sB1 = sm + C::oB1;
  const float* sWo = sm + C::oWo;
  const float* sBo = sm + C::oBo;
  const float* sSl = sm + C::oSl;
  float* sX = sm + C::oX;
  float* sY = sX + P;
  float4* sU = reinterpret_cast<float4*>(sm + C::oU);
  float4* sUp = reinterpret_cast<float4*>(sm + C::oUp);
  float* sRed = sm + C::oRed;
  float* sLoss = sm + C::oMisc;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + C::oMisc + 32);    // forward / input-adjoint MMAs
  uint64_t* mbar2 = reinterpret_cast<uint64_t*>(sm + C::oMisc + 34);   // dW MMAs
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + C::oMisc + 36);
  int* s_next = reinterpret_cast<int*>(sm + C::oMisc + 37);
  int* xcount = reinterpret_cast<int*>(sm + C::oMisc + 38);    // [kMaxPeers] peer rows of a payload chunk
  const float m1 = a.m1, m2 = a.m2;
  const uint32_t aH = smem_u32(sH), aZ = smem_u32(sZ), aW = smem_u32(sW);
#ifdef PINN_PHASE_PROF
  long long prof_acc[20] = {};
  long long prof_t0 = clock64();
  int prof_cur = 0;
#endif

  // ones column of H (bias of the forward MMA, db of the dW MMA): value rows 1,
  // derivative rows 0; columns 81..95 zero.  Activations write columns < 80 only.
  for (int e = tid; e < M * (CP - N); e += T) {
    const int r = e / (CP - N), c = N + e % (CP - N);
    sH[sw32(r, c)] = (c == N && ((r >> 3) & 3) == 0) ? 1.0f : 0.0f;
  }
  for (int e = tid; e < M * (CP - N); e += T) sZ[sw32(e / (CP - N), N + e % (CP - N))] = 0.0f;
  if (tid == 0) {
    mbar_init(mbar);
    mbar_init(mbar2);
  }
  if (tid < 32) {
    __syncwarp();
    tmem_alloc<TCOLS>(tslot);
  }
  fence_async_smem();
  tmem_fence_before();
  cta_sync();
  tmem_fence_after();
  const uint32_t tm = *tslot;
  uint32_t phase = 0, phase2 = 0;
  // one elected thread issues a group of MMAs after every thread's operand
  // writes (generic proxy) are fenced into the async proxy
  auto issue = [&](auto body) {
    fence_async_smem();
    tmem_fence_before();
    cta_sync();
    if (tid == 0) {
      tmem_fence_after();
      body();
      commit(mbar);
    }
    mbar_wait(mbar, phase);
    phase ^= 1u;
    tmem_fence_after();
  };

  // Deferred dW flush.  The reverse step of layer k leaves dW^k^T in S_k's
  // columns (lanes i, columns j); it is added into its chunk's partial only
  // when S_k is next needed -- inside the next tile's forward pass, while the
  // MMA of layer k - 1 runs (the threads would otherwise idle in its wait).
  // State (uniform, in shared memory): the pending layer mask, the partial
  // and whether that tile was its chunk's first (store instead of add).
  volatile int* dpend = reinterpret_cast<volatile int*>(sm + C::oMisc + 52);
  volatile int* dfirst = reinterpret_cast<volatile int*>(sm + C::oMisc + 53);
  float* volatile* dpc = reinterpret_cast<float* volatile*>(sm + C::oMisc + 54);
  if (tid == 0) *dpend = 0;
  // add dW^k^T (pending in S_k) into the partial; every thread reads the
  // state before anyone can change it (callers sit between CTA barriers)
  auto flush_layer = [&](int k) {
    float* P0 = *dpc;
    const bool fst = *dfirst != 0;
    if (w.q < 3) {   // lanes i = 0..95 (i < 80: W^k column i; i = 80: b^k)
      uint32_t r[5][8];
#pragma unroll
      for (int b = 0; b < 5; ++b)
        ld32x8(tm + (uint32_t(32 * w.q) << 16) + uint32_t(80 * k + 40 * w.hf + 8 * b), r[b]);
      ld_wait();
      const int i = 32 * w.q + (tid & 31);
      if (i <= N) {
        float* g = i < N ? P0 + LY::offW(k) + 40 * w.hf * N + i : P0 + LY::offB(k) + 40 * w.hf;
        const int st = i < N ? N : 1;
#pragma unroll
        for (int b = 0; b < 5; ++b)
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            float* gp = g + (8 * b + e) * st;
            if (fst)
              *gp = __uint_as_float(r[b][e]);
            else
              red_add(gp, __uint_as_float(r[b][e]));
          }
      }
    }
  };
  auto flush_pending = [&](int k) {   // flush layer k if pending (uniform branch)
    if (*dpend & (1 << k)) {
      flush_layer(k);
      tmem_fence_before();
      cta_sync();
      if (tid == 0) *dpend = *dpend & ~(1 << k);
      cta_sync();
      tmem_fence_after();
    }
  };

  int cur_sub = -1;
  const int n_pay = MODE == 2 ? a.n_chunks2 : 0;
  // peer-store exchange of the fused step: this launch's step index (receive
  // slot parity, expected arrivals) and per-peer row counts of a payload chunk
  const bool px = MODE == 2 && a.px.n > 0;
  const int xstep = px ? *reinterpret_cast<volatile int*>(a.px.step) : 0;
  const int64_t roff = px ? int64_t(xstep & 1) * a.px.n_recv : 0;
  if (tid < kMaxPeers) xcount[tid] = 0;
  volatile int* sst = reinterpret_cast<volatile int*>(sm + C::oMisc + 46);   // sticky state [6] (next_item)
  if (tid == 0) {
    sst[0] = -1;
    sst[1] = 0;
    sst[2] = -1;
    sst[3] = 0;
  }
#pragma unroll 1
  for (;;) {
    PROF_MARK(0);
    // The sticky schedule is compiled into the per-region-activation instance
    // only (C5: K1 0.324 -> 0.265 ms); in the 255-register 5x80 instance its
    // mere presence costs 9 % (C4 TF32 K1 5.61 -> 6.08 ms) and C4's big
    // chunks never use it.
    constexpr bool kSticky = MODE == 2 && ACT == kActMixed;
    if (tid == 0) *s_next = kSticky ? next_item(a, n_pay, sst) : atomicAdd(a.sched, 1);
    cta_sync();
    const int idx = *s_next;
    if (idx >= a.n_chunks + n_pay) break;
    const bool pay = MODE == 1 || (MODE == 2 && idx < n_pay);
    const int li = idx - n_pay;
    const bool direct = kSticky && a.sub_chunk_off != nullptr;   // sticky: li is the chunk index
    const int c = pay ? (MODE == 2 ? idx : (a.order ? a.order[idx] : idx)) : (direct ? li : (a.order ? a.order[li] : li));
    const Chunk ch = (MODE == 2 && pay) ? a.chunks2[c] : a.chunks[c];
    if (MODE == 2 && !pay && ch.pad) {
      wait_payload(a, n_pay, xstep);   // local payload chunks and the peers' rows
      cta_sync();
    }
    if (ch.sub != cur_sub) {
      // weights of subdomain ch.sub: W^k | b^k as tf32 operands, the rest FP32
      cta_sync();
      PROF_MARK(1);
      const float* G = a.params + size_t(ch.sub) * a.pstride;
      // every load of a layer in flight before its stores (a one-at-a-time loop
      // cannot move a load above the previous generic-pointer shared store,
      // which made a reload ~110 serial L2 round trips: 4.5 % of C4's TF32 K1)
      constexpr int WIT = (N * CP + T - 1) / T;
#pragma unroll 1
      for (int k = 2; k <= NH; ++k) {
        float* dst = sW + (k - 2) * WOPER;
        float v[WIT];
#pragma unroll
        for (int u = 0; u < WIT; ++u) {
          const int e = tid + u * T;
          const int j = e / CP, i = e % CP;
          v[u] = e >= N * CP ? 0.0f
                             : (i < N ? __ldcg(G + LY::offW(k) + j * N + i)
                                      : (i == N ? __ldcg(G + LY::offB(k) + j) : 0.0f));
        }
#pragma unroll
        for (int u = 0; u < WIT; ++u) {
          const int e = tid + u * T;
          if (e < N * CP) dst[sw32(e / CP, e % CP)] = to_tf32(v[u]);
        }
      }
      float* s1 = sm + C::oW1;
      for (int e = tid; e < 3 * N; e += T) s1[e] = G[LY::offW(1) + e];   // W^1 [N][2], b^1
      for (int e = tid; e < DO * N; e += T) sm[C::oWo + e] = G[LY::offW(NH + 1) + e];
      for (int e = tid; e < DO; e += T) sm[C::oBo + e] = G[LY::offB(NH + 1) + e];
      for (int e = tid; e < NH; e += T) sm[C::oSl + e] = a.slope_n * G[LY::offA(e + 1)];
      cur_sub = ch.sub;
    }
    PROF_MARK(0);
    const int ahead = (kSticky && !pay && tid == 0) ? sticky_ahead_issue(a, sst) : -1;
    const float4 lw = a.sub_w[ch.sub];
    const int act = ACT == kActMixed ? a.sub_act[ch.sub] : ACT;
    float* Pc = a.partial + size_t(c) * a.pstride;
    const int ntiles = (ch.count + P - 1) / P;
    if (!pay && ntiles == 0) {
      for (int e = tid; e < a.pstride; e += T) Pc[e] = 0.0f;
      if (tid < 4) a.partial_loss[size_t(c) * 4 + tid] = 0.0f;
    }

    // the chunk body is compiled once per mode; a per-subdomain-activation
    // instance branches on `act` around each activation loop only (with_act),
    // never around the MMAs, operand stores or epilogue (compiling the whole
    // body per activation tripled C5's kernel to 21 k instructions and made
    // instruction fetch its top stall)
    auto chunk_body = [&](auto mode_c) {
      constexpr int MS = decltype(mode_c)::value;   // 0 loss + gradient, 1 payload
      float lsum[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      // coordinates of the next tile are loaded into registers while the
      // current tile computes (thread p < P owns point p of a tile)
      float cx = 0.0f, cy = 0.0f;
      if (tid < min(P, ch.count)) {
        cx = a.coords[int64_t(ch.start) + tid];
        cy = a.coords[a.n_points + int64_t(ch.start) + tid];
      }
#pragma unroll 1
      for (int t = 0; t < ntiles; ++t) {
        const int64_t p0 = int64_t(ch.start) + int64_t(t) * P;
        const int np = min(P, ch.count - t * P);
        const bool first = (t == 0);
        PROF_MARK(MS == 1 ? 10 : 2);
        if (tid < P) {
          sX[tid] = cx;
          sY[tid] = cy;
          cx = cy = 0.0f;
          if (t + 1 < ntiles && tid < min(P, ch.count - (t + 1) * P)) {
            cx = a.coords[p0 + P + tid];
            cy = a.coords[a.n_points + p0 + P + tid];
          }
        }
        cta_sync();
        PROF_MARK(MS == 1 ? 10 : 3);
        // ---------------------------------------------------------- forward
        float4 z[kJT];
        {
          // layer 1 on the CUDA cores: z = W^1 x + b^1, dz/dx_i = W^1[:, i], Delta z = 0
          const float x = sX[w.pt], y = sY[w.pt];
          const float s = sSl[0];
#pragma unroll
          for (int jj = 0; jj < kJT; ++jj) {
            const int j = w.j(jj);
            const float w0 = sW1[2 * j], w1 = sW1[2 * j + 1];
            z[jj] = make_float4(fmaf(w0, x, fmaf(w1, y, sB1[j])), w0, w1, 0.0f);
          }
          with_act<ACT>(act, [&](auto act_c) {
            constexpr int AS = decltype(act_c)::value;
#pragma unroll
            for (int jj = 0; jj < kJT; ++jj) z[jj].x = stash_x<AS>(z[jj].x, s, act);
            if constexpr (MS == 0) tstore(tm, w, 80 * 1, z);
#pragma unroll
            for (int jj = 0; jj < kJT; ++jj) z[jj] = act_fwd<AS>(z[jj], s, m1, m2, act);
          });
          owrite(sH, w, z);
        }
#pragma unroll 1
        for (int k = 2; k <= NH; ++k) {
          const uint32_t wk = aW + uint32_t((k - 2) * WOPER * 4);
          PROF_MARK(MS == 1 ? 10 : 12);
          // MMA(k) into R (free during the forward pass); while it runs, add
          // the previous tile's dW^k (pending in S_k) into its chunk partial,
          // then the stash form of layer k goes into S_k
          fence_async_smem();
          tmem_fence_before();
          cta_sync();
          const int pend_k = (MS == 0) ? (*dpend & (1 << k)) : 0;
          if (tid == 0) {
            tmem_fence_after();
#pragma unroll
            for (int ks = 0; ks < KF / 8; ++ks) mma(tm, kmajor(aH, ks), kmajor(wk, ks), idesc(M, N, 0, 0), ks > 0);
            commit(mbar);
          }
          if (pend_k) {
            tmem_fence_after();
            flush_layer(k);
          }
          mbar_wait(mbar, phase);
          phase ^= 1u;
          tmem_fence_after();
          if (pend_k) {
            tmem_fence_before();
            cta_sync();   // every thread has read the state and S_k (tcgen05.wait::ld)
            if (tid == 0) *dpend = *dpend & ~(1 << k);
            tmem_fence_after();
          }
          PROF_MARK(MS == 1 ? 10 : 13);
          tload(tm, w, 0, z);
          const float s = sSl[k - 1];
          with_act<ACT>(act, [&](auto act_c) {
            constexpr int AS = decltype(act_c)::value;
#pragma unroll
            for (int jj = 0; jj < kJT; ++jj) z[jj].x = stash_x<AS>(z[jj].x, s, act);
            if constexpr (MS == 0) tstore(tm, w, 80 * k, z);   // stash form (t for tanh)
#pragma unroll
            for (int jj = 0; jj < kJT; ++jj) z[jj] = act_fwd<AS>(z[jj], s, m1, m2, act);
          });
          if (k < NH) owrite(sH, w, z);   // the MMA that read H^{k-1} has completed
        }
        PROF_MARK(MS == 1 ? 10 : 4);
        // z = H^NH of the thread's (point, 10 neurons).  Output layer on the CUDA
        // cores: partial dot products over the thread's neurons, combined over
        // the 4 lanes of a point (shuffles) and the two halves (shared memory).
#pragma unroll
        for (int o = 0; o < DO; ++o) {
          float4 acc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
          for (int jj = 0; jj < kJT; ++jj) fma4(acc, sWo[o * N + w.j(jj)], z[jj]);
#pragma unroll
          for (int off = 1; off < 4; off <<= 1) {
            acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
            acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
            acc.z += __shfl_xor_sync(0xffffffffu, acc.z, off);
            acc.w += __shfl_xor_sync(0xffffffffu, acc.w, off);
          }
          if (w.a == 0) sUp[(w.hf * P + w.pt) * DO + o] = acc;
        }
        cta_sync();
        for (int e = tid; e < P * DO; e += T) {
          const float4 u0 = sUp[e], u1 = sUp[P * DO + e];
          sU[e] = make_float4(u0.x + u1.x + sBo[e % DO], u0.y + u1.y, u0.z + u1.z, u0.w + u1.w);
        }
        cta_sync();
        PROF_MARK(MS == 1 ? 11 : 5);
        // --------------------------------------------------------- epilogue
        if constexpr (MS == 1) {
          for (int p = tid; p < np; p += T) {
            float4 U[DO];
#pragma unroll
            for (int o = 0; o < DO; ++o) U[o] = sU[p * DO + o];
            point_payload<DO>(a, p0 + p, sX[p], sY[p], U, xstep, px ? xcount : nullptr);
          }
          continue;
        } else {
          for (int p = tid; p < P; p += T) {
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
          // ------------------------------------------------------- reverse
          // output layer: Hb^NH = W^L^T Ub (thread-local); dW^L[o][j] =
          // sum_p Ub[p][o] . H^NH[p][j] (4 channels), db^L = sum_p Ub_value
          float4 hb[kJT];
#pragma unroll
          for (int jj = 0; jj < kJT; ++jj) hb[jj] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
          for (int o = 0; o < DO; ++o) {
            const float4 ub = sU[w.pt * DO + o];
#pragma unroll
            for (int jj = 0; jj < kJT; ++jj) {
              fma4(hb[jj], sWo[o * N + w.j(jj)], ub);
              float d = ub.x * z[jj].x + ub.y * z[jj].y + ub.z * z[jj].z + ub.w * z[jj].w;
              d += __shfl_xor_sync(0xffffffffu, d, 4);
              d += __shfl_xor_sync(0xffffffffu, d, 8);
              d += __shfl_xor_sync(0xffffffffu, d, 16);
              if (w.pp == 0) sRed[(w.q * N + w.j(jj)) * 4 + o] = d;
            }
          }
          cta_sync();
          for (int e = tid; e < DO * N; e += T) {
            const int o = e / N, j = e % N;
            const float v = ((sRed[(0 * N + j) * 4 + o] + sRed[(1 * N + j) * 4 + o]) + sRed[(2 * N + j) * 4 + o]) +
                            sRed[(3 * N + j) * 4 + o];
            float* g = Pc + LY::offW(NH + 1) + e;
            if (first)
              *g = v;
            else
              red_add(g, v);
          }
          if (tid < DO) {
            float v = 0.0f;
            for (int p = 0; p < P; ++p) v += sU[p * DO + tid].x;
            float* g = Pc + LY::offB(NH + 1) + tid;
            if (first)
              *g = v;
            else
              red_add(g, v);
          }
          cta_sync();   // sRed / sUp (inside the Zb buffer) are read before Zb is written
          // hidden layers k = NH .. 2.  Per step: the input-adjoint MMA commits to
          // mbar, the dW MMA to mbar2, so the dW MMA runs while the threads read
          // Hb^{k-1} and compute the next step's activation maps; its result
          // (dW^k^T in S_k: lanes i, columns j) is added to the chunk partial
          // just before the next operands overwrite its inputs.
          // this tile's dW^k^T stay in S_k after their MMAs (deferred flush; the
          // forward pass has flushed every earlier one, so dpend == 0 here)
          if (tid == 0) {
            *dpc = Pc;
            *dfirst = first ? 1 : 0;
          }
          int pend = 0;   // layer whose dW MMA may still be reading Zb / H (0 = none)
          auto wait_dw = [&]() {
            if (!pend) return;
            mbar_wait(mbar2, phase2);
            phase2 ^= 1u;
            tmem_fence_after();
            pend = 0;
          };
#pragma unroll 1
          for (int k = NH; k >= 2; --k) {
            PROF_MARK(15);
            tload(tm, w, 80 * k, z);
            {
              const float s = sSl[k - 1];
              with_act<ACT>(act, [&](auto act_c) {
                constexpr int AS = decltype(act_c)::value;
#pragma unroll
                for (int jj = 0; jj < kJT; ++jj) hb[jj] = act_bwd<AS>(z[jj], hb[jj], s, m1, m2, act);
              });
            }
            tload(tm, w, 80 * (k - 1), z);
            {
              const float s = sSl[k - 2];
              with_act<ACT>(act, [&](auto act_c) {
                constexpr int AS = decltype(act_c)::value;
#pragma unroll
                for (int jj = 0; jj < kJT; ++jj) z[jj] = act_fwd<AS>(z[jj], s, m1, m2, act);
              });
            }
            PROF_MARK(16);
            wait_dw();   // the previous dW MMA has read Zb / H: they may be overwritten
            PROF_MARK(17);
            owrite(sZ, w, hb);   // Zb^k
            owrite(sH, w, z);    // H^{k-1}
            const uint32_t wk = aW + uint32_t((k - 2) * WOPER * 4);
            PROF_MARK(18);
            fence_async_smem();
            tmem_fence_before();
            cta_sync();
            if (tid == 0) {
              tmem_fence_after();
              // Hb^{k-1} = Zb^k W^k : A = Zb (K-major, K = j), B = W^k (MN-major, N = i)
#pragma unroll
              for (int ks = 0; ks < N / 8; ++ks) mma(tm, kmajor(aZ, ks), mnmajor(wk, ks), idesc(M, N, 0, 1), ks > 0);
              commit(mbar);
              // dW^k^T = H^T Zb : A = H (MN-major, M = i + ones column), B = Zb (MN-major, N = j),
              // into S_k (consumed above)
#pragma unroll
              for (int ks = 0; ks < M / 8; ++ks)
                mma(tm + uint32_t(80 * k), mnmajor(aH, ks), mnmajor(aZ, ks), idesc(M, N, 1, 1), ks > 0);
              commit(mbar2);
              *dpend = *dpend | (1 << k);
            }
            pend = k;
            mbar_wait(mbar, phase);
            phase ^= 1u;
            tmem_fence_after();
            PROF_MARK(19);
            tload(tm, w, 0, hb);   // Hb^{k-1} from R
          }
          PROF_MARK(16);
          wait_dw();
          PROF_MARK(8);
          // layer 1: Zb^1 = act_bwd(S_1, Hb^1); dW^1[j] = sum_p (zb_v x_p + zb_{d_i}), db^1 = sum_p zb_v
          tload(tm, w, 80, z);
          {
            const float s = sSl[0];
            const float x = sX[w.pt], y = sY[w.pt];
            with_act<ACT>(act, [&](auto act_c) {
              constexpr int AS = decltype(act_c)::value;
#pragma unroll
              for (int jj = 0; jj < kJT; ++jj) hb[jj] = act_bwd<AS>(z[jj], hb[jj], s, m1, m2, act);
            });
#pragma unroll
            for (int jj = 0; jj < kJT; ++jj) {
              const float4 zb = hb[jj];
              float v0 = fmaf(zb.x, x, zb.y), v1 = fmaf(zb.x, y, zb.z), vb = zb.x;
#pragma unroll
              for (int off = 4; off < 32; off <<= 1) {
                v0 += __shfl_xor_sync(0xffffffffu, v0, off);
                v1 += __shfl_xor_sync(0xffffffffu, v1, off);
                vb += __shfl_xor_sync(0xffffffffu, vb, off);
              }
              if (w.pp == 0) {
                float* r = sRed + (w.q * N + w.j(jj)) * 4;
                r[0] = v0;
                r[1] = v1;
                r[2] = vb;
              }
            }
          }
          cta_sync();
          for (int e = tid; e < 3 * N; e += T) {
            const int j = e / 3, v = e % 3;
            const float sum = ((sRed[(0 * N + j) * 4 + v] + sRed[(1 * N + j) * 4 + v]) + sRed[(2 * N + j) * 4 + v]) +
                              sRed[(3 * N + j) * 4 + v];
            float* g = Pc + (v < 2 ? LY::offW(1) + 2 * j + v : LY::offB(1) + j);
            if (first)
              *g = sum;
            else
              red_add(g, sum);
          }
          cta_sync();
        }
      }
      PROF_MARK(9);
      if constexpr (MS == 0) {
        if (ntiles > 0) {
          block_sum<4, T>(lsum, sLoss);
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
      cta_sync();
      if (px) publish_peer_rows(a, xcount);
      if (tid == 0) {
        __threadfence();
        atomicAdd(a.sched + 4, 1);
      }
    }
    if (kSticky && tid == 0) sticky_ahead_finish(a, sst, ahead);
    cta_sync();
  }
  // the last tile's dW (pending in S_k)
  for (int k = 2; k <= NH; ++k) flush_pending(k);
#ifdef PINN_PHASE_PROF
  PROF_MARK(0);
  if (tid == 0 && blockIdx.x < 4)
    printf("PHASE N=%d NH=%d MODE=%d cta=%d: %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld "
           "%lld %lld %lld %lld %lld\n", N, NH, MODE, int(blockIdx.x), prof_acc[0], prof_acc[1], prof_acc[2],
           prof_acc[3], prof_acc[4], prof_acc[5], prof_acc[6], prof_acc[7], prof_acc[8], prof_acc[9], prof_acc[10],
           prof_acc[11], prof_acc[12], prof_acc[13], prof_acc[14], prof_acc[15], prof_acc[16], prof_acc[17],
           prof_acc[18], prof_acc[19]);
#endif
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
  tmem_fence_before();
  cta_sync();
  tmem_fence_after();
  if (tid < 32) {
    __syncwarp();
    tmem_dealloc<TCOLS>(tm);
  }
}

}  // namespace pinn
