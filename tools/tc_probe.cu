// tc_probe.cu -- standalone validation of tcgen05.mma kind::tf32 operand layouts,
// SMEM/instruction descriptors and TMEM readout (development tool).
//
// D[M x N] (+)= A[M x K] * B[K x N], fp32 accumulate, tf32 inputs (exact small ints).
// A: K-major ("a_major" = 0) or MN-major (1); B: K-major or MN-major.
// No-swizzle canonical layouts (CuTe mma_traits_sm100.hpp make_umma_desc):
//   K-major : ((8,n),2):((1,SBO),LBO) in 16-B units -> core = 8 rows x 16 B, LBO = K step
//   MN-major: ((1,n),(8,k)):((X,SBO),(1,LBO))        -> core = 8 K-rows x 16 B, SBO = MN step
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 0) {
  uint64_t d = (uint64_t)layout << 61;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                  // version 1 (Blackwell)
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}

__host__ __device__ constexpr uint32_t make_idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4)            // D format F32
       | (2u << 7)            // A TF32
       | (2u << 10)           // B TF32
       | ((uint32_t)a_mn << 15)
       | ((uint32_t)b_mn << 16)
       | ((uint32_t)(N >> 3) << 17)
       | ((uint32_t)(M >> 4) << 24);
}

// element offset (floats) in a tile stored with 8x4-element core matrices
// K-major  (rows = MN index r, cols = K index k): core(rg, kg) at (rg*KG + kg)*32 -> LBO = 128 B, SBO = KG*128 B
__host__ __device__ inline int off_kmaj(int r, int k, int KG) { return ((r >> 3) * KG + (k >> 2)) * 32 + (r & 7) * 4 + (k & 3); }
// MN-major (rows = K index k, cols = MN index c): core(kg, cg) with 8 K-rows x 4 MN: at (kg*CG + cg)*32
//   -> SBO (MN step) = 128 B, LBO (K step of 8) = CG*128 B
__host__ __device__ inline int off_mnmaj_none(int k, int c, int CG) { return ((k >> 3) * CG + (c >> 2)) * 32 + (k & 7) * 4 + (c & 3); }
// MN-major, 32-B swizzle: atom = 8 K-rows x 8 MN elements (256 B), unit(16B) ^= (row>>2)&1
//   atoms along MN at LBO = 256 B, 8-K groups at SBO = NA*256 B
__host__ __device__ inline int off_mnmaj(int k, int c, int CG) {
  const int NA = CG / 2;                 // MN atoms (8 elements each)
  const int kg = k >> 3, kr = k & 7, an = c >> 3, u = (c >> 2) & 1, e = c & 3;
  const int byte = kg * NA * 256 + an * 256 + kr * 32 + ((u ^ ((kr >> 2) & 1)) << 4) + e * 4;
  return byte >> 2;
}

template <int M, int N, int K, int AMN, int BMN>
__global__ void probe(const float* A, const float* B, float* D, int swap) {
  __shared__ __align__(1024) float sA[M * K];
  __shared__ __align__(1024) float sB[N * K];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  // A[m][k] row-major in global
  for (int e = tid; e < M * K; e += blockDim.x) {
    const int m = e / K, k = e % K;
    const int o = AMN ? off_mnmaj(k, m, M / 4) : off_kmaj(m, k, K / 4);
    sA[o] = A[e];
  }
  // B[k][n] row-major in global
  for (int e = tid; e < K * N; e += blockDim.x) {
    const int k = e / N, n = e % N;
    const int o = BMN ? off_mnmaj(k, n, N / 4) : off_kmaj(n, k, K / 4);
    sB[o] = B[e];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&mbar)));
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" :: "r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (tid == 0) {
    const uint32_t idesc = make_idesc(M, N, AMN, BMN);
    for (int ks = 0; ks < K / 8; ++ks) {
      uint64_t ad, bd;
      if (AMN) ad = make_desc(smem_u32(sA) + ks * (M / 8) * 256, 256, (M / 8) * 256, 6);
      else     ad = make_desc(smem_u32(sA) + ks * 2 * 128 /*2 K-cores*/, 128, (K / 4) * 128);
      if (BMN) bd = make_desc(smem_u32(sB) + ks * (N / 8) * 256, 256, (N / 8) * 256, 6);
      else     bd = make_desc(smem_u32(sB) + ks * 2 * 128, 128, (K / 4) * 128);
      const uint32_t acc = ks > 0 ? 1u : 0u;
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                   :: "r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&mbar)));
  }
  // wait for the MMA
  asm volatile("{\n.reg .pred P;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra WAIT_%=;\n}\n"
               :: "r"(smem_u32(&mbar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // read D: warp w reads lanes 32w..32w+31 ; N columns
  const int warp = tid >> 5, lane = tid & 31;
  if (warp < 4) {
    for (int c = 0; c < N; c += 8) {
      uint32_t r[8];
      const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + c;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   "tcgen05.wait::ld.sync.aligned;\n"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(ta));
      const int row = warp * 32 + lane;
      for (int i = 0; i < 8; ++i) D[row * N + c + i] = __uint_as_float(r[i]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" :: "r"(tmem));
}

template <int M, int N, int K, int AMN, int BMN>
int run(const char* name, int swap = 0) {
  std::vector<float> A(M * K), B(K * N), D(128 * N, -999.f), R(M * N, 0.f);
  for (int i = 0; i < M * K; ++i) A[i] = (float)((i * 7 + 3) % 11 - 5);
  for (int i = 0; i < K * N; ++i) B[i] = (float)((i * 5 + 1) % 9 - 4);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      float s = 0;
      for (int k = 0; k < K; ++k) s += A[m * K + k] * B[k * N + n];
      R[m * N + n] = s;
    }
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dD, D.data(), D.size() * 4, cudaMemcpyHostToDevice));
  probe<M, N, K, AMN, BMN><<<1, 128>>>(dA, dB, dD, swap);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0, shown = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n)
      if (D[m * N + n] != R[m * N + n]) {
        if (shown++ < 4) printf("  %s mismatch m=%d n=%d got %g want %g\n", name, m, n, D[m * N + n], R[m * N + n]);
        ++bad;
      }
  // for M=64 also report where rows landed
  if (M == 64 && bad) {
    for (int row = 0; row < 128; row += 16) printf("  lane %3d: %g %g\n", row, D[row * N], D[row * N + 1]);
  }
  printf("%s swap=%d: %s (%d mismatches)\n", name, swap, bad ? "FAIL" : "ok", bad);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return bad;
}

int main() {
  int bad = 0;
  bad += run<128, 48, 8, 0, 0>("M128 N48 K8  A-K  B-K ");
  bad += run<128, 48, 40, 0, 0>("M128 N48 K40 A-K  B-K ");
  bad += run<128, 48, 40, 0, 1>("M128 N48 K40 A-K  B-MN");
  bad += run<128, 48, 64, 1, 1>("M128 N48 K64 A-MN B-MN");
  bad += run<64, 48, 64, 1, 1>("M64  N48 K64 A-MN B-MN");
  bad += run<64, 48, 40, 0, 0>("M64  N48 K40 A-K  B-K ");
  run<128, 48, 40, 0, 1>("M128 N48 K40 A-K  B-MN", 1);
  run<128, 48, 64, 1, 0>("M128 N48 K64 A-MN B-K ", 0);
  run<128, 48, 64, 1, 0>("M128 N48 K64 A-MN B-K ", 1);
  run<128, 48, 64, 1, 1>("M128 N48 K64 A-MN B-MN", 1);
  run<128, 32, 64, 0, 1>("M128 N32 K64 A-K  B-MN", 0);
  run<128, 32, 64, 0, 1>("M128 N32 K64 A-K  B-MN", 1);
  printf("total mismatches %d\n", bad);
  return 0;
}
