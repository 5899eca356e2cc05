// tc_probe2.cu -- building blocks for a tcgen05 (kind::tf32) hidden-layer path
// (development tool):
//   1. the thread <-> (lane, column) mapping of tcgen05.ld.16x256b,
//   2. MN-major TF32 operands in the SWIZZLE_128B_BASE32B layout (layout type 1),
//      the only MN-major layout CUTLASS allows for 32-bit operands,
//   3. K-major (no swizzle) reference.
// D[M x N] = A[M x K] * B[K x N], fp32 accumulate, exact small-integer inputs.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = (uint64_t)layout << 61;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__host__ __device__ constexpr uint32_t make_idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// K-major, no swizzle: core (8 rows x 4 K) = 128 B; cores along K at 128 B (LBO), row groups at KG*128 (SBO)
__host__ __device__ inline int off_kmaj(int r, int k, int KG) { return ((r >> 3) * KG + (k >> 2)) * 32 + (r & 7) * 4 + (k & 3); }
// MN-major SW128_32B: atom = 4 K-rows x 32 MN (512 B), 32-B granule ^= k % 4.
// atoms ordered [k/4][mn/32]: MN-atom step 512 B (LBO), K-atom step NA*512 B (SBO)
__host__ __device__ inline int off_mn32(int mn, int k, int MN) {
  const int NA = MN / 32;
  const int byte_in = (k & 3) * 128 + (mn & 31) * 4;
  const int sw = byte_in ^ (((byte_in >> 7) & 3) << 5);
  return (((k >> 2) * NA + (mn >> 5)) * 512 + sw) >> 2;
}

template <int M, int N, int K, int AMN, int BMN>
__global__ void probe(const float* A, const float* B, float* D, int lbo_sbo_swap) {
  __shared__ __align__(1024) float sA[M * K];
  __shared__ __align__(1024) float sB[N * K];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  for (int e = tid; e < M * K; e += blockDim.x) {
    const int m = e / K, k = e % K;
    sA[AMN ? off_mn32(m, k, M) : off_kmaj(m, k, K / 4)] = A[e];
  }
  for (int e = tid; e < K * N; e += blockDim.x) {
    const int k = e / N, n = e % N;
    sB[BMN ? off_mn32(n, k, N) : off_kmaj(n, k, K / 4)] = B[e];
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&mbar)));
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" :: "r"(smem_u32(&tslot)));
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
      if (AMN) {
        const uint32_t lbo = 512, sbo = (M / 32) * 512;
        ad = make_desc(smem_u32(sA) + ks * 2 * sbo, lbo_sbo_swap ? sbo : lbo, lbo_sbo_swap ? lbo : sbo, 1);
      } else {
        ad = make_desc(smem_u32(sA) + ks * 2 * 128, 128, (K / 4) * 128, 0);
      }
      if (BMN) {
        const uint32_t lbo = 512, sbo = (N / 32) * 512;
        bd = make_desc(smem_u32(sB) + ks * 2 * sbo, lbo_sbo_swap ? sbo : lbo, lbo_sbo_swap ? lbo : sbo, 1);
      } else {
        bd = make_desc(smem_u32(sB) + ks * 2 * 128, 128, (K / 4) * 128, 0);
      }
      const uint32_t acc = ks > 0 ? 1u : 0u;
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                   :: "r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&mbar)));
  }
  asm volatile("{\n.reg .pred P;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra WAIT_%=;\n}\n"
               :: "r"(smem_u32(&mbar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int warp = tid >> 5, lane = tid & 31;
  if (warp < 4) {
    for (int c = 0; c < N; c += 8) {
      uint32_t r[8];
      const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + c;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                   "tcgen05.wait::ld.sync.aligned;\n"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(ta));
      for (int i = 0; i < 8; ++i) D[(warp * 32 + lane) * N + c + i] = __uint_as_float(r[i]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" :: "r"(tmem));
}

// 16x256b mapping: warp 0 writes lane t, column c := 1000 t + c (32x32b.x8 store),
// then every thread reads 16x256b at lane base 0 and 16 and reports what it got.
__global__ void map16x256b(int* out) {
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"(smem_u32(&tslot)));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  uint32_t v[8];
  for (int c = 0; c < 8; ++c) v[c] = 1000 * tid + c;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n"
               "tcgen05.wait::st.sync.aligned;\n"
               :: "r"(tmem), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
  for (int half = 0; half < 2; ++half) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];\n"
                 "tcgen05.wait::ld.sync.aligned;\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(tmem + ((uint32_t)(16 * half) << 16)));
    for (int i = 0; i < 4; ++i) out[(half * 32 + tid) * 4 + i] = (int)r[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(tmem));
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
        if (shown++ < 3) printf("  %s mismatch m=%d n=%d got %g want %g\n", name, m, n, D[m * N + n], R[m * N + n]);
        ++bad;
      }
  printf("%s swap=%d: %s (%d mismatches)\n", name, swap, bad ? "FAIL" : "ok", bad);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return bad;
}

int main() {
  int* dout;
  CK(cudaMalloc(&dout, 64 * 4 * 4));
  map16x256b<<<1, 32>>>(dout);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int> o(64 * 4);
  CK(cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost));
  printf("16x256b.x1 (value = 1000*lane + col):\n");
  for (int half = 0; half < 2; ++half)
    for (int t = 0; t < 32; t += 1) {
      printf("  base %2d thread %2d:", 16 * half, t);
      for (int i = 0; i < 4; ++i) printf(" (%d,%d)", o[(half * 32 + t) * 4 + i] / 1000, o[(half * 32 + t) * 4 + i] % 1000);
      printf("\n");
    }
  run<128, 64, 16, 0, 0>("M128 N64 K16 A-K  B-K ");
  run<128, 64, 16, 1, 0>("M128 N64 K16 A-MN B-K ");
  run<128, 64, 16, 1, 0>("M128 N64 K16 A-MN B-K ", 1);
  run<128, 64, 16, 0, 1>("M128 N64 K16 A-K  B-MN");
  run<128, 64, 16, 0, 1>("M128 N64 K16 A-K  B-MN", 1);
  run<128, 64, 16, 1, 1>("M128 N64 K16 A-MN B-MN");
  run<128, 96, 40, 1, 0>("M128 N96 K40 A-MN B-K ");
  run<128, 96, 40, 1, 0>("M128 N96 K40 A-MN B-K ", 1);
  return 0;
}
