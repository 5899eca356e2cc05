// tc_probe3.cu -- can ONE shared-memory copy of an operand serve tcgen05.mma
// kind::tf32 both as a K-major and as an MN-major operand?  (development tool
// for SURVEY 8(f) f2)
//
// A tensor T[r][c] (c contiguous) is stored in the SWIZZLE_128B_BASE32B
// arrangement (atoms of 4 rows x 32 elements = 512 B, 32-B granule ^= r % 4,
// atoms ordered [r/4][c/32]).  Round 1 found that this is the MN-major
// arrangement (MN = c, K = r).  Here T is used as a K-major operand (MN = r,
// K = c) with layout type 1 and several (LBO, SBO, k-advance) conventions.
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
// T[r][c], C = padded contiguous extent (multiple of 32): float index
__host__ __device__ inline int off32(int r, int c, int C) {
  const int NA = C / 32;
  const int byte_in = (r & 3) * 128 + (c & 31) * 4;
  const int sw = byte_in ^ (((byte_in >> 7) & 3) << 5);
  return (((r >> 2) * NA + (c >> 5)) * 512 + sw) >> 2;
}
// K-major no swizzle (known good): core 8 rows x 4 K = 128 B
__host__ __device__ inline int off_kmaj(int r, int k, int KG) { return ((r >> 3) * KG + (k >> 2)) * 32 + (r & 7) * 4 + (k & 3); }

// variant v for a K-major operand stored with off32(mn, k, KP):
//   v = 0: LBO = 512 (K-atom step), SBO = NA*512 (4-row group step), k-advance 32 B in the atom
//   v = 1: LBO = NA*512, SBO = 512
//   v = 2: LBO = 16 (ignored), SBO = NA*512
//   v = 3: LBO = 16, SBO = 2*NA*512 (8-row group semantics)
__device__ __forceinline__ uint64_t kdesc(uint32_t base, int ks, int KP, int v) {
  const int NA = KP / 32;
  const uint32_t addr = base + (ks >> 2) * 512 + (ks & 3) * 32;
  switch (v) {
    case 0: return make_desc(addr, 512, NA * 512, 1);
    case 1: return make_desc(addr, NA * 512, 512, 1);
    case 2: return make_desc(addr, 16, NA * 512, 1);
    default: return make_desc(addr, 16, 2 * NA * 512, 1);
  }
}

// MODE 0: A K-major (off32), B K-major no swizzle.   MODE 1: A K-major no swizzle, B K-major (off32).
// MODE 2: A MN-major off32 (rows k), B K-major off32 -- both from "row = k" / "row = n" storage
template <int M, int N, int K, int MODE>
__global__ void probe(const float* A, const float* B, float* D, int v) {
  constexpr int KP = (K + 31) / 32 * 32;
  constexpr int MP = (M + 31) / 32 * 32;
  constexpr int NA_ = M * KP > MP * K ? M * KP : MP * ((K + 3) / 4 * 4);
  extern __shared__ __align__(1024) float dyn[];
  float* sA = dyn;
  float* sB = dyn + NA_;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  for (int e = tid; e < NA_; e += blockDim.x) sA[e] = 0.f;
  for (int e = tid; e < N * KP; e += blockDim.x) sB[e] = 0.f;
  __syncthreads();
  for (int e = tid; e < M * K; e += blockDim.x) {
    const int m = e / K, k = e % K;
    if (MODE == 0) sA[off32(m, k, KP)] = A[e];
    else if (MODE == 1) sA[off_kmaj(m, k, KP / 4)] = A[e];
    else sA[off32(k, m, MP)] = A[e];          // A^T stored rows k, contiguous m: MN-major A
  }
  for (int e = tid; e < K * N; e += blockDim.x) {
    const int k = e / N, n = e % N;
    if (MODE == 0) sB[off_kmaj(n, k, KP / 4)] = B[e];
    else sB[off32(n, k, KP)] = B[e];
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
    const uint32_t idesc = make_idesc(M, N, MODE == 2 ? 1 : 0, 0);
    for (int ks = 0; ks < K / 8; ++ks) {
      uint64_t ad, bd;
      if (MODE == 0) {
        ad = kdesc(smem_u32(sA), ks, KP, v);
        bd = make_desc(smem_u32(sB) + ks * 2 * 128, 128, (KP / 4) * 128, 0);
      } else if (MODE == 1) {
        ad = make_desc(smem_u32(sA) + ks * 2 * 128, 128, (KP / 4) * 128, 0);
        bd = kdesc(smem_u32(sB), ks, KP, v);
      } else {
        // MN-major A (round-1 convention): LBO = MN-atom step 512, SBO = K-atom step (MP/32)*512; 8 k = 2 atoms
        const uint32_t sbo = (MP / 32) * 512;
        ad = make_desc(smem_u32(sA) + ks * 2 * sbo, 512, sbo, 1);
        bd = kdesc(smem_u32(sB), ks, KP, v);
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

template <int M, int N, int K, int MODE>
int run(const char* name, int v) {
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
  constexpr int KP = (K + 31) / 32 * 32, MP = (M + 31) / 32 * 32;
  constexpr int NA_ = M * KP > MP * K ? M * KP : MP * ((K + 3) / 4 * 4);
  const int smem = (NA_ + N * KP) * 4;
  CK(cudaFuncSetAttribute(probe<M, N, K, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe<M, N, K, MODE><<<1, 128, smem>>>(dA, dB, dD, v);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) bad += D[m * N + n] != R[m * N + n];
  printf("%s v=%d: %s (%d / %d mismatches)\n", name, v, bad ? "FAIL" : "ok", bad, M * N);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return bad;
}

int main(int argc, char** argv) {
  // one (case, variant) per process: a bad descriptor faults the context
  const int c = argc > 1 ? atoi(argv[1]) : 0, v = argc > 2 ? atoi(argv[2]) : 0;
  switch (c) {
    case 0: return run<128, 64, 32, 0>("A K-major SW32B  K=32 ", v);
    case 1: return run<128, 64, 64, 0>("A K-major SW32B  K=64 ", v);
    case 2: return run<128, 80, 80, 0>("A K-major SW32B  K=80 N=80", v);
    case 3: return run<128, 64, 64, 1>("B K-major SW32B  K=64 ", v);
    case 4: return run<128, 80, 80, 1>("B K-major SW32B  K=80 N=80", v);
    case 5: return run<128, 64, 64, 2>("A MN-major SW32B + B K-major SW32B K=64", v);
    default: return run<128, 80, 128, 2>("A MN-major SW32B + B K-major SW32B K=128 N=80", v);
  }
}
