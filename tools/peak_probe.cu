// peak_probe.cu -- measured throughput of the pipes the K1 kernel can use on this B200:
//   FFMA (FP32 CUDA cores), mma.sync m16n8k8 TF32 (legacy tensor path), MUFU.TANH.
// Every SM runs 8 warps of independent chains; time with CUDA events.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CH>
__global__ void k_ffma(float* out, int iters, float a, float b) {
  float v[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) v[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) v[i] = fmaf(v[i], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_mma_tf32(float* out, int iters) {
  uint32_t a[4], b[2];
  float c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
  b[0] = __float_as_uint(0.5f); b[1] = __float_as_uint(0.25f);
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) c[j][i] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_tanh(float* out, int iters) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 1e-4f + i * 0.1f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = tanhf(v[i]);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const int blocks = nsm * 4, threads = 256;
  float* out;
  CK(cudaMalloc(&out, blocks * threads * sizeof(float)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // warm up
  k_ffma<16><<<blocks, threads>>>(out, 1000, 0.999f, 0.001f);
  CK(cudaDeviceSynchronize());
  const int it1 = 20000;
  cudaEventRecord(e0);
  k_ffma<16><<<blocks, threads>>>(out, it1, 0.999f, 0.001f);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 16 * it1 * (double)blocks * threads;
  printf("{\"ffma_tflops\": %.2f, ", fl / (ms * 1e-3) / 1e12);
  const int it2 = 20000;
  k_mma_tf32<<<blocks, threads>>>(out, 100);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  k_mma_tf32<<<blocks, threads>>>(out, it2);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  fl = 2.0 * 16 * 8 * 8 * 4 * (double)it2 * blocks * (threads / 32);
  printf("\"mma_sync_tf32_tflops\": %.2f, ", fl / (ms * 1e-3) / 1e12);
  const int it3 = 5000;
  k_tanh<<<blocks, threads>>>(out, 100);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  k_tanh<<<blocks, threads>>>(out, it3);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  printf("\"tanhf_gops\": %.2f, \"sms\": %d, \"clock_khz_attr\": %d}\n", 8.0 * it3 * blocks * threads / (ms * 1e-3) / 1e9, nsm, clk);
  return 0;
}
