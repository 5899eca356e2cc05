// ffma2_probe.cu -- FFMA vs packed FFMA2 (fma.rn.f32x2) throughput on this B200,
// 8 and 16 warps per SM, independent chains; CUDA-event timed.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void ffma2(float2& d, float2 a, float2 b) {
  unsigned long long dd = *reinterpret_cast<unsigned long long*>(&d);
  asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(dd)
               : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  d = *reinterpret_cast<float2*>(&dd);
}

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

template <int CH>
__global__ void k_ffma2(float* out, int iters, float a, float b) {
  float2 v[CH];
  const float2 aa = make_float2(a, a * 0.5f), bb = make_float2(b, b);
#pragma unroll
  for (int i = 0; i < CH; ++i) v[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      unsigned long long dd = *reinterpret_cast<unsigned long long*>(&v[i]);
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(dd)
                   : "l"(*reinterpret_cast<const unsigned long long*>(&aa)),
                     "l"(*reinterpret_cast<const unsigned long long*>(&bb)));
      v[i] = *reinterpret_cast<float2*>(&dd);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += v[i].x + v[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, nsm * 8 * 1024 * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int it = 20000;
  for (int bpsm : {1, 2, 4}) {
    const int blocks = nsm * bpsm, threads = 256;
    float ms;
    k_ffma<16><<<blocks, threads>>>(out, 100, 0.999f, 0.001f);
    cudaEventRecord(e0);
    k_ffma<16><<<blocks, threads>>>(out, it, 0.999f, 0.001f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * it * double(blocks) * threads;
    printf("{\"probe\":\"ffma\",\"warps_per_sm\":%d,\"tflops\":%.2f}\n", bpsm * 8, fl / ms * 1e-9);
    k_ffma2<8><<<blocks, threads>>>(out, 100, 0.999f, 0.001f);
    cudaEventRecord(e0);
    k_ffma2<8><<<blocks, threads>>>(out, it, 0.999f, 0.001f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 16 * it * double(blocks) * threads;
    printf("{\"probe\":\"ffma2\",\"warps_per_sm\":%d,\"tflops\":%.2f}\n", bpsm * 8, fl / ms * 1e-9);
    k_ffma2<16><<<blocks, threads>>>(out, 100, 0.999f, 0.001f);
    cudaEventRecord(e0);
    k_ffma2<16><<<blocks, threads>>>(out, it, 0.999f, 0.001f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 32 * it * double(blocks) * threads;
    printf("{\"probe\":\"ffma2_16ch\",\"warps_per_sm\":%d,\"tflops\":%.2f}\n", bpsm * 8, fl / ms * 1e-9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
