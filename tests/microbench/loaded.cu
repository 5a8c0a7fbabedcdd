// Loaded-latency microbenchmark: one warp measures dependent 64-bit
// ld.relaxed.gpu latency (pointer chase, L2-resident) while other warps spin
// on loads like the mode-5 poll loops. Shows how polling traffic inflates the
// L2 round trip every hand-off and gather pays.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o loaded loaded.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ldr(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

__global__ void loaded(const unsigned long long* next, int steps, const unsigned long long* noise, int nmask,
                       int lanes_polling, volatile int* stop, unsigned long long* out) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // let the pollers start
    unsigned long long t = clock64();
    while (clock64() - t < 200000) {}
    unsigned long long p = 0;
    unsigned long long t0 = clock64();
    for (int i = 0; i < steps; ++i) p = ldr(next + p);
    unsigned long long t1 = clock64();
    out[0] = (t1 - t0) / steps;
    out[1] = p;
    *stop = 1;
    return;
  }
  if (blockIdx.x == 0) return;
  const int lane = threadIdx.x & 31;
  if (lane >= lanes_polling) return;
  unsigned x = (blockIdx.x * 1315423911u) ^ (threadIdx.x * 2654435761u);
  unsigned long long acc = 0;
  while (!*stop) {
    x = x * 1664525u + 1013904223u;
    acc += ldr(noise + (x & nmask));
  }
  if (acc == 42) out[2] = acc;
}

int main() {
  const int M = 1 << 16;
  unsigned long long* nx;
  cudaMallocManaged(&nx, sizeof(unsigned long long) * M);
  for (int i = 0; i < M; ++i) nx[i] = (unsigned long long)((i * 2654435761u + 12345) % M);
  const int NZ = 1 << 21;  // 16 MB of polled words (L2 resident)
  unsigned long long* noise;
  cudaMalloc(&noise, sizeof(unsigned long long) * NZ);
  cudaMemset(noise, 0, sizeof(unsigned long long) * NZ);
  unsigned long long* out;
  cudaMallocManaged(&out, 64);
  int* stop;
  cudaMalloc(&stop, 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int ctas[] = {1, 2, 149, 445, 445, 445, 445, 445, 445};
  const int lanes[] = {32, 32, 32, 4, 12, 32, 8, 8, 8};
  const int masks[] = {NZ - 1, NZ - 1, NZ - 1, NZ - 1, NZ - 1, NZ - 1, 4095, 255, 15};
  for (int k = 0; k < 9; ++k) {
    cudaMemset(stop, 0, 4);
    loaded<<<ctas[k], 256>>>(nx, 20000, noise, masks[k], lanes[k], stop, out);
    cudaDeviceSynchronize();
    printf("pollers: %4d CTAs x 8 warps x %2d lanes on %7d words -> dependent ld.relaxed.gpu: %llu cycles\n",
           ctas[k] - 1, lanes[k], masks[k] + 1, out[0]);
  }
  printf("err=%s sms=%d\n", cudaGetErrorString(cudaGetLastError()), sms);
  return 0;
}
