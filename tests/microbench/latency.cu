// Latency microbenchmarks for the design of the persistent IC(k) kernel.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o latency latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long clk() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}

// 1. pointer chase over a buffer (L2-resident): cycles per dependent load
__global__ void chase(const int* next, int steps, unsigned long long* out, int* sink) {
  int p = 0;
  unsigned long long t0 = clk();
  for (int i = 0; i < steps; ++i) p = __ldcg(next + p);
  unsigned long long t1 = clk();
  out[0] = (t1 - t0) / steps;
  sink[0] = p;
}

// 2. same-CTA producer/consumer: warp 0 writes a value to global, fences at
// CTA scope, sets a smem flag; warp 1 waits and loads it. Ping-pong N times.
__global__ void pingpong_cta(double* data, int rounds, unsigned long long* out, int mode) {
  __shared__ volatile int flag;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  unsigned long long t0 = clk();
  double acc = 0;
  for (int r = 0; r < rounds; ++r) {
    if (w == (r & 1)) {
      if (r > 0) {
        while (flag != r) {}
        __threadfence_block();
        acc += (mode == 0) ? data[lane + 64 * r - 64] : __ldcg(data + lane + 64 * r - 64);
      }
      data[lane + 64 * r] = acc + r;
      if (mode == 2) __threadfence(); else __threadfence_block();
      __syncwarp();
      if (lane == 0) flag = r + 1;
    }
  }
  unsigned long long t1 = clk();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / rounds;
  if (acc == 1234.5) data[0] = acc;
}

// 3. cross-SM ping-pong through global flags (two CTAs)
__global__ void pingpong_gpu(double* data, int* flags, int rounds, unsigned long long* out) {
  const int b = blockIdx.x, lane = threadIdx.x;
  unsigned long long t0 = clk();
  double acc = 0;
  for (int r = 0; r < rounds; ++r) {
    if (b == (r & 1)) {
      if (r > 0) {
        if (lane == 0) {
          int v;
          do { asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flags) : "memory"); } while (v != r);
        }
        __syncwarp();
        acc += data[lane + 64 * r - 64];
      }
      data[lane + 64 * r] = acc + r;
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(flags), "r"(r + 1) : "memory");
      }
      __syncwarp();
    }
  }
  unsigned long long t1 = clk();
  if (threadIdx.x == 0 && b == 0) out[0] = (t1 - t0) / rounds;
  if (acc == 1234.5) data[0] = acc;
}

// 4. atomic round trip latency (single thread)
__global__ void atom_lat(int* x, int n, unsigned long long* out) {
  int v = 0;
  unsigned long long t0 = clk();
  for (int i = 0; i < n; ++i) v += atomicAdd(x + (v & 1), 1);
  unsigned long long t1 = clk();
  out[0] = (t1 - t0) / n;
  if (v == -1) x[5] = v;
}

// 5. fences
__global__ void fence_lat(double* data, int n, unsigned long long* out, int kind) {
  unsigned long long t0 = clk();
  for (int i = 0; i < n; ++i) {
    data[threadIdx.x + 32 * (i & 7)] = i;
    if (kind == 0) __threadfence_block();
    else __threadfence();
  }
  unsigned long long t1 = clk();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / n;
}

// 6. store then load same address, same thread (write->read hazard)
__global__ void st_ld(double* data, int n, unsigned long long* out) {
  double acc = 1.0;
  unsigned long long t0 = clk();
  for (int i = 0; i < n; ++i) {
    data[threadIdx.x + 32 * (i & 15)] = acc;
    acc = data[threadIdx.x + 32 * ((i + 1) & 15)] + 1.0;
  }
  unsigned long long t1 = clk();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / n;
  if (acc == -1) data[0] = acc;
}

// 7. cross-SM hand-off through the value itself (mode 5): round r's consumer
// polls data[r-1] with 64-bit ld.relaxed.gpu until it is no longer the
// marker, then stores data[r] with st.relaxed.gpu. One round = one hand-off.
__global__ void flow_pingpong(unsigned long long* data, int rounds, unsigned long long* out) {
  const int b = blockIdx.x;
  unsigned long long t0 = clk();
  unsigned long long acc = 0;
  for (int r = 0; r < rounds; ++r) {
    if (b == (r & 1) && threadIdx.x == 0) {
      if (r > 0) {
        unsigned long long v;
        do { asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(data + r - 1)); } while (v == ~0ull);
        acc += v;
      }
      asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(data + r), "l"(acc + r) : "memory");
    }
  }
  unsigned long long t1 = clk();
  if (threadIdx.x == 0 && b == 0) out[0] = (t1 - t0) / rounds;
  if (acc == 12345) data[0] = acc;
}

// 8. dependent chase with 64-bit ld.relaxed.gpu (the mode-5 gather load)
__global__ void chase_strong(const unsigned long long* next, int steps, unsigned long long* out, int* sink) {
  unsigned long long p = 0;
  unsigned long long t0 = clk();
  for (int i = 0; i < steps; ++i)
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(p) : "l"(next + p));
  unsigned long long t1 = clk();
  out[0] = (t1 - t0) / steps;
  sink[0] = static_cast<int>(p);
}

int main() {
  unsigned long long* out;
  cudaMallocManaged(&out, 64);
  // 1
  const int N = 1 << 22;
  int* next;
  cudaMallocManaged(&next, sizeof(int) * N);
  for (int i = 0; i < N; ++i) next[i] = (int)((i * 2654435761u + 12345) % N);
  int* sink;
  cudaMallocManaged(&sink, 64);
  chase<<<1, 1>>>(next, 1000, out, sink);
  chase<<<1, 1>>>(next, 20000, out, sink);
  cudaDeviceSynchronize();
  printf("L2/DRAM pointer chase (16 MB): %llu cycles/load\n", out[0]);
  const int M = 1 << 16;  // 256 KB: L2 resident after warm-up
  for (int i = 0; i < M; ++i) next[i] = (int)((i * 2654435761u + 12345) % M);
  chase<<<1, 1>>>(next, 20000, out, sink);
  chase<<<1, 1>>>(next, 20000, out, sink);
  cudaDeviceSynchronize();
  printf("L2 pointer chase (256 KB, ldcg): %llu cycles/load\n", out[0]);
  double* data;
  cudaMalloc(&data, sizeof(double) * 64 * 4096);
  const char* m2[3] = {"ld default, fence.cta", "ld.cg, fence.cta", "ld default, fence.gpu"};
  for (int mode = 0; mode < 3; ++mode) {
    pingpong_cta<<<1, 64>>>(data, 2000, out, mode);
    cudaDeviceSynchronize();
    printf("same-CTA write->flag->read round (%s): %llu cycles\n", m2[mode], out[0]);
  }
  int* flags;
  cudaMalloc(&flags, 64);
  cudaMemset(flags, 0, 64);
  pingpong_gpu<<<2, 32>>>(data, flags, 2000, out);
  cudaDeviceSynchronize();
  printf("cross-SM write->fence->flag->read round: %llu cycles\n", out[0]);
  {
    const int R = 4000;
    unsigned long long* d;
    cudaMalloc(&d, sizeof(unsigned long long) * R);
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(d, 0xff, sizeof(unsigned long long) * R);
      flow_pingpong<<<2, 32>>>(d, R, out);
      cudaDeviceSynchronize();
    }
    printf("cross-SM value hand-off (st.relaxed -> ld.relaxed poll): %llu cycles/round\n", out[0]);
    unsigned long long* nx;
    cudaMallocManaged(&nx, sizeof(unsigned long long) * M);
    for (int i = 0; i < M; ++i) nx[i] = (unsigned long long)((i * 2654435761u + 12345) % M);
    chase_strong<<<1, 1>>>(nx, 20000, out, sink);
    chase_strong<<<1, 1>>>(nx, 20000, out, sink);
    cudaDeviceSynchronize();
    printf("L2 pointer chase (512 KB, ld.relaxed.gpu.b64): %llu cycles/load\n", out[0]);
  }
  int* x;
  cudaMalloc(&x, 64);
  atom_lat<<<1, 1>>>(x, 10000, out);
  cudaDeviceSynchronize();
  printf("atomicAdd round trip: %llu cycles\n", out[0]);
  fence_lat<<<1, 32>>>(data, 10000, out, 0);
  cudaDeviceSynchronize();
  printf("store + threadfence_block: %llu cycles\n", out[0]);
  fence_lat<<<1, 32>>>(data, 10000, out, 1);
  cudaDeviceSynchronize();
  printf("store + threadfence (gpu): %llu cycles\n", out[0]);
  st_ld<<<1, 32>>>(data, 10000, out);
  cudaDeviceSynchronize();
  printf("store then dependent load (16-line ring): %llu cycles/iter\n", out[0]);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("clock attr %d kHz; err=%s\n", clk_khz, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
