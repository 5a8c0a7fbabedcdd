// Memory-model helpers shared by the persistent kernels (sm_100a PTX).
#pragma once

#include <cuda_runtime.h>

// Device-side bounds checks of the checks build (make checked: -DTCG_DEVICE_CHECKS):
// an index outside its array traps the kernel, which the host then reports as
// a CUDA error. (compute-sanitizer is not available on the GPU pool this was
// measured on; tools/gpu_checked.sh runs the GPU tests on the checks build.)
#ifdef TCG_DEVICE_CHECKS
#define TCG_CHECK(cond) \
  do {                  \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define TCG_CHECK(cond) \
  do {                  \
  } while (0)
#endif

namespace tcbdev {

constexpr unsigned kFull = 0xffffffffu;

// Launch of a persistent kernel whose CTAs wait on one another (spin on
// values, counters or queues): a cooperative launch, so the runtime either
// makes every CTA co-resident or fails at once (cudaErrorCooperativeLaunchTooLarge,
// e.g. under MPS or beside another resident kernel) instead of leaving CTAs
// unscheduled until the watchdog.
template <class Params>
inline cudaError_t launch_resident(const void* kernel, int grid, int block, size_t smem, cudaStream_t st,
                                   const Params& p) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(static_cast<unsigned>(block));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {const_cast<Params*>(&p)};
  return cudaLaunchKernelExC(&cfg, kernel, args);
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ int atom_add_relaxed(int* p, int v) {
  int old;
  asm volatile("atom.relaxed.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_relaxed(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// 64-bit morally strong accesses (single-copy atomic): the value-flow
// schedule publishes and polls the factor values themselves.
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const void* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
// a weak load that may be served by the SM's L1 (a stale copy is possible: callers validate)
__device__ __forceinline__ unsigned long long ld_cached_u64(const void* p) {
  unsigned long long v;
  asm volatile("ld.global.ca.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
// two adjacent 64-bit values, each element single-copy atomic (16-byte aligned)
__device__ __forceinline__ void ld_relaxed_v2_u64(const void* p, unsigned long long& a, unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const void* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_relaxed_sys_u64(void* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_u64(void* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acquire_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// 16-byte asynchronous global->shared copy (LDGSTS), L2 only.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
// 8-byte variant (LDGSTS through L1; sizes below 16 need .ca)
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
// 4-byte variant
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
// barrier of the T threads of one row group (named barrier `id`; a warp: __syncwarp)
template <int T>
__device__ __forceinline__ void group_sync(int id) {
  if (T == 32) __syncwarp();
  else asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(T) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

}  // namespace tcbdev
