// ubench_mma.cu -- tcgen05.mma issue/throughput calibration (development tool).
// One CTA, one thread issues NMMA MMAs (operands in smem, 128B swizzle) and waits via
// tcgen05.commit -> mbarrier; reports cycles per MMA for several shapes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1607_07395_b200/csrc -o tools/ubench_mma tools/ubench_mma.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace cabsk;

__device__ __forceinline__ uint32_t idesc_f16(int M, int N) {  // bf16 in, f32 accumulate, K-major
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

template <int KIND, int N, int NACC>
__global__ void mma_bench(long long* out, int nmma) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 0.001f * (i % 7);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc(&tbase, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (threadIdx.x == 0) {
    const uint64_t da = tc::desc_sw128(tc::smem_u32(base));
    const uint64_t db = tc::desc_sw128(tc::smem_u32(base + 32 * 1024));
    const uint32_t idesc = KIND != 1 ? tc::idesc_tf32(128, N) : idesc_f16(128, N);
    long long t0 = clock64();
    for (int i = 0; i < nmma; ++i) {
      const uint32_t d = tbase + static_cast<uint32_t>((i % NACC) * N);
      const uint64_t off = static_cast<uint64_t>((i & 3) * 2);
      if (KIND == 2) mma_tf32_ts(d, tbase + 384 + static_cast<uint32_t>((i & 7) * 8), db + off, idesc, i >= NACC ? 1u : 0u);
      else if (KIND == 0) tc::mma_tf32(d, da + off, db + off, idesc, i >= NACC ? 1u : 0u);
      else mma_f16(d, da + off, db + off, idesc, i >= NACC ? 1u : 0u);
    }
    long long t1 = clock64();
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tbase, 512);
  }
}

template <int KIND, int N, int NACC>
void run(const char* name, long long* d) {
  const int nmma = 4096;
  auto k = mma_bench<KIND, N, NACC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  k<<<1, 128, 80 * 1024>>>(d, nmma);
  long long h[2];
  cudaError_t e = cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
  const double flop = 2.0 * 128 * N * (KIND != 1 ? 8 : 16);
  printf("%-34s issue %6.1f cyc/mma, complete %6.1f cyc/mma  (%.0f flop/cyc)\n", name, (double)h[0] / nmma,
         (double)h[1] / nmma, flop * nmma / h[1]);
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run<0, 64, 1>("tf32 M128 N64  1 acc", d);
  run<0, 64, 3>("tf32 M128 N64  3 acc", d);
  run<0, 128, 1>("tf32 M128 N128 1 acc", d);
  run<0, 256, 1>("tf32 M128 N256 1 acc", d);
  run<0, 32, 1>("tf32 M128 N32  1 acc", d);
  run<2, 64, 1>("tf32 TS (A in TMEM) M128 N64", d);
  run<2, 64, 2>("tf32 TS (A in TMEM) M128 N64 2acc", d);
  run<2, 128, 1>("tf32 TS (A in TMEM) M128 N128", d);
  run<2, 32, 1>("tf32 TS (A in TMEM) M128 N32", d);
  run<1, 64, 1>("bf16 M128 N64  1 acc", d);
  run<1, 256, 1>("bf16 M128 N256 1 acc", d);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
