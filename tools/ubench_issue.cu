// ubench_issue.cu -- tensor-pipe throughput of a single MMA-issuing thread while the other
// warps of the CTA spin on mbarrier waits (the situation of the warp-specialised kernels).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1607_07395_b200/csrc -o tools/ubench_issue tools/ubench_issue.cu
#include <cstdio>
#include <cstdint>
#include "tc_ptx.cuh"

using namespace cabsk;

__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

// spin: 0 = idle warps exit, 1 = spin on try_wait, 2 = spin with nanosleep backoff
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.b32 %0, 1, 0, P;\n}\n" : "=r"(pred));
  return pred != 0;
}

__global__ void bench(long long* out, int nk, int per, int spin, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, never;
  __shared__ uint32_t tbase;
  __shared__ volatile int done;
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 0.001f * (i % 7);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_init(&never, 1);
    done = 0;
    tc::mbar_fence_init();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 1) tc::tmem_alloc(&tbase, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (warp == 1 && mode >= 10) {
    const uint64_t db = tc::desc_sw128(tc::smem_u32(base + 64 * 1024));
    const uint32_t idesc = tc::idesc_tf32(128, 128);
    long long t0 = clock64();
    for (int k = 0; k < nk; ++k) {
      const uint64_t off = static_cast<uint64_t>((k & 3) * 2) + static_cast<uint64_t>((k >> 2) & 3) * (16384 >> 4);
      const uint32_t a = tbase + 256 + static_cast<uint32_t>((k & 15) * 8);
      if (mode == 10) {
        for (int r = 0; r < per; ++r)
          if (elect_one()) mma_tf32_ts(tbase, a + 128 * (r == 2), db + off, idesc, (k > 1 || r) ? 1u : 0u);
      } else {
        if (elect_one()) {
          for (int r = 0; r < per; ++r) mma_tf32_ts(tbase, a + 128 * (r == 2), db + off, idesc, (k > 1 || r) ? 1u : 0u);
        }
      }
      __syncwarp();
    }
    if (elect_one()) {
      tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
    if (lane == 0) {
      out[0] = clock64() - t0;
      done = 1;
      tc::mbar_arrive(&never);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint64_t db = tc::desc_sw128(tc::smem_u32(base + 64 * 1024));
      const uint32_t idesc = tc::idesc_tf32(128, mode == 6 ? 256 : 128);
      long long t0 = clock64();
      for (int k = 0; k < nk; ++k) {
        const bool va = mode == 1 || mode >= 4, vb_in = mode == 2 || mode >= 4, vb_x = mode == 3 || mode >= 4;
        const uint64_t off = (vb_in ? static_cast<uint64_t>((k & 3) * 2) : 0) +
                             (vb_x ? static_cast<uint64_t>((k >> 2) & 3) * (16384 >> 4) : 0);
        const uint32_t a = tbase + 256 + (va ? static_cast<uint32_t>((k & 15) * 8) : 0u);
        const uint32_t dd = tbase + (mode == 5 ? static_cast<uint32_t>((k & 1) * 128) : 0u);
        for (int r = 0; r < per; ++r) mma_tf32_ts(dd, a + 128 * (r == 2), db + off, idesc, (k > 1 || r) ? 1u : 0u);
      }
      tc::mma_commit(&bar);
      tc::mbar_wait(&bar, 0);
      out[0] = clock64() - t0;
      done = 1;
      tc::mbar_arrive(&never);
    }
  } else if (spin == 1) {
    tc::mbar_wait(&never, 0);
  } else if (spin == 2) {
    while (!done) __nanosleep(100);
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tbase, 512);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  const char* names[] = {"A,B fixed", "A varies", "B varies in atom", "B varies across atoms", "both vary",
                         "both vary, 2 accumulators", "both vary, N=256", "", "", "", "warp-uniform loop, elect per MMA",
                         "warp-uniform loop, elect per k step"};
  for (int mode : {0, 4, 10, 11})
    for (int per : {1, 3}) {
      const int nk = 1024;
      bench<<<1, 352, 140 * 1024>>>(d, nk, per, 0, mode);
      long long h;
      cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      printf("%-28s mmas/kstep=%d: %7.1f cyc per k step, %6.1f per MMA\n", names[mode], per, (double)h / nk,
             (double)h / nk / per);
    }
  return 0;
}
