// ubench_commit.cu -- does tcgen05.commit between MMA groups throttle the tensor pipe?
// One CTA, one thread issues NMMA tf32 MMAs (M128 N128 K8, TS or SS), with a
// tcgen05.commit -> mbarrier after every `group` MMAs (nobody waits on it except at the end).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1607_07395_b200/csrc -o tools/ubench_commit tools/ubench_commit.cu
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

template <bool TS>
__global__ void bench(long long* out, int nmma, int group, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[8];
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 0.001f * (i % 7);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) tc::mbar_init(&bar[i], 1);
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
    const uint32_t idesc = tc::idesc_tf32(128, 128);
    long long t0 = clock64();
    int nc = 0, cnt = group;
    for (int i = 0; i < nmma; ++i) {
      const uint32_t d = tbase;
      const uint64_t off = static_cast<uint64_t>((i & 3) * 2);
      if (TS) mma_tf32_ts(d, tbase + 256 + static_cast<uint32_t>((i & 7) * 8), db + off, idesc, i > 0 ? 1u : 0u);
      else tc::mma_tf32(d, da + off, db + off, idesc, i > 0 ? 1u : 0u);
      if (--cnt == 0) {
        cnt = group;
        tc::mma_commit(&bar[nc & 7]);
        ++nc;
        if (mode == 1) tc::fence_after_sync();
      }
    }
    long long t1 = clock64();
    tc::mma_commit(&bar[nc & 7]);
    // wait for the last phase of that barrier: count the commits that went to it
    const int uses = nc / 8 + ((nc & 7) >= (nc & 7) ? 1 : 0);
    (void)uses;
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  __syncthreads();
  // drain: wait for all MMAs via a fresh commit on a dedicated barrier
  __shared__ uint64_t fin;
  if (threadIdx.x == 0) {
    tc::mbar_init(&fin, 1);
    tc::mbar_fence_init();
    long long t0 = clock64();
    tc::mma_commit(&fin);
    tc::mbar_wait(&fin, 0);
    out[2] = clock64() - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tbase, 512);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  const int nmma = 3072;
  for (int ts = 0; ts < 2; ++ts)
    for (int mode = 0; mode < 2; ++mode)
      for (int group : {0, 1, 3, 12, 39}) {
        auto k = ts ? bench<true> : bench<false>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
        k<<<1, 128, 80 * 1024>>>(d, nmma, group, mode);
        long long h[3];
        cudaError_t e = cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        printf("%s fence=%d commit every %2d: issue %6.1f cyc/mma, total %6.1f cyc/mma\n", ts ? "TS" : "SS", mode,
               group, (double)h[0] / nmma, (double)(h[0] + h[2]) / nmma);
      }
  return 0;
}
