// ubench_issue2.cu -- MMA issue strategies for the residual / k-means MMA loops: how fast can
// one warp feed the tensor pipe with the 3xTF32 TS sequence (per 8-wide k step: Fh.Gh, Fh.Gl,
// Fl.Gh; G in 32-wide K chunks of a 4-slot ring)?  Reports cycles per MMA (64 = full rate for
// M128 N128 K8 tf32).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1607_07395_b200/csrc -o tools/ubench_issue2 tools/ubench_issue2.cu
#include <cstdio>
#include <cstdint>
#include "tc_ptx.cuh"

using namespace cabsk;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.b32 %0, 1, 0, P;\n}\n" : "=r"(pred));
  return pred != 0;
}

constexpr uint32_t kAtom = 16384;

template <int STRAT>
__global__ void bench(long long* out, int ntiles, int ksteps, int kp) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 0.001f * (i % 7);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tc::tmem_alloc(&tbase_s, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tbase_s;
  const uint32_t idesc = tc::idesc_tf32(128, 128);
  const uint64_t dgh0 = tc::desc_sw128(tc::smem_u32(base)), dgl0 = tc::desc_sw128(tc::smem_u32(base + 4 * kAtom));
  const int nch = (ksteps + 3) / 4;
  long long t0 = clock64();
  if (warp == 0) {
    if (STRAT == 0) {  // lane 0 only, runtime k loop (the current kernel)
      if (lane == 0) {
        int64_t j = 0;
        for (int t = 0; t < ntiles; ++t) {
          const uint32_t d = tmem + static_cast<uint32_t>((t & 1) * 128);
          const uint32_t fcol = tmem + 256;
          for (int c = 0; c < nch; ++c, ++j) {
            const int sg = static_cast<int>(j & 3);
            const int kk1 = (4 * c + 4 < ksteps) ? 4 * c + 4 : ksteps;
            for (int kk = 4 * c; kk < kk1; ++kk) {
              const uint64_t off = static_cast<uint64_t>((kk & 3) * 2);
              const uint64_t slot = static_cast<uint64_t>(sg) * (kAtom >> 4);
              const uint32_t fh = fcol + static_cast<uint32_t>(kk * 8), fl = fh + static_cast<uint32_t>(kp);
              mma_ts(d, fh, dgh0 + slot + off, idesc, kk > 0 ? 1u : 0u);
              mma_ts(d, fh, dgl0 + slot + off, idesc, 1u);
              mma_ts(d, fl, dgh0 + slot + off, idesc, 1u);
            }
          }
        }
      }
    } else {  // whole warp runs the loop (uniform), one elected lane issues; k steps unrolled
      int64_t j = 0;
      for (int t = 0; t < ntiles; ++t) {
        const uint32_t d = tmem + static_cast<uint32_t>((t & 1) * 128);
        const uint32_t fcol = tmem + 256;
        for (int c = 0; c < nch; ++c, ++j) {
          const uint64_t slot = static_cast<uint64_t>(j & 3) * (kAtom >> 4);
          const uint64_t bh = dgh0 + slot, bl = dgl0 + slot;
          const uint32_t fh0 = fcol + static_cast<uint32_t>(c * 32);
          const int nk = ksteps - 4 * c < 4 ? ksteps - 4 * c : 4;
          if (STRAT == 1) {
            if (elect_one()) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                if (q < nk) {
                  const uint32_t fh = fh0 + 8 * q;
                  mma_ts(d, fh, bh + 2 * q, idesc, (c | q) ? 1u : 0u);
                  mma_ts(d, fh, bl + 2 * q, idesc, 1u);
                  mma_ts(d, fh + kp, bh + 2 * q, idesc, 1u);
                }
              }
            }
            __syncwarp();
          } else {  // STRAT 2: lane 0 only but unrolled k steps
            if (lane == 0) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                if (q < nk) {
                  const uint32_t fh = fh0 + 8 * q;
                  mma_ts(d, fh, bh + 2 * q, idesc, (c | q) ? 1u : 0u);
                  mma_ts(d, fh, bl + 2 * q, idesc, 1u);
                  mma_ts(d, fh + kp, bh + 2 * q, idesc, 1u);
                }
              }
            }
            __syncwarp();
          }
        }
      }
    }
    if (lane == 0) {
      tc::mma_commit(&bar);
      tc::mbar_wait(&bar, 0);
      out[0] = clock64() - t0;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem, 512);
  }
}

template <int S>
void run(const char* name, long long* d, int ksteps) {
  const int ntiles = 64;
  cudaFuncSetAttribute(bench<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  bench<S><<<1, 128, 140 * 1024>>>(d, ntiles, ksteps, 128);
  long long h;
  cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  printf("%-40s ksteps=%2d: %6.1f cyc per MMA\n", name, ksteps, (double)h / (ntiles * ksteps * 3));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  for (int ks : {13, 16}) {
    run<0>("lane 0, runtime k loop", d, ks);
    run<1>("warp-uniform, elect_one, unrolled k", d, ks);
    run<2>("lane 0, unrolled k", d, ks);
  }
  return 0;
}
