// sample_gather.cu -- S1 pilot indices and the S2/S3/S9 gathers
// C = A(:,J), R = A(I,:), W = A(I,J).  Gathers are bit-exact copies.
#include "common.cuh"
#include "kernels.cuh"
#include "philox.cuh"

namespace cabsk {

constexpr int kHashBits = 12;
constexpr int kHashCap = 1 << kHashBits;  // >= 4 * CABS_KMAX / 1 load factor <= 0.25
constexpr uint32_t kEmpty = 0xFFFFFFFFu;

// ---------------------------------------------------------------- S1: Floyd
// One warp per (N, k, tag) job.  Lane 0 runs Floyd's algorithm sequentially (the
// word stream is inherently sequential: rejections consume words), keeping the
// chosen set in a shared-memory hash table; the warp then rank-sorts the result.
struct FloydJob {
  int64_t N;
  int32_t k;
  uint32_t tag;
  int64_t* out;
};

__global__ void __launch_bounds__(64) floyd_kernel(FloydJob j0, FloydJob j1, uint64_t seed) {
  __shared__ uint32_t table[2][kHashCap];
  __shared__ uint32_t vals[2][CABS_KMAX];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const FloydJob job = w == 0 ? j0 : j1;
  if (job.out == nullptr || job.k <= 0) return;
  uint32_t* tab = table[w];
  uint32_t* val = vals[w];
  for (int i = lane; i < kHashCap; i += 32) tab[i] = kEmpty;
  __syncwarp();
  if (lane == 0) {
    WordStream st(seed, job.tag);
    int cnt = 0;
    for (int64_t jj = job.N - job.k; jj < job.N; ++jj) {
      uint32_t t = static_cast<uint32_t>(lemire_bounded(st, static_cast<uint64_t>(jj) + 1));
      // insert t, or jj if t is already present
      uint32_t h = (t * 2654435761u) >> (32 - kHashBits);
      bool present = false;
      while (tab[h] != kEmpty) {
        if (tab[h] == t) { present = true; break; }
        h = (h + 1) & (kHashCap - 1);
      }
      uint32_t x = present ? static_cast<uint32_t>(jj) : t;
      if (present) {  // jj is never present (all earlier values are < jj)
        h = (x * 2654435761u) >> (32 - kHashBits);
        while (tab[h] != kEmpty) h = (h + 1) & (kHashCap - 1);
      }
      tab[h] = x;
      val[cnt++] = x;
    }
  }
  __syncwarp();
  // rank sort (values distinct)
  for (int e = lane; e < job.k; e += 32) {
    uint32_t v = val[e];
    int rank = 0;
    for (int j = 0; j < job.k; ++j) rank += val[j] < v;
    job.out[rank] = static_cast<int64_t>(v);
  }
}

int launch_floyd2(int64_t N0, int32_t k0, uint32_t tag0, int64_t* out0, int64_t N1, int32_t k1,
                  uint32_t tag1, int64_t* out1, uint64_t seed, cudaStream_t st) {
  FloydJob a{N0, k0, tag0, out0}, b{N1, k1, tag1, out1};
  note_launch();
  floyd_kernel<<<1, 64, 0, st>>>(a, b, seed);
  return 0;
}

__global__ void philox_blocks_kernel(uint64_t seed, uint32_t tag, uint64_t start, int64_t count,
                                     uint32_t* out) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= count) return;
  uint64_t c = start + static_cast<uint64_t>(b);
  uint4 r = philox4x32_10(make_uint4(static_cast<uint32_t>(c), static_cast<uint32_t>(c >> 32), tag, 0u),
                          seed_key(seed));
  reinterpret_cast<uint4*>(out)[b] = r;
}

void launch_philox_blocks(uint64_t seed, uint32_t tag, uint64_t start, int64_t count, uint32_t* out,
                          cudaStream_t st) {
  if (count <= 0) return;
  note_launch();
  philox_blocks_kernel<<<static_cast<unsigned>(ceil_div(count, 256)), 256, 0, st>>>(seed, tag, start, count,
                                                                                    out);
}

// ---------------------------------------------------------------- index validation
// For externally supplied index sets (cabs_sketch): range and distinctness.
__global__ void validate_idx_kernel(const int64_t* idx, int32_t k, int64_t N, void* ws) {
  for (int a = threadIdx.x; a < k; a += blockDim.x) {
    int64_t v = idx[a];
    if (v < 0 || v >= N) set_status(ws, CABS_DEV_RANGE);
    for (int b = a + 1; b < k; ++b)
      if (idx[b] == v) set_status(ws, CABS_DEV_DUPLICATE);
  }
}

void launch_validate_idx(const int64_t* idx, int32_t k, int64_t N, void* ws, cudaStream_t st) {
  note_launch();
  validate_idx_kernel<<<1, 256, 0, st>>>(idx, k, N, ws);
}

// ---------------------------------------------------------------- S2: row gather
// R[i, :] = A[I[i] - row_begin, :] for the rows this rank owns.  Contiguous row
// copies: 128-bit vectorised when alignment allows.
__global__ void gather_rows_kernel(const float* __restrict__ A, int64_t lda, int64_t row_begin,
                                   int64_t row_end, const int64_t* __restrict__ I, int64_t n,
                                   float* __restrict__ R, int64_t ldr, bool vec4, void* ws) {
  const int i = blockIdx.y;
  const int64_t gi = I[i];
  if (gi < row_begin || gi >= row_end) return;
  const float* src = A + (gi - row_begin) * lda;
  float* dst = R + static_cast<int64_t>(i) * ldr;
  bool bad = false;
  if (vec4) {
    const int64_t n4 = n >> 2;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n4; c += (int64_t)gridDim.x * blockDim.x) {
      float4 v = __ldg(reinterpret_cast<const float4*>(src) + c);
      bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
      reinterpret_cast<float4*>(dst)[c] = v;
    }
    for (int64_t c = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
         c += (int64_t)gridDim.x * blockDim.x) {
      float v = src[c];
      bad |= !isfinite(v);
      dst[c] = v;
    }
  } else {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
      float v = src[c];
      bad |= !isfinite(v);
      dst[c] = v;
    }
  }
  if (bad) set_status(ws, CABS_DEV_NONFINITE);
}

void launch_gather_rows(const float* A, int64_t lda, int64_t row_begin, int64_t row_end, const int64_t* I,
                        int32_t k, int64_t n, float* R, int64_t ldr, void* ws, cudaStream_t st) {
  bool vec4 = (lda % 4 == 0) && (ldr % 4 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0) &&
              ((reinterpret_cast<uintptr_t>(R) & 15) == 0);
  int64_t per = vec4 ? ceil_div(n, 4) : n;
  int gx = static_cast<int>(ceil_div(per, 256));
  if (gx > 64) gx = 64;
  if (gx < 1) gx = 1;
  dim3 grid(gx, k);
  note_launch();
  gather_rows_kernel<<<grid, 256, 0, st>>>(A, lda, row_begin, row_end, I, n, R, ldr, vec4, ws);
}

// ---------------------------------------------------------------- S3: column gather
// C[i, b] = A[i, J[b]] for every local row i.  Each element lives in its own
// 32-byte sector (random-sector bound).  A warp handles 4 rows at a
// time so each lane has 4*ceil(k/32) independent loads in flight; the C row is
// written coalesced.
constexpr int kColRowsPerWarp = 4;

__global__ void __launch_bounds__(256) gather_cols_kernel(const float* __restrict__ A, int64_t lda,
                                                          int64_t m_loc, const int64_t* __restrict__ J,
                                                          int32_t k, float* __restrict__ C, int64_t ldc,
                                                          void* ws) {
  extern __shared__ int32_t sJ[];
  for (int b = threadIdx.x; b < k; b += blockDim.x) sJ[b] = static_cast<int32_t>(J[b]);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  bool bad = false;
  for (int64_t r0 = warp * kColRowsPerWarp; r0 < m_loc; r0 += nwarps * kColRowsPerWarp) {
    for (int b0 = 0; b0 < k; b0 += 32) {
      const int b = b0 + lane;
      float v[kColRowsPerWarp];
#pragma unroll
      for (int q = 0; q < kColRowsPerWarp; ++q) {
        const int64_t r = r0 + q;
        v[q] = (b < k && r < m_loc) ? __ldg(A + r * lda + sJ[b]) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < kColRowsPerWarp; ++q) {
        const int64_t r = r0 + q;
        if (b < k && r < m_loc) {
          bad |= !isfinite(v[q]);
          C[r * ldc + b] = v[q];
        }
      }
    }
  }
  if (bad) set_status(ws, CABS_DEV_NONFINITE);
}

void launch_gather_cols(const float* A, int64_t lda, int64_t m_loc, const int64_t* J, int32_t k, float* C,
                        int64_t ldc, void* ws, cudaStream_t st) {
  if (m_loc <= 0) return;
  int64_t warps = ceil_div(m_loc, kColRowsPerWarp);
  int64_t blocks = ceil_div(warps, 8);
  if (blocks > 16 * kNumSM) blocks = 16 * kNumSM;
  note_launch();
  gather_cols_kernel<<<static_cast<unsigned>(blocks), 256, sizeof(int32_t) * k, st>>>(A, lda, m_loc, J, k, C,
                                                                                      ldc, ws);
}

// W[a, b] = R[a, J[b]]: the intersection, read from the gathered rows (no second HBM visit).
__global__ void gather_w_kernel(const float* __restrict__ R, int64_t ldr, const int64_t* __restrict__ J,
                                int32_t k, float* __restrict__ W, int64_t ldw) {
  const int a = blockIdx.x;
  for (int b = threadIdx.x; b < k; b += blockDim.x) W[a * ldw + b] = R[a * ldr + J[b]];
}

void launch_gather_w(const float* R, int64_t ldr, const int64_t* J, int32_t k, float* W, int64_t ldw,
                     cudaStream_t st) {
  note_launch();
  gather_w_kernel<<<k, 128, 0, st>>>(R, ldr, J, k, W, ldw);
}

}  // namespace cabsk
