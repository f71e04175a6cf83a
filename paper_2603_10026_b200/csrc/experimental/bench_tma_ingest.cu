// TEST-ONLY micro-benchmark (not part of librf_cuda): how many bytes per clock
// one SM can land in shared memory with TMA when every SM streams at once —
// the operand-delivery ceiling of the GEMM mainloops (profiles/r2_fp8_investigation.md).
// One CTA per SM: an elected thread keeps `stages` 32 KB loads (two 128 x 64
// bf16 SWIZZLE_128B boxes) in flight, a consumer warp frees each slot as soon
// as it lands. Modes: distinct rows per CTA (every byte from its own L2 lines),
// rows shared by groups of 2 / 4 / 8 consecutive CTAs (same lines at the same
// time), and one 4 MB panel read by everybody.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I.. -o tma_ingest bench_tma_ingest.cu ../tmap.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "../sm100.cuh"

using namespace rf::sm100;

constexpr int MAXS = 6;
constexpr int SLOT = 32768;

struct Smem {
  uint8_t buf[MAXS][SLOT];
  uint64_t full[MAXS], empty[MAXS];
};

__global__ void __launch_bounds__(64, 1)
    ingest_kernel(const __grid_constant__ CUtensorMap tm, int share, int stages, int iters, int rows_total,
                  long long* out) {
  extern __shared__ uint8_t raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  // row block of this CTA: groups of `share` CTAs read the same rows
  const int group = share > 0 ? blockIdx.x / share : 0;
  const int row_blocks = rows_total / 128;
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    if (elect_one()) {
      for (int t = 0; t < iters; ++t) {
        const int sl = t % stages;
        mbar_wait(&s.empty[sl], ((t / stages) & 1) ^ 1);
        mbar_arrive_expect_tx(&s.full[sl], SLOT);
        // share > 0: box pair idx = (group * 37 + t) mod (all box pairs), distinct per group;
        // share 0: everybody walks the same 4 MB panel (32 row blocks x 1 column pair)
        const int idx = share > 0 ? (group * 37 + t) % (row_blocks * 64) : t % 32;
        const int rb = share > 0 ? idx % row_blocks : idx;
        const int col = share > 0 ? idx / row_blocks : 0;
        tma_load_2d(s.buf[sl], &tm, &s.full[sl], col * 128, rb * 128);
        tma_load_2d(s.buf[sl] + 16384, &tm, &s.full[sl], col * 128 + 64, rb * 128);
      }
    }
  } else {
    for (int t = 0; t < iters; ++t) {
      const int sl = t % stages;
      mbar_wait(&s.full[sl], (t / stages) & 1);
      if (elect_one()) mbar_arrive(&s.empty[sl]);
      __syncwarp();
    }
    if (threadIdx.x == 32) out[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  // bf16 [rows, 8192]: 16384 rows = 256 MB (twice the L2) or 2048 rows = 32 MB (L2-resident)
  const int cols = 8192;
  void* a;
  cudaMalloc(&a, 16384ull * cols * 2);
  cudaMemset(a, 0x3c, 16384ull * cols * 2);
  long long* out;
  cudaMalloc(&out, 148 * sizeof(long long));
  const size_t smem = sizeof(Smem) + 1024;
  cudaFuncSetAttribute(ingest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  struct Case {
    int rows, share, stages;
  } cases[] = {{2048, 1, 4}, {2048, 1, 6}, {2048, 2, 4}, {2048, 4, 4}, {2048, 8, 4},
               {2048, 0, 4}, {16384, 1, 4}, {16384, 1, 6}, {16384, 8, 4}};
  for (const Case& c : cases) {
    CUtensorMap tm;
    const uint64_t dims[2] = {static_cast<uint64_t>(cols), static_cast<uint64_t>(c.rows)};
    const uint64_t str[1] = {static_cast<uint64_t>(cols) * 2};
    const uint32_t box[2] = {64, 128};
    if (!rf::make_tmap(&tm, a, 2, dims, str, box, 2)) {
      printf("tmap failed\n");
      return 1;
    }
    const int iters = 2000;
    for (int it = 0; it < 2; ++it) ingest_kernel<<<148, 64, smem>>>(tm, c.share, c.stages, iters, c.rows, out);
    if (cudaDeviceSynchronize() != cudaSuccess) {
      printf("launch failed\n");
      return 1;
    }
    long long h[148];
    cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
    double mx = 0, sum = 0;
    for (long long v : h) {
      mx = v > mx ? v : mx;
      sum += v;
    }
    const double bytes = static_cast<double>(iters) * SLOT;
    printf("rows %5d (%s) share %d stages %d: %.1f B/clk/SM mean, %.1f slowest SM, chip %.0f B/clk\n", c.rows,
           c.rows * 16384.0 > 100e6 ? "HBM" : "L2", c.share, c.stages, bytes / (sum / 148), bytes / mx,
           148 * bytes / (sum / 148));
  }
  return 0;
}
