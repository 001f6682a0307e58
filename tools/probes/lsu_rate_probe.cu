// Per-SM ingest rate from HBM: TMA box loads (one lane) vs LSU cp.async (128 threads, 16 B each) vs both
// at once, into a shared-memory ring, one CTA per SM, N CTAs.  Question: is the ~73 GB/s per-SM limit of
// DRAM-sourced TMA loads a limit of the TMA unit (then the LSU path adds bandwidth) or of the SM?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lsu_rate_probe lsu_rate_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

constexpr int STAGES = 8, TILE = 16384;
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(done) : "r"(bar), "r"(ph) : "memory");
}

// mode 0: TMA box {64 cols, 128 rows} per tile (thread 0); mode 1: LSU cp.async 16 B x 8 per thread (128 threads);
// mode 2: even tiles by TMA, odd tiles by LSU (both paths in flight at once)
__global__ void __launch_bounds__(128) probe(const __grid_constant__ CUtensorMap tile, const uint8_t *x, int rows,
                                             int kdim, int iters, int mode, unsigned long long *cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *buf = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[STAGES];
  const int tid = threadIdx.x;
  if (tid == 0)
    for (int i = 0; i < STAGES; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 129;" ::"r"(su32(full + i)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const long long t0 = clock64();
  const int nkb = kdim / 64, nmb = rows / 128;
  for (int it = 0; it < iters; ++it) {
    const int s = it % STAGES;
    const uint32_t ph = (it / STAGES) & 1;
    if (it >= STAGES) wait_bar(su32(full + s), ph ^ 1);
    const int tix = blockIdx.x + it * gridDim.x;
    const int mb = (tix / nkb) % nmb, kb = tix % nkb;
    const uint32_t dst = su32(buf + s * TILE), bar = su32(full + s);
    const bool tma = mode == 0 || (mode == 2 && (it & 1) == 0);
    if (tma) {
      // 128 plain arrivals + one expect_tx arrival: the phase completes when the TMA bytes land
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
      if (tid == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(TILE) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(dst), "l"((uint64_t)&tile), "r"(kb * 64), "r"(mb * 128), "r"(bar) : "memory");
      }
    } else {
      // tile rows r = 0..127, 128 B each at x[(mb*128 + r) * kdim + kb*64]: thread t copies 8 x 16 B
      for (int i = 0; i < 8; ++i) {
        const int u = tid + 128 * i, r = u >> 3, c = u & 7;
        const uint8_t *src = x + ((size_t)(mb * 128 + r) * kdim + kb * 64) * 2 + c * 16;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + r * 128 + ((c ^ (r & 7)) << 4)), "l"(src) : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
      if (tid == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
    }
  }
  for (int k = 0; k < STAGES; ++k) {
    const int it = iters - STAGES + k;
    if (it >= 0) wait_bar(su32(full + it % STAGES), (it / STAGES) & 1);
  }
  if (tid == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main(int argc, char **argv) {
  const int ncta = argc > 1 ? atoi(argv[1]) : 148;
  const int rows = 131072, kdim = 2880;
  void *x;
  cudaMalloc(&x, (size_t)rows * kdim * 2);
  cudaMemset(x, 1, (size_t)rows * kdim * 2);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap mt;
  cuuint64_t dims[2] = {(cuuint64_t)kdim, (cuuint64_t)rows}, str[1] = {(cuuint64_t)kdim * 2};
  cuuint32_t bt[2] = {64, 128}, es[2] = {1, 1};
  enc(&mt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, str, bt, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = STAGES * TILE + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long *cyc;
  cudaMalloc(&cyc, sizeof(unsigned long long) * ncta);
  const int iters = 4000;
  const char *names[] = {"TMA box", "LSU cp.async", "TMA + LSU alternating"};
  for (int mode = 0; mode < 3; ++mode) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    probe<<<ncta, 128, smem>>>(mt, (const uint8_t *)x, rows, kdim, 50, mode, cyc);
    cudaEventRecord(a);
    probe<<<ncta, 128, smem>>>(mt, (const uint8_t *)x, rows, kdim, iters, mode, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)ncta * iters * TILE;
    printf("{\"ctas\": %d, \"mode\": \"%s\", \"ms\": %.3f, \"GBps\": %.1f, \"per_sm_GBps\": %.1f, \"err\": \"%s\"}\n", ncta,
           names[mode], ms, bytes / ms / 1e6, bytes / ms / 1e6 / ncta, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
