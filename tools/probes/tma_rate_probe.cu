// Throughput probe: TMA tile loads vs TMA gather4 loads of [128 rows x 64 bf16] tiles into a shared-memory
// ring (no MMA), one CTA per SM.  Decides whether GEMM1 can read its A rows straight from x by gather.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather4_probe gather4_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

constexpr int MAXSTAGES = 12, TILE = 128 * 128;   // 128 rows x 128 B
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// mode 0: tile box {64, 128}; mode 1: gather4 by 32 lanes (4 rows each); mode 2: gather4, lane 0 issues all 32
__global__ void probe(const __grid_constant__ CUtensorMap tile, const __grid_constant__ CUtensorMap g4,
                      const int *__restrict__ perm, int rows, int kdim, int iters, int mode, unsigned long long *cyc,
                      const uint8_t *base, int STAGES) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *buf = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[MAXSTAGES];
  const int lane = threadIdx.x;
  if (lane == 0)
    for (int i = 0; i < STAGES; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(full + i)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const long long t0 = clock64();
  const int nkb = kdim / 64, nmb = rows / 128;
  for (int it = 0; it < iters; ++it) {
    const int s = it % STAGES;
    const uint32_t ph = (it / STAGES) & 1;
    if (it >= STAGES) {   // wait for the previous fill of this stage
      uint32_t done = 0;
      while (!done)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(done) : "r"(su32(full + s)), "r"(ph ^ 1) : "memory");
    }
    __syncwarp();
    const int tix = blockIdx.x + it * gridDim.x;
    const int mb = (tix / nkb) % nmb, kb = tix % nkb;
    const uint32_t dst = su32(buf + s * TILE), bar = su32(full + s);
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(TILE) : "memory");
    if (mode == 3) {
      if (lane == 0) {
        const uint8_t *src = base + ((size_t)tix % ((size_t)rows * kdim * 2 / TILE)) * TILE;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(dst), "l"(src), "r"(TILE), "r"(bar) : "memory");
      }
    } else if (mode == 0) {
      if (lane == 0)
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(dst), "l"((uint64_t)&tile), "r"(kb * 64), "r"(mb * 128), "r"(bar) : "memory");
    } else {
      for (int c = (mode == 1 ? lane : 0); c < 32; c += (mode == 1 ? 32 : 1)) {
        if (mode == 2 && lane != 0) break;
        const int *r = perm + mb * 128 + 4 * c;
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                     ::"r"(dst + c * 512), "l"((uint64_t)&g4), "r"(kb * 64), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(bar)
                     : "memory");
      }
    }
    __syncwarp();
  }
  for (int s = 0; s < STAGES; ++s) {   // drain
    const int it = iters - STAGES + s;
    if (it < 0) continue;
    const uint32_t ph = (it / STAGES) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(done) : "r"(su32(full + it % STAGES)), "r"(ph) : "memory");
  }
  if (lane == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main(int argc, char **argv) {
  const int ncta = argc > 1 ? atoi(argv[1]) : 0, nst = argc > 2 ? atoi(argv[2]) : 6;
  const int rows = 131072, kdim = 2880;
  void *x;
  cudaMalloc(&x, (size_t)rows * kdim * 2);
  cudaMemset(x, 1, (size_t)rows * kdim * 2);
  std::vector<int> h(rows);
  for (int i = 0; i < rows; ++i) h[i] = i;
  srand(1);
  std::vector<int> hr = h;
  for (int i = rows - 1; i > 0; --i) std::swap(hr[i], hr[rand() % (i + 1)]);
  int *perm_seq, *perm_rand;
  cudaMalloc(&perm_seq, rows * 4);
  cudaMalloc(&perm_rand, rows * 4);
  cudaMemcpy(perm_seq, h.data(), rows * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(perm_rand, hr.data(), rows * 4, cudaMemcpyHostToDevice);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap mt, mg;
  cuuint64_t dims[2] = {(cuuint64_t)kdim, (cuuint64_t)rows}, str[1] = {(cuuint64_t)kdim * 2};
  cuuint32_t bt[2] = {64, 128}, bg[2] = {64, 1}, es[2] = {1, 1};
  enc(&mt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, str, bt, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&mg, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, str, bg, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int STAGES = nst;
  const int smem = STAGES * TILE + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long *cyc;
  cudaMalloc(&cyc, sizeof(unsigned long long) * sms);
  const int iters = 4000;
  const char *names[] = {"tile box 128x64", "gather4, 32 lanes", "gather4, lane 0 only", "1D bulk 16 KB contiguous"};
  if (ncta > 0) sms = ncta;
  for (int mode : {0, 3})
    for (int pr = 0; pr < 2; ++pr) {
      if (mode == 0 && pr == 1) continue;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      const int *perm = pr ? perm_rand : perm_seq;
      probe<<<sms, 32, smem>>>(mt, mg, perm, rows, kdim, 50, mode, cyc, (const uint8_t *)x, STAGES);   // warm
      cudaEventRecord(a);
      probe<<<sms, 32, smem>>>(mt, mg, perm, rows, kdim, iters, mode, cyc, (const uint8_t *)x, STAGES);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      std::vector<unsigned long long> hc(sms);
      cudaMemcpy(hc.data(), cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
      double mc = 0;
      for (auto v : hc) mc += v;
      mc /= sms;
      const double bytes = (double)sms * iters * TILE;
      printf("{\"ctas\": %d, \"stages\": %d, \"mode\": \"%s\", \"rows\": \"%s\", \"ms\": %.3f, \"GBps\": %.1f, \"cycles_per_tile_per_sm\": %.1f, "
             "\"cycles_per_row_per_sm\": %.2f, \"err\": \"%s\"}\n",
             sms, STAGES, names[mode], pr ? "random permutation" : "sequential", ms, bytes / ms / 1e6, mc / iters, mc / iters / 128,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
