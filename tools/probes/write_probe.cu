// HBM write-bandwidth ceiling on this B200 (is the dispatch's ~4.2 TB/s of row writes at the write
// ceiling?): pure writes of 755 MB (the G120 P=1 receive arena) by cudaMemsetAsync and by a grid-stride
// kernel with 16-byte stores in three cache flavours (default, .cs streaming, .cg), plus the
// dispatch's mix (each 5760-byte row read once, written 4 times to scattered rows) for reference.
// Best of 20, CUDA events.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_probe write_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int FLAVOUR>
__global__ void fill_kernel(int4 *__restrict__ p, int64_t n16) {
  const int4 v = make_int4(1, 2, 3, 4);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    if (FLAVOUR == 0) p[i] = v;
    else if (FLAVOUR == 1) __stcs(p + i, v);
    else __stcg(p + i, v);
  }
}

// one warp per token: read the row once, write it to K scattered destination rows (like the dispatch)
__global__ void mix_kernel(const int4 *__restrict__ x, int4 *__restrict__ out, const int *__restrict__ dst,
                           int B, int K, int nv) {
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= B) return;
  for (int i0 = 0; i0 < nv; i0 += 128) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * 32 + lane;
      if (i < nv) v[u] = x[(int64_t)t * nv + i];
    }
    for (int k = 0; k < K; ++k) {
      const int r = dst[t * K + k];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * 32 + lane;
        if (i < nv) out[(int64_t)r * nv + i] = v[u];
      }
    }
  }
}

// the same mix through the TMA engine: a persistent warp loops over tokens with two 5760-byte shared
// buffers; lane 0 bulk-loads token i+1 (cp.async.bulk global->shared, mbarrier tx count) while the K
// bulk stores of token i (cp.async.bulk shared->global) drain; no register traffic
constexpr int kRow = 5760;
__global__ void __launch_bounds__(256) mix_bulk_kernel(const uint8_t *__restrict__ x, uint8_t *__restrict__ out,
                                                       const int *__restrict__ dst, int B, int K) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[8][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane != 0) return;
  uint8_t *buf0 = sm + warp * 2 * kRow;
  const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(buf0);
  const uint32_t m0 = (uint32_t)__cvta_generic_to_shared(&bar[warp][0]);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(m0));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(m0 + 8));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int gw = blockIdx.x * 8 + warp, nw = gridDim.x * 8;
  uint32_t ph[2] = {0, 0};
  int i = 0;
  auto load = [&](int t, int b) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m0 + 8 * b), "r"(kRow) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(b0 + b * kRow), "l"(x + (int64_t)t * kRow), "r"(kRow), "r"(m0 + 8 * b) : "memory");
  };
  if (gw < B) load(gw, 0);
  for (int t = gw; t < B; t += nw, ++i) {
    const int b = i & 1;
    if (t + nw < B) {
      // buffer b^1 was last stored from two tokens ago: its bulk stores must have read it
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      load(t + nw, b ^ 1);
    }
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
                 ::"r"(m0 + 8 * b), "r"(ph[b]) : "memory");
    ph[b] ^= 1;
    for (int k = 0; k < K; ++k)
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   ::"l"(out + (int64_t)dst[t * K + k] * kRow), "r"(b0 + b * kRow), "r"(kRow) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <typename F>
float best_ms(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e9f;
  for (int r = 0; r < 20; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  const int B = 32768, K = 4, D = 2880;
  const int64_t row = (int64_t)D * 2, bytes = (int64_t)B * K * row;
  int4 *out, *x;
  int *dst;
  cudaMalloc(&out, bytes);
  cudaMalloc(&x, (int64_t)B * row * 2);
  cudaMalloc(&dst, sizeof(int) * B * K);
  int *h = new int[B * K];
  uint64_t s = 12345;   // a fixed permutation of the B*K destination rows (LCG + Fisher-Yates)
  for (int i = 0; i < B * K; ++i) h[i] = i;
  for (int i = B * K - 1; i > 0; --i) {
    s = s * 6364136223846793005ULL + 1442695040888963407ULL;
    const int j = (int)((s >> 33) % (uint64_t)(i + 1));
    const int t = h[i]; h[i] = h[j]; h[j] = t;
  }
  cudaMemcpy(dst, h, sizeof(int) * B * K, cudaMemcpyHostToDevice);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t n16 = bytes / 16;
  float ms = best_ms([&] { cudaMemsetAsync(out, 1, bytes); });
  printf("{\"op\": \"cudaMemsetAsync\", \"GBps\": %.1f, \"ms\": %.4f}\n", bytes / ms / 1e6, ms);
  for (int per = 2; per <= 16; per *= 2) {
    ms = best_ms([&] { fill_kernel<0><<<sms * per, 256>>>(out, n16); });
    printf("{\"op\": \"st.global 16B, %d CTAs/SM\", \"GBps\": %.1f, \"ms\": %.4f}\n", per, bytes / ms / 1e6, ms);
  }
  ms = best_ms([&] { fill_kernel<1><<<sms * 8, 256>>>(out, n16); });
  printf("{\"op\": \"st.global.cs 16B\", \"GBps\": %.1f, \"ms\": %.4f}\n", bytes / ms / 1e6, ms);
  ms = best_ms([&] { fill_kernel<2><<<sms * 8, 256>>>(out, n16); });
  printf("{\"op\": \"st.global.cg 16B\", \"GBps\": %.1f, \"ms\": %.4f}\n", bytes / ms / 1e6, ms);
  ms = best_ms([&] { mix_kernel<<<(B + 7) / 8, 256>>>(x, out, dst, B, K, D / 8); });
  printf("{\"op\": \"dispatch mix 1:4 (row read once, 4 scattered row writes)\", \"GBps\": %.1f, \"write_GBps\": %.1f, \"ms\": %.4f}\n",
         (bytes + (int64_t)B * row) / ms / 1e6, bytes / ms / 1e6, ms);
  {  // the same mix with sequential destinations (row t*K+k): is the random row order the cost?
    int *hs = new int[B * K];
    for (int i = 0; i < B * K; ++i) hs[i] = i;
    int *dseq;
    cudaMalloc(&dseq, sizeof(int) * B * K);
    cudaMemcpy(dseq, hs, sizeof(int) * B * K, cudaMemcpyHostToDevice);
    ms = best_ms([&] { mix_kernel<<<(B + 7) / 8, 256>>>(x, out, dseq, B, K, D / 8); });
    printf("{\"op\": \"dispatch mix 1:4, sequential destinations\", \"GBps\": %.1f, \"write_GBps\": %.1f, \"ms\": %.4f}\n",
           (bytes + (int64_t)B * row) / ms / 1e6, bytes / ms / 1e6, ms);
    ms = best_ms([&] { cudaMemcpyAsync(out, x, (int64_t)B * row * 2, cudaMemcpyDeviceToDevice); });
    printf("{\"op\": \"cudaMemcpyAsync D2D 1:1 (377 MB)\", \"GBps\": %.1f, \"ms\": %.4f}\n", 2.0 * B * row * 2 / ms / 1e6, ms);
  }
  cudaFuncSetAttribute(mix_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 2 * kRow);
  for (int per = 1; per <= 2; ++per) {
    ms = best_ms([&] { mix_bulk_kernel<<<sms * per, 256, 8 * 2 * kRow>>>(reinterpret_cast<const uint8_t *>(x),
                                                                         reinterpret_cast<uint8_t *>(out), dst, B, K); });
    printf("{\"op\": \"dispatch mix 1:4, TMA bulk load + K bulk stores, %d CTAs/SM\", \"GBps\": %.1f, \"write_GBps\": %.1f, \"ms\": %.4f}\n",
           per, (bytes + (int64_t)B * row) / ms / 1e6, bytes / ms / 1e6, ms);
  }
  {  // check: every destination row equals its token's row (bytes)
    cudaMemset(out, 0, bytes);
    uint8_t *hx = new uint8_t[(int64_t)B * row];
    for (int64_t i = 0; i < (int64_t)B * row; ++i) hx[i] = (uint8_t)(i * 131 + 7);
    cudaMemcpy(x, hx, (int64_t)B * row, cudaMemcpyHostToDevice);
    mix_bulk_kernel<<<sms * 2, 256, 8 * 2 * kRow>>>(reinterpret_cast<const uint8_t *>(x), reinterpret_cast<uint8_t *>(out), dst, B, K);
    uint8_t *ho = new uint8_t[bytes];
    cudaMemcpy(ho, out, bytes, cudaMemcpyDeviceToHost);
    int64_t bad = 0;
    for (int t = 0; t < B; ++t)
      for (int k = 0; k < K; ++k)
        for (int j = 0; j < row; j += 97)
          bad += ho[(int64_t)h[t * K + k] * row + j] != hx[(int64_t)t * row + j];
    printf("{\"check\": \"bulk mix rows\", \"mismatches\": %lld}\n", (long long)bad);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
