// FMA-heavy / FMA pipe throughput microbenchmark (profiles/r1e_pipes.txt): warp-instructions per
// clock per SM for IMAD.WIDE, FFMA2, FFMA, IMAD and mixes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes profiles/pipes_microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define N 4096
__global__ void k_imadw(uint32_t* out, uint32_t s) {
  uint32_t a = threadIdx.x ^ s, b = a * 3u, c = a * 5u, d = a * 7u;
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint64_t p = (uint64_t)a * 0xD2511F53u, q = (uint64_t)b * 0xCD9E8D57u;
      uint64_t r = (uint64_t)c * 0xD2511F53u, t = (uint64_t)d * 0xCD9E8D57u;
      a = (uint32_t)(p >> 32) + (uint32_t)p; b = (uint32_t)(q >> 32) + (uint32_t)q;
      c = (uint32_t)(r >> 32) + (uint32_t)r; d = (uint32_t)(t >> 32) + (uint32_t)t;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a ^ b ^ c ^ d;
}
__global__ void k_ffma2(float* out, float s) {
  float2 a = make_float2(threadIdx.x * s, s), b = make_float2(s, 1.f), c = make_float2(1.f, s), d = make_float2(s, s);
  const float2 m = make_float2(0.999f, 1.001f), e = make_float2(0.5f, 0.25f);
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      a = __ffma2_rn(a, m, e); b = __ffma2_rn(b, m, e); c = __ffma2_rn(c, m, e); d = __ffma2_rn(d, m, e);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a.x + a.y + b.x + b.y + c.x + c.y + d.x + d.y;
}
__global__ void k_ffma(float* out, float s) {
  float a = threadIdx.x * s, b = s, c = 1.f, d = s * 2, e = s * 3, f = s * 4, g = s * 5, h = s * 6;
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      a = fmaf(a, 0.999f, 0.5f); b = fmaf(b, 0.999f, 0.5f); c = fmaf(c, 0.999f, 0.5f); d = fmaf(d, 0.999f, 0.5f);
      e = fmaf(e, 0.999f, 0.5f); f = fmaf(f, 0.999f, 0.5f); g = fmaf(g, 0.999f, 0.5f); h = fmaf(h, 0.999f, 0.5f);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d + e + f + g + h;
}
__global__ void k_mix(float* out, float s, uint32_t u) {  // 2 IMAD.WIDE + 2 FFMA2 per group
  uint32_t a = threadIdx.x ^ u, b = a * 3u;
  float2 x = make_float2(threadIdx.x * s, s), y = make_float2(s, 1.f);
  const float2 m = make_float2(0.999f, 1.001f), e = make_float2(0.5f, 0.25f);
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint64_t p = (uint64_t)a * 0xD2511F53u, q = (uint64_t)b * 0xCD9E8D57u;
      a = (uint32_t)(p >> 32) ^ (uint32_t)p; b = (uint32_t)(q >> 32) ^ (uint32_t)q;
      x = __ffma2_rn(x, m, e); y = __ffma2_rn(y, m, e);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x.x + x.y + y.x + y.y + (float)(a ^ b);
}
__global__ void k_mixs(float* out, float s, uint32_t u) {  // 2 IMAD.WIDE + 4 FFMA per group
  uint32_t a = threadIdx.x ^ u, b = a * 3u;
  float x0 = threadIdx.x * s, x1 = s, y0 = s, y1 = 1.f;
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint64_t p = (uint64_t)a * 0xD2511F53u, q = (uint64_t)b * 0xCD9E8D57u;
      a = (uint32_t)(p >> 32) ^ (uint32_t)p; b = (uint32_t)(q >> 32) ^ (uint32_t)q;
      x0 = fmaf(x0, 0.999f, 0.5f); x1 = fmaf(x1, 1.001f, 0.25f); y0 = fmaf(y0, 0.999f, 0.5f); y1 = fmaf(y1, 1.001f, 0.25f);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + y0 + y1 + (float)(a ^ b);
}
__global__ void k_imov(uint32_t* out, uint32_t s) {  // integer adds (ALU or IMAD?)
  uint32_t a = threadIdx.x ^ s, b = a * 3u, c = a * 5u, d = a * 7u;
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { a = a * 3u + b; b = b * 5u + c; c = c * 7u + d; d = d * 9u + a; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a ^ b ^ c ^ d;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  void* buf; cudaMalloc(&buf, 64 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  struct { const char* name; int kind; double ops; } ks[] = {
    {"IMAD.WIDE x4 (+IADD)", 0, 4 * 4.0}, {"FFMA2 x4", 1, 8 * 4.0}, {"FFMA x8", 2, 8 * 8.0},
    {"2 IMAD.WIDE + 2 FFMA2", 3, 8 * 4.0}, {"2 IMAD.WIDE + 4 FFMA", 4, 8 * 6.0}, {"IMAD x4", 5, 8 * 4.0}};
  for (auto& k : ks) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      switch (k.kind) {
        case 0: k_imadw<<<blocks, threads>>>((uint32_t*)buf, 1); break;
        case 1: k_ffma2<<<blocks, threads>>>((float*)buf, 1.f); break;
        case 2: k_ffma<<<blocks, threads>>>((float*)buf, 1.f); break;
        case 3: k_mix<<<blocks, threads>>>((float*)buf, 1.f, 1); break;
        case 4: k_mixs<<<blocks, threads>>>((float*)buf, 1.f, 1); break;
        case 5: k_imov<<<blocks, threads>>>((uint32_t*)buf, 1); break;
      }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double warp_instr = (double)blocks * threads / 32 * N * k.ops;
      if (rep) printf("%-24s %8.3f ms  %.2f warp-instr/clk/SM (at %d MHz)\n", k.name, ms,
                      warp_instr / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
