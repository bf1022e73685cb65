// Pipe-rate microbenchmark for the ALP search inner loop on sm_100a.
// Measures warp-instruction throughput of the candidate-evaluation idioms:
//   FADD2 (add.rn.f32x2 with scalar broadcast) + FMNMX3 (3-input min),
//   scalar FADD + FMNMX, and the LDS.128-fed masked-row loop.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void fadd2(float& v0, float& v1, float q, float b0, float b1) {
  asm volatile("{.reg .b64 x,y,z; mov.b64 x,{%2,%2}; mov.b64 y,{%3,%4}; add.rn.f32x2 z,x,y; mov.b64 {%0,%1},z;}"
               : "=f"(v0), "=f"(v1) : "f"(q), "f"(b0), "f"(b1));
}
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float d; asm volatile("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d;
}

// 8 rows x 4 columns per iteration = 32 candidates per lane-iteration, registers only.
__global__ void k_reg(const float* in, float* out, int iters) {
  float q[8], acc[8];
  for (int i = 0; i < 8; ++i) { q[i] = in[(threadIdx.x + i) & 63]; acc[i] = 3e38f; }
  float b0 = in[64], b1 = in[65], b2 = in[66], b3 = in[67];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float v0, v1, v2, v3;
      fadd2(v0, v1, q[i], b0, b1);
      fadd2(v2, v3, q[i], b2, b3);
      acc[i] = fmin3(acc[i], v0, v1);
      acc[i] = fmin3(acc[i], v2, v3);
    }
  }
  float r = 0; for (int i = 0; i < 8; ++i) r += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// scalar FADD + FMNMX (2 instr / candidate)
__global__ void k_scalar(const float* in, float* out, int iters) {
  float q[8], acc[8];
  for (int i = 0; i < 8; ++i) { q[i] = in[(threadIdx.x + i) & 63]; acc[i] = 3e38f; }
  float b0 = in[64], b1 = in[65], b2 = in[66], b3 = in[67];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float v0, v1, v2, v3;
      asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(v0) : "f"(q[i]), "f"(b0));
      asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(v1) : "f"(q[i]), "f"(b1));
      asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(v2) : "f"(q[i]), "f"(b2));
      asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(v3) : "f"(q[i]), "f"(b3));
      asm volatile("min.f32 %0, %0, %1;" : "+f"(acc[i]) : "f"(v0));
      asm volatile("min.f32 %0, %0, %1;" : "+f"(acc[i]) : "f"(v1));
      asm volatile("min.f32 %0, %0, %1;" : "+f"(acc[i]) : "f"(v2));
      asm volatile("min.f32 %0, %0, %1;" : "+f"(acc[i]) : "f"(v3));
    }
  }
  float r = 0; for (int i = 0; i < 8; ++i) r += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// LDS.128-fed: each lane reads a masked row chosen by lane (nrows distinct rows/warp),
// row stride 20 floats (bank-slot spread), 4 groups of 4 columns per "a" step, 8 rows per lane.
template <int NROWS>
__global__ void k_lds(const float* in, float* out, int iters) {
  __shared__ __align__(16) float tab[64 * 20];
  for (int i = threadIdx.x; i < 64 * 20; i += blockDim.x) tab[i] = in[i & 63];
  __syncthreads();
  float q[8], acc[8];
  for (int i = 0; i < 8; ++i) { q[i] = in[(threadIdx.x + i) & 63]; acc[i] = 3e38f; }
  int lane = threadIdx.x & 31;
  int rowoff = ((lane % NROWS) * 20) * 4;
  for (int it = 0; it < iters; ++it) {
    const char* base = reinterpret_cast<const char*>(tab) + rowoff + ((it & 7) * 20 * 4 * 0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float4 b = *reinterpret_cast<const float4*>(base + 16 * j);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float v0, v1, v2, v3;
        fadd2(v0, v1, q[i], b.x, b.y);
        fadd2(v2, v3, q[i], b.z, b.w);
        acc[i] = fmin3(acc[i], v0, v1);
        acc[i] = fmin3(acc[i], v2, v3);
      }
    }
    asm volatile("" ::: "memory");
  }
  float r = 0; for (int i = 0; i < 8; ++i) r += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d clockRate(attr) %d kHz\n", p.name, p.multiProcessorCount, clk_khz);
  float *in, *out; cudaMalloc(&in, 4096 * 4); cudaMalloc(&out, 64 << 20);
  float h[4096]; for (int i = 0; i < 4096; ++i) h[i] = 1.0f + (i % 97) * 0.01f;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int SM = p.multiProcessorCount;
  struct Cfg { const char* name; int which; int threads; int blocks_per_sm; };
  Cfg cfgs[] = {
    {"reg  FADD2+FMNMX3 256t x4", 0, 256, 4}, {"reg  FADD2+FMNMX3 512t x2", 0, 512, 2},
    {"reg  FADD2+FMNMX3 128t x4", 0, 128, 4}, {"reg  FADD2+FMNMX3 1024t x1", 0, 1024, 1},
    {"scalar FADD+FMNMX 256t x4", 1, 256, 4},
    {"lds rows=1 256t x4", 2, 256, 4}, {"lds rows=8 256t x4", 3, 256, 4}, {"lds rows=32 256t x4", 4, 256, 4},
    {"lds rows=8 512t x2", 3, 512, 2},
  };
  for (auto& c : cfgs) {
    int iters = 4096;
    dim3 g(SM * c.blocks_per_sm), b(c.threads);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      switch (c.which) {
        case 0: k_reg<<<g, b>>>(in, out, iters); break;
        case 1: k_scalar<<<g, b>>>(in, out, iters); break;
        case 2: k_lds<1><<<g, b>>>(in, out, iters); break;
        case 3: k_lds<8><<<g, b>>>(in, out, iters); break;
        case 4: k_lds<32><<<g, b>>>(in, out, iters); break;
      }
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double cand_per_it = (c.which >= 2) ? 128.0 : 32.0;
      double cands = (double)g.x * b.x * iters * cand_per_it;
      if (rep == 2)
        printf("%-28s %8.3f ms  %.3e cand/s  %.1f cand/clk/SM @1965MHz  err=%s\n", c.name, ms, cands / (ms * 1e-3),
               cands / (ms * 1e-3) / SM / 1.965e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
