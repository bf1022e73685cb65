// Pipe-rate microbenchmark v2 (no loop-invariant hoisting: b values come from shared memory at an
// iteration-dependent address).  Reports warp-instructions/clk/SMSP and candidates/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void fadd2b(float& v0, float& v1, float q, float b0, float b1) {
  asm("{.reg .b64 x,y,z; mov.b64 x,{%2,%2}; mov.b64 y,{%3,%4}; add.rn.f32x2 z,x,y; mov.b64 {%0,%1},z;}"
      : "=f"(v0), "=f"(v1) : "f"(q), "f"(b0), "f"(b1));
}
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float d; asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d;
}
template <int V, int ROWS>
__global__ void kern(const float* in, float* out, int iters, long long* clk) {
  __shared__ __align__(16) float tab[8 * 64];
  for (int i = threadIdx.x; i < 8 * 64; i += blockDim.x) tab[i] = in[i & 1023];
  __syncthreads();
  float q[ROWS], acc[ROWS], acc2[ROWS];
  for (int i = 0; i < ROWS; ++i) { q[i] = in[(threadIdx.x + i) & 1023]; acc[i] = 3e38f; acc2[i] = 0.f; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float4 b = *reinterpret_cast<const float4*>(tab + ((it * 4 + (threadIdx.x & 7) * 64) & 511));
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
      if (V == 0) {  // FADD2 + FMNMX3 (real inner loop)
        float v0, v1, v2, v3;
        fadd2b(v0, v1, q[i], b.x, b.y); fadd2b(v2, v3, q[i], b.z, b.w);
        acc[i] = fmin3(acc[i], v0, v1); acc[i] = fmin3(acc[i], v2, v3);
      } else if (V == 1) {  // scalar FADD x4 + FMNMX3 x2
        float v0 = __fadd_rn(q[i], b.x), v1 = __fadd_rn(q[i], b.y), v2 = __fadd_rn(q[i], b.z), v3 = __fadd_rn(q[i], b.w);
        acc[i] = fmin3(acc[i], v0, v1); acc[i] = fmin3(acc[i], v2, v3);
      } else if (V == 2) {  // FADD2 only (accumulate)
        float v0, v1, v2, v3;
        fadd2b(v0, v1, acc[i], b.x, b.y); fadd2b(v2, v3, acc2[i], b.z, b.w); acc[i] = v0 + 0.f * v1; acc2[i] = v2; (void)v3;
      } else if (V == 3) {  // FMNMX3 only
        acc[i] = fmin3(acc[i], b.x, b.y); acc2[i] = fmin3(acc2[i], b.z, b.w);
      } else if (V == 4) {  // scalar FADD + scalar FMNMX (2 instr / cand)
        float v0 = __fadd_rn(q[i], b.x), v1 = __fadd_rn(q[i], b.y);
        asm("min.f32 %0, %0, %1;" : "+f"(acc[i]) : "f"(v0)); asm("min.f32 %0, %0, %1;" : "+f"(acc2[i]) : "f"(v1));
      }
    }
  }
  long long t1 = clock64();
  float r = 0; for (int i = 0; i < ROWS; ++i) r += acc[i] + acc2[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}
template <int V, int ROWS> void run(const char* name, const float* in, float* out, long long* dclk, int SM, int threads, int bps, double cand_per_row_it) {
  int iters = 8192; cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); kern<V, ROWS><<<SM * bps, threads>>>(in, out, iters, dclk); cudaEventRecord(e1); cudaEventSynchronize(e1);
  }
  float ms; cudaEventElapsedTime(&ms, e0, e1); long long clk; cudaMemcpy(&clk, dclk, 8, cudaMemcpyDeviceToHost);
  double cands = (double)SM * bps * threads * iters * ROWS * cand_per_row_it;
  double f = clk / (ms * 1e-3);  // SM clock estimate from block 0
  printf("%-34s %7.3f ms  clk~%4.0f MHz  %.3e cand/s  %6.1f cand/clk/SM  err=%s\n", name, ms, f / 1e6, cands / (ms * 1e-3),
         cands / (ms * 1e-3) / SM / f, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0); int SM = p.multiProcessorCount;
  float *in, *out; long long* dclk; cudaMalloc(&in, 4096 * 4); cudaMalloc(&out, 64 << 20); cudaMalloc(&dclk, 8);
  float h[1024]; for (int i = 0; i < 1024; ++i) h[i] = 1.0f + (i % 97) * 0.01f; cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  run<0, 8>("FADD2+FMNMX3 rows=8 256x3", in, out, dclk, SM, 256, 3, 4);
  run<0, 8>("FADD2+FMNMX3 rows=8 256x4", in, out, dclk, SM, 256, 4, 4);
  run<0, 4>("FADD2+FMNMX3 rows=4 256x4", in, out, dclk, SM, 256, 4, 4);
  run<0, 8>("FADD2+FMNMX3 rows=8 256x2", in, out, dclk, SM, 256, 2, 4);
  run<1, 8>("FADDx4+FMNMX3x2 rows=8 256x3", in, out, dclk, SM, 256, 3, 4);
  run<2, 8>("FADD2 only (per 2 adds=1cand) 256x3", in, out, dclk, SM, 256, 3, 4);
  run<3, 8>("FMNMX3 only (2 folds=2cand) 256x3", in, out, dclk, SM, 256, 3, 4);
  run<4, 8>("FADD+FMNMX scalar rows=8 256x3", in, out, dclk, SM, 256, 3, 2);
  return 0;
}
