// Microbenchmark v4: where should the b operand of the inner loop live?
//   LV: lane-varying smem row (current kernel)      -> FADD2 R, Rpair, Rb
//   WU: warp-uniform smem row (broadcast LDS)       -> FADD2 R, Rpair, Rb
//   CB: warp-uniform constant bank via LDCU (UR)    -> FADD2 R, Rpair, URb
#include <cstdio>
#include <cuda_runtime.h>
__constant__ float cb[4096];
__device__ __forceinline__ void add2b(float& v0, float& v1, float q0, float q1, float b) {
  asm("{.reg .b64 x,y,z; mov.b64 x,{%2,%3}; mov.b64 y,{%4,%4}; add.rn.f32x2 z,x,y; mov.b64 {%0,%1},z;}"
      : "=f"(v0), "=f"(v1) : "f"(q0), "f"(q1), "f"(b));
}
__device__ __forceinline__ float min3(float a, float b, float c) {
  float d; asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d;
}
template <int T>
__device__ __forceinline__ void body(const float4 b, const float (&q)[T], float (&acc)[T]) {
#pragma unroll
  for (int i = 0; i < T; i += 2) {
    float a0, c0, a1, c1, a2, c2, a3, c3;
    add2b(a0, c0, q[i], q[i + 1], b.x); add2b(a1, c1, q[i], q[i + 1], b.y);
    add2b(a2, c2, q[i], q[i + 1], b.z); add2b(a3, c3, q[i], q[i + 1], b.w);
    acc[i] = min3(acc[i], a0, a1); acc[i + 1] = min3(acc[i + 1], c0, c1);
    acc[i] = min3(acc[i], a2, a3); acc[i + 1] = min3(acc[i + 1], c2, c3);
  }
}
template <int MODE, int T>
__global__ void kern(const float* in, float* out, int iters) {
  __shared__ __align__(16) float tab[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) tab[i] = in[i & 1023];
  __syncthreads();
  float q[T], acc[T];
  for (int i = 0; i < T; ++i) { q[i] = in[(threadIdx.x + i) & 1023]; acc[i] = 3e38f; }
  const int lane = threadIdx.x & 31;
  const int lrow = (MODE == 0) ? (lane & 7) * 20 : 0;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const int base = ((it & 15) * 160) + lrow;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      float4 b;
      if (MODE == 2) b = make_float4(cb[base + 4 * g], cb[base + 4 * g + 1], cb[base + 4 * g + 2], cb[base + 4 * g + 3]);
      else b = *reinterpret_cast<const float4*>(tab + base + 4 * g);
      body<T>(b, q, acc);
    }
  }
  float r = 0; for (int i = 0; i < T; ++i) r += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int MODE, int T> void run(const char* name, const float* in, float* out, int SM, int threads, int bps) {
  int iters = 4096; cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); kern<MODE, T><<<SM * bps, threads>>>(in, out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  double cands = (double)SM * bps * threads * iters * T * 16;
  printf("%-28s T=%2d %4dx%d  %7.3f ms  %6.1f cand/clk/SM @1.965GHz  err=%s\n", name, T, threads, bps, ms,
         cands / (ms * 1e-3) / SM / 1.965e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0); int SM = p.multiProcessorCount;
  float *in, *out; cudaMalloc(&in, 4096 * 4); cudaMalloc(&out, 64 << 20);
  float h[4096]; for (int i = 0; i < 4096; ++i) h[i] = 1.0f + (i % 97) * 0.01f;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice); cudaMemcpyToSymbol(cb, h, sizeof(h));
  for (int bps : {2, 3, 4}) {
    run<0, 8>("LV lane-varying smem", in, out, SM, 256, bps);
    run<1, 8>("WU warp-uniform smem", in, out, SM, 256, bps);
    run<2, 8>("CB constant bank (UR)", in, out, SM, 256, bps);
  }
  run<2, 16>("CB constant bank T=16", in, out, SM, 256, 2);
  run<1, 16>("WU warp-uniform T=16", in, out, SM, 256, 2);
  run<2, 4>("CB constant bank T=4", in, out, SM, 256, 4);
  return 0;
}
