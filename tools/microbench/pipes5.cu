// Pipe/issue microbenchmark v5: register-bank layout of the FADD2 + FMNMX3 inner loop (sm_100a).
// Same harness as pipes3 (b from a conflict-free shared row, 4 groups of 4 b per iteration, T rows
// per thread).  Variants differ only in which registers the FMNMX3 sources land in:
//   V1  row-pair FADD2 {Q_i,Q_i+1}+{b,b}; FMNMX3 acc_i = min(acc_i, lo(b0), lo(b1))  (kernel today:
//       both fresh sources of a row sit in the same bank)
//   V7  row-pair with a swapped pair {Q_i+1,Q_i} for every second b, so each FMNMX3 takes one even
//       and one odd fresh register
//   V8  Q broadcast {Q_i,Q_i}+{b0,b1}, rows inner (the b pair stays in the reuse cache)
//   V0  Q broadcast, rows outer
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void add2(float& v0, float& v1, float q, float b0, float b1) {
  asm("{.reg .b64 x,y,z; mov.b64 x,{%2,%2}; mov.b64 y,{%3,%4}; add.rn.f32x2 z,x,y; mov.b64 {%0,%1},z;}"
      : "=f"(v0), "=f"(v1) : "f"(q), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void add2b(float& v0, float& v1, float q0, float q1, float b) {
  asm("{.reg .b64 x,y,z; mov.b64 x,{%2,%3}; mov.b64 y,{%4,%4}; add.rn.f32x2 z,x,y; mov.b64 {%0,%1},z;}"
      : "=f"(v0), "=f"(v1) : "f"(q0), "f"(q1), "f"(b));
}
__device__ __forceinline__ float min3(float a, float b, float c) {
  float d; asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d;
}

template <int V, int T>
__global__ void __launch_bounds__(256, 3) kern(const float* in, float* out, int iters) {
  __shared__ __align__(16) float tab[8 * 20 * 4];
  for (int i = threadIdx.x; i < 8 * 20 * 4; i += blockDim.x) tab[i] = in[i & 1023];
  __syncthreads();
  float q[T], acc[T];
  for (int i = 0; i < T; ++i) { q[i] = in[(threadIdx.x + i) & 1023]; acc[i] = 3e38f; }
  const int lane = threadIdx.x & 31;
  const float* row = tab + (lane & 7) * 20;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const float* rp = row + ((it & 3) * 160);
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const float4 b = *reinterpret_cast<const float4*>(rp + 4 * g);
      if constexpr (V == 1) {
#pragma unroll
        for (int i = 0; i < T; i += 2) { float a0,b0,a1,b1,a2,b2,a3,b3;
          add2b(a0,b0,q[i],q[i+1],b.x); add2b(a1,b1,q[i],q[i+1],b.y); add2b(a2,b2,q[i],q[i+1],b.z); add2b(a3,b3,q[i],q[i+1],b.w);
          acc[i]=min3(acc[i],a0,a1); acc[i+1]=min3(acc[i+1],b0,b1); acc[i]=min3(acc[i],a2,a3); acc[i+1]=min3(acc[i+1],b2,b3); }
      } else if constexpr (V == 7) {
#pragma unroll
        for (int i = 0; i < T; i += 2) { float a0,b0,a1,b1,a2,b2,a3,b3;
          add2b(a0,b0,q[i],q[i+1],b.x); add2b(b1,a1,q[i+1],q[i],b.y); add2b(a2,b2,q[i],q[i+1],b.z); add2b(b3,a3,q[i+1],q[i],b.w);
          acc[i]=min3(acc[i],a0,a1); acc[i+1]=min3(acc[i+1],b0,b1); acc[i]=min3(acc[i],a2,a3); acc[i+1]=min3(acc[i+1],b2,b3); }
      } else if constexpr (V == 8) {
#pragma unroll
        for (int i = 0; i < T; ++i) { float v0, v1; add2(v0, v1, q[i], b.x, b.y); acc[i] = min3(acc[i], v0, v1); }
#pragma unroll
        for (int i = 0; i < T; ++i) { float v0, v1; add2(v0, v1, q[i], b.z, b.w); acc[i] = min3(acc[i], v0, v1); }
      } else if constexpr (V == 0) {
#pragma unroll
        for (int i = 0; i < T; ++i) { float v0, v1, v2, v3; add2(v0, v1, q[i], b.x, b.y); add2(v2, v3, q[i], b.z, b.w);
          acc[i] = min3(acc[i], v0, v1); acc[i] = min3(acc[i], v2, v3); }
      }
    }
  }
  float r = 0; for (int i = 0; i < T; ++i) r += acc[i] + q[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int V, int T> void run(const char* name, const float* in, float* out, int SM, int threads, int bps) {
  int iters = 4096; cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); kern<V, T><<<SM * bps, threads>>>(in, out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  double cands = (double)SM * bps * threads * iters * T * 16;
  printf("%-34s T=%2d %4dx%d  %7.3f ms  %6.1f cand/clk/SM @1.965GHz  err=%s\n", name, T, threads, bps, ms,
         cands / (ms * 1e-3) / SM / 1.965e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0); int SM = p.multiProcessorCount;
  float *in, *out; cudaMalloc(&in, 4096 * 4); cudaMalloc(&out, 64 << 20);
  float h[1024]; for (int i = 0; i < 1024; ++i) h[i] = 1.0f + (i % 97) * 0.01f; cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) {
    run<1, 8>("V1 row-pair (kernel today)", in, out, SM, 256, 3);
    run<7, 8>("V7 row-pair, swapped every 2nd b", in, out, SM, 256, 3);
    run<8, 8>("V8 Q-bcast, rows inner", in, out, SM, 256, 3);
    run<0, 8>("V0 Q-bcast, rows outer", in, out, SM, 256, 3);
  }
  return 0;
}
