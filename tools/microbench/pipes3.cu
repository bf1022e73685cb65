// Pipe/issue microbenchmark v3 for the ALP search inner loop on sm_100a.
// b values come from a bank-conflict-free shared-memory row (row stride 20 floats, 8 rows per warp)
// at an iteration-dependent column, so nothing can be hoisted.  Each variant is a different encoding
// of "v = Q + b; acc = min(acc, v)" (or a single-pipe stress test); prints candidates/clk/SM and the
// implied warp-instructions/clk/SMSP using the SASS instruction count per iteration.
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
__device__ __forceinline__ float min2(float a, float b) { float d; asm("min.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b)); return d; }
__device__ __forceinline__ unsigned imin(unsigned a, unsigned b) { unsigned d; asm("min.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }

template <int V, int T>
__global__ void kern(const float* in, float* out, int iters) {
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
      if constexpr (V == 0) {
#pragma unroll
        for (int i = 0; i < T; ++i) { float v0, v1, v2, v3; add2(v0, v1, q[i], b.x, b.y); add2(v2, v3, q[i], b.z, b.w);
          acc[i] = min3(acc[i], v0, v1); acc[i] = min3(acc[i], v2, v3); }
      } else if constexpr (V == 1) {
#pragma unroll
        for (int i = 0; i < T; i += 2) { float a0,b0,a1,b1,a2,b2,a3,b3;
          add2b(a0,b0,q[i],q[i+1],b.x); add2b(a1,b1,q[i],q[i+1],b.y); add2b(a2,b2,q[i],q[i+1],b.z); add2b(a3,b3,q[i],q[i+1],b.w);
          acc[i]=min3(acc[i],a0,a1); acc[i+1]=min3(acc[i+1],b0,b1); acc[i]=min3(acc[i],a2,a3); acc[i+1]=min3(acc[i+1],b2,b3); }
      } else if constexpr (V == 2) {  // FMNMX3 only: 2 per row per group
#pragma unroll
        for (int i = 0; i < T; ++i) { acc[i] = min3(acc[i], b.x + 0.f * q[i], b.y); acc[i] = min3(acc[i], b.z, b.w); }
      } else if constexpr (V == 3) {  // FADD2 only: 2 per row per group (accumulate into q pairs)
#pragma unroll
        for (int i = 0; i < T; i += 2) { float a0,b0,a1,b1; add2b(a0,b0,q[i],q[i+1],b.x); add2b(a1,b1,a0,b0,b.y); q[i]=a1; q[i+1]=b1;
          add2b(a0,b0,q[i],q[i+1],b.z); add2b(a1,b1,a0,b0,b.w); q[i]=a1; q[i+1]=b1; }
      } else if constexpr (V == 4) {  // FADD2 + FMNMX (2-input) x4
#pragma unroll
        for (int i = 0; i < T; ++i) { float v0, v1, v2, v3; add2(v0, v1, q[i], b.x, b.y); add2(v2, v3, q[i], b.z, b.w);
          acc[i] = min2(acc[i], v0); acc[i] = min2(acc[i], v1); acc[i] = min2(acc[i], v2); acc[i] = min2(acc[i], v3); }
      } else if constexpr (V == 5) {  // FADD2 + integer min on float bits (IMNMX)
#pragma unroll
        for (int i = 0; i < T; ++i) { float v0, v1, v2, v3; add2(v0, v1, q[i], b.x, b.y); add2(v2, v3, q[i], b.z, b.w);
          unsigned a = __float_as_uint(acc[i]); a = imin(a, __float_as_uint(v0)); a = imin(a, __float_as_uint(v1));
          a = imin(a, __float_as_uint(v2)); a = imin(a, __float_as_uint(v3)); acc[i] = __uint_as_float(a); }
      } else if constexpr (V == 6) {  // FADD2 (pair rows) + FMNMX3 tree over 4 then 1 fold
#pragma unroll
        for (int i = 0; i < T; i += 2) { float a0,b0,a1,b1,a2,b2,a3,b3;
          add2b(a0,b0,q[i],q[i+1],b.x); add2b(a1,b1,q[i],q[i+1],b.y); add2b(a2,b2,q[i],q[i+1],b.z); add2b(a3,b3,q[i],q[i+1],b.w);
          acc[i]=min3(acc[i],min3(a0,a1,a2),a3); acc[i+1]=min3(acc[i+1],min3(b0,b1,b2),b3); }
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
  double cands = (double)SM * bps * threads * iters * T * 16;  // 4 groups x 4 b x T rows
  printf("%-40s T=%2d %4dx%d  %7.3f ms  %6.1f cand/clk/SM @1.965GHz  err=%s\n", name, T, threads, bps, ms,
         cands / (ms * 1e-3) / SM / 1.965e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0); int SM = p.multiProcessorCount;
  float *in, *out; cudaMalloc(&in, 4096 * 4); cudaMalloc(&out, 64 << 20);
  float h[1024]; for (int i = 0; i < 1024; ++i) h[i] = 1.0f + (i % 97) * 0.01f; cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int bps : {2, 3, 4}) {
    run<0, 8>("V0 FADD2(Qbcast)+FMNMX3", in, out, SM, 256, bps);
    run<1, 8>("V1 FADD2(rowpair,bbcast)+FMNMX3", in, out, SM, 256, bps);
    run<6, 8>("V6 rowpair + FMNMX3 tree", in, out, SM, 256, bps);
    run<2, 8>("V2 FMNMX3 only (cand=fold)", in, out, SM, 256, bps);
    run<3, 8>("V3 FADD2 only (cand=add)", in, out, SM, 256, bps);
    run<4, 8>("V4 FADD2 + FMNMX x4", in, out, SM, 256, bps);
    run<5, 8>("V5 FADD2 + IMNMX x4", in, out, SM, 256, bps);
  }
  run<1, 16>("V1 rowpair T=16", in, out, SM, 256, 2);
  run<1, 4>("V1 rowpair T=4", in, out, SM, 256, 4);
  return 0;
}
