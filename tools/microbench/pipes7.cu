// Microbenchmark v7: the uniform-register inner loop in two encodings (single-warp blocks, b row in
// the constant bank at a warp-uniform index, per-a Q_a = Q + tau_a):
//   RP : row pairs   FADD2 {Q_i, Q_i+1} + {b, b}  (b: one LDCU per value; round-1 kernel form)
//   QB : Q broadcast FADD2 Q_i.F32 + {b_j, b_j+1}  (b pair: one LDCU.64 per two values; the scalar
//        vector operand is broadcast by the .F32 modifier, so no duplicated registers)
// with T rows per lane (12 or 16) and KB b values per masked row (18; 64 for long rows).
// Prints candidates/clk/SM at 1.965 GHz.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ROWS = 8, STRIDE = 68, KA = 18;
__constant__ __align__(16) float c_b[ROWS * STRIDE];
__constant__ float c_a[KA];

__device__ __forceinline__ void add2b(float &v0, float &v1, float q0, float q1, float b) {
  asm("{.reg .b64 x,y,z;\n\tmov.b64 x,{%2,%3};\n\tmov.b64 y,{%4,%4};\n\tadd.rn.f32x2 z,x,y;\n\tmov.b64 {%0,%1},z;}"
      : "=f"(v0), "=f"(v1) : "f"(q0), "f"(q1), "f"(b));
}
__device__ __forceinline__ void add2q(float &v0, float &v1, float q, float b0, float b1) {
  asm("{.reg .b64 x,y,z;\n\tmov.b64 x,{%2,%2};\n\tmov.b64 y,{%3,%4};\n\tadd.rn.f32x2 z,x,y;\n\tmov.b64 {%0,%1},z;}"
      : "=f"(v0), "=f"(v1) : "f"(q), "f"(b0), "f"(b1));
}
__device__ __forceinline__ float min3(float a, float b, float c) {
  float d; asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d;
}

template <int T, int KB, bool QB>
__global__ void __launch_bounds__(32) k_ur(const float *in, float *out, int iters) {
  float Q[T], acc[T];
  for (int i = 0; i < T; ++i) { Q[i] = in[(threadIdx.x * 7 + i) & 1023]; acc[i] = 3e38f; }
  for (int it = blockIdx.x; it < iters; it += gridDim.x) {   // uniform item sequence
#pragma unroll 2
    for (int a = 0; a < KA; ++a) {
      const float ta = c_a[a];
      const int r = (it + a * 3) & (ROWS - 1);                // uniform masked-row index
      float Qa[T];
#pragma unroll
      for (int i = 0; i < T; i += 2) add2b(Qa[i], Qa[i + 1], Q[i], Q[i + 1], ta);
      const float *rb = c_b + r * STRIDE;
      if constexpr (QB) {
#pragma unroll
        for (int j = 0; j < KB; j += 2) {
          const float2 b = *reinterpret_cast<const float2 *>(rb + j);
#pragma unroll
          for (int i = 0; i < T; ++i) {
            float x, y;
            add2q(x, y, Qa[i], b.x, b.y);
            acc[i] = min3(acc[i], x, y);
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < KB; j += 2) {
          const float b0 = rb[j], b1 = rb[j + 1];
#pragma unroll
          for (int i = 0; i < T; i += 2) {
            float x0, y0, x1, y1;
            add2b(x0, y0, Qa[i], Qa[i + 1], b0);
            add2b(x1, y1, Qa[i], Qa[i + 1], b1);
            acc[i] = min3(acc[i], x0, x1);
            acc[i + 1] = min3(acc[i + 1], y0, y1);
          }
        }
      }
    }
  }
  float s = 0; for (int i = 0; i < T; ++i) s += acc[i];
  out[blockIdx.x * 32 + threadIdx.x] = s;
}

// the same loop with the b row in shared memory (256-thread blocks, 2/SM, like k_search / the mixed
// groups): RP reads b via LDS.128 + row pairs; QB reads b pairs via LDS.64 + Q broadcast
template <int T, int KB, bool QB>
__global__ void __launch_bounds__(256, 2) k_sm(const float *in, float *out, int iters) {
  __shared__ __align__(16) float sb[ROWS * STRIDE];
  __shared__ float sa[KA];
  for (int i = threadIdx.x; i < ROWS * STRIDE; i += blockDim.x) sb[i] = in[i & 1023];
  for (int i = threadIdx.x; i < KA; i += blockDim.x) sa[i] = in[(i * 3) & 1023];
  __syncthreads();
  float Q[T], acc[T];
  for (int i = 0; i < T; ++i) { Q[i] = in[(threadIdx.x * 7 + i) & 1023]; acc[i] = 3e38f; }
  const int warps = gridDim.x * (blockDim.x >> 5);
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  for (int it = w; it < iters; it += warps) {
#pragma unroll 2
    for (int a = 0; a < KA; ++a) {
      const float ta = sa[a];
      const int r = (it + a * 3 + (threadIdx.x & 1)) & (ROWS - 1);   // lane-varying row
      float Qa[T];
#pragma unroll
      for (int i = 0; i < T; i += 2) add2b(Qa[i], Qa[i + 1], Q[i], Q[i + 1], ta);
      const float *rp = sb + r * STRIDE;
      if constexpr (QB) {
#pragma unroll
        for (int j = 0; j < KB; j += 2) {
          const float2 b = *reinterpret_cast<const float2 *>(rp + j);
#pragma unroll
          for (int i = 0; i < T; ++i) {
            float x, y;
            add2q(x, y, Qa[i], b.x, b.y);
            acc[i] = min3(acc[i], x, y);
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < KB - 3; j += 4) {
          const float4 v = *reinterpret_cast<const float4 *>(rp + j);
#pragma unroll
          for (int i = 0; i < T; i += 2) {
            float a0, b0, a1, b1, a2, b2, a3, b3;
            add2b(a0, b0, Qa[i], Qa[i + 1], v.x); add2b(a1, b1, Qa[i], Qa[i + 1], v.y);
            add2b(a2, b2, Qa[i], Qa[i + 1], v.z); add2b(a3, b3, Qa[i], Qa[i + 1], v.w);
            acc[i] = min3(acc[i], a0, a1); acc[i + 1] = min3(acc[i + 1], b0, b1);
            acc[i] = min3(acc[i], a2, a3); acc[i + 1] = min3(acc[i + 1], b2, b3);
          }
        }
        if constexpr (KB % 4 == 2) {
          const float2 v = *reinterpret_cast<const float2 *>(rp + KB - 2);
#pragma unroll
          for (int i = 0; i < T; i += 2) {
            float a0, b0, a1, b1;
            add2b(a0, b0, Qa[i], Qa[i + 1], v.x); add2b(a1, b1, Qa[i], Qa[i + 1], v.y);
            acc[i] = min3(acc[i], a0, a1); acc[i + 1] = min3(acc[i + 1], b0, b1);
          }
        }
      }
    }
  }
  float s = 0; for (int i = 0; i < T; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int T, int KB, bool QB>
void run_sm(const char *name, int SM, const float *in, float *out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k_sm<T, KB, QB>);
  const int grid = SM * 2, iters = grid * 8 * 40;
  float ms = 0;
  for (int k = 0; k < 3; ++k) { cudaEventRecord(e0); k_sm<T, KB, QB><<<grid, 256>>>(in, out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); }
  const double cand = (double)iters * 32 * T * KA * KB;
  printf("%-4s SMEM T=%2d KB=%2d regs=%3d 2x256/SM     : %7.3f ms %6.1f cand/clk/SM  %s\n", name, T, KB, fa.numRegs, ms,
         cand / (ms * 1e-3) / SM / 1.965e9, cudaGetErrorString(cudaGetLastError()));
}

template <int T, int KB, bool QB>
void run(const char *name, int SM, const float *in, float *out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int regs = 0;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k_ur<T, KB, QB>); regs = fa.numRegs;
  for (int wps : {16, 20, 24}) {
    const int grid = SM * wps, iters = grid * 40;
    float ms = 0;
    for (int k = 0; k < 3; ++k) { cudaEventRecord(e0); k_ur<T, KB, QB><<<grid, 32>>>(in, out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); }
    const double cand = (double)iters * 32 * T * KA * KB;
    printf("%-4s T=%2d KB=%2d regs=%3d %2d warps/SM: %7.3f ms %6.1f cand/clk/SM  %s\n", name, T, KB, regs, wps, ms,
           cand / (ms * 1e-3) / SM / 1.965e9, cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0); const int SM = p.multiProcessorCount;
  float *in, *out; cudaMalloc(&in, 4096 * 4); cudaMalloc(&out, 64 << 20);
  float h[1024]; for (int i = 0; i < 1024; ++i) h[i] = 1.0f + (i % 97) * 0.01f;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(c_b, h, sizeof(float) * ROWS * STRIDE);
  cudaMemcpyToSymbol(c_a, h + 300, sizeof(float) * KA);
  for (int rep = 0; rep < 2; ++rep) {
    run<12, 18, false>("RP", SM, in, out);
    run<12, 18, true>("QB", SM, in, out);
    run<16, 18, false>("RP", SM, in, out);
    run<16, 18, true>("QB", SM, in, out);
    run<12, 64, false>("RP", SM, in, out);
    run<12, 64, true>("QB", SM, in, out);
    run<16, 64, true>("QB", SM, in, out);
    run_sm<12, 18, false>("RP", SM, in, out);
    run_sm<12, 18, true>("QB", SM, in, out);
    run_sm<12, 64, false>("RP", SM, in, out);
    run_sm<12, 64, true>("QB", SM, in, out);
  }
  return 0;
}
