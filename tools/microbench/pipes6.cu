// Microbenchmark v6: the kernel's inner loop (T = 12 rows per lane, 18 b values per masked row,
// per-a Q_a = Q + tau_a, FADD2 row pairs + FMNMX3) with the b row taken from
//   UR : the constant bank at a warp-uniform index -> LDCU + FADD2 R, R.F32x2, UR
//        (single-warp blocks; row index from blockIdx + loop counter, which ptxas keeps uniform)
//   SM : shared memory (LDS.128), 256-thread blocks, row index from the same uniform sequence
// Prints candidates/clk/SM at 1.965 GHz.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int T = 12, KB = 18, ROWS = 8, STRIDE = 20, KA = 18;
__constant__ float c_b[ROWS * STRIDE];
__constant__ float c_a[KA];

__device__ __forceinline__ void add2b(float &v0, float &v1, float q0, float q1, float b) {
  asm("{.reg .b64 x,y,z;\n\tmov.b64 x,{%2,%3};\n\tmov.b64 y,{%4,%4};\n\tadd.rn.f32x2 z,x,y;\n\tmov.b64 {%0,%1},z;}"
      : "=f"(v0), "=f"(v1) : "f"(q0), "f"(q1), "f"(b));
}
__device__ __forceinline__ float min3(float a, float b, float c) {
  float d; asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d;
}
template <class BF>
__device__ __forceinline__ void row_eval(const float (&Qa)[T], float (&acc)[T], BF bval) {
#pragma unroll
  for (int j = 0; j < KB; j += 2) {
    const float b0 = bval(j), b1 = bval(j + 1);
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
      row_eval(Qa, acc, [&](int j) { return c_b[r * STRIDE + j]; });
    }
  }
  float s = 0; for (int i = 0; i < T; ++i) s += acc[i];
  out[blockIdx.x * 32 + threadIdx.x] = s;
}

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
      const int r = (it + a * 3) & (ROWS - 1);
      float Qa[T];
#pragma unroll
      for (int i = 0; i < T; i += 2) add2b(Qa[i], Qa[i + 1], Q[i], Q[i + 1], ta);
      const float *rp = sb + r * STRIDE;
      float bv[KB];
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        const float4 v = *reinterpret_cast<const float4 *>(rp + j);
        bv[j] = v.x; bv[j + 1] = v.y; bv[j + 2] = v.z; bv[j + 3] = v.w;
      }
      const float2 t2 = *reinterpret_cast<const float2 *>(rp + 16);
      bv[16] = t2.x; bv[17] = t2.y;
      row_eval(Qa, acc, [&](int j) { return bv[j]; });
    }
  }
  float s = 0; for (int i = 0; i < T; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0); const int SM = p.multiProcessorCount;
  float *in, *out; cudaMalloc(&in, 4096 * 4); cudaMalloc(&out, 64 << 20);
  float h[1024]; for (int i = 0; i < 1024; ++i) h[i] = 1.0f + (i % 97) * 0.01f;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(c_b, h, sizeof(float) * ROWS * STRIDE);
  cudaMemcpyToSymbol(c_a, h + 300, sizeof(float) * KA);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    for (int wps : {12, 16, 20, 24}) {   // warps per SM for the single-warp-block kernel
      const int grid = SM * wps, iters = grid * 40;
      float ms = 0;
      for (int k = 0; k < 3; ++k) { cudaEventRecord(e0); k_ur<<<grid, 32>>>(in, out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); }
      const double cand = (double)iters * 32 * T * KA * KB;
      printf("UR single-warp blocks, %2d warps/SM: %7.3f ms %6.1f cand/clk/SM  %s\n", wps, ms, cand / (ms * 1e-3) / SM / 1.965e9, cudaGetErrorString(cudaGetLastError()));
    }
    {
      const int grid = SM * 2, iters = grid * 8 * 40;
      float ms = 0;
      for (int k = 0; k < 3; ++k) { cudaEventRecord(e0); k_sm<<<grid, 256>>>(in, out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); }
      const double cand = (double)iters * 32 * T * KA * KB;
      printf("SM 256-thread blocks x2/SM        : %7.3f ms %6.1f cand/clk/SM  %s\n", ms, cand / (ms * 1e-3) / SM / 1.965e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
