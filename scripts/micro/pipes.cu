// Throughput probe: warp-instructions per SM per cycle for a few ops the
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/micro/pipes scripts/micro/pipes.cu
// gather's inner loop uses (F2F.F64.F32, DADD, DFMA, FFMA, integer-only f32->f64).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_f2f(const float *in, double *out, int iters) {
  float a = in[threadIdx.x & 31], b = a * 1.5f, c = a * 0.5f, d = a + 2.f;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < iters; ++i) {
    s0 += (double)a; s1 += (double)b; s2 += (double)c; s3 += (double)d;
    a += 1e-7f; b += 1e-7f; c += 1e-7f; d += 1e-7f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
__device__ __forceinline__ double f2d_int(float f) {
  const uint32_t b = __float_as_uint(f);
  const uint32_t hi = (b & 0x80000000u) | (((b & 0x7fffffffu) >> 3) + 0x38000000u);
  return __hiloint2double((int)hi, (int)(b << 29));
}
__global__ void k_f2i(const float *in, double *out, int iters) {
  float a = in[threadIdx.x & 31], b = a * 1.5f, c = a * 0.5f, d = a + 2.f;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < iters; ++i) {
    s0 += f2d_int(a); s1 += f2d_int(b); s2 += f2d_int(c); s3 += f2d_int(d);
    a += 1e-7f; b += 1e-7f; c += 1e-7f; d += 1e-7f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
__global__ void k_dadd(const float *in, double *out, int iters) {
  double a = in[threadIdx.x & 31], s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0, s6 = 0, s7 = 0;
  for (int i = 0; i < iters; ++i) {
    s0 += a; s1 += a; s2 += a; s3 += a; s4 += a; s5 += a; s6 += a; s7 += a;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3 + s4 + s5 + s6 + s7;
}
__global__ void k_fadd(const float *in, double *out, int iters) {
  float a = in[threadIdx.x & 31], s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0, s6 = 0, s7 = 0;
  for (int i = 0; i < iters; ++i) {
    s0 += a; s1 += a; s2 += a; s3 += a; s4 += a; s5 += a; s6 += a; s7 += a;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3 + s4 + s5 + s6 + s7;
}
template <typename K>
void run(const char *name, K k, int ops_per_iter, const float *in, double *out) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 4096, threads = 512, blocks = sms * 4;
  k<<<blocks, threads>>>(in, out, 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<blocks, threads>>>(in, out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double warp_ops = (double)blocks * threads / 32 * iters * ops_per_iter;
  const double cycles = ms * 1e-3 * clk * 1e3;
  printf("%-8s %.3f ms  %.2f warp-ops/SM/clk (at %d MHz nominal)\n", name, ms, warp_ops / sms / cycles, clk / 1000);
}
int main() {
  float *in; double *out;
  cudaMalloc(&in, 32 * 4); cudaMemset(in, 0, 128);
  cudaMalloc(&out, 148 * 4 * 512 * 8);
  run("f2f", k_f2f, 4, in, out);
  run("f2d_int", k_f2i, 4, in, out);
  run("dadd", k_dadd, 8, in, out);
  run("fadd", k_fadd, 8, in, out);
  return 0;
}
