// FP64 / SHFL latency and throughput on the local GPU (design input for the
// stencil kernels).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 dp_microbench.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat_dadd(double* out, double a, int n, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __dadd_rn(x, a); x = __dadd_rn(x, a); x = __dadd_rn(x, a); x = __dadd_rn(x, a); }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_dmul(double* out, double a, int n, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __dmul_rn(x, a); x = __dmul_rn(x, a); x = __dmul_rn(x, a); x = __dmul_rn(x, a); }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void lat_shfl(double* out, double a, int n, long long* cyc) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __shfl_down_sync(0xffffffff, x, 1); x = __shfl_down_sync(0xffffffff, x, 1); }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
template <int ILP>
__global__ void thr_dadd(double* out, double a, int n) {
  double x[ILP];
  for (int j = 0; j < ILP; ++j) x[j] = a * (threadIdx.x + j);
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < ILP; ++j) x[j] = __dadd_rn(x[j], a);
  double s = 0; for (int j = 0; j < ILP; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 1 << 26); cudaMalloc(&c, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int n = 1 << 16;
  long long h;
  lat_dadd<<<1, 32>>>(d, 1e-9, n, c); lat_dadd<<<1, 32>>>(d, 1e-9, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
  lat_dmul<<<1, 32>>>(d, 1.0000001, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DMUL dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
  lat_shfl<<<1, 32>>>(d, 1.0, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("SHFL(double) dependent latency: %.2f cycles\n", (double)h / (2.0 * n));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    const int it = 1 << 14;
    thr_dadd<8><<<sms, warps * 32>>>(d, 1e-9, it);
    cudaEventRecord(e0); thr_dadd<8><<<sms, warps * 32>>>(d, 1e-9, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)sms * warps * 32 * it * 8;
    printf("DADD throughput %2d warps/SM ILP8: %.1f Gop/s = %.1f lanes/clk/SM @1.965GHz\n", warps, ops / ms / 1e6, ops / (ms * 1e-3) / sms / 1.965e9);
  }
  return 0;
}
