// FP64 throughput microbenchmark for B200 (sm_100a): DFMA vs DMMA (mma.sync f64).
// Measures the roofline denominator for the FP64 congruence kernels:
// MEASURED_PEAKS.json carries no FP64 entry, so this tool measures it on the box.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int ITERS>
__global__ void dfma_kernel(double* out, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; i++) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += x[i];
  if (s == 1234.5) out[threadIdx.x] = s;
}

// m8n8k4: A 1 reg, B 1 reg, C/D 2 regs
template<int ITERS>
__global__ void dmma_884_kernel(double* out, double a0) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; i++) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = a0 + threadIdx.x, b = a0 - threadIdx.x;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += acc[i][0] + acc[i][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}

// m16n8k4: A 2 regs, B 1 reg, C/D 4 regs
template<int ITERS>
__global__ void dmma_1684_kernel(double* out, double a0) {
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) acc[i][j] = 0;
  double a = a0 + threadIdx.x, a1 = a0 * 2, b = a0 - threadIdx.x;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++) {
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3]) : "d"(a), "d"(a1), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 1234.5) out[threadIdx.x] = s;
}

// m16n8k16: A 8 regs, B 4 regs, C/D 4 regs
template<int ITERS>
__global__ void dmma_16816_kernel(double* out, double a0) {
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) acc[i][j] = 0;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; i++) a[i] = a0 + i + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 4; i++) b[i] = a0 - i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <typename F>
float timeit(F f, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int i = 0; i < reps; i++) f();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; CK(cudaMalloc(&out, 4096 * sizeof(double)));
  const int IT = 4096;
  for (int threads : {256, 512}) for (int bps : {1, 2, 4}) {
    int grid = sms * bps;
    float ms = timeit([&] { dfma_kernel<IT><<<grid, threads>>>(out, 0.999, 1e-3); }, 5);
    double fl = 2.0 * 16 * IT * (double)grid * threads;
    printf("DFMA      grid=%d thr=%d: %.3f ms  %.2f TFLOP/s\n", grid, threads, ms, fl / ms / 1e9);
    ms = timeit([&] { dmma_884_kernel<IT><<<grid, threads>>>(out, 0.5); }, 5);
    fl = 2.0 * 8 * 8 * 4 * 8 * IT * (double)grid * (threads / 32);
    printf("DMMA884   grid=%d thr=%d: %.3f ms  %.2f TFLOP/s\n", grid, threads, ms, fl / ms / 1e9);
    ms = timeit([&] { dmma_1684_kernel<IT><<<grid, threads>>>(out, 0.5); }, 5);
    fl = 2.0 * 16 * 8 * 4 * 4 * IT * (double)grid * (threads / 32);
    printf("DMMA1684  grid=%d thr=%d: %.3f ms  %.2f TFLOP/s\n", grid, threads, ms, fl / ms / 1e9);
    ms = timeit([&] { dmma_16816_kernel<IT / 4><<<grid, threads>>>(out, 0.5); }, 5);
    fl = 2.0 * 16 * 8 * 16 * 4 * (IT / 4) * (double)grid * (threads / 32);
    printf("DMMA16816 grid=%d thr=%d: %.3f ms  %.2f TFLOP/s\n", grid, threads, ms, fl / ms / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}
