// Dependent-chain latencies on one warp (cycles per op): FP64 add/mul/div,
// ceil, shared-memory load, shuffle, redux, syncwarp.  nvcc -arch=sm_100a --fmad=false
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
  __shared__ int sidx[1024];
  for (int i = threadIdx.x; i < 1024; i += 32) sidx[i] = (i * 7 + 1) & 1023;
  __syncwarp();
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) x = __dadd_rn(x, b);
  long long t1 = clock64();
  for (int i = 0; i < n; i++) x = __dmul_rn(x, b);
  long long t2 = clock64();
  for (int i = 0; i < n; i++) x = __ddiv_rn(x, b);
  long long t3 = clock64();
  for (int i = 0; i < n; i++) x = ceil(x + 0.5);
  long long t4 = clock64();
  int j = threadIdx.x;
  for (int i = 0; i < n; i++) j = sidx[j];
  long long t5 = clock64();
  int v = j;
  for (int i = 0; i < n; i++) v = __shfl_sync(0xffffffffu, v, (v + 1) & 31);
  long long t6 = clock64();
  unsigned r = v;
  for (int i = 0; i < n; i++) r = __reduce_min_sync(0xffffffffu, r + threadIdx.x);
  long long t7 = clock64();
  for (int i = 0; i < n; i++) { r += threadIdx.x; __syncwarp(); }
  long long t8 = clock64();
  double y = a;
  for (int i = 0; i < n; i++) y = (double)(long long)ceil(__dsub_rn(__ddiv_rn(y, b), 1e-12)) + a;
  long long t9 = clock64();
  out[threadIdx.x] = x + j + v + r + y;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
    cyc[5] = t6 - t5; cyc[6] = t7 - t6; cyc[7] = t8 - t7; cyc[8] = t9 - t8;
  }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMallocManaged(&c, 128);
  const int n = 1000;
  for (int rep = 0; rep < 2; rep++) { lat<<<1, 32>>>(o, c, 1.2345, 1.0001, n); cudaDeviceSynchronize(); }
  const char* nm[] = {"dadd", "dmul", "ddiv_rn", "ceil(x+.5)", "LDS chain", "SHFL chain", "REDUX chain", "syncwarp+iadd",
                      "ceil(ddiv-1e-12)+cvt"};
  for (int i = 0; i < 9; i++) printf("%-22s %6.1f cycles/op\n", nm[i], (double)c[i] / n);
  return 0;
}
