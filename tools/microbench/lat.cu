// Latency microbenchmark (single warp): cycles per dependent op on B200.
#include <cstdio>
#include <cstdint>
__global__ void k(double* out, long long* cyc, int n, double x0, int* iout) {
  __shared__ double sm[64];
  __shared__ int smi[64];
  for (int i = threadIdx.x; i < 64; i += 32) { sm[i] = i * 0.5; smi[i] = (i + 1) & 63; }
  __syncwarp();
  double x = x0, y = x0 * 0.5;
  long long t0, t1;
  // 0: DADD chain
  t0 = clock64(); for (int i = 0; i < n; ++i) x = __dadd_rn(x, y); t1 = clock64(); cyc[0] = t1 - t0;
  // 1: DMUL chain
  t0 = clock64(); for (int i = 0; i < n; ++i) x = __dmul_rn(x, 1.0000001); t1 = clock64(); cyc[1] = t1 - t0;
  // 2: DADD.RD chain
  t0 = clock64(); for (int i = 0; i < n; ++i) x = __dadd_rd(x, y); t1 = clock64(); cyc[2] = t1 - t0;
  // 3: LDS dependent chain (int index)
  int j = threadIdx.x & 63;
  t0 = clock64(); for (int i = 0; i < n; ++i) j = smi[j]; t1 = clock64(); cyc[3] = t1 - t0;
  // 4: IADD chain
  int a = j;
  t0 = clock64(); for (int i = 0; i < n; ++i) a = a * 3 + 1; t1 = clock64(); cyc[4] = t1 - t0;
  // 5: DSETP + branch chain
  double z = x;
  t0 = clock64(); for (int i = 0; i < n; ++i) { if (z < y) z = __dadd_rn(z, 1.0); else z = __dsub_rn(z, 0.5); } t1 = clock64(); cyc[5] = t1 - t0;
  // 6: shfl chain
  int b = threadIdx.x;
  t0 = clock64(); for (int i = 0; i < n; ++i) b = __shfl_sync(0xffffffffu, b, (b + 1) & 31); t1 = clock64(); cyc[6] = t1 - t0;
  // 7: REDUX chain
  unsigned c = threadIdx.x;
  t0 = clock64(); for (int i = 0; i < n; ++i) c = __reduce_min_sync(0xffffffffu, c + threadIdx.x); t1 = clock64(); cyc[7] = t1 - t0;
  // 8: I2F.F64 + F2I chain
  long long q = j;
  t0 = clock64(); for (int i = 0; i < n; ++i) q = (long long)((double)q * 1.0) + 1; t1 = clock64(); cyc[8] = t1 - t0;
  // 9: 64-bit int mul chain
  long long m = q | 1;
  t0 = clock64(); for (int i = 0; i < n; ++i) m = m * 7 + 3; t1 = clock64(); cyc[9] = t1 - t0;
  // 10: LDS double dependent (address from value)
  double v = sm[j & 63];
  t0 = clock64(); for (int i = 0; i < n; ++i) v = sm[((int)v) & 63]; t1 = clock64(); cyc[10] = t1 - t0;
  // 11: __syncwarp overhead
  t0 = clock64(); for (int i = 0; i < n; ++i) { __syncwarp(); a += 1; } t1 = clock64(); cyc[11] = t1 - t0;
  // 12: ballot+ffs chain
  unsigned bb = threadIdx.x;
  t0 = clock64(); for (int i = 0; i < n; ++i) bb = __ffs(__ballot_sync(0xffffffffu, (threadIdx.x ^ bb) & 1)) ; t1 = clock64(); cyc[12] = t1 - t0;
  // 13: DSETP only chain (compare -> select)
  double w = x;
  t0 = clock64(); for (int i = 0; i < n; ++i) w = (w < y) ? w + 0.0 : y; t1 = clock64(); cyc[13] = t1 - t0;
  // 14: DDIV
  double dv = x;
  t0 = clock64(); for (int i = 0; i < n; ++i) dv = __ddiv_rn(dv, 1.0000001); t1 = clock64(); cyc[14] = t1 - t0;
  out[threadIdx.x] = x + v + z + w + dv + (double)(a + b + c + q + m + bb);
  iout[threadIdx.x] = j;
}
int main() {
  double* out; long long* cyc; int* io;
  cudaMalloc(&out, 256); cudaMallocManaged(&cyc, 32 * 8); cudaMalloc(&io, 128);
  const int n = 4096;
  k<<<1, 32>>>(out, cyc, n, 1.5, io);
  k<<<1, 32>>>(out, cyc, n, 1.5, io);
  cudaDeviceSynchronize();
  const char* names[] = {"DADD", "DMUL", "DADD.RD", "LDS int chain", "IMAD int chain", "DSETP+branch+DADD", "SHFL", "REDUX.MIN", "I2F.F64+F2I", "IMAD.64 chain", "LDS f64 + F2I", "syncwarp+iadd", "ballot+ffs", "DSETP+select", "DDIV"};
  for (int i = 0; i < 15; ++i) printf("%-22s %.2f cyc/op\n", names[i], (double)cyc[i] / n);
  return 0;
}
