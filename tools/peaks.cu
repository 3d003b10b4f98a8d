// K9: FP64 peak microbenchmarks for the B200 roofline denominators.
// DFMA loop, DMMA (mma.sync f64) loops for every f64 shape ptxas accepts on sm_100a, and an HBM copy.
// Prints one JSON object. Standalone executable; not part of libhdg.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void dfma_loop(double* out, double s) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = s, c = 1e-9;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) r += a[i];
  if (r == 12345.0) out[0] = r;
}

__global__ void dmma_m8n8k4(double* out, double s) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = threadIdx.x * 1e-3 + s, b = 1e-3;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += acc[i][0] + acc[i][1];
  if (r == 12345.0) out[0] = r;
}

__global__ void dmma_m16n8k4(double* out, double s) {
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  double a0 = threadIdx.x * 1e-3 + s, a1 = 2e-3, b = 1e-3;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) r += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (r == 12345.0) out[0] = r;
}

__global__ void dmma_m16n8k16(double* out, double s) {
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + s + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1e-3 * i;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) r += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (r == 12345.0) out[0] = r;
}

__global__ void copy_kernel(const double2* __restrict__ in, double2* __restrict__ out, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) out[i] = in[i];
}

template <class F>
static float time_it(F f, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main(int argc, char** argv) {
  const bool fp64_only = argc > 1;
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 64));
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\"", p.name, sms, p.major, p.minor);
  // DFMA: per thread 16*ITERS fma = 2 flops each
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * (2048 / tpb);
    float ms = time_it([&] { dfma_loop<<<blocks, tpb>>>(out, 0.999); }, 5);
    double fl = 2.0 * 16 * ITERS * (double)blocks * tpb;
    printf(", \"dfma_tflops_tpb%d\": %.3f", tpb, fl / ms / 1e9);
  }
  CK(cudaGetLastError());
  for (int tpb : {128, 256, 512}) {
    int blocks = sms * (2048 / tpb);
    float ms = time_it([&] { dmma_m8n8k4<<<blocks, tpb>>>(out, 0.5); }, 5);
    double fl = 2.0 * 8 * 8 * 4 * 8 * ITERS * (double)blocks * (tpb / 32);
    printf(", \"dmma_m8n8k4_tflops_tpb%d\": %.3f", tpb, fl / ms / 1e9);
    ms = time_it([&] { dmma_m16n8k4<<<blocks, tpb>>>(out, 0.5); }, 5);
    fl = 2.0 * 16 * 8 * 4 * 4 * ITERS * (double)blocks * (tpb / 32);
    printf(", \"dmma_m16n8k4_tflops_tpb%d\": %.3f", tpb, fl / ms / 1e9);
    ms = time_it([&] { dmma_m16n8k16<<<blocks, tpb>>>(out, 0.5); }, 5);
    fl = 2.0 * 16 * 8 * 16 * 4 * (ITERS / 4) * (double)blocks * (tpb / 32);
    printf(", \"dmma_m16n8k16_tflops_tpb%d\": %.3f", tpb, fl / ms / 1e9);
  }
  CK(cudaGetLastError());
  if (fp64_only) { printf("}\n"); return 0; }
  size_t n = (size_t)1 << 30;  // 1 Gi doubles in, 8 GiB
  double2 *a, *b; CK(cudaMalloc(&a, n * 8)); CK(cudaMalloc(&b, n * 8));
  cudaMemset(a, 0, n * 8);
  float ms = time_it([&] { copy_kernel<<<sms * 8, 512>>>(a, b, n / 2); }, 10);
  printf(", \"copy_gbs\": %.1f", 2.0 * n * 8 / ms / 1e6);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf(", \"clock_khz_attr\": %d}\n", clk);
  CK(cudaGetLastError());
  return 0;
}
