// Do the FP64 tensor pipe (DMMA) and the FP64 pipe (DFMA) share their throughput on sm_100a?
// Each CTA runs 8 warps; warps whose (warp & 1) == 0 issue DMMA m8n8k4 chains, the others DFMA chains.
// Printed: TF/s of the DMMA-only, DFMA-only and mixed kernels (flops counted per executed instruction).
// If the mixed kernel reaches ~2x the single-pipe rate the pipes are independent and the FP64 roofline of a
// kernel that uses both is their sum; if it stays near one pipe's peak they share the units.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mix tools/micro/dmma_dfma_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__device__ __forceinline__ void dmma_work(double* out, double s) {
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

// ITERS x 16 x DFMAS_PER_DMMA dependent-free FMAs per thread
template <int REP>
__device__ __forceinline__ void dfma_work(double* out, double s) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = s, c = 1e-9;
  for (int it = 0; it < ITERS * REP; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) r += a[i];
  if (r == 12345.0) out[0] = r;
}

// mode 0: all warps DMMA, 1: all warps DFMA, 2: even warps DMMA / odd warps DFMA
template <int MODE, int REP>
__global__ void __launch_bounds__(256) mix(double* out, double s) {
  const int warp = threadIdx.x >> 5;
  const bool mm = MODE == 0 || (MODE == 2 && (warp & 1) == 0);
  if (mm) dmma_work(out, s);
  else dfma_work<REP>(out, s);
}

template <class F>
float time_it(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  double* out;
  cudaMalloc(&out, 64);
  const int tpb = 256;
  const double thr = tpb * 1.0;
  printf("{\"gpu\": \"%s\", \"sms\": %d", p.name, sms);
  for (int ctas_per_sm : {1, 2, 4}) {
    const int blocks = sms * ctas_per_sm;
    // flops: DMMA m8n8k4 = 512 flops per warp instruction (16 per thread); DFMA = 2 flops per thread
    const double fl_mm = 16.0 * 8 * ITERS * blocks * thr;       // per thread: 8 MMAs x ITERS x 16 flops
    const double fl_fm1 = 2.0 * 16 * ITERS * blocks * thr;      // REP = 1
    float t0 = time_it([&] { mix<0, 1><<<blocks, tpb>>>(out, 0.5); }, 5);
    float t1 = time_it([&] { mix<1, 4><<<blocks, tpb>>>(out, 0.999); }, 5);
    // mixed: half the warps each; DFMA warps do REP = 4 so both halves take similar time alone
    float t2 = time_it([&] { mix<2, 4><<<blocks, tpb>>>(out, 0.5); }, 5);
    const double mm_tf = fl_mm / t0 / 1e9, fm_tf = 4 * fl_fm1 / t1 / 1e9;
    const double mix_fl = 0.5 * fl_mm + 0.5 * 4 * fl_fm1;
    printf(", \"ctas%d\": {\"dmma_tf\": %.2f, \"dfma_tf\": %.2f, \"mixed_tf\": %.2f, \"ms\": [%.3f, %.3f, %.3f]}",
           ctas_per_sm, mm_tf, fm_tf, mix_fl / t2 / 1e9, t0, t1, t2);
  }
  printf("}\n");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { fprintf(stderr, "%s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
