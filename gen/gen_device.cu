// gen/gen_device.cu — device side of the seeded synthetic-input generator (shared test infrastructure).
//
// Same generator as gen/gen_host.c (gen/philox_normal.h), compiled with --fmad=false so every double is
// bit-identical to the host build. Used by bench.py and the full-size GPU tests to create the BASELINE.json
// workloads directly in HBM (C3/C4 inputs are ~30 GB; generating them on the host and copying would
// dominate the run). Holds none of the method's arithmetic. Not part of libhdg.
#include <cuda_runtime.h>
#include <stdint.h>

#include "philox_normal.h"

namespace {

__global__ void gen_blocks_kernel(uint64_t seed, int64_t e0, int64_t n, int kind, const int32_t* __restrict__ ne,
                                  const int32_t* __restrict__ nf, const int64_t* __restrict__ off,
                                  int uniform_ne, int uniform_nf, int64_t uniform_stride, double* __restrict__ out) {
  for (int64_t l = blockIdx.x; l < n; l += gridDim.x) {
    const int a = ne ? ne[l] : uniform_ne;
    const int f = nf ? nf[l] : uniform_nf;
    int rows, cols;
    switch (kind) {
      case GEN_KIND_A: rows = a; cols = a; break;
      case GEN_KIND_B: rows = a; cols = f; break;
      case GEN_KIND_C: rows = f; cols = a; break;
      case GEN_KIND_D: rows = f; cols = f; break;
      case GEN_KIND_RE: rows = a; cols = 1; break;
      default: rows = f; cols = 1; break;
    }
    double* o = out + (off ? off[l] : l * uniform_stride);
    const uint32_t id = (uint32_t)(e0 + l);
    const int total = rows * cols;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
      const int i = t / cols, j = t - i * cols;
      o[t] = gen_block_value(seed, id, kind, a, f, cols, i, j);
    }
  }
}

__global__ void gen_lambda_kernel(uint64_t seed, int64_t F, const int32_t* __restrict__ face_ndof,
                                  const int64_t* __restrict__ face_off, double* __restrict__ lam) {
  int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; f < F; f += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < face_ndof[f]; ++k)
      lam[face_off[f] + k] = gen_normal(seed, (uint32_t)f, GEN_TAG_LAMBDA, (uint64_t)k);
}

__global__ void philox_raw_kernel(const uint32_t* ctr, const uint32_t* key, uint32_t* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  gen_u32x4 c;
  for (int k = 0; k < 4; ++k) c.x[k] = ctr[4 * i + k];
  gen_u32x4 r = gen_philox4x32_10(c, key[2 * i], key[2 * i + 1]);
  for (int k = 0; k < 4; ++k) out[4 * i + k] = r.x[k];
}

}  // namespace

extern "C" {

// kind: GEN_KIND_*; ne/nf/off may be NULL for a uniform batch (uniform_* used instead). Returns cudaError_t.
int gen_dev_blocks(uint64_t seed, int64_t e0, int64_t n, int kind, const int32_t* ne, const int32_t* nf,
                   const int64_t* off, int uniform_ne, int uniform_nf, int64_t uniform_stride, double* out,
                   cudaStream_t stream) {
  if (n <= 0) return 0;
  int64_t grid = n < 148 * 64 ? n : 148 * 64;
  gen_blocks_kernel<<<(unsigned)grid, 256, 0, stream>>>(seed, e0, n, kind, ne, nf, off, uniform_ne, uniform_nf,
                                                          uniform_stride, out);
  return (int)cudaGetLastError();
}

int gen_dev_lambda(uint64_t seed, int64_t F, const int32_t* face_ndof, const int64_t* face_off, double* lam,
                   cudaStream_t stream) {
  if (F <= 0) return 0;
  gen_lambda_kernel<<<(unsigned)((F + 255) / 256 < 65535 ? (F + 255) / 256 : 65535), 256, 0, stream>>>(
      seed, F, face_ndof, face_off, lam);
  return (int)cudaGetLastError();
}

int gen_dev_philox_raw(const uint32_t* ctr, const uint32_t* key, uint32_t* out, int n, cudaStream_t stream) {
  philox_raw_kernel<<<(n + 127) / 128, 128, 0, stream>>>(ctr, key, out, n);
  return (int)cudaGetLastError();
}

}  // extern "C"
