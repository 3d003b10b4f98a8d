/* gen/gen_host.c — host side of the seeded synthetic-input generator (shared test infrastructure).
 *
 * Holds none of the method's arithmetic. It produces:
 *   - the periodic annulus triangulation of SURVEY.md Appendix A (the connectivity stand-in for the paper's
 *     unstructured triangulations T_h / Gamma_h, §3.1),
 *   - the per-element degree map (uniform p, or BASELINE.json configs[4]'s i.i.d. draw) and the hp sizes
 *     n_e = m_e n(p), n(p) = (p+1)(p+2)/2, face degree p_f = max(p_K-, p_K+),
 *   - the element blocks A, B, C, D, r_e, r_f and the trace vector lambda, with the value distributions of
 *     BASELINE.json configs (gen/philox_normal.h).
 * Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (see gen/build.py). Compiled with the same
 * formulas as gen/gen_device.cu so both produce bit-identical doubles.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "philox_normal.h"

/* Annulus of Nr radial x Nt angular quads, periodic in theta, each quad split into 2 triangles.
 * vertex v(i,j) = i*Nt + (j mod Nt); element e = 2(j*Nr + i) + t;
 * T0 = (v(i,j), v(i+1,j), v(i+1,j+1)), T1 = (v(i,j), v(i+1,j+1), v(i,j+1)); slot k = edge {a_k, a_(k+1)%3}.
 * Faces are numbered in order of first encounter scanning e = 0..E-1, k = 0..2;
 * face_elem[f] = (first element, second element or -1). Returns the face count F. */
int64_t gen_annulus(int32_t Nr, int32_t Nt, int32_t* elem_face, int32_t* face_elem) {
  const int64_t E = 2LL * Nr * Nt;
  const int64_t V = (int64_t)(Nr + 1) * Nt;
  /* edge lookup: for each vertex, list of (other vertex, face id) with other > vertex; degree <= 6 */
  int32_t* nb_v = (int32_t*)malloc(sizeof(int32_t) * V * 8);
  int32_t* nb_f = (int32_t*)malloc(sizeof(int32_t) * V * 8);
  int32_t* nb_n = (int32_t*)calloc((size_t)V, sizeof(int32_t));
  int64_t F = 0;
  for (int64_t e = 0; e < E; ++e) {
    const int64_t q = e / 2, t = e % 2;
    const int32_t j = (int32_t)(q / Nr), i = (int32_t)(q % Nr);
    const int32_t jp = (j + 1) % Nt;
    int32_t a[3];
    if (t == 0) { a[0] = i * Nt + j; a[1] = (i + 1) * Nt + j; a[2] = (i + 1) * Nt + jp; }
    else        { a[0] = i * Nt + j; a[1] = (i + 1) * Nt + jp; a[2] = i * Nt + jp; }
    for (int k = 0; k < 3; ++k) {
      int32_t u = a[k], w = a[(k + 1) % 3];
      if (u > w) { int32_t s = u; u = w; w = s; }
      int32_t fid = -1;
      for (int s = 0; s < nb_n[u]; ++s)
        if (nb_v[(int64_t)u * 8 + s] == w) { fid = nb_f[(int64_t)u * 8 + s]; break; }
      if (fid < 0) {
        fid = (int32_t)F++;
        nb_v[(int64_t)u * 8 + nb_n[u]] = w;
        nb_f[(int64_t)u * 8 + nb_n[u]] = fid;
        nb_n[u]++;
        face_elem[2 * (int64_t)fid] = (int32_t)e;
        face_elem[2 * (int64_t)fid + 1] = -1;
      } else {
        face_elem[2 * (int64_t)fid + 1] = (int32_t)e;
      }
      elem_face[3 * e + k] = fid;
    }
  }
  free(nb_v); free(nb_f); free(nb_n);
  return F;
}

/* Per-element degree: p_fixed > 0 -> constant; p_fixed == 0 -> BASELINE.json configs[4] draw
 * from {1:0.1, 2:0.3, 3:0.3, 4:0.2, 5:0.1} with u from Philox tag 7. */
void gen_degrees(uint64_t seed, int64_t E, int32_t p_fixed, int32_t* p) {
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < E; ++e) {
    if (p_fixed > 0) { p[e] = p_fixed; continue; }
    const double u = gen_uniform(seed, (uint32_t)e, GEN_TAG_P, 0);
    p[e] = u < 0.1 ? 1 : u < 0.4 ? 2 : u < 0.7 ? 3 : u < 0.9 ? 4 : 5;
  }
}

/* Fill blocks for elements [e0, e0+n) into dense row-major buffers at the given offsets (in doubles,
 * indexed by local element e - e0). Any output pointer may be NULL to skip that block. */
void gen_blocks(uint64_t seed, int64_t e0, int64_t n, const int32_t* ne, const int32_t* nf,
                const int64_t* offA, const int64_t* offB, const int64_t* offC, const int64_t* offD,
                const int64_t* offRe, const int64_t* offRf,
                double* A, double* B, double* C, double* D, double* Re, double* Rf) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t l = 0; l < n; ++l) {
    const uint32_t id = (uint32_t)(e0 + l);
    const int a = ne[l], f = nf[l];
    if (A) { double* o = A + offA[l]; for (int i = 0; i < a; ++i) for (int j = 0; j < a; ++j) o[i * a + j] = gen_block_value(seed, id, GEN_KIND_A, a, f, a, i, j); }
    if (B) { double* o = B + offB[l]; for (int i = 0; i < a; ++i) for (int j = 0; j < f; ++j) o[i * f + j] = gen_block_value(seed, id, GEN_KIND_B, a, f, f, i, j); }
    if (C) { double* o = C + offC[l]; for (int i = 0; i < f; ++i) for (int j = 0; j < a; ++j) o[i * a + j] = gen_block_value(seed, id, GEN_KIND_C, a, f, a, i, j); }
    if (D) { double* o = D + offD[l]; for (int i = 0; i < f; ++i) for (int j = 0; j < f; ++j) o[i * f + j] = gen_block_value(seed, id, GEN_KIND_D, a, f, f, i, j); }
    if (Re) { double* o = Re + offRe[l]; for (int i = 0; i < a; ++i) o[i] = gen_block_value(seed, id, GEN_KIND_RE, a, f, 1, i, 0); }
    if (Rf) { double* o = Rf + offRf[l]; for (int i = 0; i < f; ++i) o[i] = gen_block_value(seed, id, GEN_KIND_RF, a, f, 1, i, 0); }
  }
}

/* Trace vector lambda ~ N(0,1): dof k of face f is draw k of stream (seed, f, tag 8). */
void gen_lambda(uint64_t seed, int64_t F, const int32_t* face_ndof, const int64_t* face_off, double* lam) {
#pragma omp parallel for schedule(static)
  for (int64_t f = 0; f < F; ++f)
    for (int k = 0; k < face_ndof[f]; ++k)
      lam[face_off[f] + k] = gen_normal(seed, (uint32_t)f, GEN_TAG_LAMBDA, (uint64_t)k);
}

/* Raw access for pins (Philox known-answer tests, normal draws). */
void gen_philox_raw(const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
  gen_u32x4 c; for (int i = 0; i < 4; ++i) c.x[i] = ctr[i];
  gen_u32x4 r = gen_philox4x32_10(c, key[0], key[1]);
  for (int i = 0; i < 4; ++i) out[i] = r.x[i];
}

void gen_normals(uint64_t seed, uint32_t id, uint32_t tag, int64_t n, double* out) {
  for (int64_t t = 0; t < n; ++t) out[t] = gen_normal(seed, id, tag, (uint64_t)t);
}

double gen_ln_det(double x) { return gen_ln(x); }
void gen_sincos_2pi_det(double u, double* s, double* c) { gen_sincos_2pi(u, s, c); }
