/* oracle/oracle.c — the CPU oracle for the hybridization hot path. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load this.
 * It shares no code with the CUDA path (paper_1308_3995_b200/csrc); neither includes the other.
 *
 * What it computes (§3.4 "Hybridization", Eqs. 44-48): for every element e, with the local
 * matrix A_e = [[A,B],[C,D]]|_e, the local->trace block B_e = [R;S]|_e, the trace->local block C_e = [L M]|_e,
 * the element's trace-trace contribution D_e to N and right-hand sides r_e = [F;G]|_e, r_f (its part of H):
 *     S_e = D_e - C_e A_e^-1 B_e,      g_e = r_f - C_e A_e^-1 r_e          (Eq. hybridsystem)
 * assembled edge-wise into K, E, and the element-wise reconstruction
 *     u_e = A_e^-1 (r_e - B_e lambda_e)                                      (Eq. ls)
 * plus the monolithic solve of the uncondensed system Eq. 44 for pins.
 *
 * The method is an algebraic identity (block elimination), so the oracle is the plain definitions, written as
 * explicit loops in the order SURVEY.md §8(c) O1-O7 fixes: dense LU with partial pivoting per element
 * (SPEC.md:345), first index on ties, a true division for each multiplier, ascending-order sums in a separate
 * accumulator. No BLAS, no blocking, no reordering. Build: gcc -O2 -ffp-contract=off -fopenmp (no FMA).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------------------------------------------
 * O1 factor: P A = L U in place (row-major n x n), LAPACK getrf conventions: piv[k] = row swapped with k.
 * Returns 0, or k+1 if the k-th pivot is exactly zero or NaN (R7: NaN pivots fail too). */
int oracle_lu(int n, double* a, int32_t* piv) {
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = fabs(a[(int64_t)k * n + k]);
    for (int i = k + 1; i < n; ++i) {
      const double v = fabs(a[(int64_t)i * n + k]);
      if (v > best) { best = v; p = i; }            /* strict '>' : first index on ties */
    }
    piv[k] = p;
    if (a[(int64_t)p * n + k] == 0.0 || a[(int64_t)p * n + k] != a[(int64_t)p * n + k]) return k + 1;
    if (p != k)
      for (int j = 0; j < n; ++j) {
        const double t = a[(int64_t)k * n + j];
        a[(int64_t)k * n + j] = a[(int64_t)p * n + j];
        a[(int64_t)p * n + j] = t;
      }
    for (int i = k + 1; i < n; ++i) {
      const double l = a[(int64_t)i * n + k] / a[(int64_t)k * n + k];
      a[(int64_t)i * n + k] = l;
      for (int j = k + 1; j < n; ++j) a[(int64_t)i * n + j] = a[(int64_t)i * n + j] - l * a[(int64_t)k * n + j];
    }
  }
  return 0;
}

/* O2 solve: X = A^-1 X for nrhs right-hand sides stored row-major n x nrhs (column c = one right-hand side).
 * Apply piv in order k = 0..n-1, then unit-lower forward and upper backward substitution. */
void oracle_lu_solve(int n, const double* lu, const int32_t* piv, int nrhs, double* x) {
  for (int c = 0; c < nrhs; ++c) {
    for (int k = 0; k < n; ++k) {
      const int p = piv[k];
      if (p != k) { const double t = x[(int64_t)k * nrhs + c]; x[(int64_t)k * nrhs + c] = x[(int64_t)p * nrhs + c]; x[(int64_t)p * nrhs + c] = t; }
    }
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int j = 0; j < i; ++j) acc = acc + lu[(int64_t)i * n + j] * x[(int64_t)j * nrhs + c];
      x[(int64_t)i * nrhs + c] = x[(int64_t)i * nrhs + c] - acc;
    }
    for (int i = n - 1; i >= 0; --i) {
      double acc = 0.0;
      for (int j = i + 1; j < n; ++j) acc = acc + lu[(int64_t)i * n + j] * x[(int64_t)j * nrhs + c];
      x[(int64_t)i * nrhs + c] = (x[(int64_t)i * nrhs + c] - acc) / lu[(int64_t)i * n + i];
    }
  }
}

/* ---------------------------------------------------------------------------------------------------------
 * O1-O3 for one element. A (ne x ne), B (ne x nf), C (nf x ne), D (nf x nf) row-major; re (ne), rf (nf).
 * Outputs S (nf x nf), g (nf), LU (ne x ne) + piv (ne) for the back-substitution. Returns info. */
int oracle_condense_one(int ne, int nf, const double* A, const double* B, const double* C, const double* D,
                        const double* re, const double* rf, double* S, double* g, double* LU, int32_t* piv) {
  memcpy(LU, A, sizeof(double) * (size_t)ne * ne);
  const int info = oracle_lu(ne, LU, piv);
  if (info) {
    /* S7 / DESIGN.md R7: a singular element has no Schur complement and no reconstruction. Its S, g are NaN, and
     * its saved factors are NaN with the unreached interchanges set to none, so O6 returns NaN for u (instead of
     * reading pivots the factorization never wrote). */
    for (int64_t i = 0; i < (int64_t)nf * nf; ++i) S[i] = NAN;
    for (int i = 0; i < nf; ++i) g[i] = NAN;
    for (int k = info - 1; k < ne; ++k) piv[k] = k;
    for (int64_t i = 0; i < (int64_t)ne * ne; ++i) LU[i] = NAN;
    return info;
  }
  const int w = nf + 1;                                /* X = A^-1 [B | r_e] */
  double* X = (double*)malloc(sizeof(double) * (size_t)ne * w);
  for (int i = 0; i < ne; ++i) {
    for (int j = 0; j < nf; ++j) X[(int64_t)i * w + j] = B[(int64_t)i * nf + j];
    X[(int64_t)i * w + nf] = re[i];
  }
  oracle_lu_solve(ne, LU, piv, w, X);
  for (int i = 0; i < nf; ++i) {                       /* O3: S = D - C X, g = r_f - C y */
    for (int j = 0; j < nf; ++j) {
      double acc = 0.0;
      for (int k = 0; k < ne; ++k) acc = acc + C[(int64_t)i * ne + k] * X[(int64_t)k * w + j];
      S[(int64_t)i * nf + j] = D[(int64_t)i * nf + j] - acc;
    }
    double acc = 0.0;
    for (int k = 0; k < ne; ++k) acc = acc + C[(int64_t)i * ne + k] * X[(int64_t)k * w + nf];
    g[i] = rf[i] - acc;
  }
  free(X);
  return 0;
}

/* Batched O1-O3 over n elements with dense-packed offsets (in doubles; offPiv in int32 units). OpenMP over
 * elements; each element's arithmetic is independent of the batch. Returns the number of failed elements. */
int64_t oracle_condense(int64_t n, const int32_t* ne, const int32_t* nf,
                        const int64_t* offA, const int64_t* offB, const int64_t* offC, const int64_t* offD,
                        const int64_t* offRe, const int64_t* offRf, const int64_t* offS, const int64_t* offG,
                        const int64_t* offLU, const int64_t* offPiv,
                        const double* A, const double* B, const double* C, const double* D,
                        const double* re, const double* rf, double* S, double* g, double* LU, int32_t* piv,
                        int32_t* info) {
  int64_t nbad = 0;
#pragma omp parallel for schedule(dynamic, 8) reduction(+ : nbad)
  for (int64_t e = 0; e < n; ++e) {
    info[e] = oracle_condense_one(ne[e], nf[e], A + offA[e], B + offB[e], C + offC[e], D + offD[e], re + offRe[e],
                                  rf + offRf[e], S + offS[e], g + offG[e], LU + offLU[e], piv + offPiv[e]);
    nbad += info[e] != 0;
  }
  return nbad;
}

/* ---------------------------------------------------------------------------------------------------------
 * O4 symbolic: block-CSR of the skeleton matrix K over face rows [f0, f1) (one diagonal block and
 * the blocks of the other edges of the neighbouring elements per row). Row f's columns = sorted unique union
 * of elem_face of its left and right elements (slots of -1 skipped). row_ptr counts blocks (0-based,
 * row_ptr[0] = 0); blk_off (int64, in doubles) is the running sum of n_fp(row) * n_fp(col).
 * Pass NULL col_idx/blk_off to only count: returns nnzb. */
int64_t oracle_skeleton_symbolic(int64_t f0, int64_t f1, const int32_t* elem_face, const int32_t* face_elem,
                                 const int32_t* face_ndof, int32_t* row_ptr, int32_t* col_idx, int64_t* blk_off) {
  int64_t nnzb = 0, vals = 0;
  if (row_ptr) row_ptr[0] = 0;
  if (blk_off) blk_off[0] = 0;
  for (int64_t f = f0; f < f1; ++f) {
    int32_t cols[6];
    int nc = 0;
    for (int side = 0; side < 2; ++side) {
      const int32_t e = face_elem[2 * f + side];
      if (e < 0) continue;
      for (int k = 0; k < 3; ++k) {
        const int32_t c = elem_face[3 * (int64_t)e + k];
        if (c < 0) continue;
        int dup = 0;
        for (int q = 0; q < nc; ++q) if (cols[q] == c) dup = 1;
        if (!dup) cols[nc++] = c;
      }
    }
    for (int a = 1; a < nc; ++a)                        /* insertion sort, ascending */
      for (int b = a; b > 0 && cols[b - 1] > cols[b]; --b) { const int32_t t = cols[b]; cols[b] = cols[b - 1]; cols[b - 1] = t; }
    for (int q = 0; q < nc; ++q) {
      if (col_idx) col_idx[nnzb] = cols[q];
      vals += (int64_t)face_ndof[f] * face_ndof[cols[q]];
      nnzb++;
      if (blk_off) blk_off[nnzb] = vals;
    }
    if (row_ptr) row_ptr[f - f0 + 1] = (int32_t)nnzb;
  }
  return nnzb;
}

/* O4 numeric: K = 0, E = 0; visit elements in ascending global id; for every slot pair (a, b) add the (a, b)
 * sub-block of S_e into K[f_a, f_b] and the a-part of g_e into E[f_a] ("assembled ... in an
 * element-wise fashion"). Only rows in [f0, f1) are stored. Elements are given as a global id range
 * [e0, e0+n) with blocks at offS/offG (local index e - e0). face_off: trace dof offsets (int64, F+1). */
void oracle_assemble(int64_t f0, int64_t f1, int64_t e0, int64_t n, const int32_t* elem_face,
                     const int32_t* face_ndof, const int64_t* face_off, const int32_t* nf,
                     const int64_t* offS, const int64_t* offG, const double* S, const double* g,
                     const int32_t* row_ptr, const int32_t* col_idx, const int64_t* blk_off, double* K, double* E) {
  const int64_t nvals = blk_off[row_ptr[f1 - f0]];
  for (int64_t i = 0; i < nvals; ++i) K[i] = 0.0;
  for (int64_t i = face_off[f0]; i < face_off[f1]; ++i) E[i - face_off[f0]] = 0.0;
  for (int64_t l = 0; l < n; ++l) {
    const int64_t e = e0 + l;
    const int32_t* ef = elem_face + 3 * e;
    int soff[3], so = 0;
    for (int k = 0; k < 3; ++k) { soff[k] = so; if (ef[k] >= 0) so += face_ndof[ef[k]]; }
    const int n_f = nf[l];
    for (int a = 0; a < 3; ++a) {
      const int32_t fa = ef[a];
      if (fa < 0 || fa < f0 || fa >= f1) continue;
      const int na = face_ndof[fa];
      for (int i = 0; i < na; ++i) E[face_off[fa] - face_off[f0] + i] = E[face_off[fa] - face_off[f0] + i] + g[offG[l] + soff[a] + i];
      for (int b = 0; b < 3; ++b) {
        const int32_t fb = ef[b];
        if (fb < 0) continue;
        const int nb = face_ndof[fb];
        int64_t blk = -1;
        for (int32_t q = row_ptr[fa - f0]; q < row_ptr[fa - f0 + 1]; ++q) if (col_idx[q] == fb) blk = q;
        double* kb = K + blk_off[blk];
        const double* sb = S + offS[l];
        for (int i = 0; i < na; ++i)
          for (int j = 0; j < nb; ++j)
            kb[(int64_t)i * nb + j] = kb[(int64_t)i * nb + j] + sb[(int64_t)(soff[a] + i) * n_f + soff[b] + j];
      }
    }
  }
}

/* ---------------------------------------------------------------------------------------------------------
 * O6 back-substitution: gather lambda_e in slot order, t = r_e - B_e lambda_e (ascending sum), u_e = A_e^-1 t
 * with the saved LU + piv (O2). Elements [e0, e0+n). */
void oracle_backsub(int64_t e0, int64_t n, const int32_t* elem_face, const int32_t* face_ndof, const int64_t* face_off,
                    const int32_t* ne, const int32_t* nf, const int64_t* offLU, const int64_t* offPiv,
                    const int64_t* offB, const int64_t* offRe, const int64_t* offU, const double* LU,
                    const int32_t* piv, const double* B, const double* re, const double* lambda, double* u) {
#pragma omp parallel for schedule(dynamic, 8)
  for (int64_t l = 0; l < n; ++l) {
    const int64_t e = e0 + l;
    const int n_e = ne[l], n_f = nf[l];
    double* lam = (double*)malloc(sizeof(double) * (size_t)(n_f > 0 ? n_f : 1));
    int q = 0;
    for (int k = 0; k < 3; ++k) {
      const int32_t f = elem_face[3 * e + k];
      if (f < 0) continue;
      for (int i = 0; i < face_ndof[f]; ++i) lam[q++] = lambda[face_off[f] + i];
    }
    double* x = u + offU[l];
    for (int i = 0; i < n_e; ++i) {
      double acc = 0.0;
      for (int j = 0; j < n_f; ++j) acc = acc + B[offB[l] + (int64_t)i * n_f + j] * lam[j];
      x[i] = re[offRe[l] + i] - acc;
    }
    oracle_lu_solve(n_e, LU + offLU[l], piv + offPiv[l], 1, x);
    free(lam);
  }
}

/* ---------------------------------------------------------------------------------------------------------
 * O7 monolithic (tiny meshes): the uncondensed system of Eq. 44 as one dense matrix over
 * [element unknowns of e = 0..E-1 ; trace unknowns in face_off order]:
 *   element rows:  A_e (element cols), B_e (its faces' trace cols)          = r_e
 *   trace rows:    C_e (element cols) summed over elements, sum of D_e       = sum of r_f
 * Returns the dense matrix (row-major N x N, N = sum n_e + n_trace) and right-hand side. */
void oracle_monolithic_build(int64_t E, const int32_t* elem_face, const int32_t* face_ndof, const int64_t* face_off,
                             const int32_t* ne, const int32_t* nf, const int64_t* offA, const int64_t* offB,
                             const int64_t* offC, const int64_t* offD, const int64_t* offRe, const int64_t* offRf,
                             const double* A, const double* B, const double* C, const double* D, const double* re,
                             const double* rf, int64_t N, double* M, double* rhs) {
  for (int64_t i = 0; i < N * N; ++i) M[i] = 0.0;
  for (int64_t i = 0; i < N; ++i) rhs[i] = 0.0;
  int64_t nel = 0;
  for (int64_t e = 0; e < E; ++e) nel += ne[e];
  int64_t eo = 0;
  for (int64_t e = 0; e < E; ++e) {
    const int n_e = ne[e], n_f = nf[e];
    int64_t tcol[512];                                  /* global trace index of local trace dof q */
    int q = 0;
    for (int k = 0; k < 3; ++k) {
      const int32_t f = elem_face[3 * e + k];
      if (f < 0) continue;
      for (int i = 0; i < face_ndof[f]; ++i) tcol[q++] = nel + face_off[f] + i;
    }
    for (int i = 0; i < n_e; ++i) {
      for (int j = 0; j < n_e; ++j) M[(eo + i) * N + eo + j] = A[offA[e] + (int64_t)i * n_e + j];
      for (int j = 0; j < n_f; ++j) M[(eo + i) * N + tcol[j]] = B[offB[e] + (int64_t)i * n_f + j];
      rhs[eo + i] = re[offRe[e] + i];
    }
    for (int i = 0; i < n_f; ++i) {
      for (int j = 0; j < n_e; ++j) M[tcol[i] * N + eo + j] = M[tcol[i] * N + eo + j] + C[offC[e] + (int64_t)i * n_e + j];
      for (int j = 0; j < n_f; ++j) M[tcol[i] * N + tcol[j]] = M[tcol[i] * N + tcol[j]] + D[offD[e] + (int64_t)i * n_f + j];
      rhs[tcol[i]] = rhs[tcol[i]] + rf[offRf[e] + i];
    }
    eo += n_e;
  }
}

/* Dense solve with O1/O2 (used for O7 and for O5 on tiny meshes). Returns info. */
int oracle_dense_solve(int n, double* M, double* rhs) {
  int32_t* piv = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  const int info = oracle_lu(n, M, piv);
  if (!info) oracle_lu_solve(n, M, piv, 1, rhs);
  free(piv);
  return info;
}
