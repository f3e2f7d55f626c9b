/*
 * The INTEGRATION.md sequence in plain C, compiled against include/bddc_b200.h
 * and linked with libbddc_b200.so by tests/test_c_integration.py.
 *
 *   integration host        host-only calls (no GPU): create, structure, maps,
 *                           a caller-built constraint set; the device call
 *                           must fail with BDDC_B200_CUDA_ERROR
 *   integration device      the reference's run_items sequence
 *                           (experiment.cpp:116-205): create, analysis,
 *                           arithmetic constraints, enrich, preconditioner,
 *                           then the reference's own PCG loop (pcg.cpp:28-77)
 *                           over the two LinearOperator seams, compared with
 *                           the device-resident bddc_b200_pcg, and recover
 *
 * Prints "key value" lines the test parses; exit code 0 on success.
 */
#include <bddc_b200.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define CHECK(call)                                                                         \
  do {                                                                                      \
    int rc_ = (call);                                                                       \
    if (rc_ != BDDC_B200_OK) {                                                              \
      fprintf(stderr, "%s:%d: %s -> %d (%s)\n", __FILE__, __LINE__, #call, rc_,             \
              bddc_b200_last_error());                                                      \
      return 1;                                                                             \
    }                                                                                       \
  } while (0)

static double dot(const double* a, const double* b, int64_t n) {
  double s = 0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* 2x2x2 substructures of 2^3 elements, elasticity, clamped on x = 0, traction
 * (0,0,-1) on x = max: tests/support.hpp:32-48 */
static void cube_problem(bddc_b200_problem* p, int* faces, int* comps) {
  static int load_face[1] = {1};
  static double traction[3] = {0.0, 0.0, -1.0};
  static double flux[1] = {1.0};
  memset(p, 0, sizeof(*p));
  p->subdomains[0] = p->subdomains[1] = p->subdomains[2] = 2;
  p->elements_per_edge = 2;
  p->physics = 1;
  faces[0] = 0;
  comps[0] = comps[1] = comps[2] = 1;
  p->n_dirichlet = 1;
  p->dirichlet_face = faces;
  p->dirichlet_components = comps;
  p->n_loads = 1;
  p->load_face = load_face;
  p->load_traction = traction;
  p->load_flux = flux;
  p->tolerance = 1e-8;
  p->max_iterations = 500;
}

int main(int argc, char** argv) {
  const int device = argc > 1 && strcmp(argv[1], "device") == 0;
  bddc_b200_problem prob;
  int faces[1], comps[3];
  cube_problem(&prob, faces, comps);
  bddc_b200_t* h = NULL;
  CHECK(bddc_b200_create(&prob, &h));
  bddc_b200_structure st;
  CHECK(bddc_b200_structure_get(h, &st));
  printf("free_dofs %lld\ninterface_dofs %lld\nsubdomains %lld\n", (long long)st.free_dofs,
         (long long)st.interface_dofs, (long long)st.subdomains);
  int64_t n = 0;
  CHECK(bddc_b200_interface_size(h, &n));
  if (n != st.interface_dofs) return 2;

  if (!device) {
    /* caller-built ConstraintSet (tests/test_constraints.cpp:83-100): the
     * arithmetic average of the first face glob, twice -- the second is
     * dependent and must be dropped by the rank filter */
    int64_t ng = 0;
    CHECK(bddc_b200_glob_count(h, &ng));
    int face = -1;
    int64_t nn = 0, nsub = 0;
    for (int g = 0; g < ng && face < 0; ++g) {
      int kind = 0;
      CHECK(bddc_b200_glob_info(h, g, &kind, &nn, &nsub));
      if (kind == 2) face = g;
    }
    if (face < 0) return 3;
    CHECK(bddc_b200_constraints_arithmetic(h, 1, 1));
    int64_t n_before = 0, nw = 0;
    CHECK(bddc_b200_constraint_count(h, &n_before));
    /* weights of the first average living on that face */
    int found = -1;
    for (int a = 0; a < n_before && found < 0; ++a) {
      int g = 0;
      CHECK(bddc_b200_constraint_get(h, a, &g, &nw, NULL));
      if (g == face) found = a;
    }
    if (found < 0) return 4;
    double* w = (double*)malloc(sizeof(double) * (size_t)nw);
    int g = 0;
    CHECK(bddc_b200_constraint_get(h, found, &g, &nw, w));
    CHECK(bddc_b200_constraints_clear(h));
    int kept1 = -1, kept2 = -1;
    CHECK(bddc_b200_constraint_add(h, face, w, nw, 0, &kept1));
    CHECK(bddc_b200_constraint_add(h, face, w, nw, 0, &kept2));
    int64_t rows = 0;
    CHECK(bddc_b200_constraint_rows(h, &rows));
    printf("kept %d %d\nrows %lld\n", kept1, kept2, (long long)rows);
    free(w);
    if (bddc_b200_device_count() == 0) {
      const int rc = bddc_b200_analysis(h);
      printf("analysis_rc %d\n", rc);
      if (rc != BDDC_B200_CUDA_ERROR) return 5; /* no CPU fallback */
    }
    bddc_b200_destroy(h);
    return 0;
  }

  /* --- device sequence --- */
  CHECK(bddc_b200_analysis(h));
  CHECK(bddc_b200_constraints_arithmetic(h, 1, 0));
  double omega = NAN;
  CHECK(bddc_b200_enrich(h, 10.0, 15, 0, -1, 0, &omega));
  CHECK(bddc_b200_setup_preconditioner(h));
  int64_t rows = 0;
  CHECK(bddc_b200_constraint_rows(h, &rows));
  printf("constraint_rows %lld\nomega_tilde %.17g\n", (long long)rows, omega);

  double* b = (double*)malloc(sizeof(double) * (size_t)n * 6);
  double *x = b + n, *r = b + 2 * n, *z = b + 3 * n, *p = b + 4 * n, *q = b + 5 * n;
  CHECK(bddc_b200_rhs(h, b));
  /* the reference's pcg over the two seams (pcg.cpp:28-77), zero guess */
  const double tol = 1e-8;
  const int max_it = 500;
  memset(x, 0, sizeof(double) * (size_t)n);
  memcpy(r, b, sizeof(double) * (size_t)n);
  const double ref = sqrt(dot(b, b, n));
  CHECK(bddc_b200_precond_apply(h, r, z));
  memcpy(p, z, sizeof(double) * (size_t)n);
  double rz = dot(r, z, n);
  int it = 0;
  double relres = 1.0;
  while (it < max_it) {
    CHECK(bddc_b200_schur_apply(h, p, q));
    const double alpha = rz / dot(p, q, n);
    for (int64_t i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * q[i];
    }
    ++it;
    relres = sqrt(dot(r, r, n)) / ref;
    if (relres <= tol) break;
    CHECK(bddc_b200_precond_apply(h, r, z));
    const double rz_next = dot(r, z, n);
    const double beta = rz_next / rz;
    rz = rz_next;
    for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
  printf("host_pcg_iterations %d\nhost_pcg_relres %.3e\n", it, relres);

  bddc_b200_pcg_result res;
  double* xd = (double*)malloc(sizeof(double) * (size_t)n);
  double* ab = (double*)malloc(sizeof(double) * 2 * max_it);
  CHECK(bddc_b200_pcg(h, NULL, xd, tol, max_it, 0, &res, ab, ab + max_it));
  double kappa = 0;
  CHECK(bddc_b200_lanczos(ab, ab + max_it, res.iterations, &kappa));
  double diff = 0, nrm = 0;
  for (int64_t i = 0; i < n; ++i) {
    diff += (x[i] - xd[i]) * (x[i] - xd[i]);
    nrm += xd[i] * xd[i];
  }
  printf("device_pcg_iterations %lld\ndevice_pcg_kappa %.12g\nlanczos_kappa %.12g\nconverged %d\n",
         (long long)res.iterations, res.condition_estimate, kappa, res.converged);
  printf("host_vs_device_solution %.3e\n", sqrt(diff / nrm));

  double* u = (double*)malloc(sizeof(double) * (size_t)st.free_dofs);
  CHECK(bddc_b200_recover(h, xd, u));
  double un = 0;
  for (int64_t i = 0; i < st.free_dofs; ++i) un += u[i] * u[i];
  printf("solution_norm %.12g\n", sqrt(un));

  /* the whole work item in one call (experiment.cpp:143-205) */
  bddc_b200_row row;
  CHECK(bddc_b200_run_item(h, "adaptive", 10.0, 15, 0, 0, &row));
  printf("row_constraint_rows %lld\nrow_iterations %lld\nrow_kappa %.12g\n", (long long)row.constraint_rows,
         (long long)row.iterations, row.kappa);
  /* capped iterations: partial result + MAX_ITERATIONS (pcg.hpp:40-45) */
  const int rc = bddc_b200_pcg(h, NULL, xd, 1e-14, 2, 0, &res, NULL, NULL);
  printf("capped_rc %d\ncapped_iterations %lld\n", rc, (long long)res.iterations);
  free(u);
  free(ab);
  free(xd);
  free(b);
  bddc_b200_destroy(h);
  return rc == BDDC_B200_MAX_ITERATIONS ? 0 : 6;
}
