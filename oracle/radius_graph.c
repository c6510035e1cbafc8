/*
 * CPU oracle for the exact radius graph -- TEST INFRASTRUCTURE ONLY.
 *
 * Restates complexes.build_graph's edge rule (/root/reference/pkg/src/
 * fusionscreen/complexes.py:237-246) in plain C so the GPU radius graph can be
 * checked edge-for-edge on tens of thousands of poses (the numpy restatement
 * in fusion_oracle.radius_pairs takes ~25 ms per 1,064-atom pose; this takes
 * ~1 ms single-threaded).  Only tests/, smoke() and bench.py's CPU legs load
 * it (via ctypes); the product never does.
 *
 * Rule (float64, no FMA contraction -- build with -ffp-contract=off):
 *   candidate i<j iff d2 <= r*r, d2 = (dx*dx + dy*dy) + dz*dz, r = max(t_cov,
 *   t_ncov)  (scipy cKDTree.query_pairs, scipy 1.18.1: complexes.py:237-238);
 *   d = sqrt(d2)  (== np.linalg.norm bitwise, complexes.py:241);
 *   covalent iff same role and d <= t_cov; non-covalent iff different role
 *   and d <= t_ncov  (complexes.py:242-244).
 * Output: per pose, i<j pairs in lexicographic (i, j) order -- the canonical
 * order parity compares in (the reference emits kd-tree traversal order).
 * Pinned against fusion_oracle.radius_pairs and the reference goldens by
 * tests/test_oracle_golden.py.
 */
#include <math.h>
#include <stdint.h>

/* Brute force over i<j of one pose.  When `cov_ij` is NULL only counts. */
static void pose_pairs(const double* xyz, const int64_t* role, int64_t n, double tc, double tn,
                       int64_t* n_cov, int64_t* n_ncov, int64_t* cov_ij, double* cov_d, int64_t* ncov_ij,
                       double* ncov_d) {
  const double r = tc > tn ? tc : tn;
  const double r2 = r * r;
  int64_t c = 0, m = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double xi = xyz[3 * i], yi = xyz[3 * i + 1], zi = xyz[3 * i + 2];
    const int64_t ri = role[i];
    for (int64_t j = i + 1; j < n; ++j) {
      const double dx = xi - xyz[3 * j], dy = yi - xyz[3 * j + 1], dz = zi - xyz[3 * j + 2];
      const double d2 = (dx * dx + dy * dy) + dz * dz;
      if (!(d2 <= r2)) continue;
      const double d = sqrt(d2);
      if (ri == role[j]) {
        if (d <= tc) {
          if (cov_ij) { cov_ij[2 * c] = i; cov_ij[2 * c + 1] = j; cov_d[c] = d; }
          ++c;
        }
      } else if (d <= tn) {
        if (ncov_ij) { ncov_ij[2 * m] = i; ncov_ij[2 * m + 1] = j; ncov_d[m] = d; }
        ++m;
      }
    }
  }
  *n_cov = c;
  *n_ncov = m;
}

/* Pass 1: edge counts of every pose (atoms atom_off[p] .. atom_off[p+1]). */
void rg_count(const double* xyz, const int64_t* role, const int64_t* atom_off, int64_t n_poses, double tc,
              double tn, int64_t* n_cov, int64_t* n_ncov) {
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t p = 0; p < n_poses; ++p) {
    const int64_t a = atom_off[p];
    pose_pairs(xyz + 3 * a, role + a, atom_off[p + 1] - a, tc, tn, &n_cov[p], &n_ncov[p], 0, 0, 0, 0);
  }
}

/* Pass 2: pose p's edges at rows cov_off[p] .. (exclusive scans of pass 1),
 * pose-local node ids. */
void rg_fill(const double* xyz, const int64_t* role, const int64_t* atom_off, int64_t n_poses, double tc,
             double tn, const int64_t* cov_off, const int64_t* ncov_off, int64_t* cov_ij, double* cov_d,
             int64_t* ncov_ij, double* ncov_d) {
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t p = 0; p < n_poses; ++p) {
    const int64_t a = atom_off[p];
    int64_t c, m;
    pose_pairs(xyz + 3 * a, role + a, atom_off[p + 1] - a, tc, tn, &c, &m, cov_ij + 2 * cov_off[p],
               cov_d + cov_off[p], ncov_ij + 2 * ncov_off[p], ncov_d + ncov_off[p]);
  }
}
