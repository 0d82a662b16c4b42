/* headroom_count.c — brute-force image counts per integer delay for tests/test_poly_headroom.py (CPU test
 * infrastructure; shares nothing with the library or the oracle).
 *
 * For a shoebox room (Eq. 1: along each axis the images sit at n L + s for even n and (n + 1) L - s
 * for odd n), every lattice image within distance T c of the receiver is visited and counted on its integer
 * delay j = floor(d fs / c).  Output: one line per delay with a nonzero count, "j count".
 *
 *   headroom_count Lx Ly Lz sx sy sz rx ry rz fs T [c]
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

static double coord(long n, double L, double s) { return (n % 2 == 0) ? n * L + s : (n + 1) * L - s; }

int main(int argc, char** argv) {
  if (argc < 12) {
    fprintf(stderr, "usage: %s Lx Ly Lz sx sy sz rx ry rz fs T [c]\n", argv[0]);
    return 2;
  }
  double L[3], s[3], r[3];
  for (int a = 0; a < 3; a++) {
    L[a] = atof(argv[1 + a]);
    s[a] = atof(argv[4 + a]);
    r[a] = atof(argv[7 + a]);
  }
  const double fs = atof(argv[10]), T = atof(argv[11]), c = argc > 12 ? atof(argv[12]) : 343.0;
  const double dmax = T * c, d2max = dmax * dmax, k = fs / c;
  const long nbin = (long)(dmax * k) + 2;
  long long* cnt = calloc((size_t)nbin, sizeof(long long));
  if (!cnt) return 1;
  long kx = (long)(dmax / L[0]) + 3, ky = (long)(dmax / L[1]) + 3, kz = (long)(dmax / L[2]) + 3;
#pragma omp parallel
  {
    long long* loc = calloc((size_t)nbin, sizeof(long long));
#pragma omp for schedule(dynamic, 4)
    for (long nx = -kx; nx <= kx; nx++) {
      const double dx = coord(nx, L[0], s[0]) - r[0];
      if (dx * dx >= d2max) continue;
      for (long ny = -ky; ny <= ky; ny++) {
        const double dy = coord(ny, L[1], s[1]) - r[1];
        const double rho2 = dx * dx + dy * dy;
        if (rho2 >= d2max) continue;
        for (long nz = -kz; nz <= kz; nz++) {
          const double dz = coord(nz, L[2], s[2]) - r[2];
          const double d2 = rho2 + dz * dz;
          if (d2 >= d2max) continue;
          loc[(long)floor(sqrt(d2) * k)]++;
        }
      }
    }
#pragma omp critical
    for (long j = 0; j < nbin; j++) cnt[j] += loc[j];
    free(loc);
  }
  for (long j = 0; j < nbin; j++)
    if (cnt[j]) printf("%ld %lld\n", j, cnt[j]);
  free(cnt);
  return 0;
}
