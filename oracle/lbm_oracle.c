/* TEST INFRASTRUCTURE ONLY — the CPU oracle (see lbm_oracle.h).
 *
 * Plain-C restatement of the reference D3Q19 path. Compiled with
 * -ffp-contract=off like the reference (p/CMakeLists.txt:17-21) so the
 * collision reproduces TrtOperator::collide bit for bit.
 */
#include "lbm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* D3Q19 canonical order (p/src/stencil.cpp:18-57): rest, +x,-x,+y,-y,+z,-z,
 * then the 12 diagonals sorted lexicographically by (cx,cy,cz). */
static const int C[19][3] = {
    {0, 0, 0},   {1, 0, 0},  {-1, 0, 0}, {0, 1, 0},  {0, -1, 0}, {0, 0, 1},  {0, 0, -1},
    {-1, -1, 0}, {-1, 0, -1}, {-1, 0, 1}, {-1, 1, 0}, {0, -1, -1}, {0, -1, 1}, {0, 1, -1},
    {0, 1, 1},   {1, -1, 0}, {1, 0, -1}, {1, 0, 1},  {1, 1, 0}};
static const int OPP[19] = {0, 2, 1, 4, 3, 6, 5, 18, 17, 16, 15, 14, 13, 12, 11, 10, 9, 8, 7};
/* direction_pairs (p/src/stencil.cpp:70-76): (i, opp i), i < opp i, ascending */
static const int PI[9] = {1, 3, 5, 7, 8, 9, 10, 11, 12};
static const int PJ[9] = {2, 4, 6, 18, 17, 16, 15, 14, 13};

static double weight(int i) {
  /* p/src/stencil.cpp:63-66 */
  if (i == 0) return 1.0 / 3.0;
  if (i <= 6) return 1.0 / 18.0;
  return 1.0 / 36.0;
}

void orc_stencil(int* c, double* w, int* opp) {
  for (int i = 0; i < 19; ++i) {
    for (int k = 0; k < 3; ++k) c[i * 3 + k] = C[i][k];
    w[i] = weight(i);
    opp[i] = OPP[i];
  }
}

/* p/src/collision.cpp:8-11 */
double orc_lambda_odd(double lambda_even, double magic) {
  const double tau_e_m = 1.0 / lambda_even - 0.5;
  return 1.0 / (magic / tau_e_m + 0.5);
}

/* TrtOperator ctor + build (p/src/collision.cpp:50-93) */
void orc_trt_init(orc_trt* op, double lambda_even, double lambda_odd, const double* g) {
  op->lambda_e = lambda_even;
  op->le_half = 0.5 * lambda_even;
  op->lo_half = 0.5 * lambda_odd;
  op->w0 = weight(0);
  for (int p = 0; p < 9; ++p) {
    const int i = PI[p];
    double cg = 0.0;
    for (int k = 0; k < 3; ++k) {
      const int ck = C[i][k];
      if (ck == 0) continue;
      cg += ck * g[k];
    }
    op->w2[p] = 2.0 * weight(i);
    op->f3w[p] = 3.0 * weight(i) * cg;
  }
}

/* TrtOperator::collide (p/src/collision.cpp:95-139), same operand order. */
void orc_collide(const orc_trt* op, double* f) {
  double fsum[9], fdif[9];
  double rho = f[0];
  for (int p = 0; p < 9; ++p) {
    const double fi = f[PI[p]], fj = f[PJ[p]];
    fsum[p] = fi + fj;
    fdif[p] = fi - fj;
    rho += fsum[p];
  }
  double u[3];
  for (int k = 0; k < 3; ++k) {
    /* momentum gather in pair order, sign of c_i (collision.cpp:108-114) */
    double m = 0.0;
    for (int p = 0; p < 9; ++p) {
      const int ck = C[PI[p]][k];
      if (ck > 0) m += fdif[p];
      else if (ck < 0) m += -fdif[p];
    }
    u[k] = m / rho;
  }
  double usq = u[0] * u[0];
  usq += u[1] * u[1];
  usq += u[2] * u[2];
  const double base = 1.0 - 1.5 * usq;
  const double wr0 = op->w0 * rho;
  const double e0 = wr0 * base;
  f[0] -= op->lambda_e * (f[0] - e0);
  for (int p = 0; p < 9; ++p) {
    const int i = PI[p], j = PJ[p];
    double cu = 0.0;
    int first = 1;
    for (int k = 0; k < 3; ++k) {
      const int ck = C[i][k];
      if (ck == 0) continue;
      const double t = ck > 0 ? u[k] : -u[k];
      if (first) {
        cu = t;
        first = 0;
      } else {
        cu += t;
      }
    }
    const double cu3 = 3.0 * cu;
    const double cusq45 = 0.5 * (cu3 * cu3);
    const double wr2 = op->w2[p] * rho;
    const double esum = wr2 * (base + cusq45);
    const double edif = wr2 * cu3;
    const double dp = op->le_half * (fsum[p] - esum);
    const double dm = op->lo_half * (fdif[p] - edif);
    const double dmf = dm - op->f3w[p] * rho;
    f[i] = f[i] - dp - dmf;
    f[j] = f[j] - dp + dmf;
  }
}

/* p/src/collision.cpp:38-45 */
double orc_equilibrium(double rho, const double* u, int i) {
  double cu = 0.0, usq = 0.0;
  for (int k = 0; k < 3; ++k) {
    cu += C[i][k] * u[k];
    usq += u[k] * u[k];
  }
  return weight(i) * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * usq);
}

/* TrtOperator::flops_per_update (p/src/collision.cpp:141-149) */
int orc_flops_per_update(void) {
  int n = 3 * 9;
  for (int k = 0; k < 3; ++k) {
    int nm = 0;
    for (int p = 0; p < 9; ++p) nm += C[PI[p]][k] != 0;
    n += nm + 1;
  }
  n += 3 + 2;
  n += 2;
  n += 5;
  for (int p = 0; p < 9; ++p) {
    int nt = 0;
    for (int k = 0; k < 3; ++k) nt += C[PI[p]][k] != 0;
    n += 17 + (nt - 1);
  }
  return n;
}

static size_t gidx(const orc_geometry* g, int x, int y, int z) {
  return (size_t)x + (size_t)g->nx * ((size_t)y + (size_t)g->ny * (size_t)z);
}

static int is_fluid(const orc_geometry* g, size_t cell) { return !g->mask || g->mask[cell]; }

/* resolve_link (p/src/geometry.cpp:49-60): wall face -> bounce, periodic wrap,
 * solid target -> bounce. Returns 1 on bounce, else 0 with t[3] = target. */
int orc_resolve_link(const orc_geometry* g, int x, int y, int z, int i, int* t) {
  const int n[3] = {g->nx, g->ny, g->nz};
  int p[3] = {x + C[i][0], y + C[i][1], z + C[i][2]};
  for (int k = 0; k < 3; ++k) {
    if (p[k] >= 0 && p[k] < n[k]) continue;
    if (g->policy[k] == 1) return 1;
    p[k] = p[k] < 0 ? p[k] + n[k] : p[k] - n[k];
  }
  if (!is_fluid(g, gidx(g, p[0], p[1], p[2]))) return 1;
  t[0] = p[0];
  t[1] = p[1];
  t[2] = p[2];
  return 0;
}

size_t orc_fluid_count(const orc_geometry* g) {
  const size_t cells = (size_t)g->nx * g->ny * g->nz;
  if (!g->mask) return cells;
  size_t n = 0;
  for (size_t c = 0; c < cells; ++c) n += g->mask[c] != 0;
  return n;
}

/* build_sparse (p/src/geometry.cpp:173-207): x-fastest fluid enumeration and
 * node-major adjacency[n*18 + (i-1)], bounce = n itself.
 * Returns -1 when the fluid count exceeds the 32-bit range. */
int orc_build_sparse(const orc_geometry* g, uint32_t* adjacency, uint32_t* node_of) {
  const size_t cells = (size_t)g->nx * g->ny * g->nz;
  const size_t nfluid = orc_fluid_count(g);
  if (nfluid >= ((size_t)1 << 31)) return -1;
  uint32_t* nof = node_of ? node_of : (uint32_t*)malloc(cells * sizeof(uint32_t));
  uint32_t n = 0;
  for (size_t c = 0; c < cells; ++c) nof[c] = is_fluid(g, c) ? n++ : ~(uint32_t)0;
  size_t cell = 0;
  n = 0;
  for (int z = 0; z < g->nz; ++z)
    for (int y = 0; y < g->ny; ++y)
      for (int x = 0; x < g->nx; ++x, ++cell) {
        if (!is_fluid(g, cell)) continue;
        for (int i = 1; i < 19; ++i) {
          int t[3];
          const int b = orc_resolve_link(g, x, y, z, i, t);
          adjacency[(size_t)n * 18 + (i - 1)] = b ? n : nof[gidx(g, t[0], t[1], t[2])];
        }
        ++n;
      }
  if (!node_of) free(nof);
  return 0;
}

/* ET indirect remote table (p/src/scheme_et.cpp:42-62): rem[n*9+p] = neighbour
 * along c_i, or a mailbox slot N + k (k = running count per pair) when the
 * i-link bounces; bit 31 set when the j-link bounces. Returns max mailbox count. */
uint32_t orc_et_rem(uint32_t nodes, const uint32_t* adjacency, uint32_t* rem) {
  uint32_t mail[9] = {0};
  for (uint32_t n = 0; n < nodes; ++n) {
    const uint32_t* row = adjacency + (size_t)n * 18;
    for (int p = 0; p < 9; ++p) {
      uint32_t r = row[PI[p] - 1];
      if (r == n) r = nodes + mail[p]++;
      const int ub = row[PJ[p] - 1] == n;
      rem[(size_t)n * 9 + p] = r | (ub ? 0x80000000u : 0u);
    }
  }
  uint32_t nm = 0;
  for (int p = 0; p < 9; ++p) nm = mail[p] > nm ? mail[p] : nm;
  return nm;
}

/* Two-step reference (p/src/scheme_ts.cpp:59-112): collide sweep A -> B,
 * then pull-stream B -> A with bounce B[opp i][cell]. Direction-major arrays
 * over all cells; canonical snapshot = fluid nodes x-fastest, node-major. */
int orc_ts_run(const orc_geometry* g, double lambda_even, double lambda_odd,
               const double* force, const double* f_in, long long steps, double* f_out,
               int threads) {
  const size_t cells = (size_t)g->nx * g->ny * g->nz;
  double* A = (double*)malloc(cells * 19 * sizeof(double));
  double* B = (double*)malloc(cells * 19 * sizeof(double));
  int32_t* links = (int32_t*)malloc(cells * 19 * sizeof(int32_t)); /* src of pull, -1 bounce */
  if (!A || !B || !links) {
    free(A);
    free(B);
    free(links);
    return -1;
  }
  orc_trt op;
  orc_trt_init(&op, lambda_even, lambda_odd, force);
  if (threads < 1) threads = 1;

  size_t n = 0;
  for (size_t c = 0; c < cells; ++c) {
    if (!is_fluid(g, c)) continue;
    for (int i = 0; i < 19; ++i) A[(size_t)i * cells + c] = f_in[n * 19 + i];
    ++n;
  }
  const long long nzy = (long long)g->nz * g->ny;
#pragma omp parallel for schedule(static) num_threads(threads)
  for (long long zy = 0; zy < nzy; ++zy) {
    const int z = (int)(zy / g->ny), y = (int)(zy % g->ny);
    for (int x = 0; x < g->nx; ++x) {
      const size_t c = gidx(g, x, y, z);
      for (int i = 1; i < 19; ++i) {
        int t[3];
        links[c * 19 + i] = orc_resolve_link(g, x, y, z, OPP[i], t)
                                ? -1
                                : (int32_t)gidx(g, t[0], t[1], t[2]);
      }
    }
  }
  for (long long s = 0; s < steps; ++s) {
#pragma omp parallel for schedule(static) num_threads(threads)
    for (long long c = 0; c < (long long)cells; ++c) {
      if (!is_fluid(g, (size_t)c)) continue;
      double tmp[19];
      for (int i = 0; i < 19; ++i) tmp[i] = A[(size_t)i * cells + c];
      orc_collide(&op, tmp);
      for (int i = 0; i < 19; ++i) B[(size_t)i * cells + c] = tmp[i];
    }
#pragma omp parallel for schedule(static) num_threads(threads)
    for (long long c = 0; c < (long long)cells; ++c) {
      if (!is_fluid(g, (size_t)c)) continue;
      A[c] = B[c];
      for (int i = 1; i < 19; ++i) {
        const int32_t src = links[c * 19 + i];
        A[(size_t)i * cells + c] =
            src < 0 ? B[(size_t)OPP[i] * cells + c] : B[(size_t)i * cells + src];
      }
    }
  }
  n = 0;
  for (size_t c = 0; c < cells; ++c) {
    if (!is_fluid(g, c)) continue;
    for (int i = 0; i < 19; ++i) f_out[n * 19 + i] = A[(size_t)i * cells + c];
    ++n;
  }
  free(A);
  free(B);
  free(links);
  return 0;
}

/* traffic() element counts (p/src/perfmodel.cpp:12-75); families in
 * SchemeFamily order ts, os, osnt, cg, swap, aap, et. out = loads,
 * write_allocates, stores, idx_halves, pdf_bytes(8), idx_bytes(4). */
int orc_traffic(int family, int addressing, int* out, double* bytes_per_lup) {
  const int q = 19;
  int loads = 0, wa = 0, stores = 0, idx = 0, halves = 0;
  switch (family) {
    case 0: loads = 2 * q; wa = 2 * q; stores = 2 * q; idx = 2 * (q - 1); break;
    case 1: loads = q; wa = q; stores = q; idx = q - 1; break;
    case 2: loads = q; wa = 0; stores = q; idx = q - 1; break;
    case 3: loads = q; wa = q - 1; stores = q; idx = q - 1; break;
    case 4: loads = (3 * q - 1) / 2; wa = 0; stores = (3 * q - 1) / 2; idx = (q - 1) / 2; break;
    case 5: loads = q; wa = 0; stores = q; idx = 0; halves = addressing ? q - 1 : 0; break;
    case 6: loads = q; wa = 0; stores = q; idx = (q + 1) / 2; break;
    default: return -1;
  }
  if (family != 5 && addressing) halves = 2 * idx;
  out[0] = loads;
  out[1] = wa;
  out[2] = stores;
  out[3] = halves;
  out[4] = 8;
  out[5] = 4;
  *bytes_per_lup = (double)(loads + wa + stores) * 8 + (double)halves * 4 / 2.0;
  return 0;
}

/* std::mt19937_64 (Matsumoto & Nishimura 2000; the C++ standard's engine) */
void orc_mt64_seed(orc_mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->mti = 312;
}

uint64_t orc_mt64_next(orc_mt64* s) {
  static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (s->mti >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ mag[(int)(x & 1ULL)];
    }
    for (; i < 311; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ mag[(int)(x & 1ULL)];
    }
    x = (s->mt[311] & UM) | (s->mt[0] & LM);
    s->mt[311] = s->mt[155] ^ (x >> 1) ^ mag[(int)(x & 1ULL)];
    s->mti = 0;
  }
  uint64_t y = s->mt[s->mti++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

/* make_seeded_geometry (p/src/bench.cpp:259-273): 16x8x8, periodic x/z, wall
 * y, ~12% solids away from the y walls. */
void orc_make_seeded_geometry(uint64_t seed, uint8_t* mask, uint8_t* policy) {
  const int nx = 16, ny = 8, nz = 8;
  memset(mask, 1, (size_t)nx * ny * nz);
  policy[0] = 0;
  policy[1] = 1;
  policy[2] = 0;
  orc_mt64 r;
  orc_mt64_seed(&r, seed);
  for (int z = 0; z < nz; ++z)
    for (int y = 1; y < ny - 1; ++y)
      for (int x = 0; x < nx; ++x)
        if (orc_mt64_next(&r) % 100 < 12) mask[x + nx * (y + ny * z)] = 0;
}

/* random_field (p/tests/test_schemes.cpp:29-39) with a rho0 scale
 * (p/src/bench.cpp:283-289 uses w_i * rho0 * (0.9 + 0.2u)). */
void orc_random_field(uint64_t seed, size_t nodes, double scale, double* f) {
  orc_mt64 r;
  orc_mt64_seed(&r, seed);
  for (size_t n = 0; n < nodes; ++n)
    for (int i = 0; i < 19; ++i) {
      const double u = (double)(orc_mt64_next(&r) >> 11) * 0x1.0p-53;
      f[n * 19 + i] = weight(i) * scale * (0.9 + 0.2 * u);
    }
}

/* Seeded initial fields of the BASELINE configs: the
 * definition the product's device init (paper_1111_0922_b200/csrc/
 * kernels_util.cu node_values) implements, restated here so both sides can be
 * checked bit for bit and so the reference can be started from the same
 * snapshot.
 *   U(stream)  = splitmix64(seed + 0x9e3779b97f4a7c15 * (stream + 1)),
 *                (z >> 11) * 2^-52 - 1  in [-1, 1)
 *   stream     = 20 * global_cell + k, global_cell = x + gnx (y + gny (z + z0))
 *   rest       f_i = w_i rho0                           (p/src/scheme_aap.cpp:32-36)
 *   taylor     rho = rho0 + drho U(.., 19), u = u0 (sin X cos Y cos Z,
 *              -cos X sin Y cos Z, 0), X = (2 pi) x / gnx (libm sin / cos),
 *              f_i = equilibrium(rho, u, i) + noise U(.., i)  (p/src/collision.cpp:38-45)
 *   random     f_i = w_i rho0 (0.9 + 0.2 (U(.., i) + 1) / 2)
 * Fluid nodes only, x-fastest (the canonical snapshot order, p/include/lbmlab/
 * stepper.hpp:66-69). */
static uint64_t splitmix_bits(uint64_t seed, uint64_t stream) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
#define ORC_TWO_PI 6.283185307179586476925286766559 /* 2 pi, rounded once */
static double urand_pm1(uint64_t seed, uint64_t stream) {
  return (double)(splitmix_bits(seed, stream) >> 11) * 0x1.0p-52 - 1.0;
}

void orc_trig_table(int n, double* s, double* c) {
  for (int x = 0; x < n; ++x) {
    const double a = ORC_TWO_PI * (double)x / (double)n;
    s[x] = sin(a);
    c[x] = cos(a);
  }
}

int orc_init_field(const orc_geometry* g, int kind, int gnx, int gny, int gnz, int z0,
                   uint64_t seed, double rho0, double u0, double drho, double noise,
                   double* out) {
  double *sx = NULL, *cx = NULL, *sy = NULL, *cy = NULL, *sz = NULL, *cz = NULL;
  if (kind == 1) {
    sx = malloc(sizeof(double) * (size_t)(2 * (gnx + gny + gnz)));
    if (!sx) return -1;
    cx = sx + gnx;
    sy = cx + gnx;
    cy = sy + gny;
    sz = cy + gny;
    cz = sz + gnz;
    orc_trig_table(gnx, sx, cx);
    orc_trig_table(gny, sy, cy);
    orc_trig_table(gnz, sz, cz);
  }
  size_t n = 0;
  for (int z = 0; z < g->nz; ++z)
    for (int y = 0; y < g->ny; ++y)
      for (int x = 0; x < g->nx; ++x) {
        if (!is_fluid(g, gidx(g, x, y, z))) continue;
        const int gz = z + z0;
        const uint64_t gcell = (uint64_t)x + (uint64_t)gnx * ((uint64_t)y + (uint64_t)gny * gz);
        double* f = out + n * 19;
        ++n;
        if (kind == 0) {
          for (int i = 0; i < 19; ++i) f[i] = weight(i) * rho0;
        } else if (kind == 2) {
          for (int i = 0; i < 19; ++i) {
            const double u01 = 0.5 * (urand_pm1(seed, gcell * 20 + i) + 1.0);
            f[i] = weight(i) * rho0 * (0.9 + 0.2 * u01);
          }
        } else {
          const double rho = rho0 + drho * urand_pm1(seed, gcell * 20 + 19);
          const double u[3] = {u0 * sx[x] * cy[y] * cz[gz], -u0 * cx[x] * sy[y] * cz[gz], 0.0};
          for (int i = 0; i < 19; ++i)
            f[i] = orc_equilibrium(rho, u, i) + noise * urand_pm1(seed, gcell * 20 + i);
        }
      }
  free(sx);
  return 0;
}
