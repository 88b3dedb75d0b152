/* TEST INFRASTRUCTURE ONLY — the CPU oracle. Never linked into the product.
 *
 * A plain-C restatement of the reference (lbmlab, arXiv 1111.0922 lab) for the
 * D3Q19 collide+propagate path. Every function cites the reference file:line it
 * follows (p/ = /root/reference/proj/). It is pinned against the reference
 * itself (oracle/_ref/libref.so, built from the reference sources by
 * oracle/Makefile) and against the golden fixtures in tests/golden/.
 */
#ifndef LBM_ORACLE_H
#define LBM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int nx, ny, nz;
  uint8_t policy[3]; /* 0 periodic, 1 wall (p/include/lbmlab/geometry.hpp:13) */
  const uint8_t* mask; /* x-fastest, 1 = fluid; NULL = all fluid */
} orc_geometry;

typedef struct {
  /* TrtOperator state (p/include/lbmlab/collision.hpp:67-79) */
  double lambda_e, le_half, lo_half, w0;
  double w2[9], f3w[9];
} orc_trt;

void orc_stencil(int* c /*19*3*/, double* w /*19*/, int* opp /*19*/);
double orc_lambda_odd(double lambda_even, double magic);
void orc_trt_init(orc_trt* op, double lambda_even, double lambda_odd, const double* g);
void orc_collide(const orc_trt* op, double* f);
double orc_equilibrium(double rho, const double* u, int i);
int orc_flops_per_update(void);

int orc_resolve_link(const orc_geometry* g, int x, int y, int z, int i, int* t);
size_t orc_fluid_count(const orc_geometry* g);
int orc_build_sparse(const orc_geometry* g, uint32_t* adjacency /*N*18*/,
                     uint32_t* node_of /*cells or NULL*/);
uint32_t orc_et_rem(uint32_t nodes, const uint32_t* adjacency, uint32_t* rem /*N*9*/);

/* TS direct (p/src/scheme_ts.cpp): canonical snapshot in, `steps` steps, out. */
int orc_ts_run(const orc_geometry* g, double lambda_even, double lambda_odd,
               const double* force, const double* f_in, long long steps, double* f_out,
               int threads);

int orc_traffic(int family, int addressing, int* out /*6*/, double* bytes_per_lup);

/* mt19937_64 (std::mt19937_64) and the reference's seeded inputs */
typedef struct {
  uint64_t mt[312];
  int mti;
} orc_mt64;
void orc_mt64_seed(orc_mt64* s, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* s);
void orc_make_seeded_geometry(uint64_t seed, uint8_t* mask /*1024*/, uint8_t* policy /*3*/);
void orc_random_field(uint64_t seed, size_t nodes, double scale, double* f);

/* seeded initial fields (kind 0 rest, 1 Taylor-Green, 2 random); see lbm_oracle.c */
void orc_trig_table(int n, double* s, double* c);
int orc_init_field(const orc_geometry* g, int kind, int gnx, int gny, int gnz, int z0,
                   uint64_t seed, double rho0, double u0, double drho, double noise,
                   double* out);

#ifdef __cplusplus
}
#endif
#endif
