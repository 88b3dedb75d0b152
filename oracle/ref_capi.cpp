// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C shim over the UNMODIFIED reference library (lbmlab, /root/reference/proj),
// compiled from the reference sources where they lie by oracle/Makefile into
// oracle/_ref/libref.so. Used by tests/ (golden generation, parity checks) and
// by bench.py's reference arm / cpu_baseline leg. Every entry point forwards to
// the reference's own public API:
//   create_stepper        p/src/stepper.cpp:155-180
//   Stepper::step/...     p/include/lbmlab/stepper.hpp:70-106
//   build_sparse          p/src/geometry.cpp:173-207
//   TrtOperator::collide  p/src/collision.cpp:95-139
//   run_bench             p/src/bench.cpp:155-198
//   verify_suite          p/src/bench.cpp:275-341
//   traffic               p/src/perfmodel.cpp:12-75

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>

#include "lbmlab/bench.hpp"
#include "lbmlab/collision.hpp"
#include "lbmlab/geometry.hpp"
#include "lbmlab/perfmodel.hpp"
#include "lbmlab/stencil.hpp"
#include "lbmlab/stepper.hpp"

using namespace lbmlab;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int kind) {
  g_err = e.what();
  return kind;
}

// status: 0 ok, 1 invalid_argument, 2 runtime_error, 3 domain_error, 4 bad_alloc, 9 other
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  } catch (const std::domain_error& e) {
    return fail(e, 3);
  } catch (const std::bad_alloc& e) {
    return fail(e, 4);
  } catch (const std::runtime_error& e) {
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e, 9);
  }
}

GridGeometry make_geo(int nx, int ny, int nz, const std::uint8_t* policy,
                      const std::uint8_t* mask) {
  GridGeometry g;
  g.nx = nx;
  g.ny = ny;
  g.nz = nz;
  for (int k = 0; k < 3; ++k) g.axis_policy[k] = static_cast<AxisPolicy>(policy[k]);
  if (mask)
    g.mask.assign(mask, mask + g.cells());
  else
    g.mask.assign(g.cells(), 1);
  return g;
}

FlowParams make_flow(double lambda_even, double magic, const double* g, double rho0) {
  FlowParams p;
  p.lambda_even = lambda_even;
  p.magic_lambda = magic;
  p.body_force = {g[0], g[1], g[2]};
  p.rho0 = rho0;
  return p;
}

struct Handle {
  std::unique_ptr<Stepper> st;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

double ref_lambda_odd(double lambda_even, double magic) {
  FlowParams p;
  p.lambda_even = lambda_even;
  p.magic_lambda = magic;
  return lambda_odd(p);
}

int ref_flops_per_update() {
  return TrtOperator(make_stencil("d3q19"), FlowParams{}).flops_per_update();
}

// TrtOperator(s, lambda_even, lambda_odd, g).collide(f) on count nodes of 19
void ref_collide(double lambda_even, double lambda_odd_, const double* g, double* f,
                 long long count) {
  const TrtOperator op(make_stencil("d3q19"), lambda_even, lambda_odd_, {g[0], g[1], g[2]});
  for (long long n = 0; n < count; ++n) op.collide(f + n * 19);
}

double ref_equilibrium(double rho, const double* u, int i) {
  return equilibrium(make_stencil("d3q19"), rho, {u[0], u[1], u[2]}, i);
}

// stencil tables: c[19*3], w[19], opposite[19]
void ref_stencil(int* c, double* w, int* opp) {
  const Stencil s = make_stencil("d3q19");
  for (int i = 0; i < s.q; ++i) {
    for (int k = 0; k < 3; ++k) c[i * 3 + k] = s.c[i][k];
    w[i] = s.w[i];
    opp[i] = s.opposite[i];
  }
}

int ref_create(int scheme, int addressing, int nx, int ny, int nz,
               const std::uint8_t* policy, const std::uint8_t* mask, double lambda_even,
               double magic, const double* g, double rho0, int workers, int chunk_length,
               int streaming_stores, int swap_deferred_fixup, int zero_collision,
               void** out) {
  return guard([&] {
    auto h = std::make_unique<Handle>();
    StepperOptions o;
    o.workers = workers;
    o.chunk_length = chunk_length;
    o.streaming_stores = streaming_stores != 0;
    o.swap_deferred_fixup = swap_deferred_fixup != 0;
    o.zero_collision = zero_collision != 0;
    h->st = create_stepper(static_cast<SchemeId>(scheme), static_cast<Addressing>(addressing),
                           make_geo(nx, ny, nz, policy, mask), make_stencil("d3q19"),
                           make_flow(lambda_even, magic, g, rho0), o);
    *out = h.release();
  });
}

int ref_step(void* h, long long n) {
  return guard([&] {
    for (long long k = 0; k < n; ++k) static_cast<Handle*>(h)->st->step();
  });
}

int ref_extract(void* h, double* out) {
  return guard([&] { static_cast<Handle*>(h)->st->extract_natural(out); });
}

int ref_load(void* h, const double* in) {
  return guard([&] { static_cast<Handle*>(h)->st->load_natural(in); });
}

long long ref_time_step(void* h) { return static_cast<Handle*>(h)->st->time_step(); }
unsigned long long ref_node_count(void* h) { return static_cast<Handle*>(h)->st->node_count(); }
int ref_layout_phase(void* h) {
  return static_cast<int>(static_cast<Handle*>(h)->st->layout_phase());
}
int ref_exchange_opposite_handles(void* h) {
  return static_cast<Handle*>(h)->st->exchange_opposite_handles() ? 1 : 0;
}
void ref_destroy(void* h) { delete static_cast<Handle*>(h); }

// save_geo / load_geo (p/src/geometry.cpp:123-171)
int ref_save_geo(int nx, int ny, int nz, const std::uint8_t* policy, const std::uint8_t* mask,
                 const char* path) {
  return guard([&] { save_geo(make_geo(nx, ny, nz, policy, mask), path); });
}
int ref_load_geo_dims(const char* path, int* dims, std::uint8_t* policy) {
  return guard([&] {
    const GridGeometry g = load_geo(path);
    dims[0] = g.nx, dims[1] = g.ny, dims[2] = g.nz;
    for (int k = 0; k < 3; ++k) policy[k] = static_cast<std::uint8_t>(g.axis_policy[k]);
  });
}

int ref_kernel_available(int scheme, int addressing) {
  return kernel_available(static_cast<SchemeId>(scheme), static_cast<Addressing>(addressing))
             ? 1
             : 0;
}

// adjacency: node-major [N*18] (may be null), node_of: [cells] (may be null)
int ref_build_sparse(int nx, int ny, int nz, const std::uint8_t* policy,
                     const std::uint8_t* mask, unsigned* fluid_count, unsigned* adjacency,
                     unsigned* node_of) {
  return guard([&] {
    const SparseRepresentation sp =
        build_sparse(make_geo(nx, ny, nz, policy, mask), make_stencil("d3q19"));
    *fluid_count = sp.fluid_count;
    if (adjacency)
      std::memcpy(adjacency, sp.adjacency.data(), sp.adjacency.size() * sizeof(unsigned));
    if (node_of) std::memcpy(node_of, sp.node_of.data(), sp.node_of.size() * sizeof(unsigned));
  });
}

// make_seeded_geometry: 16x8x8; mask[1024], policy[3]
void ref_make_seeded_geometry(unsigned long long seed, std::uint8_t* mask,
                              std::uint8_t* policy) {
  const GridGeometry g = make_seeded_geometry(seed);
  std::memcpy(mask, g.mask.data(), g.mask.size());
  for (int k = 0; k < 3; ++k) policy[k] = static_cast<std::uint8_t>(g.axis_policy[k]);
}

// traffic(family, addressing): out[0..5] = loads, write_allocates, stores,
// idx_halves, pdf_bytes, idx_bytes; bytes_per_lup returned via *bytes
int ref_traffic(int family, int addressing, int* out, double* bytes) {
  return guard([&] {
    const TrafficSpec t = traffic(static_cast<SchemeFamily>(family),
                                  static_cast<Addressing>(addressing), make_stencil("d3q19"));
    out[0] = t.pdf_loads;
    out[1] = t.pdf_write_allocates;
    out[2] = t.pdf_stores;
    out[3] = t.idx_loads_halves;
    out[4] = t.pdf_bytes;
    out[5] = t.idx_bytes;
    *bytes = t.bytes_per_lup();
  });
}

// run_bench with fixed bandwidths (no host STREAM measurement); returns the
// median seconds and MLUPs of `timed_runs` runs of `steps` steps each
int ref_run_bench(int scheme, int addressing, int nx, int ny, int nz,
                  const std::uint8_t* policy, const std::uint8_t* mask, double lambda_even,
                  double magic, const double* g, double rho0, int steps, int workers,
                  int warmup, int timed_runs, double* seconds, double* mlups,
                  int* workers_used) {
  return guard([&] {
    BenchOptions bo;
    bo.timed_runs = timed_runs;
    bo.gbps_allocate = 1.0;
    bo.gbps_streaming = 1.0;
    const BenchResult r = run_bench(static_cast<SchemeId>(scheme),
                                    static_cast<Addressing>(addressing),
                                    make_geo(nx, ny, nz, policy, mask), make_stencil("d3q19"),
                                    make_flow(lambda_even, magic, g, rho0), steps, workers,
                                    warmup, bo);
    *seconds = r.seconds;
    *mlups = r.mlups;
    *workers_used = r.workers;
  });
}

// verify_suite(seed, steps): returns number of entries; per entry
// (scheme, addressing, bitwise, pass) and max_rel
int ref_verify_suite(unsigned long long seed, int steps, int* ids, double* max_rel,
                     int* all_pass) {
  int n = 0;
  const int rc = guard([&] {
    const VerifyReport rep = verify_suite(seed, steps);
    for (const VerifyEntry& e : rep.entries) {
      ids[n * 4 + 0] = static_cast<int>(e.scheme);
      ids[n * 4 + 1] = static_cast<int>(e.addressing);
      ids[n * 4 + 2] = e.bitwise ? 1 : 0;
      ids[n * 4 + 3] = e.pass ? 1 : 0;
      max_rel[n] = e.max_rel_linf;
      ++n;
    }
    *all_pass = rep.all_pass ? 1 : 0;
  });
  return rc == 0 ? n : -rc;
}

}  // extern "C"
