// C ABI of include/lbmgpu.h over the host runtime: status codes with a
// thread-local message (the reference's exception kinds and texts), the
// create_stepper dispatch, standalone IDX construction, run_bench and
// verify_suite on the GPU.
#include <cstring>

#include "runtime.h"

namespace lbmgpu {

// create_stepper (p/src/stepper.cpp:155-180)
std::unique_ptr<Stepper> create(const lbmgpu_geometry* gg, const lbmgpu_flow* p,
                                       const lbmgpu_options* o) {
  if (!p || !o) throw std::invalid_argument("null argument");
  if (!available(o->scheme, o->addressing, o->extensions != 0))
    throw std::invalid_argument("kernel not implemented; traffic model only");
  if (o->workers < 0) throw std::invalid_argument("workers must be >= 0");
  if (o->chunk_length < 1) throw std::invalid_argument("chunk_length must be >= 1");
  if (o->precision != 8 && o->precision != 4)
    throw std::invalid_argument("precision must be 8 (fp64) or 4 (fp32)");
  if (o->layout != LBMGPU_SOA && o->layout != LBMGPU_AOS)
    throw std::invalid_argument("unknown layout");
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (o->device < 0 || o->device >= ndev) throw std::invalid_argument("no such CUDA device");
  const HostGeo g = copy_geo(gg);
  if (o->z_end != 0 || o->z_begin != 0) return create_slab(g, *p, *o);
  return create_single(g, *p, *o);
}

// ---------------------------------------------------------------------------
// standalone IDX construction (build_sparse on the device)
// ---------------------------------------------------------------------------
struct IdxBuild {
  uint32_t n = 0;
  DevMem adj, node_of, rem;
  uint32_t nmail = 0;
};

void build_idx(const lbmgpu_geometry* gg, int device, bool want_node_of, bool want_rem,
                      IdxBuild& out, cudaStream_t st) {
  const HostGeo g = copy_geo(gg);
  CK(cudaSetDevice(device));
  const uint64_t cells = g.cells();
  DevMem mask, cofn;
  uint64_t n = cells;
  if (g.solids || want_node_of) {
    mask.alloc(cells);
    if (g.solids)
      CK(cudaMemcpyAsync(mask.get(), g.mask.data(), cells, cudaMemcpyHostToDevice, st));
    else
      CK(cudaMemsetAsync(mask.get(), 1, cells, st));
    out.node_of.alloc(cells * 4);
    cofn.alloc(cells * 4);
    DevMem scratch(scan_scratch_elems(cells) * sizeof(uint32_t));
    n = build_node_maps(st, mask.get<uint8_t>(), cells, out.node_of.get<uint32_t>(),
                        cofn.get<uint32_t>(), scratch.get<uint32_t>(), 0);
    ck_launch();
  }
  // guard of build_sparse (p/src/geometry.cpp:177-179)
  if (n >= (uint64_t{1} << 31)) throw std::runtime_error("fluid count exceeds 32-bit index range");
  out.n = (uint32_t)n;
  out.adj.alloc(n * 18 * 4);
  launch_adjacency(st, g.solids ? mask.get<uint8_t>() : nullptr, make_lat(g, nullptr, 0, 0, 0, 0),
                   g.solids ? out.node_of.get<uint32_t>() : nullptr,
                   g.solids ? cofn.get<uint32_t>() : nullptr, out.n, out.adj.get<uint32_t>());
  ck_launch();
  if (want_rem) {
    out.rem.alloc(n * 9 * 4);
    DevMem scratch(scan_scratch_elems(n) * sizeof(uint32_t));
    out.nmail = build_et_rem(st, out.adj.get<uint32_t>(), out.n, out.rem.get<uint32_t>(),
                             scratch.get<uint32_t>(), 0);
  }
  CK(cudaStreamSynchronize(st));
}


// ---------------------------------------------------------------------------
// Harness (p/src/bench.cpp): run_bench and verify_suite on the GPU.
// ---------------------------------------------------------------------------
// make_seeded_geometry (p/src/bench.cpp:259-273): 16x8x8, periodic x/z, wall y
HostGeo seeded_geometry(uint64_t seed) {
  HostGeo g;
  g.nx = 16, g.ny = 8, g.nz = 8;
  g.policy[0] = 0, g.policy[1] = 1, g.policy[2] = 0;
  g.mask.assign(g.cells(), 1);
  std::mt19937_64 rng(seed);
  for (int z = 0; z < g.nz; ++z)
    for (int y = 1; y < g.ny - 1; ++y)
      for (int x = 0; x < g.nx; ++x)
        if (rng() % 100 < 12) g.mask[g.idx(x, y, z)] = 0;
  g.solids = std::find(g.mask.begin(), g.mask.end(), 0) != g.mask.end();
  if (!g.solids) g.mask.clear();
  return g;
}

lbmgpu_geometry c_geo(const HostGeo& g) {
  lbmgpu_geometry c{};
  c.nx = g.nx, c.ny = g.ny, c.nz = g.nz;
  for (int k = 0; k < 3; ++k) c.axis_policy[k] = g.policy[k];
  c.mask = g.mask.empty() ? nullptr : g.mask.data();
  return c;
}

}  // namespace lbmgpu

// ===========================================================================
// C ABI
// ===========================================================================
using namespace lbmgpu;

struct lbmgpu_stepper {
  std::unique_ptr<Stepper> s;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return LBMGPU_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return LBMGPU_INVALID_ARGUMENT;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return LBMGPU_DOMAIN_ERROR;
  } catch (const std::bad_alloc& e) {
    g_err = e.what();
    return LBMGPU_BAD_ALLOC;
  } catch (const CudaError& e) {
    g_err = e.what();
    return LBMGPU_CUDA_ERROR;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return LBMGPU_RUNTIME_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return LBMGPU_RUNTIME_ERROR;
  }
}

void check_ok(int rc) {
  if (rc != LBMGPU_OK) throw std::runtime_error(g_err);
}

Stepper& S(lbmgpu_stepper* h) {
  if (!h || !h->s) throw std::invalid_argument("null stepper");
  return *h->s;
}
}  // namespace

extern "C" {

void lbmgpu_default_options(lbmgpu_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->scheme = LBMGPU_AAP;
  o->addressing = LBMGPU_DIRECT;
  o->layout = LBMGPU_SOA;
  o->precision = 8;
  o->device = 0;
  o->workers = 1;
  o->chunk_length = 150;
  o->streaming_stores = 1;
}

int lbmgpu_create(const lbmgpu_geometry* g, const lbmgpu_flow* p, const lbmgpu_options* o,
                  lbmgpu_stepper** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("null output handle");
    auto h = std::make_unique<lbmgpu_stepper>();
    h->s = create(g, p, o);
    *out = h.release();
  });
}

int lbmgpu_destroy(lbmgpu_stepper* h) {
  return guard([&] {
    if (h) {
      if (h->s) cudaSetDevice(h->s->opt_.device);
      delete h;
    }
  });
}

int lbmgpu_step(lbmgpu_stepper* h, int64_t n) {
  return guard([&] {
    if (n < 0) throw std::invalid_argument("steps must be >= 0");
    S(h).step(n);
  });
}

int lbmgpu_synchronize(lbmgpu_stepper* h) { return guard([&] { S(h).sync(); }); }

int lbmgpu_step_timed(lbmgpu_stepper* h, int64_t n, double* ms) {
  return guard([&] {
    if (n < 0) throw std::invalid_argument("steps must be >= 0");
    Stepper& s = S(h);
    CK(cudaSetDevice(s.opt_.device));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    struct EvGuard {
      cudaEvent_t a, b;
      ~EvGuard() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
      }
    } eg{e0, e1};
    s.sync();
    CK(cudaEventRecord(e0, s.stream_));
    s.step(n);
    CK(cudaEventRecord(e1, s.stream_));
    CK(cudaEventSynchronize(e1));
    float f = 0.f;
    CK(cudaEventElapsedTime(&f, e0, e1));
    *ms = (double)f;
  });
}

int lbmgpu_extract_natural(lbmgpu_stepper* h, double* out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("null output buffer");
    S(h).extract(out, false);
  });
}
int lbmgpu_extract_natural_range(lbmgpu_stepper* h, uint64_t first, uint64_t count, double* out,
                                 int32_t out_on_device) {
  return guard([&] {
    if (!out) throw std::invalid_argument("null output buffer");
    S(h).extract(out, out_on_device != 0, first, count);
  });
}

int lbmgpu_load_natural(lbmgpu_stepper* h, const double* in) {
  return guard([&] {
    if (!in) throw std::invalid_argument("null input buffer");
    S(h).load(in, false);
  });
}
int lbmgpu_extract_natural_device(lbmgpu_stepper* h, double* out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("null output buffer");
    S(h).extract(out, true);
  });
}
int lbmgpu_load_natural_device(lbmgpu_stepper* h, const double* in) {
  return guard([&] {
    if (!in) throw std::invalid_argument("null input buffer");
    S(h).load(in, true);
  });
}

int lbmgpu_init_field(lbmgpu_stepper* h, int32_t kind, uint64_t seed, double u0, double drho,
                      double noise) {
  return guard([&] {
    Stepper& s = S(h);
    int src;
    switch (kind) {
      case 0: src = kSrcRest; break;
      case 1: src = kSrcTaylorGreen; break;
      case 2: src = kSrcRandom; break;
      default: throw std::invalid_argument("unknown init kind");
    }
    InitSpec in = slab_init_spec(s, src);
    in.seed = seed, in.u0 = u0, in.drho = drho, in.noise = noise;
    s.init(in);
  });
}

int lbmgpu_layout_phase(lbmgpu_stepper* h, int32_t* phase) {
  return guard([&] { *phase = S(h).layout_phase(); });
}
int lbmgpu_exchange_opposite_handles(lbmgpu_stepper* h, int32_t* had) {
  return guard([&] { *had = S(h).exchange_opposite_handles() ? 1 : 0; });
}
int lbmgpu_time_step(lbmgpu_stepper* h, int64_t* t) {
  return guard([&] { *t = S(h).t_; });
}
int lbmgpu_node_count(lbmgpu_stepper* h, uint64_t* n) {
  return guard([&] { *n = S(h).snapshot_nodes(); });
}
int lbmgpu_storage_bytes(lbmgpu_stepper* h, uint64_t* pdf, uint64_t* idx) {
  return guard([&] {
    *pdf = S(h).pdf_bytes();
    *idx = S(h).idx_bytes();
  });
}
int lbmgpu_stream(lbmgpu_stepper* h, void** st) {
  return guard([&] { *st = (void*)S(h).stream_; });
}
int lbmgpu_launches_per_step(lbmgpu_stepper* h, int32_t* n) {
  return guard([&] { *n = S(h).launches_per_step(); });
}

int lbmgpu_scheme_halo_plan(int32_t scheme, int32_t nzl, int32_t* ops, int32_t* count) {
  return guard([&] {
    const std::vector<int32_t> rows = scheme_halo_plan(scheme, nzl);
    if (count) *count = (int32_t)(rows.size() / 5);
    if (ops) std::copy(rows.begin(), rows.end(), ops);
  });
}

int lbmgpu_halo_plan(int32_t nzl, int32_t* ops, int32_t* count) {
  return lbmgpu_scheme_halo_plan(LBMGPU_AAP, nzl, ops, count);
}

int lbmgpu_nccl_unique_id(uint8_t* id) {
  return guard([&] { nccl_unique_id(id); });
}

int lbmgpu_slab_connect_nccl(lbmgpu_stepper* h, const uint8_t* id, int32_t nranks,
                             int32_t rank) {
  return guard([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank");
    slab_connect_nccl(S(h), id, nranks, rank);
  });
}

int lbmgpu_slab_comm_info(lbmgpu_stepper* h, int32_t* count, int32_t* rank, int32_t* version) {
  return guard([&] {
    if (!count || !rank || !version) throw std::invalid_argument("null output");
    slab_comm_info(S(h), count, rank, version);
  });
}

int lbmgpu_slab_sync_ghosts(lbmgpu_stepper* h) {
  return guard([&] { slab_sync_ghosts(S(h)); });
}

int lbmgpu_slab_group_step(lbmgpu_stepper** hs, int32_t n, int64_t steps) {
  return guard([&] {
    if (n < 1 || !hs) throw std::invalid_argument("empty slab group");
    std::vector<Stepper*> v;
    for (int k = 0; k < n; ++k) v.push_back(&S(hs[k]));
    slab_group_step(v, steps);
  });
}

int lbmgpu_slab_group_connect_p2p(lbmgpu_stepper** hs, int32_t n) {
  return guard([&] {
    if (n < 1 || !hs) throw std::invalid_argument("empty slab group");
    std::vector<Stepper*> v;
    for (int k = 0; k < n; ++k) v.push_back(&S(hs[k]));
    slab_group_connect_p2p(v);
  });
}

int lbmgpu_slab_p2p_export(lbmgpu_stepper* h, uint8_t* blob) {
  return guard([&] {
    if (!blob) throw std::invalid_argument("null blob");
    slab_p2p_export(S(h), blob);
  });
}

int lbmgpu_slab_p2p_connect(lbmgpu_stepper* h, const uint8_t* lower, const uint8_t* upper,
                            int32_t nranks, int32_t rank) {
  return guard([&] {
    if (!lower || !upper) throw std::invalid_argument("null blob");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank");
    slab_p2p_connect(S(h), lower, upper, nranks, rank, 0u);
  });
}

int lbmgpu_slab_p2p_connect_ex(lbmgpu_stepper* h, const uint8_t* lower, const uint8_t* upper,
                               int32_t nranks, int32_t rank, uint32_t flags) {
  return guard([&] {
    if (!lower || !upper) throw std::invalid_argument("null blob");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank");
    if (flags & ~LBMGPU_P2P_HOST_ORDERED) throw std::invalid_argument("unknown p2p flags");
    slab_p2p_connect(S(h), lower, upper, nranks, rank, flags);
  });
}

int lbmgpu_slab_group_sync_ghosts(lbmgpu_stepper** hs, int32_t n) {
  return guard([&] {
    if (n < 1 || !hs) throw std::invalid_argument("empty slab group");
    std::vector<Stepper*> v;
    for (int k = 0; k < n; ++k) v.push_back(&S(hs[k]));
    slab_group_sync_ghosts(v);
  });
}

int lbmgpu_run_bench(const lbmgpu_geometry* g, const lbmgpu_flow* p, const lbmgpu_options* o,
                     int32_t steps, int32_t warmup, int32_t timed_runs, double hbm_gbs,
                     lbmgpu_bench_result* r) {
  return guard([&] {
    if (steps < 1) throw std::invalid_argument("steps must be at least 1");
    if (!r) throw std::invalid_argument("null result");
    auto st = create(g, p, o);
    st->init(st->base_init(kSrcRest));
    st->step(warmup);
    st->sync();
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    std::vector<double> times;
    for (int k = 0; k < std::max(1, timed_runs); ++k) {
      CK(cudaEventRecord(e0, st->stream_));
      st->step(steps);
      CK(cudaEventRecord(e1, st->stream_));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      times.push_back(ms * 1e-3);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    std::sort(times.begin(), times.end());
    const size_t n = times.size();
    const double sec = n % 2 ? times[n / 2] : 0.5 * (times[n / 2 - 1] + times[n / 2]);
    std::memset(r, 0, sizeof(*r));
    r->scheme = o->scheme, r->addressing = o->addressing, r->layout = o->layout;
    r->precision = o->precision;
    r->fluid_count = st->snapshot_nodes();
    r->steps = steps;
    r->seconds = sec;
    r->mlups = (double)st->snapshot_nodes() * steps / sec / 1.0e6;  // p/src/bench.cpp:184
    static const int fam[10] = {0, 1, 1, 2, 2, 3, 4, 4, 5, 6};
    int32_t cnt[6];
    double bpl = 0, gbpl = 0;
    check_ok(lbmgpu_traffic(fam[o->scheme], o->addressing, o->precision, cnt, &bpl));
    check_ok(lbmgpu_gpu_bytes_per_lup(o->scheme, o->addressing, o->precision, &gbpl));
    r->bytes_per_lup = bpl;
    r->gpu_bytes_per_lup = gbpl;
    r->predicted_mlups = hbm_gbs > 0 ? hbm_gbs * 1e9 / gbpl / 1e6 : 0;
    r->model_fraction = r->predicted_mlups > 0 ? r->mlups / r->predicted_mlups : 0;
    r->achieved_gbs = r->mlups * 1e6 * gbpl / 1e9;
  });
}

// verify_suite (p/src/bench.cpp:275-341) on the GPU: every implemented pair
// (optionally also AoS and fp32) against the GPU two-step reference on the
// seeded geometry, compared after every step; fp64 must be bitwise (1e-13
// relative is the reference's recorded fallback), fp32 within 1e-5.
int lbmgpu_stream_bandwidth(int32_t device, uint64_t bytes, int32_t inplace, int32_t reps,
                            double* gbps) {
  return guard([&] {
    if (!gbps) throw std::invalid_argument("null output");
    CK(cudaSetDevice(device));
    *gbps = stream_bandwidth(bytes, inplace, reps);
  });
}

int lbmgpu_selftest_division(uint64_t n, uint64_t seed, int32_t device, uint64_t* mismatches) {
  return guard([&] {
    CK(cudaSetDevice(device));
    const uint64_t m = selftest_division(n, seed);
    if (mismatches) *mismatches = m;
  });
}

int lbmgpu_verify_suite(uint64_t seed, int32_t steps, int32_t device, int32_t all_variants,
                        lbmgpu_verify_entry* entries, int32_t capacity, int32_t* count,
                        int32_t* all_pass) {
  return guard([&] {
    const HostGeo hg = seeded_geometry(seed);
    const lbmgpu_geometry g = c_geo(hg);
    lbmgpu_flow p{};
    p.lambda_even = 1.0 / 0.9;
    p.lambda_odd = lbmgpu_lambda_odd(p.lambda_even, 3.0 / 16.0);
    p.body_force[0] = 1e-5;
    p.rho0 = 1.0;
    lbmgpu_options o;
    lbmgpu_default_options(&o);
    o.device = device;
    o.scheme = LBMGPU_TS;
    auto ref = create(&g, &p, &o);
    const uint64_t nodes = ref->nodes_;
    const size_t nv = nodes * 19;
    std::vector<double> f0(nv), want(nv), got(nv);
    std::mt19937_64 rng(seed ^ 0x9e3779b97f4a7c15ull);
    for (uint64_t n = 0; n < nodes; ++n)
      for (int i = 0; i < 19; ++i) {
        const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
        f0[n * 19 + i] = w_of(i) * p.rho0 * (0.9 + 0.2 * u);
      }
    ref->load(f0.data(), false);
    struct Probe {
      lbmgpu_verify_entry e;
      std::unique_ptr<Stepper> st;
    };
    std::vector<Probe> probes;
    for (int sc = 0; sc < 10; ++sc)
      for (int ad = 0; ad < 2; ++ad)
        for (int lay = 0; lay < (all_variants ? 2 : 1); ++lay)
          for (int pr : {8, 4}) {
            if (pr == 4 && !all_variants) continue;
            if (!available(sc, ad, false)) continue;
            if (sc == LBMGPU_TS && ad == 0 && lay == 0 && pr == 8) continue;  // the reference
            lbmgpu_options q = o;
            q.scheme = sc, q.addressing = ad, q.layout = lay, q.precision = pr;
            Probe pb{};
            pb.e.scheme = sc, pb.e.addressing = ad, pb.e.layout = lay, pb.e.precision = pr;
            pb.e.bitwise = 1, pb.e.pass = 1;
            pb.st = create(&g, &p, &q);
            pb.st->load(f0.data(), false);
            probes.push_back(std::move(pb));
          }
    for (int k = 0; k < steps; ++k) {
      ref->step(1);
      ref->extract(want.data(), false);
      for (Probe& pb : probes) {
        pb.st->step(1);
        pb.st->extract(got.data(), false);
        if (std::memcmp(want.data(), got.data(), nv * sizeof(double)) == 0) continue;
        pb.e.bitwise = 0;
        for (size_t v = 0; v < nv; ++v) {
          const double d = std::fabs(got[v] - want[v]) / std::max(std::fabs(want[v]), 1e-300);
          pb.e.max_rel_linf = std::max(pb.e.max_rel_linf, d);
        }
      }
    }
    int ap = 1;
    int n = 0;
    for (Probe& pb : probes) {
      const double tol = pb.e.precision == 8 ? 1e-13 : 1e-5;
      pb.e.pass = pb.e.bitwise || pb.e.max_rel_linf <= tol;
      ap &= pb.e.pass;
      if (entries && n < capacity) entries[n] = pb.e;
      ++n;
    }
    if (count) *count = n;
    if (all_pass) *all_pass = ap;
  });
}

int lbmgpu_kernel_available(int32_t s, int32_t a) { return available(s, a, false) ? 1 : 0; }
int lbmgpu_kernel_available_ext(int32_t s, int32_t a) { return available(s, a, true) ? 1 : 0; }

int lbmgpu_build_sparse(const lbmgpu_geometry* g, int32_t device, uint32_t* fluid_count,
                        uint32_t* adjacency, uint32_t* node_of) {
  return guard([&] {
    cudaStream_t st;
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    IdxBuild b;
    build_idx(g, device, node_of != nullptr, false, b, st);
    if (fluid_count) *fluid_count = b.n;
    if (adjacency && b.n) {
      DevMem nm((size_t)b.n * 18 * 4);
      launch_transpose_u32(st, b.adj.get<uint32_t>(), 18, b.n, nm.get<uint32_t>());
      ck_launch();
      CK(cudaMemcpyAsync(adjacency, nm.get(), (size_t)b.n * 18 * 4, cudaMemcpyDeviceToHost, st));
    }
    if (node_of)
      CK(cudaMemcpyAsync(node_of, b.node_of.get(), (size_t)g->nx * g->ny * g->nz * 4,
                         cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int lbmgpu_build_et_rem(const lbmgpu_geometry* g, int32_t device, uint32_t* fluid_count,
                        uint32_t* rem, uint32_t* mailboxes) {
  return guard([&] {
    cudaStream_t st;
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    IdxBuild b;
    build_idx(g, device, false, true, b, st);
    if (fluid_count) *fluid_count = b.n;
    if (mailboxes) *mailboxes = b.nmail;
    if (rem && b.n) {
      DevMem nm((size_t)b.n * 9 * 4);
      launch_transpose_u32(st, b.rem.get<uint32_t>(), 9, b.n, nm.get<uint32_t>());
      ck_launch();
      CK(cudaMemcpyAsync(rem, nm.get(), (size_t)b.n * 9 * 4, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
  });
}

// traffic() restated (p/src/perfmodel.cpp:12-75)
int lbmgpu_traffic(int32_t family, int32_t addressing, int32_t pdf_bytes, int32_t* out,
                   double* bytes_per_lup) {
  return guard([&] {
    const int q = 19;
    int loads = 0, wa = 0, stores = 0, idx = 0, halves = 0;
    switch (family) {
      case 0: loads = 2 * q, wa = 2 * q, stores = 2 * q, idx = 2 * (q - 1); break;
      case 1: loads = q, wa = q, stores = q, idx = q - 1; break;
      case 2: loads = q, wa = 0, stores = q, idx = q - 1; break;
      case 3: loads = q, wa = q - 1, stores = q, idx = q - 1; break;
      case 4: loads = (3 * q - 1) / 2, wa = 0, stores = (3 * q - 1) / 2, idx = (q - 1) / 2; break;
      case 5: loads = q, wa = 0, stores = q, idx = 0, halves = addressing ? q - 1 : 0; break;
      case 6: loads = q, wa = 0, stores = q, idx = (q + 1) / 2; break;
      default: throw std::invalid_argument("unknown scheme");
    }
    if (family != 5 && addressing) halves = 2 * idx;
    if (pdf_bytes != 8 && pdf_bytes != 4) throw std::invalid_argument("pdf_bytes must be 8 or 4");
    if (out) {
      out[0] = loads, out[1] = wa, out[2] = stores, out[3] = halves, out[4] = pdf_bytes,
      out[5] = 4;
    }
    *bytes_per_lup = (double)(loads + wa + stores) * pdf_bytes + (double)halves * 4 / 2.0;
  });
}

// compulsory DRAM bytes per fluid-node update:
// PDF loads + stores + IDX, no write-allocate.
int lbmgpu_gpu_bytes_per_lup(int32_t scheme, int32_t addressing, int32_t pdf_bytes,
                             double* bytes_per_lup) {
  return guard([&] {
    if (scheme < 0 || scheme > 9) throw std::invalid_argument("unknown scheme");
    if (pdf_bytes != 8 && pdf_bytes != 4) throw std::invalid_argument("pdf_bytes must be 8 or 4");
    const int pdfs = scheme == LBMGPU_TS ? 4 * 19 : 2 * 19;
    double idx = 0;
    if (addressing) {
      switch (scheme) {
        case LBMGPU_TS: idx = 18; break;
        case LBMGPU_OS_PUSH:
        case LBMGPU_OS_PULL:
        case LBMGPU_OSNT_PULL_1S:
        case LBMGPU_OSNT_PULL_2S:
        case LBMGPU_CG: idx = 18; break;
        default: idx = 9; break;  // SWAP, AA (odd steps only), ET rem
      }
    }
    *bytes_per_lup = (double)pdfs * pdf_bytes + idx * 4;
  });
}

double lbmgpu_lambda_odd(double lambda_even, double magic) {
  const double tau_e_m = 1.0 / lambda_even - 0.5;
  return 1.0 / (magic / tau_e_m + 0.5);
}

int lbmgpu_host_alloc(uint64_t bytes, void** p) {
  return guard([&] {
    if (!p) throw std::invalid_argument("null output pointer");
    CK(cudaHostAlloc(p, bytes ? bytes : 1, cudaHostAllocPortable));
  });
}
int lbmgpu_host_free(void* p) {
  return guard([&] {
    if (p) CK(cudaFreeHost(p));
  });
}

const char* lbmgpu_last_error(void) { return g_err.c_str(); }

int lbmgpu_device_count(int32_t* count) {
  return guard([&] {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    *count = n;
  });
}

const char* lbmgpu_version(void) { return "lbmgpu 0.1 (sm_100a)"; }

}  // extern "C"
