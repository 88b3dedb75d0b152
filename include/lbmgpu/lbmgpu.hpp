// lbmgpu.hpp — C++ mirror of the reference's lattice/propagation API
// (lbmlab, /root/reference/proj/include/lbmlab; p/ below) on top of the C ABI
// of include/lbmgpu.h. Header-only: link liblbmgpu.so.
//
// A user of the reference switches by replacing `lbmlab::` with `lbmgpu::`
// and `#include "lbmlab/stepper.hpp"` with this header. Names, argument
// meaning, defaults, exception types and messages follow:
//   Stencil / make_stencil / direction_pairs   p/include/lbmlab/stencil.hpp:14-32
//   FlowParams / lambda_odd                    p/include/lbmlab/collision.hpp:10-18
//   AxisPolicy / GridGeometry / gen_channel    p/include/lbmlab/geometry.hpp:13-44
//   SparseRepresentation / build_sparse        p/include/lbmlab/geometry.hpp:72-84
//   SchemeId / Addressing / LayoutPhase /
//   StepperOptions / Stepper / create_stepper /
//   kernel_available / parse_* / to_string     p/include/lbmlab/stepper.hpp:15-113
//   TrafficSpec / traffic / predict_mlups      p/include/lbmlab/perfmodel.hpp:17-60
//   Moments / moments                          p/include/lbmlab/collision.hpp:25-33
//   MacroFields / macroscopic_fields           p/include/lbmlab/stepper.hpp:115-120
// GPU additions: StepperOptions::{layout, precision, device, extensions,
// z_begin, z_end}; Stepper::{step_n, synchronize, step_timed, init_field,
// slab_connect_nccl, slab_sync_ghosts, slab_p2p_export, slab_p2p_connect};
// nccl_unique_id, slab_group_step, slab_group_sync_ghosts, slab_group_connect_p2p.
// Differences: Stepper::step() is synchronous (as the reference's); the
// `workers` option is validated but unused (no CPU threads); CG and SWAP run in
// parallel on the GPU, so "scheme is sequential; workers must be 1" never fires.
#pragma once

#include <algorithm>
#include <array>
#include <cctype>
#include <cstdint>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "../lbmgpu.h"

namespace lbmgpu {

namespace detail {
inline void check(int rc) {
  if (rc == LBMGPU_OK) return;
  const std::string msg = lbmgpu_last_error();
  switch (rc) {
    case LBMGPU_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case LBMGPU_DOMAIN_ERROR: throw std::domain_error(msg);
    case LBMGPU_BAD_ALLOC: throw std::bad_alloc();
    default: throw std::runtime_error(msg);
  }
}
inline std::string normalize(std::string_view s) {
  std::string out(s);
  std::transform(out.begin(), out.end(), out.begin(), [](unsigned char c) {
    return c == '_' ? '-' : static_cast<char>(std::tolower(c));
  });
  return out;
}
}  // namespace detail

// ---- stencil (D3Q19 only: the GPU path has no D2Q9 kernels) ----------------
struct Stencil {
  std::string_view name;
  int d = 0, q = 0;
  std::vector<std::array<int, 3>> c;
  std::vector<double> w;
  std::vector<int> opposite;
  int pairs() const { return (q - 1) / 2; }
};

inline Stencil make_stencil(std::string_view name) {
  if (detail::normalize(name) != "d3q19")
    throw std::invalid_argument("unsupported stencil: " + std::string(name));
  Stencil s;
  s.name = "d3q19";
  s.d = 3;
  s.q = 19;
  s.c = {{0, 0, 0},   {1, 0, 0},   {-1, 0, 0}, {0, 1, 0},  {0, -1, 0},  {0, 0, 1},  {0, 0, -1},
         {-1, -1, 0}, {-1, 0, -1}, {-1, 0, 1}, {-1, 1, 0}, {0, -1, -1}, {0, -1, 1}, {0, 1, -1},
         {0, 1, 1},   {1, -1, 0},  {1, 0, -1}, {1, 0, 1},  {1, 1, 0}};
  s.w.assign(19, 1.0 / 36.0);
  s.w[0] = 1.0 / 3.0;
  for (int i = 1; i <= 6; ++i) s.w[i] = 1.0 / 18.0;
  s.opposite = {0, 2, 1, 4, 3, 6, 5, 18, 17, 16, 15, 14, 13, 12, 11, 10, 9, 8, 7};
  return s;
}

inline std::vector<std::pair<int, int>> direction_pairs(const Stencil& s) {
  std::vector<std::pair<int, int>> out;
  for (int i = 1; i < s.q; ++i)
    if (i < s.opposite[i]) out.emplace_back(i, s.opposite[i]);
  return out;
}

// ---- flow parameters ---------------------------------------------------------
struct FlowParams {
  double lambda_even = 1.0 / 0.9;
  double magic_lambda = 3.0 / 16.0;
  std::array<double, 3> body_force{1e-5, 0.0, 0.0};
  double rho0 = 1.0;
};

inline double lambda_odd(const FlowParams& p) {
  return lbmgpu_lambda_odd(p.lambda_even, p.magic_lambda);
}

// ---- geometry ------------------------------------------------------------------
enum class AxisPolicy : std::uint8_t { periodic = 0, wall = 1 };

struct GridGeometry {
  int nx = 0, ny = 0, nz = 0;
  std::array<AxisPolicy, 3> axis_policy{AxisPolicy::periodic, AxisPolicy::periodic,
                                        AxisPolicy::periodic};
  std::vector<std::uint8_t> mask;

  std::size_t cells() const {
    return static_cast<std::size_t>(nx) * static_cast<std::size_t>(ny) *
           static_cast<std::size_t>(nz);
  }
  std::size_t index(int x, int y, int z) const {
    return static_cast<std::size_t>(x) +
           static_cast<std::size_t>(nx) *
               (static_cast<std::size_t>(y) + static_cast<std::size_t>(ny) * z);
  }
  bool is_fluid(int x, int y, int z) const { return mask[index(x, y, z)] != 0; }
  std::size_t fluid_count() const {
    std::size_t n = 0;
    for (auto m : mask) n += (m != 0);
    return n;
  }
  bool operator==(const GridGeometry&) const = default;

  lbmgpu_geometry c_view() const {
    lbmgpu_geometry g{};
    g.nx = nx, g.ny = ny, g.nz = nz;
    for (int k = 0; k < 3; ++k) g.axis_policy[k] = static_cast<std::uint8_t>(axis_policy[k]);
    g.mask = mask.empty() ? nullptr : mask.data();
    return g;
  }
};

inline GridGeometry gen_channel(int nx, int ny, int nz) {
  if (nx < 1 || ny < 1 || nz < 1) throw std::invalid_argument("zero dimension");
  GridGeometry g;
  g.nx = nx, g.ny = ny, g.nz = nz;
  g.axis_policy = {AxisPolicy::periodic, AxisPolicy::wall, AxisPolicy::wall};
  g.mask.assign(g.cells(), 1);
  return g;
}

struct SparseRepresentation {
  std::uint32_t fluid_count = 0;
  int q = 0;
  std::vector<std::array<std::int32_t, 3>> coords;
  std::vector<std::uint32_t> adjacency;
  std::vector<std::uint32_t> node_of;
  std::uint32_t neighbor(std::uint32_t node, int dir) const {
    return adjacency[static_cast<std::size_t>(node) * (q - 1) + (dir - 1)];
  }
};

// build_sparse on the GPU (device 0 unless given)
inline SparseRepresentation build_sparse(const GridGeometry& g, const Stencil& s,
                                         int device = 0) {
  if (s.q != 19) throw std::invalid_argument("stencil/geometry dimension mismatch");
  const lbmgpu_geometry cg = g.c_view();
  SparseRepresentation sp;
  sp.q = s.q;
  detail::check(lbmgpu_build_sparse(&cg, device, &sp.fluid_count, nullptr, nullptr));
  sp.adjacency.resize(static_cast<std::size_t>(sp.fluid_count) * 18);
  sp.node_of.resize(g.cells());
  detail::check(lbmgpu_build_sparse(&cg, device, &sp.fluid_count, sp.adjacency.data(),
                                    sp.node_of.data()));
  sp.coords.resize(sp.fluid_count);
  for (int z = 0; z < g.nz; ++z)
    for (int y = 0; y < g.ny; ++y)
      for (int x = 0; x < g.nx; ++x) {
        const std::uint32_t n = sp.node_of[g.index(x, y, z)];
        if (n != ~std::uint32_t{0}) sp.coords[n] = {x, y, z};
      }
  return sp;
}

// ---- schemes -------------------------------------------------------------------
enum class SchemeId { ts, os_push, os_pull, osnt_pull_1s, osnt_pull_2s, cg, swap_push, swap_pull, aap, et };
enum class SchemeFamily { ts, os, osnt, cg, swap, aap, et };
enum class Addressing { direct, indirect };
enum class LayoutPhase { natural, opposed, shifted_even, shifted_odd, twisted, swap_partial };
enum class Layout { soa, aos };

inline const std::vector<SchemeId>& all_schemes() {
  static const std::vector<SchemeId> ids = {
      SchemeId::ts,           SchemeId::os_push,      SchemeId::os_pull, SchemeId::osnt_pull_1s,
      SchemeId::osnt_pull_2s, SchemeId::cg,           SchemeId::swap_push, SchemeId::swap_pull,
      SchemeId::aap,          SchemeId::et};
  return ids;
}

inline SchemeFamily family_of(SchemeId id) {
  switch (id) {
    case SchemeId::ts: return SchemeFamily::ts;
    case SchemeId::os_push:
    case SchemeId::os_pull: return SchemeFamily::os;
    case SchemeId::osnt_pull_1s:
    case SchemeId::osnt_pull_2s: return SchemeFamily::osnt;
    case SchemeId::cg: return SchemeFamily::cg;
    case SchemeId::swap_push:
    case SchemeId::swap_pull: return SchemeFamily::swap;
    case SchemeId::aap: return SchemeFamily::aap;
    case SchemeId::et: return SchemeFamily::et;
  }
  throw std::invalid_argument("unknown scheme");
}

inline std::string_view to_string(SchemeId id) {
  static constexpr std::string_view n[] = {"ts", "os-push", "os-pull", "osnt-pull-1s",
                                           "osnt-pull-2s", "cg", "swap-push", "swap-pull",
                                           "aap", "et"};
  const int k = static_cast<int>(id);
  if (k < 0 || k > 9) throw std::invalid_argument("unknown scheme");
  return n[k];
}
inline std::string_view to_string(Addressing a) {
  return a == Addressing::direct ? "direct" : "indirect";
}
inline std::string_view to_string(LayoutPhase p) {
  static constexpr std::string_view n[] = {"natural", "opposed", "shifted_even",
                                           "shifted_odd", "twisted", "swap_partial"};
  return n[static_cast<int>(p)];
}
inline SchemeId parse_scheme(std::string_view name) {
  const std::string k = detail::normalize(name);
  for (SchemeId id : all_schemes())
    if (k == to_string(id)) return id;
  throw std::invalid_argument("unknown scheme: " + std::string(name));
}
inline Addressing parse_addressing(std::string_view name) {
  const std::string k = detail::normalize(name);
  if (k == "direct" || k == "full") return Addressing::direct;
  if (k == "indirect" || k == "sparse") return Addressing::indirect;
  throw std::invalid_argument("unknown addressing: " + std::string(name));
}

inline bool kernel_available(SchemeId id, Addressing a) {
  return lbmgpu_kernel_available(static_cast<int>(id), static_cast<int>(a)) != 0;
}

struct StepperOptions {
  int workers = 1;
  int chunk_length = 150;
  bool streaming_stores = true;
  bool swap_deferred_fixup = false;
  bool zero_collision = false;
  // GPU selectors
  Layout layout = Layout::soa;
  int precision = 8;  // 8 fp64, 4 fp32
  int device = 0;
  bool extensions = false;  // TS / SWAP indirect (no reference kernel)
  int z_begin = 0, z_end = 0;
};

class Stepper {
 public:
  Stepper(const Stepper&) = delete;
  Stepper& operator=(const Stepper&) = delete;
  ~Stepper() {
    if (h_) lbmgpu_destroy(h_);
  }

  // one time step, synchronous (Stepper::step, p/include/lbmlab/stepper.hpp:74)
  void step() {
    detail::check(lbmgpu_step(h_, 1));
    detail::check(lbmgpu_synchronize(h_));
  }
  void step_n(long long n) { detail::check(lbmgpu_step(h_, n)); }  // asynchronous
  void synchronize() { detail::check(lbmgpu_synchronize(h_)); }
  double step_timed(long long n) {
    double ms = 0;
    detail::check(lbmgpu_step_timed(h_, n, &ms));
    return ms;
  }
  void extract_natural(double* out) const {
    detail::check(lbmgpu_extract_natural(h_, out));
  }
  void load_natural(const double* in) { detail::check(lbmgpu_load_natural(h_, in)); }
  std::vector<double> extract_natural() const {
    std::vector<double> out(values());
    extract_natural(out.data());
    return out;
  }
  LayoutPhase layout_phase() const {
    std::int32_t p = 0;
    detail::check(lbmgpu_layout_phase(h_, &p));
    return static_cast<LayoutPhase>(p);
  }
  bool exchange_opposite_handles() {
    std::int32_t had = 0;
    detail::check(lbmgpu_exchange_opposite_handles(h_, &had));
    return had != 0;
  }
  void init_field(int kind, std::uint64_t seed, double u0 = 0.01, double drho = 1e-3,
                  double noise = 1e-4) {
    detail::check(lbmgpu_init_field(h_, kind, seed, u0, drho, noise));
  }

  SchemeId scheme() const { return scheme_; }
  Addressing addressing() const { return addressing_; }
  long long time_step() const {
    std::int64_t t = 0;
    detail::check(lbmgpu_time_step(h_, &t));
    return t;
  }
  std::size_t node_count() const { return nodes_; }
  int q() const { return 19; }
  std::size_t values() const { return nodes_ * 19; }
  lbmgpu_stepper* handle() const { return h_; }

  // ---- z-slab of a multi-GPU decomposition (options.z_begin / z_end) ----
  // one rank per GPU over NCCL: every rank passes rank 0's nccl_unique_id()
  void slab_connect_nccl(const std::array<std::uint8_t, LBMGPU_NCCL_ID_BYTES>& id, int nranks,
                         int rank) {
    detail::check(lbmgpu_slab_connect_nccl(h_, id.data(), nranks, rank));
  }
  // ghosts <- owners before an extraction that gathers from them (collective)
  void slab_sync_ghosts() { detail::check(lbmgpu_slab_sync_ghosts(h_)); }
  // peer-memory AA transport: publish this slab, then connect to the lower
  // and upper neighbours' blobs (collective; nranks 1: this slab's own twice)
  std::array<std::uint8_t, LBMGPU_P2P_BLOB_BYTES> slab_p2p_export() {
    std::array<std::uint8_t, LBMGPU_P2P_BLOB_BYTES> b{};
    detail::check(lbmgpu_slab_p2p_export(h_, b.data()));
    return b;
  }
  void slab_p2p_connect(const std::array<std::uint8_t, LBMGPU_P2P_BLOB_BYTES>& lower,
                        const std::array<std::uint8_t, LBMGPU_P2P_BLOB_BYTES>& upper, int nranks,
                        int rank, bool host_ordered = false) {
    // host_ordered: no flag-word barrier; the caller synchronizes and barriers
    // the ranks after every step (ranks sharing one GPU)
    detail::check(lbmgpu_slab_p2p_connect_ex(h_, lower.data(), upper.data(), nranks, rank,
                                             host_ordered ? LBMGPU_P2P_HOST_ORDERED : 0u));
  }

 private:
  friend std::unique_ptr<Stepper> create_stepper(SchemeId, Addressing, const GridGeometry&,
                                                 const Stencil&, const FlowParams&,
                                                 const StepperOptions&);
  Stepper(lbmgpu_stepper* h, SchemeId s, Addressing a) : h_(h), scheme_(s), addressing_(a) {
    std::uint64_t n = 0;
    detail::check(lbmgpu_node_count(h_, &n));
    nodes_ = n;
  }
  lbmgpu_stepper* h_ = nullptr;
  SchemeId scheme_;
  Addressing addressing_;
  std::size_t nodes_ = 0;
};

// create_stepper (p/src/stepper.cpp:155-180): starts at w_i * rho0
inline std::unique_ptr<Stepper> create_stepper(SchemeId id, Addressing a, const GridGeometry& g,
                                               const Stencil& s, const FlowParams& p,
                                               const StepperOptions& opt = {}) {
  if (s.q != 19) throw std::invalid_argument("unsupported stencil: " + std::string(s.name));
  const lbmgpu_geometry cg = g.c_view();
  lbmgpu_flow f{};
  f.lambda_even = p.lambda_even;
  f.lambda_odd = lambda_odd(p);
  for (int k = 0; k < 3; ++k) f.body_force[k] = p.body_force[k];
  f.rho0 = p.rho0;
  lbmgpu_options o;
  lbmgpu_default_options(&o);
  o.scheme = static_cast<int>(id);
  o.addressing = static_cast<int>(a);
  o.layout = opt.layout == Layout::aos ? LBMGPU_AOS : LBMGPU_SOA;
  o.precision = opt.precision;
  o.device = opt.device;
  o.workers = opt.workers;
  o.chunk_length = opt.chunk_length;
  o.streaming_stores = opt.streaming_stores;
  o.swap_deferred_fixup = opt.swap_deferred_fixup;
  o.zero_collision = opt.zero_collision;
  o.extensions = opt.extensions;
  o.z_begin = opt.z_begin;
  o.z_end = opt.z_end;
  lbmgpu_stepper* h = nullptr;
  detail::check(lbmgpu_create(&cg, &f, &o, &h));
  return std::unique_ptr<Stepper>(new Stepper(h, id, a));
}

// ---- macroscopic diagnostics (host side, over the extracted snapshot) ----------
// moments (p/src/collision.cpp:24-36): rho = sum f_i, u = (sum f_i c_i) / rho
// + g / 2; std::domain_error("vacuum node") when rho <= 0
struct Moments {
  double rho = 0.0;
  std::array<double, 3> u{0.0, 0.0, 0.0};
};
inline Moments moments(const Stencil& s, const double* f, const std::array<double, 3>& g) {
  double rho = 0.0;
  std::array<double, 3> m{0.0, 0.0, 0.0};
  for (int i = 0; i < s.q; ++i) {
    rho += f[i];
    for (int k = 0; k < s.d; ++k) m[k] += f[i] * s.c[i][k];
  }
  if (!(rho > 0.0)) throw std::domain_error("vacuum node");
  Moments out;
  out.rho = rho;
  for (int k = 0; k < 3; ++k) out.u[k] = m[k] / rho + 0.5 * g[k];
  return out;
}
// MacroFields / macroscopic_fields (p/include/lbmlab/stepper.hpp:115-120,
// p/src/stepper.cpp:182-193): per fluid node, canonical node order
struct MacroFields {
  std::vector<double> rho;
  std::vector<std::array<double, 3>> u;
};
inline MacroFields macroscopic_fields(const Stepper& st, const Stencil& s, const FlowParams& p) {
  const std::vector<double> f = st.extract_natural();
  MacroFields out;
  out.rho.resize(st.node_count());
  out.u.resize(st.node_count());
  for (std::size_t n = 0; n < st.node_count(); ++n) {
    const Moments m = moments(s, f.data() + n * s.q, p.body_force);
    out.rho[n] = m.rho;
    out.u[n] = m.u;
  }
  return out;
}

// ---- traffic model (p/src/perfmodel.cpp:12-75, 115-119) ------------------------
struct TrafficSpec {
  SchemeFamily scheme;
  Addressing addressing;
  int pdf_loads = 0, pdf_write_allocates = 0, pdf_stores = 0, idx_loads_halves = 0;
  int pdf_bytes = 8, idx_bytes = 4;
  int pdf_elements() const { return pdf_loads + pdf_write_allocates + pdf_stores; }
  double idx_loads() const { return idx_loads_halves / 2.0; }
  double bytes_per_lup() const {
    return static_cast<double>(pdf_elements()) * pdf_bytes +
           static_cast<double>(idx_loads_halves) * idx_bytes / 2.0;
  }
};

inline TrafficSpec traffic(SchemeFamily f, Addressing a, int pdf_bytes = 8) {
  std::int32_t out[6];
  double b = 0;
  detail::check(lbmgpu_traffic(static_cast<int>(f), static_cast<int>(a), pdf_bytes, out, &b));
  TrafficSpec t{f, a, out[0], out[1], out[2], out[3], out[4], out[5]};
  return t;
}
inline TrafficSpec traffic(SchemeId id, Addressing a, int pdf_bytes = 8) {
  return traffic(family_of(id), a, pdf_bytes);
}
inline double predict_mlups(double bandwidth_gbps, double bytes_per_lup) {
  if (bandwidth_gbps <= 0 || bytes_per_lup <= 0)
    throw std::invalid_argument("bandwidth and bytes/LUP must be positive");
  return bandwidth_gbps * 1.0e9 / bytes_per_lup / 1.0e6;
}

// ---- z-slabs: NCCL id and in-process groups --------------------------------
inline std::array<std::uint8_t, LBMGPU_NCCL_ID_BYTES> nccl_unique_id() {
  std::array<std::uint8_t, LBMGPU_NCCL_ID_BYTES> id{};
  detail::check(lbmgpu_nccl_unique_id(id.data()));
  return id;
}
namespace detail {
inline std::vector<lbmgpu_stepper*> handles(const std::vector<Stepper*>& slabs) {
  std::vector<lbmgpu_stepper*> h;
  for (Stepper* s : slabs) h.push_back(s->handle());
  return h;
}
}  // namespace detail
// several slabs of one process (ring in list order), stepped in lockstep
inline void slab_group_step(const std::vector<Stepper*>& slabs, long long steps) {
  auto h = detail::handles(slabs);
  detail::check(lbmgpu_slab_group_step(h.data(), (std::int32_t)h.size(), steps));
}
inline void slab_group_sync_ghosts(const std::vector<Stepper*>& slabs) {
  auto h = detail::handles(slabs);
  detail::check(lbmgpu_slab_group_sync_ghosts(h.data(), (std::int32_t)h.size()));
}
inline void slab_group_connect_p2p(const std::vector<Stepper*>& slabs) {
  auto h = detail::handles(slabs);
  detail::check(lbmgpu_slab_group_connect_p2p(h.data(), (std::int32_t)h.size()));
}

}  // namespace lbmgpu
