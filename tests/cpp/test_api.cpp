// C++ drop-in check: the reference's own test scenarios written against the
// C++ mirror (include/lbmgpu/lbmgpu.hpp) exactly as they are written against
// lbmlab in p/tests/test_schemes.cpp — only the namespace differs. Runs on a
// GPU (tests/test_cpp_api.py, -m gpu). Exit 0 iff every check passes.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "lbmgpu/lbmgpu.hpp"

using namespace lbmgpu;

namespace {

int failures = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (!(cond)) {                                                         \
      std::fprintf(stderr, "[FAIL] %s:%d %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                          \
    }                                                                      \
  } while (0)

// make_seeded_geometry (p/src/bench.cpp:259-273)
GridGeometry seeded_geometry(std::uint64_t seed) {
  GridGeometry g;
  g.nx = 16, g.ny = 8, g.nz = 8;
  g.axis_policy = {AxisPolicy::periodic, AxisPolicy::wall, AxisPolicy::periodic};
  g.mask.assign(g.cells(), 1);
  std::mt19937_64 rng(seed);
  for (int z = 0; z < g.nz; ++z)
    for (int y = 1; y < g.ny - 1; ++y)
      for (int x = 0; x < g.nx; ++x)
        if (rng() % 100 < 12) g.mask[g.index(x, y, z)] = 0;
  return g;
}

// random_field (p/tests/test_schemes.cpp:29-39)
std::vector<double> random_field(const Stencil& s, std::size_t nodes, std::uint64_t seed) {
  std::vector<double> f(nodes * s.q);
  std::mt19937_64 rng(seed);
  for (std::size_t n = 0; n < nodes; ++n)
    for (int i = 0; i < s.q; ++i) {
      const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
      f[n * s.q + i] = s.w[i] * (0.9 + 0.2 * u);
    }
  return f;
}

bool bitwise_equal(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * 8) == 0;
}

}  // namespace

int main() {
  const Stencil s = make_stencil("d3q19");
  const GridGeometry g = seeded_geometry(42);
  const FlowParams p;

  // availability matrix (p/tests/test_schemes.cpp:65-95)
  int pairs = 0;
  for (SchemeId id : all_schemes())
    for (Addressing a : {Addressing::direct, Addressing::indirect}) pairs += kernel_available(id, a);
  CHECK(pairs == 16);
  CHECK(parse_scheme("OSNT_pull_1s") == SchemeId::osnt_pull_1s);
  try {
    create_stepper(SchemeId::cg, Addressing::indirect, g, s, p);
    CHECK(false);
  } catch (const std::invalid_argument& e) {
    CHECK(std::string(e.what()) == "kernel not implemented; traffic model only");
  }

  // every implemented pair tracks TS bitwise for 10 steps (test_schemes.cpp:145-183)
  auto ref = create_stepper(SchemeId::ts, Addressing::direct, g, s, p);
  const std::vector<double> f0 = random_field(s, ref->node_count(), 4242);
  ref->load_natural(f0.data());
  std::vector<std::unique_ptr<Stepper>> probes;
  for (SchemeId id : all_schemes())
    for (Addressing a : {Addressing::direct, Addressing::indirect}) {
      if (!kernel_available(id, a) || (id == SchemeId::ts && a == Addressing::direct)) continue;
      for (Layout lay : {Layout::soa, Layout::aos}) {
        StepperOptions o;
        o.layout = lay;
        probes.push_back(create_stepper(id, a, g, s, p, o));
        probes.back()->load_natural(f0.data());
      }
    }
  CHECK(probes.size() == 30);
  for (int t = 1; t <= 10; ++t) {
    ref->step();
    const std::vector<double> want = ref->extract_natural();
    for (auto& st : probes) {
      st->step();
      CHECK(st->time_step() == t);
      const bool same = bitwise_equal(st->extract_natural(), want);
      if (!same)
        std::fprintf(stderr, "  %s/%s differs at t=%d\n", std::string(to_string(st->scheme())).c_str(),
                     std::string(to_string(st->addressing())).c_str(), t);
      CHECK(same);
    }
  }

  // layout phases (test_schemes.cpp:358-396)
  {
    const GridGeometry ch = gen_channel(8, 4, 4);
    auto aa = create_stepper(SchemeId::aap, Addressing::direct, ch, s, p);
    aa->step();
    CHECK(aa->layout_phase() == LayoutPhase::opposed);
    auto et = create_stepper(SchemeId::et, Addressing::indirect, ch, s, p);
    CHECK(et->exchange_opposite_handles());
    CHECK(et->layout_phase() == LayoutPhase::twisted);
  }

  // build_sparse reciprocity (p/tests/test_geometry.cpp:155-170)
  {
    const SparseRepresentation sp = build_sparse(g, s);
    CHECK(sp.fluid_count == g.fluid_count());
    for (std::uint32_t n = 0; n < sp.fluid_count; ++n)
      for (int i = 1; i < 19; ++i) {
        const std::uint32_t m = sp.neighbor(n, i);
        if (m != n) CHECK(sp.neighbor(m, s.opposite[i]) == n);
      }
  }

  // traffic table (p/tests/acceptance.cpp:69-98)
  CHECK(traffic(SchemeFamily::aap, Addressing::indirect).bytes_per_lup() == 340);
  CHECK(traffic(SchemeFamily::ts, Addressing::direct).bytes_per_lup() == 912);

  // z-slabs in one process (NCCL-free transports): two AA slabs over peer
  // memory reproduce one domain bitwise at odd and even t
  {
    GridGeometry box;
    box.nx = 40, box.ny = 12, box.nz = 10;
    auto one = create_stepper(SchemeId::aap, Addressing::direct, box, s, p);
    StepperOptions lo, hi;
    lo.z_begin = 0, lo.z_end = 4, hi.z_begin = 4, hi.z_end = 10;
    auto a = create_stepper(SchemeId::aap, Addressing::direct, box, s, p, lo);
    auto b = create_stepper(SchemeId::aap, Addressing::direct, box, s, p, hi);
    const std::vector<double> f0 = random_field(s, one->node_count(), 7);
    one->load_natural(f0.data());
    const std::size_t split = a->values();
    a->load_natural(f0.data());
    b->load_natural(f0.data() + split);
    std::vector<Stepper*> group{a.get(), b.get()};
    slab_group_connect_p2p(group);
    for (int steps : {3, 4}) {  // t = 3 (odd), 7 (odd) ...
      for (int k = 0; k < steps; ++k) one->step();
      slab_group_step(group, steps);
      if (one->time_step() % 2) slab_group_sync_ghosts(group);
      std::vector<double> got = a->extract_natural();
      const std::vector<double> tail = b->extract_natural();
      got.insert(got.end(), tail.begin(), tail.end());
      CHECK(bitwise_equal(got, one->extract_natural()));
    }
    for (int k = 0; k < 1; ++k) one->step();
    slab_group_step(group, 1);  // t = 8 (even)
    std::vector<double> got = a->extract_natural();
    const std::vector<double> tail = b->extract_natural();
    got.insert(got.end(), tail.begin(), tail.end());
    CHECK(bitwise_equal(got, one->extract_natural()));
  }

  // macroscopic_fields (p/src/stepper.cpp:182-193) and moments' domain_error
  // "vacuum node" (p/src/collision.cpp:31)
  {
    auto st = create_stepper(SchemeId::aap, Addressing::direct, g, s, p);
    const MacroFields m0 = macroscopic_fields(*st, s, p);
    CHECK(m0.rho.size() == st->node_count() && m0.u.size() == st->node_count());
    for (std::size_t n = 0; n < m0.rho.size(); ++n) {  // rest start: rho0, u = g/2
      CHECK(std::abs(m0.rho[n] - p.rho0) < 1e-14);
      CHECK(std::abs(m0.u[n][0] - 0.5 * p.body_force[0]) < 1e-14);
    }
    std::vector<double> f = st->extract_natural();
    for (int i = 0; i < 19; ++i) f[3 * 19 + i] = 0.0;
    st->load_natural(f.data());
    bool threw = false;
    try {
      (void)macroscopic_fields(*st, s, p);
    } catch (const std::domain_error& e) {
      threw = std::string(e.what()) == "vacuum node";
    }
    CHECK(threw);
  }

  std::printf("%s: %d failure(s)\n", failures ? "FAIL" : "PASS", failures);
  return failures ? 1 : 0;
}
