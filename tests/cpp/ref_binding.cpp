// The reference's own callers, run on the GPU through the reference-side
// binding (include/lbmgpu/lbmlab_gpu.hpp: GpuStepper : lbmlab::Stepper).
//
// Built against the UNMODIFIED reference headers and library (oracle/_ref,
// compiled from /root/reference by oracle/Makefile) and liblbmgpu.so; run by
// tests/test_gpu_ref_binding.py on the GPU box. Each check restates one
// reference caller with create_stepper replaced by create_gpu_stepper and is
// otherwise the reference's own logic:
//
//   verify      verify_suite's loop (p/src/bench.cpp:275-341): every
//               implemented pair against the reference's CPU two-step
//               stepper on make_seeded_geometry(42), memcmp after each of 10
//               steps; also every layout/precision variant (fp32 <= 1e-5)
//   conserve    acceptance criterion 4 (p/tests/acceptance.cpp:140-169):
//               closed 8^3 box, 1000 steps, |mass drift| <= 1e-10, every pair
//   channel     acceptance criterion 5 (:173-230): force-driven channel to
//               steady state, profiled with the reference's macroscopic_fields
//               on the GPU stepper, parabola to 1e-6
//   chunks      acceptance criterion 8 (:285-310): chunk-length invariance
//   errors      the reference's exception types and texts through the binding,
//               incl. macroscopic_fields' domain_error("vacuum node")
//   bench       run_bench's timing loop (p/src/bench.cpp:155-198) over the
//               GPU stepper: warm-up, timed_runs x steps of synchronous step()
//
// Prints one [PASS]/[FAIL] line per check; exit 0 iff all selected pass.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "lbmgpu/lbmlab_gpu.hpp"
#include "lbmlab/bench.hpp"
#include "lbmlab/collision.hpp"
#include "lbmlab/geometry.hpp"
#include "lbmlab/stencil.hpp"
#include "lbmlab/stepper.hpp"

using lbmgpu::binding::create_gpu_stepper;
using lbmgpu::binding::GpuOptions;
using lbmlab::Addressing;
using lbmlab::SchemeId;

namespace {

#define REQUIRE(cond, msg)                                                            \
  do {                                                                                \
    if (!(cond)) {                                                                    \
      std::fprintf(stderr, "[FAIL] %s:%d %s\n", __FILE__, __LINE__,                   \
                   std::string(msg).c_str());                                         \
      return false;                                                                   \
    }                                                                                 \
  } while (0)

std::string name(SchemeId id, Addressing a) {
  return std::string(lbmlab::to_string(id)) + "/" + std::string(lbmlab::to_string(a));
}
std::string num(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.6g", v);
  return b;
}

double max_rel(const std::vector<double>& got, const std::vector<double>& want) {
  double m = 0.0;
  for (std::size_t v = 0; v < want.size(); ++v)
    m = std::max(m, std::abs(got[v] - want[v]) / std::max(std::abs(want[v]), 1.0e-300));
  return m;
}

// verify_suite (p/src/bench.cpp:275-341) with GPU probes
bool check_verify() {
  const lbmlab::Stencil s = lbmlab::make_stencil("d3q19");
  const lbmlab::GridGeometry g = lbmlab::make_seeded_geometry(42);
  const lbmlab::FlowParams p;
  const std::size_t nvals = g.fluid_count() * s.q;
  std::vector<double> f0(nvals);
  std::mt19937_64 rng(42 ^ 0x9e3779b97f4a7c15ull);
  for (std::size_t n = 0; n < g.fluid_count(); ++n)
    for (int i = 0; i < s.q; ++i) {
      const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
      f0[n * s.q + i] = s.w[i] * p.rho0 * (0.9 + 0.2 * u);
    }
  auto ref = lbmlab::create_stepper(SchemeId::ts, Addressing::direct, g, s, p);  // CPU
  ref->load_natural(f0.data());

  struct Probe {
    std::string label;
    int precision;
    std::unique_ptr<lbmlab::Stepper> st;
    bool bitwise = true;
    double max_rel = 0.0;
  };
  std::vector<Probe> probes;
  int pairs = 0;
  for (SchemeId id : lbmlab::all_schemes())
    for (Addressing a : {Addressing::direct, Addressing::indirect}) {
      if (!lbmlab::kernel_available(id, a)) continue;
      ++pairs;
      for (int layout : {LBMGPU_SOA, LBMGPU_AOS})
        for (int prec : {8, 4}) {
          GpuOptions gpu;
          gpu.layout = layout;
          gpu.precision = prec;
          Probe pr;
          pr.label = name(id, a) + (layout == LBMGPU_SOA ? "/soa" : "/aos") +
                     (prec == 8 ? "/f64" : "/f32");
          pr.precision = prec;
          pr.st = create_gpu_stepper(id, a, g, s, p, {}, gpu);
          pr.st->load_natural(f0.data());
          probes.push_back(std::move(pr));
        }
    }
  REQUIRE(pairs == 16, "expected the reference's 16 implemented pairs, got " + num(pairs));
  std::vector<double> want(nvals), got(nvals);
  for (int k = 0; k < 10; ++k) {
    ref->step();
    ref->extract_natural(want.data());
    for (Probe& pr : probes) {
      pr.st->step();
      pr.st->extract_natural(got.data());
      if (std::memcmp(want.data(), got.data(), nvals * sizeof(double)) == 0) continue;
      pr.bitwise = false;
      pr.max_rel = std::max(pr.max_rel, max_rel(got, want));
    }
  }
  for (const Probe& pr : probes) {
    if (pr.precision == 8)
      REQUIRE(pr.bitwise, pr.label + " not bitwise (max rel " + num(pr.max_rel) + ")");
    else
      REQUIRE(pr.max_rel <= 1e-5, pr.label + " fp32 max rel " + num(pr.max_rel));
  }
  std::printf("  %zu GPU probes (16 pairs x SoA/AoS x fp64/fp32) vs the reference's CPU "
              "two-step stepper, 10 steps\n", probes.size());
  // and the reference's own verify_suite on its CPU kernels still passes
  const lbmlab::VerifyReport rep = lbmlab::verify_suite(42, 10);
  REQUIRE(rep.all_pass && rep.entries.size() == 15, "reference verify_suite failed");
  return true;
}

std::vector<double> random_positive_field(const lbmlab::Stencil& s, std::size_t nodes,
                                          std::uint64_t seed) {
  std::vector<double> f(nodes * s.q);
  std::mt19937_64 rng(seed);
  for (std::size_t n = 0; n < nodes; ++n)
    for (int i = 0; i < s.q; ++i) {
      const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
      f[n * s.q + i] = s.w[i] * (0.9 + 0.2 * u);
    }
  return f;
}

// acceptance criterion 4 (p/tests/acceptance.cpp:140-169)
bool check_conserve() {
  const lbmlab::Stencil s = lbmlab::make_stencil("d3q19");
  lbmlab::GridGeometry g;
  g.nx = g.ny = g.nz = 8;
  g.axis_policy = {lbmlab::AxisPolicy::wall, lbmlab::AxisPolicy::wall, lbmlab::AxisPolicy::wall};
  g.mask.assign(g.cells(), 1);
  lbmlab::FlowParams p;
  p.body_force = {0.0, 0.0, 0.0};
  int n = 0;
  for (SchemeId id : lbmlab::all_schemes())
    for (Addressing a : {Addressing::direct, Addressing::indirect}) {
      if (!lbmlab::kernel_available(id, a)) continue;
      for (int layout : {LBMGPU_SOA, LBMGPU_AOS}) {
        GpuOptions gpu;
        gpu.layout = layout;
        auto st = create_gpu_stepper(id, a, g, s, p, {}, gpu);
        const auto f0 = random_positive_field(s, st->node_count(), 2026);
        st->load_natural(f0.data());
        double mass0 = 0.0;
        for (double v : f0) mass0 += v;
        for (int t = 0; t < 1000; ++t) st->step();
        REQUIRE(st->time_step() == 1000, "time_step");
        const std::vector<double> f1 = st->extract_natural();
        double mass1 = 0.0;
        for (double v : f1) mass1 += v;
        const double drift = std::abs(mass1 - mass0) / mass0;
        REQUIRE(drift <= 1e-10, name(id, a) + " mass drift " + num(drift));
        ++n;
      }
    }
  std::printf("  %d GPU steppers, 1000 steps each, closed 8^3 box\n", n);
  return true;
}

// acceptance criterion 5 (p/tests/acceptance.cpp:173-230), profiled through the
// reference's own macroscopic_fields on the GPU stepper
bool channel_for(SchemeId id) {
  const lbmlab::Stencil s = lbmlab::make_stencil("d3q19");
  lbmlab::GridGeometry g;
  g.nx = 16;
  g.ny = 32;
  g.nz = 4;
  g.axis_policy = {lbmlab::AxisPolicy::periodic, lbmlab::AxisPolicy::wall,
                   lbmlab::AxisPolicy::periodic};
  g.mask.assign(g.cells(), 1);
  const lbmlab::FlowParams p;
  auto st = create_gpu_stepper(id, Addressing::direct, g, s, p);
  auto profile = [&]() {
    const lbmlab::MacroFields m = lbmlab::macroscopic_fields(*st, s, p);
    std::vector<double> prof(g.ny, 0.0);
    std::size_t n = 0;
    for (int z = 0; z < g.nz; ++z)
      for (int y = 0; y < g.ny; ++y)
        for (int x = 0; x < g.nx; ++x, ++n) prof[y] += m.u[n][0];
    for (double& v : prof) v /= static_cast<double>(g.nx) * g.nz;
    return prof;
  };
  std::vector<double> prev = profile();
  int t = 0;
  double change = 1.0;
  for (; t < 200000; ++t) {
    st->step();
    const std::vector<double> cur = profile();
    double dmax = 0.0, umax = 0.0;
    for (int y = 0; y < g.ny; ++y) {
      dmax = std::max(dmax, std::abs(cur[y] - prev[y]));
      umax = std::max(umax, std::abs(cur[y]));
    }
    prev = cur;
    change = dmax / umax;
    if (change < 1e-12) break;
  }
  REQUIRE(change < 1e-12, "no steady state after 200000 steps (" + num(change) + ")");
  const double nu = (1.0 / p.lambda_even - 0.5) / 3.0;
  const double gx = p.body_force[0];
  const double h = g.ny;
  double err = 0.0, scale = 0.0;
  for (int y = 0; y < g.ny; ++y) {
    const double yc = y + 0.5 - h / 2;
    const double ana = gx / (2 * nu) * (h * h / 4 - yc * yc);
    err = std::max(err, std::abs(prev[y] - ana));
    scale = std::max(scale, std::abs(ana));
  }
  REQUIRE(err / scale <= 1e-6, std::string(lbmlab::to_string(id)) + " profile rel Linf " +
                                   num(err / scale) + " after " + num(t) + " steps");
  std::printf("  %s: steady after %d steps, parabola rel Linf %.3g\n",
              std::string(lbmlab::to_string(id)).c_str(), t, err / scale);
  return true;
}
bool check_channel() { return channel_for(SchemeId::ts) && channel_for(SchemeId::aap); }

// acceptance criterion 8 (p/tests/acceptance.cpp:285-310)
bool check_chunks() {
  const lbmlab::Stencil s = lbmlab::make_stencil("d3q19");
  const lbmlab::GridGeometry g = lbmlab::make_seeded_geometry(42);
  const lbmlab::FlowParams p;
  const int chunks[] = {1, 150, static_cast<int>(g.fluid_count())};
  for (SchemeId id : {SchemeId::osnt_pull_1s, SchemeId::osnt_pull_2s})
    for (Addressing a : {Addressing::direct, Addressing::indirect}) {
      std::vector<std::vector<double>> outs;
      for (int chunk : chunks) {
        lbmlab::StepperOptions opt;
        opt.chunk_length = chunk;
        auto st = create_gpu_stepper(id, a, g, s, p, opt);
        for (int t = 0; t < 5; ++t) st->step();
        outs.push_back(st->extract_natural());
      }
      // and the reference's CPU kernel from the same start
      auto cpu = lbmlab::create_stepper(id, a, g, s, p);
      for (int t = 0; t < 5; ++t) cpu->step();
      outs.push_back(cpu->extract_natural());
      for (std::size_t k = 1; k < outs.size(); ++k)
        REQUIRE(std::memcmp(outs[k].data(), outs[0].data(), outs[0].size() * sizeof(double)) == 0,
                name(id, a) + " differs (variant " + num(k) + ")");
    }
  return true;
}

template <class E, class F>
bool throws(F&& f, const std::string& text) {
  try {
    f();
  } catch (const E& e) {
    return std::string(e.what()) == text;
  } catch (...) {
    return false;
  }
  return false;
}

bool check_errors() {
  const lbmlab::Stencil s = lbmlab::make_stencil("d3q19");
  const lbmlab::GridGeometry g = lbmlab::make_seeded_geometry(42);
  const lbmlab::FlowParams p;
  REQUIRE((throws<std::invalid_argument>(
              [&] { create_gpu_stepper(SchemeId::cg, Addressing::indirect, g, s, p); },
              "kernel not implemented; traffic model only")),
          "unsupported pair");
  lbmlab::StepperOptions bad;
  bad.workers = -1;
  REQUIRE((throws<std::invalid_argument>(
              [&] { create_gpu_stepper(SchemeId::aap, Addressing::direct, g, s, p, bad); },
              "workers must be >= 0")),
          "workers");
  bad = {};
  bad.chunk_length = 0;
  REQUIRE((throws<std::invalid_argument>(
              [&] { create_gpu_stepper(SchemeId::osnt_pull_1s, Addressing::direct, g, s, p, bad); },
              "chunk_length must be >= 1")),
          "chunk_length");
  REQUIRE((throws<std::invalid_argument>(
              [&] {
                create_gpu_stepper(SchemeId::aap, Addressing::direct, g,
                                   lbmlab::make_stencil("d2q9"), p);
              },
              "unsupported stencil: d2q9")),
          "stencil");
  // a vacuum node: the reference's macroscopic_fields (moments,
  // p/src/collision.cpp:31) throws domain_error on the GPU stepper's state
  auto st = create_gpu_stepper(SchemeId::aap, Addressing::direct, g, s, p);
  std::vector<double> f = st->extract_natural();
  for (int i = 0; i < 19; ++i) f[5 * 19 + i] = 0.0;
  st->load_natural(f.data());
  REQUIRE((throws<std::domain_error>([&] { lbmlab::macroscopic_fields(*st, s, p); },
                                     "vacuum node")),
          "vacuum node");
  // ET's handle table through the base-class virtual
  auto et = create_gpu_stepper(SchemeId::et, Addressing::direct, g, s, p);
  auto os = create_gpu_stepper(SchemeId::os_pull, Addressing::direct, g, s, p);
  REQUIRE(et->exchange_opposite_handles() && !os->exchange_opposite_handles(), "handles");
  return true;
}

// run_bench's loop (p/src/bench.cpp:155-198) over the GPU stepper
bool check_bench() {
  const lbmlab::Stencil s = lbmlab::make_stencil("d3q19");
  const lbmlab::GridGeometry g = lbmlab::gen_channel(128, 128, 128);
  const lbmlab::FlowParams p;
  for (SchemeId id : {SchemeId::aap, SchemeId::os_pull, SchemeId::et}) {
    auto st = create_gpu_stepper(id, Addressing::direct, g, s, p);
    st->step();  // warm-up
    std::vector<double> times;
    for (int r = 0; r < 3; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      for (int i = 0; i < 20; ++i) st->step();
      times.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    std::sort(times.begin(), times.end());
    const double mlups = static_cast<double>(g.fluid_count()) * 20 / times[1] / 1e6;
    std::printf("  %-8s run_bench loop (synchronous step()): %.0f MFLUP/s on 128^3\n",
                std::string(lbmlab::to_string(id)).c_str(), mlups);
    REQUIRE(mlups > 0, "timing");
  }
  return true;
}

struct Check {
  const char* id;
  bool (*fn)();
};
const Check kChecks[] = {{"verify", check_verify},   {"conserve", check_conserve},
                         {"channel", check_channel}, {"chunks", check_chunks},
                         {"errors", check_errors},   {"bench", check_bench}};

}  // namespace

int main(int argc, char** argv) {
  int failed = 0, ran = 0;
  for (const Check& c : kChecks) {
    bool sel = argc < 2;
    for (int k = 1; k < argc; ++k) sel = sel || std::string(argv[k]) == c.id;
    if (!sel) continue;
    ++ran;
    bool ok = false;
    try {
      ok = c.fn();
    } catch (const std::exception& e) {
      std::fprintf(stderr, "[FAIL] %s: exception %s\n", c.id, e.what());
    }
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.id);
    std::fflush(stdout);
    failed += !ok;
  }
  return (ran > 0 && failed == 0) ? 0 : 1;
}
