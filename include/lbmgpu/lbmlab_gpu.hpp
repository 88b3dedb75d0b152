// lbmlab_gpu.hpp — the reference-side binding: a GPU `lbmlab::Stepper`.
//
// For code built against the REFERENCE's own headers (lbmlab,
// p/include/lbmlab/stepper.hpp): `GpuStepper` derives from lbmlab::Stepper
// (p/include/lbmlab/stepper.hpp:70-106) and forwards every virtual to the C
// ABI of liblbmgpu.so (include/lbmgpu.h), so any reference caller that takes
// a `Stepper&` — the verify loop of verify_suite (p/src/bench.cpp:275-341),
// the timing loop of run_bench (:155-198), acceptance's checks
// (p/tests/acceptance.cpp:128-230), macroscopic_fields (p/src/stepper.cpp:182-193)
// — runs the sm_100a kernels unchanged. `create_gpu_stepper` has
// create_stepper's signature (p/src/stepper.cpp:155-180) plus the GPU
// selectors; a maintainer wires it into create_stepper with one branch
// (INTEGRATION.md section 2).
//
// Include path: the reference's include/ (for lbmlab/*.hpp) and this repo's
// include/ (for lbmgpu.h); link the reference library and -llbmgpu.
// tests/cpp/ref_binding.cpp builds and runs it against the unmodified
// reference (tests/test_gpu_ref_binding.py).
#pragma once

#include <cstdint>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>

#include "lbmgpu.h"
#include "lbmlab/collision.hpp"
#include "lbmlab/geometry.hpp"
#include "lbmlab/stencil.hpp"
#include "lbmlab/stepper.hpp"

namespace lbmgpu::binding {

// GPU selectors that lbmlab::StepperOptions has no field for
struct GpuOptions {
  int layout = LBMGPU_SOA;  // LBMGPU_SOA (the reference's layout) or LBMGPU_AOS
  int precision = 8;        // 8 = fp64 (the reference's), 4 = fp32
  int device = 0;
  bool extensions = false;  // also allow TS / SWAP indirect (no reference kernel)
};

// status -> the reference's exception types and texts
inline void check(int rc) {
  switch (rc) {
    case LBMGPU_OK: return;
    case LBMGPU_INVALID_ARGUMENT: throw std::invalid_argument(lbmgpu_last_error());
    case LBMGPU_DOMAIN_ERROR: throw std::domain_error(lbmgpu_last_error());
    case LBMGPU_BAD_ALLOC: throw std::bad_alloc();
    default: throw std::runtime_error(lbmgpu_last_error());
  }
}

class GpuStepper final : public lbmlab::Stepper {
 public:
  GpuStepper(lbmlab::SchemeId id, lbmlab::Addressing a, const lbmlab::GridGeometry& g,
             const lbmlab::Stencil& s, const lbmlab::FlowParams& p,
             const lbmlab::StepperOptions& opt, const GpuOptions& gpu)
      : lbmlab::Stepper(id, a, s.q, 0) {
    if (s.q != 19 || s.d != 3)
      throw std::invalid_argument("unsupported stencil: " + std::string(s.name));
    if (g.mask.size() != g.cells()) throw std::invalid_argument("mask size != nx*ny*nz");
    lbmgpu_geometry cg{g.nx, g.ny, g.nz,
                       {static_cast<std::uint8_t>(g.axis_policy[0]),
                        static_cast<std::uint8_t>(g.axis_policy[1]),
                        static_cast<std::uint8_t>(g.axis_policy[2])},
                       g.mask.data()};
    // the reference's own lambda_odd: both sides relax with the same double
    lbmgpu_flow f{p.lambda_even, lbmlab::lambda_odd(p),
                  {p.body_force[0], p.body_force[1], p.body_force[2]}, p.rho0};
    lbmgpu_options o;
    lbmgpu_default_options(&o);
    o.scheme = static_cast<std::int32_t>(id);
    o.addressing = static_cast<std::int32_t>(a);
    o.layout = gpu.layout;
    o.precision = gpu.precision;
    o.device = gpu.device;
    o.extensions = gpu.extensions;
    o.workers = opt.workers;
    o.chunk_length = opt.chunk_length;
    o.streaming_stores = opt.streaming_stores;
    o.swap_deferred_fixup = opt.swap_deferred_fixup;
    o.zero_collision = opt.zero_collision;
    check(lbmgpu_create(&cg, &f, &o, &h_));
    std::uint64_t n = 0;
    check(lbmgpu_node_count(h_, &n));
    nodes_ = static_cast<std::size_t>(n);
  }
  GpuStepper(const GpuStepper&) = delete;
  GpuStepper& operator=(const GpuStepper&) = delete;
  ~GpuStepper() override {
    if (h_) lbmgpu_destroy(h_);
  }

  // synchronous, like the reference's step(): run_bench's wall clock and
  // every caller that extracts after step() see a finished step
  void step() override {
    check(lbmgpu_step(h_, 1));
    check(lbmgpu_synchronize(h_));
    ++t_;
  }
  void extract_natural(double* out) const override {
    check(lbmgpu_extract_natural(h_, out));
  }
  void load_natural(const double* in) override {
    check(lbmgpu_load_natural(h_, in));
    t_ = 0;
  }
  lbmlab::LayoutPhase layout_phase() const override {
    std::int32_t v = 0;
    check(lbmgpu_layout_phase(h_, &v));
    return static_cast<lbmlab::LayoutPhase>(v);
  }
  bool exchange_opposite_handles() override {
    std::int32_t v = 0;
    check(lbmgpu_exchange_opposite_handles(h_, &v));
    return v != 0;
  }
  using lbmlab::Stepper::extract_natural;

  // GPU additions: n steps enqueued on the stepper's stream, then a sync;
  // device-timed steps (CUDA events on that stream)
  void step_n(long long n) {
    check(lbmgpu_step(h_, n));
    t_ += n;
  }
  void synchronize() { check(lbmgpu_synchronize(h_)); }
  double step_timed(long long n) {
    double ms = 0.0;
    check(lbmgpu_step_timed(h_, n, &ms));
    t_ += n;
    return ms;
  }
  // the library's own count (equals time_step() unless steps bypassed this object)
  long long device_time_step() const {
    std::int64_t t = 0;
    check(lbmgpu_time_step(h_, &t));
    return t;
  }
  lbmgpu_stepper* handle() const { return h_; }

 private:
  lbmgpu_stepper* h_ = nullptr;
};

// create_stepper's signature (p/include/lbmlab/stepper.hpp:110-113) + GPU selectors;
// unsupported pairs throw invalid_argument("kernel not implemented; traffic model only")
inline std::unique_ptr<lbmlab::Stepper> create_gpu_stepper(
    lbmlab::SchemeId id, lbmlab::Addressing a, const lbmlab::GridGeometry& g,
    const lbmlab::Stencil& s, const lbmlab::FlowParams& p,
    const lbmlab::StepperOptions& opt = {}, const GpuOptions& gpu = {}) {
  return std::make_unique<GpuStepper>(id, a, g, s, p, opt, gpu);
}

}  // namespace lbmgpu::binding
