// Host runtime of liblbmgpu.so: one C++ class per propagation scheme, each
// owning its device storage, index tables and CUDA stream, plus the C ABI of
// include/lbmgpu.h. Mirrors the reference's Stepper hierarchy
// (p/include/lbmlab/stepper.hpp:70-106, p/src/scheme_*.cpp): same state
// machine (time step, fresh/pending flags, ET handle table, layout phases),
// with every sweep a sm_100a kernel launch.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <random>
#include <cstring>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/lbmgpu.h"
#include "launch.h"

namespace lbmgpu {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

static void ck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    throw std::bad_alloc();
  }
  throw CudaError(std::string("cuda: ") + what + ": " + cudaGetErrorString(e));
}
#define CK(x) ck((x), #x)
static void ck_launch() { ck(cudaGetLastError(), "kernel launch"); }

// ---------------------------------------------------------------------------
// device memory
// ---------------------------------------------------------------------------
class DevMem {
 public:
  DevMem() = default;
  explicit DevMem(size_t bytes) { alloc(bytes); }
  ~DevMem() { release(); }
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
  DevMem(DevMem&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr, o.n_ = 0; }
  DevMem& operator=(DevMem&& o) noexcept {
    release();
    p_ = o.p_, n_ = o.n_;
    o.p_ = nullptr, o.n_ = 0;
    return *this;
  }
  void alloc(size_t bytes) {
    release();
    if (bytes == 0) bytes = 256;
    CK(cudaMalloc(&p_, bytes));
    n_ = bytes;
  }
  void release() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  template <class T = void>
  T* get() const {
    return static_cast<T*>(p_);
  }
  size_t bytes() const { return n_; }

 private:
  void* p_ = nullptr;
  size_t n_ = 0;
};

// ---------------------------------------------------------------------------
// host-side restatements used to set up kernels
// ---------------------------------------------------------------------------
static constexpr int kC[19][3] = {
    {0, 0, 0},   {1, 0, 0},   {-1, 0, 0}, {0, 1, 0},   {0, -1, 0}, {0, 0, 1},  {0, 0, -1},
    {-1, -1, 0}, {-1, 0, -1}, {-1, 0, 1}, {-1, 1, 0},  {0, -1, -1}, {0, -1, 1}, {0, 1, -1},
    {0, 1, 1},   {1, -1, 0},  {1, 0, -1}, {1, 0, 1},   {1, 1, 0}};
static constexpr int kPi[9] = {1, 3, 5, 7, 8, 9, 10, 11, 12};
static constexpr int kPj[9] = {2, 4, 6, 18, 17, 16, 15, 14, 13};
static double w_of(int i) { return i == 0 ? 1.0 / 3.0 : (i <= 6 ? 1.0 / 18.0 : 1.0 / 36.0); }

// TrtOperator ctor/build (p/src/collision.cpp:50-93), including the
// zero-collision identity operator (p/src/stepper_common.hpp:104-108).
static TrtHost make_trt(const lbmgpu_flow& p, bool zero_collision) {
  const double le = zero_collision ? 0.0 : p.lambda_even;
  const double lo = zero_collision ? 0.0 : p.lambda_odd;
  const double g[3] = {zero_collision ? 0.0 : p.body_force[0],
                       zero_collision ? 0.0 : p.body_force[1],
                       zero_collision ? 0.0 : p.body_force[2]};
  TrtHost t{};
  t.lambda_e = le;
  t.le_half = 0.5 * le;
  t.lo_half = 0.5 * lo;
  t.w0 = w_of(0);
  for (int q = 0; q < 9; ++q) {
    const int i = kPi[q];
    double cg = 0.0;
    for (int k = 0; k < 3; ++k) {
      const int ck_ = kC[i][k];
      if (ck_ == 0) continue;
      cg += ck_ * g[k];
    }
    t.w2[q] = 2.0 * w_of(i);
    t.f3w[q] = 3.0 * w_of(i) * cg;
  }
  return t;
}

struct HostGeo {
  int nx = 0, ny = 0, nz = 0;
  uint8_t policy[3] = {0, 0, 0};
  std::vector<uint8_t> mask;  // empty = all fluid
  bool solids = false;
  uint64_t cells() const { return (uint64_t)nx * ny * nz; }
  bool fluid(uint64_t c) const { return mask.empty() || mask[c]; }
  uint64_t idx(int x, int y, int z) const {
    return (uint64_t)x + (uint64_t)nx * ((uint64_t)y + (uint64_t)ny * z);
  }
  // resolve_link (p/src/geometry.cpp:49-60); returns false on bounce
  bool link(int x, int y, int z, int i, int* t) const {
    const int n[3] = {nx, ny, nz};
    int p[3] = {x + kC[i][0], y + kC[i][1], z + kC[i][2]};
    for (int k = 0; k < 3; ++k) {
      if (p[k] >= 0 && p[k] < n[k]) continue;
      if (policy[k] == 1) return false;
      p[k] = p[k] < 0 ? p[k] + n[k] : p[k] - n[k];
    }
    if (!fluid(idx(p[0], p[1], p[2]))) return false;
    t[0] = p[0], t[1] = p[1], t[2] = p[2];
    return true;
  }
};

static HostGeo copy_geo(const lbmgpu_geometry* g) {
  if (!g) throw std::invalid_argument("null geometry");
  if (g->nx < 1 || g->ny < 1 || g->nz < 1) throw std::invalid_argument("zero dimension");
  for (int k = 0; k < 3; ++k)
    if (g->axis_policy[k] > 1) throw std::invalid_argument("unknown axis policy");
  HostGeo h;
  h.nx = g->nx, h.ny = g->ny, h.nz = g->nz;
  for (int k = 0; k < 3; ++k) h.policy[k] = g->axis_policy[k];
  if (h.cells() >= (uint64_t{1} << 32))
    throw std::runtime_error("grid exceeds 32-bit cell index range");
  if (g->mask) {
    h.mask.assign(g->mask, g->mask + h.cells());
    for (auto& m : h.mask) m = m != 0;
    h.solids = std::find(h.mask.begin(), h.mask.end(), 0) != h.mask.end();
    if (!h.solids) h.mask.clear();
  }
  return h;
}

static dev::Lat make_lat(const HostGeo& g, const uint32_t* linkmask, int hx, int hy, int hz,
                         int origin) {
  dev::Lat L{};
  L.nx = g.nx, L.ny = g.ny, L.nz = g.nz;
  L.sx = g.nx + 2 * hx;
  L.sy = g.ny + 2 * hy;
  L.sxy = (long long)L.sx * L.sy;
  L.ox = hx + origin, L.oy = hy + origin, L.oz = hz + origin;
  L.ncells = (uint32_t)g.cells();
  for (int k = 0; k < 3; ++k) L.wall[k] = g.policy[k];
  L.zghost = 0;
  L.linkmask = linkmask;
  L.divx.init((uint32_t)g.nx);
  L.divy.init((uint32_t)g.ny);
  return L;
}

// kernel availability (p/src/stepper.cpp:140-153)
static bool available(int s, int a, bool ext) {
  if (s < 0 || s > 9 || a < 0 || a > 1) return false;
  if (a == LBMGPU_DIRECT) return true;
  switch (s) {
    case LBMGPU_OS_PUSH:
    case LBMGPU_OS_PULL:
    case LBMGPU_OSNT_PULL_1S:
    case LBMGPU_OSNT_PULL_2S:
    case LBMGPU_AAP:
    case LBMGPU_ET:
      return true;
    case LBMGPU_TS:
    case LBMGPU_SWAP_PUSH:
    case LBMGPU_SWAP_PULL:
      return ext;
    default:
      return false;
  }
}

// ---------------------------------------------------------------------------
// Stepper base: geometry on the device, node maps, canonical conversion
// ---------------------------------------------------------------------------
class Stepper {
 public:
  Stepper(const HostGeo& g, const lbmgpu_flow& p, const lbmgpu_options& o)
      : geo_(g), opt_(o), op_(make_trt(p, o.zero_collision != 0)), rho0_(p.rho0) {
    prec_ = o.precision == 4 ? Prec::f32 : Prec::f64;
    aos_ = o.layout == LBMGPU_AOS;
    CK(cudaSetDevice(o.device));
    CK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    setup_nodes();
  }
  virtual ~Stepper() {
    if (stream_) {
      cudaStreamSynchronize(stream_);
      cudaStreamDestroy(stream_);
    }
  }

  virtual void step_one() = 0;
  virtual int launches_per_step() const { return 1; }
  virtual void extract_range(uint32_t n0, uint32_t cnt, double* dbuf) = 0;
  virtual void load_range(uint32_t n0, uint32_t cnt, const double* dbuf, const InitSpec& in) = 0;
  virtual void after_load() { t_ = 0; }
  virtual void before_extract() {}
  virtual void finish() {}  // join side streams into stream_ after a step() batch
  virtual void after_extract() {}
  virtual int layout_phase() const { return LBMGPU_NATURAL; }
  virtual bool exchange_opposite_handles() { return false; }
  virtual uint64_t pdf_bytes() const = 0;
  virtual uint64_t idx_bytes() const { return 0; }
  // nodes of the canonical snapshot (a z-slab on indirect addressing stores
  // ghost-plane nodes besides its own)
  virtual uint64_t snapshot_nodes() const { return nodes_; }

  void step(long long n) {
    CK(cudaSetDevice(opt_.device));
    for (long long k = 0; k < n; ++k) {
      if (nodes_ > 0) step_one();
      ++t_;
    }
    finish();
    ck_launch();
  }

  void sync() { CK(cudaStreamSynchronize(stream_)); }

  // canonical snapshot <-> storage, in chunks through a device staging buffer;
  // [first, first + count) selects a node range (out holds count*19 values)
  void extract(double* out, bool out_on_device, uint64_t first = 0, uint64_t count = ~0ull) {
    CK(cudaSetDevice(opt_.device));
    const uint64_t nsnap = snapshot_nodes();
    if (count == ~0ull) count = nsnap - std::min(first, nsnap);
    if (first > nsnap || count > nsnap - first)
      throw std::invalid_argument("node range outside the snapshot");
    before_extract();
    const uint64_t ch = chunk_nodes();
    for (uint64_t k = 0; k < count; k += ch) {
      const uint32_t n0 = (uint32_t)(first + k);
      const uint32_t cnt = (uint32_t)std::min<uint64_t>(ch, count - k);
      double* d = out_on_device ? out + (size_t)k * 19 : stage();
      extract_range(n0, cnt, d);
      ck_launch();
      if (!out_on_device) {
        CK(cudaMemcpyAsync(out + (size_t)k * 19, d, (size_t)cnt * 19 * sizeof(double),
                           cudaMemcpyDeviceToHost, stream_));
        sync();
      }
    }
    after_extract();
    sync();
  }

  void load(const double* in, bool in_on_device) {
    CK(cudaSetDevice(opt_.device));
    InitSpec spec;
    spec.source = kSrcBuffer;
    for_chunks([&](uint32_t n0, uint32_t cnt) {
      const double* d = in + (size_t)n0 * 19;
      if (!in_on_device) {
        double* s = stage();
        CK(cudaMemcpyAsync(s, d, (size_t)cnt * 19 * sizeof(double), cudaMemcpyHostToDevice,
                           stream_));
        d = s;
      }
      load_range(n0, cnt, d, spec);
      ck_launch();
      if (!in_on_device) sync();
    });
    after_load();
    sync();
  }

  void init(const InitSpec& spec) {
    CK(cudaSetDevice(opt_.device));
    for_chunks([&](uint32_t n0, uint32_t cnt) {
      load_range(n0, cnt, nullptr, spec);
      ck_launch();
    });
    after_load();
    sync();
  }

  InitSpec base_init(int source) const {
    InitSpec s;
    s.source = source;
    s.rho0 = rho0_;
    s.gnx = geo_.nx, s.gny = geo_.ny, s.gnz = geo_.nz;
    s.z0 = 0;
    return s;
  }

  long long t_ = 0;
  uint64_t nodes_ = 0;
  cudaStream_t stream_ = nullptr;
  lbmgpu_options opt_;

 protected:
  DField field(DevMem& m, long long stride) const {
    DField f;
    f.p = m.get();
    f.stride = stride;
    f.aos = aos_;
    f.prec = prec_;
    return f;
  }
  size_t esize() const { return prec_ == Prec::f64 ? 8 : 4; }
  long long soa_stride(uint64_t storage) const {
    return (long long)((storage + 31) & ~uint64_t{31});
  }
  uint64_t field_elems(uint64_t storage) const {
    return aos_ ? storage * 19 + 32 : (uint64_t)soa_stride(storage) * 19;
  }
  void alloc_field(DevMem& m, uint64_t storage) {
    m.alloc(field_elems(storage) * esize());
    CK(cudaMemsetAsync(m.get(), 0, m.bytes(), stream_));
  }

  double* stage() {
    if (!stage_.get()) stage_.alloc((size_t)chunk_nodes() * 19 * sizeof(double));
    return stage_.get<double>();
  }
  uint32_t chunk_nodes() const {
    return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(snapshot_nodes(), uint64_t{1} << 20));
  }
  template <class F>
  void for_chunks(F&& f) {
    const uint32_t ch = chunk_nodes();
    const uint64_t nsnap = snapshot_nodes();
    for (uint64_t n0 = 0; n0 < nsnap; n0 += ch)
      f((uint32_t)n0, (uint32_t)std::min<uint64_t>(ch, nsnap - n0));
  }

  // fluid enumeration x-fastest (build_sparse, p/src/geometry.cpp:187-194)
  void setup_nodes() {
    const uint64_t cells = geo_.cells();
    if (!geo_.solids) {
      nodes_ = cells;
      return;
    }
    mask_d_.alloc(cells);
    CK(cudaMemcpyAsync(mask_d_.get(), geo_.mask.data(), cells, cudaMemcpyHostToDevice, stream_));
    cell_of_node_.alloc(cells * sizeof(uint32_t));
    node_of_.alloc(cells * sizeof(uint32_t));
    DevMem scratch(scan_scratch_elems(cells) * sizeof(uint32_t));
    nodes_ = build_node_maps(stream_, mask_d_.get<uint8_t>(), cells, node_of_.get<uint32_t>(),
                             cell_of_node_.get<uint32_t>(), scratch.get<uint32_t>(), 0);
    ck_launch();
  }
  void setup_linkmask() {
    if (!geo_.solids) return;
    linkmask_.alloc(geo_.cells() * sizeof(uint32_t));
    const dev::Lat L = make_lat(geo_, nullptr, 0, 0, 0, 0);
    launch_linkmask(stream_, mask_d_.get<uint8_t>(), L, linkmask_.get<uint32_t>());
    ck_launch();
  }
  const uint32_t* linkmask() const { return geo_.solids ? linkmask_.get<uint32_t>() : nullptr; }
  const uint32_t* cell_of_node() const {
    return geo_.solids ? cell_of_node_.get<uint32_t>() : nullptr;
  }

  HostGeo geo_;
  TrtHost op_;
  double rho0_;
  Prec prec_ = Prec::f64;
  bool aos_ = false;
  DevMem mask_d_, cell_of_node_, node_of_, linkmask_, stage_;
};

// ---------------------------------------------------------------------------
// direct schemes
// ---------------------------------------------------------------------------
class DirectStepper : public Stepper {
 public:
  DirectStepper(const HostGeo& g, const lbmgpu_flow& p, const lbmgpu_options& o)
      : Stepper(g, p, o) {
    setup_linkmask();
    L_ = make_lat(geo_, linkmask(), 0, 0, 0, 0);
  }

 protected:
  void ex(const DField& f, const dev::Lat& L, int mode, uint32_t n0, uint32_t cnt, double* d,
          const EtBase& b = EtBase{}) {
    launch_extract(stream_, f, L, cell_of_node(), n0, cnt, mode, b, d);
  }
  void ld(const DField& f, const dev::Lat& L, int mode, uint32_t n0, uint32_t cnt,
          const double* d, const InitSpec& in) {
    launch_load(stream_, f, L, cell_of_node(), n0, cnt, mode, d, in);
  }
  dev::Lat L_;
};

// TS: collide A -> B, stream B -> A (p/src/scheme_ts.cpp)
class TsDirect final : public DirectStepper {
 public:
  TsDirect(const HostGeo& g, const lbmgpu_flow& p, const lbmgpu_options& o) : DirectStepper(g, p, o) {
    alloc_field(a_, g.cells());
    alloc_field(b_, g.cells());
    init(base_init(kSrcRest));
  }
  void step_one() override {
    const long long s = soa_stride(geo_.cells());
    launch_local(stream_, field(a_, s), field(b_, s), L_, op_, false, false);
    launch_ts_stream(stream_, field(a_, s), field(b_, s), L_);
  }
  int launches_per_step() const override { return 2; }
  void extract_range(uint32_t n0, uint32_t c, double* d) override {
    ex(field(a_, soa_stride(geo_.cells())), L_, kExNatural, n0, c, d);
  }
  void load_range(uint32_t n0, uint32_t c, const double* d, const InitSpec& in) override {
    ld(field(a_, soa_stride(geo_.cells())), L_, kExNatural, n0, c, d, in);
  }
  uint64_t pdf_bytes() const override { return a_.bytes() + b_.bytes(); }

 private:
  DevMem a_, b_;
};

// OS push/pull and OSNT pull (p/src/scheme_os.cpp, p/src/scheme_osnt.cpp)
class OsDirect final : public DirectStepper {
 public:
  OsDirect(const HostGeo& g, const lbmgpu_flow& p, const lbmgpu_options& o)
      : DirectStepper(g, p, o) {
    const int s = o.scheme;
    pull_ = s != LBMGPU_OS_PUSH;
    nt_ = (s == LBMGPU_OSNT_PULL_1S || s == LBMGPU_OSNT_PULL_2S) && o.streaming_stores;
    two_s_ = s == LBMGPU_OSNT_PULL_2S;
    alloc_field(g_[0], g.cells());
    alloc_field(g_[1], g.cells());
    init(base_init(kSrcRest));
  }
  void step_one() override {
    const long long s = soa_stride(geo_.cells());
    DField a = field(g_[active_], s), b = field(g_[active_ ^ 1], s);
    if (pull_ && fresh_) {
      launch_local(stream_, a, a, L_, op_, false, false);
      fresh_ = false;
    }
    if (pull_)
      launch_os_pull(stream_, a, b, L_, op_, nt_, two_s_);
    else
      launch_os_push(stream_, a, b, L_, op_);
    active_ ^= 1;
  }
  void extract_range(uint32_t n0, uint32_t c, double* d) override {
    const long long s = soa_stride(geo_.cells());
    if (!pull_ || fresh_)
      ex(field(g_[active_], s), L_, kExNatural, n0, c, d);
    else
      ex(field(g_[active_ ^ 1], s), L_, kExGather, n0, c, d);
  }
  void load_range(uint32_t n0, uint32_t c, const double* d, const InitSpec& in) override {
    ld(field(g_[active_], soa_stride(geo_.cells())), L_, kExNatural, n0, c, d, in);
  }
  void after_load() override {
    t_ = 0;
    fresh_ = pull_;
  }
  uint64_t pdf_bytes() const override { return g_[0].bytes() + g_[1].bytes(); }

 private:
  bool pull_, nt_, two_s_;
  bool fresh_ = false;
  int active_ = 0;
  DevMem g_[2];
};

// AA pattern (p/src/scheme_aap.cpp)
class AaDirect final : public DirectStepper {
 public:
  AaDirect(const HostGeo& g, const lbmgpu_flow& p, const lbmgpu_options& o)
      : DirectStepper(g, p, o) {
    alloc_field(f_, g.cells());
    init(base_init(kSrcRest));
  }
  void step_one() override {
    const DField f = field(f_, soa_stride(geo_.cells()));
    if ((t_ & 1) == 0)
      launch_local(stream_, f, f, L_, op_, false, true);
    else
      launch_aa_odd(stream_, f, L_, op_);
  }
  void extract_range(uint32_t n0, uint32_t c, double* d) override {
    ex(field(f_, soa_stride(geo_.cells())), L_, (t_ & 1) ? kExAaOdd : kExNatural, n0, c, d);
  }
  void load_range(uint32_t n0, uint32_t c, const double* d, const InitSpec& in) override {
    ld(field(f_, soa_stride(geo_.cells())), L_, kExNatural, n0, c, d, in);
  }
  int layout_phase() const override { return (t_ & 1) ? LBMGPU_OPPOSED : LBMGPU_NATURAL; }
  uint64_t pdf_bytes() const override { return f_.bytes(); }

 private:
  DevMem f_;
};

// ET (p/src/scheme_et.cpp): extended grid with a halo plane on wall axes
class EtDirect final : public DirectStepper {
 public:
  EtDirect(const HostGeo& g, const lbmgpu_flow& p, const lbmgpu_options& o)
      : DirectStepper(g, p, o) {
    for (int k = 0; k < 3; ++k) halo_[k] = g.policy[k] == 1 ? 1 : 0;
    Le_ = make_lat(geo_, linkmask(), halo_[0], halo_[1], halo_[2], 0);
    ext_ = (uint64_t)(g.nx + 2 * halo_[0]) * (g.ny + 2 * halo_[1]) * (g.nz + 2 * halo_[2]);
    alloc_field(f_, ext_);
    reset_base();
    init(base_init(kSrcRest));
  }
  void step_one() override {
    launch_et(stream_, field(f_, soa_stride(ext_)), Le_, op_, base_);
    swap_base();
  }
  void extract_range(uint32_t n0, uint32_t c, double* d) override {
    ex(field(f_, soa_stride(ext_)), Le_, kExEt, n0, c, d, base_);
  }
  void load_range(uint32_t n0, uint32_t c, const double* d, const InitSpec& in) override {
    reset_base();
    ld(field(f_, soa_stride(ext_)), Le_, kExEt, n0, c, d, in);
  }
  bool exchange_opposite_handles() override {
    swap_base();
    return true;
  }
  int layout_phase() const override {
    for (int i = 0; i < 19; ++i)
      if (base_.b[i] != i) return LBMGPU_TWISTED;
    return LBMGPU_NATURAL;
  }
  uint64_t pdf_bytes() const override { return f_.bytes(); }

 private:
  void reset_base() {
    for (int i = 0; i < 20; ++i) base_.b[i] = (int8_t)(i < 19 ? i : 0);
  }
  void swap_base() {
    for (int q = 0; q < 9; ++q) std::swap(base_.b[kPi[q]], base_.b[kPj[q]]);
  }
  int halo_[3];
  uint64_t ext_ = 0;
  dev::Lat Le_;
  EtBase base_;
  DevMem f_;
};

// periodic-seam links (targets wrapped by resolve_link), from fluid cells
// along `dirs` (CG: all 18, p/src/scheme_cg.cpp:31-41; SWAP: back half,
// p/src/scheme_swap.cpp:48-65)
struct SeamLink {
  int x, y, z, tx, ty, tz, lx, ly, lz, dir;
};
static std::vector<SeamLink> seam_links(const HostGeo& g, const int* dirs, int ndirs) {
  std::vector<SeamLink> out;
  for (int z = 0; z < g.nz; ++z)
    for (int y = 0; y < g.ny; ++y)
      for (int x = 0; x < g.nx; ++x) {
        if (x > 0 && x < g.nx - 1 && y > 0 && y < g.ny - 1 && z > 0 && z < g.nz - 1) continue;
        if (!g.fluid(g.idx(x, y, z))) continue;
        for (int k = 0; k < ndirs; ++k) {
          const int i = dirs[k];
          int t[3];
          if (!g.link(x, y, z, i, t)) continue;
          const int tx = x + kC[i][0], ty = y + kC[i][1], tz = z + kC[i][2];
          if (tx == t[0] && ty == t[1] && tz == t[2]) continue;
          out.push_back({x, y, z, tx, ty, tz, t[0], t[1], t[2], i});
        }
      }
  return out;
}

// CG (p/src/scheme_cg.cpp): one grid, two origins S planes apart, sweeps
// alternate the read origin (even: read S, write 0, ascending plane groups;
// odd: read 0, write S, descending), each plane group of P < S planes one
// push launch (P = nz/4 clamped to [16, 64]); z-periodic seam values land in
// padding planes and are copied to their wrapped planes after the sweep.
// Storage: nz + S + 2 planes
// (planes 0 and nz+S+1 pad; origin o's plane z at storage z + 1 + o).
class CgDirect final : public DirectStepper {
 public:
  CgDirect(const HostGeo& g, const lbmgpu_flow& p, const lbmgpu_options& o)
      : DirectStepper(g, p, o) {
    // planes per launch: more planes, fewer launch tails, but S = P + 1
    // extra storage planes (C1 256^3: P 16 / 32 / 64 / 128 -> 0.83 / 0.92 /
    // 0.95 / 0.96 of the roofline fp64, 0.74 / 0.82 / 0.85 / 0.87 fp32).
    // Default nz/4 in [16, 64]: +25% storage on 256^3; LBMGPU_CG_PLANES overrides.
    int planes = std::max(16, std::min(64, g.nz / 4));
    if (const char* e = std::getenv("LBMGPU_CG_PLANES")) planes = std::max(1, std::atoi(e));
    P_ = std::min(planes, g.nz);
    S_ = P_ + 1;
    plane_ = (uint64_t)g.nx * g.ny;
    storage_ = plane_ * (uint64_t)(g.nz + S_ + 2);
    if (storage_ >= (uint64_t{1} << 32))
      throw std::runtime_error("grid exceeds 32-bit cell index range");
    alloc_field(f_, storage_);
    init(base_init(kSrcRest));
    sync();
  }
  dev::Lat frame(int origin) const {
    dev::Lat L = L_;
    L.oz = 1 + origin;
    L.znowrap = 1;
    return L;
  }
  void step_one() override {
    const DField f = field(f_, soa_stride(storage_));
    const bool even = (t_ & 1) == 0;
    const int R = even ? S_ : 0, W = even ? 0 : S_;
    const int delta = (W - R) * (int)plane_;
    const dev::Lat Lr = frame(R);
    const int ngroups = (geo_.nz + P_ - 1) / P_;
    for (int k = 0; k < ngroups; ++k) {
      const int gi = even ? k : ngroups - 1 - k;
      dev::Lat L = Lr;
      L.cell_begin = (uint32_t)(gi * P_ * plane_);
      L.ncells = (uint32_t)(std::min(geo_.nz, (gi + 1) * P_) * plane_);
      launch_cg_push(stream_, f, L, op_, delta);
    }
    if (geo_.policy[2] == 0) {  // z-periodic seam fix-up
      static const int zm[5] = {6, 8, 11, 13, 16}, zp[5] = {5, 9, 12, 14, 17};
      const uint32_t pl = (uint32_t)plane_;
      launch_plane_copy(stream_, f, L_, zm, (uint32_t)W * pl, (uint32_t)(geo_.nz + W) * pl, 0);
      launch_plane_copy(stream_, f, L_, zp, (uint32_t)(geo_.nz + 1 + W) * pl,
                        (uint32_t)(1 + W) * pl, geo_.nz - 1);
    }
  }
  int launches_per_step() const override {
    return (geo_.nz + P_ - 1) / P_ + (geo_.policy[2] == 0 ? 2 : 0);
  }
  void extract_range(uint32_t n0, uint32_t c, double* d) override {
    ex(field(f_, soa_stride(storage_)), frame((t_ & 1) ? 0 : S_), kExNatural, n0, c, d);
  }
  void load_range(uint32_t n0, uint32_t c, const double* d, const InitSpec& in) override {
    ld(field(f_, soa_stride(storage_)), frame(S_), kExNatural, n0, c, d, in);
  }
  int layout_phase() const override {
    return (t_ & 1) ? LBMGPU_SHIFTED_EVEN : LBMGPU_SHIFTED_ODD;
  }
  uint64_t pdf_bytes() const override { return f_.bytes(); }

 private:
  int P_, S_;
  uint64_t plane_, storage_;
  DevMem f_;
};

// SWAP push/pull (p/src/scheme_swap.cpp): collide pass + link-exchange pass
// + the periodic-seam fix-up list (post-sweep for push, or deferred; pre-sweep
// for pull), exactly the reference's state machine. Fused single-sweep
// variants (ticketed tiles, a lagged pipeline, z-plane stage launches, a
// cooperative persistent sweep) were measured slower on B200.
class SwapDirect final : public DirectStepper {
 public:
  SwapDirect(const HostGeo& g, const lbmgpu_flow& p, const lbmgpu_options& o)
      : DirectStepper(g, p, o) {
    pull_ = o.scheme == LBMGPU_SWAP_PULL;
    defer_ = o.swap_deferred_fixup != 0;
    static const int back[9] = {2, 4, 6, 7, 8, 11, 13, 15, 16};
    const auto links = seam_links(geo_, back, 9);
    nfix_ = (long long)links.size();
    if (nfix_) {
      std::vector<long long> a(nfix_), b(nfix_);
      std::vector<int8_t> d(nfix_);
      for (long long k = 0; k < nfix_; ++k) {
        a[k] = (long long)geo_.idx(links[k].x, links[k].y, links[k].z);
        b[k] = (long long)geo_.idx(links[k].lx, links[k].ly, links[k].lz);
        d[k] = (int8_t)links[k].dir;
      }
      fa_.alloc(nfix_ * 8), fb_.alloc(nfix_ * 8), fd_.alloc(nfix_);
      CK(cudaMemcpyAsync(fa_.get(), a.data(), nfix_ * 8, cudaMemcpyHostToDevice, stream_));
      CK(cudaMemcpyAsync(fb_.get(), b.data(), nfix_ * 8, cudaMemcpyHostToDevice, stream_));
      CK(cudaMemcpyAsync(fd_.get(), d.data(), nfix_, cudaMemcpyHostToDevice, stream_));
    }
    alloc_field(f_, g.cells());
    init(base_init(kSrcRest));
    sync();
  }
  void fixup(const DField& f) {
    launch_swap_list(stream_, f, fa_.get<long long>(), fb_.get<long long>(), fd_.get<int8_t>(),
                     nfix_);
  }
  void step_one() override {
    const DField f = field(f_, soa_stride(geo_.cells()));
    if (pull_) {
      if (fresh_) {
        launch_local(stream_, f, f, L_, op_, false, false);
        fresh_ = false;
        return;
      }
      fixup(f);
      sweep(f, false);
    } else {
      if (pending_) {
        fixup(f);
        pending_ = false;
      }
      sweep(f, true);
      if (defer_ && nfix_)
        pending_ = true;
      else
        fixup(f);
    }
  }
  // all collisions then all swaps (push) / all swaps then all collisions
  // (pull): the swapped slot pairs are disjoint and independent of the
  // sweep's collisions, so this equals the sequential sweep bit for bit.
  void sweep(const DField& f, bool push) {
    if (push) {
      launch_local(stream_, f, f, L_, op_, true, false);
      launch_swap(stream_, f, L_, 1);
    } else {
      launch_swap(stream_, f, L_, 1);
      launch_local(stream_, f, f, L_, op_, true, false);
    }
  }
  int launches_per_step() const override { return 2 + (nfix_ ? 1 : 0); }
  void before_extract() override {
    if (!pull_ && pending_) fixup(field(f_, soa_stride(geo_.cells())));
  }
  void after_extract() override {
    if (!pull_ && pending_) fixup(field(f_, soa_stride(geo_.cells())));
  }
  void extract_range(uint32_t n0, uint32_t c, double* d) override {
    const DField f = field(f_, soa_stride(geo_.cells()));
    if (pull_)
      ex(f, L_, fresh_ ? kExNatural : kExGather, n0, c, d);
    else
      ex(f, L_, kExOpposed, n0, c, d);
  }
  void load_range(uint32_t n0, uint32_t c, const double* d, const InitSpec& in) override {
    ld(field(f_, soa_stride(geo_.cells())), L_, pull_ ? kExNatural : kExOpposed, n0, c, d, in);
  }
  void after_load() override {
    t_ = 0;
    fresh_ = pull_;
    pending_ = false;
  }
  int layout_phase() const override {
    if (pull_) return LBMGPU_NATURAL;
    return pending_ ? LBMGPU_SWAP_PARTIAL : LBMGPU_OPPOSED;
  }
  uint64_t pdf_bytes() const override { return f_.bytes(); }

 private:
  bool pull_, defer_;
  bool fresh_ = false, pending_ = false;
  long long nfix_ = 0;
  DevMem f_, fa_, fb_, fd_;
};

// ---------------------------------------------------------------------------
// indirect schemes: IDX built on the device (build_sparse restated)
// ---------------------------------------------------------------------------
class IndirectStepper : public Stepper {
 public:
  IndirectStepper(const HostGeo& g, const lbmgpu_flow& p, const lbmgpu_options& o)
      : Stepper(g, p, o) {
    if (nodes_ >= (uint64_t{1} << 31))
      throw std::runtime_error("fluid count exceeds 32-bit index range");
    adj_.alloc((size_t)nodes_ * 18 * sizeof(uint32_t));
    const dev::Lat L = make_lat(geo_, nullptr, 0, 0, 0, 0);
    Lcells_ = L;
    launch_adjacency(stream_, geo_.solids ? mask_d_.get<uint8_t>() : nullptr, L,
                     geo_.solids ? node_of_.get<uint32_t>() : nullptr, cell_of_node(),
                     (uint32_t)nodes_, adj_.get<uint32_t>());
    ck_launch();
    I_.adj = adj_.get<uint32_t>();
    I_.rem = nullptr;
    I_.n = (uint32_t)nodes_;
  }

 protected:
  void ex(const DField& f, int mode, uint32_t n0, uint32_t cnt, double* d,
          const EtBase& b = EtBase{}) {
    launch_extract_idx(stream_, f, I_, n0, cnt, mode, b, d);
  }
  void ld(const DField& f, int mode, uint32_t n0, uint32_t cnt, const double* d,
          const InitSpec& in) {
    launch_load_idx(stream_, f, I_, Lcells_, cell_of_node(), n0, cnt, mode, d, in);
  }
  uint64_t idx_bytes() const override { return adj_.bytes(); }
  DevMem adj_;
  Idx I_;
  dev::Lat Lcells_;
};

class TsIndirect final : public IndirectStepper {
 public:
  TsIndirect(const HostGeo& g, const lbmgpu_flow& p, const lbmgpu_options& o)
      : IndirectStepper(g, p, o) {
    alloc_field(a_, nodes_);
    alloc_field(b_, nodes_);
    init(base_init(kSrcRest));
  }
  void step_one() override {
    const long long s = soa_stride(nodes_);
    launch_local_idx(stream_, field(a_, s), field(b_, s), I_.n, op_, false, false);
    launch_ts_stream_idx(stream_, field(a_, s), field(b_, s), I_);
  }
  int launches_per_step() const override { return 2; }
  void extract_range(uint32_t n0, uint32_t c, double* d) override {
    ex(field(a_, soa_stride(nodes_)), kExNatural, n0, c, d);
  }
  void load_range(uint32_t n0, uint32_t c, const double* d, const InitSpec& in) override {
    ld(field(a_, soa_stride(nodes_)), kExNatural, n0, c, d, in);
  }
  uint64_t pdf_bytes() const override { return a_.bytes() + b_.bytes(); }

 private:
  DevMem a_, b_;
};

class OsIndirect final : public IndirectStepper {
 public:
  OsIndirect(const HostGeo& g, const lbmgpu_flow& p, const lbmgpu_options& o)
      : IndirectStepper(g, p, o) {
    const int s = o.scheme;
    pull_ = s != LBMGPU_OS_PUSH;
    nt_ = (s == LBMGPU_OSNT_PULL_1S || s == LBMGPU_OSNT_PULL_2S) && o.streaming_stores;
    two_s_ = s == LBMGPU_OSNT_PULL_2S;
    alloc_field(g_[0], nodes_);
    alloc_field(g_[1], nodes_);
    init(base_init(kSrcRest));
  }
  void step_one() override {
    const long long s = soa_stride(nodes_);
    DField a = field(g_[active_], s), b = field(g_[active_ ^ 1], s);
    if (pull_ && fresh_) {
      launch_local_idx(stream_, a, a, I_.n, op_, false, false);
      fresh_ = false;
    }
    if (pull_)
      launch_os_pull_idx(stream_, a, b, I_, op_, nt_, two_s_);
    else
      launch_os_push_idx(stream_, a, b, I_, op_);
    active_ ^= 1;
  }
  void extract_range(uint32_t n0, uint32_t c, double* d) override {
    const long long s = soa_stride(nodes_);
    if (!pull_ || fresh_)
      ex(field(g_[active_], s), kExNatural, n0, c, d);
    else
      ex(field(g_[active_ ^ 1], s), kExGather, n0, c, d);
  }
  void load_range(uint32_t n0, uint32_t c, const double* d, const InitSpec& in) override {
    ld(field(g_[active_], soa_stride(nodes_)), kExNatural, n0, c, d, in);
  }
  void after_load() override {
    t_ = 0;
    fresh_ = pull_;
  }
  uint64_t pdf_bytes() const override { return g_[0].bytes() + g_[1].bytes(); }

 private:
  bool pull_, nt_, two_s_;
  bool fresh_ = false;
  int active_ = 0;
  DevMem g_[2];
};

class AaIndirect final : public IndirectStepper {
 public:
  AaIndirect(const HostGeo& g, const lbmgpu_flow& p, const lbmgpu_options& o)
      : IndirectStepper(g, p, o) {
    alloc_field(f_, nodes_);
    init(base_init(kSrcRest));
  }
  void step_one() override {
    const DField f = field(f_, soa_stride(nodes_));
    if ((t_ & 1) == 0)
      launch_local_idx(stream_, f, f, I_.n, op_, false, true);
    else
      launch_aa_odd_idx(stream_, f, I_, op_);
  }
  void extract_range(uint32_t n0, uint32_t c, double* d) override {
    ex(field(f_, soa_stride(nodes_)), (t_ & 1) ? kExAaOdd : kExNatural, n0, c, d);
  }
  void load_range(uint32_t n0, uint32_t c, const double* d, const InitSpec& in) override {
    ld(field(f_, soa_stride(nodes_)), kExNatural, n0, c, d, in);
  }
  int layout_phase() const override { return (t_ & 1) ? LBMGPU_OPPOSED : LBMGPU_NATURAL; }
  uint64_t pdf_bytes() const override { return f_.bytes(); }

 private:
  DevMem f_;
};

class EtIndirect final : public IndirectStepper {
 public:
  EtIndirect(const HostGeo& g, const lbmgpu_flow& p, const lbmgpu_options& o)
      : IndirectStepper(g, p, o) {
    rem_.alloc((size_t)nodes_ * 9 * sizeof(uint32_t));
    {
      DevMem scratch(scan_scratch_elems(nodes_) * sizeof(uint32_t));
      nmail_ = build_et_rem(stream_, adj_.get<uint32_t>(), (uint32_t)nodes_, rem_.get<uint32_t>(),
                            scratch.get<uint32_t>(), 0);
    }
    I_.rem = rem_.get<uint32_t>();
    storage_ = nodes_ + nmail_;
    alloc_field(f_, storage_);
    reset_base();
    init(base_init(kSrcRest));
  }
  void step_one() override {
    launch_et_idx(stream_, field(f_, soa_stride(storage_)), I_, op_, base_);
    swap_base();
  }
  void extract_range(uint32_t n0, uint32_t c, double* d) override {
    ex(field(f_, soa_stride(storage_)), kExEt, n0, c, d, base_);
  }
  void load_range(uint32_t n0, uint32_t c, const double* d, const InitSpec& in) override {
    reset_base();
    ld(field(f_, soa_stride(storage_)), kExEt, n0, c, d, in);
  }
  bool exchange_opposite_handles() override {
    swap_base();
    return true;
  }
  int layout_phase() const override {
    for (int i = 0; i < 19; ++i)
      if (base_.b[i] != i) return LBMGPU_TWISTED;
    return LBMGPU_NATURAL;
  }
  uint64_t pdf_bytes() const override { return f_.bytes(); }
  uint64_t idx_bytes() const override { return adj_.bytes() + rem_.bytes(); }

 private:
  void reset_base() {
    for (int i = 0; i < 20; ++i) base_.b[i] = (int8_t)(i < 19 ? i : 0);
  }
  void swap_base() {
    for (int q = 0; q < 9; ++q) std::swap(base_.b[kPi[q]], base_.b[kPj[q]]);
  }
  uint32_t nmail_ = 0;
  uint64_t storage_ = 0;
  EtBase base_;
  DevMem rem_, f_;
};

class SwapIndirect final : public IndirectStepper {
 public:
  SwapIndirect(const HostGeo& g, const lbmgpu_flow& p, const lbmgpu_options& o)
      : IndirectStepper(g, p, o) {
    pull_ = o.scheme == LBMGPU_SWAP_PULL;
    alloc_field(f_, nodes_);
    init(base_init(kSrcRest));
  }
  void step_one() override {
    const DField f = field(f_, soa_stride(nodes_));
    if (pull_) {
      if (fresh_) {
        launch_local_idx(stream_, f, f, I_.n, op_, false, false);
        fresh_ = false;
      } else {
        launch_swap_idx(stream_, f, I_);
        launch_local_idx(stream_, f, f, I_.n, op_, true, false);
      }
    } else {
      launch_local_idx(stream_, f, f, I_.n, op_, true, false);
      launch_swap_idx(stream_, f, I_);
    }
  }
  int launches_per_step() const override { return 2; }
  void extract_range(uint32_t n0, uint32_t c, double* d) override {
    const DField f = field(f_, soa_stride(nodes_));
    if (pull_)
      ex(f, fresh_ ? kExNatural : kExGather, n0, c, d);
    else
      ex(f, kExOpposed, n0, c, d);
  }
  void load_range(uint32_t n0, uint32_t c, const double* d, const InitSpec& in) override {
    ld(field(f_, soa_stride(nodes_)), pull_ ? kExNatural : kExOpposed, n0, c, d, in);
  }
  void after_load() override {
    t_ = 0;
    fresh_ = pull_;
  }
  int layout_phase() const override { return pull_ ? LBMGPU_NATURAL : LBMGPU_OPPOSED; }
  uint64_t pdf_bytes() const override { return f_.bytes(); }

 private:
  bool pull_;
  bool fresh_ = false;
  DevMem f_;
};


// ---------------------------------------------------------------------------
// Multi-GPU z-slab decomposition of the AA pattern.
//
// A slab owns global planes [z0, z1) plus one ghost plane below and above
// (storage plane 0 and nzl+1). The even sweep is node-local. The odd sweep
// of a bottom-plane cell reads and rewrites exactly the cz = -1 slots
// {6,8,11,13,16} of the plane below it, and a top-plane cell the cz = +1
// slots {5,9,12,14,17} of the plane above (p/src/scheme_aap.cpp:133-173
// with X - c_i / X + c_j crossing the slab face). Within an odd sweep no one
// else touches those slots, so the exchange is: before the sweep copy the
// owners' face slots into the neighbours' ghosts, after it copy them back.
// The plan (order included) is one table used by every transport: NCCL
// (ncclSend/ncclRecv in one group per phase, over NVLink/NVSwitch), an
// in-process device-to-device transport (several slabs on one or more
// devices of one process), and the CPU gloo test (tests/test_slab_plan.py).
// ---------------------------------------------------------------------------
static constexpr int kZm[5] = {6, 8, 11, 13, 16};  // cz = -1
static constexpr int kZp[5] = {5, 9, 12, 14, 17};  // cz = +1

struct HaloOp {
  int phase;  // 0: before the odd sweep (owner -> ghost); 1: after it (ghost -> owner)
  int send;   // 1 send, 0 recv
  int peer;   // -1 lower neighbour (rank - 1), +1 upper neighbour (rank + 1), periodic ring
  int plane;  // local plane: -1 lower ghost, 0 bottom, nzl-1 top, nzl upper ghost
  int slot;   // direction slot (a whole nx*ny slot plane)
};

enum SlabKind {
  kSlabAA = 0,
  kSlabOsPull = 1,
  kSlabOsPush = 2,
  kSlabEt = 3,
  kSlabTs = 4,
  kSlabSwap = 5,
  kSlabCg = 6
};
// ET remote slots crossing a face (logical directions, mapped through the
// handle table base[] when executed): a top cell reads and rewrites the second
// members j of the pairs whose first member points up (5,9,12 -> 6,16,13) one
// plane above; a bottom cell those of the pairs pointing down (8,11 -> 17,14)
static constexpr int kEtUp[3] = {6, 16, 13};
static constexpr int kEtDown[2] = {17, 14};

// Exchange plan per scheme. phase 0 runs before a sweep, phase 1 after it.
//  AA (odd sweeps only): 0 = owners' face slots -> neighbours' ghosts (the
//     opposed slots the odd gather reads), 1 = ghosts -> owners
//  OS pull (every step, active grid): 0 = the slots the pull gathers across
//     the face (bottom cells read cz=+1 slots below, top cells cz=-1 above)
//  OS push (every step, destination grid): 1 = the slots pushed into the
//     ghosts (top cells push cz=+1 up, bottom cells cz=-1 down) -> owners
//  TS (every step, post-collision grid B between collide and stream): the
//     OS pull plan (the stream pass is a pull gather from B)
//  CG (every sweep, write frame): the OS push plan — a sweep's cross-face
//     pushes land in the write frame's padding planes (the single-domain
//     z-seam fix-up becomes this exchange)
//  SWAP (every swap pass): the pairs crossing a face are the bottom cells'
//     back links with cz=-1 against the lower neighbour's top-plane cz=+1
//     slots: 0 = those slots -> the lower ghost, 1 = swapped values -> owner
static std::vector<HaloOp> halo_plan(int kind, int nzl) {
  std::vector<HaloOp> v;
  auto add = [&](int ph, int send, int peer, int plane, const int* slots) {
    for (int k = 0; k < 5; ++k) v.push_back({ph, send, peer, plane, slots[k]});
  };
  if (kind == kSlabAA) {
    // phase 0: sends [up: top cz-] [down: bottom cz+]; recvs [down: lower ghost cz-] [up: upper ghost cz+]
    add(0, 1, +1, nzl - 1, kZm);
    add(0, 1, -1, 0, kZp);
    add(0, 0, -1, -1, kZm);
    add(0, 0, +1, nzl, kZp);
  }
  if (kind == kSlabOsPull || kind == kSlabTs) {
    // phase 0: sends [up: top cz+] [down: bottom cz-]; recvs [down: lower ghost cz+] [up: upper ghost cz-]
    add(0, 1, +1, nzl - 1, kZp);
    add(0, 1, -1, 0, kZm);
    add(0, 0, -1, -1, kZp);
    add(0, 0, +1, nzl, kZm);
  }
  if (kind == kSlabSwap) {
    add(0, 1, +1, nzl - 1, kZp);
    add(0, 0, -1, -1, kZp);
    add(1, 1, -1, -1, kZp);
    add(1, 0, +1, nzl - 1, kZp);
  }
  if (kind == kSlabEt) {
    // every sweep. phase 0: sends [up: top {17,14}] [down: bottom {6,16,13}];
    // recvs [down: lower ghost {17,14}] [up: upper ghost {6,16,13}]; phase 1 back
    auto addn = [&](int ph, int send, int peer, int plane, const int* slots, int n) {
      for (int k = 0; k < n; ++k) v.push_back({ph, send, peer, plane, slots[k]});
    };
    addn(0, 1, +1, nzl - 1, kEtDown, 2);
    addn(0, 1, -1, 0, kEtUp, 3);
    addn(0, 0, -1, -1, kEtDown, 2);
    addn(0, 0, +1, nzl, kEtUp, 3);
    addn(1, 1, -1, -1, kEtDown, 2);
    addn(1, 1, +1, nzl, kEtUp, 3);
    addn(1, 0, +1, nzl - 1, kEtDown, 2);
    addn(1, 0, -1, 0, kEtUp, 3);
  }
  if (kind == kSlabAA || kind == kSlabOsPush || kind == kSlabCg) {
    // phase 1: sends [down: lower ghost cz-] [up: upper ghost cz+]; recvs [up: top cz-] [down: bottom cz+]
    add(1, 1, -1, -1, kZm);
    add(1, 1, +1, nzl, kZp);
    add(1, 0, +1, nzl - 1, kZm);
    add(1, 0, -1, 0, kZp);
  }
  return v;
}
static std::vector<HaloOp> halo_plan(int nzl) { return halo_plan(kSlabAA, nzl); }

// NCCL, loaded on first use (dlopen) so processes that never decompose do not
// map it; inside a torch process this resolves to torch's libnccl.so.2.
#include <dlfcn.h>
#include <nccl.h>
struct Nccl {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
  static Nccl& get() {
    static Nccl n;
    if (!n.h) {
      n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!n.h) n.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
      if (!n.h) throw std::runtime_error(std::string("cannot load NCCL: ") + dlerror());
#define LBM_SYM(f, name)                                                    \
  n.f = reinterpret_cast<decltype(n.f)>(dlsym(n.h, name));                  \
  if (!n.f) throw std::runtime_error("NCCL symbol missing: " name);
      LBM_SYM(getUniqueId, "ncclGetUniqueId")
      LBM_SYM(commInitRank, "ncclCommInitRank")
      LBM_SYM(commDestroy, "ncclCommDestroy")
      LBM_SYM(send, "ncclSend")
      LBM_SYM(recv, "ncclRecv")
      LBM_SYM(groupStart, "ncclGroupStart")
      LBM_SYM(groupEnd, "ncclGroupEnd")
      LBM_SYM(errStr, "ncclGetErrorString")
#undef LBM_SYM
    }
    return n;
  }
  void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw CudaError(std::string("nccl: ") + what + ": " + errStr(r));
  }
};

class SlabStepper final : public Stepper {
 public:
  SlabStepper(const HostGeo& g, const lbmgpu_flow& p, const lbmgpu_options& o)
      : Stepper(slab_geo(g, o), p, o), gnz_(g.nz), z0_(o.z_begin), z1_(o.z_end) {
    kind_ = o.scheme == LBMGPU_AAP    ? kSlabAA
            : o.scheme == LBMGPU_ET   ? kSlabEt
            : o.scheme == LBMGPU_TS   ? kSlabTs
            : (o.scheme == LBMGPU_SWAP_PUSH || o.scheme == LBMGPU_SWAP_PULL) ? kSlabSwap
            : o.scheme == LBMGPU_CG   ? kSlabCg
            : o.scheme == LBMGPU_OS_PUSH ? kSlabOsPush
                                         : kSlabOsPull;
    for (int i = 0; i < 20; ++i) base_.b[i] = (int8_t)(i < 19 ? i : 0);
    nt_ = (o.scheme == LBMGPU_OSNT_PULL_1S || o.scheme == LBMGPU_OSNT_PULL_2S) && o.streaming_stores;
    swap_pull_ = o.scheme == LBMGPU_SWAP_PULL;
    two_s_ = o.scheme == LBMGPU_OSNT_PULL_2S;
    nzl_ = z1_ - z0_;
    plane_ = (uint64_t)g.nx * g.ny;
    idx_ = o.addressing == LBMGPU_INDIRECT;
    if (idx_) {
      // geo_ is the slab plus one ghost plane per face (slab_geo); its fluid
      // nodes in x-fastest order are [lower ghost | own planes | upper ghost]
      poff_.assign((size_t)nzl_ + 3, 0);
      for (int k = 0; k < nzl_ + 2; ++k) {
        uint64_t c = plane_;
        if (geo_.solids) {
          c = 0;
          for (uint64_t q = 0; q < plane_; ++q) c += geo_.mask[(uint64_t)k * plane_ + q] ? 1 : 0;
        }
        poff_[k + 1] = poff_[k] + c;
      }
      if (nodes_ >= (uint64_t{1} << 31))
        throw std::runtime_error("fluid count exceeds 32-bit index range");
      storage_ = nodes_;
      adj_.alloc((size_t)nodes_ * 18 * sizeof(uint32_t));
      Lcells_ = make_lat(geo_, nullptr, 0, 0, 0, 0);
      launch_adjacency(stream_, geo_.solids ? mask_d_.get<uint8_t>() : nullptr, Lcells_,
                       geo_.solids ? node_of_.get<uint32_t>() : nullptr, cell_of_node(),
                       (uint32_t)nodes_, adj_.get<uint32_t>());
      ck_launch();
      I_.adj = adj_.get<uint32_t>();
      I_.rem = nullptr;
      I_.n = (uint32_t)nodes_;
      if (kind_ == kSlabEt) {
        // ET remote table over the extended numbering; bounced links get
        // mailbox slots after all nodes, touched only by their own node
        rem_.alloc((size_t)nodes_ * 9 * sizeof(uint32_t));
        DevMem scratch(scan_scratch_elems(nodes_) * sizeof(uint32_t));
        const uint32_t nmail = build_et_rem(stream_, adj_.get<uint32_t>(), (uint32_t)nodes_,
                                            rem_.get<uint32_t>(), scratch.get<uint32_t>(), 0);
        I_.rem = rem_.get<uint32_t>();
        storage_ = nodes_ + nmail;
      }
    } else {
      L_ = make_lat(geo_, nullptr, 0, 0, 0, 0);
      L_.zghost = 1;
      L_.oz = 1;
      L_.wall[2] = 0;
      storage_ = plane_ * (nzl_ + 2);
      if (kind_ == kSlabCg) {  // CgDirect's layout over the slab: nzl + S + 2 planes
        cg_p_ = std::min(std::max(16, std::min(64, nzl_ / 4)), nzl_);
        cg_s_ = cg_p_ + 1;
        storage_ = plane_ * (uint64_t)(nzl_ + cg_s_ + 2);
        if (storage_ >= (uint64_t{1} << 32))
          throw std::runtime_error("grid exceeds 32-bit cell index range");
      }
    }
    ngrids_ = (kind_ == kSlabAA || kind_ == kSlabEt || kind_ == kSlabSwap || kind_ == kSlabCg) ? 1
                                                                                            : 2;
    for (int k = 0; k < ngrids_; ++k) alloc_field(g_[k], storage_);
    // an owner node whose link towards the neighbour slab bounces (x/y wall,
    // solid) writes that face slot itself: phase 1 then merges, not copies
    // (SWAP: a face pair exists only between two fluid nodes, so the returned
    // values are always the swapped ones: plain copies)
    merge_ = kind_ != kSlabSwap &&
             (geo_.policy[0] == 1 || geo_.policy[1] == 1 || (idx_ && geo_.solids));
    if (merge_) {
      maxcount_ = 0;
      for (int pl : {0, nzl_ - 1}) maxcount_ = std::max(maxcount_, plane_count(pl));
      rbuf_.alloc(std::max<uint64_t>(1, maxcount_) * 10 * esize());
    }
    CK(cudaStreamCreateWithFlags(&comm_, cudaStreamNonBlocking));
    for (auto* e : {&ev_c_, &ev_halo_, &ev_odd_, &ev_back_})
      CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    CK(cudaEventRecord(ev_back_, comm_));
    init(base_init(kSrcRest));
  }
  ~SlabStepper() override {
    if (stream_) cudaStreamSynchronize(stream_);
    if (comm_) {
      cudaStreamSynchronize(comm_);
      cudaStreamDestroy(comm_);
    }
    for (auto e : {ev_c_, ev_halo_, ev_odd_, ev_back_})
      if (e) cudaEventDestroy(e);
    if (nccl_) Nccl::get().commDestroy(nccl_);
  }

  static HostGeo slab_geo(const HostGeo& g, const lbmgpu_options& o) {
    const bool ok_scheme = o.scheme == LBMGPU_AAP || o.scheme == LBMGPU_ET || o.scheme == LBMGPU_TS ||
                           o.scheme == LBMGPU_SWAP_PUSH || o.scheme == LBMGPU_SWAP_PULL ||
                           o.scheme == LBMGPU_CG || o.scheme == LBMGPU_OS_PUSH ||
                           o.scheme == LBMGPU_OS_PULL || o.scheme == LBMGPU_OSNT_PULL_1S ||
                           o.scheme == LBMGPU_OSNT_PULL_2S;
    const bool idx = o.addressing == LBMGPU_INDIRECT;
    if (!ok_scheme || o.layout != LBMGPU_SOA)
      throw std::invalid_argument(
          "z-slab decomposition supports every scheme (CG direct only), SoA");
    if ((o.scheme == LBMGPU_SWAP_PUSH || o.scheme == LBMGPU_SWAP_PULL) && o.swap_deferred_fixup)
      throw std::invalid_argument("SWAP z-slabs swap every link each sweep (swap_deferred_fixup = 0)");
    if (g.solids && !idx)
      throw std::invalid_argument("z-slab decomposition needs an all-fluid box (direct)");
    if (g.policy[2] != 0) throw std::invalid_argument("z-slab decomposition needs periodic z");
    if (o.scheme == LBMGPU_ET && (g.policy[0] != 0 || g.policy[1] != 0))
      throw std::invalid_argument("ET z-slabs need periodic x and y (no mailbox halo)");
    if (o.z_begin < 0 || o.z_end > g.nz || o.z_end <= o.z_begin)
      throw std::invalid_argument("z-slab range must satisfy 0 <= z_begin < z_end <= nz");
    HostGeo s = g;
    const int nzl = o.z_end - o.z_begin;
    if (!idx) {
      s.nz = nzl;
      return s;
    }
    // indirect: planes z_begin-1 .. z_end (wrapped) with a wall policy in z,
    // so build_sparse links own nodes to the ghost planes and never wraps
    s.nz = nzl + 2;
    s.policy[2] = 1;
    if (g.solids) {
      const uint64_t pl = (uint64_t)g.nx * g.ny;
      s.mask.assign(pl * (uint64_t)(nzl + 2), 0);
      for (int k = 0; k < nzl + 2; ++k) {
        const int gz = ((o.z_begin - 1 + k) % g.nz + g.nz) % g.nz;
        std::copy(g.mask.begin() + (size_t)(gz * pl), g.mask.begin() + (size_t)((gz + 1) * pl),
                  s.mask.begin() + (size_t)(k * pl));
      }
    }
    return s;
  }

  InitSpec slab_init(int source) const {
    InitSpec s = base_init(source);
    s.gnz = gnz_;
    s.z0 = z0_;
    return s;
  }

  // ---- transports ----------------------------------------------------------
  void connect_nccl(const ncclUniqueId& id, int nranks, int rank) {
    CK(cudaSetDevice(opt_.device));
    Nccl& N = Nccl::get();
    if (nccl_) N.commDestroy(nccl_), nccl_ = nullptr;
    N.check(N.commInitRank(&nccl_, nranks, id, rank), "ncclCommInitRank");
    nranks_ = nranks, rank_ = rank;
    transport_ = kNccl;
  }
  void set_local(int transport) { transport_ = transport; }

  // the grid an exchange phase applies to: AA its one grid; OS pull the
  // active grid (read by the coming pull); OS push the grid just written
  int phase_grid(int phase) const {
    if (kind_ == kSlabAA || kind_ == kSlabEt || kind_ == kSlabSwap || kind_ == kSlabCg) return 0;
    if (kind_ == kSlabTs) return 1;  // B, the post-collision grid the stream reads
    if (kind_ == kSlabOsPull) return active_;
    return phase == 1 ? active_ ^ 1 : active_;
  }
  // local plane -1 .. nzl (ghost planes -1 and nzl): direct, storage plane
  // + 1; indirect, the plane's node range of the extended numbering
  // (CG: planes of the current exchange frame, zoff_ = its origin)
  uint64_t plane_first(int plane) const {
    return idx_ ? poff_[plane + 1] : (uint64_t)(plane + 1 + zoff_) * plane_;
  }
  uint64_t plane_count(int plane) const {
    return idx_ ? poff_[plane + 2] - poff_[plane + 1] : plane_;
  }
  void* slot_ptr(int grid, int slot, int plane) const {
    return static_cast<char*>(g_[grid].get()) +
           ((size_t)slot * soa_stride(storage_) + plane_first(plane)) * esize();
  }
  uint64_t snapshot_nodes() const override {
    return idx_ ? poff_[nzl_ + 1] - poff_[1] : nodes_;
  }
  uint64_t idx_bytes() const override { return adj_.bytes() + rem_.bytes(); }
  size_t elem_bytes() const { return esize(); }
  // storage plane of a logical slot (ET: through the handle table)
  int phys_slot(int slot) const { return kind_ == kSlabEt ? base_.b[slot] : slot; }
  void swap_base() {
    for (int q = 0; q < 9; ++q) std::swap(base_.b[kPi[q]], base_.b[kPj[q]]);
  }

  // phase-1 receive into an owner plane that must be merged (see merge_)
  bool merged(const HaloOp& op) const { return merge_ && op.phase == 1 && !op.send; }
  void* rbuf_slot(int q) const { return static_cast<char*>(rbuf_.get()) + (size_t)q * maxcount_ * esize(); }
  // the link of the owner node pointing at the slot's writer in the other
  // slab: AA / OS push slot k is written by R - c_k; ET slot j by R + c_j
  int merge_dir(const HaloOp& op) const { return kind_ == kSlabEt ? op.slot : dev::opp(op.slot); }
  void merge_into(cudaStream_t st, int grid, const HaloOp& op, const void* src) {
    launch_slab_merge(st, prec_, slot_ptr(grid, phys_slot(op.slot), op.plane), src,
                      (uint32_t)plane_count(op.plane), merge_dir(op), (uint32_t)plane_first(op.plane),
                      idx_ ? I_.adj : nullptr, idx_ ? I_.n : 0u, geo_.nx, geo_.ny,
                      geo_.policy[0] == 1, geo_.policy[1] == 1);
  }

  // NCCL phase: the plan's sends and receives in plan order, one group
  // the plan that refreshes the ghosts an extraction gathers from (SWAP pull
  // gathers like OS pull)
  int sync_kind() const { return kind_ == kSlabSwap ? kSlabOsPull : kind_; }
  void nccl_phase(int phase, int grid, int plan_kind = -1) {
    Nccl& N = Nccl::get();
    const ncclDataType_t ty = prec_ == Prec::f64 ? ncclDouble : ncclFloat;
    const std::vector<HaloOp> plan = halo_plan(plan_kind < 0 ? kind_ : plan_kind, nzl_);
    N.check(N.groupStart(), "ncclGroupStart");
    int q = 0;
    for (const HaloOp& op : plan) {
      if (op.phase != phase) continue;
      const int peer = (rank_ + op.peer + nranks_) % nranks_;
      void* p = merged(op) ? rbuf_slot(q++) : slot_ptr(grid, phys_slot(op.slot), op.plane);
      const size_t cnt = plane_count(op.plane);
      if (op.send)
        N.check(N.send(p, cnt, ty, peer, nccl_, comm_), "ncclSend");
      else
        N.check(N.recv(p, cnt, ty, peer, nccl_, comm_), "ncclRecv");
    }
    N.check(N.groupEnd(), "ncclGroupEnd");
    q = 0;
    for (const HaloOp& op : plan)
      if (op.phase == phase && merged(op)) merge_into(comm_, grid, op, rbuf_slot(q++));
  }
  // comm stream runs `phase` after everything enqueued on stream_ so far
  void enqueue_phase(int phase, int grid, cudaEvent_t done, int plan_kind = -1) {
    CK(cudaEventRecord(ev_c_, stream_));
    CK(cudaStreamWaitEvent(comm_, ev_c_, 0));
    nccl_phase(phase, grid, plan_kind);
    CK(cudaEventRecord(done, comm_));
  }

  dev::Lat planes(int za, int zb) const {  // local planes [za, zb)
    dev::Lat L = L_;
    L.cell_begin = (uint32_t)(za * plane_);
    L.ncells = (uint32_t)(zb * plane_);
    return L;
  }

  // one sweep of the scheme's kernel over local planes [za, zb)
  void sweep(int za, int zb) {
    if (zb <= za) return;
    const long long st = soa_stride(storage_);
    if (idx_) {
      Idx I = I_;
      I.first = (uint32_t)poff_[za + 1];
      I.last = (uint32_t)poff_[zb + 1];
      if (kind_ == kSlabAA) {
        const DField f = field(g_[0], st);
        if ((t_ & 1) == 0)
          launch_local_idx_range(stream_, f, f, I.first, I.last, op_, false, true);
        else
          launch_aa_odd_idx(stream_, f, I, op_);
      } else if (kind_ == kSlabTs) {
        launch_ts_stream_idx(stream_, field(g_[0], st), field(g_[1], st), I);
      } else if (kind_ == kSlabEt) {
        launch_et_idx(stream_, field(g_[0], st), I, op_, base_);
      } else if (kind_ == kSlabSwap) {
        launch_swap_idx(stream_, field(g_[0], st), I);
      } else {
        const DField a = field(g_[active_], st), b = field(g_[active_ ^ 1], st);
        if (kind_ == kSlabOsPull)
          launch_os_pull_idx(stream_, a, b, I, op_, nt_, two_s_);
        else
          launch_os_push_idx(stream_, a, b, I, op_);
      }
      return;
    }
    const dev::Lat L = planes(za, zb);
    if (kind_ == kSlabAA) {
      const DField f = field(g_[0], st);
      if ((t_ & 1) == 0)
        launch_local(stream_, f, f, L, op_, false, true);
      else
        launch_aa_odd(stream_, f, L, op_);
    } else if (kind_ == kSlabEt) {
      launch_et(stream_, field(g_[0], st), L, op_, base_);
    } else if (kind_ == kSlabTs) {
      launch_ts_stream(stream_, field(g_[0], st), field(g_[1], st), L);
    } else if (kind_ == kSlabSwap) {
      launch_swap(stream_, field(g_[0], st), L, 0);  // z never wraps inside a slab
    } else {
      const DField a = field(g_[active_], st), b = field(g_[active_ ^ 1], st);
      if (kind_ == kSlabOsPull)
        launch_os_pull(stream_, a, b, L, op_, nt_, two_s_);
      else
        launch_os_push(stream_, a, b, L, op_);
    }
  }
  // the interior planes never touch ghost planes or exchanged face slots
  void sweep_split(cudaEvent_t wait_before_boundary) {
    const int zi0 = 1, zi1 = std::max(1, nzl_ - 1);
    sweep(zi0, zi1);
    CK(cudaStreamWaitEvent(stream_, wait_before_boundary, 0));
    sweep(0, 1);
    if (nzl_ > 1) sweep(nzl_ - 1, nzl_);
  }

  // CG (CgDirect over the slab): frame(origin) addresses plane z at storage
  // z + 1 + origin; a sweep is a sequence of plane-group push launches from
  // the read origin to the write origin; the pushes across the slab faces land
  // in the write frame's padding planes, which phase 1 delivers
  dev::Lat cg_frame(int origin) const {
    dev::Lat L = L_;
    L.zghost = 0;
    L.oz = 1 + origin;
    L.znowrap = 1;
    return L;
  }
  void cg_sweep() {
    const DField f = field(g_[0], soa_stride(storage_));
    const bool even = (t_ & 1) == 0;
    const int R = even ? cg_s_ : 0, W = even ? 0 : cg_s_;
    const int ngroups = (nzl_ + cg_p_ - 1) / cg_p_;
    for (int k = 0; k < ngroups; ++k) {
      const int gi = even ? k : ngroups - 1 - k;
      dev::Lat L = cg_frame(R);
      L.cell_begin = (uint32_t)(gi * cg_p_ * plane_);
      L.ncells = (uint32_t)(std::min(nzl_, (gi + 1) * cg_p_) * plane_);
      launch_cg_push(stream_, f, L, op_, (W - R) * (int)plane_);
    }
    cg_w_ = W;
  }

  // TS collide sweep A -> B over the own planes (p/src/scheme_ts.cpp:59-80)
  void ts_collide() {
    const long long st = soa_stride(storage_);
    const DField a = field(g_[0], st), b = field(g_[1], st);
    if (idx_)
      launch_local_idx_range(stream_, a, b, (uint32_t)poff_[1], (uint32_t)poff_[nzl_ + 1], op_,
                             false, false);
    else
      launch_local(stream_, a, b, planes(0, nzl_), op_, false, false);
  }

  // SWAP collide pass: opposed slots in, natural out (push: before the swaps;
  // pull: after them); the first pull step only precollides (natural in place)
  void swap_collide(bool first_pull = false) {
    const long long st = soa_stride(storage_);
    const DField f = field(g_[0], st);
    if (idx_)
      launch_local_idx_range(stream_, f, f, (uint32_t)poff_[1], (uint32_t)poff_[nzl_ + 1], op_,
                             !first_pull, false);
    else
      launch_local(stream_, f, f, planes(0, nzl_), op_, !first_pull, false);
  }

  void precollide_if_fresh() {
    if (kind_ == kSlabOsPull && fresh_) {
      const DField a = field(g_[active_], soa_stride(storage_));
      if (idx_)
        launch_local_idx_range(stream_, a, a, (uint32_t)poff_[1], (uint32_t)poff_[nzl_ + 1], op_,
                               false, false);
      else
        launch_local(stream_, a, a, planes(0, nzl_), op_, false, false);
      fresh_ = false;
    }
  }

  void step_one() override {
    if (transport_ == kNccl) {
      if (kind_ == kSlabEt) {
        if (owners_stale_) {  // values a load parked in the ghosts -> owners
          enqueue_phase(1, 0, ev_back_);
          owners_stale_ = false;
        }
        enqueue_phase(0, 0, ev_halo_);
        sweep_split(ev_halo_);
        enqueue_phase(1, 0, ev_back_);
        swap_base();
      } else if (kind_ == kSlabAA) {
        if ((t_ & 1) == 0) {
          sweep_split(ev_back_);
        } else {
          enqueue_phase(0, 0, ev_halo_);
          sweep_split(ev_halo_);
          enqueue_phase(1, 0, ev_back_);
        }
      } else if (kind_ == kSlabOsPull) {
        precollide_if_fresh();
        enqueue_phase(0, active_, ev_halo_);
        sweep_split(ev_halo_);
        active_ ^= 1;
      } else if (kind_ == kSlabTs) {
        ts_collide();
        enqueue_phase(0, 1, ev_halo_);
        sweep_split(ev_halo_);
      } else if (kind_ == kSlabCg) {
        CK(cudaStreamWaitEvent(stream_, ev_back_, 0));  // my read frame got its face values
        cg_sweep();
        zoff_ = cg_w_;
        enqueue_phase(1, 0, ev_back_);
        zoff_ = 0;
      } else if (kind_ == kSlabSwap) {
        CK(cudaStreamWaitEvent(stream_, ev_back_, 0));  // last phase 1 reached my top plane
        if (swap_pull_ && fresh_) {
          swap_collide(true);
          fresh_ = false;
        } else {
          if (!swap_pull_) swap_collide();
          enqueue_phase(0, 0, ev_halo_);
          sweep_split(ev_halo_);
          enqueue_phase(1, 0, ev_back_);
          if (swap_pull_) {
            CK(cudaStreamWaitEvent(stream_, ev_back_, 0));
            swap_collide();
          }
        }
      } else {  // push: interior and boundary, then ghosts -> owners of the new grid
        sweep_split(ev_back_);
        enqueue_phase(1, active_ ^ 1, ev_back_);
        active_ ^= 1;
      }
      ghosts_fresh_ = false;
      return;
    }
    if (transport_ != kLocalGroup)
      throw std::runtime_error("slab stepper has no transport: connect NCCL or step as a group");
    // in-process group: group_step runs the exchange phases around the sweep
    if (kind_ == kSlabSwap && swap_pull_ && fresh_) {
      swap_collide(true);
      fresh_ = false;
      return;
    }
    if (kind_ == kSlabCg) {
      cg_sweep();
      return;
    }
    sweep(0, nzl_);
    if (kind_ == kSlabEt)
      swap_base();
    else if (kind_ == kSlabOsPull || kind_ == kSlabOsPush)
      active_ ^= 1;
  }
  int launches_per_step() const override {
    if (kind_ == kSlabCg) return (nzl_ + cg_p_ - 1) / cg_p_;
    const int collide = (kind_ == kSlabTs || kind_ == kSlabSwap) ? 1 : 0;
    if (transport_ != kNccl) return 1 + collide;
    return (nzl_ > 2 ? 3 : nzl_) + collide;
  }

  void finish() override {
    if (transport_ == kNccl) CK(cudaStreamWaitEvent(stream_, ev_back_, 0));
  }

  // ghost planes the extraction gathers from: AA at odd t, OS pull once it
  // streams the idle grid (phase-0 slot set applied to that grid)
  bool extract_needs_ghosts() const {
    if (kind_ == kSlabAA) return (t_ & 1) != 0;
    if (kind_ == kSlabSwap) return swap_pull_ && !fresh_;
    if (kind_ == kSlabEt) return true;
    if (kind_ == kSlabOsPull) return !fresh_;
    return false;
  }
  int ghost_grid() const { return kind_ == kSlabOsPull ? active_ ^ 1 : 0; }

  void sync_ghosts_nccl() {
    if (transport_ != kNccl) throw std::runtime_error("slab stepper is not connected to NCCL");
    enqueue_phase(0, ghost_grid(), ev_halo_, sync_kind());
    CK(cudaStreamWaitEvent(stream_, ev_halo_, 0));
    ghosts_fresh_ = true;
  }

  void before_extract() override {
    if (extract_needs_ghosts() && !ghosts_fresh_)
      throw std::runtime_error(
          "slab extract reads the ghost planes at this time step: call "
          "lbmgpu_slab_sync_ghosts (or the group variant) first");
  }
  void extract_range(uint32_t n0, uint32_t c, double* d) override {
    const long long st = soa_stride(storage_);
    if (idx_) {
      const uint32_t n = (uint32_t)poff_[1] + n0;
      if (kind_ == kSlabAA)
        launch_extract_idx(stream_, field(g_[0], st), I_, n, c, (t_ & 1) ? kExAaOdd : kExNatural,
                           EtBase{}, d);
      else if (kind_ == kSlabSwap)
        launch_extract_idx(stream_, field(g_[0], st), I_, n, c,
                           !swap_pull_ ? kExOpposed : (fresh_ ? kExNatural : kExGather), EtBase{},
                           d);
      else if (kind_ == kSlabEt)
        launch_extract_idx(stream_, field(g_[0], st), I_, n, c, kExEt, base_, d);
      else if (kind_ == kSlabOsPull && !fresh_)
        launch_extract_idx(stream_, field(g_[active_ ^ 1], st), I_, n, c, kExGather, EtBase{}, d);
      else
        launch_extract_idx(stream_, field(g_[active_], st), I_, n, c, kExNatural, EtBase{}, d);
      return;
    }
    if (kind_ == kSlabAA)
      launch_extract(stream_, field(g_[0], st), L_, nullptr, n0, c,
                     (t_ & 1) ? kExAaOdd : kExNatural, EtBase{}, d);
    else if (kind_ == kSlabSwap)
      launch_extract(stream_, field(g_[0], st), L_, nullptr, n0, c,
                     !swap_pull_ ? kExOpposed : (fresh_ ? kExNatural : kExGather), EtBase{}, d);
    else if (kind_ == kSlabCg)
      launch_extract(stream_, field(g_[0], st), cg_frame((t_ & 1) ? 0 : cg_s_), nullptr, n0, c,
                     kExNatural, EtBase{}, d);
    else if (kind_ == kSlabEt)
      launch_extract(stream_, field(g_[0], st), L_, nullptr, n0, c, kExEt, base_, d);
    else if (kind_ == kSlabOsPull && !fresh_)
      launch_extract(stream_, field(g_[active_ ^ 1], st), L_, nullptr, n0, c, kExGather,
                     EtBase{}, d);
    else
      launch_extract(stream_, field(g_[active_], st), L_, nullptr, n0, c, kExNatural,
                     EtBase{}, d);
  }
  void load_range(uint32_t n0, uint32_t c, const double* d, const InitSpec& in) override {
    InitSpec s = in;
    if (s.source != kSrcBuffer) s.gnz = gnz_, s.z0 = z0_;
    if (idx_) {
      s.z0 = z0_ - 1;  // extended plane 0 is global plane z_begin - 1
      int mode = (kind_ == kSlabSwap && !swap_pull_) ? kExOpposed : kExNatural;
      if (kind_ == kSlabEt) {
        for (int i = 0; i < 20; ++i) base_.b[i] = (int8_t)(i < 19 ? i : 0);
        mode = kExEt;
      }
      launch_load_idx(stream_, field(g_[active_], soa_stride(storage_)), I_, Lcells_,
                      cell_of_node(), (uint32_t)poff_[1] + n0, c, mode, d, s);
      return;
    }
    if (kind_ == kSlabEt) {
      for (int i = 0; i < 20; ++i) base_.b[i] = (int8_t)(i < 19 ? i : 0);
      launch_load(stream_, field(g_[0], soa_stride(storage_)), L_, nullptr, n0, c, kExEt, d, s);
      return;
    }
    launch_load(stream_, field(g_[active_], soa_stride(storage_)),
                kind_ == kSlabCg ? cg_frame(cg_s_) : L_, nullptr, n0, c,
                (kind_ == kSlabSwap && !swap_pull_) ? kExOpposed : kExNatural, d, s);
  }
  void after_load() override {
    t_ = 0;
    fresh_ = kind_ == kSlabOsPull || (kind_ == kSlabSwap && swap_pull_);
    // ET's load writes the remote slots of the boundary cells into the ghost
    // planes: they are fresh, and their owners get them before the first sweep
    ghosts_fresh_ = kind_ == kSlabEt;
    owners_stale_ = kind_ == kSlabEt;
  }
  bool exchange_opposite_handles() override {
    if (kind_ != kSlabEt) return false;
    swap_base();
    return true;
  }
  int layout_phase() const override {
    if (kind_ == kSlabEt) {
      for (int i = 0; i < 19; ++i)
        if (base_.b[i] != i) return LBMGPU_TWISTED;
      return LBMGPU_NATURAL;
    }
    if (kind_ == kSlabSwap) return swap_pull_ ? LBMGPU_NATURAL : LBMGPU_OPPOSED;
    if (kind_ == kSlabCg) return (t_ & 1) ? LBMGPU_SHIFTED_EVEN : LBMGPU_SHIFTED_ODD;
    return (kind_ == kSlabAA && (t_ & 1)) ? LBMGPU_OPPOSED : LBMGPU_NATURAL;
  }
  uint64_t pdf_bytes() const override { return g_[0].bytes() + g_[1].bytes(); }

  enum { kNone = 0, kLocalGroup = 1, kNccl = 2 };
  int kind_ = kSlabAA;
  int transport_ = kNone;
  int nzl_ = 0, gnz_ = 0, z0_ = 0, z1_ = 0;
  int ngrids_ = 1, active_ = 0;
  bool nt_ = false, two_s_ = false, fresh_ = false, swap_pull_ = false;
  int cg_p_ = 1, cg_s_ = 2, cg_w_ = 0, zoff_ = 0;
  bool ghosts_fresh_ = false, owners_stale_ = false;
  EtBase base_;
  bool idx_ = false;
  bool merge_ = false;
  uint64_t maxcount_ = 0;
  DevMem rbuf_;
  std::vector<uint64_t> poff_;  // indirect: node offset of extended plane k
  DevMem adj_, rem_;
  Idx I_{};
  dev::Lat Lcells_{};
  uint64_t plane_ = 0, storage_ = 0;
  dev::Lat L_;
  DevMem g_[2];
  cudaStream_t comm_ = nullptr;
  cudaEvent_t ev_c_ = nullptr, ev_halo_ = nullptr, ev_odd_ = nullptr, ev_back_ = nullptr;
  ncclComm_t nccl_ = nullptr;
  int nranks_ = 1, rank_ = 0;
};

// In-process transport: executes one plan phase for a ring of slabs (rank k
// = slab k) by matching each rank's sends with its peer's receives in plan
// order — NCCL's point-to-point matching rule — as device-to-device copies.
static void local_phase(std::vector<SlabStepper*>& S, int phase, bool use_ghost_grid = false) {
  const int n = (int)S.size();
  for (auto* s : S) s->sync();
  std::vector<std::vector<HaloOp>> plans(n);
  for (int k = 0; k < n; ++k)
    plans[k] = halo_plan(use_ghost_grid ? S[k]->sync_kind() : S[k]->kind_, S[k]->nzl_);
  // receives that merge: (peer, op, scratch slot) applied after all copies
  struct Pending {
    int peer;
    HaloOp op;
    int q;
  };
  std::vector<Pending> pend;
  std::vector<int> nq(n, 0);
  for (int k = 0; k < n; ++k) {
    std::vector<size_t> cursor(n, 0);
    const int gk = use_ghost_grid ? S[k]->ghost_grid() : S[k]->phase_grid(phase);
    for (const HaloOp& op : plans[k]) {
      if (op.phase != phase || !op.send) continue;
      const int peer = (k + op.peer + n) % n;
      // the next receive the peer posts from rank k in this phase
      size_t& c = cursor[peer];
      const std::vector<HaloOp>& pp = plans[peer];
      for (; c < pp.size(); ++c) {
        const HaloOp& r = pp[c];
        if (r.phase == phase && !r.send && (peer + r.peer + n) % n == k) break;
      }
      if (c == pp.size()) throw std::runtime_error("halo plan: unmatched send");
      const HaloOp& r = pp[c++];
      const int gp = use_ghost_grid ? S[peer]->ghost_grid() : S[peer]->phase_grid(phase);
      const uint64_t cnt = S[k]->plane_count(op.plane);
      if (cnt != S[peer]->plane_count(r.plane))
        throw std::runtime_error("halo plan: message sizes differ between neighbours");
      void* dst = S[peer]->slot_ptr(gp, S[peer]->phys_slot(r.slot), r.plane);
      if (S[peer]->merged(r)) {
        dst = S[peer]->rbuf_slot(nq[peer]);
        pend.push_back({peer, r, nq[peer]++});
      }
      CK(cudaMemcpyPeerAsync(dst, S[peer]->opt_.device,
                             S[k]->slot_ptr(gk, S[k]->phys_slot(op.slot), op.plane),
                             S[k]->opt_.device, cnt * S[k]->elem_bytes(), S[k]->stream_));
    }
  }
  for (auto* s : S) s->sync();
  for (const Pending& m : pend) {
    SlabStepper* R = S[m.peer];
    CK(cudaSetDevice(R->opt_.device));
    const int g = use_ghost_grid ? R->ghost_grid() : R->phase_grid(phase);
    R->merge_into(R->stream_, g, m.op, R->rbuf_slot(m.q));
  }
  for (auto* s : S) s->sync();
}

static void group_step(std::vector<SlabStepper*>& S, long long steps) {
  for (auto* s : S) {
    if (s->transport_ == SlabStepper::kNccl) throw std::invalid_argument("slab is NCCL-connected");
    if (s->kind_ != S[0]->kind_) throw std::invalid_argument("slabs of different schemes");
    s->set_local(SlabStepper::kLocalGroup);
  }
  const int kind = S[0]->kind_;
  for (long long k = 0; k < steps; ++k) {
    const bool odd = (S[0]->t_ & 1) != 0;
    for (auto* s : S)
      if (((s->t_ & 1) != 0) != odd) throw std::invalid_argument("slabs out of step");
    if (kind == kSlabCg) {
      for (auto* s : S) s->step(1);  // the plane-group sweep
      for (auto* s : S) s->zoff_ = s->cg_w_;
      local_phase(S, 1);
      for (auto* s : S) s->zoff_ = 0;
      continue;
    }
    if (kind == kSlabSwap) {
      const bool fresh = S[0]->swap_pull_ && S[0]->fresh_;
      if (!fresh && !S[0]->swap_pull_)
        for (auto* s : S) s->swap_collide();
      if (!fresh) local_phase(S, 0);
      for (auto* s : S) s->step(1);  // the swap pass (first pull step: precollide)
      if (!fresh) {
        local_phase(S, 1);
        if (S[0]->swap_pull_)
          for (auto* s : S) s->swap_collide();
      }
      for (auto* s : S) s->ghosts_fresh_ = false;
      continue;
    }
    if (kind == kSlabOsPull) {
      for (auto* s : S) s->precollide_if_fresh();
    }
    if (kind == kSlabTs) {
      for (auto* s : S) s->ts_collide();
    }
    if (kind == kSlabEt && S[0]->owners_stale_) {
      local_phase(S, 1);
      for (auto* s : S) s->owners_stale_ = false;
    }
    const bool pre = (kind == kSlabAA && odd) || kind == kSlabOsPull || kind == kSlabEt ||
                     kind == kSlabTs;
    const bool post = (kind == kSlabAA && odd) || kind == kSlabOsPush || kind == kSlabEt;
    if (pre) local_phase(S, 0);
    for (auto* s : S) s->step(1);
    // phase 1 of push applies to the grid just written (now active)
    if (post) {
      if (kind == kSlabOsPush)
        for (auto* s : S) s->active_ ^= 1;  // phase_grid(1) = active ^ 1 = written grid
      if (kind == kSlabEt)  // the sweep's handle table (step() already swapped it)
        for (auto* s : S) s->swap_base();
      local_phase(S, 1);
      if (kind == kSlabOsPush)
        for (auto* s : S) s->active_ ^= 1;
      if (kind == kSlabEt)
        for (auto* s : S) s->swap_base();
    }
    for (auto* s : S) s->ghosts_fresh_ = false;
  }
  for (auto* s : S) s->sync();
}

// create_stepper (p/src/stepper.cpp:155-180)
static std::unique_ptr<Stepper> create(const lbmgpu_geometry* gg, const lbmgpu_flow* p,
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
  if (o->z_end != 0 || o->z_begin != 0) return std::make_unique<SlabStepper>(g, *p, *o);
  if (o->addressing == LBMGPU_DIRECT) {
    switch (o->scheme) {
      case LBMGPU_TS: return std::make_unique<TsDirect>(g, *p, *o);
      case LBMGPU_OS_PUSH:
      case LBMGPU_OS_PULL:
      case LBMGPU_OSNT_PULL_1S:
      case LBMGPU_OSNT_PULL_2S: return std::make_unique<OsDirect>(g, *p, *o);
      case LBMGPU_CG: return std::make_unique<CgDirect>(g, *p, *o);
      case LBMGPU_SWAP_PUSH:
      case LBMGPU_SWAP_PULL: return std::make_unique<SwapDirect>(g, *p, *o);
      case LBMGPU_AAP: return std::make_unique<AaDirect>(g, *p, *o);
      case LBMGPU_ET: return std::make_unique<EtDirect>(g, *p, *o);
    }
  } else {
    switch (o->scheme) {
      case LBMGPU_TS: return std::make_unique<TsIndirect>(g, *p, *o);
      case LBMGPU_OS_PUSH:
      case LBMGPU_OS_PULL:
      case LBMGPU_OSNT_PULL_1S:
      case LBMGPU_OSNT_PULL_2S: return std::make_unique<OsIndirect>(g, *p, *o);
      case LBMGPU_SWAP_PUSH:
      case LBMGPU_SWAP_PULL: return std::make_unique<SwapIndirect>(g, *p, *o);
      case LBMGPU_AAP: return std::make_unique<AaIndirect>(g, *p, *o);
      case LBMGPU_ET: return std::make_unique<EtIndirect>(g, *p, *o);
    }
  }
  throw std::invalid_argument("unknown scheme");
}

// ---------------------------------------------------------------------------
// standalone IDX construction (build_sparse on the device)
// ---------------------------------------------------------------------------
struct IdxBuild {
  uint32_t n = 0;
  DevMem adj, node_of, rem;
  uint32_t nmail = 0;
};

static void build_idx(const lbmgpu_geometry* gg, int device, bool want_node_of, bool want_rem,
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
static HostGeo seeded_geometry(uint64_t seed) {
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

static lbmgpu_geometry c_geo(const HostGeo& g) {
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
    InitSpec in;
    switch (kind) {
      case 0: in = s.base_init(kSrcRest); break;
      case 1: in = s.base_init(kSrcTaylorGreen); break;
      case 2: in = s.base_init(kSrcRandom); break;
      default: throw std::invalid_argument("unknown init kind");
    }
    if (auto* sl = dynamic_cast<SlabStepper*>(&s)) {
      const int src = in.source;
      in = sl->slab_init(src);
    }
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
    if (nzl < 1) throw std::invalid_argument("slab needs at least one plane");
    int kind;
    switch (scheme) {
      case LBMGPU_AAP: kind = kSlabAA; break;
      case LBMGPU_OS_PUSH: kind = kSlabOsPush; break;
      case LBMGPU_OS_PULL:
      case LBMGPU_OSNT_PULL_1S:
      case LBMGPU_OSNT_PULL_2S: kind = kSlabOsPull; break;
      case LBMGPU_ET: kind = kSlabEt; break;
      case LBMGPU_TS: kind = kSlabTs; break;
      case LBMGPU_SWAP_PUSH:
      case LBMGPU_SWAP_PULL: kind = kSlabSwap; break;
      case LBMGPU_CG: kind = kSlabCg; break;
      default: throw std::invalid_argument("no z-slab decomposition for this scheme");
    }
    const auto plan = halo_plan(kind, nzl);
    if (count) *count = (int32_t)plan.size();
    if (ops)
      for (size_t k = 0; k < plan.size(); ++k) {
        ops[k * 5 + 0] = plan[k].phase;
        ops[k * 5 + 1] = plan[k].send;
        ops[k * 5 + 2] = plan[k].peer;
        ops[k * 5 + 3] = plan[k].plane;
        ops[k * 5 + 4] = plan[k].slot;
      }
  });
}

int lbmgpu_halo_plan(int32_t nzl, int32_t* ops, int32_t* count) {
  return lbmgpu_scheme_halo_plan(LBMGPU_AAP, nzl, ops, count);
}

int lbmgpu_nccl_unique_id(uint8_t* id) {
  return guard([&] {
    ncclUniqueId u;
    Nccl& N = Nccl::get();
    N.check(N.getUniqueId(&u), "ncclGetUniqueId");
    static_assert(sizeof(u) == LBMGPU_NCCL_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id, &u, sizeof(u));
  });
}

static SlabStepper& slab(lbmgpu_stepper* h) {
  auto* s = dynamic_cast<SlabStepper*>(&S(h));
  if (!s) throw std::invalid_argument("not a z-slab stepper");
  return *s;
}

int lbmgpu_slab_connect_nccl(lbmgpu_stepper* h, const uint8_t* id, int32_t nranks,
                             int32_t rank) {
  return guard([&] {
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank");
    slab(h).connect_nccl(u, nranks, rank);
  });
}

int lbmgpu_slab_sync_ghosts(lbmgpu_stepper* h) {
  return guard([&] { slab(h).sync_ghosts_nccl(); });
}

int lbmgpu_slab_group_step(lbmgpu_stepper** hs, int32_t n, int64_t steps) {
  return guard([&] {
    if (n < 1 || !hs) throw std::invalid_argument("empty slab group");
    std::vector<SlabStepper*> S;
    for (int k = 0; k < n; ++k) S.push_back(&slab(hs[k]));
    group_step(S, steps);
  });
}

int lbmgpu_slab_group_sync_ghosts(lbmgpu_stepper** hs, int32_t n) {
  return guard([&] {
    if (n < 1 || !hs) throw std::invalid_argument("empty slab group");
    std::vector<SlabStepper*> S;
    for (int k = 0; k < n; ++k) S.push_back(&slab(hs[k]));
    local_phase(S, 0, true);
    for (auto* s : S) s->ghosts_fresh_ = true;
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
