// Host runtime of liblbmgpu.so (shared by steppers.cu, slabs.cu, capi.cu):
// errors, device memory, host geometry, and the Stepper base class that
// mirrors the reference's (p/include/lbmlab/stepper.hpp:70-106): time step,
// canonical snapshot conversion in chunks, device-side init. One subclass per
// propagation scheme lives in steppers.cu (single domain) and slabs.cu (z-slab
// decomposition); capi.cu is the C ABI of include/lbmgpu.h.
#pragma once
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

inline void ck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    throw std::bad_alloc();
  }
  throw CudaError(std::string("cuda: ") + what + ": " + cudaGetErrorString(e));
}
#define CK(x) ck((x), #x)
inline void ck_launch() { ck(cudaGetLastError(), "kernel launch"); }

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
    // + 64 bytes: kernels may over-read up to 15 bytes past a row for
    // 16-byte-aligned bulk copies (kernels_aos.cu copy_in_bulk_superset)
    CK(cudaMalloc(&p_, bytes + 64));
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
inline constexpr int kC[19][3] = {
    {0, 0, 0},   {1, 0, 0},   {-1, 0, 0}, {0, 1, 0},   {0, -1, 0}, {0, 0, 1},  {0, 0, -1},
    {-1, -1, 0}, {-1, 0, -1}, {-1, 0, 1}, {-1, 1, 0},  {0, -1, -1}, {0, -1, 1}, {0, 1, -1},
    {0, 1, 1},   {1, -1, 0},  {1, 0, -1}, {1, 0, 1},   {1, 1, 0}};
inline constexpr int kPi[9] = {1, 3, 5, 7, 8, 9, 10, 11, 12};
inline constexpr int kPj[9] = {2, 4, 6, 18, 17, 16, 15, 14, 13};
inline double w_of(int i) { return i == 0 ? 1.0 / 3.0 : (i <= 6 ? 1.0 / 18.0 : 1.0 / 36.0); }

// TrtOperator ctor/build (p/src/collision.cpp:50-93), including the
// zero-collision identity operator (p/src/stepper_common.hpp:104-108).
inline TrtHost make_trt(const lbmgpu_flow& p, bool zero_collision) {
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
  t.rho0 = p.rho0;
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

inline HostGeo copy_geo(const lbmgpu_geometry* g) {
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

inline dev::Lat make_lat(const HostGeo& g, const uint32_t* linkmask, int hx, int hy, int hz,
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
inline bool available(int s, int a, bool ext) {
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

  void sync() {
    CK(cudaStreamSynchronize(stream_));
    check_health();
  }
  // errors a transport records on the device instead of trapping (z-slab p2p)
  virtual void check_health() {}

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
    spec.rho0 = rho0_;  // the fp32 storage offset
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

  void init(const InitSpec& spec_in) {
    CK(cudaSetDevice(opt_.device));
    InitSpec spec = spec_in;
    double* trig = nullptr;
    if (spec.source == kSrcTaylorGreen) {
      std::vector<double> tab(2 * ((size_t)spec.gnx + spec.gny + spec.gnz));
      taylor_green_table(spec.gnx, spec.gny, spec.gnz, tab.data());
      CK(cudaMalloc(&trig, tab.size() * sizeof(double)));
      CK(cudaMemcpy(trig, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice));
      spec.trig = trig;
    }
    for_chunks([&](uint32_t n0, uint32_t cnt) {
      load_range(n0, cnt, nullptr, spec);
      ck_launch();
    });
    after_load();
    sync();
    if (trig) CK(cudaFree(trig));
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
    f.shift = rho0_;
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
// factories and z-slab entry points (defined in steppers.cu / slabs.cu)
// ---------------------------------------------------------------------------
std::unique_ptr<Stepper> create_single(const HostGeo& g, const lbmgpu_flow& p,
                                       const lbmgpu_options& o);
std::unique_ptr<Stepper> create_slab(const HostGeo& g, const lbmgpu_flow& p,
                                     const lbmgpu_options& o);
bool is_slab(const Stepper& s);
// a device-side init spec of the global box for a slab (unchanged otherwise)
InitSpec slab_init_spec(const Stepper& s, int source);
// the exchange table of a scheme on an nzl-plane slab, rows of 5 int32
std::vector<int32_t> scheme_halo_plan(int scheme, int nzl);
void nccl_unique_id(uint8_t* id);
void slab_connect_nccl(Stepper& s, const uint8_t* id, int nranks, int rank);
void slab_sync_ghosts(Stepper& s);
void slab_comm_info(const Stepper& s, int32_t* count, int32_t* rank, int32_t* version);
void slab_group_step(const std::vector<Stepper*>& slabs, long long steps);
void slab_group_sync_ghosts(const std::vector<Stepper*>& slabs);
// p2p transport (AA direct): in one process over a ring of slabs, or one rank
// per process through exported blobs (CUDA IPC handles of field and flags)
void slab_group_connect_p2p(const std::vector<Stepper*>& slabs);
void slab_p2p_export(Stepper& s, uint8_t* blob);
void slab_p2p_connect(Stepper& s, const uint8_t* lo, const uint8_t* hi, int nranks, int rank,
                      unsigned flags);

}  // namespace lbmgpu
