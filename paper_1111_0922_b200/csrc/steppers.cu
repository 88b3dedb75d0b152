// Single-domain steppers: one class per propagation scheme and addressing,
// each owning its device storage, index tables and sweep sequence
// (p/src/scheme_*.cpp state machines: time step, fresh/pending flags, ET
// handle table, layout phases), every sweep a sm_100a kernel launch.
#include "runtime.h"

namespace lbmgpu {

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
    // AoS: face-buffer kernels (kernels_aos_fb.cu); the face slots' home
    const DField f = field(f_, soa_stride(g.cells()));
    if (aa_fb_ok(f, L_)) {
      h_.alloc(aa_fb_face_elems(f, L_) * esize());
      fb_ = true;
    }
    init(base_init(kSrcRest));
  }
  void step_one() override {
    const DField f = field(f_, soa_stride(geo_.cells()));
    if (fb_) {
      if (!h_valid_) {
        launch_aa_fb_faces(stream_, f, L_, true, h_.get());
        h_valid_ = true;
      }
      launch_aa_fb(stream_, f, L_, op_, (t_ & 1) != 0, h_.get());
      return;
    }
    if ((t_ & 1) == 0)
      launch_local(stream_, f, f, L_, op_, false, true);
    else
      launch_aa_odd(stream_, f, L_, op_);
  }
  void before_extract() override {  // the face slots back into their records
    if (fb_ && h_valid_)
      launch_aa_fb_faces(stream_, field(f_, soa_stride(geo_.cells())), L_, false, h_.get());
  }
  void after_load() override {
    t_ = 0;
    h_valid_ = false;
  }
  void extract_range(uint32_t n0, uint32_t c, double* d) override {
    ex(field(f_, soa_stride(geo_.cells())), L_, (t_ & 1) ? kExAaOdd : kExNatural, n0, c, d);
  }
  void load_range(uint32_t n0, uint32_t c, const double* d, const InitSpec& in) override {
    ld(field(f_, soa_stride(geo_.cells())), L_, kExNatural, n0, c, d, in);
  }
  int layout_phase() const override { return (t_ & 1) ? LBMGPU_OPPOSED : LBMGPU_NATURAL; }
  uint64_t pdf_bytes() const override { return f_.bytes() + h_.bytes(); }

 private:
  DevMem f_, h_;
  bool fb_ = false, h_valid_ = false;
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
std::vector<SeamLink> seam_links(const HostGeo& g, const int* dirs, int ndirs) {
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
    win_ = aos_ && aos_push_planes_ok(field(f_, soa_stride(storage_)),
                                      make_lat(geo_, linkmask(), 0, 0, 0, 0));
    init(base_init(kSrcRest));
    sync();
  }
  dev::Lat frame(int origin) const {
    dev::Lat L = L_;
    L.oz = 1 + origin;
    L.znowrap = 1;
    return L;
  }
  // AoS: each plane group runs as the OS-push tile window (pull form of the
  // push: gather post-collision values from the read frame into whole
  // write-frame records). Within a group the read and write storage ranges
  // are disjoint; a periodic z wrap reads copies of the read frame's planes
  // 0 and nz-1 taken before the sweep, so no seam fix-up is needed.
  bool aos_window_step(bool even) {
    const DField base = field(f_, soa_stride(storage_));
    const dev::Lat Lc = make_lat(geo_, linkmask(), 0, 0, 0, 0);
    if (!aos_push_planes_ok(base, Lc)) return false;
    const size_t pl = (size_t)plane_ * 19 * esize();
    auto framed = [&](int origin) {
      DField d = base;
      d.p = static_cast<char*>(base.p) + (size_t)(1 + origin) * pl;
      return d;
    };
    const int R = even ? S_ : 0, W = even ? 0 : S_;
    const void *wlo = nullptr, *whi = nullptr;
    if (geo_.policy[2] == 0) {
      if (!side_.get()) side_.alloc(2 * pl);
      const char* r = static_cast<const char*>(framed(R).p);
      CK(cudaMemcpyAsync(side_.get(), r + (size_t)(geo_.nz - 1) * pl, pl, cudaMemcpyDeviceToDevice,
                         stream_));
      CK(cudaMemcpyAsync(static_cast<char*>(side_.get()) + pl, r, pl, cudaMemcpyDeviceToDevice,
                         stream_));
      wlo = side_.get();
      whi = static_cast<char*>(side_.get()) + pl;
    }
    const int ngroups = (geo_.nz + P_ - 1) / P_;
    for (int k = 0; k < ngroups; ++k) {
      const int gi = even ? k : ngroups - 1 - k;
      launch_aos_push_planes(stream_, framed(R), framed(W), Lc, op_, gi * P_,
                             std::min(geo_.nz, (gi + 1) * P_), wlo, whi);
    }
    return true;
  }
  void step_one() override {
    const DField f = field(f_, soa_stride(storage_));
    const bool even = (t_ & 1) == 0;
    if (win_ && aos_window_step(even)) return;
    const int R = even ? S_ : 0, W = even ? 0 : S_;
    const int delta = (W - R) * (int)plane_;
    const dev::Lat Lr = frame(R);
    const int ngroups = (geo_.nz + P_ - 1) / P_;
    for (int k = 0; k < ngroups; ++k) {
      const int gi = even ? k : ngroups - 1 - k;
      dev::Lat L = Lr;
      L.cell_begin = (uint32_t)(gi * P_ * plane_);
      L.ncells = (uint32_t)(std::min(geo_.nz, (gi + 1) * P_) * plane_);
      launch_cg_push(stream_, f, L, op_, delta, k > 0);
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
    return (geo_.nz + P_ - 1) / P_ + (!win_ && geo_.policy[2] == 0 ? 2 : 0);
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
  bool win_ = false;  // AoS plane groups through the tile window
  uint64_t plane_, storage_;
  DevMem f_, side_;
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
    // one-launch sweep (kernels_swap.cu), opt-in with LBMGPU_SWAP_FUSED=1: it
    // moves only the compulsory bytes but runs slower than the two passes
    const char* e = std::getenv("LBMGPU_SWAP_FUSED");
    const int rows = swap_fused_rows(L_);
    if (!aos_ && rows > 0 && e && std::atoi(e) == 1) {
      const size_t words = 1 + (size_t)((g.ny + rows - 1) / rows);
      sync_.alloc(words * 8);
      CK(cudaMemsetAsync(sync_.get(), 0, words * 8, stream_));
      fused_ = true;
    }
    // single pass with face buffers (kernels_swap1.cu), SoA: two parities
    // (when the two face buffers, ~18 % of the field each, do not fit in the
    // free device memory, the two passes run instead)
    if (!fused_ && swap1_ok(field(f_, soa_stride(g.cells())), L_, !pull_)) {
      hn_ = swap1_face_elems(field(f_, soa_stride(g.cells())), L_, !pull_);
      size_t fr = 0, tot = 0;
      CK(cudaMemGetInfo(&fr, &tot));
      if (2 * hn_ * esize() + (size_t(1) << 28) < fr) {
        h_[0].alloc(hn_ * esize());
        h_[1].alloc(hn_ * esize());
        single_ = true;
      }
    }
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
    if (single_) {
      if (!h_valid_) {  // the last sweep's face values, gathered from the field
        launch_swap1_faces(stream_, f, L_, push, true, h_[hpar_ ^ 1].get());
        h_valid_ = true;
      }
      launch_swap1(stream_, f, L_, op_, push, h_[hpar_].get(), h_[hpar_ ^ 1].get());
      hpar_ ^= 1;
      return;
    }
    if (fused_ && launch_swap_fused(stream_, f, L_, op_, push,
                                    sync_.get<unsigned long long>(), ++epoch_))
      return;
    if (push) {
      launch_local(stream_, f, f, L_, op_, true, false);
      launch_swap(stream_, f, L_, 1);
    } else {
      launch_swap(stream_, f, L_, 1);
      launch_local(stream_, f, f, L_, op_, true, false);
    }
  }
  int launches_per_step() const override { return (fused_ || single_ ? 1 : 2) + (nfix_ ? 1 : 0); }
  void before_extract() override {
    if (!pull_ && pending_) fixup(field(f_, soa_stride(geo_.cells())));
    // push: the face links of the last sweep live in the face buffer only
    if (single_ && h_valid_ && !pull_)
      launch_swap1_faces(stream_, field(f_, soa_stride(geo_.cells())), L_, true, false,
                         h_[hpar_ ^ 1].get());
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
    h_valid_ = false;
  }
  int layout_phase() const override {
    if (pull_) return LBMGPU_NATURAL;
    return pending_ ? LBMGPU_SWAP_PARTIAL : LBMGPU_OPPOSED;
  }
  uint64_t pdf_bytes() const override { return f_.bytes() + h_[0].bytes() + h_[1].bytes(); }

 private:
  bool pull_, defer_;
  bool fresh_ = false, pending_ = false, fused_ = false;
  bool single_ = false, h_valid_ = false;
  int hpar_ = 0;     // face buffer the next sweep writes
  size_t hn_ = 0;    // face-buffer elements per parity
  DevMem h_[2];
  long long nfix_ = 0;
  unsigned long long epoch_ = 0;
  DevMem f_, fa_, fb_, fd_, sync_;
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
    if (!geo_.solids) I_.bx = geo_.nx, I_.by = geo_.ny, I_.bz = geo_.nz;
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
  uint64_t pdf_bytes() const override { return f_.bytes() + h_.bytes(); }

 private:
  DevMem f_, h_;
  bool fb_ = false, h_valid_ = false;
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


std::unique_ptr<Stepper> create_single(const HostGeo& g, const lbmgpu_flow& p,
                                       const lbmgpu_options& o) {
  if (o.addressing == LBMGPU_DIRECT) {
    switch (o.scheme) {
      case LBMGPU_TS: return std::make_unique<TsDirect>(g, p, o);
      case LBMGPU_OS_PUSH:
      case LBMGPU_OS_PULL:
      case LBMGPU_OSNT_PULL_1S:
      case LBMGPU_OSNT_PULL_2S: return std::make_unique<OsDirect>(g, p, o);
      case LBMGPU_CG: return std::make_unique<CgDirect>(g, p, o);
      case LBMGPU_SWAP_PUSH:
      case LBMGPU_SWAP_PULL: return std::make_unique<SwapDirect>(g, p, o);
      case LBMGPU_AAP: return std::make_unique<AaDirect>(g, p, o);
      case LBMGPU_ET: return std::make_unique<EtDirect>(g, p, o);
    }
  } else {
    switch (o.scheme) {
      case LBMGPU_TS: return std::make_unique<TsIndirect>(g, p, o);
      case LBMGPU_OS_PUSH:
      case LBMGPU_OS_PULL:
      case LBMGPU_OSNT_PULL_1S:
      case LBMGPU_OSNT_PULL_2S: return std::make_unique<OsIndirect>(g, p, o);
      case LBMGPU_SWAP_PUSH:
      case LBMGPU_SWAP_PULL: return std::make_unique<SwapIndirect>(g, p, o);
      case LBMGPU_AAP: return std::make_unique<AaIndirect>(g, p, o);
      case LBMGPU_ET: return std::make_unique<EtIndirect>(g, p, o);
    }
  }
  throw std::invalid_argument("unknown scheme");
}

}  // namespace lbmgpu
