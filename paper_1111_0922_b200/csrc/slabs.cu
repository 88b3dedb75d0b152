// Multi-GPU z-slab decomposition of every scheme: halo plans, the NCCL and
// in-process transports, and SlabStepper (direct and indirect addressing).
#include "runtime.h"

#include <dlfcn.h>
#include <nccl.h>
#include <unistd.h>

#include <cstring>

namespace lbmgpu {

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

// NCCL, loaded on first use (dlopen) so processes that never decompose do not
// map it; inside a torch process this resolves to torch's libnccl.so.2.
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
  decltype(&ncclCommCount) commCount = nullptr;
  decltype(&ncclCommUserRank) commUserRank = nullptr;
  decltype(&ncclGetVersion) getVersion = nullptr;
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
      LBM_SYM(commCount, "ncclCommCount")
      LBM_SYM(commUserRank, "ncclCommUserRank")
      LBM_SYM(getVersion, "ncclGetVersion")
#undef LBM_SYM
    }
    return n;
  }
  void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw CudaError(std::string("nccl: ") + what + ": " + errStr(r));
  }
};

// ---------------------------------------------------------------------------
// Peer-memory transport for AA slabs ("p2p"): no ghost exchange. The face
// planes' odd sweep (launch_aa_odd_face) reads and rewrites the neighbour's
// face-plane slots in place over NVLink (the AA partition makes the slots of
// a sweep disjoint between the two sides), so a step only needs ordering:
// a face-plane sweep of step t starts after both neighbours finished step
// t - 1. In one process (kP2PGroup) that is a stream wait on the neighbours'
// step events; across processes (kP2PIpc: field and flag buffers shared with
// CUDA IPC handles) a one-thread kernel on the side stream publishes "step
// t - 1 done" into the neighbours' flag words (st.release.sys) and spins on
// its own (ld.acquire.sys) while the interior planes run on the main stream.
// ---------------------------------------------------------------------------
// mine[0] / mine[1]: step counts published by the lower / upper neighbour;
// mine[2]: error word. Epochs carry the connect generation in their high bits
// (see connect_p2p_ipc), so flag words are never reset while a neighbour may
// already be storing into them. A neighbour silent for 60 s sets the error
// word and the barrier returns (no __trap: the context stays usable and
// Stepper::sync reports the failure).
__global__ void k_slab_flag_barrier(unsigned long long* mine, unsigned long long* to_lo,
                                    unsigned long long* to_hi, unsigned long long epoch) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(to_lo), "l"(epoch) : "memory");
  asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(to_hi), "l"(epoch) : "memory");
  unsigned long long t0, now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int k = 0; k < 2; ++k) {
    unsigned long long v = 0;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(mine + k) : "memory");
      if (v >= epoch) break;
      __nanosleep(256);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > 60ull * 1000000000ull) {  // a neighbour stopped stepping
        atomicExch(mine + 2, epoch);
        return;
      }
    }
  }
}

// what a rank publishes so its neighbours can address its field and flags
struct P2PBlob {
  char magic[8];
  cudaIpcMemHandle_t field, flags;
  int64_t stride;  // SoA slot stride (elements)
  int64_t plane;   // cells per plane
  int32_t nzl, esize, device, pid;
};
static_assert(sizeof(P2PBlob) <= LBMGPU_P2P_BLOB_BYTES, "p2p blob size");

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
    for (auto e : ev_step_)
      if (e) cudaEventDestroy(e);
    close_ipc();
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

  // ---- p2p transport (AA, direct) ----------------------------------------
  void p2p_check() const {
    if (kind_ != kSlabAA || idx_)
      throw std::invalid_argument("p2p slab transport: AA on direct addressing only");
    if (nzl_ < 2) throw std::invalid_argument("p2p slab transport: at least 2 planes per slab");
  }
  void ensure_step_events() {
    for (auto& e : ev_step_)
      if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto e : ev_step_) CK(cudaEventRecord(e, stream_));
  }
  // in-process ring: lower / upper are the neighbouring slabs (may be this one)
  void connect_p2p_group(SlabStepper& lo, SlabStepper& hi) {
    p2p_check();
    if (lo.plane_ != plane_ || hi.plane_ != plane_ || lo.prec_ != prec_ || hi.prec_ != prec_)
      throw std::invalid_argument("p2p slab transport: slabs of different boxes or precisions");
    CK(cudaSetDevice(opt_.device));
    for (SlabStepper* n : {&lo, &hi}) {
      if (n->opt_.device == opt_.device) continue;
      int ok = 0;
      CK(cudaDeviceCanAccessPeer(&ok, opt_.device, n->opt_.device));
      if (!ok) throw std::runtime_error("p2p slab transport: devices without peer access");
      const cudaError_t e = cudaDeviceEnablePeerAccess(n->opt_.device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled)
        cudaGetLastError();
      else
        CK(e);
    }
    for (int k = 0; k < 19; ++k) {
      rem_lo_[k] = lo.slot_ptr(0, k, lo.nzl_ - 1);
      rem_hi_[k] = hi.slot_ptr(0, k, 0);
    }
    ensure_step_events();
    nb_ev_lo_ = lo.ev_step_;
    nb_ev_hi_ = hi.ev_step_;
    transport_ = kP2PGroup;
  }
  void p2p_export(P2PBlob& b) {
    p2p_check();
    CK(cudaSetDevice(opt_.device));
    if (!flags_.get()) {  // zeroed once, before any neighbour can address it
      flags_.alloc(3 * sizeof(unsigned long long));
      CK(cudaMemset(flags_.get(), 0, 3 * sizeof(unsigned long long)));
      CK(cudaDeviceSynchronize());
    }
    std::memset(&b, 0, sizeof(b));
    std::memcpy(b.magic, "LBMP2P1", 8);
    CK(cudaIpcGetMemHandle(&b.field, g_[0].get()));
    CK(cudaIpcGetMemHandle(&b.flags, flags_.get()));
    b.stride = soa_stride(storage_);
    b.plane = (int64_t)plane_;
    b.nzl = nzl_;
    b.esize = (int32_t)esize();
    b.device = opt_.device;
    b.pid = (int32_t)getpid();
  }
  void close_ipc() {
    for (void* p : ipc_open_) cudaIpcCloseMemHandle(p);
    ipc_open_.clear();
  }
  // one rank per process: lo / hi = the neighbours' blobs (nranks 1: this
  // slab's own, opened without IPC). Collective (every rank connects before
  // any rank steps), but with no host handshake needed: the flag words are
  // not reset here. Each connect starts a new generation g (the same on every
  // rank: connects are collective) and epochs count on from g << 40, so
  // values a neighbour stored for an earlier generation never satisfy a
  // barrier of this one, and a neighbour that connected and stepped first
  // cannot have its stores wiped.
  void connect_p2p_ipc(const P2PBlob& lo, const P2PBlob& hi, int nranks, int rank,
                       bool host_ordered = false) {
    p2p_check();
    for (const P2PBlob* b : {&lo, &hi}) {
      if (std::memcmp(b->magic, "LBMP2P1", 8) != 0)
        throw std::invalid_argument("p2p slab transport: not a p2p blob");
      if (b->plane != (int64_t)plane_ || b->esize != (int32_t)esize())
        throw std::invalid_argument("p2p slab transport: slabs of different boxes or precisions");
    }
    CK(cudaSetDevice(opt_.device));
    if (!flags_.get()) {
      P2PBlob mine;
      p2p_export(mine);
    }
    close_ipc();
    auto open = [&](const P2PBlob& b, char*& field, unsigned long long*& flags) {
      if (nranks == 1) {
        field = static_cast<char*>(g_[0].get());
        flags = flags_.get<unsigned long long>();
        return;
      }
      void* f = nullptr;
      void* g = nullptr;
      CK(cudaIpcOpenMemHandle(&f, b.field, cudaIpcMemLazyEnablePeerAccess));
      CK(cudaIpcOpenMemHandle(&g, b.flags, cudaIpcMemLazyEnablePeerAccess));
      ipc_open_.push_back(f);
      ipc_open_.push_back(g);
      field = static_cast<char*>(f);
      flags = static_cast<unsigned long long*>(g);
    };
    char *flo = nullptr, *fhi = nullptr;
    unsigned long long *glo = nullptr, *ghi = nullptr;
    open(lo, flo, glo);
    if (nranks == 2) {  // the same rank is both neighbours
      fhi = flo;
      ghi = glo;
    } else {
      open(hi, fhi, ghi);
    }
    const size_t es = esize();
    for (int k = 0; k < 19; ++k) {
      rem_lo_[k] = flo + ((size_t)k * lo.stride + (size_t)lo.nzl * lo.plane) * es;  // its plane nzl-1
      rem_hi_[k] = fhi + ((size_t)k * hi.stride + (size_t)hi.plane) * es;            // its plane 0
    }
    flag_to_lo_ = glo + 1;  // I am my lower neighbour's upper neighbour
    flag_to_hi_ = ghi + 0;
    CK(cudaDeviceSynchronize());
    ++generation_;
    epoch_ = (unsigned long long)generation_ << 40;
    nranks_ = nranks, rank_ = rank;
    host_ordered_ = host_ordered;
    transport_ = kP2PIpc;
  }
  void check_health() override {
    if (transport_ != kP2PIpc || !flags_.get()) return;
    unsigned long long err = 0;
    CK(cudaMemcpy(&err, flags_.get<unsigned long long>() + 2, sizeof(err),
                  cudaMemcpyDeviceToHost));
    if (err)
      throw std::runtime_error("p2p slab transport: a neighbour rank stopped stepping "
                               "(flag barrier timed out after 60 s at epoch " +
                               std::to_string(err & ((1ull << 40) - 1)) + ")");
  }
  void flag_barrier(cudaStream_t st) {
    ++epoch_;
    if (host_ordered_) return;  // the caller's host barrier orders the ranks
    k_slab_flag_barrier<<<1, 32, 0, st>>>(flags_.get<unsigned long long>(), flag_to_lo_, flag_to_hi_,
                                         epoch_);
  }
  // the two face planes of the current AA step (odd: over peer memory)
  void face_sweeps(cudaStream_t st) {
    const DField f = field(g_[0], soa_stride(storage_));
    if ((t_ & 1) == 0) {
      launch_local(st, f, f, planes(0, 1), op_, false, true);
      launch_local(st, f, f, planes(nzl_ - 1, nzl_), op_, false, true);
    } else {
      launch_aa_odd_face(st, f, planes(0, 1), op_, rem_lo_, -1, 0u);
      launch_aa_odd_face(st, f, planes(nzl_ - 1, nzl_), op_, rem_hi_, +1,
                         (uint32_t)((nzl_ + 1) * plane_));
    }
  }
  void step_p2p() {
    sweep(1, nzl_ - 1);  // interior planes: nothing crosses a face
    if (transport_ == kP2PGroup) {
      const int prev = (int)((t_ + 1) & 1);  // parity of step t - 1
      CK(cudaStreamWaitEvent(stream_, nb_ev_lo_[prev], 0));
      CK(cudaStreamWaitEvent(stream_, nb_ev_hi_[prev], 0));
      face_sweeps(stream_);
      CK(cudaEventRecord(ev_step_[t_ & 1], stream_));
      return;
    }
    // kP2PIpc: side stream after my step t - 1: barrier, then the face planes
    CK(cudaStreamWaitEvent(comm_, ev_back_, 0));
    flag_barrier(comm_);
    face_sweeps(comm_);
    CK(cudaEventRecord(ev_halo_, comm_));
    CK(cudaStreamWaitEvent(stream_, ev_halo_, 0));
    CK(cudaEventRecord(ev_back_, stream_));
  }
  // extraction at odd t reads the ghost planes: copy the neighbours' face
  // slots the odd gather reads (the AA phase-0 receives) over peer memory
  void sync_ghosts_p2p() {
    CK(cudaSetDevice(opt_.device));
    CK(cudaEventRecord(ev_c_, stream_));
    CK(cudaStreamWaitEvent(comm_, ev_c_, 0));
    flag_barrier(comm_);
    const size_t bytes = plane_ * esize();
    for (int k = 1; k < 19; ++k) {
      if (dev::cz(k) < 0)
        CK(cudaMemcpyAsync(slot_ptr(0, k, -1), rem_lo_[k], bytes, cudaMemcpyDefault, comm_));
      if (dev::cz(k) > 0)
        CK(cudaMemcpyAsync(slot_ptr(0, k, nzl_), rem_hi_[k], bytes, cudaMemcpyDefault, comm_));
    }
    CK(cudaEventRecord(ev_halo_, comm_));
    CK(cudaStreamWaitEvent(stream_, ev_halo_, 0));
    CK(cudaEventRecord(ev_back_, stream_));
    ghosts_fresh_ = true;
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
  // what the communicator itself reports (ncclCommCount / ncclCommUserRank)
  void comm_info(int32_t* count, int32_t* rank, int32_t* version) const {
    if (transport_ != kNccl || !nccl_) throw std::invalid_argument("slab has no NCCL communicator");
    Nccl& N = Nccl::get();
    int c = 0, r = 0, v = 0;
    N.check(N.commCount(nccl_, &c), "ncclCommCount");
    N.check(N.commUserRank(nccl_, &r), "ncclCommUserRank");
    N.check(N.getVersion(&v), "ncclGetVersion");
    *count = c, *rank = r, *version = v;
  }

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
      launch_cg_push(stream_, f, L, op_, (W - R) * (int)plane_, k > 0);
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
    if (transport_ == kP2PGroup || transport_ == kP2PIpc) {
      step_p2p();
      ghosts_fresh_ = false;
      return;
    }
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
    if (transport_ == kP2PGroup) return 3;
    if (transport_ == kP2PIpc) return 4;  // interior, barrier, two face planes
    if (transport_ != kNccl) return 1 + collide;
    return (nzl_ > 2 ? 3 : nzl_) + collide;
  }

  void finish() override {
    if (transport_ == kNccl || transport_ == kP2PIpc) CK(cudaStreamWaitEvent(stream_, ev_back_, 0));
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
    if (transport_ == kP2PIpc) return sync_ghosts_p2p();
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

  enum { kNone = 0, kLocalGroup = 1, kNccl = 2, kP2PGroup = 3, kP2PIpc = 4 };
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
  // p2p transport: base of the neighbours' face-plane slot k (lower: its top
  // owned plane, upper: its bottom one), step-done events (kP2PGroup: the
  // neighbours' ev_step_), flag words (kP2PIpc)
  void* rem_lo_[19] = {};
  void* rem_hi_[19] = {};
  cudaEvent_t ev_step_[2] = {nullptr, nullptr};
  const cudaEvent_t* nb_ev_lo_ = nullptr;
  const cudaEvent_t* nb_ev_hi_ = nullptr;
  DevMem flags_;
  unsigned long long* flag_to_lo_ = nullptr;
  unsigned long long* flag_to_hi_ = nullptr;
  unsigned long long epoch_ = 0;
  bool host_ordered_ = false;  // kP2PIpc without the flag-word barrier kernel
  int generation_ = 0;  // p2p connects so far (collective, so equal on every rank)
  std::vector<void*> ipc_open_;
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
  if (S[0]->transport_ == SlabStepper::kP2PGroup) {  // ordering by the step events only
    for (auto* s : S)
      if (s->transport_ != SlabStepper::kP2PGroup)
        throw std::invalid_argument("slab group mixes transports");
    for (long long k = 0; k < steps; ++k) {
      for (auto* s : S)
        if (s->t_ != S[0]->t_) throw std::invalid_argument("slabs out of step");
      for (auto* s : S) s->step(1);
    }
    for (auto* s : S) s->sync();
    return;
  }
  for (auto* s : S) {
    if (s->transport_ == SlabStepper::kNccl || s->transport_ == SlabStepper::kP2PIpc)
      throw std::invalid_argument("slab is connected to other processes");
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

// ---- entry points for capi.cu ---------------------------------------------
static SlabStepper& as_slab(Stepper& s) {
  auto* p = dynamic_cast<SlabStepper*>(&s);
  if (!p) throw std::invalid_argument("not a z-slab stepper");
  return *p;
}

std::unique_ptr<Stepper> create_slab(const HostGeo& g, const lbmgpu_flow& p,
                                     const lbmgpu_options& o) {
  return std::make_unique<SlabStepper>(g, p, o);
}

bool is_slab(const Stepper& s) { return dynamic_cast<const SlabStepper*>(&s) != nullptr; }

InitSpec slab_init_spec(const Stepper& s, int source) {
  if (auto* sl = dynamic_cast<const SlabStepper*>(&s)) return sl->slab_init(source);
  return s.base_init(source);
}

std::vector<int32_t> scheme_halo_plan(int scheme, int nzl) {
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
  std::vector<int32_t> rows;
  for (const HaloOp& op : halo_plan(kind, nzl))
    rows.insert(rows.end(), {op.phase, op.send, op.peer, op.plane, op.slot});
  return rows;
}

void nccl_unique_id(uint8_t* id) {
  ncclUniqueId u;
  Nccl& N = Nccl::get();
  N.check(N.getUniqueId(&u), "ncclGetUniqueId");
  static_assert(sizeof(u) == LBMGPU_NCCL_ID_BYTES, "ncclUniqueId size");
  std::memcpy(id, &u, sizeof(u));
}

void slab_connect_nccl(Stepper& s, const uint8_t* id, int nranks, int rank) {
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  as_slab(s).connect_nccl(u, nranks, rank);
}

void slab_sync_ghosts(Stepper& s) { as_slab(s).sync_ghosts_nccl(); }

void slab_comm_info(const Stepper& s, int32_t* count, int32_t* rank, int32_t* version) {
  auto* sl = dynamic_cast<const SlabStepper*>(&s);
  if (!sl) throw std::invalid_argument("not a z-slab stepper");
  sl->comm_info(count, rank, version);
}

void slab_group_step(const std::vector<Stepper*>& slabs, long long steps) {
  std::vector<SlabStepper*> S;
  for (Stepper* s : slabs) S.push_back(&as_slab(*s));
  group_step(S, steps);
}

void slab_group_connect_p2p(const std::vector<Stepper*>& slabs) {
  std::vector<SlabStepper*> S;
  for (Stepper* s : slabs) S.push_back(&as_slab(*s));
  const int n = (int)S.size();
  for (auto* s : S) s->sync();
  for (int k = 0; k < n; ++k) S[k]->connect_p2p_group(*S[(k - 1 + n) % n], *S[(k + 1) % n]);
}

void slab_p2p_export(Stepper& s, uint8_t* blob) {
  P2PBlob b;
  as_slab(s).p2p_export(b);
  std::memset(blob, 0, LBMGPU_P2P_BLOB_BYTES);
  std::memcpy(blob, &b, sizeof(b));
}

void slab_p2p_connect(Stepper& s, const uint8_t* lo, const uint8_t* hi, int nranks, int rank,
                      unsigned flags) {
  P2PBlob a, b;
  std::memcpy(&a, lo, sizeof(a));
  std::memcpy(&b, hi, sizeof(b));
  as_slab(s).connect_p2p_ipc(a, b, nranks, rank, (flags & LBMGPU_P2P_HOST_ORDERED) != 0);
}

void slab_group_sync_ghosts(const std::vector<Stepper*>& slabs) {
  std::vector<SlabStepper*> S;
  for (Stepper* s : slabs) S.push_back(&as_slab(*s));
  local_phase(S, 0, true);
  for (auto* s : S) s->ghosts_fresh_ = true;
}

}  // namespace lbmgpu
