// AoS "window" kernels (direct addressing, record layout f[s*19 + i]).
//
// The per-thread AoS kernels in kernels_direct.cu read or write one field of
// 32 different 152-byte records per warp instruction: every gather/scatter
// moves a 32-byte L2 sector for 8 useful bytes, so the streamed side runs at
// a quarter of the sector rate (profiles/r01_sweep_c1_final2.jsonl: OS pull
// 0.45, OS push 0.23, AA 0.32 of the HBM roofline). Here a block owns a
// 32 x 8 x-y tile and marches through a chunk of z planes. Each plane of the
// tile plus a one-cell halo (34 x 10 records) is copied whole into a 4-plane
// shared-memory ring, one bulk copy (TMA engine) per row issued by one lane
// of the loading warp (the row phase in shared memory matches the record's
// global byte phase, so the copy is 16-byte congruent); all neighbour accesses are
// shared-memory accesses, and the tile's output records leave as contiguous
// 16-byte stores. DRAM sees each record once per sweep (the halo rows/planes
// are L2 hits of the neighbouring tiles), L2 sees 1.33x the record bytes.
//
// Modes (bitwise the same arithmetic as the per-thread kernels):
//   kWinPull   OS / OSNT pull: gather A[X - c_i][i] (bounce A[X][opp i]),
//              collide, store B[X]                  (p/src/scheme_os.cpp:141-174)
//   kWinStream TS stream: B[X][i] = A[X - c_i][i]   (p/src/scheme_ts.cpp:82-112)
//   kWinPush   OS push: collide every window record in place, then
//              B[X][i] = bounce(opp i) ? post(X)[opp i] : post(X - c_i)[i],
//              the same values the scatter B[i][Y + c_i] = post(Y)[i] writes
//              (p/src/scheme_os.cpp:104-139); halo records are collided
//              redundantly by both tiles (deterministic, identical)
//   kWinPushS  OS push, scatter form (fp64): each tile node collides its own
//              record and stores post(X)[i] into slot i of X + c_i in the
//              ring; the output leaves through the AA-odd ownership
//              write-back into the other grid
//   kWinAaOdd  AA odd sweep in place (p/src/scheme_aap.cpp:133-173). Node X
//              reads and rewrites the slot set {(opp i, X - c_i)} (bounce:
//              (i, X)); those sets partition the grid, so the owner of slot
//              (k, R) is R if link opp k of R bounces, else R - c_k. A record
//              whose 19 owners all lie in this block's tile and z chunk is
//              written back whole; the others (tile rim, halo ring, chunk
//              faces) slot by slot, only the owned slots.
//   kWinSwap   SWAP link exchange in place (p/src/scheme_swap.cpp:172-235,
//              kernels_direct k_swap mode 1: non-wrapped links): node X swaps
//              (i, X) <-> (opp i, X + c_i) for its back directions, so slot
//              (k, R) is swapped by R (k back) or by R + c_k (k forward).
//   kWinEt*    ET sweep in place (p/src/scheme_et.cpp:191-239) with the handle
//              table's parity as the mode: physical slot s of R holds logical
//              direction d (s = b_d); it is written by R when d is 0 or a first
//              pair member, else (second member j of pair (i, j)) by R + c_j =
//              R - c_i, or by R itself when link j of R bounces. Solid and
//              wall-halo records are mailboxes: their second-member slots are
//              written by the fluid neighbour R + c_j.
// CG runs each plane group as a kWinPush window between its two frames
// (launch_aos_push_planes; a periodic z wrap reads copies of the read
// frame's planes 0 and nz-1 taken before the sweep). The local sweeps (AA
// even, TS collide, precollide, SWAP collide) have no neighbour accesses and
// stream 256-record runs through a two-slot cp.async ring (k_local_stream).
#include "dispatch.h"
#include "launch.h"

#include <algorithm>
#include <atomic>
#include <cstdlib>

namespace lbmgpu {
using namespace dev;

namespace {

// Phase trace (experiments only, -DLBM_WIN_TRACE): thread 0 of every window
// block accumulates clock64 cycles per phase of the plane loop; read back
// with lbmgpu_debug_win_trace (tools/win_trace.py).
#ifdef LBM_WIN_TRACE
__device__ unsigned long long g_win_trace[16];
#define WIN_T0() long long _tt = clock64()
#define WIN_T(k)                                                                 \
  do {                                                                           \
    const long long _n = clock64();                                              \
    if (threadIdx.x == 0) atomicAdd(&g_win_trace[k], (unsigned long long)(_n - _tt)); \
    _tt = _n;                                                                    \
  } while (0)
#else
#define WIN_T0()
#define WIN_T(k)
#endif

constexpr int kTX = 32, kTY = 8;             // tile: one warp per x-row
constexpr int kWC = kTX + 2, kWR = kTY + 2;  // window columns / rows (1-cell halo)
constexpr int kNB = 4;                       // plane buffers in the ring

enum WinMode : int {
  kWinPull = 0,
  kWinStream = 1,
  kWinPush = 2,
  kWinAaOdd = 3,
  kWinSwap = 4,
  kWinEtI = 5,  // ET, identity handle table
  kWinEtS = 6,  // ET, all pairs swapped
  kWinPushS = 7 // OS push, scatter form
};
constexpr bool is_et(int mode) { return mode == kWinEtI || mode == kWinEtS; }
constexpr bool in_place(int mode) { return mode == kWinAaOdd || mode == kWinSwap || is_et(mode); }
// modes whose output leaves through the ownership write-back (in place, or
// the scatter-form push into the other grid)
constexpr bool owned_wb(int mode) { return in_place(mode) || mode == kWinPushS; }

// threads per block: one warp per tile row computes; fp64 runs one block per
// SM (the ring takes 207 KB) and adds 3 warps that only load and store
// (11 x 32 = 352 threads <= 184 registers; C1 OS pull 0.62 -> 0.67) ...
// for the gather modes (OS push's ring collisions need more than 184
// registers; AA odd measured no better)
#ifndef LBM_WIN_GATHER_THREADS
#define LBM_WIN_GATHER_THREADS 352
#endif
// LBM_WIN_LOADER > 0 (experiments): that many extra warps in the modes that
// have none; the first of them issues the ring's plane loads (load_plane).
// Measured slower for the in-place modes (the register cap of the larger
// block), so off by default.
#ifndef LBM_WIN_LOADER
#define LBM_WIN_LOADER 0
#endif
template <class T, int MODE>
struct WinThreads {
  // kWinPush (CG plane groups) collides the whole (kTY + 2) x 34 window
  // before its gathers: enough warps for one round
  static constexpr int value = (sizeof(T) == 8 && (MODE == kWinPull || MODE == kWinStream)) ||
                                       MODE == kWinPush
                                   ? LBM_WIN_GATHER_THREADS
                                   : kTX * kTY + 32 * LBM_WIN_LOADER;
  static constexpr int warps = value / 32;
};

template <class T>
struct WinSz {
  static constexpr int V = 16 / (int)sizeof(T);                    // elements per 16 B
  static constexpr int ROW = ((kWC * 19 + V + V - 1) / V) * V;     // + phase slack
  static constexpr int BUF = kWR * ROW;
  static constexpr size_t kBytes = (size_t)kNB * BUF * sizeof(T);
};
static_assert(WinSz<double>::kBytes <= 227 * 1024 - 256, "fp64 ring exceeds shared memory");

// one warp copies n elements global -> shared; s and g congruent mod 16 bytes
template <class T>
__device__ __forceinline__ void copy_in(T* s, const T* g, int n, int lane) {
  constexpr int V = 16 / (int)sizeof(T);
  int head = (int)(((16u - (uint32_t)(reinterpret_cast<uintptr_t>(g) & 15u)) & 15u) / sizeof(T));
  if (head > n) head = n;
  const int nv = (n - head) / V;
  if (lane < head) cp_async<sizeof(T)>(s + lane, g + lane);
  uint32_t sa = smem_u32(s + head) + 16u * (uint32_t)lane;
  const char* ga = reinterpret_cast<const char*>(g + head) + 16 * lane;
  for (int c = lane; c < nv; c += 32, sa += 512u, ga += 512)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(ga) : "memory");
  const int t0 = head + nv * V;
  if (t0 + lane < n) cp_async<sizeof(T)>(s + t0 + lane, g + t0 + lane);
}
// one record from another phase (a wrapped halo column)
template <class T>
__device__ __forceinline__ void copy_in_rec(T* s, const T* g, int lane) {
  if (lane < 19) cp_async<sizeof(T)>(s + lane, g + lane);
}
// one warp copies n elements shared -> global; congruent mod 16 bytes
template <class T>
__device__ __forceinline__ void copy_out(T* g, const T* s, int n, int lane) {
  constexpr int V = 16 / (int)sizeof(T);
  int head = (int)(((16u - (uint32_t)(reinterpret_cast<uintptr_t>(g) & 15u)) & 15u) / sizeof(T));
  if (head > n) head = n;
  const int nv = (n - head) / V;
  if (lane < head) g[lane] = s[lane];
  const float4* sv = reinterpret_cast<const float4*>(s + head) + lane;
  float4* gv = reinterpret_cast<float4*>(g + head) + lane;
  for (int c = lane; c < nv; c += 32, sv += 32, gv += 32) *gv = *sv;
  const int t0 = head + nv * V;
  if (t0 + lane < n) g[t0 + lane] = s[t0 + lane];
}

// Bulk (TMA engine) forms, selected by LBM_AOS_BULK (default on): the
// 16-byte-aligned middle of a row moves as one cp.async.bulk issued by lane 0
// (loads count their bytes on the ring slot's mbarrier, stores join a bulk
// group), the unaligned head / tail elements as before.
#ifndef LBM_AOS_BULK
#define LBM_AOS_BULK 1
#endif
constexpr bool kBulk = LBM_AOS_BULK != 0;

// one warp: n elements global -> shared (congruent mod 16 bytes). Arrivals on
// bar (kRowArrivals per row): every lane once when its cp.async copies (the
// unaligned head / tail, and any the caller issued before) have landed, lane 0
// once more with the bulk bytes.
constexpr uint32_t kRowArrivals = 33;
template <class T>
__device__ __forceinline__ void copy_in_bulk(T* s, const T* g, int n, int lane, uint64_t* bar) {
  constexpr int V = 16 / (int)sizeof(T);
  int head = (int)(((16u - (uint32_t)(reinterpret_cast<uintptr_t>(g) & 15u)) & 15u) / sizeof(T));
  if (head > n) head = n;
  const int nmid = (n - head) / V * V;
#ifdef LBM_WIN_TRACE
  long long c0 = clock64();
#define WIN_T2(k)                                                        \
  do {                                                                   \
    const long long c1 = clock64();                                      \
    if (lane == 0) atomicAdd(&g_win_trace[k], (unsigned long long)(c1 - c0)); \
    c0 = c1;                                                             \
  } while (0)
#else
#define WIN_T2(k)
#endif
  if (lane < head) cp_async<sizeof(T)>(s + lane, g + lane);
  const int t0 = head + nmid;
  if (t0 + lane < n) cp_async<sizeof(T)>(s + t0 + lane, g + t0 + lane);
  WIN_T2(8);
  cp_async_mbar_arrive(bar);
  WIN_T2(9);
  if (lane == 0) {
    const uint32_t bytes = (uint32_t)nmid * (uint32_t)sizeof(T);
    mbar_arrive_tx(bar, bytes);
    WIN_T2(10);
    if (bytes) bulk_g2s(s + head, g + head, bytes, bar);
    WIN_T2(11);
#ifdef LBM_WIN_TRACE
    atomicAdd(&g_win_trace[12], 1ull);
#endif
  }
#undef WIN_T2
}
// The same as one bulk copy of the 16-byte-aligned superset of the range
// (at most 15 bytes more on either side, landing in the row's phase slack):
// lane 0 issues everything, no per-lane cp.async and no per-lane arrival.
// Only where the superset's extra bytes in shared memory are not also written
// by another copy (a row without separately copied wrap records). Global
// over-reads stay inside the allocation (DevMem pads every buffer).
template <class T>
__device__ __forceinline__ void copy_in_bulk_superset(T* s, const T* g, int n, int lane,
                                                      uint64_t* bar) {
  if (lane == 0) {
    const uintptr_t gb = reinterpret_cast<uintptr_t>(g), lo = gb & ~(uintptr_t)15;
    const uintptr_t hi = (gb + (uintptr_t)n * sizeof(T) + 15) & ~(uintptr_t)15;
    char* sa = reinterpret_cast<char*>(s) - (gb - lo);
    mbar_arrive(bar, kRowArrivals - 1);
    mbar_arrive_tx(bar, (uint32_t)(hi - lo));
    bulk_g2s(sa, reinterpret_cast<const void*>(lo), (uint32_t)(hi - lo), bar);
  }
}
#ifndef LBM_AOS_SUPERSET
#define LBM_AOS_SUPERSET 1
#endif

// one warp: n elements shared -> global (congruent mod 16 bytes). The lanes'
// own shared-memory writes must precede it (each lane fences them for the
// async proxy here); lane 0 later waits for the group's reads (bulk_wait_read)
// before the staging area is reused.
template <class T>
__device__ __forceinline__ void copy_out_bulk(T* g, const T* s, int n, int lane) {
  constexpr int V = 16 / (int)sizeof(T);
  int head = (int)(((16u - (uint32_t)(reinterpret_cast<uintptr_t>(g) & 15u)) & 15u) / sizeof(T));
  if (head > n) head = n;
  const int nmid = (n - head) / V * V;
  fence_async_smem();
  __syncwarp();
  if (lane < head) g[lane] = s[lane];
  const int t0 = head + nmid;
  if (t0 + lane < n) g[t0 + lane] = s[t0 + lane];
  if (lane == 0 && nmid) {
    bulk_s2g(g + head, s + head, (uint32_t)nmid * (uint32_t)sizeof(T));
    bulk_commit();
  }
}

// window position p on one axis (cell coordinate, may be -1 or n) -> storage
// coordinate; false when no record is stored there (a wall axis without a
// halo). Halo axes (ET: wall axes carry one mailbox layer, o = 1) keep the
// position, periodic axes wrap.
__device__ __forceinline__ bool axis_pos(int p, int n, bool wall, int o, int& st) {
  if ((p < 0 || p >= n) && !o) {
    if (wall) return false;
    p = p < 0 ? p + n : p - n;
  }
  st = p + o;
  return true;
}
// storage index of the record at storage x = 0 of window row (y, z)
__device__ __forceinline__ bool row_base(const Lat& L, int y, int z, uint32_t& rb) {
  int ys, zs;
  if (!axis_pos(y, L.ny, L.wall[1], L.oy, ys) || !axis_pos(z, L.nz, L.wall[2], L.oz, zs))
    return false;
  rb = (uint32_t)L.sx * ((uint32_t)ys + (uint32_t)L.sy * (uint32_t)zs);
  return true;
}
// storage x of window column rx
__device__ __forceinline__ bool col_xs(const Lat& L, int x0, int rx, int& xs) {
  return axis_pos(x0 - 1 + rx, L.nx, L.wall[0], L.ox, xs);
}
// cell coordinate (wrapped) of a window position, false outside the domain
__device__ __forceinline__ bool axis_cell(int p, int n, bool wall, int o, int& c) {
  if (p < 0 || p >= n) {
    if (o || wall) return false;
    p = p < 0 ? p + n : p - n;
  }
  c = p;
  return true;
}
// links of an in-range cell (resolve_link, p/src/geometry.cpp:49-60)
__device__ __forceinline__ bool cell_links(const Lat& L, int x, int y, int z, uint32_t& bounce) {
  if (L.linkmask) {
    const uint32_t lm = L.linkmask[(uint32_t)x + (uint32_t)L.nx * ((uint32_t)y + (uint32_t)L.ny * (uint32_t)z)];
    bounce = lm & ~1u;
    return lm & 1u;
  }
  uint32_t b = 0;
  if (L.wall[0]) b |= (x == 0 ? kMxm : 0u) | (x == L.nx - 1 ? kMxp : 0u);
  if (L.wall[1]) b |= (y == 0 ? kMym : 0u) | (y == L.ny - 1 ? kMyp : 0u);
  if (L.wall[2]) b |= (z == 0 ? kMzm : 0u) | (z == L.nz - 1 ? kMzp : 0u);
  bounce = b;
  return true;
}

struct Tile {
  int x0, y0, txv, tyv, zb, ze;
};

// the record at window (rx, r, z) is an in-domain fluid cell; its links
__device__ __forceinline__ bool win_cell(const Lat& L, const Tile& t, int rx, int r, int z,
                                         uint32_t& bounce) {
  int x, y, zc;
  if (!axis_cell(t.x0 - 1 + rx, L.nx, L.wall[0], L.ox, x) ||
      !axis_cell(t.y0 - 1 + r, L.ny, L.wall[1], L.oy, y) ||
      !axis_cell(z, L.nz, L.wall[2], L.oz, zc))
    return false;
  return cell_links(L, x, y, zc, bounce);
}
__device__ __forceinline__ bool in_block(const Tile& t, int rx, int r, int z) {
  return rx >= 1 && rx <= t.txv && r >= 1 && r <= t.tyv && z >= t.zb && z < t.ze;
}

// One lane copies one window row: n elements at g -> s (congruent mod 16 B)
// as one bulk copy of the 16-byte-aligned part plus cp.async for the
// unaligned head / tail elements; where the row's neighbouring shared memory
// is not written by anyone else (lo_free / hi_free: no wrap record next to
// it) the bulk copy takes the aligned superset instead and there are no
// head / tail copies. Plus the wrap records (19 elements each, cp.async).
// Arrivals on bar: kRowArrivals per row, like the warp form.
template <class T>
__device__ __forceinline__ void copy_row_lane(T* s, const T* g, int n, bool lo_free, bool hi_free,
                                              T* sl, const T* gl, T* sr, const T* gr,
                                              uint64_t* bar) {
  const uintptr_t gb = reinterpret_cast<uintptr_t>(g);
  const uintptr_t ge = gb + (uintptr_t)n * sizeof(T);
  const uintptr_t lo = lo_free ? (gb & ~(uintptr_t)15) : ((gb + 15) & ~(uintptr_t)15);
  const uintptr_t hi = hi_free ? ((ge + 15) & ~(uintptr_t)15) : (ge & ~(uintptr_t)15);
  bool cp = false;
  if (gl) {
    for (int i = 0; i < 19; ++i) cp_async<sizeof(T)>(sl + i, gl + i);
    cp = true;
  }
  if (gr) {
    for (int i = 0; i < 19; ++i) cp_async<sizeof(T)>(sr + i, gr + i);
    cp = true;
  }
  const int nh = (int)((lo > gb ? lo - gb : 0) / sizeof(T));
  for (int i = 0; i < nh && i < n; ++i) cp_async<sizeof(T)>(s + i, g + i), cp = true;
  if (hi < lo) {  // a row shorter than one aligned vector: all elements by cp.async
    for (int i = nh; i < n; ++i) cp_async<sizeof(T)>(s + i, g + i), cp = true;
    mbar_arrive(bar, kRowArrivals - 1);
    cp_async_mbar_arrive(bar);
    return;
  }
  const int nt = (int)((ge > hi ? ge - hi : 0) / sizeof(T));
  for (int i = n - nt; i < n; ++i) cp_async<sizeof(T)>(s + i, g + i), cp = true;
  mbar_arrive(bar, kRowArrivals - 1 - (cp ? 1u : 0u));
  if (cp) cp_async_mbar_arrive(bar);
  char* sa = reinterpret_cast<char*>(s) + (lo - gb);
  mbar_arrive_tx(bar, (uint32_t)(hi - lo));
  if (hi > lo) bulk_g2s(sa, reinterpret_cast<const void*>(lo), (uint32_t)(hi - lo), bar);
}
#ifndef LBM_AOS_LANELOAD
#define LBM_AOS_LANELOAD 1
#endif

// issue the cp.async copies of window plane z (cell z, may be -1 / nz)
template <class T>
__device__ __forceinline__ void load_plane(const Lat& L, const T* __restrict__ g, T* buf,
                                           int* ph, const Tile& t, int z, const T* wlo,
                                           const T* whi, uint64_t* bar, int loader = -1) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // a periodic z wrap may read a saved copy of the wrapped plane (CG groups:
  // the plane itself may already be overwritten by an earlier group)
  if (z < 0 && wlo) {
    g = wlo - (size_t)L.sxy * (size_t)(L.nz - 1) * 19;
  } else if (z >= L.nz && whi) {
    g = whi;
  }
  if constexpr (kBulk && LBM_AOS_LANELOAD) {
    // warp 0, one lane per window row: a plane costs the loading warp a few
    // dozen instructions instead of every warp a row loop
    // the loading warp: the first warp beyond the tile rows where there is
    // one (the fp64 gather modes' extra warps: loads overlap the compute
    // warps' work, C1 OS pull 0.68 -> 0.76), else warp 0
    const int lw = loader >= 0 ? loader : ((int)(blockDim.x >> 5) > kTY ? kTY : 0);
    if (warp != lw) return;
    const int r = lane;
    if (r >= t.tyv + 2) return;
    uint32_t rb;
    int phase = 0;
    if (row_base(L, t.y0 - 1 + r, z, rb)) {
      const uintptr_t a0 = reinterpret_cast<uintptr_t>(g) +
                           (uintptr_t)(((long long)rb + L.ox + t.x0 - 1) * 19 * (long long)sizeof(T));
      phase = (int)((a0 & 15u) / sizeof(T));
      T* srow = buf + r * WinSz<T>::ROW + phase;
      const int xa = max(t.x0 - 1, -L.ox), xb = min(t.x0 + t.txv, L.nx - 1 + L.ox);
      const T *gl = nullptr, *gr = nullptr;
      if (!L.wall[0] && !L.ox) {
        if (t.x0 == 0) gl = g + ((size_t)rb + (size_t)(L.nx - 1)) * 19;
        if (t.x0 + t.txv == L.nx) gr = g + (size_t)rb * 19;
      }
      ph[r] = phase;  // before the arrivals: readers acquire it through the barrier
      copy_row_lane(srow + (xa - t.x0 + 1) * 19, g + ((size_t)rb + (size_t)(xa + L.ox)) * 19,
                    (xb - xa + 1) * 19, gl == nullptr, gr == nullptr, srow, gl,
                    srow + (t.txv + 1) * 19, gr, bar);
    } else {
      ph[r] = phase;
      mbar_arrive(bar, kRowArrivals);
    }
  } else {
  for (int r = warp; r < t.tyv + 2; r += (int)(blockDim.x >> 5)) {
    uint32_t rb;
    int phase = 0;
    if (row_base(L, t.y0 - 1 + r, z, rb)) {
      // byte phase of the record under window column 0 (from its address: g
      // may be a saved plane copy)
      const uintptr_t a0 = reinterpret_cast<uintptr_t>(g) +
                           (uintptr_t)(((long long)rb + L.ox + t.x0 - 1) * 19 * (long long)sizeof(T));
      phase = (int)((a0 & 15u) / sizeof(T));
      T* srow = buf + r * WinSz<T>::ROW + phase;
      const int xa = max(t.x0 - 1, -L.ox), xb = min(t.x0 + t.txv, L.nx - 1 + L.ox);
      bool wrapx = false;
      if (!L.wall[0] && !L.ox) {
        if (t.x0 == 0) copy_in_rec(srow, g + ((size_t)rb + (size_t)(L.nx - 1)) * 19, lane);
        if (t.x0 + t.txv == L.nx) copy_in_rec(srow + (t.txv + 1) * 19, g + (size_t)rb * 19, lane);
        wrapx = t.x0 == 0 || t.x0 + t.txv == L.nx;
      }
      if constexpr (kBulk) {
        if (LBM_AOS_SUPERSET && !wrapx)
          copy_in_bulk_superset(srow + (xa - t.x0 + 1) * 19,
                                g + ((size_t)rb + (size_t)(xa + L.ox)) * 19, (xb - xa + 1) * 19,
                                lane, bar);
        else
          copy_in_bulk(srow + (xa - t.x0 + 1) * 19, g + ((size_t)rb + (size_t)(xa + L.ox)) * 19,
                       (xb - xa + 1) * 19, lane, bar);
      }
      else
        copy_in(srow + (xa - t.x0 + 1) * 19, g + ((size_t)rb + (size_t)(xa + L.ox)) * 19,
                (xb - xa + 1) * 19, lane);
    } else if (kBulk && lane == 0) {
      mbar_arrive(bar, kRowArrivals);  // every window row arrives fully once per load
    }
    if (lane == 0) ph[r] = phase;
  }
  }
}

// OS push: collide every fluid record of a window plane in place
template <class T>
__device__ __forceinline__ void collide_plane(const Lat& L, const Trt<T>& op, T* buf,
                                              const int* ph, const Tile& t, int z) {
  const int w = t.txv + 2, n = w * (t.tyv + 2);
  for (int q = threadIdx.x; q < n; q += (int)blockDim.x) {
    const int r = q / w, rx = q - r * w;
    uint32_t bounce;
    if (!win_cell(L, t, rx, r, z, bounce)) continue;
    T* rec = buf + r * WinSz<T>::ROW + ph[r] + rx * 19;
    T f[19];
#pragma unroll
    for (int i = 0; i < 19; ++i) f[i] = rec[i];
    collide(op, f);
#pragma unroll
    for (int i = 0; i < 19; ++i) rec[i] = f[i];
  }
}

// AA odd: write back window plane z of the in-place field (owned slots only).
// Work items, round-robin over the 8 warps: the halves (by column) of the
// rows that are written slot by slot throughout, then the rows whose interior
// records are owned whole (one 16-byte vector run plus the 4 rim columns
// 0, 1, txv, txv+1 slot by slot). Lanes first compute the 19-bit ownership
// mask of each of the item's columns (into msk), then store element-parallel
// (coalesced, with holes). A slot is written back when the node that writes
// it in this sweep belongs to the block (AA odd: slot (k, R) is written by R
// if link opp k of R bounces, else by R - c_k; SWAP and ET: see the mode list
// at the top).
// slot k's owner, as a window position offset from R (no bounce at R)
template <int MODE>
__device__ __forceinline__ constexpr int owner_sign(int k) {
  if constexpr (MODE == kWinSwap) {
    // back slot: swapped by R itself; forward slot: by R + c_k
    return (cz(k) < 0 || (cz(k) == 0 && (cy(k) < 0 || (cy(k) == 0 && cx(k) < 0)))) ? 0 : 1;
  } else {
    return -1;  // AA odd: R - c_k
  }
}
// ET: logical direction held in physical slot s, and whether it is the
// second member of its pair
template <int MODE>
__device__ __forceinline__ constexpr int et_dir(int s) {
  return MODE == kWinEtS ? opp(s) : s;
}
// the directions with c_z = +1
__device__ constexpr int kUp[5] = {5, 9, 12, 14, 17};
__device__ __forceinline__ constexpr bool second_member(int d) {
  return d == 2 || d == 4 || d == 6 || (d >= 13 && d <= 18);
}
template <int MODE>
__device__ __forceinline__ uint32_t owned_slots(const Lat& L, const Tile& t, int rx, int r, int z) {
  uint32_t bR = 0;
  const bool fR = win_cell(L, t, rx, r, z, bR);
  const bool selfin = in_block(t, rx, r, z);
  uint32_t m = 0;
  if constexpr (is_et(MODE)) {
#pragma unroll
    for (int s = 0; s < 19; ++s) {
      const int d = et_dir<MODE>(s);
      bool own;
      if (!second_member(d))
        own = fR && selfin;  // written by R itself (mailboxes: by nobody)
      else if (fR && ((bR >> d) & 1u))
        own = selfin;
      else
        own = in_block(t, rx + cx(d), r + cy(d), z + cz(d));
      m |= own ? (1u << s) : 0u;
    }
    return m;
  }
  if (!fR) return 0;  // AA / SWAP: solids and halo records are never written
  m = selfin ? 1u : 0u;
#pragma unroll
  for (int k = 1; k < 19; ++k) {
    bool own;
    const int sg = owner_sign<MODE>(k);
    if ((MODE == kWinAaOdd || MODE == kWinPushS) && ((bR >> opp(k)) & 1u))
      own = selfin;  // AA odd: a bounced link's slot is written by R itself
    else
      own = in_block(t, rx + sg * cx(k), r + sg * cy(k), z + sg * cz(k));
    m |= own ? (1u << k) : 0u;
  }
  return m;
}
// the same for a fluid record with no bounce link on a plane strictly inside
// the chunk: depends on the window position only (one table per block)
template <int MODE>
__device__ __forceinline__ uint32_t owned_slots_xy(const Tile& t, int rx, int r) {
  auto in_xy = [&](int a, int b) { return a >= 1 && a <= t.txv && b >= 1 && b <= t.tyv; };
  uint32_t m = 0;
  if constexpr (is_et(MODE)) {
#pragma unroll
    for (int s = 0; s < 19; ++s) {
      const int d = et_dir<MODE>(s);
      const bool own = second_member(d) ? in_xy(rx + cx(d), r + cy(d)) : in_xy(rx, r);
      m |= own ? (1u << s) : 0u;
    }
    return m;
  }
  m = in_xy(rx, r) ? 1u : 0u;
#pragma unroll
  for (int k = 1; k < 19; ++k) {
    const int sg = owner_sign<MODE>(k);
    m |= in_xy(rx + sg * cx(k), r + sg * cy(k)) ? (1u << k) : 0u;
  }
  return m;
}

// the z part of the ownership rule for window plane z of a chunk [zb, ze):
// slot k's writer sits at z + dz(k), dz = 0 (written by the record itself) or
// the owner offset's z component; all ones strictly inside the chunk
template <int MODE>
__device__ __forceinline__ uint32_t zmask_of(const Tile& t, int z) {
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < 19; ++k) {
    int dz;
    if constexpr (is_et(MODE)) {
      const int d = et_dir<MODE>(k);
      dz = second_member(d) ? cz(d) : 0;
    } else {
      dz = k == 0 ? 0 : owner_sign<MODE>(k) * cz(k);
    }
    m |= (z + dz >= t.zb && z + dz < t.ze) ? (1u << k) : 0u;
  }
  return m;
}

template <int MODE, class T>
__device__ __forceinline__ void writeback_plane(const Lat& L, T* __restrict__ g, const T* buf,
                                                const int* ph, uint32_t* msk, int* mcol,
                                                const uint32_t* gmask, const Tile& t, int z,
                                                int warp0 = 0, int nwarps = 0) {
  // the warps [warp0, warp0 + nwarps) do the work (default: the whole block)
  if (nwarps == 0) nwarps = (int)(blockDim.x >> 5);
  const int warp = (int)(threadIdx.x >> 5) - warp0, lane = threadIdx.x & 31;
  const bool zin = z >= t.zb + 1 && z <= t.ze - 2;
  const int w = t.txv + 2, rows = t.tyv + 2;
  const bool can_run = zin && t.txv >= 3;
  // rows with a run: r in [2, tyv-1] when can_run; the others are split in two
  const int nrun = can_run ? max(0, t.tyv - 2) : 0;
  const int nfull = rows - nrun;
  const int nitems = 2 * nfull + nrun;
  for (int it = warp; it < nitems; it += nwarps) {
    int r, c0, c1;  // row, column range [c0, c1) for the slot-by-slot pass
    bool run;
    if (it < 2 * nfull) {
      const int fr = it >> 1;  // fr-th row without a run
      r = (!can_run || fr < 2) ? fr : fr + nrun;
      const int half = (w + 1) / 2;
      c0 = (it & 1) ? half : 0;
      c1 = (it & 1) ? w : half;
      run = false;
    } else {
      r = 2 + (it - 2 * nfull);
      c0 = 0;
      c1 = 4;
      run = true;
    }
    uint32_t rb;
    if (!row_base(L, t.y0 - 1 + r, z, rb)) continue;
    const T* srow = buf + r * WinSz<T>::ROW + ph[r];
    // per column q of the item (the range [c0, c1), or the rim list of a run
    // row): ownership mask and storage x
    uint32_t* mk = msk + warp * kWC;
    int* mc = mcol + warp * kWC;
    auto col_of = [&](int q) { return run ? (q < 2 ? q : t.txv + q - 2) : q; };
    for (int q = c0 + lane; q < c1; q += 32) {
      const int rx = col_of(q);
      int xs = 0;
      uint32_t m = 0;
      if (col_xs(L, t.x0, rx, xs)) {
        uint32_t bR = 0;
        if (zin && win_cell(L, t, rx, r, z, bR) && bR == 0)
          m = gmask[r * kWC + rx];
        else
          m = owned_slots<MODE>(L, t, rx, r, z);
      }
      mk[q - c0] = m;
      mc[q - c0] = xs;
    }
    __syncwarp();
    if (run)
      copy_out(g + ((size_t)rb + (size_t)(L.ox + t.x0 + 1)) * 19, srow + 2 * 19, (t.txv - 2) * 19,
               lane);
    const int n = (c1 - c0) * 19;
    // element e = lane + 32 j: column qq = e / 19, slot k = e % 19 (stepped)
    int qq = lane / 19, k = lane - qq * 19;
    for (int e = lane; e < n; e += 32) {
      if ((mk[qq] >> k) & 1u) {
        const int rx = col_of(c0 + qq), xs = mc[qq];
        g[((size_t)rb + (size_t)xs) * 19 + k] = srow[rx * 19 + k];
      }
      k += 13;  // 32 = 19 + 13
      qq += 1;
      if (k >= 19) {
        k -= 19;
        qq += 1;
      }
    }
    __syncwarp();
  }
}

// Compact write-back (in-place modes, the planes strictly inside the chunk of
// a block whose tile touches no x/y wall, all-fluid lattice): every record of
// such a plane has no bounce link, so its owned slots depend on the window
// position only (gmask). The block lists, once, the owned (row, column, slot)
// elements outside the whole-record runs; a plane's write-back is then the
// runs (16-byte vectors, one warp per row) plus one strided pass of all
// threads over the list. Entry: row << 12 | column class << 10 | column * 19
// + slot; class 1 / 2 = window column 0 / w - 1 (their storage x may wrap),
// 0 = the others.
constexpr int kListMax = 4 * kWC * 19 + (kWR - 4) * 4 * 19;  // tyv >= 3: 4 full rows + rims
// static shared memory of an in-place window block (k_win below); fp32 must
// keep two blocks per SM (228 KB per SM, 1 KB reserved per block)
constexpr size_t kInPlaceStatic = kNB * kWR * 4 + 8 * kWC * 4 * 2 + kWR * kWC * 4 + kListMax * 2 +
                                  (kWR + 1) * 4 + kWR * 8 + kWR * 4 + kNB * 8;
static_assert(2 * (WinSz<float>::kBytes + kInPlaceStatic + 1024) <= 228 * 1024,
              "fp32 in-place window no longer fits two blocks per SM");

struct WbList {
  uint16_t* e;      // entries: row << 11 | column << 5 | slot
  int n;            // entry count
  long long colb0;  // element offset of window column 0 (unwrapped): storage x of column q = x0 - 1 + ox + q
  int d1, d2;       // + element correction of column 0 / column w - 1 when their x wraps
};

// fast-path eligibility of the block (uniform)
__device__ __forceinline__ bool wb_fast_ok(const Lat& L, const Tile& t) {
  if (L.linkmask || t.txv < 3 || t.tyv < 3) return false;
  if (L.wall[0] && (t.x0 == 0 || t.x0 + t.txv == L.nx)) return false;
  if (L.wall[1] && (t.y0 == 0 || t.y0 + t.tyv == L.ny)) return false;
  return true;
}

// build the block's list (all threads; cnt = kWR + 1 ints of scratch)
__device__ __forceinline__ int wb_build(const Lat& L, const Tile& t, const uint32_t* gmask,
                                        uint16_t* list, int* cnt) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = (int)(blockDim.x >> 5);
  const int w = t.txv + 2, rows = t.tyv + 2;
  auto row_cols = [&](int r, int j) {  // j-th slot-by-slot column of row r
    const bool run = r >= 2 && r <= t.tyv - 1;
    return run ? (j < 2 ? j : t.txv + j - 2) : j;
  };
  auto row_ncols = [&](int r) { return (r >= 2 && r <= t.tyv - 1) ? 4 : w; };
  for (int pass = 0; pass < 2; ++pass) {
    for (int r = warp; r < rows; r += nw) {
      const int ne = row_ncols(r) * 19;
      int pos = pass ? cnt[r] : 0;
      for (int b = 0; b < ne; b += 32) {
        const int e = b + lane;
        bool own = false;
        int q = 0, k = 0;
        if (e < ne) {
          const int j = e / 19;
          k = e - j * 19;
          q = row_cols(r, j);
          own = (gmask[r * kWC + q] >> k) & 1u;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, own);
        if (pass && own)
          list[pos + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)((r << 11) | (q << 5) | k);
        pos += __popc(bal);
      }
      if (!pass && lane == 0) cnt[r] = pos;
    }
    __syncthreads();
    if (!pass && threadIdx.x == 0) {  // counts -> offsets
      int s = 0;
      for (int r = 0; r < rows; ++r) {
        const int c = cnt[r];
        cnt[r] = s;
        s += c;
      }
      cnt[rows] = s;
    }
    __syncthreads();
  }
  return cnt[rows];
}

// one plane's write-back from its ring slot (rbp / sbp: the plane's per-row
// element offset of window column 0 in storage and in the ring, published
// before the barrier). zm = the plane's z ownership mask: all ones strictly
// inside the chunk (the run records leave whole), else (a chunk face or halo
// plane of a bounce-free block) only the slots in zm, runs included.
template <class T>
__device__ __forceinline__ void writeback_fast(T* __restrict__ g, const T* ring, const WbList& wl,
                                               const long long* rbp, const int* sbp,
                                               const Tile& t, uint32_t zm = ~0u, int warp0 = 0,
                                               int nwarps = 0) {
  // the warps [warp0, warp0 + nwarps) do the work (default: the whole block)
  if (nwarps == 0) nwarps = (int)(blockDim.x >> 5);
  const int warp = (int)(threadIdx.x >> 5) - warp0, lane = threadIdx.x & 31, nw = nwarps;
  const int tid = (int)threadIdx.x - 32 * warp0, nthr = 32 * nwarps;
  const int w = t.txv + 2;
  if (zm == ~0u) {  // runs: rows 2 .. tyv-1, columns 2 .. txv-1, whole records
    for (int r = 2 + warp; r <= t.tyv - 1; r += nw)
      if constexpr (kBulk)
        copy_out_bulk(g + rbp[r] + 2 * 19, ring + sbp[r] + 2 * 19, (t.txv - 2) * 19, lane);
      else
        copy_out(g + rbp[r] + 2 * 19, ring + sbp[r] + 2 * 19, (t.txv - 2) * 19, lane);
  } else {  // the run records' zm slots
    const int nk = __popc(zm), ncol = t.txv - 2, nrun = max(0, t.tyv - 2);
    const int n = nrun * ncol * nk;
    for (int e = tid; e < n; e += nthr) {
      const int kk = e % nk, rc = e / nk, r = 2 + rc / ncol, q = 2 + rc % ncol;
      const int off = q * 19 + (int)__fns(zm, 0, kk + 1);
      g[rbp[r] + off] = ring[sbp[r] + off];
    }
  }
  for (int e = tid; e < wl.n; e += nthr) {
    const uint32_t v = wl.e[e];
    const int r = (int)(v >> 11), q = (int)((v >> 5) & 63u), k = (int)(v & 31u);
    if (!((zm >> k) & 1u)) continue;
    const int off = q * 19 + k;
    const int dq = q == 0 ? wl.d1 : (q == w - 1 ? wl.d2 : 0);
    g[rbp[r] + (off + dq)] = ring[sbp[r] + off];
  }
}

// per-node body: gather (pull form) or in-place AA odd, BB = some lane of the
// warp has a bounce link
template <int MODE, bool BB, class T, class At>
__device__ __forceinline__ void win_node(const Trt<T>& op, uint32_t bounce, T (&f)[19], At at,
                                         uint32_t wrapped = 0) {
  if constexpr (is_et(MODE)) {
    constexpr bool SW = MODE == kWinEtS;
    f[0] = at(0, 0);
#pragma unroll
    for (int p = 0; p < 9; ++p) {
      const int i = pair_i(p), j = pair_j(p);
      f[i] = at(0, hb<SW>(i));
      f[j] = at(i, (BB && ((bounce >> i) & 1u)) ? hb<SW>(i) : hb<SW>(j));
    }
    collide(op, f);
    at(0, 0) = f[0];
#pragma unroll
    for (int p = 0; p < 9; ++p) {
      const int i = pair_i(p), j = pair_j(p);
      at(0, (BB && ((bounce >> j) & 1u)) ? hb<SW>(j) : hb<SW>(i)) = f[j];
      at(i, hb<SW>(j)) = f[i];
    }
  } else if constexpr (MODE == kWinSwap) {
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const int i = back_dir(k);
      if ((BB && ((bounce >> i) & 1u)) || ((wrapped >> i) & 1u)) continue;
      T& a = at(0, i);
      T& b = at(i, opp(i));
      const T va = a;
      a = b;
      b = va;
    }
  } else if constexpr (MODE == kWinAaOdd) {
    f[0] = at(0, 0);
#pragma unroll
    for (int i = 1; i < 19; ++i) {
      const int j = opp(i);
      f[i] = (BB && ((bounce >> j) & 1u)) ? at(0, i) : at(j, j);
    }
    collide(op, f);
    at(0, 0) = f[0];
#pragma unroll
    for (int j = 1; j < 19; ++j) {
      if (BB && ((bounce >> j) & 1u))
        at(0, opp(j)) = f[j];
      else
        at(j, j) = f[j];
    }
  } else {
    f[0] = at(0, 0);
#pragma unroll
    for (int i = 1; i < 19; ++i) {
      const int j = opp(i);
      f[i] = (BB && ((bounce >> j) & 1u)) ? at(0, j) : at(j, i);
    }
    if constexpr (MODE == kWinPull) collide(op, f);
  }
}

template <class T, int MODE>
__global__ void __launch_bounds__(WinThreads<T, MODE>::value, sizeof(T) == 8 ? 1 : 2)
    k_win(Fld<T, true> src, Fld<T, true> dst, Lat L, Trt<T> op, int tiles_x, int tiles_y, int zc,
          int z0, int z1, const T* wlo, const T* whi) {
  extern __shared__ __align__(16) unsigned char win_smem[];
  T* sm = reinterpret_cast<T*>(win_smem);
  __shared__ int ph[kNB][kWR];
  __shared__ uint32_t msk[owned_wb(MODE) ? WinThreads<T, MODE>::warps * kWC : 1];
  __shared__ int mcol[owned_wb(MODE) ? WinThreads<T, MODE>::warps * kWC : 1];
  __shared__ uint32_t gmask[owned_wb(MODE) ? kWR * kWC : 1];
  __shared__ uint16_t wlist[owned_wb(MODE) ? kListMax : 1];
  __shared__ int wcnt[kWR + 1];
  __shared__ long long rbp[kWR];  // write-back plane: row storage bases (elements)
  __shared__ int sbp[kWR];        // ... and ring offsets
  __shared__ __align__(8) uint64_t lbar[kNB];  // ring slot s: bulk bytes of its current load
  constexpr int BUF = WinSz<T>::BUF, ROW = WinSz<T>::ROW;

  const int ntile = tiles_x * tiles_y;
  const int tile = (int)blockIdx.x % ntile, chunk = (int)blockIdx.x / ntile;
  Tile t;
  t.x0 = (tile % tiles_x) * kTX;
  t.y0 = (tile / tiles_x) * kTY;
  t.txv = min(kTX, L.nx - t.x0);
  t.tyv = min(kTY, L.ny - t.y0);
  t.zb = z0 + chunk * zc;  // planes [z0, z1) in chunks of zc
  t.ze = min(z1, t.zb + zc);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const bool valid = tx < t.txv && ty < t.tyv;
  const T* gin = src.p;
  if constexpr (owned_wb(MODE)) {  // ownership masks of no-bounce records inside the chunk
    for (int q = threadIdx.x; q < kWR * kWC; q += blockDim.x)
      gmask[q] = owned_slots_xy<MODE>(t, q % kWC, q / kWC);
  }
  WbList wl{wlist, 0, 0, 0, 0};
  bool fast = false;
  if constexpr (owned_wb(MODE)) {
    fast = wb_fast_ok(L, t);
    if (fast) {
      __syncthreads();  // gmask
      wl.n = wb_build(L, t, gmask, wlist, wcnt);
      int xs0 = 0, xs1 = 0;
      col_xs(L, t.x0, 0, xs0);
      col_xs(L, t.x0, t.txv + 1, xs1);
      wl.colb0 = (long long)(t.x0 - 1 + L.ox) * 19;
      wl.d1 = (xs0 - (t.x0 - 1 + L.ox)) * 19;
      wl.d2 = (xs1 - (t.x0 + t.txv + L.ox)) * 19;
    }
  }
  // plane zp is written back by the compact pass
  auto fast_plane = [&](int zp) { return fast && zp >= t.zb + 1 && zp <= t.ze - 2; };
  // a fast block's other planes: gmask & zmask when the plane is a bounce-free
  // domain plane (not a z-wall face, not an ET mailbox halo plane)
  auto face_zm = [&](int zp) -> uint32_t {
    int zcell;
    if (!fast || !axis_cell(zp, L.nz, L.wall[2], L.oz, zcell)) return 0u;
    if (L.wall[2] && (zcell == 0 || zcell == L.nz - 1)) return 0u;
    return zmask_of<MODE>(t, zp);
  };
  // ring slot of window plane z (z in [zb - 1, ze])
  auto slot = [&](int z) { return (z - t.zb + 1) & (kNB - 1); };
  auto load = [&](int z) {
    load_plane(L, gin, sm + slot(z) * BUF, ph[slot(z)], t, z, wlo, whi, &lbar[slot(z)]);
  };
  // parity of the k-th load into a slot: k & 1
  auto wait_plane = [&](int z) { mbar_wait(&lbar[slot(z)], (uint32_t)((z - t.zb + 1) >> 2) & 1u); };
  if constexpr (kBulk) {
    if (threadIdx.x == 0) {
      for (int b = 0; b < kNB; ++b) mbar_init(&lbar[b], (uint32_t)(t.tyv + 2) * kRowArrivals);
      mbar_fence_init();
    }
    __syncthreads();
  }

  // Schedule per plane z: wait for plane z + 1, barrier (every warp has also
  // finished plane z - 1, so slot(z + 2) = slot(z - 2) is free), prefetch
  // plane z + 2, compute, barrier (plane z - 1 fully read), then each warp
  // stages / writes back its rows of plane z - 1's slot.
  load(t.zb - 1);
  load(t.zb);
  cp_commit();
  T pc[19];             // kWinPushS: post-collision values of this thread's node, plane z
  bool pc_live = false;
  T pd[5];              // ... and the deferred cz = +1 values of plane z - 1
  bool pd_live = false;
  uint32_t pd_mask = 0;
  WIN_T0();
  for (int z = t.zb; z < t.ze; ++z) {
    if (z == t.zb) load(z + 1);
    WIN_T(0);
    if constexpr (kBulk) {
      // every warp is done with plane z - 2's slot (compute of z - 1, write-back
      // of z - 2 and its bulk stores' reads): refill it with plane z + 2, then
      // wait for plane z + 1 (two planes in flight while waiting)
      bulk_wait_read();
      fence_async_smem();
      __syncthreads();
      WIN_T(1);  // previous plane's stragglers (barrier)
      if (z + 2 <= t.ze) load(z + 2);
      WIN_T(2);  // issuing the prefetch
      if (z == t.zb) {
        wait_plane(z - 1);
        wait_plane(z);
      }
      wait_plane(z + 1);
      WIN_T(3);  // waiting for plane z + 1
    } else {
      cp_commit();
      if (z == t.zb) cp_wait1(); else cp_wait0();
      __syncthreads();
      if (z == t.zb) {
        cp_wait0();  // plane z + 1 of the prologue
        __syncthreads();
      }
      if (z + 2 <= t.ze) load(z + 2);
    }
    if constexpr (MODE == kWinPush) {
      if (z == t.zb) {
        collide_plane(L, op, sm + slot(z - 1) * BUF, ph[slot(z - 1)], t, z - 1);
        collide_plane(L, op, sm + slot(z) * BUF, ph[slot(z)], t, z);
      }
      collide_plane(L, op, sm + slot(z + 1) * BUF, ph[slot(z + 1)], t, z + 1);
      __syncthreads();
    }
    T f[19];
    bool live = false;
    if constexpr (MODE == kWinPushS) {
      // Scatter form of OS push: this thread's node X at plane z writes
      // post(X)[i] into slot i of X + c_i (bounce: slot opp i of X) in the
      // ring; plane z - 1 is then complete and leaves through the ownership
      // write-back (the owner of slot (k, R) is R - c_k, as for AA odd), so
      // no halo node is collided. The cz = +1 values land one iteration
      // later (pd), after every tile record of plane z + 1 has been read
      // (this iteration, before the barrier); cz <= 0 targets were read in
      // earlier iterations.
      const int x = t.x0 + tx, y = t.y0 + ty;
      auto own = [&](int zp) -> const T* {
        const int sl = slot(zp);
        return sm + sl * BUF + (ty + 1) * ROW + ph[sl][ty + 1] + (tx + 1) * 19;
      };
      auto nbr = [&](int zp) {  // element offsets of the 3 x 3 (z, y) neighbourhood
        int rp[3][3];
#pragma unroll
        for (int dz = 0; dz < 3; ++dz)
#pragma unroll
          for (int dy = 0; dy < 3; ++dy) {
            const int sl = slot(zp - 1 + dz), r = ty + dy;
            rp[dz][dy] = sl * BUF + r * ROW + ph[sl][r] + (tx + 1) * 19;
          }
        return [=](int i, int k) -> T& { return sm[rp[1 + cz(i)][1 + cy(i)] + cx(i) * 19 + k]; };
      };
      uint32_t bz = 0;
      if (z == t.zb) {  // plane zb's post values
        pc_live = valid && cell_links(L, x, y, z, bz);
        if (pc_live) {
          const T* rec = own(z);
#pragma unroll
          for (int i = 0; i < 19; ++i) pc[i] = rec[i];
          collide(op, pc);
        }
      }
      T fr[19];  // plane z + 1, pristine: nothing has landed in it yet
      bool rlive = false;
      if (z + 1 < t.ze && valid) rlive = cell_links(L, x, y, z + 1, bz);
      if (rlive) {
        const T* rec = own(z + 1);
#pragma unroll
        for (int i = 0; i < 19; ++i) fr[i] = rec[i];
      }
      if (pd_live) {  // plane z - 1's deferred cz = +1 values into plane z
        auto at = nbr(z - 1);
#pragma unroll
        for (int q = 0; q < 5; ++q)
          if ((pd_mask >> kUp[q]) & 1u) at(kUp[q], kUp[q]) = pd[q];
      }
      if (pc_live) {
        auto at = nbr(z);
        uint32_t bounce = 0;
        cell_links(L, x, y, z, bounce);
        at(0, 0) = pc[0];
#pragma unroll
        for (int i = 1; i < 19; ++i) {
          if ((bounce >> i) & 1u)
            at(0, opp(i)) = pc[i];
          else if (cz(i) <= 0)
            at(i, i) = pc[i];
        }
        // a bounced cz = +1 link was written above; the deferred store of its
        // slot is skipped
#pragma unroll
        for (int q = 0; q < 5; ++q) pd[q] = pc[kUp[q]];
        pd_mask = ~bounce;
      }
      pd_live = pc_live;
      if (rlive) {
        collide(op, fr);
#pragma unroll
        for (int i = 0; i < 19; ++i) pc[i] = fr[i];
      }
      pc_live = rlive;
    } else if (ty < kTY) {  // warps beyond the tile rows only move data
      // element offsets of the 3 x 3 (z, y) neighbourhood at this thread's column
      int rp[3][3];
#pragma unroll
      for (int dz = 0; dz < 3; ++dz)
#pragma unroll
        for (int dy = 0; dy < 3; ++dy) {
          const int s = slot(z - 1 + dz), r = ty + dy;
          rp[dz][dy] = s * BUF + r * ROW + ph[s][r] + (tx + 1) * 19;
        }
      auto at = [&](int i, int k) -> T& {  // slot k of the record at X + c_i
        return sm[rp[1 + cz(i)][1 + cy(i)] + cx(i) * 19 + k];
      };
      uint32_t bounce = 0;
      if (valid) live = cell_links(L, t.x0 + tx, t.y0 + ty, z, bounce);
      const bool interior = __all_sync(0xffffffffu, bounce == 0u);
      uint32_t wrapped = 0;
      if constexpr (MODE == kWinSwap) {  // periodic-seam links are the fix-up list's
        const int x = t.x0 + tx, y = t.y0 + ty;
        const bool px = !L.wall[0], py = !L.wall[1], pz = !L.wall[2];
        if (px && x == 0) wrapped |= kMxm;
        if (px && x == L.nx - 1) wrapped |= kMxp;
        if (py && y == 0) wrapped |= kMym;
        if (py && y == L.ny - 1) wrapped |= kMyp;
        if (pz && z == 0) wrapped |= kMzm;
        if (pz && z == L.nz - 1) wrapped |= kMzp;
      }
#ifdef LBM_WIN_NO_COMPUTE
      live = false;  // experiment: load + write-back pipeline only (wrong results)
#endif
      if (live) {
        if (interior)
          win_node<MODE, false>(op, bounce, f, at, wrapped);
        else
          win_node<MODE, true>(op, bounce, f, at, wrapped);
      }
    }
    if constexpr (owned_wb(MODE)) {
      if ((fast_plane(z - 1) || face_zm(z - 1)) && (int)threadIdx.x < t.tyv + 2) {
        const int r = threadIdx.x;
        uint32_t rb = 0;
        row_base(L, t.y0 - 1 + r, z - 1, rb);
        rbp[r] = (long long)rb * 19 + wl.colb0;
        sbp[r] = slot(z - 1) * BUF + r * ROW + ph[slot(z - 1)][r];
      }
      if constexpr (kBulk) fence_async_smem();  // ring writes before the runs' bulk stores
    }
    WIN_T(4);  // compute (+ per-node stores into the ring)
    __syncthreads();  // every read of plane z - 1 is done
    WIN_T(5);  // waiting for the slowest warp's compute
#ifdef LBM_WIN_NO_WB
    if (false)  // experiment: load + compute only (wrong results)
#endif
    if constexpr (owned_wb(MODE)) {
      if (fast_plane(z - 1))
        writeback_fast(dst.p, sm, wl, rbp, sbp, t);
      else if (const uint32_t zm = face_zm(z - 1))
        writeback_fast(dst.p, sm, wl, rbp, sbp, t, zm);
      else
        writeback_plane<MODE>(L, dst.p, sm + slot(z - 1) * BUF, ph[slot(z - 1)], msk, mcol, gmask,
                              t, z - 1);
    } else if (ty < t.tyv) {
      // stage the tile row in plane z - 1's slot with the phase of dst's row
      uint32_t rb;
      row_base(L, t.y0 + ty, z, rb);
      const long long v0 = (long long)rb + L.ox + t.x0;
      const int phase =
          (int)(((reinterpret_cast<uintptr_t>(dst.p) + (uintptr_t)(v0 * 19 * (long long)sizeof(T))) &
                 15u) / sizeof(T));
      T* srow = sm + slot(z - 1) * BUF + ty * ROW + phase;
      if (tx < t.txv) {
#pragma unroll
        for (int i = 0; i < 19; ++i) srow[tx * 19 + i] = live ? f[i] : T(0);
      }
      __syncwarp();
      if constexpr (kBulk)
        copy_out_bulk(dst.p + (size_t)v0 * 19, srow, t.txv * 19, tx);
      else
        copy_out(dst.p + (size_t)v0 * 19, srow, t.txv * 19, tx);
    }
    WIN_T(6);  // write-back / staging of plane z - 1
  }
  if constexpr (kBulk) bulk_wait_all();
  if constexpr (MODE == kWinPushS) {  // plane ze - 1's deferred values into the halo plane
    __syncthreads();
    if (pd_live) {
      const int zp = t.ze - 1;
      auto at = [&](int i, int k) -> T& {
        const int sl = slot(zp + cz(i)), r = ty + 1 + cy(i);
        return sm[sl * BUF + r * ROW + ph[sl][r] + (tx + 1 + cx(i)) * 19 + k];
      };
#pragma unroll
      for (int q = 0; q < 5; ++q)
        if ((pd_mask >> kUp[q]) & 1u) at(kUp[q], kUp[q]) = pd[q];
    }
  }
  if constexpr (owned_wb(MODE)) {  // the chunk's top plane and the halo plane above
    for (int zp = t.ze - 1; zp <= t.ze; ++zp) {
      const uint32_t zm = face_zm(zp);
      __syncthreads();
      if (zm && (int)threadIdx.x < t.tyv + 2) {
        const int r = threadIdx.x;
        uint32_t rb = 0;
        row_base(L, t.y0 - 1 + r, zp, rb);
        rbp[r] = (long long)rb * 19 + wl.colb0;
        sbp[r] = slot(zp) * BUF + r * ROW + ph[slot(zp)][r];
      }
      __syncthreads();
      if (zm)
        writeback_fast(dst.p, sm, wl, rbp, sbp, t, zm);
      else
        writeback_plane<MODE>(L, dst.p, sm + slot(zp) * BUF, ph[slot(zp)], msk, mcol, gmask, t, zp);
    }
  }
}

// ---------------------------------------------------------------------------
// Register-carried z pipeline for the gather modes (OS / OSNT pull, TS
// stream). Node X at plane q reads its 19 values from plane q - 1 (the five
// c_z = +1 directions), plane q (c_z = 0, the rest value and every bounced
// link: own record) and plane q + 1 (c_z = -1). A thread owns one (x, y)
// column of the tile and collects while the planes pass: with plane p in
// the ring it takes the c_z = -1 values of its node p - 1 (then complete:
// collide, stage, store), the c_z = 0 values of node p and the c_z = +1
// values of node p + 1 (five registers carried to the next plane). Every
// plane is read during ONE iteration, so of the NS ring slots one holds the
// plane being read, one (the previous plane's) stages this iteration's
// output records and NS - 2 are loads in flight; k_win keeps three planes
// resident for its gathers and has one in flight. One block barrier per
// plane (the previous slot's reads and the bulk stores' reads of the slot
// before it are done before that slot is refilled).
// ---------------------------------------------------------------------------
#ifndef LBM_ZP_NS64
#define LBM_ZP_NS64 4
#endif
#ifndef LBM_ZP_NS32
#define LBM_ZP_NS32 4
#endif
#ifndef LBM_ZP_TY64
#define LBM_ZP_TY64 8
#endif
#ifndef LBM_ZP_TY32
#define LBM_ZP_TY32 8
#endif
template <class T>
struct ZpCfg {
  static constexpr int TY = sizeof(T) == 8 ? LBM_ZP_TY64 : LBM_ZP_TY32;  // tile rows (row warps)
  static constexpr int NS = sizeof(T) == 8 ? LBM_ZP_NS64 : LBM_ZP_NS32;  // ring slots
  static constexpr int ROW = WinSz<T>::ROW;
  static constexpr int BUF = (TY + 2) * ROW;
  static constexpr size_t kBytes = (size_t)NS * BUF * sizeof(T);
  static constexpr int kThreads = 32 * (TY + 1);  // + one loading warp
  static constexpr int kBlocks = (int)((227 * 1024) / (kBytes + 2048)) > 0 ? (int)((227 * 1024) / (kBytes + 2048)) : 1;
};
// OS push collides every window record of a plane ((TY + 2) x 34) before the
// gathers: extra warps so that is one round of the block, not two
#ifndef LBM_ZP_PUSH_EXTRA
#define LBM_ZP_PUSH_EXTRA 2
#endif
template <class T, int MODE>
struct ZpThreads {
  static constexpr int value =
      MODE == kWinPush ? 32 * (ZpCfg<T>::TY + 1 + LBM_ZP_PUSH_EXTRA) : ZpCfg<T>::kThreads;
};
static_assert(ZpCfg<double>::kBytes <= 227 * 1024 - 1024, "fp64 z-pipeline ring too large");
static_assert(ZpCfg<float>::kBytes <= 227 * 1024 - 1024, "fp32 z-pipeline ring too large");
static_assert(ZpCfg<double>::NS >= 3 && ZpCfg<float>::NS >= 3, "z pipeline: at least one plane in flight");

// the gathers of one plane: node p - 1 (c_z = -1), node p (c_z = 0 and the
// bounced links of every direction), node p + 1 (c_z = +1 into g5)
template <bool BB, class T, class At>
__device__ __forceinline__ void zp_take_prev(T (&f)[19], uint32_t b, At at) {
#pragma unroll
  for (int i = 1; i < 19; ++i)
    if (cz(i) == -1 && !(BB && ((b >> opp(i)) & 1u))) f[i] = at(opp(i), i);
}
template <bool BB, class T, class At>
__device__ __forceinline__ void zp_take_cur(T (&f)[19], const T (&g5)[5], uint32_t b, At at) {
  f[0] = at(0, 0);
#pragma unroll
  for (int i = 1; i < 19; ++i) {
    const int j = opp(i);
    const bool bj = BB && ((b >> j) & 1u);
    if (cz(i) == 0) {
      f[i] = bj ? at(0, j) : at(j, i);
    } else if (cz(i) == 1) {
      int q = 0;
#pragma unroll
      for (int k = 1; k < i; ++k) q += cz(k) == 1 ? 1 : 0;
      f[i] = bj ? at(0, j) : g5[q];
    } else if (bj) {
      f[i] = at(0, j);
    }
  }
}
template <class T, class At>
__device__ __forceinline__ void zp_take_next(T (&g5)[5], At at) {
  int q = 0;
#pragma unroll
  for (int i = 1; i < 19; ++i)
    if (cz(i) == 1) g5[q++] = at(opp(i), i);
}

template <class T, int MODE>
__global__ void __launch_bounds__(ZpThreads<T, MODE>::value, ZpCfg<T>::kBlocks)
    k_win_zp(Fld<T, true> src, Fld<T, true> dst, Lat L, Trt<T> op, int tiles_x, int tiles_y,
             int zc, int z0, int z1, const T* wlo, const T* whi) {
  static_assert(MODE == kWinPull || MODE == kWinStream || MODE == kWinPush,
                "z pipeline: gather modes");
  constexpr int TY = ZpCfg<T>::TY, NS = ZpCfg<T>::NS, ROW = ZpCfg<T>::ROW, BUF = ZpCfg<T>::BUF;
  extern __shared__ __align__(16) unsigned char win_smem[];
  T* sm = reinterpret_cast<T*>(win_smem);
  __shared__ int ph[NS][TY + 2];
  __shared__ __align__(8) uint64_t full[NS];

  const int ntile = tiles_x * tiles_y;
  const int tile = (int)blockIdx.x % ntile, chunk = (int)blockIdx.x / ntile;
  Tile t;
  t.x0 = (tile % tiles_x) * kTX;
  t.y0 = (tile / tiles_x) * TY;
  t.txv = min(kTX, L.nx - t.x0);
  t.tyv = min(TY, L.ny - t.y0);
  t.zb = z0 + chunk * zc;  // planes [z0, z1) in chunks of zc (CG: one plane group)
  t.ze = min(z1, t.zb + zc);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int b = 0; b < NS; ++b) mbar_init(&full[b], (uint32_t)(t.tyv + 2) * kRowArrivals);
    mbar_fence_init();
  }
  __syncthreads();
  const int pb = t.zb - 1, pe = t.ze;  // window planes pb .. pe
  auto slot = [&](int p) { return (p - pb) % NS; };
  auto par = [&](int p) { return (uint32_t)((p - pb) / NS) & 1u; };
  auto load = [&](int p) {
    load_plane(L, (const T*)src.p, sm + slot(p) * BUF, ph[slot(p)], t, p, wlo, whi,
               &full[slot(p)], TY);
  };
  if (warp == TY)
    for (int p = pb; p <= min(pe, pb + NS - 1); ++p) load(p);

  const int tx = lane, ty = warp;
  const bool valid = ty < t.tyv && tx < t.txv;
  const int x = t.x0 + tx, y = t.y0 + ty;
  T f[19], g5[5];
  uint32_t bq = 0;   // bounce mask of the node held in f
  bool lq = false;   // ... and whether it is a fluid cell
  // OS push as a gather of post-collision values: every window record of a
  // plane collides in place before its gathers (the halo records redundantly
  // in both neighbouring tiles: deterministic, identical). Plane p + 1
  // collides in iteration p, after the row warps' gathers from plane p (a
  // different ring slot), so one block barrier per plane orders both and the
  // warps without gathers collide while the row warps gather (LBM_ZP_PUSH_LAG
  // = 0: collide plane p at the top of iteration p, between two barriers)
#ifndef LBM_ZP_PUSH_LAG
#define LBM_ZP_PUSH_LAG 1
#endif
  // the row warps' part of iteration p (gathers from plane p, output of p - 1)
  auto zp_row = [&](int p) {
    mbar_wait(&full[slot(p)], par(p));
    const int s = slot(p);
    int rp[3];
#pragma unroll
    for (int dy = 0; dy < 3; ++dy) rp[dy] = s * BUF + (ty + dy) * ROW + ph[s][ty + dy] + (tx + 1) * 19;
    // slot k of the record at (x + cx(i), y + cy(i)) in plane p
    auto at = [&](int i, int k) -> T { return sm[rp[1 + cy(i)] + cx(i) * 19 + k]; };
    if (p - 1 >= t.zb) {  // node p - 1: its last five values, then collide and store
      const bool plain = __all_sync(0xffffffffu, !lq || bq == 0u);
      if (lq) {
        if (plain)
          zp_take_prev<false>(f, bq, at);
        else
          zp_take_prev<true>(f, bq, at);
        if constexpr (MODE == kWinPull) collide(op, f);
      }
      uint32_t rb;
      row_base(L, y, p - 1, rb);
      const long long v0 = (long long)rb + L.ox + t.x0;
      const int phase = (int)(((reinterpret_cast<uintptr_t>(dst.p) +
                                (uintptr_t)(v0 * 19 * (long long)sizeof(T))) & 15u) / sizeof(T));
      T* srow = sm + slot(p - 1) * BUF + ty * ROW + phase;
      if (tx < t.txv) {
#pragma unroll
        for (int i = 0; i < 19; ++i) srow[tx * 19 + i] = lq ? f[i] : T(0);
      }
      __syncwarp();
      copy_out_bulk(dst.p + (size_t)v0 * 19, srow, t.txv * 19, tx);
    }
    if (p >= t.zb && p < t.ze) {  // node p: c_z = 0, bounced links, c_z = +1 from g5
      uint32_t b = 0;
      const bool l = valid && cell_links(L, x, y, p, b);
      const bool plain = __all_sync(0xffffffffu, !l || b == 0u);
      if (l) {
        if (plain)
          zp_take_cur<false>(f, g5, b, at);
        else
          zp_take_cur<true>(f, g5, b, at);
      }
      bq = b;
      lq = l;
    }
    if (p + 1 >= t.zb && p + 1 < t.ze && valid) zp_take_next(g5, at);  // node p + 1
  };
  constexpr bool kLag = MODE == kWinPush && LBM_ZP_PUSH_LAG;
  if constexpr (kLag) {
    mbar_wait(&full[slot(pb)], par(pb));
    collide_plane(L, op, sm + slot(pb) * BUF, ph[slot(pb)], t, pb);
  }
  for (int p = pb; p <= pe; ++p) {
    // slot(p - 2) staged iteration p - 1's output: its bulk stores must have
    // read it, and every thread is done with plane p - 1 (slot(p - 1) stages
    // this iteration's output)
    bulk_wait_read();
    fence_async_smem();
    __syncthreads();
    if (warp == TY && p - 2 >= pb && p - 2 + NS <= pe) load(p - 2 + NS);
    if constexpr (MODE == kWinPush && !kLag) {
      mbar_wait(&full[slot(p)], par(p));
      collide_plane(L, op, sm + slot(p) * BUF, ph[slot(p)], t, p);
      __syncthreads();
    }
    if (warp != TY && ty < t.tyv) zp_row(p);
    if constexpr (kLag) {
      if (p + 1 <= pe) {
        mbar_wait(&full[slot(p + 1)], par(p + 1));
        collide_plane(L, op, sm + slot(p + 1) * BUF, ph[slot(p + 1)], t, p + 1);
      }
    }
  }
  bulk_wait_all();
}

// ---------------------------------------------------------------------------
// Warp-specialised in-place window (AA odd, ET, SWAP exchange; fp64). The
// plain k_win runs load issue, compute and write-back of a plane in series
// between block barriers (C1 fp64 AA odd: load pipeline alone 0.60 ms, +
// compute 0.31, + write-back 0.43 = 1.35 ms; they add up). Here a 32 x 6
// tile's six row warps compute plane z while the write-back warps (ten)
// write back plane z - 2
// (final once every row warp has computed z - 1) and then refill its ring
// slot with plane z + 3: a 5-plane ring (34 x 8 records per plane, 207 KB
// fp64), hand-offs through mbarriers only:
//   full[s]  the plane in slot s has landed (bulk-copy bytes + cp.async)
//   comp[s]  the six row warps have computed the plane in slot s
// Every slot (k, R) is read and rewritten by exactly one node of an in-place
// sweep, so the row warps need no ordering among themselves; a plane is
// final (write-back) once the row warps computed the plane above it, and a
// row warp can be at most three planes ahead of the write-back (it waits for
// loads that follow the write-back), inside the 5-use parity window.
constexpr int kNBw = 5;
// tile rows (= row warps): fp64 6 (a 34 x 8 window, 5 planes = 207 KB); fp32
// records are half as long, so LBM_WS_TY32 rows (34 x 16 window: the
// slot-by-slot rim rows are 4 of 16 instead of 4 of 8)
#ifndef LBM_WS_TY32
#define LBM_WS_TY32 14
#endif
#ifndef LBM_WS_TY64
#define LBM_WS_TY64 6
#endif
// write-back warps (measured on C1 fp64: 2 -> AA 0.51, 4 -> 0.66, 6 -> 0.67,
// 8 -> 0.74, 10 -> 0.77 of the roofline; the row warps' register cap at 512
// threads costs a few spills); storing the rim slots straight from the row
// warps instead of a list pass measured 0.70
#ifndef LBM_WS_WB
#define LBM_WS_WB 10
#endif
constexpr int kWsWb = LBM_WS_WB;
template <class T>
struct WinSzW {
  static constexpr int TY = sizeof(T) == 8 ? LBM_WS_TY64 : LBM_WS_TY32;  // row warps
  static constexpr int WR = TY + 2;
  static constexpr int kThreads = 32 * (TY + kWsWb);
  static constexpr int kList = 4 * kWC * 19 + (WR - 4) * 4 * 19;
  static constexpr int ROW = WinSz<T>::ROW;
  static constexpr int BUF = WR * ROW;
  static constexpr size_t kBytes = (size_t)kNBw * BUF * sizeof(T);
};
static_assert(WinSzW<double>::kBytes <= 227 * 1024 - 12 * 1024, "fp64 ws ring too large");
static_assert(WinSzW<float>::kBytes <= 227 * 1024 - 16 * 1024, "fp32 ws ring too large");
static_assert(WinSzW<float>::WR <= 32, "one loading lane per window row");

__device__ __forceinline__ void wb_group_sync() {
  asm volatile("bar.sync 1, %0;\n" ::"r"(32 * kWsWb) : "memory");
}

#ifndef LBM_WS_F32
#define LBM_WS_F32 0
#endif
#ifndef LBM_WS_F32_BLOCKS
#define LBM_WS_F32_BLOCKS 1
#endif
template <class T, int MODE>
__global__ void __launch_bounds__(WinSzW<T>::kThreads, sizeof(T) == 8 ? 1 : LBM_WS_F32_BLOCKS)
    k_win_ws(Fld<T, true> fld_, Lat L, Trt<T> op, int tiles_x, int tiles_y, int zc) {
  static_assert(in_place(MODE), "warp-specialised window: in-place modes only");
  extern __shared__ __align__(16) unsigned char win_smem[];
  T* sm = reinterpret_cast<T*>(win_smem);
  T* const g = fld_.p;
  constexpr int kTYw = WinSzW<T>::TY, kWRw = WinSzW<T>::WR, kWsCompute = kTYw;
  __shared__ int ph[kNBw][kWRw];
  __shared__ uint32_t msk[kWsWb * kWC];
  __shared__ int mcol[kWsWb * kWC];
  __shared__ uint32_t gmask[kWRw * kWC];
  __shared__ uint16_t wlist[WinSzW<T>::kList];
  __shared__ int wcnt[kWRw + 1];
  __shared__ long long rbp[kWRw];
  __shared__ int sbp[kWRw];
  __shared__ __align__(8) uint64_t full[kNBw];
  __shared__ __align__(8) uint64_t comp[kNBw];
  constexpr int BUF = WinSzW<T>::BUF, ROW = WinSzW<T>::ROW;

  const int ntile = tiles_x * tiles_y;
  const int tile = (int)blockIdx.x % ntile, chunk = (int)blockIdx.x / ntile;
  Tile t;
  t.x0 = (tile % tiles_x) * kTX;
  t.y0 = (tile / tiles_x) * kTYw;
  t.txv = min(kTX, L.nx - t.x0);
  t.tyv = min(kTYw, L.ny - t.y0);
  t.zb = chunk * zc;
  t.ze = min(L.nz, t.zb + zc);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int q = threadIdx.x; q < kWRw * kWC; q += blockDim.x)
    gmask[q] = owned_slots_xy<MODE>(t, q % kWC, q / kWC);
  WbList wl{wlist, 0, 0, 0, 0};
  const bool fast = wb_fast_ok(L, t);
  if (threadIdx.x == 0) {
    for (int b = 0; b < kNBw; ++b) {
      mbar_init(&full[b], (uint32_t)(t.tyv + 2) * kRowArrivals);
      mbar_init(&comp[b], (uint32_t)kWsCompute);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (fast) {
    wl.n = wb_build(L, t, gmask, wlist, wcnt);  // all threads, block barriers inside
    int xs0 = 0, xs1 = 0;
    col_xs(L, t.x0, 0, xs0);
    col_xs(L, t.x0, t.txv + 1, xs1);
    wl.colb0 = (long long)(t.x0 - 1 + L.ox) * 19;
    wl.d1 = (xs0 - (t.x0 - 1 + L.ox)) * 19;
    wl.d2 = (xs1 - (t.x0 + t.txv + L.ox)) * 19;
  }
  auto slot = [&](int z) { return (z - t.zb + 1) % kNBw; };
  // parity of plane z's phase of full[slot(z)] (every plane zb - 1 .. ze is
  // loaded once) and of comp[slot(z)] (only planes zb .. ze - 1 are computed;
  // slot 0's first plane, zb - 1, is not)
  auto use = [&](int z) { return (uint32_t)((z - t.zb + 1) / kNBw) & 1u; };
  auto cuse = [&](int z) {
    return (uint32_t)((z - t.zb + 1) / kNBw - (slot(z) == 0 ? 1 : 0)) & 1u;
  };
  auto fast_plane = [&](int zp) { return fast && zp >= t.zb + 1 && zp <= t.ze - 2; };
  auto face_zm = [&](int zp) -> uint32_t {
    int zcell;
    if (!fast || !axis_cell(zp, L.nz, L.wall[2], L.oz, zcell)) return 0u;
    if (L.wall[2] && (zcell == 0 || zcell == L.nz - 1)) return 0u;
    return zmask_of<MODE>(t, zp);
  };
  constexpr int kLoader = kWsCompute + kWsWb - 1;  // the last write-back warp issues loads
  auto load = [&](int z) {
    load_plane(L, (const T*)g, sm + slot(z) * BUF, ph[slot(z)], t, z, (const T*)nullptr,
               (const T*)nullptr, &full[slot(z)], kLoader);
  };

  if (warp < kWsCompute) {
    // ---- row warps: compute planes zb .. ze - 1 --------------------------------
    const int tx = lane, ty = warp;
    const bool valid = tx < t.txv && ty < t.tyv;
    for (int z = t.zb; z < t.ze; ++z) {
      if (z == t.zb) {
        mbar_wait(&full[slot(z - 1)], use(z - 1));
        mbar_wait(&full[slot(z)], use(z));
      }
      mbar_wait(&full[slot(z + 1)], use(z + 1));
      int rp[3][3];
#pragma unroll
      for (int dz = 0; dz < 3; ++dz)
#pragma unroll
        for (int dy = 0; dy < 3; ++dy) {
          const int sl = slot(z - 1 + dz), r = ty + dy;
          rp[dz][dy] = sl * BUF + r * ROW + ph[sl][r] + (tx + 1) * 19;
        }
      auto at = [&](int i, int k) -> T& { return sm[rp[1 + cz(i)][1 + cy(i)] + cx(i) * 19 + k]; };
      uint32_t bounce = 0;
      bool live = false;
      if (valid) live = cell_links(L, t.x0 + tx, t.y0 + ty, z, bounce);
      const bool interior = __all_sync(0xffffffffu, bounce == 0u);
      uint32_t wrapped = 0;
      if constexpr (MODE == kWinSwap) {
        const int x = t.x0 + tx, y = t.y0 + ty;
        if (!L.wall[0] && x == 0) wrapped |= kMxm;
        if (!L.wall[0] && x == L.nx - 1) wrapped |= kMxp;
        if (!L.wall[1] && y == 0) wrapped |= kMym;
        if (!L.wall[1] && y == L.ny - 1) wrapped |= kMyp;
        if (!L.wall[2] && z == 0) wrapped |= kMzm;
        if (!L.wall[2] && z == L.nz - 1) wrapped |= kMzp;
      }
      T f[19];
      if (live) {
        if (interior)
          win_node<MODE, false>(op, bounce, f, at, wrapped);
        else
          win_node<MODE, true>(op, bounce, f, at, wrapped);
      }
      if constexpr (kBulk) fence_async_smem();  // ring writes before the write-back's bulk stores
      __syncwarp();
      if (lane == 0) mbar_arrive(&comp[slot(z)], 1);
    }
    return;
  }

  // ---- write-back warps: plane zp once the row warps computed zp + 1, then
  // refill its slot with plane zp + kNBw ------------------------------------
  const int w0 = kWsCompute;
  if (warp == kLoader)
    for (int z = t.zb - 1; z <= min(t.ze, t.zb - 1 + kNBw - 1); ++z) load(z);
  auto writeback = [&](int zp) {
    const uint32_t zm = fast_plane(zp) ? ~0u : face_zm(zp);
    if (zm) {
      const int r = (int)threadIdx.x - 32 * w0;
      if (r < t.tyv + 2) {
        uint32_t rb = 0;
        row_base(L, t.y0 - 1 + r, zp, rb);
        rbp[r] = (long long)rb * 19 + wl.colb0;
        sbp[r] = slot(zp) * BUF + r * ROW + ph[slot(zp)][r];
      }
      wb_group_sync();
      writeback_fast(g, sm, wl, rbp, sbp, t, zm, w0, kWsWb);
    } else {
      writeback_plane<MODE>(L, g, sm + slot(zp) * BUF, ph[slot(zp)], msk, mcol, gmask, t, zp, w0,
                            kWsWb);
    }
    if constexpr (kBulk) bulk_wait_read();  // the slot's bulk stores have read it
    wb_group_sync();
  };
  for (int z = t.zb; z < t.ze; ++z) {
    mbar_wait(&comp[slot(z)], cuse(z));
    writeback(z - 1);
    if (warp == kLoader && z - 1 + kNBw <= t.ze) load(z - 1 + kNBw);
  }
  writeback(t.ze - 1);
  writeback(t.ze);
  if constexpr (kBulk) bulk_wait_all();
}

// ---------------------------------------------------------------------------
// Local AoS sweep (AA even, TS collide, OS precollide, SWAP collide) as a
// persistent stream: each block walks 256-record runs with a two-slot
// cp.async ring, so the next run's loads are in flight while this run
// collides in shared memory and leaves as 16-byte vector stores.
// ---------------------------------------------------------------------------
constexpr int kRun = 256;
template <class T>
struct RunSz {
  static constexpr int V = 16 / (int)sizeof(T);
  static constexpr int SLOT = ((kRun * 19 + V + V - 1) / V) * V;
  static constexpr size_t kBytes = 2 * (size_t)SLOT * sizeof(T);
};

template <class T, bool RD_OPP, bool WR_OPP>
__global__ void __launch_bounds__(kRun, MinBlocks<T>::value)
    k_local_stream(Fld<T, true> src, Fld<T, true> dst, Lat L, Trt<T> op, uint32_t soff,
                   uint32_t nruns) {
  extern __shared__ __align__(16) unsigned char run_smem[];
  T* sm = reinterpret_cast<T*>(run_smem);
  constexpr int SLOT = RunSz<T>::SLOT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto phase_of = [&](uint32_t c0) {
    return (int)((((unsigned long long)(c0 + soff) * 19ull * sizeof(T)) & 15ull) / sizeof(T));
  };
  // the block's k-th run and its record count
  auto run_c0 = [&](uint32_t k) { return L.cell_begin + (blockIdx.x + k * gridDim.x) * kRun; };
  auto issue = [&](uint32_t k) {
    const uint32_t c0 = run_c0(k);
    const uint32_t nrec = min((uint32_t)kRun, L.ncells - c0);
    // 8 warps split the contiguous run into 8 pieces
    const uint32_t nel = nrec * 19, per = (nel + 7) / 8;
    const uint32_t e0 = min(nel, (uint32_t)warp * per), e1 = min(nel, e0 + per);
    T* s = sm + (k & 1) * SLOT + phase_of(c0);
    if (e1 > e0) copy_in(s + e0, src.p + (size_t)(c0 + soff) * 19 + e0, (int)(e1 - e0), lane);
  };
  uint32_t nmine = 0;
  while (blockIdx.x + nmine * gridDim.x < nruns) ++nmine;
  if (nmine == 0) return;
  auto compute = [&](uint32_t k) {
    const uint32_t c0 = run_c0(k);
    const uint32_t nrec = min((uint32_t)kRun, L.ncells - c0);
    T* s = sm + (k & 1) * SLOT + phase_of(c0);
    const uint32_t r = threadIdx.x;
    if (r < nrec && (L.linkmask ? (L.linkmask[c0 + r] & 1u) != 0 : true)) {
      T f[19];
#pragma unroll
      for (int i = 0; i < 19; ++i) f[i] = s[r * 19 + (RD_OPP ? opp(i) : i)];
      collide(op, f);
#pragma unroll
      for (int i = 0; i < 19; ++i) s[r * 19 + (WR_OPP ? opp(i) : i)] = f[i];
    }
  };
  if constexpr (kBulk) {
    // warp 0 moves each run: one bulk copy in (bytes on the slot's mbarrier,
    // head / tail by cp.async) and one bulk copy out
    __shared__ __align__(8) uint64_t rbar[2];
    if (threadIdx.x == 0) {
      mbar_init(&rbar[0], kRowArrivals);
      mbar_init(&rbar[1], kRowArrivals);
      mbar_fence_init();
    }
    __syncthreads();
    auto issue_bulk = [&](uint32_t k) {
      const uint32_t c0 = run_c0(k);
      const uint32_t nrec = min((uint32_t)kRun, L.ncells - c0);
      if (LBM_AOS_SUPERSET)
        copy_in_bulk_superset(sm + (k & 1) * SLOT + phase_of(c0),
                              src.p + (size_t)(c0 + soff) * 19, (int)(nrec * 19), lane,
                              &rbar[k & 1]);
      else
        copy_in_bulk(sm + (k & 1) * SLOT + phase_of(c0), src.p + (size_t)(c0 + soff) * 19,
                     (int)(nrec * 19), lane, &rbar[k & 1]);
    };
    if (warp == 0) issue_bulk(0);
    for (uint32_t k = 0; k < nmine; ++k) {
      // run k - 1's slot: its collisions are done and its bulk store has read it
      bulk_wait_read();
      fence_async_smem();
      __syncthreads();
      if (warp == 0 && k + 1 < nmine) issue_bulk(k + 1);
      mbar_wait(&rbar[k & 1], (k >> 1) & 1u);
      compute(k);
      fence_async_smem();
      __syncthreads();
      if (warp == 0) {
        const uint32_t c0 = run_c0(k);
        const uint32_t nrec = min((uint32_t)kRun, L.ncells - c0);
        copy_out_bulk(dst.p + (size_t)(c0 + soff) * 19, sm + (k & 1) * SLOT + phase_of(c0),
                      (int)(nrec * 19), lane);
      }
    }
    bulk_wait_all();
    return;
  }
  issue(0);
  cp_commit();
  for (uint32_t k = 0; k < nmine; ++k) {
    if (k + 1 < nmine) issue(k + 1);
    cp_commit();
    cp_wait1();
    __syncthreads();
    compute(k);
    __syncthreads();
    const uint32_t c0 = run_c0(k);
    const uint32_t nrec = min((uint32_t)kRun, L.ncells - c0);
    T* s = sm + (k & 1) * SLOT + phase_of(c0);
    const uint32_t nel = nrec * 19, per = (nel + 7) / 8;
    const uint32_t e0 = min(nel, (uint32_t)warp * per), e1 = min(nel, e0 + per);
    if (e1 > e0) copy_out(dst.p + (size_t)(c0 + soff) * 19 + e0, s + e0, (int)(e1 - e0), lane);
    __syncthreads();  // the slot is refilled two runs later
  }
}

// z planes per block of a z-marching window: blocks of equal length run in
// waves of `resident`, a block's time ~ its planes + `halo` prologue planes,
// so pick the chunk (4 .. 64 planes) minimising waves x (chunk + halo)
// (C4: nz = 200 over 175 tiles: 34-plane chunks = 7.1 waves -> 8; 40-plane
// chunks = 5.9 -> 6 waves), ties to the longer chunk
static long long wave_chunk(long long nz, long long tiles, long long resident, int halo,
                            long long zmax = 64) {
  zmax = std::max(1LL, std::min({zmax, nz, 64LL}));
  long long best = zmax, best_cost = -1;
  for (long long zc = zmax; zc >= std::min(zmax, 4LL); --zc) {
    const long long nzc = (nz + zc - 1) / zc, blocks = tiles * nzc;
    const long long waves = (blocks + resident - 1) / resident;
    const long long cost = waves * (zc + halo);
    if (best_cost < 0 || cost < best_cost) best = zc, best_cost = cost;
  }
  return best;
}

// opt Kernel into more than 48 KB of dynamic shared memory on the current
// device, once per (kernel, device): the attribute is per device and a
// process may drive several GPUs. Returns the resident blocks per SM.
template <auto Kernel>
int ensure_smem(int threads, size_t bytes) {
  static std::atomic<int> per_sm[64];  // 0 = not yet set on that device
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  int n = per_sm[dev].load(std::memory_order_acquire);
  if (n > 0) return n;
  cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, Kernel, threads, bytes) != cudaSuccess ||
      n < 1)
    n = 1;
  per_sm[dev].store(n, std::memory_order_release);
  return n;
}

bool window_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("LBMGPU_AOS_WINDOW");
    return !(e && e[0] == '0');
  }();
  return on;
}

#ifndef LBM_AOS_WS
#define LBM_AOS_WS 1
#endif
template <class T, int MODE>
void launch_win_ws(cudaStream_t st, const DField& f, const Lat& L, const TrtHost& op) {
  const int per_sm = ensure_smem<k_win_ws<T, MODE>>(WinSzW<T>::kThreads, WinSzW<T>::kBytes);
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int tiles_x = (L.nx + kTX - 1) / kTX, tiles_y = (L.ny + WinSzW<T>::TY - 1) / WinSzW<T>::TY;
  // z planes per block: about 7 waves of resident blocks, 4 .. 64 planes, and
  // at least two chunks on a periodic z axis (the halo plane is not one of
  // the chunk's own planes)
  const long long tiles = (long long)tiles_x * tiles_y, resident = (long long)sms * per_sm;
  long long zc = wave_chunk(L.nz, tiles, resident, 2, L.wall[2] ? 64 : L.nz - 2);
  if (const char* e = std::getenv("LBMGPU_AOS_ZCHUNK"))
    if (std::atoi(e) > 0) zc = std::atoi(e);
  if (!L.wall[2]) zc = std::min<long long>(zc, L.nz - 2);
  zc = std::max(1LL, std::min<long long>(zc, L.nz));
  const int nzc = (int)((L.nz + zc - 1) / zc);
  k_win_ws<T, MODE><<<(unsigned)(tiles * nzc), WinSzW<T>::kThreads, WinSzW<T>::kBytes, st>>>(
      fld<T, true>(f), L, cast_op<T>(op), tiles_x, tiles_y, (int)zc);
}

template <class T, int MODE>
void launch_win(cudaStream_t st, const DField& a, const DField& b, const Lat& L,
                const TrtHost& op, int zc, int z0, int z1, const void* wlo = nullptr,
                const void* whi = nullptr) {
  ensure_smem<k_win<T, MODE>>(WinThreads<T, MODE>::value, WinSz<T>::kBytes);
  const int tiles_x = (L.nx + kTX - 1) / kTX, tiles_y = (L.ny + kTY - 1) / kTY;
  const int nzc = (z1 - z0 + zc - 1) / zc;
  const unsigned grid = (unsigned)(tiles_x * tiles_y * nzc);
  k_win<T, MODE><<<grid, WinThreads<T, MODE>::value, WinSz<T>::kBytes, st>>>(
      fld<T, true>(a), fld<T, true>(b), L, cast_op<T>(op), tiles_x, tiles_y, zc, z0, z1,
      static_cast<const T*>(wlo), static_cast<const T*>(whi));
}

template <class T, int MODE>
void launch_win_zp(cudaStream_t st, const DField& a, const DField& b, const Lat& L,
                   const TrtHost& op, int z0 = 0, int z1 = -1, const void* wlo = nullptr,
                   const void* whi = nullptr) {
  if (z1 < 0) z1 = L.nz;
  using C = ZpCfg<T>;
  constexpr int kThr = ZpThreads<T, MODE>::value;
  const int per_sm = ensure_smem<k_win_zp<T, MODE>>(kThr, C::kBytes);
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int tiles_x = (L.nx + kTX - 1) / kTX, tiles_y = (L.ny + C::TY - 1) / C::TY;
  // z planes per block: about 7 waves of resident blocks, 4 .. 64 planes
  const long long tiles = (long long)tiles_x * tiles_y, resident = (long long)sms * per_sm;
  long long zc = wave_chunk(z1 - z0, tiles, resident, 2);
  if (const char* e = std::getenv("LBMGPU_AOS_ZCHUNK"))
    if (std::atoi(e) > 0) zc = std::atoi(e);
  zc = std::max(1LL, std::min<long long>(zc, z1 - z0));
  const int nzc = (int)((z1 - z0 + zc - 1) / zc);
  k_win_zp<T, MODE><<<(unsigned)(tiles * nzc), kThr, C::kBytes, st>>>(
      fld<T, true>(a), fld<T, true>(b), L, cast_op<T>(op), tiles_x, tiles_y, (int)zc, z0, z1,
      static_cast<const T*>(wlo), static_cast<const T*>(whi));
}

// OS push through the z pipeline (every window record of a plane collided in
// place by 11 warps, then the stream gathers): C1 fp64 0.46 vs 0.54 for the
// scatter form (the halo ring's redundant collisions and the extra barrier
// per plane), fp32 0.51 vs 0.47 for the k_win gather; LBMGPU_AOS_ZPIPE_PUSH
// = 1 / 0 forces it on / off for both precisions
// fp32 in-place modes through the warp-specialised window (LBMGPU_AOS_WS32=1
// or -DLBM_WS_F32=1)
bool ws_f32() {
  static const bool on = [] {
    const char* e = std::getenv("LBMGPU_AOS_WS32");
    return e ? e[0] == '1' : LBM_WS_F32 != 0;
  }();
  return on;
}

// default: fp32 only (C1 fp32 0.47 -> 0.51, C4 0.42 -> 0.46 with the extra
// collision warps; fp64 keeps the scatter form, 0.54 vs 0.46)
bool zpipe_push(bool f64) {
  static const int env = [] {
    const char* e = std::getenv("LBMGPU_AOS_ZPIPE_PUSH");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  return env < 0 ? !f64 : env == 1;
}

// CG plane groups through the z pipeline's push (LBMGPU_AOS_ZPIPE_CG = 1 / 0)
bool zpipe_cg(bool f64) {
  static const int env = [] {
    const char* e = std::getenv("LBMGPU_AOS_ZPIPE_CG");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  return env < 0 ? !f64 : env == 1;
}

bool zpipe_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("LBMGPU_AOS_ZPIPE");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace

// z planes per block: enough blocks for ~7 waves of resident blocks (one
// fp64 / two fp32 per SM), at most 64 planes, and for the in-place mode at
// least two chunks on a periodic z axis (a chunk's halo plane must not be
// one of its own planes)
static int window_chunk(const Lat& L, bool fp64, bool inplace) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long tiles = (long long)((L.nx + kTX - 1) / kTX) * ((L.ny + kTY - 1) / kTY);
  const long long resident = (long long)sms * (fp64 ? 1 : 2);
  long long zc = wave_chunk(L.nz, tiles, resident, 2, inplace && !L.wall[2] ? L.nz - 2 : 64);
  if (const char* e = std::getenv("LBMGPU_AOS_ZCHUNK"))  // tests: long chunks on small boxes
    if (std::atoi(e) > 0) zc = std::atoi(e);
  if (inplace && !L.wall[2]) zc = std::min<long long>(zc, L.nz - 2);
  return (int)std::max(1LL, std::min<long long>(zc, L.nz));
}

// Applicability: AoS, x-fastest storage (a one-layer halo is allowed on wall
// axes), the whole lattice in one launch. In place additionally needs every
// window position to be a distinct record (periodic nx >= 34, ny >= 10,
// nz >= 3).
bool launch_aos_window(cudaStream_t st, int mode, const DField& a, const DField& b,
                       const Lat& L, const TrtHost& op) {
  if (!a.aos || !window_enabled()) return false;
  const int o[3] = {L.ox, L.oy, L.oz};
  for (int k = 0; k < 3; ++k)
    if (o[k] < 0 || o[k] > 1 || (o[k] && !L.wall[k])) return false;
  if (L.sx != L.nx + 2 * L.ox || L.sy != L.ny + 2 * L.oy || L.zghost || L.znowrap) return false;
  if (L.cell_begin != 0 || (unsigned long long)L.ncells != (unsigned long long)L.nx * L.ny * L.nz)
    return false;
  // every window position a distinct record (the ownership write-back)
  const bool distinct = (L.wall[0] || L.nx >= kTX + 2) && (L.wall[1] || L.ny >= kTY + 2) &&
                        (L.wall[2] || L.nz >= 3);
  if (in_place(mode) && !distinct) return false;
  const bool f64 = a.prec == Prec::f64;
  // OS push: the scatter form (no redundant halo collisions, ownership
  // write-back) for fp64; fp32 keeps the gather form (C1 fp64 0.44 -> 0.49,
  // fp32 0.43 -> 0.38; profiles/r01_variants.md)
  // (its bulk write-back runs use the source rows' 16-byte phase)
  const bool congruent = ((reinterpret_cast<uintptr_t>(a.p) ^ reinterpret_cast<uintptr_t>(b.p)) & 15u) == 0;
  if (mode == kWinPush && distinct && f64 && congruent && !(zpipe_enabled() && zpipe_push(f64)))
    mode = kWinPushS;
  // fp64 in-place modes: the warp-specialised window where its 32 x 6 tile
  // keeps every window position a distinct record (a 34 x 8 window on
  // periodic y); fp32 measured no better with it (C1 AA 0.61 -> 0.62, C4 0.51
  // -> 0.52) and keeps k_win at two blocks per SM
  if (LBM_AOS_WS && (f64 || ws_f32()) && in_place(mode) &&
      (L.wall[1] || L.ny >= (f64 ? WinSzW<double>::TY : WinSzW<float>::TY) + 2)) {
#define LBM_WS_CASES(T)                                                   \
  switch (mode) {                                                         \
    case kWinAaOdd: launch_win_ws<T, kWinAaOdd>(st, a, L, op); break;     \
    case kWinSwap: launch_win_ws<T, kWinSwap>(st, a, L, op); break;       \
    case kWinEtI: launch_win_ws<T, kWinEtI>(st, a, L, op); break;         \
    default: launch_win_ws<T, kWinEtS>(st, a, L, op); break;              \
  }
    if (f64) {
      LBM_WS_CASES(double)
    } else {
      LBM_WS_CASES(float)
    }
#undef LBM_WS_CASES
    return true;
  }
  // gather modes: the register-carried z pipeline
  if ((mode == kWinPull || mode == kWinStream || (mode == kWinPush && zpipe_push(f64))) &&
      zpipe_enabled()) {
    if (f64) {
      if (mode == kWinPull) launch_win_zp<double, kWinPull>(st, a, b, L, op);
      else if (mode == kWinPush) launch_win_zp<double, kWinPush>(st, a, b, L, op);
      else launch_win_zp<double, kWinStream>(st, a, b, L, op);
    } else {
      if (mode == kWinPull) launch_win_zp<float, kWinPull>(st, a, b, L, op);
      else if (mode == kWinPush) launch_win_zp<float, kWinPush>(st, a, b, L, op);
      else launch_win_zp<float, kWinStream>(st, a, b, L, op);
    }
    return true;
  }
  const int zc = window_chunk(L, f64, owned_wb(mode));
#define LBM_WIN_CASES(T)                                                              \
  switch (mode) {                                                                     \
    case kWinPull: launch_win<T, kWinPull>(st, a, b, L, op, zc, 0, L.nz); break;     \
    case kWinStream: launch_win<T, kWinStream>(st, a, b, L, op, zc, 0, L.nz); break; \
    case kWinPush: launch_win<T, kWinPush>(st, a, b, L, op, zc, 0, L.nz); break;     \
    case kWinAaOdd: launch_win<T, kWinAaOdd>(st, a, b, L, op, zc, 0, L.nz); break;   \
    case kWinSwap: launch_win<T, kWinSwap>(st, a, b, L, op, zc, 0, L.nz); break;     \
    case kWinEtI: launch_win<T, kWinEtI>(st, a, b, L, op, zc, 0, L.nz); break;       \
    case kWinPushS: launch_win<T, kWinPushS>(st, a, b, L, op, zc, 0, L.nz); break;   \
    default: launch_win<T, kWinEtS>(st, a, b, L, op, zc, 0, L.nz); break;            \
  }
  if (f64) {
    LBM_WIN_CASES(double)
  } else {
    LBM_WIN_CASES(float)
  }
#undef LBM_WIN_CASES
  return true;
}

// OS-push window over planes [z0, z1) only (CG plane groups: src and dst are
// the read and write frames of one grid; wlo / whi = saved copies of the
// planes a periodic z wrap reads, or null)
bool aos_push_planes_ok(const DField& src, const Lat& L) {
  if (!src.aos || !window_enabled()) return false;
  if (L.sx != L.nx || L.sy != L.ny || L.ox || L.oy || L.oz || L.zghost || L.znowrap) return false;
  return L.cell_begin == 0 &&
         (unsigned long long)L.ncells == (unsigned long long)L.nx * L.ny * L.nz;
}
void launch_aos_push_planes(cudaStream_t st, const DField& src, const DField& dst, const Lat& L,
                            const TrtHost& op, int z0, int z1, const void* wlo, const void* whi) {
  if (z1 <= z0) return;
  // the z pipeline's push (the OS-push kernel) on the group's planes
  if (zpipe_enabled() && zpipe_cg(src.prec == Prec::f64)) {
    if (src.prec == Prec::f64)
      launch_win_zp<double, kWinPush>(st, src, dst, L, op, z0, z1, wlo, whi);
    else
      launch_win_zp<float, kWinPush>(st, src, dst, L, op, z0, z1, wlo, whi);
    return;
  }
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // about two waves of resident blocks over the group's planes
  const long long tiles = (long long)((L.nx + kTX - 1) / kTX) * ((L.ny + kTY - 1) / kTY);
  const long long resident = (long long)sms * (src.prec == Prec::f64 ? 1 : 2);
  const int zc = (int)std::max(4LL, std::min<long long>(z1 - z0, ((z1 - z0) * tiles) / (2 * resident) + 1));
  if (src.prec == Prec::f64)
    launch_win<double, kWinPush>(st, src, dst, L, op, zc, z0, z1, wlo, whi);
  else
    launch_win<float, kWinPush>(st, src, dst, L, op, zc, z0, z1, wlo, whi);
}

template <class T, bool RD, bool WR>
static void launch_stream_t(cudaStream_t st, const DField& a, const DField& b, const Lat& L,
                            const TrtHost& op, uint32_t soff) {
  // resident blocks per SM (registers and the two-slot ring)
  const int per_sm = ensure_smem<k_local_stream<T, RD, WR>>(kRun, RunSz<T>::kBytes);
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t nruns = (L.ncells - L.cell_begin + kRun - 1) / kRun;
  const uint32_t grid = std::min<uint32_t>(nruns, (uint32_t)(sms * per_sm));
  k_local_stream<T, RD, WR><<<grid, kRun, RunSz<T>::kBytes, st>>>(
      fld<T, true>(a), fld<T, true>(b), L, cast_op<T>(op), soff, nruns);
}

// contiguous AoS local sweep: storage index = cell + soff for every cell
bool launch_aos_local_stream(cudaStream_t st, const DField& a, const DField& b, const Lat& L,
                             const TrtHost& op, bool rd_opp, bool wr_opp, uint32_t soff) {
  if (!a.aos || !window_enabled()) return false;
  if (a.prec == Prec::f64) {
    if (!rd_opp && !wr_opp) launch_stream_t<double, false, false>(st, a, b, L, op, soff);
    if (!rd_opp && wr_opp) launch_stream_t<double, false, true>(st, a, b, L, op, soff);
    if (rd_opp && !wr_opp) launch_stream_t<double, true, false>(st, a, b, L, op, soff);
    if (rd_opp && wr_opp) launch_stream_t<double, true, true>(st, a, b, L, op, soff);
  } else {
    if (!rd_opp && !wr_opp) launch_stream_t<float, false, false>(st, a, b, L, op, soff);
    if (!rd_opp && wr_opp) launch_stream_t<float, false, true>(st, a, b, L, op, soff);
    if (rd_opp && !wr_opp) launch_stream_t<float, true, false>(st, a, b, L, op, soff);
    if (rd_opp && wr_opp) launch_stream_t<float, true, true>(st, a, b, L, op, soff);
  }
  return true;
}

}  // namespace lbmgpu

#ifdef LBM_WIN_TRACE
extern "C" int lbmgpu_debug_win_trace(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, lbmgpu::g_win_trace, sizeof(unsigned long long) * 16);
  if (reset) {
    static const unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(lbmgpu::g_win_trace, z, sizeof(z));
  }
  return 0;
}
#endif
