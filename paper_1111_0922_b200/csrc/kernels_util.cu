// Geometry/IDX construction, canonical-snapshot conversion and initial
// fields, all on the device (sm_100a).
//
//   build_node_maps  exclusive scan of the fluid mask -> node_of / cell_of_node
//                    (the x-fastest enumeration of build_sparse,
//                    p/src/geometry.cpp:187-194)
//   launch_adjacency resolve_link per (node, dir) -> transposed IDX
//                    (p/src/geometry.cpp:49-60, 196-205)
//   build_et_rem     ET remote table with per-pair mailbox running counts
//                    (p/src/scheme_et.cpp:42-62) as 9 exclusive scans
//   launch_extract / launch_load
//                    canonical snapshot <-> scheme storage (the
//                    copy_out/gather_out/load_in helpers, p/src/stepper.cpp:207-289,
//                    and the per-scheme extract_natural/load_natural)
#include "dispatch.h"
#include "launch.h"

#include <cmath>
#include <stdexcept>
#include <string>

namespace lbmgpu {
using namespace dev;

namespace {

inline unsigned grid_for(uint64_t n) { return (unsigned)((n + kBlock - 1) / kBlock); }

__device__ __forceinline__ double weight(int i) {
  return i == 0 ? 1.0 / 3.0 : (i <= 6 ? 1.0 / 18.0 : 1.0 / 36.0);
}

// splitmix64 of (seed, stream)
__device__ __forceinline__ unsigned long long urand_bits(unsigned long long seed,
                                                         unsigned long long stream) {
  unsigned long long z = seed + 0x9e3779b97f4a7c15ull * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
// counter-based uniform in [-1, 1)
__device__ __forceinline__ double urand(unsigned long long seed, unsigned long long stream) {
  const unsigned long long z = urand_bits(seed, stream);
  return __dsub_rn(__dmul_rn((double)(z >> 11), 0x1.0p-52), 1.0);
}

// equilibrium (p/src/collision.cpp:38-45)
__device__ __forceinline__ double equilibrium(double rho, double ux, double uy, double uz, int i) {
  double cu = 0.0, usq = 0.0;
  cu = __dadd_rn(cu, __dmul_rn((double)cx(i), ux));
  usq = __dadd_rn(usq, __dmul_rn(ux, ux));
  cu = __dadd_rn(cu, __dmul_rn((double)cy(i), uy));
  usq = __dadd_rn(usq, __dmul_rn(uy, uy));
  cu = __dadd_rn(cu, __dmul_rn((double)cz(i), uz));
  usq = __dadd_rn(usq, __dmul_rn(uz, uz));
  const double a = __dadd_rn(__dadd_rn(1.0, __dmul_rn(3.0, cu)), __dmul_rn(__dmul_rn(4.5, cu), cu));
  return __dmul_rn(__dmul_rn(weight(i), rho), __dsub_rn(a, __dmul_rn(1.5, usq)));
}

// canonical value of direction i <-> stored value (fp32 fields hold
// f_i - w_i shift, lbm_device.cuh kShifted; fp64 fields hold f_i)
template <class T>
__device__ __forceinline__ T to_store(double v, int i, double shift) {
  if constexpr (kShifted<T>)
    return (T)__dsub_rn(v, __dmul_rn(weight(i), shift));
  else
    return (T)v;
}
template <class T>
__device__ __forceinline__ double from_store(T s, int i, double shift) {
  if constexpr (kShifted<T>)
    return __dadd_rn((double)s, __dmul_rn(weight(i), shift));
  else
    return (double)s;
}

// Initial canonical values of one node (host buffer or a generator).
//  Rest:        w_i rho0 (every reference stepper's start, e.g. scheme_aap.cpp:32-36)
//  TaylorGreen: equilibrium(rho, u) + noise*U, rho = rho0 + drho*U,
//               u = u0 (sin X cos Y cos Z, -cos X sin Y cos Z, 0),
//               X = (2 pi) x / gnx (cell index x, likewise Y, Z); sin/cos
//               come from the host's libm table (InitSpec::trig)
//  Random:      w_i rho0 (0.9 + 0.2 U01)  (shape of test_schemes.cpp:29-39)
// U draws are keyed by the GLOBAL cell index, so z-slabs reproduce the
// single-domain field exactly.
__device__ __forceinline__ void node_values(const InitSpec& in, const double* buf, uint32_t k,
                                            int x, int y, int z, double (&v)[19]) {
  if (in.source == kSrcBuffer) {
#pragma unroll
    for (int i = 0; i < 19; ++i) v[i] = buf[(size_t)k * 19 + i];
    return;
  }
  if (in.source == kSrcRest) {
#pragma unroll
    for (int i = 0; i < 19; ++i) v[i] = __dmul_rn(weight(i), in.rho0);
    return;
  }
  const int gz = z + in.z0;
  const unsigned long long gcell =
      (unsigned long long)x + (unsigned long long)in.gnx * ((unsigned long long)y + (unsigned long long)in.gny * gz);
  if (in.source == kSrcRandom) {
#pragma unroll
    for (int i = 0; i < 19; ++i) {
      const double u01 = __dmul_rn(0.5, __dadd_rn(urand(in.seed, gcell * 20 + i), 1.0));
      v[i] = __dmul_rn(__dmul_rn(weight(i), in.rho0), __dadd_rn(0.9, __dmul_rn(0.2, u01)));
    }
    return;
  }
  const double* tx = in.trig;
  const double* ty = tx + 2 * in.gnx;
  const double* tz = ty + 2 * in.gny;
  const double sx = tx[x], cxv = tx[in.gnx + x];
  const double sy = ty[y], cyv = ty[in.gny + y];
  const double czv = tz[in.gnz + gz];
  const double rho = __dadd_rn(in.rho0, __dmul_rn(in.drho, urand(in.seed, gcell * 20 + 19)));
  const double ux = __dmul_rn(__dmul_rn(__dmul_rn(in.u0, sx), cyv), czv);
  const double uy = __dmul_rn(__dmul_rn(__dmul_rn(-in.u0, cxv), sy), czv);
  const double uz = 0.0;
#pragma unroll
  for (int i = 0; i < 19; ++i)
    v[i] = __dadd_rn(equilibrium(rho, ux, uy, uz, i), __dmul_rn(in.noise, urand(in.seed, gcell * 20 + i)));
}

template <class T, bool AOS>
__global__ void k_extract(Fld<T, AOS> F, Lat L, const uint32_t* cell_of_node, uint32_t n0,
                          uint32_t count, int mode, EtBase B, double* buf, double shift) {
  const uint32_t k = blockIdx.x * kBlock + threadIdx.x;
  if (k >= count) return;
  const uint32_t node = n0 + k;
  const uint32_t cell = cell_of_node ? cell_of_node[node] : node;
  const Ctx c = make_ctx(L, cell);
  double* o = buf + (size_t)k * 19;
  switch (mode) {
    case kExNatural:
#pragma unroll
      for (int i = 0; i < 19; ++i) o[i] = from_store(*F.at(i, c.s), i, shift);
      break;
    case kExOpposed:
#pragma unroll
      for (int i = 0; i < 19; ++i) o[i] = from_store(*F.at(opp(i), c.s), i, shift);
      break;
    case kExGather:  // gather_out_direct (p/src/stepper.cpp:228-252)
      o[0] = from_store(*F.at(0, c.s), 0, shift);
#pragma unroll
      for (int i = 1; i < 19; ++i) {
        const int j = opp(i);
        o[i] = from_store(*(c.bb(j) ? F.at(j, c.s) : F.at(i, c.nb(j))), i, shift);
      }
      break;
    case kExAaOdd:  // AapStepper::extract_natural, odd (p/src/scheme_aap.cpp:57-75)
      o[0] = from_store(*F.at(0, c.s), 0, shift);
#pragma unroll
      for (int i = 1; i < 19; ++i) {
        const int j = opp(i);
        o[i] = from_store(*(c.bb(j) ? F.at(i, c.s) : F.at(j, c.nb(j))), i, shift);
      }
      break;
    case kExEt:  // EtStepper::extract_natural, direct (p/src/scheme_et.cpp:83-109)
      o[0] = from_store(*F.at(0, c.s), 0, shift);
#pragma unroll
      for (int p = 0; p < 9; ++p) {
        const int i = pair_i(p), j = pair_j(p);
        o[i] = from_store(*F.at(B.b[i], c.s), i, shift);
        o[j] = from_store(*F.at(c.bb(i) ? B.b[i] : B.b[j], c.nb(i)), j, shift);
      }
      break;
  }
}

template <class T, bool AOS>
__global__ void k_load(Fld<T, AOS> F, Lat L, const uint32_t* cell_of_node, uint32_t n0,
                       uint32_t count, int mode, const double* buf, InitSpec in) {
  const uint32_t k = blockIdx.x * kBlock + threadIdx.x;
  if (k >= count) return;
  const uint32_t node = n0 + k;
  const uint32_t cell = cell_of_node ? cell_of_node[node] : node;
  const Ctx c = make_ctx(L, cell);
  double v[19];
  node_values(in, buf, k, c.x, c.y, c.z, v);
  switch (mode) {
    case kExNatural:
#pragma unroll
      for (int i = 0; i < 19; ++i) *F.at(i, c.s) = to_store<T>(v[i], i, in.rho0);
      break;
    case kExOpposed:
#pragma unroll
      for (int i = 0; i < 19; ++i) *F.at(opp(i), c.s) = to_store<T>(v[i], i, in.rho0);
      break;
    case kExEt:  // EtStepper::fill, direct (p/src/scheme_et.cpp:152-169), identity handles
      *F.at(0, c.s) = to_store<T>(v[0], 0, in.rho0);
#pragma unroll
      for (int p = 0; p < 9; ++p) {
        const int i = pair_i(p), j = pair_j(p);
        *F.at(i, c.s) = to_store<T>(v[i], i, in.rho0);
        *F.at(c.bb(i) ? i : j, c.nb(i)) = to_store<T>(v[j], j, in.rho0);
      }
      break;
  }
}

template <class T, bool AOS>
__global__ void k_extract_idx(Fld<T, AOS> F, Idx I, uint32_t n0, uint32_t count, int mode,
                              EtBase B, double* buf, double shift) {
  const uint32_t k = blockIdx.x * kBlock + threadIdx.x;
  if (k >= count) return;
  const uint32_t node = n0 + k;
  double* o = buf + (size_t)k * 19;
  switch (mode) {
    case kExNatural:
#pragma unroll
      for (int i = 0; i < 19; ++i) o[i] = from_store(*F.at(i, node), i, shift);
      break;
    case kExOpposed:
#pragma unroll
      for (int i = 0; i < 19; ++i) o[i] = from_store(*F.at(opp(i), node), i, shift);
      break;
    case kExGather:  // gather_out_indirect (p/src/stepper.cpp:254-271)
      o[0] = from_store(*F.at(0, node), 0, shift);
#pragma unroll
      for (int i = 1; i < 19; ++i) {
        const int j = opp(i);
        const uint32_t src = I.adj[(size_t)(j - 1) * I.n + node];
        o[i] = from_store(*(src == node ? F.at(j, node) : F.at(i, src)), i, shift);
      }
      break;
    case kExAaOdd:  // p/src/scheme_aap.cpp:81-97
      o[0] = from_store(*F.at(0, node), 0, shift);
#pragma unroll
      for (int i = 1; i < 19; ++i) {
        const int j = opp(i);
        const uint32_t e = I.adj[(size_t)(j - 1) * I.n + node];
        o[i] = from_store(*(e == node ? F.at(i, node) : F.at(j, e)), i, shift);
      }
      break;
    case kExEt:  // p/src/scheme_et.cpp:110-123
      o[0] = from_store(*F.at(0, node), 0, shift);
#pragma unroll
      for (int p = 0; p < 9; ++p) {
        const int i = pair_i(p), j = pair_j(p);
        const uint32_t r = I.rem[(size_t)p * I.n + node] & 0x7fffffffu;
        o[i] = from_store(*F.at(B.b[i], node), i, shift);
        o[j] = from_store(*F.at(r >= I.n ? B.b[i] : B.b[j], r), j, shift);
      }
      break;
  }
}

template <class T, bool AOS>
__global__ void k_load_idx(Fld<T, AOS> F, Idx I, Lat L, const uint32_t* cell_of_node,
                           uint32_t n0, uint32_t count, int mode, const double* buf, InitSpec in) {
  const uint32_t k = blockIdx.x * kBlock + threadIdx.x;
  if (k >= count) return;
  const uint32_t node = n0 + k;
  int x = 0, y = 0, z = 0;
  if (in.source != kSrcBuffer) {
    const uint32_t cell = cell_of_node ? cell_of_node[node] : node;
    const uint32_t row = L.divx.div(cell);
    x = (int)(cell - row * (uint32_t)L.nx);
    const uint32_t zz = L.divy.div(row);
    y = (int)(row - zz * (uint32_t)L.ny);
    z = (int)zz;
  }
  double v[19];
  node_values(in, buf, k, x, y, z, v);
  switch (mode) {
    case kExNatural:
#pragma unroll
      for (int i = 0; i < 19; ++i) *F.at(i, node) = to_store<T>(v[i], i, in.rho0);
      break;
    case kExOpposed:
#pragma unroll
      for (int i = 0; i < 19; ++i) *F.at(opp(i), node) = to_store<T>(v[i], i, in.rho0);
      break;
    case kExEt:  // EtStepper::fill, indirect (p/src/scheme_et.cpp:170-183)
      *F.at(0, node) = to_store<T>(v[0], 0, in.rho0);
#pragma unroll
      for (int p = 0; p < 9; ++p) {
        const int i = pair_i(p), j = pair_j(p);
        const uint32_t r = I.rem[(size_t)p * I.n + node] & 0x7fffffffu;
        *F.at(i, node) = to_store<T>(v[i], i, in.rho0);
        *F.at(r >= I.n ? i : j, r) = to_store<T>(v[j], j, in.rho0);
      }
      break;
  }
}

template <class T>
__global__ void k_fill(T* p, long long count, T v) {
  for (long long k = (long long)blockIdx.x * kBlock + threadIdx.x; k < count;
       k += (long long)gridDim.x * kBlock)
    p[k] = v;
}

// ---------------------------------------------------------------------------
// Device-wide exclusive scan (3 phases: tile reduce, scan of tile sums in one
// block, tile re-scan + offset). Tiles of 1024 threads x 16 items.
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 16;
constexpr uint64_t kScanTile = (uint64_t)kScanThreads * kScanItems;

__device__ __forceinline__ uint32_t warp_incl(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// exclusive block scan of one value per thread; returns exclusive prefix, total in *tot
__device__ uint32_t block_excl(uint32_t v, uint32_t* tot) {
  __shared__ uint32_t ws[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t inc = warp_incl(v);
  if (lane == 31) ws[w] = inc;
  __syncthreads();
  if (w == 0) {
    const uint32_t x = ws[lane];
    ws[lane] = warp_incl(x) - x;
  }
  __syncthreads();
  const uint32_t r = ws[w] + inc - v;
  if (tot) *tot = ws[31] + __shfl_sync(0xffffffffu, inc, 31);  // valid for the last warp
  __syncthreads();
  return r;
}

struct MaskFlag {
  const uint8_t* m;
  __device__ uint32_t operator()(uint64_t k) const { return m[k] != 0; }
};
struct BounceFlag {  // ET: i-link of pair p bounces
  const uint32_t* adj_i;
  __device__ uint32_t operator()(uint64_t k) const { return adj_i[k] == (uint32_t)k; }
};

template <class Flag>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(Flag fl, uint64_t n, uint32_t* part) {
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  uint32_t s = 0;
#pragma unroll
  for (int t = 0; t < kScanItems; ++t)
    if (base + t < n) s += fl(base + t);
  uint32_t tot = 0;
  block_excl(s, &tot);
  if (threadIdx.x == kScanThreads - 1) part[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_parts(uint32_t* part, uint32_t np,
                                                             unsigned long long* total) {
  const uint32_t per = (np + kScanThreads - 1) / kScanThreads;
  const uint32_t b0 = threadIdx.x * per;
  uint32_t s = 0;
  for (uint32_t k = 0; k < per; ++k)
    if (b0 + k < np) s += part[b0 + k];
  uint32_t tot = 0;
  uint32_t run = block_excl(s, &tot);
  for (uint32_t k = 0; k < per; ++k)
    if (b0 + k < np) {
      const uint32_t v = part[b0 + k];
      part[b0 + k] = run;
      run += v;
    }
  if (threadIdx.x == kScanThreads - 1) *total = tot;
}

template <class Flag, class Sink>
__global__ void __launch_bounds__(kScanThreads) k_scan_apply(Flag fl, uint64_t n,
                                                             const uint32_t* part, Sink sink) {
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  uint32_t f[kScanItems];
  uint32_t s = 0;
#pragma unroll
  for (int t = 0; t < kScanItems; ++t) {
    f[t] = (base + t < n) ? fl(base + t) : 0u;
    s += f[t];
  }
  uint32_t run = block_excl(s, nullptr) + part[blockIdx.x];
#pragma unroll
  for (int t = 0; t < kScanItems; ++t)
    if (base + t < n) {
      sink(base + t, f[t], run);
      run += f[t];
    }
}

struct NodeMapSink {
  uint32_t* node_of;
  uint32_t* cell_of_node;
  __device__ void operator()(uint64_t cell, uint32_t flag, uint32_t idx) const {
    if (node_of) node_of[cell] = flag ? idx : ~0u;
    if (flag && cell_of_node) cell_of_node[idx] = (uint32_t)cell;
  }
};

struct EtRemSink {
  const uint32_t* adj_i;
  const uint32_t* adj_j;
  uint32_t* rem_p;
  uint32_t n;
  __device__ void operator()(uint64_t node, uint32_t flag, uint32_t idx) const {
    const uint32_t r = flag ? n + idx : adj_i[node];
    const bool ub = adj_j[node] == (uint32_t)node;
    rem_p[node] = r | (ub ? 0x80000000u : 0u);
  }
};

template <class Flag, class Sink>
uint64_t device_scan(cudaStream_t st, Flag fl, uint64_t n, Sink sink, uint32_t* scratch) {
  const uint32_t np = (uint32_t)((n + kScanTile - 1) / kScanTile);
  unsigned long long* total = reinterpret_cast<unsigned long long*>(scratch);
  uint32_t* part = scratch + 2;
  if (np == 0) return 0;
  k_scan_reduce<<<np, kScanThreads, 0, st>>>(fl, n, part);
  k_scan_parts<<<1, kScanThreads, 0, st>>>(part, np, total);
  k_scan_apply<<<np, kScanThreads, 0, st>>>(fl, n, part, sink);
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, total, sizeof(h), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  return h;
}

// resolve_link on the device (p/src/geometry.cpp:49-60); returns target cell or -1 (bounce)
__device__ __forceinline__ long long resolve(const uint8_t* mask, const Lat& L, int x, int y,
                                             int z, int i) {
  int t[3] = {x + cx(i), y + cy(i), z + cz(i)};
  const int n[3] = {L.nx, L.ny, L.nz};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (t[k] >= 0 && t[k] < n[k]) continue;
    if (L.wall[k]) return -1;
    t[k] = t[k] < 0 ? t[k] + n[k] : t[k] - n[k];
  }
  const long long cell = (long long)t[0] + (long long)L.nx * ((long long)t[1] + (long long)L.ny * t[2]);
  if (mask && !mask[cell]) return -1;
  return cell;
}

__global__ void k_linkmask(const uint8_t* mask, Lat L, uint32_t* out) {
  const uint32_t cell = blockIdx.x * kBlock + threadIdx.x;
  if (cell >= L.ncells) return;
  if (mask && !mask[cell]) {
    out[cell] = 0;
    return;
  }
  const uint32_t row = L.divx.div(cell);
  const int x = (int)(cell - row * (uint32_t)L.nx);
  const uint32_t z = L.divy.div(row);
  const int y = (int)(row - z * (uint32_t)L.ny);
  uint32_t m = 1u;
#pragma unroll
  for (int i = 1; i < 19; ++i)
    if (resolve(mask, L, x, y, (int)z, i) < 0) m |= 1u << i;
  out[cell] = m;
}

__global__ void k_adjacency(const uint8_t* mask, Lat L, const uint32_t* node_of,
                            const uint32_t* cell_of_node, uint32_t n, uint32_t* adjT) {
  const uint32_t node = blockIdx.x * kBlock + threadIdx.x;
  if (node >= n) return;
  const uint32_t cell = cell_of_node ? cell_of_node[node] : node;
  const uint32_t row = L.divx.div(cell);
  const int x = (int)(cell - row * (uint32_t)L.nx);
  const uint32_t z = L.divy.div(row);
  const int y = (int)(row - z * (uint32_t)L.ny);
#pragma unroll
  for (int i = 1; i < 19; ++i) {
    const long long t = resolve(mask, L, x, y, (int)z, i);
    adjT[(size_t)(i - 1) * n + node] =
        t < 0 ? node : (node_of ? node_of[t] : (uint32_t)t);
  }
}

__global__ void k_transpose(const uint32_t* inT, uint32_t rows, uint32_t n, uint32_t* out) {
  const uint64_t k = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
  if (k >= (uint64_t)rows * n) return;
  const uint32_t node = (uint32_t)(k / rows), r = (uint32_t)(k % rows);
  out[k] = inT[(size_t)r * n + node];
}

}  // namespace

uint64_t scan_scratch_elems(uint64_t n) { return 2 + (n + kScanTile - 1) / kScanTile + 2; }

uint64_t build_node_maps(cudaStream_t st, const uint8_t* mask, uint64_t ncells,
                         uint32_t* node_of, uint32_t* cell_of_node, uint32_t* scratch,
                         uint64_t) {
  return device_scan(st, MaskFlag{mask}, ncells, NodeMapSink{node_of, cell_of_node}, scratch);
}

uint32_t build_et_rem(cudaStream_t st, const uint32_t* adjT, uint32_t n, uint32_t* remT,
                      uint32_t* scratch, uint64_t) {
  uint32_t nmail = 0;
  for (int p = 0; p < 9; ++p) {
    const uint32_t* ai = adjT + (size_t)(pair_i(p) - 1) * n;
    const uint32_t* aj = adjT + (size_t)(pair_j(p) - 1) * n;
    const uint64_t cnt =
        device_scan(st, BounceFlag{ai}, n, EtRemSink{ai, aj, remT + (size_t)p * n, n}, scratch);
    if (cnt > nmail) nmail = (uint32_t)cnt;
  }
  return nmail;
}

void launch_linkmask(cudaStream_t st, const uint8_t* mask, const dev::Lat& L, uint32_t* out) {
  k_linkmask<<<grid_for(L.ncells), kBlock, 0, st>>>(mask, L, out);
}

void launch_adjacency(cudaStream_t st, const uint8_t* mask, const dev::Lat& L,
                      const uint32_t* node_of, const uint32_t* cell_of_node, uint32_t n,
                      uint32_t* adjT) {
  if (n == 0) return;
  k_adjacency<<<grid_for(n), kBlock, 0, st>>>(mask, L, node_of, cell_of_node, n, adjT);
}

void launch_transpose_u32(cudaStream_t st, const uint32_t* inT, uint32_t rows, uint32_t n,
                          uint32_t* out) {
  const uint64_t tot = (uint64_t)rows * n;
  if (tot == 0) return;
  k_transpose<<<grid_for(tot), kBlock, 0, st>>>(inT, rows, n, out);
}

void launch_extract(cudaStream_t st, const DField& f, const dev::Lat& L,
                    const uint32_t* cell_of_node, uint32_t n0, uint32_t count, int mode,
                    const EtBase& base, double* buf) {
  if (count == 0) return;
  LBM_DISPATCH(f, {
    k_extract<T, A><<<grid_for(count), kBlock, 0, st>>>(fld<T, A>(f), L, cell_of_node, n0,
                                                        count, mode, base, buf, f.shift);
  });
}

// sin/cos of (2 pi) x / n with the host libm, the oracle's orc_trig_table
// (oracle/lbm_oracle.c) operation for operation
void taylor_green_table(int gnx, int gny, int gnz, double* out) {
  const double two_pi = 6.283185307179586476925286766559;
  for (int n : {gnx, gny, gnz}) {
    for (int x = 0; x < n; ++x) {
      const double a = two_pi * (double)x / (double)n;
      out[x] = std::sin(a);
      out[n + x] = std::cos(a);
    }
    out += 2 * n;
  }
}

void launch_load(cudaStream_t st, const DField& f, const dev::Lat& L,
                 const uint32_t* cell_of_node, uint32_t n0, uint32_t count, int mode,
                 const double* buf, const InitSpec& init) {
  if (count == 0) return;
  LBM_DISPATCH(f, {
    k_load<T, A><<<grid_for(count), kBlock, 0, st>>>(fld<T, A>(f), L, cell_of_node, n0, count,
                                                     mode, buf, init);
  });
}

void launch_extract_idx(cudaStream_t st, const DField& f, const Idx& I, uint32_t n0,
                        uint32_t count, int mode, const EtBase& base, double* buf) {
  if (count == 0) return;
  LBM_DISPATCH(f, {
    k_extract_idx<T, A><<<grid_for(count), kBlock, 0, st>>>(fld<T, A>(f), I, n0, count, mode,
                                                            base, buf, f.shift);
  });
}

void launch_load_idx(cudaStream_t st, const DField& f, const Idx& I, const dev::Lat& Lcells,
                     const uint32_t* cell_of_node, uint32_t n0, uint32_t count, int mode,
                     const double* buf, const InitSpec& init) {
  if (count == 0) return;
  LBM_DISPATCH(f, {
    k_load_idx<T, A><<<grid_for(count), kBlock, 0, st>>>(fld<T, A>(f), I, Lcells, cell_of_node,
                                                         n0, count, mode, buf, init);
  });
}

// ---- z-slab phase-1 merge ---------------------------------------------------
namespace {
template <class T>
__global__ void k_slab_merge(T* dst, const T* src, uint32_t count, int dir, uint32_t first,
                             const uint32_t* adj, uint32_t n, int nx, uint8_t wx, uint8_t wy,
                             int ny) {
  const uint32_t q = blockIdx.x * kBlock + threadIdx.x;
  if (q >= count) return;
  bool bounce;
  if (adj) {
    const uint32_t node = first + q;
    bounce = adj[(size_t)(dir - 1) * n + node] == node;
  } else {
    const int x = (int)(q % (uint32_t)nx), y = (int)(q / (uint32_t)nx);
    bounce = (wx && ((x == 0 && dev::cx(dir) < 0) || (x == nx - 1 && dev::cx(dir) > 0))) ||
             (wy && ((y == 0 && dev::cy(dir) < 0) || (y == ny - 1 && dev::cy(dir) > 0)));
  }
  if (!bounce) dst[q] = src[q];
}
}  // namespace

void launch_slab_merge(cudaStream_t st, Prec prec, void* dst, const void* src, uint32_t count,
                       int dir, uint32_t first, const uint32_t* adj, uint32_t n, int nx, int ny,
                       bool wx, bool wy) {
  if (count == 0) return;
  if (prec == Prec::f64)
    k_slab_merge<double><<<grid_for(count), kBlock, 0, st>>>(
        static_cast<double*>(dst), static_cast<const double*>(src), count, dir, first, adj, n, nx,
        wx, wy, ny);
  else
    k_slab_merge<float><<<grid_for(count), kBlock, 0, st>>>(
        static_cast<float*>(dst), static_cast<const float*>(src), count, dir, first, adj, n, nx,
        wx, wy, ny);
}

// ---- division self-test -----------------------------------------------------
namespace {
__device__ double test_value(uint64_t h, int kind) {
  const uint64_t r = h >> 11;
  const double u = (double)r * 0x1.0p-53;  // [0, 1)
  switch (kind) {
    case 0: return __longlong_as_double((long long)h);                       // any bit pattern
    case 1: return 1.0 + (u - 0.5) * 1e-2;                                   // rho-like
    case 2: return (u - 0.5) * ldexp(1.0, (int)(h & 127) - 100);             // momenta, wide range
    case 3: return (h & 1) ? -0.0 : 0.0;                                     // signed zeros
    case 4: return ldexp(u, -1030);                                          // denormals
    case 5: return (h & 1) ? -INFINITY : INFINITY;
    case 6: return __longlong_as_double(0x7ff8000000000000LL | (long long)(h & 0xfffff));
    default: return ldexp(1.0 + u, (int)(h % 2046) - 1022);                  // any normal
  }
}
__global__ void k_selftest_div(uint64_t n, uint64_t seed, unsigned long long* bad) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t h1 = urand_bits(seed, 2 * k), h2 = urand_bits(seed, 2 * k + 1);
    // numerator kinds weighted towards the collision's (2, 3), denominator rho-like
    const int ka = (int)((h1 >> 3) % 10), kb = (int)((h2 >> 3) % 10);
    const int kinds_a[10] = {0, 2, 2, 2, 3, 4, 5, 6, 7, 1};
    const int kinds_b[10] = {1, 1, 1, 1, 1, 7, 0, 4, 5, 2};
    const double a = test_value(h1, kinds_a[ka]), b = test_value(h2 * 0x9e3779b97f4a7c15ull, kinds_b[kb]);
    const double want = __ddiv_rn(a, b);
    const double got = dev::div_by(a, dev::rcp_prep(b));
    if (__double_as_longlong(got) != __double_as_longlong(want)) atomicAdd(bad, 1ull);
    // fp32: the same inputs rounded to float, plus float-range momenta
    const float af = (k & 1) ? (float)a : (float)test_value(h1 ^ 0x5bd1e995ull, 2) * 1e-3f;
    const float bf = (float)b;
    const float wantf = __fdiv_rn(af, bf);
    const float gotf = dev::div_by(af, dev::rcp_prep(bf));
    if (__float_as_int(gotf) != __float_as_int(wantf)) atomicAdd(bad, 1ull);
  }
}
}  // namespace

uint64_t selftest_division(uint64_t n, uint64_t seed) {
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, sizeof(*d)) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
  cudaMemset(d, 0, sizeof(*d));
  k_selftest_div<<<1184, 256>>>(n, seed, d);
  unsigned long long h = 0;
  const cudaError_t e = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
  return h;
}

// ---- streaming-bandwidth probe (the roofline denominator, measured live) ----
// copy b <- a, or the sweeps' own in-place pattern a <- f(a) (every 16-byte
// line read once and written back, like the AA / ET / OS-pull stores over the
// slots they read). Three launch shapes; the probe reports the best:
//   0  persistent grid (8 x 256 threads per SM), grid-stride, 4 loads in flight
//   1  one 16-byte element per thread, one block per 256 elements
//   2  four 16-byte elements per thread (warp-contiguous), one block per 1024
namespace {
__device__ __forceinline__ uint4 bump(uint4 v) {
  v.x += 1u;
  return v;
}
__global__ void __launch_bounds__(256) k_bw0(const uint4* a, uint4* b, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    const uint4 v0 = a[i], v1 = a[i + stride], v2 = a[i + 2 * stride], v3 = a[i + 3 * stride];
    b[i] = bump(v0), b[i + stride] = bump(v1), b[i + 2 * stride] = bump(v2),
    b[i + 3 * stride] = bump(v3);
  }
  for (; i < n; i += stride) b[i] = bump(a[i]);
}
__global__ void __launch_bounds__(256) k_bw1(const uint4* a, uint4* b, size_t n) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = bump(a[i]);
}
__global__ void __launch_bounds__(256) k_bw2(const uint4* a, uint4* b, size_t n) {
  const size_t base = (size_t)blockIdx.x * 1024 + (threadIdx.x / 32) * 128 + (threadIdx.x % 32);
  uint4 v[4];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (base + 32 * k < n) v[k] = a[base + 32 * k];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (base + 32 * k < n) b[base + 32 * k] = bump(v[k]);
}
}  // namespace

double stream_bandwidth(uint64_t bytes, int inplace, int reps) {
  const size_t n = bytes / 16;
  if (n == 0 || reps < 1) throw std::invalid_argument("bandwidth probe needs bytes >= 16, reps >= 1");
  uint4 *a = nullptr, *b = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  auto release = [&] {
    if (a) cudaFree(a);
    if (b) cudaFree(b);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (st) cudaStreamDestroy(st);
  };
  if (cudaMalloc(&a, n * 16) != cudaSuccess ||
      (!inplace && cudaMalloc(&b, n * 16) != cudaSuccess)) {
    release();
    throw std::bad_alloc();
  }
  uint4* dst = inplace ? a : b;
  auto CK = [&](cudaError_t e) {
    if (e != cudaSuccess) {
      release();
      throw std::runtime_error(std::string("bandwidth probe: ") + cudaGetErrorString(e));
    }
  };
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaMemsetAsync(a, 0, n * 16, st));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float best = 1e30f;
  for (int shape = 0; shape < 3; ++shape)
    for (int r = 0; r < reps + 1; ++r) {  // the first launch of a shape is a warm-up
      CK(cudaEventRecord(e0, st));
      if (shape == 0)
        k_bw0<<<(unsigned)sms * 8, 256, 0, st>>>(a, dst, n);
      else if (shape == 1)
        k_bw1<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a, dst, n);
      else
        k_bw2<<<(unsigned)((n + 1023) / 1024), 256, 0, st>>>(a, dst, n);
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r > 0) best = std::min(best, ms);
    }
  CK(cudaGetLastError());
  release();
  return 2.0 * (double)n * 16.0 / (best * 1e-3) / 1e9;
}

void launch_fill(cudaStream_t st, const DField& f, long long count, double v) {
  if (count <= 0) return;
  const unsigned g = (unsigned)std::min<long long>((count + kBlock - 1) / kBlock, 148 * 64);
  if (f.prec == Prec::f64)
    k_fill<double><<<g, kBlock, 0, st>>>(static_cast<double*>(f.p), count, v);
  else
    k_fill<float><<<g, kBlock, 0, st>>>(static_cast<float*>(f.p), count, (float)v);
}

}  // namespace lbmgpu
