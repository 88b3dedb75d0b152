// AA pattern on AoS records with face buffers (direct addressing, full grid).
//
// The AoS window kernels (kernels_aos.cu) run the in-place odd sweep over a
// tile plus a one-cell halo ring and write back by slot ownership: a record
// on the tile rim is partly written by the neighbouring tile, so rim and halo
// records leave slot by slot (C1 fp64: ten write-back warps, 0.77 of the
// roofline for the AA pair). Here a slot whose two accessors sit in different
// blocks never lives in a record at all:
//   slot (k, R) is accessed by R in the even sweep and by R - c_k in the odd
//   sweep (AA, p/src/scheme_aap.cpp:100-173); when R - c_k is a fluid cell
//   outside R's block box (x-y tile x z chunk, unwrapped coordinates) the
//   slot's home is a face-buffer entry (faces.cuh), read and rewritten there
//   by both sweeps, one sweep at a time.
// Every block then reads and writes only its own records, whole: a plane of
// the tile is a few contiguous rows, one bulk copy in and one out per row
// (TMA engine), no halo records, no ownership lists. The record copies of
// face slots go stale; extraction first writes the face buffer back into
// the records (launch_aa_fb_faces flush), a load refills the buffer (fill).
//
// Odd sweep, node X at plane p: reads and rewrites slot (j, X + c_j) for
// every j (bounce: (opp j, X)), i.e. records of planes p - 1 .. p + 1 of the
// same block, or face entries. A 5-slot ring holds the block's planes:
// iteration p waits for plane p + 1, computes plane p, and (after the block
// barrier) stores plane p - 1, which no later node touches; the slot is
// refilled with plane p - 1 + 5 in the next iteration, so two planes are in
// flight while a plane is computed. The even sweep (local) stores plane p in
// iteration p.
#include "dispatch.h"
#include "faces.cuh"
#include "launch.h"

#include <algorithm>
#include <cstdlib>

namespace lbmgpu {
using namespace dev;

namespace {

template <class T>
struct AaFb {
  static constexpr int NS = 5;                                  // ring slots
  static constexpr int ROWF = kFbX * 19 + 32 / (int)sizeof(T);  // row + 16-byte phase slack
  static constexpr int BUF = kFbY * ROWF;
  // + one record before and after the ring: the odd sweep's record reads
  // towards a target outside the box (its value comes from the face buffer)
  // may index one record beyond a row
  static constexpr size_t kBytes = ((size_t)NS * BUF + 40) * sizeof(T);
  static constexpr int kThreads = 32 * kFbY;  // one warp per tile row; warp 0's lanes also load
  static constexpr int kBlocks = sizeof(T) == 8 ? 1 : 2;
};
static_assert(AaFb<double>::kBytes <= 227 * 1024 - 1024, "fp64 AA face-buffer ring too large");
static_assert(2 * (AaFb<float>::kBytes + 1024) <= 228 * 1024, "fp32 AA ring: two blocks per SM");

// bit k: slot (k, R) of home R = (x, y, z) lives in the face buffer (its
// odd-sweep accessor R - c_k is a fluid cell outside the block box)
__device__ __forceinline__ uint32_t fb_home_mask(const FbBlock& b, int x, int y, int z,
                                                 uint32_t bounce) {
  uint32_t m = 0;
  if (x == b.x0) m |= kMxp;
  if (x == b.x0 + b.txv - 1) m |= kMxm;
  if (y == b.y0) m |= kMyp;
  if (y == b.y0 + b.tyv - 1) m |= kMym;
  if (z == b.zb) m |= kMzp;
  if (z == b.ze - 1) m |= kMzm;
  uint32_t ob = 0;  // bit k = bounce bit opp(k)
#pragma unroll
  for (int k = 1; k < 19; ++k) ob |= ((bounce >> opp(k)) & 1u) << k;
  return m & ~ob;
}
// bit j: slot (j, X + c_j) that node X accesses in the odd sweep lives in the
// face buffer (X + c_j outside the box, link j not a bounce)
__device__ __forceinline__ uint32_t fb_nb_mask(const FbBlock& b, int x, int y, int z,
                                               uint32_t bounce) {
  uint32_t m = 0;
  if (x == b.x0) m |= kMxm;
  if (x == b.x0 + b.txv - 1) m |= kMxp;
  if (y == b.y0) m |= kMym;
  if (y == b.y0 + b.tyv - 1) m |= kMyp;
  if (z == b.zb) m |= kMzm;
  if (z == b.ze - 1) m |= kMzp;
  return m & ~bounce;
}
// face-buffer entry of slot (K, R), R = (x, y, z) in block b
template <int K>
__device__ __forceinline__ long long fb_home_slot(const FbGeo& G, const FbBlock& b, int x, int y,
                                                  int z) {
  return fb_slot<K>(G, b, x, y, z, x - cx(K), y - cy(K), z - cz(K));
}
// ... for the target (xr, yr, zr) = X + c_K of an odd-sweep access from block
// b, outside b's box (may wrap): the neighbouring block, tile indices wrapped
template <int K>
__device__ __forceinline__ long long fb_target_slot(const Lat& L, const FbGeo& G, const FbBlock& b,
                                                    int xr, int yr, int zr) {
  int tix = b.tix, tiy = b.tiy, ch = b.ch;
  if (xr < b.x0) {
    --tix;
    if (xr < 0) xr += L.nx, tix = G.tiles_x - 1;
  } else if (xr >= b.x0 + b.txv) {
    ++tix;
    if (xr >= L.nx) xr -= L.nx, tix = 0;
  }
  if (yr < b.y0) {
    --tiy;
    if (yr < 0) yr += L.ny, tiy = G.tiles_y - 1;
  } else if (yr >= b.y0 + b.tyv) {
    ++tiy;
    if (yr >= L.ny) yr -= L.ny, tiy = 0;
  }
  if (zr < b.zb) {
    --ch;
    if (zr < 0) zr += L.nz, ch = G.nchunks - 1;
  } else if (zr >= b.ze) {
    ++ch;
    if (zr >= L.nz) zr -= L.nz, ch = 0;
  }
  const FbBlock rb = fb_block(L, G, tix, tiy, ch);
  return fb_home_slot<K>(G, rb, xr, yr, zr);
}

// one warp: n elements shared -> global, s and g congruent mod 16 bytes: the
// 16-byte-aligned middle as one bulk copy (lane 0), head / tail elements by
// the lanes (a record row must not be stored as a superset: the bytes beyond
// it belong to other blocks' records)
template <class T>
__device__ __forceinline__ void fb_copy_out(T* g, const T* s, int n, int lane) {
  constexpr int V = 16 / (int)sizeof(T);
  int head = (int)(((16u - (uint32_t)(reinterpret_cast<uintptr_t>(g) & 15u)) & 15u) / sizeof(T));
  if (head > n) head = n;
  const int nmid = (n - head) / V * V;
  if (lane < head) g[lane] = s[lane];
  const int t0 = head + nmid;
  if (t0 + lane < n) g[t0 + lane] = s[t0 + lane];
  if (lane == 0 && nmid) {
    bulk_s2g(g + head, s + head, (uint32_t)nmid * (uint32_t)sizeof(T));
    bulk_commit();
  }
}

// Face-slot passes with compile-time directions: per face of the block box a
// warp-uniform (y rows, z planes) or lane (x columns) branch visits the five
// directions crossing it; a link crossing several faces is taken by the
// first of y, x, z (the order of fb_slot). No loops, no indirect branches.
// crosses_y(J) / crosses_x(J): the link from X along c_J leaves the box
// through a y / x face (masks ylo..: X on that face).
#define FB_FACE5(D0, D1, D2, D3, D4, OP) OP(D0) OP(D1) OP(D2) OP(D3) OP(D4)
#define FB_CY_M 4, 7, 11, 12, 15   /* c_y = -1 */
#define FB_CY_P 3, 10, 13, 14, 18  /* c_y = +1 */
#define FB_CX_M 2, 7, 8, 9, 10     /* c_x = -1 */
#define FB_CX_P 1, 15, 16, 17, 18  /* c_x = +1 */
#define FB_CZ_M 6, 8, 11, 13, 16   /* c_z = -1 */
#define FB_CZ_P 5, 9, 12, 14, 17   /* c_z = +1 */
#define FB_APPLY(M, OP) FB_APPLY_(M, OP)
#define FB_APPLY_(D0, D1, D2, D3, D4, OP) FB_FACE5(D0, D1, D2, D3, D4, OP)

template <class T, bool ODD>
__global__ void __launch_bounds__(AaFb<T>::kThreads, AaFb<T>::kBlocks)
    k_aa_fb(Fld<T, true> F, Lat L, Trt<T> op, FbGeo G, T* __restrict__ H) {
  using C = AaFb<T>;
  constexpr int NS = C::NS, ROWF = C::ROWF, BUF = C::BUF;
  extern __shared__ __align__(16) unsigned char fb_smem[];
  T* sm = reinterpret_cast<T*>(fb_smem) + 20;  // 16-byte aligned, a record of slack before
  __shared__ __align__(8) uint64_t full[NS];
  const int ntile = G.tiles_x * G.tiles_y;
  const int tile = (int)blockIdx.x % ntile, ch = (int)blockIdx.x / ntile;
  const FbBlock b = fb_block(L, G, tile % G.tiles_x, tile / G.tiles_x, ch);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&full[s], (uint32_t)b.tyv);
    mbar_fence_init();
  }
  __syncthreads();
  auto slot = [&](int p) { return (p - b.zb) % NS; };
  auto par = [&](int p) { return (uint32_t)((p - b.zb) / NS) & 1u; };
  // element offset of record (x0, y, p) and its 16-byte phase (elements)
  auto rowg = [&](int y, int p) {
    return ((long long)L.sx * ((long long)y + (long long)L.sy * p) + b.x0) * 19;
  };
  auto phase = [&](long long g) { return (int)(g & (long long)(16 / sizeof(T) - 1)); };
  // the loading warp: lane r copies row r of plane p (16-byte superset; the
  // over-read bytes land in the row's slack)
  auto load = [&](int p) {
    const int r = lane;
    if (r >= b.tyv) return;
    const long long g = rowg(b.y0 + r, p);
    const uintptr_t lo = reinterpret_cast<uintptr_t>(F.p + g) & ~(uintptr_t)15;
    const uintptr_t hi =
        (reinterpret_cast<uintptr_t>(F.p + g + (long long)b.txv * 19) + 15) & ~(uintptr_t)15;
    T* dst = sm + slot(p) * BUF + r * ROWF;  // data at dst + ph
    mbar_arrive_tx(&full[slot(p)], (uint32_t)(hi - lo));
    bulk_g2s(dst, reinterpret_cast<const void*>(lo), (uint32_t)(hi - lo), &full[slot(p)]);
  };
  if (warp == 0)
    for (int p = b.zb; p < min(b.ze, b.zb + NS); ++p) load(p);

  const int tx = lane, ty = warp;
  const bool act = ty < b.tyv && tx < b.txv;
  const int x = b.x0 + tx, y = b.y0 + ty;
  const int last = b.ze - 1 + (ODD ? 1 : 0);
  for (int p = b.zb; p <= last; ++p) {
    bulk_wait_read();
    fence_async_smem();
    __syncthreads();  // (A) iteration p - 1 done; its stores have read their slot
    if (warp == 0) {
      const int q = p - (ODD ? 2 : 1);  // the plane stored in iteration p - 1
      if (q >= b.zb && q + NS < b.ze) load(q + NS);
    }
    if (ty < b.tyv && p < b.ze) {
      if (ODD) {
        if (p == b.zb) mbar_wait(&full[slot(p)], par(p));
        if (p + 1 < b.ze) mbar_wait(&full[slot(p + 1)], par(p + 1));
      } else {
        mbar_wait(&full[slot(p)], par(p));
      }
      uint32_t bounce = 0;
      const bool live = act && fb_cell(L, x, y, p, bounce);
      if (live) {
        if constexpr (ODD) {
          // record rows of planes p - 1 .. p + 1, rows ty - 1 .. ty + 1 (a
          // row outside the box: a harmless dummy inside the ring; no access
          // through it survives the face-buffer fix-ups below)
          int rp[3][3];
#pragma unroll
          for (int dz = 0; dz < 3; ++dz)
#pragma unroll
            for (int dy = 0; dy < 3; ++dy) {
              const int pz = p - 1 + dz, r = ty - 1 + dy;
              rp[dz][dy] = (pz >= b.zb && pz < b.ze && r >= 0 && r < b.tyv)
                               ? slot(pz) * BUF + r * ROWF + phase(rowg(b.y0 + r, pz)) + tx * 19
                               : 19;
            }
          // slot k of the record at X + c_i (in the block box)
          auto at = [&](int i, int k) -> T& {
            return sm[rp[1 + cz(i)][1 + cy(i)] + cx(i) * 19 + k];
          };
          const uint32_t hm = fb_nb_mask(b, x, y, p, bounce);
          T f[19];
          f[0] = at(0, 0);
#pragma unroll
          for (int i = 1; i < 19; ++i) {
            const int j = opp(i);
            f[i] = ((bounce >> j) & 1u) ? at(0, i) : at(j, j);
          }
          // face slots (odd access of X: slot J of X + c_J outside the box)
          const bool ylo = ty == 0, yhi = ty == b.tyv - 1, xlo = tx == 0, xhi = tx == b.txv - 1;
          const bool zlo = p == b.zb, zhi = p == b.ze - 1;
          auto cyo = [&](int J) { return (cy(J) < 0 && ylo) || (cy(J) > 0 && yhi); };
          auto cxo = [&](int J) { return (cx(J) < 0 && xlo) || (cx(J) > 0 && xhi); };
#define FB_ORD(J)                                                                     \
  if (!((bounce >> J) & 1u)) f[opp(J)] = H[fb_target_slot<J>(L, G, b, x + cx(J), y + cy(J), p + cz(J))];
#define FB_ORD_X(J) if (!cyo(J)) { FB_ORD(J) }
#define FB_ORD_Z(J) if (!cyo(J) && !cxo(J)) { FB_ORD(J) }
          if (ylo) { FB_APPLY(FB_CY_M, FB_ORD) }
          if (yhi) { FB_APPLY(FB_CY_P, FB_ORD) }
          if (xlo) { FB_APPLY(FB_CX_M, FB_ORD_X) }
          if (xhi) { FB_APPLY(FB_CX_P, FB_ORD_X) }
          if (zlo) { FB_APPLY(FB_CZ_M, FB_ORD_Z) }
          if (zhi) { FB_APPLY(FB_CZ_P, FB_ORD_Z) }
#undef FB_ORD
#undef FB_ORD_X
#undef FB_ORD_Z
          collide(op, f);
          at(0, 0) = f[0];
#pragma unroll
          for (int j = 1; j < 19; ++j) {
            if ((bounce >> j) & 1u)
              at(0, opp(j)) = f[j];
            else if (!((hm >> j) & 1u))
              at(j, j) = f[j];
          }
#define FB_OWR(J)                                                                     \
  if (!((bounce >> J) & 1u)) H[fb_target_slot<J>(L, G, b, x + cx(J), y + cy(J), p + cz(J))] = f[J];
#define FB_OWR_X(J) if (!cyo(J)) { FB_OWR(J) }
#define FB_OWR_Z(J) if (!cyo(J) && !cxo(J)) { FB_OWR(J) }
          if (ylo) { FB_APPLY(FB_CY_M, FB_OWR) }
          if (yhi) { FB_APPLY(FB_CY_P, FB_OWR) }
          if (xlo) { FB_APPLY(FB_CX_M, FB_OWR_X) }
          if (xhi) { FB_APPLY(FB_CX_P, FB_OWR_X) }
          if (zlo) { FB_APPLY(FB_CZ_M, FB_OWR_Z) }
          if (zhi) { FB_APPLY(FB_CZ_P, FB_OWR_Z) }
#undef FB_OWR
#undef FB_OWR_X
#undef FB_OWR_Z
        } else {
          T* rec = sm + slot(p) * BUF + ty * ROWF + phase(rowg(y, p)) + tx * 19;
          T f[19];
#pragma unroll
          for (int i = 0; i < 19; ++i) f[i] = rec[i];
          // face slots of home R: slot K whose source R - c_K is outside the box
          const bool ylo = ty == 0, yhi = ty == b.tyv - 1, xlo = tx == 0, xhi = tx == b.txv - 1;
          const bool zlo = p == b.zb, zhi = p == b.ze - 1;
          auto cyh = [&](int K) { return (cy(K) > 0 && ylo) || (cy(K) < 0 && yhi); };
          auto cxh = [&](int K) { return (cx(K) > 0 && xlo) || (cx(K) < 0 && xhi); };
#define FB_ERD(K) if (!((bounce >> opp(K)) & 1u)) f[K] = H[fb_home_slot<K>(G, b, x, y, p)];
#define FB_ERD_X(K) if (!cyh(K)) { FB_ERD(K) }
#define FB_ERD_Z(K) if (!cyh(K) && !cxh(K)) { FB_ERD(K) }
          if (ylo) { FB_APPLY(FB_CY_P, FB_ERD) }
          if (yhi) { FB_APPLY(FB_CY_M, FB_ERD) }
          if (xlo) { FB_APPLY(FB_CX_P, FB_ERD_X) }
          if (xhi) { FB_APPLY(FB_CX_M, FB_ERD_X) }
          if (zlo) { FB_APPLY(FB_CZ_P, FB_ERD_Z) }
          if (zhi) { FB_APPLY(FB_CZ_M, FB_ERD_Z) }
#undef FB_ERD
#undef FB_ERD_X
#undef FB_ERD_Z
          collide(op, f);
          // post_i -> slot (opp i, R); a face slot's record copy is stale anyway
#pragma unroll
          for (int i = 0; i < 19; ++i) rec[opp(i)] = f[i];
#define FB_EWR(K) if (!((bounce >> opp(K)) & 1u)) H[fb_home_slot<K>(G, b, x, y, p)] = f[opp(K)];
#define FB_EWR_X(K) if (!cyh(K)) { FB_EWR(K) }
#define FB_EWR_Z(K) if (!cyh(K) && !cxh(K)) { FB_EWR(K) }
          if (ylo) { FB_APPLY(FB_CY_P, FB_EWR) }
          if (yhi) { FB_APPLY(FB_CY_M, FB_EWR) }
          if (xlo) { FB_APPLY(FB_CX_P, FB_EWR_X) }
          if (xhi) { FB_APPLY(FB_CX_M, FB_EWR_X) }
          if (zlo) { FB_APPLY(FB_CZ_P, FB_EWR_Z) }
          if (zhi) { FB_APPLY(FB_CZ_M, FB_EWR_Z) }
#undef FB_EWR
#undef FB_EWR_X
#undef FB_EWR_Z
        }
      }
    }
    fence_async_smem();
    __syncthreads();  // (B) every write into the plane stored below is done
    const int q = ODD ? p - 1 : p;
    if (warp < b.tyv && q >= b.zb && q < b.ze) {
      const long long g = rowg(b.y0 + warp, q);
      fb_copy_out(F.p + g, sm + slot(q) * BUF + warp * ROWF + phase(g), b.txv * 19, lane);
    }
  }
  bulk_wait_all();
}

// face buffer <-> records: fill (records -> buffer, after a load) or flush
// (buffer -> records, before an extraction)
template <class T, bool FILL>
__global__ void __launch_bounds__(kFbThreads)
    k_aa_fb_faces(Fld<T, true> F, Lat L, FbGeo G, T* __restrict__ H) {
  const int ntile = G.tiles_x * G.tiles_y;
  const int tile = (int)blockIdx.x % ntile, ch = (int)blockIdx.x / ntile;
  const FbBlock b = fb_block(L, G, tile % G.tiles_x, tile / G.tiles_x, ch);
  const int tx = threadIdx.x % kFbX, ty = threadIdx.x / kFbX;
  if (tx >= b.txv || ty >= b.tyv) return;
  const int x = b.x0 + tx, y = b.y0 + ty;
  for (int z = b.zb; z < b.ze; ++z) {
    uint32_t bounce = 0;
    if (!fb_cell(L, x, y, z, bounce)) continue;
    const uint32_t hm = fb_home_mask(b, x, y, z, bounce);
    if (!hm) continue;
    T* rec = F.p + ((size_t)x + (size_t)L.sx * ((size_t)y + (size_t)L.sy * z)) * 19;
#define FB_FACE(K)                                   \
  if ((hm >> K) & 1u) {                              \
    T* h = H + fb_home_slot<K>(G, b, x, y, z);       \
    if (FILL) *h = rec[K]; else rec[K] = *h;         \
  }
    FB_FACE(1) FB_FACE(2) FB_FACE(3) FB_FACE(4) FB_FACE(5) FB_FACE(6) FB_FACE(7) FB_FACE(8)
    FB_FACE(9) FB_FACE(10) FB_FACE(11) FB_FACE(12) FB_FACE(13) FB_FACE(14) FB_FACE(15)
    FB_FACE(16) FB_FACE(17) FB_FACE(18)
#undef FB_FACE
  }
}

template <class T>
FbGeo aa_fb_geo(const Lat& L) {
  return fb_geo(L, AaFb<T>::kBlocks);
}

template <class T, bool ODD>
void launch_aa_fb_t(cudaStream_t st, const DField& f, const Lat& L, const TrtHost& op, void* h) {
  using C = AaFb<T>;
  static int set_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (set_dev != dev) {
    cudaFuncSetAttribute(k_aa_fb<T, ODD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kBytes);
    set_dev = dev;
  }
  const FbGeo G = aa_fb_geo<T>(L);
  const unsigned grid = (unsigned)(G.tiles_x * G.tiles_y * G.nchunks);
  k_aa_fb<T, ODD><<<grid, C::kThreads, C::kBytes, st>>>(fld<T, true>(f), L, cast_op<T>(op), G,
                                                        static_cast<T*>(h));
}

}  // namespace

// AoS, full grid, no halo or ghost planes; opt-in (LBMGPU_AOS_FB=1) until it
// beats the ownership windows
bool aa_fb_ok(const DField& f, const Lat& L) {
  if (!f.aos) return false;
  const char* e = std::getenv("LBMGPU_AOS_FB");
  if (!(e && e[0] == '1')) return false;
  if (L.ox || L.oy || L.oz || L.zghost || L.znowrap || L.sx != L.nx || L.sy != L.ny) return false;
  return L.cell_begin == 0 && (unsigned long long)L.ncells == (unsigned long long)L.nx * L.ny * L.nz;
}

size_t aa_fb_face_elems(const DField& f, const Lat& L) {
  const FbGeo G = f.prec == Prec::f64 ? aa_fb_geo<double>(L) : aa_fb_geo<float>(L);
  return (size_t)G.tiles_x * G.tiles_y * G.nchunks * (size_t)G.region;
}

void launch_aa_fb(cudaStream_t st, const DField& f, const Lat& L, const TrtHost& op, bool odd,
                  void* h) {
  if (f.prec == Prec::f64) {
    if (odd) launch_aa_fb_t<double, true>(st, f, L, op, h);
    else launch_aa_fb_t<double, false>(st, f, L, op, h);
  } else {
    if (odd) launch_aa_fb_t<float, true>(st, f, L, op, h);
    else launch_aa_fb_t<float, false>(st, f, L, op, h);
  }
}

void launch_aa_fb_faces(cudaStream_t st, const DField& f, const Lat& L, bool fill, void* h) {
  if (f.prec == Prec::f64) {
    const FbGeo G = aa_fb_geo<double>(L);
    const unsigned grid = (unsigned)(G.tiles_x * G.tiles_y * G.nchunks);
    if (fill)
      k_aa_fb_faces<double, true><<<grid, kFbThreads, 0, st>>>(fld<double, true>(f), L, G, (double*)h);
    else
      k_aa_fb_faces<double, false><<<grid, kFbThreads, 0, st>>>(fld<double, true>(f), L, G, (double*)h);
  } else {
    const FbGeo G = aa_fb_geo<float>(L);
    const unsigned grid = (unsigned)(G.tiles_x * G.tiles_y * G.nchunks);
    if (fill)
      k_aa_fb_faces<float, true><<<grid, kFbThreads, 0, st>>>(fld<float, true>(f), L, G, (float*)h);
    else
      k_aa_fb_faces<float, false><<<grid, kFbThreads, 0, st>>>(fld<float, true>(f), L, G, (float*)h);
  }
}

}  // namespace lbmgpu
