// SWAP in one sweep with face buffers (SoA, direct addressing).
//
// What a SWAP sweep computes (p/src/scheme_swap.cpp:172-235), independent of
// its sequential order:
//   push  (opposed layout in and out): X collides from its opposed slots
//         (opp i, X) and its post value of direction k lands in (opp k, X+c_k),
//         or in (k, X) when link k bounces or wraps (a periodic-seam link: the
//         fix-up list exchanges it, exactly as before);
//   pull  (natural layout in and out, fix-up list applied first): X collides
//         from (i, X - c_i), or (opp i, X) when that link bounces or wraps,
//         and stores natural (i, X).
// Both are an in-place streaming step: every slot is read by one node and
// rewritten by one (other) node within the sweep. The two-pass GPU form
// (collide, then exchange) moves 2 x 19 values twice (0.52 of the roofline,
// its bound). Here ONE pass moves each value once:
//   * a block owns a 32 x 8 x-y tile and a z chunk and marches through z;
//     inside the block every read of a plane's slots happens in an earlier
//     iteration, or before the block barrier that precedes the writes into
//     that plane (push: node p+1's inputs are read before node p's outputs
//     land; pull: node p's inputs from plane p+1 are read one iteration
//     before plane p+1's nodes rewrite it), so in-block links are exchanged
//     in place with no other ordering;
//   * links between blocks (tile faces, chunk faces; ~9 % of the links of a
//     32 x 8 tile with 64-plane chunks) never go in place: the sender writes
//     its value into the receiver's face buffer of this sweep's parity,
//     H[t & 1], and the receiver reads it in the NEXT sweep from the same
//     buffer, while this sweep's receiver reads the other parity. No block
//     ever waits for another one. (Pull also stores the value naturally, so
//     the natural state stays complete for the gathering extraction.)
// A face-buffer slot is (receiver block, face, incoming direction, position
// on the face, plane): Hy (rows y0 - 1 / y0 + TY), Hx (columns x0 - 1 /
// x0 + TX), Hz (the chunk's planes zb - 1 / ze), first match in that order.
// After a load the incoming face values are gathered once from the field
// (launch_swap1_fill); before a push extraction they are written back into
// their opposed slots (launch_swap1_flush). Bit-identical to the reference:
// every node collides exactly the values the sequential sweep gives it.
#include "dispatch.h"
#include "launch.h"
#include "faces.cuh"

#include <algorithm>
#include <cstdlib>
#include <utility>

namespace lbmgpu {
using namespace dev;

namespace {

// Per-thread frame of the sweep: the node's position in the block box and
// the strides of the neighbouring blocks' face regions, and per plane two
// link masks (bit k: the link along c_k from the node):
//   local  the link bounces or leaves the domain (a periodic wrap: the fix-up
//          list's) — its value stays in the node's own column;
//   cross  the other end is inside the domain but outside the block box — its
//          value goes through a face buffer.
// Both come from the stencil's per-axis direction masks (kMxm ... kMzp)
// selected by the x (per lane), y (per row) and z (per plane) flags, so the
// per-direction work is a bit test; the face-buffer slot is the one fb_slot
// (faces.cuh) names, with the receiver block and its coordinates derived
// from the flags instead of recomputed from cell coordinates.
struct S1Frame {
  bool fxl, fxh, fyl, fyh, fzl, fzh;  // on the box's low / high face
  bool dxl, dxh, dyl, dyh, dzl, dzh;  // on the domain's low / high face
  int tx, ty, pz;                     // position in the box
  int zc;
  // face-buffer element offsets (32-bit: a whole buffer is < 2^32 elements):
  // this block's region and its neighbours' strides; the input slots of this
  // thread on its y / x faces at the current plane and on its z faces
  uint32_t base, rx, ry, rz, hy, hx, hz;
  uint32_t iy, ix, iz;
  uint32_t box;  // LBM_S1_CROSSMASK: links leaving the block box at this plane
};
// the link along (CX, CY, CZ) leaves the domain / crosses the block box;
// only the flags of the direction's nonzero components are tested (y / z
// flags are uniform over a warp, x flags per lane)
template <int CX, int CY, int CZ>
__device__ __forceinline__ bool s1_leaves(const S1Frame& q) {
  return (CX < 0 && q.dxl) || (CX > 0 && q.dxh) || (CY < 0 && q.dyl) || (CY > 0 && q.dyh) ||
         (CZ < 0 && q.dzl) || (CZ > 0 && q.dzh);
}
template <int CX, int CY, int CZ>
__device__ __forceinline__ bool s1_crosses(const S1Frame& q) {
  return (CX < 0 && q.fxl) || (CX > 0 && q.fxh) || (CY < 0 && q.fyl) || (CY > 0 && q.fyh) ||
         (CZ < 0 && q.fzl) || (CZ > 0 && q.fzh);
}
// link K (along (CX, CY, CZ)) stays local: it bounces or leaves the domain.
// LBM_S1_LOCALMASK: `bounce` already holds the leaving links (one mask per
// plane, a bit test per link) instead of testing the edge flags per link
#ifndef LBM_S1_LOCALMASK
#define LBM_S1_LOCALMASK 1
#endif
template <int K, int CX, int CY, int CZ>
__device__ __forceinline__ bool s1_local(const S1Frame& q, uint32_t bounce) {
  if (LBM_S1_LOCALMASK) return (bounce >> K) & 1u;
  return ((bounce >> K) & 1u) || s1_leaves<CX, CY, CZ>(q);
}
// link K crosses the block box: a bit of the plane's box mask (CM) or the
// face flags of the direction's components
template <bool CM, int K, int CX, int CY, int CZ>
__device__ __forceinline__ bool s1_cross(const S1Frame& q) {
  if (CM) return (q.box >> K) & 1u;
  return s1_crosses<CX, CY, CZ>(q);
}
// Per kernel (measured on C1 / C4, the choices only change registers and
// schedule): the box as a mask for fp64 push (no spills: C1 0.77 -> 0.81);
// pull keeps a second frame for the next node across the barrier (C1 fp64
// 0.53 -> 0.56), push recomputes the plane fields instead (fp64 0.58 -> 0.77)
#ifndef LBM_S1_PULL_CM
#define LBM_S1_PULL_CM 0
#endif
#ifndef LBM_S1_F32_CM
#define LBM_S1_F32_CM 0
#endif
template <class T, bool PUSH>
struct S1Cfg {
  static constexpr bool kCrossMask =
      sizeof(T) == 8 ? (PUSH || LBM_S1_PULL_CM) : (PUSH && LBM_S1_F32_CM);
  static constexpr bool kTwoFrames = !PUSH;
};
__device__ __forceinline__ uint32_t s1_axis_mask(bool lo, bool hi, uint32_t mlo, uint32_t mhi) {
  return (lo ? mlo : 0u) | (hi ? mhi : 0u);
}
// plane bases of the field (kernel parameters, so constant-bank operands):
// pl[i] = plane i; sh[i] = push: the store target of output i, plane opp i
// shifted by +c_i (pl[opp i] + off_i); pull: the load source of input i,
// plane i shifted by -c_i. Every plain access is then one IMAD.WIDE.U32 of
// the 32-bit storage index.
template <class T>
struct S1Tab {
  T* pl[19];
  T* sh[19];
};
// slot of the value this node receives along direction I from S = X - c_I
// (outside the box): in this block's region, keyed by the face S lies across
#ifndef LBM_S1_SLOT_INLINE
#define LBM_S1_SLOT_INLINE __forceinline__
#endif
template <int I>
__device__ LBM_S1_SLOT_INLINE uint32_t s1_in_slot(const S1Frame& q) {
  constexpr int X = cx(I), Y = cy(I), Z = cz(I);
  if ((Y > 0 && q.fyl) || (Y < 0 && q.fyh)) {
    constexpr int side = Y > 0 ? 0 : 1, qq = face_q(1, Y > 0 ? 1 : -1, I);
    return q.iy + (uint32_t)((side * 5 + qq) * kFbX);
  }
  if ((X > 0 && q.fxl) || (X < 0 && q.fxh)) {
    constexpr int side = X > 0 ? 0 : 1, qq = face_q(0, X > 0 ? 1 : -1, I);
    return q.ix + (uint32_t)((side * 5 + qq) * kFbY);
  }
  constexpr int side = Z > 0 ? 0 : 1, qq = face_q(2, Z > 0 ? 1 : -1, I);
  return q.iz + (uint32_t)((side * 5 + qq) * kFbY * kFbX);
}
// slot of the value this node sends along direction K to R = X + c_K (outside
// the box): in the receiving block's region, keyed by the face X lies across
template <int K>
__device__ LBM_S1_SLOT_INLINE uint32_t s1_out_slot(const S1Frame& q) {
  constexpr int X = cx(K), Y = cy(K), Z = cz(K);
  const int ex = (X < 0 && q.fxl) ? -1 : ((X > 0 && q.fxh) ? 1 : 0);
  const int ey = (Y < 0 && q.fyl) ? -1 : ((Y > 0 && q.fyh) ? 1 : 0);
  const int ez = (Z < 0 && q.fzl) ? -1 : ((Z > 0 && q.fzh) ? 1 : 0);
  const uint32_t rb = q.base + (uint32_t)ex * q.rx + (uint32_t)ey * q.ry + (uint32_t)ez * q.rz;
  const int px = ex > 0 ? 0 : (ex < 0 ? kFbX - 1 : q.tx + X);
  const int py = ey > 0 ? 0 : (ey < 0 ? kFbY - 1 : q.ty + Y);
  const int pz = ez > 0 ? 0 : (ez < 0 ? q.zc - 1 : q.pz + Z);
  if (ey != 0) {
    constexpr int side = Y > 0 ? 0 : 1, qq = face_q(1, Y > 0 ? 1 : -1, K);
    return rb + q.hy + (uint32_t)(((pz * 2 + side) * 5 + qq) * kFbX + px);
  }
  if (ex != 0) {
    constexpr int side = X > 0 ? 0 : 1, qq = face_q(0, X > 0 ? 1 : -1, K);
    return rb + q.hx + (uint32_t)(((pz * 2 + side) * 5 + qq) * kFbY + py);
  }
  constexpr int side = Z > 0 ? 0 : 1, qq = face_q(2, Z > 0 ? 1 : -1, K);
  return rb + q.hz + (uint32_t)(((side * 5 + qq) * kFbY + py) * kFbX + px);
}

// the 19 inputs of the node: push (opp i, X); pull (i, X - c_i), or (opp i, X)
// when that link (opp i from X) is local; a crossing input comes from the
// face buffer of the last sweep (the field load is issued regardless, so the
// loads of a node leave together)
template <bool PUSH, bool CM, int I, class T>
__device__ __forceinline__ void s1_in(const S1Tab<T>& F, const T* hprev, const FbGeo& G,
                                      const S1Frame& q, uint32_t s, uint32_t bounce, T (&v)[19]) {
  constexpr int X = cx(I), Y = cy(I), Z = cz(I), J = opp(I);
  const bool local = s1_local<J, -X, -Y, -Z>(q, bounce);
  if (!local && s1_cross<CM, J, -X, -Y, -Z>(q))
    v[I] = hprev[s1_in_slot<I>(q)];
  else if (PUSH || local)
    v[I] = F.pl[J][s];
  else
    v[I] = F.sh[I][s];
}
// the 19 outputs: push (opp k, X + c_k), or (k, X) when link k is local;
// pull (k, X); a crossing output goes to the receiver's face buffer instead
// (push) or as well (pull)
template <bool PUSH, bool CM, int K, class T>
__device__ __forceinline__ void s1_out(const S1Tab<T>& F, T* hcur, const FbGeo& G,
                                       const S1Frame& q, uint32_t s, uint32_t bounce,
                                       const T (&v)[19]) {
  constexpr int X = cx(K), Y = cy(K), Z = cz(K);
  const bool local = s1_local<K, X, Y, Z>(q, bounce);
  const bool cross = !local && s1_cross<CM, K, X, Y, Z>(q);
  if (cross) hcur[s1_out_slot<K>(q)] = v[K];
  if (!PUSH || local)
    F.pl[K][s] = v[K];
  else if (!cross)
    F.sh[K][s] = v[K];
}
template <bool PUSH, bool CM, class T, int... Is>
__device__ __forceinline__ void s1_read(const S1Tab<T>& F, const T* hprev, const FbGeo& G,
                                        const S1Frame& q, uint32_t s, uint32_t bounce, T (&v)[19],
                                        std::integer_sequence<int, Is...>) {
  v[0] = F.pl[0][s];
  (s1_in<PUSH, CM, Is + 1>(F, hprev, G, q, s, bounce, v), ...);
}
// the inputs of the node read one iteration ahead (SEL 1) or in the node's
// own iteration (SEL 2, with the rest value). Pull: sources one plane below
// (c_z = +1) must be read ahead (node z - 1 rewrites them); the others are
// rewritten in the node's own iteration or later and may be read either way.
// LBM_S1_PULL_AHEAD = 1: only the c_z = +1 inputs ahead; 2: every c_z != 0
// input ahead (the nine in-plane ones in the node's iteration; C1 fp64 0.58
// -> 0.51: more registers live across the barrier)
#ifndef LBM_S1_PULL_AHEAD
#define LBM_S1_PULL_AHEAD 1
#endif
__host__ __device__ constexpr bool s1_early(int i) {
  return LBM_S1_PULL_AHEAD == 1 ? cz(i) == 1 : cz(i) != 0;
}
template <bool PUSH, bool CM, int SEL, int I, class T>
__device__ __forceinline__ void s1_in_sel(const S1Tab<T>& F, const T* hprev, const FbGeo& G,
                                          const S1Frame& q, uint32_t s, uint32_t bounce,
                                          T (&v)[19]) {
  if constexpr ((SEL == 1) == s1_early(I)) s1_in<PUSH, CM, I>(F, hprev, G, q, s, bounce, v);
}
template <bool PUSH, bool CM, int SEL, class T, int... Is>
__device__ __forceinline__ void s1_read_sel(const S1Tab<T>& F, const T* hprev, const FbGeo& G,
                                            const S1Frame& q, uint32_t s, uint32_t bounce,
                                            T (&v)[19], std::integer_sequence<int, Is...>) {
  if (SEL == 2) v[0] = F.pl[0][s];
  (s1_in_sel<PUSH, CM, SEL, Is + 1>(F, hprev, G, q, s, bounce, v), ...);
}
template <bool PUSH, bool CM, class T, int... Ks>
__device__ __forceinline__ void s1_write(const S1Tab<T>& F, T* hcur, const FbGeo& G,
                                         const S1Frame& q, uint32_t s, uint32_t bounce,
                                         const T (&v)[19], std::integer_sequence<int, Ks...>) {
  F.pl[0][s] = v[0];
  (s1_out<PUSH, CM, Ks + 1>(F, hcur, G, q, s, bounce, v), ...);
}

// resident 256-thread blocks per SM (the register budget; the z chunks are
// sized for these waves): fp64 2 (<= 128 registers), fp32 LBM_S1_BLOCKS32
#ifndef LBM_S1_BLOCKS
#define LBM_S1_BLOCKS 2
#endif
#ifndef LBM_S1_BLOCKS32
#define LBM_S1_BLOCKS32 3
#endif
// warp-uniform inner fast path of k_swap1's push (per precision)
#ifndef LBM_S1_PUSH_FAST32
#define LBM_S1_PUSH_FAST32 0
#endif
#ifndef LBM_S1_PUSH_FAST64
#define LBM_S1_PUSH_FAST64 0
#endif
template <class T>
struct S1PushFast {
  static constexpr bool value = sizeof(T) == 8 ? LBM_S1_PUSH_FAST64 != 0 : LBM_S1_PUSH_FAST32 != 0;
};
template <class T>
struct S1Blocks {
  static constexpr int value = sizeof(T) == 8 ? LBM_S1_BLOCKS : LBM_S1_BLOCKS32;
};
static int s1_blocks(Prec p) { return p == Prec::f64 ? LBM_S1_BLOCKS : LBM_S1_BLOCKS32; }
// AoS: the staged ring (one fp64 / two fp32 blocks per SM)
static int s1_blocks(const DField& f) {
  return f.aos ? (f.prec == Prec::f64 ? 1 : 2) : s1_blocks(f.prec);
}

// One sweep over a block's planes. Iteration z reads node z + 1's inputs
// (push: its own slots in plane z + 1; pull: planes z .. z + 2), then, after
// the block barrier, node z collides and writes (push: planes z - 1 .. z + 1;
// pull: plane z). Every in-block read of a slot precedes the barrier before
// which the slot is rewritten: push plane z + 1 is read before node z's
// outputs land, pull plane z is read by nodes z - 1 .. z + 1 in iterations
// <= z.
template <class T, bool PUSH>
__global__ void __launch_bounds__(kFbThreads, S1Blocks<T>::value)
    k_swap1(const __grid_constant__ S1Tab<T> F, Lat L, Trt<T> op, FbGeo G, T* __restrict__ hcur,
            const T* __restrict__ hprev) {
  const int ntile = G.tiles_x * G.tiles_y;
  const int tile = (int)blockIdx.x % ntile, ch = (int)blockIdx.x / ntile;
  const FbBlock b = fb_block(L, G, tile % G.tiles_x, tile / G.tiles_x, ch);
  const int tx = threadIdx.x % kFbX, ty = threadIdx.x / kFbX;
  const bool act = tx < b.txv && ty < b.tyv;
  const int x = b.x0 + tx, y = b.y0 + ty;
  const uint32_t sxy = (uint32_t)L.sxy;
  const uint32_t s0 = (uint32_t)x + (uint32_t)L.sx * (uint32_t)y;
  const auto seq = std::make_integer_sequence<int, 18>{};
  constexpr bool CM = S1Cfg<T, PUSH>::kCrossMask, TWO = S1Cfg<T, PUSH>::kTwoFrames;
  S1Frame qf;
  qf.fxl = tx == 0, qf.fxh = tx == b.txv - 1, qf.fyl = ty == 0, qf.fyh = ty == b.tyv - 1;
  qf.dxl = x == 0, qf.dxh = x == L.nx - 1, qf.dyl = y == 0, qf.dyh = y == L.ny - 1;
  qf.tx = tx, qf.ty = ty, qf.zc = G.zc;
  qf.base = (uint32_t)b.base;
  qf.rx = (uint32_t)G.region;
  qf.ry = (uint32_t)((long long)G.tiles_x * G.region);
  qf.rz = (uint32_t)((long long)G.tiles_x * G.tiles_y * G.region);
  qf.hy = (uint32_t)G.hy, qf.hx = (uint32_t)G.hx, qf.hz = (uint32_t)G.hz;
  qf.iz = qf.base + qf.hz + (uint32_t)(ty * kFbX + tx);
  const uint32_t leave_xy = s1_axis_mask(qf.dxl, qf.dxh, kMxm, kMxp) | s1_axis_mask(qf.dyl, qf.dyh, kMym, kMyp);
  const uint32_t box_xy = s1_axis_mask(qf.fxl, qf.fxh, kMxm, kMxp) | s1_axis_mask(qf.fyl, qf.fyh, kMym, kMyp);
  auto at_plane = [&](S1Frame& q, int z) {
    q.pz = z - b.zb;
    q.fzl = z == b.zb, q.fzh = z == b.ze - 1;
    q.dzl = z == 0, q.dzh = z == L.nz - 1;
    q.iy = q.base + q.hy + (uint32_t)(q.pz * 10 * kFbX + tx);
    q.ix = q.base + q.hx + (uint32_t)(q.pz * 10 * kFbY + ty);
    if (CM) q.box = box_xy | s1_axis_mask(q.fzl, q.fzh, kMzm, kMzp);
  };
  T f[19];
  uint32_t bf = 0, bg = 0;
  bool lf = false, lg = false;
  if constexpr (!PUSH) {
    // Pull: only the five inputs of node z + 1 from plane z (c_z = +1) must
    // be read before node z's stores (iteration z); its other inputs (planes
    // z + 1, z + 2) are rewritten only by nodes z + 1, z + 2, so they are read
    // in iteration z + 1 itself. Five values cross the barrier instead of 19.
    if (act) {
      lf = fb_cell(L, x, y, b.zb, bf);
      if (LBM_S1_LOCALMASK) bf |= leave_xy | s1_axis_mask(b.zb == 0, b.zb == L.nz - 1, kMzm, kMzp);
      at_plane(qf, b.zb);
      if (lf) s1_read_sel<PUSH, CM, 1>(F, hprev, G, qf, s0 + (uint32_t)b.zb * sxy, bf, f, seq);
    }
    for (int z = b.zb; z < b.ze; ++z) {
      if (lf) {
        at_plane(qf, z);
        s1_read_sel<PUSH, CM, 2>(F, hprev, G, qf, s0 + (uint32_t)z * sxy, bf, f, seq);
      }
      T g[19];
      lg = false;
      if (act && z + 1 < b.ze) {
        lg = fb_cell(L, x, y, z + 1, bg);
        if (LBM_S1_LOCALMASK) bg |= leave_xy | s1_axis_mask(z + 1 == 0, z + 1 == L.nz - 1, kMzm, kMzp);
        at_plane(qf, z + 1);
        if (lg) s1_read_sel<PUSH, CM, 1>(F, hprev, G, qf, s0 + (uint32_t)(z + 1) * sxy, bg, g, seq);
      }
      __syncthreads();
      if (lf) {
        collide(op, f);
        at_plane(qf, z);
        s1_write<PUSH, CM>(F, hcur, G, qf, s0 + (uint32_t)z * sxy, bf, f, seq);
      }
#pragma unroll
      for (int i = 1; i < 19; ++i)
        if (s1_early(i)) f[i] = g[i];
      bf = bg;
      lf = lg;
    }
    return;
  }
  // push: node z + 1's inputs (its own column) are all read in iteration z;
  // qg: the frame of node z + 1 (TWO), else qf's per-plane fields are
  // recomputed (at_plane) before each node's reads and writes
  S1Frame qg = qf;
  T g[19];
  // warp-uniform inner case (as in k_swap1_pa below): the y / z flags and the
  // link mask as constants, only the end lanes' x-crossing links remain
  constexpr bool kFast = S1PushFast<T>::value;
  const bool row_inner = ty > 0 && ty < b.tyv - 1;
  auto inner = [&](int z, bool l, uint32_t bm) {
    if (!kFast) return false;
    return __all_sync(0xffffffffu, l && bm == 0u && row_inner && z > b.zb && z < b.ze - 1) != 0;
  };
  auto inner_frame = [&](int z) {
    S1Frame qi = qf;
    at_plane(qi, z);
    qi.fyl = qi.fyh = qi.fzl = qi.fzh = false;
    return qi;
  };
  bool ff = false, fg = false;
  if (act) {
    lf = fb_cell(L, x, y, b.zb, bf);
    if (LBM_S1_LOCALMASK) bf |= leave_xy | s1_axis_mask(b.zb == 0, b.zb == L.nz - 1, kMzm, kMzp);
    at_plane(qf, b.zb);
    if (lf) s1_read<PUSH, CM>(F, hprev, G, qf, s0 + (uint32_t)b.zb * sxy, bf, f, seq);
  }
  for (int z = b.zb; z < b.ze; ++z) {
    lg = false;
    const bool more = act && z + 1 < b.ze;
    if (more) {
      lg = fb_cell(L, x, y, z + 1, bg);
      if (LBM_S1_LOCALMASK) bg |= leave_xy | s1_axis_mask(z + 1 == 0, z + 1 == L.nz - 1, kMzm, kMzp);
    }
    fg = inner(z + 1, lg, bg);
    if (fg) {
      const S1Frame qi = inner_frame(z + 1);
      s1_read<PUSH, false>(F, hprev, G, qi, s0 + (uint32_t)(z + 1) * sxy, 0u, g, seq);
    } else if (more) {
      S1Frame& qn = TWO ? qg : qf;
      at_plane(qn, z + 1);
      if (lg) s1_read<PUSH, CM>(F, hprev, G, qn, s0 + (uint32_t)(z + 1) * sxy, bg, g, seq);
    }
    __syncthreads();
    if (ff) {
      collide(op, f);
      const S1Frame qi = inner_frame(z);
      s1_write<PUSH, false>(F, hcur, G, qi, s0 + (uint32_t)z * sxy, 0u, f, seq);
    } else if (lf) {
      collide(op, f);
      if (!TWO) at_plane(qf, z);
      s1_write<PUSH, CM>(F, hcur, G, qf, s0 + (uint32_t)z * sxy, bf, f, seq);
    }
#pragma unroll
    for (int i = 0; i < 19; ++i) f[i] = g[i];
    bf = bg;
    lf = lg;
    ff = fg;
    if (TWO) qf = qg;
  }
}

// ---------------------------------------------------------------------------
// SWAP pull in one sweep, SoA, with the inputs staged by cp.async two nodes
// ahead. k_swap1's pull reads 14 of a node's 19 inputs in the node's own
// iteration and collides right after the barrier, so their latency is exposed
// once per plane (C1 fp64 0.58); reading all 19 one node ahead in registers
// spills (0.51). Here node z + 2's 19 inputs are copied asynchronously into a
// thread-private shared-memory column right after iteration z's barrier (the
// column node z just emptied) and complete before iteration z + 1's barrier:
// they fly across node z's collision and stores and hold no registers.
// In-place order: node z + 2's inputs lie in planes z + 1 .. z + 3, rewritten
// only by their own nodes after barriers z + 1 .. z + 3, and the copies have
// landed (wait_group 0) before barrier z + 1; crossing inputs come from the
// last sweep's face buffer as in k_swap1. The same schedule for push (node
// z + 2's own column staged; LBMGPU_S1_PUSH_ASYNC=1) measured slower than
// k_swap1's register-held push (C1 fp64 0.82 -> 0.75, fp32 0.53 -> 0.49).
// ---------------------------------------------------------------------------
// the address s1_in reads input I from
template <bool PUSH, bool CM, int I, class T>
__device__ __forceinline__ const T* s1_src(const S1Tab<T>& F, const T* hprev, const S1Frame& q,
                                           uint32_t s, uint32_t bounce) {
  constexpr int X = cx(I), Y = cy(I), Z = cz(I), J = opp(I);
  const bool local = s1_local<J, -X, -Y, -Z>(q, bounce);
  if (!local && s1_cross<CM, J, -X, -Y, -Z>(q)) return hprev + s1_in_slot<I>(q);
  return (PUSH || local) ? F.pl[J] + s : F.sh[I] + s;
}
// LBM_S1_PA_SPLIT (pull): a node's copies leave in two groups. EARLY: the
// five c_z = +1 inputs (plane z - 1 of the node: rewritten by the node below
// one iteration earlier, so they must land before that iteration's barrier);
// LATE: the other 14 (the node's own plane and the one above, rewritten in
// the node's own iteration or later), which may stay in flight one iteration
// longer (wait_group 1 at the top of the loop). Measured slower (C1 fp64 0.74
// -> 0.64, C4 0.62 -> 0.56; fp32 unchanged), so off: one group, wait_group 0.
#ifndef LBM_S1_PA_SPLIT
#define LBM_S1_PA_SPLIT 0
#endif
template <bool PUSH>
__host__ __device__ constexpr bool s1_pa_early(int i) {
  return PUSH || !LBM_S1_PA_SPLIT || cz(i) == 1;
}
template <bool PUSH, bool CM, bool EARLY, int I, class T>
__device__ __forceinline__ void s1_issue_one(const S1Tab<T>& F, const T* hprev, const S1Frame& q,
                                             uint32_t s, uint32_t bounce, T* col) {
  if constexpr (s1_pa_early<PUSH>(I) == EARLY)
    cp_async<(int)sizeof(T)>(col + I * kFbThreads, s1_src<PUSH, CM, I>(F, hprev, q, s, bounce));
}
template <bool PUSH, bool CM, bool EARLY, class T, int... Is>
__device__ __forceinline__ void s1_issue(const S1Tab<T>& F, const T* hprev, const S1Frame& q,
                                         uint32_t s, uint32_t bounce, T* col,
                                         std::integer_sequence<int, Is...>) {
  if constexpr (s1_pa_early<PUSH>(0) == EARLY) cp_async<(int)sizeof(T)>(col, F.pl[0] + s);
  (s1_issue_one<PUSH, CM, EARLY, Is + 1>(F, hprev, q, s, bounce, col), ...);
}
template <class T>
constexpr size_t kS1PaBytes = 2 * 19 * kFbThreads * sizeof(T);
// resident blocks per SM: fp64 as k_swap1 (2), fp32 4 (C1 pull 0.51 -> 0.56,
// C4 0.48 -> 0.50 against 3; the face-buffer geometry keeps k_swap1's waves)
#ifndef LBM_S1_PA_BLOCKS32
#define LBM_S1_PA_BLOCKS32 4
#endif
// warp-uniform inner fast path of k_swap1_pa (per precision)
// (C1 fp64 pull 0.69 -> 0.74, C4 0.60 -> 0.62; fp32 0.51 -> 0.50: off)
#ifndef LBM_S1_PA_FAST32
#define LBM_S1_PA_FAST32 0
#endif
#ifndef LBM_S1_PA_FAST64
#define LBM_S1_PA_FAST64 1
#endif
// y-face classes (a tile's two edge rows specialised as well): four code
// paths per block measured far slower (C1 fp64 0.74 -> 0.36, fp32 0.51 ->
// 0.38: the warps of a block then run different instruction streams), off
#ifndef LBM_S1_PA_YFACE
#define LBM_S1_PA_YFACE 0
#endif
template <class T>
struct S1PaFast {
  static constexpr bool value = sizeof(T) == 8 ? LBM_S1_PA_FAST64 != 0 : LBM_S1_PA_FAST32 != 0;
};
template <class T>
struct S1PaBlocks {
  static constexpr int value = sizeof(T) == 8 ? LBM_S1_BLOCKS : LBM_S1_PA_BLOCKS32;
};

template <class T, bool PUSH>
__global__ void __launch_bounds__(kFbThreads, S1PaBlocks<T>::value)
    k_swap1_pa(const __grid_constant__ S1Tab<T> F, Lat L, Trt<T> op, FbGeo G, T* __restrict__ hcur,
               const T* __restrict__ hprev) {
  extern __shared__ __align__(16) unsigned char s1pa_smem[];
  T* stg = reinterpret_cast<T*>(s1pa_smem);
  const int ntile = G.tiles_x * G.tiles_y;
  const int tile = (int)blockIdx.x % ntile, ch = (int)blockIdx.x / ntile;
  const FbBlock b = fb_block(L, G, tile % G.tiles_x, tile / G.tiles_x, ch);
  const int tx = threadIdx.x % kFbX, ty = threadIdx.x / kFbX;
  const bool act = tx < b.txv && ty < b.tyv;
  const int x = b.x0 + tx, y = b.y0 + ty;
  const uint32_t sxy = (uint32_t)L.sxy;
  const uint32_t s0 = (uint32_t)x + (uint32_t)L.sx * (uint32_t)y;
  const auto seq = std::make_integer_sequence<int, 18>{};
  constexpr bool CM = S1Cfg<T, PUSH>::kCrossMask;
  S1Frame qf;
  qf.fxl = tx == 0, qf.fxh = tx == b.txv - 1, qf.fyl = ty == 0, qf.fyh = ty == b.tyv - 1;
  qf.dxl = x == 0, qf.dxh = x == L.nx - 1, qf.dyl = y == 0, qf.dyh = y == L.ny - 1;
  qf.tx = tx, qf.ty = ty, qf.zc = G.zc;
  qf.base = (uint32_t)b.base;
  qf.rx = (uint32_t)G.region;
  qf.ry = (uint32_t)((long long)G.tiles_x * G.region);
  qf.rz = (uint32_t)((long long)G.tiles_x * G.tiles_y * G.region);
  qf.hy = (uint32_t)G.hy, qf.hx = (uint32_t)G.hx, qf.hz = (uint32_t)G.hz;
  qf.iz = qf.base + qf.hz + (uint32_t)(ty * kFbX + tx);
  const uint32_t leave_xy = s1_axis_mask(qf.dxl, qf.dxh, kMxm, kMxp) | s1_axis_mask(qf.dyl, qf.dyh, kMym, kMyp);
  const uint32_t box_xy = s1_axis_mask(qf.fxl, qf.fxh, kMxm, kMxp) | s1_axis_mask(qf.fyl, qf.fyh, kMym, kMyp);
  auto at_plane = [&](S1Frame& q, int z) {
    q.pz = z - b.zb;
    q.fzl = z == b.zb, q.fzh = z == b.ze - 1;
    q.dzl = z == 0, q.dzh = z == L.nz - 1;
    q.iy = q.base + q.hy + (uint32_t)(q.pz * 10 * kFbX + tx);
    q.ix = q.base + q.hx + (uint32_t)(q.pz * 10 * kFbY + ty);
    if (CM) q.box = box_xy | s1_axis_mask(q.fzl, q.fzh, kMzm, kMzp);
  };
  // node z's fluid flag and local-link mask
  auto cell = [&](int z, uint32_t& bm) {
    bm = 0;
    if (!act || z >= b.ze) return false;
    const bool l = fb_cell(L, x, y, z, bm);
    if (LBM_S1_LOCALMASK) bm |= leave_xy | s1_axis_mask(z == 0, z == L.nz - 1, kMzm, kMzp);
    return l;
  };
  auto col = [&](int z) { return stg + ((z - b.zb) & 1) * 19 * kFbThreads + threadIdx.x; };
  // Warp-uniform inner case (LBM_S1_PA_FAST): the warp's row is not on a y
  // face of the box, the plane not on a z face and no lane has a local link,
  // so only the x-crossing directions of the warp's end lanes use the face
  // buffers. The same templates with the y / z flags and the link mask as
  // constants: the per-direction tests and slot arithmetic fold away.
  constexpr bool kFast = S1PaFast<T>::value;
  constexpr bool kSplit = !PUSH && LBM_S1_PA_SPLIT != 0;
  const bool row_inner = ty > 0 && ty < b.tyv - 1;  // uniform over a warp (kFbX % 32 == 0)
  // class of the warp's node at plane z: 0 generic, 1 inner, 2 / 3 the box's
  // low / high y face (LBM_S1_PA_YFACE: the two edge rows of a tile otherwise
  // run the generic path and the block's per-plane barrier waits for them)
  const int row_class = row_inner ? 1 : (!LBM_S1_PA_YFACE || b.tyv < 2 ? 0 : (ty == 0 ? 2 : 3));
  auto inner = [&](int z, bool l, uint32_t bm) {
    if (!kFast) return 0;
    const bool ok = __all_sync(0xffffffffu, l && bm == 0u && z > b.zb && z < b.ze - 1) != 0;
    return ok ? row_class : 0;
  };
  auto inner_frame = [&](int z, auto yl, auto yh) {
    S1Frame qi = qf;
    at_plane(qi, z);
    qi.fyl = decltype(yl)::value, qi.fyh = decltype(yh)::value;
    qi.fzl = qi.fzh = false;
    return qi;
  };
  auto issue_class = [&](int z, auto yl, auto yh) {
    const S1Frame qi = inner_frame(z, yl, yh);
    s1_issue<PUSH, false, true>(F, hprev, qi, s0 + (uint32_t)z * sxy, 0u, col(z), seq);
    if (kSplit) cp_commit();
    s1_issue<PUSH, false, false>(F, hprev, qi, s0 + (uint32_t)z * sxy, 0u, col(z), seq);
  };
  auto write_class = [&](int z, const T(&v)[19], auto yl, auto yh) {
    const S1Frame qi = inner_frame(z, yl, yh);
    s1_write<PUSH, false>(F, hcur, G, qi, s0 + (uint32_t)z * sxy, 0u, v, seq);
  };
  using No = std::false_type;
  using Yes = std::true_type;
  auto issue = [&](int z, bool l, uint32_t bm, int fast) {
    if (fast == 1) {
      issue_class(z, No{}, No{});
    } else if (fast == 2) {
      issue_class(z, Yes{}, No{});
    } else if (fast == 3) {
      issue_class(z, No{}, Yes{});
    } else if (l) {
      at_plane(qf, z);
      s1_issue<PUSH, CM, true>(F, hprev, qf, s0 + (uint32_t)z * sxy, bm, col(z), seq);
      if (kSplit) cp_commit();
      s1_issue<PUSH, CM, false>(F, hprev, qf, s0 + (uint32_t)z * sxy, bm, col(z), seq);
    } else if (kSplit) {
      cp_commit();
    }
    cp_commit();
  };
  uint32_t bf, bg;
  bool lf = cell(b.zb, bf), lg = cell(b.zb + 1, bg);
  int ff = inner(b.zb, lf, bf), fg = inner(b.zb + 1, lg, bg);
  issue(b.zb, lf, bf, ff);
  issue(b.zb + 1, lg, bg, fg);
  for (int z = b.zb; z < b.ze; ++z) {
    // node z has all its inputs and node z + 1 its plane-z ones before barrier
    // z; split: node z + 1's late group may still be in flight
    if (kSplit)
      cp_wait1();
    else
      cp_wait0();
    __syncthreads();
    T f[19];
    if (lf) {
      const T* c = col(z);
#pragma unroll
      for (int i = 0; i < 19; ++i) f[i] = c[i * kFbThreads];
    }
    uint32_t bh;
    const bool lh = cell(z + 2, bh);
    const int fh = inner(z + 2, lh, bh);
    issue(z + 2, lh, bh, fh);  // into the column node z just emptied
    if (ff) {
      collide(op, f);
      if (ff == 1)
        write_class(z, f, No{}, No{});
      else if (ff == 2)
        write_class(z, f, Yes{}, No{});
      else
        write_class(z, f, No{}, Yes{});
    } else if (lf) {
      collide(op, f);
      at_plane(qf, z);
      s1_write<PUSH, CM>(F, hcur, G, qf, s0 + (uint32_t)z * sxy, bf, f, seq);
    }
    bf = bg, lf = lg, ff = fg;
    bg = bh, lg = lh, fg = fh;
  }
}

// ---------------------------------------------------------------------------
// SWAP push in one sweep on AoS records. The same face buffers as the SoA
// kernel: a block never writes a record outside its box, so its box planes
// can be staged in shared memory whole and leave whole — each record row of
// a plane (txv records, contiguous) arrives as one bulk copy (TMA) and, once
// final, leaves as one (head / tail elements by the lanes: the bytes around
// a row belong to other blocks). A 5-plane ring, one row per warp:
//   iteration z: node z + 1 reads its record (plane z + 1) into registers;
//   block barrier; plane z - 2 (last written in iteration z - 1) leaves and
//   its slot is refilled with plane z + 3; node z collides and writes its
//   outputs into the staged records of planes z - 1 .. z + 1 (or a face
//   buffer, or its own slot on a local link).
// ---------------------------------------------------------------------------
template <class T>
struct S1Aos {
  static constexpr int NS = 5;
  static constexpr int ROWF = kFbX * 19 + 32 / (int)sizeof(T);  // a row + 16-byte phase slack
  static constexpr int BUF = kFbY * ROWF;
  static constexpr size_t kBytes = (size_t)NS * BUF * sizeof(T);
  static constexpr int kBlocks = sizeof(T) == 8 ? 1 : 2;
};
static_assert(S1Aos<double>::kBytes <= 227 * 1024 - 1024, "fp64 AoS swap ring too large");
static_assert(2 * (S1Aos<float>::kBytes + 1024) <= 228 * 1024, "fp32 AoS swap ring: two blocks");

// one warp: n elements shared -> global, s and g congruent mod 16 bytes
template <class T>
__device__ __forceinline__ void s1_copy_out(T* g, const T* s, int n, int lane) {
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

template <bool CM, int I, class T>
__device__ __forceinline__ void s1a_in(const T* rec, const T* hprev, const S1Frame& q,
                                       uint32_t bounce, T (&v)[19]) {
  constexpr int X = cx(I), Y = cy(I), Z = cz(I), J = opp(I);
  const bool local = s1_local<J, -X, -Y, -Z>(q, bounce);
  if (!local && s1_cross<CM, J, -X, -Y, -Z>(q))
    v[I] = hprev[s1_in_slot<I>(q)];
  else
    v[I] = rec[J];
}
// nb(K): the staged record X + c_K (in the box)
template <bool CM, int K, class T, class Nb>
__device__ __forceinline__ void s1a_out(T* rec, Nb nb, T* hcur, const S1Frame& q, uint32_t bounce,
                                        const T (&v)[19]) {
  constexpr int X = cx(K), Y = cy(K), Z = cz(K);
  const bool local = s1_local<K, X, Y, Z>(q, bounce);
  const bool cross = !local && s1_cross<CM, K, X, Y, Z>(q);
  if (cross)
    hcur[s1_out_slot<K>(q)] = v[K];
  else if (local)
    rec[K] = v[K];
  else
    nb(K)[opp(K)] = v[K];
}
template <bool CM, class T, int... Is>
__device__ __forceinline__ void s1a_read(const T* rec, const T* hprev, const S1Frame& q,
                                         uint32_t bounce, T (&v)[19],
                                         std::integer_sequence<int, Is...>) {
  v[0] = rec[0];
  (s1a_in<CM, Is + 1>(rec, hprev, q, bounce, v), ...);
}
template <bool CM, class T, class Nb, int... Ks>
__device__ __forceinline__ void s1a_write(T* rec, Nb nb, T* hcur, const S1Frame& q,
                                          uint32_t bounce, const T (&v)[19],
                                          std::integer_sequence<int, Ks...>) {
  rec[0] = v[0];
  (s1a_out<CM, Ks + 1>(rec, nb, hcur, q, bounce, v), ...);
}

// pull on AoS: input I of X is slot I of the staged record X - c_I (src(I)),
// or its own slot opp I on a local link; outputs stay in its own record (and
// go to the face buffer as well when they cross)
template <bool CM, int SEL, int I, class T, class Src>
__device__ __forceinline__ void s1a_in_pull(const T* rec, Src src, const T* hprev,
                                            const S1Frame& q, uint32_t bounce, T (&v)[19]) {
  if constexpr ((SEL == 1) == s1_early(I)) {
    constexpr int X = cx(I), Y = cy(I), Z = cz(I), J = opp(I);
    const bool local = s1_local<J, -X, -Y, -Z>(q, bounce);
    if (local)
      v[I] = rec[J];
    else if (s1_cross<CM, J, -X, -Y, -Z>(q))
      v[I] = hprev[s1_in_slot<I>(q)];
    else
      v[I] = src(I)[I];
  }
}
template <bool CM, int SEL, class T, class Src, int... Is>
__device__ __forceinline__ void s1a_read_pull(const T* rec, Src src, const T* hprev,
                                              const S1Frame& q, uint32_t bounce, T (&v)[19],
                                              std::integer_sequence<int, Is...>) {
  if (SEL == 2) v[0] = rec[0];
  (s1a_in_pull<CM, SEL, Is + 1>(rec, src, hprev, q, bounce, v), ...);
}
template <bool CM, int K, class T>
__device__ __forceinline__ void s1a_out_pull(T* rec, T* hcur, const S1Frame& q, uint32_t bounce,
                                             const T (&v)[19]) {
  constexpr int X = cx(K), Y = cy(K), Z = cz(K);
  rec[K] = v[K];
  if (!s1_local<K, X, Y, Z>(q, bounce) && s1_cross<CM, K, X, Y, Z>(q))
    hcur[s1_out_slot<K>(q)] = v[K];
}
template <bool CM, class T, int... Ks>
__device__ __forceinline__ void s1a_write_pull(T* rec, T* hcur, const S1Frame& q, uint32_t bounce,
                                               const T (&v)[19], std::integer_sequence<int, Ks...>) {
  rec[0] = v[0];
  (s1a_out_pull<CM, Ks + 1>(rec, hcur, q, bounce, v), ...);
}

template <class T, bool PUSH>
__global__ void __launch_bounds__(kFbThreads, S1Aos<T>::kBlocks)
    k_swap1_aos(T* __restrict__ fp, Lat L, Trt<T> op, FbGeo G, T* __restrict__ hcur,
                const T* __restrict__ hprev) {
  using C = S1Aos<T>;
  constexpr int NS = C::NS, ROWF = C::ROWF, BUF = C::BUF;
  constexpr bool CM = sizeof(T) == 8;
  extern __shared__ __align__(16) unsigned char s1a_smem[];
  T* sm = reinterpret_cast<T*>(s1a_smem);
  __shared__ __align__(8) uint64_t full[NS];
  const int ntile = G.tiles_x * G.tiles_y;
  const int tile = (int)blockIdx.x % ntile, ch = (int)blockIdx.x / ntile;
  const FbBlock b = fb_block(L, G, tile % G.tiles_x, tile / G.tiles_x, ch);
  const int tx = threadIdx.x % kFbX, ty = threadIdx.x / kFbX, lane = tx;
  if (threadIdx.x == 0) {
    for (int k = 0; k < NS; ++k) mbar_init(&full[k], (uint32_t)b.tyv);
    mbar_fence_init();
  }
  __syncthreads();
  auto slot = [&](int p) { return (p - b.zb) % NS; };
  auto par = [&](int p) { return (uint32_t)((p - b.zb) / NS) & 1u; };
  // element offset of record (x0, y, p) and its 16-byte phase in elements
  auto rowg = [&](int y, int p) {
    return ((long long)L.sx * ((long long)y + (long long)L.sy * p) + b.x0) * 19;
  };
  auto phase = [&](long long g) { return (int)(g & (long long)(16 / sizeof(T) - 1)); };
  // row r of plane p (lane 0 of warp r): one bulk copy of the row's 16-byte
  // superset (the over-read lands in the row's slack)
  auto load = [&](int p, int r) {
    const long long g = rowg(b.y0 + r, p);
    const uintptr_t lo = reinterpret_cast<uintptr_t>(fp + g) & ~(uintptr_t)15;
    const uintptr_t hi = (reinterpret_cast<uintptr_t>(fp + g + (long long)b.txv * 19) + 15) & ~(uintptr_t)15;
    mbar_arrive_tx(&full[slot(p)], (uint32_t)(hi - lo));
    bulk_g2s(sm + slot(p) * BUF + r * ROWF, reinterpret_cast<const void*>(lo), (uint32_t)(hi - lo),
             &full[slot(p)]);
  };
  const bool rowv = ty < b.tyv;
  if (rowv && lane == 0)
    for (int p = b.zb; p < min(b.ze, b.zb + NS); ++p) load(p, ty);
  auto store = [&](int p) {
    if (!rowv) return;
    const long long g = rowg(b.y0 + ty, p);
    s1_copy_out(fp + g, sm + slot(p) * BUF + ty * ROWF + phase(g), b.txv * 19, lane);
  };
  // staged record (tx + dx, ty + dy) of the plane in ring slot sl (the row's
  // phase from its 32-bit cell index: records are 19 elements, 16 / sizeof(T)
  // elements per phase)
  const uint32_t sxy32 = (uint32_t)L.sxy, sx32 = (uint32_t)L.sx;
  auto rowoff = [&](int sl, int p, int dy) -> int {
    const uint32_t c = (uint32_t)(b.y0 + ty + dy) * sx32 + (uint32_t)p * sxy32 + (uint32_t)b.x0;
    const int ph = (int)((c * 19u) & (uint32_t)(16 / sizeof(T) - 1));
    return sl * BUF + (ty + dy) * ROWF + ph + tx * 19;
  };
  auto srec = [&](int p, int dx, int dy) -> T* {
    return sm + rowoff(slot(p), p, dy) + dx * 19;
  };

  const bool act = tx < b.txv && rowv;
  const int x = b.x0 + tx, y = b.y0 + ty;
  const auto seq = std::make_integer_sequence<int, 18>{};
  S1Frame qf;
  qf.fxl = tx == 0, qf.fxh = tx == b.txv - 1, qf.fyl = ty == 0, qf.fyh = ty == b.tyv - 1;
  qf.dxl = x == 0, qf.dxh = x == L.nx - 1, qf.dyl = y == 0, qf.dyh = y == L.ny - 1;
  qf.tx = tx, qf.ty = ty, qf.zc = G.zc;
  qf.base = (uint32_t)b.base;
  qf.rx = (uint32_t)G.region;
  qf.ry = (uint32_t)((long long)G.tiles_x * G.region);
  qf.rz = (uint32_t)((long long)G.tiles_x * G.tiles_y * G.region);
  qf.hy = (uint32_t)G.hy, qf.hx = (uint32_t)G.hx, qf.hz = (uint32_t)G.hz;
  qf.iz = qf.base + qf.hz + (uint32_t)(ty * kFbX + tx);
  const uint32_t leave_xy = s1_axis_mask(qf.dxl, qf.dxh, kMxm, kMxp) | s1_axis_mask(qf.dyl, qf.dyh, kMym, kMyp);
  const uint32_t box_xy = s1_axis_mask(qf.fxl, qf.fxh, kMxm, kMxp) | s1_axis_mask(qf.fyl, qf.fyh, kMym, kMyp);
  auto at_plane = [&](S1Frame& q, int z) {
    q.pz = z - b.zb;
    q.fzl = z == b.zb, q.fzh = z == b.ze - 1;
    q.dzl = z == 0, q.dzh = z == L.nz - 1;
    q.iy = q.base + q.hy + (uint32_t)(q.pz * 10 * kFbX + tx);
    q.ix = q.base + q.hx + (uint32_t)(q.pz * 10 * kFbY + ty);
    if (CM) q.box = box_xy | s1_axis_mask(q.fzl, q.fzh, kMzm, kMzp);
  };
  if constexpr (!PUSH) {
    // Pull: node z reads the staged records of planes z - 1 .. z + 1 and
    // rewrites only its own; the five inputs of node z + 1 from plane z
    // (c_z = +1) are read before node z's stores (iteration z), the others in
    // node z + 1's own iteration. Plane z - 1 is final once iteration z - 1
    // wrote it: it leaves after iteration z's barrier.
    T f[19];
    uint32_t bf = 0, bg = 0;
    bool lf = false, lg = false;
    if (rowv) mbar_wait(&full[slot(b.zb)], par(b.zb));
    if (act) {
      lf = fb_cell(L, x, y, b.zb, bf);
      if (LBM_S1_LOCALMASK) bf |= leave_xy | s1_axis_mask(b.zb == 0, b.zb == L.nz - 1, kMzm, kMzp);
      at_plane(qf, b.zb);
      auto src = [&](int i) -> const T* { return srec(b.zb - cz(i), -cx(i), -cy(i)); };
      if (lf) s1a_read_pull<CM, 1>(srec(b.zb, 0, 0), src, hprev, qf, bf, f, seq);
    }
    for (int z = b.zb; z < b.ze; ++z) {
      if (z + 1 < b.ze && rowv) mbar_wait(&full[slot(z + 1)], par(z + 1));
      if (lf) {
        at_plane(qf, z);
        auto src = [&](int i) -> const T* { return srec(z - cz(i), -cx(i), -cy(i)); };
        s1a_read_pull<CM, 2>(srec(z, 0, 0), src, hprev, qf, bf, f, seq);
      }
      T g[19];
      lg = false;
      if (act && z + 1 < b.ze) {
        lg = fb_cell(L, x, y, z + 1, bg);
        if (LBM_S1_LOCALMASK) bg |= leave_xy | s1_axis_mask(z + 1 == 0, z + 1 == L.nz - 1, kMzm, kMzp);
        at_plane(qf, z + 1);
        auto src = [&](int i) -> const T* { return srec(z + 1 - cz(i), -cx(i), -cy(i)); };
        if (lg) s1a_read_pull<CM, 1>(srec(z + 1, 0, 0), src, hprev, qf, bg, g, seq);
      }
      fence_async_smem();
      __syncthreads();
      if (z - 1 >= b.zb) {
        store(z - 1);
        if (lane == 0 && rowv && z - 1 + NS < b.ze) {
          bulk_wait_read();
          load(z - 1 + NS, ty);
        }
      }
      if (lf) {
        collide(op, f);
        at_plane(qf, z);
        s1a_write_pull<CM>(srec(z, 0, 0), hcur, qf, bf, f, seq);
      }
#pragma unroll
      for (int i = 1; i < 19; ++i)
        if (s1_early(i)) f[i] = g[i];
      bf = bg;
      lf = lg;
    }
    fence_async_smem();
    __syncthreads();
    store(b.ze - 1);
    bulk_wait_all();
    return;
  }
  T f[19], g[19];
  uint32_t bf = 0, bg = 0;
  bool lf = false, lg = false;
  if (rowv) mbar_wait(&full[slot(b.zb)], par(b.zb));
  if (act) {
    lf = fb_cell(L, x, y, b.zb, bf);
    if (LBM_S1_LOCALMASK) bf |= leave_xy | s1_axis_mask(b.zb == 0, b.zb == L.nz - 1, kMzm, kMzp);
    at_plane(qf, b.zb);
    if (lf) s1a_read<CM>(srec(b.zb, 0, 0), hprev, qf, bf, f, seq);
  }
  int sz = 0;  // ring slot of plane z
  for (int z = b.zb; z < b.ze; ++z) {
    lg = false;
    if (z + 1 < b.ze) {
      const int s1 = sz == NS - 1 ? 0 : sz + 1;
      if (rowv) mbar_wait(&full[s1], par(z + 1));
      if (act) {
        lg = fb_cell(L, x, y, z + 1, bg);
        if (LBM_S1_LOCALMASK) bg |= leave_xy | s1_axis_mask(z + 1 == 0, z + 1 == L.nz - 1, kMzm, kMzp);
        at_plane(qf, z + 1);
        if (lg) s1a_read<CM>(sm + rowoff(s1, z + 1, 0), hprev, qf, bg, g, seq);
      }
    }
    // one barrier per plane: node z + 1's record is in registers before node
    // z writes into it, and iteration z - 1's writes (the last into plane
    // z - 2) are done, so plane z - 2 leaves now
    fence_async_smem();
    __syncthreads();
    if (z - 2 >= b.zb) {
      store(z - 2);
      if (lane == 0 && rowv && z - 2 + NS < b.ze) {
        bulk_wait_read();  // the slot's store has read it
        load(z - 2 + NS, ty);
      }
    }
    if (lf) {
      collide(op, f);
      at_plane(qf, z);
      if constexpr (sizeof(T) == 4) {
        // the nine (plane, row) offsets the node's outputs land in, once per
        // node (fp32: C1 0.45 -> 0.46; fp64 measured better recomputing them)
        const int s0r = sz == 0 ? NS - 1 : sz - 1, s2r = sz == NS - 1 ? 0 : sz + 1;
        int ro[3][3];
#pragma unroll
        for (int dz = 0; dz < 3; ++dz)
#pragma unroll
          for (int dy = 0; dy < 3; ++dy) {
            if ((dz == 0 && z == b.zb) || (dz == 2 && z + 1 >= b.ze)) continue;  // never used
            ro[dz][dy] = rowoff(dz == 0 ? s0r : (dz == 1 ? sz : s2r), z - 1 + dz, dy - 1);
          }
        auto nb = [&](int k) -> T* { return sm + ro[1 + cz(k)][1 + cy(k)] + cx(k) * 19; };
        s1a_write<CM>(sm + ro[1][1], nb, hcur, qf, bf, f, seq);
      } else {
        auto nb = [&](int k) -> T* { return srec(z + cz(k), cx(k), cy(k)); };
        s1a_write<CM>(srec(z, 0, 0), nb, hcur, qf, bf, f, seq);
      }
    }
#pragma unroll
    for (int i = 0; i < 19; ++i) f[i] = g[i];
    bf = bg;
    lf = lg;
    sz = sz == NS - 1 ? 0 : sz + 1;
  }
  fence_async_smem();
  __syncthreads();
  if (b.ze - 2 >= b.zb) store(b.ze - 2);
  store(b.ze - 1);
  bulk_wait_all();
}

// face buffer <-> field: every crossing input slot of every node.
// fill: h = the input the sweep would read in place (push (opp i, X); pull
// (i, X - c_i)); flush (push only): (opp i, X) = h.
template <class T, bool PUSH, bool FILL, bool AOS>
__global__ void __launch_bounds__(kFbThreads)
    k_swap1_faces(Fld<T, AOS> F, Lat L, FbGeo G, T* __restrict__ h) {
  const int ntile = G.tiles_x * G.tiles_y;
  const int tile = (int)blockIdx.x % ntile, ch = (int)blockIdx.x / ntile;
  const FbBlock b = fb_block(L, G, tile % G.tiles_x, tile / G.tiles_x, ch);
  const int tx = threadIdx.x % kFbX, ty = threadIdx.x / kFbX;
  if (tx >= b.txv || ty >= b.tyv) return;
  const int x = b.x0 + tx, y = b.y0 + ty;
  for (int z = b.zb; z < b.ze; ++z) {
    uint32_t bounce = 0;
    if (!fb_cell(L, x, y, z, bounce)) continue;
    const uint32_t s = (uint32_t)x + (uint32_t)L.sx * ((uint32_t)y + (uint32_t)L.sy * (uint32_t)z);
#define S1_FACE(I)                                                                       \
  {                                                                                      \
    constexpr int J = opp(I);                                                            \
    const int sx = x - cx(I), sy = y - cy(I), sz = z - cz(I);                            \
    const bool local = ((bounce >> J) & 1u) || !fb_inside(L, sx, sy, sz);                \
    if (!local && !fb_in_block(b, sx, sy, sz)) {                                         \
      T* hp = h + fb_slot<I>(G, b, x, y, z, sx, sy, sz);                                 \
      T* fp = PUSH ? F.at(J, s)                                                          \
                   : F.at_off(I, s, -cx(I) - cy(I) * L.sx - cz(I) * (int)L.sxy);         \
      if (FILL) *hp = *fp; else *fp = *hp;                                               \
    }                                                                                    \
  }
    S1_FACE(1) S1_FACE(2) S1_FACE(3) S1_FACE(4) S1_FACE(5) S1_FACE(6) S1_FACE(7) S1_FACE(8)
    S1_FACE(9) S1_FACE(10) S1_FACE(11) S1_FACE(12) S1_FACE(13) S1_FACE(14) S1_FACE(15)
    S1_FACE(16) S1_FACE(17) S1_FACE(18)
#undef S1_FACE
  }
}

}  // namespace

// SoA through k_swap1_pa (LBMGPU_S1_PULL_ASYNC / LBMGPU_S1_PUSH_ASYNC = 1 / 0).
// Default: pull in both precisions; push in fp32 only (four blocks per SM:
// C1 0.52 -> 0.54, C4 0.47 -> 0.49; fp64 push stays register-held, 0.81
// against 0.74 staged)
static bool s1_async(bool push, Prec p) {
  static const int on[2] = {[] {
                              const char* e = std::getenv("LBMGPU_S1_PULL_ASYNC");
                              return e ? (e[0] == '1' ? 1 : 0) : 1;
                            }(),
                            [] {
                              const char* e = std::getenv("LBMGPU_S1_PUSH_ASYNC");
                              return e ? (e[0] == '1' ? 1 : 0) : -1;
                            }()};
  const int v = on[push ? 1 : 0];
  return v < 0 ? p != Prec::f64 : v != 0;
}
// resident blocks per SM of the kernel that will run (the z chunks of the
// face-buffer geometry are sized for its waves): the staged pull runs four
// fp32 blocks per SM where k_swap1 runs three (chunks for three: C1 fp32 pull
// 0.51, for four: 0.55)
static int s1_blocks(const DField& f, bool push) {
  if (!f.aos && s1_async(push, f.prec)) return f.prec == Prec::f64 ? LBM_S1_BLOCKS : LBM_S1_PA_BLOCKS32;
  return s1_blocks(f);
}
// SoA, full-grid direct lattice without halo or ghost planes
bool swap1_ok(const DField& f, const Lat& L, bool push) {
  if (f.aos) {
    // AoS push and pull in one sweep (staged box planes): C1 fp64 0.39 ->
    // 0.52, fp32 0.33 -> 0.46-0.47, C4 0.34 -> 0.46 / 0.32 -> 0.40-0.41
    // against the two-pass windows; LBMGPU_SWAP_SINGLE_AOS=0 restores those
    const char* a = std::getenv("LBMGPU_SWAP_SINGLE_AOS");
    if (a && a[0] == '0') return false;
    if (L.ox || L.oy || L.oz || L.zghost || L.znowrap || L.sx != L.nx || L.sy != L.ny) return false;
    if (L.cell_begin != 0 || (unsigned long long)L.ncells != (unsigned long long)L.nx * L.ny * L.nz)
      return false;
    const FbGeo G = fb_geo(L, s1_blocks(f, push));
    return (long long)G.tiles_x * G.tiles_y * G.nchunks * G.region < (1LL << 32);
  }
  // default: SWAP push in one sweep (C1 fp64 0.81 / fp32 0.53, C4 0.68 / 0.47
  // vs the two passes' 0.51 / 0.49, 0.50 / 0.47); pull in one sweep through
  // the cp.async-staged k_swap1_pa (C1 fp64 0.70 / fp32 0.51, C4 0.61 / 0.48
  // vs the two passes' 0.51 / 0.49, 0.50 / 0.47; k_swap1's register-held pull,
  // LBMGPU_S1_PULL_ASYNC=0, is one sweep only in fp64 with whole 32-wide x
  // tiles: C1 0.58). LBMGPU_SWAP_SINGLE=1 / 0 forces it on / off for both.
  const char* e = std::getenv("LBMGPU_SWAP_SINGLE");
  const bool on = e ? e[0] == '1'
                    : (push || s1_async(false, f.prec) || (f.prec == Prec::f64 && L.nx % kFbX == 0));
  if (!on) return false;
  if (L.ox || L.oy || L.oz || L.zghost || L.znowrap || L.sx != L.nx || L.sy != L.ny) return false;
  if (L.cell_begin != 0 || (unsigned long long)L.ncells != (unsigned long long)L.nx * L.ny * L.nz)
    return false;
  // face-buffer slots are 32-bit element offsets
  const FbGeo G = fb_geo(L, s1_blocks(f, push));
  return (long long)G.tiles_x * G.tiles_y * G.nchunks * G.region < (1LL << 32);
}

size_t swap1_face_elems(const DField& f, const Lat& L, bool push) {
  const FbGeo G = fb_geo(L, s1_blocks(f, push));
  return (size_t)G.tiles_x * G.tiles_y * G.nchunks * (size_t)G.region;
}

template <class T>
static S1Tab<T> s1_tab(const DField& f, const Lat& L, bool push) {
  S1Tab<T> t;
  T* p = static_cast<T*>(f.p);
  for (int i = 0; i < 19; ++i) t.pl[i] = p + (long long)i * f.stride;
  for (int i = 0; i < 19; ++i) {
    const long long off = cx(i) + (long long)cy(i) * L.sx + (long long)cz(i) * L.sxy;
    t.sh[i] = push ? t.pl[opp(i)] + off : t.pl[i] - off;
  }
  t.sh[0] = t.pl[0];
  return t;
}

template <class T, bool PUSH>
static void launch_swap1_aos_t(cudaStream_t st, const DField& f, const Lat& L, const TrtHost& op,
                               const FbGeo& G, T* hcur, const T* hprev) {
  static int set_dev = -1;  // the attribute is per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (set_dev != dev) {
    cudaFuncSetAttribute(k_swap1_aos<T, PUSH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)S1Aos<T>::kBytes);
    set_dev = dev;
  }
  const unsigned grid = (unsigned)(G.tiles_x * G.tiles_y * G.nchunks);
  k_swap1_aos<T, PUSH><<<grid, kFbThreads, S1Aos<T>::kBytes, st>>>(static_cast<T*>(f.p), L, cast_op<T>(op),
                                                            G, hcur, hprev);
}

template <class T, bool PUSH>
static void launch_swap1_pa(cudaStream_t st, const DField& f, const Lat& L, const TrtHost& op,
                            const FbGeo& G, T* hcur, const T* hprev) {
  static int set_dev = -1;  // the attribute is per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (set_dev != dev) {
    cudaFuncSetAttribute(k_swap1_pa<T, PUSH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kS1PaBytes<T>);
    set_dev = dev;
  }
  const unsigned grid = (unsigned)(G.tiles_x * G.tiles_y * G.nchunks);
  k_swap1_pa<T, PUSH><<<grid, kFbThreads, kS1PaBytes<T>, st>>>(s1_tab<T>(f, L, PUSH), L, cast_op<T>(op),
                                                                G, hcur, hprev);
}

void launch_swap1(cudaStream_t st, const DField& f, const Lat& L, const TrtHost& op, bool push,
                  void* hcur, const void* hprev) {
  const FbGeo G = fb_geo(L, s1_blocks(f, push));
  const unsigned grid = (unsigned)(G.tiles_x * G.tiles_y * G.nchunks);
  if (f.aos) {
    if (f.prec == Prec::f64) {
      if (push) launch_swap1_aos_t<double, true>(st, f, L, op, G, (double*)hcur, (const double*)hprev);
      else launch_swap1_aos_t<double, false>(st, f, L, op, G, (double*)hcur, (const double*)hprev);
    } else {
      if (push) launch_swap1_aos_t<float, true>(st, f, L, op, G, (float*)hcur, (const float*)hprev);
      else launch_swap1_aos_t<float, false>(st, f, L, op, G, (float*)hcur, (const float*)hprev);
    }
    return;
  }
  if (s1_async(push, f.prec)) {
    if (f.prec == Prec::f64) {
      if (push) launch_swap1_pa<double, true>(st, f, L, op, G, (double*)hcur, (const double*)hprev);
      else launch_swap1_pa<double, false>(st, f, L, op, G, (double*)hcur, (const double*)hprev);
    } else {
      if (push) launch_swap1_pa<float, true>(st, f, L, op, G, (float*)hcur, (const float*)hprev);
      else launch_swap1_pa<float, false>(st, f, L, op, G, (float*)hcur, (const float*)hprev);
    }
    return;
  }
  if (f.prec == Prec::f64) {
    if (push)
      k_swap1<double, true><<<grid, kFbThreads, 0, st>>>(s1_tab<double>(f, L, true), L, cast_op<double>(op), G,
                                                        (double*)hcur, (const double*)hprev);
    else
      k_swap1<double, false><<<grid, kFbThreads, 0, st>>>(s1_tab<double>(f, L, false), L, cast_op<double>(op), G,
                                                         (double*)hcur, (const double*)hprev);
  } else {
    if (push)
      k_swap1<float, true><<<grid, kFbThreads, 0, st>>>(s1_tab<float>(f, L, true), L, cast_op<float>(op), G,
                                                       (float*)hcur, (const float*)hprev);
    else
      k_swap1<float, false><<<grid, kFbThreads, 0, st>>>(s1_tab<float>(f, L, false), L, cast_op<float>(op), G,
                                                        (float*)hcur, (const float*)hprev);
  }
}

void launch_swap1_faces(cudaStream_t st, const DField& f, const Lat& L, bool push, bool fill,
                        void* h) {
  const FbGeo G = fb_geo(L, s1_blocks(f, push));
  const unsigned grid = (unsigned)(G.tiles_x * G.tiles_y * G.nchunks);
#define S1_F(T, P, FL)                                                                          \
  do {                                                                                          \
    if (f.aos) k_swap1_faces<T, P, FL, true><<<grid, kFbThreads, 0, st>>>(fld<T, true>(f), L, G, (T*)h); \
    else k_swap1_faces<T, P, FL, false><<<grid, kFbThreads, 0, st>>>(fld<T, false>(f), L, G, (T*)h); \
  } while (0)
  if (f.prec == Prec::f64) {
    if (push && fill) S1_F(double, true, true);
    if (push && !fill) S1_F(double, true, false);
    if (!push && fill) S1_F(double, false, true);
  } else {
    if (push && fill) S1_F(float, true, true);
    if (push && !fill) S1_F(float, true, false);
    if (!push && fill) S1_F(float, false, true);
  }
#undef S1_F
}

}  // namespace lbmgpu
