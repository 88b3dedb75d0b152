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

namespace lbmgpu {
using namespace dev;

namespace {

// Per-face passes with compile-time directions (as kernels_aos_fb.cu): a
// warp-uniform (y rows, z planes) or lane (x columns) branch per face of the
// block box visits the five directions crossing it; a link crossing several
// faces is taken by the first of y, x, z (the order of fb_slot). A link
// leaving the domain (bounce or periodic wrap: the fix-up list's) never
// crosses. F: the node's face flags.
struct S1Face {
  bool ylo, yhi, xlo, xhi, zlo, zhi;
};
#define S1_5(D0, D1, D2, D3, D4, OP) OP(D0) OP(D1) OP(D2) OP(D3) OP(D4)
#define S1_APPLY(M, OP) S1_APPLY_(M, OP)
#define S1_APPLY_(D0, D1, D2, D3, D4, OP) S1_5(D0, D1, D2, D3, D4, OP)
#define S1_CY_M 4, 7, 11, 12, 15
#define S1_CY_P 3, 10, 13, 14, 18
#define S1_CX_M 2, 7, 8, 9, 10
#define S1_CX_P 1, 15, 16, 17, 18
#define S1_CZ_M 6, 8, 11, 13, 16
#define S1_CZ_P 5, 9, 12, 14, 17
// the link from the node along c (dx, dy, dz) leaves the box through a y / x face
__device__ __forceinline__ bool s1_ycross(const S1Face& q, int dy) {
  return (dy < 0 && q.ylo) || (dy > 0 && q.yhi);
}
__device__ __forceinline__ bool s1_xcross(const S1Face& q, int dx) {
  return (dx < 0 && q.xlo) || (dx > 0 && q.xhi);
}
__device__ __forceinline__ bool s1_cross(const S1Face& q, int dx, int dy, int dz) {
  return s1_ycross(q, dy) || s1_xcross(q, dx) || (dz < 0 && q.zlo) || (dz > 0 && q.zhi);
}

// the 19 inputs of node (x, y, z): push (opp i, X); pull (i, X - c_i), or
// (opp i, X) on a bounce / wrap; a crossing input then comes from the face
// buffer of the last sweep
template <bool PUSH, class T>
__device__ __forceinline__ void s1_read(const Fld<T, false>& F, const T* hprev, const Lat& L,
                                        const FbGeo& G, const FbBlock& b, int x, int y, int z,
                                        uint32_t s, uint32_t bounce, const S1Face& q, T (&v)[19]) {
  v[0] = *F.at(0, s);
#pragma unroll
  for (int i = 1; i < 19; ++i) {
    const int j = opp(i);
    if (PUSH) {
      v[i] = *F.at(j, s);
    } else {
      const int off = -cx(i) - cy(i) * L.sx - cz(i) * (int)L.sxy;
      const bool loc = ((bounce >> j) & 1u) || !fb_inside(L, x - cx(i), y - cy(i), z - cz(i));
      v[i] = *(loc ? F.at(j, s) : F.at(i, s) + off);
    }
  }
  // input I crosses when its source X - c_I is in the domain, outside the box
#define S1_RD(I)                                                                        \
  if (!((bounce >> opp(I)) & 1u) && fb_inside(L, x - cx(I), y - cy(I), z - cz(I)))       \
    v[I] = hprev[fb_slot<I>(G, b, x, y, z, x - cx(I), y - cy(I), z - cz(I))];
#define S1_RD_X(I) if (!s1_ycross(q, -cy(I))) { S1_RD(I) }
#define S1_RD_Z(I) if (!s1_ycross(q, -cy(I)) && !s1_xcross(q, -cx(I))) { S1_RD(I) }
  if (q.ylo) { S1_APPLY(S1_CY_P, S1_RD) }
  if (q.yhi) { S1_APPLY(S1_CY_M, S1_RD) }
  if (q.xlo) { S1_APPLY(S1_CX_P, S1_RD_X) }
  if (q.xhi) { S1_APPLY(S1_CX_M, S1_RD_X) }
  if (q.zlo) { S1_APPLY(S1_CZ_P, S1_RD_Z) }
  if (q.zhi) { S1_APPLY(S1_CZ_M, S1_RD_Z) }
#undef S1_RD
#undef S1_RD_X
#undef S1_RD_Z
}
// the 19 outputs: push (opp k, X + c_k), or (k, X) on a bounce / wrap; pull
// (k, X); a crossing link's value goes to the receiver's face buffer instead
// (push) or as well (pull)
template <bool PUSH, class T>
__device__ __forceinline__ void s1_write(const Fld<T, false>& F, T* hcur, const Lat& L,
                                         const FbGeo& G, const FbBlock& b, int x, int y, int z,
                                         uint32_t s, uint32_t bounce, const S1Face& q,
                                         const T (&v)[19]) {
  *F.at(0, s) = v[0];
#pragma unroll
  for (int k = 1; k < 19; ++k) {
    if (!PUSH) {
      *F.at(k, s) = v[k];
    } else {
      const bool loc = ((bounce >> k) & 1u) || !fb_inside(L, x + cx(k), y + cy(k), z + cz(k));
      if (loc) {
        *F.at(k, s) = v[k];
      } else if (!s1_cross(q, cx(k), cy(k), cz(k))) {
        const int off = cx(k) + cy(k) * L.sx + cz(k) * (int)L.sxy;
        *(F.at(opp(k), s) + off) = v[k];
      }
    }
  }
#define S1_WR(K)                                                                         \
  if (!((bounce >> K) & 1u) && fb_inside(L, x + cx(K), y + cy(K), z + cz(K))) {          \
    const int rx = x + cx(K), ry = y + cy(K), rz = z + cz(K);                             \
    hcur[fb_slot<K>(G, fb_block_of(L, G, b, rx, ry, rz), rx, ry, rz, x, y, z)] = v[K];    \
  }
#define S1_WR_X(K) if (!s1_ycross(q, cy(K))) { S1_WR(K) }
#define S1_WR_Z(K) if (!s1_ycross(q, cy(K)) && !s1_xcross(q, cx(K))) { S1_WR(K) }
  if (q.ylo) { S1_APPLY(S1_CY_M, S1_WR) }
  if (q.yhi) { S1_APPLY(S1_CY_P, S1_WR) }
  if (q.xlo) { S1_APPLY(S1_CX_M, S1_WR_X) }
  if (q.xhi) { S1_APPLY(S1_CX_P, S1_WR_X) }
  if (q.zlo) { S1_APPLY(S1_CZ_M, S1_WR_Z) }
  if (q.zhi) { S1_APPLY(S1_CZ_P, S1_WR_Z) }
#undef S1_WR
#undef S1_WR_X
#undef S1_WR_Z
}

#ifndef LBM_S1_BLOCKS
#define LBM_S1_BLOCKS 2
#endif

// One sweep over a block's planes. Iteration z reads node z + 1's inputs
// (push: its own slots in plane z + 1; pull: planes z .. z + 2), then, after
// the block barrier, node z collides and writes (push: planes z - 1 .. z + 1;
// pull: plane z). Every in-block read of a slot precedes the barrier before
// which the slot is rewritten: push plane z + 1 is read before node z's
// outputs land, pull plane z is read by nodes z - 1 .. z + 1 in iterations
// <= z.
template <class T, bool PUSH>
__global__ void __launch_bounds__(kFbThreads, LBM_S1_BLOCKS)
    k_swap1(Fld<T, false> F, Lat L, Trt<T> op, FbGeo G, T* __restrict__ hcur,
            const T* __restrict__ hprev) {
  const int ntile = G.tiles_x * G.tiles_y;
  const int tile = (int)blockIdx.x % ntile, ch = (int)blockIdx.x / ntile;
  const FbBlock b = fb_block(L, G, tile % G.tiles_x, tile / G.tiles_x, ch);
  const int tx = threadIdx.x % kFbX, ty = threadIdx.x / kFbX;
  const bool act = tx < b.txv && ty < b.tyv;
  const int x = b.x0 + tx, y = b.y0 + ty;
  const uint32_t s0 = (uint32_t)x + (uint32_t)L.sx * (uint32_t)y;
  const uint32_t sxy = (uint32_t)L.sxy;
  S1Face qf{ty == 0, ty == b.tyv - 1, tx == 0, tx == b.txv - 1, false, false}, qg = qf;
  T f[19], g[19];
  uint32_t bf = 0, bg = 0;
  bool lf = false, lg = false;
  if (act) {
    lf = fb_cell(L, x, y, b.zb, bf);
    qf.zlo = true;
    qf.zhi = b.zb == b.ze - 1;
    if (lf) s1_read<PUSH>(F, hprev, L, G, b, x, y, b.zb, s0 + (uint32_t)b.zb * sxy, bf, qf, f);
  }
  for (int z = b.zb; z < b.ze; ++z) {
    lg = false;
    if (act && z + 1 < b.ze) {
      lg = fb_cell(L, x, y, z + 1, bg);
      qg.zlo = false;
      qg.zhi = z + 1 == b.ze - 1;
      if (lg) s1_read<PUSH>(F, hprev, L, G, b, x, y, z + 1, s0 + (uint32_t)(z + 1) * sxy, bg, qg, g);
    }
    __syncthreads();
    if (lf) {
      collide(op, f);
      s1_write<PUSH>(F, hcur, L, G, b, x, y, z, s0 + (uint32_t)z * sxy, bf, qf, f);
    }
#pragma unroll
    for (int i = 0; i < 19; ++i) f[i] = g[i];
    bf = bg;
    lf = lg;
    qf = qg;
  }
}

// face buffer <-> field: every crossing input slot of every node.
// fill: h = the input the sweep would read in place (push (opp i, X); pull
// (i, X - c_i)); flush (push only): (opp i, X) = h.
template <class T, bool PUSH, bool FILL>
__global__ void __launch_bounds__(kFbThreads)
    k_swap1_faces(Fld<T, false> F, Lat L, FbGeo G, T* __restrict__ h) {
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
                   : F.at(I, s) + (-cx(I) - cy(I) * L.sx - cz(I) * (int)L.sxy);          \
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

// SoA, full-grid direct lattice without halo or ghost planes
bool swap1_ok(const DField& f, const Lat& L) {
  if (f.aos) return false;
  const char* e = std::getenv("LBMGPU_SWAP_SINGLE");  // opt-in until it beats two passes
  if (!(e && e[0] == '1')) return false;
  if (L.ox || L.oy || L.oz || L.zghost || L.znowrap || L.sx != L.nx || L.sy != L.ny) return false;
  return L.cell_begin == 0 && (unsigned long long)L.ncells == (unsigned long long)L.nx * L.ny * L.nz;
}

size_t swap1_face_elems(const Lat& L) {
  const FbGeo G = fb_geo(L, LBM_S1_BLOCKS);
  return (size_t)G.tiles_x * G.tiles_y * G.nchunks * (size_t)G.region;
}

void launch_swap1(cudaStream_t st, const DField& f, const Lat& L, const TrtHost& op, bool push,
                  void* hcur, const void* hprev) {
  const FbGeo G = fb_geo(L, LBM_S1_BLOCKS);
  const unsigned grid = (unsigned)(G.tiles_x * G.tiles_y * G.nchunks);
  if (f.prec == Prec::f64) {
    if (push)
      k_swap1<double, true><<<grid, kFbThreads, 0, st>>>(fld<double, false>(f), L, cast_op<double>(op), G,
                                                        (double*)hcur, (const double*)hprev);
    else
      k_swap1<double, false><<<grid, kFbThreads, 0, st>>>(fld<double, false>(f), L, cast_op<double>(op), G,
                                                         (double*)hcur, (const double*)hprev);
  } else {
    if (push)
      k_swap1<float, true><<<grid, kFbThreads, 0, st>>>(fld<float, false>(f), L, cast_op<float>(op), G,
                                                       (float*)hcur, (const float*)hprev);
    else
      k_swap1<float, false><<<grid, kFbThreads, 0, st>>>(fld<float, false>(f), L, cast_op<float>(op), G,
                                                        (float*)hcur, (const float*)hprev);
  }
}

void launch_swap1_faces(cudaStream_t st, const DField& f, const Lat& L, bool push, bool fill,
                        void* h) {
  const FbGeo G = fb_geo(L, LBM_S1_BLOCKS);
  const unsigned grid = (unsigned)(G.tiles_x * G.tiles_y * G.nchunks);
#define S1_F(T, P, FL) k_swap1_faces<T, P, FL><<<grid, kFbThreads, 0, st>>>(fld<T, false>(f), L, G, (T*)h)
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
