// Face buffers (shared by the single-pass SWAP and the AoS face-buffer
// kernels). A block owns an x-y tile of kFbX x kFbY cells and a chunk of z
// planes; a link whose other end lies outside the block's box (unwrapped
// coordinates) is a crossing link, and the value travelling along it lives
// in a face-buffer slot of the block holding the link's home cell R, keyed by
// (face, direction, position on the face, plane). Hy holds the links whose
// other end is in row y0 - 1 / y0 + tyv, else Hx (column x0 - 1 / x0 + txv),
// else Hz (plane zb - 1 / ze).
#pragma once

#include "lbm_device.cuh"

#include <algorithm>
#include <cstdlib>

#ifndef LBM_S1_BLOCKS_DEFAULT
#define LBM_S1_BLOCKS_DEFAULT 2
#endif

namespace lbmgpu {
namespace dev {

#ifndef LBM_FB_X
#define LBM_FB_X 32
#endif
#ifndef LBM_FB_Y
#define LBM_FB_Y 8
#endif
constexpr int kFbX = LBM_FB_X, kFbY = LBM_FB_Y, kFbThreads = kFbX * kFbY;

// direction lists of the faces (ascending): incoming from y - 1 (c_y = +1),
// from y + 1 (c_y = -1), and likewise for x and z
__host__ __device__ constexpr int face_q(int axis, int sign, int i) {
  // position of direction i among the directions with c_axis = sign
  int q = 0;
  for (int k = 1; k < i; ++k) {
    const int c = axis == 0 ? cx(k) : (axis == 1 ? cy(k) : cz(k));
    q += c == sign ? 1 : 0;
  }
  return q;
}

struct FbGeo {
  int tiles_x, tiles_y, zc, nchunks;
  long long region;  // elements of one block's face region
  long long hy, hx, hz;  // offsets of the three parts inside a region
};

struct FbBlock {
  int tix, tiy, ch;
  int x0, y0, zb, txv, tyv, ze;
  long long base;  // element offset of the block's region
};

__device__ __forceinline__ FbBlock fb_block(const Lat& L, const FbGeo& G, int tx_, int ty_, int ch) {
  FbBlock b;
  b.tix = tx_, b.tiy = ty_, b.ch = ch;
  b.x0 = tx_ * kFbX;
  b.y0 = ty_ * kFbY;
  b.zb = ch * G.zc;
  b.txv = min(kFbX, L.nx - b.x0);
  b.tyv = min(kFbY, L.ny - b.y0);
  b.ze = min(L.nz, b.zb + G.zc);
  b.base = ((long long)ch * G.tiles_y * G.tiles_x + (long long)ty_ * G.tiles_x + tx_) * G.region;
  return b;
}

// Face-buffer slot of receiver R = (x, y, z) in block b, incoming direction i
// from source (sx, sy, sz) outside the block (and inside the domain).
template <int I>
__device__ __forceinline__ long long fb_slot(const FbGeo& G, const FbBlock& b, int x, int y, int z,
                                             int sx, int sy, int sz) {
  const int pz = z - b.zb;
  if (sy < b.y0 || sy >= b.y0 + b.tyv) {
    const int side = sy < b.y0 ? 0 : 1;
    const int q = side == 0 ? face_q(1, 1, I) : face_q(1, -1, I);
    return b.base + G.hy + ((long long)(pz * 2 + side) * 5 + q) * kFbX + (x - b.x0);
  }
  if (sx < b.x0 || sx >= b.x0 + b.txv) {
    const int side = sx < b.x0 ? 0 : 1;
    const int q = side == 0 ? face_q(0, 1, I) : face_q(0, -1, I);
    return b.base + G.hx + ((long long)(pz * 2 + side) * 5 + q) * kFbY + (y - b.y0);
  }
  const int side = sz < b.zb ? 0 : 1;
  const int q = side == 0 ? face_q(2, 1, I) : face_q(2, -1, I);
  return b.base + G.hz + ((long long)(side * 5 + q) * kFbY + (y - b.y0)) * kFbX + (x - b.x0);
}

// cell (x, y, z) of the lattice: fluid, and its bounce mask
__device__ __forceinline__ bool fb_cell(const Lat& L, int x, int y, int z, uint32_t& bounce) {
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

__device__ __forceinline__ bool fb_inside(const Lat& L, int x, int y, int z) {
  return x >= 0 && x < L.nx && y >= 0 && y < L.ny && z >= 0 && z < L.nz;
}
__device__ __forceinline__ bool fb_in_block(const FbBlock& b, int x, int y, int z) {
  return x >= b.x0 && x < b.x0 + b.txv && y >= b.y0 && y < b.y0 + b.tyv && z >= b.zb && z < b.ze;
}

// the block holding cell (x, y, z), a neighbour of block b
__device__ __forceinline__ FbBlock fb_block_of(const Lat& L, const FbGeo& G, const FbBlock& b,
                                               int x, int y, int z) {
  const int dx = x < b.x0 ? -1 : (x >= b.x0 + b.txv ? 1 : 0);
  const int dy = y < b.y0 ? -1 : (y >= b.y0 + b.tyv ? 1 : 0);
  const int dz = z < b.zb ? -1 : (z >= b.ze ? 1 : 0);
  return fb_block(L, G, b.tix + dx, b.tiy + dy, b.ch + dz);
}

// blocks_per_sm: resident blocks of the kernel using the layout (the chunk
// length is chosen for its waves)
inline FbGeo fb_geo(const Lat& L, int blocks_per_sm = LBM_S1_BLOCKS_DEFAULT) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  FbGeo G{};
  G.tiles_x = (L.nx + kFbX - 1) / kFbX;
  G.tiles_y = (L.ny + kFbY - 1) / kFbY;
  const long long tiles = (long long)G.tiles_x * G.tiles_y, resident = (long long)sms * blocks_per_sm;
  // chunk length: waves of resident blocks x (chunk + 1 prologue plane),
  // 8 .. 64 planes (longer chunks: fewer chunk-face links)
  long long best = std::min(64, L.nz), cost = -1;
  for (long long zc = std::min(64, L.nz); zc >= std::min(8, L.nz); --zc) {
    const long long n = tiles * ((L.nz + zc - 1) / zc);
    const long long c = ((n + resident - 1) / resident) * (zc + 1);
    if (cost < 0 || c < cost) best = zc, cost = c;
  }
  if (const char* e = std::getenv("LBMGPU_SWAP1_ZCHUNK"))
    if (std::atoi(e) > 0) best = std::min<long long>(std::atoi(e), L.nz);
  G.zc = (int)best;
  G.nchunks = (L.nz + G.zc - 1) / G.zc;
  G.hy = 0;
  G.hx = (long long)G.zc * 10 * kFbX;
  G.hz = G.hx + (long long)G.zc * 10 * kFbY;
  G.region = G.hz + 10LL * kFbX * kFbY;
  return G;
}


}  // namespace dev
}  // namespace lbmgpu
