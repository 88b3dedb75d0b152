// SWAP in one sweep (SoA, direct addressing): collisions and link exchanges
// of p/src/scheme_swap.cpp:172-235 fused into a single launch per time step.
//
// The reference sweeps cells in lexicographic order; cell X collides from its
// opposed slots, stores natural, then swaps (i, X) <-> (opp i, X + c_i) for
// the back half i (the neighbour is lexicographically earlier, so it already
// collided). The swapped pairs are disjoint and never depend on the sweep's
// collisions, so any order is bit-identical as long as each pair is swapped
// after both of its cells collided (push) or before either collides (pull).
//
// Here a block owns a tile of full x rows [y0, y0 + H) and marches through
// z. Pairs stay inside the tile except those reaching row y0 - 1 (tile T-1)
// and the c = (0,1,-1) pairs from the tile's last row into tile T+1's first
// row; the latter are executed by tile T+1 (it "owns" the row y + 1 side), so
// a tile only ever touches its own slots and tile T-1's. One flag word per
// tile publishes its progress (release/acquire at gpu scope):
//   push (z ascending, k_swap_push_staged): collide(z); in-tile exchanges of
//        plane z-1; cross-tile exchanges of plane z-KC once tile T-1
//        published it (publishes every KG planes).
//   pull (z descending, tiles descending, k_swap_pull_fused): exchange plane
//        z -> publish; collide(z+1) after tile T+1 published plane z+1.
// A tile waits only for one neighbour, and blocks take tiles in ticket order
// (atomic counter), so that neighbour is resident or done: no deadlock
// without a co-residency assumption. Periodic-seam pairs stay with the
// fix-up list (k_swap mode 1 semantics), exactly as the two-pass path.
//
// DRAM traffic is the compulsory 2q elements per node (ncu on C1: 5.08 GB per
// step for 5.10 GB algorithmic): the exchanges' reads and second writes hit
// L2. Speed is another matter: each tile is one serial chain of plane
// iterations (barrier, flag, L2 round trips; ~6.5-11 k cycles per 256-node
// plane measured with clock64 traces), and only ~2 tiles fit per SM, so the
// sweep runs at 0.50 (C1) / 0.36 (C4) of the fp64 roofline against 0.47 /
// 0.44 for the two streaming passes (profiles/r01_variants.md). It is
// therefore opt-in (LBMGPU_SWAP_FUSED=1); the default stays two passes.
#include "dispatch.h"
#include "launch.h"

#include <algorithm>
#include <cstdlib>

namespace lbmgpu {
using namespace dev;

namespace {

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
// wait until *p >= want (thread 0 polls; the barrier hands the acquire on)
__device__ __forceinline__ void wait_flag(const unsigned long long* p, unsigned long long want) {
  if (threadIdx.x == 0)
    while (ld_acquire(p) < want) __nanosleep(64);
  __syncthreads();
}
__device__ __forceinline__ void publish(unsigned long long* p, unsigned long long v) {
  __syncthreads();
  if (threadIdx.x == 0) st_release(p, v);
}

struct SwapTile {
  int T, ntiles, y0, rows;
  int x, r;  // this thread's column and row inside the tile
  bool active;
  unsigned long long* flag;  // flag[T] = tile T's progress
};

__device__ __forceinline__ uint32_t cell_at(const Lat& L, int x, int y, int z) {
  return (uint32_t)x + (uint32_t)L.nx * ((uint32_t)y + (uint32_t)L.ny * (uint32_t)z);
}

// Exchange every non-wrapped back-half pair whose back endpoint lies in this
// tile's plane z, except the (0,1,-1) pairs of the last row (tile T+1's), plus
// the (0,1,-1) pairs of tile T-1's last row (ours: their row y + 1 is our first).
// All loads are issued before any store (the compiler cannot prove the pairs
// disjoint, so load-store-load order would serialise ten L2 round trips).
template <class T>
__device__ __forceinline__ void swap_plane(const Fld<T, false>& F, const Lat& L,
                                           const SwapTile& t, int z) {
  if (!t.active) return;
  uint32_t sa[10], sb[10];  // storage indices of the pair's two slots
  T va[10], vb[10];
  uint32_t use = 0;
  const Ctx c = make_ctx(L, cell_at(L, t.x, t.y0 + t.r, z));
  const bool last = t.r == t.rows - 1;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const int i = back_dir(k);
    sa[k] = c.s;
    sb[k] = c.nb(i);
    if (c.fluid && !(i == 13 && last) && !c.bb(i) && !c.wrapped(L, i)) use |= 1u << k;
  }
  if (t.r == 0 && t.T > 0) {
    const Ctx p = make_ctx(L, cell_at(L, t.x, t.y0 - 1, z));
    sa[9] = p.s;
    sb[9] = p.nb(13);
    if (p.fluid && !p.bb(13) && !p.wrapped(L, 13)) use |= 1u << 9;
  }
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    const int i = k < 9 ? back_dir(k) : 13;
    if (use & (1u << k)) va[k] = __ldcg(F.at(i, sa[k])), vb[k] = __ldcg(F.at(opp(i), sb[k]));
  }
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    const int i = k < 9 ? back_dir(k) : 13;
    if (use & (1u << k)) *F.at(i, sa[k]) = vb[k], *F.at(opp(i), sb[k]) = va[k];
  }
}

// Push, staged. Plane z + NS - 1 streams into shared memory (bulk copies of
// the tile's 19 direction rows on an mbarrier when rows are 16-byte
// multiples, else per-element cp.async) while the block collides plane z.
// Pairs inside the tile are exchanged one plane later: a node keeps its
// back-half post-collision values in registers until then, so the exchange
// reads only the partner slot (L2) and the back-half natural stores it would
// overwrite are never issued; the block barrier that ends each iteration
// orders them. Pairs reaching tile T-1 (the first row's c_y = -1 links and
// the (0,1,-1) pairs of T-1's last row) are exchanged KC planes later from
// L2, both slots, after tile T-1 published that plane. A tile publishes its
// collided planes every KG planes (one release per KG iterations), and KC >
// KG, so in lock step the flag a tile needs was published an iteration ago:
// no tile waits and no skew accumulates along the chain of tiles. Everything
// that does not depend on z is hoisted (storage index = s0 + z nx ny; partner
// offsets c_x + c_y nx + c_z nx ny, since exchanged pairs never wrap).
constexpr int kSwapKG = 4;  // planes per publish
constexpr int kSwapKC = 6;  // lag of the cross-tile exchanges (> kSwapKG)
template <class T, int NS, bool BULK>
__global__ void __launch_bounds__(512, 1)
    k_swap_push_staged(Fld<T, false> F, Lat L, Trt<T> op, unsigned long long* sync, int H,
                       int ntiles, unsigned long long epoch) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t full[NS];
  __shared__ int s_tile;
  const uint32_t tid = threadIdx.x;
  if (tid == 0) {
    s_tile = (int)(atomicAdd(&sync[0], 1ull) % (unsigned long long)ntiles);
    for (int k = 0; k < NS; ++k) mbar_init(&full[k], BULK ? 1u : blockDim.x);
    mbar_fence_init();
  }
  __syncthreads();
  const int T_ = s_tile;
  const int nx = L.nx, ny = L.ny, nz = L.nz;
  const int y0 = T_ * H, rows = min(H, ny - y0);
  const uint32_t P = (uint32_t)(nx * rows);           // tile nodes per plane
  const uint32_t PS = (uint32_t)(nx * H + 3) & ~3u;   // stage row pitch (16 B multiple)
  T* stg = reinterpret_cast<T*>(smraw);               // [NS][19][PS]
  const int x = (int)(tid % (uint32_t)nx), r = (int)(tid / (uint32_t)nx), y = y0 + r;
  const bool active = tid < P;
  const bool last = r == rows - 1;
  const bool xrow = r == 0 && T_ > 0;  // first row of a tile with a predecessor
  const uint32_t plane = (uint32_t)nx * (uint32_t)ny;
  const uint32_t s0 = (uint32_t)x + (uint32_t)nx * (uint32_t)y;
  const uint32_t* lm = L.linkmask;
  unsigned long long* flag = sync + 1;
  const unsigned long long base = epoch * (unsigned long long)(nz + 1);
  const uint32_t nwarps = blockDim.x >> 5;

  // exchanged pairs that x, y and the tile split allow (bit k: back_dir(k)):
  // in-tile (register-held) and cross-tile (first row, c_y = -1)
  uint32_t use_in = 0, use_x = 0, zmask = 0;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const int i = back_dir(k);
    const int xn = x + cx(i), yn = y + cy(i);
    const bool ok = xn >= 0 && xn < nx && yn >= 0 && yn < ny && !(i == 13 && last);
    if (ok && xrow && cy(i) < 0) use_x |= 1u << k;
    else if (ok) use_in |= 1u << k;
    if (cz(i) < 0) zmask |= 1u << k;
  }
  auto boff = [&](int i) -> int { return cx(i) + cy(i) * nx + cz(i) * (int)plane; };
  // pairs of the node at storage index s on plane z, masked by the link mask
  auto pairs = [&](uint32_t set, uint32_t s, int z, bool& fl) -> uint32_t {
    uint32_t u = set & (z == 0 ? ~zmask : 0x1ffu);
    fl = true;
    if (lm) {
      const uint32_t w = lm[s];
      fl = w & 1u;
      if (!fl) return 0;
#pragma unroll
      for (int k = 0; k < 9; ++k)
        if ((w >> back_dir(k)) & 1u) u &= ~(1u << k);
    }
    return u;
  };

  auto issue = [&](int z) {
    if (z >= nz) return;
    const int sg = z % NS;
    T* d = stg + (size_t)sg * 19 * PS;
    if (BULK) {
      // direction row i is issued by lane i / nwarps of warp i % nwarps
      const uint32_t w = tid >> 5, lane = tid & 31;
      const uint32_t i = lane * nwarps + w;
      if (tid == 0) mbar_arrive_tx(&full[sg], 19u * P * (uint32_t)sizeof(T));
      if (i < 19) {
        fence_async_smem();
        const uint32_t c0 = (uint32_t)nx * (uint32_t)y0 + (uint32_t)z * plane;
        bulk_g2s(d + (size_t)i * PS, F.at((int)i, c0), P * (uint32_t)sizeof(T), &full[sg]);
      }
    } else {
      if (active) {
        const uint32_t s = s0 + (uint32_t)z * plane;
#pragma unroll
        for (int i = 0; i < 19; ++i) cp_async<sizeof(T)>(d + (size_t)i * PS + tid, F.at(i, s));
      }
      cp_async_mbar_arrive(&full[sg]);
    }
  };

#pragma unroll 1
  for (int j = 0; j < NS - 1; ++j) issue(j);

  T bk[9];
  uint32_t use_prev = 0;
  unsigned long long fv = 0;
  const int zend = nz - 1 + kSwapKC;  // last iteration: the last cross-tile exchange
#pragma unroll 1
  for (int z = 0; z <= zend; ++z) {
    issue(z + NS - 1);
    const uint32_t s = s0 + (uint32_t)z * plane;  // this plane's node
    const uint32_t sp = s - plane;                // plane z-1's node
    // plane zc's cross-tile exchanges first (tile T-1 published plane zc before
    // the last barrier): their L2 round trip overlaps the other tile's work
    // on this SM, and their registers are free again before the collision
    const int zc = z - kSwapKC;
    if (zc >= 0 && active && xrow) {
      const uint32_t sc = s0 + (uint32_t)zc * plane;
      bool fc;
      const uint32_t ux = pairs(use_x, sc, zc, fc);
      T va[5], vv[5];
      uint32_t pa9 = sc - (uint32_t)nx;  // tile T-1's last-row node on plane zc
      bool x9 = false;
      if (zc >= 1) x9 = lm ? ((lm[pa9] & 1u) && !((lm[pa9] >> 13) & 1u)) : true;
#pragma unroll
      for (int k = 0, q = 0; k < 9; ++k) {
        const int i = back_dir(k);
        if (cy(i) >= 0) continue;
        if (ux & (1u << k)) va[q] = __ldcg(F.at(i, sc)), vv[q] = __ldcg(F.at(opp(i), sc + (uint32_t)boff(i)));
        ++q;
      }
      T a9 = T(0), b9 = T(0);
      if (x9) a9 = __ldcg(F.at(13, pa9)), b9 = __ldcg(F.at(12, sc - plane));
#pragma unroll
      for (int k = 0, q = 0; k < 9; ++k) {
        const int i = back_dir(k);
        if (cy(i) >= 0) continue;
        if (ux & (1u << k)) F.at(i, sc)[0] = vv[q], F.at(opp(i), sc + (uint32_t)boff(i))[0] = va[q];
        ++q;
      }
      if (x9) F.at(13, pa9)[0] = b9, F.at(12, sc - plane)[0] = a9;
    }
    // in-tile partner slots of plane z-1 (collided before the last barrier)
    T vb[9];
    if (z >= 1 && z <= nz && active) {
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const int i = back_dir(k);
        if (use_prev & (1u << k)) vb[k] = __ldcg(F.at(opp(i), sp + (uint32_t)boff(i)));
      }
    }
    // collide plane z from its stage
    T fb[9];
    uint32_t use_z = 0;
    bool fl = false;
    if (z < nz) {
      const int sg = z % NS;
      mbar_wait(&full[sg], (uint32_t)(z / NS) & 1u);
      if (active) {
        use_z = pairs(use_in, s, z, fl);
        if (fl) {
          const T* src = stg + (size_t)sg * 19 * PS + tid;
          T f[19];
#pragma unroll
          for (int i = 0; i < 19; ++i) f[i] = src[(size_t)opp(i) * PS];
          collide(op, f);
          F.at(0, s)[0] = f[0];
#pragma unroll
          for (int k = 0; k < 9; ++k) {
            const int i = back_dir(k);
            F.at(opp(i), s)[0] = f[opp(i)];
            fb[k] = f[i];
          }
        }
      }
    }
    // plane z-1's in-tile exchanges
    if (z >= 1 && z <= nz && active) {
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const int i = back_dir(k);
        if (use_prev & (1u << k)) {
          F.at(i, sp)[0] = vb[k];
          F.at(opp(i), sp + (uint32_t)boff(i))[0] = bk[k];
        }
      }
    }
    // plane z's back-half slots that no register-held exchange rewrites
    if (fl) {
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        if (!(use_z & (1u << k))) F.at(back_dir(k), s)[0] = fb[k];
        bk[k] = fb[k];
      }
    }
    use_prev = use_z;
    // next iteration's cross-tile plane must be published by tile T-1
    const int zn = z + 1 - kSwapKC;
    if (tid == 0 && T_ > 0 && zn >= 0 && zn < nz) {
      const unsigned long long want = base + (unsigned long long)zn + 1;
      while (fv < want) fv = ld_acquire(&flag[T_ - 1]);
    }
    __syncthreads();
    if (tid == 0 && z < nz && ((z + 1) % kSwapKG == 0 || z == nz - 1))
      st_release(&flag[T_], base + (unsigned long long)z + 1);
  }
}

// Pull, one sweep: z descending, tiles descending (tile T waits for T+1).
template <class T>
__global__ void __launch_bounds__(512, 1)
    k_swap_pull_fused(Fld<T, false> F, Lat L, Trt<T> op, unsigned long long* sync, int H, int ntiles,
                 unsigned long long epoch) {
  __shared__ int s_tile;
  if (threadIdx.x == 0) s_tile = (int)(atomicAdd(&sync[0], 1ull) % (unsigned long long)ntiles);
  __syncthreads();
  SwapTile t;
  t.ntiles = ntiles;
  t.T = ntiles - 1 - s_tile;
  t.y0 = t.T * H;
  t.rows = min(H, L.ny - t.y0);
  t.x = (int)threadIdx.x % L.nx;
  t.r = (int)threadIdx.x / L.nx;
  t.active = (int)threadIdx.x < L.nx * t.rows;
  t.flag = sync + 1;
  const int nz = L.nz;
  const unsigned long long base = epoch * (unsigned long long)(nz + 1);

  {
    for (int z = nz - 1; z >= -1; --z) {
      if (z >= 0) {
        swap_plane(F, L, t, z);
        publish(&t.flag[t.T], base + (unsigned long long)(nz - z));
      }
      const int zc = z + 1;
      if (zc <= nz - 1) {
        if (t.T < ntiles - 1) wait_flag(&t.flag[t.T + 1], base + (unsigned long long)(nz - zc));
        if (t.active) {
          const Ctx c = make_ctx(L, cell_at(L, t.x, t.y0 + t.r, zc));
          if (c.fluid) {
            T f[19];
#pragma unroll
            for (int i = 0; i < 19; ++i) f[i] = __ldcg(F.at(opp(i), c.s));
            collide(op, f);
#pragma unroll
            for (int i = 0; i < 19; ++i) F.at(i, c.s)[0] = f[i];
          }
        }
      }
    }
  }
}

}  // namespace

int swap_fused_rows(const dev::Lat& L) {
  if (L.nx > 512 || L.zghost || L.ox || L.oy || L.oz || L.sx != L.nx || L.sy != L.ny) return 0;
  return std::max(1, std::min(L.ny, 256 / L.nx));
}

template <class T>
void launch_push_staged(cudaStream_t st, const DField& f, const dev::Lat& L, const TrtHost& op,
                        unsigned long long* sync, int H, int ntiles, unsigned long long epoch,
                        unsigned threads) {
  const size_t smem = (size_t)2 * 19 * (size_t)((L.nx * H + 3) & ~3) * sizeof(T);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<ntiles, threads, smem, st>>>(fld<T, false>(f), L, cast_op<T>(op), sync, H, ntiles,
                                        epoch);
  };
  if ((L.nx * sizeof(T)) % 16 == 0)
    go(k_swap_push_staged<T, 2, true>);
  else
    go(k_swap_push_staged<T, 2, false>);
}

bool launch_swap_fused(cudaStream_t st, const DField& f, const dev::Lat& L, const TrtHost& op,
                       bool push, unsigned long long* sync, unsigned long long epoch) {
  const int H = swap_fused_rows(L);
  if (f.aos || H == 0 || L.cell_begin != 0) return false;
  const int ntiles = (L.ny + H - 1) / H;
  const unsigned threads = (unsigned)((L.nx * H + 31) / 32 * 32);
  if (f.prec == Prec::f64) {
    if (push)
      launch_push_staged<double>(st, f, L, op, sync, H, ntiles, epoch, threads);
    else
      k_swap_pull_fused<double><<<ntiles, threads, 0, st>>>(fld<double, false>(f), L,
                                                            cast_op<double>(op), sync, H, ntiles,
                                                            epoch);
  } else {
    if (push)
      launch_push_staged<float>(st, f, L, op, sync, H, ntiles, epoch, threads);
    else
      k_swap_pull_fused<float><<<ntiles, threads, 0, st>>>(fld<float, false>(f), L,
                                                           cast_op<float>(op), sync, H, ntiles,
                                                           epoch);
  }
  return true;
}

}  // namespace lbmgpu
