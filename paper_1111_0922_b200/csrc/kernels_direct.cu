// sm_100a kernels for direct (full-grid) addressing: one thread per lattice
// cell, threads x-contiguous so every direction plane (SoA) is read and written
// as coalesced, 256-byte aligned warp rows (the +-1 x shift of a neighbour
// access costs one extra L2 sector per warp, never an extra DRAM byte).
//
// Each kernel restates one reference sweep (cited per kernel); the collision
// is dev::collide (p/src/collision.cpp:95-139, bit-exact).
#include "dispatch.h"
#include "launch.h"

namespace lbmgpu {
using namespace dev;

namespace {

template <class T>
Trt<T> cast_op(const TrtHost& h) {
  Trt<T> o;
  o.lambda_e = (T)h.lambda_e;
  o.le_half = (T)h.le_half;
  o.lo_half = (T)h.lo_half;
  o.w0 = (T)h.w0;
  for (int p = 0; p < 9; ++p) {
    o.w2[p] = (T)h.w2[p];
    o.f3w[p] = (T)h.f3w[p];
  }
  return o;
}

inline unsigned grid_for(uint64_t n) { return (unsigned)((n + kBlock - 1) / kBlock); }

// ---------------------------------------------------------------------------
// Local collision sweep. Covers
//   TS collide_sweep A -> B            (p/src/scheme_ts.cpp:59-80)
//   OS/OSNT precollide, in place        (p/src/scheme_os.cpp:79-102)
//   AA even sweep: write opposite slots (p/src/scheme_aap.cpp:114-131)
//   SWAP collide from opposed slots     (p/src/scheme_swap.cpp:187-190, 228-231)
// ---------------------------------------------------------------------------
template <class T, bool AOS, bool RD_OPP, bool WR_OPP>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value) k_local(Fld<T, AOS> src, Fld<T, AOS> dst, Lat L,
                                                  Trt<T> op) {
  const uint32_t cell = L.cell_begin + blockIdx.x * kBlock + threadIdx.x;
  if (cell >= L.ncells) return;
  const Ctx c = make_ctx(L, cell);
  if (!c.fluid) return;
  T f[19];
#pragma unroll
  for (int i = 0; i < 19; ++i) f[i] = ld(src.at(RD_OPP ? opp(i) : i, c.s));
  collide(op, f);
#pragma unroll
  for (int i = 0; i < 19; ++i) st<false>(dst.at(WR_OPP ? opp(i) : i, c.s), f[i]);
}

// TS stream_sweep: pull B -> A with bounce B[opp i][cell] (p/src/scheme_ts.cpp:82-112)
template <bool BB, class T, bool AOS>
__device__ __forceinline__ void ts_stream_body(const Fld<T, AOS>& a, const Fld<T, AOS>& b,
                                               const Ctx& c) {
  T v[19];
  v[0] = ld(b.at(0, c.s));
#pragma unroll
  for (int i = 1; i < 19; ++i) {
    const int j = opp(i);
    v[i] = ld((BB && c.bb(j)) ? b.at(j, c.s) : b.at(i, c.nb(j)));
  }
#pragma unroll
  for (int i = 0; i < 19; ++i) st<false>(a.at(i, c.s), v[i]);
}
template <class T, bool AOS>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value) k_ts_stream(Fld<T, AOS> a, Fld<T, AOS> b, Lat L) {
  const uint32_t cell = L.cell_begin + blockIdx.x * kBlock + threadIdx.x;
  if (cell >= L.ncells) return;
  const Ctx c = make_ctx(L, cell);
  if (!c.fluid) return;
  if (warp_interior(c))
    ts_stream_body<false>(a, b, c);
  else
    ts_stream_body<true>(a, b, c);
}

// OS pull (p/src/scheme_os.cpp:141-174) and OSNT pull with streaming stores
// (p/src/scheme_osnt.cpp:131-173, 175-217: 1S = one store loop per direction,
// 2S = rest then one per opposing pair; st.global.cs replaces _mm_stream_si64).
template <bool BB, bool NT, bool TWO_S, class T, bool AOS>
__device__ __forceinline__ void os_pull_body(const Fld<T, AOS>& a, const Fld<T, AOS>& b,
                                             const Ctx& c, const Trt<T>& op) {
  T f[19];
  f[0] = ld(a.at(0, c.s));
#pragma unroll
  for (int i = 1; i < 19; ++i) {
    const int j = opp(i);
    f[i] = ld((BB && c.bb(j)) ? a.at(j, c.s) : a.at(i, c.nb(j)));
  }
  collide(op, f);
  if (!TWO_S) {
#pragma unroll
    for (int i = 0; i < 19; ++i) st<NT>(b.at(i, c.s), f[i]);
  } else {
    st<NT>(b.at(0, c.s), f[0]);
#pragma unroll
    for (int p = 0; p < 9; ++p) {
      st<NT>(b.at(pair_i(p), c.s), f[pair_i(p)]);
      st<NT>(b.at(pair_j(p), c.s), f[pair_j(p)]);
    }
  }
}
template <class T, bool AOS, bool NT, bool TWO_S>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value) k_os_pull(Fld<T, AOS> a, Fld<T, AOS> b, Lat L,
                                                    Trt<T> op) {
  const uint32_t cell = L.cell_begin + blockIdx.x * kBlock + threadIdx.x;
  if (cell >= L.ncells) return;
  const Ctx c = make_ctx(L, cell);
  if (!c.fluid) return;
  if (warp_interior(c))
    os_pull_body<false, NT, TWO_S>(a, b, c, op);
  else
    os_pull_body<true, NT, TWO_S>(a, b, c, op);
}

// OS push (p/src/scheme_os.cpp:104-139)
template <bool BB, class T, bool AOS>
__device__ __forceinline__ void os_push_body(const Fld<T, AOS>& a, const Fld<T, AOS>& b,
                                             const Ctx& c, const Trt<T>& op) {
  T f[19];
#pragma unroll
  for (int i = 0; i < 19; ++i) f[i] = ld(a.at(i, c.s));
  collide(op, f);
  st<false>(b.at(0, c.s), f[0]);
#pragma unroll
  for (int i = 1; i < 19; ++i)
    st<false>((BB && c.bb(i)) ? b.at(opp(i), c.s) : b.at_off(i, c.s, c.off(i)), f[i]);
}
template <class T, bool AOS>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value) k_os_push(Fld<T, AOS> a, Fld<T, AOS> b, Lat L,
                                                    Trt<T> op) {
  const uint32_t cell = L.cell_begin + blockIdx.x * kBlock + threadIdx.x;
  if (cell >= L.ncells) return;
  const Ctx c = make_ctx(L, cell);
  if (!c.fluid) return;
  if (warp_interior(c))
    os_push_body<false>(a, b, c, op);
  else
    os_push_body<true>(a, b, c, op);
}

// AA pattern odd sweep (p/src/scheme_aap.cpp:133-173): gather
// f[opp i][x - c_i] (bounce: f[i][x]), collide, scatter f[j][x + c_j]
// (bounce: f[opp j][x]). Every slot is read and rewritten by one thread.
template <bool BB, class T, bool AOS>
__device__ __forceinline__ void aa_odd_body(const Fld<T, AOS>& F, const Ctx& c,
                                            const Trt<T>& op) {
  T f[19];
  f[0] = ld(F.at(0, c.s));
#pragma unroll
  for (int i = 1; i < 19; ++i) {
    const int j = opp(i);
    f[i] = ld((BB && c.bb(j)) ? F.at(i, c.s) : F.at(j, c.nb(j)));
  }
  collide(op, f);
  st<false>(F.at(0, c.s), f[0]);
#pragma unroll
  for (int j = 1; j < 19; ++j)
    st<false>((BB && c.bb(j)) ? F.at(opp(j), c.s) : F.at_off(j, c.s, c.off(j)), f[j]);
}
template <class T, bool AOS>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value) k_aa_odd(Fld<T, AOS> F, Lat L, Trt<T> op) {
  const uint32_t cell = L.cell_begin + blockIdx.x * kBlock + threadIdx.x;
  if (cell >= L.ncells) return;
  const Ctx c = make_ctx(L, cell);
  if (!c.fluid) return;
  if (warp_interior(c))
    aa_odd_body<false>(F, c, op);
  else
    aa_odd_body<true>(F, c, op);
}

// Esoteric twist sweep (p/src/scheme_et.cpp:191-239). For pair (i, j):
// tmp_i = F[b_i][X], tmp_j = F[b_(db?i:j)][X + c_i]; collide;
// F[b_(ub?j:i)][X] = tmp_j, F[b_j][X + c_i] = tmp_i. Wall axes carry a halo
// plane, solid cells act as mailboxes, so X + c_i is always a storage slot.
template <bool BB, class T, bool AOS>
__device__ __forceinline__ void et_body(const Fld<T, AOS>& F, const Ctx& c, const Trt<T>& op,
                                        const EtBase& B) {
  T f[19];
  f[0] = ld(F.at(0, c.s));
#pragma unroll
  for (int p = 0; p < 9; ++p) {
    const int i = pair_i(p), j = pair_j(p);
    f[i] = ld(F.at(B.b[i], c.s));
    f[j] = ld(F.at((BB && c.bb(i)) ? B.b[i] : B.b[j], c.nb(i)));
  }
  collide(op, f);
  st<false>(F.at(0, c.s), f[0]);
#pragma unroll
  for (int p = 0; p < 9; ++p) {
    const int i = pair_i(p), j = pair_j(p);
    st<false>(F.at((BB && c.bb(j)) ? B.b[j] : B.b[i], c.s), f[j]);
    st<false>(F.at_off(B.b[j], c.s, c.off(i)), f[i]);
  }
}
template <class T, bool AOS>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value) k_et(Fld<T, AOS> F, Lat L, Trt<T> op, EtBase B) {
  const uint32_t cell = L.cell_begin + blockIdx.x * kBlock + threadIdx.x;
  if (cell >= L.ncells) return;
  const Ctx c = make_ctx(L, cell);
  if (!c.fluid) return;
  if (warp_interior(c))
    et_body<false>(F, c, op, B);
  else
    et_body<true>(F, c, op, B);
}

// SWAP link exchange (p/src/scheme_swap.cpp:172-235, fix-ups :127-131).
// The set of swapped slot pairs {(i, X), (opp i, X + c_i)}, i in the back
// half, is identical for push and pull, pairwise disjoint, and never depends
// on the current sweep's collisions — so the reference's strictly sequential
// sweep equals "all collisions, then all swaps" (push) or "all swaps, then all
// collisions" (pull), bit for bit. mode: 0 all, 1 non-wrapped, 2 wrapped only.
template <class T, bool AOS>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value) k_swap(Fld<T, AOS> F, Lat L, int mode) {
  const uint32_t cell = L.cell_begin + blockIdx.x * kBlock + threadIdx.x;
  if (cell >= L.ncells) return;
  const Ctx c = make_ctx(L, cell);
  if (!c.fluid) return;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const int i = back_dir(k);
    if (c.bb(i)) continue;
    const bool w = c.wrapped(L, i);
    if ((mode == 1 && w) || (mode == 2 && !w)) continue;
    T* a = F.at(i, c.s);
    T* b = F.at(opp(i), c.nb(i));
    const T va = ld(a), vb = ld(b);
    st<false>(a, vb);
    st<false>(b, va);
  }
}

// swap a list of slot pairs (i, a) <-> (opp i, b): SWAP periodic-seam fix-ups
// (p/src/scheme_swap.cpp:127-131)
template <class T, bool AOS>
__global__ void k_swap_list(Fld<T, AOS> F, const long long* a, const long long* b,
                            const int8_t* dir, long long count) {
  const long long k = (long long)blockIdx.x * kBlock + threadIdx.x;
  if (k >= count) return;
  const int i = dir[k];
  T* pa = F.at(i, (uint32_t)a[k]);
  T* pb = F.at(opp(i), (uint32_t)b[k]);
  const T va = *pa, vb = *pb;
  *pa = vb;
  *pb = va;
}

template <class T, bool AOS>
__global__ void k_cg_fixup(Fld<T, AOS> F, const long long* src, const long long* dst,
                           const int8_t* dir, long long count, long long shift) {
  const long long k = (long long)blockIdx.x * kBlock + threadIdx.x;
  if (k >= count) return;
  const int i = dir[k];
  *F.at(i, (uint32_t)(dst[k] - shift)) = *F.at(i, (uint32_t)(src[k] - shift));
}


// ---------------------------------------------------------------------------
// AoS variants with shared-memory staging of the record-contiguous (local)
// side: the block's 256 records are read and/or written as one coalesced
// 16-byte-vector run. Used when storage index = cell + soff (no x/y halo).
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool cell_fluid(const Lat& L, uint32_t cell) {
  return L.linkmask ? (L.linkmask[cell] & 1u) != 0 : true;
}

template <class T, bool RD_OPP, bool WR_OPP>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value)
    k_local_aos(Fld<T, true> src, Fld<T, true> dst, Lat L, Trt<T> op, uint32_t soff) {
  __shared__ __align__(16) T sm[kBlock * 19];
  const uint32_t c0 = L.cell_begin + blockIdx.x * kBlock;
  const uint32_t nrec = min((uint32_t)kBlock, L.ncells - c0);
  aos_stage_in(sm, src.p + (size_t)(c0 + soff) * 19, nrec);
  __syncthreads();
  const uint32_t k = threadIdx.x;
  if (k < nrec && cell_fluid(L, c0 + k)) {
    T f[19];
#pragma unroll
    for (int i = 0; i < 19; ++i) f[i] = sm[k * 19 + (RD_OPP ? opp(i) : i)];
    collide(op, f);
#pragma unroll
    for (int i = 0; i < 19; ++i) sm[k * 19 + (WR_OPP ? opp(i) : i)] = f[i];
  }
  __syncthreads();
  aos_stage_out(dst.p + (size_t)(c0 + soff) * 19, sm, nrec);
}

// OS/OSNT pull, AoS: gather per field (neighbour records), staged local store
template <class T>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value)
    k_os_pull_aos(Fld<T, true> a, Fld<T, true> b, Lat L, Trt<T> op, uint32_t soff) {
  __shared__ __align__(16) T sm[kBlock * 19];
  const uint32_t c0 = L.cell_begin + blockIdx.x * kBlock;
  const uint32_t nrec = min((uint32_t)kBlock, L.ncells - c0);
  const uint32_t k = threadIdx.x;
  T f[19];
  bool live = false;
  if (k < nrec) {
    const Ctx c = make_ctx(L, c0 + k);
    live = c.fluid;
    if (live) {
      f[0] = ld(a.at(0, c.s));
#pragma unroll
      for (int i = 1; i < 19; ++i) {
        const int j = opp(i);
        f[i] = ld(c.bb(j) ? a.at(j, c.s) : a.at(i, c.nb(j)));
      }
      collide(op, f);
    }
  }
#pragma unroll
  for (int i = 0; i < 19; ++i)
    if (k < nrec) sm[k * 19 + i] = live ? f[i] : T(0);
  __syncthreads();
  aos_stage_out(b.p + (size_t)(c0 + soff) * 19, sm, nrec);
}

// OS push, AoS: staged local load, scatter per field
template <class T>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value)
    k_os_push_aos(Fld<T, true> a, Fld<T, true> b, Lat L, Trt<T> op, uint32_t soff) {
  __shared__ __align__(16) T sm[kBlock * 19];
  const uint32_t c0 = L.cell_begin + blockIdx.x * kBlock;
  const uint32_t nrec = min((uint32_t)kBlock, L.ncells - c0);
  aos_stage_in(sm, a.p + (size_t)(c0 + soff) * 19, nrec);
  __syncthreads();
  const uint32_t k = threadIdx.x;
  if (k >= nrec) return;
  const Ctx c = make_ctx(L, c0 + k);
  if (!c.fluid) return;
  T f[19];
#pragma unroll
  for (int i = 0; i < 19; ++i) f[i] = sm[k * 19 + i];
  collide(op, f);
  st<false>(b.at(0, c.s), f[0]);
#pragma unroll
  for (int i = 1; i < 19; ++i)
    st<false>(c.bb(i) ? b.at(opp(i), c.s) : b.at_off(i, c.s, c.off(i)), f[i]);
}

// TS stream, AoS: gather per field, staged local store
template <class T>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value)
    k_ts_stream_aos(Fld<T, true> a, Fld<T, true> b, Lat L, uint32_t soff) {
  __shared__ __align__(16) T sm[kBlock * 19];
  const uint32_t c0 = L.cell_begin + blockIdx.x * kBlock;
  const uint32_t nrec = min((uint32_t)kBlock, L.ncells - c0);
  const uint32_t k = threadIdx.x;
  if (k < nrec) {
    const Ctx c = make_ctx(L, c0 + k);
    if (c.fluid) {
      sm[k * 19] = ld(b.at(0, c.s));
#pragma unroll
      for (int i = 1; i < 19; ++i) {
        const int j = opp(i);
        sm[k * 19 + i] = ld(c.bb(j) ? b.at(j, c.s) : b.at(i, c.nb(j)));
      }
    } else {
#pragma unroll
      for (int i = 0; i < 19; ++i) sm[k * 19 + i] = T(0);
    }
  }
  __syncthreads();
  aos_stage_out(a.p + (size_t)(c0 + soff) * 19, sm, nrec);
}

// storage index = cell + soff for every cell (no x/y halo or padding)?
inline bool aos_contiguous(const DField& f, const dev::Lat& L, uint32_t* soff) {
  if (!f.aos || L.sx != L.nx || L.sy != L.ny || L.ox != 0 || L.oy != 0) return false;
  *soff = (uint32_t)(L.oz * L.sxy);
  return true;
}


// ---------------------------------------------------------------------------
// Ticketed tiles (used by the compressed-grid sweep): blocks take tickets in
// the reference traversal order, publish per-tile progress with st.release,
// and wait with ld.acquire only on tiles holding earlier tickets, so the
// waits cannot deadlock. Loads of data another SM rewrote during the sweep
// use ld.global.cg (L2) so they are never served from a stale L1 line.
template <class T>
__device__ __forceinline__ T ldcg(const T* p) { return __ldcg(p); }

__device__ __forceinline__ uint32_t take_ticket(unsigned long long* ticket, unsigned epoch,
                                                uint32_t ntiles, bool reverse) {
  __shared__ uint32_t s_tile;
  if (threadIdx.x == 0) {
    const unsigned long long k =
        atomicAdd(ticket, 1ull) - (unsigned long long)(epoch - 1) * ntiles;
    s_tile = reverse ? ntiles - 1 - (uint32_t)k : (uint32_t)k;
  }
  __syncthreads();
  return s_tile;
}
__device__ __forceinline__ void publish_tile(unsigned* flags, uint32_t tile, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + tile), "r"(epoch) : "memory");
  }
}
// Compressed grid, lagged pipeline (p/src/scheme_cg.cpp:118-158). Ticket tau
// (reference traversal order: reverse lex for even sweeps, forward for odd)
// runs phase A on its tile — read the 19 slots at the read origin, collide,
// park the result in an L2-resident ring slot, publish "read" — and phase B on
// the tile lag tickets behind: wait until every tile whose read slots it
// overwrites has published "read" (X + (1,1,1) + c_i even / X - (1,1,1) + c_i
// odd, all earlier tickets), then write the parked values at the write origin
// and publish "ring slot free". The only hazards in a CG sweep are
// write-after-read (every slot is read before it is overwritten), so these
// waits reproduce the sequential result bit for bit.
template <class T, bool AOS, bool EVEN>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value)
    k_cg_lag(Fld<T, AOS> F, Lat L, Trt<T> op, unsigned long long* ticket, unsigned* flagsA,
             unsigned* flagsB, unsigned epoch, uint32_t ntiles, uint32_t lag, T* ring,
             uint32_t R) {
  const uint32_t tau = take_ticket(ticket, epoch, ntiles + lag, false);
  // ---- phase A ----
  if (tau < ntiles) {
    const uint32_t a = EVEN ? ntiles - 1 - tau : tau;
    if (tau >= R) {  // the ring slot's previous tile must have been written out
      if (threadIdx.x == 0) {
        const uint32_t prev = EVEN ? ntiles - 1 - (tau - R) : tau - R;
        unsigned v;
        while (true) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flagsB + prev) : "memory");
          if (v == epoch) break;
          __nanosleep(32);
        }
      }
      __syncthreads();
    }
    const uint32_t cell = a * kBlock + threadIdx.x;
    T* slot = ring + (size_t)(tau % R) * 19 * kBlock + threadIdx.x;
    if (cell < L.ncells) {
      const Ctx c = make_ctx(L, cell);  // L.o* = read origin (1 even, 2 odd)
      if (c.fluid) {
        T f[19];
#pragma unroll
        for (int i = 0; i < 19; ++i) f[i] = ld(F.at(i, c.s));
        collide(op, f);
#pragma unroll
        for (int i = 0; i < 19; ++i) slot[i * kBlock] = f[i];
      }
    }
    publish_tile(flagsA, a, epoch);
  }
  // ---- phase B ----
  if (tau >= lag) {
    const uint32_t ub = tau - lag;
    const uint32_t b = EVEN ? ntiles - 1 - ub : ub;
    if (threadIdx.x < 38) {
      const int d = threadIdx.x >> 1;
      const int sgn = EVEN ? 1 : -1;
      const long long D = (long long)(sgn + cx(d)) + (long long)L.nx * (sgn + cy(d)) +
                          (long long)L.nx * L.ny * (sgn + cz(d));
      const long long tgt = (long long)b * kBlock + D + ((threadIdx.x & 1) ? kBlock - 1 : 0);
      if (tgt >= 0 && tgt < (long long)L.ncells) {
        const unsigned* fl = flagsA + (uint32_t)(tgt / kBlock);
        unsigned v;
        while (true) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(fl) : "memory");
          if (v == epoch) break;
          __nanosleep(32);
        }
      }
    } else if (threadIdx.x == 38) {  // the tile's own phase A (ring contents)
      unsigned v;
      while (true) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flagsA + b) : "memory");
        if (v == epoch) break;
        __nanosleep(32);
      }
    }
    __syncthreads();
    const uint32_t cell = b * kBlock + threadIdx.x;
    const T* slot = ring + (size_t)(ub % R) * 19 * kBlock + threadIdx.x;
    if (cell < L.ncells) {
      const Ctx c = make_ctx(L, cell);
      if (c.fluid) {
        T f[19];
#pragma unroll
        for (int i = 0; i < 19; ++i) f[i] = __ldcg(slot + i * kBlock);
        const uint32_t sh = 1u + (uint32_t)L.sx + (uint32_t)L.sxy;  // shift1
        const uint32_t wr = EVEN ? c.s + sh : c.s - sh;
        st<false>(F.at(0, wr), f[0]);
#pragma unroll
        for (int i = 1; i < 19; ++i) {
          const int po = cx(i) + L.sx * cy(i) + (int)L.sxy * cz(i);
          T* dst = c.bb(i) ? F.at(opp(i), wr) : F.at(i, wr + (uint32_t)po);
          st<false>(dst, f[i]);
        }
      }
    }
    publish_tile(flagsB, b, epoch);
  }
}



}  // namespace

void launch_local(cudaStream_t st, const DField& src, const DField& dst, const dev::Lat& L,
                  const TrtHost& op, bool rd_opp, bool wr_opp) {
  if (L.ncells <= L.cell_begin) return;
  uint32_t soff = 0;
  if (aos_contiguous(src, L, &soff)) {
    const unsigned g = grid_for(L.ncells - L.cell_begin);
    LBM_DISPATCH(src, {
      if constexpr (A) {
        auto a = fld<T, true>(src);
        auto b = fld<T, true>(dst);
        const auto o = cast_op<T>(op);
        if (!rd_opp && !wr_opp) k_local_aos<T, false, false><<<g, kBlock, 0, st>>>(a, b, L, o, soff);
        if (!rd_opp && wr_opp) k_local_aos<T, false, true><<<g, kBlock, 0, st>>>(a, b, L, o, soff);
        if (rd_opp && !wr_opp) k_local_aos<T, true, false><<<g, kBlock, 0, st>>>(a, b, L, o, soff);
        if (rd_opp && wr_opp) k_local_aos<T, true, true><<<g, kBlock, 0, st>>>(a, b, L, o, soff);
      }
    });
    return;
  }
  LBM_DISPATCH(src, {
    auto a = fld<T, A>(src);
    auto b = fld<T, A>(dst);
    const auto o = cast_op<T>(op);
    const unsigned g = grid_for(L.ncells - L.cell_begin);
    if (!rd_opp && !wr_opp) k_local<T, A, false, false><<<g, kBlock, 0, st>>>(a, b, L, o);
    if (!rd_opp && wr_opp) k_local<T, A, false, true><<<g, kBlock, 0, st>>>(a, b, L, o);
    if (rd_opp && !wr_opp) k_local<T, A, true, false><<<g, kBlock, 0, st>>>(a, b, L, o);
    if (rd_opp && wr_opp) k_local<T, A, true, true><<<g, kBlock, 0, st>>>(a, b, L, o);
  });
}

void launch_ts_stream(cudaStream_t st, const DField& a, const DField& b, const dev::Lat& L) {
  if (L.ncells <= L.cell_begin) return;
  uint32_t soff = 0;
  if (aos_contiguous(a, L, &soff)) {
    LBM_DISPATCH(a, {
      if constexpr (A)
        k_ts_stream_aos<T><<<grid_for(L.ncells - L.cell_begin), kBlock, 0, st>>>(
            fld<T, true>(a), fld<T, true>(b), L, soff);
    });
    return;
  }
  LBM_DISPATCH(a, {
    k_ts_stream<T, A><<<grid_for(L.ncells - L.cell_begin), kBlock, 0, st>>>(fld<T, A>(a), fld<T, A>(b), L);
  });
}

void launch_os_pull(cudaStream_t st, const DField& a, const DField& b, const dev::Lat& L,
                    const TrtHost& op, bool streaming, bool two_s) {
  if (L.ncells <= L.cell_begin) return;
  uint32_t soff = 0;
  if (aos_contiguous(a, L, &soff)) {
    // the staged store writes whole 16-byte vectors: store order (1S/2S) and
    // streaming hints are properties of the record run, not of single slots
    LBM_DISPATCH(a, {
      if constexpr (A)
        k_os_pull_aos<T><<<grid_for(L.ncells - L.cell_begin), kBlock, 0, st>>>(
            fld<T, true>(a), fld<T, true>(b), L, cast_op<T>(op), soff);
    });
    return;
  }
  LBM_DISPATCH(a, {
    auto fa = fld<T, A>(a);
    auto fb = fld<T, A>(b);
    const auto o = cast_op<T>(op);
    const unsigned g = grid_for(L.ncells - L.cell_begin);
    if (!streaming && !two_s) k_os_pull<T, A, false, false><<<g, kBlock, 0, st>>>(fa, fb, L, o);
    if (!streaming && two_s) k_os_pull<T, A, false, true><<<g, kBlock, 0, st>>>(fa, fb, L, o);
    if (streaming && !two_s) k_os_pull<T, A, true, false><<<g, kBlock, 0, st>>>(fa, fb, L, o);
    if (streaming && two_s) k_os_pull<T, A, true, true><<<g, kBlock, 0, st>>>(fa, fb, L, o);
  });
}

void launch_os_push(cudaStream_t st, const DField& a, const DField& b, const dev::Lat& L,
                    const TrtHost& op) {
  if (L.ncells <= L.cell_begin) return;
  uint32_t soff = 0;
  if (aos_contiguous(a, L, &soff)) {
    LBM_DISPATCH(a, {
      if constexpr (A)
        k_os_push_aos<T><<<grid_for(L.ncells - L.cell_begin), kBlock, 0, st>>>(
            fld<T, true>(a), fld<T, true>(b), L, cast_op<T>(op), soff);
    });
    return;
  }
  LBM_DISPATCH(a, {
    k_os_push<T, A><<<grid_for(L.ncells - L.cell_begin), kBlock, 0, st>>>(fld<T, A>(a), fld<T, A>(b), L,
                                                           cast_op<T>(op));
  });
}

void launch_aa_odd(cudaStream_t st, const DField& f, const dev::Lat& L, const TrtHost& op) {
  if (L.ncells <= L.cell_begin) return;
  LBM_DISPATCH(f, {
    k_aa_odd<T, A><<<grid_for(L.ncells - L.cell_begin), kBlock, 0, st>>>(fld<T, A>(f), L, cast_op<T>(op));
  });
}

void launch_et(cudaStream_t st, const DField& f, const dev::Lat& L, const TrtHost& op,
               const EtBase& base) {
  if (L.ncells <= L.cell_begin) return;
  LBM_DISPATCH(f, {
    k_et<T, A><<<grid_for(L.ncells - L.cell_begin), kBlock, 0, st>>>(fld<T, A>(f), L, cast_op<T>(op), base);
  });
}

void launch_swap(cudaStream_t st, const DField& f, const dev::Lat& L, int mode) {
  if (L.ncells <= L.cell_begin) return;
  LBM_DISPATCH(f, { k_swap<T, A><<<grid_for(L.ncells - L.cell_begin), kBlock, 0, st>>>(fld<T, A>(f), L, mode); });
}

uint32_t cg_lag(const dev::Lat& L) {
  const uint64_t reach = (2ull * L.nx * L.ny + 2ull * L.nx + 2 + kBlock - 1) / kBlock + 2;
  return (uint32_t)(reach + 148 * 2);
}

void launch_cg_lag(cudaStream_t st, const DField& f, const dev::Lat& L, const TrtHost& op,
                   bool even, unsigned long long* ticket, unsigned* flagsA, unsigned* flagsB,
                   unsigned epoch, void* ring, uint32_t R) {
  if (L.ncells <= L.cell_begin) return;
  const uint32_t ntiles = grid_for(L.ncells);
  const uint32_t lag = cg_lag(L);
  LBM_DISPATCH(f, {
    if (even)
      k_cg_lag<T, A, true><<<ntiles + lag, kBlock, 0, st>>>(fld<T, A>(f), L, cast_op<T>(op), ticket,
                                                            flagsA, flagsB, epoch, ntiles, lag,
                                                            static_cast<T*>(ring), R);
    else
      k_cg_lag<T, A, false><<<ntiles + lag, kBlock, 0, st>>>(fld<T, A>(f), L, cast_op<T>(op),
                                                             ticket, flagsA, flagsB, epoch, ntiles,
                                                             lag, static_cast<T*>(ring), R);
  });
}

void launch_swap_list(cudaStream_t st, const DField& f, const long long* a, const long long* b,
                      const int8_t* dir, long long count) {
  if (count <= 0) return;
  LBM_DISPATCH(f, {
    k_swap_list<T, A><<<grid_for(count), kBlock, 0, st>>>(fld<T, A>(f), a, b, dir, count);
  });
}

void launch_cg_fixup(cudaStream_t st, const DField& f, const long long* src,
                     const long long* dst, const int8_t* dir, long long count, long long shift) {
  if (count <= 0) return;
  LBM_DISPATCH(f, {
    k_cg_fixup<T, A><<<grid_for(count), kBlock, 0, st>>>(fld<T, A>(f), src, dst, dir, count,
                                                         shift);
  });
}

}  // namespace lbmgpu
