// sm_100a kernels for direct (full-grid) addressing: one thread per lattice
// cell, threads x-contiguous so every direction plane (SoA) is read and written
// as coalesced, 256-byte aligned warp rows (the +-1 x shift of a neighbour
// access costs one extra L2 sector per warp, never an extra DRAM byte).
//
// Each kernel restates one reference sweep (cited per kernel); the collision
// is dev::collide (p/src/collision.cpp:95-139, bit-exact).
#include "dispatch.h"
#include "launch.h"

#include <stdexcept>

namespace lbmgpu {
using namespace dev;

namespace {

inline unsigned grid_for(uint64_t n) { return (unsigned)((n + kBlock - 1) / kBlock); }

// shifted plane table of an SoA field (unused for AoS): n[j] = plane j +
// sign * (c_x + c_y sx + c_z sxy)(j); sign 0 gives the plain plane bases
template <class T>
SoaNb<T> soa_nb(const DField& f, const Lat& L, int sign = 1) {
  SoaNb<T> N;
  for (int j = 0; j < 19; ++j) {
    const long long off = (long long)cx(j) + (long long)cy(j) * L.sx + (long long)cz(j) * L.sxy;
    const uintptr_t b = reinterpret_cast<uintptr_t>(f.p) +
                        (uintptr_t)((long long)j * f.stride + sign * off) * sizeof(T);
    N.n[j] = reinterpret_cast<T*>(f.aos ? reinterpret_cast<uintptr_t>(f.p) : b);
  }
  return N;
}
// ET: n[p] = plane hb(pair_j(p)) shifted by c_(pair_i(p)), p = 0..8
template <class T>
SoaNb<T> et_nb(const DField& f, const Lat& L, bool sw) {
  SoaNb<T> N{};
  for (int p = 0; p < 9; ++p) {
    const int i = pair_i(p), j = pair_j(p), k = sw ? opp(j) : j;
    const long long off = (long long)cx(i) + (long long)cy(i) * L.sx + (long long)cz(i) * L.sxy;
    N.n[p] = reinterpret_cast<T*>(
        f.aos ? reinterpret_cast<uintptr_t>(f.p)
              : reinterpret_cast<uintptr_t>(f.p) +
                    (uintptr_t)((long long)k * f.stride + off) * sizeof(T));
  }
  return N;
}

// per-lane indices of a plain warp: s, and s with the x wrap of a -x / +x shift
#define LBM_PLAIN_IX(c, s, sm, sp)                                             \
  const uint32_t s = (c).s, sm = s + (uint32_t)((c).xm + 1), sp = s + (uint32_t)((c).xp - 1)

// ---------------------------------------------------------------------------
// Local collision sweep. Covers
//   TS collide_sweep A -> B            (p/src/scheme_ts.cpp:59-80)
//   OS/OSNT precollide, in place        (p/src/scheme_os.cpp:79-102)
//   AA even sweep: write opposite slots (p/src/scheme_aap.cpp:114-131)
//   SWAP collide from opposed slots     (p/src/scheme_swap.cpp:187-190, 228-231)
// ---------------------------------------------------------------------------
template <class T, bool AOS, bool RD_OPP, bool WR_OPP>
__global__ void __launch_bounds__(kBlock, SoaMinBlocks<T, AOS>::value) k_local(Fld<T, AOS> src, Fld<T, AOS> dst, Lat L,
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
// plain warp: Bm = b shifted by -c_i, A0 = a's plane bases
template <class T>
__device__ __forceinline__ void ts_stream_plain(const SoaNb<T>& A0, const SoaNb<T>& Bm, const Ctx& c) {
  LBM_PLAIN_IX(c, s, sm, sp);
  T v[19];
#pragma unroll
  for (int i = 0; i < 19; ++i) v[i] = ld(Bm.n[i] + nb_ix(-cx(i), s, sm, sp));
#pragma unroll
  for (int i = 0; i < 19; ++i) A0.n[i][s] = v[i];
}
template <class T, bool AOS>
__global__ void __launch_bounds__(kBlock, SoaMinBlocks<T, AOS>::value)
    k_ts_stream(Fld<T, AOS> a, Fld<T, AOS> b, Lat L, SoaNb<T> A0, SoaNb<T> Bm) {
  const uint32_t cell = L.cell_begin + blockIdx.x * kBlock + threadIdx.x;
  if (cell >= L.ncells) return;
  const Ctx c = make_ctx(L, cell);
  if (!c.fluid) return;
  if (!AOS && warp_plain(L, c))
    ts_stream_plain(A0, Bm, c);
  else if (warp_interior(c))
    ts_stream_body<false>(a, b, c);
  else
    ts_stream_body<true>(a, b, c);
}

// OS pull (p/src/scheme_os.cpp:141-174) and OSNT pull with streaming stores
// (p/src/scheme_osnt.cpp:131-173, 175-217: 1S = one store loop per direction,
// 2S = rest then one per opposing pair; st.global.cs replaces _mm_stream_si64).
template <bool BB, bool NT, bool TWO_S, class FA, class T>
__device__ __forceinline__ void os_pull_body(const FA& a, const FA& b, const Ctx& c,
                                             const Trt<T>& op) {
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
// plain warp: Am = a shifted by -c_i, B0 = b's plane bases
template <bool NT, bool TWO_S, class T>
__device__ __forceinline__ void os_pull_plain(const SoaNb<T>& Am, const SoaNb<T>& B0, const Ctx& c,
                                              const Trt<T>& op) {
  LBM_PLAIN_IX(c, s, sm, sp);
  T f[19];
#pragma unroll
  for (int i = 0; i < 19; ++i) f[i] = ld(Am.n[i] + nb_ix(-cx(i), s, sm, sp));
  collide(op, f);
  if (!TWO_S) {
#pragma unroll
    for (int i = 0; i < 19; ++i) st<NT>(B0.n[i] + s, f[i]);
  } else {
    st<NT>(B0.n[0] + s, f[0]);
#pragma unroll
    for (int p = 0; p < 9; ++p) {
      st<NT>(B0.n[pair_i(p)] + s, f[pair_i(p)]);
      st<NT>(B0.n[pair_j(p)] + s, f[pair_j(p)]);
    }
  }
}
// fp32 SoA OSNT (streaming stores) addresses through plane bases (FldT:
// C1 1S 0.99 -> 1.01, 2S 0.98 -> 1.01, measured)
template <class T, bool NT>
constexpr bool kOsPullTab = sizeof(T) == 4 && NT;
// fp32 SoA OSNT at 6 blocks per SM (<= 40 registers; with the deviation
// collision C1 1S 0.95 -> 1.01), the plain pull keeps 5 (1.03 vs 1.01)
template <class T, bool AOS, bool NT>
constexpr int kOsPullBlocks = (NT && sizeof(T) == 4 && !AOS) ? 6 : OsMinBlocks<T, AOS>::value;
template <class T, bool AOS, bool NT, bool TWO_S>
__global__ void __launch_bounds__(kBlock, kOsPullBlocks<T, AOS, NT>)
    k_os_pull(FldSel<T, AOS, kOsPullTab<T, NT>> a, FldSel<T, AOS, kOsPullTab<T, NT>> b, Lat L,
              Trt<T> op, SoaNb<T> Am, SoaNb<T> B0) {
  const uint32_t cell = L.cell_begin + blockIdx.x * kBlock + threadIdx.x;
  if (cell >= L.ncells) return;
  const Ctx c = make_ctx(L, cell);
  if (!c.fluid) return;
  // (the streaming-store OSNT forms keep the generic path: measured slower
  // with the table at their 5-block register budget)
  if (!AOS && !NT && warp_plain(L, c))
    os_pull_plain<NT, TWO_S>(Am, B0, c, op);
  else if (warp_interior(c))
    os_pull_body<false, NT, TWO_S>(a, b, c, op);
  else
    os_pull_body<true, NT, TWO_S>(a, b, c, op);
}

// OS push (p/src/scheme_os.cpp:104-139)
template <bool BB, class FA, class T>
__device__ __forceinline__ void os_push_body(const FA& a, const FA& b, const Ctx& c,
                                             const Trt<T>& op) {
  T f[19];
#pragma unroll
  for (int i = 0; i < 19; ++i) f[i] = ld(a.at(i, c.s));
  collide(op, f);
  st<false>(b.at(0, c.s), f[0]);
#pragma unroll
  for (int i = 1; i < 19; ++i)
    st<false>((BB && c.bb(i)) ? b.at(opp(i), c.s) : b.at_off(i, c.s, c.off(i)), f[i]);
}
// plain warp: A0 = a's plane bases, Bp = b shifted by +c_i
template <class T>
__device__ __forceinline__ void os_push_plain(const SoaNb<T>& A0, const SoaNb<T>& Bp, const Ctx& c,
                                              const Trt<T>& op) {
  LBM_PLAIN_IX(c, s, sm, sp);
  T f[19];
#pragma unroll
  for (int i = 0; i < 19; ++i) f[i] = ld(A0.n[i] + s);
  collide(op, f);
#pragma unroll
  for (int i = 0; i < 19; ++i) Bp.n[i][nb_ix(cx(i), s, sm, sp)] = f[i];
}
// fp32 SoA takes its generic-path fields with plane bases (FldT: C1 0.92 ->
// 0.99 of the roofline, measured; the kernel-wide register allocation is what
// moves)
template <class T, bool AOS>
constexpr bool kOsPushTab = sizeof(T) == 4;
template <class T, bool AOS>
__global__ void __launch_bounds__(kBlock, OsMinBlocks<T, AOS>::value)
    k_os_push(FldSel<T, AOS, kOsPushTab<T, AOS>> a, FldSel<T, AOS, kOsPushTab<T, AOS>> b, Lat L,
              Trt<T> op, SoaNb<T> A0, SoaNb<T> Bp) {
  const uint32_t cell = L.cell_begin + blockIdx.x * kBlock + threadIdx.x;
  if (cell >= L.ncells) return;
  const Ctx c = make_ctx(L, cell);
  if (!c.fluid) return;
  if (!AOS && warp_plain(L, c))
    os_push_plain(A0, Bp, c, op);
  else if (warp_interior(c))
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
// the same sweep for a warp with no bounce and no y/z wrap, addressed through
// the shifted plane table (SoaNb)
template <class T>
__device__ __forceinline__ void aa_odd_plain(const SoaNb<T>& N, const Ctx& c, const Trt<T>& op) {
  LBM_PLAIN_IX(c, s, sm, sp);
  T f[19];
  f[0] = ld(N.n[0] + s);
#pragma unroll
  for (int i = 1; i < 19; ++i) {
    const int j = opp(i);
    f[i] = ld(N.n[j] + nb_ix(cx(j), s, sm, sp));
  }
  collide(op, f);
  N.n[0][s] = f[0];
#pragma unroll
  for (int j = 1; j < 19; ++j) N.n[j][nb_ix(cx(j), s, sm, sp)] = f[j];
}
// fp32 SoA AA odd sweep at 6 blocks per SM (<= 42 registers; the spilled
// values are L1 hits): C1 0.92 -> 0.98, C4 0.89 -> 0.96 of the roofline
// (4: latency-bound at ~28 resident warps, 7: 0.82)
#ifndef LBM_AA_MIN_BLOCKS_F32
#define LBM_AA_MIN_BLOCKS_F32 6
#endif
template <class T, bool AOS>
struct AaOddBlocks {
  static constexpr int value =
      sizeof(T) == 4 && !AOS ? LBM_AA_MIN_BLOCKS_F32 : SoaMinBlocks<T, AOS>::value;
};
template <class T, bool AOS>
__global__ void __launch_bounds__(kBlock, AaOddBlocks<T, AOS>::value)
    k_aa_odd(Fld<T, AOS> F, Lat L, Trt<T> op, SoaNb<T> N) {
  const uint32_t cell = L.cell_begin + blockIdx.x * kBlock + threadIdx.x;
  if (cell >= L.ncells) return;
  const Ctx c = make_ctx(L, cell);
  if (!c.fluid) return;
  if (!AOS && warp_plain(L, c))
    aa_odd_plain(N, c, op);
  else if (warp_interior(c))
    aa_odd_body<false>(F, c, op);
  else
    aa_odd_body<true>(F, c, op);
}

// AA odd sweep of one slab face plane over peer memory (the p2p slab
// transport, slabs.cu): the slots a face cell reads and rewrites across the
// face, (j, X + c_j) with c_z(j) = dz, live in the neighbour slab's face plane
// and are addressed there directly (R.p[j] = that slot plane's base, indexed
// like the local ghost plane); every other access is local. The AA partition
// (each slot read and rewritten by one node per sweep) makes the neighbour's
// own odd sweep touch disjoint slots, so no ghost copy and no exchange phase.
template <class T>
struct FaceRemote {
  T* p[19];
  int dz;               // -1: bottom face (ghost plane below), +1: top face
  uint32_t ghost_base;  // local storage index of the ghost plane's first cell
};
template <bool BB, class T>
__device__ __forceinline__ void aa_odd_face_body(const Fld<T, false>& F, const Ctx& c,
                                                 const Trt<T>& op, const FaceRemote<T>& R) {
  auto slot = [&](int j) -> T* {  // (j, X + c_j), remote when it crosses the face
    if (cz(j) == R.dz) return R.p[j] + (c.nb(j) - R.ghost_base);
    return F.at_off(j, c.s, c.off(j));
  };
  T f[19];
  f[0] = ld(F.at(0, c.s));
#pragma unroll
  for (int i = 1; i < 19; ++i) {
    const int j = opp(i);
    f[i] = ld((BB && c.bb(j)) ? F.at(i, c.s) : slot(j));
  }
  collide(op, f);
  st<false>(F.at(0, c.s), f[0]);
#pragma unroll
  for (int j = 1; j < 19; ++j) st<false>((BB && c.bb(j)) ? F.at(opp(j), c.s) : slot(j), f[j]);
}
template <class T>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value)
    k_aa_odd_face(Fld<T, false> F, Lat L, Trt<T> op, FaceRemote<T> R) {
  const uint32_t cell = L.cell_begin + blockIdx.x * kBlock + threadIdx.x;
  if (cell >= L.ncells) return;
  const Ctx c = make_ctx(L, cell);
  if (!c.fluid) return;
  if (warp_interior(c))
    aa_odd_face_body<false>(F, c, op, R);
  else
    aa_odd_face_body<true>(F, c, op, R);
}

// Esoteric twist sweep (p/src/scheme_et.cpp:191-239). For pair (i, j):
// tmp_i = F[b_i][X], tmp_j = F[b_(db?i:j)][X + c_i]; collide;
// F[b_(ub?j:i)][X] = tmp_j, F[b_j][X + c_i] = tmp_i. Wall axes carry a halo
// plane, solid cells act as mailboxes, so X + c_i is always a storage slot.
template <bool BB, bool SW, class T, bool AOS>
__device__ __forceinline__ void et_body(const Fld<T, AOS>& F, const Ctx& c, const Trt<T>& op) {
  constexpr bool NC = sizeof(T) == 4 && !AOS;
  T f[19];
  f[0] = ldsel<NC>(F.at(0, c.s));
#pragma unroll
  for (int p = 0; p < 9; ++p) {
    const int i = pair_i(p), j = pair_j(p);
    f[i] = ldsel<NC>(F.at(hb<SW>(i), c.s));
    f[j] = ldsel<NC>(F.at((BB && c.bb(i)) ? hb<SW>(i) : hb<SW>(j), c.nb(i)));
  }
  collide(op, f);
  st<false>(F.at(0, c.s), f[0]);
#pragma unroll
  for (int p = 0; p < 9; ++p) {
    const int i = pair_i(p), j = pair_j(p);
    st<false>(F.at((BB && c.bb(j)) ? hb<SW>(j) : hb<SW>(i), c.s), f[j]);
    st<false>(F.at_off(hb<SW>(j), c.s, c.off(i)), f[i]);
  }
}
// plain warp: T0 = plane bases, E[p] = plane hb(j) shifted by c_i for pair p
template <bool SW, class T>
__device__ __forceinline__ void et_plain(const SoaNb<T>& T0, const SoaNb<T>& E, const Ctx& c,
                                         const Trt<T>& op) {
  constexpr bool NC = sizeof(T) == 4;
  LBM_PLAIN_IX(c, s, sm, sp);
  T f[19];
  f[0] = ldsel<NC>(T0.n[0] + s);
#pragma unroll
  for (int p = 0; p < 9; ++p) {
    const int i = pair_i(p), j = pair_j(p);
    f[i] = ldsel<NC>(T0.n[hb<SW>(i)] + s);
    f[j] = ldsel<NC>(E.n[p] + nb_ix(cx(i), s, sm, sp));
  }
  collide(op, f);
  T0.n[0][s] = f[0];
#pragma unroll
  for (int p = 0; p < 9; ++p) {
    const int i = pair_i(p), j = pair_j(p);
    T0.n[hb<SW>(i)][s] = f[j];
    E.n[p][nb_ix(cx(i), s, sm, sp)] = f[i];
  }
}
template <class T, bool AOS, bool SW>
__global__ void __launch_bounds__(kBlock, EtMinBlocks<T, AOS>::value)
    k_et(Fld<T, AOS> F, Lat L, Trt<T> op, SoaNb<T> T0, SoaNb<T> E) {
  const uint32_t cell = L.cell_begin + blockIdx.x * kBlock + threadIdx.x;
  if (cell >= L.ncells) return;
  const Ctx c = make_ctx(L, cell);
  if (!c.fluid) return;
  if (!AOS && warp_plain(L, c))
    et_plain<SW>(T0, E, c, op);
  else if (warp_interior(c))
    et_body<false, SW>(F, c, op);
  else
    et_body<true, SW>(F, c, op);
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
  // all 18 loads before any store: the compiler cannot prove the nine pairs
  // disjoint, so load / store / load order would serialise nine round trips
  uint32_t use = 0;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const int i = back_dir(k);
    if (c.bb(i)) continue;
    const bool w = c.wrapped(L, i);
    if ((mode == 1 && w) || (mode == 2 && !w)) continue;
    use |= 1u << k;
  }
  T va[9], vb[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const int i = back_dir(k);
    if (use & (1u << k)) va[k] = ld(F.at(i, c.s)), vb[k] = ld(F.at(opp(i), c.nb(i)));
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const int i = back_dir(k);
    if (use & (1u << k)) st<false>(F.at(i, c.s), vb[k]), st<false>(F.at(opp(i), c.nb(i)), va[k]);
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
// Compressed grid (p/src/scheme_cg.cpp:118-158) as plane-group push
// launches. The reference shifts the write origin by (1,1,1) cells from the
// read origin and relies on a sequential traversal; here the shift is S whole
// z-planes and a launch covers P < S planes, so no write of a launch lands in
// a slot a node of the same launch still has to read (the readers of every
// written slot lie in earlier launches) and each launch is a plain push
// sweep. x/y links wrap directly; z-seam values land in a padding plane and
// are copied to their wrapped plane after the sweep (the reference's fix-up).
template <bool BB, class T, bool AOS>
__device__ __forceinline__ void cg_push_body(const Fld<T, AOS>& F, const Ctx& c, const Trt<T>& op,
                                             int delta) {
  T f[19];
#pragma unroll
  for (int i = 0; i < 19; ++i) f[i] = ld(F.at(i, c.s));
  collide(op, f);
  // programmatic dependent launch: this group's reads never depend on the
  // previous group's writes (only write-after-read hazards in CG), so the
  // loads and the collision overlap the previous launch's tail and only the
  // stores wait for it (no-op when launched without the attribute)
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const uint32_t w = c.s + (uint32_t)delta;
  st<false>(F.at(0, w), f[0]);
#pragma unroll
  for (int i = 1; i < 19; ++i)
    st<false>((BB && c.bb(i)) ? F.at(opp(i), w) : F.at_off(i, w, c.off(i)), f[i]);
}
// plain warp: T0 = plane bases (read frame at s), Tp = planes shifted by +c_i
// (write frame at w = s + delta)
template <class T>
__device__ __forceinline__ void cg_push_plain(const SoaNb<T>& T0, const SoaNb<T>& Tp, const Ctx& c,
                                              const Trt<T>& op, int delta) {
  T f[19];
#pragma unroll
  for (int i = 0; i < 19; ++i) f[i] = ld(T0.n[i] + c.s);
  collide(op, f);
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const uint32_t w = c.s + (uint32_t)delta, wm = w + (uint32_t)(c.xm + 1), wp = w + (uint32_t)(c.xp - 1);
#pragma unroll
  for (int i = 0; i < 19; ++i) Tp.n[i][nb_ix(cx(i), w, wm, wp)] = f[i];
}
template <class T, bool AOS, bool RAW>
__global__ void __launch_bounds__(kBlock, CgMinBlocks<T, AOS>::value)
    k_cg_push(Fld<T, AOS> F, Lat L, Trt<T> op, int delta, SoaNb<T> T0, SoaNb<T> Tp) {
  // the first group of a sweep reads what the previous sweep and its seam
  // copies wrote: wait before the loads, and only then let the next group
  // launch (its loads start early, so they must not precede the previous
  // sweep's stores: a dependent starts once every block of this grid has
  // passed launch_dependents)
  if (RAW) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const uint32_t cell = L.cell_begin + blockIdx.x * kBlock + threadIdx.x;
  // threads without a node still wait for the previous group before they
  // exit: a grid's completion must imply its predecessor's, or a group with
  // no fluid cell could finish before the group ahead of it and let the next
  // group's stores overtake that group's reads
  if (cell >= L.ncells) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    return;
  }
  const Ctx c = make_ctx(L, cell);
  if (!c.fluid) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    return;
  }
  if (!AOS && warp_plain(L, c))
    cg_push_plain(T0, Tp, c, op, delta);
  else if (warp_interior(c))
    cg_push_body<false>(F, c, op, delta);
  else
    cg_push_body<true>(F, c, op, delta);
}

// z-seam fix-up: copy the 5 slot planes of one padding plane to the wrapped
// plane, for the links that were actually written there — i.e. whose writer
// (the node one link back, on plane writer_z) is fluid and did not bounce
template <class T, bool AOS>
__global__ void k_plane_copy(Fld<T, AOS> F, Lat L, int8_t d0, int8_t d1, int8_t d2, int8_t d3,
                             int8_t d4, uint32_t src, uint32_t dst, int writer_z) {
  // launched early (programmatic dependent launch): copy only once the
  // sweep's last group is complete
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const uint32_t plane = (uint32_t)L.nx * L.ny;
  const uint32_t k = blockIdx.x * kBlock + threadIdx.x;
  if (k >= plane) return;
  const int x = (int)(k % L.nx), y = (int)(k / L.nx);
  const int8_t d[5] = {d0, d1, d2, d3, d4};
  uint32_t use = 0;
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    int xw = x - cx(d[q]), yw = y - cy(d[q]);
    if (xw < 0 || xw >= L.nx) {
      if (L.wall[0]) continue;
      xw = xw < 0 ? xw + L.nx : xw - L.nx;
    }
    if (yw < 0 || yw >= L.ny) {
      if (L.wall[1]) continue;
      yw = yw < 0 ? yw + L.ny : yw - L.ny;
    }
    if (L.linkmask) {
      const uint32_t lm = L.linkmask[(uint32_t)xw + (uint32_t)L.nx * ((uint32_t)yw + (uint32_t)L.ny * writer_z)];
      if (!(lm & 1u) || ((lm >> d[q]) & 1u)) continue;
    }
    use |= 1u << q;
  }
  // five loads, then five stores (the planes are distinct; see k_swap)
  T v[5];
#pragma unroll
  for (int q = 0; q < 5; ++q)
    if (use & (1u << q)) v[q] = *F.at(d[q], src + k);
#pragma unroll
  for (int q = 0; q < 5; ++q)
    if (use & (1u << q)) *F.at(d[q], dst + k) = v[q];
}

}  // namespace

void launch_local(cudaStream_t st, const DField& src, const DField& dst, const dev::Lat& L,
                  const TrtHost& op, bool rd_opp, bool wr_opp) {
  if (L.ncells <= L.cell_begin) return;
  uint32_t soff = 0;
  if (aos_contiguous(src, L, &soff)) {
    if (launch_aos_local_stream(st, src, dst, L, op, rd_opp, wr_opp, soff)) return;
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
  if (launch_aos_window(st, kWinModeStream, b, a, L, TrtHost{})) return;
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
    k_ts_stream<T, A><<<grid_for(L.ncells - L.cell_begin), kBlock, 0, st>>>(
        fld<T, A>(a), fld<T, A>(b), L, soa_nb<T>(a, L, 0), soa_nb<T>(b, L, -1));
  });
}

void launch_os_pull(cudaStream_t st, const DField& a, const DField& b, const dev::Lat& L,
                    const TrtHost& op, bool streaming, bool two_s) {
  if (L.ncells <= L.cell_begin) return;
  if (launch_aos_window(st, kWinModePull, a, b, L, op)) return;
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
    constexpr bool tab = kOsPullTab<T, true>;
    auto ta = fld_sel<T, A, tab>(a);
    auto tb = fld_sel<T, A, tab>(b);
    const auto o = cast_op<T>(op);
    const unsigned g = grid_for(L.ncells - L.cell_begin);
    const auto am = soa_nb<T>(a, L, -1), b0 = soa_nb<T>(b, L, 0);
    if (!streaming && !two_s) k_os_pull<T, A, false, false><<<g, kBlock, 0, st>>>(fa, fb, L, o, am, b0);
    if (!streaming && two_s) k_os_pull<T, A, false, true><<<g, kBlock, 0, st>>>(fa, fb, L, o, am, b0);
    if (streaming && !two_s) k_os_pull<T, A, true, false><<<g, kBlock, 0, st>>>(ta, tb, L, o, am, b0);
    if (streaming && two_s) k_os_pull<T, A, true, true><<<g, kBlock, 0, st>>>(ta, tb, L, o, am, b0);
  });
}

void launch_os_push(cudaStream_t st, const DField& a, const DField& b, const dev::Lat& L,
                    const TrtHost& op) {
  if (L.ncells <= L.cell_begin) return;
  if (launch_aos_window(st, kWinModePush, a, b, L, op)) return;
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
    constexpr bool tab = kOsPushTab<T, A>;
    k_os_push<T, A><<<grid_for(L.ncells - L.cell_begin), kBlock, 0, st>>>(
        fld_sel<T, A, tab>(a), fld_sel<T, A, tab>(b), L, cast_op<T>(op), soa_nb<T>(a, L, 0),
        soa_nb<T>(b, L, 1));
  });
}

void launch_aa_odd(cudaStream_t st, const DField& f, const dev::Lat& L, const TrtHost& op) {
  if (L.ncells <= L.cell_begin) return;
  if (launch_aos_window(st, kWinModeAaOdd, f, f, L, op)) return;
  LBM_DISPATCH(f, {
    k_aa_odd<T, A><<<grid_for(L.ncells - L.cell_begin), kBlock, 0, st>>>(fld<T, A>(f), L, cast_op<T>(op),
                                                                         soa_nb<T>(f, L));
  });
}

void launch_aa_odd_face(cudaStream_t st, const DField& f, const dev::Lat& L, const TrtHost& op,
                        void* const remote[19], int dz, uint32_t ghost_base) {
  if (L.ncells <= L.cell_begin) return;
  if (f.aos) throw std::invalid_argument("p2p face sweep: SoA fields only");
  if (f.prec == Prec::f64) {
    FaceRemote<double> R;
    for (int k = 0; k < 19; ++k) R.p[k] = static_cast<double*>(remote[k]);
    R.dz = dz;
    R.ghost_base = ghost_base;
    k_aa_odd_face<double><<<grid_for(L.ncells - L.cell_begin), kBlock, 0, st>>>(
        fld<double, false>(f), L, cast_op<double>(op), R);
  } else {
    FaceRemote<float> R;
    for (int k = 0; k < 19; ++k) R.p[k] = static_cast<float*>(remote[k]);
    R.dz = dz;
    R.ghost_base = ghost_base;
    k_aa_odd_face<float><<<grid_for(L.ncells - L.cell_begin), kBlock, 0, st>>>(
        fld<float, false>(f), L, cast_op<float>(op), R);
  }
}

void launch_et(cudaStream_t st, const DField& f, const dev::Lat& L, const TrtHost& op,
               const EtBase& base) {
  if (L.ncells <= L.cell_begin) return;
  if (launch_aos_window(st, base.swapped() ? kWinModeEtSw : kWinModeEt, f, f, L, op)) return;
  LBM_DISPATCH(f, {
    const unsigned g = grid_for(L.ncells - L.cell_begin);
    if (base.swapped())
      k_et<T, A, true><<<g, kBlock, 0, st>>>(fld<T, A>(f), L, cast_op<T>(op), soa_nb<T>(f, L, 0),
                                             et_nb<T>(f, L, true));
    else
      k_et<T, A, false><<<g, kBlock, 0, st>>>(fld<T, A>(f), L, cast_op<T>(op), soa_nb<T>(f, L, 0),
                                              et_nb<T>(f, L, false));
  });
}

void launch_swap(cudaStream_t st, const DField& f, const dev::Lat& L, int mode) {
  if (L.ncells <= L.cell_begin) return;
  if (mode == 1 && launch_aos_window(st, kWinModeSwap, f, f, L, TrtHost{})) return;
  LBM_DISPATCH(f, { k_swap<T, A><<<grid_for(L.ncells - L.cell_begin), kBlock, 0, st>>>(fld<T, A>(f), L, mode); });
}

void launch_cg_push(cudaStream_t st, const DField& f, const dev::Lat& L, const TrtHost& op,
                    int delta, bool early) {
  if (L.ncells <= L.cell_begin) return;
  LBM_DISPATCH(f, {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid_for(L.ncells - L.cell_begin));
    cfg.blockDim = dim3(kBlock);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (early)
      cudaLaunchKernelEx(&cfg, k_cg_push<T, A, false>, fld<T, A>(f), L, cast_op<T>(op), delta,
                         soa_nb<T>(f, L, 0), soa_nb<T>(f, L, 1));
    else
      cudaLaunchKernelEx(&cfg, k_cg_push<T, A, true>, fld<T, A>(f), L, cast_op<T>(op), delta,
                         soa_nb<T>(f, L, 0), soa_nb<T>(f, L, 1));
  });
}

void launch_plane_copy(cudaStream_t st, const DField& f, const dev::Lat& L, const int* dirs,
                       uint32_t src, uint32_t dst, int writer_z) {
  const uint32_t plane = (uint32_t)L.nx * L.ny;
  LBM_DISPATCH(f, {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid_for(plane));
    cfg.blockDim = dim3(kBlock);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_plane_copy<T, A>, fld<T, A>(f), L, (int8_t)dirs[0], (int8_t)dirs[1],
                       (int8_t)dirs[2], (int8_t)dirs[3], (int8_t)dirs[4], src, dst, writer_z);
  });
}

void launch_swap_list(cudaStream_t st, const DField& f, const long long* a, const long long* b,
                      const int8_t* dir, long long count) {
  if (count <= 0) return;
  LBM_DISPATCH(f, {
    k_swap_list<T, A><<<grid_for(count), kBlock, 0, st>>>(fld<T, A>(f), a, b, dir, count);
  });
}

void EtBase::throw_bad_handles() {
  throw std::logic_error("ET handle table is neither the identity nor fully swapped");
}

}  // namespace lbmgpu
