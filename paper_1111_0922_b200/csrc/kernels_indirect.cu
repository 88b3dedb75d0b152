// sm_100a kernels for indirect (IDX) addressing: fluid nodes only, enumerated
// x-fastest, one thread per node. The adjacency is stored transposed,
// adj[(i-1)*N + n], so the 18 index loads of a warp are 18 coalesced 128-byte
// rows (the reference's node-major adjacency[n*18 + i-1], geometry.cpp:196-205,
// is exported bit-identically by lbmgpu_build_sparse). A bounce link stores
// the node itself.
#include "dispatch.h"
#include "launch.h"

#include <algorithm>
#include <cstdlib>

#include <algorithm>

namespace lbmgpu {
using namespace dev;

namespace {

inline unsigned grid_for(uint64_t n) { return (unsigned)((n + kBlock - 1) / kBlock); }

__device__ __forceinline__ uint32_t ldidx(const uint32_t* p) { return __ldg(p); }

// local collision over nodes (TS collide, precollide, AA even, SWAP collide);
// no indirection, so the direct k_local's register budget (fp64 SoA at 3
// blocks per SM)
template <class T, bool AOS, bool RD_OPP, bool WR_OPP>
__global__ void __launch_bounds__(kBlock, SoaMinBlocks<T, AOS>::value) k_local_idx(Fld<T, AOS> src, Fld<T, AOS> dst,
                                                      uint32_t first, uint32_t n, Trt<T> op) {
  const uint32_t node = first + blockIdx.x * kBlock + threadIdx.x;
  if (node >= n) return;
  T f[19];
#pragma unroll
  for (int i = 0; i < 19; ++i) f[i] = ld(src.at(RD_OPP ? opp(i) : i, node));
  collide(op, f);
#pragma unroll
  for (int i = 0; i < 19; ++i) st<false>(dst.at(WR_OPP ? opp(i) : i, node), f[i]);
}

// TS streaming over the IDX graph (GPU extension; the reference's TS is
// direct-only, stepper.cpp:140-153): A[i][n] = src == n ? B[opp i][n] : B[i][src]
template <class T, bool AOS>
__device__ __forceinline__ void ts_stream_idx_node(const Fld<T, AOS>& a, const Fld<T, AOS>& b,
                                                   const Idx& I, uint32_t node) {
  T v[19];
  v[0] = ld(b.at(0, node));
#pragma unroll
  for (int i = 1; i < 19; ++i) {
    const int j = opp(i);
    const uint32_t src = ldidx(I.adj + (size_t)(j - 1) * I.n + node);
    v[i] = ld(src == node ? b.at(j, node) : b.at(i, src));
  }
#pragma unroll
  for (int i = 0; i < 19; ++i) st<false>(a.at(i, node), v[i]);
}
template <class T, bool AOS>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value) k_ts_stream_idx(Fld<T, AOS> a, Fld<T, AOS> b, Idx I) {
  const uint32_t node = I.first + blockIdx.x * kBlock + threadIdx.x;
  if (node >= I.end()) return;
  ts_stream_idx_node(a, b, I, node);
}

// OS / OSNT pull, indirect (p/src/scheme_os.cpp:203-226, scheme_osnt.cpp:219-260)
template <class T, bool AOS, bool NT, bool TWO_S>
__global__ void __launch_bounds__(kBlock, SoaMinBlocks<T, AOS>::value) k_os_pull_idx(Fld<T, AOS> a, Fld<T, AOS> b, Idx I,
                                                        Trt<T> op) {
  const uint32_t node = I.first + blockIdx.x * kBlock + threadIdx.x;
  if (node >= I.end()) return;
  T f[19];
  f[0] = ld(a.at(0, node));
#pragma unroll
  for (int i = 1; i < 19; ++i) {
    const int j = opp(i);
    const uint32_t src = ldidx(I.adj + (size_t)(j - 1) * I.n + node);
    f[i] = ld(src == node ? a.at(j, node) : a.at(i, src));
  }
  collide(op, f);
  if (!TWO_S) {
#pragma unroll
    for (int i = 0; i < 19; ++i) st<NT>(b.at(i, node), f[i]);
  } else {
    st<NT>(b.at(0, node), f[0]);
#pragma unroll
    for (int p = 0; p < 9; ++p) {
      st<NT>(b.at(pair_i(p), node), f[pair_i(p)]);
      st<NT>(b.at(pair_j(p), node), f[pair_j(p)]);
    }
  }
}

// OS push, indirect (p/src/scheme_os.cpp:176-201)
template <class T, bool AOS>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value) k_os_push_idx(Fld<T, AOS> a, Fld<T, AOS> b, Idx I,
                                                        Trt<T> op) {
  const uint32_t node = I.first + blockIdx.x * kBlock + threadIdx.x;
  if (node >= I.end()) return;
  // fp64: the scatter targets first, so their loads overlap the PDF loads and
  // the collision instead of stalling each store (C2 0.86 -> 0.94 of the
  // roofline); fp32 loads them at the store (its 64-register budget spills)
  constexpr bool kEarly = sizeof(T) == 8;
  uint32_t e[19];
  if (kEarly) {
#pragma unroll
    for (int i = 1; i < 19; ++i) e[i] = ldidx(I.adj + (size_t)(i - 1) * I.n + node);
  }
  T f[19];
#pragma unroll
  for (int i = 0; i < 19; ++i) f[i] = ld(a.at(i, node));
  collide(op, f);
  st<false>(b.at(0, node), f[0]);
#pragma unroll
  for (int i = 1; i < 19; ++i) {
    const uint32_t nb = kEarly ? e[i] : ldidx(I.adj + (size_t)(i - 1) * I.n + node);
    st<false>(nb == node ? b.at(opp(i), node) : b.at(i, nb), f[i]);
  }
}

// AA odd sweep, indirect (p/src/scheme_aap.cpp:175-201). The gather uses
// row[opp i - 1] for i = 1..18 and the scatter row[j - 1] for j = 1..18: the
// same 18 entries, loaded once.
template <class FA, class T>
__device__ __forceinline__ void aa_odd_idx_node(const FA& F, const Idx& I, const Trt<T>& op,
                                                uint32_t node) {
  uint32_t e[19];
#pragma unroll
  for (int i = 1; i < 19; ++i) e[i] = ldidx(I.adj + (size_t)(i - 1) * I.n + node);
  T f[19];
  f[0] = ld(F.at(0, node));
#pragma unroll
  for (int i = 1; i < 19; ++i) {
    const int j = opp(i);
    f[i] = ld(e[j] == node ? F.at(i, node) : F.at(j, e[j]));
  }
  collide(op, f);
  st<false>(F.at(0, node), f[0]);
#pragma unroll
  for (int j = 1; j < 19; ++j) st<false>(e[j] == node ? F.at(opp(j), node) : F.at(j, e[j]), f[j]);
}
// fp32 SoA addresses through plane bases (FldT: C4 0.97 -> 0.98, C2 0.91 ->
// 0.94 of the roofline, measured)
template <class T>
constexpr bool kAaIdxTab = sizeof(T) == 4;
template <class T, bool AOS>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value)
    k_aa_odd_idx(FldSel<T, AOS, kAaIdxTab<T>> F, Idx I, Trt<T> op) {
  const uint32_t node = I.first + blockIdx.x * kBlock + threadIdx.x;
  if (node >= I.end()) return;
  aa_odd_idx_node(F, I, op, node);
}

// Persistent-block pipeline over 256-node batches: ROWS rows of a transposed
// per-node table (adjacency or ET rem) for the NEXT batch are staged in shared
// memory by cp.async while the current batch computes, so the PDF accesses do
// not wait behind their index loads. body(node, row) with row(r) = table[r][node].
template <int ROWS, bool VEC, class Body>
__device__ __forceinline__ void staged_batches(const uint32_t* __restrict__ table, const Idx& I,
                                               uint32_t nbatch, uint32_t (*sm)[ROWS][kBlock],
                                               Body body) {
  const uint32_t tid = threadIdx.x;
  auto issue = [&](uint32_t k) {
    const uint32_t bt = blockIdx.x + k * gridDim.x;
    if (bt >= nbatch) return;
    const uint32_t n0 = I.first + bt * kBlock;
    const uint32_t cnt = min((uint32_t)kBlock, I.end() - n0);
    uint32_t* dst = &sm[k & 1][0][0];
    if (VEC && cnt == kBlock) {
      for (uint32_t q = tid; q < ROWS * (kBlock / 4); q += kBlock) {
        const uint32_t row = q / (kBlock / 4), c = q - row * (kBlock / 4);
        cp_async<16>(dst + row * kBlock + c * 4, table + (size_t)row * I.n + n0 + c * 4);
      }
    } else {
      for (uint32_t q = tid; q < ROWS * cnt; q += kBlock) {
        const uint32_t row = q / cnt, c = q - row * cnt;
        cp_async<4>(dst + row * kBlock + c, table + (size_t)row * I.n + n0 + c);
      }
    }
  };
  issue(0);
  cp_commit();
  for (uint32_t k = 0; blockIdx.x + k * gridDim.x < nbatch; ++k) {
    issue(k + 1);
    cp_commit();
    cp_wait1();
    __syncthreads();
    const uint32_t node = I.first + (blockIdx.x + k * gridDim.x) * kBlock + tid;
    if (node < I.end()) body(node, [&](int r) { return sm[k & 1][r][tid]; });
    __syncthreads();  // the slot is refilled two batches later
  }
}

template <int ROWS, bool VEC, class Body>
__device__ __forceinline__ void staged_rows(const uint32_t* __restrict__ table, const Idx& I,
                                            uint32_t nbatch, Body body) {
  __shared__ __align__(16) uint32_t sb[2][ROWS][kBlock];
  staged_batches<ROWS, VEC>(table, I, nbatch, sb, body);
}

// Staged-table kernels (fp64): resident blocks per SM, and whether the staged
// rows are read from shared memory at each use instead of being held in
// registers across the collision (measured: ET C2 0.73 -> 0.76, C4 0.87 ->
// 0.96 of the roofline, AA unchanged; 3 blocks per SM and warp-private
// staging without block barriers both measured slower)
#ifndef LBM_IDX_PF_MIN_BLOCKS
#define LBM_IDX_PF_MIN_BLOCKS 2
#endif
#ifndef LBM_IDX_PF_LAZY
#define LBM_IDX_PF_LAZY 1
#endif
// AA odd (fp64 SoA): the software-pipelined staged kernel (k_aa_odd_idx_pp)
#ifndef LBM_IDX_PP
#define LBM_IDX_PP 1
#endif

// AA odd sweep with the adjacency staged (fp64; C4 0.94 -> 0.97 of the
// roofline; fp32 spills at its register budget and keeps k_aa_odd_idx)
template <class T, bool VEC>
__global__ void __launch_bounds__(kBlock, LBM_IDX_PF_MIN_BLOCKS)
    k_aa_odd_idx_pf(Fld<T, false> F, Idx I, Trt<T> op, uint32_t nbatch) {
  staged_rows<18, VEC>(I.adj, I, nbatch, [&](uint32_t node, auto row) {
    uint32_t e[19] = {};
    if (!LBM_IDX_PF_LAZY) {
#pragma unroll
      for (int i = 1; i < 19; ++i) e[i] = row(i - 1);
    }
    auto nb = [&](int k) { return LBM_IDX_PF_LAZY ? row(k - 1) : e[k]; };
    T f[19];
    f[0] = ld(F.at(0, node));
#pragma unroll
    for (int i = 1; i < 19; ++i) {
      const int j = opp(i);
      const uint32_t ej = nb(j);
      f[i] = ld(ej == node ? F.at(i, node) : F.at(j, ej));
    }
    collide(op, f);
    st<false>(F.at(0, node), f[0]);
#pragma unroll
    for (int j = 1; j < 19; ++j) {
      const uint32_t ej = nb(j);
      st<false>(ej == node ? F.at(opp(j), node) : F.at(j, ej), f[j]);
    }
  });
}

// Software pipeline over the staged batches (AA odd, ET; fp64 SoA): the
// table rows (adjacency / rem) are staged two batches ahead (three buffers)
// and the gathers of batch k + 1 are issued before batch k collides and
// scatters, so a thread keeps one node's loads in flight across its other
// node's collision. In place but race-free: every slot is read and
// rewritten by exactly one node per sweep. gather(node, row, f) / finish(node,
// row, f) with row(r) = table[r][node].
template <class T, int ROWS, bool VEC, class Gather, class Finish>
__device__ __forceinline__ void pp_batches(const uint32_t* __restrict__ table, const Idx& I,
                                           uint32_t nbatch, unsigned char* smem, Gather gather,
                                           Finish finish) {
  uint32_t(*sb)[ROWS][kBlock] = reinterpret_cast<uint32_t(*)[ROWS][kBlock]>(smem);
  const uint32_t tid = threadIdx.x;
  auto bat = [&](uint32_t k) { return blockIdx.x + k * gridDim.x; };
  auto issue = [&](uint32_t k) {
    const uint32_t bt = bat(k);
    if (bt >= nbatch) return;
    const uint32_t n0 = I.first + bt * kBlock;
    const uint32_t cnt = min((uint32_t)kBlock, I.end() - n0);
    uint32_t* dst = &sb[k % 3][0][0];
    if (VEC && cnt == kBlock) {
      for (uint32_t q = tid; q < ROWS * (kBlock / 4); q += kBlock) {
        const uint32_t row = q / (kBlock / 4), c = q - row * (kBlock / 4);
        cp_async<16>(dst + row * kBlock + c * 4, table + (size_t)row * I.n + n0 + c * 4);
      }
    } else {
      for (uint32_t q = tid; q < ROWS * cnt; q += kBlock) {
        const uint32_t row = q / cnt, c = q - row * cnt;
        cp_async<4>(dst + row * kBlock + c, table + (size_t)row * I.n + n0 + c);
      }
    }
  };
  if (bat(0) >= nbatch) return;
  issue(0);
  cp_commit();
  issue(1);
  cp_commit();
  cp_wait1();
  __syncthreads();
  T fc[19];
  uint32_t nc = I.first + bat(0) * kBlock + tid;
  if (nc < I.end()) gather(nc, [&](int r) { return sb[0][r][tid]; }, fc);
  for (uint32_t k = 0; bat(k) < nbatch; ++k) {
    __syncthreads();  // batch k - 1 is done with its rows: buffer (k + 2) % 3 is free
    issue(k + 2);
    cp_commit();
    cp_wait1();       // rows of batch k + 1
    __syncthreads();
    T fn[19];
    const uint32_t nn = I.first + bat(k + 1) * kBlock + tid;
    const bool hn = bat(k + 1) < nbatch && nn < I.end();
    if (hn) gather(nn, [&](int r) { return sb[(k + 1) % 3][r][tid]; }, fn);
    if (nc < I.end()) finish(nc, [&](int r) { return sb[k % 3][r][tid]; }, fc);
#pragma unroll
    for (int i = 0; i < 19; ++i) fc[i] = fn[i];
    nc = hn ? nn : I.end();
  }
}
template <int ROWS>
constexpr int kPpBytes = 3 * ROWS * kBlock * 4;
// resident blocks per SM of the pipelined kernels: fp64 2 (<= 128 registers),
// fp32 LBM_IDX_PP32_BLOCKS
#ifndef LBM_IDX_PP32_BLOCKS
#define LBM_IDX_PP32_BLOCKS 4
#endif
// fp32 through the pipeline (-DLBM_IDX_PP32=1): measured slower on C2 (AA
// 0.93 -> 0.75-0.88, ET 0.80 -> 0.73-0.78) at 3-4 blocks per SM
#ifndef LBM_IDX_PP32
#define LBM_IDX_PP32 0
#endif
template <class T>
struct PpBlocks {
  static constexpr int value = sizeof(T) == 8 ? LBM_IDX_PF_MIN_BLOCKS : LBM_IDX_PP32_BLOCKS;
};

template <class T, bool VEC>
__global__ void __launch_bounds__(kBlock, PpBlocks<T>::value)
    k_aa_odd_idx_pp(Fld<T, false> F, Idx I, Trt<T> op, uint32_t nbatch) {
  extern __shared__ __align__(16) unsigned char pp_smem[];
  auto gather = [&](uint32_t node, auto row, T(&f)[19]) {
    f[0] = ld(F.at(0, node));
#pragma unroll
    for (int i = 1; i < 19; ++i) {
      const int j = opp(i);
      const uint32_t ej = row(j - 1);
      f[i] = ld(ej == node ? F.at(i, node) : F.at(j, ej));
    }
  };
  auto finish = [&](uint32_t node, auto row, T(&f)[19]) {
    collide(op, f);
    st<false>(F.at(0, node), f[0]);
#pragma unroll
    for (int j = 1; j < 19; ++j) {
      const uint32_t ej = row(j - 1);
      st<false>(ej == node ? F.at(opp(j), node) : F.at(j, ej), f[j]);
    }
  };
  pp_batches<T, 18, VEC>(I.adj, I, nbatch, pp_smem, gather, finish);
}

template <class T, bool SW, bool VEC>
__global__ void __launch_bounds__(kBlock, PpBlocks<T>::value)
    k_et_idx_pp(Fld<T, false> F, Idx I, Trt<T> op, uint32_t nbatch) {
  extern __shared__ __align__(16) unsigned char pp_smem[];
  auto gather = [&](uint32_t node, auto row, T(&f)[19]) {
    f[0] = ld(F.at(0, node));
#pragma unroll
    for (int p = 0; p < 9; ++p) {
      const int i = pair_i(p), j = pair_j(p);
      const uint32_t r = row(p) & 0x7fffffffu;
      f[i] = ld(F.at(hb<SW>(i), node));
      f[j] = ld(F.at(r >= I.n ? hb<SW>(i) : hb<SW>(j), r));
    }
  };
  auto finish = [&](uint32_t node, auto row, T(&f)[19]) {
    collide(op, f);
    st<false>(F.at(0, node), f[0]);
#pragma unroll
    for (int p = 0; p < 9; ++p) {
      const int i = pair_i(p), j = pair_j(p);
      const uint32_t rv = row(p);
      const bool ub = (rv & 0x80000000u) != 0;
      st<false>(F.at(ub ? hb<SW>(j) : hb<SW>(i), node), f[j]);
      st<false>(F.at(hb<SW>(j), rv & 0x7fffffffu), f[i]);
    }
  };
  pp_batches<T, 9, VEC>(I.rem, I, nbatch, pp_smem, gather, finish);
}

// ET sweep with the rem rows staged (fp64)
template <class T, bool SW, bool VEC>
__global__ void __launch_bounds__(kBlock, LBM_IDX_PF_MIN_BLOCKS)
    k_et_idx_pf(Fld<T, false> F, Idx I, Trt<T> op, uint32_t nbatch) {
  staged_rows<9, VEC>(I.rem, I, nbatch, [&](uint32_t node, auto row) {
    uint32_t rs[9] = {};
    auto rm = [&](int p) { return LBM_IDX_PF_LAZY ? row(p) : rs[p]; };
    T f[19];
    f[0] = ld(F.at(0, node));
#pragma unroll
    for (int p = 0; p < 9; ++p) {
      const int i = pair_i(p), j = pair_j(p);
      if (!LBM_IDX_PF_LAZY) rs[p] = row(p);
      const uint32_t r = rm(p) & 0x7fffffffu;
      f[i] = ld(F.at(hb<SW>(i), node));
      f[j] = ld(F.at(r >= I.n ? hb<SW>(i) : hb<SW>(j), r));
    }
    collide(op, f);
    st<false>(F.at(0, node), f[0]);
#pragma unroll
    for (int p = 0; p < 9; ++p) {
      const int i = pair_i(p), j = pair_j(p);
      const uint32_t rv = rm(p);
      const bool ub = (rv & 0x80000000u) != 0;
      st<false>(F.at(ub ? hb<SW>(j) : hb<SW>(i), node), f[j]);
      st<false>(F.at(hb<SW>(j), rv & 0x7fffffffu), f[i]);
    }
  });
}

// ---------------------------------------------------------------------------
// Asynchronous-gather pipeline (SoA, in-place sweeps over the IDX graph: AA
// odd, ET). The register-held gathers of the kernels above leave a warp's
// loads in flight only until its collision starts (C2 porous: 16 warps per
// SM, long-scoreboard 8-9 stalls per issue, 0.75-0.89 of the roofline).
// Here every gather is a cp.async into shared memory, one batch ahead: while
// batch k collides from shared memory and scatters its results, the 19
// gathers of batch k + 1 and the index rows (adjacency / rem) of batch k + 2
// are in flight, without holding registers. Each thread gathers, and later
// reads, only its own node's column, so only the index rows (copied as
// 16-byte vectors by the whole block) need the block barrier. In-place
// safety: the slots a node gathers are exactly the slots it rewrites (AA odd
// and ET partition the slots among nodes), so batch k + 1's gathers and
// batch k's stores never touch the same slot.
// ---------------------------------------------------------------------------
constexpr int kAgB = 128;  // nodes per batch = threads per block
template <class T>
struct AgCfg {
  static constexpr int kBlocks = sizeof(T) == 8 ? 3 : 4;  // resident blocks per SM
};
template <int ROWS, class T>
constexpr size_t ag_smem_bytes() {
  return (size_t)3 * ROWS * kAgB * 4 + (size_t)2 * 19 * kAgB * sizeof(T);
}

template <class T, bool ET, bool SW, bool VEC>
__global__ void __launch_bounds__(kAgB, AgCfg<T>::kBlocks)
    k_idx_ag(Fld<T, false> F, Idx I, Trt<T> op, uint32_t nbatch) {
  constexpr int ROWS = ET ? 9 : 18;
  extern __shared__ __align__(16) unsigned char ag_smem[];
  auto tab = reinterpret_cast<uint32_t(*)[ROWS][kAgB]>(ag_smem);  // [3]
  auto gs = reinterpret_cast<T(*)[19][kAgB]>(ag_smem + (size_t)3 * ROWS * kAgB * 4);  // [2]
  const uint32_t* table = ET ? I.rem : I.adj;
  const uint32_t tid = threadIdx.x;
  auto batch = [&](uint32_t k) { return blockIdx.x + k * gridDim.x; };
  auto issue_tab = [&](uint32_t k) {
    const uint32_t bt = batch(k);
    if (bt >= nbatch) return;
    const uint32_t n0 = I.first + bt * kAgB, cnt = min((uint32_t)kAgB, I.end() - n0);
    uint32_t* dst = &tab[k % 3][0][0];
    if (VEC && cnt == kAgB) {
      for (uint32_t q = tid; q < ROWS * (kAgB / 4); q += kAgB) {
        const uint32_t row = q / (kAgB / 4), c = q - row * (kAgB / 4);
        cp_async<16>(dst + row * kAgB + c * 4, table + (size_t)row * I.n + n0 + c * 4);
      }
    } else {
      for (uint32_t q = tid; q < ROWS * cnt; q += kAgB) {
        const uint32_t row = q / cnt, c = q - row * cnt;
        cp_async<4>(dst + row * kAgB + c, table + (size_t)row * I.n + n0 + c);
      }
    }
  };
  auto node_of = [&](uint32_t k) { return I.first + batch(k) * kAgB + tid; };
  auto issue_gather = [&](uint32_t k) {
    if (batch(k) >= nbatch) return;
    const uint32_t node = node_of(k);
    if (node >= I.end()) return;
    T* g = &gs[k & 1][0][tid];
    const uint32_t(&row)[ROWS][kAgB] = tab[k % 3];
    cp_async<sizeof(T)>(g, F.at(0, node));
    if constexpr (!ET) {  // AA odd: slot j of the neighbour along c_j (bounce: own slot i)
#pragma unroll
      for (int i = 1; i < 19; ++i) {
        const int j = opp(i);
        const uint32_t ej = row[j - 1][tid];
        cp_async<sizeof(T)>(g + i * kAgB, ej == node ? F.at(i, node) : F.at(j, ej));
      }
    } else {  // ET: own slot b_i, and slot b_j of the neighbour along c_i (or mailbox)
#pragma unroll
      for (int p = 0; p < 9; ++p) {
        const int i = pair_i(p), j = pair_j(p);
        const uint32_t r = row[p][tid] & 0x7fffffffu;
        cp_async<sizeof(T)>(g + i * kAgB, F.at(hb<SW>(i), node));
        cp_async<sizeof(T)>(g + j * kAgB, F.at(r >= I.n ? hb<SW>(i) : hb<SW>(j), r));
      }
    }
  };
  issue_tab(0);
  issue_tab(1);
  cp_commit();
  cp_wait0();
  __syncthreads();
  issue_gather(0);
  cp_commit();
  for (uint32_t k = 0; batch(k) < nbatch; ++k) {
    // batch k's gathers and batch k + 1's rows have landed; every thread is
    // done with batch k - 1 (its row slot is refilled with batch k + 2, its
    // gather slot with batch k + 1)
    cp_wait0();
    __syncthreads();
    issue_tab(k + 2);
    issue_gather(k + 1);
    cp_commit();
    const uint32_t node = node_of(k);
    if (node >= I.end()) continue;
    const T* g = &gs[k & 1][0][tid];
    const uint32_t(&row)[ROWS][kAgB] = tab[k % 3];
    T f[19];
#pragma unroll
    for (int i = 0; i < 19; ++i) f[i] = g[i * kAgB];
    collide(op, f);
    st<false>(F.at(0, node), f[0]);
    if constexpr (!ET) {
#pragma unroll
      for (int j = 1; j < 19; ++j) {
        const uint32_t ej = row[j - 1][tid];
        st<false>(ej == node ? F.at(opp(j), node) : F.at(j, ej), f[j]);
      }
    } else {
#pragma unroll
      for (int p = 0; p < 9; ++p) {
        const int i = pair_i(p), j = pair_j(p);
        const uint32_t rv = row[p][tid];
        const bool ub = (rv & 0x80000000u) != 0;
        st<false>(F.at(ub ? hb<SW>(j) : hb<SW>(i), node), f[j]);
        st<false>(F.at(hb<SW>(j), rv & 0x7fffffffu), f[i]);
      }
    }
  }
}

// ET sweep, indirect (p/src/scheme_et.cpp:241-272): rem[p][n] = neighbour
// along c_i or a mailbox slot >= N (i-link bounces), bit 31 = j-link bounces.
template <class T, bool AOS, bool SW>
__device__ __forceinline__ void et_idx_node(const Fld<T, AOS>& F, const Idx& I, const Trt<T>& op,
                                            uint32_t node) {
  uint32_t rs[9];
  T f[19];
  f[0] = ld(F.at(0, node));
#pragma unroll
  for (int p = 0; p < 9; ++p) {
    const int i = pair_i(p), j = pair_j(p);
    rs[p] = ldidx(I.rem + (size_t)p * I.n + node);
    const uint32_t r = rs[p] & 0x7fffffffu;
    const bool db = r >= I.n;
    f[i] = ld(F.at(hb<SW>(i), node));
    f[j] = ld(F.at(db ? hb<SW>(i) : hb<SW>(j), r));
  }
  collide(op, f);
  st<false>(F.at(0, node), f[0]);
#pragma unroll
  for (int p = 0; p < 9; ++p) {
    const int i = pair_i(p), j = pair_j(p);
    // fp32 SoA (6 blocks per SM, <= 42 registers): re-read the rem entry (an
    // L1 hit) instead of keeping nine live across the collision
    const uint32_t rv = (sizeof(T) == 4 && !AOS) ? ldidx(I.rem + (size_t)p * I.n + node) : rs[p];
    const bool ub = (rv & 0x80000000u) != 0;
    st<false>(F.at(ub ? hb<SW>(j) : hb<SW>(i), node), f[j]);
    st<false>(F.at(hb<SW>(j), rv & 0x7fffffffu), f[i]);
  }
}
template <class T, bool AOS, bool SW>
__global__ void __launch_bounds__(kBlock, EtMinBlocks<T, AOS>::value) k_et_idx(Fld<T, AOS> F, Idx I, Trt<T> op) {
  const uint32_t node = I.first + blockIdx.x * kBlock + threadIdx.x;
  if (node >= I.end()) return;
  et_idx_node<T, AOS, SW>(F, I, op, node);
}

// SWAP link exchange over the IDX graph (GPU extension, see k_swap): every
// non-bounce back-half link swaps (i, n) <-> (opp i, adj[i][n]).
template <class T, bool AOS>
__device__ __forceinline__ void swap_idx_node(const Fld<T, AOS>& F, const Idx& I, uint32_t node) {
  // all loads before any store (the pairs are disjoint, which the compiler
  // cannot prove: load / store / load order serialises nine round trips)
  uint32_t nb[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) nb[k] = ldidx(I.adj + (size_t)(back_dir(k) - 1) * I.n + node);
  T va[9], vb[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const int i = back_dir(k);
    if (nb[k] != node) va[k] = ld(F.at(i, node)), vb[k] = ld(F.at(opp(i), nb[k]));
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    const int i = back_dir(k);
    if (nb[k] != node) st<false>(F.at(i, node), vb[k]), st<false>(F.at(opp(i), nb[k]), va[k]);
  }
}
template <class T, bool AOS>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value) k_swap_idx(Fld<T, AOS> F, Idx I) {
  const uint32_t node = I.first + blockIdx.x * kBlock + threadIdx.x;
  if (node >= I.end()) return;
  swap_idx_node(F, I, node);
}


// ---------------------------------------------------------------------------
// AoS variants: the node-contiguous (local) side is staged through shared
// memory as coalesced 16-byte vectors (see aos_stage_in / aos_stage_out).
// ---------------------------------------------------------------------------
template <class T, bool RD_OPP, bool WR_OPP>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value)
    k_local_idx_aos(Fld<T, true> src, Fld<T, true> dst, uint32_t first, uint32_t n, Trt<T> op) {
  __shared__ __align__(16) T sm[kBlock * 19];
  const uint32_t n0 = first + blockIdx.x * kBlock;
  const uint32_t nrec = min((uint32_t)kBlock, n - n0);
  aos_stage_in(sm, src.p + (size_t)n0 * 19, nrec);
  __syncthreads();
  const uint32_t k = threadIdx.x;
  if (k < nrec) {
    T f[19];
#pragma unroll
    for (int i = 0; i < 19; ++i) f[i] = sm[k * 19 + (RD_OPP ? opp(i) : i)];
    collide(op, f);
#pragma unroll
    for (int i = 0; i < 19; ++i) sm[k * 19 + (WR_OPP ? opp(i) : i)] = f[i];
  }
  __syncthreads();
  aos_stage_out(dst.p + (size_t)n0 * 19, sm, nrec);
}

template <class T>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value)
    k_os_pull_idx_aos(Fld<T, true> a, Fld<T, true> b, Idx I, Trt<T> op) {
  __shared__ __align__(16) T sm[kBlock * 19];
  const uint32_t n0 = I.first + blockIdx.x * kBlock;
  const uint32_t nrec = min((uint32_t)kBlock, I.end() - n0);
  const uint32_t k = threadIdx.x;
  if (k < nrec) {
    const uint32_t node = n0 + k;
    T f[19];
    f[0] = ld(a.at(0, node));
#pragma unroll
    for (int i = 1; i < 19; ++i) {
      const int j = opp(i);
      const uint32_t src = ldidx(I.adj + (size_t)(j - 1) * I.n + node);
      f[i] = ld(src == node ? a.at(j, node) : a.at(i, src));
    }
    collide(op, f);
#pragma unroll
    for (int i = 0; i < 19; ++i) sm[k * 19 + i] = f[i];
  }
  __syncthreads();
  aos_stage_out(b.p + (size_t)n0 * 19, sm, nrec);
}

// AoS pull on an all-fluid box, nodes walked in 32 x 8 x-y tiles marching
// through a z chunk (one warp per tile row): the records a warp gathers from
// (planes z - 1 .. z + 1 of its tile and halo) stay in L1 while the chunk
// moves on, so most 8-byte gathers hit sectors already on the SM instead of
// fetching a 32-byte L2 sector each. Same per-node arithmetic and adjacency
// reads as k_os_pull_idx_aos; outputs leave per warp as 16-byte vectors.
constexpr int kIdxTX = 32, kIdxTY = 8;
template <class T, bool COLLIDE>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value)
    k_os_pull_idx_aos_tiled(Fld<T, true> a, Fld<T, true> b, Idx I, Trt<T> op, int tiles_x,
                            int tiles_y, int zc) {
  __shared__ __align__(16) T sm[kBlock * 19 + 8];
  const int ntile = tiles_x * tiles_y;
  const int tile = (int)blockIdx.x % ntile, chunk = (int)blockIdx.x / ntile;
  const int x0 = (tile % tiles_x) * kIdxTX, y = (tile / tiles_x) * kIdxTY + (int)(threadIdx.x >> 5);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x = x0 + lane, txv = min(kIdxTX, I.bx - x0);
  const int zb = chunk * zc, ze = min(I.bz, zb + zc);
  T* srow = sm + warp * (kIdxTX * 19);
  for (int z = zb; z < ze; ++z) {
    const bool live = x < I.bx && y < I.by;
    const uint32_t node = (uint32_t)x + (uint32_t)I.bx * ((uint32_t)y + (uint32_t)I.by * (uint32_t)z);
    if (live) {
      T f[19];
      f[0] = ld(a.at(0, node));
#pragma unroll
      for (int i = 1; i < 19; ++i) {
        const int j = opp(i);
        const uint32_t src = ldidx(I.adj + (size_t)(j - 1) * I.n + node);
        f[i] = ld(src == node ? a.at(j, node) : a.at(i, src));
      }
      if constexpr (COLLIDE) collide(op, f);
#pragma unroll
      for (int i = 0; i < 19; ++i) srow[lane * 19 + i] = f[i];
    }
    __syncwarp();
    if (y < I.by) {
      const uint32_t n0 = (uint32_t)x0 + (uint32_t)I.bx * ((uint32_t)y + (uint32_t)I.by * (uint32_t)z);
      T* g = b.p + (size_t)n0 * 19;
      const int n = txv * 19;
      for (int e = lane; e < n; e += 32) g[e] = srow[e];
    }
    __syncwarp();
  }
}

// The same walk for the in-place sweeps (AoS, all-fluid box): AA odd and ET
// (C4 fp64 AA 0.33 -> 0.39, ET 0.24 -> 0.29; the SWAP exchange measured
// slower tiled and keeps the block order; the TS stream uses the staged pull
// walk without collision). A block is a 32 x 8 tile of one z chunk.
enum IdxTiledKind : int { kTiledAa = 1, kTiledEt = 2, kTiledEtSw = 3 };
template <class T, int KIND>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value)
    k_idx_aos_tiled(Fld<T, true> a, Fld<T, true> b, Idx I, Trt<T> op, int tiles_x, int tiles_y,
                    int zc) {
  const int ntile = tiles_x * tiles_y;
  const int tile = (int)blockIdx.x % ntile, chunk = (int)blockIdx.x / ntile;
  const int x = (tile % tiles_x) * kIdxTX + (int)(threadIdx.x & 31);
  const int y = (tile / tiles_x) * kIdxTY + (int)(threadIdx.x >> 5);
  if (x >= I.bx || y >= I.by) return;
  const int zb = chunk * zc, ze = min(I.bz, zb + zc);
  for (int z = zb; z < ze; ++z) {
    const uint32_t node = (uint32_t)x + (uint32_t)I.bx * ((uint32_t)y + (uint32_t)I.by * (uint32_t)z);
    if constexpr (KIND == kTiledAa) aa_odd_idx_node(a, I, op, node);
    if constexpr (KIND == kTiledEt) et_idx_node<T, true, false>(a, I, op, node);
    if constexpr (KIND == kTiledEtSw) et_idx_node<T, true, true>(a, I, op, node);
  }
}

template <class T>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value)
    k_os_push_idx_aos(Fld<T, true> a, Fld<T, true> b, Idx I, Trt<T> op) {
  __shared__ __align__(16) T sm[kBlock * 19];
  const uint32_t n0 = I.first + blockIdx.x * kBlock;
  const uint32_t nrec = min((uint32_t)kBlock, I.end() - n0);
  aos_stage_in(sm, a.p + (size_t)n0 * 19, nrec);
  __syncthreads();
  const uint32_t k = threadIdx.x;
  if (k >= nrec) return;
  const uint32_t node = n0 + k;
  T f[19];
#pragma unroll
  for (int i = 0; i < 19; ++i) f[i] = sm[k * 19 + i];
  collide(op, f);
  st<false>(b.at(0, node), f[0]);
#pragma unroll
  for (int i = 1; i < 19; ++i) {
    const uint32_t nb = ldidx(I.adj + (size_t)(i - 1) * I.n + node);
    st<false>(nb == node ? b.at(opp(i), node) : b.at(i, nb), f[i]);
  }
}

// SWAP link exchange, AoS: a node's own side of its nine pairs (its back
// slots) is staged with the block's contiguous records (coalesced 16-byte
// vectors in) and only the back slots go out again, as element runs; the
// partner side (opp i, adj[i][n]) stays a scattered access. Nobody but the
// node itself writes its back slots (a partner exchange writes front slots),
// so the staged copies of the back slots are current and no front slot is
// written back.
constexpr uint32_t kBackMask = (1u << 2) | (1u << 4) | (1u << 6) | (1u << 7) | (1u << 8) |
                               (1u << 11) | (1u << 13) | (1u << 15) | (1u << 16);
template <class T>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value)
    k_swap_idx_aos(Fld<T, true> F, Idx I) {
  __shared__ __align__(16) T sm[kBlock * 19];
  const uint32_t n0 = I.first + blockIdx.x * kBlock;
  const uint32_t nrec = min((uint32_t)kBlock, I.end() - n0);
  aos_stage_in(sm, F.p + (size_t)n0 * 19, nrec);
  __syncthreads();
  const uint32_t k = threadIdx.x;
  if (k < nrec) {
    const uint32_t node = n0 + k;
    uint32_t nb[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) nb[q] = ldidx(I.adj + (size_t)(back_dir(q) - 1) * I.n + node);
    T vb[9];
#pragma unroll
    for (int q = 0; q < 9; ++q)
      if (nb[q] != node) vb[q] = ld(F.at(opp(back_dir(q)), nb[q]));
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      const int i = back_dir(q);
      if (nb[q] != node) {
        st<false>(F.at(opp(i), nb[q]), sm[k * 19 + i]);
        sm[k * 19 + i] = vb[q];
      }
    }
  }
  __syncthreads();
  T* g = F.p + (size_t)n0 * 19;
  for (uint32_t e = threadIdx.x; e < nrec * 19; e += blockDim.x)
    if ((kBackMask >> (e % 19)) & 1u) g[e] = sm[e];
}

// ET sweep, AoS, the nodes' own records staged (coalesced in). A node's own
// slots that it writes this sweep — hb(i) of every pair, or hb(j) when its
// j-link bounces — are written by nobody else, so they go out again from the
// staged copies (element runs, per-node mask); the slots hb(j) its partners
// rewrite are never written back from here.
template <class T, bool SW>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value)
    k_et_idx_aos(Fld<T, true> F, Idx I, Trt<T> op) {
  __shared__ __align__(16) T sm[kBlock * 19];
  __shared__ uint32_t wmask[kBlock];
  const uint32_t n0 = I.first + blockIdx.x * kBlock;
  const uint32_t nrec = min((uint32_t)kBlock, I.end() - n0);
  aos_stage_in(sm, F.p + (size_t)n0 * 19, nrec);
  __syncthreads();
  const uint32_t k = threadIdx.x;
  if (k < nrec) {
    const uint32_t node = n0 + k;
    T* rec = sm + k * 19;
    uint32_t rs[9];
    T f[19];
    f[0] = rec[0];
#pragma unroll
    for (int p = 0; p < 9; ++p) {
      const int i = pair_i(p), j = pair_j(p);
      rs[p] = ldidx(I.rem + (size_t)p * I.n + node);
      const uint32_t r = rs[p] & 0x7fffffffu;
      const bool db = r >= I.n;
      f[i] = rec[hb<SW>(i)];
      f[j] = ld(F.at(db ? hb<SW>(i) : hb<SW>(j), r));
    }
    collide(op, f);
    rec[0] = f[0];
    uint32_t m = 1u;
#pragma unroll
    for (int p = 0; p < 9; ++p) {
      const int i = pair_i(p), j = pair_j(p);
      const uint32_t rv = rs[p];
      const bool ub = (rv & 0x80000000u) != 0;
      const int own = ub ? hb<SW>(j) : hb<SW>(i);
      rec[own] = f[j];
      m |= 1u << own;
      st<false>(F.at(hb<SW>(j), rv & 0x7fffffffu), f[i]);
    }
    wmask[k] = m;
  }
  __syncthreads();
  T* g = F.p + (size_t)n0 * 19;
  for (uint32_t e = threadIdx.x; e < nrec * 19; e += blockDim.x) {
    const uint32_t r = e / 19, sl = e - r * 19;
    if ((wmask[r] >> sl) & 1u) g[e] = sm[e];
  }
}

// The same staged ET on an all-fluid box in the tiled walk (x-y tiles
// marching through z, k_idx_aos_tiled): each warp stages its row of 32
// records per plane (one contiguous run), so the neighbour gathers keep
// their L1 reuse and the own side is coalesced.
template <class T, bool SW>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value)
    k_et_idx_aos_tiled(Fld<T, true> F, Idx I, Trt<T> op, int tiles_x, int tiles_y, int zc) {
  __shared__ __align__(16) T sm[kBlock * 19];
  const int ntile = tiles_x * tiles_y;
  const int tile = (int)blockIdx.x % ntile, chunk = (int)blockIdx.x / ntile;
  const int lane = (int)(threadIdx.x & 31), warp = (int)(threadIdx.x >> 5);
  const int x0 = (tile % tiles_x) * kIdxTX, y = (tile / tiles_x) * kIdxTY + warp;
  const int x = x0 + lane;
  const int txv = y < I.by ? min(kIdxTX, I.bx - x0) : 0;
  const bool live = lane < txv;
  T* rec = sm + warp * (kIdxTX * 19) + lane * 19;
  T* srow = sm + warp * (kIdxTX * 19);
  const int zb = chunk * zc, ze = min(I.bz, zb + zc);
  for (int z = zb; z < ze; ++z) {
    const uint32_t n0 = (uint32_t)x0 + (uint32_t)I.bx * ((uint32_t)y + (uint32_t)I.by * (uint32_t)z);
    T* g = F.p + (size_t)n0 * 19;
    const int nel = txv * 19;
    for (int e = lane; e < nel; e += 32) srow[e] = g[e];
    __syncwarp();
    uint32_t m = 0;
    if (live) {
      const uint32_t node = n0 + (uint32_t)lane;
      uint32_t rs[9];
      T f[19];
      f[0] = rec[0];
#pragma unroll
      for (int p = 0; p < 9; ++p) {
        const int i = pair_i(p), j = pair_j(p);
        rs[p] = ldidx(I.rem + (size_t)p * I.n + node);
        const uint32_t r = rs[p] & 0x7fffffffu;
        const bool db = r >= I.n;
        f[i] = rec[hb<SW>(i)];
        f[j] = ld(F.at(db ? hb<SW>(i) : hb<SW>(j), r));
      }
      collide(op, f);
      rec[0] = f[0];
      m = 1u;
#pragma unroll
      for (int p = 0; p < 9; ++p) {
        const int i = pair_i(p), j = pair_j(p);
        const uint32_t rv = rs[p];
        const bool ub = (rv & 0x80000000u) != 0;
        const int own = ub ? hb<SW>(j) : hb<SW>(i);
        rec[own] = f[j];
        m |= 1u << own;
        st<false>(F.at(hb<SW>(j), rv & 0x7fffffffu), f[i]);
      }
    }
    __syncwarp();
    for (int e = lane; e < ((nel + 31) & ~31); e += 32) {
      const int r = e / 19, sl = e - r * 19;
      const uint32_t mr = __shfl_sync(0xffffffffu, m, r < 32 ? r : 31);
      if (e < nel && ((mr >> sl) & 1u)) g[e] = srow[e];
    }
    __syncwarp();
  }
}

// The staged SWAP exchange in the tiled walk (all-fluid boxes): each warp
// stages its row of 32 records per plane; the partners' records stay in L1
// while the tile marches through z.
template <class T>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value)
    k_swap_idx_aos_tiled(Fld<T, true> F, Idx I, int tiles_x, int tiles_y, int zc) {
  __shared__ __align__(16) T sm[kBlock * 19];
  const int ntile = tiles_x * tiles_y;
  const int tile = (int)blockIdx.x % ntile, chunk = (int)blockIdx.x / ntile;
  const int lane = (int)(threadIdx.x & 31), warp = (int)(threadIdx.x >> 5);
  const int x0 = (tile % tiles_x) * kIdxTX, y = (tile / tiles_x) * kIdxTY + warp;
  const int txv = y < I.by ? min(kIdxTX, I.bx - x0) : 0;
  const bool live = lane < txv;
  T* rec = sm + warp * (kIdxTX * 19) + lane * 19;
  T* srow = sm + warp * (kIdxTX * 19);
  const int zb = chunk * zc, ze = min(I.bz, zb + zc);
  for (int z = zb; z < ze; ++z) {
    const uint32_t n0 = (uint32_t)x0 + (uint32_t)I.bx * ((uint32_t)y + (uint32_t)I.by * (uint32_t)z);
    T* g = F.p + (size_t)n0 * 19;
    const int nel = txv * 19;
    for (int e = lane; e < nel; e += 32) srow[e] = g[e];
    __syncwarp();
    if (live) {
      const uint32_t node = n0 + (uint32_t)lane;
      uint32_t nb[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) nb[q] = ldidx(I.adj + (size_t)(back_dir(q) - 1) * I.n + node);
      T vb[9];
#pragma unroll
      for (int q = 0; q < 9; ++q)
        if (nb[q] != node) vb[q] = ld(F.at(opp(back_dir(q)), nb[q]));
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const int i = back_dir(q);
        if (nb[q] != node) {
          st<false>(F.at(opp(i), nb[q]), rec[i]);
          rec[i] = vb[q];
        }
      }
    }
    __syncwarp();
    for (int e = lane; e < nel; e += 32)
      if ((kBackMask >> (e % 19)) & 1u) g[e] = srow[e];
    __syncwarp();
  }
}

template <class T>
__global__ void __launch_bounds__(kBlock, MinBlocks<T>::value)
    k_ts_stream_idx_aos(Fld<T, true> a, Fld<T, true> b, Idx I) {
  __shared__ __align__(16) T sm[kBlock * 19];
  const uint32_t n0 = I.first + blockIdx.x * kBlock;
  const uint32_t nrec = min((uint32_t)kBlock, I.end() - n0);
  const uint32_t k = threadIdx.x;
  if (k < nrec) {
    const uint32_t node = n0 + k;
    sm[k * 19] = ld(b.at(0, node));
#pragma unroll
    for (int i = 1; i < 19; ++i) {
      const int j = opp(i);
      const uint32_t src = ldidx(I.adj + (size_t)(j - 1) * I.n + node);
      sm[k * 19 + i] = ld(src == node ? b.at(j, node) : b.at(i, src));
    }
  }
  __syncthreads();
  aos_stage_out(a.p + (size_t)n0 * 19, sm, nrec);
}

}  // namespace


// tiled walk of an all-fluid box (Idx.bx > 0) over the whole node range:
// grid and z chunk (about 6 waves of 2 resident blocks per SM)
static bool idx_tiled_grid(const Idx& I, int& tx, int& ty, int& zc, unsigned& grid) {
  if (I.bx <= 0 || I.first != 0 || I.end() != I.n) return false;
  if (const char* e = std::getenv("LBMGPU_IDX_TILED"))
    if (e[0] == '0') return false;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  tx = (I.bx + kIdxTX - 1) / kIdxTX;
  ty = (I.by + kIdxTY - 1) / kIdxTY;
  zc = std::max(1, std::min(I.bz, (int)((long long)I.bz * tx * ty / ((long long)sms * 2 * 6) + 1)));
  grid = (unsigned)(tx * ty * ((I.bz + zc - 1) / zc));
  return true;
}
template <int KIND>
static bool launch_idx_tiled(cudaStream_t st, const DField& a, const DField& b, const Idx& I,
                             const TrtHost& op) {
  int tx, ty, zc;
  unsigned g;
  if (!a.aos || !idx_tiled_grid(I, tx, ty, zc, g)) return false;
  if (a.prec == Prec::f64)
    k_idx_aos_tiled<double, KIND><<<g, kBlock, 0, st>>>(fld<double, true>(a), fld<double, true>(b), I,
                                                       cast_op<double>(op), tx, ty, zc);
  else
    k_idx_aos_tiled<float, KIND><<<g, kBlock, 0, st>>>(fld<float, true>(a), fld<float, true>(b), I,
                                                      cast_op<float>(op), tx, ty, zc);
  return true;
}

void launch_local_idx(cudaStream_t st, const DField& src, const DField& dst, uint32_t n,
                      const TrtHost& op, bool rd_opp, bool wr_opp) {
  launch_local_idx_range(st, src, dst, 0, n, op, rd_opp, wr_opp);
}

void launch_local_idx_range(cudaStream_t st, const DField& src, const DField& dst, uint32_t first,
                            uint32_t n, const TrtHost& op, bool rd_opp, bool wr_opp) {
  if (n <= first) return;
  const unsigned g = grid_for(n - first);
  if (src.aos) {
    // node records are contiguous: the streamed AoS local sweep applies
    dev::Lat L{};
    L.cell_begin = first;
    L.ncells = n;
    L.linkmask = nullptr;
    if (launch_aos_local_stream(st, src, dst, L, op, rd_opp, wr_opp, 0)) return;
    LBM_DISPATCH(src, {
      if constexpr (A) {
        auto a = fld<T, true>(src);
        auto b = fld<T, true>(dst);
        const auto o = cast_op<T>(op);
        if (!rd_opp && !wr_opp) k_local_idx_aos<T, false, false><<<g, kBlock, 0, st>>>(a, b, first, n, o);
        if (!rd_opp && wr_opp) k_local_idx_aos<T, false, true><<<g, kBlock, 0, st>>>(a, b, first, n, o);
        if (rd_opp && !wr_opp) k_local_idx_aos<T, true, false><<<g, kBlock, 0, st>>>(a, b, first, n, o);
        if (rd_opp && wr_opp) k_local_idx_aos<T, true, true><<<g, kBlock, 0, st>>>(a, b, first, n, o);
      }
    });
    return;
  }
  LBM_DISPATCH(src, {
    auto a = fld<T, A>(src);
    auto b = fld<T, A>(dst);
    const auto o = cast_op<T>(op);
    if (!rd_opp && !wr_opp) k_local_idx<T, A, false, false><<<g, kBlock, 0, st>>>(a, b, first, n, o);
    if (!rd_opp && wr_opp) k_local_idx<T, A, false, true><<<g, kBlock, 0, st>>>(a, b, first, n, o);
    if (rd_opp && !wr_opp) k_local_idx<T, A, true, false><<<g, kBlock, 0, st>>>(a, b, first, n, o);
    if (rd_opp && wr_opp) k_local_idx<T, A, true, true><<<g, kBlock, 0, st>>>(a, b, first, n, o);
  });
}

void launch_ts_stream_idx(cudaStream_t st, const DField& a, const DField& b, const Idx& I) {
  if (I.count() == 0) return;
  int tx = 0, ty = 0, zc = 0;
  unsigned g = 0;
  // fp64 AoS on an all-fluid box: the tiled gather without collision
  // (A <- gathered B; C4 0.56 -> 0.66; fp32 keeps the block order, 0.76 vs 0.73)
  if (a.aos && a.prec == Prec::f64 && idx_tiled_grid(I, tx, ty, zc, g)) {
    k_os_pull_idx_aos_tiled<double, false><<<g, kBlock, 0, st>>>(
        fld<double, true>(b), fld<double, true>(a), I, Trt<double>{}, tx, ty, zc);
    return;
  }
  if (a.aos) {
    LBM_DISPATCH(a, {
      if constexpr (A)
        k_ts_stream_idx_aos<T><<<grid_for(I.count()), kBlock, 0, st>>>(fld<T, true>(a), fld<T, true>(b), I);
    });
    return;
  }
  LBM_DISPATCH(a, {
    k_ts_stream_idx<T, A><<<grid_for(I.count()), kBlock, 0, st>>>(fld<T, A>(a), fld<T, A>(b), I);
  });
}

void launch_os_pull_idx(cudaStream_t st, const DField& a, const DField& b, const Idx& I,
                        const TrtHost& op, bool streaming, bool two_s) {
  if (I.count() == 0) return;
  if (a.aos) {
    int tx = 0, ty = 0, zc = 0;
    unsigned g = 0;
    // the tiled walk pays for fp64 (C4 0.54 -> 0.60); fp32 keeps the block order (0.68 vs 0.64)
    const bool tiled = a.prec == Prec::f64 && idx_tiled_grid(I, tx, ty, zc, g);
    LBM_DISPATCH(a, {
      if constexpr (A) {
        if (tiled) {
          k_os_pull_idx_aos_tiled<T, true><<<g, kBlock, 0, st>>>(fld<T, true>(a), fld<T, true>(b), I,
                                                                  cast_op<T>(op), tx, ty, zc);
        } else {
          k_os_pull_idx_aos<T><<<grid_for(I.count()), kBlock, 0, st>>>(fld<T, true>(a), fld<T, true>(b), I,
                                                                 cast_op<T>(op));
        }
      }
    });
    return;
  }
  LBM_DISPATCH(a, {
    auto fa = fld<T, A>(a);
    auto fb = fld<T, A>(b);
    const auto o = cast_op<T>(op);
    const unsigned g = grid_for(I.count());
    if (!streaming && !two_s) k_os_pull_idx<T, A, false, false><<<g, kBlock, 0, st>>>(fa, fb, I, o);
    if (!streaming && two_s) k_os_pull_idx<T, A, false, true><<<g, kBlock, 0, st>>>(fa, fb, I, o);
    if (streaming && !two_s) k_os_pull_idx<T, A, true, false><<<g, kBlock, 0, st>>>(fa, fb, I, o);
    if (streaming && two_s) k_os_pull_idx<T, A, true, true><<<g, kBlock, 0, st>>>(fa, fb, I, o);
  });
}

void launch_os_push_idx(cudaStream_t st, const DField& a, const DField& b, const Idx& I,
                        const TrtHost& op) {
  if (I.count() == 0) return;
  if (a.aos) {
    LBM_DISPATCH(a, {
      if constexpr (A)
        k_os_push_idx_aos<T><<<grid_for(I.count()), kBlock, 0, st>>>(fld<T, true>(a), fld<T, true>(b), I,
                                                               cast_op<T>(op));
    });
    return;
  }
  LBM_DISPATCH(a, {
    k_os_push_idx<T, A><<<grid_for(I.count()), kBlock, 0, st>>>(fld<T, A>(a), fld<T, A>(b), I,
                                                          cast_op<T>(op));
  });
}

// persistent grid of the staged-batch kernels: resident fp64 blocks
static unsigned staged_grid(uint32_t nbatch) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return std::min<uint32_t>(nbatch, (uint32_t)(sms * LBM_IDX_PF_MIN_BLOCKS));
}

// the asynchronous-gather pipeline (k_idx_ag), SoA, opt-in LBMGPU_IDX_AG=1:
// measured slower than the register gathers on C2 (AA odd fp64 0.88 -> 0.80,
// fp32 0.94 -> 0.87; ET fp64 0.74 -> 0.74, fp32 0.81 -> 0.66)
static bool idx_ag_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("LBMGPU_IDX_AG");
    return e && e[0] == '1';
  }();
  return on;
}
template <class T, bool ET, bool SW, bool VEC>
static void launch_ag_t(cudaStream_t st, const DField& f, const Idx& I, const TrtHost& op) {
  constexpr size_t bytes = ag_smem_bytes<ET ? 9 : 18, T>();
  static int set_dev = -1;  // the attribute is per device
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (set_dev != dev) {
    cudaFuncSetAttribute(k_idx_ag<T, ET, SW, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    set_dev = dev;
  }
  const uint32_t nbatch = (I.count() + kAgB - 1) / kAgB;
  const unsigned g = std::min<uint32_t>(nbatch, (uint32_t)(sms * AgCfg<T>::kBlocks));
  k_idx_ag<T, ET, SW, VEC><<<g, kAgB, bytes, st>>>(fld<T, false>(f), I, cast_op<T>(op), nbatch);
}
template <bool ET, bool SW>
static bool launch_ag(cudaStream_t st, const DField& f, const Idx& I, const TrtHost& op) {
  if (f.aos || !idx_ag_enabled()) return false;
  const bool vec = I.n % 4 == 0 && I.first % 4 == 0;
  if (f.prec == Prec::f64) {
    if (vec) launch_ag_t<double, ET, SW, true>(st, f, I, op);
    else launch_ag_t<double, ET, SW, false>(st, f, I, op);
  } else {
    if (vec) launch_ag_t<float, ET, SW, true>(st, f, I, op);
    else launch_ag_t<float, ET, SW, false>(st, f, I, op);
  }
  return true;
}

void launch_aa_odd_idx(cudaStream_t st, const DField& f, const Idx& I, const TrtHost& op) {
  if (I.count() == 0) return;
  if (launch_ag<false, false>(st, f, I, op)) return;
  if (LBM_IDX_PP32 && !f.aos && f.prec == Prec::f32) {
    const uint32_t nbatch = (I.count() + kBlock - 1) / kBlock;
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned g = std::min<uint32_t>(nbatch, (uint32_t)(sms * LBM_IDX_PP32_BLOCKS));
    constexpr int bytes = kPpBytes<18>;
    cudaFuncSetAttribute(k_aa_odd_idx_pp<float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    cudaFuncSetAttribute(k_aa_odd_idx_pp<float, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (I.n % 4 == 0 && I.first % 4 == 0)
      k_aa_odd_idx_pp<float, true><<<g, kBlock, bytes, st>>>(fld<float, false>(f), I, cast_op<float>(op), nbatch);
    else
      k_aa_odd_idx_pp<float, false><<<g, kBlock, bytes, st>>>(fld<float, false>(f), I, cast_op<float>(op), nbatch);
    return;
  }
  if (!f.aos && f.prec == Prec::f64) {  // fp32 spills at its register budget
    const uint32_t nbatch = (I.count() + kBlock - 1) / kBlock;
    const unsigned g = staged_grid(nbatch);
    const auto F = fld<double, false>(f);
    const auto o = cast_op<double>(op);
    const bool vec = I.n % 4 == 0 && I.first % 4 == 0;
    if (LBM_IDX_PP) {
      constexpr int bytes = kPpBytes<18>;
      static int set_dev = -1;  // the attribute is per device
      int dev = 0;
      cudaGetDevice(&dev);
      if (set_dev != dev) {
        cudaFuncSetAttribute(k_aa_odd_idx_pp<double, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        cudaFuncSetAttribute(k_aa_odd_idx_pp<double, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        set_dev = dev;
      }
      if (vec) k_aa_odd_idx_pp<double, true><<<g, kBlock, bytes, st>>>(F, I, o, nbatch);
      else k_aa_odd_idx_pp<double, false><<<g, kBlock, bytes, st>>>(F, I, o, nbatch);
      return;
    }
    if (vec)
      k_aa_odd_idx_pf<double, true><<<g, kBlock, 0, st>>>(F, I, o, nbatch);
    else
      k_aa_odd_idx_pf<double, false><<<g, kBlock, 0, st>>>(F, I, o, nbatch);
    return;
  }
  if (I.count() == 0) return;
  if (launch_idx_tiled<kTiledAa>(st, f, f, I, op)) return;
  LBM_DISPATCH(f, {
    k_aa_odd_idx<T, A><<<grid_for(I.count()), kBlock, 0, st>>>(fld_sel<T, A, kAaIdxTab<T>>(f), I,
                                                              cast_op<T>(op));
  });
}

// ET on AoS with the own records staged (k_et_idx_aos), also on all-fluid
// boxes instead of the tiled walk; LBMGPU_IDX_ET_STAGED=0 restores the
// per-thread kernels
static bool et_aos_staged() {
  static const bool on = [] {
    const char* e = std::getenv("LBMGPU_IDX_ET_STAGED");
    return !(e && e[0] == '0');
  }();
  return on;
}

void launch_et_idx(cudaStream_t st, const DField& f, const Idx& I, const TrtHost& op,
                   const EtBase& base) {
  if (I.count() == 0) return;
  if (!(f.aos && et_aos_staged()) &&
      (base.swapped() ? launch_idx_tiled<kTiledEtSw>(st, f, f, I, op)
                      : launch_idx_tiled<kTiledEt>(st, f, f, I, op)))
    return;
  if (base.swapped() ? launch_ag<true, true>(st, f, I, op) : launch_ag<true, false>(st, f, I, op))
    return;
  if (LBM_IDX_PP32 && !f.aos && f.prec == Prec::f32) {
    const uint32_t nbatch = (I.count() + kBlock - 1) / kBlock;
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned g = std::min<uint32_t>(nbatch, (uint32_t)(sms * LBM_IDX_PP32_BLOCKS));
    constexpr int bytes = kPpBytes<9>;
    const auto F = fld<float, false>(f);
    const auto o = cast_op<float>(op);
    const bool vec = I.n % 4 == 0 && I.first % 4 == 0, sw = base.swapped();
    if (vec && sw) k_et_idx_pp<float, true, true><<<g, kBlock, bytes, st>>>(F, I, o, nbatch);
    if (vec && !sw) k_et_idx_pp<float, false, true><<<g, kBlock, bytes, st>>>(F, I, o, nbatch);
    if (!vec && sw) k_et_idx_pp<float, true, false><<<g, kBlock, bytes, st>>>(F, I, o, nbatch);
    if (!vec && !sw) k_et_idx_pp<float, false, false><<<g, kBlock, bytes, st>>>(F, I, o, nbatch);
    return;
  }
  if (!f.aos && f.prec == Prec::f64) {
    const uint32_t nbatch = (I.count() + kBlock - 1) / kBlock;
    const unsigned g = staged_grid(nbatch);
    const auto F = fld<double, false>(f);
    const auto o = cast_op<double>(op);
    const bool vec = I.n % 4 == 0 && I.first % 4 == 0, sw = base.swapped();
    if (LBM_IDX_PP) {
      constexpr int bytes = kPpBytes<9>;
      if (vec && sw) k_et_idx_pp<double, true, true><<<g, kBlock, bytes, st>>>(F, I, o, nbatch);
      if (vec && !sw) k_et_idx_pp<double, false, true><<<g, kBlock, bytes, st>>>(F, I, o, nbatch);
      if (!vec && sw) k_et_idx_pp<double, true, false><<<g, kBlock, bytes, st>>>(F, I, o, nbatch);
      if (!vec && !sw) k_et_idx_pp<double, false, false><<<g, kBlock, bytes, st>>>(F, I, o, nbatch);
      return;
    }
    if (vec && sw) k_et_idx_pf<double, true, true><<<g, kBlock, 0, st>>>(F, I, o, nbatch);
    if (vec && !sw) k_et_idx_pf<double, false, true><<<g, kBlock, 0, st>>>(F, I, o, nbatch);
    if (!vec && sw) k_et_idx_pf<double, true, false><<<g, kBlock, 0, st>>>(F, I, o, nbatch);
    if (!vec && !sw) k_et_idx_pf<double, false, false><<<g, kBlock, 0, st>>>(F, I, o, nbatch);
    return;
  }
  if (f.aos && et_aos_staged()) {
    const bool sw = base.swapped();
    int tx, ty, zc;
    unsigned gt;
    if (idx_tiled_grid(I, tx, ty, zc, gt)) {
      if (f.prec == Prec::f64) {
        if (sw) k_et_idx_aos_tiled<double, true><<<gt, kBlock, 0, st>>>(fld<double, true>(f), I, cast_op<double>(op), tx, ty, zc);
        else k_et_idx_aos_tiled<double, false><<<gt, kBlock, 0, st>>>(fld<double, true>(f), I, cast_op<double>(op), tx, ty, zc);
      } else {
        if (sw) k_et_idx_aos_tiled<float, true><<<gt, kBlock, 0, st>>>(fld<float, true>(f), I, cast_op<float>(op), tx, ty, zc);
        else k_et_idx_aos_tiled<float, false><<<gt, kBlock, 0, st>>>(fld<float, true>(f), I, cast_op<float>(op), tx, ty, zc);
      }
      return;
    }
    if (f.prec == Prec::f64) {
      if (sw) k_et_idx_aos<double, true><<<grid_for(I.count()), kBlock, 0, st>>>(fld<double, true>(f), I, cast_op<double>(op));
      else k_et_idx_aos<double, false><<<grid_for(I.count()), kBlock, 0, st>>>(fld<double, true>(f), I, cast_op<double>(op));
    } else {
      if (sw) k_et_idx_aos<float, true><<<grid_for(I.count()), kBlock, 0, st>>>(fld<float, true>(f), I, cast_op<float>(op));
      else k_et_idx_aos<float, false><<<grid_for(I.count()), kBlock, 0, st>>>(fld<float, true>(f), I, cast_op<float>(op));
    }
    return;
  }
  LBM_DISPATCH(f, {
    if (base.swapped())
      k_et_idx<T, A, true><<<grid_for(I.count()), kBlock, 0, st>>>(fld<T, A>(f), I, cast_op<T>(op));
    else
      k_et_idx<T, A, false><<<grid_for(I.count()), kBlock, 0, st>>>(fld<T, A>(f), I, cast_op<T>(op));
  });
}

void launch_swap_idx(cudaStream_t st, const DField& f, const Idx& I) {
  if (I.count() == 0) return;
  if (f.aos) {
    int tx, ty, zc;
    unsigned gt;
    if (idx_tiled_grid(I, tx, ty, zc, gt)) {
      if (f.prec == Prec::f64)
        k_swap_idx_aos_tiled<double><<<gt, kBlock, 0, st>>>(fld<double, true>(f), I, tx, ty, zc);
      else
        k_swap_idx_aos_tiled<float><<<gt, kBlock, 0, st>>>(fld<float, true>(f), I, tx, ty, zc);
      return;
    }
    if (f.prec == Prec::f64)
      k_swap_idx_aos<double><<<grid_for(I.count()), kBlock, 0, st>>>(fld<double, true>(f), I);
    else
      k_swap_idx_aos<float><<<grid_for(I.count()), kBlock, 0, st>>>(fld<float, true>(f), I);
    return;
  }
  LBM_DISPATCH(f, { k_swap_idx<T, A><<<grid_for(I.count()), kBlock, 0, st>>>(fld<T, A>(f), I); });
}

}  // namespace lbmgpu
