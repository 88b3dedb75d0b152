// Host-side launchers for the sm_100a kernels (internal to liblbmgpu.so).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "lbm_device.cuh"

namespace lbmgpu {

enum class Prec { f64 = 8, f32 = 4 };

// A PDF field in device memory: SoA (direction planes of `stride` elements)
// or AoS (node-major records of 19), fp64 or fp32.
struct DField {
  void* p = nullptr;
  long long stride = 0;
  bool aos = false;
  Prec prec = Prec::f64;
  double shift = 0.0;  // rho0 of the stepper: fp32 slots hold f_i - w_i shift (kShifted)
};

// TrtOperator coefficients in double (cast per launch for fp32)
struct TrtHost {
  double lambda_e, le_half, lo_half, w0;
  double w2[9], f3w[9];
  double rho0;  // fp32 fields store f_i - w_i rho0 (lbm_device.cuh kShifted)
};

struct EtBase {
  int8_t b[20];
  // the table is the identity or all pairs swapped (see dev::hb)
  bool swapped() const {
    const bool sw = b[1] == 2;
    for (int i = 1; i < 19; ++i)
      if (b[i] != (sw ? dev::opp(i) : i)) throw_bad_handles();
    return sw;
  }
  [[noreturn]] static void throw_bad_handles();
};

constexpr int kBlock = 256;
// Resident 256-thread blocks per SM that the register budget must allow
// (__launch_bounds__ min blocks): fp64 kernels 2 (<= 128 registers, no
// spills), fp32 kernels 4 (<= 64). Measured on B200: tools/sweep.py c1,
// profiles/r01_variants.md.
#ifndef LBM_MIN_BLOCKS_F64
#define LBM_MIN_BLOCKS_F64 2
#endif
#ifndef LBM_MIN_BLOCKS_F32
#define LBM_MIN_BLOCKS_F32 4
#endif
template <class T>
struct MinBlocks {
  static constexpr int value = sizeof(T) == 8 ? LBM_MIN_BLOCKS_F64 : LBM_MIN_BLOCKS_F32;
};
// SoA kernels of the direct path (and the indirect OS pull) under their own
// budgets, measured per kernel (tools/sweep.py, profiles/r01_variants.md):
// fp64 at 3 blocks (<= 85 registers; C1 AA 1.01 -> 1.04, ET 0.95 -> 1.02, CG
// 0.98 -> 1.02, OS push 1.00 -> 1.03 of the roofline, a few spilled values
// land in L1); the indirect OS push / AA / ET lose with it and keep 2. fp32
// OS pull/push and ET at 5 blocks (<= 51 registers; C1 OS pull 0.99 -> 1.02,
// ET 0.89 -> 0.91). AoS per-thread kernels keep MinBlocks.
#ifndef LBM_SOA_MIN_BLOCKS_F64
#define LBM_SOA_MIN_BLOCKS_F64 3
#endif
#ifndef LBM_OS_MIN_BLOCKS_F32
#define LBM_OS_MIN_BLOCKS_F32 5
#endif
#ifndef LBM_ET_MIN_BLOCKS_F32
#define LBM_ET_MIN_BLOCKS_F32 6
#endif
// fp32 CG push at 6 (C1 0.92 -> 0.94; 4: 0.91)
#ifndef LBM_CG_MIN_BLOCKS_F32
#define LBM_CG_MIN_BLOCKS_F32 6
#endif
template <class T, bool AOS>
struct SoaMinBlocks {
  static constexpr int value =
      sizeof(T) == 8 && !AOS ? LBM_SOA_MIN_BLOCKS_F64 : MinBlocks<T>::value;
};
template <class T, bool AOS>
struct OsMinBlocks {
  static constexpr int value =
      sizeof(T) == 4 && !AOS ? LBM_OS_MIN_BLOCKS_F32 : SoaMinBlocks<T, AOS>::value;
};
template <class T, bool AOS>
struct CgMinBlocks {
  static constexpr int value =
      sizeof(T) == 4 && !AOS ? LBM_CG_MIN_BLOCKS_F32 : SoaMinBlocks<T, AOS>::value;
};
template <class T, bool AOS = false>
struct EtMinBlocks {
  static constexpr int value =
      sizeof(T) == 4 && !AOS ? LBM_ET_MIN_BLOCKS_F32 : SoaMinBlocks<T, AOS>::value;
};

// ---- direct (full-grid) addressing -----------------------------------------
// collide every fluid cell locally: dst[wr(i)][s] = collide(src[rd(i)][s])
void launch_local(cudaStream_t st, const DField& src, const DField& dst, const dev::Lat& L,
                  const TrtHost& op, bool rd_opp, bool wr_opp);
// TS streaming sweep: A[i][s] = B[i][s - c_i] (bounce: B[opp i][s])
void launch_ts_stream(cudaStream_t st, const DField& a, const DField& b, const dev::Lat& L);
// OS / OSNT pull: gather from a, collide, store local into b
void launch_os_pull(cudaStream_t st, const DField& a, const DField& b, const dev::Lat& L,
                    const TrtHost& op, bool streaming, bool two_s);
// OS push: read local from a, collide, scatter into b
void launch_os_push(cudaStream_t st, const DField& a, const DField& b, const dev::Lat& L,
                    const TrtHost& op);
// AA-pattern odd sweep (the even sweep is launch_local(rd natural, wr opposed))
void launch_aa_odd(cudaStream_t st, const DField& f, const dev::Lat& L, const TrtHost& op);
// one slab face plane of the AA odd sweep; the slots crossing the face
// (c_z = dz) are addressed in peer memory: remote[k] = base of the neighbour's
// face-plane slot k, indexed like the local ghost plane at ghost_base
void launch_aa_odd_face(cudaStream_t st, const DField& f, const dev::Lat& L, const TrtHost& op,
                        void* const remote[19], int dz, uint32_t ghost_base);
// Esoteric twist sweep with the current handle table
void launch_et(cudaStream_t st, const DField& f, const dev::Lat& L, const TrtHost& op,
               const EtBase& base);
// SWAP link exchange: mode 0 all links, 1 only non-wrapped, 2 only wrapped
void launch_swap(cudaStream_t st, const DField& f, const dev::Lat& L, int mode);
// SWAP collisions + non-wrapped link exchanges in one launch (SoA, storage =
// cells; kernels_swap.cu). rows of a tile (0: not applicable). sync = 1 +
// ntiles zeroed words per stepper; epoch >= 1 increments per launch.
int swap_fused_rows(const dev::Lat& L);
bool launch_swap_fused(cudaStream_t st, const DField& f, const dev::Lat& L, const TrtHost& op,
                       bool push, unsigned long long* sync, unsigned long long epoch);
// single-pass SWAP with face buffers (SoA direct; kernels_swap1.cu): whether
// the lattice qualifies, the face-buffer length per parity (elements), one
// sweep (hcur: this sweep's buffer, hprev: the last sweep's), and the
// field <-> buffer transfers (fill: field -> hprev after a load; flush (push):
// latest buffer -> field before an extraction)
bool swap1_ok(const DField& f, const dev::Lat& L, bool push);
size_t swap1_face_elems(const DField& f, const dev::Lat& L, bool push);
void launch_swap1(cudaStream_t st, const DField& f, const dev::Lat& L, const TrtHost& op, bool push,
                  void* hcur, const void* hprev);
void launch_swap1_faces(cudaStream_t st, const DField& f, const dev::Lat& L, bool push, bool fill,
                        void* h);
// AA pattern on AoS records with face buffers (kernels_aos_fb.cu): whether
// the lattice qualifies, the face-buffer length (elements), one sweep (even
// or odd), and the buffer <-> record transfers (fill after a load, flush
// before an extraction)
bool aa_fb_ok(const DField& f, const dev::Lat& L);
size_t aa_fb_face_elems(const DField& f, const dev::Lat& L);
void launch_aa_fb(cudaStream_t st, const DField& f, const dev::Lat& L, const TrtHost& op, bool odd,
                  void* h);
void launch_aa_fb_faces(cudaStream_t st, const DField& f, const dev::Lat& L, bool fill, void* h);
void launch_swap_list(cudaStream_t st, const DField& f, const long long* a, const long long* b,
                      const int8_t* dir, long long count);
// CG as a plane-group push launch: read at the cell's storage index, write at
// + delta (the other origin); copy of 5 slot planes src -> dst (seam fix-up)
// launched with programmatic dependent launch: early = a later group of the
// same sweep (loads and collision overlap the previous group's tail, stores
// wait for it); otherwise the kernel waits for its predecessors before loading
void launch_cg_push(cudaStream_t st, const DField& f, const dev::Lat& L, const TrtHost& op,
                    int delta, bool early = false);
void launch_plane_copy(cudaStream_t st, const DField& f, const dev::Lat& L, const int* dirs,
                       uint32_t src, uint32_t dst, int writer_z);
// AoS window kernels (kernels_aos.cu): tile + halo planes staged in shared
// memory. Returns false (nothing launched) where they do not apply.
enum WinModeId : int {
  kWinModePull = 0,
  kWinModeStream = 1,
  kWinModePush = 2,
  kWinModeAaOdd = 3,
  kWinModeSwap = 4,  // SWAP link exchange, non-wrapped links (k_swap mode 1)
  kWinModeEt = 5,    // ET sweep, identity handle table
  kWinModeEtSw = 6   // ET sweep, all pairs swapped
};
bool launch_aos_window(cudaStream_t st, int mode, const DField& src, const DField& dst,
                       const dev::Lat& L, const TrtHost& op);
// AoS OS-push window over planes [z0, z1) from src to dst (CG plane groups);
// wlo / whi: saved copies of the planes a periodic z wrap reads (or null)
bool aos_push_planes_ok(const DField& src, const dev::Lat& L);
void launch_aos_push_planes(cudaStream_t st, const DField& src, const DField& dst,
                            const dev::Lat& L, const TrtHost& op, int z0, int z1,
                            const void* wlo, const void* whi);
// local AoS sweep over contiguous records (storage index = cell + soff)
bool launch_aos_local_stream(cudaStream_t st, const DField& src, const DField& dst,
                             const dev::Lat& L, const TrtHost& op, bool rd_opp, bool wr_opp,
                             uint32_t soff);
// ---- indirect (IDX) addressing ---------------------------------------------
struct Idx {
  const uint32_t* adj;  // transposed [18][n]: adj[(i-1)*n + node]
  const uint32_t* rem;  // ET: transposed [9][n] (bit 31 = j-link bounces)
  uint32_t n;           // nodes in storage (the stride of adj / rem)
  uint32_t first = 0;   // sweeps update nodes [first, min(last, n)) (z-slabs:
  uint32_t last = ~0u;  // the slab's own nodes, not its ghost planes)
  // all-fluid box (node = x + nx (y + ny z)): the AoS kernels may walk the
  // nodes in x-y tiles marching through z (0 = not available)
  int bx = 0, by = 0, bz = 0;
  __host__ __device__ uint32_t end() const { return last < n ? last : n; }
  __host__ __device__ uint32_t count() const { return end() > first ? end() - first : 0; }
};
void launch_local_idx(cudaStream_t st, const DField& src, const DField& dst, uint32_t n,
                      const TrtHost& op, bool rd_opp, bool wr_opp);
// the same over nodes [first, last)
void launch_local_idx_range(cudaStream_t st, const DField& src, const DField& dst, uint32_t first,
                            uint32_t last, const TrtHost& op, bool rd_opp, bool wr_opp);
void launch_ts_stream_idx(cudaStream_t st, const DField& a, const DField& b, const Idx& I);
void launch_os_pull_idx(cudaStream_t st, const DField& a, const DField& b, const Idx& I,
                        const TrtHost& op, bool streaming, bool two_s);
void launch_os_push_idx(cudaStream_t st, const DField& a, const DField& b, const Idx& I,
                        const TrtHost& op);
void launch_aa_odd_idx(cudaStream_t st, const DField& f, const Idx& I, const TrtHost& op);
void launch_et_idx(cudaStream_t st, const DField& f, const Idx& I, const TrtHost& op,
                   const EtBase& base);
void launch_swap_idx(cudaStream_t st, const DField& f, const Idx& I);

// ---- canonical snapshot <-> scheme storage ---------------------------------
enum ExMode : int {
  kExNatural = 0,   // o[i] = F[i][s]
  kExOpposed = 1,   // o[i] = F[opp i][s]
  kExGather = 2,    // o[i] = F[i][s - c_i] (bounce F[opp i][s]): stream the stored post-collision state
  kExAaOdd = 3,     // o[i] = F[opp i][s - c_i] (bounce F[i][s])
  kExEt = 4,        // twisted handles
};
enum LdSource : int { kSrcBuffer = 0, kSrcRest = 1, kSrcTaylorGreen = 2, kSrcRandom = 3 };
struct InitSpec {
  int source = kSrcBuffer;
  double rho0 = 1.0;
  unsigned long long seed = 0;
  double u0 = 0.01, drho = 1e-3, noise = 1e-4;
  int gnx = 0, gny = 0, gnz = 0;  // global box for Taylor-Green phase
  int z0 = 0;                     // global z of local plane 0 (slabs)
  // Taylor-Green phase table on the device: sin/cos of (2 pi) x / gnx for
  // x < gnx, then y, then z ([sx | cx | sy | cy | sz | cz]), computed on the
  // host with libm (Stepper::init) so the field equals the oracle's bit for bit
  const double* trig = nullptr;
};
// host side of the table above (runtime.h)
void taylor_green_table(int gnx, int gny, int gnz, double* out);
// nodes [n0, n0+count) of the canonical order; buf[(n-n0)*19 + i] (fp64)
void launch_extract(cudaStream_t st, const DField& f, const dev::Lat& L,
                    const uint32_t* cell_of_node, uint32_t n0, uint32_t count, int mode,
                    const EtBase& base, double* buf);
void launch_load(cudaStream_t st, const DField& f, const dev::Lat& L,
                 const uint32_t* cell_of_node, uint32_t n0, uint32_t count, int mode,
                 const double* buf, const InitSpec& init);
void launch_extract_idx(cudaStream_t st, const DField& f, const Idx& I, uint32_t n0,
                        uint32_t count, int mode, const EtBase& base, double* buf);
void launch_load_idx(cudaStream_t st, const DField& f, const Idx& I, const dev::Lat& Lcells,
                     const uint32_t* cell_of_node, uint32_t n0, uint32_t count, int mode,
                     const double* buf, const InitSpec& init);
// z-slab phase 1 into an owner plane: dst[q] = src[q] unless the owner node's
// link `dir` bounces (then the owner wrote that slot itself). Indirect: node
// first + q, bounce = adj[dir-1][node] == node; direct: cell q of an nx*ny
// plane against the x/y walls.
void launch_slab_merge(cudaStream_t st, Prec prec, void* dst, const void* src, uint32_t count,
                       int dir, uint32_t first, const uint32_t* adj, uint32_t n, int nx, int ny,
                       bool wx, bool wy);
// mismatches of the shared-reciprocal division against __ddiv_rn (synchronous)
uint64_t selftest_division(uint64_t n, uint64_t seed);
// best-of-reps GB/s (read + write bytes) of a 16-byte streaming copy / in-place update
double stream_bandwidth(uint64_t bytes, int inplace, int reps);
void launch_fill(cudaStream_t st, const DField& f, long long count, double v);

// ---- geometry / IDX construction -------------------------------------------
// exclusive scan of (mask != 0) over ncells -> node_of (~0u for solids),
// cell_of_node; returns the fluid count (synchronises)
uint64_t build_node_maps(cudaStream_t st, const uint8_t* mask, uint64_t ncells,
                         uint32_t* node_of, uint32_t* cell_of_node, uint32_t* scratch,
                         uint64_t scratch_elems);
uint64_t scan_scratch_elems(uint64_t n);
void launch_linkmask(cudaStream_t st, const uint8_t* mask, const dev::Lat& L, uint32_t* out);
void launch_adjacency(cudaStream_t st, const uint8_t* mask, const dev::Lat& L,
                      const uint32_t* node_of, const uint32_t* cell_of_node, uint32_t n,
                      uint32_t* adjT);
// ET remote table: returns max mailbox count (synchronises)
uint32_t build_et_rem(cudaStream_t st, const uint32_t* adjT, uint32_t n, uint32_t* remT,
                      uint32_t* scratch, uint64_t scratch_elems);
void launch_transpose_u32(cudaStream_t st, const uint32_t* inT, uint32_t rows, uint32_t n,
                          uint32_t* out_nodemajor);

}  // namespace lbmgpu
