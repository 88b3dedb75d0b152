/*
 * lbmgpu.h — C ABI of the B200-native D3Q19 collide+propagate library
 * (liblbmgpu.so, hand-written sm_100a CUDA).
 *
 * This is the drop-in boundary below the reference's C++ lattice/propagation
 * API (lbmlab, /root/reference/proj; p/ below). Each entry point names the
 * reference interface it replaces. Plain pointers and sizes only; no CUDA or
 * torch types. The C++ mirror of the reference API (include/lbmgpu/lbmgpu.hpp)
 * and the Python mirror (paper_1111_0922_b200) are thin layers over it.
 *
 * Errors: every function returns an lbmgpu_status; on failure
 * lbmgpu_last_error() holds the message (thread-local). Kinds mirror the
 * reference's exception types (std::invalid_argument, std::runtime_error,
 * std::domain_error, std::bad_alloc) plus CUDA failures, and the messages are
 * the reference's texts where one exists.
 */
#ifndef LBMGPU_H
#define LBMGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LBMGPU_OK = 0,
  LBMGPU_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  LBMGPU_RUNTIME_ERROR = 2,    /* std::runtime_error */
  LBMGPU_DOMAIN_ERROR = 3,     /* std::domain_error */
  LBMGPU_BAD_ALLOC = 4,        /* std::bad_alloc / cudaErrorMemoryAllocation */
  LBMGPU_CUDA_ERROR = 5        /* any other CUDA runtime failure */
} lbmgpu_status;

/* lbmlab::SchemeId order (p/include/lbmlab/stepper.hpp:15-26) */
typedef enum {
  LBMGPU_TS = 0,
  LBMGPU_OS_PUSH = 1,
  LBMGPU_OS_PULL = 2,
  LBMGPU_OSNT_PULL_1S = 3,
  LBMGPU_OSNT_PULL_2S = 4,
  LBMGPU_CG = 5,
  LBMGPU_SWAP_PUSH = 6,
  LBMGPU_SWAP_PULL = 7,
  LBMGPU_AAP = 8,
  LBMGPU_ET = 9
} lbmgpu_scheme;

/* lbmlab::Addressing (stepper.hpp:31) */
typedef enum { LBMGPU_DIRECT = 0, LBMGPU_INDIRECT = 1 } lbmgpu_addressing;
/* storage layout of the PDF field (new: the reference is SoA-only,
 * p/src/stepper_common.hpp:17-44) */
typedef enum { LBMGPU_SOA = 0, LBMGPU_AOS = 1 } lbmgpu_layout;
/* lbmlab::LayoutPhase order (stepper.hpp:41-48) */
typedef enum {
  LBMGPU_NATURAL = 0,
  LBMGPU_OPPOSED = 1,
  LBMGPU_SHIFTED_EVEN = 2,
  LBMGPU_SHIFTED_ODD = 3,
  LBMGPU_TWISTED = 4,
  LBMGPU_SWAP_PARTIAL = 5
} lbmgpu_phase;

/* lbmlab::GridGeometry (p/include/lbmlab/geometry.hpp:19-38): x-fastest
 * mask, 1 = fluid (NULL = all fluid); axis_policy 0 periodic, 1 wall. The
 * stepper copies what it needs; the caller keeps ownership. */
typedef struct {
  int32_t nx, ny, nz;
  uint8_t axis_policy[3];
  const uint8_t* mask;
} lbmgpu_geometry;

/* Relaxation rates and force. The C++ mirror fills lambda_odd with the
 * reference's lambda_odd(FlowParams) (p/src/collision.cpp:8-11) so both
 * sides use the same double — TrtOperator's explicit-rate constructor
 * (collision.hpp:46-47). */
typedef struct {
  double lambda_even;
  double lambda_odd;
  double body_force[3];
  double rho0;
} lbmgpu_flow;

/* lbmlab::StepperOptions (stepper.hpp:55-64) + the GPU selectors. */
typedef struct {
  int32_t scheme;              /* lbmgpu_scheme */
  int32_t addressing;          /* lbmgpu_addressing */
  int32_t layout;              /* lbmgpu_layout */
  int32_t precision;           /* 8 = fp64 (reference), 4 = fp32 */
  int32_t device;              /* CUDA device ordinal */
  int32_t workers;             /* reference CPU threads: validated (>= 0), unused */
  int32_t chunk_length;        /* OSNT staging block: validated (>= 1); no effect on results */
  int32_t streaming_stores;    /* OSNT: st.global.cs streaming stores */
  int32_t swap_deferred_fixup; /* SWAP push: defer the periodic-seam exchange */
  int32_t zero_collision;      /* identity collision (property tests) */
  int32_t extensions;          /* 1: also allow TS/SWAP indirect (no reference kernel) */
  /* z-slab of a multi-GPU decomposition (AA direct only): owned global planes
   * [z_begin, z_end) of a box of nz planes; z_end == 0 means the whole box */
  int32_t z_begin, z_end;
} lbmgpu_options;

typedef struct lbmgpu_stepper lbmgpu_stepper;

/* Fills *o with the reference defaults (stepper.hpp:55-64): AAP direct SoA
 * fp64, device 0, workers 1, chunk_length 150, streaming stores on. */
void lbmgpu_default_options(lbmgpu_options* o);

/* create_stepper (p/src/stepper.cpp:155-180). Unsupported pairs fail with
 * LBMGPU_INVALID_ARGUMENT "kernel not implemented; traffic model only". The
 * field starts at rest equilibrium w_i*rho0 like every reference stepper. */
int lbmgpu_create(const lbmgpu_geometry* g, const lbmgpu_flow* p, const lbmgpu_options* o,
                  lbmgpu_stepper** out);
int lbmgpu_destroy(lbmgpu_stepper* h);

/* Stepper::step() (stepper.hpp:74), n times, enqueued asynchronously on the
 * stepper's CUDA stream. */
int lbmgpu_step(lbmgpu_stepper* h, int64_t n);
int lbmgpu_synchronize(lbmgpu_stepper* h);
/* n steps bracketed by CUDA events recorded on the stepper's own (launching)
 * stream, synchronised on both sides; *ms = device time of the n steps */
int lbmgpu_step_timed(lbmgpu_stepper* h, int64_t n, double* ms);

/* Stepper::extract_natural / load_natural (stepper.hpp:75-76): canonical
 * snapshot, fluid nodes x-fastest, out[n*19 + i], fp64, caller-owned host
 * memory of node_count*19 doubles. Both synchronise; load resets t to 0. */
int lbmgpu_extract_natural(lbmgpu_stepper* h, double* out);
int lbmgpu_load_natural(lbmgpu_stepper* h, const double* in);
/* nodes [first, first + count) of the canonical snapshot only (count*19
 * doubles, host or device memory): extract a large lattice in pieces */
int lbmgpu_extract_natural_range(lbmgpu_stepper* h, uint64_t first, uint64_t count, double* out,
                                 int32_t out_on_device);
/* the same with a device pointer (node_count*19 doubles on the stepper's device) */
int lbmgpu_extract_natural_device(lbmgpu_stepper* h, double* dev_out);
int lbmgpu_load_natural_device(lbmgpu_stepper* h, const double* dev_in);

/* Device-side initial fields (t reset to 0), keyed by GLOBAL cell index so
 * z-slabs reproduce the single-domain field:
 *   kind 0: rest            w_i rho0
 *   kind 1: Taylor-Green    equilibrium(rho0 + drho U, u0 (sin X cos Y cos Z,
 *                           -cos X sin Y cos Z, 0)) + noise U, X = 2 pi x/nx
 *   kind 2: random          w_i rho0 (0.9 + 0.2 U01)
 * U: splitmix64(seed, 20*cell + i) uniform in [-1, 1). */
int lbmgpu_init_field(lbmgpu_stepper* h, int32_t kind, uint64_t seed, double u0, double drho,
                      double noise);

int lbmgpu_layout_phase(lbmgpu_stepper* h, int32_t* phase);     /* Stepper::layout_phase */
int lbmgpu_exchange_opposite_handles(lbmgpu_stepper* h, int32_t* had_handles);
int lbmgpu_time_step(lbmgpu_stepper* h, int64_t* t);            /* Stepper::time_step */
int lbmgpu_node_count(lbmgpu_stepper* h, uint64_t* n);          /* Stepper::node_count */
/* device bytes of the PDF field(s) + index tables */
int lbmgpu_storage_bytes(lbmgpu_stepper* h, uint64_t* pdf_bytes, uint64_t* idx_bytes);
/* the stepper's cudaStream_t, for event timing on the launching stream */
int lbmgpu_stream(lbmgpu_stepper* h, void** cuda_stream);
/* kernels enqueued by one step() at the current parity */
int lbmgpu_launches_per_step(lbmgpu_stepper* h, int32_t* launches);

/* ---- harness (p/src/bench.cpp) ---------------------------------------------
 * run_bench (bench.cpp:155-198): rest start, warmup steps, then timed_runs x
 * steps, median device time (CUDA events on the stepper's stream).
 * MLUPs = fluid * steps / s / 1e6 (bench.cpp:184); bytes_per_lup = the paper's
 * traffic(); gpu_bytes_per_lup = compulsory bytes; predicted = hbm_gbs /
 * gpu_bytes_per_lup (hbm_gbs <= 0: no prediction). */
typedef struct {
  int32_t scheme, addressing, layout, precision;
  uint64_t fluid_count;
  int32_t steps;
  double seconds, mlups, bytes_per_lup, gpu_bytes_per_lup, predicted_mlups, model_fraction,
      achieved_gbs;
} lbmgpu_bench_result;
int lbmgpu_run_bench(const lbmgpu_geometry* g, const lbmgpu_flow* p, const lbmgpu_options* o,
                     int32_t steps, int32_t warmup, int32_t timed_runs, double hbm_gbs,
                     lbmgpu_bench_result* result);

/* verify_suite (bench.cpp:275-341): make_seeded_geometry(seed), seeded start,
 * every implemented pair (all_variants: x {SoA, AoS} x {fp64, fp32}) against
 * the GPU two-step reference after every step. fp64 passes bitwise (or
 * max_rel <= 1e-13, the reference's fallback), fp32 at max_rel <= 1e-5. */
typedef struct {
  int32_t scheme, addressing, layout, precision;
  int32_t bitwise, pass;
  double max_rel_linf;
} lbmgpu_verify_entry;
int lbmgpu_verify_suite(uint64_t seed, int32_t steps, int32_t device, int32_t all_variants,
                        lbmgpu_verify_entry* entries, int32_t capacity, int32_t* count,
                        int32_t* all_pass);

/* Device self-test of the collision's shared-reciprocal division against
 * __ddiv_rn (fp64) and __fdiv_rn (fp32): n seeded inputs (random bit
 * patterns, collision-like ranges, signed zeros, denormals, infinities,
 * NaNs); *mismatches = results whose bit patterns differ. */
int lbmgpu_selftest_division(uint64_t n, uint64_t seed, int32_t device, uint64_t* mismatches);
/* HBM streaming probe: best of `reps` launches of a 16-byte-vector copy over
 * `bytes` (inplace = 0) or an in-place read-modify-write of one buffer
 * (inplace = 1, the AA/ET/OS sweeps' pattern); GB/s counts read + write bytes.
 * bench.py reports it beside MEASURED_PEAKS.json as a second denominator. */
int lbmgpu_stream_bandwidth(int32_t device, uint64_t bytes, int32_t inplace, int32_t reps,
                            double* gbps);

/* kernel_available (p/src/stepper.cpp:140-153): 10 direct + 6 indirect */
int lbmgpu_kernel_available(int32_t scheme, int32_t addressing);
/* the same including the GPU extensions (TS / SWAP indirect) */
int lbmgpu_kernel_available_ext(int32_t scheme, int32_t addressing);

/* build_sparse (p/src/geometry.cpp:173-207) on the device: fluid count, and
 * when non-NULL the node-major adjacency[n*18 + (i-1)] (bounce = n) and
 * node_of[cell] (~0u for solids), bit-identical to the reference. Two-call
 * pattern: pass NULL arrays first to learn *fluid_count. Fails with
 * LBMGPU_RUNTIME_ERROR "fluid count exceeds 32-bit index range". */
int lbmgpu_build_sparse(const lbmgpu_geometry* g, int32_t device, uint32_t* fluid_count,
                        uint32_t* adjacency, uint32_t* node_of);
/* ET indirect remote table (p/src/scheme_et.cpp:42-62), node-major rem[n*9+p] */
int lbmgpu_build_et_rem(const lbmgpu_geometry* g, int32_t device, uint32_t* fluid_count,
                        uint32_t* rem, uint32_t* mailboxes);

/* traffic() (p/src/perfmodel.cpp:12-75): family in SchemeFamily order
 * (ts, os, osnt, cg, swap, aap, et); out[6] = loads, write_allocates, stores,
 * idx_halves, pdf_bytes, idx_bytes; bytes_per_lup for pdf_bytes (8 or 4).
 * gpu_bytes_per_lup: the compulsory DRAM bytes of THIS library's kernels
 * (loads + stores + IDX, no write-allocate). */
int lbmgpu_traffic(int32_t family, int32_t addressing, int32_t pdf_bytes, int32_t* out,
                   double* bytes_per_lup);
int lbmgpu_gpu_bytes_per_lup(int32_t scheme, int32_t addressing, int32_t pdf_bytes,
                             double* bytes_per_lup);

/* lambda_odd (p/src/collision.cpp:8-11) */
double lbmgpu_lambda_odd(double lambda_even, double magic_lambda);

/* ---- multi-GPU z-slabs (AA, OS push/pull, OSNT; direct, SoA; options.z_begin/z_end) ----
 * A slab stepper owns global planes [z_begin, z_end) of the geometry's box
 * (periodic z). Its canonical snapshot is that contiguous range of the global
 * one. Exchanges follow one plan: phase 0 (before each odd sweep) copies the
 * owners' face slots into the neighbours' ghost planes, phase 1 (after it)
 * copies them back; ops[k*5 + {phase, send, peer(-1 lower/+1 upper), plane
 * (-1 lower ghost .. nzl upper ghost), slot}], posted in this order. */
int lbmgpu_halo_plan(int32_t nzl, int32_t* ops, int32_t* count);
/* the plan of any decomposable scheme: AA (phases around odd sweeps), OS/OSNT
 * pull (phase 0 before every sweep, on the active grid), OS push (phase 1
 * after every sweep, on the grid just written) */
int lbmgpu_scheme_halo_plan(int32_t scheme, int32_t nzl, int32_t* ops, int32_t* count);
#define LBMGPU_NCCL_ID_BYTES 128
int lbmgpu_nccl_unique_id(uint8_t* id);
/* one rank per GPU: ring over ranks, rank r owns the r-th slab; collective */
int lbmgpu_slab_connect_nccl(lbmgpu_stepper* h, const uint8_t* id, int32_t nranks, int32_t rank);
/* the slab's communicator as NCCL reports it: ncclCommCount, ncclCommUserRank,
 * ncclGetVersion (evidence of the N-rank ring in bench output) */
int lbmgpu_slab_comm_info(lbmgpu_stepper* h, int32_t* count, int32_t* rank, int32_t* version);
/* ghosts <- owners (phase 0), needed before extract_natural at odd t; collective */
int lbmgpu_slab_sync_ghosts(lbmgpu_stepper* h);
/* several slabs in ONE process (any devices): step them in lockstep, the
 * exchanges as device-to-device copies following the same plan */
int lbmgpu_slab_group_step(lbmgpu_stepper** hs, int32_t n, int64_t steps);
int lbmgpu_slab_group_sync_ghosts(lbmgpu_stepper** hs, int32_t n);

/* peer-memory transport for AA slabs on direct addressing ("p2p"): no ghost
 * exchange and no collective. The face planes' odd sweep reads and rewrites
 * the neighbour slab's face-plane slots in place through peer pointers
 * (NVLink loads/stores inside the collision kernel); steps are ordered by
 * stream events (one process) or by flag words the ranks write into each
 * other's memory (one rank per process). The reference has no multi-node
 * path; this replaces the ghost exchange of lbmgpu_slab_connect_nccl. */
#define LBMGPU_P2P_BLOB_BYTES 256
/* several slabs of one process (ring in the given order, any devices with
 * peer access); then lbmgpu_slab_group_step as usual */
int lbmgpu_slab_group_connect_p2p(lbmgpu_stepper** hs, int32_t n);
/* one rank per process: publish this slab (CUDA IPC handles + layout) ... */
int lbmgpu_slab_p2p_export(lbmgpu_stepper* h, uint8_t* blob);
/* ... and connect to the lower / upper neighbours' blobs (nranks 1: pass
 * this slab's own blob twice). Collective: every rank connects before any
 * rank steps; lbmgpu_slab_sync_ghosts works as with NCCL. */
int lbmgpu_slab_p2p_connect(lbmgpu_stepper* h, const uint8_t* lower, const uint8_t* upper,
                            int32_t nranks, int32_t rank);
/* the same with flags. LBMGPU_P2P_HOST_ORDERED: no flag-word barrier kernel;
 * the CALLER orders the ranks (after every step / sync_ghosts: synchronize,
 * then a host barrier across the ranks before the next call). For ranks that
 * share one GPU, where kernels of different processes that spin on each
 * other's flags are not guaranteed to run concurrently. */
#define LBMGPU_P2P_HOST_ORDERED 1u
int lbmgpu_slab_p2p_connect_ex(lbmgpu_stepper* h, const uint8_t* lower, const uint8_t* upper,
                               int32_t nranks, int32_t rank, uint32_t flags);

/* page-locked host memory (cudaHostAlloc) for the canonical snapshot, so
 * extract/load run at full host-link bandwidth */
int lbmgpu_host_alloc(uint64_t bytes, void** p);
int lbmgpu_host_free(void* p);

const char* lbmgpu_last_error(void);
int lbmgpu_device_count(int32_t* count);
const char* lbmgpu_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LBMGPU_H */
