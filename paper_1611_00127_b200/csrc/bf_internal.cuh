// bf_internal.cuh -- internal data structures of libbf.so (not part of the ABI).
//
// Device data layout (HBM, fp64 values, int32 indices):
//   J        : canonical point-interleaved 2x2 BSR, row_ptr[n+1], col[nnzb],
//              vals as double2 pairs [nnzb][2] = {(a_pp,a_ps),(a_sp,a_ss)} (32 B / block)
//   blocks   : A_pp, A_ps, A_sp, A_ss, S~ as scalar CSR (int32 rp/ci, f64 v)
//   AMG      : per level A_l, P_l, R_l = P_l^T (CSR), cf[n_l] (int8), dl1[n_l] (f64),
//              work vectors b_l, x_l, r_l, t_l (f64[n_l]); coarsest: dense LU (smem-staged)
//   GMRES    : V (restart+1) x N (column-contiguous), w, z, r, x (f64[N]), N = 2 n
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <deque>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/bf.h"
#include <nvtx3/nvToolsExt.h>

#define BF_MAXL 64

namespace bf {

// Windowed jagged-diagonal form of a CSR matrix (k_csr_win.cuh).  Kept behind a pointer: DCsr is a
// by-value kernel parameter of the setup kernels.
struct WJds {
  int32_t wrows = 0;          // rows per block (one CTA of wrows threads; power of two, 32..256)
  int32_t wmax_used = 0;      // largest window of any block (doubles)
  int32_t cap_ne = 0;         // largest entry count of any block (its bulk-copy stage; multiple of 8)
  int4 *meta = nullptr;       // per block: entry offset, entries (padded to 8), window length, longest row
  uint16_t *jdo = nullptr;    // per block: 256 slots, offset of jagged diagonal e within the block
  uint32_t *rowinfo = nullptr;// per sorted position: (row length << 16) | row within the block (0xffff: none)
  double *wv = nullptr;       // values by block and jagged diagonal
  uint16_t *lc = nullptr;     // per entry: position of its column in the block's window
  int32_t wstride = 0;        // slots per block in wcol: wmax_used rounded up to 256
  int32_t *wcol = nullptr;    // per block: wstride slots, the sorted distinct columns (zero padded)
};

struct DCsr {
  int32_t n = 0, m = 0;  // rows, cols
  int64_t nnz = 0;
  int32_t rpt = 0, cap = 0;  // TMA tiling: rows per tile, max nonzeros per tile (0: not tiled)
  int32_t g = 1;             // lanes per row in the TMA kernel
  bool short_rows = false;   // thread-per-row kernel (k_csr_short): large P / R with mean row length <= 4
  double *dia_v = nullptr;   // DIA storage of a grid-structured finest-level matrix (k_dia.cuh)
  int32_t dia_k = 0;
  int32_t *dia_off = nullptr;  // host array of dia_k offsets (kept out of the by-value kernel struct)
  int32_t *rp = nullptr, *ci = nullptr;
  double *v = nullptr;
  WJds *ws = nullptr;  // windowed jagged-diagonal form (k_csr_win.cuh), host object; null: none
};

struct Level {
  DCsr A, P, R;          // the solve-phase operators (coarse levels renumbered for locality, below)
  DCsr A_io, P_io;       // the hierarchy in the construction (= oracle) numbering when A / P were
                         // renumbered (k_amg_setup.cu reorder_levels); empty otherwise
  int32_t *perm = nullptr;  // solve-phase position -> construction index of this level's points
  DCsr Rf;  // fused restriction R (I - beta A D^-1) of the seeded pre-smoother's residual (k_amg_setup.cu)
  int8_t *cf = nullptr;
  double *dl1 = nullptr;
  double *b = nullptr, *x = nullptr, *r = nullptr, *t = nullptr;
  double *d = nullptr;  // 1 / dl1 (smoother scaling)
  int smoother = 0;      // 0 l1-Jacobi, 1 Chebyshev: the hierarchy's smoother (reading R22)
  double cheb_hi = 1.0;  // upper end of the Chebyshev interval [cheb_lo hi, hi] (reading R21)
  double beta0 = 1.0;    // first smoothing step from zero: x0 = beta0 b ./ dl1 (1/theta for Chebyshev)
};

struct Hier {
  int nlev = 0;
  int smoother = 0;       // this hierarchy's smoother (opt.smoother or, pressure-type, opt.smoother_p; R22)
  Level lv[BF_MAXL];
  double *lu = nullptr;  // nL x nL row-major LU (unit lower L below the diagonal)
  int32_t *piv = nullptr;
  double *inv = nullptr;  // explicit inverse of the coarsest matrix (nL x nL, row-major)
  int32_t nL = 0;
  int tail = -1;          // first level handled by the cooperative tail kernel (-1: none)
  int dtail = -1;         // first level whose whole sub-V-cycle is applied as a dense operator T (-1: none)
  double *tmat = nullptr; // T (n_dtail x n_dtail, row-major): the exact linear map b -> x of that sub-V-cycle
  bool dense = false;  // coarsest level solved by LU (else 4 l1-Jacobi sweeps)
};

// Solve-path variants and tiling heuristics.  Every default is the measured choice (DESIGN.md
// section 8b); the environment overrides (BF_NO_TMA, BF_NO_DTAIL, BF_TAIL_NNZ, ...) exist for
// the parity tests of the path variants (tests/test_gpu_parity.py VARIANTS) and for tuning
// experiments.  They are read ONCE per bf_setup into the handle (tuning_from_env), never cached
// in process-wide statics, so handles are independent.  Not part of the ABI.
struct Tuning {
  bool verbose = false;
  bool tma = true;          // TMA-pipelined CSR kernels (else the warp-staged k_csr)
  bool pdl = true;          // programmatic dependent launch
  bool dia = true;          // DIA storage of grid-structured finest-level operators and of J
  bool tail = true;         // cooperative single-kernel V-cycle tail
  int64_t tail_nnz = 3000;  // levels with at most this many nonzeros go to the cooperative tail
  int tail_bps = 1;         // cooperative tail CTAs per SM
  bool reorder = true;      // coarse levels renumbered in (x/8, y, z)-Morton order for gather locality
  bool dtail = true;        // dense tail operator below dtail_n rows
  int dtail_n = 2048;
  bool rfuse = true;        // fused restriction R (I - beta A D) on the CSR levels
  bool rfuse_l0 = false;    // ... also on the finest level (measured slower)
  bool merge_fuse = true;   // S~ finest post-sweep fused with the merge
  double short_lim = 8.0;   // thread-per-row kernel for P / R with mean row length <= short_lim ...
  double short_k4 = 3.0;    // ... with 4 register slots per row up to this mean row length, 8 above
  int64_t short_nmin = 65536;  // ... and at least this many rows
  double stencil_g2 = 8.0;  // stencil rows longer than this on average get 2 lanes per row
  double tma_g_div = 4.0;   // Galerkin rows: lanes per row ~ mean row length / tma_g_div
  double tma_tile = 1024.0; // target nonzeros per TMA tile
  int tma_ctas = 8;         // TMA kernel CTAs per SM (upper bound; shared memory decides)
  int64_t tma_min_nnz = 0;  // matrices with fewer nonzeros use the warp-staged kernel (no TMA pipeline)
  bool spread_small = true; // small matrices: >= 2 TMA tiles per SM (more lanes per row)
  bool win = true;          // windowed jagged-diagonal form of the coarse-level operators (k_csr_win.cuh)
  int win_rows = 256;       // rows per block at most
  int win_stage = 36 * 1024; // block size: mean bytes of a block's matrix stream
  double win_minlen = 8.0;  // matrices with shorter mean rows (the level transfers) keep the CSR kernels
  int64_t win_nmin = 16384; // matrices with fewer rows keep the CSR kernels
  double win_ratio = 0.35;   // the form is dropped if the windows hold more than this many entries per nonzero
  int tma_g_p = 0, tma_g_r = 0;  // forced lanes per row for P / R (0: heuristic)
  int spgemm = 0;           // 0 auto (thread-per-row, hash, ESC fallback), 1 hash, 2 ESC
  double interp_warp_min = 16.0;  // interpolation: warp per row above this mean row length of A, thread per row below
  bool hash_large = true;   // ... and with the 1024-slot table for rows of up to 640 columns before falling back to ESC
  double hash_large_min = 500.0;  // mean products per row from which the count starts with the large table
  bool hash_small = true;   // warp-hash fill kernel with the small table when the product's longest row allows
  double wk_amin = 14.0;    // ... and the lane-per-entry warp kernels (k_spgemm_wk_*) above this mean row length of A
  double tpr_bmax = 6.0;    // thread-per-row / lane-per-entry SpGEMM only for B with at most this mean row length
  double tpr_amax = 200.0;  // ... and A with at most this mean row length (longer: warp-hash kernels)
  int ilu_ctas = 4;         // generic ILU sweep CTAs per SM
  bool ilu_pencil = true;   // pencil-wavefront ILU sweeps on grid-structured J
  bool ilu_flags = false;   // flag-array sweeps instead of value flags (generic path)
  int pencil_tk = 8, pencil_tj = 0;  // pencil tile (0: 128 / tk)
};
Tuning tuning_from_env();

struct Timer {
  double ms = 0.0;
  int64_t launches = 0;
  double bytes = 0.0;
  std::vector<cudaEvent_t> pending;  // pairs (start, stop)
};

class Error {
 public:
  bf_status st;
  std::string msg;
  Error(bf_status s, std::string m) : st(s), msg(std::move(m)) {}
};

}  // namespace bf

struct bf_ctx {
  bf_options opt{};
  cudaStream_t stream = nullptr;
  std::string err;
  int32_t n = 0;  // cells
  int32_t nx = 0, ny = 0, nz = 0;
  int64_t nnzb = 0;
  int32_t var_order = 0;
  int32_t block_order = 0;
  int32_t *brp = nullptr, *bci = nullptr;
  double *bv = nullptr;  // canonical (p,s) row-major blocks
  double *jdia = nullptr;  // DIA copy of J (7 block diagonals), k_spmv.cu
  int32_t jdia_k = 0, jdia_off[8] = {0};
  bf::DCsr blk[5];       // A_pp, A_ps, A_sp, A_ss, S~
  double *dss = nullptr;
  bf::Hier h[4];         // AMG hierarchies: 0 A_ss, 1 S~ (BF), 2 A_pp (CPR), 3 J as a scalar matrix (coupled AMG)
  bf::DCsr jsc;          // J as a point-ordered scalar CSR (precond 3)
  // CPR-AMG(1)/(2) block ILU(0) of J (k_ilu.cu)
  int32_t *ilu_perm = nullptr, *ilu_dpos = nullptr;  // level-sorted row schedule, diagonal block positions
  int32_t ilu_levels = 0;
  double *ilu_lu = nullptr, *ilu_dinv = nullptr;     // factors on J's block pattern, inverse pivot blocks
  int *ilu_flag = nullptr;                           // per-row completion flags of the sync-free sweeps
  unsigned *ilu_sync = nullptr;                      // tickets / epoch of the sweeps
  double *ilu_y = nullptr, *ilu_u = nullptr;         // forward result, CPR first-stage solution (canonical)
  bool ilu_vflag = true;                             // value-flag sweeps (default) or flag-array sweeps
  bool ilu_pencil = false, ilu_pencil_checked = false;  // pencil-wavefront sweeps (grid-structured J)
  double *ilu_ld = nullptr, *ilu_ud = nullptr;       // DIA copies of L (k-1, j-1, i-1) and U (i+1, j+1, k+1)
  int2 *ilu_order = nullptr;                         // tile order (anti-diagonals)
  int ilu_geom[7] = {0};                             // nx, ny, nz, TJ, TK, NJ, NK
  // solve workspace
  int32_t Vm = 0;
  double *Z = nullptr;  // preconditioned basis z_j = M^-1 v_j (restart x N)
  double *V = nullptr, *w = nullptr, *z = nullptr, *r = nullptr, *xd = nullptr, *bd = nullptr;
  double *vp = nullptr, *vs = nullptr, *sv = nullptr, *pv = nullptr;  // BF apply split vectors
  double *red = nullptr;        // reduction partials
  double *hdev = nullptr;       // reduced coefficients (device)
  double *hpin = nullptr;       // pinned host mirror
  size_t hpin_bytes = 0;
  unsigned long long *nonfinite = nullptr;  // first non-finite index (error reporting)
  unsigned int *counter = nullptr;
  cudaEvent_t step_ev[2] = {nullptr, nullptr};  // per-Arnoldi-step completion (pipelined GMRES)
  int red_blocks = 0;
  // bookkeeping
  std::vector<std::pair<void *, size_t>> allocs;
  std::vector<std::pair<void *, size_t>> pending_free;  // reusable after the next sync
  int64_t dev_bytes = 0;
  int64_t launches = 0;
  bf::Timer timers[4];
  std::vector<cudaEvent_t> event_pool;
  // CUDA graph of the BF apply (k_vcycle.cu)
  cudaStream_t cap_stream = nullptr;
  cudaGraph_t apply_graph = nullptr;
  cudaGraphExec_t apply_exec = nullptr;
  struct PatchNode {
    cudaGraphNode_t node;
    cudaKernelNodeParams params;
    int nargs = 0;
    std::vector<std::pair<int, int>> roles;  // (argument index, 0 v | 1 nrm2 | 2 z)
  };
  std::vector<PatchNode> apply_patch;
  int64_t apply_graph_kernels = 0;
  int num_sms = 148;
  int device = 0;
  bf::Tuning tune;      // solve-path variants / heuristics, read once at bf_setup
  bool use_tma = true;
  bool use_pdl = true;  // programmatic dependent launch for the TMA CSR kernels
  std::unordered_map<const void *, int> occ_cache;  // resident CTAs per SM of a kernel (this device)
  std::deque<std::vector<int32_t>> dia_offsets;  // storage behind DCsr::dia_off
  double alloc_ms = 0.0;
  double alg_bytes = 0.0;       // running algorithmic-bytes counter (csr_op, vector kernels)
  double apply_bytes = 0.0;     // algorithmic bytes of one BF apply (set at graph capture)
  int64_t syncs = 0;
  double sync_ms = 0.0;
  bool fuse_post0 = false;      // BF apply: S~ finest post-sweep fused with the merge (k_vcycle.cu)
  bool timing_skip = false;     // opt.timing = k > 1: only every k-th Arnoldi step is timed
  int64_t timing_step = 0;      // Arnoldi steps enqueued since setup (sampling counter)
};

namespace bf {

// ---- error / allocation helpers (bf_api.cu) --------------------------------------
void cuda_check(cudaError_t e, const char *what);
void *dalloc(bf_ctx *c, size_t bytes);
void dfree(bf_ctx *c, void *p);
template <class T>
T *dalloc_t(bf_ctx *c, size_t count) {
  return static_cast<T *>(dalloc(c, count * sizeof(T) + 16));
}
void free_csr(bf_ctx *c, DCsr &A);
// checked build: validate row pointers / column range / ascending columns of A on the device
void check_csr(bf_ctx *c, const DCsr &A, const char *what);
// checked build: read every translation unit's device-check flag (throws on a failed check)
void check_device_flags(bf_ctx *c, const char *call);
// pinned host buffers of at least `bytes` (pooled process-wide; *got = the block's size)
double *pinned_acquire(size_t bytes, size_t *got);
void pinned_release(double *p, size_t bytes);
void timer_begin(bf_ctx *c, int k, cudaEvent_t *start);
void timer_end(bf_ctx *c, int k, cudaEvent_t start, double alg_bytes = 0.0);
void timer_flush(bf_ctx *c);
void sync(bf_ctx *c);  // counted, timed cudaStreamSynchronize
void release_all(bf_ctx *c);  // return every block of c to the cache (after a sync)

#define BF_CUDA(x) ::bf::cuda_check((x), #x)

// NVTX range for profilers (ncu --nvtx / nsys); a no-op without an attached tool
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};
#define BF_LAUNCH(c) ((c)->launches++)

// ---- scans (k_util.cu) ------------------------------------------------------------
// exclusive prefix sum of int32 counts[0..n) into out[0..n], returns out[n] (host sync)
int64_t exclusive_scan_i32(bf_ctx *c, const int32_t *counts, int32_t *out, int32_t n);
int64_t exclusive_scan_i64(bf_ctx *c, const int64_t *counts, int64_t *out, int64_t n);
void sort_pairs_u64_f64(bf_ctx *c, uint64_t *keys, double *vals, int64_t count, int end_bit);
void sort_pairs_u64_i32(bf_ctx *c, uint64_t *keys, int32_t *vals, int64_t count, int end_bit);

// ---- setup kernels -----------------------------------------------------------------
void validate_and_ingest(bf_ctx *c, const bf_bsr2 *J);                 // k_split.cu
void build_split(bf_ctx *c);                                            // k_split.cu
void reingest_values(bf_ctx *c, const double *vals, int mem);            // k_split.cu
void refresh_finest(bf_ctx *c, int which, const DCsr &A0);              // k_amg_setup.cu
void drop_apply_graph(bf_ctx *c);                                       // k_vcycle.cu
void build_schur(bf_ctx *c);                                            // k_split.cu
void build_hierarchy(bf_ctx *c, int which, const DCsr &A0);             // k_amg_setup.cu
void free_hierarchy(bf_ctx *c, Hier &h);
void plan_tail(bf_ctx *c, Hier &h);
void set_level_beta(const bf_options &o, Level &L);                      // k_vcycle.cu
// smoother of hierarchy `which` (0 A_ss, 1 S~, 2 A_pp, 3 J): all but A_ss take smoother_p (R22)
inline int hier_smoother(const bf_options &o, int which) {
  return (which != 0 && o.smoother_p >= 0) ? o.smoother_p : o.smoother;
}
void build_dense_tail(bf_ctx *c, Hier &h);                               // k_vcycle.cu
void build_rfuse(bf_ctx *c, Hier &h, bool finest_only);                 // k_amg_setup.cu
double apply_model_bytes(bf_ctx *c);                                    // k_vcycle.cu
void tile_csr(bf_ctx *c, DCsr &A, bool stencil = false, int force_g = 0);  // k_vcycle.cu
void window_csr(bf_ctx *c, DCsr &A);                                    // k_vcycle.cu
void free_window(bf_ctx *c, DCsr &A);                                   // k_vcycle.cu
void build_windows(bf_ctx *c, Hier &h);                                 // k_vcycle.cu
void setup_dia(bf_ctx *c, DCsr &A);                                     // k_vcycle.cu

// ---- solve kernels -------------------------------------------------------------
void bsr_spmv(bf_ctx *c, const double *x, double *y);                   // k_spmv.cu
void setup_bsr_dia(bf_ctx *c);                                          // k_spmv.cu
void csr_spmv(bf_ctx *c, const DCsr &A, const double *x, double *y);    // k_spmv.cu
void vcycle(bf_ctx *c, int which, const double *b, double *x);          // k_vcycle.cu
void bf_apply(bf_ctx *c, const double *v, double *z, const double *nrm2 = nullptr);                   // k_vcycle.cu
void bf_apply_graph(bf_ctx *c, const double *v, double *z, const double *nrm2 = nullptr);             // k_vcycle.cu
void alloc_solve_workspace(bf_ctx *c, int restart);                     // k_gmres.cu
void assemble(bf_ctx *c, const bf_twophase *P, const double *p, const double *sn, int32_t *rp, int32_t *ci,
              double *vals, double *R);                                   // k_assemble.cu
void newton_update(bf_ctx *c, int n, double *p, double *sn, const double *delta, double chop);
void build_ilu(bf_ctx *c);                                              // k_ilu.cu
void build_jscalar(bf_ctx *c, DCsr &A);                                 // k_ilu.cu
void cpr_apply(bf_ctx *c, const double *v, double *z, const double *nrm2);
double cpr_model_bytes(bf_ctx *c);
bool cpr_patch_roles(const void *func, int &nargs, std::vector<std::pair<int, int>> &roles);
void ilu_solve_into(bf_ctx *c, const double *r, double *x);              // x = (LU)^-1 r, caller order
void gmres(bf_ctx *c, const double *b, double *x, double tol, int restart, int maxit,
           int *iters, double *hist, int *converged, double *relres);   // k_gmres.cu

// resident CTAs per SM of `kernel` at `threads` threads and `smem` dynamic shared memory on the
// handle's device (cached in the handle)
int occupancy(bf_ctx *c, const void *kernel, int threads, size_t smem);
// cudaFuncAttributeMaxDynamicSharedMemorySize of `kernel` raised to `bytes` on the current
// device (once per kernel and device; thread-safe)
void ensure_smem_attr(const void *kernel, int bytes);

// number of parameters of a kernel (graph-node argument patching, k_vcycle.cu)
template <typename... A>
constexpr int nargs_of(void (*)(A...)) {
  return (int)sizeof...(A);
}

inline int div_up(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// programmatic dependent launch (PDL): the kernel may begin while its stream predecessor is
// still running; it touches that predecessor's outputs only after pdl_wait().  Data written
// before the predecessor started (setup matrices, older Krylov vectors) may be read earlier.
// Both are no-ops for a kernel launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void launch_pdl(bf_ctx *c, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = c->use_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BF_CUDA(cudaLaunchKernelEx(&cfg, kernel, ((KArgs)args)...));
}

}  // namespace bf

// ---- checked build (-DBF_CHECKED, libbf_checked.so) ---------------------------------------
// compute-sanitizer is closed on the GPU pool this was developed on, so memory safety is shown
// with the library's own checks: BF_CHK(cond) records the source line of the first failed
// device-side check in a per-translation-unit flag (the access is then clamped, never made);
// every public call of a checked build reads all flags after its work and fails with
// BF_ERR_CUDA "device check failed ..." if one is set.  check_csr() validates a built matrix
// (row pointers, column range and order) on the device.  In the normal build all of it
// compiles to nothing.
#ifdef BF_CHECKED
static __device__ unsigned int bf_chk_line = 0;
#define BF_CHK(cond) ((cond) ? true : (atomicCAS(&bf_chk_line, 0u, (unsigned)__LINE__), false))
namespace bf {
int register_check_reader(unsigned (*reader)(), const char *tu);
}  // namespace bf
static unsigned bf_chk_read() {
  unsigned v = 0, z = 0;
  cudaMemcpyFromSymbol(&v, bf_chk_line, sizeof v);
  if (v) cudaMemcpyToSymbol(bf_chk_line, &z, sizeof z);
  return v;
}
#define BF_CHECK_TU(name) static int bf_chk_registered = ::bf::register_check_reader(&bf_chk_read, name);
#else
#define BF_CHK(cond) true
#define BF_CHECK_TU(name)
#endif
// a gathered column index, bounds-checked (and clamped) in the checked build
#define BF_COL(col, m) (BF_CHK((unsigned)(col) < (unsigned)(m)) ? (col) : 0)
// a polling loop of the sync-free sweeps: bounded in the checked build (a dependency that never
// completes is reported instead of hanging the GPU)
#ifdef BF_CHECKED
#define BF_SPIN_OK(s) BF_CHK(++(s) < (1u << 26))
#else
#define BF_SPIN_OK(s) true
#endif

