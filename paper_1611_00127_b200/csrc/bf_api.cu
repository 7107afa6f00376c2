// bf_api.cu -- the C-ABI entry points of libbf.so (include/bf.h), handle and memory
// management, error translation.  No exception crosses the ABI.
#include <chrono>
#include <functional>
#include <map>
#include <set>
#include <algorithm>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>

#include "bf_internal.cuh"
BF_CHECK_TU("bf_api.cu")

static thread_local std::string g_setup_err;

namespace bf {

void cuda_check(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation) {
    (void)cudaGetLastError();
    throw Error(BF_ERR_OOM, std::string("device allocation failed: ") + what);
  }
  throw Error(BF_ERR_CUDA, std::string(cudaGetErrorString(e)) + " at " + what);
}

// process-wide pool of small pinned host buffers (cudaMallocHost costs milliseconds; a
// setup+solve step must not pay it every time).  Thread-safe; one buffer per live handle.
static std::mutex g_pin_mu;
static std::multimap<size_t, double *> g_pin_free;  // size -> block

double *pinned_acquire(size_t bytes, size_t *got) {
  size_t sz = 4096;
  while (sz < bytes) sz <<= 1;
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    auto it = g_pin_free.lower_bound(sz);
    if (it != g_pin_free.end()) {
      double *p = it->second;
      *got = it->first;
      g_pin_free.erase(it);
      return p;
    }
  }
  void *p = nullptr;
  cuda_check(cudaMallocHost(&p, sz), "cudaMallocHost");
  *got = sz;
  return static_cast<double *>(p);
}

void pinned_release(double *p, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_free.emplace(bytes, p);
}

// Process-wide caching device allocator.  cudaMallocAsync/cudaFreeAsync were measured to
// block the host for up to ~1.5 s per setup when the stream-ordered pool had to remap; the
// setup allocates and frees ~2000 temporaries.  Blocks are cached by size class and never
// returned to the driver.  A block freed by a handle is reused only after that handle's next
// stream synchronisation (bf::sync), so queued work can never see its memory recycled.
static std::mutex g_dev_mu;
static std::multimap<size_t, void *> g_dev_free;  // size class -> block

static size_t size_class(size_t bytes) {
  if (bytes <= 4096) {
    size_t s = 256;
    while (s < bytes) s <<= 1;
    return s;
  }
  if (bytes <= (1u << 20)) return (bytes + 4095) & ~size_t(4095);
  return (bytes + (1u << 20) - 1) & ~size_t((1u << 20) - 1);
}

void *dalloc(bf_ctx *c, size_t bytes) {
  size_t sc = size_class(bytes);
  void *p = nullptr;
  auto t0 = std::chrono::steady_clock::now();
  {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    auto it = g_dev_free.lower_bound(sc);
    if (it != g_dev_free.end() && it->first <= sc + sc / 4) {  // accept <= 25 % slack
      sc = it->first;
      p = it->second;
      g_dev_free.erase(it);
    }
  }
  if (!p) {
    cudaError_t e = cudaMalloc(&p, sc);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      {  // release the cache and retry once
        std::lock_guard<std::mutex> lk(g_dev_mu);
        for (auto &f : g_dev_free) cudaFree(f.second);
        g_dev_free.clear();
      }
      e = cudaMalloc(&p, sc);
      if (e != cudaSuccess) {
        (void)cudaGetLastError();
        throw Error(BF_ERR_OOM, "cudaMalloc of " + std::to_string(sc) + " bytes failed (" +
                                    cudaGetErrorString(e) + ")");
      }
    }
  }
  c->alloc_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  c->allocs.emplace_back(p, sc);
  c->dev_bytes += (int64_t)sc;
  return p;
}

void release_all(bf_ctx *c) {  // caller has synchronised
  for (auto &a : c->allocs) c->pending_free.push_back(a);
  c->allocs.clear();
  {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    for (auto &f : c->pending_free) g_dev_free.emplace(f.second, f.first);
  }
  c->pending_free.clear();
}

// blocks freed since the last sync of this handle become reusable after the sync
static void release_pending(bf_ctx *c) {
  if (c->pending_free.empty()) return;
  std::lock_guard<std::mutex> lk(g_dev_mu);
  for (auto &f : c->pending_free) g_dev_free.emplace(f.second, f.first);
  c->pending_free.clear();
}

void dfree(bf_ctx *c, void *p) {
  if (!p) return;
  for (size_t i = 0; i < c->allocs.size(); i++) {
    if (c->allocs[i].first == p) {
      c->dev_bytes -= (int64_t)c->allocs[i].second;
      c->pending_free.push_back(c->allocs[i]);
      c->allocs[i] = c->allocs.back();
      c->allocs.pop_back();
      return;
    }
  }
}

void free_csr(bf_ctx *c, DCsr &A) {
  dfree(c, A.rp);
  dfree(c, A.ci);
  dfree(c, A.v);
  dfree(c, A.dia_v);
  free_window(c, A);
  A = DCsr();
}

static cudaEvent_t event_get(bf_ctx *c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  BF_CUDA(cudaEventCreate(&e));
  return e;
}

void timer_begin(bf_ctx *c, int k, cudaEvent_t *start) {
  *start = nullptr;
  if (!c->opt.timing || (k != 3 && c->timing_skip)) return;
  *start = event_get(c);
  BF_CUDA(cudaEventRecord(*start, c->stream));
}

void timer_end(bf_ctx *c, int k, cudaEvent_t start, double alg_bytes) {
  if (!c->opt.timing || !start) return;
  c->timers[k].bytes += alg_bytes;
  cudaEvent_t stop = event_get(c);
  BF_CUDA(cudaEventRecord(stop, c->stream));
  c->timers[k].pending.push_back(start);
  c->timers[k].pending.push_back(stop);
  c->timers[k].launches++;
}

void sync(bf_ctx *c) {
  auto t0 = std::chrono::steady_clock::now();
  cuda_check(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
  release_pending(c);
  c->sync_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  c->syncs++;
}

void timer_flush(bf_ctx *c) {
  for (auto &t : c->timers) {
    for (size_t i = 0; i + 1 < t.pending.size(); i += 2) {
      BF_CUDA(cudaEventSynchronize(t.pending[i + 1]));
      float ms = 0.f;
      BF_CUDA(cudaEventElapsedTime(&ms, t.pending[i], t.pending[i + 1]));
      t.ms += ms;
      c->event_pool.push_back(t.pending[i]);
      c->event_pool.push_back(t.pending[i + 1]);
    }
    t.pending.clear();
  }
}

// ---- checked build --------------------------------------------------------------------
#ifdef BF_CHECKED
static std::vector<std::pair<unsigned (*)(), const char *>> &check_registry() {
  static std::vector<std::pair<unsigned (*)(), const char *>> r;
  return r;
}
int register_check_reader(unsigned (*reader)(), const char *tu) {
  check_registry().emplace_back(reader, tu);
  return 1;
}
static __global__ void k_check_csr(DCsr A, int *bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0 && (A.rp[0] != 0 || A.rp[A.n] != A.nnz)) atomicCAS(bad, 0, -1);
  if (i >= A.n) return;
  int lo = A.rp[i], hi = A.rp[i + 1];
  if (hi < lo || lo < 0 || hi > A.nnz) {
    atomicCAS(bad, 0, i + 1);
    return;
  }
  for (int q = lo; q < hi; q++)
    if (A.ci[q] < 0 || A.ci[q] >= A.m || (q > lo && A.ci[q] <= A.ci[q - 1])) atomicCAS(bad, 0, i + 1);
}
#endif

void check_csr(bf_ctx *c, const DCsr &A, const char *what) {
#ifdef BF_CHECKED
  if (A.n == 0 || !A.rp) return;
  int *bad = dalloc_t<int>(c, 1);
  BF_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), c->stream));
  k_check_csr<<<div_up(A.n, 256), 256, 0, c->stream>>>(A, bad);
  int hb = 0;
  BF_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  dfree(c, bad);
  if (hb)
    throw Error(BF_ERR_CUDA, std::string("checked build: malformed CSR ") + what +
                                 (hb < 0 ? " (row pointer ends)" : " at row " + std::to_string(hb - 1)));
#else
  (void)c, (void)A, (void)what;
#endif
}

void check_device_flags(bf_ctx *c, const char *call) {
#ifdef BF_CHECKED
  BF_CUDA(cudaStreamSynchronize(c->stream));
  for (auto &r : check_registry()) {
    unsigned line = r.first();
    if (line)
      throw Error(BF_ERR_CUDA, std::string("checked build: device check failed in ") + r.second + " line " +
                                   std::to_string(line) + " during " + call);
  }
#else
  (void)c, (void)call;
#endif
}

#ifdef BF_CHECKED
// self-test of the checking mechanism (BF_CHECK_SELFTEST=1, checked build only): one gather one
// past the end of a vector of m entries must be reported by the next check_device_flags
static __global__ void k_check_selftest(const double *x, int m, double *y) {
  if (threadIdx.x == 0 && blockIdx.x == 0) y[0] = x[BF_COL(m, m)];
}
#endif

// checked build: every matrix the handle holds is well formed
static void check_handle(bf_ctx *c) {
#ifdef BF_CHECKED
  if (getenv("BF_CHECK_SELFTEST")) {
    k_check_selftest<<<1, 32, 0, c->stream>>>(c->xd, 2 * c->n, c->w);
    BF_CUDA(cudaGetLastError());
  }
  static const char *bn[5] = {"A_pp", "A_ps", "A_sp", "A_ss", "S~"};
  for (int b = 0; b < 5; b++) check_csr(c, c->blk[b], bn[b]);
  check_csr(c, c->jsc, "J scalar");
  for (int w = 0; w < 4; w++)
    for (int l = 0; l < c->h[w].nlev; l++) {
      const Level &L = c->h[w].lv[l];
      std::string t = "hierarchy " + std::to_string(w) + " level " + std::to_string(l) + " ";
      check_csr(c, L.A, (t + "A").c_str());
      check_csr(c, L.P, (t + "P").c_str());
      check_csr(c, L.R, (t + "R").c_str());
      check_csr(c, L.Rf, (t + "Rf").c_str());
      check_csr(c, L.A_io, (t + "A (construction order)").c_str());
      check_csr(c, L.P_io, (t + "P (construction order)").c_str());
    }
#else
  (void)c;
#endif
}

static bool env_flag(const char *name) { return getenv(name) != nullptr; }
static double env_num(const char *name, double dflt) {
  const char *e = getenv(name);
  return e ? atof(e) : dflt;
}

Tuning tuning_from_env() {
  Tuning t;
  t.verbose = env_flag("BF_VERBOSE");
  t.tma = !env_flag("BF_NO_TMA");
  t.pdl = !env_flag("BF_NO_PDL");
  t.dia = !env_flag("BF_NO_DIA");
  t.tail = !env_flag("BF_NO_TAIL");
  t.tail_nnz = (int64_t)env_num("BF_TAIL_NNZ", (double)t.tail_nnz);
  t.tail_bps = std::max(1, (int)env_num("BF_TAIL_BPS", t.tail_bps));
  t.reorder = !env_flag("BF_NO_REORDER");
  t.dtail = !env_flag("BF_NO_DTAIL");
  t.dtail_n = (int)env_num("BF_DTAIL_N", t.dtail_n);
  t.rfuse = !env_flag("BF_NO_RFUSE");
  t.rfuse_l0 = env_flag("BF_RFUSE_L0");
  t.merge_fuse = !env_flag("BF_NO_MERGE_FUSE");
  t.short_lim = env_num("BF_SHORT", t.short_lim);
  t.short_nmin = (int64_t)env_num("BF_SHORT_N", (double)t.short_nmin);
  t.short_k4 = env_num("BF_SHORT_K4", t.short_k4);
  t.stencil_g2 = env_num("BF_STENCIL_G2", t.stencil_g2);
  t.tma_g_div = env_num("BF_TMA_G", t.tma_g_div);
  t.tma_tile = env_num("BF_TMA_TILE", t.tma_tile);
  t.tma_ctas = std::max(1, (int)env_num("BF_TMA_CTAS", t.tma_ctas));
  t.tma_min_nnz = (int64_t)env_num("BF_TMA_MIN_NNZ", (double)t.tma_min_nnz);
  t.spread_small = !env_flag("BF_NO_SPREAD");
  t.win = !env_flag("BF_NO_WIN");
  t.win_rows = std::max(32, (int)env_num("BF_WIN_ROWS", t.win_rows));
  t.win_nmin = (int64_t)env_num("BF_WIN_NMIN", (double)t.win_nmin);
  t.win_ratio = env_num("BF_WIN_RATIO", t.win_ratio);
  t.win_minlen = env_num("BF_WIN_MINLEN", t.win_minlen);
  t.win_stage = std::max(1024, (int)env_num("BF_WIN_STAGE", t.win_stage));
  t.tma_g_p = (int)env_num("BF_TMA_G_P", 0);
  t.tma_g_r = (int)env_num("BF_TMA_G_R", 0);
  t.spgemm = env_flag("BF_SPGEMM_ESC") ? 2 : (env_flag("BF_SPGEMM_HASH") ? 1 : 0);
  t.wk_amin = env_num("BF_WK_AMIN", t.wk_amin);
  t.hash_small = !env_flag("BF_NO_HASH_SMALL");
  t.hash_large = !env_flag("BF_NO_HASH_LARGE");
  t.ilu_ctas = std::max(1, (int)env_num("BF_ILU_CTAS", t.ilu_ctas));
  t.ilu_pencil = env_num("BF_ILU_PENCIL", 1.0) != 0.0;
  t.ilu_flags = env_flag("BF_ILU_FLAGS");
  t.pencil_tk = std::max(1, (int)env_num("BF_PENCIL_TK", t.pencil_tk));
  t.pencil_tj = (int)env_num("BF_PENCIL_TJ", 0);
  return t;
}

int occupancy(bf_ctx *c, const void *kernel, int threads, size_t smem) {
  auto it = c->occ_cache.find(kernel);
  if (it != c->occ_cache.end()) return it->second;
  int per_sm = 0;
  BF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
  c->occ_cache[kernel] = per_sm;
  return per_sm;
}

static std::mutex g_attr_mu;
static std::set<std::pair<int, const void *>> g_attr_done;

void ensure_smem_attr(const void *kernel, int bytes) {
  int dev = 0;
  BF_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_attr_mu);
  if (g_attr_done.count({dev, kernel})) return;
  BF_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  g_attr_done.insert({dev, kernel});
}

}  // namespace bf

using namespace bf;

static void destroy_ctx(bf_ctx *c) {
  if (!c) return;
  cudaStreamSynchronize(c->stream);
  for (auto &t : c->timers)
    for (auto e : t.pending) cudaEventDestroy(e);
  for (auto e : c->event_pool) cudaEventDestroy(e);
  for (auto &a : c->allocs) c->pending_free.push_back(a);
  c->allocs.clear();
  bf::release_pending(c);
  if (c->hpin) bf::pinned_release(c->hpin, c->hpin_bytes);
  for (auto e : c->step_ev)
    if (e) cudaEventDestroy(e);
  if (c->apply_exec) cudaGraphExecDestroy(c->apply_exec);
  if (c->apply_graph) cudaGraphDestroy(c->apply_graph);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  cudaStreamSynchronize(c->stream);
  delete c;
}

#define BF_GUARD_BEGIN try {
#define BF_GUARD_END(ctx)                                           \
  }                                                                 \
  catch (const Error &e) {                                          \
    if (ctx) (ctx)->err = e.msg;                                    \
    return e.st;                                                    \
  }                                                                 \
  catch (const std::exception &e) {                                 \
    if (ctx) (ctx)->err = std::string("internal error: ") + e.what(); \
    return BF_ERR_CUDA;                                             \
  }


// the two AMG hierarchies of a preconditioner, built one after the other on the handle's stream
// (building them concurrently on two host threads was measured: ~5 ms faster on C3 but with
// 60-120 ms setup outliers from interleaved allocator requests -- not kept)
static void build_two_hierarchies(bf_ctx *c, int w0, const DCsr &A0, int w1, const DCsr &A1) {
  build_hierarchy(c, w0, A0);
  build_hierarchy(c, w1, A1);
}

extern "C" {

bf_status bf_default_options(bf_options *o) {
  if (!o) return BF_ERR_ARG;
  memset(o, 0, sizeof *o);
  o->theta = 0.25;
  o->max_levels = 25;
  o->max_coarse = 64;
  o->smoother = 1;  // R22: Chebyshev(2) on [0.1, 1] for A_ss, l1-Jacobi for S~ (and A_pp, J)
  o->nu_pre = 1;
  o->nu_post = 1;
  o->cheb_degree = 2;
  o->cheb_lo = 0.1;
  o->seed = 0x1611ULL;
  o->orth = 0;
  o->schur_as_printed = 0;
  o->interp_norm = 1;
  o->timing = 0;
  o->precond = 0;
  o->cheb_eig = 0;
  o->smoother_p = 0;
  o->cheb_levels = 0;
  o->diag_stop = 1;  // R23
  return BF_OK;
}

static const char *check_options(const bf_options *o) {
  if (!(o->theta > 0.0 && o->theta <= 1.0)) return "theta must be in (0, 1]";
  if (o->max_levels < 1 || o->max_levels > BF_MAXL) return "max_levels must be in [1, 64]";
  if (o->max_coarse < 1 || o->max_coarse > 128) return "max_coarse must be in [1, 128]";
  if (o->smoother != 0 && o->smoother != 1) return "smoother must be 0 or 1";
  if (o->smoother_p < -1 || o->smoother_p > 1) return "smoother_p must be -1, 0 or 1";
  if (o->cheb_levels < 0) return "cheb_levels must be >= 0";
  if (o->diag_stop != 0 && o->diag_stop != 1) return "diag_stop must be 0 or 1";
  if (o->nu_pre < 0 || o->nu_post < 0 || o->nu_pre > 8 || o->nu_post > 8) return "nu_pre/nu_post in [0, 8]";
  const bool cheb = o->smoother == 1 || o->smoother_p == 1;
  if (cheb && (o->cheb_degree < 1 || o->cheb_degree > 8)) return "cheb_degree in [1, 8]";
  if (cheb && !(o->cheb_lo > 0.0 && o->cheb_lo < 1.0)) return "cheb_lo in (0, 1)";
  if (o->orth != 0 && o->orth != 1) return "orth must be 0 or 1";
  if (o->cheb_eig < 0 || o->cheb_eig > 64) return "cheb_eig in [0, 64]";
  if (o->precond < 0 || o->precond > 3)
    return "precond must be 0 (BF), 1 (CPR-AMG(1)), 2 (CPR-AMG(2)) or 3 (coupled AMG)";
  return nullptr;
}

bf_status bf_setup(const bf_bsr2 *J, const bf_options *opt, void *stream, bf_handle *out) {
  if (out) *out = nullptr;
  g_setup_err.clear();
  if (!J || !out) {
    g_setup_err = "bf_setup: J and out must be non-NULL";
    return BF_ERR_ARG;
  }
  bf_ctx *c = new bf_ctx();
  c->stream = (cudaStream_t)stream;
  if (opt) c->opt = *opt;
  else bf_default_options(&c->opt);
  if (const char *m = check_options(&c->opt)) {
    g_setup_err = std::string("bf_setup: ") + m;
    delete c;
    return BF_ERR_ARG;
  }
  try {
    BF_CUDA(cudaGetDevice(&c->device));
    BF_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
    c->tune = tuning_from_env();
    c->use_tma = c->tune.tma;
    c->use_pdl = c->tune.pdl;
    const bool verbose = c->tune.verbose;
    auto t0 = std::chrono::steady_clock::now();
    auto lap = [&](const char *what) {
      if (!verbose) return;
      BF_CUDA(cudaStreamSynchronize(c->stream));
      auto t1 = std::chrono::steady_clock::now();
      fprintf(stderr, "[bf_setup] %-12s %8.2f ms  (alloc/free %.2f ms, %lld syncs waiting %.2f ms)\n", what,
              std::chrono::duration<double, std::milli>(t1 - t0).count(), c->alloc_ms, (long long)c->syncs,
              c->sync_ms);
      t0 = t1;
    };
    NvtxRange r_setup("bf_setup");
    {
      NvtxRange r("bf_setup: ingest + validate (a1)");
      validate_and_ingest(c, J);
      setup_bsr_dia(c);
    }
    lap("ingest");
    {
      NvtxRange r("bf_setup: field split (a2)");
      build_split(c);
    }
    lap("split");
    const int pc = c->opt.precond;
    if (pc == 0) {  // BF (Algorithm 3): S~, the A_ps coupling, hierarchies A_ss and S~
      {
        NvtxRange r("bf_setup: S~ (a3)");
        build_schur(c);
      }
      lap("schur");
      tile_csr(c, c->blk[1]);
      setup_dia(c, c->blk[1]);
      {
        NvtxRange r("bf_setup: AMG A_ss + S~ (a4)");
        build_two_hierarchies(c, 0, c->blk[3], 1, c->blk[4]);
      }
      lap("amg A_ss + S~");
    } else if (pc == 3) {  // coupled point AMG on J
      build_jscalar(c, c->jsc);
      build_hierarchy(c, 3, c->jsc);
      lap("amg J");
    } else {  // CPR-AMG(1)/(2) (Algorithms 1, 2): A_pp [and A_ss] hierarchies, ILU(0) of J
      if (pc == 2) {
        build_two_hierarchies(c, 2, c->blk[0], 0, c->blk[3]);
      } else {
        build_hierarchy(c, 2, c->blk[0]);
      }
      lap("amg A_pp [+ A_ss]");
      build_ilu(c);
      lap("ilu0");
    }
    alloc_solve_workspace(c, 30);
    BF_CUDA(cudaStreamSynchronize(c->stream));
    lap("workspace");
    check_handle(c);
    check_device_flags(c, "bf_setup");
  } catch (const Error &e) {
    g_setup_err = e.msg;
    bf_status st = e.st;
    destroy_ctx(c);
    return st;
  } catch (const std::exception &e) {
    g_setup_err = std::string("internal error: ") + e.what();
    destroy_ctx(c);
    return BF_ERR_CUDA;
  }
  *out = c;
  return BF_OK;
}

bf_status bf_update(bf_handle c, const double *vals, int32_t mem, void *stream) {
  if (!c || !vals || (mem != 0 && mem != 1)) {
    if (c) c->err = "bf_update: vals must be non-NULL and mem 0|1";
    return BF_ERR_ARG;
  }
  BF_GUARD_BEGIN
  NvtxRange r_update("bf_update");
  c->stream = (cudaStream_t)stream;
  c->err.clear();
  reingest_values(c, vals, mem);  // validation first: the handle is untouched on BF_ERR_NONFINITE
  setup_bsr_dia(c);
  drop_apply_graph(c);
  for (int b = 0; b < 5; b++) free_csr(c, c->blk[b]);
  dfree(c, c->dss);
  c->dss = nullptr;
  build_split(c);
  if (c->opt.precond == 0) {
    build_schur(c);
    tile_csr(c, c->blk[1]);
    setup_dia(c, c->blk[1]);
    refresh_finest(c, 0, c->blk[3]);
    refresh_finest(c, 1, c->blk[4]);
  } else if (c->opt.precond == 3) {
    free_csr(c, c->jsc);
    build_jscalar(c, c->jsc);
    refresh_finest(c, 3, c->jsc);
  } else {
    refresh_finest(c, 2, c->blk[0]);
    if (c->opt.precond == 2) refresh_finest(c, 0, c->blk[3]);
    build_ilu(c);  // numeric refactorization on the kept schedule
  }
  sync(c);
  check_handle(c);
  check_device_flags(c, "bf_update");
  return BF_OK;
  BF_GUARD_END(c)
}

int64_t bf_assemble_nnzb(int32_t nx, int32_t ny, int32_t nz) {
  int64_t n = (int64_t)nx * ny * nz;
  int64_t faces = (int64_t)(nx - 1) * ny * nz + (int64_t)nx * (ny - 1) * nz + (int64_t)nx * ny * (nz - 1);
  return n + 2 * faces;
}

// stand-alone calls (no handle): a transient context for the stream, scratch memory and errors
static bf_status run_transient(void *stream, const std::function<void(bf_ctx *)> &fn) {
  g_setup_err.clear();
  bf_ctx c;
  c.stream = (cudaStream_t)stream;
  try {
    fn(&c);
    bf::sync(&c);
  } catch (const Error &e) {
    g_setup_err = e.msg;
    cudaStreamSynchronize(c.stream);
    bf::release_all(&c);
    return e.st;
  }
  bf::release_all(&c);
  return BF_OK;
}

bf_status bf_assemble(const bf_twophase *P, const double *p, const double *sn, int32_t *row_ptr, int32_t *col_idx,
                      double *vals, double *residual, void *stream) {
  if (!P) {
    g_setup_err = "bf_assemble: prob must be non-NULL";
    return BF_ERR_ARG;
  }
  return run_transient(stream, [&](bf_ctx *c) { assemble(c, P, p, sn, row_ptr, col_idx, vals, residual); });
}

bf_status bf_newton_update(int32_t n, double *p, double *sn, const double *delta, double chop, void *stream) {
  if (n < 1 || !p || !sn || !delta) {
    g_setup_err = "bf_newton_update: bad argument";
    return BF_ERR_ARG;
  }
  return run_transient(stream, [&](bf_ctx *c) { newton_update(c, n, p, sn, delta, chop); });
}

bf_status bf_destroy(bf_handle h) {
  destroy_ctx(h);
  return BF_OK;
}

const char *bf_last_error(bf_handle h) { return h ? h->err.c_str() : g_setup_err.c_str(); }

// copy a 2n vector in or out; returns a device pointer (the handle's buffer when host)
static const double *vec_in(bf_ctx *c, const double *p, int mem, double *tmp) {
  if (mem == 1) return p;
  BF_CUDA(cudaMemcpyAsync(tmp, p, sizeof(double) * 2 * (size_t)c->n, cudaMemcpyHostToDevice, c->stream));
  return tmp;
}

bf_status bf_solve(bf_handle c, const double *rhs, double *x, double tol, int32_t restart,
                   int32_t maxit, int32_t vec_mem, int32_t *iters, double *res_hist,
                   int32_t *converged, double *relres, void *stream) {
  if (!c) return BF_ERR_ARG;
  if (!rhs || !x || !iters || !converged || !relres || restart < 1 || restart > 256 || maxit < 0 ||
      !(tol >= 0.0) || (vec_mem != 0 && vec_mem != 1)) {
    c->err = "bf_solve: bad argument (rhs/x/iters/converged/relres non-NULL, 1 <= restart <= 256, maxit >= 0, tol >= 0, vec_mem 0|1)";
    return BF_ERR_ARG;
  }
  BF_GUARD_BEGIN
  NvtxRange r_solve("bf_solve");
  c->stream = (cudaStream_t)stream;
  c->err.clear();
  cudaEvent_t t0;
  timer_begin(c, 3, &t0);
  alloc_solve_workspace(c, restart);
  const double *b = vec_in(c, rhs, vec_mem, c->bd);
  double *xd = x;
  if (vec_mem == 0) {
    BF_CUDA(cudaMemcpyAsync(c->xd, x, sizeof(double) * 2 * (size_t)c->n, cudaMemcpyHostToDevice, c->stream));
    xd = c->xd;
  }
  gmres(c, b, xd, tol, restart, maxit, iters, res_hist, converged, relres);
  if (vec_mem == 0)
    BF_CUDA(cudaMemcpyAsync(x, c->xd, sizeof(double) * 2 * (size_t)c->n, cudaMemcpyDeviceToHost, c->stream));
  timer_end(c, 3, t0);
  BF_CUDA(cudaStreamSynchronize(c->stream));
  timer_flush(c);
  check_device_flags(c, "bf_solve");
  return BF_OK;
  BF_GUARD_END(c)
}

bf_status bf_spmv(bf_handle c, const double *x, double *y, int32_t vec_mem, void *stream) {
  if (!c || !x || !y || (vec_mem != 0 && vec_mem != 1)) return BF_ERR_ARG;
  BF_GUARD_BEGIN
  c->stream = (cudaStream_t)stream;
  const double *xd = vec_in(c, x, vec_mem, c->bd);
  double *yd = vec_mem ? y : c->xd;
  cudaEvent_t t0;
  timer_begin(c, 0, &t0);
  bsr_spmv(c, xd, yd);
  timer_end(c, 0, t0, 36.0 * c->nnzb + 36.0 * c->n);
  if (!vec_mem)
    BF_CUDA(cudaMemcpyAsync(y, yd, sizeof(double) * 2 * (size_t)c->n, cudaMemcpyDeviceToHost, c->stream));
  BF_CUDA(cudaStreamSynchronize(c->stream));
  timer_flush(c);
  check_device_flags(c, "bf_spmv");
  return BF_OK;
  BF_GUARD_END(c)
}

bf_status bf_apply_precond(bf_handle c, const double *r, double *z, int32_t vec_mem, void *stream) {
  if (!c || !r || !z || (vec_mem != 0 && vec_mem != 1)) return BF_ERR_ARG;
  BF_GUARD_BEGIN
  c->stream = (cudaStream_t)stream;
  const double *rd = vec_in(c, r, vec_mem, c->bd);
  double *zd = vec_mem ? z : c->xd;
  cudaEvent_t t0;
  timer_begin(c, 2, &t0);
  bf_apply(c, rd, zd);
  timer_end(c, 2, t0);
  if (!vec_mem)
    BF_CUDA(cudaMemcpyAsync(z, zd, sizeof(double) * 2 * (size_t)c->n, cudaMemcpyDeviceToHost, c->stream));
  BF_CUDA(cudaStreamSynchronize(c->stream));
  timer_flush(c);
  check_device_flags(c, "bf_apply_precond");
  return BF_OK;
  BF_GUARD_END(c)
}

bf_status bf_vcycle(bf_handle c, int32_t which, const double *b, double *x, int32_t vec_mem, void *stream) {
  if (!c) return BF_ERR_ARG;
  if (!b || !x || which < 0 || which > 3 || c->h[which].nlev == 0 || (vec_mem != 0 && vec_mem != 1)) {
    c->err = "bf_vcycle: bad argument or hierarchy not built by this handle's preconditioner";
    return BF_ERR_ARG;
  }
  BF_GUARD_BEGIN
  c->stream = (cudaStream_t)stream;
  size_t bytes = sizeof(double) * (size_t)c->h[which].lv[0].A.n;
  const double *bd = b;
  double *xd = x;
  if (!vec_mem) {
    BF_CUDA(cudaMemcpyAsync(c->bd, b, bytes, cudaMemcpyHostToDevice, c->stream));
    bd = c->bd;
    xd = c->xd;
  }
  vcycle(c, which, bd, xd);
  if (!vec_mem) BF_CUDA(cudaMemcpyAsync(x, xd, bytes, cudaMemcpyDeviceToHost, c->stream));
  BF_CUDA(cudaStreamSynchronize(c->stream));
  check_device_flags(c, "bf_vcycle");
  return BF_OK;
  BF_GUARD_END(c)
}

bf_status bf_num_levels(bf_handle c, int32_t which, int32_t *nlev) {
  if (!c || !nlev || which < 0 || which > 3) return BF_ERR_ARG;
  *nlev = c->h[which].nlev;
  return BF_OK;
}

static void copy_csr_out(bf_ctx *c, const DCsr &A, int32_t *rp, int32_t *ci, double *v) {
  if (rp) BF_CUDA(cudaMemcpyAsync(rp, A.rp, sizeof(int32_t) * (A.n + 1), cudaMemcpyDeviceToHost, c->stream));
  if (ci && A.nnz) BF_CUDA(cudaMemcpyAsync(ci, A.ci, sizeof(int32_t) * A.nnz, cudaMemcpyDeviceToHost, c->stream));
  if (v && A.nnz) BF_CUDA(cudaMemcpyAsync(v, A.v, sizeof(double) * A.nnz, cudaMemcpyDeviceToHost, c->stream));
}

bf_status bf_get_level(bf_handle c, int32_t which, int32_t level, int32_t *n, int64_t *nnz_A,
                       int64_t *nnz_P, int32_t *A_rowptr, int32_t *A_col, double *A_val, int8_t *cf,
                       int32_t *P_rowptr, int32_t *P_col, double *P_val, double *dl1) {
  if (!c || which < 0 || which > 3 || level < 0 || level >= c->h[which].nlev) return BF_ERR_ARG;
  BF_GUARD_BEGIN
  const Level &L = c->h[which].lv[level];
  bool coarsest = level == c->h[which].nlev - 1;
  // the construction (= oracle) numbering: the copies kept when the solve-phase operators were renumbered
  const DCsr &A = L.A_io.n ? L.A_io : L.A;
  const DCsr &P = L.P_io.n ? L.P_io : L.P;
  if (n) *n = A.n;
  if (nnz_A) *nnz_A = A.nnz;
  if (nnz_P) *nnz_P = coarsest ? 0 : P.nnz;
  copy_csr_out(c, A, A_rowptr, A_col, A_val);
  if (!coarsest) {
    if (cf) BF_CUDA(cudaMemcpyAsync(cf, L.cf, A.n, cudaMemcpyDeviceToHost, c->stream));
    copy_csr_out(c, P, P_rowptr, P_col, P_val);
  }
  if (dl1) BF_CUDA(cudaMemcpyAsync(dl1, L.dl1, sizeof(double) * L.A.n, cudaMemcpyDeviceToHost, c->stream));
  BF_CUDA(cudaStreamSynchronize(c->stream));
  return BF_OK;
  BF_GUARD_END(c)
}

bf_status bf_get_level_smoother(bf_handle c, int32_t which, int32_t level, double *cheb_hi, double *beta0) {
  if (!c || which < 0 || which > 3 || level < 0 || level >= c->h[which].nlev) return BF_ERR_ARG;
  if (cheb_hi) *cheb_hi = c->h[which].lv[level].cheb_hi;
  if (beta0) *beta0 = c->h[which].lv[level].beta0;
  return BF_OK;
}

bf_status bf_get_block(bf_handle c, int32_t which, int64_t *nnz, int32_t *rowptr, int32_t *col, double *val) {
  if (!c || which < 0 || which > 4) return BF_ERR_ARG;
  BF_GUARD_BEGIN
  if (nnz) *nnz = c->blk[which].nnz;
  copy_csr_out(c, c->blk[which], rowptr, col, val);
  BF_CUDA(cudaStreamSynchronize(c->stream));
  return BF_OK;
  BF_GUARD_END(c)
}

bf_status bf_get_ilu(bf_handle c, double *lu, double *dinv, int32_t *levels) {
  if (!c) return BF_ERR_ARG;
  if (!c->ilu_lu) {
    c->err = "bf_get_ilu: the handle has no ILU(0) (only CPR handles, precond 1 or 2)";
    return BF_ERR_ARG;
  }
  BF_GUARD_BEGIN
  if (lu) BF_CUDA(cudaMemcpyAsync(lu, c->ilu_lu, sizeof(double) * 4 * (size_t)c->nnzb, cudaMemcpyDeviceToHost, c->stream));
  if (dinv) BF_CUDA(cudaMemcpyAsync(dinv, c->ilu_dinv, sizeof(double) * 4 * (size_t)c->n, cudaMemcpyDeviceToHost, c->stream));
  if (levels) *levels = c->ilu_levels;
  BF_CUDA(cudaStreamSynchronize(c->stream));
  return BF_OK;
  BF_GUARD_END(c)
}

bf_status bf_ilu_solve(bf_handle c, const double *r, double *x, int32_t vec_mem, void *stream) {
  if (!c) return BF_ERR_ARG;
  if (!r || !x || !c->ilu_lu || (vec_mem != 0 && vec_mem != 1)) {
    c->err = "bf_ilu_solve: needs a CPR handle (precond 1 or 2), non-NULL r and x, vec_mem 0|1";
    return BF_ERR_ARG;
  }
  BF_GUARD_BEGIN
  c->stream = (cudaStream_t)stream;
  const double *rd = vec_in(c, r, vec_mem, c->bd);
  double *xd = vec_mem ? x : c->xd;
  ilu_solve_into(c, rd, xd);
  if (!vec_mem)
    BF_CUDA(cudaMemcpyAsync(x, xd, sizeof(double) * 2 * (size_t)c->n, cudaMemcpyDeviceToHost, c->stream));
  BF_CUDA(cudaStreamSynchronize(c->stream));
  check_device_flags(c, "bf_ilu_solve");
  return BF_OK;
  BF_GUARD_END(c)
}

bf_status bf_kernel_time(bf_handle c, int32_t k, double *ms, int64_t *launches, double *alg_bytes) {
  if (!c || k < 0 || k > 3) return BF_ERR_ARG;
  if (ms) *ms = c->timers[k].ms;
  if (launches) *launches = c->timers[k].launches;
  if (alg_bytes) *alg_bytes = c->timers[k].bytes;
  return BF_OK;
}

bf_status bf_launch_count(bf_handle c, int64_t *launches) {
  if (!c || !launches) return BF_ERR_ARG;
  *launches = c->launches;
  return BF_OK;
}

bf_status bf_device_bytes(bf_handle c, int64_t *bytes) {
  if (!c || !bytes) return BF_ERR_ARG;
  *bytes = c->dev_bytes;
  return BF_OK;
}

}  // extern "C"
