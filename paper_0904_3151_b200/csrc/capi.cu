// capi.cu -- extern "C" entry points of libepsgraph_b200.so (see
// include/epsgraph_b200.h) and the host-side launch logic around the
// kernels.  Single translation unit: nvcc -gencode arch=compute_100a,
// code=sm_100a -O3 -lineinfo -shared.
#include <stdarg.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "msm.cuh"
#include "plan.cuh"
#include "project_h16.cuh"
#include "exact.cuh"
#include "format.cuh"
#include "project.cuh"
#include "project_tc.cuh"
#include <cudaTypedefs.h>
#include "scan_sort.cuh"
#include "verify.cuh"

namespace eg {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// ------------------------------------------------------- instrumentation
struct ProfRec {
  int cls;
  cudaEvent_t a, b;
};
static std::mutex g_prof_mu;
static std::atomic<long long> g_launches{0};
static std::atomic<int> g_prof_on{0};
static std::vector<ProfRec> g_prof_open[PC_COUNT];   // per class stack (nesting)
static std::vector<ProfRec> g_prof_done;
static std::vector<cudaEvent_t> g_event_pool;
static const char *g_prof_names[PC_COUNT] = {
    "row_stats", "project", "fixup", "msm_hist", "msm_scan", "msm_scatter", "msm_group",
    "msm_spill", "msm_batch", "sort_upsweep", "scan", "sort_downsweep", "verify", "compact",
    "misc", "msm_stage", "sort_stage", "verify_stage"};

static cudaEvent_t take_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void prof_begin(int cls, cudaStream_t st, int launches) {
  g_launches += launches;
  if (!g_prof_on.load()) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  ProfRec r{cls, take_event(), take_event()};
  cudaEventRecord(r.a, st);
  g_prof_open[cls].push_back(r);
}

void prof_end(int cls, cudaStream_t st) {
  if (!g_prof_on.load()) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (g_prof_open[cls].empty()) return;
  ProfRec r = g_prof_open[cls].back();
  g_prof_open[cls].pop_back();
  cudaEventRecord(r.b, st);
  g_prof_done.push_back(r);
}

static int arg_error(const char *msg) {
  set_error("%s", msg);
  return EG_ERR_ARG;
}

static int num_sms() {
  static int cached[64];
  int dev = 0;
  cudaGetDevice(&dev);
  dev &= 63;
  if (!cached[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v < 1)
      v = 148;
    cached[dev] = v;
  }
  return cached[dev];
}

Options &options() {
  static Options o;
  return o;
}

// Dynamic shared-memory opt-in.  The attribute lives in the device context,
// so the record of what was already set is kept per (device, kernel): a
// process that builds on cuda:0 and then on cuda:1 sets it on both.
static cudaError_t smem_optin(const void *func, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  static std::mutex mu;
  static std::map<std::pair<int, const void *>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t &have = done[std::make_pair(dev, func)];
  if (bytes <= have) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}
#define EG_SMEM_OPTIN(func, bytes) EG_CUDA_TRY(smem_optin((const void *)(func), (size_t)(bytes)))

// ------------------------------------------------------------ projection
static int project_tn(int cols) {
  int g = (cols + 31) / 32;
  return g > 8 ? 8 : g;
}

static double projection_tau(int dim) {
  // |s_fp32 - s_exact| <= ((dim+2) u + O(u^2)) sum|x_q r_q| <= ... ||x|| ||r||
  // (u = 2^-24: rounding of x and r to fp32, FMA accumulation); plus the
  // reference's own fp64 error dim * 2^-53; 25% safety margin.
  return 1.25 * ((double)(dim + 2) * ldexp(1.0, -24) + (double)dim * ldexp(1.0, -52));
}

static unsigned long long fixup_cap(int64_t n, int cols) {
  unsigned long long c = (unsigned long long)n * cols / 32;
  c = c < (1ull << 20) ? (1ull << 20) : c;
  const long long forced = options().fixup_cap;   // tests: force the overflow path
  return forced > 0 && (unsigned long long)forced < c ? (unsigned long long)forced : c;
}

template <typename TX, int TN>
static void launch_project(const TX *x, int64_t n, int dim, const float *rt, int cols,
                           int cols_pad, const double *norms, const double *rnorm, double tau,
                           int L, int W, uint64_t *codes, FixupList fl, cudaStream_t st) {
  unsigned grid = (unsigned)((n + PJ_BM - 1) / PJ_BM);
  EG_PROF(PC_PROJECT, st);
  k_project<TX, TN><<<grid, PJ_NT, 0, st>>>(x, n, dim, rt, cols, cols_pad, norms, rnorm, tau, L,
                                            W, codes, fl);
}

template <typename TX>
static void dispatch_project(int tn, const TX *x, int64_t n, int dim, const float *rt, int cols,
                             int cols_pad, const double *norms, const double *rnorm, double tau,
                             int L, int W, uint64_t *codes, FixupList fl, cudaStream_t st) {
  switch (tn) {
#define EG_TN(T)                                                                              \
  case T:                                                                                     \
    launch_project<TX, T>(x, n, dim, rt, cols, cols_pad, norms, rnorm, tau, L, W, codes, fl, \
                          st);                                                                \
    break;
    EG_TN(1) EG_TN(2) EG_TN(3) EG_TN(4) EG_TN(5) EG_TN(6) EG_TN(7) EG_TN(8)
#undef EG_TN
  }
}

// ------------------------------------------------------------------ MSM

// Small pinned host staging area per device (results read after a sync the
// call performs anyway, so the copy does not add a synchronisation).
static unsigned long long *pinned_small() {
  static unsigned long long *buf[64];
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!buf[dev] && cudaHostAlloc(&buf[dev], 4096, cudaHostAllocPortable) != cudaSuccess)
    buf[dev] = nullptr;
  return buf[dev];
}

static int msm_buckets(int64_t n) {
  // mean bucket size: the tuned target, but never above 70% of the small
  // tier's capacity.  Buckets are hash-balanced (Poisson, sd = sqrt(mean)),
  // so the ones that overflow hold a large group on top of their share
  // (coarse design keys: config 3 has groups of 500-1500 rows) and go to the
  // medium tier; 70% leaves room for groups up to ~600 rows (cfg3 stage at
  // 80% / 70% / 60% / 50%: 2.58 / 2.51 / 2.56 / 2.71 ms).
  const int64_t cap_mean = (int64_t)(0.7 * SmallCfg<1>::CAP);
  const int64_t tgt = std::min<int64_t>(MSM_TARGET, cap_mean);
  int64_t b = (n + tgt - 1) / tgt;
  if (b < 1) b = 1;
  return (int)std::min<int64_t>(b, (int64_t)1 << MSM_MAX_LGB);
}

static int msm_batch_units(int64_t n) {
  // keep the per-batch scratch (elems + gcnt: 12 B/row/unit) under ~2 GiB
  int64_t per = n * 12;
  int64_t u = per > 0 ? (int64_t)(2ll << 30) / per : MSM_MAXU;
  if (u < 1) u = 1;
  return (int)(u > MSM_MAXU ? MSM_MAXU : u);
}

struct MsmLayout {
  int lgB, B, U, sets;
  size_t bytes;
};

static MsmLayout msm_layout(int64_t n, int reps) {
  MsmLayout l;
  l.B = msm_buckets(n);
  l.lgB = ilog2_ceil((uint64_t)l.B);
  l.U = msm_batch_units(n);
  // two scratch sets: batch i+1's hist/scatter overlap batch i's grouping
  l.sets = options().msm_streams >= 2 ? 2 : 1;
  size_t b = 0;
  b += ws_bytes((size_t)l.U * l.B, 4);            // counts
  b += ws_bytes((size_t)l.U * (l.B + 1), 4);      // starts
  b += ws_bytes((size_t)l.U * l.B, 4);            // cursor
  b += ws_bytes((size_t)l.U * n, 8);              // elems
  b += ws_bytes((size_t)l.U * n, 4);              // gcnt
  b += ws_bytes(EG_MAX_LENGTH, 1);                // bit2blk
  b += ws_bytes(3 + 2 * (size_t)reps, 8);         // counters
  b += ws_bytes((size_t)l.U * (l.B + 1) * 9, 4);  // spill list (<= 3 entries/bucket)
  b += ws_bytes(2, 8);                            // spill counters
  l.bytes = (b + 4096) * l.sets;
  return l;
}

template <int W>
static int msm_run(MsmArgs *sets, const MsmLayout &lay, const std::vector<UnitBatch> &batches,
                   cudaStream_t st) {
  MsmArgs a = sets[0];
  // histograms of several units side by side (<= 96 KB), staging for scatter
  const size_t smem_hist =
      std::min<size_t>((size_t)128 << 10, (size_t)lay.B * 4 * lay.U) / ((size_t)lay.B * 4) *
      ((size_t)lay.B * 4);
  a.hist_smem = (int)smem_hist;
  // smem-staged coalesced runs only pay when a tile holds several rows per
  // bucket; for large B the scatter writes directly
  const bool staged = lay.B <= MSM_STAGE_MAX_B;
  a.scatter_staged = staged ? 1 : 0;
  const size_t smem_scatter =
      staged ? (size_t)MSM_TILE * 10 + (size_t)lay.B * 12 : (size_t)lay.B * 8;
  const size_t smem_group =
      sizeof(HGroupSmem<W, SmallCfg<W>::CAP, SmallCfg<W>::NT, SmallCfg<W>::MDIV>);

  const size_t smem_medium = sizeof(HGroupSmem<W, MediumCfg<W>::CAP, MediumCfg<W>::NT, 1>);
  a.gcnt_min = MediumCfg<W>::CAP;
  EG_SMEM_OPTIN(k_msm_hist<W>, smem_hist);
  EG_SMEM_OPTIN(k_msm_scatter<W>, smem_scatter);
  EG_SMEM_OPTIN(k_msm_group<W>, smem_group);
  EG_SMEM_OPTIN(k_msm_medium<W>, smem_medium);
  const unsigned tiles = (unsigned)((a.n + MSM_TILE - 1) / MSM_TILE);
  const unsigned spill_grid = (unsigned)num_sms() * 8;
  // Two scratch sets on two streams: the caller's stream runs hist / scan /
  // scatter of batch i+1 while a side stream groups batch i (the first is
  // L2/atomic bound, the second issue bound).  Events order the reuse of a
  // set and the final join.
  // A third stream runs the tail tiers (medium / spill / max group) of
  // batch i concurrently with the small-tier group kernel of batch i+1:
  // the tails occupy few SMs (a handful of heavy buckets) and would
  // otherwise serialise behind it.
  // Priorities: the partition stream (hist / scan / scatter of the next
  // batch) and the tail stream outrank the group stream, so their CTAs take
  // the SM slots the group kernel frees first -- the next batch is ready
  // when the group kernel ends, and a batch's heavy buckets do not queue
  // behind the next group kernel.
  static cudaStream_t side[64], tail[64], part[64];
  static cudaEvent_t ev_scat[64][2], ev_grp[64][2], ev_done[64][2], ev_end[64];
  int dev = 0;
  cudaGetDevice(&dev);
  const bool two = lay.sets == 2;
  if (two && !side[dev]) {
    int prio_lo = 0, prio_hi = 0;
    EG_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    EG_CUDA_TRY(cudaStreamCreateWithPriority(&side[dev], cudaStreamNonBlocking, prio_lo));
    EG_CUDA_TRY(cudaStreamCreateWithPriority(&tail[dev], cudaStreamNonBlocking, prio_hi));
    EG_CUDA_TRY(cudaStreamCreateWithPriority(&part[dev], cudaStreamNonBlocking, prio_hi));
    for (int i = 0; i < 2; ++i) {
      EG_CUDA_TRY(cudaEventCreateWithFlags(&ev_scat[dev][i], cudaEventDisableTiming));
      EG_CUDA_TRY(cudaEventCreateWithFlags(&ev_grp[dev][i], cudaEventDisableTiming));
      EG_CUDA_TRY(cudaEventCreateWithFlags(&ev_done[dev][i], cudaEventDisableTiming));
    }
    EG_CUDA_TRY(cudaEventCreateWithFlags(&ev_end[dev], cudaEventDisableTiming));
  }
  cudaStream_t gs = two ? side[dev] : st;
  cudaStream_t ts = two ? tail[dev] : st;
  cudaStream_t ps = two ? part[dev] : st;
  if (two) {   // the side streams start after everything already on st
    EG_CUDA_TRY(cudaEventRecord(ev_scat[dev][0], st));
    EG_CUDA_TRY(cudaStreamWaitEvent(gs, ev_scat[dev][0], 0));
    EG_CUDA_TRY(cudaStreamWaitEvent(ts, ev_scat[dev][0], 0));
    EG_CUDA_TRY(cudaStreamWaitEvent(ps, ev_scat[dev][0], 0));
  }
#ifdef EG_MSM_TIMELINE
  std::vector<std::pair<const char *, cudaEvent_t>> tl;
  auto mark = [&](const char *what, cudaStream_t s) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    tl.push_back({what, e});
  };
  mark("start", st);
#define EG_TL(what, s) mark(what, s)
#else
#define EG_TL(what, s)
#endif
  for (size_t bi = 0; bi < batches.size(); ++bi) {
    const UnitBatch &ub = batches[bi];
    const int si = two ? (int)(bi & 1) : 0;
    MsmArgs &x = sets[si];
    x.hist_smem = a.hist_smem;
    x.scatter_staged = a.scatter_staged;
    x.gcnt_min = a.gcnt_min;
    x.small_cap = SmallCfg<W>::CAP;
    if (two && bi >= 2) EG_CUDA_TRY(cudaStreamWaitEvent(ps, ev_done[dev][si], 0));
    dim3 g1(tiles, ub.count);
    {
      EG_PROF(PC_MSM_HIST, ps);
      k_msm_hist<W><<<tiles, MSM_NT, smem_hist, ps>>>(x, ub);
    }
    EG_CUDA_TRY(cudaMemsetAsync(x.spill_ctr, 0, 16, ps));   // spill list reset for this batch
    {
      EG_PROF(PC_MSM_SCAN, ps);
      k_msm_scan<<<ub.count, 1024, 0, ps>>>(x);
    }
    {
      EG_PROF(PC_MSM_SCATTER, ps);
      k_msm_scatter<W><<<g1, MSM_SC_NT, smem_scatter, ps>>>(x, ub);
    }
    EG_TL("scatter_end", ps);
    if (two) {
      EG_CUDA_TRY(cudaEventRecord(ev_scat[dev][si], ps));
      EG_CUDA_TRY(cudaStreamWaitEvent(gs, ev_scat[dev][si], 0));
    }
    // persistent medium-tier CTAs: as many as are resident (two per SM when
    // the tier's shared memory fits twice)
    const unsigned per_sm = smem_medium * 2 + 2048 <= (size_t)227 * 1024 ? EG_MEDIUM_MINCTAS : 1;
    const unsigned medium_grid = (unsigned)num_sms() * per_sm;
    if (two) EG_CUDA_TRY(cudaStreamWaitEvent(ts, ev_scat[dev][si], 0));
    {   // oversized buckets: beside the small tier, not behind it
      EG_PROF(PC_MSM_SPILL, ts);
      k_msm_medium<W><<<medium_grid, MediumCfg<W>::NT, smem_medium, ts>>>(x, ub, 0);
    }
    dim3 g4(lay.B, ub.count);
    EG_TL("group_start", gs);
    {
      EG_PROF(PC_MSM_GROUP, gs);
      k_msm_group<W><<<g4, SmallCfg<W>::NT, smem_group, gs>>>(x, ub);
    }
    EG_TL("group_end", gs);
    if (two) {
      EG_CUDA_TRY(cudaEventRecord(ev_grp[dev][si], gs));
      EG_CUDA_TRY(cudaStreamWaitEvent(ts, ev_grp[dev][si], 0));
    }
    {
      EG_PROF(PC_MSM_SPILL, ts);
      k_msm_medium<W><<<medium_grid, MediumCfg<W>::NT, smem_medium, ts>>>(x, ub, 1);
    }
    EG_TL("medium_end", ts);
    {
      EG_PROF(PC_MSM_SPILL, ts);
      k_msm_spill<W><<<spill_grid, MSM_SPILL_T, 0, ts>>>(x, ub);
    }
    EG_TL("spill_end", ts);
    {
      EG_PROF(PC_MSM_SPILL, ts);
      k_msm_spill_maxgroup<<<64, 256, 0, ts>>>(x);
    }
    if (two) EG_CUDA_TRY(cudaEventRecord(ev_done[dev][si], ts));
    EG_LAUNCH_CHECK();
  }
  if (two) {   // join: the tails are last on ts, the group kernels on gs
    EG_CUDA_TRY(cudaEventRecord(ev_done[dev][0], ts));
    EG_CUDA_TRY(cudaStreamWaitEvent(st, ev_done[dev][0], 0));
    EG_CUDA_TRY(cudaEventRecord(ev_end[dev], gs));
    EG_CUDA_TRY(cudaStreamWaitEvent(st, ev_end[dev], 0));
  }
#ifdef EG_MSM_TIMELINE
  mark("joined", st);
  cudaStreamSynchronize(st);
  for (size_t i = 1; i < tl.size(); ++i) {
    float ms = 0;
    cudaEventElapsedTime(&ms, tl[0].second, tl[i].second);
    fprintf(stderr, "[msm timeline] %-12s %.3f ms\n", tl[i].first, ms);
  }
  for (auto &t : tl) cudaEventDestroy(t.second);
#endif
  return EG_OK;
}

}  // namespace eg

using namespace eg;

extern "C" {

const char *eg_last_error(void) { return g_err; }

int eg_set_option(const char *name, long long value) {
  if (!name) return arg_error("eg_set_option: null name");
  Options &o = options();
  if (!strcmp(name, "project_path") && value >= 0 && value <= 4) o.project_path = (int)value;
  else if (!strcmp(name, "fixup_force_seq")) o.fixup_force_seq = value != 0;
  else if (!strcmp(name, "fixup_cap") && value >= 0) o.fixup_cap = value;
  else if (!strcmp(name, "msm_blocks") &&
           ((value >= -1 && value <= EG_MAX_BLOCKS) || (value >= 10000 && value < 20000)))
    o.msm_blocks = (int)value;
  else if (!strcmp(name, "msm_designs") && (value == 0 || value == 1)) o.msm_designs = (int)value;
  else if (!strcmp(name, "msm_streams") && (value == 1 || value == 2)) o.msm_streams = (int)value;
  else if (!strcmp(name, "plan_debug")) o.plan_debug = value != 0;
  else if (!strcmp(name, "msm_batches") && value >= 0 && value <= 64) o.msm_batches = (int)value;
  else if (!strcmp(name, "verify_wide")) o.verify_wide = value != 0;
  else if (!strcmp(name, "sort_path") && value >= -1 && value <= 1) o.sort_path = (int)value;
  else return arg_error("eg_set_option: unknown option or value out of range");
  return EG_OK;
}

void eg_reset_options(void) { options() = Options(); }

long long eg_launch_count(void) { return g_launches.load(); }

void eg_profile_enable(int on) {
  if (on) {
    // pre-create the event pool (and the record list) so that the first
    // profiled builds do not pay for cudaEventCreate / vector growth
    std::lock_guard<std::mutex> lk(g_prof_mu);
    while (g_event_pool.size() < 8192) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) break;
      g_event_pool.push_back(e);
    }
    g_prof_done.reserve(8192);
  }
  g_prof_on = on ? 1 : 0;
}

const char *eg_profile_class_name(int cls) {
  return (cls >= 0 && cls < PC_COUNT) ? g_prof_names[cls] : "";
}

int eg_profile_read(double *ms_out, long long *count_out, int max_classes) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (int c = 0; c < max_classes && c < PC_COUNT; ++c) {
    ms_out[c] = 0.0;
    count_out[c] = 0;
  }
  for (ProfRec &r : g_prof_done) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    if (r.cls < max_classes) {
      ms_out[r.cls] += ms;
      count_out[r.cls] += 1;
    }
    g_event_pool.push_back(r.a);
    g_event_pool.push_back(r.b);
  }
  g_prof_done.clear();
  return PC_COUNT;
}
int eg_version(void) { return 1; }
int eg_device_sm_count(void) { return num_sms(); }

// ------------------------------------------------------------ row stats
int eg_row_stats(const void *d_x, int x_is_f64, int64_t n, int32_t dim, double *d_norms,
                 uint64_t *d_bad, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || dim < 1 || !d_bad) return arg_error("eg_row_stats: bad shape");
  EG_CUDA_TRY(cudaMemsetAsync(d_bad, 0xff, 16, st));
  if (n == 0) return EG_OK;
  unsigned grid = (unsigned)((n + ROWST_WARPS * 32 - 1) / (ROWST_WARPS * 32));
  EG_PROF(PC_ROW_STATS, st);
  if (x_is_f64)
    k_row_stats<double><<<grid, ROWST_WARPS * 32, 0, st>>>((const double *)d_x, n, dim, d_norms,
                                                        (unsigned long long *)d_bad);
  else
    k_row_stats<float><<<grid, ROWST_WARPS * 32, 0, st>>>((const float *)d_x, n, dim, d_norms,
                                                       (unsigned long long *)d_bad);
  EG_LAUNCH_CHECK();
  return EG_OK;
}

// ----------------------------------------------------------- projection
size_t eg_project_workspace(int64_t n, int32_t dim, int32_t length, int32_t replicates) {
  int cols = length * replicates;
  int cols_pad = (cols + 31) / 32 * 32;
  int npad = (cols + 15) / 16 * 16;
  return ws_bytes((size_t)dim * cols_pad, 4) + ws_bytes(1, 8) +
         ws_bytes(fixup_cap(n, cols), 8) +
         ws_bytes((size_t)((dim + TC_BK - 1) / TC_BK) * 2 * npad * TC_BK, 4) +
         ws_bytes((size_t)replicates * n * ((length + 63) / 64), 8) + ws_bytes(TC_MAXN, 8) +
         2048;
}

// TMA descriptor of the row-major fp32 rows: box = 32 columns (128 B, one
// swizzle row) x 128 rows, SWIZZLE_128B, out-of-bounds rows zero-filled.
static bool make_x_tensor_map(CUtensorMap *map, const void *d_x, int64_t n, int dim) {
  static PFN_cuTensorMapEncodeTiled encode = nullptr;
  if (!encode) {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = (PFN_cuTensorMapEncodeTiled)fn;
  }
  if (((uintptr_t)d_x & 15) || (dim * 4) % 16) return false;
  cuuint64_t gdim[2] = {(cuuint64_t)dim, (cuuint64_t)n};
  cuuint64_t gstride[1] = {(cuuint64_t)dim * 4};
  cuuint32_t box[2] = {TC_BK, TC_M};
  cuuint32_t estride[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(d_x), gdim,
                      gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Test hook: when set, the tensor-core projection also writes its raw fp32
// accumulator (n x cols) here (used to validate the error band).
static float *g_tc_debug = nullptr;
extern "C" void eg_debug_set_tc_dump(float *d_buf) { g_tc_debug = d_buf; }
// Debug: copy (and optionally reset) the MSM bucket counters (all zero
// unless the library was compiled with -DEG_MSM_STATS=1).
extern "C" int eg_debug_msm_stats(unsigned long long *out16, int reset) {
  if (cudaMemcpyFromSymbol(out16, eg::g_msm_stats, sizeof(unsigned long long) * 8) != cudaSuccess)
    return EG_ERR_CUDA;
  for (int i = 8; i < 16; ++i) out16[i] = 0;
  if (reset) {
    static const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (cudaMemcpyToSymbol(eg::g_msm_stats, z, sizeof(z)) != cudaSuccess) return EG_ERR_CUDA;
  }
  return EG_OK;
}

// Shared body of eg_project / eg_project_rows.  d_bad != nullptr: also
// produce the row norms into d_norms (and the bad-row flags) -- fused into
// the tensor-core kernel where that path runs, else k_row_stats first.
static int project_impl(const void *d_x, int x_is_f64, int64_t n, int32_t dim, double *d_norms,
                        const double *d_r, const double *d_rnorm, int32_t length,
                        int32_t replicates, uint64_t *d_codes, void *d_workspace,
                        size_t workspace_bytes, uint64_t *d_fixups, uint64_t *d_bad,
                        cudaStream_t st);

int eg_project(const void *d_x, int x_is_f64, int64_t n, int32_t dim, const double *d_norms,
               const double *d_r, const double *d_rnorm, int32_t length, int32_t replicates,
               uint64_t *d_codes, void *d_workspace, size_t workspace_bytes, uint64_t *d_fixups,
               void *stream) {
  return project_impl(d_x, x_is_f64, n, dim, const_cast<double *>(d_norms), d_r, d_rnorm, length,
                      replicates, d_codes, d_workspace, workspace_bytes, d_fixups, nullptr,
                      (cudaStream_t)stream);
}

int eg_project_rows(const void *d_x, int x_is_f64, int64_t n, int32_t dim, double *d_norms,
                    uint64_t *d_bad, const double *d_r, const double *d_rnorm, int32_t length,
                    int32_t replicates, uint64_t *d_codes, void *d_workspace,
                    size_t workspace_bytes, uint64_t *d_fixups, void *stream) {
  if (!d_bad || !d_norms) return arg_error("eg_project_rows: d_norms and d_bad are required");
  return project_impl(d_x, x_is_f64, n, dim, d_norms, d_r, d_rnorm, length, replicates, d_codes,
                      d_workspace, workspace_bytes, d_fixups, d_bad, (cudaStream_t)stream);
}

// Exact recompute of the band entries flagged in `unc` (the codes layout):
// entry list (k_collect_bits), warp-per-entry fix-up, and the bitmap pass
// that redoes everything if the list overflowed.
static int run_band_fixup(const void *d_x, int32_t dim, const double *d_r, int64_t n,
                          int32_t length, int W, int32_t replicates, int cols, uint64_t *d_codes,
                          uint64_t *unc, unsigned long long *items, unsigned long long *cnt,
                          unsigned long long cap, uint64_t *d_fixups, cudaStream_t st) {
  {
    EG_PROF(PC_FIXUP, st);
    const int64_t words = (int64_t)replicates * n * W;
    const int64_t per = (int64_t)COLLECT_NT * COLLECT_WPT;
    k_collect_bits<<<(unsigned)std::min<int64_t>((words + per - 1) / per,
                                                 (int64_t)num_sms() * 8),
                     COLLECT_NT, 0, st>>>(unc, n, W, length, replicates, items, cnt, cap);
    {
      const size_t fws = (size_t)(FIXW_NT / 32) * dim * 8;
      EG_SMEM_OPTIN(k_fixup_warp, fws);
      k_fixup_warp<<<(unsigned)num_sms() * 8, FIXW_NT, fws, st>>>(
          (const float *)d_x, dim, d_r, n, length, W, d_codes, items, cnt, cap,
          options().fixup_force_seq);
    }
    const size_t fsm = (size_t)8 * dim * 8;   // 8 warps x dim doubles
    EG_SMEM_OPTIN(k_fixup_bits, fsm);
    const unsigned fg = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8);
    k_fixup_bits<<<fg, 256, fsm, st>>>((const float *)d_x, n, dim, d_r, length, W,
                                       replicates, d_codes, unc, cnt, cap);
  }
  EG_LAUNCH_CHECK();
  if (d_fixups)
    EG_CUDA_TRY(cudaMemcpyAsync(d_fixups, cnt, 8, cudaMemcpyDeviceToDevice, st));
  return EG_OK;
}

static int project_impl(const void *d_x, int x_is_f64, int64_t n, int32_t dim, double *d_norms,
                        const double *d_r, const double *d_rnorm, int32_t length,
                        int32_t replicates, uint64_t *d_codes, void *d_workspace,
                        size_t workspace_bytes, uint64_t *d_fixups, uint64_t *d_bad,
                        cudaStream_t st) {
  if (n < 0 || dim < 1 || length < 1 || replicates < 1)
    return arg_error("eg_project: bad shape");
  if ((int64_t)length * replicates >= (1ll << 31) || n >= (1ll << 32))
    return arg_error("eg_project: too large");
  const int W = (length + 63) / 64;
  const int cols = length * replicates;
  const int cols_pad = (cols + 31) / 32 * 32;
  EG_CUDA_TRY(cudaMemsetAsync(d_codes, 0, (size_t)replicates * n * W * 8, st));
  if (d_fixups) EG_CUDA_TRY(cudaMemsetAsync(d_fixups, 0, 8, st));
  if (n == 0) {
    if (d_bad) EG_CUDA_TRY(cudaMemsetAsync(d_bad, 0xff, 16, st));
    return EG_OK;
  }
  Arena ar(d_workspace, workspace_bytes);
  float *rt = ar.take<float>((size_t)dim * cols_pad);
  unsigned long long *cnt = ar.take<unsigned long long>(1);
  const unsigned long long cap = fixup_cap(n, cols);
  unsigned long long *items = ar.take<unsigned long long>(cap);
  if (!rt || !cnt || !items) {
    set_error("eg_project: workspace too small");
    return EG_ERR_WORKSPACE;
  }
  EG_CUDA_TRY(cudaMemsetAsync(cnt, 0, 8, st));
  FixupList fl{cnt, items, cap};
  const int npad = (cols + 15) / 16 * 16;
  const int path = options().project_path;
  const bool use_tc = !x_is_f64 && dim % 4 == 0 && npad <= TC_MAXN && path != 1;
  CUtensorMap xmap;
  const bool tma_ok = use_tc && path != 4 &&
                      make_x_tensor_map(&xmap, d_x, n, dim);
  const bool fuse = d_bad && tma_ok && path != 3;
  if (d_bad && !fuse) {   // norms first, then the projection reads them
    int rc = eg_row_stats(d_x, x_is_f64, n, dim, d_norms, d_bad, st);
    if (rc) return rc;
  } else if (fuse) {
    EG_CUDA_TRY(cudaMemsetAsync(d_bad, 0xff, 16, st));
  }
  if (use_tc) {
    float *img = ar.take<float>((size_t)((dim + TC_BK - 1) / TC_BK) * 2 * npad * TC_BK);
    if (!img) {
      set_error("eg_project: workspace too small");
      return EG_ERR_WORKSPACE;
    }
    {
      EG_PROF(PC_MISC, st);
      k_tc_prep_directions<<<256, 256, 0, st>>>(d_r, cols, dim, npad, img);
    }
    EG_LAUNCH_CHECK();
    const int64_t ntiles = (n + TC_M - 1) / TC_M;
    const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)num_sms());
    const int h16_no = 2;
#ifndef EG_H16_NPAD_MIN
#define EG_H16_NPAD_MIN 0   // experiments: pad the direction columns (MMA N) to at least this
#endif
    const int h16_npad = std::max(npad, EG_H16_NPAD_MIN);
    const bool h16 = tma_ok && path != 2 && h16_fits(h16_npad, h16_no);
    if (h16) {
      // kind::f16 (2-term fp16 splits): the production path for fp32 rows
      double *colscale = ar.take<double>(TC_MAXN);
      uint64_t *unc = ar.take<uint64_t>((size_t)replicates * n * W);
      if (!colscale || !unc) {
        set_error("eg_project: workspace too small");
        return EG_ERR_WORKSPACE;
      }
      __half *himg = reinterpret_cast<__half *>(img);
      {
        EG_PROF(PC_MISC, st);
        k_h16_prep_directions<<<h16_npad, 128, 0, st>>>(d_r, cols, dim, h16_npad, himg, colscale);
      }
      EG_LAUNCH_CHECK();
      const size_t ob = h16_oslot_bytes(h16_npad);
      const int no = h16_no;
      const size_t budget = ((size_t)220 << 10) - sizeof(H16Bars) - 1024;
      const int nx = (int)std::min<size_t>(H16_MAXSLOTS, (budget - no * ob) / H16_XSLOT);
      if (nx < 2) return arg_error("eg_project: too many direction columns for the f16 path");
      const size_t smem = nx * H16_XSLOT + no * ob + sizeof(H16Bars) + 1024;
      EG_SMEM_OPTIN(k_project_h16, smem);
      {
        EG_PROF(PC_PROJECT, st);
        k_project_h16<<<grid, H16_THREADS, smem, st>>>(
            xmap, n, dim, himg, colscale, cols, h16_npad, nx, no, d_norms, d_rnorm, h16_tau(dim),
            length, W, d_codes, unc, g_tc_debug, fuse ? d_norms : nullptr,
            fuse ? (unsigned long long *)d_bad : nullptr);
      }
      EG_LAUNCH_CHECK();
      return run_band_fixup(d_x, dim, d_r, n, length, W, replicates, cols, d_codes, unc, items,
                            cnt, cap, d_fixups, st);
    }
    if (tma_ok) {
      const size_t sbytes = tc2_stage_bytes(npad);
      const int nstages = (int)std::min<size_t>(4, ((size_t)212 << 10) / sbytes);
      const size_t smem = nstages * sbytes + sizeof(Tc2Bars) + 1024;
      EG_SMEM_OPTIN(k_project_tc2, smem);
      uint64_t *unc = ar.take<uint64_t>((size_t)replicates * n * W);
      if (!unc) {
        set_error("eg_project: workspace too small");
        return EG_ERR_WORKSPACE;
      }
      {
        EG_PROF(PC_PROJECT, st);
        k_project_tc2<<<grid, TC2_THREADS, smem, st>>>(xmap, n, dim, img, cols, npad, nstages,
                                                       d_norms, d_rnorm, tc_tau(dim), length, W,
                                                       d_codes, unc, g_tc_debug,
                                                       fuse ? d_norms : nullptr,
                                                       fuse ? (unsigned long long *)d_bad
                                                            : nullptr);
      }
      EG_LAUNCH_CHECK();
      return run_band_fixup(d_x, dim, d_r, n, length, W, replicates, cols, d_codes, unc, items,
                            cnt, cap, d_fixups, st);
    } else {
      const size_t smem = 2 * tc_stage_bytes(npad) + sizeof(TcSmem) + 1024;
      EG_SMEM_OPTIN(k_project_tc, smem);
      EG_PROF(PC_PROJECT, st);
      k_project_tc<<<grid, TC_NT, smem, st>>>((const float *)d_x, n, dim, img, cols, npad,
                                              d_norms, d_rnorm, tc_tau(dim), length, W, d_codes,
                                              fl, g_tc_debug);
    }
    EG_LAUNCH_CHECK();
  } else {
    {
      int64_t tot = (int64_t)dim * cols_pad;
      EG_PROF(PC_MISC, st);
      k_prep_directions<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(d_r, cols, dim, cols_pad,
                                                                      rt);
      EG_LAUNCH_CHECK();
    }
    const double tau = projection_tau(dim);
    const int tn = project_tn(cols);
    if (x_is_f64)
      dispatch_project<double>(tn, (const double *)d_x, n, dim, rt, cols, cols_pad, d_norms,
                               d_rnorm, tau, length, W, d_codes, fl, st);
    else
      dispatch_project<float>(tn, (const float *)d_x, n, dim, rt, cols, cols_pad, d_norms,
                              d_rnorm, tau, length, W, d_codes, fl, st);
    EG_LAUNCH_CHECK();
  }
  const unsigned fgrid = (unsigned)num_sms() * 8;
  {
    EG_PROF(PC_FIXUP, st);
    if (x_is_f64) {
      k_fixup<double><<<fgrid, 128, 0, st>>>((const double *)d_x, n, dim, d_r, length, W, d_codes,
                                             items, cnt, cap, cols);
      k_fixup_overflow<double><<<fgrid, 128, 0, st>>>((const double *)d_x, n, dim, d_r, length,
                                                      W, d_codes, cnt, cap, cols);
    } else {
      k_fixup<float><<<fgrid, 128, 0, st>>>((const float *)d_x, n, dim, d_r, length, W, d_codes,
                                            items, cnt, cap, cols);
      k_fixup_overflow<float><<<fgrid, 128, 0, st>>>((const float *)d_x, n, dim, d_r, length, W,
                                                     d_codes, cnt, cap, cols);
    }
  }
  EG_LAUNCH_CHECK();
  if (d_fixups)
    EG_CUDA_TRY(cudaMemcpyAsync(d_fixups, cnt, 8, cudaMemcpyDeviceToDevice, st));
  return EG_OK;
}


// ------------------------------------------------------------- MSM plan
// Block count for eg_msm_pairs (see plan.cuh).  Blocks follow the
// reference's partition rule (first length % k blocks one bit wider,
// bitpool.py:44-69) for every candidate k'.
static double comb_sat(int a, int b) {
  double r = 1;
  for (int i = 0; i < b; ++i) r = r * (a - i) / (i + 1);
  return r;
}

static void plan_kept(int length, int kk, uint64_t dropped_blocks, uint64_t kept[4]) {
  const int base = length / kk, rem = length % kk;
  for (int w = 0; w < 4; ++w) kept[w] = 0;
  int t = 0;
  for (int b = 0; b < kk; ++b) {
    const int wd = base + (b < rem ? 1 : 0);
    for (int q = 0; q < wd; ++q, ++t)
      if (!(dropped_blocks >> b & 1)) kept[t >> 6] |= 1ull << (t & 63);
  }
}


#include "designs.inc"
constexpr int PLAN_DESIGN_BASE = 10000;   // plan code of a table design: BASE + 100 v + m

static const DesignEntry *find_design(int v, int m, int t) {
  for (const DesignEntry &e : kDesigns)
    if (e.v == v && e.m == m && e.t == t) return &e;
  return nullptr;
}

int eg_msm_design(int32_t v, int32_t m, int32_t t, uint64_t *h_masks, int32_t capacity) {
  const DesignEntry *e = find_design(v, m, t);
  if (!e) return 0;
  if (h_masks)
    for (int i = 0; i < e->count && i < capacity; ++i) h_masks[i] = kDesignMasks[e->offset + i];
  return e->count;
}

constexpr int PLAN_REF_MAX = 4096;     // reference masks probed for the oversize check
constexpr int PLAN_PER_K = 12;         // masks probed per candidate block count
constexpr int PLAN_PER_DESIGN = 16;    // members probed per candidate design
constexpr int PLAN_MIN_ROWS = 65536;   // smaller pools keep the reference blocks

size_t eg_msm_plan_workspace(int32_t length, int32_t k, int32_t d) {
  (void)length; (void)k; (void)d;
  const size_t P = PLAN_REF_MAX + PLAN_PER_K * EG_MAX_BLOCKS +
                   PLAN_PER_DESIGN * (sizeof(kDesigns) / sizeof(kDesigns[0]));
  return ws_bytes(P * 4, 8) + ws_bytes(P, 8) + ws_bytes(P, 4) + ws_bytes(P, 4) + 1024;
}

int eg_msm_plan(const uint64_t *d_codes, int64_t n, int32_t length, int32_t k, int32_t d,
                double oversized_fraction, int32_t *h_k_out, double *h_cost, void *d_workspace,
                size_t workspace_bytes, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!h_k_out) return arg_error("eg_msm_plan: h_k_out is null");
  if (n < 1 || length < 1 || length > EG_MAX_LENGTH)
    return arg_error("eg_msm_plan: need n >= 1 and 1 <= length <= 256");
  if (!(0 <= d && d < k && k <= length) || k > EG_MAX_BLOCKS)
    return arg_error("eg_msm_plan: need 0 <= d < k <= min(length, 64)");
  *h_k_out = k;
  if (h_cost) h_cost[0] = h_cost[1] = 0;
  const int kmax = std::min(length, EG_MAX_BLOCKS);
  const int forced = options().msm_blocks;
  if (forced > 0) {
    if (forced > d && forced <= kmax) *h_k_out = forced;
    if (forced >= PLAN_DESIGN_BASE) {
      const int fv = (forced - PLAN_DESIGN_BASE) / 100, fm = (forced - PLAN_DESIGN_BASE) % 100;
      if (fv <= kmax && find_design(fv, fm, d)) *h_k_out = forced;
    }
    return EG_OK;
  }
  if (forced < 0 || n < PLAN_MIN_ROWS) return EG_OK;
  const double nref = comb_sat(k, d);
  if (nref > PLAN_REF_MAX) return EG_OK;
  const int W = (length + 63) / 64;
  const int S = (int)std::min<int64_t>(n, PLAN_SAMPLE);
  const int SR = (int)std::min<int64_t>(n, PLAN_REF_SAMPLE);
  // probes: every reference mask (oversize check), then PLAN_PER_K masks of
  // every candidate block count
  std::vector<uint64_t> kept;
  std::vector<int> probe_k;
  auto add = [&](int kk, uint64_t dropped, int label = 0) {
    uint64_t kw[4];
    plan_kept(length, kk, dropped, kw);
    kept.insert(kept.end(), kw, kw + 4);
    probe_k.push_back(label ? label : kk);
  };
  {
    std::vector<int> c(d);
    for (int i = 0; i < d; ++i) c[i] = i;
    while (true) {
      uint64_t m = 0;
      for (int i = 0; i < d; ++i) m |= 1ull << c[i];
      add(k, m);
      probe_k.back() = -1;     // reference probe: oversize check only
      int i = d - 1;
      while (i >= 0 && c[i] == k - d + i) --i;
      if (i < 0) break;
      ++c[i];
      for (int j = i + 1; j < d; ++j) c[j] = c[j - 1] + 1;
    }
  }
  const int nref_probes = (int)probe_k.size();
  // candidates: d < k' <= k + 2 (finer blocks than the reference's only pay
  // off marginally; coarser ones are where skewed or clustered codes win)
  const double lgn = std::log2((double)n);
  auto width_fits = [&](double kept_bits) {   // key widths worth a probe
    return kept_bits >= lgn - 1.0 && kept_bits <= lgn + 10.0;
  };
  for (int kk = d + 1; kk <= std::min(kmax, k + 2); ++kk) {
    const double units = comb_sat(kk, d);
    if (units > 8192) break;
    if (kk != k && !width_fits((double)length * (kk - d) / kk)) continue;
    if (units <= PLAN_PER_K) {
      std::vector<int> c(d);
      for (int i = 0; i < d; ++i) c[i] = i;
      while (true) {
        uint64_t m = 0;
        for (int i = 0; i < d; ++i) m |= 1ull << c[i];
        add(kk, m);
        int i = d - 1;
        while (i >= 0 && c[i] == kk - d + i) --i;
        if (i < 0) break;
        ++c[i];
        for (int j = i + 1; j < d; ++j) c[j] = c[j - 1] + 1;
      }
    } else {
      uint64_t rng = 0x9e3779b97f4a7c15ULL * (uint64_t)(kk + 1);
      std::vector<uint64_t> seen;
      while ((int)seen.size() < PLAN_PER_K) {
        uint64_t m = 0;
        int cnt = 0;
        while (cnt < d) {   // random d-subset of [0, kk)
          rng = rng * 6364136223846793005ULL + 1442695040888963407ULL;
          const int b = (int)((rng >> 33) % (uint64_t)kk);
          if (!(m >> b & 1)) { m |= 1ull << b; ++cnt; }
        }
        if (std::find(seen.begin(), seen.end(), m) != seen.end()) continue;
        seen.push_back(m);
        add(kk, m);
      }
    }
  }
  // covering designs of the table (t = d): fewer units than the complete
  // design of similar key width; PLAN_PER_DESIGN members probed each
  std::vector<double> design_units;      // by plan code - PLAN_DESIGN_BASE
  if (d >= 1 && options().msm_designs) {
    for (const DesignEntry &e : kDesigns) {
      if (e.t != d || e.v > kmax) continue;
      if (!width_fits((double)length * (e.v - e.m) / e.v)) continue;
      const int code = PLAN_DESIGN_BASE + 100 * e.v + e.m;
      const int np = std::min<int>(e.count, PLAN_PER_DESIGN);
      for (int i = 0; i < np; ++i)
        add(e.v, kDesignMasks[e.offset + (int64_t)i * e.count / np], code);
      if ((int)design_units.size() <= code - PLAN_DESIGN_BASE)
        design_units.resize(code - PLAN_DESIGN_BASE + 1, 0.0);
      design_units[code - PLAN_DESIGN_BASE] = e.count;
    }
  }
  const int P = (int)probe_k.size();
  std::vector<int> samples(P);
  for (int p = 0; p < P; ++p) samples[p] = p < nref_probes ? SR : S;
  Arena ar(d_workspace, workspace_bytes);
  unsigned long long *d_kept = ar.take<unsigned long long>((size_t)P * 4);
  unsigned long long *d_pairs = ar.take<unsigned long long>((size_t)P);
  uint32_t *d_max = ar.take<uint32_t>((size_t)P);
  int *d_samp = ar.take<int>((size_t)P);
  if (!d_kept || !d_pairs || !d_max || !d_samp) {
    set_error("eg_msm_plan: workspace too small");
    return EG_ERR_WORKSPACE;
  }
  EG_CUDA_TRY(cudaMemcpyAsync(d_kept, kept.data(), (size_t)P * 32, cudaMemcpyHostToDevice, st));
  EG_CUDA_TRY(cudaMemcpyAsync(d_samp, samples.data(), (size_t)P * 4, cudaMemcpyHostToDevice, st));
  const size_t smem = (size_t)PLAN_TABLE * 12;
  {
    EG_PROF(PC_MISC, st);
#define EG_PLAN_CASE(WW)                                                                     \
  case WW:                                                                                   \
    EG_SMEM_OPTIN(k_msm_plan<WW>, smem);                                                     \
    k_msm_plan<WW><<<P, PLAN_NT, smem, st>>>(d_codes, n, d_samp, d_kept, d_pairs, d_max);    \
    break;
    switch (W) {
      EG_PLAN_CASE(1)
      EG_PLAN_CASE(2)
      EG_PLAN_CASE(3)
      EG_PLAN_CASE(4)
    }
#undef EG_PLAN_CASE
  }
  EG_LAUNCH_CHECK();
  std::vector<unsigned long long> pairs(P);
  std::vector<uint32_t> mx(P);
  EG_CUDA_TRY(cudaMemcpyAsync(pairs.data(), d_pairs, (size_t)P * 8, cudaMemcpyDeviceToHost, st));
  EG_CUDA_TRY(cudaMemcpyAsync(mx.data(), d_max, (size_t)P * 4, cudaMemcpyDeviceToHost, st));
  EG_CUDA_TRY(cudaStreamSynchronize(st));
  // oversize check on the reference blocks: keep them whenever the
  // reference's warning (largest group > fraction * n) could fire, so the
  // caller's max_group is the reference's own
  uint32_t rmax = 0;
  for (int p = 0; p < nref_probes; ++p) rmax = std::max(rmax, mx[p]);
  if (SR == n) {
    if (n > 16 && rmax > oversized_fraction * (double)n) return EG_OK;
  } else if (oversized_fraction * SR < 200 || rmax >= 0.5 * oversized_fraction * SR) {
    return EG_OK;
  }
  // s per row per unit and per visited in-group pair: marginal costs fitted
  // on config 3 over the complete and the covering designs (tools/
  // design_sweep.sh; the member-parallel pair loop made visits cheap)
  const double ce = 14.0e-12;
  const double cp = 1.2e-12;
  const double scale = S > 1 ? (double)n * (double)(n - 1) / ((double)S * (double)(S - 1)) : 0;
  double best = -1, ref_cost = -1;
  int best_k = k;
  for (int p = nref_probes; p < P;) {
    const int kk = probe_k[p];
    double sum = 0;
    int cnt = 0;
    for (; p < P && probe_k[p] == kk; ++p, ++cnt) sum += (double)pairs[p];
    const double est_pairs = sum / cnt * scale;
    const double units =
        kk >= PLAN_DESIGN_BASE ? design_units[kk - PLAN_DESIGN_BASE] : comb_sat(kk, d);
    const double cost = units * ((double)n * ce + est_pairs * cp);
    if (options().plan_debug)
      fprintf(stderr, "[msm plan] code %d units %.0f probes %d est_pairs/unit %.3g cost %.3f ms\n",
              kk, units, cnt, est_pairs, cost * 1e3);
    if (kk == k) ref_cost = cost;
    if (best < 0 || cost < best) {
      best = cost;
      best_k = kk;
    }
  }
  if (ref_cost >= 0 && best >= 0.95 * ref_cost) best_k = k;   // not worth a change
  *h_k_out = best_k;
  if (h_cost) {
    h_cost[0] = (best_k == k ? ref_cost : best) * 1e3;
    h_cost[1] = ref_cost * 1e3;
  }
  return EG_OK;
}

// ------------------------------------------------------- output estimate
int eg_msm_estimate_pairs(const uint64_t *d_codes, int64_t n, int32_t W, int32_t replicates,
                          int32_t d, double *h_estimate, void *d_workspace,
                          size_t workspace_bytes, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!h_estimate || n < 0 || W < 1 || W > 4 || replicates < 1 || d < 0)
    return arg_error("eg_msm_estimate_pairs: bad arguments");
  h_estimate[0] = h_estimate[1] = 0.0;
  if (n < 2) return EG_OK;
  Arena ar(d_workspace, workspace_bytes);
  unsigned long long *cnt = ar.take<unsigned long long>(1);
  if (!cnt) return EG_ERR_WORKSPACE;
  const int S = (int)std::min<int64_t>(n, EST_SAMPLE);
  const int probed = std::min(replicates, EST_MAXREPS);
  const int nt = (S + EST_T - 1) / EST_T;
  EG_CUDA_TRY(cudaMemsetAsync(cnt, 0, 8, st));
  {
    EG_PROF(PC_MISC, st);
    k_est_pairs<<<dim3((unsigned)(nt * (nt + 1) / 2), (unsigned)probed), EST_T, 0, st>>>(
        d_codes, n, W, S, d, cnt);
  }
  EG_LAUNCH_CHECK();
  unsigned long long c = 0;
  EG_CUDA_TRY(cudaMemcpyAsync(&c, cnt, 8, cudaMemcpyDeviceToHost, st));
  EG_CUDA_TRY(cudaStreamSynchronize(st));
  const double scale = S > 1 ? (double)n * (double)(n - 1) / ((double)S * (double)(S - 1)) : 1.0;
  const double per_rep = (double)replicates / (double)probed;
  h_estimate[0] = (double)c * scale * per_rep;
  // ~4 sigma upper bound (sampled pairs ~ Poisson) plus 10 %
  h_estimate[1] = 1.1 * ((double)c + 4.0 * sqrt((double)c) + 4.0) * scale * per_rep;
  return EG_OK;
}

// ------------------------------------------------------------------ MSM
size_t eg_msm_workspace(int64_t n, int32_t length, int32_t replicates) {
  (void)length;
  return msm_layout(n, replicates).bytes;
}

int eg_msm_pairs(const uint64_t *d_codes, int64_t n, int32_t length, int32_t replicates,
                 const int32_t *h_block_bounds, int32_t k, int32_t d, const int32_t *h_unit_rep,
                 const uint64_t *h_unit_mask, int64_t n_units, uint64_t *d_out_keys,
                 uint16_t *d_out_rep, int64_t capacity, int64_t *h_counts, void *d_workspace,
                 size_t workspace_bytes, void *stream) {
  return eg_msm_pairs_design(d_codes, n, length, replicates, h_block_bounds, k, d, h_unit_rep,
                             h_unit_mask, n_units, nullptr, 0, d_out_keys, d_out_rep, capacity,
                             h_counts, d_workspace, workspace_bytes, stream);
}

// Does every d-subset of the k blocks lie inside a member of the family?
static bool design_covers(const uint64_t *fam, int nf, int k, int d) {
  if (d == 0) return nf > 0;
  std::vector<int> c(d);
  for (int i = 0; i < d; ++i) c[i] = i;
  while (true) {
    uint64_t m = 0;
    for (int i = 0; i < d; ++i) m |= 1ull << c[i];
    bool ok = false;
    for (int q = 0; q < nf && !ok; ++q) ok = (fam[q] & m) == m;
    if (!ok) return false;
    int i = d - 1;
    while (i >= 0 && c[i] == k - d + i) --i;
    if (i < 0) return true;
    ++c[i];
    for (int j = i + 1; j < d; ++j) c[j] = c[j - 1] + 1;
  }
}

int eg_msm_pairs_design(const uint64_t *d_codes, int64_t n, int32_t length, int32_t replicates,
                        const int32_t *h_block_bounds, int32_t k, int32_t d,
                        const int32_t *h_unit_rep, const uint64_t *h_unit_mask, int64_t n_units,
                        const uint64_t *h_design, int32_t n_design, uint64_t *d_out_keys,
                        uint16_t *d_out_rep, int64_t capacity, int64_t *h_counts,
                        void *d_workspace, size_t workspace_bytes, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n_design < 0 || n_design > MSM_MAXDESIGN || (n_design > 0 && !h_design))
    return arg_error("eg_msm_pairs: design of more than 64 members (or null)");
  if (n < 1 || n >= (1ll << 32)) return arg_error("eg_msm_pairs: need 1 <= n < 2^32");
  if (length < 1 || length > EG_MAX_LENGTH)
    return arg_error("eg_msm_pairs: length outside [1, 256]");
  if (!(0 <= d && d < k && k <= length) || k > EG_MAX_BLOCKS)
    return arg_error("eg_msm_pairs: need 0 <= d < k <= min(length, 64)");
  if (replicates < 1 || replicates > EG_MAX_REPLICATES)
    return arg_error("eg_msm_pairs: replicates outside [1, 65535] (the pair tag is 16 bits)");
  const int W = (length + 63) / 64;
  if (h_block_bounds[0] != 0 || h_block_bounds[k] != length)
    return arg_error("eg_msm_pairs: block bounds must span [0, length]");
  uint8_t b2b[EG_MAX_LENGTH];
  memset(b2b, 0, sizeof(b2b));
  for (int b = 0; b < k; ++b) {
    if (h_block_bounds[b + 1] <= h_block_bounds[b])
      return arg_error("eg_msm_pairs: block bounds must increase");
    for (int t = h_block_bounds[b]; t < h_block_bounds[b + 1]; ++t) b2b[t] = (uint8_t)b;
  }
  uint64_t all_bits[4] = {0, 0, 0, 0};
  for (int t = 0; t < length; ++t) all_bits[t >> 6] |= 1ull << (t & 63);
  auto kept_of = [&](uint64_t mb, unsigned long long *kept) {
    for (int w = 0; w < 4; ++w) kept[w] = all_bits[w];
    for (int b = 0; b < k; ++b)
      if (mb >> b & 1)
        for (int t = h_block_bounds[b]; t < h_block_bounds[b + 1]; ++t)
          kept[t >> 6] &= ~(1ull << (t & 63));
  };
  if (n_design > 0) {
    for (int q = 0; q < n_design; ++q)
      if (__builtin_popcountll(h_design[q]) < d || (k < 64 && (h_design[q] >> k)))
        return arg_error("eg_msm_pairs: design members must mask >= d of the k blocks");
    if (comb_sat(k, d) > 1048576.0 || !design_covers(h_design, n_design, k, d))
      return arg_error("eg_msm_pairs: the design does not cover every d-subset of the blocks");
  }

  MsmLayout lay = msm_layout(n, replicates);
  Arena ar(d_workspace, workspace_bytes);
  MsmArgs a;
  memset(&a, 0, sizeof(a));
  a.codes = d_codes;
  a.n = n;
  a.L = length;
  a.W = W;
  a.k = k;
  a.d = d;
  a.lgB = lay.lgB;
  a.B = lay.B;
  a.reps = replicates;
  uint8_t *b2b_d = ar.take<uint8_t>(EG_MAX_LENGTH);
  a.bit2blk = b2b_d;
  a.ctr = ar.take<unsigned long long>(3 + 2 * (size_t)replicates);
  a.spill_cap = (int64_t)lay.U * (lay.B + 1) * 3;   // a bucket is queued at most 3 times
  a.out_keys = (unsigned long long *)d_out_keys;
  a.out_rep = replicates > 1 ? d_out_rep : nullptr;
  a.out_cap = capacity > 0 ? (unsigned long long)capacity : 0ull;
  if (!b2b_d || !a.ctr) {
    set_error("eg_msm_pairs: workspace too small (%zu < %zu)", workspace_bytes, lay.bytes);
    return EG_ERR_WORKSPACE;
  }
  MsmArgs sets[2];
  for (int si = 0; si < lay.sets; ++si) {
    MsmArgs &x = sets[si];
    x = a;
    x.counts = ar.take<uint32_t>((size_t)lay.U * lay.B);
    x.starts = ar.take<uint32_t>((size_t)lay.U * (lay.B + 1));
    x.cursor = ar.take<uint32_t>((size_t)lay.U * lay.B);
    x.elems = ar.take<uint64_t>((size_t)lay.U * n);
    x.gcnt = ar.take<uint32_t>((size_t)lay.U * n);
    x.spill = ar.take<uint32_t>((size_t)lay.U * (lay.B + 1) * 9);
    x.spill_ctr = ar.take<unsigned long long>(2);
    if (!x.counts || !x.starts || !x.cursor || !x.elems || !x.gcnt || !x.spill || !x.spill_ctr) {
      set_error("eg_msm_pairs: workspace too small (%zu < %zu)", workspace_bytes, lay.bytes);
      return EG_ERR_WORKSPACE;
    }
    EG_CUDA_TRY(cudaMemsetAsync(x.counts, 0, (size_t)lay.U * lay.B * 4, st));
  }
  if (lay.sets == 1) sets[1] = sets[0];
  EG_CUDA_TRY(cudaMemsetAsync(a.ctr, 0, (3 + 2 * (size_t)replicates) * 8, st));
  EG_CUDA_TRY(cudaMemcpyAsync(b2b_d, b2b, EG_MAX_LENGTH, cudaMemcpyHostToDevice, st));

  // balanced batches of <= lay.U units; at least two when there are a few
  // units (a sharded rank's share), so the second batch's hist / scatter
  // overlap the first batch's grouping on the side stream
  std::vector<UnitBatch> batches;
  const int64_t min_batches = (n_units + lay.U - 1) / lay.U;   // scratch capacity
  int64_t nbatch = min_batches;
  if (lay.sets == 2 && n_units >= 4)
    nbatch = std::max<int64_t>(nbatch, std::min<int64_t>(2, n_units / 2));
  if (options().msm_batches > 0)
    nbatch = std::max<int64_t>(min_batches, std::min<int64_t>(options().msm_batches, n_units));
  const int64_t per_batch = nbatch > 0 ? (n_units + nbatch - 1) / nbatch : lay.U;
  for (int64_t u0 = 0; u0 < n_units; u0 += per_batch) {
    UnitBatch ub;
    memset(&ub, 0, sizeof(ub));
    ub.count = (int)std::min<int64_t>(per_batch, n_units - u0);
    ub.ndesign = n_design;
    for (int q = 0; q < n_design; ++q) kept_of(h_design[q], ub.dkept[q]);
    for (int j = 0; j < ub.count; ++j) {
      const int rep = h_unit_rep[u0 + j];
      const uint64_t mb = h_unit_mask[u0 + j];
      if (rep < 0 || rep >= replicates) return arg_error("eg_msm_pairs: unit replicate out of range");
      if (n_design > 0) {
        const uint64_t *hit = std::find(h_design, h_design + n_design, mb);
        if (hit == h_design + n_design)
          return arg_error("eg_msm_pairs: unit mask is not a member of the design");
        ub.dq[j] = (uint8_t)(hit - h_design);
      } else if (__builtin_popcountll(mb) != d || (k < 64 && (mb >> k))) {
        return arg_error("eg_msm_pairs: unit mask must select exactly d of the k blocks");
      }
      ub.rep[j] = rep;
      ub.maskbits[j] = mb;
      kept_of(mb, ub.kept[j]);
      ub.salt[j] = 0x2545f4914f6cdd1dULL * (uint64_t)(u0 + j + 1);
      // tail blocks: masked blocks above the lowest kept block
      int lowest_kept = 0;
      while (lowest_kept < k && (mb >> lowest_kept & 1)) ++lowest_kept;
      int nt = 0;
      for (int b = lowest_kept + 1; b < k; ++b) {
        if (!(mb >> b & 1)) continue;
        if (nt < MSM_MAXT) {
          ub.tail_lo[j][nt] = (uint16_t)h_block_bounds[b];
          ub.tail_hi[j][nt] = (uint16_t)h_block_bounds[b + 1];
        }
        ++nt;
      }
      ub.ntail[j] = (uint8_t)std::min(nt, 255);
    }
    batches.push_back(ub);
  }
  int rc = EG_OK;
  {
    EG_PROF_GROUP(PC_MSM_STAGE, st);
    switch (W) {
      case 1: rc = msm_run<1>(sets, lay, batches, st); break;
      case 2: rc = msm_run<2>(sets, lay, batches, st); break;
      case 3: rc = msm_run<3>(sets, lay, batches, st); break;
      default: rc = msm_run<4>(sets, lay, batches, st); break;
    }
  }
  if (rc) return rc;
  std::vector<unsigned long long> hc(3 + 2 * (size_t)replicates);
  EG_CUDA_TRY(cudaMemcpyAsync(hc.data(), a.ctr, hc.size() * 8, cudaMemcpyDeviceToHost, st));
  EG_CUDA_TRY(cudaStreamSynchronize(st));
  h_counts[0] = (int64_t)hc[0];
  h_counts[1] = (int64_t)hc[1];
  for (int h = 0; h < 2 * replicates; ++h) h_counts[2 + h] = (int64_t)hc[3 + h];
  if (hc[0] > a.out_cap) {
    set_error("eg_msm_pairs: %llu pairs exceed capacity %llu", hc[0], a.out_cap);
    return EG_ERR_CAPACITY;
  }
  return EG_OK;
}

int eg_xrep_filter_async(const uint64_t *d_keys, const uint16_t *d_reps, int64_t m,
                         const uint64_t *d_codes, int64_t n, int32_t W, int32_t d,
                         int32_t replicates, uint8_t *d_keep, uint64_t *d_new_counts,
                         void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (replicates < 1 || replicates > EG_MAX_REPLICATES || W < 1 || m < 0)
    return arg_error("eg_xrep_filter: bad arguments");
  EG_CUDA_TRY(cudaMemsetAsync(d_new_counts, 0, 8 * (size_t)replicates, st));
  if (m > 0) {
    unsigned grid = (unsigned)std::min<int64_t>((m + 255) / 256, (int64_t)num_sms() * 16);
    EG_PROF(PC_MISC, st);
    k_xrep_filter<<<grid, 256, 0, st>>>(const_cast<uint64_t *>(d_keys), d_reps, m, d_codes, n, W,
                                        d, replicates, d_keep,
                                        (unsigned long long *)d_new_counts);
    EG_LAUNCH_CHECK();
  }
  return EG_OK;
}

int eg_xrep_filter(const uint64_t *d_keys, const uint16_t *d_reps, int64_t m,
                   const uint64_t *d_codes, int64_t n, int32_t W, int32_t d, int32_t replicates,
                   uint8_t *d_keep, int64_t *h_new_counts, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (replicates < 1 || replicates > EG_MAX_REPLICATES)
    return arg_error("eg_xrep_filter: replicates outside [1, 65535]");
  // per-device counter block, allocated once: a stream-ordered allocation
  // here released its pool at every synchronise and stalled some calls by
  // tens of ms.  The mutex covers the call up to its final synchronise.
  static std::mutex mu;
  static unsigned long long *small[64];
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  EG_CUDA_TRY(cudaGetDevice(&dev));
  if (!small[dev]) EG_CUDA_TRY(cudaMalloc(&small[dev], 8 * (size_t)EG_MAX_REPLICATES));
  unsigned long long *nc = small[dev];
  EG_CUDA_TRY(cudaMemsetAsync(nc, 0, 8 * (size_t)replicates, st));
  if (m > 0) {
    unsigned grid = (unsigned)std::min<int64_t>((m + 255) / 256, (int64_t)num_sms() * 16);
    EG_PROF(PC_MISC, st);
    k_xrep_filter<<<grid, 256, 0, st>>>(const_cast<uint64_t *>(d_keys), d_reps, m, d_codes, n, W,
                                        d, replicates, d_keep, nc);
    EG_LAUNCH_CHECK();
  }
  std::vector<unsigned long long> h(replicates);
  EG_CUDA_TRY(cudaMemcpyAsync(h.data(), nc, 8 * (size_t)replicates, cudaMemcpyDeviceToHost, st));
  EG_CUDA_TRY(cudaStreamSynchronize(st));
  for (int i = 0; i < replicates; ++i) h_new_counts[i] = (int64_t)h[i];
  return EG_OK;
}

// ---------------------------------------------------- full-code filter
int eg_hamming_filter_async(const uint64_t *d_keys, const uint16_t *d_reps, int64_t m,
                            const uint64_t *d_codes, int64_t n, int32_t W, int32_t d,
                            int32_t replicates, uint8_t *d_keep, uint64_t *d_raw_counts,
                            void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (replicates < 1 || replicates > EG_MAX_REPLICATES || W < 1 || m < 0 || d < 0)
    return arg_error("eg_hamming_filter: bad arguments");
  EG_CUDA_TRY(cudaMemsetAsync(d_raw_counts, 0, 8 * (size_t)replicates, st));
  if (m > 0) {
    unsigned grid = (unsigned)std::min<int64_t>((m + 255) / 256, (int64_t)num_sms() * 16);
    EG_PROF(PC_MISC, st);
    k_hamming_filter<<<grid, 256, 0, st>>>(d_keys, d_reps, m, d_codes, n, W, d, replicates,
                                           d_keep, (unsigned long long *)d_raw_counts);
    EG_LAUNCH_CHECK();
  }
  return EG_OK;
}

// --------------------------------------------------------- grouped sort
size_t eg_grouped_sort_workspace(int64_t n, int32_t chunk_bits) {
  const int cb = chunk_bits < 1 ? 1 : (chunk_bits > 24 ? 24 : chunk_bits);
  return ws_bytes(n, 8) + 2 * ws_bytes(n, 4) + ws_bytes(n, 1) + ws_bytes(n, 8) +
         ws_bytes((size_t)1 << cb, 4) + ws_bytes(EG_MAX_LENGTH, 4) +
         radix_workspace(n, true) + compact_workspace(n) + 4096;
}

int eg_grouped_sort(const uint64_t *d_codes, int64_t n, int32_t length,
                    const int32_t *h_block_bounds, int32_t k, uint64_t mask_bits,
                    int32_t chunk_bits, uint32_t *d_perm, int64_t *d_bounds, int64_t *h_groups,
                    void *d_workspace, size_t workspace_bytes, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 1 || n >= (1ll << 32)) return arg_error("eg_grouped_sort: need 1 <= n < 2^32");
  if (length < 1 || length > EG_MAX_LENGTH || k < 1 || k > length || k > EG_MAX_BLOCKS)
    return arg_error("eg_grouped_sort: bad length/k");
  if (chunk_bits < 1 || chunk_bits > 24) return arg_error("chunk_bits must be in [1, 24]");
  const int W = (length + 63) / 64;
  // kept bit positions in ascending order (bitpool._kept_positions)
  std::vector<int32_t> cols;
  UnitBatch ub;
  memset(&ub, 0, sizeof(ub));
  ub.count = 1;
  for (int b = 0; b < k; ++b) {
    if (mask_bits >> b & 1) continue;
    for (int t = h_block_bounds[b]; t < h_block_bounds[b + 1]; ++t) {
      cols.push_back(t);
      ub.kept[0][t >> 6] |= 1ull << (t & 63);
    }
  }
  const int ncols = (int)cols.size();
  Arena ar(d_workspace, workspace_bytes);
  uint64_t *key = ar.take<uint64_t>(n);
  uint32_t *val = ar.take<uint32_t>(n);
  uint32_t *vbuf = ar.take<uint32_t>(n);
  uint8_t *flags = ar.take<uint8_t>(n);
  uint64_t *idx = ar.take<uint64_t>(n);
  uint32_t *first = ar.take<uint32_t>((size_t)1 << chunk_bits);
  int32_t *d_cols = ar.take<int32_t>(EG_MAX_LENGTH);
  if (!key || !val || !vbuf || !flags || !idx || !first || !d_cols) {
    set_error("eg_grouped_sort: workspace too small");
    return EG_ERR_WORKSPACE;
  }
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 4096);
  {
    EG_PROF(PC_MISC, st);
    k_iota<<<grid, 256, 0, st>>>(d_perm, n);
  }
  EG_LAUNCH_CHECK();
  if (ncols == 0) {   // every block masked: one group
    int64_t b2[2] = {0, n};
    EG_CUDA_TRY(cudaMemcpyAsync(d_bounds, b2, 16, cudaMemcpyHostToDevice, st));
    EG_CUDA_TRY(cudaStreamSynchronize(st));
    *h_groups = 1;
    return EG_OK;
  }
  EG_CUDA_TRY(cudaMemcpyAsync(d_cols, cols.data(), (size_t)ncols * 4, cudaMemcpyHostToDevice, st));
  const int nch = (ncols + chunk_bits - 1) / chunk_bits;
  int shifts[8], np = 0;
  for (int sft = 0; sft < ilog2_ceil((uint64_t)std::max<int64_t>(n, 2)); sft += 8) shifts[np++] = sft;
  size_t mark = ar.used;
  for (int c = nch - 1; c >= 0; --c) {   // last chunk first (hamming_join.py:267)
    EG_CUDA_TRY(cudaMemsetAsync(first, 0xff, ((size_t)1 << chunk_bits) * 4, st));
    {
      EG_PROF(PC_MISC, st);
      k_chunk_first<<<grid, 256, 0, st>>>(d_codes, d_perm, n, W, d_cols, c * chunk_bits,
                                          chunk_bits, ncols, first, vbuf);
      k_chunk_rank<<<grid, 256, 0, st>>>(vbuf, first, d_perm, n, key, val);
    }
    EG_LAUNCH_CHECK();
    ar.used = mark;
    int rc = radix_sort(key, val, n, shifts, np, ar, st);
    if (rc) return rc;
    EG_CUDA_TRY(cudaMemcpyAsync(d_perm, val, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
  }
  ar.used = mark;
  {
    EG_PROF(PC_MISC, st);
    k_group_flags<4><<<grid, 256, 0, st>>>(d_codes, d_perm, n, W, ub, flags, idx);
  }
  EG_LAUNCH_CHECK();
  int64_t groups = 0;
  int rc = compact<uint32_t>(idx, (const uint32_t *)nullptr, flags, n, (uint64_t *)d_bounds,
                             (uint32_t *)nullptr, &groups, ar, st);
  if (rc) return rc;
  int64_t nn = n;
  EG_CUDA_TRY(cudaMemcpyAsync(d_bounds + groups, &nn, 8, cudaMemcpyHostToDevice, st));
  EG_CUDA_TRY(cudaStreamSynchronize(st));
  *h_groups = groups;
  return EG_OK;
}

// -------------------------------------------------------- first witness
int eg_first_witness(const uint64_t *d_keys, int64_t m, const uint64_t *const *d_pools,
                     int32_t n_pools, int32_t W, int32_t d, uint8_t *d_keep, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (m <= 0) return EG_OK;
  unsigned grid = (unsigned)std::min<int64_t>((m + 255) / 256, 8192);
  EG_PROF(PC_MISC, st);
  k_first_witness<<<grid, 256, 0, st>>>(d_keys, m, d_pools, n_pools, W, d, d_keep);
  EG_LAUNCH_CHECK();
  return EG_OK;
}

// ----------------------------------------------------------------- sort
size_t eg_sort_workspace(int64_t m, int with_values) { return radix_workspace(m, with_values != 0); }

int eg_sort_keys(uint64_t *d_keys, uint32_t *d_vals, int64_t m, int32_t key_bits,
                 void *d_workspace, size_t workspace_bytes, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (key_bits < 0 || key_bits > 64) return arg_error("eg_sort_keys: key_bits outside [0, 64]");
  int shifts[8], np = 0;
  for (int s = 0; s < key_bits; s += 8) shifts[np++] = s;
  Arena ar(d_workspace, workspace_bytes);
  return radix_sort(d_keys, d_vals, m, shifts, np, ar, st);
}

int eg_sort_pair_keys(uint64_t *d_keys, int64_t m, int64_t n, void *d_workspace,
                      size_t workspace_bytes, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int shifts[8];
  int np = pair_key_shifts(n, shifts);
  Arena ar(d_workspace, workspace_bytes);
  EG_PROF_GROUP(PC_SORT_STAGE, st);
  return radix_sort(d_keys, nullptr, m, shifts, np, ar, st);
}

// ----------------------------------------------------------- merge runs
size_t eg_merge_runs_workspace(int64_t m, int with_values) {
  return ws_bytes(m, 8) * (with_values ? 2 : 1) + 1024;
}

int eg_merge_runs(uint64_t *d_keys, uint64_t *d_vals, const int64_t *h_offsets, int32_t runs,
                  void *d_workspace, size_t workspace_bytes, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (runs < 1 || !h_offsets) return arg_error("eg_merge_runs: need >= 1 run");
  const int64_t m = h_offsets[runs] - h_offsets[0];
  if (m < 0) return arg_error("eg_merge_runs: offsets must increase");
  for (int r = 0; r < runs; ++r)
    if (h_offsets[r + 1] < h_offsets[r]) return arg_error("eg_merge_runs: offsets must increase");
  if (runs == 1 || m == 0) return EG_OK;
  Arena ar(d_workspace, workspace_bytes);
  uint64_t *tk = ar.take<uint64_t>(m);
  uint64_t *tv = d_vals ? ar.take<uint64_t>(m) : nullptr;
  if (!tk || (d_vals && !tv)) {
    set_error("eg_merge_runs: workspace too small");
    return EG_ERR_WORKSPACE;
  }
  std::vector<int64_t> off(h_offsets, h_offsets + runs + 1);
  for (int64_t &o : off) o -= h_offsets[0];
  uint64_t *src = d_keys, *srcv = d_vals, *dst = tk, *dstv = tv;
  while (off.size() > 2) {   // one round: merge neighbouring runs pairwise
    std::vector<int64_t> next;
    for (size_t r = 0; r + 1 < off.size(); r += 2) {
      next.push_back(off[r]);
      if (r + 2 < off.size()) {
        const int64_t na = off[r + 1] - off[r], nb = off[r + 2] - off[r + 1];
        const int64_t tot = na + nb;
        const unsigned grid = (unsigned)std::max<int64_t>(
            1, std::min<int64_t>((tot + MP_NT * MP_IT - 1) / (MP_NT * MP_IT),
                                 (int64_t)num_sms() * 16));
        EG_PROF(PC_SORT_DOWNSWEEP, st);
        k_merge_path<<<grid, MP_NT, 0, st>>>(src + off[r], srcv ? srcv + off[r] : nullptr, na,
                                             src + off[r + 1], srcv ? srcv + off[r + 1] : nullptr,
                                             nb, dst + off[r], dstv ? dstv + off[r] : nullptr);
      } else {   // odd run out: carried over
        const int64_t len = off[r + 1] - off[r];
        EG_CUDA_TRY(cudaMemcpyAsync(dst + off[r], src + off[r], len * 8, cudaMemcpyDeviceToDevice, st));
        if (srcv)
          EG_CUDA_TRY(cudaMemcpyAsync(dstv + off[r], srcv + off[r], len * 8,
                                      cudaMemcpyDeviceToDevice, st));
      }
    }
    next.push_back(off.back());
    off.swap(next);
    std::swap(src, dst);
    std::swap(srcv, dstv);
  }
  EG_LAUNCH_CHECK();
  if (src != d_keys) {
    EG_CUDA_TRY(cudaMemcpyAsync(d_keys, src, m * 8, cudaMemcpyDeviceToDevice, st));
    if (d_vals) EG_CUDA_TRY(cudaMemcpyAsync(d_vals, srcv, m * 8, cudaMemcpyDeviceToDevice, st));
  }
  return EG_OK;
}

// ------------------------------------------------------------ compaction
size_t eg_compact_workspace(int64_t m) { return compact_workspace(m); }

int eg_compact_keys(const uint64_t *d_keys, const uint8_t *d_flags, int64_t m, uint64_t *d_out,
                    int64_t *h_count, void *d_workspace, size_t workspace_bytes, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  Arena ar(d_workspace, workspace_bytes);
  return compact<uint32_t>(d_keys, (const uint32_t *)nullptr, d_flags, m, d_out,
                           (uint32_t *)nullptr, h_count, ar, st);
}

// --------------------------------------------------------------- verify
size_t eg_verify_workspace(int64_t m) {
  return ws_bytes(m, 1) + ws_bytes(m, 8) + ws_bytes(1, 8) + compact_workspace(m) + 1024;
}

int eg_verify(const void *d_x, int x_is_f64, int64_t n, int32_t dim, const double *d_norms,
              const uint64_t *d_keys, int64_t m, int32_t metric, double eps, uint64_t *d_out_keys,
              double *d_out_dist, int64_t *h_count, void *d_workspace, size_t workspace_bytes,
              void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  *h_count = 0;
  if (m <= 0) return EG_OK;
  if (metric != EG_METRIC_COSINE && metric != EG_METRIC_EUCLIDEAN)
    return arg_error("eg_verify: unknown metric");
  Arena ar(d_workspace, workspace_bytes);
  uint8_t *flags = ar.take<uint8_t>(m);
  double *dist = ar.take<double>(m);
  unsigned long long *bad = ar.take<unsigned long long>(1);
  if (!flags || !dist || !bad) return EG_ERR_WORKSPACE;
  EG_PROF_GROUP(PC_VERIFY_STAGE, st);
  EG_CUDA_TRY(cudaMemsetAsync(bad, 0xff, 8, st));
  unsigned grid = (unsigned)std::min<int64_t>((m + 7) / 8, (int64_t)num_sms() * 64);
  {
  EG_PROF(PC_VERIFY, st);
  const int vu = (!x_is_f64 && dim % 4 == 0 && dim <= 128 * VER_VU) ? (dim + 127) / 128 : 0;
  const bool narrow = !x_is_f64 && dim % 4 == 0 && dim <= 128 && !options().verify_wide;
  if (narrow) {
    // eight lanes per pair, four pairs per warp step (measured: 4 lanes per
    // pair is slower on configs 4 and 5)
    const int lp = 8;
    const unsigned g8 = (unsigned)std::min<int64_t>((m * lp + 255) / 256, (int64_t)num_sms() * 64);
    const int v8 = (dim / 4 + lp - 1) / lp;
#define EG_V8(LP, V)                                                                           \
  k_verify8<LP, V><<<g8, 256, 0, st>>>((const float *)d_x, n, dim, d_norms, d_keys, m, metric, \
                                       eps, flags, dist, bad)
    if (v8 <= 1) EG_V8(8, 1); else if (v8 == 2) EG_V8(8, 2); else if (v8 == 3) EG_V8(8, 3);
    else EG_V8(8, 4);
#undef EG_V8
  } else if (x_is_f64)
    k_verify<double, 0><<<grid, 256, 0, st>>>((const double *)d_x, n, dim, d_norms, d_keys, m,
                                              metric, eps, flags, dist, bad);
  else if (vu == 1)
    k_verify<float, 1><<<grid, 256, 0, st>>>((const float *)d_x, n, dim, d_norms, d_keys, m,
                                             metric, eps, flags, dist, bad);
  else if (vu == 2)
    k_verify<float, 2><<<grid, 256, 0, st>>>((const float *)d_x, n, dim, d_norms, d_keys, m,
                                             metric, eps, flags, dist, bad);
  else if (vu == 3)
    k_verify<float, 3><<<grid, 256, 0, st>>>((const float *)d_x, n, dim, d_norms, d_keys, m,
                                             metric, eps, flags, dist, bad);
  else if (vu == 4)
    k_verify<float, 4><<<grid, 256, 0, st>>>((const float *)d_x, n, dim, d_norms, d_keys, m,
                                             metric, eps, flags, dist, bad);
  else
    k_verify<float, 0><<<grid, 256, 0, st>>>((const float *)d_x, n, dim, d_norms, d_keys, m,
                                             metric, eps, flags, dist, bad);
  }
  EG_LAUNCH_CHECK();
  // the out-of-range flag rides on the compaction's synchronisation
  unsigned long long *pin = pinned_small();
  if (pin) EG_CUDA_TRY(cudaMemcpyAsync(pin, bad, 8, cudaMemcpyDeviceToHost, st));
  int rc = compact<double>(d_keys, dist, flags, m, d_out_keys, d_out_dist, h_count, ar, st);
  if (rc) return rc;
  unsigned long long hb = 0;
  if (pin) {
    hb = pin[0];
  } else {
    EG_CUDA_TRY(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, st));
    EG_CUDA_TRY(cudaStreamSynchronize(st));
  }
  if (hb != ~0ull) {
    set_error("eg_verify: candidate %llu has an index out of range", hb);
    return EG_ERR_ARG;
  }
  return EG_OK;
}


// ------------------------------------------------------ exhaustive oracle
// TMA descriptor of the fp16 unit rows (row stride dp): box 64 x rows, SW128.
static bool make_f16_map(CUtensorMap *map, const void *d_u, int64_t n, int dp, int rows) {
  static PFN_cuTensorMapEncodeTiled encode = nullptr;
  if (!encode) {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = (PFN_cuTensorMapEncodeTiled)fn;
  }
  cuuint64_t gdim[2] = {(cuuint64_t)dp, (cuuint64_t)n};
  cuuint64_t gstride[1] = {(cuuint64_t)dp * 2};
  cuuint32_t box[2] = {BF_BK, (cuuint32_t)rows};
  cuuint32_t estride[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void *>(d_u), gdim, gstride,
                box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

size_t eg_bf_cosine_workspace(int64_t n, int32_t dim) {
  return ws_bytes((size_t)n * bf_dpad(dim), 2) + ws_bytes(1, 8) + 1024;
}

int eg_bf_cosine_candidates(const void *d_x, int x_is_f64, int64_t n, int32_t dim,
                            const double *d_norms, double eps, uint64_t *d_keys, int64_t cap,
                            int64_t *h_count, void *d_workspace, size_t workspace_bytes,
                            void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  *h_count = 0;
  if (n < 0 || dim < 1 || cap < 0) return arg_error("eg_bf_cosine_candidates: bad shape");
  if (n >= (1ll << 31)) return arg_error("eg_bf_cosine_candidates: too many rows");
  const int dp = bf_dpad(dim);
  if (dp > 512)
    {
      set_error("eg_bf_cosine_candidates: dim > 512 (the A tile is kept in shared memory)");
      return EG_ERR_UNSUPPORTED;
    }
  if (n < 2) return EG_OK;
  Arena ar(d_workspace, workspace_bytes);
  __half *u = ar.take<__half>((size_t)n * dp);
  unsigned long long *cnt = ar.take<unsigned long long>(1);
  if (!u || !cnt) {
    set_error("eg_bf_cosine_candidates: workspace too small");
    return EG_ERR_WORKSPACE;
  }
  EG_CUDA_TRY(cudaMemsetAsync(cnt, 0, 8, st));
  const unsigned g = (unsigned)std::min<int64_t>((n * dp + 255) / 256, (int64_t)num_sms() * 16);
  if (x_is_f64)
    k_unit_f16<double><<<g, 256, 0, st>>>((const double *)d_x, n, dim, dp, d_norms, u);
  else
    k_unit_f16<float><<<g, 256, 0, st>>>((const float *)d_x, n, dim, dp, d_norms, u);
  EG_LAUNCH_CHECK();
  CUtensorMap amap, bmap;
  if (!make_f16_map(&amap, u, n, dp, BF_BM) || !make_f16_map(&bmap, u, n, dp, BF_BN))
    {
    set_error("eg_bf_cosine_candidates: tensor map encoding failed");
    return EG_ERR_UNSUPPORTED;
  }
  // screen: fp16 unit rows (2 x 2^-11 relative each, 2^-25 subnormal floor)
  // and fp32 accumulation over dp / 16 MMAs -- |error| < 1.1e-3 for unit
  // rows; 4x margin
  const double delta = 4.0 * (2.0 * ldexp(1.0, -11) + ldexp(1.0, -22) +
                              sqrt((double)dp) * ldexp(1.0, -24) +
                              (dp / 16) * ldexp(1.0, -22));
  const float thr = (float)(1.0 - eps - delta);
  const int nkc = dp / BF_BK;
  const size_t budget = ((size_t)220 << 10) - sizeof(BfBars) - 1024;
  const int nb = (int)std::min<size_t>(BF_MAXSTAGES, (budget - nkc * BF_ACHUNK) / BF_BSTAGE);
  const size_t smem = nkc * BF_ACHUNK + nb * BF_BSTAGE + sizeof(BfBars) + 1024;
  EG_SMEM_OPTIN(k_bf_cosine_tc, smem);
  const int64_t ti = (n + BF_BM - 1) / BF_BM;
  const unsigned grid = (unsigned)std::min<int64_t>(ti, (int64_t)num_sms());
  {
    EG_PROF(PC_VERIFY, st);
    k_bf_cosine_tc<<<grid, BF_THREADS, smem, st>>>(amap, bmap, n, dp, nb, thr,
                                                   (unsigned long long *)d_keys,
                                                   (unsigned long long)cap, cnt);
  }
  EG_LAUNCH_CHECK();
  EG_CUDA_TRY(cudaMemcpyAsync(h_count, cnt, 8, cudaMemcpyDeviceToHost, st));
  EG_CUDA_TRY(cudaStreamSynchronize(st));
  return EG_OK;
}

size_t eg_bf_hamming_workspace(void) { return ws_bytes(1, 8) + 256; }

int eg_bf_hamming(const uint64_t *d_codes, int64_t n, int32_t words, int32_t d, uint64_t *d_keys,
                  int64_t cap, int64_t *h_count, void *d_workspace, size_t workspace_bytes,
                  void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  *h_count = 0;
  if (n < 0 || words < 1 || words > BFH_MAXW || d < 0 || cap < 0)
    return arg_error("eg_bf_hamming: bad arguments");
  if (n >= (1ll << 32)) return arg_error("eg_bf_hamming: too many rows");
  if (n < 2) return EG_OK;
  Arena ar(d_workspace, workspace_bytes);
  unsigned long long *cnt = ar.take<unsigned long long>(1);
  if (!cnt) {
    set_error("eg_bf_hamming: workspace too small");
    return EG_ERR_WORKSPACE;
  }
  EG_CUDA_TRY(cudaMemsetAsync(cnt, 0, 8, st));
  const int64_t nblk = (n + BFH_ROWS - 1) / BFH_ROWS;
  dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((n + BFH_NT - 1) / BFH_NT, 64)),
            (unsigned)std::min<int64_t>(nblk, 65535));
  {
    EG_PROF(PC_MSM_GROUP, st);
    k_bf_hamming<<<grid, BFH_NT, 0, st>>>(d_codes, n, words, d, (unsigned long long *)d_keys,
                                          (unsigned long long)cap, cnt);
  }
  EG_LAUNCH_CHECK();
  EG_CUDA_TRY(cudaMemcpyAsync(h_count, cnt, 8, cudaMemcpyDeviceToHost, st));
  EG_CUDA_TRY(cudaStreamSynchronize(st));
  return EG_OK;
}


// --------------------------------------------------------- edge text
size_t eg_format_edges_workspace(int64_t m) {
  return ws_bytes(m + 1, 4) + scan_workspace(m + 1) + ws_bytes(1, 8) + 1024;
}

int eg_format_edges(const uint64_t *d_keys, const double *d_dist, int64_t m, char *d_out,
                    int64_t out_cap, int64_t *h_bytes, void *d_workspace,
                    size_t workspace_bytes, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  *h_bytes = 0;
  if (m < 0 || m > EG_FORMAT_MAX_EDGES) return arg_error("eg_format_edges: 0 <= m <= 2^26");
  if (m == 0) return EG_OK;
  Arena ar(d_workspace, workspace_bytes);
  uint32_t *len = ar.take<uint32_t>(m + 1);
  unsigned long long *bad = ar.take<unsigned long long>(1);
  if (!len || !bad) {
    set_error("eg_format_edges: workspace too small");
    return EG_ERR_WORKSPACE;
  }
  EG_CUDA_TRY(cudaMemsetAsync(bad, 0xff, 8, st));
  EG_CUDA_TRY(cudaMemsetAsync(len + m, 0, 4, st));
  const unsigned g = (unsigned)std::min<int64_t>((m + 255) / 256, (int64_t)num_sms() * 16);
  k_edge_len<<<g, 256, 0, st>>>(d_keys, d_dist, m, len, bad);
  EG_LAUNCH_CHECK();
  int rc = scan_exclusive_u32(len, len, m + 1, ar, st);
  if (rc) return rc;
  unsigned long long *pin = pinned_small();
  uint32_t total = 0;
  unsigned long long hb = 0;
  if (pin) {
    EG_CUDA_TRY(cudaMemcpyAsync(pin, len + m, 4, cudaMemcpyDeviceToHost, st));
    EG_CUDA_TRY(cudaMemcpyAsync(pin + 1, bad, 8, cudaMemcpyDeviceToHost, st));
    EG_CUDA_TRY(cudaStreamSynchronize(st));
    total = (uint32_t)(pin[0] & 0xffffffffull);
    hb = pin[1];
  } else {
    EG_CUDA_TRY(cudaMemcpyAsync(&total, len + m, 4, cudaMemcpyDeviceToHost, st));
    EG_CUDA_TRY(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, st));
    EG_CUDA_TRY(cudaStreamSynchronize(st));
  }
  if (hb != ~0ull) {
    set_error("eg_format_edges: distance of edge %llu is outside the %%.9f range", hb);
    return EG_ERR_UNSUPPORTED;
  }
  *h_bytes = (int64_t)total;
  if ((int64_t)total > out_cap) {
    set_error("eg_format_edges: %u bytes exceed capacity %lld", total, (long long)out_cap);
    return EG_ERR_CAPACITY;
  }
  k_edge_write<<<g, 256, 0, st>>>(d_keys, d_dist, m, len, d_out);
  EG_LAUNCH_CHECK();
  return EG_OK;
}

}  // extern "C"
