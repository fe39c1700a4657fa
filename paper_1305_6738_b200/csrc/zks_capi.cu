// C ABI of the engine (include/zipfks_b200.h): engine / table lifetime, launches, errors.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <tuple>
#include <vector>
#include <string>

#include "../../include/zipfks_b200.h"
#include "zks_replicate.cuh"
#include "zks_batch.cuh"
#include "zks_rows.cuh"
#include "zks_lanes.cuh"
#include "zks_samples.cuh"
#include "zks_select.cuh"
#include "zks_probe.cuh"

namespace {

thread_local std::string g_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_error = buf;
  return code;
}

#define ZKS_CUDA(call)                                                                            \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      return fail(ZKS_ECUDA, "%s failed at zks_capi.cu:%d: %s", #call, __LINE__, cudaGetErrorString(e_)); \
  } while (0)

constexpr int64_t kLogsLen = 65537;                   // ln k for k = 0..65536
#ifndef ZKS_SELECT_PER_SM
#define ZKS_SELECT_PER_SM 2
#endif
constexpr size_t kSlabBudget = size_t(4) << 30;       // overflow-slab memory cap (bytes)
constexpr int kStagingSlots = 8;                      // pinned staging slots for table uploads
constexpr int64_t kStagingLen = 65536;                // doubles per slot
constexpr uint64_t kPreBytes = uint64_t(48) << 30;    // pre-drawn rows per chunk (bytes), at most
constexpr double kPreFreeFrac = 0.4;                  // ... and at most this share of the free memory
constexpr uint64_t kPreMaxRows = uint64_t(1) << 20;   // ... and at most this many rows per cell: 8.8 fit-kernel
                                                      // waves; larger chunks only cost allocation time
constexpr int kLaneL2SetAside = 24 << 20;             // persisting L2 for lane_row_kernel's words (bytes)
constexpr double kLaneHeavyTail = 40.0;                // expected values above 64 that make a lane row cell "heavy"
constexpr uint32_t kBatchHist = 512;                  // batch / retry histogram bins above K = 1024

}  // namespace

struct zks_engine {
  int device = 0;
  int sms = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  double* logs = nullptr;
  // pinned staging ring: table uploads stay asynchronous w.r.t. queued kernels
  double* staging = nullptr;
  cudaEvent_t staging_done[kStagingSlots] = {};
  int staging_next = 0;
  unsigned long long* counters = nullptr;  // optional work counters (diagnostics)
  int mle_mode = ZKS_MLE_TABLE;
  int rng = ZKS_RNG_NUMPY;  // replicate streams: numpy's (bit-exact) or the opt-in fast one
  uint64_t pre_cap = 0;   // pre-drawn rows per chunk (zks_engine_set_chunk_bytes; 0 = from the free memory)
  uint64_t pre_auto = 0;  // ... that budget, measured at the first use
  std::map<int, zks::FitTable> fit_tables;  // per support K (0 = unbounded)
  std::map<std::tuple<const void*, size_t, int>, int> occupancy;  // (kernel, smem, threads) -> blocks per SM
  // per-stream scratch: everything a launch writes besides its caller-owned outputs (the work
  // counter, the pre-drawn rows of the two-kernel path, the overflow slab of replicate_kernel, the
  // selection state, its candidates and single-call outputs), so cells and selections enqueued
  // on different streams run concurrently without sharing any of it
  struct Scratch {
    unsigned long long* work = nullptr;
    void* pre = nullptr;
    size_t pre_bytes = 0;
    uint16_t* slab = nullptr;
    size_t slab_bytes = 0;
    zks::SelectState* sel = nullptr;
    double* sel_out = nullptr;
    void* cand = nullptr;  // selection candidates (keys matching a 16-bit prefix)
    size_t cand_bytes = 0;
    uint32_t* words = nullptr;  // lane_row_kernel: per resident warp n x 32 top words
    size_t words_bytes = 0;
  };
  std::map<cudaStream_t, Scratch> scratch;
  unsigned long long launches = 0;  // kernels enqueued by this engine (zks_engine_launches)
  int select_blocks = 0;
  int l2_persist_max = -1;  // cudaDevAttrMaxPersistingL2CacheSize (queried at the first lane launch)
  int l2_window_max = 0;    // cudaDevAttrMaxAccessPolicyWindowSize            // resident grid of the cooperative selection kernel
  zks::SelectBatch dist{};          // the distributed selection in progress (zks_select_dist_*)
  zks::SelectState* dist_sel = nullptr;  // ... and the state it works in (its stream's scratch)
  bool dist_active = false;
  int dist_blocks = 1;
  // per-kernel timing (zks_engine_set_timing): event pairs around launches on the engine stream
  bool timing = false;
  std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> timed;
  std::vector<cudaEvent_t> event_pool;
};

namespace {

// Top words t = x >> 32 of Philox words x, u = 1 - (x >> 11) 2^-53 (stream.py:57-63):
// u > h <=> m = x >> 11 < M(h), M(h) = #{m : 1 - m 2^-53 > h} (exact, by bisection on m).
// Hence t < M >> 21 decides u > h, t > M >> 21 decides u <= h, and t == M >> 21 is undecided.
uint32_t word_cut(double h) {
  uint64_t lo = 0, hi = uint64_t(1) << 53;  // smallest m with 1 - m 2^-53 <= h in [lo, hi]
  while (lo < hi) {
    const uint64_t mid = (lo + hi) / 2;
    if (1.0 - static_cast<double>(mid) * 0x1p-53 <= h)
      hi = mid;
    else
      lo = mid + 1;
  }
  return static_cast<uint32_t>(std::min<uint64_t>(lo >> 21, 0xffffffffu));
}

// RAII timer of one launch: events on the engine stream before and after (timing mode only)
struct Timed {
  zks_engine* e;
  int kind;
  cudaEvent_t a = nullptr;
  static cudaEvent_t take(zks_engine* e) {
    cudaEvent_t ev = nullptr;
    if (!e->event_pool.empty()) {
      ev = e->event_pool.back();
      e->event_pool.pop_back();
    } else if (cudaEventCreate(&ev) != cudaSuccess) {
      ev = nullptr;
    }
    return ev;
  }
  Timed(zks_engine* eng, int k) : e(eng), kind(k) {
    if (e->timing && (a = take(e))) cudaEventRecord(a, e->stream);
  }
  ~Timed() {
    if (!a) return;
    cudaEvent_t b = take(e);
    if (!b) {
      e->event_pool.push_back(a);
      return;
    }
    cudaEventRecord(b, e->stream);
    e->timed.emplace_back(kind, a, b);
  }
};

// the calling stream's scratch (created on first use)
cudaError_t scratch_for(zks_engine* e, zks_engine::Scratch** out) {
  auto it = e->scratch.find(e->stream);
  if (it == e->scratch.end()) {
    zks_engine::Scratch sc;
    cudaError_t err = cudaMalloc(&sc.work, sizeof(unsigned long long));
    if (err == cudaSuccess) err = cudaMalloc(&sc.sel, sizeof(zks::SelectState));
    if (err == cudaSuccess) err = cudaMalloc(&sc.sel_out, zks::kMaxRanks * sizeof(double));
    if (err != cudaSuccess) {
      cudaFree(sc.work);
      cudaFree(sc.sel);
      return err;
    }
    it = e->scratch.emplace(e->stream, sc).first;
  }
  *out = &it->second;
  return cudaSuccess;
}

// every kernel launch goes through here: the error check and the engine's launch count
cudaError_t launched(zks_engine* e) {
  ++e->launches;
  return cudaGetLastError();
}

// exponent-fit table of support K, built on the engine stream on first use
int fit_table_for(zks_engine* e, int K, zks::FitTable** out) {
  auto it = e->fit_tables.find(K);
  if (it == e->fit_tables.end()) {
    zks::FitTable T = zks::fit_layout(K);
    double* coef = nullptr;
    ZKS_CUDA(cudaMalloc(&coef, size_t(T.intervals) * zks::kFitStride * sizeof(double)));
    T.coef = coef;
    const int threads = 128;
    const int blocks = (T.intervals * 32 + threads - 1) / threads;
    {
      Timed tm(e, ZKS_KERNEL_OTHER);
      zks::fit_table_kernel<<<blocks, threads, 0, e->stream>>>(T, coef, e->logs);
      ZKS_CUDA(launched(e));
    }
    it = e->fit_tables.emplace(K, T).first;
  }
  *out = &it->second;
  return ZKS_OK;
}

}  // namespace

struct zks_table {
  zks_engine* engine = nullptr;
  double* cdf = nullptr;
  uint16_t* guide = nullptr;
  uint32_t len = 0;
  double head[4] = {0, 0, 0, 0};  // cdf[0..3], +inf from L-1 on (draw_stats_kernel's head test)
  double tail_mass = 0.0;          // P(X > 64) = 1 - cdf[63]: the row kernel's cost estimate
  uint32_t tcut[4] = {0, 0, 0, 0};  // the same tests on the top 32 bits of Philox words
  unsigned long long* mcut = nullptr;  // exact 53-bit cuts of cdf[0..kCutMax) (row_draw_kernel)
  zks::LaneCut* lanecut = nullptr;     // top-32-bit head cuts + bucket brackets (lane_row_kernel)
  // stream ordering: the upload (and guide build) runs on `home`; another stream's first use
  // waits on `ready`; the free waits on every stream that used the table
  cudaStream_t home = nullptr;
  cudaEvent_t ready = nullptr;
  mutable std::vector<cudaStream_t> users;
};

namespace {
// order the engine stream's coming use of table t after its upload
cudaError_t table_use(zks_engine* e, const zks_table* t) {
  if (e->stream == t->home) return cudaSuccess;
  if (std::find(t->users.begin(), t->users.end(), e->stream) != t->users.end()) return cudaSuccess;
  const cudaError_t err = cudaStreamWaitEvent(e->stream, t->ready, 0);
  if (err == cudaSuccess) t->users.push_back(e->stream);
  return err;
}
}  // namespace

extern "C" {

int zks_version(void) { return 3; }

const char* zks_last_error(void) { return g_error.c_str(); }

int zks_engine_create(int device, const double* logs_host, int64_t logs_len, zks_engine** out) {
  if (!out) return fail(ZKS_EINVAL, "out is NULL");
  *out = nullptr;
  if (!logs_host || logs_len < kLogsLen) return fail(ZKS_EINVAL, "log table needs >= %lld entries", (long long)kLogsLen);
  int ndev = 0;
  ZKS_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(ZKS_EINVAL, "device %d out of range (%d devices)", device, ndev);
  ZKS_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  ZKS_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10) return fail(ZKS_EINVAL, "device %d is sm_%d%d; this build targets sm_100a", device, prop.major, prop.minor);
  zks_engine* e = new zks_engine();
  e->device = device;
  e->sms = prop.multiProcessorCount;
  cudaError_t err = cudaStreamCreateWithFlags(&e->own, cudaStreamNonBlocking);
  if (err == cudaSuccess) err = cudaMalloc(&e->logs, kLogsLen * sizeof(double));
  if (err == cudaSuccess) err = cudaMemcpy(e->logs, logs_host, kLogsLen * sizeof(double), cudaMemcpyHostToDevice);
  if (err == cudaSuccess) err = cudaMallocHost(&e->staging, kStagingSlots * kStagingLen * sizeof(double));
  for (int i = 0; i < kStagingSlots && err == cudaSuccess; ++i)
    err = cudaEventCreateWithFlags(&e->staging_done[i], cudaEventDisableTiming);
  if (err != cudaSuccess) {
    zks_engine_destroy(e);
    return fail(ZKS_ECUDA, "engine allocation failed: %s", cudaGetErrorString(err));
  }
  // the engine's scratch (pre-drawn rows: tens of GB for large rows) comes from the device's
  // default memory pool; keep freed blocks mapped in the pool instead of returning them to the
  // driver at every synchronisation, so that a chunk buffer regrown for a larger row reuses them
  // (re-mapping tens of GB stalled the enqueue for seconds, e.g. config 5's K = inf grid)
  {
    cudaMemPool_t pool = nullptr;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = ~uint64_t(0);
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  e->stream = e->own;
  *out = e;
  return ZKS_OK;
}

void zks_engine_destroy(zks_engine* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  if (e->stream) cudaStreamSynchronize(e->stream);
  cudaDeviceSynchronize();  // queued work on every stream that used this engine's scratch
  cudaFree(e->logs);
  for (auto& kv : e->scratch) {
    zks_engine::Scratch& sc = kv.second;
    cudaFree(sc.work);
    if (sc.pre) cudaFree(sc.pre);
    cudaFree(sc.slab);
    cudaFree(sc.sel);
    cudaFree(sc.sel_out);
    if (sc.cand) cudaFree(sc.cand);
    if (sc.words) cudaFree(sc.words);
  }
  for (auto& kv : e->fit_tables) cudaFree(const_cast<double*>(kv.second.coef));
  if (e->staging) cudaFreeHost(e->staging);
  for (auto& t : e->timed) {
    cudaEventDestroy(std::get<1>(t));
    cudaEventDestroy(std::get<2>(t));
  }
  for (cudaEvent_t ev : e->event_pool) cudaEventDestroy(ev);
  for (int i = 0; i < kStagingSlots; ++i)
    if (e->staging_done[i]) cudaEventDestroy(e->staging_done[i]);
  if (e->own) cudaStreamDestroy(e->own);
  delete e;
}

int zks_engine_set_stream(zks_engine* e, void* stream) {
  if (!e) return fail(ZKS_EINVAL, "engine is NULL");
  e->stream = static_cast<cudaStream_t>(stream);  // NULL = the legacy default stream
  return ZKS_OK;
}

int zks_engine_sync(zks_engine* e) {
  if (!e) return fail(ZKS_EINVAL, "engine is NULL");
  ZKS_CUDA(cudaSetDevice(e->device));
  ZKS_CUDA(cudaStreamSynchronize(e->stream));
  return ZKS_OK;
}

int zks_engine_set_chunk_bytes(zks_engine* e, uint64_t bytes) {
  if (!e) return fail(ZKS_EINVAL, "engine is NULL");
  e->pre_cap = bytes;
  return ZKS_OK;
}

int zks_engine_set_rng(zks_engine* e, int rng) {
  if (!e) return fail(ZKS_EINVAL, "engine is NULL");
  if (rng != ZKS_RNG_NUMPY && rng != ZKS_RNG_PHILOX4X32) return fail(ZKS_EINVAL, "unknown stream kind %d", rng);
  e->rng = rng;
  return ZKS_OK;
}

int zks_engine_set_timing(zks_engine* e, int on) {
  if (!e) return fail(ZKS_EINVAL, "engine is NULL");
  e->timing = on != 0;
  return ZKS_OK;
}

int zks_engine_kernel_times(zks_engine* e, double* ms_out, unsigned long long* launches_out) {
  if (!e || !ms_out || !launches_out) return fail(ZKS_EINVAL, "NULL argument");
  ZKS_CUDA(cudaSetDevice(e->device));
  ZKS_CUDA(cudaStreamSynchronize(e->stream));
  for (int k = 0; k < ZKS_KERNEL_KINDS; ++k) {
    ms_out[k] = 0.0;
    launches_out[k] = 0;
  }
  cudaError_t err = cudaSuccess;
  for (auto& t : e->timed) {
    float ms = 0.0f;
    if (err == cudaSuccess) err = cudaEventElapsedTime(&ms, std::get<1>(t), std::get<2>(t));
    ms_out[std::get<0>(t)] += ms;
    ++launches_out[std::get<0>(t)];
    e->event_pool.push_back(std::get<1>(t));
    e->event_pool.push_back(std::get<2>(t));
  }
  e->timed.clear();
  ZKS_CUDA(err);
  return ZKS_OK;
}

int zks_engine_launches(zks_engine* e, unsigned long long* out) {
  if (!e || !out) return fail(ZKS_EINVAL, "engine/out is NULL");
  *out = e->launches;
  return ZKS_OK;
}

int zks_table_create(zks_engine* e, const double* cdf_host, int64_t len, zks_table** out) {
  if (!e || !out) return fail(ZKS_EINVAL, "engine/out is NULL");
  *out = nullptr;
  if (!cdf_host || len < 2 || len > 65535) return fail(ZKS_EINVAL, "cdf length %lld outside [2, 65535]", (long long)len);
  ZKS_CUDA(cudaSetDevice(e->device));
  zks_table* t = new zks_table();
  t->engine = e;
  t->len = static_cast<uint32_t>(len);
  for (int j = 0; j < 4; ++j) {
    t->head[j] = j + 1 < len ? cdf_host[j] : __builtin_huge_val();
    t->tail_mass = len > 64 ? std::max(0.0, 1.0 - cdf_host[63]) : 0.0;
    t->tcut[j] = word_cut(t->head[j]);
  }
  // one stream-ordered allocation (cdf then guide): no device-wide synchronisation
  void* mem = nullptr;
  const int64_t cdf_slots = (len + 1) & ~int64_t(1);  // guide 16-byte aligned (vector copies)
  const size_t guide_bytes = (size_t(zks::kGuideEntries) * sizeof(uint16_t) + 15) & ~size_t(15);
  cudaError_t err =
      cudaMallocAsync(&mem,
                      cdf_slots * sizeof(double) + guide_bytes + zks::kCutMax * sizeof(unsigned long long) +
                          sizeof(zks::LaneCut),
                      e->stream);
  if (err == cudaSuccess) {
    t->cdf = static_cast<double*>(mem);
    t->guide = reinterpret_cast<uint16_t*>(t->cdf + cdf_slots);
    t->mcut = reinterpret_cast<unsigned long long*>(reinterpret_cast<unsigned char*>(t->guide) + guide_bytes);
    t->lanecut = reinterpret_cast<zks::LaneCut*>(t->mcut + zks::kCutMax);
  }
  if (err == cudaSuccess) {
    // stage through a pinned slot so the copy never waits for kernels already queued
    const int slot = e->staging_next;
    e->staging_next = (slot + 1) % kStagingSlots;
    err = cudaEventSynchronize(e->staging_done[slot]);
    double* stage = e->staging + slot * kStagingLen;
    if (err == cudaSuccess) {
      std::memcpy(stage, cdf_host, len * sizeof(double));
      err = cudaMemcpyAsync(t->cdf, stage, len * sizeof(double), cudaMemcpyHostToDevice, e->stream);
    }
    if (err == cudaSuccess) err = cudaEventRecord(e->staging_done[slot], e->stream);
  }
  if (err == cudaSuccess) {
    {
      Timed tm(e, ZKS_KERNEL_OTHER);
      zks::guide_kernel<<<(zks::kGuideEntries + 255) / 256, 256, 0, e->stream>>>(t->cdf, t->len, t->guide);
      err = launched(e);
    }
    if (err == cudaSuccess) {
      Timed tm(e, ZKS_KERNEL_OTHER);
      zks::cut_kernel<<<zks::kCutMax / 256, 256, 0, e->stream>>>(t->cdf, t->len, t->mcut);
      err = launched(e);
    }
    if (err == cudaSuccess) {
      Timed tm(e, ZKS_KERNEL_OTHER);
      zks::lane_cut_kernel<<<16, 256, 0, e->stream>>>(t->mcut, t->lanecut);
      err = launched(e);
    }
  }
  t->home = e->stream;
  if (err == cudaSuccess) err = cudaEventCreateWithFlags(&t->ready, cudaEventDisableTiming);
  if (err == cudaSuccess) err = cudaEventRecord(t->ready, e->stream);
  if (err != cudaSuccess) {
    zks_table_destroy(t);
    return fail(ZKS_ECUDA, "table upload failed: %s", cudaGetErrorString(err));
  }
  *out = t;
  return ZKS_OK;
}

void zks_table_destroy(zks_table* t) {
  if (!t) return;
  if (t->engine && t->cdf) {
    zks_engine* e = t->engine;
    cudaSetDevice(e->device);
    // the free runs on the engine's current stream after every queued use on the others
    std::vector<cudaStream_t> others = t->users;
    others.push_back(t->home);
    for (cudaStream_t s : others) {
      if (s == e->stream) continue;
      cudaEvent_t ev = nullptr;
      if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
        cudaDeviceSynchronize();
        break;
      }
      cudaEventRecord(ev, s);
      cudaStreamWaitEvent(e->stream, ev, 0);
      cudaEventDestroy(ev);
    }
    cudaFreeAsync(t->cdf, e->stream);
  }
  if (t->ready) cudaEventDestroy(t->ready);
  delete t;
}

}  // extern "C"

namespace {

int check_cell(const zks_table* t, const zks_cell* c) {
  if (!t || !c) return fail(ZKS_EINVAL, "table/cell is NULL");
  if (c->n < 1) return fail(ZKS_EINVAL, "sample size must be >= 1, got %lld", (long long)c->n);
  if (c->support_k < 0 || c->support_k == 1 || c->support_k > 32766)
    return fail(ZKS_EINVAL, "finite support bound must be in [2, 32766], got %d", c->support_k);
  const uint32_t L = c->support_k ? static_cast<uint32_t>(c->support_k) : 65535u;
  if (t->len != L) return fail(ZKS_EINVAL, "table length %u does not match support (%u)", t->len, L);
  return ZKS_OK;
}

// the per-cell launch arguments every replicate kernel shares
int cell_args(zks_engine* e, const zks_table* t, const zks_cell* c, double* ks_dev, double* gh_dev, uint8_t* st_dev,
              zks_engine::Scratch* sc, zks::ReplicateArgs& a) {
  const uint32_t L = t->len;
  a = zks::ReplicateArgs{};
  a.cdf = t->cdf;
  a.guide = t->guide;
  a.guide_fine = t->guide + 2 * zks::kGuideLevel;
  for (int j = 0; j < 4; ++j) {
    a.cdf_head[j] = t->head[j];
    a.tcut[j] = t->tcut[j];
  }
  a.logs = e->logs;
  a.L = L;
  a.K = c->support_k;
  a.H = static_cast<int32_t>(std::min<uint32_t>(L, zks::kHistMax));
  a.hist_words = zks::round_up(std::max(a.H, 4) + 1, 4);
  a.gamma = c->gamma;
  a.n = c->n;
  a.inv_n = 1.0 / static_cast<double>(c->n);
  a.seed = c->base_seed;
  a.rep = c->repetition;
  a.first = c->first;
  a.count = c->count;
  a.ks_out = ks_dev;
  a.gh_out = gh_dev;
  a.st_out = st_dev;
  a.work = sc->work;
  a.counters = e->counters;
  a.guide_levels = L > 4096u ? 2 : 1;
  a.rng = e->rng;
  a.use_table = e->mle_mode == ZKS_MLE_TABLE;
  if (a.use_table) {
    zks::FitTable* T = nullptr;
    const int rc = fit_table_for(e, c->support_k, &T);
    if (rc) return rc;
    a.fit = *T;
  }
  return ZKS_OK;
}

// the chunk budget of pre-drawn rows: the caller's, else min(kPreBytes, kPreFreeFrac of the free
// memory + what this stream's buffer already holds) -- larger chunks mean fewer, fuller launches
// memory once per engine (the driver query stalls the enqueue; repeated per call it let the device
// idle: sweep times varied 90-108 ms)
uint64_t pre_budget(zks_engine* e, const zks_engine::Scratch* sc) {
  if (e->pre_cap) return e->pre_cap;
  if (!e->pre_auto) {
    size_t free_b = 0, total_b = 0;
    e->pre_auto = cudaMemGetInfo(&free_b, &total_b) == cudaSuccess
                      ? std::min<uint64_t>(kPreBytes, uint64_t(kPreFreeFrac * double(free_b + sc->pre_bytes)))
                      : uint64_t(4) << 30;
  }
  return e->pre_auto;
}

// blocks per SM of a kernel at a dynamic shared-memory size (cached; sets the opt-in ceiling)
int occupancy_of(zks_engine* e, const void* kernel, size_t smem, int threads, int* per) {
  const auto key = std::make_tuple(kernel, smem, threads);
  auto it = e->occupancy.find(key);
  if (it == e->occupancy.end()) {
    int optin = 0;
    ZKS_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, e->device));
    cudaFuncAttributes fa;
    ZKS_CUDA(cudaFuncGetAttributes(&fa, kernel));
    const int dyn_max = optin - static_cast<int>(fa.sharedSizeBytes);  // dynamic ceiling next to the static smem
    if (smem > size_t(dyn_max)) return fail(ZKS_EINVAL, "kernel needs %zu B of shared memory (%d available)", smem, dyn_max);
    ZKS_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max));
    int p = 0;
    ZKS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p, kernel, threads, smem));
    if (p < 1) return fail(ZKS_ECUDA, "kernel does not fit (smem %zu)", smem);
    it = e->occupancy.emplace(key, p).first;
  }
  *per = it->second;
  return ZKS_OK;
}

// The two-kernel layout (kLaneDrawMaxN <= n <= kPreMaxN, table MLE) for ncells cells of one row
// (equal n, support, seed, repetition and replicate range; gammas differ): per chunk of
// replicates the draw phase writes every cell's pre-drawn rows -- row_draw_kernel (n <=
// kRowMaxN: each stream drawn and sorted once for all cells) or draw_stats_kernel per cell --
// then per cell fit_ks_kernel and retry_kernel.
int run_pre_rows(zks_engine* e, int ncells, const zks_table* const* tables, const zks_cell* cells,
                 double* const* ks_dev, double* const* gh_dev, uint8_t* const* st_dev) {
  const zks_cell& c0 = cells[0];
  zks_engine::Scratch* sc = nullptr;
  ZKS_CUDA(scratch_for(e, &sc));
  const bool rows = c0.n <= zks::kRowMaxN;
  std::vector<zks::ReplicateArgs> args(ncells);
  for (int j = 0; j < ncells; ++j) {
    ZKS_CUDA(table_use(e, tables[j]));
    const int rc = cell_args(e, tables[j], &cells[j], ks_dev[j], gh_dev[j], st_dev[j], sc, args[j]);
    if (rc) return rc;
  }
  // finite supports up to 1024 fit the retry histogram whole; otherwise 512 bins + ordered overflow
  const uint32_t L = tables[0]->len;
  int H = static_cast<int>(L <= 1024u ? L : kBatchHist);
  int hist_words = std::max(zks::round_up(std::max(H, 4) + 1, 4), zks::kLaneHistWords);
  int vals_stride = zks::round_up(static_cast<int>(c0.n), 4);
  int dense_words = 0;
  // finite supports above the head and up to kDenseMaxK: dense counts instead of value lists
  if (c0.support_k > static_cast<int>(zks::kKsHead) && c0.support_k <= zks::kDenseMaxK) {
    dense_words = c0.support_k - static_cast<int>(zks::kKsHead);
    vals_stride = std::max(vals_stride, zks::round_up(2 * dense_words, 4));
  }
  for (auto& a : args) {
    a.H = H;
    a.hist_words = hist_words;
    a.vals_stride = vals_stride;
    a.batch = 32;
    a.dense_words = dense_words;
    a.slab = nullptr;
    a.slab_cap = 0;
  }
  const bool counting = e->counters != nullptr;
  const size_t guide_bytes = zks::round_up(args[0].guide_levels * zks::kGuideLevel * 2, 16);
  // per row and cell: u16 head counts (128 B), log-sum, min / max / m, the tail slot, a
  // retry-list slot, a long-tail-list slot with its head state (44 B); per cell region 256-byte
  // aligned
  const uint64_t row_bytes = zks::kKsHead * 2 + 8 + 12 + uint64_t(vals_stride) * 2 + 4 + 48;
  const uint64_t chunk = std::max<uint64_t>(
      1, std::min<uint64_t>(std::min<uint64_t>(c0.count, kPreMaxRows), pre_budget(e, sc) / (row_bytes * uint64_t(ncells))));
  const size_t region = (size_t(chunk) * row_bytes + 64 + 255) & ~size_t(255);
  const size_t need = region * size_t(ncells);
  if (need > sc->pre_bytes) {
    if (sc->pre) ZKS_CUDA(cudaFreeAsync(sc->pre, e->stream));
    sc->pre = nullptr;
    sc->pre_bytes = 0;
    ZKS_CUDA(cudaMallocAsync(&sc->pre, need, e->stream));
    sc->pre_bytes = need;
  }
  struct Pre {
    uint16_t* head;
    double* ls;
    uint32_t *mn, *mx, *m;
    uint16_t* tail;
    uint32_t* retry;
    zks::TailList tl;
  };
  std::vector<Pre> pre(ncells);
  for (int j = 0; j < ncells; ++j) {
    unsigned char* base = static_cast<unsigned char*>(sc->pre) + region * j;
    Pre& p = pre[j];
    p.head = reinterpret_cast<uint16_t*>(base);
    p.ls = reinterpret_cast<double*>(p.head + chunk * zks::kKsHead);
    p.mn = reinterpret_cast<uint32_t*>(p.ls + chunk);
    p.mx = p.mn + chunk;
    p.m = p.mx + chunk;
    p.tail = reinterpret_cast<uint16_t*>(p.m + chunk);
    p.retry = reinterpret_cast<uint32_t*>(p.tail + chunk * vals_stride);  // vals_stride % 4 == 0
    double* st = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(p.retry + chunk + 1) + 7) & ~uintptr_t(7));
    p.tl.S = st;
    p.tl.D = st + chunk;
    p.tl.g = st + 2 * chunk;
    p.tl.norm = st + 3 * chunk;
    p.tl.C = reinterpret_cast<uint32_t*>(st + 4 * chunk);
    p.tl.kmax = p.tl.C + chunk;
    p.tl.list = p.tl.kmax + chunk;
  }
  // the retry kernel's per-warp sample store grows with n: fewer warps per block for large n
  const int rwarps = static_cast<int>(std::max<size_t>(
      1, std::min<size_t>(zks::kWarps, (size_t(227) * 1024 - guide_bytes) /
                                           size_t(zks::retry_warp_bytes(hist_words, vals_stride)))));
  auto fit = counting ? zks::fit_ks_kernel<true> : zks::fit_ks_kernel<false>;
  auto again = counting ? zks::retry_kernel<true> : zks::retry_kernel<false>;
  auto longk = counting ? zks::long_tail_kernel<true> : zks::long_tail_kernel<false>;
  const size_t fsmem = size_t(zks::kWarps) * zks::kFitWarpWords * 4;
  const size_t lsmem = size_t(zks::kWarps) * (zks::kFitHistWords + zks::kKsQueueWords) * 4;
  const size_t rsmem = guide_bytes + size_t(rwarps) * zks::retry_warp_bytes(hist_words, vals_stride);
  int fper = 0, rper = 0, lper = 0;
  if (int rc = occupancy_of(e, reinterpret_cast<const void*>(fit), fsmem, zks::kThreads, &fper)) return rc;
  if (int rc = occupancy_of(e, reinterpret_cast<const void*>(longk), lsmem, zks::kThreads, &lper)) return rc;
  if (int rc = occupancy_of(e, reinterpret_cast<const void*>(again), rsmem, 32 * rwarps, &rper)) return rc;
  // draw phase
  const bool wide = c0.n > zks::kNarrowBinsMaxN;
  auto draw = counting ? (wide ? zks::draw_stats_kernel<true, true> : zks::draw_stats_kernel<true, false>)
                       : (wide ? zks::draw_stats_kernel<false, true> : zks::draw_stats_kernel<false, false>);
  const size_t dsmem = zks::round_up(zks::kGuideLevel * 2, 16) + (size_t(4) << zks::kCutTabBits) +
                       size_t(zks::kWarps) * (zks::draw_warp_bytes(wide) + size_t(dense_words) * 4);
  auto rowk = counting ? zks::row_draw_kernel<true> : zks::row_draw_kernel<false>;
  // warps per row block (the cells are spread over them by the schedule below)
  int row_warps = std::max(4, std::min(zks::kWarps, ncells));
  int row_bits = zks::row_bucket_bits(static_cast<int>(c0.n));
  if (rows && row_warps > 4 && c0.n <= 1024) {
    // blocks of 4 warps when they keep as many warps resident: more, smaller blocks per SM leave
    // fewer warps idle at a row's barriers (measured, 21-cell rows: n = 128..1000 5-8 % faster,
    // with 512 buckets for 512 < n <= 1024 so that 8 such blocks fit; n = 1500..3000: no gain)
    int p8 = 0, p4 = 0;
    const int n = static_cast<int>(c0.n);
    if (int rc = occupancy_of(e, reinterpret_cast<const void*>(rowk), zks::row_smem_bytes(n, dense_words, row_warps, row_bits),
                              32 * row_warps, &p8))
      return rc;
    if (int rc = occupancy_of(e, reinterpret_cast<const void*>(rowk), zks::row_smem_bytes(n, dense_words, 4, row_bits), 128, &p4))
      return rc;
    if (p4 * 4 >= p8 * row_warps) row_warps = 4;
  }
  const size_t rsmem_row = zks::row_smem_bytes(static_cast<int>(c0.n), dense_words, row_warps, row_bits);
  int dper = 0;
  if (rows) {
    if (int rc = occupancy_of(e, reinterpret_cast<const void*>(rowk), rsmem_row, 32 * row_warps, &dper)) return rc;
  } else {
    if (int rc = occupancy_of(e, reinterpret_cast<const void*>(draw), dsmem, zks::kThreads, &dper)) return rc;
  }
  zks::RowArgs ra{};
  if (rows) {
    ra.seed = c0.base_seed;
    ra.rep = c0.repetition;
    ra.n = static_cast<int>(c0.n);
    ra.vals_stride = vals_stride;
    ra.dense_words = dense_words;
    ra.ncells = ncells;
    ra.bucket_bits = row_bits;
    ra.logs = e->logs;
    ra.counters = e->counters;
    ra.rng = e->rng;
    // longest processing time first: a cell costs its 64 cut positions and reductions (~one
    // 32-lane round) plus a guide + cdf search per 32 tail draws (about three rounds each)
    auto cell_cost = [&](int j) { return 1.0 + 3.0 * double(c0.n) * tables[j]->tail_mass / 32.0; };
    std::vector<std::pair<double, int>> cost(ncells);
    for (int j = 0; j < ncells; ++j) cost[j] = {cell_cost(j), j};
    std::sort(cost.begin(), cost.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
    std::vector<std::vector<int>> lists(row_warps);
    std::vector<double> load(row_warps, 0.0);
    for (const auto& cj : cost) {
      int w = 0;
      for (int v = 1; v < row_warps; ++v)
        if (load[v] < load[w]) w = v;
      lists[w].push_back(cj.second);
      load[w] += cj.first;
    }
    // the least loaded list last (that warp also derives the next row's stream key)
    auto list_cost = [&](const std::vector<int>& l) {
      double c = 0.0;
      for (int j : l) c += cell_cost(j);
      return c;
    };
    std::stable_sort(lists.begin(), lists.end(),
                     [&](const auto& x, const auto& y) { return list_cost(x) > list_cost(y); });
    int at = 0;
    for (int w = 0; w < row_warps; ++w) {
      ra.wbeg[w] = static_cast<uint8_t>(at);
      for (int j : lists[w]) ra.order[at++] = static_cast<uint8_t>(j);
    }
    for (int w = row_warps; w <= zks::kWarps; ++w) ra.wbeg[w] = static_cast<uint8_t>(at);
    for (int j = 0; j < ncells; ++j) {
      zks::RowCell& rc = ra.cell[j];
      rc.cdf = tables[j]->cdf;
      rc.guide = tables[j]->guide;
      rc.guide_fine = tables[j]->guide + 2 * zks::kGuideLevel;
      rc.mcut = tables[j]->mcut;
      rc.L = tables[j]->len;
      rc.guide_levels = args[j].guide_levels;
    }
  }
  for (uint64_t off = 0; off < c0.count; off += chunk) {
    const uint64_t cnt = std::min<uint64_t>(chunk, c0.count - off);
    std::vector<zks::ReplicateArgs> sub(args);
    for (int j = 0; j < ncells; ++j) {
      zks::ReplicateArgs& s = sub[j];
      s.first = c0.first + off;
      s.count = cnt;
      s.ks_out = ks_dev[j] + off;
      s.gh_out = gh_dev[j] + off;
      s.st_out = st_dev[j] + off;
      s.pre_head = pre[j].head;
      s.pre_tail = pre[j].tail;
      s.pre_m = pre[j].m;
      s.pre_ls = pre[j].ls;
      s.pre_min = pre[j].mn;
      s.pre_max = pre[j].mx;
      s.pre_first = s.first;
    }
    if (rows) {
      ra.first = c0.first + off;
      ra.count = cnt;
      for (int j = 0; j < ncells; ++j) {
        zks::RowCell& rc = ra.cell[j];
        rc.head = pre[j].head;
        rc.tail = pre[j].tail;
        rc.m = pre[j].m;
        rc.ls = pre[j].ls;
        rc.mn = pre[j].mn;
        rc.mx = pre[j].mx;
      }
      const int64_t rblocks = std::max<int64_t>(1, std::min<int64_t>(int64_t(e->sms) * dper, (int64_t)cnt));
      Timed tm(e, ZKS_KERNEL_ROW);
      rowk<<<(unsigned)rblocks, 32 * row_warps, rsmem_row, e->stream>>>(ra);
      ZKS_CUDA(launched(e));
    } else {
      for (int j = 0; j < ncells; ++j) {
        const zks::ReplicateArgs& s = sub[j];
        const int64_t dblocks =
            std::max<int64_t>(1, std::min<int64_t>(int64_t(e->sms) * dper, (int64_t)((cnt + 7) / 8)));
        Timed tm(e, ZKS_KERNEL_DRAW);
        draw<<<(unsigned)dblocks, zks::kThreads, dsmem, e->stream>>>(s, pre[j].head, pre[j].tail, pre[j].m,
                                                                     pre[j].ls, pre[j].mn, pre[j].mx);
        ZKS_CUDA(launched(e));
      }
    }
    const int64_t fblocks = std::max<int64_t>(1, std::min<int64_t>(int64_t(e->sms) * fper, (int64_t)((cnt + 255) / 256)));
    for (int j = 0; j < ncells; ++j) {
      ZKS_CUDA(cudaMemsetAsync(sub[j].work, 0, sizeof(unsigned long long), e->stream));
      ZKS_CUDA(cudaMemsetAsync(pre[j].retry, 0, sizeof(uint32_t), e->stream));
      ZKS_CUDA(cudaMemsetAsync(pre[j].tl.list, 0, sizeof(uint32_t), e->stream));
      {
        Timed tm(e, ZKS_KERNEL_FIT);
        fit<<<(unsigned)fblocks, zks::kThreads, fsmem, e->stream>>>(sub[j], pre[j].retry, pre[j].tl);
        ZKS_CUDA(launched(e));
      }
      if (!dense_words) {  // the listed paged tails, one warp each (exits at once on an empty list)
        Timed tm(e, ZKS_KERNEL_FIT);
        longk<<<(unsigned)(e->sms * lper), zks::kThreads, lsmem, e->stream>>>(sub[j], pre[j].tl);
        ZKS_CUDA(launched(e));
      }
      {
        Timed tm(e, ZKS_KERNEL_RETRY);
        again<<<(unsigned)e->sms, 32 * rwarps, rsmem, e->stream>>>(sub[j], pre[j].retry);
        ZKS_CUDA(launched(e));
      }
    }
  }
  return ZKS_OK;
}

// Small samples (n < kLaneDrawMaxN, table MLE) for ncells cells of one row (equal n, support,
// seed, repetition and replicate range; gammas differ): one lane_row_kernel launch, each replicate
// stream drawn once per work item for the cells of its group.  A single cell runs through here
// too (ncells = 1), so a cell's results do not depend on whether it was computed alone or in a row.
template <int C>
int run_lane_launch_t(zks_engine* e, int ncells, const zks_table* const* tables, const zks_cell* cells,
                      double* const* ks_dev, double* const* gh_dev, uint8_t* const* st_dev) {
  const zks_cell& c0 = cells[0];
  zks_engine::Scratch* sc = nullptr;
  ZKS_CUDA(scratch_for(e, &sc));
  thread_local zks::LaneArgsT<C> la;  // up to 18 KB: kept off the host stack
  std::memset(&la, 0, sizeof la);
  const uint32_t L = tables[0]->len;
  const int H = static_cast<int>(L <= 1024u ? L : kBatchHist);
  // a lane's tail buffer: the tails a lane scores itself (ks_tail_lane), longer ones go to the
  // warp.  kLaneTailMax values, or the whole sample when a cell of the row expects long tails
  // (n P(X > 64) > 40: K = 500 / 1000 at n = 100, gamma < 1) -- then one warp-serial tail per
  // replicate would cost more than a resident block less (measured: K = 1000, n = 100, 31 cells
  // 95 -> 85 ms; at n = 50 the same rule cost 13 %)
  double tail_max = 0.0;
  for (int j = 0; j < ncells; ++j) tail_max = std::max(tail_max, double(c0.n) * tables[j]->tail_mass);
  const int vals_stride = tail_max > kLaneHeavyTail
                              ? zks::round_up(static_cast<int>(c0.n), 4)
                              : std::min(zks::round_up(static_cast<int>(c0.n), 4), zks::round_up(int(zks::kLaneTailMax), 4));
  for (int j = 0; j < ncells; ++j) {
    ZKS_CUDA(table_use(e, tables[j]));
    zks::ReplicateArgs& a = la.cell[j];
    if (int rc = cell_args(e, tables[j], &cells[j], ks_dev[j], gh_dev[j], st_dev[j], sc, a)) return rc;
    // finite supports up to 1024 fit the histogram whole; otherwise 512 bins + ordered overflow
    a.H = H;
    a.hist_words = std::max(zks::round_up(std::max(H, 4) + 1, 4), zks::kLaneHistWords);
    a.vals_stride = vals_stride;
    a.batch = 32;
    a.slab = nullptr;
    a.slab_cap = 0;
    la.cut[j] = tables[j]->lanecut;
  }
  la.ncells = ncells;
  const bool counting = e->counters != nullptr;
  auto kernel = counting ? zks::lane_row_kernel<true, C> : zks::lane_row_kernel<false, C>;
  const zks::ReplicateArgs& a0 = la.cell[0];
  const size_t smem = zks::kLaneLnBytes + size_t(zks::kWarps) * zks::batch_warp_bytes(a0.hist_words, a0.vals_stride,
                                                                                       int(c0.n));
  int per_sm = 0;
  if (int rc = occupancy_of(e, reinterpret_cast<const void*>(kernel), smem, zks::kThreads, &per_sm)) return rc;
  const int64_t tiles = (c0.count + 31) / 32;
  int64_t blocks = std::min<int64_t>(int64_t(e->sms) * per_sm, (tiles + zks::kWarps - 1) / zks::kWarps);
  // enough work items for about two per resident warp: short launches split the cells into
  // groups (each group redraws its tiles)
  const int64_t warps = int64_t(e->sms) * per_sm * zks::kWarps;
  int groups = static_cast<int>(std::min<int64_t>(ncells, std::max<int64_t>(1, (2 * warps + tiles - 1) / tiles)));
  la.per_group = (ncells + groups - 1) / groups;
  la.groups = (ncells + la.per_group - 1) / la.per_group;
  blocks = std::min<int64_t>(int64_t(e->sms) * per_sm, (tiles * la.groups + zks::kWarps - 1) / zks::kWarps);
  const size_t need = size_t(blocks) * zks::kWarps * size_t(c0.n) * 32 * sizeof(uint32_t);
  if (need > sc->words_bytes) {
    if (sc->words) ZKS_CUDA(cudaFreeAsync(sc->words, e->stream));
    sc->words = nullptr;
    sc->words_bytes = 0;
    ZKS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&sc->words), need, e->stream));
    sc->words_bytes = need;
  }
  la.words = sc->words;
  ZKS_CUDA(cudaMemsetAsync(a0.work, 0, sizeof(unsigned long long), e->stream));
  {
    Timed tm(e, ZKS_KERNEL_BATCH);
    // the words are re-read once per cell: keep them in L2 as persisting lines (an access-policy
    // window on this launch; the device's persisting set-aside is raised once per engine)
    if (e->l2_persist_max < 0) {
      // a set-aside of 24 MB of the 79 MB allowed: larger ones cost the row and fit kernels of
      // the larger rows L2 they need (config 3: 2.61 s at 24 MB, 2.66 s at 79 MB; config 2 best
      // at 24-48 MB, 1 % slower without).  A performance hint only: where the device refuses it
      // (queries or the limit fail), the launch goes without the window
      int maxp = 0, maxw = 0;
      if (cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, e->device) != cudaSuccess ||
          cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, e->device) != cudaSuccess)
        maxp = maxw = 0;
      maxp = std::min(maxp, kLaneL2SetAside);
      if (maxp > 0 && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, size_t(maxp)) != cudaSuccess) maxp = 0;
      cudaGetLastError();  // clear a refused hint
      e->l2_persist_max = maxp;
      e->l2_window_max = maxw;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3(zks::kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = e->stream;
    cudaLaunchAttribute at[1];
    if (e->l2_persist_max > 0 && e->l2_window_max > 0) {
      at[0].id = cudaLaunchAttributeAccessPolicyWindow;
      at[0].val.accessPolicyWindow.base_ptr = sc->words;
      at[0].val.accessPolicyWindow.num_bytes = std::min<size_t>(need, size_t(e->l2_window_max));
      at[0].val.accessPolicyWindow.hitRatio =
          std::min(1.0f, float(e->l2_persist_max) / float(at[0].val.accessPolicyWindow.num_bytes));
      at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cfg.attrs = at;
      cfg.numAttrs = 1;
    }
    ZKS_CUDA(cudaLaunchKernelEx(&cfg, kernel, la));
    ZKS_CUDA(launched(e));
  }
  if (need >= (size_t(16) << 20)) {  // large word buffers are dropped from L2 (no write-back of scratch)
    Timed tm(e, ZKS_KERNEL_OTHER);
    zks::lane_release_kernel<<<(unsigned)e->sms, 256, 0, e->stream>>>(sc->words, need & ~size_t(127));
    ZKS_CUDA(launched(e));
  }
  return ZKS_OK;
}

int run_lane_launch(zks_engine* e, int ncells, const zks_table* const* tables, const zks_cell* cells,
                    double* const* ks_dev, double* const* gh_dev, uint8_t* const* st_dev) {
  if (ncells == 1) return run_lane_launch_t<1>(e, ncells, tables, cells, ks_dev, gh_dev, st_dev);
  return run_lane_launch_t<zks::kLaneMaxCells>(e, ncells, tables, cells, ks_dev, gh_dev, st_dev);
}

// The row's cells that expect long tails (n P(X > 64) > kLaneHeavyTail) run one launch each,
// the others together: heavy cells spend most of their time in warp-scored tails and long KS
// scans, and mixed with light cells in one launch the warps' phases and tables thrash the
// instruction cache and L1 (K = 1000, n = 100, 31 cells: 84 ms in one launch, 69 ms split;
// K = 500: 63 -> 53 ms).  Results do not depend on the grouping.
int run_lane_rows(zks_engine* e, int ncells, const zks_table* const* tables, const zks_cell* cells,
                  double* const* ks_dev, double* const* gh_dev, uint8_t* const* st_dev) {
  std::vector<int> light;
  for (int j = 0; j < ncells; ++j) {
    if (ncells > 1 && double(cells[j].n) * tables[j]->tail_mass > kLaneHeavyTail) {
      if (int rc = run_lane_launch(e, 1, tables + j, cells + j, ks_dev + j, gh_dev + j, st_dev + j)) return rc;
    } else {
      light.push_back(j);
    }
  }
  if (light.empty()) return ZKS_OK;
  if (int(light.size()) == ncells) return run_lane_launch(e, ncells, tables, cells, ks_dev, gh_dev, st_dev);
  std::vector<const zks_table*> t;
  std::vector<zks_cell> c;
  std::vector<double*> k, g;
  std::vector<uint8_t*> st;
  for (int j : light) {
    t.push_back(tables[j]);
    c.push_back(cells[j]);
    k.push_back(ks_dev[j]);
    g.push_back(gh_dev[j]);
    st.push_back(st_dev[j]);
  }
  return run_lane_launch(e, int(light.size()), t.data(), c.data(), k.data(), g.data(), st.data());
}

int run_replicates_impl(zks_engine* e, const zks_table* t, const zks_cell* c, double* ks_dev, double* gh_dev,
                        uint8_t* st_dev) {
  if (!e) return fail(ZKS_EINVAL, "engine is NULL");
  if (int rc = check_cell(t, c)) return rc;
  if (c->count == 0) return ZKS_OK;
  if (!ks_dev || !gh_dev || !st_dev) return fail(ZKS_EINVAL, "output pointer is NULL");
  ZKS_CUDA(cudaSetDevice(e->device));
  const bool table_mode = e->mle_mode == ZKS_MLE_TABLE;
  if (table_mode && c->n >= zks::kLaneDrawMaxN && c->n <= zks::kPreMaxN)
    return run_pre_rows(e, 1, &t, c, &ks_dev, &gh_dev, &st_dev);
  if (table_mode && c->n < zks::kLaneDrawMaxN) return run_lane_rows(e, 1, &t, c, &ks_dev, &gh_dev, &st_dev);
  ZKS_CUDA(table_use(e, t));
  zks_engine::Scratch* sc = nullptr;
  ZKS_CUDA(scratch_for(e, &sc));
  zks::ReplicateArgs a;
  if (int rc = cell_args(e, t, c, ks_dev, gh_dev, st_dev, sc, a)) return rc;
  const uint32_t L = t->len;
  const bool counting = e->counters != nullptr;
  // replicate_kernel: direct-sum MLE at any n, table MLE above kPreMaxN (one warp per replicate)
  const size_t guide_bytes = zks::round_up(a.guide_levels * zks::kGuideLevel * 2, 16);
  a.batch = 1;
  a.vals_stride = 0;
  auto kernel = counting ? zks::replicate_kernel<true> : zks::replicate_kernel<false>;
  const size_t smem = guide_bytes + size_t(zks::kWarps) * (a.hist_words + 3 * zks::kKsQueue) * 4;
  const int64_t per_block = zks::kWarps;  // replicates one block takes per work item round
  int per_sm = 0;
  if (int rc = occupancy_of(e, reinterpret_cast<const void*>(kernel), smem, zks::kThreads, &per_sm)) return rc;
  int64_t blocks = int64_t(e->sms) * std::max(per_sm, 1);
  blocks = std::min<int64_t>(blocks, (int64_t)((c->count + per_block - 1) / per_block));
  a.slab = nullptr;
  a.slab_cap = 0;
  if (L > static_cast<uint32_t>(a.H)) {
    // worst case every draw of a replicate lands above the histogram, so
    // capacity n per warp
    const size_t per_warp = size_t(c->n) * sizeof(uint16_t);
    int64_t max_blocks = int64_t(kSlabBudget / (per_warp * zks::kWarps));
    if (max_blocks < 1) return fail(ZKS_EINVAL, "sample size %lld too large for the overflow slab", (long long)c->n);
    blocks = std::min(blocks, max_blocks);
    const size_t need = per_warp * zks::kWarps * size_t(blocks);
    if (need > sc->slab_bytes) {  // stream-ordered: no device-wide synchronisation
      if (sc->slab) ZKS_CUDA(cudaFreeAsync(sc->slab, e->stream));
      sc->slab = nullptr;
      sc->slab_bytes = 0;
      ZKS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&sc->slab), need, e->stream));
      sc->slab_bytes = need;
    }
    a.slab = sc->slab;
    a.slab_cap = c->n;
  }
  ZKS_CUDA(cudaMemsetAsync(a.work, 0, sizeof(unsigned long long), e->stream));
  {
    Timed tm(e, ZKS_KERNEL_SINGLE);
    kernel<<<(unsigned)blocks, zks::kThreads, smem, e->stream>>>(a);
    ZKS_CUDA(launched(e));
  }
  return ZKS_OK;
}

}  // namespace

extern "C" {

int zks_run_replicates(zks_engine* e, const zks_table* t, const zks_cell* c, double* ks_dev, double* gh_dev,
                       uint8_t* st_dev) {
  return run_replicates_impl(e, t, c, ks_dev, gh_dev, st_dev);
}

int zks_run_cells(zks_engine* e, int32_t ncells, const zks_table* const* tables, const zks_cell* cells,
                  double* const* ks_dev, double* const* gh_dev, uint8_t* const* st_dev) {
  if (!e || !tables || !cells || !ks_dev || !gh_dev || !st_dev) return fail(ZKS_EINVAL, "NULL argument");
  if (ncells < 1 || ncells > zks::kRowMaxCells)
    return fail(ZKS_EINVAL, "ncells %d outside [1, %d]", ncells, zks::kRowMaxCells);
  const zks_cell& c0 = cells[0];
  for (int j = 0; j < ncells; ++j) {
    if (int rc = check_cell(tables[j], &cells[j])) return rc;
    const zks_cell& c = cells[j];
    if (c.support_k != c0.support_k || c.n != c0.n || c.base_seed != c0.base_seed || c.repetition != c0.repetition ||
        c.first != c0.first || c.count != c0.count)
      return fail(ZKS_EINVAL, "cells of one call must differ only in gamma (cell %d)", j);
    if (c.count && (!ks_dev[j] || !gh_dev[j] || !st_dev[j])) return fail(ZKS_EINVAL, "output pointer %d is NULL", j);
  }
  if (c0.count == 0) return ZKS_OK;
  ZKS_CUDA(cudaSetDevice(e->device));
  if (e->mle_mode == ZKS_MLE_TABLE && c0.n >= zks::kLaneDrawMaxN && c0.n <= zks::kRowMaxN)
    return run_pre_rows(e, ncells, tables, cells, ks_dev, gh_dev, st_dev);
  if (e->mle_mode == ZKS_MLE_TABLE && c0.n < zks::kLaneDrawMaxN)
    return run_lane_rows(e, ncells, tables, cells, ks_dev, gh_dev, st_dev);
  for (int j = 0; j < ncells; ++j)  // other sizes: cell by cell (independent streams per launch)
    if (int rc = run_replicates_impl(e, tables[j], &cells[j], ks_dev[j], gh_dev[j], st_dev[j])) return rc;
  return ZKS_OK;
}

}  // extern "C"

namespace {
// the batch of a selection call (validation, candidate buffer); `global_counts` (optional) are
// the full arrays' lengths the ranks refer to when this GPU holds shards
int select_batch(zks_engine* e, const double* const* values_dev, const int64_t* counts, int32_t narrays,
                 const int64_t* ranks_host, int32_t nranks, double* const* out_dev, const uint8_t* const* status_dev,
                 uint8_t* const* worst_dev, const int64_t* global_counts, zks::SelectBatch* out,
                 zks::SelectState** sel, double** sel_out) {
  if (!e || !values_dev || !counts || !ranks_host || !out_dev) return fail(ZKS_EINVAL, "NULL argument");
  if (narrays < 1 || narrays > zks::kSelMaxArrays)
    return fail(ZKS_EINVAL, "narrays %d outside [1, %d]", narrays, zks::kSelMaxArrays);
  if (nranks < 1 || nranks > zks::kMaxRanks) return fail(ZKS_EINVAL, "nranks %d outside [1, %d]", nranks, zks::kMaxRanks);
  zks::SelectBatch& B = *out;
  std::memset(&B, 0, sizeof B);
  B.narrays = narrays;
  B.nr = nranks;
  for (int a = 0; a < narrays; ++a) {
    const int64_t full = global_counts ? global_counts[a] : counts[a];
    if (!out_dev[a] || (counts[a] > 0 && !values_dev[a])) return fail(ZKS_EINVAL, "NULL array %d", a);
    if (full < 1 || counts[a] < 0 || counts[a] > full) return fail(ZKS_EINVAL, "cannot take quantiles of an empty array");
    B.keys[a] = reinterpret_cast<const unsigned long long*>(values_dev[a]);
    B.count[a] = counts[a];
    B.out[a] = out_dev[a];
    B.status[a] = status_dev ? status_dev[a] : nullptr;
    B.worst[a] = (status_dev && status_dev[a] && worst_dev) ? worst_dev[a] : nullptr;
    for (int i = 0; i < nranks; ++i) {
      const int64_t r = ranks_host[int64_t(a) * nranks + i];
      if (r < 0 || r >= full)
        return fail(ZKS_EINVAL, "rank %lld out of range for %lld values", (long long)r, (long long)full);
      B.rank[a][i] = static_cast<unsigned long long>(r);
    }
  }
  ZKS_CUDA(cudaSetDevice(e->device));
  zks_engine::Scratch* sc = nullptr;
  ZKS_CUDA(scratch_for(e, &sc));
  int64_t total = 0;
  for (int a = 0; a < narrays; ++a) total += counts[a];
  if (size_t(total) * 8 > sc->cand_bytes) {
    if (sc->cand) ZKS_CUDA(cudaFreeAsync(sc->cand, e->stream));
    sc->cand = nullptr;
    sc->cand_bytes = 0;
    ZKS_CUDA(cudaMallocAsync(&sc->cand, std::max<size_t>(size_t(total) * 8, 8), e->stream));
    sc->cand_bytes = std::max<size_t>(size_t(total) * 8, 8);
  }
  B.cand = static_cast<unsigned long long*>(sc->cand);
  *sel = sc->sel;
  *sel_out = sc->sel_out;
  return ZKS_OK;
}

}  // namespace

extern "C" {

int zks_select_ranks_batch(zks_engine* e, const double* const* values_dev, const int64_t* counts, int32_t narrays,
                           const int64_t* ranks_host, int32_t nranks, double* const* out_dev,
                           const uint8_t* const* status_dev, uint8_t* const* worst_dev) {
  zks::SelectBatch B;
  zks::SelectState* st = nullptr;
  double* unused = nullptr;
  const int rc = select_batch(e, values_dev, counts, narrays, ranks_host, nranks, out_dev, status_dev, worst_dev,
                              nullptr, &B, &st, &unused);
  if (rc) return rc;
  int64_t most = 0;
  for (int a = 0; a < narrays; ++a) most = std::max<int64_t>(most, counts[a]);
  // one cooperative launch: every block resident (grid barriers between the radix passes)
  if (e->select_blocks == 0) {
    int per = 0;
    ZKS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, zks::select_kernel, 256, 0));
    e->select_blocks = std::max(1, std::min(per, ZKS_SELECT_PER_SM)) * e->sms;
  }
  const int blocks = static_cast<int>(
      std::max<int64_t>(1, std::min<int64_t>(e->select_blocks, (most * narrays + 255) / 256)));
  {
    Timed tm(e, ZKS_KERNEL_SELECT);
    void* args[] = {&B, &st};
    ZKS_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(zks::select_kernel), dim3(blocks), dim3(256),
                                         args, 0, e->stream));
    ZKS_CUDA(launched(e));
  }
  return ZKS_OK;
}

int zks_select_ranks_async(zks_engine* e, const double* values_dev, int64_t count, const int64_t* ranks_host,
                           int32_t nranks, double* out_dev) {
  return zks_select_ranks_batch(e, &values_dev, &count, 1, ranks_host, nranks, &out_dev, nullptr, nullptr);
}

int zks_select_dist_begin(zks_engine* e, const double* const* values_dev, const int64_t* counts,
                          const int64_t* global_counts, int32_t narrays, const int64_t* ranks_host, int32_t nranks,
                          double* const* out_dev, const uint8_t* const* status_dev, uint8_t* const* worst_dev) {
  if (!global_counts) return fail(ZKS_EINVAL, "NULL argument");
  zks::SelectBatch B;
  double* unused = nullptr;
  const int rc = select_batch(e, values_dev, counts, narrays, ranks_host, nranks, out_dev, status_dev, worst_dev,
                              global_counts, &B, &e->dist_sel, &unused);
  if (rc) return rc;
  e->dist = B;
  e->dist_active = true;
  int64_t most = 0;
  for (int a = 0; a < narrays; ++a) most = std::max<int64_t>(most, counts[a]);
  e->dist_blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(int64_t(e->sms) * 2, (most * narrays + 255) / 256)));
  Timed tm(e, ZKS_KERNEL_SELECT);
  zks::select_init_kernel<<<1, 256, 0, e->stream>>>(e->dist, e->dist_sel);
  ZKS_CUDA(launched(e));
  return ZKS_OK;
}

int zks_select_dist_count(zks_engine* e, int32_t pass, uint32_t* hist_dev) {
  if (!e || !hist_dev) return fail(ZKS_EINVAL, "NULL argument");
  if (!e->dist_active || pass < 0 || pass >= zks::kSelectPasses) return fail(ZKS_EINVAL, "no selection pass %d", pass);
  ZKS_CUDA(cudaSetDevice(e->device));
  Timed tm(e, ZKS_KERNEL_SELECT);
  zks::select_count_kernel<<<(unsigned)e->dist_blocks, 256, 0, e->stream>>>(e->dist, e->dist_sel, pass, hist_dev);
  ZKS_CUDA(launched(e));
  return ZKS_OK;
}

int zks_select_dist_pick(zks_engine* e, int32_t pass, const uint32_t* hist_dev) {
  if (!e || !hist_dev) return fail(ZKS_EINVAL, "NULL argument");
  if (!e->dist_active || pass < 0 || pass >= zks::kSelectPasses) return fail(ZKS_EINVAL, "no selection pass %d", pass);
  ZKS_CUDA(cudaSetDevice(e->device));
  {
    Timed tm(e, ZKS_KERNEL_SELECT);
    const int slots = e->dist.narrays * e->dist.nr;
    zks::select_pick_kernel<<<(unsigned)((slots + 7) / 8), 256, 0, e->stream>>>(e->dist, e->dist_sel, pass, hist_dev);
    ZKS_CUDA(launched(e));
  }
  if (pass == 1) {
    Timed tm(e, ZKS_KERNEL_SELECT);
    zks::select_compact_kernel<<<(unsigned)e->dist_blocks, 256, 0, e->stream>>>(e->dist, e->dist_sel);
    ZKS_CUDA(launched(e));
  }
  return ZKS_OK;
}

int zks_select_dist_end(zks_engine* e) {
  if (!e) return fail(ZKS_EINVAL, "engine is NULL");
  if (!e->dist_active) return fail(ZKS_EINVAL, "no selection in progress");
  ZKS_CUDA(cudaSetDevice(e->device));
  e->dist_active = false;
  Timed tm(e, ZKS_KERNEL_SELECT);
  zks::select_out_kernel<<<1, 256, 0, e->stream>>>(e->dist, e->dist_sel);
  ZKS_CUDA(launched(e));
  return ZKS_OK;
}

int zks_select_ranks(zks_engine* e, const double* values_dev, int64_t count, const int64_t* ranks_host,
                     int32_t nranks, double* out_host) {
  if (!e || !out_host) return fail(ZKS_EINVAL, "NULL argument");
  ZKS_CUDA(cudaSetDevice(e->device));
  zks_engine::Scratch* sc = nullptr;
  ZKS_CUDA(scratch_for(e, &sc));
  const int rc = zks_select_ranks_async(e, values_dev, count, ranks_host, nranks, sc->sel_out);
  if (rc) return rc;
  ZKS_CUDA(cudaMemcpyAsync(out_host, sc->sel_out, nranks * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
  ZKS_CUDA(cudaStreamSynchronize(e->stream));
  return ZKS_OK;
}

int zks_normaliser(zks_engine* e, double gamma, int32_t support_k, double* out_host) {
  if (!e || !out_host) return fail(ZKS_EINVAL, "NULL argument");
  if (support_k < 0 || support_k == 1 || support_k > 32766)
    return fail(ZKS_EINVAL, "finite support bound must be in [2, 32766], got %d", support_k);
  if (!(gamma == gamma) || gamma - gamma != 0.0) return fail(ZKS_EINVAL, "exponent must be finite, got %g", gamma);
  if (support_k == 0 && gamma < zks::kMinUnboundedGamma)
    return fail(ZKS_EINVAL, "unbounded support requires gamma >= 1.05, got %g", gamma);
  ZKS_CUDA(cudaSetDevice(e->device));
  zks_engine::Scratch* sc = nullptr;
  ZKS_CUDA(scratch_for(e, &sc));
  {
    Timed tm(e, ZKS_KERNEL_OTHER);
    zks::normaliser_kernel<<<1, 32, 0, e->stream>>>(gamma, support_k, e->logs, sc->sel_out);
    ZKS_CUDA(launched(e));
  }
  ZKS_CUDA(cudaMemcpyAsync(out_host, sc->sel_out, sizeof(double), cudaMemcpyDeviceToHost, e->stream));
  ZKS_CUDA(cudaStreamSynchronize(e->stream));
  return ZKS_OK;
}

int zks_engine_set_mle_mode(zks_engine* e, int mode) {
  if (!e) return fail(ZKS_EINVAL, "engine is NULL");
  if (mode != ZKS_MLE_TABLE && mode != ZKS_MLE_DIRECT) return fail(ZKS_EINVAL, "unknown MLE mode %d", mode);
  e->mle_mode = mode;
  return ZKS_OK;
}

int zks_fit_eval(zks_engine* e, int32_t support_k, const double* x_dev, int64_t count, double* mu_dev,
                 double* m2_dev, double* norm_dev) {
  if (!e || !x_dev || !mu_dev || !m2_dev || !norm_dev) return fail(ZKS_EINVAL, "NULL argument");
  if (support_k < 0 || support_k == 1 || support_k > 32766)
    return fail(ZKS_EINVAL, "finite support bound must be in [2, 32766], got %d", support_k);
  if (count <= 0) return ZKS_OK;
  ZKS_CUDA(cudaSetDevice(e->device));
  zks::FitTable* T = nullptr;
  const int rc = fit_table_for(e, support_k, &T);
  if (rc) return rc;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(int64_t(e->sms) * 4, (count + 255) / 256));
  {
    Timed tm(e, ZKS_KERNEL_OTHER);
    zks::fit_eval_kernel<<<(unsigned)blocks, 256, 0, e->stream>>>(*T, x_dev, count, mu_dev, m2_dev, norm_dev);
    ZKS_CUDA(launched(e));
  }
  return ZKS_OK;
}

int zks_engine_set_counters(zks_engine* e, unsigned long long* counters_dev) {
  if (!e) return fail(ZKS_EINVAL, "engine is NULL");
  e->counters = counters_dev;
  return ZKS_OK;
}

int zks_probe_peaks(zks_engine* e, double* out_host) {
  if (!e || !out_host) return fail(ZKS_EINVAL, "NULL argument");
  ZKS_CUDA(cudaSetDevice(e->device));
  return zks::probe_peaks(e->stream, e->sms, out_host) ? ZKS_OK : fail(ZKS_ECUDA, "peak probe failed");
}

int zks_stream_uniforms(zks_engine* e, uint64_t seed, uint64_t rep, uint64_t idx, int64_t count, double* out_dev) {
  if (!e || !out_dev) return fail(ZKS_EINVAL, "NULL argument");
  if (count < 0) return fail(ZKS_EINVAL, "count must be >= 0");
  if (count == 0) return ZKS_OK;
  ZKS_CUDA(cudaSetDevice(e->device));
  const int64_t nb = (count + 3) / 4;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(int64_t(e->sms) * 8, (nb + 255) / 256));
  {
    Timed tm(e, ZKS_KERNEL_OTHER);
    zks::uniforms_kernel<<<(unsigned)blocks, 256, 0, e->stream>>>(seed, rep, idx, 0, count, out_dev);
    ZKS_CUDA(launched(e));
  }
  return ZKS_OK;
}

int zks_stream_uniforms_key(zks_engine* e, uint64_t k0, uint64_t k1, int64_t count, double* out_dev) {
  if (!e || !out_dev) return fail(ZKS_EINVAL, "NULL argument");
  if (count < 0) return fail(ZKS_EINVAL, "count must be >= 0");
  if (count == 0) return ZKS_OK;
  ZKS_CUDA(cudaSetDevice(e->device));
  const int64_t nb = (count + 3) / 4;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(int64_t(e->sms) * 8, (nb + 255) / 256));
  {
    Timed tm(e, ZKS_KERNEL_OTHER);
    zks::uniforms_kernel<<<(unsigned)blocks, 256, 0, e->stream>>>(k0, k1, 0, 1, count, out_dev);
    ZKS_CUDA(launched(e));
  }
  return ZKS_OK;
}

int zks_draw(zks_engine* e, const zks_table* t, const double* u_dev, int64_t count, int64_t* out_dev) {
  if (!e || !t || !u_dev || !out_dev) return fail(ZKS_EINVAL, "NULL argument");
  if (count < 0) return fail(ZKS_EINVAL, "count must be >= 0");
  if (count == 0) return ZKS_OK;
  ZKS_CUDA(cudaSetDevice(e->device));
  ZKS_CUDA(table_use(e, t));
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(int64_t(e->sms) * 8, (count + 255) / 256));
  {
    Timed tm(e, ZKS_KERNEL_OTHER);
    zks::draw_kernel<<<(unsigned)blocks, 256, 0, e->stream>>>(t->cdf, t->guide, t->len, u_dev, count, out_dev);
    ZKS_CUDA(launched(e));
  }
  return ZKS_OK;
}

}  // extern "C"

namespace {

zks::MleParams mle_params(const zks_mle_settings* s) {
  zks::MleParams P;
  if (s) {
    P.x0 = s->initial_guess;
    P.tol = s->absolute_tolerance;
    P.max_iter = s->max_iterations;
    P.lo = s->bracket_lo;
    P.hi = s->bracket_hi;
  }
  return P;
}

int check_support(int32_t k) {
  if (k < 0 || k == 1 || k > 32766) return fail(ZKS_EINVAL, "finite support bound must be in [2, 32766], got %d", k);
  return ZKS_OK;
}

}  // namespace

extern "C" {

int zks_fit_samples(zks_engine* e, int32_t support_k, const int64_t* values_dev, const int64_t* offsets_dev,
                    int64_t nsamples, int32_t mode, const zks_mle_settings* settings, const double* gamma_in_dev,
                    const double* norm_in_dev, double* log_mean_dev, double* gamma_dev, double* ks_dev,
                    int64_t* argmax_dev, uint8_t* status_dev) {
  if (!e || !offsets_dev || !log_mean_dev || !gamma_dev || !ks_dev || !argmax_dev || !status_dev)
    return fail(ZKS_EINVAL, "NULL argument");
  if (int rc = check_support(support_k)) return rc;
  if (nsamples < 0) return fail(ZKS_EINVAL, "nsamples must be >= 0");
  if (!(mode & ZKS_FIT_EXPONENT) && (mode & ZKS_FIT_KS) && !gamma_in_dev)
    return fail(ZKS_EINVAL, "scoring without a fit needs the model exponents");
  const zks::MleParams P = mle_params(settings);
  if (settings && (P.tol <= 0.0 || P.max_iter < 1 || !(P.lo < P.x0 && P.x0 < P.hi)))
    return fail(ZKS_EINVAL, "invalid MLE settings");
  if (nsamples == 0) return ZKS_OK;
  ZKS_CUDA(cudaSetDevice(e->device));
  zks::SamplesArgs a{};
  a.values = values_dev;
  a.offsets = offsets_dev;
  a.nsamples = nsamples;
  a.K = support_k;
  a.logs = e->logs;
  a.mle = P;
  a.mode = mode;
  a.gamma_in = gamma_in_dev;
  a.norm_in = norm_in_dev;
  a.log_mean_out = log_mean_dev;
  a.gamma_out = gamma_dev;
  a.ks_out = ks_dev;
  a.argmax_out = argmax_dev;
  a.status_out = status_dev;
  a.hist_words = zks::round_up(zks::kSamplesHist + 1, 4);
  zks_engine::Scratch* sc = nullptr;
  ZKS_CUDA(scratch_for(e, &sc));
  a.work = sc->work;
  // the fit tables cover [-20, 20] (finite) and [1.05, 20] (unbounded): wider brackets sum directly
  a.use_table = e->mle_mode == ZKS_MLE_TABLE && (support_k == 0 || (P.lo >= -20.0 && P.hi <= 20.0));
  if (a.use_table) {
    zks::FitTable* T = nullptr;
    if (int rc = fit_table_for(e, support_k, &T)) return rc;
    a.fit = *T;
  }
  const size_t smem = size_t(zks::kWarps) * (a.hist_words + zks::kKsQueueWords) * 4;
  ZKS_CUDA(cudaFuncSetAttribute(zks::samples_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(int64_t(e->sms) * 2, (nsamples + zks::kWarps - 1) / zks::kWarps));
  ZKS_CUDA(cudaMemsetAsync(a.work, 0, sizeof(unsigned long long), e->stream));
  {
    Timed tm(e, ZKS_KERNEL_OTHER);
    zks::samples_kernel<<<(unsigned)blocks, zks::kThreads, smem, e->stream>>>(a);
    ZKS_CUDA(launched(e));
  }
  return ZKS_OK;
}

int zks_series_eval(zks_engine* e, int32_t support_k, const double* gamma_dev, int64_t count, double* out_dev) {
  if (!e || !gamma_dev || !out_dev) return fail(ZKS_EINVAL, "NULL argument");
  if (int rc = check_support(support_k)) return rc;
  if (count <= 0) return ZKS_OK;
  ZKS_CUDA(cudaSetDevice(e->device));
  const int64_t blocks = (count * 32 + 255) / 256;
  {
    Timed tm(e, ZKS_KERNEL_OTHER);
    zks::series_kernel<<<(unsigned)blocks, 256, 0, e->stream>>>(gamma_dev, count, support_k, e->logs, out_dev);
    ZKS_CUDA(launched(e));
  }
  return ZKS_OK;
}

int zks_tail_mass(zks_engine* e, double gamma, const double* start_dev, int64_t count, double* out_dev) {
  if (!e || !start_dev || !out_dev) return fail(ZKS_EINVAL, "NULL argument");
  if (count <= 0) return ZKS_OK;
  ZKS_CUDA(cudaSetDevice(e->device));
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(int64_t(e->sms) * 4, (count + 255) / 256));
  {
    Timed tm(e, ZKS_KERNEL_OTHER);
    zks::tail_mass_kernel<<<(unsigned)blocks, 256, 0, e->stream>>>(gamma, start_dev, count, out_dev);
    ZKS_CUDA(launched(e));
  }
  return ZKS_OK;
}

int zks_solve_exponents(zks_engine* e, int32_t support_k, const double* target_dev, int64_t count,
                        const zks_mle_settings* settings, int32_t bisect_only, double* gamma_dev, uint8_t* status_dev) {
  if (!e || !target_dev || !gamma_dev || !status_dev) return fail(ZKS_EINVAL, "NULL argument");
  if (int rc = check_support(support_k)) return rc;
  if (count <= 0) return ZKS_OK;
  ZKS_CUDA(cudaSetDevice(e->device));
  const int64_t blocks = (count * 32 + 255) / 256;
  {
    Timed tm(e, ZKS_KERNEL_OTHER);
    zks::solve_kernel<<<(unsigned)blocks, 256, 0, e->stream>>>(target_dev, count, support_k, e->logs, mle_params(settings),
                                                               bisect_only, gamma_dev, status_dev);
    ZKS_CUDA(launched(e));
  }
  return ZKS_OK;
}

}  // extern "C"
