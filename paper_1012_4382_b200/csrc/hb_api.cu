// C ABI of libheomb200.so (see include/heom_b200.h).
//
// The handle owns the device state of one propagation: the hierarchy tables
// (built on the device, hb_graph.cu), four AoSoA state buffers (sigma, Y2, Y3,
// Y4), the control block, the record buffer, a private CUDA stream and a CUDA
// graph of `chunk_steps` RK4 steps (4 stage kernels each).  hb_run replays the
// graph and synchronises once per chunk to drain records and read the status
// written by the last CTA of each stage-4 kernel (hb_stage.cu).
#include <dlfcn.h>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>
#include "hb_handle.h"

using namespace hb;

static thread_local std::string g_err;

int hb::fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int hb::cuda_fail(cudaError_t e, const char* where) {
  cudaGetLastError();  // clear sticky-free errors
  return fail(HB_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// Host<->device bytes moved by the library (every copy goes through hb_memcpy):
// the end-to-end benchmark reads them around a propagate() call.
static std::atomic<long long> g_io_h2d{0}, g_io_d2h{0};

cudaError_t hb::hb_memcpy(void* dst, const void* src, size_t n, cudaMemcpyKind kind,
                           cudaStream_t s) {
  if (kind == cudaMemcpyHostToDevice) g_io_h2d += (long long)n;
  if (kind == cudaMemcpyDeviceToHost) g_io_d2h += (long long)n;
  return cudaMemcpyAsync(dst, src, n, kind, s);
}

void hb_io_bytes(int64_t* h2d, int64_t* d2h) {
  if (h2d) *h2d = g_io_h2d.load();
  if (d2h) *d2h = g_io_d2h.load();
}

// Device hierarchy tables are immutable, so handles with the same
// (modes, n_max, ordering, device) share one copy -- the analogue of the
// reference's lru_cache'd _graph (heom.py:222-224).
namespace {
using GraphKey = std::tuple<int, int, int, int>;
std::mutex g_graph_mu;
std::map<GraphKey, std::shared_ptr<CachedGraph>> g_graphs;  // LRU of 8, like lru_cache(8)
std::vector<GraphKey> g_graph_lru;

cudaError_t shared_graph(int modes, int n_max, int ordering, int device, cudaStream_t s,
                         std::shared_ptr<CachedGraph>* out) {
  std::lock_guard<std::mutex> lk(g_graph_mu);
  const GraphKey key{modes, n_max, ordering, device};
  auto touch = [&] {
    for (size_t i = 0; i < g_graph_lru.size(); ++i)
      if (g_graph_lru[i] == key) {
        g_graph_lru.erase(g_graph_lru.begin() + i);
        break;
      }
    g_graph_lru.push_back(key);
  };
  auto it = g_graphs.find(key);
  if (it != g_graphs.end()) {
    *out = it->second;
    touch();
    return cudaSuccess;
  }
  auto sp = std::make_shared<CachedGraph>();
  cudaError_t e = build_graph(modes, n_max, ordering, s, nullptr, nullptr, nullptr, nullptr,
                              nullptr, &sp->gt);
  if (e != cudaSuccess) return e;
  g_graphs[key] = sp;
  touch();
  while (g_graph_lru.size() > 8) {  // handles still using an evicted graph keep it alive
    g_graphs.erase(g_graph_lru.front());
    g_graph_lru.erase(g_graph_lru.begin());
  }
  *out = sp;
  return cudaSuccess;
}
}  // namespace

// definitions take C linkage from the extern "C" declarations in heom_b200.h

const char* hb_last_error(void) { return g_err.c_str(); }

int hb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int64_t hb_hierarchy_size(int modes, int n_max) { return hierarchy_size(modes, n_max); }

static int check_graph_args(int modes, int n_max, int64_t* n_tot) {
  if (modes < 1) return fail(HB_ERR_ARG, "need at least one site");
  if (n_max < 0) return fail(HB_ERR_ARG, "truncation tier must be >= 0");
  if (modes > MAX_MODES) return fail(HB_ERR_ARG, "more than 64 modes is not supported");
  const int64_t n = hierarchy_size(modes, n_max);
  if (n < 0 || n > INT32_MAX) {
    char buf[160];
    if (n < 0)
      snprintf(buf, sizeof buf, "hierarchy with more than 2^63 indices exceeds the supported index range");
    else
      snprintf(buf, sizeof buf, "hierarchy with %lld indices exceeds the supported index range",
               (long long)n);
    return fail(HB_ERR_RANGE, buf);
  }
  *n_tot = n;
  return HB_OK;
}

int hb_graph_build(int modes, int n_max, int device, int32_t* indices, int32_t* tiers,
                   int32_t* plus, int32_t* minus, int32_t* perm_or_null) {
  int64_t n_tot = 0;
  int rc = check_graph_args(modes, n_max, &n_tot);
  if (rc) return rc;
  CK(cudaSetDevice(device));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaError_t e = build_graph(modes, n_max, HB_ORDER_LEX, s, indices, tiers, plus, minus,
                              perm_or_null, nullptr);
  cudaStreamDestroy(s);
  if (e != cudaSuccess) return cuda_fail(e, "build_graph");
  return HB_OK;
}

// ---------------------------------------------------------------------------
// Level-2 kernel ABI shims

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() { if (p) cudaFree(p); }
  cudaError_t alloc(size_t n) { return cudaMalloc(&p, n ? n : 8); }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

static int rhs_impl(double* out, const double* sig, int64_t n_tot, int d, const double* h,
                    const int32_t* site_of, const int32_t* plus, const int32_t* minus, int modes,
                    const double* nvec, const double* tier_damp, double a_comm, double b_anti,
                    const double* decay, int n_refill, const int32_t* refill_dst,
                    const int32_t* refill_src, const double* refill_rate, int device) {
  if (n_refill < 0 || n_refill > MAXT) return fail(HB_ERR_ARG, "too many refill channels");
  if (d < 1 || d > MAXD) return fail(HB_ERR_ARG, "block dimension must be 1..9");
  if (n_tot < 1 || n_tot > INT32_MAX) return fail(HB_ERR_ARG, "bad n_tot");
  if (modes < 1 || modes > MAX_MODES) return fail(HB_ERR_ARG, "bad mode count");
  std::vector<uint8_t> nv((size_t)n_tot * modes);
  for (size_t i = 0; i < nv.size(); ++i) {
    const double v = nvec[i];
    if (!(v >= 0.0 && v <= 255.0 && v == std::floor(v)))
      return fail(HB_ERR_ARG, "nvec must hold integers 0..255");
    nv[i] = (uint8_t)v;
  }
  CK(cudaSetDevice(device));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct SG { cudaStream_t s; ~SG() { cudaStreamDestroy(s); } } sg{s};
  GraphTables gt;
  struct GG { GraphTables* g; ~GG() { free_graph(g); } } gg{&gt};
  CK(upload_tables(modes, (int)n_tot, plus, minus, nv.data(), s, &gt));
  KParams p{};
  p.d = d;
  p.n_sites = modes;
  p.kp1 = 1;
  p.modes = modes;
  p.n_tot = (int)n_tot;
  p.n_tiles = gt.n_tiles;
  p.n_tiles_total = gt.n_tiles;
  p.hermitian = 0;
  p.n_planes = 2 * d * d;
  for (int i = 0; i < d; ++i) {
    for (int j = 0; j < d; ++j) p.h[i * MAXD + j] = h[i * d + j];
    p.site_of[i] = site_of[i];
    p.decay[i] = decay[i];
  }
  p.a[0] = a_comm;
  p.b[0] = b_anti;
  p.n_refill = n_refill;
  for (int q = 0; q < n_refill; ++q) {
    if (refill_dst[q] < 0 || refill_dst[q] >= d || refill_src[q] < 0 || refill_src[q] >= d)
      return fail(HB_ERR_ARG, "refill channel out of range");
    p.refill_dst[q] = refill_dst[q];
    p.refill_src[q] = refill_src[q];
    p.refill_rate[q] = refill_rate[q];
  }
  const size_t n_pad = (size_t)gt.n_tiles * TILE;
  const size_t ref_bytes = (size_t)n_tot * d * d * 2 * sizeof(double);
  const size_t dev_bytes = n_pad * p.n_planes * sizeof(double);
  DevBuf dref, din, dout, ddamp;
  CK(dref.alloc(ref_bytes));
  CK(din.alloc(dev_bytes));
  CK(dout.alloc(dev_bytes));
  CK(ddamp.alloc(n_pad * sizeof(double)));
  CK(cudaMemsetAsync(ddamp.p, 0, n_pad * sizeof(double), s));
  CK(hb_memcpy(ddamp.p, tier_damp, (size_t)n_tot * sizeof(double), cudaMemcpyHostToDevice, s));
  CK(hb_memcpy(dref.p, sig, ref_bytes, cudaMemcpyHostToDevice, s));
  CK(launch_pack(p, dref.as<double>(), gt.dev2ref, din.as<double>(), s));
  p.Yin = din.as<double>();
  p.Yout = dout.as<double>();
  p.plus = gt.plus_t;
  p.minus = gt.minus_t;
  p.nvec = gt.nvec_t;
  p.damp_plane = ddamp.as<double>();
  CK(configure_stages(p));
  CK(launch_rhs_only(p, s));
  CK(launch_unpack(p, dout.as<double>(), gt.dev2ref, dref.as<double>(), s));
  CK(hb_memcpy(out, dref.p, ref_bytes, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return HB_OK;
}

int hb_rhs(double* out, const double* sig, int64_t n_tot, int d, const double* h,
           const int32_t* site_of, const int32_t* plus, const int32_t* minus, int modes,
           const double* nvec, const double* tier_damp, double a_comm, double b_anti,
           const double* decay, int device) {
  return rhs_impl(out, sig, n_tot, d, h, site_of, plus, minus, modes, nvec, tier_damp, a_comm,
                  b_anti, decay, 0, nullptr, nullptr, nullptr, device);
}

int hb_heom_rhs(double* out, const double* sig, int64_t n_tot, int d, const double* h,
                const int32_t* site_of, const int32_t* plus, const int32_t* minus, int modes,
                const double* nvec, const double* tier_damp, double a_comm, double b_anti,
                const double* decay, int n_refill, const int32_t* refill_dst,
                const int32_t* refill_src, const double* refill_rate, int device) {
  return rhs_impl(out, sig, n_tot, d, h, site_of, plus, minus, modes, nvec, tier_damp, a_comm,
                  b_anti, decay, n_refill, refill_dst, refill_src, refill_rate, device);
}

static int elementwise(int op, double* out, const double* x, const double* y, const double* z,
                       const double* w, double c, int64_t n, int device) {
  if (n < 0) return fail(HB_ERR_ARG, "negative size");
  if (n == 0) return HB_OK;
  CK(cudaSetDevice(device));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct SG { cudaStream_t s; ~SG() { cudaStreamDestroy(s); } } sg{s};
  const size_t bytes = (size_t)n * 2 * sizeof(double);
  DevBuf o, a, b, cc, dd;
  CK(o.alloc(bytes));
  CK(a.alloc(bytes));
  CK(b.alloc(bytes));
  CK(hb_memcpy(a.p, x, bytes, cudaMemcpyHostToDevice, s));
  CK(hb_memcpy(b.p, y, bytes, cudaMemcpyHostToDevice, s));
  if (op == 1) {
    CK(cc.alloc(bytes));
    CK(dd.alloc(bytes));
    CK(hb_memcpy(o.p, out, bytes, cudaMemcpyHostToDevice, s));
    CK(hb_memcpy(cc.p, z, bytes, cudaMemcpyHostToDevice, s));
    CK(hb_memcpy(dd.p, w, bytes, cudaMemcpyHostToDevice, s));
  }
  CK(launch_elementwise(op, n, o.as<double>(), a.as<double>(), b.as<double>(), cc.as<double>(),
                        dd.as<double>(), c, s));
  CK(hb_memcpy(out, o.p, bytes, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return HB_OK;
}

int hb_add_scaled(double* out, const double* x, const double* y, double c, int64_t n, int device) {
  return elementwise(0, out, x, y, nullptr, nullptr, c, n, device);
}

int hb_rk4_update(double* sig, const double* k1, const double* k2, const double* k3,
                  const double* k4, double w, int64_t n, int device) {
  return elementwise(1, sig, k1, k2, k3, k4, w, n, device);
}

int hb_max_abs2(const double* x, int64_t n, double* result, int device) {
  if (n < 0) return fail(HB_ERR_ARG, "negative size");
  *result = 0.0;
  if (n == 0) return HB_OK;
  CK(cudaSetDevice(device));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct SG { cudaStream_t s; ~SG() { cudaStreamDestroy(s); } } sg{s};
  const size_t bytes = (size_t)n * 2 * sizeof(double);
  DevBuf a, r;
  CK(a.alloc(bytes));
  CK(r.alloc(sizeof(unsigned long long)));
  CK(cudaMemsetAsync(r.p, 0, sizeof(unsigned long long), s));
  CK(hb_memcpy(a.p, x, bytes, cudaMemcpyHostToDevice, s));
  CK(launch_max_abs2(n, a.as<double>(), r.as<unsigned long long>(), s));
  unsigned long long bits = 0;
  CK(hb_memcpy(&bits, r.p, sizeof bits, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  std::memcpy(result, &bits, sizeof(double));
  return HB_OK;
}

// ---------------------------------------------------------------------------
// Level-1 propagator

// Device buffer pool: propagate() creates and destroys a handle per call, and
// cudaMalloc/cudaFree of the 4-5 state buffers (125 MB each at config 4) is
// synchronous and costs milliseconds; released buffers are kept per (device,
// size) up to kPoolCap bytes and handed to the next handle of the same shape
// (which zeroes them, alloc_state).
struct BufPool {
  std::mutex mu;
  std::multimap<std::pair<int, size_t>, void*> idle;
  size_t cached = 0;
};
static BufPool& buf_pool() {
  static BufPool* p = new BufPool();  // never destroyed: the driver reclaims at exit
  return *p;
}
constexpr size_t kPoolCap = size_t(24) << 30;

static void pool_trim_device(int device) {
  BufPool& P = buf_pool();
  std::lock_guard<std::mutex> lk(P.mu);
  for (auto it = P.idle.begin(); it != P.idle.end();) {
    if (device < 0 || it->first.first == device) {
      int cur = 0;
      cudaGetDevice(&cur);
      cudaSetDevice(it->first.first);
      cudaFree(it->second);
      cudaSetDevice(cur);
      P.cached -= it->first.second;
      it = P.idle.erase(it);
    } else {
      ++it;
    }
  }
}

cudaError_t hb::pool_alloc(int device, size_t bytes, void** out) {
  {
    BufPool& P = buf_pool();
    std::lock_guard<std::mutex> lk(P.mu);
    auto it = P.idle.find({device, bytes});
    if (it != P.idle.end()) {
      *out = it->second;
      P.idle.erase(it);
      P.cached -= bytes;
      return cudaSuccess;
    }
  }
  cudaError_t e = cudaMalloc(out, bytes);
  if (e == cudaErrorMemoryAllocation) {  // idle pooled buffers may be what is missing
    cudaGetLastError();
    pool_trim_device(device);
    e = cudaMalloc(out, bytes);
  }
  return e;
}

void hb::pool_release(int device, size_t bytes, void* p) {
  BufPool& P = buf_pool();
  std::lock_guard<std::mutex> lk(P.mu);
  if (P.cached + bytes > kPoolCap) {
    cudaFree(p);
    return;
  }
  P.idle.insert({{device, bytes}, p});
  P.cached += bytes;
}

// Streams and pinned control blocks are pooled too: propagate() creates a
// handle per call, and cudaStreamCreate / cudaMallocHost cost tens of
// microseconds to milliseconds each.
struct HostPool {
  std::mutex mu;
  std::multimap<int, cudaStream_t> streams;
  std::vector<Ctl*> pinned;
};
static HostPool& host_pool() {
  static HostPool* p = new HostPool();
  return *p;
}

static cudaError_t stream_acquire(int device, cudaStream_t* s) {
  {
    HostPool& H = host_pool();
    std::lock_guard<std::mutex> lk(H.mu);
    auto it = H.streams.find(device);
    if (it != H.streams.end()) {
      *s = it->second;
      H.streams.erase(it);
      return cudaSuccess;
    }
  }
  return cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
}

static void stream_release(int device, cudaStream_t s) {
  HostPool& H = host_pool();
  std::lock_guard<std::mutex> lk(H.mu);
  if (H.streams.count(device) >= 64) {
    cudaStreamDestroy(s);
    return;
  }
  H.streams.insert({device, s});
}

static cudaError_t pinned_acquire(Ctl** c) {
  {
    HostPool& H = host_pool();
    std::lock_guard<std::mutex> lk(H.mu);
    if (!H.pinned.empty()) {
      *c = H.pinned.back();
      H.pinned.pop_back();
      return cudaSuccess;
    }
  }
  return cudaMallocHost(reinterpret_cast<void**>(c), sizeof(Ctl));
}

static void pinned_release(Ctl* c) {
  HostPool& H = host_pool();
  std::lock_guard<std::mutex> lk(H.mu);
  if (H.pinned.size() >= 256) {
    cudaFreeHost(c);
    return;
  }
  H.pinned.push_back(c);
}

// Frees every idle pooled device buffer (all devices).  Buffers of live handles
// are untouched.
void hb_pool_trim(void) { pool_trim_device(-1); }

// The device's L2 set-aside for persisting accesses: grown to the largest
// window a handle asked for (capped at the device maximum) -- a larger set-aside
// than the window costs the streamed accesses L2 capacity (measured: the
// 83 MB maximum against a 45 MB window makes config 4 17 % slower).
static size_t persisting_l2(int device, size_t want, size_t max_persist) {
  static std::mutex mu;
  static std::map<int, size_t> cur;
  std::lock_guard<std::mutex> lk(mu);
  size_t& c = cur[device];
  const size_t w = std::min(want, max_persist);
  if (w > c) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, w) == cudaSuccess) {
      size_t got = 0;
      cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize);
      c = got;
    }
    cudaGetLastError();
    cudaSetDevice(prev);
  }
  return c;
}

// Instantiated step graphs, keyed by the bytes of the four stages' kernel
// parameters (+ chunk and device): instantiating 4 x chunk_steps kernel nodes
// costs ~20 ms at chunk 64, as much as a few hundred steps of a small
// hierarchy.  With pooled buffers a repeated propagate() of the same shape sees
// identical parameters and replays the cached graph.  A graph is owned by at
// most one handle at a time (identical parameters mean identical buffers, which
// the pool never hands to two live handles).
struct GraphCache {
  std::mutex mu;
  struct Entry {
    std::string key;
    cudaGraphExec_t exec;
    int64_t nodes;
  };
  std::vector<Entry> lru;  // most recent last
};
static GraphCache& graph_cache() {
  static GraphCache* c = new GraphCache();
  return *c;
}
constexpr size_t kGraphCacheCap = 8;

// step graphs launched per host synchronisation in hb_run (records buffer sized
// for all of them)
constexpr int kGraphsPerSync = 2;
// RK4 steps per WHILE-body (PDL-chained inside a body; a run stops within the
// body of its stop step)
constexpr int kDefaultBodySteps = 16;


static void graph_cache_put(hb_handle* h) {
  if (!h->graph) return;
  GraphCache& G = graph_cache();
  std::lock_guard<std::mutex> lk(G.mu);
  G.lru.push_back({h->graph_key, h->graph, h->graph_nodes});
  if (G.lru.size() > kGraphCacheCap) {
    cudaGraphExecDestroy(G.lru.front().exec);
    G.lru.erase(G.lru.begin());
  }
  h->graph = nullptr;
}

static cudaGraphExec_t graph_cache_take(const std::string& key, int64_t* nodes) {
  GraphCache& G = graph_cache();
  std::lock_guard<std::mutex> lk(G.mu);
  for (auto it = G.lru.rbegin(); it != G.lru.rend(); ++it)
    if (it->key == key) {
      cudaGraphExec_t g = it->exec;
      *nodes = it->nodes;
      G.lru.erase(std::next(it).base());
      return g;
    }
  return nullptr;
}

static void free_state(hb_handle* h) {
  if (h->stream) cudaStreamSynchronize(h->stream);  // no work in flight on the buffers
  for (auto& b : h->buf) {
    if (b) pool_release(h->device, h->buf_bytes, b);
    b = nullptr;
  }
  graph_cache_put(h);
  h->graph_layout = -1;
}


void hb_destroy(hb_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  free_shard(h);
  free_state(h);
  h->graph_ref.reset();
  if (h->ctl) pool_release(h->device, sizeof(Ctl), h->ctl);
  if (h->ctl_host) pinned_release(h->ctl_host);
  if (h->rec_step) pool_release(h->device, h->rec_cap * sizeof(long long), h->rec_step);
  if (h->rec_pops) pool_release(h->device, h->rec_cap * h->prm.d_full * sizeof(double), h->rec_pops);
  if (h->rec_mats)
    pool_release(h->device, h->rec_cap * h->prm.d_full * h->prm.d_full * 2 * sizeof(double),
                 h->rec_mats);
  if (h->stream) stream_release(h->device, h->stream);
  delete h;
}

// T != null: a shard (hb_create_shard) with caller-built local tables
static int create_impl(const hb_params* P, const hb_shard_tables* T, hb_handle** out) {
  *out = nullptr;
  if (!P) return fail(HB_ERR_ARG, "null params");
  const hb_params& q = *P;
  if (q.d < 1 || q.d > MAXD) return fail(HB_ERR_ARG, "block dimension must be 1..9");
  if (q.kp1 < 1 || q.kp1 > MAXKP1) return fail(HB_ERR_ARG, "n_matsubara must be 0..7");
  if (q.n_max > 255) return fail(HB_ERR_ARG, "n_max > 255 is not supported");
  if (q.n_sinks < 0 || q.n_sinks > MAXS) return fail(HB_ERR_ARG, "too many sinks");
  if (q.n_site_pos < 0 || q.n_site_pos > MAXD) return fail(HB_ERR_ARG, "bad site positions");
  if (q.d_full < q.d) return fail(HB_ERR_ARG, "d_full < d");
  if (q.d_full > MAXFULL) return fail(HB_ERR_ARG, "full basis dimension above 16 is not supported");
  if (!(q.dt > 0)) return fail(HB_ERR_ARG, "dt must be > 0");
  if (q.record_stride < 1) return fail(HB_ERR_ARG, "record stride must be >= 1");
  if (q.ordering < HB_ORDER_LEX || q.ordering > HB_ORDER_LEX_SPLIT)
    return fail(HB_ERR_ARG, "ordering must be 'lex', 'lex-split' or 'reference'");
  if (q.precision != HB_PREC_DOUBLE && q.precision != HB_PREC_SINGLE)
    return fail(HB_ERR_ARG, "precision must be 'double' or 'single'");
  int nterms = 0;
  for (int s = 0; s < q.n_sinks; ++s) nterms += q.sink_nterms[s];
  if (nterms > MAXT) return fail(HB_ERR_ARG, "too many sink terms");
  const int modes = q.n_sites * q.kp1;
  int64_t n_tot = 0;
  int rc = check_graph_args(modes, q.n_max, &n_tot);
  if (rc) return rc;
  if (T) {
    if (T->n_local < TILE || T->n_local % TILE != 0)
      return fail(HB_ERR_ARG, "shard: n_local must be a positive multiple of 32");
    if (T->own_tiles < 1 || T->own_tiles > T->n_local / TILE)
      return fail(HB_ERR_ARG, "shard: own_tiles outside the local slots");
    if (!q.has_t_end) return fail(HB_ERR_ARG, "sharded runs need the t_end stop policy");
    int gsum = 0;
    for (int g = 0; g < 4; ++g) {
      if (T->group_count[g] < 0) return fail(HB_ERR_ARG, "shard: negative group size");
      gsum += T->group_count[g];
    }
    if (gsum != T->own_tiles) return fail(HB_ERR_ARG, "shard: the groups must partition the owned tiles");
    for (int i = 0; i < gsum; ++i)
      if (T->groups[i] < 0 || T->groups[i] >= T->own_tiles)
        return fail(HB_ERR_ARG, "shard: group tile outside the owned tiles");
    n_tot = T->n_local;
  }

  hb_handle* h = new hb_handle();
  h->prm = q;
  h->device = q.device;
  h->modes = modes;
  h->n_tot = (int)n_tot;
  // steps per CUDA-graph body (ensure_graph); a graph launch runs up to
  // loop_iters bodies: 128 records' worth of steps at stride 1, more for sparse
  // records (fewer host synchronisations), at most 16,384
  h->chunk = q.chunk_steps > 0 ? q.chunk_steps : kDefaultBodySteps;
  {
    const int64_t want = std::max<int64_t>(h->chunk, std::min<int64_t>(128 * q.record_stride, 16384));
    h->loop_iters = (want + h->chunk - 1) / h->chunk;
  }
  const int d = q.d;
  h->h.assign(q.h, q.h + d * d);
  h->decay.assign(q.decay, q.decay + d);
  h->site_of.assign(q.site_of, q.site_of + d);
  h->nu.assign(q.nu, q.nu + q.kp1);
  h->a.assign(q.a, q.a + q.kp1);
  h->b.assign(q.b, q.b + q.kp1);
  h->sink_nterms.assign(q.sink_nterms, q.sink_nterms + q.n_sinks);
  h->sink_rate.assign(q.sink_rate, q.sink_rate + nterms);
  h->sink_pos.assign(q.sink_pos, q.sink_pos + nterms);
  h->site_pos.assign(q.site_pos, q.site_pos + q.n_site_pos);
  h->block_full.assign(q.block_full, q.block_full + d);
  h->sink_full.assign(q.sink_full, q.sink_full + q.n_sinks);
  for (int i = 0; i < d; ++i)
    if (h->site_of[i] >= q.n_sites) {
      delete h;
      return fail(HB_ERR_ARG, "site_of out of range");
    }
  auto bail = [&](cudaError_t e, const char* w) {
    int r = cuda_fail(e, w);
    hb_destroy(h);
    return r;
  };
  cudaError_t e = cudaSetDevice(h->device);
  if (e) return bail(e, "cudaSetDevice");
  e = stream_acquire(h->device, &h->stream);
  if (e) return bail(e, "cudaStreamCreate");
  if (T) {
    std::vector<uint8_t> nv(T->nvec, T->nvec + (size_t)T->n_local * modes);
    e = upload_tables(modes, T->n_local, T->plus, T->minus, nv.data(), h->stream, &h->own_gt);
    if (e) return bail(e, "upload shard tables");
    h->gt = h->own_gt;
    h->n_tiles = h->gt.n_tiles;
    h->own_tiles = T->own_tiles;
    h->shard = true;
    int rs = init_shard(h, T);
    if (rs) {
      hb_destroy(h);
      return rs;
    }
  } else {
    e = shared_graph(modes, q.n_max, q.ordering, h->device, h->stream, &h->graph_ref);
    if (e) return bail(e, "build_graph");
    h->gt = h->graph_ref->gt;
    h->n_tiles = h->gt.n_tiles;
    h->own_tiles = h->n_tiles;
  }
  // small per-handle buffers come from the pool too: a handle of the same shape
  // then gets the same pointers, hence byte-identical kernel parameters, and can
  // reuse a cached instantiated CUDA graph (ensure_graph)
  e = pool_alloc(h->device, sizeof(Ctl), reinterpret_cast<void**>(&h->ctl));
  if (e) return bail(e, "cudaMalloc(ctl)");
  e = pinned_acquire(&h->ctl_host);
  if (e) return bail(e, "cudaMallocHost(ctl)");
  std::memset(h->ctl_host, 0, sizeof(Ctl));  // pooled: may hold a previous handle's block
  // records of kGraphsPerSync launches between two drains (+ the final sample)
  h->rec_cap = (int64_t)kGraphsPerSync * (h->loop_iters * h->chunk / q.record_stride + 2) + 4;
  e = pool_alloc(h->device, h->rec_cap * sizeof(long long), reinterpret_cast<void**>(&h->rec_step));
  if (!e)
    e = pool_alloc(h->device, h->rec_cap * q.d_full * sizeof(double),
                   reinterpret_cast<void**>(&h->rec_pops));
  if (!e && q.record_matrices)
    e = pool_alloc(h->device, h->rec_cap * q.d_full * q.d_full * 2 * sizeof(double),
                   reinterpret_cast<void**>(&h->rec_mats));
  if (e) return bail(e, "cudaMalloc(records)");

  KParams& p = h->base;
  p.d = d;
  p.n_sites = q.n_sites;
  p.kp1 = q.kp1;
  p.modes = modes;
  p.n_tot = h->n_tot;
  p.n_tiles = h->own_tiles;
  p.n_tiles_total = h->n_tiles;
  p.tile_begin = 0;
  p.root = T ? T->root != 0 : 1;
  for (int i = 0; i < d; ++i) {
    for (int j = 0; j < d; ++j) p.h[i * MAXD + j] = h->h[i * d + j];
    p.decay[i] = h->decay[i];
    p.site_of[i] = h->site_of[i];
    p.block_full[i] = h->block_full[i];
  }
  for (int k = 0; k < q.kp1; ++k) {
    p.nu[k] = h->nu[k];
    p.a[k] = h->a[k];
    p.b[k] = h->b[k];
  }
  // single precision: the RHS operands rounded once, like the reference's float32
  // h_block / decay / nvec arrays (heom.py:235-275 with rdtype = float32)
  p.single = q.precision == HB_PREC_SINGLE;
  for (int i = 0; i < MAXD * MAXD; ++i) p.hf[i] = (float)p.h[i];
  for (int i = 0; i < MAXD; ++i) p.decayf[i] = (float)p.decay[i];
  for (int k = 0; k < MAXKP1; ++k) {
    p.nuf[k] = (float)p.nu[k];
    p.af[k] = (float)p.a[k];
    p.bf[k] = (float)p.b[k];
  }
  p.plus = h->gt.plus_t;
  p.minus = h->gt.minus_t;
  p.nvec = h->gt.nvec_t;
  p.damp_plane = nullptr;
  p.tile_list = nullptr;
  // tier-major order: the top tier (no raise links) is the last
  // C(N_max + M - 1, N_max) positions; tiles wholly inside it skip the raise table
  p.top_tile = h->n_tiles;
  if (T) {
    p.top_tile = T->top_tile;
  } else if (q.ordering == HB_ORDER_REFERENCE) {
    const int64_t top_count = hierarchy_size(modes - 1, q.n_max);  // |n| = N_max exactly
    const int64_t first_top = n_tot - top_count;
    p.top_tile = (int)((first_top + TILE - 1) / TILE);
  }
  // small hierarchies: k_mm4ab (phase A and phase B of a tile on separate warps,
  // hb_mm4.cu) while the tiles fill at most ~4 per SM; decided on the whole
  // hierarchy's size, so every shard of a run makes the same choice
  {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
    const int64_t all_tiles = (hierarchy_size(modes, q.n_max) + TILE - 1) / TILE;
    p.split = d > 7 || sms <= 0 ? 0 : all_tiles <= sms ? 2 : all_tiles <= 4 * sms ? 1 : 0;
  }
  // L2 persisting window over the stage input's tiers below N_max (tier-major
  // order: one contiguous prefix, 36 % of the ADOs at N_max = 8, K = 1): the
  // targets of the top tier's lower-link gathers stay in L2 while the state
  // streams past them (-7 % per step at config 4).  Shards: their owned tiles
  // below the top tier.  Only where a state buffer exceeds half the L2.
  {
    int64_t first = 0, tiles = 0;
    if (T) {
      tiles = T->top_tile;
    } else if (q.ordering == HB_ORDER_REFERENCE && q.n_max >= 1) {
      tiles = (hierarchy_size(modes, q.n_max - 1) + TILE - 1) / TILE;
    }
    const size_t buf_bytes = (size_t)h->n_tiles * TILE * q.d * q.d *
                             (q.precision == HB_PREC_SINGLE ? 4 : 8);
    int l2 = 0, max_persist = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, h->device);
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, h->device);
    if (tiles > 0 && max_persist > 0 && buf_bytes > (size_t)l2 / 2) {
      const size_t want = (size_t)tiles * TILE * q.d * q.d * (q.precision == HB_PREC_SINGLE ? 4 : 8);
      const size_t lim = persisting_l2(h->device, want, (size_t)max_persist);
      if (lim > 0) {
        p.apw_first_tile = first;
        p.apw_tiles = tiles;
        p.apw_hit = (float)std::min(1.0, (double)lim / (double)want);
      }
    }
  }
  p.dt = q.dt;
  p.ctl = h->ctl;
  p.n_sinks = q.n_sinks;
  for (int s = 0; s < q.n_sinks; ++s) {
    p.sink_nterms[s] = h->sink_nterms[s];
    p.sink_full[s] = h->sink_full[s];
  }
  for (int t = 0; t < nterms; ++t) {
    p.sink_rate[t] = h->sink_rate[t];
    p.sink_pos[t] = h->sink_pos[t];
  }
  p.n_site_pos = q.n_site_pos;
  for (int k = 0; k < q.n_site_pos; ++k) p.site_pos[k] = h->site_pos[k];
  p.d_full = q.d_full;
  for (int f = 0; f < MAXFULL; ++f) p.full2blk[f] = p.full2sink[f] = -1;
  for (int i = 0; i < d; ++i) p.full2blk[h->block_full[i]] = i;
  for (int s = 0; s < q.n_sinks; ++s) p.full2sink[h->sink_full[s]] = s;
  p.has_t_end = q.has_t_end;
  p.has_residual = q.has_residual;
  p.record_matrices = q.record_matrices;
  p.t_end = q.t_end;
  p.residual = q.residual;
  p.hard_cap = q.hard_cap;
  p.blow2 = q.blowup_norm * q.blowup_norm;
  p.stride = q.record_stride;
  p.rec_cap = h->rec_cap;
  p.rec_step = h->rec_step;
  p.rec_pops = h->rec_pops;
  p.rec_mats = h->rec_mats;
  *out = h;
  return HB_OK;
}

int hb_create(const hb_params* P, hb_handle** out) { return create_impl(P, nullptr, out); }

int hb_create_shard(const hb_params* P, const hb_shard_tables* T, hb_handle** out) {
  if (!T) return fail(HB_ERR_ARG, "null shard tables");
  return create_impl(P, T, out);
}

KParams hb::stage_params(hb_handle* h, int stage) {
  KParams p;
  std::memcpy(&p, &h->base, sizeof p);  // byte-exact (padding too): GraphCache keys
  double* S = h->buf[0];
  double* Y2 = h->buf[1];
  double* Y3 = h->buf[2];
  double* Y4 = h->buf[3];
  p.sig = S;
  p.Y2 = Y2;
  p.Y3 = Y3;
  p.Bbuf = h->buf[4];
  const double dt = h->prm.dt;
  switch (stage) {
    case 1: p.Yin = S;  p.Yout = Y2; p.coef = 0.5 * dt; break;
    case 2: p.Yin = Y2; p.Yout = Y3; p.coef = 0.5 * dt; break;
    case 3: p.Yin = Y3; p.Yout = Y4; p.coef = dt; break;
    default: p.Yin = Y4; p.Yout = S; p.coef = dt; break;
  }
  return p;
}

// bytes per state element: float for HB_PREC_SINGLE, double otherwise
size_t hb::elem_size(const hb_handle* h) { return h->base.single ? sizeof(float) : sizeof(double); }

static int alloc_state(hb_handle* h, int layout) {
  if (h->layout == layout && h->buf[0]) return HB_OK;
  free_state(h);
  h->layout = layout;
  const int d = h->prm.d;
  h->n_planes = layout == HB_LAYOUT_HERMITIAN ? d * d : 2 * d * d;
  // one extra all-zero tile per buffer: target of absent links (never written)
  if (h->base.single) {
    bool identity = h->prm.n_sites == d;
    for (int i = 0; i < d; ++i) identity = identity && h->site_of[i] == i;
    if (layout != HB_LAYOUT_HERMITIAN || !identity || !mm4_supported(d, h->prm.kp1) ||
        h->prm.kernel_variant != HB_KERNEL_AUTO)
      return fail(HB_ERR_ARG,
                  "precision='single' needs a Hermitian rho0, every block level a site, "
                  "d <= 8, n_matsubara <= 1 and kernel='auto'");
  }
  const size_t bytes = (size_t)(h->n_tiles + 1) * TILE * h->n_planes * elem_size(h);
  h->buf_bytes = bytes;
  for (auto& b : h->buf) {
    void* p = nullptr;
    CK(pool_alloc(h->device, bytes, &p));
    b = static_cast<double*>(p);
    CK(cudaMemsetAsync(b, 0, bytes, h->stream));
  }
  h->base.hermitian = layout == HB_LAYOUT_HERMITIAN;
  h->base.n_planes = h->n_planes;
  bool identity = h->prm.n_sites == d;
  for (int i = 0; i < d; ++i) identity = identity && h->site_of[i] == i;
  // the unrolled kernels address a buffer with int32 element offsets
  const bool fits32 = (h->n_tiles + 1) * (int64_t)TILE * h->n_planes < INT32_MAX;
  h->base.fast = h->base.hermitian && identity && mm4_supported(d, h->prm.kp1) &&
                 h->prm.kernel_variant == HB_KERNEL_AUTO && fits32;
  CK(configure_stages(h->base));
  return HB_OK;
}

int hb::drain(hb_handle* h) {
  // ctl_host is current (caller synchronised)
  const long long n = h->ctl_host->n_rec;
  if (n <= 0) return HB_OK;
  const int df = h->prm.d_full;
  const size_t s0 = h->steps.size();
  h->steps.resize(s0 + n);
  h->pops.resize((s0 + n) * df);
  std::vector<long long> st(n);
  CK(hb_memcpy(st.data(), h->rec_step, n * sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
  CK(hb_memcpy(h->pops.data() + s0 * df, h->rec_pops, n * df * sizeof(double),
                     cudaMemcpyDeviceToHost, h->stream));
  if (h->prm.record_matrices) {
    h->mats.resize((s0 + n) * df * df * 2);
    CK(hb_memcpy(h->mats.data() + s0 * df * df * 2, h->rec_mats,
                       n * df * df * 2 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  }
  const long long zero = 0;
  CK(hb_memcpy(&h->ctl->n_rec, &zero, sizeof zero, cudaMemcpyHostToDevice, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  for (long long i = 0; i < n; ++i) h->steps[s0 + i] = st[i];
  h->ctl_host->n_rec = 0;
  return HB_OK;
}

int hb::sync_ctl(hb_handle* h) {
  CK(hb_memcpy(h->ctl_host, h->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return HB_OK;
}

// (re)starts the run on the state in buffer 0: control block, t = 0 sample and
// stop policy before the first step (heom.py:355-368)
static int start_run(hb_handle* h, const double* sink_pops) {
  h->launches_base += h->ctl_host->launches;  // the device count restarts with the block
  h->host_step = 0;
  for (bool& b : h->packed_once) b = false;
  Ctl c{};
  c.status = ST_RUNNING;
  for (int s = 0; s < h->prm.n_sinks; ++s) c.sink_pops[s] = sink_pops[s];
  std::memcpy(h->ctl_host, &c, sizeof c);
  CK(hb_memcpy(h->ctl, h->ctl_host, sizeof(Ctl), cudaMemcpyHostToDevice, h->stream));
  h->steps.clear();
  h->pops.clear();
  h->mats.clear();
  KParams p = stage_params(h, 4);
  CK(launch_init(p, h->stream));
  h->launches += 1;
  int rc = sync_ctl(h);
  if (rc) return rc;
  rc = drain(h);
  if (rc) return rc;
  h->ready = true;
  return HB_OK;
}

int hb_set_rho0(hb_handle* h, const double* rho0, const double* sink_pops) {
  if (!h) return fail(HB_ERR_ARG, "null handle");
  CK(cudaSetDevice(h->device));
  if (h->comm) CK(cudaStreamSynchronize(h->comm));  // no exchange in flight on the buffers
  const int d = h->prm.d;
  int layout = h->prm.layout;
  if (layout == HB_LAYOUT_AUTO) {
    bool herm = true;
    for (int i = 0; i < d && herm; ++i)
      for (int j = 0; j < d; ++j) {
        const double re = rho0[2 * (i * d + j)], im = rho0[2 * (i * d + j) + 1];
        const double rt = rho0[2 * (j * d + i)], it = rho0[2 * (j * d + i) + 1];
        if (re != rt || im != -it) {
          herm = false;
          break;
        }
      }
    layout = herm ? HB_LAYOUT_HERMITIAN : HB_LAYOUT_GENERAL;
  }
  int rc = alloc_state(h, layout);
  if (rc) return rc;
  // sigma: auxiliaries zero, sigma^0 = rho0 block in tile 0, lane 0
  const size_t bytes = (size_t)h->n_tiles * TILE * h->n_planes * elem_size(h);
  CK(cudaMemsetAsync(h->buf[0], 0, bytes, h->stream));
  std::vector<double> tile0((size_t)h->n_planes * TILE, 0.0);
  if (layout == HB_LAYOUT_HERMITIAN) {
    int e = d;
    for (int i = 0; i < d; ++i) tile0[(size_t)i * TILE] = rho0[2 * (i * d + i)];
    for (int i = 0; i < d; ++i)
      for (int j = i + 1; j < d; ++j, ++e) {
        const int pr = d + 2 * (e - d);
        tile0[herm_off(d, pr, 0)] = rho0[2 * (i * d + j)];
        tile0[herm_off(d, pr + 1, 0)] = rho0[2 * (i * d + j) + 1];
      }
  } else {
    for (int k = 0; k < d * d; ++k) {
      tile0[(size_t)(2 * k) * TILE] = rho0[2 * k];
      tile0[(size_t)(2 * k + 1) * TILE] = rho0[2 * k + 1];
    }
  }
  if (!h->base.root) {  // a shard without ADO 0: auxiliaries only, all zero
  } else if (h->base.single) {  // pageable source: the copy is staged before the call returns
    std::vector<float> tile0f(tile0.begin(), tile0.end());
    CK(hb_memcpy(h->buf[0], tile0f.data(), tile0f.size() * sizeof(float),
                 cudaMemcpyHostToDevice, h->stream));
  } else {
    CK(hb_memcpy(h->buf[0], tile0.data(), tile0.size() * sizeof(double),
                 cudaMemcpyHostToDevice, h->stream));
  }
  if (h->shard) h->halo_primed = false;
  return start_run(h, sink_pops);
}

int hb_set_state(hb_handle* h, const double* sig, const double* sink_pops) {
  if (!h) return fail(HB_ERR_ARG, "null handle");
  if (h->shard) return fail(HB_ERR_ARG, "hb_set_state needs an unsharded handle");
  CK(cudaSetDevice(h->device));
  const int d = h->prm.d;
  int layout = h->prm.layout;
  if (layout == HB_LAYOUT_AUTO) {  // Hermitian-packed only if every ADO is exactly Hermitian
    bool herm = true;
    for (int64_t k = 0; k < h->n_tot && herm; ++k) {
      const double* m = sig + (size_t)k * d * d * 2;
      for (int i = 0; i < d && herm; ++i)
        for (int j = i; j < d; ++j)
          if (m[2 * (i * d + j)] != m[2 * (j * d + i)] ||
              m[2 * (i * d + j) + 1] != -m[2 * (j * d + i) + 1]) {
            herm = false;
            break;
          }
    }
    layout = herm ? HB_LAYOUT_HERMITIAN : HB_LAYOUT_GENERAL;
  }
  int rc = alloc_state(h, layout);
  if (rc) return rc;
  const size_t ref_bytes = (size_t)h->n_tot * d * d * 2 * sizeof(double);
  DevBuf tmp;
  CK(tmp.alloc(ref_bytes));
  CK(hb_memcpy(tmp.p, sig, ref_bytes, cudaMemcpyHostToDevice, h->stream));
  CK(launch_pack(h->base, tmp.as<double>(), h->gt.dev2ref, h->buf[0], h->stream));
  h->launches += 1;
  return start_run(h, sink_pops);  // synchronises before tmp is freed
}

// One graph launch = a CUDA-graph WHILE node whose body is `chunk` RK4 steps
// (5 PDL-chained kernels each); the step-finish kernel of the body's last step
// re-arms the loop while the run is RUNNING and fewer than loop_iters bodies of
// this launch have run (hb_mm4.cu k_step_finish).  A run therefore stops within
// the body of its stop step: at most chunk - 1 no-op steps, each a CTA launch
// per stage that exits on the status (k_mm4), instead of whole graphs of them.
// Kernels that cannot re-arm the loop (the generic k_stage) get a plain graph of
// `chunk` steps per launch.
static cudaError_t capture_steps(hb_handle* h, int n_steps, bool set_cond,
                                 cudaGraphConditionalHandle cond) {
  cudaError_t err = cudaSuccess;
  // k_mm4ab graphs fold each step's bookkeeping into the next step's stage 1
  // (an extra CTA; one launch less per step), except the last step of the
  // graph, whose k_step_finish closes the body; the sink rates alternate by
  // step parity.  (us per step: K = 0 twin 17.5 -> 15.4; K = 1, N_max = 4
  // 24.0 -> 21.4; N_max = 5 34.4 -> 32.0.)
  const bool fold = h->base.fast && h->base.split;
  for (int c = 0; c < n_steps && !err; ++c)
    for (int s = 1; s <= 4 && !err; ++s) {
      KParams p = stage_params(h, s);
      if (fold) {
        p.rpar = c & 1;
        p.fold = (s == 1 && c > 0) || (s == 4 && c < n_steps - 1);
      }
      if (set_cond && s == 4 && c == n_steps - 1) {
        p.set_cond = 1;
        p.cond = (unsigned long long)cond;
        p.loop_iters = h->loop_iters;
      }
      err = launch_stage(s, p, h->stream);
    }
  return err;
}

static int build_while_graph(hb_handle* h, cudaGraphExec_t* exec, int64_t* nodes) {
  cudaGraph_t g = nullptr;
  CK(cudaGraphCreate(&g, 0));
  struct GD { cudaGraph_t g; ~GD() { if (g) cudaGraphDestroy(g); } } gd{g};
  cudaGraphConditionalHandle cond;
  CK(cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = cond;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, nullptr, 0, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(h->stream, body, nullptr, nullptr, 0,
                                   cudaStreamCaptureModeThreadLocal));
  cudaError_t err = capture_steps(h, h->chunk, true, cond);
  cudaGraph_t out = nullptr;
  cudaError_t e2 = cudaStreamEndCapture(h->stream, &out);
  if (err) return cuda_fail(err, "capture stage kernels");
  if (e2) return cuda_fail(e2, "cudaStreamEndCapture");
  *nodes = (int64_t)5 * h->chunk;
  CK(cudaGraphInstantiate(exec, g, 0));
  return HB_OK;
}

static int build_plain_graph(hb_handle* h, cudaGraphExec_t* exec, int64_t* nodes) {
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  cudaError_t err = capture_steps(h, h->chunk, false, 0);
  cudaError_t e2 = cudaStreamEndCapture(h->stream, &g);
  if (err) return cuda_fail(err, "capture stage kernels");
  if (e2) return cuda_fail(e2, "cudaStreamEndCapture");
  size_t n = 0;
  err = cudaGraphGetNodes(g, nullptr, &n);
  if (!err) err = cudaGraphInstantiate(exec, g, 0);
  cudaGraphDestroy(g);
  if (err) return cuda_fail(err, "cudaGraphInstantiate");
  *nodes = (int64_t)n;
  return HB_OK;
}

static int ensure_graph(hb_handle* h) {
  if (h->graph && h->graph_layout == h->layout) return HB_OK;
  graph_cache_put(h);
  h->graph_while = h->base.fast != 0;
  std::string key(reinterpret_cast<const char*>(&h->device), sizeof(int));
  key.append(reinterpret_cast<const char*>(&h->chunk), sizeof(int));
  key.append(reinterpret_cast<const char*>(&h->loop_iters), sizeof(h->loop_iters));
  key.append(1, h->graph_while ? 'w' : 'p');
  for (int s = 1; s <= 4; ++s) {
    const KParams p = stage_params(h, s);
    key.append(reinterpret_cast<const char*>(&p), sizeof(KParams));
  }
  h->graph_key = key;
  h->graph = graph_cache_take(key, &h->graph_nodes);
  if (h->graph) {
    h->graph_layout = h->layout;
    return HB_OK;
  }
  int rc = h->graph_while ? build_while_graph(h, &h->graph, &h->graph_nodes)
                          : build_plain_graph(h, &h->graph, &h->graph_nodes);
  if (rc) {
    h->graph = nullptr;
    return rc;
  }
  h->graph_layout = h->layout;
  return HB_OK;
}

// smallest step s with s * dt >= t_end - 1e-9 (the t_end test of heom.py:359-361)
static long long t_end_step(double t_end, double dt) {
  long long s = (long long)std::floor((t_end - 1e-9) / dt) - 2;
  if (s < 0) s = 0;
  while ((double)s * dt < t_end - 1e-9) ++s;
  return s;
}

// steps one graph launch covers at most (the record buffer holds a sync's worth)
static int64_t launch_steps(const hb_handle* h) {
  return h->graph_while ? h->loop_iters * h->chunk : h->chunk;
}

int hb_run(hb_handle* h, hb_result* res) {
  if (!h || !h->ready) return fail(HB_ERR_ARG, "hb_set_rho0 must be called first");
  if (h->shard) return fail(HB_ERR_ARG, "shard handles step with hb_shard_steps");
  CK(cudaSetDevice(h->device));
  int rc = ensure_graph(h);
  if (rc) return rc;
  const long long stop = h->prm.has_t_end ? t_end_step(h->prm.t_end, h->prm.dt) : -1;
  while (h->ctl_host->status == ST_RUNNING) {
    // kGraphsPerSync launches back to back: the device never idles while the host
    // drains records and relaunches; a launch past the stop is a no-op body.  A
    // t_end run that one launch finishes gets exactly one.
    int n = kGraphsPerSync;
    if (stop >= 0 && stop - h->ctl_host->step <= launch_steps(h)) n = 1;
    for (int g = 0; g < n; ++g) CK(cudaGraphLaunch(h->graph, h->stream));
    rc = sync_ctl(h);
    if (rc) return rc;
    rc = drain(h);
    if (rc) return rc;
  }
  const Ctl& c = *h->ctl_host;
  if (res) {
    res->stop_reason = c.status == ST_T_END ? HB_STOP_T_END
                       : c.status == ST_RESIDUAL ? HB_STOP_RESIDUAL : HB_STOP_NONE;
    res->layout = h->layout;
    res->steps = c.step;
    res->n_records = (int64_t)h->steps.size();
    res->n_tot = h->n_tot;
  }
  if (c.status == ST_DIVERGED) return fail(HB_DIVERGED, "matrix norm exceeded the blow-up bound");
  if (c.status == ST_HARDCAP) return fail(HB_HARDCAP, "residual policy not reached within the cap");
  return HB_OK;
}

int hb_get_records(hb_handle* h, int64_t* steps, double* pops, double* mats_or_null, int64_t cap) {
  if (!h) return fail(HB_ERR_ARG, "null handle");
  const int64_t n = (int64_t)h->steps.size();
  if (cap < n) return fail(HB_ERR_ARG, "record buffer too small");
  const int df = h->prm.d_full;
  if (steps) std::memcpy(steps, h->steps.data(), n * sizeof(int64_t));
  if (pops) std::memcpy(pops, h->pops.data(), n * df * sizeof(double));
  if (mats_or_null) {
    if (!h->prm.record_matrices) return fail(HB_ERR_ARG, "matrices were not recorded");
    std::memcpy(mats_or_null, h->mats.data(), n * df * df * 2 * sizeof(double));
  }
  return HB_OK;
}

int64_t hb_record_count(hb_handle* h) { return h ? (int64_t)h->steps.size() : 0; }

int hb_get_state(hb_handle* h, double* sig, double* sink_pops) {
  if (!h || !h->ready) return fail(HB_ERR_ARG, "no state");
  CK(cudaSetDevice(h->device));
  const int d = h->prm.d;
  const size_t ref_bytes = (size_t)h->n_tot * d * d * 2 * sizeof(double);
  if (sig) {
    DevBuf tmp;
    CK(tmp.alloc(ref_bytes));
    KParams p = h->base;
    CK(launch_unpack(p, h->buf[0], h->gt.dev2ref, tmp.as<double>(), h->stream));
    CK(hb_memcpy(sig, tmp.p, ref_bytes, cudaMemcpyDeviceToHost, h->stream));
  }
  int rc = sync_ctl(h);
  if (rc) return rc;
  if (sink_pops)
    for (int s = 0; s < h->prm.n_sinks; ++s) sink_pops[s] = h->ctl_host->sink_pops[s];
  return HB_OK;
}

int hb_get_sigma0(hb_handle* h, double* sig0, double* sink_pops) {
  if (!h || !h->ready) return fail(HB_ERR_ARG, "no state");
  CK(cudaSetDevice(h->device));
  const int d = h->prm.d;
  std::vector<double> tile0((size_t)h->n_planes * TILE);
  std::vector<float> tile0f(h->base.single ? tile0.size() : 0);
  if (h->base.single)
    CK(hb_memcpy(tile0f.data(), h->buf[0], tile0f.size() * sizeof(float),
                       cudaMemcpyDeviceToHost, h->stream));
  else
    CK(hb_memcpy(tile0.data(), h->buf[0], tile0.size() * sizeof(double),
                       cudaMemcpyDeviceToHost, h->stream));
  int rc = sync_ctl(h);
  if (rc) return rc;
  if (h->base.single) tile0.assign(tile0f.begin(), tile0f.end());
  const bool herm = h->layout == HB_LAYOUT_HERMITIAN;
  auto at = [&](int plane) { return tile0[plane_off(herm, d, plane, 0)]; };  // lane 0 = ADO 0
  if (h->layout == HB_LAYOUT_HERMITIAN) {
    for (int i = 0; i < d; ++i) {
      sig0[2 * (i * d + i)] = at(i);
      sig0[2 * (i * d + i) + 1] = 0.0;
    }
    int e = d;
    for (int i = 0; i < d; ++i)
      for (int j = i + 1; j < d; ++j, ++e) {
        const int pr = d + 2 * (e - d);
        sig0[2 * (i * d + j)] = at(pr);
        sig0[2 * (i * d + j) + 1] = at(pr + 1);
        sig0[2 * (j * d + i)] = at(pr);
        sig0[2 * (j * d + i) + 1] = -at(pr + 1);
      }
  } else {
    for (int k = 0; k < 2 * d * d; ++k) sig0[k] = at(k);
  }
  if (sink_pops)
    for (int s = 0; s < h->prm.n_sinks; ++s) sink_pops[s] = h->ctl_host->sink_pops[s];
  return HB_OK;
}

int hb_time_steps(hb_handle* h, int64_t n_steps, double* ms, double* stage_ms) {
  if (!h || !h->ready) return fail(HB_ERR_ARG, "hb_set_rho0 must be called first");
  if (h->shard) return fail(HB_ERR_ARG, "shard handles step with hb_shard_steps");
  if (h->ctl_host->status != ST_RUNNING) return fail(HB_ERR_ARG, "run already stopped");
  if (n_steps < 0) return fail(HB_ERR_ARG, "negative step count");
  // the records of the timed steps stay on the device until the next sync
  if (n_steps / h->prm.record_stride + 1 >= h->rec_cap)
    return fail(HB_ERR_ARG, "record_stride too small for the timed step count (records would be dropped)");
  CK(cudaSetDevice(h->device));
  int rc = ensure_graph(h);
  if (rc) return rc;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  struct EG { cudaEvent_t a, b; ~EG() { cudaEventDestroy(a); cudaEventDestroy(b); } } eg{e0, e1};
  CK(cudaEventRecord(e0, h->stream));
  int64_t left = n_steps;
  const int64_t per_launch = launch_steps(h);
  while (left >= per_launch) {
    CK(cudaGraphLaunch(h->graph, h->stream));
    left -= per_launch;
  }
  for (; left > 0; --left)
    for (int s = 1; s <= 4; ++s) CK(launch_stage(s, stage_params(h, s), h->stream));
  CK(cudaEventRecord(e1, h->stream));
  CK(cudaEventSynchronize(e1));
  float f = 0.f;
  CK(cudaEventElapsedTime(&f, e0, e1));
  *ms = f;
  if (stage_ms) {
    // per-stage kernel durations: events around individual launches (these
    // break the PDL overlap between stages, so they sum to more than a step)
    const int reps = 8;
    std::vector<cudaEvent_t> ev(reps * 5);
    for (auto& x : ev) CK(cudaEventCreate(&x));
    for (int r = 0; r < reps; ++r) {
      CK(cudaEventRecord(ev[r * 5], h->stream));
      for (int s = 1; s <= 4; ++s) {
        CK(launch_stage(s, stage_params(h, s), h->stream));
        CK(cudaEventRecord(ev[r * 5 + s], h->stream));
      }
    }
    CK(cudaEventSynchronize(ev.back()));
    for (int s = 0; s < 4; ++s) stage_ms[s] = 0.0;
    for (int r = 0; r < reps; ++r)
      for (int s = 1; s <= 4; ++s) {
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, ev[r * 5 + s - 1], ev[r * 5 + s]));
        stage_ms[s - 1] += t / reps;
      }
    for (auto& x : ev) cudaEventDestroy(x);
  }
  rc = sync_ctl(h);
  if (rc) return rc;
  rc = drain(h);
  if (rc) return rc;
  if (h->ctl_host->status != ST_RUNNING)
    return fail(HB_ERR_ARG, "stop policy fired during timing; use a t_end beyond the timed steps");
  return HB_OK;
}

// kernels that did work: host-launched ones plus the step kernels the device
// counted (current as of the handle's last synchronisation)
int64_t hb_launch_count(hb_handle* h) {
  return h ? h->launches + h->launches_base + (h->ctl_host ? h->ctl_host->launches : 0) : 0;
}

