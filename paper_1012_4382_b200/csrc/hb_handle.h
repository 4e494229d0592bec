// The run handle (hb_handle of include/heom_b200.h) and the host helpers shared
// by the translation units of the C ABI: hb_api.cu (create / run / state /
// Level-2 shims) and hb_shard.cu (sharded runs, halos, NCCL).
#pragma once
#include <cstdint>
#include <memory>
#include <string>
#include <vector>
#include "hb_internal.h"

namespace hb {

int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);
// every host<->device copy of the library goes through here (byte counters)
cudaError_t hb_memcpy(void* dst, const void* src, size_t n, cudaMemcpyKind kind, cudaStream_t s);

struct CachedGraph {
  GraphTables gt;
  ~CachedGraph() { free_graph(&gt); }
};

}  // namespace hb

#define CK(x)                                              \
  do {                                                     \
    cudaError_t e_ = (x);                                  \
    if (e_ != cudaSuccess) return hb::cuda_fail(e_, #x);   \
  } while (0)

struct hb_handle {
  hb_params prm{};
  std::vector<double> h, decay, nu, a, b, sink_rate;
  std::vector<int32_t> site_of, sink_nterms, sink_pos, site_pos, block_full, sink_full;
  int device = 0;
  int modes = 0, n_tot = 0, n_tiles = 0;  // n_tot / n_tiles: every ADO slot of the buffers
  int chunk = 64;
  cudaStream_t stream = nullptr;
  std::shared_ptr<hb::CachedGraph> graph_ref;  // shared device tables (unsharded)
  hb::GraphTables gt;                          // the tables in use (non-owning)
  hb::GraphTables own_gt;                      // shard handles: their local tables (owned)
  int layout = 0;  // HB_LAYOUT_HERMITIAN / GENERAL once allocated
  int n_planes = 0;
  double* buf[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // sigma, Y2, Y3, Y4, B
  size_t buf_bytes = 0;
  hb::Ctl* ctl = nullptr;
  hb::Ctl* ctl_host = nullptr;  // pinned
  long long* rec_step = nullptr;
  double* rec_pops = nullptr;
  double* rec_mats = nullptr;
  long long rec_cap = 0;
  hb::KParams base{};
  cudaGraphExec_t graph = nullptr;
  int graph_layout = -1;
  std::string graph_key;     // GraphCache key of `graph`
  int64_t graph_nodes = 0;   // kernel launches in one body (WHILE) / replay (plain) of `graph`
  bool graph_while = false;  // `graph` is a WHILE node over a body of `chunk` steps
  long long loop_iters = 1;  // WHILE-body iterations per graph launch
  std::vector<int64_t> steps;
  std::vector<double> pops, mats;
  int64_t launches = 0;       // host-counted kernels (init, pack/unpack, extra shard launches)
  int64_t launches_base = 0;  // device-counted step kernels of earlier runs of the handle
  bool ready = false;         // rho0 / state set

  // ---- sharded runs (hb_shard.cu) ----
  bool shard = false;         // created by hb_create_shard: local ADO numbering
  int own_tiles = 0;          // tiles [0, own_tiles) are computed here; the rest is halo
  int32_t* groups = nullptr;  // device tile lists of the four launch groups
  int group_off[5] = {0, 0, 0, 0, 0};
  int group_first[4] = {-1, -1, -1, -1};  // first tile of a contiguous group, else -1
  void* nccl_comm = nullptr;
  cudaStream_t comm = nullptr;  // halo exchange + guard all-reduce stream
  // events: ev_send[s-1] stage s's send tiles done (compute); ev_halo[b] halo of
  // buffer b unpacked (comm); ev_packed[b] the sends of buffer b packed (comm);
  // ev_s4 / ev_guard: stage 4 done (compute) / guard all-reduce done (comm)
  cudaEvent_t ev_send[4] = {}, ev_halo[4] = {}, ev_packed[4] = {}, ev_s4 = nullptr,
              ev_guard = nullptr;
  bool halo_primed = false;  // buffer 0's halo exchanged since the state was set
  int64_t host_step = 0;     // steps enqueued since the state was set (guard steps)
  bool packed_once[4] = {false, false, false, false};
  // compressed halo plan (hb_halo_set): segments of (local position, site) entries
  struct Halo {
    int nc = 0;                                    // planes per cross (2d - 1)
    std::vector<int> peer, is_send, count, off;    // per segment; off in entries
    int32_t* pos = nullptr;                        // device, all segments
    int32_t* site = nullptr;
    int16_t* planes = nullptr;                     // device, [site][nc] plane index
    void* packed = nullptr;                        // device staging, [entry][nc]
  } halo;
};

namespace hb {

KParams stage_params(hb_handle* h, int stage);
size_t elem_size(const hb_handle* h);
int sync_ctl(hb_handle* h);
int drain(hb_handle* h);
cudaError_t pool_alloc(int device, size_t bytes, void** out);
void pool_release(int device, size_t bytes, void* p);
// hb_shard.cu
int init_shard(hb_handle* h, const hb_shard_tables* T);
void free_shard(hb_handle* h);
void nccl_destroy(void* comm);

}  // namespace hb
