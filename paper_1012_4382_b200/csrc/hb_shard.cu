// Sharded propagation of ONE hierarchy (new -- the reference
// declares distribution a non-goal).
//
// A shard (hb_create_shard) numbers its ADO slots locally: its owned ADOs first
// -- those below the top tier, then the top-tier ones in whole tiles, so the
// paired gather rounds of k_mm4 survive -- then halo slots for the neighbours
// owned by other shards.  Buffers hold only owned + halo slots.  The host side
// (shard.py) builds the local tables, the halo plan and four launch groups that
// partition the owned tiles:
//   0 send-only  -- tiles holding crosses other shards read, no halo reads
//   1 interior   -- neither
//   2 send+halo  -- both
//   3 halo-only  -- tiles that read halo slots, nothing sent
// A stage runs 0 and 1 at once, waits for the halo of its input (exchanged on
// the second stream during the previous stage), runs 2, hands its output
// crosses to the exchange stream (pack, grouped ncclSend/ncclRecv, unpack into
// the consumers' halo slots) and runs 3 while they travel.  Every 25th step the
// whole-state divergence max (heom.py:386-389) is all-reduced so that every
// shard stops at the same step.  The root shard (local slot 0 = ADO 0) does the
// sinks, records and stop policy; the others advance the step and stop at t_end.
#include <dlfcn.h>
#include <cstring>
#include <string>
#include <vector>
#include "hb_handle.h"

using namespace hb;

namespace {

// ---- NCCL, resolved at run time so the library loads without it ----
struct NcclUniqueId { char internal[128]; };
struct NcclApi {
  typedef int (*GetUniqueId)(void*);
  typedef int (*CommInitRank)(void**, int, NcclUniqueId, int);
  typedef int (*SendRecv)(const void*, size_t, int, int, void*, cudaStream_t);
  typedef int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t);
  typedef int (*Group)();
  typedef int (*CommDestroy)(void*);
  typedef const char* (*ErrStr)(int);
  GetUniqueId get_id = nullptr;
  CommInitRank init_rank = nullptr;
  SendRecv send = nullptr;
  SendRecv recv = nullptr;
  AllReduce allreduce = nullptr;
  Group group_start = nullptr, group_end = nullptr;
  CommDestroy destroy = nullptr;
  ErrStr err = nullptr;
  bool ok = false;
};
constexpr int kNcclInt8 = 0, kNcclUint64 = 5, kNcclMax = 2;  // nccl.h enums

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return a;
    a.get_id = (NcclApi::GetUniqueId)dlsym(lib, "ncclGetUniqueId");
    a.init_rank = (NcclApi::CommInitRank)dlsym(lib, "ncclCommInitRank");
    a.send = (NcclApi::SendRecv)dlsym(lib, "ncclSend");
    a.recv = (NcclApi::SendRecv)dlsym(lib, "ncclRecv");
    a.allreduce = (NcclApi::AllReduce)dlsym(lib, "ncclAllReduce");
    a.group_start = (NcclApi::Group)dlsym(lib, "ncclGroupStart");
    a.group_end = (NcclApi::Group)dlsym(lib, "ncclGroupEnd");
    a.destroy = (NcclApi::CommDestroy)dlsym(lib, "ncclCommDestroy");
    a.err = (NcclApi::ErrStr)dlsym(lib, "ncclGetErrorString");
    a.ok = a.get_id && a.init_rank && a.send && a.recv && a.allreduce && a.group_start &&
           a.group_end;
    return a;
  }();
  return api;
}

int nccl_fail(int r, const char* where) {
  const char* m = nccl().err ? nccl().err(r) : "nccl error";
  return fail(HB_ERR_CUDA, std::string(where) + ": " + m);
}

void free_halo(hb_handle* h) {
  cudaFree(h->halo.pos);
  cudaFree(h->halo.site);
  cudaFree(h->halo.planes);
  cudaFree(h->halo.packed);
  h->halo = hb_handle::Halo{};
}

void* seg_packed(hb_handle* h, int i) {
  return static_cast<char*>(h->halo.packed) + (size_t)h->halo.off[i] * h->halo.nc * elem_size(h);
}

cudaError_t pack_seg(hb_handle* h, int i, int b, cudaStream_t s) {
  auto& H = h->halo;
  return launch_halo(0, h->base.single != 0, nullptr, h->buf[b], H.count[i], H.pos + H.off[i],
                     H.site + H.off[i], H.planes, H.nc, h->n_planes, seg_packed(h, i), s);
}

// unpack consumer segment i of h from `packed` (the owner's staging or h's own)
cudaError_t unpack_seg(hb_handle* h, int i, int b, void* packed, cudaStream_t s) {
  auto& H = h->halo;
  return launch_halo(1, h->base.single != 0, h->buf[b], nullptr, H.count[i], H.pos + H.off[i],
                     H.site + H.off[i], H.planes, H.nc, h->n_planes, packed, s);
}

// one launch group of a stage (no step bookkeeping); empty groups launch nothing
cudaError_t launch_group(hb_handle* h, int stage, int g, cudaStream_t s, int* n_launched) {
  const int n = h->group_off[g + 1] - h->group_off[g];
  if (n == 0) return cudaSuccess;
  KParams p = stage_params(h, stage);
  if (h->group_first[g] >= 0) {  // a contiguous run of tiles: a plain range launch
    p.tile_begin = h->group_first[g];
  } else {
    p.tile_list = h->groups + h->group_off[g];
  }
  p.n_tiles = n;
  ++*n_launched;
  return launch_mm4_only(stage, p, s);
}

// pack the sends of buffer b, grouped NCCL send/recv, unpack the receives; all
// on the exchange stream (ev_packed[b] after the packs, ev_halo[b] at the end)
int exchange_nccl(hb_handle* h, int b) {
  auto& H = h->halo;
  for (size_t i = 0; i < H.count.size(); ++i)
    if (H.is_send[i] && H.count[i] > 0) {
      CK(pack_seg(h, (int)i, b, h->comm));
      h->launches += 1;
    }
  CK(cudaEventRecord(h->ev_packed[b], h->comm));
  h->packed_once[b] = true;
  if (!H.count.empty()) {
    int r = nccl().group_start();
    if (r) return nccl_fail(r, "ncclGroupStart");
    for (size_t i = 0; i < H.count.size(); ++i) {
      if (H.count[i] == 0) continue;  // both sides list the same (empty) entries
      const size_t bytes = (size_t)H.count[i] * H.nc * elem_size(h);
      void* p = seg_packed(h, (int)i);
      r = H.is_send[i] ? nccl().send(p, bytes, kNcclInt8, H.peer[i], h->nccl_comm, h->comm)
                       : nccl().recv(p, bytes, kNcclInt8, H.peer[i], h->nccl_comm, h->comm);
      if (r) {
        nccl().group_end();
        return nccl_fail(r, H.is_send[i] ? "ncclSend" : "ncclRecv");
      }
    }
    r = nccl().group_end();
    if (r) return nccl_fail(r, "ncclGroupEnd");
  }
  for (size_t i = 0; i < H.count.size(); ++i)
    if (!H.is_send[i] && H.count[i] > 0) {
      CK(unpack_seg(h, (int)i, b, seg_packed(h, (int)i), h->comm));
      h->launches += 1;
    }
  CK(cudaEventRecord(h->ev_halo[b], h->comm));
  return HB_OK;
}

int check_shard(hb_handle* h) {
  if (!h || !h->ready) return fail(HB_ERR_ARG, "hb_set_rho0 must be called first");
  if (!h->shard) return fail(HB_ERR_ARG, "not a shard handle (hb_create_shard)");
  if (!h->base.fast || h->layout != HB_LAYOUT_HERMITIAN)
    return fail(HB_ERR_ARG, "sharded runs need the Hermitian production layout");
  return HB_OK;
}

}  // namespace

namespace hb {

int init_shard(hb_handle* h, const hb_shard_tables* T) {
  int total = 0;
  for (int g = 0; g < 4; ++g) {
    h->group_off[g] = total;
    total += T->group_count[g];
  }
  h->group_off[4] = total;
  for (int g = 0; g < 4; ++g) {  // contiguous ascending groups launch as ranges
    const int32_t* t = T->groups + h->group_off[g];
    bool run = T->group_count[g] > 0;
    for (int i = 1; i < T->group_count[g] && run; ++i) run = t[i] == t[0] + i;
    h->group_first[g] = run ? t[0] : -1;
  }
  CK(cudaMalloc(&h->groups, (size_t)(total > 0 ? total : 1) * sizeof(int32_t)));
  CK(hb_memcpy(h->groups, T->groups, (size_t)total * sizeof(int32_t), cudaMemcpyHostToDevice,
               h->stream));
  CK(cudaStreamCreateWithFlags(&h->comm, cudaStreamNonBlocking));
  for (int i = 0; i < 4; ++i) {
    CK(cudaEventCreateWithFlags(&h->ev_send[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_halo[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_packed[i], cudaEventDisableTiming));
  }
  CK(cudaEventCreateWithFlags(&h->ev_s4, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&h->ev_guard, cudaEventDisableTiming));
  CK(cudaStreamSynchronize(h->stream));
  return HB_OK;
}

void nccl_destroy(void* comm) {
  if (nccl().destroy) nccl().destroy(comm);
}

void free_shard(hb_handle* h) {
  if (h->comm) cudaStreamSynchronize(h->comm);
  if (h->nccl_comm) nccl_destroy(h->nccl_comm);
  h->nccl_comm = nullptr;
  free_halo(h);
  cudaFree(h->groups);
  h->groups = nullptr;
  if (h->shard) free_graph(&h->own_gt);
  for (int i = 0; i < 4; ++i) {
    if (h->ev_send[i]) cudaEventDestroy(h->ev_send[i]);
    if (h->ev_halo[i]) cudaEventDestroy(h->ev_halo[i]);
    if (h->ev_packed[i]) cudaEventDestroy(h->ev_packed[i]);
    h->ev_send[i] = h->ev_halo[i] = h->ev_packed[i] = nullptr;
  }
  if (h->ev_s4) cudaEventDestroy(h->ev_s4);
  if (h->ev_guard) cudaEventDestroy(h->ev_guard);
  h->ev_s4 = h->ev_guard = nullptr;
  if (h->comm) cudaStreamDestroy(h->comm);
  h->comm = nullptr;
}

}  // namespace hb

// definitions take C linkage from the extern "C" declarations in heom_b200.h

int hb_sync(hb_handle* h, int* status, int64_t* step) {
  if (!h || !h->ready) return fail(HB_ERR_ARG, "hb_set_rho0 must be called first");
  CK(cudaSetDevice(h->device));
  if (h->comm) CK(cudaStreamSynchronize(h->comm));
  int rc = sync_ctl(h);
  if (rc) return rc;
  rc = drain(h);
  if (rc) return rc;
  if (status) *status = h->ctl_host->status;
  if (step) *step = h->ctl_host->step;
  return HB_OK;
}

int hb_nccl_unique_id(char* id128) {
  if (!nccl().ok) return fail(HB_ERR_CUDA, "libnccl.so.2 not found");
  const int r = nccl().get_id(id128);
  return r ? nccl_fail(r, "ncclGetUniqueId") : HB_OK;
}

int hb_nccl_init(hb_handle* h, const char* id128, int nranks, int rank) {
  if (!h) return fail(HB_ERR_ARG, "null handle");
  if (!nccl().ok) return fail(HB_ERR_CUDA, "libnccl.so.2 not found");
  CK(cudaSetDevice(h->device));
  NcclUniqueId id;
  std::memcpy(id.internal, id128, sizeof id.internal);
  void* comm = nullptr;
  const int r = nccl().init_rank(&comm, nranks, id, rank);
  if (r) return nccl_fail(r, "ncclCommInitRank");
  h->nccl_comm = comm;
  return HB_OK;
}

int hb_halo_set(hb_handle* h, int n_seg, const int32_t* peer, const int32_t* is_send,
                const int32_t* count, const int32_t* pos, const int32_t* site) {
  if (!h || !h->ready) return fail(HB_ERR_ARG, "hb_set_rho0 must be called first");
  if (!h->shard) return fail(HB_ERR_ARG, "halo plans belong to shard handles (hb_create_shard)");
  if (!h->base.fast || h->layout != HB_LAYOUT_HERMITIAN)
    return fail(HB_ERR_ARG, "compressed halos need the Hermitian production layout");
  if (n_seg < 0) return fail(HB_ERR_ARG, "negative segment count");
  CK(cudaSetDevice(h->device));
  CK(cudaStreamSynchronize(h->stream));
  CK(cudaStreamSynchronize(h->comm));
  free_halo(h);
  const int d = h->prm.d, nc = 2 * d - 1;
  auto& H = h->halo;
  H.nc = nc;
  int64_t total = 0;
  for (int i = 0; i < n_seg; ++i) {
    if (count[i] < 0) return fail(HB_ERR_ARG, "negative segment size");
    H.peer.push_back(peer[i]);
    H.is_send.push_back(is_send[i] != 0);
    H.count.push_back(count[i]);
    H.off.push_back((int)total);
    total += count[i];
  }
  if (total > INT32_MAX / nc) return fail(HB_ERR_ARG, "halo plan too large");
  const int own_slots = h->own_tiles * TILE;
  for (int i = 0; i < n_seg; ++i)
    for (int64_t e = H.off[i]; e < H.off[i] + (int64_t)H.count[i]; ++e) {
      const bool ok = is_send[i] ? (pos[e] >= 0 && pos[e] < own_slots)
                                 : (pos[e] >= own_slots && pos[e] < h->n_tot);
      if (!ok) return fail(HB_ERR_ARG, is_send[i] ? "send entry outside the owned slots"
                                                  : "receive entry outside the halo slots");
      if (site[e] < 0 || site[e] >= d) return fail(HB_ERR_ARG, "halo site outside the block");
    }
  // Hermitian-packed planes of the cross of block position s (row/column s)
  std::vector<int16_t> planes((size_t)d * nc);
  auto packed_off = [&](int a, int b) {  // a < b
    int e = 0;
    for (int r = 0; r < a; ++r) e += d - 1 - r;
    return e + (b - a - 1);
  };
  for (int s = 0; s < d; ++s) {
    int q = 0;
    planes[(size_t)s * nc + q++] = (int16_t)s;
    for (int o = 0; o < d; ++o) {
      if (o == s) continue;
      const int re = d + 2 * packed_off(s < o ? s : o, s < o ? o : s);
      planes[(size_t)s * nc + q++] = (int16_t)re;
      planes[(size_t)s * nc + q++] = (int16_t)(re + 1);
    }
  }
  const size_t ib = (size_t)std::max<int64_t>(total, 1) * sizeof(int32_t);
  CK(cudaMalloc(&H.pos, ib));
  CK(cudaMalloc(&H.site, ib));
  CK(cudaMalloc(&H.planes, planes.size() * sizeof(int16_t)));
  CK(cudaMalloc(&H.packed, (size_t)std::max<int64_t>(total, 1) * nc * elem_size(h)));
  if (total) {
    CK(hb_memcpy(H.pos, pos, total * sizeof(int32_t), cudaMemcpyHostToDevice, h->stream));
    CK(hb_memcpy(H.site, site, total * sizeof(int32_t), cudaMemcpyHostToDevice, h->stream));
  }
  CK(hb_memcpy(H.planes, planes.data(), planes.size() * sizeof(int16_t), cudaMemcpyHostToDevice,
               h->stream));
  CK(cudaStreamSynchronize(h->stream));
  h->halo_primed = false;
  return HB_OK;
}

// NCCL: one shard per process and GPU, exchange overlapped with the interior
int hb_shard_steps(hb_handle* h, int64_t n_steps, double* ms) {
  int rc = check_shard(h);
  if (rc) return rc;
  if (!h->nccl_comm) return fail(HB_ERR_ARG, "hb_nccl_init must be called first");
  if (n_steps < 0) return fail(HB_ERR_ARG, "negative step count");
  CK(cudaSetDevice(h->device));
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  if (ms) {
    CK(cudaEventCreate(&t0));
    CK(cudaEventCreate(&t1));
    CK(cudaEventRecord(t0, h->stream));
  }
  if (!h->halo_primed) {  // the halo of sigma (buffer 0) before the first stage
    CK(cudaEventRecord(h->ev_send[3], h->stream));
    CK(cudaStreamWaitEvent(h->comm, h->ev_send[3], 0));
    rc = exchange_nccl(h, 0);
    if (rc) return rc;
    h->halo_primed = true;
  }
  // a shard without a halo plan (one rank) runs its stages back to back, keeping
  // the programmatic-launch overlap between them
  bool has_halo = false;
  for (size_t i = 0; i < h->halo.count.size(); ++i) has_halo = has_halo || h->halo.count[i] > 0;
  for (int64_t it = 0; it < n_steps; ++it) {
    int n_launched = 0;
    for (int s = 1; s <= 4; ++s) {
      const int b_in = s - 1, b_out = s % 4;
      if (!has_halo) {
        for (int g = 0; g < 4; ++g) CK(launch_group(h, s, g, h->stream, &n_launched));
        continue;
      }
      // the previous pack of b_out must have read it before this stage rewrites it
      if (h->packed_once[b_out]) CK(cudaStreamWaitEvent(h->stream, h->ev_packed[b_out], 0));
      CK(launch_group(h, s, 0, h->stream, &n_launched));
      CK(launch_group(h, s, 1, h->stream, &n_launched));
      CK(cudaStreamWaitEvent(h->stream, h->ev_halo[b_in], 0));
      CK(launch_group(h, s, 2, h->stream, &n_launched));
      CK(cudaEventRecord(h->ev_send[s - 1], h->stream));
      CK(cudaStreamWaitEvent(h->comm, h->ev_send[s - 1], 0));
      rc = exchange_nccl(h, b_out);
      if (rc) return rc;
      CK(launch_group(h, s, 3, h->stream, &n_launched));
    }
    const long long step_next = h->host_step + 1;
    if (step_next % 25 == 0) {  // every shard sees the global max|x|^2 (heom.py:386-389)
      CK(cudaEventRecord(h->ev_s4, h->stream));
      CK(cudaStreamWaitEvent(h->comm, h->ev_s4, 0));
      const int r = nccl().allreduce(&h->ctl->maxabs2_bits, &h->ctl->maxabs2_bits, 1, kNcclUint64,
                                     kNcclMax, h->nccl_comm, h->comm);
      if (r) return nccl_fail(r, "ncclAllReduce");
      CK(cudaEventRecord(h->ev_guard, h->comm));
      CK(cudaStreamWaitEvent(h->stream, h->ev_guard, 0));
    }
    CK(launch_step_finish(stage_params(h, 4), h->stream));
    h->host_step = step_next;
    h->launches += n_launched + 1 - 5;  // k_step_finish counts 5 on the device
  }
  if (ms) {
    CK(cudaEventRecord(t1, h->stream));
    CK(cudaEventSynchronize(t1));
    float f = 0.f;
    CK(cudaEventElapsedTime(&f, t0, t1));
    *ms = f;
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
  }
  return HB_OK;
}

// In-process shards on one device: the same launch groups, the exchange as
// device copies of the packed crosses (owner pack -> consumer unpack), every
// stage serialised across the shards.  The bit-exactness check of the
// partition, the local numbering and the halo plan.
static int exchange_local(hb_handle** S, int n, int b) {
  for (int q = 0; q < n; ++q) CK(cudaEventRecord(S[q]->ev_send[0], S[q]->stream));
  for (int q = 0; q < n; ++q) {
    hb_handle* c = S[q];
    auto& H = c->halo;
    for (size_t i = 0; i < H.count.size(); ++i) {
      if (H.is_send[i]) continue;
      const int o = H.peer[i];
      if (o < 0 || o >= n || o == q) return fail(HB_ERR_ARG, "halo peer outside the shard set");
      hb_handle* w = S[o];
      int j = -1;
      for (size_t k = 0; k < w->halo.count.size(); ++k)
        if (w->halo.is_send[k] && w->halo.peer[k] == q) j = (int)k;
      if (j < 0 || w->halo.count[j] != H.count[i])
        return fail(HB_ERR_ARG, "halo plans of the owner and the consumer disagree");
      CK(cudaStreamWaitEvent(c->stream, w->ev_send[0], 0));
      if (H.count[i] == 0) continue;
      CK(pack_seg(w, j, b, c->stream));
      CK(unpack_seg(c, (int)i, b, seg_packed(w, j), c->stream));
      c->launches += 2;
    }
  }
  for (int q = 0; q < n; ++q) CK(cudaEventRecord(S[q]->ev_send[1], S[q]->stream));
  for (int o = 0; o < n; ++o)
    for (int q = 0; q < n; ++q)
      if (q != o) CK(cudaStreamWaitEvent(S[o]->stream, S[q]->ev_send[1], 0));
  return HB_OK;
}

int hb_shard_steps_local(hb_handle** S, int n, int64_t n_steps, double* ms) {
  if (!S || n < 1 || n > 64) return fail(HB_ERR_ARG, "need 1..64 shard handles");
  for (int q = 0; q < n; ++q) {
    int rc = check_shard(S[q]);
    if (rc) return rc;
    if (S[q]->device != S[0]->device) return fail(HB_ERR_ARG, "in-process shards share one device");
  }
  if (n_steps < 0) return fail(HB_ERR_ARG, "negative step count");
  CK(cudaSetDevice(S[0]->device));
  for (int q = 0; q < n; ++q) CK(cudaStreamSynchronize(S[q]->comm));
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  if (ms) {
    CK(cudaEventCreate(&t0));
    CK(cudaEventCreate(&t1));
    CK(cudaEventRecord(t0, S[0]->stream));
    for (int q = 1; q < n; ++q) CK(cudaStreamWaitEvent(S[q]->stream, t0, 0));
  }
  bool primed = true;
  for (int q = 0; q < n; ++q) primed = primed && S[q]->halo_primed;
  if (!primed) {
    int rc = exchange_local(S, n, 0);
    if (rc) return rc;
    for (int q = 0; q < n; ++q) S[q]->halo_primed = true;
  }
  std::vector<unsigned long long*> bits(n);
  for (int q = 0; q < n; ++q) bits[q] = &S[q]->ctl->maxabs2_bits;
  for (int64_t it = 0; it < n_steps; ++it) {
    for (int s = 1; s <= 4; ++s) {
      for (int q = 0; q < n; ++q) {
        int n_launched = 0;
        for (int g = 0; g < 4; ++g) CK(launch_group(S[q], s, g, S[q]->stream, &n_launched));
        S[q]->launches += n_launched;
      }
      int rc = exchange_local(S, n, s % 4);
      if (rc) return rc;
    }
    const long long step_next = S[0]->host_step + 1;
    if (step_next % 25 == 0 && n > 1) {
      for (int q = 1; q < n; ++q) {
        CK(cudaEventRecord(S[q]->ev_s4, S[q]->stream));
        CK(cudaStreamWaitEvent(S[0]->stream, S[q]->ev_s4, 0));
      }
      CK(launch_guard_max(bits.data(), n, S[0]->stream));
      S[0]->launches += 1;
      CK(cudaEventRecord(S[0]->ev_guard, S[0]->stream));
      for (int q = 1; q < n; ++q) CK(cudaStreamWaitEvent(S[q]->stream, S[0]->ev_guard, 0));
    }
    for (int q = 0; q < n; ++q) {
      CK(launch_step_finish(stage_params(S[q], 4), S[q]->stream));
      S[q]->launches += 1 - 5;  // k_step_finish counts 5 per step on the device
      S[q]->host_step = step_next;
    }
  }
  if (ms) {
    for (int q = 1; q < n; ++q) {
      CK(cudaEventRecord(S[q]->ev_s4, S[q]->stream));
      CK(cudaStreamWaitEvent(S[0]->stream, S[q]->ev_s4, 0));
    }
    CK(cudaEventRecord(t1, S[0]->stream));
    CK(cudaEventSynchronize(t1));
    float f = 0.f;
    CK(cudaEventElapsedTime(&f, t0, t1));
    *ms = f;
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
  }
  return HB_OK;
}
