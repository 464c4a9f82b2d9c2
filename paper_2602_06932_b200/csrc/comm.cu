// comm.cu — communicator creation and the three collectives of the VP / DP modes
// over NCCL or the single-device loopback transport.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>

#include "comm.h"
#include "internal.h"

namespace aur {

// ------------------------------------------------------------------ NCCL (dlopen)
namespace nccl {
typedef int Result;
typedef void* Comm;
struct UniqueId { char internal[128]; };
enum { ncclInt32 = 2, ncclFloat32 = 7 };
enum { ncclSum = 0 };
struct Api {
  bool ok = false;
  Result (*GetUniqueId)(UniqueId*) = nullptr;
  Result (*CommInitRank)(Comm*, int, UniqueId, int) = nullptr;
  Result (*CommDestroy)(Comm) = nullptr;
  Result (*CommSplit)(Comm, int, int, Comm*, void*) = nullptr;
  Result (*AllReduce)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  Result (*AllGather)(const void*, void*, size_t, int, Comm, cudaStream_t) = nullptr;
  Result (*ReduceScatter)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
};
Api& api() {
  static Api a;
  static bool tried = false;
  if (tried) return a;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy torch already loaded
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return a;
  a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
  a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
  a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
  a.CommSplit = reinterpret_cast<decltype(a.CommSplit)>(dlsym(h, "ncclCommSplit"));
  a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(h, "ncclAllReduce"));
  a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
  a.ReduceScatter = reinterpret_cast<decltype(a.ReduceScatter)>(dlsym(h, "ncclReduceScatter"));
  a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.CommSplit && a.AllReduce && a.AllGather &&
         a.ReduceScatter;
  return a;
}
int nccl_type(int dt) { return dt == DT_I32 ? ncclInt32 : ncclFloat32; }
}  // namespace nccl

// ------------------------------------------------------------------ loopback transport
namespace {

// Ordered sum over the n member slots (member 0 first): deterministic.
template <typename T>
__global__ void k_loop_sum(const T* __restrict__ stage, int n, size_t count, size_t stride, T* __restrict__ out) {
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    T acc = stage[i];
    for (int q = 1; q < n; ++q) acc += stage[static_cast<size_t>(q) * stride + i];
    out[i] = acc;
  }
}

template <typename F>
bool barrier(LoopGroup* g, F&& leader) {
  std::unique_lock<std::mutex> lk(g->mu);
  const uint64_t gen = g->gen;
  if (++g->arrived == g->n) {
    if (!leader()) g->failed = true;
    g->arrived = 0;
    ++g->gen;
    g->cv.notify_all();
  } else {
    g->cv.wait(lk, [&] { return g->gen != gen; });
  }
  return !g->failed;
}

enum { OP_AG = 0, OP_AR = 1, OP_RS = 2 };

// Per member: (1) host barrier — the last arrival grows the staging buffer; (2) wait for
// every member's previous copy-out, stage this member's contribution, record in_ev[me];
// (3) host barrier — every in_ev of this collective is recorded; (4) wait for all of
// them, copy out / reduce, record done_ev[me].  Event reuse is race-free: a member
// re-records in_ev only after barrier (1) of the next collective, which every member
// reaches after its step (4) of this one.
aurora_status_t loop_coll(LoopGroup* g, int me, int op, const void* send, void* recv, size_t count, int dt,
                          cudaStream_t s) {
  const size_t esz = 4;
  const size_t B = count * esz;
  const size_t contrib = (op == OP_RS) ? static_cast<size_t>(g->n) * B : B;
  const size_t need = static_cast<size_t>(g->n) * contrib;
  if (count == 0) return AURORA_OK;
  if (!barrier(g, [&] {
        if (g->stage_bytes >= need) return true;
        if (g->stage) cudaFree(g->stage);  // synchronising; growth only
        g->stage = nullptr;
        g->stage_bytes = 0;
        if (cudaMalloc(&g->stage, need) != cudaSuccess) return false;
        g->stage_bytes = need;
        return true;
      }))
    return AURORA_ERR_CUDA;
  char* st = static_cast<char*>(g->stage);
  for (int q = 0; q < g->n; ++q)
    if (cudaStreamWaitEvent(s, g->done_ev[q], 0) != cudaSuccess) return AURORA_ERR_CUDA;
  if (cudaMemcpyAsync(st + static_cast<size_t>(me) * contrib, send, contrib, cudaMemcpyDeviceToDevice, s) !=
      cudaSuccess)
    return AURORA_ERR_CUDA;
  if (cudaEventRecord(g->in_ev[me], s) != cudaSuccess) return AURORA_ERR_CUDA;
  if (!barrier(g, [] { return true; })) return AURORA_ERR_CUDA;
  for (int q = 0; q < g->n; ++q)
    if (cudaStreamWaitEvent(s, g->in_ev[q], 0) != cudaSuccess) return AURORA_ERR_CUDA;
  const int blocks = static_cast<int>(std::min<size_t>((count + 255) / 256, 4 * kNumSMs));
  if (op == OP_AG) {
    if (cudaMemcpyAsync(recv, st, need, cudaMemcpyDeviceToDevice, s) != cudaSuccess) return AURORA_ERR_CUDA;
  } else {
    const char* base = st + (op == OP_RS ? static_cast<size_t>(me) * B : 0);
    const size_t stride = contrib / esz;
    if (dt == DT_I32)
      k_loop_sum<int32_t><<<blocks, 256, 0, s>>>(reinterpret_cast<const int32_t*>(base), g->n, count, stride,
                                                 static_cast<int32_t*>(recv));
    else
      k_loop_sum<float><<<blocks, 256, 0, s>>>(reinterpret_cast<const float*>(base), g->n, count, stride,
                                               static_cast<float*>(recv));
    count_launch();
    if (cudaGetLastError() != cudaSuccess) return AURORA_ERR_CUDA;
  }
  if (cudaEventRecord(g->done_ev[me], s) != cudaSuccess) return AURORA_ERR_CUDA;
  return AURORA_OK;
}

LoopGroup* loop_group_new(int n) {
  auto* g = new LoopGroup();
  g->n = n;
  g->in_ev.resize(n);
  g->done_ev.resize(n);
  for (int i = 0; i < n; ++i) {
    if (cudaEventCreateWithFlags(&g->in_ev[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->done_ev[i], cudaEventDisableTiming) != cudaSuccess) {
      delete g;
      return nullptr;
    }
  }
  return g;
}

void loop_group_release(LoopGroup* g) {
  if (!g) return;
  bool last;
  {
    std::lock_guard<std::mutex> lk(g->mu);
    last = --g->refs == 0;
  }
  if (!last) return;
  for (auto e : g->in_ev) cudaEventDestroy(e);
  for (auto e : g->done_ev) cudaEventDestroy(e);
  if (g->stage) cudaFree(g->stage);
  delete g;
}

aurora_status_t dispatch(aurora_comm_t c, int group, int op, const void* send, void* recv, size_t count, int dt,
                         cudaStream_t s) {
  if (!c) return AURORA_ERR_INVALID_ARG;
  if (c->kind == 1) {
    LoopGroup* g = group == G_VP ? c->lvp : c->ldp;
    return loop_coll(g, group_rank(c, group), op, send, recv, count, dt, s);
  }
  auto& A = nccl::api();
  nccl::Comm nc = group == G_VP ? c->vp : c->dp;
  int r = 0;
  if (op == OP_AG) r = A.AllGather(send, recv, count, nccl::nccl_type(dt), nc, s);
  else if (op == OP_AR) r = A.AllReduce(send, recv, count, nccl::nccl_type(dt), nccl::ncclSum, nc, s);
  else r = A.ReduceScatter(send, recv, count, nccl::nccl_type(dt), nccl::ncclSum, nc, s);
  return r == 0 ? AURORA_OK : AURORA_ERR_NCCL;
}

}  // namespace

aurora_status_t coll_allgather(aurora_comm_t c, int group, const void* send, void* recv, size_t count, int dt,
                               cudaStream_t s) {
  return dispatch(c, group, OP_AG, send, recv, count, dt, s);
}
aurora_status_t coll_allreduce(aurora_comm_t c, int group, const void* send, void* recv, size_t count, int dt,
                               cudaStream_t s) {
  return dispatch(c, group, OP_AR, send, recv, count, dt, s);
}
aurora_status_t coll_reduce_scatter(aurora_comm_t c, int group, const void* send, void* recv, size_t count, int dt,
                                    cudaStream_t s) {
  return dispatch(c, group, OP_RS, send, recv, count, dt, s);
}

}  // namespace aur

using namespace aur;

extern "C" {

aurora_status_t aurora_comm_get_unique_id(void* id_out) {
  if (!id_out) return AURORA_ERR_INVALID_ARG;
  auto& A = nccl::api();
  if (!A.ok) return AURORA_ERR_NCCL;
  nccl::UniqueId id;
  if (A.GetUniqueId(&id) != 0) return AURORA_ERR_NCCL;
  std::memcpy(id_out, &id, sizeof(id));
  return AURORA_OK;
}

static bool layout_ok(int nranks, int vp_size, int dp_size) {
  return nranks >= 1 && vp_size >= 1 && dp_size >= 1 && vp_size * dp_size == nranks;
}

aurora_status_t aurora_comm_create(const void* id_in, int nranks, int rank, int vp_size, int dp_size,
                                   aurora_comm_t* out) {
  if (!id_in || !out || rank < 0 || rank >= nranks || !layout_ok(nranks, vp_size, dp_size))
    return AURORA_ERR_INVALID_ARG;
  auto& A = nccl::api();
  if (!A.ok) return AURORA_ERR_NCCL;
  auto* c = new aurora_comm_s();
  c->nranks = nranks;
  c->rank = rank;
  c->vp_size = vp_size;
  c->dp_size = dp_size;
  c->vp_rank = rank % vp_size;
  c->dp_rank = rank / vp_size;
  c->kind = 0;
  nccl::UniqueId id;
  std::memcpy(&id, id_in, sizeof(id));
  if (A.CommInitRank(&c->world, nranks, id, rank) != 0) {
    delete c;
    return AURORA_ERR_NCCL;
  }
  if (A.CommSplit(c->world, c->dp_rank, c->vp_rank, &c->vp, nullptr) != 0 ||
      A.CommSplit(c->world, c->vp_rank, c->dp_rank, &c->dp, nullptr) != 0) {
    A.CommDestroy(c->world);
    delete c;
    return AURORA_ERR_NCCL;
  }
  *out = c;
  return AURORA_OK;
}

aurora_status_t aurora_comm_create_loopback(int nranks, int vp_size, int dp_size, aurora_comm_t* out) {
  if (!out || !layout_ok(nranks, vp_size, dp_size) || nranks > 64) return AURORA_ERR_INVALID_ARG;
  std::vector<LoopGroup*> vpg(dp_size, nullptr), dpg(vp_size, nullptr);
  bool ok = true;
  for (auto& g : vpg) ok = ok && (g = loop_group_new(vp_size)) != nullptr;
  for (auto& g : dpg) ok = ok && (g = loop_group_new(dp_size)) != nullptr;
  if (!ok) {
    for (auto g : vpg) delete g;
    for (auto g : dpg) delete g;
    return AURORA_ERR_CUDA;
  }
  for (int r = 0; r < nranks; ++r) {
    auto* c = new aurora_comm_s();
    c->nranks = nranks;
    c->rank = r;
    c->vp_size = vp_size;
    c->dp_size = dp_size;
    c->vp_rank = r % vp_size;
    c->dp_rank = r / vp_size;
    c->kind = 1;
    c->lvp = vpg[c->dp_rank];
    c->ldp = dpg[c->vp_rank];
    c->lvp->refs++;
    c->ldp->refs++;
    out[r] = c;
  }
  return AURORA_OK;
}

aurora_status_t aurora_comm_destroy(aurora_comm_t c) {
  if (!c) return AURORA_ERR_INVALID_ARG;
  if (c->kind == 0) {
    auto& A = nccl::api();
    if (c->vp) A.CommDestroy(c->vp);
    if (c->dp) A.CommDestroy(c->dp);
    if (c->world) A.CommDestroy(c->world);
  } else {
    loop_group_release(c->lvp);
    loop_group_release(c->ldp);
  }
  if (c->scratch) cudaFree(c->scratch);
  for (auto& e : c->side_ev)
    if (e) cudaEventDestroy(e);
  if (c->side) cudaStreamDestroy(c->side);
  delete c;
  return AURORA_OK;
}

}  // extern "C"
