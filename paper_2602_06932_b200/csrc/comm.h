// comm.h — the library's communicator: a VP group and a DP group per rank,
// served by one of two transports behind the same three collectives:
//   * NCCL (one process per GPU; dlopen'd, bootstrapped from a broadcast unique id);
//   * loopback: P virtual ranks on ONE device, one host thread + stream per rank, the
//     collectives done as device copies into a group-shared staging buffer ordered by
//     CUDA events and a host barrier.  It exists so the multi-rank code of the library
//     (C1 merge, F2 triple merge, P-way row combine, C2/C4/C5 sums, the DP reduce-scatter
//     + sharded optimizer) runs and is checked against the oracle on a one-GPU box.
#pragma once
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <mutex>
#include <vector>

#include "../../include/aurora.h"

namespace aur {

enum CollGroup : int { G_VP = 0, G_DP = 1 };
enum CollType : int { DT_F32 = 0, DT_I32 = 1 };

// Loopback group shared by the virtual ranks of one VP or DP group.
struct LoopGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  void* stage = nullptr;  // [n][bytes] staging buffer (device)
  size_t stage_bytes = 0;
  std::vector<cudaEvent_t> in_ev, done_ev;  // per member: contribution staged / copy-out done
  int refs = 0;
  bool failed = false;
};

}  // namespace aur

struct aurora_comm_s {
  int nranks, rank, vp_size, dp_size, vp_rank, dp_rank;
  // A 1-rank communicator runs every exchange (identity collectives); it exists to
  // exercise the collective plumbing on one GPU.  Otherwise a group exchanges iff size > 1.
  bool vp_x() const { return nranks == 1 || vp_size > 1; }
  bool dp_x() const { return nranks == 1 || dp_size > 1; }
  int kind = 0;  // 0 NCCL, 1 loopback
  void* world = nullptr;
  void* vp = nullptr;
  void* dp = nullptr;  // ncclComm_t (NCCL)
  aur::LoopGroup* lvp = nullptr;
  aur::LoopGroup* ldp = nullptr;  // loopback groups
  void* scratch = nullptr;        // comm-owned device scratch for gathered candidates / stats
  size_t scratch_bytes = 0;
  // comm-owned side stream + fork / join events (created on first use on the calling device):
  // the C4 dH allreduce runs there, overlapped with the last dW GEMM
  cudaStream_t side = nullptr;
  cudaEvent_t side_ev[2] = {nullptr, nullptr};
};

namespace aur {
// All three enqueue on `s` and return AURORA_ERR_NCCL / AURORA_ERR_CUDA on failure.
// allgather: recv = [member][count] (rank order); allreduce: recv = sum over members (send
// and recv may alias); reduce_scatter: recv[count] = sum over members of send[member
// slot: this rank's index * count .. +count).
aurora_status_t coll_allgather(aurora_comm_t c, int group, const void* send, void* recv, size_t count, int dt,
                               cudaStream_t s);
aurora_status_t coll_allreduce(aurora_comm_t c, int group, const void* send, void* recv, size_t count, int dt,
                               cudaStream_t s);
aurora_status_t coll_reduce_scatter(aurora_comm_t c, int group, const void* send, void* recv, size_t count, int dt,
                                    cudaStream_t s);
inline int group_size(aurora_comm_t c, int g) { return g == G_VP ? c->vp_size : c->dp_size; }
inline int group_rank(aurora_comm_t c, int g) { return g == G_VP ? c->vp_rank : c->dp_rank; }
}  // namespace aur
