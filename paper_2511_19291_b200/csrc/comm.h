// comm.h -- the transport under the sharded state (§4.2):
// the remap exchange (grouped point-to-point block swaps) and the scalar /
// vector sum reductions.  Two implementations:
//
//   * NcclComm: one process per GPU, NCCL over NVLink / NVSwitch (the product
//     path for world > 1);
//   * LoopComm: W ranks emulated inside ONE process on ONE device, one host
//     thread per rank.  Blocks move with device-to-device cudaMemcpyAsync between
//     the ranks' buffers after a host barrier; no kernel ever waits on another
//     rank's kernel (host threads synchronise, then copy).  It exists so the
//     multi-rank device path (rank-bit conditioned sweeps, remap pack / unpack,
//     sharded expval / adjoint / readback) can be checked on a 1-GPU machine.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace tqd {

enum CommElem { CE_F32 = 0, CE_F64 = 1 };

class Comm {
  public:
    virtual ~Comm() {}
    // grouped point-to-point: every send to peer p pairs with p's recv from us,
    // in posting order; the group executes at group_end (stream-ordered)
    virtual int group_start() = 0;
    virtual int send(const void *buf, size_t bytes, int peer, cudaStream_t s) = 0;
    virtual int recv(void *buf, size_t bytes, int peer, cudaStream_t s) = 0;
    virtual int group_end(cudaStream_t s) = 0;
    // in-place elementwise sum over all ranks of a device buffer
    virtual int allreduce_sum(void *buf, size_t count, CommElem t, cudaStream_t s) = 0;
    // make nbuf local device allocations addressable by every rank (peer memory):
    // table[r * nbuf + i] = rank r's buffer i, usable in this process's kernels.
    // NCCL: CUDA IPC handles exchanged with an all-gather (NVLink P2P); loopback:
    // plain pointers (same device).  Collective.  Returns 0, 1 (error) or 2 (peer
    // memory unavailable on some rank -- the same answer on every rank).
    virtual int share_buffers(void *const *local, int nbuf, std::vector<void *> &table, cudaStream_t s) = 0;
    virtual void release_buffers(std::vector<void *> &table, int nbuf) {}
    // returns once the work every rank queued before it has completed (host-blocking)
    virtual int barrier(cudaStream_t s) = 0;
    int rank = 0, world = 1;
    std::string err;
};

// 128-byte ids: NCCL's unique id, or a loopback id (magic prefix + hub key)
bool comm_is_loopback_id(const void *id128);
void comm_make_loopback_id(void *id128);
// returns nullptr and sets err on failure
Comm *comm_create(const void *id128, int world, int rank, std::string &err);

}  // namespace tqd
