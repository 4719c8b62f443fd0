// gtcp_comm.cuh -- the library's communication layer (private).
//
// Every exchange step of the decomposed hot path (§3.2: ghost-plane
// charge merge, particle-replica / section allreduce, flux-surface sums,
// potential halos, shift counts and payload) goes through these calls.  Two
// transports sit behind one interface:
//   - NCCL (the product): one process per GPU, communicators over NVLink /
//     NVSwitch, all work enqueued on the context stream;
//   - loopback (test-only): K contexts of one process on ONE device, one host
//     thread per context, each message one cudaMemcpyAsync between the two
//     contexts' device buffers, each reduction one small kernel summing the
//     members' staged buffers in member order.  It lets the decomposition
//     logic (every byte the library exchanges) run and be checked on a single
//     GPU (SURVEY §4 "test-only loopback transport").
// Both count the bytes they move (NCCL bus-byte convention: send/recv payload,
// allreduce 2(n-1)/n x size, broadcast size) into the caller's accumulator.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstddef>

namespace gtcp {

struct LoopShared;  // state shared by the members of one loopback communicator
struct LoopHub;     // one per loopback "job": owns every LoopShared

struct Comm {
    ncclComm_t nc = nullptr;
    LoopShared* ls = nullptr;
    int rank = 0, size = 1;
    bool valid() const { return nc != nullptr || ls != nullptr; }
};

LoopHub* loop_hub_create(int nranks);
void loop_hub_destroy(LoopHub* h);
int loop_hub_size(const LoopHub* h);
Comm loop_world(LoopHub* h, int rank);

ncclResult_t comm_init_nccl(Comm* out, int nranks, const ncclUniqueId& id, int rank);
ncclResult_t comm_split(const Comm& parent, int color, int key, Comm* out);
void comm_destroy(Comm* c);

ncclResult_t comm_group_start();
ncclResult_t comm_group_end();
ncclResult_t comm_send(const Comm& c, const void* buf, size_t count, ncclDataType_t ty, int peer, cudaStream_t st,
                       long long* acct);
ncclResult_t comm_recv(const Comm& c, void* buf, size_t count, ncclDataType_t ty, int peer, cudaStream_t st,
                       long long* acct);
ncclResult_t comm_allreduce(const Comm& c, const void* sbuf, void* rbuf, size_t count, ncclDataType_t ty,
                            ncclRedOp_t op, cudaStream_t st, long long* acct);
ncclResult_t comm_bcast(const Comm& c, const void* sbuf, void* rbuf, size_t count, ncclDataType_t ty, int root,
                        cudaStream_t st, long long* acct);
const char* comm_error_string(ncclResult_t r);

}  // namespace gtcp
