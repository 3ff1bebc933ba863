// transport.h -- point-to-point + all-reduce between the z-slab ranks.
//
// Two implementations behind one interface:
//   * NcclTransport  : one process per GPU, NCCL (libnccl.so.2 loaded with dlopen, the copy
//                      torch already mapped is reused), grouped ncclSend/ncclRecv on the
//                      engine's stream, ncclAllReduce in place.
//   * LocalTransport : several contexts of ONE process (host threads, possibly one GPU)
//                      exchanging through a process-wide registry with D2D copies and CUDA
//                      events.  Used to run the multi-rank device path on a single B200 in the
//                      tests; selected by an id starting with "LJMDLOCAL".
//   * ShmTransport   : several PROCESSES on one GPU (NCCL refuses two ranks per device):
//                      transfers staged through host files under /dev/shm; selected by an id
//                      "LJMDSHM:<key>".  Tests and bench.py's one-GPU multi-process run.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace ljmd {

struct Xfer {
    int peer;
    void* ptr;
    size_t bytes;
};

class Transport {
public:
    virtual ~Transport() {}
    // Grouped exchange: every send is matched, per (src, dst) pair in posting order, with the
    // peer's recv.  Completion is ordered on `stream` (no host sync implied for NCCL).
    virtual bool exchange(cudaStream_t stream, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs,
                          std::string& err) = 0;
    // In-place all-reduce of n doubles in device memory (sum or max), ordered on `stream`.
    virtual bool allreduce(cudaStream_t stream, double* dbuf, int n, bool max, std::string& err) = 0;
    virtual const char* name() const = 0;
};

// nccl_id: 128 bytes.  Returns nullptr and sets err on failure.
Transport* make_transport(const void* nccl_id, int rank, int nranks, int device, std::string& err);
// ncclGetUniqueId through the dlopen'ed NCCL (rank 0 calls it, the caller broadcasts it)
bool nccl_unique_id(void* out128, std::string& err);

}  // namespace ljmd
