// NCCL transport for the dense merges (north_star (2): the fused peer-store
// gather vs an NCCL all-gather / reduce-scatter, chosen by measured NVLink
// GB/s).  libnccl.so.2 is opened at run time (dlopen), only when a session
// asks for this backend, so the product library has no link-time NCCL
// dependency.  One communicator per sub-module over its devices (rank =
// position in the sub-module's device list, the reference's contributor
// order), single process, all ranks driven from this thread inside an NCCL
// group (ncclCommInitAll / ncclGroupStart..End).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

namespace ppb {

struct NcclGroup {
    std::vector<int> ordinals;  // CUDA ordinal of each rank
    std::vector<void*> comms;   // ncclComm_t per rank
    // every rank on ONE GPU (how multi-device plans are tested on a one-GPU
    // box; NCCL cannot hold a GPU twice): the collectives' exact semantics
    // emulated with device copies / an ascending-rank sum on ranks[0]'s
    // stream, so the NCCL data layout (packing, unpacking) is exercised
    bool loopback = false;
    ~NcclGroup();
};

// Throws std::runtime_error (with NCCL's message) when the library or the
// communicator cannot be created, std::invalid_argument when some but not
// all ranks share a GPU.
std::unique_ptr<NcclGroup> nccl_group_create(const std::vector<int>& ordinals);

// recv[r] = [send[0] | send[1] | ... | send[n-1]] (count floats each), on
// streams[r], as one NCCL group.
cudaError_t nccl_all_gather(const NcclGroup& g, const std::vector<const float*>& send,
                            const std::vector<float*>& recv, size_t count, const std::vector<cudaStream_t>& streams);
// recv[r] = sum over ranks of send[rank][r-th block of rows x u floats].
cudaError_t nccl_reduce_scatter(const NcclGroup& g, const std::vector<const float*>& send,
                                const std::vector<float*>& recv, int rows, int u,
                                const std::vector<cudaStream_t>& streams);

}  // namespace ppb
