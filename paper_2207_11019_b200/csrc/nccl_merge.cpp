// NCCL transport for the dense merges; see nccl_merge.h.
#include "nccl_merge.h"

#include "kernels.h"

#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <stdexcept>

namespace ppb {

namespace {

struct Api {
    bool ok = false;
    std::string err;
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                   cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const Api& api() {
    static Api a;
    static std::once_flag once;
    std::call_once(once, [] {
        // the process may already hold an NCCL (e.g. torch's): reuse that soname
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h == nullptr) {
            a.err = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (fn == nullptr && a.err.empty()) a.err = std::string("libnccl.so.2 lacks ") + name;
        };
        sym(a.comm_init_all, "ncclCommInitAll");
        sym(a.comm_destroy, "ncclCommDestroy");
        sym(a.group_start, "ncclGroupStart");
        sym(a.group_end, "ncclGroupEnd");
        sym(a.all_gather, "ncclAllGather");
        sym(a.reduce_scatter, "ncclReduceScatter");
        sym(a.error_string, "ncclGetErrorString");
        a.ok = a.err.empty();
    });
    return a;
}

// NCCL failures surface as a CUDA error code at the launch site (the op
// machinery reports it with the op's context).
cudaError_t to_cuda(ncclResult_t r) { return r == ncclSuccess ? cudaSuccess : cudaErrorUnknown; }

}  // namespace

NcclGroup::~NcclGroup() {
    if (loopback || comms.empty()) return;
    const Api& a = api();
    if (!a.ok) return;
    for (void* c : comms)
        if (c != nullptr) a.comm_destroy(static_cast<ncclComm_t>(c));
}

std::unique_ptr<NcclGroup> nccl_group_create(const std::vector<int>& ordinals) {
    auto g = std::make_unique<NcclGroup>();
    g->ordinals = ordinals;
    bool all_same = true;
    for (int o : ordinals) all_same = all_same && o == ordinals.front();
    if (all_same) {
        g->loopback = true;
        return g;
    }
    const Api& a = api();
    if (!a.ok) throw std::runtime_error("NCCL merge backend: " + a.err);
    for (size_t i = 0; i < ordinals.size(); ++i)
        for (size_t k = 0; k < i; ++k)
            if (ordinals[i] == ordinals[k])
                throw std::invalid_argument("NCCL merge backend needs one plan device per GPU (GPU " +
                                            std::to_string(ordinals[i]) + " appears twice)");
    std::vector<ncclComm_t> comms(ordinals.size(), nullptr);
    const ncclResult_t r = a.comm_init_all(comms.data(), static_cast<int>(ordinals.size()), ordinals.data());
    if (r != ncclSuccess) throw std::runtime_error(std::string("ncclCommInitAll: ") + a.error_string(r));
    g->comms.assign(comms.begin(), comms.end());
    return g;
}

cudaError_t nccl_all_gather(const NcclGroup& g, const std::vector<const float*>& send,
                            const std::vector<float*>& recv, size_t count,
                            const std::vector<cudaStream_t>& streams) {
    if (g.loopback) {  // every send buffer was produced before the collective's op (its stream waited)
        for (size_t r = 0; r < recv.size(); ++r)
            for (size_t k = 0; k < send.size(); ++k) {
                const cudaError_t e = cudaMemcpyAsync(recv[r] + k * count, send[k], sizeof(float) * count,
                                                      cudaMemcpyDeviceToDevice, streams[0]);
                if (e != cudaSuccess) return e;
            }
        return cudaSuccess;
    }
    const Api& a = api();
    if (!a.ok) return cudaErrorUnknown;
    ncclResult_t r = a.group_start();
    for (size_t k = 0; k < g.comms.size() && r == ncclSuccess; ++k)
        r = a.all_gather(send[k], recv[k], count, ncclFloat32, static_cast<ncclComm_t>(g.comms[k]), streams[k]);
    const ncclResult_t e = a.group_end();
    return to_cuda(r != ncclSuccess ? r : e);
}

cudaError_t nccl_reduce_scatter(const NcclGroup& g, const std::vector<const float*>& send,
                                const std::vector<float*>& recv, int rows, int u,
                                const std::vector<cudaStream_t>& streams) {
    const size_t count = static_cast<size_t>(rows) * u;
    if (g.loopback) {  // ascending-rank sum of block r (the reference's order)
        for (size_t r = 0; r < recv.size(); ++r) {
            ReduceSlots rs;
            for (size_t k = 0; k < send.size(); ++k) rs.slot[rs.n++] = send[k] + r * count;
            const cudaError_t e = launch_reduce_mask(rs, u, rows, u, nullptr, 0, recv[r], u, streams[0]);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    const Api& a = api();
    if (!a.ok) return cudaErrorUnknown;
    ncclResult_t r = a.group_start();
    for (size_t k = 0; k < g.comms.size() && r == ncclSuccess; ++k)
        r = a.reduce_scatter(send[k], recv[k], count, ncclFloat32, ncclSum, static_cast<ncclComm_t>(g.comms[k]),
                             streams[k]);
    const ncclResult_t e = a.group_end();
    return to_cuda(r != ncclSuccess ? r : e);
}

}  // namespace ppb
