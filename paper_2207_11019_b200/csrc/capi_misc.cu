// Misc C entry points: error slot, version, device count, defaults.
#include <cuda_runtime.h>

#include <string>

#include "capi_common.h"

namespace {
thread_local std::string g_last_error;
}

void ppb_set_error(const std::string& msg) { g_last_error = msg; }

extern "C" const char* ppb_last_error(void) { return g_last_error.c_str(); }

extern "C" const char* ppb_version(void) { return "pipeplan_b200 0.1 (sm_100a, tcgen05 tf32)"; }

extern "C" int ppb_device_count(int* out_count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *out_count = 0;
        ppb_set_error(std::string("no CUDA device: ") + cudaGetErrorString(e));
        return PPB_ERR_NO_DEVICE;
    }
    *out_count = n;
    return PPB_OK;
}

extern "C" void ppb_default_options(ppb_options* o) {
    *o = ppb_options{};
    o->receive_timeout_s = 30.0;
    o->precision = PPB_PRECISION_TF32;
    o->multiclass_accuracy = 0;
    o->use_graph = 1;
    o->pipeline_gate = 2;
}

extern "C" void ppb_default_config(ppb_train_config* c) {
    // TrainConfig defaults, include/pipeplan/tinynet.hpp:76-82.
    c->alpha0 = 1e-4;
    c->decay = 1e-2;
    c->loss = PPB_LOSS_CE;
    c->iterations = 50;
    c->seed = 1;
}
