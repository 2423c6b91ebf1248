// fmha_errors.hpp -- per-thread error/launch state shared by the C ABI
// translation units (fmha_api.cu, fmha_host.cpp).
#pragma once
#include <cstdint>
#include <string>

#include "../../include/fmha/fmha.h"

namespace fmha_b200 {
inline thread_local std::string g_last_error;
inline thread_local int g_last_launches = 0;

// fmha_fwd_host's pipeline with a hook: prepare(ctx, b0, b1) runs on the
// calling thread right before batches [b0, b1) of Q/K/V are copied to the
// device, while earlier chunks' copies and kernels proceed (fmha_forward_f32
// quantises its float inputs there).
fmha_status fwd_host_pipeline(const fmha_fwd_params* p, const void* q, const void* k, const void* v, void* o,
                              float* lse, int device, void (*prepare)(void* ctx, int64_t b0, int64_t b1),
                              void* ctx);
}  // namespace fmha_b200
