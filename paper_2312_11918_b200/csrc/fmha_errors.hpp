// fmha_errors.hpp -- per-thread error/launch state shared by the C ABI
// translation units (fmha_api.cu, fmha_host.cpp).
#pragma once
#include <cstdint>
#include <string>

#include "../../include/fmha/fmha.h"

namespace fmha_b200 {
inline thread_local std::string g_last_error;
inline thread_local int g_last_launches = 0;

// A piece of the host pipeline's output: batches [b0, b1) x heads [h0, h1)
// x query rows [n0, n1) of O (and the matching LSE rows), complete on the host.
struct OutPiece {
  int64_t b0, b1, h0, h1, n0, n1;
};

// fmha_fwd_host's pipeline with two hooks:
//  * prepare(ctx, b0, b1) runs on the calling thread right before batches
//    [b0, b1) of Q/K/V are copied to the device, while earlier chunks' copies
//    and kernels proceed (fmha_forward_f32 quantises its float inputs there);
//  * consume(ctx, piece) runs on the calling thread, in issue order, as soon
//    as a piece of O / LSE has landed in the host buffers, while later pieces
//    are still computed and copied (fmha_forward_f32 dequantises there).
fmha_status fwd_host_pipeline(const fmha_fwd_params* p, const void* q, const void* k, const void* v, void* o,
                              float* lse, int device, void (*prepare)(void* ctx, int64_t b0, int64_t b1),
                              void* ctx, void (*consume)(void* ctx, const OutPiece& piece) = nullptr);
}  // namespace fmha_b200
