// fmha_errors.hpp -- per-thread error/launch state shared by the C ABI
// translation units (fmha_api.cu, fmha_host.cpp).
#pragma once
#include <string>

namespace fmha_b200 {
inline thread_local std::string g_last_error;
inline thread_local int g_last_launches = 0;
}  // namespace fmha_b200
