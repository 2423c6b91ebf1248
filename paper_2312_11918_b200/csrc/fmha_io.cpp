// fmha_io.cpp -- FHMT fixture files: the reference's self-describing tensor
// dump (save_tensor / load_tensor, /root/reference/proj/src/tensor.cpp:30-84):
//   u32 magic 0x544D4846 ("FHMT"), u32 version 1, i64 L, N, h, d,
//   u32 precision (0 = f32, 1 = f16), then the values in row-major
//   (b, n, head, k) order as f32 or as RNE-rounded (saturating) binary16.
// Files written here load in the reference and vice versa
// (tests/test_fixture_io.py checks both directions against oracle/_ref).
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fmha/fmha.h"
#include "../../include/fmha/fmha.hpp"
#include "fmha_errors.hpp"

extern "C" uint16_t fmha_host_f32_to_16(float x, int bf16);
extern "C" float fmha_host_16_to_f32(uint16_t x, int bf16);

namespace {
constexpr uint32_t kMagic = 0x544D4846u;
constexpr uint32_t kVersion = 1;

fmha_status io_fail(const std::string& msg) {
  fmha_b200::g_last_error = msg;
  return FMHA_ERR_CONFIG;
}

struct File {
  std::FILE* f = nullptr;
  File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
};
}  // namespace

extern "C" {

fmha_status fmha_tensor_save(const char* path, const float* data, int64_t L, int64_t N, int64_t h,
                             int64_t d, int f16) {
  if (!path || !data || L < 0 || N < 0 || h < 0 || d < 0) return io_fail("fmha_tensor_save: bad arguments");
  File out(path, "wb");
  if (!out.f) return io_fail(std::string("save_tensor: cannot open ") + path);
  const uint32_t prec = f16 ? 1u : 0u;
  const int64_t dims[4] = {L, N, h, d};
  bool ok = std::fwrite(&kMagic, 4, 1, out.f) == 1 && std::fwrite(&kVersion, 4, 1, out.f) == 1 &&
            std::fwrite(dims, 8, 4, out.f) == 4 && std::fwrite(&prec, 4, 1, out.f) == 1;
  const int64_t n = L * N * h * d;
  if (ok && f16) {
    std::vector<uint16_t> buf(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) buf[i] = fmha_host_f32_to_16(data[i], 0);
    ok = std::fwrite(buf.data(), 2, buf.size(), out.f) == buf.size();
  } else if (ok) {
    ok = std::fwrite(data, 4, static_cast<size_t>(n), out.f) == static_cast<size_t>(n);
  }
  if (!ok) return io_fail(std::string("save_tensor: write failed for ") + path);
  return FMHA_OK;
}

fmha_status fmha_tensor_load_header(const char* path, int64_t dims[4], int* f16) {
  if (!path || !dims) return io_fail("fmha_tensor_load_header: bad arguments");
  File in(path, "rb");
  if (!in.f) return io_fail(std::string("load_tensor: cannot open ") + path);
  uint32_t magic = 0, version = 0, prec = 0;
  if (std::fread(&magic, 4, 1, in.f) != 1) return io_fail("tensor file truncated");
  if (magic != kMagic) return io_fail(std::string("load_tensor: bad magic in ") + path);
  if (std::fread(&version, 4, 1, in.f) != 1) return io_fail("tensor file truncated");
  if (version != kVersion) return io_fail(std::string("load_tensor: unsupported version in ") + path);
  if (std::fread(dims, 8, 4, in.f) != 4 || std::fread(&prec, 4, 1, in.f) != 1)
    return io_fail("tensor file truncated");
  if (f16) *f16 = prec == 1 ? 1 : 0;
  return FMHA_OK;
}

fmha_status fmha_tensor_load(const char* path, float* data, int64_t count) {
  int64_t dims[4];
  int f16 = 0;
  fmha_status s = fmha_tensor_load_header(path, dims, &f16);
  if (s != FMHA_OK) return s;
  const int64_t n = dims[0] * dims[1] * dims[2] * dims[3];
  if (!data || count < n) return io_fail("fmha_tensor_load: destination too small");
  File in(path, "rb");
  std::fseek(in.f, 4 + 4 + 32 + 4, SEEK_SET);
  if (f16) {
    std::vector<uint16_t> buf(static_cast<size_t>(n));
    if (std::fread(buf.data(), 2, buf.size(), in.f) != buf.size()) return io_fail("tensor file truncated");
    for (int64_t i = 0; i < n; ++i) data[i] = fmha_host_16_to_f32(buf[i], 0);
  } else if (std::fread(data, 4, static_cast<size_t>(n), in.f) != static_cast<size_t>(n)) {
    return io_fail("tensor file truncated");
  }
  return FMHA_OK;
}

}  // extern "C"

namespace fmha_b200 {

void save_tensor(const Tensor4& t, const std::string& path, const std::string& precision) {
  if (precision != "f32" && precision != "f16")
    throw std::invalid_argument("save_tensor: unknown precision " + precision);
  if (fmha_tensor_save(path.c_str(), t.data.data(), t.L, t.N, t.h, t.d, precision == "f16") != FMHA_OK)
    throw std::runtime_error(g_last_error);
}

Tensor4 load_tensor(const std::string& path) {
  int64_t dims[4];
  int f16 = 0;
  if (fmha_tensor_load_header(path.c_str(), dims, &f16) != FMHA_OK) throw std::runtime_error(g_last_error);
  Tensor4 t(dims[0], dims[1], dims[2], dims[3]);
  if (fmha_tensor_load(path.c_str(), t.data.data(), t.elements()) != FMHA_OK)
    throw std::runtime_error(g_last_error);
  return t;
}

}  // namespace fmha_b200
