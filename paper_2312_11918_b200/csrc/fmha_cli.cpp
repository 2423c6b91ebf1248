// fmha_cli.cpp -- `fmha-b200`, the GPU counterpart of the reference CLI
// `fmha-sim` (/root/reference/proj/tools/fmha_cli.cpp).  Same flag names and
// exit codes (0 ok, 2 config error, 3 verification failure; 5 is new: CUDA
// failure):
//
//   fmha-b200 verify [--seqlen N] [--headdim d] [--heads h] [--batch L]
//                    [--tile-q bM] [--tile-k bN] [--precision f16emu|bf16]
//                    [--seed S] [--iterations I] [--format text|csv|json]
//                    [--out FILE] [--device D] [--load-prefix P] [--dump-prefix P]
//   fmha-b200 sweep  [--precision ...] [--iterations I] [--format ...] [--out FILE]
//
// verify (fmha_cli.cpp:105-145): seeded Gaussian Q/K/V (seeds S, S+1, S+2,
// fmha_cli.cpp:79-84 -- std::mt19937_64 + Box-Muller, so the inputs are the
// reference's own fixtures bit for bit), rounded to the 16-bit type, run on
// the tensor-core kernel, checked against the independent fp32 CUDA-core
// attention (fmha_fwd_reference, the standard_attention semantics) with the
// north-star tolerance (O max abs <= 1e-2, mean abs <= 1e-3, LSE rel <= 1e-4)
// and the reference's own metric |a-b|/max(|b|,1) reported beside it.
// --load-prefix P reads P_q.fhmt / P_k.fhmt / P_v.fhmt instead; --dump-prefix
// writes the inputs and P_o.fhmt (FHMT, tensor.cpp:30-84).
// sweep reproduces the paper's Table-1 shapes (L=4, N=4096, (d,h) in
// {(64,32),(128,16),(256,8)}) and reports TFLOP/s.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/fmha/fmha.h"
#include "../../include/fmha/fmha.hpp"

extern "C" uint16_t fmha_host_f32_to_16(float x, int bf16);
extern "C" float fmha_host_16_to_f32(uint16_t x, int bf16);

namespace {

constexpr int kExitOk = 0;
constexpr int kExitConfig = 2;
constexpr int kExitVerify = 3;
constexpr int kExitCuda = 5;

struct Options {
  std::string cmd;
  int64_t N = 256, d = 64, h = 2, L = 1, bM = 64, bN = 64;
  std::string precision = "f16emu";
  uint64_t seed = 42;
  int iterations = 1;
  std::string format = "text";
  std::string out, load_prefix, dump_prefix;
  int device = 0;
};

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

void usage() {
  std::fprintf(stderr,
               "usage: fmha-b200 <verify|sweep> [--seqlen N] [--headdim d] [--heads h] [--batch L]\n"
               "                 [--tile-q bM] [--tile-k bN] [--precision f16emu|bf16] [--seed S]\n"
               "                 [--iterations I] [--format text|csv|json] [--out FILE] [--device D]\n"
               "                 [--load-prefix P] [--dump-prefix P]\n");
}

Options parse(int argc, char** argv) {
  if (argc < 2) throw ConfigError("missing subcommand");
  Options o;
  o.cmd = argv[1];
  if (o.cmd != "verify" && o.cmd != "sweep") throw ConfigError("unknown subcommand " + o.cmd);
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) throw ConfigError(a + " needs a value");
      return argv[++i];
    };
    auto num = [&]() -> int64_t {
      const std::string v = val();
      char* end = nullptr;
      const long long x = std::strtoll(v.c_str(), &end, 10);
      if (end == v.c_str() || *end != '\0') throw ConfigError(a + ": not an integer: " + v);
      return x;
    };
    if (a == "--seqlen") o.N = num();
    else if (a == "--headdim") o.d = num();
    else if (a == "--heads") o.h = num();
    else if (a == "--batch") o.L = num();
    else if (a == "--tile-q") o.bM = num();
    else if (a == "--tile-k") o.bN = num();
    else if (a == "--seed") o.seed = static_cast<uint64_t>(num());
    else if (a == "--iterations") o.iterations = static_cast<int>(num());
    else if (a == "--device") o.device = static_cast<int>(num());
    else if (a == "--precision") o.precision = val();
    else if (a == "--format") o.format = val();
    else if (a == "--out") o.out = val();
    else if (a == "--load-prefix") o.load_prefix = val();
    else if (a == "--dump-prefix") o.dump_prefix = val();
    else throw ConfigError("unknown flag " + a);
  }
  if (o.precision != "f16emu" && o.precision != "f16" && o.precision != "bf16")
    throw ConfigError("--precision must be f16emu or bf16 (the GPU path is 16-bit)");
  if (o.format != "text" && o.format != "csv" && o.format != "json")
    throw ConfigError("--format must be text, csv or json");
  if (o.iterations < 1) throw ConfigError("--iterations must be >= 1");
  if (o.N < 1 || o.d < 1 || o.h < 1 || o.L < 1)
    throw ConfigError("AttentionProblem: need N >= 1 and d >= 1");
  // validate_tiling, attention.cpp:21-27 (same inputs rejected)
  if (o.bM < 1 || o.bN < 1 || o.N % o.bM != 0 || o.N % o.bN != 0)
    throw ConfigError("TileConfig: N = " + std::to_string(o.N) + " must be divisible by bM = " +
                      std::to_string(o.bM) + " and bN = " + std::to_string(o.bN));
  if (o.d != 64 && o.d != 128 && o.d != 256)
    throw ConfigError("head dim " + std::to_string(o.d) + " unsupported by the sm_100a kernel (64, 128, 256)");
  return o;
}

// Seeded standard normals in storage order: std::mt19937_64, 53-bit uniforms
// and the Box-Muller pair (cos first, sin kept), as the reference's
// GaussianSource (random.hpp:14-42) so fixtures match for the same seed.
void gaussian_fill(std::vector<float>& out, uint64_t seed) {
  std::mt19937_64 rng(seed);
  auto uni = [&]() { return static_cast<double>(rng() >> 11) * (1.0 / 9007199254740992.0); };
  bool have = false;
  float spare = 0.f;
  for (auto& x : out) {
    if (have) {
      x = spare;
      have = false;
      continue;
    }
    double u1;
    do {
      u1 = uni();
    } while (u1 <= 0.0);
    const double u2 = uni();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double th = 2.0 * M_PI * u2;
    spare = static_cast<float>(r * std::sin(th));
    have = true;
    x = static_cast<float>(r * std::cos(th));
  }
}

void emit(const Options& o, const std::string& text) {
  if (o.out.empty()) {
    std::cout << text;
    return;
  }
  std::ofstream os(o.out);
  if (!os) throw std::runtime_error("cannot open output file " + o.out);
  os << text;
}

struct Result {
  double ms = 0, tflops = 0;
  double max_rel = 0, max_abs = 0, mean_abs = 0, lse_rel = 0;
  bool pass = true;
  int64_t worst = 0;
};

// Runs the kernel `iters` times on device-resident inputs (first call
// warms up), optionally checks it against fmha_fwd_reference.
Result run_case(const Options& o, int64_t L, int64_t N, int64_t h, int64_t d, bool check,
                const std::vector<float>* qf, const std::vector<float>* kf,
                const std::vector<float>* vf, std::vector<float>* o_out) {
  const bool bf = o.precision == "bf16";
  const int64_t n = L * N * h * d;
  std::vector<float> q(n), k(n), v(n);
  if (qf) {
    q = *qf;
    k = *kf;
    v = *vf;
  } else {
    gaussian_fill(q, o.seed);
    gaussian_fill(k, o.seed + 1);
    gaussian_fill(v, o.seed + 2);
  }
  std::vector<uint16_t> hq(n), hk(n), hv(n);
  for (int64_t i = 0; i < n; ++i) {
    hq[i] = fmha_host_f32_to_16(q[i], bf);
    hk[i] = fmha_host_f32_to_16(k[i], bf);
    hv[i] = fmha_host_f32_to_16(v[i], bf);
  }
  fmha_fwd_params p;
  fmha_params_dense(&p, L, N, h, d, bf ? FMHA_BF16 : FMHA_F16, 0.0f);
  void *dq, *dk, *dv, *dO;
  float *dl, *dref, *dlref;
  cuda_check(cudaSetDevice(o.device), "cudaSetDevice");
  cuda_check(cudaMalloc(&dq, n * 2), "cudaMalloc");
  cuda_check(cudaMalloc(&dk, n * 2), "cudaMalloc");
  cuda_check(cudaMalloc(&dv, n * 2), "cudaMalloc");
  cuda_check(cudaMalloc(&dO, n * 2), "cudaMalloc");
  cuda_check(cudaMalloc(&dl, L * h * N * 4), "cudaMalloc");
  cuda_check(cudaMemcpy(dq, hq.data(), n * 2, cudaMemcpyHostToDevice), "H2D");
  cuda_check(cudaMemcpy(dk, hk.data(), n * 2, cudaMemcpyHostToDevice), "H2D");
  cuda_check(cudaMemcpy(dv, hv.data(), n * 2, cudaMemcpyHostToDevice), "H2D");
  auto launch = [&]() {
    if (fmha_fwd(&p, dq, dk, dv, dO, dl, nullptr) != FMHA_OK) throw CudaError(fmha_last_error());
  };
  launch();  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int it = 0; it < o.iterations; ++it) launch();
  cudaEventRecord(e1);
  cuda_check(cudaEventSynchronize(e1), "kernel execution");
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  Result r;
  r.ms = ms / o.iterations;
  r.tflops = static_cast<double>(fmha_attention_flops(L, N, h, d)) / (r.ms * 1e-3) / 1e12;
  std::vector<uint16_t> ho(n);
  std::vector<float> lse(L * h * N);
  cuda_check(cudaMemcpy(ho.data(), dO, n * 2, cudaMemcpyDeviceToHost), "D2H");
  cuda_check(cudaMemcpy(lse.data(), dl, lse.size() * 4, cudaMemcpyDeviceToHost), "D2H");
  if (o_out) {
    o_out->resize(n);
    for (int64_t i = 0; i < n; ++i) (*o_out)[i] = fmha_host_16_to_f32(ho[i], bf);
  }
  if (check) {
    cuda_check(cudaMalloc(&dref, n * 4), "cudaMalloc");
    cuda_check(cudaMalloc(&dlref, L * h * N * 4), "cudaMalloc");
    if (fmha_fwd_reference(&p, dq, dk, dv, dref, dlref, nullptr) != FMHA_OK)
      throw CudaError(fmha_last_error());
    std::vector<float> ref(n), lref(L * h * N);
    cuda_check(cudaMemcpy(ref.data(), dref, n * 4, cudaMemcpyDeviceToHost), "D2H");
    cuda_check(cudaMemcpy(lref.data(), dlref, lref.size() * 4, cudaMemcpyDeviceToHost), "D2H");
    double sum = 0;
    for (int64_t i = 0; i < n; ++i) {
      const double got = fmha_host_16_to_f32(ho[i], bf), want = ref[i];
      const double ad = std::abs(got - want);
      const double rel = ad / std::max(std::abs(want), 1.0);  // fmha_cli.cpp:63-77 metric
      if (!(ad <= r.max_abs)) {
        r.max_abs = ad;
        r.worst = i;
      }
      r.max_rel = std::max(r.max_rel, rel);
      sum += ad;
    }
    r.mean_abs = sum / n;
    for (size_t i = 0; i < lref.size(); ++i)
      r.lse_rel = std::max(r.lse_rel, std::abs(static_cast<double>(lse[i]) - lref[i]) / std::abs(lref[i]));
    r.pass = r.max_abs <= 1e-2 && r.mean_abs <= 1e-3 && r.lse_rel <= 1e-4;
    cudaFree(dref);
    cudaFree(dlref);
  }
  cudaFree(dq);
  cudaFree(dk);
  cudaFree(dv);
  cudaFree(dO);
  cudaFree(dl);
  return r;
}

std::string config_name(const Options& o, int64_t L, int64_t N, int64_t h, int64_t d) {
  std::ostringstream os;
  os << "L=" << L << ",N=" << N << ",h=" << h << ",d=" << d << "," << (o.precision == "bf16" ? "bf16" : "fp16");
  return os.str();
}

int cmd_verify(const Options& o) {
  std::vector<float> q, k, v;
  int64_t L = o.L, N = o.N, h = o.h, d = o.d;
  const bool loaded = !o.load_prefix.empty();
  if (loaded) {
    fmha_b200::Tensor4 tq = fmha_b200::load_tensor(o.load_prefix + "_q.fhmt");
    fmha_b200::Tensor4 tk = fmha_b200::load_tensor(o.load_prefix + "_k.fhmt");
    fmha_b200::Tensor4 tv = fmha_b200::load_tensor(o.load_prefix + "_v.fhmt");
    fmha_b200::AttentionProblem prob(tq, tk, tv);  // shape checks (attention.cpp:13-17)
    L = tq.L, N = tq.N, h = tq.h, d = tq.d;
    fmha_b200::validate_tiling(prob, fmha_b200::TileConfig{o.bM, o.bN});
    q = std::move(tq.data);
    k = std::move(tk.data);
    v = std::move(tv.data);
  }
  std::vector<float> out;
  Result r = run_case(o, L, N, h, d, true, loaded ? &q : nullptr, loaded ? &k : nullptr,
                      loaded ? &v : nullptr, o.dump_prefix.empty() ? nullptr : &out);
  if (!o.dump_prefix.empty()) {
    if (!loaded) {
      q.resize(L * N * h * d);
      k.resize(q.size());
      v.resize(q.size());
      gaussian_fill(q, o.seed);
      gaussian_fill(k, o.seed + 1);
      gaussian_fill(v, o.seed + 2);
    }
    const int f16 = o.precision == "bf16" ? 0 : 1;
    fmha_tensor_save((o.dump_prefix + "_q.fhmt").c_str(), q.data(), L, N, h, d, f16);
    fmha_tensor_save((o.dump_prefix + "_k.fhmt").c_str(), k.data(), L, N, h, d, f16);
    fmha_tensor_save((o.dump_prefix + "_v.fhmt").c_str(), v.data(), L, N, h, d, f16);
    fmha_tensor_save((o.dump_prefix + "_o.fhmt").c_str(), out.data(), L, N, h, d, 0);
  }
  const std::string cfg = config_name(o, L, N, h, d);
  std::ostringstream os;
  char buf[512];
  if (o.format == "csv") {
    os << "config,ms,tflops,max_rel_error,max_abs_error,mean_abs_error,lse_rel_error,pass\n";
    std::snprintf(buf, sizeof(buf), "\"%s\",%.6f,%.3f,%.6g,%.6g,%.6g,%.6g,%d\n", cfg.c_str(), r.ms, r.tflops,
                  r.max_rel, r.max_abs, r.mean_abs, r.lse_rel, r.pass ? 1 : 0);
    os << buf;
  } else if (o.format == "json") {
    std::snprintf(buf, sizeof(buf),
                  "{\"config\": \"%s\", \"ms\": %.6f, \"tflops\": %.3f, \"max_rel_error\": %.6g, "
                  "\"max_abs_error\": %.6g, \"mean_abs_error\": %.6g, \"lse_rel_error\": %.6g, \"pass\": %s}\n",
                  cfg.c_str(), r.ms, r.tflops, r.max_rel, r.max_abs, r.mean_abs, r.lse_rel,
                  r.pass ? "true" : "false");
    os << buf;
  } else {
    os << "config: " << cfg << '\n';
    std::snprintf(buf, sizeof(buf),
                  "max relative error: %.9g (reference metric |a-b|/max(|b|,1))\n"
                  "O max abs error: %.3g (tol 1e-2)  mean abs error: %.3g (tol 1e-3)  LSE rel error: %.3g "
                  "(tol 1e-4)\n"
                  "timing: %.4f ms/iteration over %d iterations, %.1f TFLOP/s\n",
                  r.max_rel, r.max_abs, r.mean_abs, r.lse_rel, r.ms, o.iterations, r.tflops);
    os << buf << (r.pass ? "PASS" : "FAIL") << '\n';
  }
  emit(o, os.str());
  if (!r.pass) {
    std::cerr << "verification failed (worst element " << r.worst << ")\n";
    return kExitVerify;
  }
  return kExitOk;
}

int cmd_sweep(const Options& o) {
  struct Shape {
    int64_t d, h;
  };
  const Shape shapes[] = {{64, 32}, {128, 16}, {256, 8}};
  std::ostringstream os;
  if (o.format == "csv") os << "config,ms,tflops\n";
  if (o.format == "json") os << "[";
  bool first = true;
  for (const auto& s : shapes) {
    const int64_t L = 4, N = 4096;
    Options oo = o;
    oo.iterations = std::max(o.iterations, 20);
    Result r = run_case(oo, L, N, s.h, s.d, false, nullptr, nullptr, nullptr, nullptr);
    const std::string cfg = config_name(o, L, N, s.h, s.d);
    char buf[256];
    if (o.format == "csv") {
      std::snprintf(buf, sizeof(buf), "\"%s\",%.6f,%.3f\n", cfg.c_str(), r.ms, r.tflops);
    } else if (o.format == "json") {
      std::snprintf(buf, sizeof(buf), "%s{\"config\": \"%s\", \"ms\": %.6f, \"tflops\": %.3f}", first ? "" : ", ",
                    cfg.c_str(), r.ms, r.tflops);
    } else {
      std::snprintf(buf, sizeof(buf), "%-32s %9.4f ms  %8.1f TFLOP/s\n", cfg.c_str(), r.ms, r.tflops);
    }
    os << buf;
    first = false;
  }
  if (o.format == "json") os << "]\n";
  emit(o, os.str());
  return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
  Options o;
  try {
    o = parse(argc, argv);
  } catch (const ConfigError& e) {
    std::cerr << "error: " << e.what() << '\n';
    usage();
    return kExitConfig;
  }
  try {
    return o.cmd == "verify" ? cmd_verify(o) : cmd_sweep(o);
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kExitConfig;
  } catch (const CudaError& e) {
    std::cerr << "CUDA error: " << e.what() << '\n';
    return kExitCuda;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kExitConfig;
  }
}
