/*
 * fmha.h -- C ABI of the B200-native (sm_100a) fused multi-head attention
 * forward pass.  This is the drop-in boundary for the reference's C++ FMHA
 * entry point
 *
 *     Tensor4 fmhasim::fmha_forward(const AttentionProblem&, const TileConfig&,
 *                                   Precision)
 *         /root/reference/proj/include/fmhasim/attention.hpp:58-59
 *         /root/reference/proj/src/attention.cpp:153-173
 *
 * and for the pybind entry `_fmhasim.fmha_forward(q, k, v, bM, bN, precision)`
 * (/root/reference/proj/src/bindings.cpp:81-91).  The C++ adapter in
 * include/fmha/fmha.hpp keeps the reference's call shape on top of this ABI.
 *
 * No C++ or torch types cross this boundary: plain pointers, sizes, strides.
 *
 * Layout (same as the reference's Tensor4, tensor.hpp:12-22): Q, K, V, O are
 * BSHD -- element (b, n, head, k) at  b*stride[0] + n*stride[1] + head*stride[2] + k
 * (strides in ELEMENTS, head-dim stride 1).  The reference's dense Tensor4 is
 * stride = {N*h*d, h*d, d}.  LSE is fp32 [L][h][N] (the reference keeps
 * rowMaxNew/rowSum in SoftmaxState, attention.cpp:29-34, and discards them;
 * lse = rowMaxNew + ln(rowSum) in scaled-score units, natural log).
 *
 * Numerics: 16-bit inputs (fp16 or bf16), fp32 accumulation in Tensor Memory,
 * P rounded to the input type before GEMM-II (as the reference's F16Emu mode
 * rounds it inside gemm_nt_accumulate, attention.cpp:82), row sums over the
 * unrounded fp32 P (attention.cpp:50-55), O = O_acc * (1/Sigma)
 * (attention.cpp:68-73), O stored in the input type.
 *
 * Errors (no CPU fallback exists):
 *   FMHA_ERR_CONFIG      -- what the reference rejects with
 *                           std::invalid_argument (N < 1, d < 1,
 *                           attention.cpp:16-17) and malformed arguments
 *                           (null pointers, misaligned strides).
 *   FMHA_ERR_UNSUPPORTED -- valid for the reference but not for this kernel
 *                           (head dim not in {64, 128, 256}).
 *   FMHA_ERR_CUDA        -- a CUDA runtime / driver failure.
 * fmha_last_error() returns a thread-local message for the last failure.
 */
#ifndef FMHA_B200_FMHA_H_
#define FMHA_B200_FMHA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FMHA_OK = 0,
  FMHA_ERR_CONFIG = 2,      /* same code as the reference CLI's config exit (fmha_cli.cpp:19-22) */
  FMHA_ERR_CUDA = 5,
  FMHA_ERR_UNSUPPORTED = 6
} fmha_status;

typedef enum { FMHA_F16 = 0, FMHA_BF16 = 1 } fmha_dtype;

typedef struct {
  int64_t L, N, h, d;     /* batch, sequence length, heads, head dim             */
  int64_t q_stride[3];    /* (b, n, head) strides in elements; head-dim stride 1  */
  int64_t k_stride[3];
  int64_t v_stride[3];
  int64_t o_stride[3];
  float scale;            /* softmax scale; <= 0 selects the reference default
                             float(1/sqrt(double(d))) (attention.cpp:18)        */
  fmha_dtype dtype;       /* fp16 or bf16 for Q, K, V and O                      */
} fmha_fwd_params;

/* Fill `p` for dense BSHD tensors (the reference Tensor4 layout). */
void fmha_params_dense(fmha_fwd_params* p, int64_t L, int64_t N, int64_t h, int64_t d,
                       fmha_dtype dtype, float scale);

/* Check a parameter block without launching (FMHA_OK when launchable). */
fmha_status fmha_fwd_check(const fmha_fwd_params* p);

/*
 * Device entry point.  q, k, v, o: device pointers (16-B aligned);
 * lse: device pointer to L*h*N floats or NULL; cuda_stream: cudaStream_t or
 * NULL for the legacy default stream.  Asynchronous; allocates nothing.
 * Replaces the arithmetic of fmhasim::fmha_forward (attention.cpp:153-173).
 */
fmha_status fmha_fwd(const fmha_fwd_params* p, const void* q, const void* k, const void* v,
                     void* o, float* lse, void* cuda_stream);

/*
 * Host entry point (the reference-facing call: host buffers in, host buffers
 * out, like fmhasim::fmha_forward returning a Tensor4 by value).  q, k, v, o
 * are HOST pointers to 16-bit BSHD data in the dtype of `p` (pinned memory
 * is fastest); lse is a host pointer or NULL.  Copies in, runs, copies back,
 * synchronises.  Uses a per-device cached workspace.
 */
fmha_status fmha_fwd_host(const fmha_fwd_params* p, const void* q, const void* k, const void* v,
                          void* o, float* lse, int device);

/*
 * Host entry point over float32 BSHD buffers with the reference's tiling
 * contract: bM, bN must divide N (validate_tiling, attention.cpp:21-27) even
 * though the kernel picks its own tile shape.  Inputs are rounded RNE to
 * `dtype` (fp16 rounding saturates like the reference's f16_round,
 * half.hpp:12-42); O is returned as float32.  This is what the C++ adapter
 * fmha_b200::fmha_forward and the Python `fmha_forward` call.
 */
fmha_status fmha_forward_f32(const float* q, const float* k, const float* v, int64_t L, int64_t N,
                             int64_t h, int64_t d, int64_t bM, int64_t bN, fmha_dtype dtype,
                             float scale, float* o, float* lse, int device);

/*
 * Verification path (NOT the hot path): an independent fp32 CUDA-core
 * attention with the reference's standard_attention semantics
 * (attention.cpp:137-151; exact expf, unrounded P).  q, k, v: 16-bit device
 * tensors described by `p`; o: dense fp32 [L][N][h][d] device buffer; lse:
 * [L][h][N] or NULL.  Used by the `fmha-b200 verify` CLI as its checker.
 */
fmha_status fmha_fwd_reference(const fmha_fwd_params* p, const void* q, const void* k,
                               const void* v, float* o, float* lse, void* cuda_stream);

/*
 * FHMT fixture files -- the reference's save_tensor / load_tensor format
 * (tensor.hpp:36-38, tensor.cpp:30-84): magic "FHMT", version 1, int64
 * L, N, h, d, precision tag (0 f32, 1 f16), values in (b, n, head, k) order.
 */
fmha_status fmha_tensor_save(const char* path, const float* data, int64_t L, int64_t N, int64_t h,
                             int64_t d, int f16);
fmha_status fmha_tensor_load_header(const char* path, int64_t dims[4], int* f16);
fmha_status fmha_tensor_load(const char* path, float* data, int64_t count);

/* Host quantisers used by fmha_forward_f32 (threaded; F16C when the CPU has it):
 * float -> fp16 with the reference's semantics (half.hpp:12-42: round to nearest
 * even, finite overflow saturates to +-65504, subnormals kept) or -> bf16 (RNE),
 * and back.  Bit-identical to an element-wise loop. */
void fmha_host_quantize(const float* src, uint16_t* dst, int64_t n, fmha_dtype dtype);
void fmha_host_dequantize(const uint16_t* src, float* dst, int64_t n, fmha_dtype dtype);

/* 4 * N^2 * d * h * L (attention_flops, attention.cpp:191-193). */
int64_t fmha_attention_flops(int64_t L, int64_t N, int64_t h, int64_t d);

/* Name of the kernel fmha_fwd would launch for this problem (host-only, no
 * CUDA call; NULL when fmha_fwd_check rejects the parameters).  The choice
 * depends on d and N (and on FMHA_TUNE_* environment overrides). */
const char* fmha_kernel_for(const fmha_fwd_params* p);

/* Number of kernel launches the last fmha_fwd call on this thread issued. */
int fmha_last_launch_count(void);

/* Thread-local description of the last error ("" when none). */
const char* fmha_last_error(void);

/* Library version string. */
const char* fmha_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FMHA_B200_FMHA_H_ */
