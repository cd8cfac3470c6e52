/*
 * pact_cuda.h — C-ABI of the B200 (sm_100a) implementation of the NF-APACT
 * hot path.  This is the drop-in boundary: the reference library `pact`
 * (/root/reference/proj/include/pact/ headers) is header-only C++; its hot entry
 * points are re-exported here as plain `extern "C"` functions over POD structs,
 * raw pointers and sizes.  The C++ host API in
 * paper_2409_10876_b200/include/pact/ (same names/types as the reference)
 * is a thin layer over these calls, and so is the Python ctypes binding.
 *
 * Conventions
 *  - Every compute entry point works on DEVICE pointers (cudaMalloc'd, or
 *    torch CUDA tensors) and is asynchronous on the context's stream.  Host
 *    staging is done with pact_upload/pact_download (pinned or pageable).
 *  - Return value: PACT_OK (0), PACT_E_VALIDATION (2, the reference's
 *    ValidationError, CLI exit 2), PACT_E_NUMERICAL (3, NumericalError,
 *    CLI exit 3), PACT_E_CUDA (4, a CUDA runtime error), PACT_E_UNSUPPORTED (5).
 *    The message is available from pact_last_error() (thread-local).
 *  - Arithmetic on device is fp32 (fp64 where the reference's index math needs
 *    it); geometry scalars cross the boundary as double like the reference.
 *  - The reference's `workers` argument has no meaning here; it is accepted
 *    by the C++ layer and ignored.
 */
#ifndef PACT_CUDA_H
#define PACT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PACT_OK 0
#define PACT_E_VALIDATION 2
#define PACT_E_NUMERICAL 3
#define PACT_E_CUDA 4
#define PACT_E_UNSUPPORTED 5

#define PACT_ABI_VERSION 1

/* ---- geometry PODs (field meaning identical to the reference types) ---- */

/* RingGeometry, core.hpp:152-173: transducer n at angle 2*pi*n/N + angle_offset. */
typedef struct pact_ring {
  int32_t n_transducers;
  double radius;       /* mm */
  double angle_offset; /* rad */
} pact_ring;

/* GridSpec, core.hpp:58-89: pixel (0,0) centre at origin; row-major rasters. */
typedef struct pact_grid {
  int32_t width;
  int32_t height;
  double pitch;    /* mm */
  double origin_x; /* mm */
  double origin_y; /* mm */
} pact_grid;

/* SignalSet metadata, core.hpp:284-313 (the data is a separate N x T array). */
typedef struct pact_signal_meta {
  int32_t n_samples;
  double dt;             /* s */
  double t0;             /* s */
  double background_sos; /* m/s */
} pact_signal_meta;

/* CircularMask, core.hpp:175-180. */
typedef struct pact_mask {
  double center_x;
  double center_y;
  double radius; /* mm */
} pact_mask;

/* PatchLayout, core.hpp:222-281 (offsets are regenerated from nx/ny/stride). */
typedef struct pact_layout {
  pact_grid grid;
  int32_t patch_pixels;
  int32_t stride_pixels;
  int32_t nx;
  int32_t ny;
  int32_t last_x; /* clamped last offset along x (= width - P, or 0) */
  int32_t last_y;
} pact_layout;

/* ---- context, errors, memory ---- */

typedef struct pact_ctx pact_ctx;

int pact_abi_version(void);
const char* pact_last_error(void);

/* Creates a context on `device` with its own non-blocking stream. */
int pact_ctx_create(int device, pact_ctx** out);
int pact_ctx_destroy(pact_ctx* ctx);
/* Returns the cudaStream_t the context launches on (as void*). */
void* pact_ctx_stream(pact_ctx* ctx);
/* Makes the context launch on a caller-owned stream.  NULL is the legacy
 * default stream (e.g. torch's default stream); pact_ctx_use_own_stream
 * switches back to the context's private non-blocking stream. */
int pact_ctx_set_stream(pact_ctx* ctx, void* stream);
int pact_ctx_use_own_stream(pact_ctx* ctx);
int pact_ctx_synchronize(pact_ctx* ctx);
/* Number of kernels this library launched on the context so far. */
int64_t pact_ctx_launch_count(pact_ctx* ctx);

int pact_device_alloc(pact_ctx* ctx, size_t bytes, void** out);
int pact_device_free(pact_ctx* ctx, void* ptr);
int pact_host_alloc_pinned(size_t bytes, void** out);
int pact_host_free_pinned(void* ptr);
int pact_upload(pact_ctx* ctx, void* dst_device, const void* src_host, size_t bytes);
int pact_download(pact_ctx* ctx, void* dst_host, const void* src_device, size_t bytes);
int pact_memset(pact_ctx* ctx, void* dst_device, int value, size_t bytes);

/* ---- part 1: delay-and-sum stack ---- */

/* make_delays, beamform.hpp:113-120: `count` evenly spaced delays in [lo, hi]. */
int pact_make_delays(double lo, double hi, int32_t count, double* out);

/* das_stack, beamform.hpp:77-110 (and das, beamform.hpp:56-75, as K = 1).
 *   signals : device fp32 [n_transducers][n_samples] (SignalSet::data layout)
 *   delays  : HOST double[K], strictly increasing (mm)
 *   out     : device fp32 [K][grid.height][grid.width]
 * y_j(r) = sum_n S_n((|r - r_n| - d_j)/v0) with SignalSet::sample semantics
 * (linear interpolation, zero outside [0, n_samples-1], core.hpp:296-304). */
int pact_das_stack(pact_ctx* ctx, const pact_ring* ring, const pact_signal_meta* meta,
                   const float* signals, const pact_grid* grid, double v0,
                   const double* delays, int32_t n_delays, float* out);

#ifdef __cplusplus
}
#endif

#endif /* PACT_CUDA_H */
