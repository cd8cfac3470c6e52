// The NF-APACT iteration engine: joint_reconstruct (optimize.hpp:367-494) on
// one B200.
//
// One-time (optimize.hpp:369-405): patch layout, DAS stack, fp32 patch
// spectra (the reference also caches them as complex<float>), SIREN init,
// Fourier tables.  Each iteration (optimize.hpp:412-471) is one sequence on
// the engine's stream, captured once as a CUDA graph:
//   siren_forward -> finite(SOS) -> wavefront -> fused loss/dL/dw ->
//   ray backward (dL/dv) -> TV -> report -> siren_backward -> finite(grad) ->
//   Adam (fp64 master parameters, fp32 working copy)
// The host reads back only the three loss terms and the NumericalError flags
// once per reported epoch.  Results are deterministic: every reduction has a
// fixed order except the dL/dv scatter, which accumulates in fp64.
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "geom.cuh"
#include "nccl_api.cuh"
#include "siren.cuh"
#include "train_ops.cuh"

namespace {
// PACT_TRACE=1: host-side phase timings of trainer creation on stderr.
struct HostTrace {
  bool on = std::getenv("PACT_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[pact] %-28s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};
}  // namespace

namespace pactgpu {
Status merge_window(double fwhm, int P, double pitch, std::vector<float>& w);
Status launch_sos_from_dev(pact_ctx* ctx, const float* dv, size_t n, double v0, float* out);
}  // namespace pactgpu

using namespace pactgpu;

struct pact_trainer {
  pact_ctx* user = nullptr;  // caller's context (its stream orders inputs/outputs)
  pact_ctx eng;              // engine context: private stream
  pact_ring ring{};
  pact_signal_meta meta{};
  pact_grid grid{};
  pact_mask mask{};
  pact_train_config cfg{};
  std::vector<double> delays;
  double v0 = 0.0;
  pact_layout lay{};
  int n_patches = 0, P = 0, K = 0, A = 0, n_params = 0;
  // partition: this rank owns patches [p_lo, p_hi) (whole
  // patch rows) and masked pixels [m_lo, m_hi) of the row-major list; the
  // caller all-reduces dv, dL/dv, the report and the gradient between phases
  int rank = 0, world = 1, p_lo = 0, p_hi = 0, n_local = 0, m_lo = 0, m_hi = 0;
  int row0 = 0, rows = 0;  // the stack's row band [row0, row0 + rows) of the grid
  float* num = nullptr;  // merge accumulators of the final image (world > 1)
  float* den = nullptr;
  double loss_scale = 0.0;
  SirenShape shape;
  MaskedPixels mp;
  SirenWork sw;
  FourierTable ftab;
  RayArgs ray{};
  RayPlan ray_plan;
  int n_tv = 0;
  // device state
  void* arena = nullptr;
  float* stack = nullptr;
  float2* Y = nullptr;
  float* dv = nullptr;
  float* w = nullptr;
  float* dw = nullptr;
  double* loss_patch = nullptr;
  double* gv = nullptr;
  float* gtv = nullptr;
  double* tv_partial = nullptr;
  unsigned char* inmask = nullptr;
  double* theta = nullptr;
  double* m = nullptr;
  double* v = nullptr;
  float* theta32 = nullptr;
  double* grad = nullptr;
  unsigned* flags = nullptr;
  double* report = nullptr;
  long long* t = nullptr;
  double2* centers = nullptr;
  float* win = nullptr;
  cudaGraphExec_t graph = nullptr;
  int64_t graph_kernels = 0;
  int steps_done = 0;
  // pact_trainer_step_nccl: the collectives' stream and its two ordering events
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_eng = nullptr, ev_comm = nullptr;
};

namespace {

// The iteration in four phases; a partitioned trainer (world > 1) runs them
// one at a time with the caller's all-reduces in between:
//   0 render    -> all-reduce dv (SUM; each pixel has one owner)
//   1 rays/loss -> all-reduce dL/dv (SUM), report[0..3) (SUM), flags (MAX)
//     (= 6 wavefronts, loss, ray adjoint -> the dL/dv collective can start,
//      then 7 TV + report, which overlaps it)
//   2 SIREN bwd -> all-reduce the gradient (SUM)
//   3 Adam (replicated)
Status enqueue_phase(pact_trainer* tr, int phase) {
  pact_ctx* ctx = &tr->eng;
  const size_t npx = static_cast<size_t>(tr->grid.width) * tr->grid.height;
  switch (phase) {
    case 0:
      // render_sos (optimize.hpp:413) + finiteness (414-417)
      if (tr->world > 1)  // foreign pixels stay 0 for the all-reduce
        PACT_CUDA_S(cudaMemsetAsync(tr->dv, 0, sizeof(float) * npx, ctx->stream));
      PACT_TRY_S(siren_forward(ctx, tr->shape, tr->theta32, tr->sw, tr->dv));
      PACT_TRY_S(launch_check_finite_f32(ctx, tr->dv, tr->sw.idx, tr->mp.n, kFlagSos, tr->flags));
      return {};
    case 1:
      PACT_TRY_S(enqueue_phase(tr, 6));
      return enqueue_phase(tr, 7);
    case 6:
      // wavefront_profile for every (local) patch (431-433)
      PACT_TRY_S(launch_wavefront(ctx, tr->ray, tr->w));
      // fused_patch_loss_grad (434-436)
      PACT_TRY_S(launch_loss_grad(ctx, tr->ftab.tab, tr->Y, tr->w, tr->n_local,
                                  tr->cfg.eps_deconv, tr->loss_scale,
                                  tr->cfg.implicit_xhat_grad != 0, tr->loss_patch, tr->dw));
      // wavefront_grad_trace into dL/dv (437-438)
      PACT_CUDA_S(cudaMemsetAsync(tr->gv, 0, sizeof(double) * npx, ctx->stream));
      PACT_TRY_S(launch_ray_backward(ctx, tr->ray, tr->dw, tr->gv));
      return {};
    case 7:
      // tv_loss (448) and the loss report / checks (442-451)
      PACT_TRY_S(launch_tv(ctx, tr->dv, tr->inmask, tr->sw.idx, tr->mp.n, tr->grid.width,
                           tr->grid.height, tr->cfg.lambda_tv, tr->gtv, tr->tv_partial, tr->n_tv));
      PACT_TRY_S(launch_step_report(ctx, tr->loss_patch, tr->n_local, tr->tv_partial, tr->n_tv,
                                    tr->cfg.lambda_tv, tr->report, tr->flags));
      return {};
    case 2:
      // backprop_sos of (dL/dv at masked pixels + TV gradient) (453-461)
      return siren_backward(ctx, tr->shape, tr->theta32, tr->sw, tr->gv, tr->gtv, tr->grad);
    case 3:
      PACT_TRY_S(launch_check_finite_f64(ctx, tr->grad, tr->n_params, kFlagGrad, tr->flags));
      // adam_step (466-467)
      return launch_adam(ctx, tr->n_params, tr->theta, tr->grad, tr->m, tr->v, tr->t,
                         tr->cfg.learning_rate, tr->cfg.beta1, tr->cfg.beta2, tr->cfg.adam_eps,
                         tr->flags, tr->theta32, true);
    default:
      return validation("pact_trainer_phase: unknown phase");
  }
}

Status enqueue_step(pact_trainer* tr) {
  for (int ph = 0; ph < 4; ++ph) PACT_TRY_S(enqueue_phase(tr, ph));
  return {};
}

// One eager step with events between the stages of enqueue_step (same kernels,
// same order): render, wavefront, loss, ray backward, TV + report, SIREN
// backward, Adam.
Status profile_step(pact_trainer* tr, float* ms) {
  pact_ctx* ctx = &tr->eng;
  cudaStream_t s = ctx->stream;
  const size_t npx = static_cast<size_t>(tr->grid.width) * tr->grid.height;
  cudaEvent_t ev[8];
  for (auto& e : ev) PACT_CUDA_S(cudaEventCreate(&e));
  PACT_CUDA_S(cudaEventRecord(ev[0], s));
  PACT_TRY_S(siren_forward(ctx, tr->shape, tr->theta32, tr->sw, tr->dv));
  PACT_TRY_S(launch_check_finite_f32(ctx, tr->dv, tr->sw.idx, tr->mp.n, kFlagSos, tr->flags));
  PACT_CUDA_S(cudaEventRecord(ev[1], s));
  PACT_TRY_S(launch_wavefront(ctx, tr->ray, tr->w));
  PACT_CUDA_S(cudaEventRecord(ev[2], s));
  PACT_TRY_S(launch_loss_grad(ctx, tr->ftab.tab, tr->Y, tr->w, tr->n_local, tr->cfg.eps_deconv,
                              tr->loss_scale, tr->cfg.implicit_xhat_grad != 0, tr->loss_patch,
                              tr->dw));
  PACT_CUDA_S(cudaEventRecord(ev[3], s));
  PACT_CUDA_S(cudaMemsetAsync(tr->gv, 0, sizeof(double) * npx, s));
  PACT_TRY_S(launch_ray_backward(ctx, tr->ray, tr->dw, tr->gv));
  PACT_CUDA_S(cudaEventRecord(ev[4], s));
  PACT_TRY_S(launch_tv(ctx, tr->dv, tr->inmask, tr->sw.idx, tr->mp.n, tr->grid.width,
                       tr->grid.height, tr->cfg.lambda_tv, tr->gtv, tr->tv_partial, tr->n_tv));
  PACT_TRY_S(launch_step_report(ctx, tr->loss_patch, tr->n_local, tr->tv_partial, tr->n_tv,
                                tr->cfg.lambda_tv, tr->report, tr->flags));
  PACT_CUDA_S(cudaEventRecord(ev[5], s));
  PACT_TRY_S(siren_backward(ctx, tr->shape, tr->theta32, tr->sw, tr->gv, tr->gtv, tr->grad));
  PACT_TRY_S(launch_check_finite_f64(ctx, tr->grad, tr->n_params, kFlagGrad, tr->flags));
  PACT_CUDA_S(cudaEventRecord(ev[6], s));
  PACT_TRY_S(launch_adam(ctx, tr->n_params, tr->theta, tr->grad, tr->m, tr->v, tr->t,
                         tr->cfg.learning_rate, tr->cfg.beta1, tr->cfg.beta2, tr->cfg.adam_eps,
                         tr->flags, tr->theta32, true));
  PACT_CUDA_S(cudaEventRecord(ev[7], s));
  PACT_CUDA_S(cudaEventSynchronize(ev[7]));
  for (int i = 0; i < 7; ++i) PACT_CUDA_S(cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1]));
  for (auto& e : ev) cudaEventDestroy(e);
  return {};
}

Status capture_graph(pact_trainer* tr) {
  cudaStream_t s = tr->eng.stream;
  PACT_CUDA_S(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  int64_t before = tr->eng.launches.load();
  Status st = enqueue_step(tr);
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(s, &g);
  if (!st.ok()) {
    if (g) cudaGraphDestroy(g);
    return st;
  }
  PACT_CUDA_S(e);
  // kernels inside the graph are counted per replay, not per capture
  tr->eng.launches.store(before);
  e = cudaGraphInstantiate(&tr->graph, g, 0);
  cudaGraphDestroy(g);
  return cuda_status(e, "cudaGraphInstantiate");
}

template <typename T>
T* carve(char*& p, size_t count) {
  T* r = reinterpret_cast<T*>(p);
  p += (sizeof(T) * count + 255) & ~size_t(255);
  return r;
}

// ---- the partitioned frame over NCCL (pact_trainer_step_nccl) ------------------
struct NcclRun {
  pact_trainer* tr;
  const NcclApi* api;
  NcclComm c;
  bool slab;      // equal raster slabs: all-gather / reduce-scatter
  size_t npx, lo;  // raster pixels, this rank's slab start
  // the communication stream waits for the engine's work so far, or the reverse
  Status comm_after_engine() {
    PACT_CUDA_S(cudaEventRecord(tr->ev_eng, tr->eng.stream));
    PACT_CUDA_S(cudaStreamWaitEvent(tr->comm_stream, tr->ev_eng, 0));
    return {};
  }
  Status engine_after_comm() {
    PACT_CUDA_S(cudaEventRecord(tr->ev_comm, tr->comm_stream));
    PACT_CUDA_S(cudaStreamWaitEvent(tr->eng.stream, tr->ev_comm, 0));
    return {};
  }
  Status all_reduce(void* buf, size_t n, ncclDataType_t t, ncclRedOp_t op, const char* what) {
    return nccl_status(api->all_reduce(buf, buf, n, t, op, c.comm, tr->comm_stream), what);
  }
  // dv (f32): the rank's slab to everyone, or the all-reduce of the zeroed rasters
  Status share_dv() {
    if (!slab) return all_reduce(tr->dv, npx, ncclFloat32, ncclSum, "all-reduce dv");
    const size_t cnt = npx / c.world;
    return nccl_status(api->all_gather(tr->dv + lo, tr->dv, cnt, ncclFloat32, c.comm, tr->comm_stream),
                       "all-gather dv");
  }
  // dL/dv (f64) to the slab owners (in place), or everywhere
  Status reduce_gv() {
    if (!slab) return all_reduce(tr->gv, npx, ncclFloat64, ncclSum, "all-reduce dL/dv");
    const size_t cnt = npx / c.world;
    return nccl_status(api->reduce_scatter(tr->gv, tr->gv + lo, cnt, ncclFloat64, ncclSum, c.comm,
                                           tr->comm_stream),
                       "reduce-scatter dL/dv");
  }
};

Status nccl_run(pact_trainer* tr, NcclRun& r) {
  r.tr = tr;
  r.api = nccl_api();
  if (!r.api) return internal_error("the NCCL path needs libnccl.so.2");
  r.c = ctx_nccl(tr->user);
  if (!r.c.comm) return validation("pact_trainer_step_nccl: no NCCL communicator attached to the context");
  if (r.c.world != tr->world || r.c.rank != tr->rank)
    return validation("pact_trainer_step_nccl: the communicator's rank / world differ from the trainer's");
  if (!tr->comm_stream) {
    PACT_CUDA_S(cudaStreamCreateWithFlags(&tr->comm_stream, cudaStreamNonBlocking));
    PACT_CUDA_S(cudaEventCreateWithFlags(&tr->ev_eng, cudaEventDisableTiming));
    PACT_CUDA_S(cudaEventCreateWithFlags(&tr->ev_comm, cudaEventDisableTiming));
  }
  r.npx = static_cast<size_t>(tr->grid.width) * tr->grid.height;
  const size_t W = static_cast<size_t>(tr->world);
  r.slab = static_cast<size_t>(tr->mp.n) == r.npx && r.npx % W == 0 &&
           static_cast<size_t>(tr->m_lo) == tr->rank * r.npx / W &&
           static_cast<size_t>(tr->m_hi) == (tr->rank + 1) * r.npx / W;
  r.lo = r.slab ? static_cast<size_t>(tr->m_lo) : 0;
  return {};
}

__global__ void merge_divide_kernel(const float* __restrict__ num, const float* __restrict__ den,
                                    int n, float* __restrict__ img) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) img[i] = den[i] > 0.f ? num[i] / den[i] : 0.f;  // merge_patches (deconv.hpp:158-163)
}

}  // namespace

extern "C" {

int pact_train_config_default(pact_train_config* c) {
  // TrainConfig defaults, optimize.hpp:48-69
  static double delays[32];
  for (int j = 0; j < 32; ++j) delays[j] = -0.8 + (0.8 - -0.8) * j / 31;
  if (!c) return validation("pact_train_config_default: null").code;
  std::memset(c, 0, sizeof(*c));
  c->epochs = 10;
  c->steps_per_epoch = 30;
  c->learning_rate = 1e-3;
  c->beta1 = 0.9;
  c->beta2 = 0.999;
  c->adam_eps = 1e-8;
  c->lambda_tv = 3e9;
  c->n_delays = 32;
  c->delays = delays;
  c->eps_deconv = 1e-3;
  c->n_angles = 512;
  c->ray_step = 0.05;
  c->seed = 0;
  c->hidden = 64;
  c->sine_layers = 2;
  c->omega0 = 30.0;
  c->out_scale = 100.0;
  c->patch_mm = 3.2;
  c->overlap = 0.75;
  c->merge_fwhm = 1.5;
  c->implicit_xhat_grad = 1;
  c->workers = 0;
  c->use_cuda_graph = 1;
  return PACT_OK;
}

// sync_end: wait for the one-time device work (DAS, spectra) before returning,
// so the caller may release `signals` (the public entry points); the batch
// entry point keeps the signals alive and lets the frames' setup overlap.
static int trainer_create(pact_ctx* ctx, const pact_ring* ring, const pact_signal_meta* meta,
                          const float* signals, const pact_grid* grid, const pact_mask* mask,
                          const pact_train_config* cfg, const pact_partition* part,
                          pact_trainer** out, bool sync_end);

int pact_trainer_create_partitioned(pact_ctx* ctx, const pact_ring* ring,
                                    const pact_signal_meta* meta, const float* signals,
                                    const pact_grid* grid, const pact_mask* mask,
                                    const pact_train_config* cfg, const pact_partition* part,
                                    pact_trainer** out) {
  return trainer_create(ctx, ring, meta, signals, grid, mask, cfg, part, out, true);
}

static int trainer_create(pact_ctx* ctx, const pact_ring* ring, const pact_signal_meta* meta,
                          const float* signals, const pact_grid* grid, const pact_mask* mask,
                          const pact_train_config* cfg, const pact_partition* part,
                          pact_trainer** out, bool sync_end) {
  if (!ctx || !ring || !meta || !signals || !grid || !mask || !cfg || !out || !part)
    return validation("pact_trainer_create: null argument").code;
  if (part->world < 1 || part->rank < 0 || part->rank >= part->world)
    return validation("pact_trainer_create: invalid partition").code;
  *out = nullptr;
  // TrainConfig::validate (optimize.hpp:71-77), SignalSet::validate, v0 (369-371)
  if (cfg->epochs < 1) return validation("train: epochs must be >= 1").code;
  if (cfg->steps_per_epoch < 1) return validation("train: steps_per_epoch must be >= 1").code;
  if (!(cfg->learning_rate > 0.0)) return validation("train: learning rate must be > 0").code;
  if (!(cfg->lambda_tv >= 0.0)) return validation("train: lambda_tv must be >= 0").code;
  if (cfg->n_delays < 1 || !cfg->delays) return validation("train: need at least one delay").code;
  if (ring->n_transducers < 3) return validation("ring: need at least 3 transducers").code;
  if (!(ring->radius > 0.0)) return validation("ring: radius must be > 0").code;
  if (meta->n_samples < 2) return validation("signals: need at least 2 samples").code;
  if (!(meta->dt > 0.0)) return validation("signals: dt must be > 0").code;
  const double v0 = meta->background_sos;
  if (!(v0 > 0.0)) return validation("joint_reconstruct: non-positive background SOS").code;

  HostTrace trace;
  auto* tr = new pact_trainer();
  tr->user = ctx;
  tr->eng.device = ctx->device;
  tr->eng.num_sms = ctx->num_sms;
  cudaError_t ce = cudaStreamCreateWithFlags(&tr->eng.own_stream, cudaStreamNonBlocking);
  if (ce != cudaSuccess) {
    delete tr;
    return cuda_status(ce, "cudaStreamCreateWithFlags").code;
  }
  tr->eng.stream = tr->eng.own_stream;
  auto fail = [&](int code) {
    pact_trainer_destroy(tr);
    return code;
  };
  tr->ring = *ring;
  tr->meta = *meta;
  tr->grid = *grid;
  tr->mask = *mask;
  tr->cfg = *cfg;
  tr->delays.assign(cfg->delays, cfg->delays + cfg->n_delays);
  tr->cfg.delays = tr->delays.data();
  tr->v0 = v0;
  Status st = make_layout(*grid, cfg->patch_mm, cfg->overlap, tr->lay);
  if (!st.ok()) return fail(st.code);
  tr->n_patches = tr->lay.nx * tr->lay.ny;
  if (part->world > tr->lay.ny) return fail(validation("partition: more ranks than patch rows").code);
  tr->rank = part->rank;
  tr->world = part->world;
  tr->p_lo = (tr->lay.ny * part->rank / part->world) * tr->lay.nx;
  tr->p_hi = (tr->lay.ny * (part->rank + 1) / part->world) * tr->lay.nx;
  tr->n_local = tr->p_hi - tr->p_lo;
  // the grid rows the local patches cover: only they are beamformed (SURVEY
  // §8(e): DAS split by image-row tiles; each DAS pixel is independent,
  // beamform.hpp:96-108, so the band equals those rows of the full stack)
  {
    auto oy = [&](int py) { return py == tr->lay.ny - 1 ? tr->lay.last_y : py * tr->lay.stride_pixels; };
    const int py_lo = tr->p_lo / tr->lay.nx, py_hi = (tr->p_hi - 1) / tr->lay.nx;
    tr->row0 = tr->n_local > 0 ? oy(py_lo) : 0;
    tr->rows = tr->n_local > 0 ? oy(py_hi) + tr->lay.patch_pixels - tr->row0 : 1;
  }
  tr->P = tr->lay.patch_pixels;
  tr->K = cfg->n_delays;
  tr->A = cfg->n_angles;
  tr->loss_scale = 1.0 / (static_cast<double>(tr->n_patches) * tr->K * tr->P * tr->P);
  tr->shape.hidden = cfg->hidden;
  tr->shape.layers = cfg->sine_layers;
  tr->shape.omega0 = cfg->omega0;
  tr->shape.out_scale = cfg->out_scale;
  tr->shape.v0 = v0;
  tr->n_params = static_cast<int>(tr->shape.count());
  std::vector<double> centers(2 * tr->n_patches);
  layout_centers(tr->lay, centers.data());
  st = ray_args(*ring, *grid, v0, *mask, cfg->n_angles, cfg->ray_step, tr->ray);
  if (!st.ok()) return fail(st.code);
  st = validate_centers(*ring, tr->n_patches, centers.data());
  if (!st.ok()) return fail(st.code);
  std::vector<float> win;
  st = merge_window(cfg->merge_fwhm, tr->P, grid->pitch, win);
  if (!st.ok()) return fail(st.code);
  trace.mark("layout + window");
  const MaskedPixels mp_all = masked_pixels(*grid, *mask);
  if (mp_all.n < tr->world) return fail(validation("partition: fewer masked pixels than ranks").code);
  tr->m_lo = static_cast<int>(static_cast<int64_t>(mp_all.n) * tr->rank / tr->world);
  tr->m_hi = static_cast<int>(static_cast<int64_t>(mp_all.n) * (tr->rank + 1) / tr->world);
  if (tr->world == 1) {
    tr->mp = mp_all;
  } else {
    tr->mp.n = tr->m_hi - tr->m_lo;
    tr->mp.idx.assign(mp_all.idx.begin() + tr->m_lo, mp_all.idx.begin() + tr->m_hi);
    tr->mp.coords.assign(mp_all.coords.begin() + 2 * tr->m_lo, mp_all.coords.begin() + 2 * tr->m_hi);
  }
  trace.mark("masked pixels");

  // ---- device arena ----
  const size_t npx = static_cast<size_t>(grid->width) * grid->height;
  const size_t P2 = static_cast<size_t>(tr->P) * tr->P;
  tr->n_tv = std::max(1, std::min(div_up(std::max(tr->mp.n, 1), 256), ctx->num_sms * 4));
  size_t bytes = 0;
  auto add = [&](size_t b) { bytes += (b + 255) & ~size_t(255); };
  add(sizeof(float) * tr->K * grid->width * tr->rows);           // stack (the local row band)
  add(sizeof(float2) * tr->n_local * tr->K * P2);                // Y (local patches)
  add(sizeof(float) * npx);                                      // dv
  add(sizeof(float) * tr->n_local * tr->A);                      // w
  add(sizeof(float) * tr->n_local * tr->A);                      // dw
  add(sizeof(double) * tr->n_local);                             // loss_patch
  add(sizeof(double) * npx);                                     // gv
  add(sizeof(float) * std::max(tr->mp.n, 1));                    // gtv
  add(sizeof(double) * tr->n_tv);                                // tv_partial
  add(npx);                                                      // inmask
  add(sizeof(double) * tr->n_params * 4);                        // theta m v grad
  add(sizeof(float) * tr->n_params);                             // theta32
  add(64);                                                       // flags
  add(sizeof(double) * 4);                                       // report
  add(sizeof(long long));                                        // t
  add(sizeof(double2) * tr->n_local);                            // centers
  add(sizeof(float) * P2);                                       // window
  if (tr->world > 1) add(sizeof(float) * 2 * npx);               // num, den
  bytes += 64 * 256;  // per-carve alignment slack
  st = pool_alloc(&tr->arena, bytes, tr->eng.stream);
  if (!st.ok()) return fail(st.code);
  char* p = static_cast<char*>(tr->arena);
  tr->stack = carve<float>(p, static_cast<size_t>(tr->K) * grid->width * tr->rows);
  tr->Y = carve<float2>(p, tr->n_local * tr->K * P2);
  tr->dv = carve<float>(p, npx);
  tr->w = carve<float>(p, tr->n_local * tr->A);
  tr->dw = carve<float>(p, tr->n_local * tr->A);
  tr->loss_patch = carve<double>(p, tr->n_local);
  tr->gv = carve<double>(p, npx);
  tr->gtv = carve<float>(p, std::max(tr->mp.n, 1));
  tr->tv_partial = carve<double>(p, tr->n_tv);
  tr->inmask = carve<unsigned char>(p, npx);
  tr->theta = carve<double>(p, tr->n_params);
  tr->m = carve<double>(p, tr->n_params);
  tr->v = carve<double>(p, tr->n_params);
  tr->grad = carve<double>(p, tr->n_params);
  tr->theta32 = carve<float>(p, tr->n_params);
  tr->flags = carve<unsigned>(p, 16);
  tr->report = carve<double>(p, 4);
  tr->t = carve<long long>(p, 1);
  tr->centers = carve<double2>(p, tr->n_local);
  tr->win = carve<float>(p, P2);
  if (tr->world > 1) {
    tr->num = carve<float>(p, npx);
    tr->den = carve<float>(p, npx);
  }

  trace.mark("arena");
  pact_ctx* e = &tr->eng;
  cudaStream_t s = e->stream;
  // inputs produced on the caller's stream must be visible to the engine
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  cudaEventRecord(ev, ctx->stream);
  cudaStreamWaitEvent(s, ev, 0);
  cudaEventDestroy(ev);

  std::vector<unsigned char> flag(npx, 0);
  for (int i : mp_all.idx) flag[i] = 1;
  std::vector<double> theta(tr->n_params);
  pact_siren sp{2, cfg->hidden, cfg->sine_layers, cfg->omega0, cfg->out_scale, v0};
  int rc = pact_init_siren(cfg->seed, &sp, theta.data());
  if (rc) return fail(rc);
  std::vector<float> theta32(theta.begin(), theta.end());
#define TRY_CU(x)                                        \
  do {                                                   \
    cudaError_t _e = (x);                                \
    if (_e != cudaSuccess) return fail(cuda_status(_e, #x).code); \
  } while (0)
#define TRY_ST(x)                                        \
  do {                                                   \
    Status _s = (x);                                     \
    if (!_s.ok()) return fail(_s.code);                  \
  } while (0)
  trace.mark("init_siren + flags");
  TRY_CU(cudaMemcpyAsync(tr->inmask, flag.data(), npx, cudaMemcpyHostToDevice, s));
  TRY_CU(cudaMemcpyAsync(tr->theta, theta.data(), sizeof(double) * tr->n_params,
                         cudaMemcpyHostToDevice, s));
  TRY_CU(cudaMemcpyAsync(tr->theta32, theta32.data(), sizeof(float) * tr->n_params,
                         cudaMemcpyHostToDevice, s));
  TRY_CU(cudaMemcpyAsync(tr->centers, centers.data() + 2 * tr->p_lo,
                         sizeof(double2) * tr->n_local, cudaMemcpyHostToDevice, s));
  TRY_CU(cudaMemcpyAsync(tr->win, win.data(), sizeof(float) * P2, cudaMemcpyHostToDevice, s));
  TRY_CU(cudaMemsetAsync(tr->m, 0, sizeof(double) * tr->n_params, s));
  TRY_CU(cudaMemsetAsync(tr->v, 0, sizeof(double) * tr->n_params, s));
  TRY_CU(cudaMemsetAsync(tr->flags, 0, 64, s));
  TRY_CU(cudaMemsetAsync(tr->t, 0, sizeof(long long), s));
  TRY_CU(cudaMemsetAsync(tr->dv, 0, sizeof(float) * npx, s));
  tr->ray.dv = tr->dv;
  tr->ray.centers = tr->centers;
  tr->ray.n_rays = tr->n_local * tr->A;
  make_raster_texture(tr->dv, grid->width, grid->height, &tr->ray.tex);
  TRY_ST(ray_plan_get(ctx, e, tr->ray, centers.data() + 2 * tr->p_lo, tr->n_local, tr->ray_plan));
  trace.mark("uploads + texture + ray plan");
  // pageable uploads first: a pageable cudaMemcpyAsync waits for the stream,
  // which is still idle here (after the DAS launch it would wait for the DAS)
  TRY_ST(siren_work_alloc(tr->sw, tr->mp, tr->shape, s));
  trace.mark("siren work");
  TRY_ST(fourier_table(e, tr->ftab, tr->P, grid->pitch, tr->A, tr->delays.data(), tr->K));
  trace.mark("fourier table");
  // DAS stack + spectra, once (optimize.hpp:380-392)
  // host signals (pinned: asynchronous) are uploaded on the engine's own
  // stream, so a batch's frames overlap their copies with each other's compute
  const float* dsig = signals;
  void* staged = nullptr;
  if (is_host_pointer(signals)) {
    const size_t nb = sizeof(float) * static_cast<size_t>(ring->n_transducers) * meta->n_samples;
    TRY_ST(pool_alloc(&staged, nb, s));
    cudaError_t ce2 = cudaMemcpyAsync(staged, signals, nb, cudaMemcpyHostToDevice, s);
    if (ce2 != cudaSuccess) {
      pool_free(staged, s);
      return fail(cuda_status(ce2, "signals H2D").code);
    }
    dsig = static_cast<const float*>(staged);
  }
  {
    Status sd = das_stack_device(e, *ring, *meta, dsig, *grid, v0, tr->delays.data(), tr->K,
                                 tr->stack, tr->row0, tr->rows);
    if (staged) pool_free(staged, s);
    if (sd.code) return fail(sd.code);
  }
  TRY_ST(launch_patch_fft(e, tr->lay, tr->stack, tr->K, tr->Y, tr->p_lo, tr->p_hi, tr->row0,
                          tr->rows));
  trace.mark("DAS + FFT launched");
  if (sync_end) TRY_CU(cudaStreamSynchronize(s));
  trace.mark("final sync");
  *out = tr;
  return PACT_OK;
#undef TRY_CU
#undef TRY_ST
}

int pact_trainer_create(pact_ctx* ctx, const pact_ring* ring, const pact_signal_meta* meta,
                        const float* signals, const pact_grid* grid, const pact_mask* mask,
                        const pact_train_config* cfg, pact_trainer** out) {
  const pact_partition whole{0, 1};
  return pact_trainer_create_partitioned(ctx, ring, meta, signals, grid, mask, cfg, &whole, out);
}

int pact_trainer_phase(pact_trainer* tr, int32_t phase) {
  if (!tr) return validation("pact_trainer_phase: null trainer").code;
  pact_ctx* e = &tr->eng;
  const size_t npx = static_cast<size_t>(tr->grid.width) * tr->grid.height;
  const size_t P2 = static_cast<size_t>(tr->P) * tr->P;
  if ((phase >= 0 && phase <= 3) || phase == 6 || phase == 7) {
    PACT_TRY(enqueue_phase(tr, phase));
    if (phase == 3) ++tr->steps_done;
    return PACT_OK;
  }
  if (phase == 4) {  // final render (optimize.hpp:478): local pixels into a cleared dv
    if (tr->world > 1) PACT_CUDA(cudaMemsetAsync(tr->dv, 0, sizeof(float) * npx, e->stream));
    PACT_TRY(siren_forward(e, tr->shape, tr->theta32, tr->sw, tr->dv));
    return PACT_OK;
  }
  if (phase == 5) {  // final deconvolution of the local patches -> merge accumulators
    if (tr->world == 1) return validation("pact_trainer_phase: phase 5 needs a partition").code;
    PACT_TRY(launch_wavefront(e, tr->ray, tr->w));
    void* tmp = nullptr;
    PACT_TRY(scratch_get(e, kScratchGeneric1, sizeof(float2) * tr->n_local * P2 +
                                                  sizeof(float) * tr->n_local * P2 + 256,
                         &tmp));
    float2* X = static_cast<float2*>(tmp);
    float* patches = reinterpret_cast<float*>(X + tr->n_local * P2);
    PACT_TRY(launch_wiener(e, tr->ftab.tab, tr->Y, tr->w, tr->n_local, tr->cfg.eps_deconv, X));
    PACT_TRY(launch_patch_ifft_real(e, tr->P, tr->n_local, X, patches));
    PACT_TRY(launch_merge_partial(e, tr->lay, patches, tr->win, tr->p_lo, tr->p_hi, tr->num,
                                  tr->den));
    return PACT_OK;
  }
  return validation("pact_trainer_phase: unknown phase").code;
}

int pact_trainer_local(pact_trainer* tr, int32_t* info) {
  if (!tr || !info) return validation("pact_trainer_local: null argument").code;
  info[0] = tr->p_lo;
  info[1] = tr->p_hi;
  info[2] = tr->m_lo;
  info[3] = tr->m_hi;
  info[4] = tr->n_patches;
  info[5] = tr->rank;
  info[6] = tr->world;
  info[7] = tr->row0;
  info[8] = tr->rows;
  return PACT_OK;
}

int pact_trainer_step(pact_trainer* tr, int32_t n_steps) {
  if (!tr) return validation("pact_trainer_step: null trainer").code;
  if (tr->world > 1)
    return validation("pact_trainer_step: a partitioned trainer steps by phases").code;
  for (int i = 0; i < n_steps; ++i) {
    if (tr->graph) {
      PACT_CUDA(cudaGraphLaunch(tr->graph, tr->eng.stream));
      tr->eng.launches.fetch_add(tr->graph_kernels);
    } else {
      int64_t before = tr->eng.launches.load();
      PACT_TRY(enqueue_step(tr));
      // the first (eager) step configures kernel attributes and scratch; later
      // steps replay it as one graph
      if (tr->cfg.use_cuda_graph && tr->steps_done == 0) {
        tr->graph_kernels = tr->eng.launches.load() - before;
        PACT_TRY(capture_graph(tr));
      }
    }
    ++tr->steps_done;
  }
  return PACT_OK;
}

int pact_trainer_report(pact_trainer* tr, int32_t epoch, double* report3) {
  if (!tr) return validation("pact_trainer_report: null trainer").code;
  double rep[4];
  unsigned flags = 0;
  PACT_CUDA(cudaMemcpyAsync(rep, tr->report, sizeof(double) * 3, cudaMemcpyDeviceToHost,
                            tr->eng.stream));
  PACT_CUDA(cudaMemcpyAsync(&flags, tr->flags, sizeof(unsigned), cudaMemcpyDeviceToHost,
                            tr->eng.stream));
  PACT_CUDA(cudaStreamSynchronize(tr->eng.stream));
  if (flags) {
    const char* what = (flags & kFlagSos)    ? "non-finite rendered SOS"
                       : (flags & kFlagLoss) ? "non-finite data loss"
                       : (flags & kFlagTv)   ? "non-finite TV loss"
                                             : "non-finite parameter gradient";
    set_error("joint_reconstruct: %s at epoch %d", what, epoch);
    return PACT_E_NUMERICAL;
  }
  if (report3) std::memcpy(report3, rep, sizeof(double) * 3);
  return PACT_OK;
}

int pact_trainer_run_epoch(pact_trainer* tr, int32_t epoch, double* report4) {
  if (!tr) return validation("pact_trainer_run_epoch: null trainer").code;
  auto t0 = std::chrono::steady_clock::now();
  int rc = pact_trainer_step(tr, tr->cfg.steps_per_epoch);
  if (rc) return rc;
  double rep[3];
  rc = pact_trainer_report(tr, epoch, rep);
  if (rc) return rc;
  double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (report4) {
    report4[0] = rep[0];
    report4[1] = rep[1];
    report4[2] = rep[2];
    report4[3] = wall;
  }
  return PACT_OK;
}

int pact_trainer_finish(pact_trainer* tr, float* image, float* sos) {
  if (!tr) return validation("pact_trainer_finish: null trainer").code;
  if (tr->world > 1)
    return validation("pact_trainer_finish: a partitioned trainer finishes by phases 4/5").code;
  pact_ctx* e = &tr->eng;
  const size_t npx = static_cast<size_t>(tr->grid.width) * tr->grid.height;
  const size_t P2 = static_cast<size_t>(tr->P) * tr->P;
  // render_sos + deconvolve_image with the learned field (optimize.hpp:478-486)
  PACT_TRY(siren_forward(e, tr->shape, tr->theta32, tr->sw, tr->dv));
  PACT_TRY(launch_wavefront(e, tr->ray, tr->w));
  void* tmp = nullptr;
  PACT_TRY(scratch_get(e, kScratchGeneric1, sizeof(float2) * tr->n_patches * P2 +
                                                sizeof(float) * tr->n_patches * P2 + 256,
                       &tmp));
  float2* X = static_cast<float2*>(tmp);
  float* patches = reinterpret_cast<float*>(X + tr->n_patches * P2);
  // host outputs (pinned: asynchronous) are written through a pooled device
  // buffer and copied back on the engine stream
  auto emit = [&](float* dst, auto&& produce) -> int {
    if (!is_host_pointer(dst)) return produce(dst);
    void* dev = nullptr;
    PACT_TRY(pool_alloc(&dev, sizeof(float) * npx, e->stream));
    int rc = produce(static_cast<float*>(dev));
    if (!rc && cudaMemcpyAsync(dst, dev, sizeof(float) * npx, cudaMemcpyDeviceToHost,
                               e->stream) != cudaSuccess)
      rc = cuda_status(cudaGetLastError(), "output D2H").code;  // (message set)
    pool_free(dev, e->stream);
    return rc;
  };
  if (image) {
    PACT_TRY(launch_wiener(e, tr->ftab.tab, tr->Y, tr->w, tr->n_patches, tr->cfg.eps_deconv, X));
    PACT_TRY(launch_patch_ifft_real(e, tr->P, tr->n_patches, X, patches));
    int rc = emit(image, [&](float* d) { return launch_merge(e, tr->lay, patches, tr->win, d).code; });
    if (rc) return rc;
  }
  if (sos) {
    int rc = emit(sos, [&](float* d) { return launch_sos_from_dev(e, tr->dv, npx, tr->v0, d).code; });
    if (rc) return rc;
  }
  // outputs visible on the caller's stream
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  cudaEventRecord(ev, e->stream);
  cudaStreamWaitEvent(tr->user->stream, ev, 0);
  cudaEventDestroy(ev);
  tr->user->launches.fetch_add(e->launches.exchange(0));
  return PACT_OK;
}

int pact_trainer_get_theta(pact_trainer* tr, double* theta) {
  if (!tr || !theta) return validation("pact_trainer_get_theta: null argument").code;
  PACT_CUDA(cudaMemcpyAsync(theta, tr->theta, sizeof(double) * tr->n_params,
                            cudaMemcpyDeviceToHost, tr->eng.stream));
  PACT_CUDA(cudaStreamSynchronize(tr->eng.stream));
  return PACT_OK;
}

int pact_trainer_set_theta(pact_trainer* tr, const double* theta) {
  if (!tr || !theta) return validation("pact_trainer_set_theta: null argument").code;
  std::vector<float> t32(theta, theta + tr->n_params);
  PACT_CUDA(cudaMemcpyAsync(tr->theta, theta, sizeof(double) * tr->n_params,
                            cudaMemcpyHostToDevice, tr->eng.stream));
  PACT_CUDA(cudaMemcpyAsync(tr->theta32, t32.data(), sizeof(float) * tr->n_params,
                            cudaMemcpyHostToDevice, tr->eng.stream));
  PACT_CUDA(cudaStreamSynchronize(tr->eng.stream));
  return PACT_OK;
}

void* pact_trainer_buffer(pact_trainer* tr, int32_t what) {
  if (!tr) return nullptr;
  switch (what) {
    case 0: return tr->stack;
    case 1: return tr->Y;
    case 2: return tr->dv;
    case 3: return tr->w;
    case 4: return tr->dw;
    case 5: return tr->gv;
    case 6: return tr->grad;
    case 7: return tr->theta;
    case 8: return tr->report;
    case 9: return tr->flags;
    case 10: return tr->num;
    case 11: return tr->den;
    case 12: return tr->theta32;
    default: return nullptr;
  }
}

int pact_trainer_destroy(pact_trainer* tr) {
  if (!tr) return PACT_OK;
  if (tr->eng.stream) cudaStreamSynchronize(tr->eng.stream);
  if (tr->user) tr->user->launches.fetch_add(tr->eng.launches.exchange(0));
  if (tr->graph) cudaGraphExecDestroy(tr->graph);
  if (tr->comm_stream) {
    cudaStreamSynchronize(tr->comm_stream);
    cudaStreamDestroy(tr->comm_stream);
  }
  if (tr->ev_eng) cudaEventDestroy(tr->ev_eng);
  if (tr->ev_comm) cudaEventDestroy(tr->ev_comm);
  if (tr->ray.tex) cudaDestroyTextureObject(tr->ray.tex);
  ray_plan_release(tr->ray_plan, tr->eng.stream);
  siren_work_free(tr->sw);
  fourier_table_free(tr->ftab);
  for (auto& sc : tr->eng.scratch) pool_free(sc.ptr, tr->eng.stream);
  pool_free(tr->arena, tr->eng.stream);
  if (tr->eng.stream) cudaStreamSynchronize(tr->eng.stream);
  if (tr->eng.own_stream) cudaStreamDestroy(tr->eng.own_stream);
  delete tr;
  return PACT_OK;
}

int pact_trainer_step_nccl(pact_trainer* tr, int32_t n_steps) {
  if (!tr) return validation("pact_trainer_step_nccl: null trainer").code;
  NcclRun r;
  PACT_TRY(nccl_run(tr, r));
  for (int i = 0; i < n_steps; ++i) {
    PACT_TRY(enqueue_phase(tr, 0));  // render own pixels -> dv
    PACT_TRY(r.comm_after_engine());
    PACT_TRY(r.share_dv());
    PACT_TRY(r.engine_after_comm());
    PACT_TRY(enqueue_phase(tr, 6));  // wavefronts, loss, ray adjoint -> dL/dv
    PACT_TRY(r.comm_after_engine());
    PACT_TRY(r.reduce_gv());         // ... while the engine runs TV + the report
    PACT_TRY(enqueue_phase(tr, 7));
    PACT_TRY(r.comm_after_engine());
    PACT_TRY(r.all_reduce(tr->report, 3, ncclFloat64, ncclSum, "all-reduce report"));
    PACT_TRY(r.all_reduce(tr->flags, 1, ncclUint32, ncclMax, "all-reduce flags"));
    PACT_TRY(r.engine_after_comm());
    PACT_TRY(enqueue_phase(tr, 2));  // SIREN backward of own pixels -> gradient
    PACT_TRY(r.comm_after_engine());
    PACT_TRY(r.all_reduce(tr->grad, static_cast<size_t>(tr->n_params), ncclFloat64, ncclSum,
                          "all-reduce gradient"));
    PACT_TRY(r.engine_after_comm());
    PACT_TRY(enqueue_phase(tr, 3));  // Adam, replicated: theta stays identical on every rank
    ++tr->steps_done;
  }
  return PACT_OK;
}

int pact_trainer_finish_nccl(pact_trainer* tr, float* image, float* sos) {
  if (!tr) return validation("pact_trainer_finish_nccl: null trainer").code;
  if (tr->world == 1) return pact_trainer_finish(tr, image, sos);
  NcclRun r;
  PACT_TRY(nccl_run(tr, r));
  pact_ctx* e = &tr->eng;
  if (int rc = pact_trainer_phase(tr, 4)) return rc;  // final render of own pixels
  PACT_TRY(r.comm_after_engine());
  PACT_TRY(r.share_dv());
  PACT_TRY(r.engine_after_comm());
  if (image) {
    if (int rc = pact_trainer_phase(tr, 5)) return rc;  // own patches -> merge accumulators
    PACT_TRY(r.comm_after_engine());
    PACT_TRY(r.all_reduce(tr->num, r.npx, ncclFloat32, ncclSum, "all-reduce merge numerator"));
    PACT_TRY(r.all_reduce(tr->den, r.npx, ncclFloat32, ncclSum, "all-reduce merge weights"));
    PACT_TRY(r.engine_after_comm());
    merge_divide_kernel<<<div_up(static_cast<int>(r.npx), 256), 256, 0, e->stream>>>(
        tr->num, tr->den, static_cast<int>(r.npx), image);
    PACT_TRY(after_launch(e, "merge_divide_kernel"));
  }
  if (sos) PACT_TRY(launch_sos_from_dev(e, tr->dv, r.npx, tr->v0, sos));
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  cudaEventRecord(ev, e->stream);
  cudaStreamWaitEvent(tr->user->stream, ev, 0);
  cudaEventDestroy(ev);
  tr->user->launches.fetch_add(e->launches.exchange(0));
  return PACT_OK;
}

int64_t pact_trainer_launch_count(pact_trainer* tr) { return tr ? tr->eng.launches.load() : -1; }

void* pact_trainer_stream(pact_trainer* tr) { return tr ? (void*)tr->eng.stream : nullptr; }

int pact_trainer_profile_step(pact_trainer* tr, float* stage_ms) {
  if (!tr || !stage_ms) return validation("pact_trainer_profile_step: null argument").code;
  if (tr->steps_done == 0) {  // configure kernels / capture the graph first
    int rc = pact_trainer_step(tr, 1);
    if (rc) return rc;
  }
  PACT_TRY(profile_step(tr, stage_ms));
  ++tr->steps_done;
  return PACT_OK;
}

int pact_joint_reconstruct(pact_ctx* ctx, const pact_ring* ring, const pact_signal_meta* meta,
                           const float* signals, const pact_grid* grid, const pact_mask* mask,
                           const pact_train_config* cfg, double* reports, float* image,
                           float* sos, double* theta) {
  pact_trainer* tr = nullptr;
  int rc0 = pact_trainer_create(ctx, ring, meta, signals, grid, mask, cfg, &tr);
  if (rc0) return rc0;
  for (int e = 1; e <= cfg->epochs; ++e) {
    int rc = pact_trainer_run_epoch(tr, e, reports ? reports + 4 * (e - 1) : nullptr);
    if (rc) {
      pact_trainer_destroy(tr);
      return rc;
    }
  }
  int rc = pact_trainer_finish(tr, image, sos);
  if (!rc && theta) rc = pact_trainer_get_theta(tr, theta);
  pact_trainer_destroy(tr);
  return rc;
}

int pact_joint_reconstruct_batch(pact_ctx* ctx, int32_t n_frames, const pact_ring* ring,
                                 const pact_signal_meta* meta, const float* const* signals,
                                 const pact_grid* grid, const pact_mask* mask,
                                 const pact_train_config* cfgs, double* reports,
                                 float* const* images, float* const* sos, double* thetas) {
  if (!ctx || n_frames < 0 || (n_frames > 0 && (!signals || !cfgs)))
    return validation("pact_joint_reconstruct_batch: null argument").code;
  std::vector<pact_trainer*> trs(n_frames, nullptr);
  auto cleanup = [&](int rc) {
    for (pact_trainer* t : trs) pact_trainer_destroy(t);
    return rc;
  };
  const int epochs = n_frames > 0 ? cfgs[0].epochs : 0;
  for (int f = 0; f < n_frames; ++f) {
    if (cfgs[f].epochs != epochs)
      return cleanup(validation("pact_joint_reconstruct_batch: frames need equal epochs").code);
    // `thetas` is strided by one parameter count: every frame needs the same network
    if (cfgs[f].hidden != cfgs[0].hidden || cfgs[f].sine_layers != cfgs[0].sine_layers)
      return cleanup(
          validation("pact_joint_reconstruct_batch: frames need the same SIREN shape").code);
    const pact_partition whole{0, 1};
    int rc = trainer_create(ctx, ring, meta, signals[f], grid, mask, &cfgs[f], &whole, &trs[f],
                            false);
    // the frame's first epoch is enqueued at once: its iterations run while
    // the host prepares the next frames
    if (!rc) rc = pact_trainer_step(trs[f], trs[f]->cfg.steps_per_epoch);
    if (rc) return cleanup(rc);
  }
  int n_params = 0;
  if (n_frames > 0) n_params = trs[0]->n_params;
  auto t0 = std::chrono::steady_clock::now();
  for (int e = 1; e <= epochs; ++e) {
    // a frame's next epoch (after the last: its final render + deconvolution)
    // is enqueued as soon as its report is read, so the other frames' streams
    // keep the GPU busy across the host round trip
    for (int f = 0; f < n_frames; ++f) {
      double rep[3];
      int rc = pact_trainer_report(trs[f], e, rep);
      if (!rc)
        rc = e < epochs ? pact_trainer_step(trs[f], trs[f]->cfg.steps_per_epoch)
                        : pact_trainer_finish(trs[f], images ? images[f] : nullptr,
                                              sos ? sos[f] : nullptr);
      if (rc) return cleanup(rc);
      if (reports) {
        double* r = reports + (static_cast<size_t>(f) * epochs + (e - 1)) * 4;
        r[0] = rep[0];
        r[1] = rep[1];
        r[2] = rep[2];
        r[3] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      }
    }
    t0 = std::chrono::steady_clock::now();
  }
  // every frame's final render + deconvolution was enqueued with its last
  // report, before any theta read waits on a frame
  for (int f = 0; thetas && f < n_frames; ++f) {
    int rc = pact_trainer_get_theta(trs[f], thetas + static_cast<size_t>(f) * n_params);
    if (rc) return cleanup(rc);
  }
  return cleanup(PACT_OK);
}

}  // extern "C"
