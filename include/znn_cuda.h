/*
 * znn_cuda.h — C-ABI of the B200-native ZNN training hot path
 * (libznn_cuda.so, built from paper_1510_06706_b200/csrc/).
 *
 * The reference (arXiv 1510.06706 / proj/include/znn) calls its hot-path
 * operators per EDGE and per SAMPLE as C++ templates on host volumes. This
 * boundary is per LAYER and per BATCH (one call covers all f x f' edges of a
 * fully connected layer and every patch) because per-edge calls cannot fill
 * a B200. Plain C types only: device pointers, int64 dims {x,y,z}, enums.
 *
 * Layout at the boundary (reference volume.hpp:21-24): a batch tensor is
 * [B][maps][x][y][z] fp32 with each map a contiguous x-major volume
 * (flat index (i*ny + j)*nz + l). Argmax masks are int32 flat indices into
 * the per-map INPUT volume (maxops.hpp:24-25), bit-comparable with the
 * reference's argmax_record.
 *
 * Status codes (reference tools/znn.cpp:182-191 exit codes):
 *   0 ok, 1 shape/config error (reference structural_error, types.hpp:57-74),
 *   2 CUDA/runtime error (reference std::runtime_error). Details via
 *   znn_last_error(). There is no CPU fallback: without a CUDA device every
 *   compute entry point returns 2.
 */
#ifndef ZNN_CUDA_H
#define ZNN_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ZNN_OK 0
#define ZNN_ERR_SHAPE 1
#define ZNN_ERR_RUNTIME 2

/* transfer kinds: transfer.hpp:11 transfer_kind {logistic, tanh, relu};
 * ZNN_ACT_NONE = identity (no transfer edge fused). */
#define ZNN_ACT_LOGISTIC 0
#define ZNN_ACT_TANH 1
#define ZNN_ACT_RELU 2
#define ZNN_ACT_NONE 3

/* convolution engines: engine.hpp:31 conv_engine {direct, fft} (+ auto = the
 * device autotuner, trainer.hpp:181-250). Direct = tensor-core implicit GEMM
 * (3xTF32) where the shape allows it, SIMT fp32 otherwise. */
#define ZNN_CONV_DIRECT 0
#define ZNN_CONV_FFT 1
#define ZNN_CONV_AUTO 2
#define ZNN_CONV_DIRECT_SIMT 3

/* losses: taskgraph.hpp:116-126 half-L2; binomial cross-entropy on logistic
 * outputs is the extension BASELINE configs 2-5 need. */
#define ZNN_LOSS_L2 0
#define ZNN_LOSS_CE 1

typedef struct znn_ctx_s* znn_ctx;
typedef struct znn_net_s* znn_net;

/* ---- library / context ---------------------------------------------- */
const char* znn_version(void);
/* number of CUDA devices visible (0 on a CPU-only host; never an error) */
int znn_device_count(void);
int znn_ctx_create(int device, znn_ctx* out);
int znn_ctx_destroy(znn_ctx ctx);
/* run all subsequent work of ctx on this cudaStream_t (NULL = legacy default) */
int znn_ctx_set_stream(znn_ctx ctx, void* cuda_stream);
int znn_ctx_synchronize(znn_ctx ctx);
const char* znn_last_error(znn_ctx ctx);
/* number of kernels this context has launched so far (evidence counter) */
int64_t znn_ctx_launch_count(znn_ctx ctx);

int znn_malloc(znn_ctx ctx, size_t bytes, void** dptr);
int znn_free(znn_ctx ctx, void* dptr);
int znn_memcpy_h2d(znn_ctx ctx, void* dst, const void* src, size_t bytes);
int znn_memcpy_d2h(znn_ctx ctx, void* dst, const void* src, size_t bytes);

/* ---- per-layer operators (device pointers) ---------------------------
 * conv: replaces conv_valid_direct (conv_direct.hpp:39-68) summed over the
 * f_in edges converging on each head node (engine.hpp:345-353 merge_payload,
 * sum_accumulator.hpp:51-95) plus the fused transfer edge
 * (transfer.hpp:58-73). x [B][f_in][n], w [f_out][f_in][k], bias [f_out]
 * (NULL = 0), y [B][f_out][n - s*(k-1)]. act = ZNN_ACT_*. */
int znn_conv_fwd(znn_ctx ctx, const float* x, int64_t B, int64_t f_in, const int64_t n[3],
                 const float* w, int64_t f_out, const int64_t k[3], const int64_t s[3],
                 const float* bias, int act, float* y, int engine);
/* dgrad: replaces conv_full_direct(g, reflect(k), s) (conv_direct.hpp:74-101,
 * called at engine.hpp:681-682) summed over the f_out edges leaving each
 * tail node. g [B][f_out][m], dx [B][f_in][m + s*(k-1)] (overwritten). */
int znn_conv_dgrad(znn_ctx ctx, const float* g, int64_t B, int64_t f_out, const int64_t m[3],
                   const float* w, int64_t f_in, const int64_t k[3], const int64_t s[3],
                   float* dx, int engine);
/* wgrad: replaces kernel_gradient_direct (conv_direct.hpp:108-132, called at
 * engine.hpp:791-792) summed over the batch. dw [f_out][f_in][k] =
 * scale * sum_b kernel_gradient(x_b, g_b) (overwritten). */
int znn_conv_wgrad(znn_ctx ctx, const float* x, int64_t B, int64_t f_in, const int64_t n[3],
                   const float* g, int64_t f_out, const int64_t k[3], const int64_t s[3],
                   float* dw, float scale, int engine);

/* transfer.hpp:58-73: y = phi(x + bias[map]); kinds: host array [f] of ZNN_ACT_* */
int znn_transfer_fwd(znn_ctx ctx, const float* x, int64_t B, int64_t f, int64_t voxels,
                     const int32_t* kinds_host, const float* bias, float* y);
/* transfer.hpp:77-121: gx = g * phi'(.) and dbias[map] = sum g * phi'(.).
 * If from_output != 0, phi' is evaluated from the transfer OUTPUT y
 * (relu: y>0, logistic: y(1-y), tanh: 1-y^2); otherwise from x + bias.
 * gx may alias g. dbias may be NULL. */
int znn_transfer_bwd(znn_ctx ctx, const float* g, const float* xy, int from_output, int64_t B,
                     int64_t f, int64_t voxels, const int32_t* kinds_host, const float* bias,
                     float* gx, float* dbias);

/* maxops.hpp:60-104. maps = B*f independent volumes. */
int znn_maxpool_fwd(znn_ctx ctx, const float* x, int64_t maps, const int64_t n[3],
                    const int64_t p[3], float* y, int32_t* mask);
int znn_maxpool_bwd(znn_ctx ctx, const float* g, const int32_t* mask, int64_t maps,
                    const int64_t m[3], const int64_t p[3], float* dx);
/* maxops.hpp:111-182. Dilated sliding max; ties -> lowest flat index. */
int znn_maxfilter_fwd(znn_ctx ctx, const float* x, int64_t maps, const int64_t n[3],
                      const int64_t k[3], const int64_t s[3], float* y, int32_t* mask);
int znn_maxfilter_bwd(znn_ctx ctx, const float* g, const int32_t* mask, int64_t maps,
                      const int64_t m[3], const int64_t k[3], const int64_t s[3],
                      float* dx);

/* loss over count voxels: L2 -> grad = scale*(a - d); CE -> grad_pre =
 * scale*(a - d) w.r.t. the logistic PRE-activation. loss_out (host) gets the
 * unscaled sum. */
int znn_loss(znn_ctx ctx, int kind, const float* a, const float* d, int64_t count,
             float scale, float* grad, double* loss_out);
/* engine.hpp:795,800 SGD extended with momentum: v = mu*v + g; w -= lr*v */
int znn_sgd_momentum(znn_ctx ctx, float* w, float* v, const float* g, int64_t count,
                     float lr, float mu);

/* ---- network executor (drop-in for engine<float>::run + train) --------
 * Builds the per-layer GPU executor from the reference netspec text
 * (netspec.hpp:13-27 format). out_dims NULL = take them from the spec. */
typedef struct {
    int64_t batch;        /* patches per step on this rank */
    int64_t global_batch; /* patches per step over all ranks (gradient mean) */
    float learning_rate;  /* trainer.hpp:39 default 0.01 */
    float momentum;       /* 0 = the reference's plain SGD */
    int loss;             /* ZNN_LOSS_* */
    int engine;           /* ZNN_CONV_* default for every conv layer */
    int sliding;          /* 1 = apply to_sliding_equivalent (netgraph.hpp:321-354) */
} znn_train_cfg;

int znn_net_create(znn_ctx ctx, const char* netspec, const int64_t* out_dims,
                   const znn_train_cfg* cfg, znn_net* out);
int znn_net_destroy(znn_net net);
/* textual summary of the layer program (one line per layer) */
const char* znn_net_describe(znn_net net);
int znn_net_num_params(znn_net net, int64_t* count);
/* input / output tensor element counts per patch (all input / output maps) */
int znn_net_io_sizes(znn_net net, int64_t* in_per_patch, int64_t* out_per_patch);
/* parameters in the reference's flat order: edges by id, conv -> k-volume,
 * transfer -> bias (test_engine.cpp:57-67 collect_params) */
int znn_net_set_params(znn_net net, const float* host_params);
int znn_net_get_params(znn_net net, float* host_params);
int znn_net_get_gradients(znn_net net, float* host_grads);
int znn_net_reset_momentum(znn_net net);
/* per-conv-layer engine choice; layer index as listed by describe() */
int znn_net_set_layer_engine(znn_net net, int conv_layer, int engine);
/* device autotuner (trainer.hpp:181-250): times fwd+bwd+upd of every conv
 * layer with each engine and keeps the faster. Returns chosen engines. */
int znn_net_autotune(znn_net net, int trials, int32_t* chosen, int max_layers);

/* FFT transform counters of conv layer `conv_layer` (fft.hpp:19-49 phases x
 * kinds): out[9] = {fwd image, fwd kernel, fwd inverse, bwd image, bwd kernel,
 * bwd inverse, upd image, upd kernel, upd inverse}. Status 1 if the layer
 * has not run on the FFT engine. */
int znn_net_fft_counts(znn_net net, int conv_layer, int64_t* out);

/* Roofline probe (bench.py): average device time of one frequency-domain
 * CMAC launch of the FFT engine for a conv layer (B patches, f_in -> f_out
 * maps, input dims n, kernel k, sparsity s; the engine's own pads give the
 * bin count, returned in *bins), `which` = 0 forward (Y = X conj K, the
 * merge_payload sum of conv_fft.hpp:38-60), 1 data gradient
 * (conv_fft.hpp:67-96), 2 kernel-gradient product (conv_fft.hpp:98-125);
 * timed with CUDA events on the context stream over `reps` launches on
 * synthetic spectra it allocates ((B f_in + B f_out + f_in f_out) x bins x 8 bytes). */
int znn_fft_cmac_time(znn_ctx ctx, int which, int64_t B, int64_t f_in, int64_t f_out, const int64_t n[3],
                      const int64_t k[3], const int64_t s[3], int reps, float* ms, int64_t* bins);
/* Measured FP32 FMA throughput of the device (TFLOP/s) for 3-register FFMA
 * (d = a*b + c, all operands in registers, the form the CMACs issue; 16
 * independent chains per thread, 2 CTAs of 1024 threads per SM): the
 * denominator of the CMAC roofline, since MEASURED_PEAKS.json carries HBM
 * and bf16 only. */
int znn_fma_peak_tflops(znn_ctx ctx, float* tflops);

/* Full SGD step through HOST buffers (H2D of inputs/labels, fwd, loss,
 * bwd, update, D2H of the loss): the reference engine::run round. */
int znn_net_step_host(znn_net net, const float* inputs, const float* labels, double* loss);
/* Phase split for data-parallel training (gradient allreduce between):
 * forward + loss + backward from DEVICE buffers, gradients into the flat
 * device gradient buffer, no update. */
int znn_net_forward_backward(znn_net net, const float* inputs_dev, const float* labels_dev,
                             double* loss);
int znn_net_apply_update(znn_net net);
/* Single-process SGD step from DEVICE buffers: forward + loss + backward with
 * the SGD+momentum update applied layer by layer as each gradient becomes
 * final (fused into the tensor-core weight-gradient epilogue; the weights a
 * layer's data gradient reads are updated only after it). Same result as
 * znn_net_forward_backward + znn_net_apply_update; the reference likewise
 * updates each edge as soon as its gradient task ran (run_update_body,
 * engine.hpp:772-829). */
int znn_net_train_step(znn_net net, const float* inputs_dev, const float* labels_dev, double* loss);
/* device pointer + length of the flat gradient buffer (allreduce target) */
int znn_net_grad_buffer(znn_net net, float** dptr, int64_t* count);
/* forward only; outputs [B][f_out][m] copied to host when host_out != NULL */
int znn_net_forward(znn_net net, const float* inputs_dev, float* host_out);
/* node-group images for tests: group index as in describe(); which = 0
 * forward image, 1 backward image (valid after forward_backward). */
int znn_net_group_info(znn_net net, int group, int64_t* maps, int64_t dims[3]);
int znn_net_get_group_image(znn_net net, int group, int which, float* host);
int znn_net_get_mask(znn_net net, int group, int32_t* host);

/* ---- FFT engine per layer ---------------------------------------------
 * A plan is the reference's fft_plan_cache + memo_store for one fully
 * connected layer (fft.hpp:57-192, conv_fft.hpp:127-192): pads, memoised
 * image spectra X of the layer input and kernel spectra K.
 * znn_fft_conv_fwd = fwd_image_fft + fwd_kernel_fft + fft_conv_valid_pre
 *   (conv_fft.hpp:25-60) summed over the f_in converging edges, + bias and
 *   transfer; memoises X and K.
 * znn_fft_conv_bwd = fwd_image_fft(g) + fft_conv_full_adjoint_pre
 *   (conv_fft.hpp:67-96, dx; NULL = skip, e.g. for the input layer) +
 *   fft_kernel_gradient_pre (conv_fft.hpp:98-125, dw = sum over the batch),
 *   from the memo of the preceding znn_fft_conv_fwd (status 1 without one).
 * Shapes and layouts as znn_conv_fwd / _dgrad / _wgrad. */
typedef struct znn_fft_plan_s* znn_fft_plan;
int znn_fft_plan_create(znn_ctx ctx, int64_t B, int64_t f_in, int64_t f_out, const int64_t n[3],
                        const int64_t k[3], const int64_t s[3], znn_fft_plan* out);
int znn_fft_plan_destroy(znn_fft_plan p);
/* pads (x, y, z), bins = px*py*(pz/2+1), bytes of the kernel spectra */
int znn_fft_plan_info(znn_fft_plan p, int64_t pads[3], int64_t* bins, int64_t* kernel_spectrum_bytes);
int znn_fft_conv_fwd(znn_fft_plan p, const float* x, const float* w, const float* bias, int act, float* y);
int znn_fft_conv_bwd(znn_fft_plan p, const float* g, const float* w, float* dw, float* dx);
/* transform counters as znn_net_fft_counts */
int znn_fft_plan_counts(znn_fft_plan p, int64_t out[9]);

/* ---- autotune one layer (trainer.hpp:181-250 autotune_modes) -----------
 * Median-of-`trials` device time of fwd + dgrad + wgrad for the layer at
 * batch B with each candidate engine (tensor-core direct, FFT, SIMT direct
 * for thin layers); *chosen = the fastest ZNN_CONV_*, ms[3] = {direct, fft,
 * simt} (-1 = not a candidate or failed). */
int znn_autotune_layer(znn_ctx ctx, int64_t B, int64_t f_in, int64_t f_out, const int64_t n[3],
                       const int64_t k[3], const int64_t s[3], int trials, int* chosen, float ms[3]);

/* ---- data parallelism over NCCL (the reference has none) ---
 * One communicator per rank. Rank 0 creates the 128-byte unique id and the
 * caller distributes it (MPI, a file, torch.distributed). */
#define ZNN_COMM_ID_BYTES 128
typedef struct znn_comm_s* znn_comm;
int znn_comm_unique_id(void* id /* ZNN_COMM_ID_BYTES */);
int znn_comm_create(znn_ctx ctx, const void* id, int nranks, int rank, znn_comm* out);
int znn_comm_destroy(znn_comm comm);
/* in-place sum over ranks on the context stream (fp32) */
int znn_allreduce(znn_comm comm, float* buf, int64_t count);
/* one data-parallel SGD step on this rank's shard (device buffers): forward,
 * loss (scaled by 1/global_batch), backward with one allreduce per layer
 * issued on a communication stream as soon as that layer's gradient is final
 * (overlapping the remaining backward), then the SGD+momentum update. */
int znn_net_train_step_dp(znn_net net, znn_comm comm, const float* inputs_dev, const float* labels_dev,
                          double* loss);

/* ---- CUDA graph + memory ------------------------------------------------
 * Graph mode: znn_net_train_step / step_host / step_loader run the first
 * step eagerly, then capture the whole step once per input buffer pair and
 * replay it (no per-launch host work, no allocation: the scratch arena is
 * frozen and a step that would need more fails with status 2). */
int znn_net_set_graph(znn_net net, int on);
int znn_net_graph_captured(znn_net net, int* yes);
/* out = {device free bytes, device total bytes, device allocations made by
 * the library so far, bytes of those allocations} */
int znn_mem_stats(znn_ctx ctx, int64_t out[4]);

/* In-step kernel timing: with profiling on, the library records a CUDA
 * event pair around each launch of its dominant kernels (FFT CMACs, kernel
 * spectra, transforms, tensor-core convolutions, max-filter) on the launch
 * stream (never inside a graph capture). report: JSON array of {kernel,
 * launches, ms (sum of event durations), bytes, flops (algorithmic, summed
 * over launches)} since the last report; status 1 if buf is too small. */
int znn_profile_enable(znn_ctx ctx, int on);
int znn_profile_report(znn_ctx ctx, char* buf, int64_t len);

/* ---- volume files and the data provider ---------------------------------
 * ZNNV format (volume_io.hpp:15-86): "ZNNV", u32 version 1, u32 nx, ny, nz,
 * float32 x-major, little-endian. read: data NULL -> dims only. */
int znn_volume_write(const char* path, const int64_t dims[3], const float* data);
int znn_volume_read(const char* path, int64_t dims[3], float* data, int64_t capacity);
/* Data provider (trainer.hpp:87-166): patch b of step t is sample
 * (t * global_batch + shard_offset + b) mod samples. From a directory with
 * inputs/ and labels/ ZNNV files paired by sorted name (every input node
 * gets the input volume, every output node the label, as from_files does),
 * or from host arrays [samples][in maps][in vol] / [samples][out maps][out
 * vol] (pin them for asynchronous copies). Two pinned/device slots: the
 * next step's files and H2D overlap the current step. */
typedef struct znn_loader_s* znn_loader;
int znn_loader_open_dir(znn_net net, const char* dir, int64_t shard_offset, znn_loader* out);
int znn_loader_open_host(znn_net net, const float* inputs, const float* labels, int64_t samples,
                         int64_t shard_offset, znn_loader* out);
int znn_loader_size(znn_loader ld, int64_t* samples);
int znn_loader_destroy(znn_loader ld);
/* one SGD step on the loader's next batch (single process; fused update) */
int znn_net_step_loader(znn_net net, znn_loader ld, double* loss);

#ifdef __cplusplus
}
#endif
#endif
