/* mixgraph_b200 — C ABI of the B200-native batched audio-graph renderer.
 *
 * This is the drop-in boundary for the reference's render path. The reference exposes a
 * C++ API (no FFI in the snapshot: its pybind11 module `mixgraph._core`,
 * proj/CMakeLists.txt:47-74, is absent); every entry point below is what such a binding
 * would call, and cites the reference interface it replaces. Conventions:
 *  - every function returns MG_OK (0) or an error code; mg_last_error() gives the
 *    message (thread-local). MG_EINVAL corresponds to the reference's
 *    std::invalid_argument and carries the same message text (tests match substrings
 *    such as "cycle", "channel", "homogeneity", "causality", "empty", "beam");
 *  - node types are the reference enum values (proj/include/mixgraph/types.hpp:12-23):
 *    0 in, 1 out, 2 mix, 3 gain, 4 eq, 5 compressor, 6 noisegate, 7 imager, 8 reverb, 9 delay;
 *  - edges are int32 quadruples [src, dst, outlet, inlet] in insertion order;
 *  - parameter tables are passed as `const double* const tables[10]` indexed by node type
 *    (NULL for absent types) with `rows[10]`; each table is row-major
 *    [rows][param_width(type)] (widths: gain 2, eq 1024, compressor/noisegate 4,
 *    imager 1, reverb 768, delay 880, others 0);
 *  - audio buffers are [batch][2][length] per signal, signals concatenated.
 * No function falls back to the CPU: without a CUDA device the render/process calls
 * return MG_ERUNTIME.
 */
#ifndef MIXGRAPH_B200_H
#define MIXGRAPH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MG_OK 0
#define MG_EINVAL 1
#define MG_ERUNTIME 2

#define MG_STRATEGY_ONE_BY_ONE 0
#define MG_STRATEGY_GREEDY 1
#define MG_STRATEGY_BEAM 2
#define MG_STRATEGY_OPTIMAL 3

typedef struct mg_plan mg_plan;             /* RenderData (+ its device step table) */
typedef struct mg_processors mg_processors; /* ProcessorSet (device constants) */
typedef struct mg_graph mg_graph;           /* one captured device render (CUDA graph) */
typedef struct mg_pipeline mg_pipeline;     /* streaming host-buffer renders (RenderPipeline) */

const char* mg_last_error(void);
int32_t mg_abi_version(void);
int32_t mg_param_width(int32_t node_type); /* types.cpp:14-25 */

/* Graph::validate (graph.cpp:48-114) on an edge list; MG_EINVAL with "cycle"/"channel"/... */
int32_t mg_graph_validate(const int32_t* node_types, int32_t num_nodes, const int32_t* edges, int32_t num_edges);

/* to_flat (graph.cpp:188-199) + compute_render_data (schedule.cpp:473-525). */
int32_t mg_plan_create(const int32_t* node_types, int32_t num_nodes, const int32_t* edges, int32_t num_edges,
                       int32_t strategy, int32_t beam_width, int32_t optimal_node_cap, mg_plan** out);
void mg_plan_destroy(mg_plan* plan);
/* info[6] = num_steps, buffer_rows, num_inputs, output_begin, num_edges, type string length */
int32_t mg_plan_info(const mg_plan* plan, int32_t* info);
/* Schedule::type_codes (schedule.cpp:301-306), NUL-terminated */
int32_t mg_plan_type_codes(const mg_plan* plan, char* buf, int32_t cap);
/* Schedule::subsets (original rows): sizes[type string length], rows concatenated */
int32_t mg_plan_subsets(const mg_plan* plan, int32_t* sizes, int32_t* rows);
/* RenderData::sigma (old row -> new row) */
int32_t mg_plan_sigma(const mg_plan* plan, int32_t* sigma);
/* RenderData::flat (reorder_flat, schedule.cpp:421-452): node types and edges */
int32_t mg_plan_flat(const mg_plan* plan, int32_t* node_types, int32_t* edges);
/* StepIndex k (schedule.hpp:60-68): head[6] = type, param_begin, param_end, store_begin,
 * store_end, |gather|; gather / aggregate may be NULL. */
int32_t mg_plan_step(const mg_plan* plan, int32_t k, int32_t* head, int32_t* gather, int32_t* aggregate);
/* RenderData::param_source_rows[type] (schedule.cpp:515-523); returns the count (>= 0) */
int32_t mg_plan_param_source_rows(const mg_plan* plan, int32_t node_type, int32_t* out);
/* RenderData::reorder_params (schedule.cpp:454-471): original-order tables -> render order */
int32_t mg_plan_reorder_params(const mg_plan* plan, const double* const* original, const int32_t* rows,
                               double* const* reordered);
/* validate_schedule (schedule.cpp:351-395) */
int32_t mg_validate_schedule(const int32_t* node_types, int32_t num_nodes, const int32_t* edges, int32_t num_edges,
                             const int32_t* type_string, int32_t num_subsets, const int32_t* subset_sizes,
                             const int32_t* subset_rows);

/* ProcessorSet(ProcessorConfig) (processors.cpp:151-160) on CUDA device `device`. */
int32_t mg_processors_create(double sample_rate, uint32_t reverb_seed, int32_t envelope_taps, double energy_floor,
                             int32_t device, mg_processors** out);
void mg_processors_destroy(mg_processors* procs);
/* info[3] = delay_span, delay_window, reverb_length */
int32_t mg_processors_info(const mg_processors* procs, int64_t* info);

/* render(rd, procs, params, sources, {keep_intermediates}) (render.cpp:14-81): host double
 * buffers; tables in render (reordered) row order; sources [K][B][2][L]; outputs
 * [num_outputs][B][2][L]; intermediates [buffer_rows][B][2][L] in ORIGINAL row order or NULL. */
int32_t mg_render(const mg_plan* plan, const mg_processors* procs, const double* const* tables, const int32_t* rows,
                  const double* sources, int32_t num_sources, int32_t batch, int64_t length, double sample_rate,
                  double* outputs, double* intermediates);

/* Device-resident render (the hot path): d_tables are device fp64 tables in render order;
 * d_arena holds buffer_rows x [B][2][L] fp32 with the sources in rows [0, num_inputs);
 * outputs are rows [output_begin, buffer_rows). Asynchronous on `stream` (cudaStream_t). */
int32_t mg_plan_workspace_bytes(const mg_plan* plan, const mg_processors* procs, int32_t batch, int64_t length,
                                uint64_t* bytes);
int32_t mg_plan_kernel_count(const mg_plan* plan, int32_t batch, int64_t length, int32_t* count);
/* owner[k] (num_steps entries) = the step whose kernel launch computes step k in a render:
 * k itself, the first step of a fused run of small pointwise steps, or the scan / pointwise
 * step whose epilogue computes it (measurement: per-kernel attribution of the render's work).
 * No reference counterpart (the reference runs one step at a time, render.cpp:40-80). */
int32_t mg_plan_step_owners(const mg_plan* plan, int32_t batch, int64_t length, int32_t* owner);
/* pairs[k] (num_steps entries) = the number of step k's slots that reuse the signal spectrum of a
 * slot of step k-1 in a render with these processors / batch / length (adjacent delay and
 * reverb steps on common source rows; 0 = step k transforms all its inputs). Measurement and
 * tests; no reference counterpart (the reference transforms every input, dsp.cpp:64-86). */
int32_t mg_plan_shared_pairs(const mg_plan* plan, const mg_processors* procs, int32_t batch, int64_t length,
                             int32_t* pairs);
/* Host-side plan analysis (no device needed), num_steps entries each: share_pairs[k] = slots
 * of step k that pair with a slot of step k-1 on a common single source row (both long
 * convolutions; used when the transforms match, mg_plan_shared_pairs), reads_prev_rows[k] = 1
 * when step k reads exactly step k-1's rows slot by slot (a compressor -> noisegate pair runs
 * as one kernel then). */
int32_t mg_plan_fusion_candidates(const mg_plan* plan, int32_t* share_pairs, int32_t* reads_prev_rows);
int32_t mg_render_arena(const mg_plan* plan, const mg_processors* procs, const double* const* d_tables, float* d_arena,
                        int32_t batch, int64_t length, void* d_workspace, uint64_t workspace_bytes, void* stream);

/* Same as mg_render_arena with, when step_ms is non-NULL, a device event pair recorded around
 * every step (each step then launches on its own): the call synchronises `stream` and writes
 * each step's duration (ms). hoist = 0 runs every parameter prologue inline and nothing on
 * side streams: the render's kernels serialised on `stream` (per-kernel costs in a trace). */
int32_t mg_render_arena_profiled(const mg_plan* plan, const mg_processors* procs, const double* const* d_tables,
                                 float* d_arena, int32_t batch, int64_t length, void* d_workspace,
                                 uint64_t workspace_bytes, void* stream, float* step_ms, int32_t hoist);

/* Capture one device render (same arguments as mg_render_arena) into a CUDA graph whose
 * kernel nodes keep their stream priorities (main path high, parameter prologues low);
 * mg_render_graph_launch replays it on `stream`. Arena, tables and workspace are baked in. */
int32_t mg_render_graph_create(const mg_plan* plan, const mg_processors* procs, const double* const* d_tables,
                               float* d_arena, int32_t batch, int64_t length, void* d_workspace,
                               uint64_t workspace_bytes, mg_graph** out);
int32_t mg_render_graph_launch(const mg_graph* graph, void* stream);
void mg_render_graph_destroy(mg_graph* graph);

/* Streaming host-buffer renders: submit() enqueues H2D (params + sources), the render graph
 * and D2H (outputs) on three chained streams over `depth` rotating arenas, so consecutive
 * renders overlap their PCIe copies with kernels. f32_io selects float host audio (else
 * double, as render()). sources [K][B][2][L], outputs [num_outputs][B][2][L]; tables in
 * render order, validated like mg_render. Host buffers must stay valid until sync(). */
int32_t mg_pipeline_create(const mg_plan* plan, const mg_processors* procs, int32_t batch, int64_t length,
                           int32_t f32_io, int32_t depth, int32_t host_threads, mg_pipeline** out);
int32_t mg_pipeline_submit(mg_pipeline* pipe, const double* const* tables, const int32_t* rows, const void* sources,
                           void* outputs);
int32_t mg_pipeline_sync(mg_pipeline* pipe);
void mg_pipeline_destroy(mg_pipeline* pipe);

/* Reverse-mode pass over a device render (parameter gradients, BASELINE configs 4/5; the
 * reference has no autodiff — fit.cpp:70-82 takes central differences, which the tests
 * compare against). d_arena / d_workspace: those of the mg_render_arena call that produced
 * the forward, the workspace sized by mg_backward_workspace_bytes (>= the forward's).
 * d_adjoint [rows][B][2][L] fp32: rows [output_begin, rows) hold dL/d(outputs) on entry;
 * on return rows [0, num_inputs) hold dL/d(sources) (other rows: dL/d(node inputs)).
 * d_grad_tables[t]: device fp64 tables shaped like d_tables[t] (render order), overwritten.
 * Delay tap positions are piecewise constant: their (Re z, Im z) gradients are 0. */
int32_t mg_backward_workspace_bytes(const mg_plan* plan, const mg_processors* procs, int32_t batch, int64_t length,
                                    uint64_t* bytes);
int32_t mg_render_backward_arena(const mg_plan* plan, const mg_processors* procs, const double* const* d_tables,
                                 const float* d_arena, float* d_adjoint, double* const* d_grad_tables, int32_t batch,
                                 int64_t length, void* d_workspace, uint64_t workspace_bytes, void* stream);

/* Execution-strategy switch for the long convolutions (diagnostics and tests): -1 chooses
 * per step (default: kernel spectra over 64 MiB fuse their row stage into the signal's row
 * pass), 0 always runs the separate kernel-spectrum row pass, 1 always fuses. Process-wide;
 * results agree either way. */
void mg_set_conv_fuse(int32_t mode);

/* Execution-strategy switch for the compressor / noisegate scans (diagnostics and tests): -1
 * chooses per step (default: steps with a full wave of dense sequences stream one sequence per
 * CTA, others run the chained look-back scan), 0 always chained, 1 streaming wherever legal
 * (dense steps, L % 4 == 0). Process-wide; results agree to fp64 rounding of the envelope. */
void mg_set_dyn_stream(int32_t mode);
/* A compressor / noisegate step followed by one reading exactly its rows (a console track's
 * compressor -> noisegate), both on the streaming scan, runs as ONE kernel (-1 / 1, default);
 * 0 runs them as two launches (tests). Process-wide. */
void mg_set_dyn_pair(int32_t mode);

/* Transform-size switch for the long convolutions (tests): 0 (default) picks per step the
 * cheapest segmented overlap-save size (one next_pow2(L + taps - 1) transform, as the
 * reference's fft_convolve `dsp.cpp:64-86`, whenever that is cheapest); 13..22 forces 2^log_n
 * points per segment. Applies to plans whose device workspace is sized after the call. */
void mg_set_conv_log(int32_t log_n);

/* Transform geometry a long convolution of `length` samples with a `taps`-tap kernel uses:
 * out = [log2 N, log2 N1 (columns), log2 N2 (rows), segments, output samples per segment]. */
int32_t mg_conv_geometry(int64_t length, int64_t taps, int64_t* out);

/* Arithmetic precision of the FFT-based steps (EQ, reverb, delay): 32 or 64 bits; the arena
 * stays fp32. Process-wide. */
void mg_set_fft_precision(int32_t bits);
int32_t mg_fft_precision(void);

/* Optimisation helpers on device buffers (fit.cpp:25-96 with analytic gradients): the MSE
 * loss mean((y - t)^2) into *d_loss (fp64, deterministic) and d_grad = 2 (y - t) / n;
 * d_scratch >= mg_mse_scratch_bytes(). mg_sgd_step: table -= lr * grad over rows x width,
 * then fit.cpp:13-21's projection of compressor/noisegate rows into their legal ranges. */
uint64_t mg_mse_scratch_bytes(void);
int32_t mg_mse_loss_grad(const float* d_y, const float* d_target, int64_t n, float* d_grad, double* d_loss,
                         void* d_scratch, void* stream);
int32_t mg_sgd_step(int32_t node_type, double* d_table, const double* d_grad, int32_t rows, double learning_rate,
                    void* stream);

/* Renders of plans whose topology changes every batch (BASELINE config 3), no per-plan
 * allocation or synchronisation: device pools sized once from a capacity (cap[4] = arena
 * rows, workspace bytes, step-table ints, parameter doubles; mg_batch_capacity gives one
 * plan's needs, take the max over the plans to render), `depth` rotating slots. submit()
 * takes parameter tables in ORIGINAL row order (reorder_params is done on the device,
 * schedule.cpp:454-471; missing/misshaped tables fail like it), validates them when
 * `validate` (processors.cpp:132-149), and sources fp32 [source_rows][B][2][L] (input k
 * takes row k % source_rows; device or host memory); outputs: host fp32
 * [num_outputs][B][2][L] or NULL. The plan must stay alive until its slot is reused
 * (`depth` submits later) or mg_batch_sync. Replaces, per batch, compute_render_data's
 * consumer loop in bench.cpp:52-57 with a re-drawn graph. */
typedef struct mg_batch mg_batch;
int32_t mg_batch_capacity(const mg_plan* plan, const mg_processors* procs, int32_t batch, int64_t length, uint64_t* cap);
int32_t mg_batch_create(const mg_processors* procs, int32_t batch, int64_t length, const uint64_t* cap, int32_t depth,
                        mg_batch** out);
int32_t mg_batch_submit(mg_batch* b, const mg_plan* plan, const double* const* tables, const int32_t* rows,
                        int32_t validate, const float* sources, int32_t source_rows, int32_t sources_on_device,
                        float* outputs);
int32_t mg_batch_sync(mg_batch* b);
int32_t mg_batch_last_arena(const mg_batch* b, void** arena);
void mg_batch_destroy(mg_batch* b);

/* Per-step device time (ms; prologue + audio pass of step k) averaged over `reps`
 * back-to-back repetitions replayed as one CUDA graph between one event pair, after one full
 * render. Synchronous. */
int32_t mg_profile_steps(const mg_plan* plan, const mg_processors* procs, const double* const* d_tables,
                         float* d_arena, int32_t batch, int64_t length, void* d_workspace, uint64_t workspace_bytes,
                         void* stream, int32_t reps, float* step_ms);

/* ProcessorSet::process (processors.cpp:229-282): in/out [slots][B][2][L] host double;
 * params [param_rows][width] (NULL for in/out/mix). */
int32_t mg_process(const mg_processors* procs, int32_t node_type, const double* in, double* out, int32_t slots,
                   int32_t batch, int64_t length, const double* params, int32_t param_rows, int32_t param_offset);
/* ProcessorSet::reverb_kernel (processors.cpp:162-187): left/right hold reverb_length samples */
int32_t mg_reverb_kernel(const mg_processors* procs, const double* row, double* left, double* right);
/* ProcessorSet::delay_kernel / delay_positions (processors.cpp:189-227) */
int32_t mg_delay_kernel(const mg_processors* procs, const double* row, int32_t channel, double* kernel,
                        int64_t* positions);
/* compressor_gain_log / noisegate_gain_log (processors.cpp:110-130) */
double mg_compressor_gain_log(double g_u, double threshold, double knee_half_width, double ratio);
double mg_noisegate_gain_log(double g_u, double threshold, double knee_half_width, double ratio);
/* check_param_row (processors.cpp:132-149) */
int32_t mg_check_param_row(int32_t node_type, const double* row);

/* default_param_row (graph.cpp:130-155) and dsp::uniform_noise (dsp.cpp:222-230). The
 * synthetic workload generators (console, random_legal_params) are test/bench support:
 * workloads/libmgbwork.so, not part of this library. */
int32_t mg_default_param_row(int32_t node_type, double* row);
int32_t mg_uniform_noise(int64_t n, uint32_t seed, double* out);

/* ---- File-level I/O (host only) -------------------------------------------------------
 * Graph documents: graph_to_json / graph_from_json / save_graph / load_graph
 * (proj/include/mixgraph/graph_io.hpp:20-24, proj/src/graph_io.cpp:19-127); DOT export
 * (graph_io.hpp:28, graph_io.cpp:129-143); 32-bit float stereo WAV (wav.hpp:11-12,
 * wav.cpp:39-133). Text outputs use the two-call idiom: *len receives the byte count
 * (without the terminating NUL); the text is copied only when cap > *len. Document errors
 * are MG_EINVAL ("graph document: ..."), WAV errors MG_ERUNTIME ("read_wav: ...",
 * "write_wav: ..."), as the reference's std::invalid_argument / std::runtime_error. */
typedef struct mg_doc mg_doc;     /* (Graph, ParamStore) of a parsed graph document */
typedef struct mg_audio mg_audio; /* AudioBuffer read from a WAV file */
int32_t mg_graph_to_json(const int32_t* node_types, int32_t num_nodes, const int32_t* edges, int32_t num_edges,
                         const double* const* tables, const int32_t* rows, char* buf, int64_t cap, int64_t* len);
int32_t mg_save_graph(const int32_t* node_types, int32_t num_nodes, const int32_t* edges, int32_t num_edges,
                      const double* const* tables, const int32_t* rows, const char* path);
int32_t mg_graph_from_json(const char* text, int64_t len, mg_doc** out);
int32_t mg_load_graph(const char* path, mg_doc** out);
/* rows[10]: parameter rows per node type, -1 for types without a table */
int32_t mg_doc_info(const mg_doc* doc, int32_t* num_nodes, int32_t* num_edges, int32_t* rows);
int32_t mg_doc_graph(const mg_doc* doc, int32_t* node_types, int32_t* edges);
int32_t mg_doc_params(const mg_doc* doc, int32_t node_type, double* out);
void mg_doc_destroy(mg_doc* doc);
int32_t mg_export_dot(const int32_t* node_types, int32_t num_nodes, const int32_t* edges, int32_t num_edges, char* buf,
                      int64_t cap, int64_t* len);
/* samples [batch][channels][length]; batch must be 1 and channels 2 (wav.cpp:40-41) */
int32_t mg_write_wav(const double* samples, int32_t batch, int32_t channels, int64_t length, double sample_rate,
                     const char* path);
int32_t mg_read_wav(const char* path, mg_audio** out);
int32_t mg_audio_info(const mg_audio* audio, int64_t* length, double* sample_rate);
int32_t mg_audio_samples(const mg_audio* audio, double* out); /* [1][2][length] */
void mg_audio_destroy(mg_audio* audio);

#ifdef __cplusplus
}
#endif

#endif /* MIXGRAPH_B200_H */
