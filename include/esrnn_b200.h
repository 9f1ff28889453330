/*
 * esrnn_b200.h — C-ABI of the B200-native ES-RNN training / forecasting engine.
 *
 * This is the drop-in boundary for the reference's hot path: every entry point
 * below replaces one member of `esrnn::Trainer`
 * (/root/reference/proj/include/esrnn/trainer.hpp) or a free function it owns.
 * The C++ class `esrnn::Trainer` in include/esrnn_b200/trainer.hpp (same API as
 * the reference) is a thin header-only wrapper over these functions; Python
 * binds them with ctypes (paper_1907_03329_b200/_native.py).
 *
 * Conventions
 *  - Plain pointers and sizes only; every buffer is caller-owned host memory,
 *    copied in/out synchronously during the call (the engine owns all device
 *    memory).  All real-valued buffers are fp64, like the reference's Matrix.
 *  - Functions never throw across the ABI.  They return an `esrnn_status`
 *    mirroring the reference's exception hierarchy (errors.hpp:9-67); the
 *    message is available from esrnn_last_error(handle) (or NULL handle for
 *    errors raised by esrnn_trainer_create).
 *  - A handle is single-threaded, like the reference Trainer.
 *
 * The same ABI is implemented by three libraries:
 *    libesrnn_b200.so          the product (CUDA sm_100a kernels)
 *    oracle/liboracle_esrnn.so the plain-C restatement (test oracle only)
 *    oracle/_ref/libesrnn_ref.so  the reference's own headers behind a shim
 *                                 (test oracle / CPU baseline only)
 */
#ifndef ESRNN_B200_H
#define ESRNN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ESRNN_ABI_VERSION 3
#define ESRNN_MAX_BLOCKS 8
#define ESRNN_MAX_LAYERS 16
#define ESRNN_NUM_CATEGORIES 6      /* data.hpp:21 kNumCategories */

/* Status codes: one per esrnn::Error subclass (errors.hpp:9-67) plus device errors. */
typedef enum esrnn_status {
    ESRNN_OK = 0,
    ESRNN_ERROR = 1,                  /* esrnn::Error                   errors.hpp:9   */
    ESRNN_PARSE_ERROR = 2,            /* ParseError                     errors.hpp:15  */
    ESRNN_VALIDATION_ERROR = 3,       /* ValidationError                errors.hpp:22  */
    ESRNN_SHAPE_ERROR = 4,            /* ShapeError                     errors.hpp:28  */
    ESRNN_INSUFFICIENT_LENGTH = 5,    /* InsufficientLengthError        errors.hpp:34  */
    ESRNN_NUMERIC_DOMAIN_ERROR = 6,   /* NumericDomainError             errors.hpp:40  */
    ESRNN_CONFIG_ERROR = 7,           /* ConfigError                    errors.hpp:46  */
    ESRNN_CONTRACT_ERROR = 8,         /* ContractError                  errors.hpp:52  */
    ESRNN_EQUIVALENCE_ERROR = 9,      /* EquivalenceError               errors.hpp:58  */
    ESRNN_CHECKPOINT_ERROR = 10,      /* CheckpointError                errors.hpp:64  */
    ESRNN_CUDA_ERROR = 11,            /* device / driver failure (no reference analogue) */
    ESRNN_NCCL_ERROR = 12             /* collective failure (no reference analogue)      */
} esrnn_status;

/* Compute precision of the device path (B200 extension; the reference is fp64). */
/* Zero selects fp64, the reference's arithmetic; fp32 is the opt-in performance path. */
enum { ESRNN_FP64 = 0, ESRNN_FP32 = 1 };

/* esrnn::FrequencyProfile (data.hpp:60-118).  dilation_blocks is flattened:
 * block b owns layers [sum(block_len[0..b)), +block_len[b]). */
typedef struct esrnn_profile {
    int32_t frequency;            /* 0 Yearly, 1 Quarterly, 2 Monthly (data.hpp:19) */
    int32_t seasonality_length;   /* S */
    int32_t horizon;              /* O */
    int32_t input_window;         /* I */
    int32_t hidden_size;          /* H */
    int32_t min_length;           /* C */
    int32_t n_blocks;
    int32_t block_len[ESRNN_MAX_BLOCKS];
    int32_t dilations[ESRNN_MAX_LAYERS];
} esrnn_profile;

/* esrnn::TrainConfig (trainer.hpp:22-44) plus B200 extensions at the end;
 * zero-initialised extensions reproduce the reference's behaviour (precision 0 = fp64). */
typedef struct esrnn_train_config {
    int32_t epochs;
    int32_t batch_size;
    double learning_rate_network;
    double learning_rate_per_series;
    double tau;
    int32_t has_gradient_clip;    /* std::optional<double> gradient_clip */
    double gradient_clip;
    uint64_t seed;
    int32_t attach_es_state;
    int32_t patience;
    double min_delta;
    /* --- B200 extensions --- */
    int32_t precision;            /* ESRNN_FP32 | ESRNN_FP64 */
    int32_t max_batch_size;       /* 0 => 2048, the reference cap (trainer.hpp:36) */
    int32_t device;               /* CUDA device ordinal */
    int32_t use_graphs;           /* 0 => default (on); <0 => off (debug) */
    /* --- ABI 3 --- */
    double level_variability_penalty;  /* lambda >= 0; 0 = the reference's pinball-only loss
                                        * (bit-identical).  See esrnn_trainer_run_batch. */
} esrnn_train_config;

/* Series-sharded data parallelism (B200 extension).  Rank r owns dataset
 * rows [floor(r*N/W), floor((r+1)*N/W)); per-series parameters live only on their owner.
 * Per step, the shared-network gradients and the step tail (per-series squared norm, loss
 * sum, error flag) are all-reduced, then every rank finalises the identical clip scale and
 * Adam update.  Two transports:
 *   - NCCL (one process per GPU): nccl_unique_id from esrnn_nccl_unique_id() on rank 0;
 *   - an in-process group (group != NULL, from esrnn_group_create): W trainers in one
 *     process, each driven by its own host thread, on one GPU or on peer-accessible GPUs;
 *     the exchange is the engine's own fused reduce kernel (no NCCL).
 * flags: ESRNN_DIST_FORCE_COLLECTIVE runs the collective step even at world_size 1 (a
 * one-rank NCCL communicator or group): the sharded code path on a single GPU. */
typedef struct esrnn_group esrnn_group;
enum { ESRNN_DIST_FORCE_COLLECTIVE = 1 };
typedef struct esrnn_dist {
    int32_t rank;
    int32_t world_size;
    uint8_t nccl_unique_id[128];  /* from esrnn_nccl_unique_id() on rank 0 */
    /* --- ABI 2 --- */
    int32_t flags;
    esrnn_group* group;
} esrnn_dist;

/* In-process rank group of world_size ranks (see esrnn_dist).  Destroy after every trainer
 * that joined it; a trainer keeps the group alive while it exists. */
esrnn_status esrnn_group_create(int32_t world_size, esrnn_group** out);
void esrnn_group_destroy(esrnn_group* g);

/* One named network array in StackWeights::for_each_param order (network.hpp:62-74). */
typedef struct esrnn_param_info {
    char name[32];
    int32_t rows;
    int32_t cols;
    int64_t offset;               /* into the flat weight vector */
} esrnn_param_info;

typedef struct esrnn_trainer esrnn_trainer;

const char* esrnn_version(void);
int32_t esrnn_abi_version(void);
/* Message of the last failing call on `t` (t == NULL: last failing create, per thread). */
const char* esrnn_last_error(const esrnn_trainer* t);

/* Trainer::Trainer(vector<SeriesRecord>, FrequencyProfile, TrainConfig)  trainer.hpp:159-200.
 * values: n_series x length row-major; category: n_series entries in [0,6) or -1
 * (unset -> Category::Other, trainer.hpp:186).  dist may be NULL (single GPU).
 * In sharded mode every rank passes the full dataset; only the owned rows are
 * uploaded.  Consumes the trainer RNG exactly like init_stack_weights
 * (network.hpp:89-116). */
esrnn_status esrnn_trainer_create(const esrnn_profile* profile, const esrnn_train_config* cfg,
                                  int64_t n_series, int32_t length, const double* values,
                                  const int32_t* category, const esrnn_dist* dist,
                                  esrnn_trainer** out);
void esrnn_trainer_destroy(esrnn_trainer* t);

/* Rows owned by this rank (all rows when unsharded). */
esrnn_status esrnn_trainer_shard(const esrnn_trainer* t, int64_t* row_begin, int64_t* row_end);

/* StackWeights layout: number of arrays / values, and one array's info. */
esrnn_status esrnn_trainer_param_count(const esrnn_trainer* t, int32_t* n_arrays, int64_t* n_values);
esrnn_status esrnn_trainer_param_info(const esrnn_trainer* t, int32_t index, esrnn_param_info* out);

/* Trainer::weights() (trainer.hpp:205-206) as a flat vector in for_each_param order. */
esrnn_status esrnn_trainer_get_weights(esrnn_trainer* t, double* flat, int64_t count);
/* Trainer::set_weights (trainer.hpp:415-432): count mismatch -> ESRNN_CHECKPOINT_ERROR. */
esrnn_status esrnn_trainer_set_weights(esrnn_trainer* t, const double* flat, int64_t count);

/* Trainer::per_series_params(i) (trainer.hpp:210-211) for rows [row_begin, row_begin+n)
 * (global row numbers; must be owned).  seas_raw is n x S row-major. */
esrnn_status esrnn_trainer_get_per_series(esrnn_trainer* t, int64_t row_begin, int64_t n,
                                          double* alpha_raw, double* gamma_raw, double* seas_raw);
/* Collective (every rank of a sharded trainer calls it): all series' per-series parameters
 * (Trainer::per_series_params for every i, trainer.hpp:210-211), gathered from their owners
 * in dataset order -- what checkpoint.hpp's snapshot (:48-62) needs from a sharded run.
 * alpha_raw, gamma_raw [n_series], seas_raw [n_series x S].  Unsharded: every row. */
esrnn_status esrnn_trainer_gather_per_series(esrnn_trainer* t, double* alpha_raw, double* gamma_raw,
                                             double* seas_raw);
/* Trainer::set_per_series (trainer.hpp:434-445), same addressing. */
esrnn_status esrnn_trainer_set_per_series(esrnn_trainer* t, int64_t row_begin, int64_t n,
                                          const double* alpha_raw, const double* gamma_raw,
                                          const double* seas_raw);

/* Training state for exact resume (B200 extension).  The reference's checkpoint v1
 * (checkpoint.hpp:37-46, :64-88) stores weights and per-series parameters only, so a
 * reloaded trainer restarts Adam and the shuffle RNG; these two calls export / import the
 * rest of what apply_updates and make_batches consume:
 *   adam_m, adam_v [n_values]  network Adam moments in for_each_param order (trainer.hpp:625-631)
 *   net_step                   the global Adam step (trainer.hpp:617)
 *   ps_m, ps_v [n x (2+S)]     per-series moments for rows [row_begin, row_begin+n), each row
 *                              {alpha, gamma, seas[S]} like PerSeriesParams (trainer.hpp:638-650)
 *   ps_steps [n]               per-series Adam steps (trainer.hpp:639)
 *   rng_text                   the trainer RNG (matrix.hpp:173-213) as std::mt19937_64's text
 *                              form, taken before the next epoch's shuffle; NUL-terminated, at
 *                              most ESRNN_RNG_TEXT_MAX bytes
 * Every pointer is nullable (that part is skipped); rows must be owned by this rank. */
#define ESRNN_RNG_TEXT_MAX 8192
esrnn_status esrnn_trainer_get_train_state(esrnn_trainer* t, double* adam_m, double* adam_v, int64_t n_values,
                                           int64_t row_begin, int64_t n, double* ps_m, double* ps_v,
                                           int64_t* ps_steps, int64_t* net_step, char* rng_text, int64_t rng_cap);
esrnn_status esrnn_trainer_set_train_state(esrnn_trainer* t, const double* adam_m, const double* adam_v,
                                           int64_t n_values, int64_t row_begin, int64_t n, const double* ps_m,
                                           const double* ps_v, const int64_t* ps_steps, int64_t net_step,
                                           const char* rng_text);

/* Trainer::train_epoch (trainer.hpp:234-243): shuffle (make_batches, trainer.hpp:82-102)
 * with the trainer RNG, one step per batch with updates; returns the
 * mask-weighted mean pinball loss. */
esrnn_status esrnn_trainer_train_epoch(esrnn_trainer* t, double* mean_loss);

/* One batch through build_graph (trainer.hpp:484-591) — the engine behind
 * batch_loss (:338), batch_gradients (:308) and step (:593).
 *   B, rows[B], anchors[B], mask[B*O] (NULL = all ones)         in
 *   flags: ESRNN_BATCH_GRADS (backward), ESRNN_BATCH_UPDATE (apply_updates)
 *   loss, mask_count                                            out (nullable)
 *   inputs[B*(I+6)], targets[B*O], seasonality_slices[B*O], anchor_levels[B]
 *                                                               out (nullable) — WindowBatch fields
 *   net_grads[n_values] (for_each_param order, incl. the exact zeros)  out (nullable)
 *   n_slots, slot_rows[B], ps_grads[B*(2+S)] (per slot: alpha_raw, gamma_raw, seas_raw[S])
 *                                                               out (nullable; slots in first-appearance
 *                                                               order, trainer.hpp:494-501)
 * In sharded mode every rank passes the same global batch; the loss/network
 * gradients are global, per-series outputs cover the local slots only. */
enum { ESRNN_BATCH_GRADS = 1, ESRNN_BATCH_UPDATE = 2 };
esrnn_status esrnn_trainer_run_batch(esrnn_trainer* t, int32_t B, const int32_t* rows,
                                     const int32_t* anchors, const double* mask, int32_t flags,
                                     double* loss, double* mask_count, double* inputs,
                                     double* targets, double* seasonality_slices,
                                     double* anchor_levels, double* net_grads, int32_t* n_slots,
                                     int32_t* slot_rows, double* ps_grads);

/* Global shuffled window order (series row, anchor) that the last train_epoch consumed:
 * make_batches(all_windows(), ...) with the trainer RNG (trainer.hpp:82-102, 214-223,
 * matrix.hpp:203-205); batch b is entries [b*batch_size, (b+1)*batch_size).  n must equal
 * the number of windows (series x (T - O - I + 1)).  Inspection hook for the bit-exact
 * window-index contract. */
esrnn_status esrnn_trainer_last_epoch_windows(const esrnn_trainer* t, int32_t* rows, int32_t* anchors, int64_t n);

/* Trainer::forecast_at(drop_tail) (trainer.hpp:248-288): real-scale O-step
 * forecasts for the owned rows, out is n_local x O row-major. */
esrnn_status esrnn_trainer_forecast(esrnn_trainer* t, int64_t drop_tail, double* out);

/* Trainer::validate (trainer.hpp:292-305): forecasts (nullable, n_local x O),
 * per-series sMAPE (nullable, n_local) and the mean over ALL series (global). */
esrnn_status esrnn_trainer_validate(esrnn_trainer* t, double* forecasts, double* smape_per_series,
                                    double* mean_smape);

/* Scoring behind cmd_evaluate (commands.hpp:312-338) and detail::score_forecasts
 * (commands.hpp:285-308), fused into the forecast pass.  against_test != 0: model forecasts
 * are forecast_at(O), actual = the test block, in-sample = train + validation;
 * against_test == 0: forecast_at(2*O), actual = the validation block, in-sample = train.
 * Per owned series (all nullable): forecasts [n_local x O], smape (metrics.hpp:17-28),
 * mase (metrics.hpp:33-49; NaN where the in-sample seasonal-naive MAE is 0, the reference's
 * std::nullopt), and the same two scores of seasonal_naive (metrics.hpp:52-59) over the same
 * in-sample span.  totals[8] (nullable) are sums over ALL ranks: {smape, mase, mase count,
 * naive smape, naive mase, naive mase count, series, 0}. */
esrnn_status esrnn_trainer_evaluate(esrnn_trainer* t, int32_t against_test, double* forecasts, double* smape,
                                    double* mase, double* naive_smape, double* naive_mase, double* totals);

/* forward_stack (network.hpp:190-210; plain mirror :268-287) over a general input sequence
 * with this trainer's StackWeights: the dilated recurrence with full LSTM cells (forget gates,
 * recurrent matrices, (h, c) from step t - d; lstm_cell :148-163, dilated_lstm_layer :167-184)
 * that the sequence-length-1 training path never exercises.
 *   inputs [seq_len][B][I+6] row-major (one (B, I+6) matrix per step), out [B][O]
 *   out_bar [B][O] (nullable): upstream adjoint of out; then weights_bar [n_values]
 *   (for_each_param order) and inputs_bar [seq_len][B][I+6] (each nullable) receive the
 *   reverse-mode adjoints (Tape::backward of the same graph, autodiff.hpp:397-631).
 * seq_len < 1 -> ESRNN_CONTRACT_ERROR ("forward_stack: empty sequence"). */
esrnn_status esrnn_trainer_forward_stack(esrnn_trainer* t, int32_t seq_len, int32_t B, const double* inputs,
                                         double* out, const double* out_bar, double* weights_bar,
                                         double* inputs_bar);

/* HWState of hybrid_primer(values[0:t_len], per_series_params(row)) (holt_winters.hpp:66-97):
 * levels[t_len], seasonalities[t_len + S].  Inspection hook for the scan KATs. */
esrnn_status esrnn_trainer_hw_state(esrnn_trainer* t, int64_t row, int64_t t_len, double* levels,
                                    double* seasonalities);

/* Device time in ms of the last train_epoch / run_batch / forecast / validate
 * call, measured with CUDA events on the engine's stream (0 for CPU builds). */
esrnn_status esrnn_trainer_last_device_ms(const esrnn_trainer* t, double* ms);
/* Number of kernels the engine launched since creation (graph nodes counted). */
esrnn_status esrnn_trainer_kernel_launches(const esrnn_trainer* t, int64_t* n);

/* Per-kernel device timing (measurement hook for bench.py's roofline).  enable == 1:
 * train_epoch / run_batch / forecast launch kernels directly (no CUDA graph) with a CUDA
 * event pair around every launch on the engine stream.  enable == 2: train_epoch runs its
 * CUDA graph as usual (programmatic dependent launch on) and every CTA stamps the device
 * global timer after its dependency wait and at its end; a kernel's time per step is its
 * latest CTA end minus its earliest CTA start.  kernel_times returns, per kernel class, the
 * summed milliseconds and launch counts since the last reset (0 disables both).
 * Classes: 0 (unused: the training scan runs inside the tile kernel), 1 tile (scan +
 * window + stack fwd/bwd + loss), 2 finish (ES backward + weight-gradient contraction),
 * 3 (unused), 4 adam, 5 finalize, 6 forecast_scan, 7 tile (forecast). */
#define ESRNN_KERNEL_CLASSES 8
esrnn_status esrnn_trainer_profile_kernels(esrnn_trainer* t, int32_t enable);
esrnn_status esrnn_trainer_kernel_times(esrnn_trainer* t, double* total_ms, int64_t* launches);

/* The engine keeps freed device / pinned-host blocks and instantiated epoch graphs in
 * process-wide caches so that re-creating a trainer of the same configuration allocates
 * and captures nothing; this returns every cached block to CUDA and drops the cached
 * graphs (live trainers keep theirs).  No-op in the CPU oracles. */
esrnn_status esrnn_release_cached_memory(void);

/* NCCL bootstrap for esrnn_dist (returns ESRNN_NCCL_ERROR in builds without NCCL). */
esrnn_status esrnn_nccl_unique_id(uint8_t out[128]);

/* Synthetic M4-shaped data, bit-identical to the reference's
 * testutil::make_multiplicative_series (tests/helpers.hpp:148-172) consumed in
 * order from Rng(seed): values n x length, category n. */
esrnn_status esrnn_make_synthetic(uint64_t seed, int64_t n, int32_t length, int32_t season_length,
                                  double noise_sigma, double* values, int32_t* category);

/* ---- Ingestion -------------------------------------------------
 * The reference's prepare + load path in one call: parse_m4_train_csv (data.hpp:205-232),
 * parse_info_csv (:251-279), apply_info (:282-290), the frequency filter and length
 * statistics of cmd_prepare (commands.hpp:141-175), equalize_lengths (data.hpp:147-160),
 * replacing the JSON bundle round trip (save_prepared / load_prepared, commands.hpp:30-74)
 * that feeds Trainer(vector<SeriesRecord>).  The train CSV's lines are parsed by `threads`
 * host threads (0 = all) with the reference's number parser (std::from_chars: values
 * bit-identical); the kept series' last C + 2*O values land in one pinned host block,
 * row-major n x (C + 2O), ready for esrnn_trainer_create (which uploads a pinned block
 * with one async copy, no staging).  Errors: the reference's exception class and message
 * for the first failing line in file order; the message via esrnn_ingest_last_error(). */
typedef struct esrnn_dataset esrnn_dataset;
typedef struct esrnn_ingest_stats {
    int64_t raw_count;          /* series of the selected frequency before equalisation */
    int64_t kept, dropped;
    int32_t equalized_length;   /* C + 2*O */
    double len_mean, len_stddev, len_min, len_q25, len_q50, len_q75, len_max;  /* LengthStats */
} esrnn_ingest_stats;
esrnn_status esrnn_ingest_m4_csv(const char* train_csv, const char* info_csv, int32_t frequency,
                                 const esrnn_profile* profile, int32_t threads, esrnn_dataset** out,
                                 esrnn_ingest_stats* stats);
const char* esrnn_ingest_last_error(void);
esrnn_status esrnn_dataset_shape(const esrnn_dataset* d, int64_t* n, int32_t* length);
const double* esrnn_dataset_values(const esrnn_dataset* d);     /* n x length, row-major */
const int32_t* esrnn_dataset_categories(const esrnn_dataset* d); /* n, data.hpp Category order */
const char* esrnn_dataset_id(const esrnn_dataset* d, int64_t i);
void esrnn_dataset_destroy(esrnn_dataset* d);

#ifdef __cplusplus
}
#endif

#endif /* ESRNN_B200_H */
