/*
 * otfgpu.h -- C ABI of libotfgpu.so, the B200 engine for the reference's
 * virtual-clock scalability experiment.
 *
 * The reference (otfstream, pure Python) has no FFI; its drop-in boundary is
 * the Python call
 *
 *     run_experiment(config: ExperimentConfig) -> ExperimentResult
 *         /root/reference/pkg/src/otfstream/orchestrator.py:327-370
 *
 * plus the sweep driver that calls it once per grid point
 * (orchestrator.py:373-390, cli.py:52-62).  This library replaces the body of
 * that call for a whole batch of configs at once: the host lowers each
 * ExperimentConfig to an otf_scenario plus shared input tables, and
 * otf_run_batch() replays every scenario's event order on the GPU.  The
 * Python package paper_2603_08417_b200 binds these symbols with ctypes
 * (INTEGRATION.md shows the binding).
 *
 * Conventions: plain C types only; every pointer inside otf_batch is a DEVICE
 * pointer owned by the caller unless stated otherwise; calls are stateless,
 * enqueue on the given CUDA stream and return an otf_status.  The last error
 * message is kept per host thread (otf_last_error).
 */
#ifndef OTFGPU_H
#define OTFGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OTF_ABI_VERSION 3

/* ---- status codes (ValueError / RuntimeError on the Python side) ---- */
typedef enum {
    OTF_OK = 0,
    OTF_EINVAL = 1,     /* malformed batch / scenario (ConfigError-class) */
    OTF_ECUDA = 3,      /* a CUDA call failed */
} otf_status;

/* ---- per-scenario status bits (otf_batch.status[s]) ---- */
#define OTF_S_RECORD_OVERFLOW 0x1  /* record capacity too small: counts are exact, re-run with them */
#define OTF_S_EPS_OVERFLOW 0x2     /* worker noise table too short: re-run with a longer one */
#define OTF_S_INTERNAL 0x4         /* structural invariant violated (bug) */
#define OTF_S_TIE 0x8              /* windowed engine met an ordering tie it cannot resolve:
                                      the host re-runs the scenario on the exact engine */
#define OTF_S_HUNG 0x10            /* a client slept forever (starved trace), informative */
#define OTF_S_UNFIT 0x20           /* outside the windowed engine's limits (client / descriptor /
                                      worker counts, segments per sequence, simultaneous requests):
                                      the host re-runs the scenario on the exact engine */
#define OTF_S_LIST_OVERFLOW 0x80  /* windowed engine: more simultaneous requests in one window than
                                      otf_scenario.list_cap: the host re-runs it with a larger list */
#define OTF_S_TAIL_OVERFLOW 0x40   /* a summary tail buffer (nonzero latencies / stalled sessions) was
                                      too small: otf_qoe.n_lat_tail / n_stall_tail are exact, re-run */

/* ---- enums shared with the host (values are part of the ABI) ---- */
enum { OTF_PATH_STORAGE = 0, OTF_PATH_CACHE = 1, OTF_PATH_WAITED = 2, OTF_PATH_TRANSCODED = 3, OTF_PATH_ERROR = 4 };
enum { OTF_ORIGIN_DEMAND = 0, OTF_ORIGIN_SPECULATIVE = 1 };
enum { OTF_OUTCOME_PENDING = 0, OTF_OUTCOME_COMPLETED = 1, OTF_OUTCOME_DROPPED = 2 };
enum { OTF_POP_UNIFORM = 0, OTF_POP_ZIPF = 1 };
enum { OTF_ENGINE_EXACT = 0, OTF_ENGINE_WINDOWED = 1 };
enum { OTF_MODE_HISTOGRAM = 0, OTF_MODE_RECORDS = 1 };

/* stats[] slots: Backend.stats() (backend.py:228-239) and SegmentCache.stats()
 * (cache.py:83-92) as integers. */
enum {
    OTF_ST_JOBS_TOTAL = 0, OTF_ST_JOBS_DEMAND, OTF_ST_JOBS_SPEC, OTF_ST_WASTED, OTF_ST_SPEC_ENQUEUED,
    OTF_ST_SKIP_DISABLED, OTF_ST_SKIP_EOS, OTF_ST_SKIP_STORED, OTF_ST_SKIP_CACHED,
    OTF_ST_SKIP_INFLIGHT, OTF_ST_SKIP_OVERLOAD,
    OTF_ST_CACHE_CAPACITY, OTF_ST_CURRENT_BYTES, OTF_ST_ENTRIES, OTF_ST_HITS, OTF_ST_MISSES,
    OTF_ST_EVICTIONS, OTF_ST_REJECTED,
    OTF_ST_STATUS, OTF_ST_HUNG, OTF_ST_TIMER_POPS, OTF_ST_READY_CALLBACKS, OTF_ST_WINDOWS,
    /* windowed engine profile: SM cycles spent per phase (lane 0's clock) */
    OTF_ST_CYC_SCAN, OTF_ST_CYC_SORT, OTF_ST_CYC_SERVER, OTF_ST_CYC_CLIENTS, OTF_ST_CYC_TOTAL,
    OTF_ST_CYC_LOCAL,   /* client-local phase run concurrently with the server lane */
    OTF_ST_PAR_WINDOWS, /* windows whose server events took the parallel (request-only) pass */
    OTF_ST_NSLOTS = 32
};

/* One scenario = one ExperimentConfig (orchestrator.py:74-113).  Table
 * offsets index the shared pools of otf_batch (in elements). */
typedef struct otf_scenario {
    int32_t n_clients, n_workers, n_seq, n_ranks;
    int32_t max_nseg, n_samples, cache_enabled, spec_enabled;
    int32_t popularity;
    int32_t queue_bound;              /* BackendPolicy.queue_bound: 0 = unbounded (backend.py:56,160-166) */
    uint32_t stored_mask;             /* bit r set <=> rank r stored at origin (backend.py:76-82) */
    int32_t retries;                  /* ClientConfig.retries (client.py:291-305) */
    int64_t cache_capacity;           /* bytes (cache.py:27-30) */
    uint64_t seed;                    /* ExperimentConfig.seed: picks stream SS([seed, 3, cid]) */
    double horizon, latency;          /* horizon_s; ClientConfig.latency_s */
    double target, safe, panic, resume, startup;   /* BufferConfig (client.py:49-61) */
    double alpha, headroom;           /* ClientConfig.ewma_alpha / headroom */
    double noise;                     /* LatencyModel.noise_rel_std */
    double period;                    /* BandwidthTrace.period (shared timestamps) */
    double grid_step;                 /* > 0 when starts[i] == i * grid_step exactly (bisect-free lookup) */
    double retry_backoff;             /* ClientConfig.retry_backoff_s */
    int32_t demand_priority;          /* BackendPolicy.demand_priority (backend.py:103-105,174-184) */
    int32_t list_cap;                 /* windowed engine: server events one window can hold (0 = the
                                         default for n_clients, otf_list_cap); more -> OTF_S_LIST_OVERFLOW */
    int64_t off_tr_i;                 /* CSV traces (netem.trace_dir): i64 [n_clients][3] = starts offset,
                                         values offset, samples (f64 pool); -1 = synthetic traces */
    int64_t off_tr_f;                 /* f64 [n_clients][3] = period, period bits, grid step */
    int64_t off_sizes;                /* i64: [n_seq][n_ranks][max_nseg] segment bytes */
    int64_t off_bitrates;             /* i64: [n_ranks] */
    int64_t off_manifest;             /* i64: [n_seq] manifest JSON bytes */
    int64_t off_segcount;             /* i32: [n_seq] */
    int64_t off_seqdur, off_segdur;   /* f64: [n_seq] */
    int64_t off_rho;                  /* f64: [n_ranks] */
    int64_t off_zipf;                 /* f64: [n_seq] Zipf CDF (popularity == ZIPF) */
    int64_t off_starts;               /* f64: [n_samples] trace piece start times */
    int64_t off_values;               /* f64: [n_clients][n_samples] bandwidth, bit/s */
    int64_t off_pbits;                /* f64: [n_clients] bits per trace period */
    int64_t off_arrivals;             /* f64: [n_clients] arrival offsets (cumsum) */
    int64_t off_eps;                  /* f64: [n_workers][eps_stride] worker noise draws */
    int64_t eps_stride;
    int64_t scratch_off;              /* bytes into otf_batch.scratch */
    int64_t req_off, req_cap;         /* record slices (records mode) */
    int64_t sess_off, sess_cap;
    int64_t seg_off, seg_cap;
    int64_t job_off, job_cap;
    /* summary tails (both modes; see otf_batch.tail_*): the nonzero request
     * latencies, every closed session (ses_cap records, then 2 * stl_cap
     * entries where the summary pass gathers and orders the stalled ones), and
     * the startup delays */
    int64_t lat_off, lat_cap;
    int64_t ses_off, ses_cap, stl_cap;
    int64_t sup_off, sup_cap;
} otf_scenario;

/* Fused QoE / fulfillment epilogue (metrics.py:67-116, orchestrator.py:280-309).
 * Every field ExperimentResult.summary() reports is exact here, so a sweep
 * needs no per-request records:
 *   requests / sessions / jobs        n_requests, n_sessions, otf_batch.counts[3]
 *   instant_fraction                  lat_hist[0] / n_requests  (lat_hist[0] counts latency < 0.010 exactly)
 *   latency_p50_s / latency_p99_s     latency_p50 / latency_p99: sorted(latencies)[n // 2] and
 *                                     [min(n - 1, int(0.99 * n))], selected on the device
 *   stalls_mean                       n_stalls / n_sessions
 *   stall_time_total_s                stall_time_sum: the reference's left-to-right sum in
 *                                     session registration order (metrics.py:88-92)
 *   quality_fractions / mean_rank     rank_count[r] / n_segments
 * latency_sum and startup_delay_sum are correctly rounded exact sums (== math.fsum). */
#define OTF_LAT_BINS 64      /* bin 0: latency < 10 ms (instant); then 4 bins per octave from 10 ms */
#define OTF_STALL_BINS 32    /* sessions by stall count, last bin = ">= 31" */
#define OTF_RANK_BINS 32     /* segments by representation rank (rank < 32) */
/* otf_qoe.summary_flags */
#define OTF_Q_ORDER_STATS 0x1  /* latency_p50 / latency_p99 / stall_time_sum were computed */
#define OTF_Q_INEXACT_SUM 0x2  /* a value outside [2^-76, 2^64) reached an exact sum (sum approximate) */
#define OTF_Q_RANKS_CAPPED 0x4 /* a rank >= OTF_RANK_BINS was counted in the last bin */
typedef struct otf_qoe {
    int64_t lat_hist[OTF_LAT_BINS];
    int64_t path_count[8];            /* by OTF_PATH_* */
    int64_t stall_hist[OTF_STALL_BINS];
    int64_t rank_count[OTF_RANK_BINS];
    int64_t n_requests, n_sessions, n_segments, n_finished, n_started;
    int64_t n_stalls;                 /* stall events summed over sessions */
    double latency_sum, stall_time_sum, startup_delay_sum;
    double latency_p50, latency_p99;
    int64_t n_lat_tail;               /* requests with a nonzero latency */
    int64_t n_stall_tail;             /* sessions with a nonzero stall time */
    int64_t summary_flags;            /* OTF_Q_* */
    /* n_sessions / n_started count the session records and startup delays the
     * engines kept (summary tails); the summary pass derives the rest */
} otf_qoe;

/* One closed session (summary tail): the report as _sync_report left it
 * (client.py:284-288).  Registration time and session id give the
 * registration order the reference sums stall times in. */
typedef struct otf_sess_ent {
    double reg_time;
    double stall_time;
    int32_t sid;
    uint32_t stalls;                  /* stall events | OTF_SE_FINISHED */
} otf_sess_ent;
#define OTF_SE_FINISHED 0x80000000u

/* otf_batch.engine_flags */
#define OTF_BF_ENGINE_ONLY 0x1        /* otf_run_batch skips the summary pass (run it with otf_run_summary) */

typedef struct otf_batch {
    int32_t n_scenarios;
    int32_t mode;                     /* OTF_MODE_* */
    const otf_scenario *scenarios;    /* [n_scenarios] */
    const double *f64_pool;
    const int64_t *i64_pool;
    const int32_t *i32_pool;
    uint8_t *scratch;                 /* engine state, otf_scratch_bytes() per scenario */
    /* records (MODE_RECORDS; SoA slices at otf_scenario.*_off) */
    int64_t *req_id; int32_t *req_seq, *req_rep, *req_index, *req_path;
    double *req_arrival, *req_response; int64_t *req_bytes;
    int32_t *sess_client, *sess_seq, *sess_stalls, *sess_flags;
    double *sess_start, *sess_end, *sess_stall_time, *sess_startup;
    int32_t *seg_session, *seg_index, *seg_rep; double *seg_start, *seg_end;
    int32_t *job_seq, *job_rep, *job_index, *job_origin, *job_outcome;
    double *job_enq, *job_start, *job_fin;
    /* per-scenario outputs */
    int64_t *counts;                  /* [n_scenarios][4]: requests, sessions, segments, jobs */
    int64_t *stats;                   /* [n_scenarios][OTF_ST_NSLOTS] */
    otf_qoe *qoe;                     /* [n_scenarios] */
    int32_t *status;                  /* [n_scenarios] OTF_S_* bits */
    const int32_t *order;             /* optional launch order (longest first), NULL = identity */
    int64_t shared_bytes;             /* windowed engine: dynamic shared memory per scenario
                                         (max of otf_shared_bytes over the batch) */
    int32_t engine_flags;             /* OTF_BF_* */
    int32_t concurrent;               /* scenarios resident alongside this launch (its own plus those
                                         of launches running concurrently on other streams); sizes
                                         the warps per scenario.  0 = n_scenarios */
    double *tail_lat;                 /* summary tails at otf_scenario.lat_off / ses_off / sup_off */
    otf_sess_ent *tail_sess;
    double *tail_sup;
} otf_batch;

/* A segment-size table: Catalog.descriptor sizes (content.py:204-218) for one
 * catalog, generated on the device from SeedSequence([seed, key, rank, index]). */
typedef struct otf_size_table {
    int32_t n_seq, n_ranks, max_nseg, pad;
    uint64_t seed;                    /* catalog seed (= ExperimentConfig.seed) */
    double size_jitter;
    int64_t off_out;                  /* i64 pool offset of [n_seq][n_ranks][max_nseg] */
    int64_t off_keys;                 /* i64: [n_seq] sha256(seq id)[:8] big-endian */
    int64_t off_bitrates;             /* i64: [n_ranks] */
    int64_t off_seqdur, off_segdur;   /* f64: [n_seq] */
    int64_t off_segcount;             /* i32: [n_seq] */
} otf_size_table;

int otf_version(void);
const char *otf_last_error(void);
size_t otf_sizeof_scenario(void);
size_t otf_sizeof_batch(void);
size_t otf_sizeof_qoe(void);

/* Engine scratch bytes for one scenario (host-side layout helper). */
int64_t otf_scratch_bytes(int32_t engine, int32_t n_clients, int32_t n_workers, int32_t n_seq,
                          int32_t n_ranks, int32_t max_nseg);

/* 1 if the scenario (HOST pointer) is inside `engine`'s limits, else 0.  The
 * windowed engine has fixed-width ids (see OTF_S_UNFIT); the exact engine
 * takes every scenario.  Shared memory is checked separately against the
 * device's opt-in limit (otf_shared_bytes). */
int32_t otf_engine_fits(int32_t engine, const otf_scenario *sc);

/* Per-scenario dynamic shared memory of the windowed engine (host-side helper),
 * with the default server-event list capacity (otf_list_cap). */
int64_t otf_shared_bytes(int32_t engine, int32_t n_clients, int32_t n_workers, int32_t n_seq,
                         int32_t n_ranks, int32_t max_nseg);
/* The same with an explicit list capacity (otf_scenario.list_cap > 0). */
int64_t otf_shared_bytes_cap(int32_t n_clients, int32_t n_seq, int32_t n_ranks, int32_t max_nseg, int32_t list_cap);
/* The windowed engine's default server-event list capacity for n_clients. */
int32_t otf_list_cap(int32_t n_clients);

/* HOST function: synthetic traces (netem.py:179-202) + BandwidthTrace period
 * bits (netem.py:39-64) from numpy's standard-normal draws.  normals is
 * [n_traces][n_samples + 1]; starts is [n_samples]; values is
 * [n_traces][n_samples]; pbits [n_traces].  Uses glibc exp() (== math.exp)
 * and CPython 3.12's compensated sum(), so the values are bit-identical to
 * the reference's BandwidthTrace. Host pointers. */
int otf_build_traces(int64_t n_traces, int32_t n_samples, const double *normals, const double *starts,
                     double period, double mu, double sigma, double decay, double spread,
                     double floor_bps, double cap_bps, double *values, double *pbits, int32_t n_threads);

/* ---- HOST input generators: numpy Generator(PCG64(SeedSequence(entropy)))
 * streams replayed bit-for-bit (numpy 2.3.5 SeedSequence, PCG64, ziggurat
 * normal / exponential), multithreaded over independent streams.  They replace
 * the reference's per-run numpy draws; host pointers. ---- */
enum {
    OTF_DRAW_STANDARD_NORMAL = 0,     /* Generator.standard_normal(n) */
    OTF_DRAW_NORMAL = 1,              /* Generator.normal(loc, scale, n) */
    OTF_DRAW_EXPONENTIAL = 2,         /* Generator.exponential(scale, n) */
    OTF_DRAW_STANDARD_EXPONENTIAL = 3 /* Generator.standard_exponential(n) */
};

/* n draws of `kind` from Generator(PCG64(SeedSequence(entropy[0..n_entropy)))). */
int otf_np_draws(int32_t kind, const uint64_t *entropy, int32_t n_entropy, double loc, double scale, int64_t n,
                 double *out);

/* ExperimentConfig.arrival_offsets (orchestrator.py:265-268):
 * out = cumsum(SS([seed, 1]).exponential(scale, n)), sequential. */
int otf_gen_arrivals(uint64_t seed, int64_t n, double scale, double *out);

/* ServiceSampler noise (transcode.py:89-99): out[w][0..n) = SS([seed, w]).normal(0, noise, n). */
int otf_gen_noise(uint64_t seed, int32_t n_workers, double noise, int64_t n, double *out, int32_t n_threads);

/* ExperimentConfig.trace_for + synthetic_trace + BandwidthTrace (orchestrator.py:254-263,
 * netem.py:179-202,39-64) for clients 0..n_traces-1 of `seed`: normals from
 * SS([seed, 2, c]), then as otf_build_traces. */
int otf_gen_traces(uint64_t seed, int64_t n_traces, int32_t n_samples, const double *starts, double period,
                   double mu, double sigma, double decay, double spread, double floor_bps, double cap_bps,
                   double *values, double *pbits, int32_t n_threads);

/* Many trace tables in one parallel region (one per (seed, netem) of a sweep):
 * job q = otf_gen_traces(seed, n_traces, ...) for clients 0..n_traces-1. */
typedef struct otf_trace_job {
    uint64_t seed;
    int64_t n_traces;
    int32_t n_samples, pad;
    const double *starts;
    double period, mu, sigma, decay, spread, floor_bps, cap_bps;
    double *values;                   /* [n_traces][n_samples] */
    double *pbits;                    /* [n_traces] */
} otf_trace_job;
int otf_gen_traces_multi(int32_t n_jobs, const otf_trace_job *jobs, int32_t n_threads);

/* ---- the per-client model functions (csrc/otf_model.cuh) on their own, for
 * validation against the reference's known answers (tests/test_model_kat.py) ---- */

/* BandwidthTrace.completion_time (netem.py:77-118) over a looping trace of n
 * pieces; grid > 0 when starts[i] == i * grid exactly.  HOST pointers. */
double otf_model_completion_time(const double *starts, const double *values, int32_t n, double period, double pbits,
                                 double grid, double start, int64_t nbytes);

/* select_quality (client.py:134-146); bitrates[r-1] is rank r, top = n ranks. */
int32_t otf_model_select_quality(double level, int32_t cur, int32_t has_est, double est, const int64_t *bitrates,
                                 int32_t top, double panic, double safe, double headroom);

/* PlayerBuffer (client.py:74-121) from buf_reset(t0): op[i] = 1 -> on_segment(t[i],
 * dur[i]), 0 -> advance(t[i]); out[i][6] = level, phase (0 startup, 1 playing,
 * 2 stalled), stall events, stall time, started_at (NaN until playback), last sync. */
int otf_model_buffer_run(double t0, int32_t n, const int32_t *op, const double *t, const double *dur, double startup,
                         double resume, double *out);

/* HOST: the engines' exact sum (csrc/otf_xacc.cuh) of n non-negative doubles:
 * the correctly rounded sum (== math.fsum) or, with a value outside
 * [2^-76, 2^64), returns 1 (*out is then the sum of the covered values). */
int otf_model_exact_sum(const double *v, int64_t n, double *out);

/* DEVICE: completion_time for n (start, nbytes) queries over one trace (device
 * pointers), as the engines compute it (--fmad=false). */
int otf_model_completion_times(const double *starts, const double *values, int32_t n_samples, double period,
                               double pbits, double grid, const double *start, const int64_t *nbytes, int32_t n,
                               double *out, void *stream);

/* DEVICE: fill segment-size tables (one thread per entry). */
int otf_gen_sizes(const otf_size_table *tables_dev, int32_t n_tables, int64_t total_entries,
                  int64_t *i64_pool, const double *f64_pool, const int32_t *i32_pool, void *stream);

/* ---- DEVICE request generation: the reference's seeded numpy streams
 * replayed on the GPU (csrc/otf_gen.cu), bit-identical to the host
 * generators above (same otf_npdist.cuh / otf_libm.cuh arithmetic).  One
 * thread per stream; a batch of jobs runs as one launch.  Offsets index the
 * f64 pool (device pointer). ---- */
enum {
    OTF_GEN_TRACE = 0,     /* synthetic_trace + BandwidthTrace (netem.py:179-202,39-64): n_streams clients,
                              stream c = SS([seed, 2, c]).standard_normal; values [c][n], period bits [c] */
    OTF_GEN_ARRIVALS = 1,  /* arrival_offsets (orchestrator.py:265-268): cumsum(SS([seed, 1]).exponential(scale, n)) */
    OTF_GEN_NOISE = 2      /* ServiceSampler eps (transcode.py:89-99): [w][0..n) = SS([seed, w]).normal(0, scale, n) */
};
typedef struct otf_gen_job {
    int32_t kind;                     /* OTF_GEN_* */
    int32_t n;                        /* samples per trace / arrivals / draws per worker */
    int64_t n_streams;                /* traces (clients) / 1 / workers */
    int64_t first_stream;             /* sum of n_streams over the jobs before this one */
    uint64_t seed;
    int64_t off_out;                  /* f64: [n_streams][n] */
    int64_t off_pbits;                /* f64: [n_streams] trace period bits */
    int64_t off_starts;               /* f64: [n] trace sample starts */
    double period, mu, sigma, decay, spread, floor_bps, cap_bps;   /* trace parameters */
    double scale;                     /* arrivals: 1 / rate; noise: noise_rel_std */
} otf_gen_job;

/* DEVICE: run n_jobs generator jobs (device array) into f64_pool.  Job q's
 * streams are threads first_stream .. first_stream + n_streams - 1; every
 * first_stream is a multiple of OTF_GEN_ALIGN and increases with q;
 * total_streams = the last job's first_stream + n_streams. */
#define OTF_GEN_ALIGN 128
int otf_gen_tables(const otf_gen_job *jobs_dev, int32_t n_jobs, int64_t total_streams, double *f64_pool,
                   void *stream);

/* glibc's exp (fn 0) / log1p (fn 1) as restated in csrc/otf_libm.cuh, for
 * validation: otf_model_libm on HOST pointers (host build of the restatement),
 * otf_model_libm_dev on DEVICE pointers (the device build the generators use). */
int otf_model_libm(int32_t fn, const double *x, int64_t n, double *out);
int otf_model_libm_dev(int32_t fn, const double *x, int64_t n, double *out, void *stream);

/* DEVICE: run every scenario of the batch to its horizon (sim.py:347-360), then
 * the summary pass: order statistics of the latency tail and the
 * registration-order stall sum into each scenario's otf_qoe. */
int otf_run_batch(const otf_batch *batch, int32_t engine, void *stream);

/* DEVICE: the summary pass alone (after an OTF_BF_ENGINE_ONLY otf_run_batch on
 * the same stream); `engine` is the engine that produced the tails. */
int otf_run_summary(const otf_batch *batch, int32_t engine, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* OTFGPU_H */
