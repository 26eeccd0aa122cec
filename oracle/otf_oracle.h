/* otf_oracle.h -- TEST INFRASTRUCTURE ONLY (see otf_oracle.c). */
#ifndef OTF_ORACLE_H
#define OTF_ORACLE_H
#include <stdint.h>

enum { PATH_STORAGE = 0, PATH_CACHE = 1, PATH_WAITED = 2, PATH_TRANSCODED = 3, PATH_ERROR = 4 };
enum { ORIGIN_DEMAND = 0, ORIGIN_SPEC = 1 };
enum { OUT_PENDING = 0, OUT_COMPLETED = 1, OUT_DROPPED = 2, OUT_FAILED = 3 };
enum { POP_UNIFORM = 0, POP_ZIPF = 1 };
enum { SESS_FINISHED = 1, SESS_ABORTED = 2 };
enum { ORACLE_OK = 0, ORACLE_EOVERFLOW = 2 };

/* stats[] slots (backend.py:228-239, cache.py:83-92) */
enum {
    ST_JOBS_TOTAL = 0, ST_JOBS_DEMAND, ST_JOBS_SPEC, ST_WASTED, ST_SPEC_ENQUEUED,
    ST_SKIP_DISABLED, ST_SKIP_EOS, ST_SKIP_STORED, ST_SKIP_CACHED, ST_SKIP_INFLIGHT, ST_SKIP_OVERLOAD,
    ST_CACHE_CAPACITY, ST_CURRENT_BYTES, ST_ENTRIES, ST_HITS, ST_MISSES, ST_EVICTIONS, ST_REJECTED,
    ST_STATUS, ST_HUNG, ST_TIMER_POPS, ST_READY_CALLBACKS,
    ST_NSLOTS = 32
};

typedef struct {
    int32_t n_clients, n_workers, n_seq, n_ranks, max_nseg, n_samples;
    int32_t cache_enabled, spec_enabled, popularity, pad0;
    uint32_t stored_mask, pad1;           /* bit r set <=> rank r stored */
    int64_t cache_capacity;
    uint64_t seed, catalog_seed;
    double horizon, latency, target, safe, panic, resume, startup, alpha, headroom, noise;
    double size_jitter;
    double trace_mu, trace_sigma, trace_decay, trace_spread, trace_floor, trace_cap;
    double trace_step, trace_duration;
    const int64_t *bitrates;        /* [n_ranks], rank r at r-1 */
    const double *rho;              /* [n_ranks] */
    const double *seq_duration;     /* [n_seq] */
    const double *seq_segdur;       /* [n_seq] */
    const int64_t *seq_key;         /* [n_seq] sha256(id)[:8] big-endian */
    const int64_t *manifest_bytes;  /* [n_seq] */
    const double *arrival_draws;    /* [n_clients] exponential draws, cumsum done here */
    const double *trace_normals;    /* [n_clients][n_samples + 1] */
    const double *zipf_cdf;         /* [n_seq] */
    const double *eps;              /* [n_workers][eps_per_worker] */
    int64_t eps_per_worker;
    int32_t queue_bound, retries;   /* BackendPolicy.queue_bound, ClientConfig.retries */
    double retry_backoff;           /* ClientConfig.retry_backoff_s */
    int32_t demand_priority, pad2;  /* BackendPolicy.demand_priority */
    /* CSV traces (netem.trace_dir): per-client trace tables, else NULL (synthetic traces) */
    const double *tr_starts, *tr_values, *tr_period, *tr_pbits;  /* tables; [N] period, pbits */
    const int64_t *tr_off;          /* [N] offset of the client's trace in tr_starts/tr_values */
    const int32_t *tr_n;            /* [N] samples */
} oracle_scenario;

typedef struct {
    int64_t req_cap, sess_cap, seg_cap, job_cap;
    int64_t *req_id; int32_t *req_seq, *req_rep, *req_index, *req_path;
    double *req_arrival, *req_response; int64_t *req_bytes;
    int32_t *sess_client, *sess_seq, *sess_stalls, *sess_flags;
    double *sess_start, *sess_end, *sess_stall_time, *sess_startup;
    int32_t *seg_session, *seg_index, *seg_rep; double *seg_start, *seg_end;
    int32_t *job_seq, *job_rep, *job_index, *job_origin, *job_outcome;
    double *job_enq, *job_start, *job_fin;
    int64_t n_req, n_sess, n_seg, n_job;
    int64_t stats[ST_NSLOTS];
} oracle_outputs;

int oracle_sample_times(double duration, double step, double *starts, int cap);
int oracle_segment_sizes(const oracle_scenario *sc, int64_t *sizes, int32_t *counts);
int oracle_build_traces(const oracle_scenario *sc, double *values, double *pbits, double *period);
int oracle_run(const oracle_scenario *sc, oracle_outputs *out);
/* glibc exp (fn 0) / log1p (fn 1) over n values: the libm the reference and
 * numpy call, as the checker for the library's restatement (csrc/otf_libm.cuh). */
int oracle_libm(int fn, const double *x, int64_t n, double *out);

#endif
