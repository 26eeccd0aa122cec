// otf_model.cuh -- per-client model functions shared by both engines.
//
// Each function restates one reference function with its exact operation
// order (the library is compiled with --fmad=false so every double op rounds
// like CPython's):
//   completion_time / drain_from  netem.py:77-118
//   buf_advance / buf_on_segment  client.py:91-121
//   select_quality                client.py:134-146
//   segment duration              client.py:264, content.py:214
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "otfgpu.h"

// Loops that run 1-2 times are kept rolled: the engine is sensitive to its hot
// code size (instruction fetch is a third of its stall samples).
#if defined(__CUDA_ARCH__) && !defined(OTF_UNROLL_OK)
#define OTF_NOUNROLL _Pragma("unroll 1")
#else
#define OTF_NOUNROLL
#endif

#ifndef OTF_HD
#define OTF_HD __host__ __device__ __forceinline__
#endif

namespace otf {

#ifdef __CUDA_ARCH__
OTF_HD double __longlong_as_double_hd(long long v) { return __longlong_as_double(v); }
OTF_HD long long __double_as_longlong_hd(double v) { return __double_as_longlong(v); }
#else
OTF_HD double __longlong_as_double_hd(long long v) { double d; memcpy(&d, &v, 8); return d; }
OTF_HD long long __double_as_longlong_hd(double v) { long long l; memcpy(&l, &v, 8); return l; }
#endif

enum { PH_STARTUP = 0, PH_PLAYING = 1, PH_STALLED = 2, PH_FINISHED = 3 };

struct Trace {
    const double *starts;   // [n]
    const double *values;   // [n]
    double period, pbits;
    double grid;            // > 0: starts[i] == i * grid exactly
    double inv_grid;        // 1 / grid (an estimate's multiplier; exactness comes from the fix-up)
    int32_t n;
};

// bisect_right(starts, phase) - 1, clamped at 0 (netem.py:80)
OTF_HD int32_t trace_piece(const Trace &tr, double phase) {
    if (tr.grid > 0) {
        double q = phase * tr.inv_grid;                // estimate; the two loops below make it exact
        int32_t i = q < (double)tr.n ? (int32_t)q : tr.n - 1;
        if (i < 0) i = 0;
        OTF_NOUNROLL
        while (i + 1 < tr.n && (double)(i + 1) * tr.grid <= phase) i++;
        OTF_NOUNROLL
        while (i > 0 && (double)i * tr.grid > phase) i--;
        return i;
    }
    int32_t lo = 0, hi = tr.n;
    while (lo < hi) {
        int32_t mid = (lo + hi) >> 1;
        if (phase < tr.starts[mid]) hi = mid; else lo = mid + 1;
    }
    return lo > 0 ? lo - 1 : 0;
}

OTF_HD double piece_start(const Trace &tr, int32_t i) {
    return tr.grid > 0 ? (double)i * tr.grid : tr.starts[i];
}

// The first two samples a drain from `phase` reads: a caller may issue these
// loads before it knows the byte count (completion_time_at).
struct TraceAhead {
    double phase, v0, v1;
    int32_t i;
};

OTF_HD TraceAhead trace_ahead(const Trace &tr, double phase) {
    TraceAhead a;
    a.phase = phase;
    a.i = trace_piece(tr, phase);
    a.v0 = a.i < tr.n ? tr.values[a.i] : 0.0;
    a.v1 = a.i + 1 < tr.n ? tr.values[a.i + 1] : 0.0;
    return a;
}

// BandwidthTrace._drain_from (netem.py:77-95) from piece a.i, whose sample and
// the next one are already loaded; later samples load two pieces ahead.
OTF_HD void drain_from_at(const Trace &tr, const TraceAhead &a, double bits, double &spent_out, double &left_out) {
    int32_t i = a.i;
    double spent = 0.0, pos = a.phase;
    double v_here = a.v0, v_next = a.v1;
    OTF_NOUNROLL
    for (; i < tr.n; i++) {
        double seg_end = (i + 1 < tr.n) ? piece_start(tr, i + 1) : tr.period;
        double width = seg_end - pos;
        if (width > 0) {
            double v = v_here;
            if (v > 0) {
                if (v * width >= bits) { spent_out = spent + bits / v; left_out = 0.0; return; }
                bits -= v * width;
            }
            spent += width;
            pos = seg_end;
        }
        v_here = v_next;
        if (i + 2 < tr.n) v_next = tr.values[i + 2];
    }
    spent_out = spent;
    left_out = bits;
}

OTF_HD void drain_from(const Trace &tr, double phase, double bits, double &spent_out, double &left_out) {
    drain_from_at(tr, trace_ahead(tr, phase), bits, spent_out, left_out);
}

// fmod(start, period) == start for 0 <= start < period (exact)
OTF_HD double trace_phase(const Trace &tr, double start) {
    return (start >= 0.0 && start < tr.period) ? start : fmod(start, tr.period);
}

// The rest of a transfer that outlasts the trace's end (netem.py:109-118): whole
// periods, then a drain from phase 0.  Rare, so kept out of line (scalar arguments).
#ifdef __CUDA_ARCH__
static __device__ __noinline__
#else
static inline
#endif
double completion_wrap(const double *starts, const double *values, int32_t n, double period, double pbits,
                       double grid, double inv_grid, double t, double left) {
    const Trace tr{starts, values, period, pbits, grid, inv_grid, n};
    double whole = floor(left / tr.pbits);
    t += whole * tr.period;
    left -= whole * tr.pbits;
    if (left <= 0) return t;
    double spent;
    drain_from(tr, 0.0, left, spent, left);
    return t + spent;
}

// BandwidthTrace.completion_time for a looping trace (netem.py:97-118), the
// first drain starting from a = trace_ahead(tr, trace_phase(tr, start)).
OTF_HD double completion_time_at(const Trace &tr, const TraceAhead &a, double start, int64_t nbytes) {
    double bits = (double)nbytes * 8.0;
    if (bits <= 0) return start;
    if (tr.pbits <= 0) return INFINITY;
    double t = start, spent, left;
    drain_from_at(tr, a, bits, spent, left);
    t += spent;
    if (left <= 0) return t;
    return completion_wrap(tr.starts, tr.values, tr.n, tr.period, tr.pbits, tr.grid, tr.inv_grid, t, left);
}

OTF_HD double completion_time(const Trace &tr, double start, int64_t nbytes) {
    return completion_time_at(tr, trace_ahead(tr, trace_phase(tr, start)), start, nbytes);
}

struct Buffer {
    double level, last_sync, stall_time, started_at, session_start;   // (position is never observed)
    int32_t phase, stall_events;
};

// PlayerBuffer.advance (client.py:91-112)
OTF_HD void buf_advance(Buffer &b, double now) {
    double dt = now - b.last_sync;
    b.last_sync = now;
    if (b.phase == PH_PLAYING) {
        if (b.level >= dt - 1e-9) {
            double l = b.level - dt;
            b.level = (l > 0.0) ? l : 0.0;
        } else {
            double played = b.level;
            b.level = 0.0;
            b.phase = PH_STALLED;
            b.stall_events++;
            b.stall_time += dt - played;
        }
    } else if (b.phase == PH_STALLED) {
        b.stall_time += dt;
    }
}

// PlayerBuffer.on_segment (client.py:114-121)
OTF_HD void buf_on_segment(Buffer &b, double now, double duration, double startup, double resume) {
    buf_advance(b, now);
    b.level += duration;
    if (b.phase == PH_STARTUP && b.level >= startup) {
        b.phase = PH_PLAYING;
        b.started_at = now;
    } else if (b.phase == PH_STALLED && b.level >= resume) {
        b.phase = PH_PLAYING;
    }
}

OTF_HD void buf_reset(Buffer &b, double now) {
    b.level = 0.0; b.last_sync = now; b.stall_time = 0.0;
    b.started_at = NAN; b.session_start = now; b.phase = PH_STARTUP; b.stall_events = 0;
}

// select_quality (client.py:134-146); bitrates[r-1] is rank r.
OTF_HD int32_t select_quality(double level, int32_t cur, bool has_est, double est, const int64_t *bitrates,
                              int32_t top, double panic, double safe, double headroom) {
    if (level < panic) return 1;
    if (level < safe) return cur - 1 > 1 ? cur - 1 : 1;
    if (cur < top && has_est && est >= (double)bitrates[cur] * headroom) return cur + 1;
    return cur;
}

// min(segdur, duration - index * segdur)  (client.py:264, content.py:214)
OTF_HD double seg_duration(double seqdur, double segdur, int32_t index) {
    double rem = seqdur - (double)index * segdur;
    return rem < segdur ? rem : segdur;
}

// Latency histogram bin: 0 = instant (< 10 ms, metrics.py:38,77), then 4 bins
// per octave with lower edges 0.01 * (1 + q/4) * 2^o (exact in double).
OTF_HD double pow2i(int o) {                           // 2^o for 0 <= o < 1024, exact
    return __longlong_as_double_hd((long long)(o + 1023) << 52);
}
OTF_HD double lat_edge(int k) {                        // lower edge of bin 1 + k
    return (0.01 * (1.0 + 0.25 * (double)(k & 3))) * pow2i(k >> 2);
}
OTF_HD int lat_bin(double lat) {
    if (lat < 0.010) return 0;
    double x = lat * 100.0;                            // estimate of lat / 0.01; exact edges decide
    long long bitsx = __double_as_longlong_hd(x);
    int e = (int)((bitsx >> 52) & 0x7ff) - 1023;
    int k = e * 4 + (int)((bitsx >> 50) & 3);
    if (k < 0) k = 0;
    if (k > OTF_LAT_BINS - 2) k = OTF_LAT_BINS - 2;
    OTF_NOUNROLL
    while (k + 1 <= OTF_LAT_BINS - 2 && lat >= lat_edge(k + 1)) k++;
    OTF_NOUNROLL
    while (k > 0 && lat < lat_edge(k)) k--;
    return 1 + k;
}

}  // namespace otf
