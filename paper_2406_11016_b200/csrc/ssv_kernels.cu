// ssv_kernels.cu -- sm_100a kernels of the speculative-sampling verification step.
//
// k_verify<T, ACT> is the whole step in ONE persistent, warp-specialized
// launch (DESIGN.md has the derivation and the roofline):
//
//   producer warp   claims work items in order from a global counter and
//                   streams their bytes into a kStages-deep ring of shared-
//                   memory stages with TMA bulk copies (cp.async.bulk, 16-byte
//                   aligned supersets of misaligned rows) completing on mbarriers.
//   consumer warps  (8) drain the ring:
//     A-item  (exact only) one chunk of one drafted p/q row: CTA max, fp32 ex2
//             sums with fp64 carries -> chunk partial (m, s); the logit at the
//             drafted token is picked out of the stage.  The consumer group
//             that completes batch row b's LAST A-item folds the partials into
//             row statistics, evaluates tau at every drafted position in fp64,
//             runs the first-rejection scan and publishes the decision
//             (release flag, tagged with the launch epoch).
//     D-item  (sigmoid / probabilities) the same decision from the B*gamma
//             gathered logits alone -- no row reductions (paper section 3.2.2).
//     B-item  one slice of the ONE row (bonus) or row PAIR (rejected position)
//             batch row b still needs; the producer waits for b's decision
//             before fetching it.  Each consumer warp reduces one granule to
//             its residual mass max(0, p - q) (or p mass / (m, s) for the bonus
//             row).  B-items of b are ordered after the A-items of b + lag, so
//             the rejected pair is re-read from L2, not HBM.
//             The group completing b's LAST B-item runs the inverse CDF: fp64
//             granule prefix from SMEM, then an exact fp64 scan inside the
//             selected granule (dist.cpp:122-137, incl. its fallbacks).
//
// Every reduction has a fixed topology, so results are bit-identical run to
// run.  k_materialize (optional p / q / residual grids) and the synthetic-input
// generator follow.
#include <algorithm>
#include <type_traits>

#include "ssv_launch.h"
#include "ssv_device.cuh"
#include "ssv_pipe.cuh"

namespace ssv {

constexpr int kCons = 256;                 // consumer threads (8 warps)
constexpr int kConsWarps = kCons / 32;
constexpr int kBlock = kCons + 32;         // + one producer warp

// Work-item phases of one batch row, in dependency order.
enum ItemType : int { IT_A = 0, IT_D = 1, IT_B = 2, IT_L = 3, IT_STOP = 4 };
constexpr int kMaxRowsSmem = 96;  // row statistics a decide keeps in SMEM (gamma <= 47)

constexpr int kMaxRunA = 64;  // chunks per A-run (row-statistics run)
constexpr int kMaxRunB = 8;   // slices per B-run (residual / bonus run)
constexpr int kCtx = 8;       // run contexts (runs in flight per CTA; see RunInfo)

// Work-item description handed from producer to consumers.  A- and B-items
// are RUNS of consecutive chunks of one row; a run is streamed one 16 KB chunk
// per ring stage.
struct Item {
    int type, b;
    int r, q;            // A: stat row, run index within the row; B: run index
    int mode, row;       // B / L: decision
    double Mp, Sp, Mq, Sq;
};

// One ring slot (16 bytes for A/B chunks; D/L items also carry the decision).
struct Slot {
    int type, ctx, pos, b;
    int mode, row, pad0, pad1;
    double Mp, Sp, Mq, Sq;
};

// Per-run constants (written once by the producer before the run's first
// chunk is published) and the consumers' fold state.  kCtx contexts: consumer
// warps can be at most kStages chunks apart (a stage is refilled only after
// all 8 warps released it), so a context is free again long before the
// producer reuses it kCtx runs later.
struct RunInfo {
    int type, b, r, q, len, k0;  // k0: first chunk (A) / slice (B) of the run
    int mode, row, shift_p, shift_q;
    double Mp, Sp, Mq, Sq;
    double2 wpart[kConsWarps];   // A: warp partials (max, sum) of the run
    double wmin[kConsWarps];
    double2 gpart[kMaxRunB * kConsWarps];  // B: granule partials of the run
    unsigned cnt;                // warps done with the run
};

// ---------------------------------------------------------------------------
// Row addressing.  Stat rows of batch row b: r < G -> p row r, G <= r < 2G ->
// q row r-G, r == 2G -> p row G (bonus, only when p is materialized).
template <typename T>
__device__ __forceinline__ const T* p_row(const StepParams& P, int b, int c) {
    return reinterpret_cast<const T*>(P.zp) + ((size_t)b * P.PS + c) * (size_t)P.V;
}
template <typename T>
__device__ __forceinline__ const T* q_row(const StepParams& P, int b, int c) {
    return reinterpret_cast<const T*>(P.zq) + ((size_t)b * P.G + c) * (size_t)P.V;
}
template <typename T>
__device__ __forceinline__ const T* stat_row(const StepParams& P, int b, int r) {
    if (r < P.G) return p_row<T>(P, b, r);
    if (r < 2 * P.G) return q_row<T>(P, b, r - P.G);
    return p_row<T>(P, b, P.G);
}

__device__ __forceinline__ void flag(const StepParams& P, uint32_t bits) { atomicOr(P.status, bits); }

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Diagnostics: phase timestamps (ns) when a trace buffer is attached.
__device__ __forceinline__ void trace(const StepParams& P, int idx) {
    if (P.trace) P.trace[idx] = gtime();
}

__device__ __forceinline__ double ratio_clamped(double p, double q) {  // dist.cpp:104-112
    if (q <= kZeroEps) return p > kZeroEps ? 1.0 : 0.0;
    return fmin(1.0, p / q);
}

// ---- consumer-group collectives (named barrier 1, 256 threads) -------------
template <typename V, typename Op>
__device__ __forceinline__ V creduce(V v, V* sm, Op op) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(kFull, v, o));
    cbar<kCons>();
    if (lane == 0) sm[warp] = v;
    cbar<kCons>();
    V r = sm[0];
#pragma unroll
    for (int w = 1; w < kConsWarps; ++w) r = op(r, sm[w]);
    return r;
}

__device__ __forceinline__ double cscan_incl(double v, double* sm, double& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double incl = warp_scan_incl(v);
    cbar<kCons>();
    if (lane == 31) sm[warp] = incl;
    cbar<kCons>();
    double off = 0.0, tot = 0.0;
#pragma unroll
    for (int w = 0; w < kConsWarps; ++w) {
        if (w < warp) off += sm[w];
        tot += sm[w];
    }
    total = tot;
    return off + incl;
}

template <typename T>
__device__ __forceinline__ typename Elem<T>::acc lds_elem(const uint8_t* base, int i) {
    return (typename Elem<T>::acc)load_smem_elem(reinterpret_cast<const T*>(base) + i);
}

// ---------------------------------------------------------------------------
// Work-item order.  Segment t holds, in order, the A-items of batch row t,
// the decide item of t - off[1], the B-items of t - off[2] and the locate item
// of t - off[3] (each only if that row exists).  Items only ever wait on items
// with a smaller index -- claimed earlier by a running CTA -- so the schedule
// cannot deadlock, and the lags keep the waits short and the rejected pair of
// row b L2-resident when its B-items stream it again.
__device__ __forceinline__ int seg_size(const StepParams& P, int t) {
    int n = 0;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const int b = t - P.off[p];
        if (b >= 0 && b < P.B) n += P.nph[p];
    }
    return n;
}

// Position of an item: segment t, phase p, index a within the phase.
struct Cursor {
    int t, p, a;
};

__device__ __forceinline__ bool phase_active(const StepParams& P, int t, int p) {
    const int b = t - P.off[p];
    return P.nph[p] > 0 && b >= 0 && b < P.B;
}

// First active phase of segment t at or after phase p (p may be 4: next segment).
__device__ __forceinline__ void settle(const StepParams& P, Cursor& c) {
    const int tend = P.B + P.off[3];
    while (c.t < tend) {
        while (c.p < 4 && !phase_active(P, c.t, c.p)) ++c.p;
        if (c.p < 4) return;
        ++c.t;
        c.p = 0;
        c.a = 0;
    }
}

__device__ __forceinline__ Cursor decode_cursor(const StepParams& P, unsigned i) {
    Cursor c{P.B + P.off[3], 0, 0};  // past the end
    if (i >= P.n_items) return c;
    unsigned cum = 0;
    int o = 0;
    for (int q = 0; q + 1 < P.nbp; ++q) {
        const int x = P.bp[q], y = P.bp[q + 1];
        const int sz = seg_size(P, x);
        const unsigned cnt = (unsigned)(y - x) * (unsigned)sz;
        if (sz > 0 && i < cum + cnt) {
            c.t = x + (int)((i - cum) / (unsigned)sz);
            o = (int)((i - cum) % (unsigned)sz);
            break;
        }
        cum += cnt;
    }
    c.p = 0;
    c.a = 0;
    for (int p = 0; p < 4; ++p) {
        if (!phase_active(P, c.t, p)) continue;
        if (o < P.nph[p]) {
            c.p = p;
            c.a = o;
            return c;
        }
        o -= P.nph[p];
    }
    return c;
}

__device__ __forceinline__ void advance(const StepParams& P, Cursor& c) {
    if (++c.a < P.nph[c.p]) return;
    c.a = 0;
    ++c.p;
    settle(P, c);
}

__device__ __forceinline__ void cursor_item(const StepParams& P, const Cursor& c, Item& it) {
    it.type = IT_STOP;
    if (c.t >= P.B + P.off[3]) return;
    it.type = c.p;
    it.b = c.t - P.off[c.p];
    if (c.p == IT_A) {
        it.r = c.a / P.RPR;
        it.q = c.a - it.r * P.RPR;
    } else {
        it.q = c.a;
    }
}

// Bulk-copy the 16-byte-aligned superset of [lo, hi) of `row` into dst;
// returns the copied bytes and the element shift of `lo` inside it.
template <typename T>
__device__ __forceinline__ uint32_t stage_range(const T* row, int lo, int hi, uint8_t* dst, uint64_t* bar,
                                                int& shift) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(row + lo);
    const uintptr_t a1 = reinterpret_cast<uintptr_t>(row + hi);
    const uintptr_t s0 = a0 & ~uintptr_t(15), s1 = (a1 + 15) & ~uintptr_t(15);
    shift = (int)((a0 - s0) / sizeof(T));
    const uint32_t bytes = (uint32_t)(s1 - s0);
    bulk_g2s(dst, reinterpret_cast<const void*>(s0), bytes, bar);
    return bytes;
}

template <typename T>
__device__ __forceinline__ uint32_t staged_bytes(const T* row, int lo, int hi) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(row + lo);
    const uintptr_t a1 = reinterpret_cast<uintptr_t>(row + hi);
    return (uint32_t)(((a1 + 15) & ~uintptr_t(15)) - (a0 & ~uintptr_t(15)));
}

// ---------------------------------------------------------------------------
// Producer: lane 0 of the last warp.  Claims kClaim items per atomic, waits
// for an item's dependencies (acquire loads of the completion counters and the
// decision flag), then fills the next ring stage: TMA bulk copies for A- and
// B-items, a bare arrive for decide / locate items.
__device__ __forceinline__ void wait_eq(const unsigned* p, unsigned v) {
    while (ld_acquire(p) != v) __nanosleep(32);
}

__device__ __forceinline__ bool load_decision(const StepParams& P, Item& it) {
    if (P.sample_mode) {
        it.mode = MODE_BONUS;
        it.row = 0;
        it.Mp = it.Mq = 0.0;
        it.Sp = it.Sq = 1.0;
        return true;
    }
    wait_eq(&P.flag[it.b], P.epoch);
    const Decision* d = &P.dec[it.b];
    it.mode = __ldcg(&d->mode);
    if (it.mode == MODE_NONE) return false;
    it.row = __ldcg(&d->row);
    it.Mp = __ldcg(&d->Mp);
    it.Sp = __ldcg(&d->Sp);
    it.Mq = __ldcg(&d->Mq);
    it.Sq = __ldcg(&d->Sq);
    return true;
}

template <typename T, int ACT>
__device__ void producer(const StepParams& P, uint8_t* stages, uint64_t* full, uint64_t* empty, Slot* slots,
                         RunInfo* runs) {
    constexpr int CA = kStageBytes / (int)sizeof(T);
    unsigned cur = atomicAdd(P.next, 1u);
    unsigned nxt = atomicAdd(P.next, 1u);  // next item, claimed one ahead
    if (P.trace) P.trace[2 * gridDim.x + 4 * P.B + blockIdx.x] = cur;
    unsigned n = 0, runseq = 0;
    auto stage = [&](unsigned& sidx) -> uint8_t* {
        const unsigned s = n % kStages, ph = (n / kStages) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        sidx = s;
        return stages + (size_t)s * kStageStride;
    };
    for (;;) {
        Item it;
        cursor_item(P, decode_cursor(P, cur), it);
        cur = nxt;
        nxt = atomicAdd(P.next, 1u);
        if (it.type == IT_D) {
            if (ACT == ACT_SOFTMAX && !P.sample_mode) wait_eq(&P.cnt1[it.b], (unsigned)P.nph[IT_A]);
        } else if (it.type == IT_B) {
            if (!load_decision(P, it)) continue;
        } else if (it.type == IT_L) {
            if (!load_decision(P, it)) continue;
            wait_eq(&P.cnt2[it.b], (unsigned)P.nph[IT_B]);
        }
        if (it.type == IT_A || it.type == IT_B) {
            const int c = (int)(runseq++ % kCtx);
            RunInfo& ri = runs[c];
            const T* pr;
            const T* qr = nullptr;
            int k0, k1, step;
            if (it.type == IT_A) {
                pr = stat_row<T>(P, it.b, it.r);
                k0 = it.q * P.runA;
                k1 = min(k0 + P.runA, P.K);
                step = CA;
            } else {
                pr = p_row<T>(P, it.b, it.row);
                if (it.mode == MODE_REJECT) qr = q_row<T>(P, it.b, it.row);
                k0 = it.q * P.runB;
                k1 = min(k0 + P.runB, P.nBi);
                step = P.CB;
            }
            // chunk starts are 16 KB / 8 KB apart: the misalignment is constant per row
            ri.type = it.type;
            ri.b = it.b;
            ri.r = it.r;
            ri.q = it.q;
            ri.len = k1 - k0;
            ri.k0 = k0;
            ri.mode = it.mode;
            ri.row = it.row;
            ri.Mp = it.Mp;
            ri.Sp = it.Sp;
            ri.Mq = it.Mq;
            ri.Sq = it.Sq;
            ri.shift_p = (int)((reinterpret_cast<uintptr_t>(pr + (size_t)k0 * step) & 15) / sizeof(T));
            ri.shift_q = qr ? (int)((reinterpret_cast<uintptr_t>(qr + (size_t)k0 * step) & 15) / sizeof(T)) : 0;
            for (int k = k0; k < k1; ++k) {
                unsigned s;
                uint8_t* st = stage(s);
                const int lo = k * step, hi = min(lo + step, P.V);
                uint32_t bytes = staged_bytes(pr, lo, hi);
                if (qr) bytes += staged_bytes(qr, lo, hi);
                slots[s].type = it.type;
                slots[s].ctx = c;
                slots[s].pos = k - k0;
                slots[s].b = it.b;
                mbar_arrive_expect_tx(&full[s], bytes);  // publishes slot + run info (release)
                int sh;
                stage_range(pr, lo, hi, st, &full[s], sh);
                if (qr) stage_range(qr, lo, hi, st + kHalfStride, &full[s], sh);
                ++n;
            }
        } else {
            unsigned s;
            stage(s);
            Slot sl;
            sl.type = it.type;
            sl.ctx = -1;
            sl.pos = 0;
            sl.b = it.b;
            sl.mode = it.mode;
            sl.row = it.row;
            sl.Mp = it.Mp;
            sl.Sp = it.Sp;
            sl.Mq = it.Mq;
            sl.Sq = it.Sq;
            slots[s] = sl;
            mbar_arrive(&full[s]);
            ++n;
            if (it.type == IT_STOP) break;
        }
    }
}

// ---------------------------------------------------------------------------
// Decisions.  Exact: row statistics from the A-item partials (fixed order,
// fp64), tau at every drafted position from the gathered logits (fp64;
// activation.cpp:20-27 + verify_reference.cpp:87-92), first rejection
// (verify_reference.cpp:93-96, inclusive u <= tau).
template <typename T>
__device__ void decide_exact(const StepParams& P, int b, double* s_red, int* s_ired, double2* s_rs) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int G = P.G;
    // gathers and uniforms first: their latency overlaps the row statistics
    const int c = threadIdx.x;
    double zp = 0.0, zq = 0.0, u = 0.0;
    if (c < G) {
        int x = P.ids[(size_t)b * G + c];
        if (x < 0 || x >= P.V) {
            flag(P, SSV_STATUS_TOKEN_RANGE);
            x = x < 0 ? 0 : P.V - 1;
        }
        zp = load_exact(p_row<T>(P, b, c) + x);
        zq = load_exact(q_row<T>(P, b, c) + x);
    }
    if (c <= G) u = P.u[(size_t)b * (G + 1) + c];
    if (P.check_uniforms && c <= G && (!(u >= 0.0) || !(u < 1.0))) flag(P, SSV_STATUS_UNIFORM_RANGE);
    for (int r = warp; r < P.NR; r += kConsWarps) {
        const double2* part = P.part + ((size_t)b * P.NR + r) * P.RPR;
        double2 pk[4];
        double m = -CUDART_INF;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int k = lane + 32 * i;
            pk[i] = k < P.RPR ? __ldcg(&part[k]) : make_double2(-CUDART_INF, 0.0);
            m = fmax(m, pk[i].x);
        }
        for (int k = lane + 128; k < P.RPR; k += 32) m = fmax(m, __ldcg(&part[k].x));
        m = warp_max(m);
        double sm = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (pk[i].y > 0.0) sm += pk[i].y * exp(pk[i].x - m);
        for (int k = lane + 128; k < P.RPR; k += 32) {
            const double2 v = __ldcg(&part[k]);
            if (v.y > 0.0) sm += v.y * exp(v.x - m);
        }
        sm = warp_sum(sm);
        if (lane == 0) {
            P.rowstat[(size_t)b * P.NR + r] = make_double2(m, sm);
            if (r < kMaxRowsSmem) s_rs[r] = make_double2(m, sm);
        }
    }
    cbar<kCons>();
    auto rs = [&](int r) -> double2 { return r < kMaxRowsSmem ? s_rs[r] : P.rowstat[(size_t)b * P.NR + r]; };
    int rej = 0x7fffffff;
    if (c < G) {
        const double2 sp = rs(c), sq = rs(G + c);
        const double p = exp(zp - sp.x) / sp.y;   // activation.cpp:20-27, dist.cpp:46-50
        const double q = exp(zq - sq.x) / sq.y;
        const double tau = ratio_clamped(p, q);
        P.tau[(size_t)b * G + c] = tau;
        if (!(u <= tau)) rej = c;                // verify_reference.cpp:93-96 (inclusive)
    }
    const int a = min(creduce(rej, s_ired, OpMin()), G);
    if (threadIdx.x == 0) {
        P.acc[b] = a;
        Decision d{};
        if (a < G) {
            const double2 sp = rs(a), sq = rs(G + a);
            d.mode = MODE_REJECT;
            d.row = a;
            d.Mp = sp.x;
            d.Sp = sp.y;
            d.Mq = sq.x;
            d.Sq = sq.y;
        } else if (P.PS == G + 1) {
            d.mode = MODE_BONUS;
            d.row = G;
        } else {
            d.mode = MODE_NONE;
            P.fin[b] = -1;  // kNoToken, step.hpp:11
            P.rsu[b] = 0;
            P.rden[b] = 0.0;
        }
        P.dec[b] = d;
        P.cnt1[b] = 0;  // every A-item of b has been counted (the producer waited for it)
        __threadfence();
        st_release(&P.flag[b], P.epoch);
    }
}

// Sigmoid / probability decision from the gathered logits only (one warp).
// verify_sigmoid.cpp:50-58 -> verify_reference.cpp:87-96; the sigmoid is
// evaluated in fp64 exactly as dist.cpp:60-62 does.
template <typename T, int ACT>
__device__ void decide_gather(const StepParams& P, int b) {
    const int lane = threadIdx.x & 31;
    const int G = P.G;
    int accepted = G;
    for (int c0 = 0; c0 < G; c0 += 32) {
        const int c = c0 + lane;
        bool rej = false;
        if (c < G) {
            int x = P.ids[(size_t)b * G + c];
            if (x < 0 || x >= P.V) {
                flag(P, SSV_STATUS_TOKEN_RANGE);
                x = x < 0 ? 0 : P.V - 1;
            }
            const double zp = load_exact(p_row<T>(P, b, c) + x);
            const double zq = load_exact(q_row<T>(P, b, c) + x);
            double p, q;
            if (ACT == ACT_SIGMOID) {
                p = sigmoid_scaled_d(zp, P.alpha, P.width);
                q = sigmoid_scaled_d(zq, P.alpha, P.width);
            } else {
                p = zp;
                q = zq;
                if (p < 0.0 || q < 0.0) flag(P, SSV_STATUS_NEGATIVE);
            }
            const double tau = ratio_clamped(p, q);
            P.tau[(size_t)b * G + c] = tau;
            rej = !(P.u[(size_t)b * (G + 1) + c] <= tau);
        }
        const unsigned m = __ballot_sync(kFull, rej);
        if (m) {
            accepted = c0 + __ffs(m) - 1;
            break;
        }
    }
    if (P.check_uniforms) {
        for (int c = lane; c <= G; c += 32) {
            const double u = P.u[(size_t)b * (G + 1) + c];
            if (!(u >= 0.0) || !(u < 1.0)) flag(P, SSV_STATUS_UNIFORM_RANGE);
        }
    }
    if (lane == 0) {
        Decision d{};
        d.Sp = d.Sq = 1.0;
        P.acc[b] = accepted;
        if (accepted < G) {
            d.mode = MODE_REJECT;
            d.row = accepted;
        } else if (P.PS == G + 1) {
            d.mode = MODE_BONUS;
            d.row = G;
        } else {
            d.mode = MODE_NONE;
            P.fin[b] = -1;
            P.rsu[b] = 0;
            P.rden[b] = 0.0;
        }
        P.dec[b] = d;
        __threadfence();
        st_release(&P.flag[b], P.epoch);
    }
}

// ---------------------------------------------------------------------------
// Per-element values.  Streaming (acc precision) and exact (fp64) forms.
struct RowCtx {
    int mode;   // MODE_REJECT / MODE_BONUS
    bool useA;  // reject: sample the residual (else the degenerate fallback on p)
    double Mp, Sp, Mq, Sq;
    double denom;
};

template <int ACT>
__device__ __forceinline__ double exact_act(const StepParams& P, double z, double M, double S) {
    if (ACT == ACT_SOFTMAX) return exp(z - M) / S;  // dist.cpp:46-50
    if (ACT == ACT_SIGMOID) return sigmoid_scaled_d(z, P.alpha, P.width);
    return z;
}

// Value the inverse CDF scans at element i (fp64): residual max(0, p - q)
// (verify_reference.cpp:51-55) or the p row itself (fallback / bonus).
template <typename T, int ACT>
__device__ __forceinline__ double exact_value(const StepParams& P, const RowCtx& R, const T* pr, const T* qr,
                                              int i) {
    const double p = exact_act<ACT>(P, load_exact(pr + i), R.Mp, R.Sp);
    if (R.mode == MODE_REJECT && R.useA) {
        const double q = exact_act<ACT>(P, load_exact(qr + i), R.Mq, R.Sq);
        const double d = p - q;
        return d > 0.0 ? d : 0.0;
    }
    return p;
}

// ---------------------------------------------------------------------------
// Inverse CDF of batch row b (consumer group): granule partials -> SMEM ->
// fp64 granule prefix (contiguous ownership, one scan) -> exact fp64 scan
// inside the selected granule (dist.cpp:122-137, incl. both fallbacks).
template <typename T, int ACT>
__device__ void locate(const StepParams& P, const Slot& it, double2* gcache, double* s_red, int* s_ired) {
    const int b = it.b, NG = P.NG, GW = P.GW;
    const double2* gp = P.gpart + (size_t)b * NG;
    const T* pr = p_row<T>(P, b, it.row);
    const T* qr = it.mode == MODE_REJECT ? q_row<T>(P, b, it.row) : nullptr;
    const double u = __ldcg(&P.u[(size_t)b * (P.G + 1) + P.G]);  // u_final, verify_reference.cpp:98
    const int ncache = min(NG, kLocCap);
    for (int g = threadIdx.x; g < ncache; g += kCons) gcache[g] = __ldcg(&gp[g]);
    cbar<kCons>();
    auto raw = [&](int g) -> double2 { return g < kLocCap ? gcache[g] : __ldcg(&gp[g]); };

    RowCtx R;
    R.mode = it.mode;
    R.Mp = it.Mp;
    R.Sp = it.Sp;
    R.Mq = it.Mq;
    R.Sq = it.Sq;
    R.useA = false;
    R.denom = 1.0;
    double gM = 0.0, gS = 1.0;
    if (it.mode == MODE_REJECT) {
        double sa = 0.0, sp = 0.0;
        for (int g = threadIdx.x; g < NG; g += kCons) {
            const double2 v = raw(g);
            sa += v.x;
            sp += v.y;
        }
        sa = creduce(sa, s_red, OpSum());
        sp = creduce(sp, s_red, OpSum());
        R.useA = sa > kZeroEps;  // verify_reference.cpp:57-62
        R.denom = R.useA ? sa : sp;
        if (threadIdx.x == 0) {
            if (P.rsu) P.rsu[b] = 1;
            if (P.rden) P.rden[b] = R.useA ? sa : 0.0;
        }
    } else {
        if (ACT == ACT_SOFTMAX) {  // the bonus row's statistics from its granules
            double m = -CUDART_INF;
            for (int g = threadIdx.x; g < NG; g += kCons) m = fmax(m, raw(g).x);
            gM = creduce(m, s_red, OpMax());
            double sm = 0.0;
            for (int g = threadIdx.x; g < NG; g += kCons) {
                const double2 v = raw(g);
                if (v.y > 0.0) sm += v.y * exp(v.x - gM);
            }
            gS = creduce(sm, s_red, OpSum());
            R.Mp = gM;
            R.Sp = gS;
            R.denom = 1.0;  // sample_row's sequential_sum of a softmax row (1 within rounding)
        } else {
            double sm = 0.0;
            for (int g = threadIdx.x; g < NG; g += kCons) sm += raw(g).y;
            R.denom = creduce(sm, s_red, OpSum());
        }
        if (threadIdx.x == 0) {
            if (P.rsu) P.rsu[b] = 0;
            if (P.rden) P.rden[b] = 0.0;
        }
    }
    auto gmass = [&](int g) -> double {  // normalized granule mass
        const double2 v = raw(g);
        if (R.mode == MODE_REJECT) return (R.useA ? v.x : v.y) / R.denom;
        if (ACT == ACT_SOFTMAX) return v.y > 0.0 ? v.y * exp(v.x - gM) / gS : 0.0;
        return v.y / R.denom;
    };

    // Level 1: contiguous granule ownership, one block scan.
    const int gpt = (NG + kCons - 1) / kCons;
    const int ga = min(NG, threadIdx.x * gpt), gb = min(NG, ga + gpt);
    double tsum = 0.0;
    for (int g = ga; g < gb; ++g) tsum += gmass(g);
    double total;
    double run = cscan_incl(tsum, s_red, total) - tsum;
    int hit = 0x7fffffff;
    double hit_carry = 0.0;
    for (int g = ga; g < gb; ++g) {
        const double w = gmass(g);
        if (u < run + w) {
            hit = g;
            hit_carry = run;
            break;
        }
        run += w;
    }
    int gstar = creduce(hit, s_ired, OpMin());
    double carry = 0.0;
    if (gstar != 0x7fffffff) {
        if (hit == gstar) s_red[0] = hit_carry;  // creduce's barriers ordered every earlier s_red read
        cbar<kCons>();
        carry = s_red[0];
    } else {
        gstar = -1;
    }

    // Level 2: exact element scan, continuing into later granules on rounding.
    int token = -1;
    const int E = (GW + kCons - 1) / kCons;  // elements per thread (1 or 2)
    while (gstar >= 0 && gstar < NG) {
        const int lo = gstar * GW;
        const int hi = min(lo + GW, P.V);
        const int base = lo + threadIdx.x * E;
        double v0 = 0.0, v1 = 0.0;
        if (base < hi) v0 = exact_value<T, ACT>(P, R, pr, qr, base) / R.denom;
        if (E > 1 && base + 1 < hi) v1 = exact_value<T, ACT>(P, R, pr, qr, base + 1) / R.denom;
        const double ts = v0 + v1;
        double tot;
        const double incl = cscan_incl(ts, s_red, tot);
        double cum = carry + (incl - ts);
        int h = 0x7fffffff;
        cum += v0;
        if (base < hi && u < cum) h = base;
        cum += v1;
        if (h == 0x7fffffff && E > 1 && base + 1 < hi && u < cum) h = base + 1;
        const int first = creduce(h, s_ired, OpMin());
        if (first != 0x7fffffff) {
            token = first;
            break;
        }
        carry += tot;
        ++gstar;
    }
    if (token < 0) {
        // dist.cpp:135-136: last index with positive mass, else 0.
        int glast = -1;
        for (int g = threadIdx.x; g < NG; g += kCons)
            if (gmass(g) > 0.0) glast = max(glast, g);
        glast = creduce(glast, s_ired, OpMax());
        token = 0;
        if (glast >= 0) {
            int last = -1;
            for (int i = glast * GW + threadIdx.x; i < min((glast + 1) * GW, P.V); i += kCons)
                if (exact_value<T, ACT>(P, R, pr, qr, i) > 0.0) last = max(last, i);
            last = creduce(last, s_ired, OpMax());
            if (last >= 0) token = last;
        }
    }
    if (threadIdx.x == 0) {
        P.fin[b] = token;
        P.cnt2[b] = 0;  // every B-item of b has been counted (the producer waited for it)
    }
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Lane 0 of each warp counts the warp out of run `ri`; true in exactly one
// warp per run (the last), after every other warp's writes to `ri`.
__device__ __forceinline__ bool run_last_warp(RunInfo& ri) {
    unsigned old = 0;
    if ((threadIdx.x & 31) == 0) {
        __threadfence_block();
        old = atomicAdd(&ri.cnt, 1u);
        __threadfence_block();
    }
    old = __shfl_sync(kFull, old, 0);
    return old == kConsWarps - 1;
}

// Per-lane online softmax state of the A-run in flight.
template <typename A>
struct LaneRun {
    A m, mn;
    double s;
};

// A-chunk: the warp copies its 1/8 of the staged chunk into registers, frees
// the stage, then folds it into the lane's running (max, sum e^(x - max), min)
// -- fp32 ex2 within the chunk, fp64 across chunks, an fp64 exp only when the
// lane's max grows.  No cross-lane work until the run's last chunk.
template <typename T>
__device__ __forceinline__ void chunk_A(const StepParams& P, const uint8_t* st, int shift, int n,
                                        LaneRun<typename Elem<T>::acc>& L, uint64_t* empty_s) {
    using A = typename Elem<T>::acc;
    constexpr int VEC = Elem<T>::VEC;
    constexpr int WPW = kStageBytes / 16 / kConsWarps;  // 16-byte words per warp (128)
    constexpr int M = WPW / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int end = shift + n;                          // valid element range in the stage
    const int nwords = (end * (int)sizeof(T) + 15) / 16;  // <= 1025
    const int w0 = warp * WPW;
    const int w1 = min(nwords, w0 + WPW);
    uint4 w[M];
    uint4 wx;  // the 1025th word of a misaligned chunk (warp 7, lane 0)
    const bool has_x = warp == kConsWarps - 1 && lane == 0 && nwords > kConsWarps * WPW;
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const int wi = w0 + lane + 32 * m;
        if (wi < w1) w[m] = *reinterpret_cast<const uint4*>(st + (size_t)wi * 16);
    }
    if (has_x) wx = *reinterpret_cast<const uint4*>(st + (size_t)(kConsWarps * WPW) * 16);
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_s);  // the stage is free for the producer
    A cm = -INFINITY, cn = INFINITY;
    auto scan_word = [&](const uint4& v, int wi, auto&& f) {
        A x[VEC];
        unpack(v, x);
        if (wi * VEC >= shift && (wi + 1) * VEC <= end) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) f(x[e]);
        } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
                const int idx = wi * VEC + e;
                if (idx >= shift && idx < end) f(x[e]);
            }
        }
    };
    auto mm = [&](A x) {
        cm = fmax(cm, x);
        cn = fmin(cn, x);
    };
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const int wi = w0 + lane + 32 * m;
        if (wi < w1) scan_word(w[m], wi, mm);
    }
    if (has_x) scan_word(wx, kConsWarps * WPW, mm);
    if (cm > L.m) {  // the lane's max grew: rescale its running sum (fp64)
        if (L.s > 0.0) L.s *= exp((double)L.m - (double)cm);
        L.m = cm;
    }
    L.mn = fmin(L.mn, cn);
    if (L.m > -INFINITY) {
        A t = 0;
        const A mref = L.m;
        auto ex = [&](A x) { t += exp_rel(x, mref); };
#pragma unroll
        for (int m = 0; m < M; ++m) {
            const int wi = w0 + lane + 32 * m;
            if (wi < w1) scan_word(w[m], wi, ex);
        }
        if (has_x) scan_word(wx, kConsWarps * WPW, ex);
        L.s += (double)t;
    }
}

// End of an A-run: warp partial, and the run's last warp folds the 8 warp
// partials (fixed order) and publishes ONE (max, sum) per run.
template <typename A>
__device__ void finish_A(const StepParams& P, RunInfo& ri, LaneRun<A>& L) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (isnan(L.s)) flag(P, SSV_STATUS_NONFINITE);  // NaN logit (require_finite, dist.cpp:27-36)
    const double lm = (double)L.m;
    const double M = warp_max(lm);
    const double S = warp_sum(L.s > 0.0 ? L.s * exp(lm - M) : 0.0);
    const double MN = warp_min((double)L.mn);
    if (lane == 0) {
        if (isnan(S)) flag(P, SSV_STATUS_NONFINITE);  // NaN logit (require_finite, dist.cpp:27-36)
        ri.wpart[warp] = make_double2(M, S);
        ri.wmin[warp] = MN;
    }
    if (!run_last_warp(ri)) return;
    const double2 wp = lane < kConsWarps ? ri.wpart[lane] : make_double2(-CUDART_INF, 0.0);
    const double MX = warp_max(wp.x);
    const double SX = warp_sum(wp.y > 0.0 ? wp.y * exp(wp.x - MX) : 0.0);
    const double MNX = warp_min(lane < kConsWarps ? ri.wmin[lane] : CUDART_INF);
    if (lane == 0) {
        ri.cnt = 0;
        P.part[((size_t)ri.b * P.NR + ri.r) * P.RPR + ri.q] = make_double2(MX, SX);
        if (!isfinite(MX) || isnan(SX) || !isfinite(MNX)) flag(P, SSV_STATUS_NONFINITE);
        __threadfence();
        red_release_add(&P.cnt1[ri.b], 1u);
    }
}

// B-chunk: each warp copies its granule (both rows for a rejection) into
// registers, frees the stage, and reduces the granule; the run's last warp
// publishes the run's granule partials.
template <typename T, int ACT>
__device__ void chunk_B(const StepParams& P, RunInfo& ri, const uint8_t* st, int pos, int n, uint64_t* empty_s) {
    using A = typename Elem<T>::acc;
    constexpr int EPL = kStageBytes / 2 / (int)sizeof(T) / kCons;  // elements per lane per granule
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int e0 = warp * P.GW;
    const bool reject = ri.mode == MODE_REJECT;
    const A alpha = (A)P.alpha, invw = (A)(1.0 / P.width);
    A xs[EPL], xq[EPL];
#pragma unroll
    for (int t = 0; t < EPL; ++t) {
        const int e = e0 + t * 32 + lane;
        xs[t] = e < n ? lds_elem<T>(st, ri.shift_p + e) : (A)0;
        xq[t] = (reject && e < n) ? lds_elem<T>(st + kHalfStride, ri.shift_q + e) : (A)0;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty_s);
    double2 out = make_double2(0.0, 0.0);
    if (e0 < n) {
        if (!reject) {
            if (ACT == ACT_SOFTMAX) {
                A mx = -INFINITY, mn = INFINITY;
#pragma unroll
                for (int t = 0; t < EPL; ++t)
                    if (e0 + t * 32 + lane < n) {
                        mx = fmax(mx, xs[t]);
                        mn = fmin(mn, xs[t]);
                    }
                mx = warp_max(mx);
                mn = warp_min(mn);
                A sm = 0;
#pragma unroll
                for (int t = 0; t < EPL; ++t)
                    if (e0 + t * 32 + lane < n) sm += exp_rel(xs[t], mx);
                const double S = warp_sum((double)sm);
                if (lane == 0 && (!isfinite((double)mx) || isnan(S) || !isfinite((double)mn)))
                    flag(P, SSV_STATUS_NONFINITE);
                out = make_double2((double)mx, S);
            } else {
                A sm = 0;
#pragma unroll
                for (int t = 0; t < EPL; ++t) {
                    if (e0 + t * 32 + lane < n) {
                        if (ACT == ACT_SIGMOID) sm += (A)1 / ((A)1 + exp_neg((xs[t] - alpha) * invw));
                        else sm += xs[t];
                    }
                }
                out = make_double2(0.0, warp_sum((double)sm));
            }
        } else {
            const A Mp = (A)ri.Mp, Mq = (A)ri.Mq, iSp = (A)(1.0 / ri.Sp), iSq = (A)(1.0 / ri.Sq);
            A ta = 0, tp = 0;
#pragma unroll
            for (int t = 0; t < EPL; ++t) {
                if (e0 + t * 32 + lane < n) {
                    const A xp = xs[t], xqq = xq[t];
                    A a, vp;
                    if (ACT == ACT_SOFTMAX) {
                        vp = exp_rel(xp, Mp) * iSp;
                        const A vq = exp_rel(xqq, Mq) * iSq;
                        a = vp - vq > (A)0 ? vp - vq : (A)0;
                    } else if (ACT == ACT_SIGMOID) {
                        // sigma(tp) - sigma(tq) = sigma(tp) sigma(-tq) (1 - e^-(tp-tq)): no cancellation.
                        const A tp_ = (xp - alpha) * invw, tq_ = (xqq - alpha) * invw;
                        const A d = (xp - xqq) * invw;
                        vp = (A)1 / ((A)1 + exp_neg(tp_));
                        const A sqn = (A)1 / ((A)1 + exp_neg(-tq_));
                        a = d > (A)0 ? vp * sqn * (-expm1_acc(-d)) : (A)0;
                    } else {
                        vp = xp;
                        a = xp - xqq > (A)0 ? xp - xqq : (A)0;
                    }
                    ta += a;
                    tp += vp;
                }
            }
            out = make_double2(warp_sum((double)ta), warp_sum((double)tp));
        }
    }
    if (lane == 0) ri.gpart[pos * kConsWarps + warp] = out;
    if (pos != ri.len - 1) return;
    if (!run_last_warp(ri)) return;
    const int g0 = ri.q * P.runB * kConsWarps;
    const int ng = min(ri.len * kConsWarps, P.NG - g0);
    for (int i = lane; i < ng; i += 32) P.gpart[(size_t)ri.b * P.NG + g0 + i] = ri.gpart[i];
    __threadfence();
    __syncwarp();
    if (lane == 0) {
        ri.cnt = 0;
        red_release_add(&P.cnt2[ri.b], 1u);
    }
}

// ---------------------------------------------------------------------------
template <typename T, int ACT>
__global__ void __launch_bounds__(kBlock, 2) k_verify(StepParams P) {
    using A = typename Elem<T>::acc;
    constexpr int CA = kStageBytes / (int)sizeof(T);
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* stages = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)kStages * kStageStride);
    uint64_t* empty = full + kStages;
    Slot* slots = reinterpret_cast<Slot*>(empty + kStages);
    double2* gcache = reinterpret_cast<double2*>(slots + kStages);
    RunInfo* runs = reinterpret_cast<RunInfo*>(gcache + kLocCap);
    __shared__ double s_red[kConsWarps];
    __shared__ int s_ired[kConsWarps];
    __shared__ double2 s_rs[kMaxRowsSmem];

    if (threadIdx.x == 0) {
        trace(P, 2 * blockIdx.x);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsWarps);  // every consumer warp frees the stage
        }
        for (int c = 0; c < kCtx; ++c) runs[c].cnt = 0;
        mbar_fence_init();
    }
    __syncthreads();

    if (threadIdx.x >= kCons) {
        if (threadIdx.x == kCons) producer<T, ACT>(P, stages, full, empty, slots, runs);
    } else {
        const int lane = threadIdx.x & 31;
        LaneRun<A> L{(A)-INFINITY, (A)INFINITY, 0.0};
        unsigned n = 0;
        for (;;) {
            const unsigned s = n % kStages, ph = (n / kStages) & 1u;
            mbar_wait(&full[s], ph);
            const int4 hdr = *reinterpret_cast<const int4*>(&slots[s]);  // type, ctx, pos, b
            ++n;
            if (hdr.x == IT_STOP) break;
            const uint8_t* st = stages + (size_t)s * kStageStride;
            if (hdr.x == IT_A) {
                RunInfo& ri = runs[hdr.y];
                const int pos = hdr.z, len = ri.len;
                const int lo = (ri.k0 + pos) * CA;
                if (pos == 0) L = LaneRun<A>{(A)-INFINITY, (A)INFINITY, 0.0};
                chunk_A<T>(P, st, ri.shift_p, min(CA, P.V - lo), L, &empty[s]);
                if (pos == len - 1) finish_A<A>(P, ri, L);
            } else if (hdr.x == IT_B) {
                RunInfo& ri = runs[hdr.y];
                const int lo = (ri.k0 + hdr.z) * P.CB;
                chunk_B<T, ACT>(P, ri, st, hdr.z, min(P.CB, P.V - lo), &empty[s]);
            } else {
                const Slot sl = slots[s];
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                cbar<kCons>();  // the decide / locate run on the whole consumer group
                const int tb = 2 * (int)gridDim.x + 4 * sl.b + (sl.type == IT_D ? 0 : 2);
                if (threadIdx.x == 0) trace(P, tb);
                if (sl.type == IT_D) {
                    if (ACT == ACT_SOFTMAX && !P.sample_mode) decide_exact<T>(P, sl.b, s_red, s_ired, s_rs);
                    else if (threadIdx.x < 32) decide_gather<T, ACT>(P, sl.b);
                } else {
                    locate<T, ACT>(P, sl, gcache, s_red, s_ired);
                }
                if (threadIdx.x == 0) trace(P, tb + 1);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        trace(P, 2 * blockIdx.x + 1);
        __threadfence();
        const unsigned prev = atomicAdd(P.exit_cnt, 1u);
        if (prev == gridDim.x - 1) {  // last CTA out resets the work counters
            *P.exit_cnt = 0;
            *P.next = 0;
            __threadfence();
        }
    }
}

// ---------------------------------------------------------------------------
// K3: optional materialized grids (activation.cpp:20-49; verify_fused.cpp:50
// residual-in-q semantics; verify_sigmoid.cpp:39-48).
template <typename T, int ACT>
__global__ void __launch_bounds__(kThreads) k_materialize(StepParams P, void* outp, void* outq, void* outr) {
    using A = typename Elem<T>::acc;
    using O = typename std::conditional<sizeof(A) == 8, double, float>::type;
    const size_t V = (size_t)P.V;
    const size_t np = (size_t)P.B * P.PS * V, nq = (size_t)P.B * P.G * V;
    const A alpha = (A)P.alpha, invw = (A)(1.0 / P.width);
    auto act = [&](A x, const double2& st) -> A {
        if (ACT == ACT_SOFTMAX) return exp_rel(x, (A)st.x) * (A)(1.0 / st.y);
        if (ACT == ACT_SIGMOID) return (A)1 / ((A)1 + exp_neg((x - alpha) * invw));
        return x;
    };
    auto stat_of = [&](int b, int r) -> double2 {
        if (ACT != ACT_SOFTMAX) return make_double2(0.0, 1.0);
        return P.rowstat[(size_t)b * P.NR + r];
    };
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += stride) {
        const size_t rowi = i / V;
        const int b = (int)(rowi / P.PS), c = (int)(rowi % P.PS);
        const A x = load_elem(reinterpret_cast<const T*>(P.zp) + i);
        const A pv = act(x, stat_of(b, c < P.G ? c : 2 * P.G));
        if (outp) reinterpret_cast<O*>(outp)[i] = (O)pv;
    }
    if (!outq && !outr) return;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq; i += stride) {
        const size_t rowi = i / V, e = i % V;
        const int b = (int)(rowi / P.G), c = (int)(rowi % P.G);
        const A xq = load_elem(reinterpret_cast<const T*>(P.zq) + i);
        const A qv = act(xq, stat_of(b, P.G + c));
        if (outq) reinterpret_cast<O*>(outq)[i] = (O)qv;
        if (outr) {
            const A xp = load_elem(p_row<T>(P, b, c) + e);
            const A pv = act(xp, stat_of(b, c));
            reinterpret_cast<O*>(outr)[i] = (O)(pv - qv > (A)0 ? pv - qv : (A)0);
        }
    }
}

// ---------------------------------------------------------------------------
// Synthetic inputs: bench.cpp:46-74 per batch row (seed + b), using the
// counter RNG of rng.cpp:12-33 (SplitMix64 at index i, Box-Muller in fp64).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t word_at(uint64_t seed, uint64_t index) {
    return mix64(seed + (index + 1) * 0x9e3779b97f4a7c15ull);
}
__device__ __forceinline__ double uniform_at(uint64_t seed, uint64_t index) {
    return (double)(word_at(seed, index) >> 11) * 0x1.0p-53;
}
__device__ __forceinline__ double normal_at(uint64_t seed, uint64_t n) {  // n-th normal = words 2n, 2n+1
    const double u1 = ((double)(word_at(seed, 2 * n) >> 11) + 0.5) * 0x1.0p-53;
    const double u2 = (double)(word_at(seed, 2 * n + 1) >> 11) * 0x1.0p-53;
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

template <typename T>
__device__ __forceinline__ T to_store(double v);
template <>
__device__ __forceinline__ float to_store<float>(double v) { return (float)v; }
template <>
__device__ __forceinline__ double to_store<double>(double v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 to_store<__nv_bfloat16>(double v) {
    return __float2bfloat16_rn((float)v);  // double -> fp32 -> bf16, like orc_round_bf16
}

template <typename T>
__global__ void k_gen_logits(uint64_t seed, int B, int G, int V, T* zp, T* zq) {
    const size_t per_b = (size_t)(2 * G + 1) * V;
    const size_t n = (size_t)B * per_b;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int b = (int)(i / per_b);
        const size_t j = i % per_b;
        const uint64_t s = seed + (uint64_t)b;
        const size_t np = (size_t)(G + 1) * V;
        if (j < np) {
            zp[(size_t)b * np + j] = to_store<T>(4.0 * normal_at(s, j));
        } else {
            const size_t jq = j - np;  // q row c element e: z_p[c][e] + N at index np + jq
            const double v = 4.0 * normal_at(s, jq) + 1.0 * normal_at(s, np + jq);
            zq[(size_t)b * G * V + jq] = to_store<T>(v);
        }
    }
}

// Draft draws (index 2(2G+1)V + c) and acceptance/final uniforms
// (index 2(2G+1)V + G + c) of bench.cpp:66-73.
__global__ void k_gen_uniforms(uint64_t seed, int B, int G, int V, double* draft_u, double* u) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int per = 2 * G + 1;
    if (i >= B * per) return;
    const int b = i / per, c = i % per;
    const uint64_t base = 2ull * (uint64_t)(2 * G + 1) * (uint64_t)V;
    const double v = uniform_at(seed + (uint64_t)b, base + (uint64_t)c);
    if (c < G) draft_u[(size_t)b * G + c] = v;
    else u[(size_t)b * (G + 1) + (c - G)] = v;
}

// ---------------------------------------------------------------------------
// Host-side launchers.
static int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

constexpr size_t kVerifySmem = (size_t)kStages * kStageStride + 2 * kStages * sizeof(uint64_t) +
                               kStages * sizeof(Slot) + kLocCap * sizeof(double2) + kCtx * sizeof(RunInfo);

static size_t elem_size(int dtype) { return dtype == DT_F64 ? 8 : (dtype == DT_BF16 ? 2 : 4); }

void plan_geometry(int dtype, int act, StepParams& P) {
    const int s = (int)elem_size(dtype);
    const int CA = kStageBytes / s;
    P.CH = CA;
    P.CB = kStageBytes / (2 * s);
    P.GW = P.CB / kConsWarps;
    P.NG = (P.V + P.GW - 1) / P.GW;
    P.nBi = (P.V + P.CB - 1) / P.CB;
    if (P.sample_mode || act != ACT_SOFTMAX) {
        P.NR = 0;
        P.K = 0;
    } else {
        P.K = (P.V + CA - 1) / CA;
    }
    const long grid = 2L * sm_count();
    // Runs: long enough to amortize one publish over many 16 KB chunks, short
    // enough that every phase still spreads over ~4 runs per CTA.
    auto run_len = [&](long chunks_per_row, long rows, int cap) {
        if (chunks_per_row <= 0) return 1;
        long want = (chunks_per_row * rows + 4 * grid - 1) / (4 * grid);
        want = std::max<long>(1, std::min<long>({want, chunks_per_row, (long)cap}));
        const long runs = (chunks_per_row + want - 1) / want;
        return (int)((chunks_per_row + runs - 1) / runs);
    };
    P.runA = P.K > 0 ? run_len(P.K, (long)P.B * P.NR, kMaxRunA) : 1;
    P.RPR = P.K > 0 ? (P.K + P.runA - 1) / P.runA : 0;
    P.runB = run_len(P.nBi, P.B, kMaxRunB);
    P.nA = P.NR * P.RPR;
    P.nph[IT_A] = P.nA;
    P.nph[IT_D] = P.sample_mode ? 0 : 1;
    P.nph[IT_B] = (P.nBi + P.runB - 1) / P.runB;
    P.nph[IT_L] = 1;
    const long seg = (long)P.nph[0] + P.nph[1] + P.nph[2] + P.nph[3];
    P.n_items = (unsigned)((long)P.B * seg);
    const long g = std::min<long>(grid, std::max<long>(1, P.n_items));
    // Items a CTA may hold: the run in its ring and the one claimed ahead.
    // Lag between the phases of one batch row, in segments, so a phase's
    // dependency has completed when a producer reaches it.
    const long inflight = g * 3;
    P.claim = 1;
    P.lag = (int)std::max<long>(1, std::min<long>(P.B, (inflight + seg - 1) / seg + 1));
    int o = 0;
    for (int p = 0; p < 4; ++p) {
        P.off[p] = o;
        if (P.nph[p] > 0) o += P.lag;
    }
    int pts[10], n = 0;
    pts[n++] = 0;
    const int tend = P.B + P.off[3];
    pts[n++] = tend;
    for (int p = 0; p < 4; ++p) {
        if (P.nph[p] == 0) continue;
        pts[n++] = std::min(P.off[p], tend);
        pts[n++] = std::min(P.off[p] + P.B, tend);
    }
    for (int i = 1; i < n; ++i)  // insertion sort of <= 10 points
        for (int j = i; j > 0 && pts[j - 1] > pts[j]; --j) std::swap(pts[j - 1], pts[j]);
    P.nbp = 0;
    for (int i = 0; i < n; ++i)
        if (P.nbp == 0 || pts[i] != P.bp[P.nbp - 1]) P.bp[P.nbp++] = pts[i];
}

int verify_grid(const StepParams& P) { return (int)std::min<long>(2L * sm_count(), std::max<long>(1, P.n_items)); }

template <typename T, int ACT>
static void launch_verify_t(const StepParams& P, const Launch& L) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_verify<T, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kVerifySmem);
        attr = true;
    }
    const int grid = (int)std::min<long>(2L * sm_count(), std::max<long>(1, P.n_items));
    const int h = L.begin(KID_VERIFY);
    k_verify<T, ACT><<<grid, kBlock, kVerifySmem, L.st>>>(P);
    L.end(h);
}

template <typename T, int ACT>
static void launch_mat_t(const StepParams& P, void* p, void* q, void* r, const Launch& L) {
    const int h = L.begin(KID_MATERIALIZE);
    k_materialize<T, ACT><<<148 * 8, kThreads, 0, L.st>>>(P, p, q, r);
    L.end(h);
}

template <typename T>
static void dispatch_verify(int act, const StepParams& P, void* outp, void* outq, void* outr, const Launch& L) {
    const bool mat = outp || outq || outr;
    if (act == ACT_SOFTMAX) {
        launch_verify_t<T, ACT_SOFTMAX>(P, L);
        if (mat) launch_mat_t<T, ACT_SOFTMAX>(P, outp, outq, outr, L);
    } else if (act == ACT_SIGMOID) {
        launch_verify_t<T, ACT_SIGMOID>(P, L);
        if (mat) launch_mat_t<T, ACT_SIGMOID>(P, outp, outq, outr, L);
    } else {
        launch_verify_t<T, ACT_PROBS>(P, L);
        if (mat) launch_mat_t<T, ACT_PROBS>(P, outp, outq, outr, L);
    }
}

void launch_verify(int dtype, int act, const StepParams& P, void* outp, void* outq, void* outr, const Launch& L) {
    if (dtype == DT_F32) dispatch_verify<float>(act, P, outp, outq, outr, L);
    else if (dtype == DT_BF16) dispatch_verify<__nv_bfloat16>(act, P, outp, outq, outr, L);
    else dispatch_verify<double>(act, P, outp, outq, outr, L);
}

void launch_sample_softmax(int dtype, const StepParams& P, const Launch& L) {
    if (dtype == DT_F32) launch_verify_t<float, ACT_SOFTMAX>(P, L);
    else if (dtype == DT_BF16) launch_verify_t<__nv_bfloat16, ACT_SOFTMAX>(P, L);
    else launch_verify_t<double, ACT_SOFTMAX>(P, L);
}

void launch_gen_logits(int dtype, uint64_t seed, int B, int G, int V, void* zp, void* zq, const Launch& L) {
    const int blocks = 148 * 16;
    const int h = L.begin(KID_GEN);
    if (dtype == DT_F32) k_gen_logits<float><<<blocks, kThreads, 0, L.st>>>(seed, B, G, V, (float*)zp, (float*)zq);
    else if (dtype == DT_BF16)
        k_gen_logits<__nv_bfloat16><<<blocks, kThreads, 0, L.st>>>(seed, B, G, V, (__nv_bfloat16*)zp, (__nv_bfloat16*)zq);
    else k_gen_logits<double><<<blocks, kThreads, 0, L.st>>>(seed, B, G, V, (double*)zp, (double*)zq);
    L.end(h);
}

void launch_gen_uniforms(uint64_t seed, int B, int G, int V, double* draft_u, double* u, const Launch& L) {
    const int n = B * (2 * G + 1);
    const int h = L.begin(KID_GEN);
    k_gen_uniforms<<<(n + kThreads - 1) / kThreads, kThreads, 0, L.st>>>(seed, B, G, V, draft_u, u);
    L.end(h);
}

}  // namespace ssv
