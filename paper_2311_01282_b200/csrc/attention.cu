// Subsystem 1 — split-KV decode/prefill attention: host side (plans,
// workspace layout, launch policy, the C ABI).  The kernels live in
// attention_kernels.cuh, instantiated per dtype x mode in attention_*.cu.
#include <cfloat>
#include <cmath>
#include <cstring>

#include "attention_kernels.cuh"

namespace fdpp {

#define FDPP_ATTN_EXTERN(T)                                                                         \
    extern template fdpp_status by_d<T, true>(const AttnArgs &, int, int, int, cudaStream_t);       \
    extern template fdpp_status by_d<T, false>(const AttnArgs &, int, int, int, cudaStream_t);
FDPP_ATTN_EXTERN(__half)
FDPP_ATTN_EXTERN(__nv_bfloat16)
FDPP_ATTN_EXTERN(float)
#undef FDPP_ATTN_EXTERN
extern template fdpp_status launch_mma_t<__half, true>(const AttnArgs &, int, const CUtensorMap *,
                                                       const CUtensorMap *, cudaStream_t);
extern template fdpp_status launch_mma_t<__half, false>(const AttnArgs &, int, const CUtensorMap *,
                                                        const CUtensorMap *, cudaStream_t);
extern template fdpp_status launch_mma_t<__nv_bfloat16, true>(const AttnArgs &, int, const CUtensorMap *,
                                                              const CUtensorMap *, cudaStream_t);
extern template fdpp_status launch_mma_t<__nv_bfloat16, false>(const AttnArgs &, int, const CUtensorMap *,
                                                               const CUtensorMap *, cudaStream_t);

template <bool ASYNC>
static fdpp_status launch_mma(const AttnArgs &a, int dtype, int gx, const CUtensorMap *tmK,
                              const CUtensorMap *tmV, cudaStream_t st) {
    return dtype == FDPP_BF16 ? launch_mma_t<__nv_bfloat16, ASYNC>(a, gx, tmK, tmV, st)
                              : launch_mma_t<__half, ASYNC>(a, gx, tmK, tmV, st);
}

// ---------------------------------------------------------------------- host
struct AttnLayout {
    int G, GT, n_rg, p, nsub, P;
    bool mma;      // async launch on tensor cores (GQA/MQA): 16-row groups
    int n_rg_mma;  // its row groups per kv head
    float pscale;  // its power-of-two P scale
    size_t off_num, off_den, off_m, off_viol, off_cnt, off_flags, total;
};

// recompute list header (fixed offset after the ticket counters, never aliased,
// left zeroed by every launch): [0] count, [32] CTAs done, list, dedupe marks
constexpr int kFlagListOff = 64, kFlagMax = 8128;
constexpr size_t kFlagBytes = 16384 * sizeof(int);

static int pick_gt(int G) { return G >= 8 ? 8 : G >= 4 ? 4 : G >= 2 ? 2 : 1; }

// Tensor-core async path: GQA/MQA groups (G >= 4) at D = 128 in f16/bf16 over a
// contiguous [B, Hkv, Lmax, D] cache.  f16 P needs the band's dynamic range
// e^(b - a) inside fp16's normal range with margin ((b - a) log2 e <= 28);
// P is scaled by 2^(14 - ceil(b log2 e)) so e^b lands below 2^14.
// FDPP_ATTN_MMA=0 forces the CUDA-core path.
static bool mma_enabled() {
    static int v = [] {
        const char *e = getenv("FDPP_ATTN_MMA");
        return e ? atoi(e) : 1;
    }();
    return v != 0;
}

// FDPP_ATTN_INCLUSTER=0: cluster-joined launches hand flagged rows to the
// separate recompute launch (the round-1 two-launch form) instead of
// recomputing them inside the cluster.
static bool incluster_enabled() {
    static int v = [] {
        const char *e = getenv("FDPP_ATTN_INCLUSTER");
        return e ? atoi(e) : 1;
    }();
    return v != 0;
}

// An aborted group's flags come from its sync pass (band check + in-band
// exp-sums + finite outputs).  That equals the async verdict whenever the async
// numerators cannot overflow without a band violation: fp16 K/V (|v| <= 65504)
// and e^b x L x 65504 below FLT_MAX.  FDPP_ATTN_ABORT=0 disables the early stop.
static bool abort_safe(const fdpp_attn_params *p, const AttnLayout &lay) {
    static int v = [] {
        const char *e = getenv("FDPP_ATTN_ABORT");
        return e ? atoi(e) : 1;
    }();
    if (!v || p->dtype != FDPP_F16) return false;
    // worth it only for long chunks: below ~1K keys per CTA the stream is short
    // and the per-tile checks cost more (measured on the 7B B = 32 step: 512
    // keys per CTA, 98.7 vs 103.4 us per layer); FDPP_ATTN_ABORT=2 forces it
    if (v < 2 && (int64_t)p->L < 1024ll * lay.P) return false;
    return std::exp((double)p->b) * (double)p->L * 65504.0 < 1e37;
}

static bool mma_shape_ok(const fdpp_attn_params *p, int G) {
    if (!mma_enabled() || G < 4 || p->D != 128) return false;
    if (p->dtype != FDPP_F16 && p->dtype != FDPP_BF16) return false;
    return p->kv_stride_h % p->D == 0 && p->kv_stride_b == (int64_t)p->Hkv * p->kv_stride_h &&
           p->kv_stride_h >= (int64_t)p->L * p->D;
}

static bool mma_eligible(const fdpp_attn_params *p, int G, float *pscale) {
    if (p->mode != FDPP_ATTN_ASYNC || !mma_shape_ok(p, G)) return false;
    const double log2e = 1.4426950408889634;
    if (p->dtype == FDPP_F16) {
        if (!(p->b > p->a) || (double)(p->b - p->a) * log2e > 28.0) return false;
        *pscale = ldexpf(1.f, 14 - (int)ceil((double)p->b * log2e));
    } else {
        *pscale = 1.f;
    }
    return true;
}

static fdpp_status layout_for(const fdpp_attn_params *p, AttnLayout *lay) {
    FDPP_REQUIRE(p != nullptr, FDPP_ERR_VALUE, "null params");
    FDPP_REQUIRE(p->B >= 1 && p->Hq >= 1 && p->Hkv >= 1 && p->L >= 1, FDPP_ERR_SHAPE,
                 "attention dims must be >= 1 (K/V cache must hold at least one row)");
    FDPP_REQUIRE(p->Hq % p->Hkv == 0, FDPP_ERR_SHAPE, "Hq %% Hkv != 0");
    lay->G = p->Hq / p->Hkv;
    lay->GT = pick_gt(lay->G);
    lay->n_rg = (lay->G + lay->GT - 1) / lay->GT;
    const int groups = p->B * p->Hkv * lay->n_rg;  // counters (the CUDA-core grouping is the finest)
    lay->pscale = 1.f;
    lay->mma = mma_eligible(p, lay->G, &lay->pscale);
    lay->n_rg_mma = (lay->G + 15) / 16;
    const int launch_groups = lay->mma ? p->B * p->Hkv * lay->n_rg_mma : groups;
    const int sms = sm_count() > 0 ? sm_count() : 148;
    if (p->p > 0) {
        FDPP_REQUIRE(p->p <= p->L, FDPP_ERR_VALUE, "partition count must be in [1, %d], got %d",
                     p->L, p->p);
        FDPP_REQUIRE(p->p <= ATT_MAX_P, FDPP_ERR_VALUE, "partition count above %d", ATT_MAX_P);
        lay->p = p->p;
    } else if (lay->mma) {
        // auto, tensor-core path: one full wave (3 CTAs per SM: each CTA keeps
        // 64 KB of K/V in flight, so the whole wave is what saturates HBM), no
        // second partial wave, >= 128 keys per CTA (profiles/r1_attn_gqa_sweep.txt)
        int want = (3 * sms) / launch_groups;
        int maxp = p->L / 128 > 0 ? p->L / 128 : 1;
        if (maxp > 16) maxp = 16;  // the cluster (DSMEM) join takes <= 16 CTAs per row group
        lay->p = want < 1 ? 1 : (want > maxp ? maxp : want);
    } else {
        // auto: enough chunks for ~8 CTAs per SM over the launch, >= 512 keys each
        int want = (8 * sms + launch_groups - 1) / launch_groups;
        int maxp = p->L / 512 > 0 ? p->L / 512 : 1;
        lay->p = want < 1 ? 1 : (want > maxp ? maxp : want);
        if (lay->p > ATT_MAX_P) lay->p = ATT_MAX_P;
    }
    if (p->splits_per_chunk > 0) {
        lay->nsub = p->splits_per_chunk;
    } else if (lay->mma) {
        lay->nsub = 1;
    } else {
        const int per_chunk = p->L / lay->p;
        int want = (8 * sms + launch_groups * lay->p - 1) / (launch_groups * lay->p);
        // >= 128 keys per CTA: few (batch, kv-head) groups (config 1: B = 1) need the
        // splits to fill the machine; with many groups the CTA target is met first
        int maxs = per_chunk / 128 > 0 ? per_chunk / 128 : 1;
        lay->nsub = want < 1 ? 1 : (want > maxs ? maxs : want);
    }
    if (p->p <= 0 && p->splits_per_chunk <= 0 && !lay->mma) {
        // auto, CUDA-core path: one semantic chunk per CTA (the <= 16 CTAs of a row
        // group join over DSMEM as one cluster).  p0 = the fewest chunks filling half
        // a wave of the 3-per-SM slots (W = CTAs / slots >= 0.5); p0 + 1 only if it
        // fills its last wave better (W / ceil(W); W <= 1 counts as W), >= 128 keys
        // per CTA.  Measured (profiles/r1_attn_mha_splits.txt, L ~ 1K): B=1: 8, B=4: 3,
        // B=8: 1 (2 = 1.15 waves is the worst), B=16: 2, B=32: 2, B=64: 1.
        const double slots = 3.0 * sms;
        int pmax = p->L / 128 > 0 ? p->L / 128 : 1;
        if (pmax > 16) pmax = 16;
        auto fill = [&](int c) {
            const double w = (double)groups * c / slots;
            return w <= 1.0 ? w : w / std::ceil(w);
        };
        int p0 = 1;
        while (p0 < pmax && (double)groups * p0 / slots < 0.5) ++p0;
        // long rows with few row groups amortise the per-CTA cost: look two chunk
        // counts further (B=8/16, L=8K: p=3; B=32/64, L=4K keep 2/1)
        const int span = (p->L > 2048 && (double)groups * p0 / slots < 2.0) ? 2 : 1;
        int best = p0;
        for (int c = p0 + 1; c <= p0 + span && c <= pmax; ++c)
            if (fill(c) > fill(best) + 1e-9) best = c;
        lay->p = best;
        lay->nsub = 1;
    }
    lay->P = lay->p * lay->nsub;
    FDPP_REQUIRE(lay->P <= ATT_MAX_P, FDPP_ERR_VALUE,
                 "p x splits_per_chunk = %d exceeds %d partials per row", lay->P, ATT_MAX_P);
    const size_t rows = (size_t)p->B * p->Hq;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    size_t off = 0;
    FDPP_REQUIRE(groups <= kWsCounters, FDPP_ERR_SHAPE, "too many (batch, kv-head) groups: %d", groups);
    lay->off_cnt = off;  off += kWsCounterBytes;
    lay->off_flags = off; off += kFlagBytes;
    lay->off_num = off;  off += al(rows * lay->P * p->D * sizeof(float));
    lay->off_den = off;  off += al(rows * lay->P * sizeof(float));
    lay->off_m = off;    off += al(rows * lay->P * sizeof(float));
    lay->off_viol = off; off += al(rows * lay->P * sizeof(int));
    lay->total = off;
    return FDPP_OK;
}

// async launches join over DSMEM when a row group's split is <= 16 single-chunk
// CTAs and no per-chunk outputs are requested
static bool cluster_join_for(const fdpp_attn_params *p, const AttnLayout &lay) {
    if (lay.P > 16 || lay.nsub != 1 || p->viol_index || p->chunk_num || p->chunk_den) return false;
    return lay.mma || p->D <= ATT_CONSUMERS * 32;  // the producer warp reads the chunk states
}

// 2-D maps over the cache as [B * Hkv * Lmax rows, D]: 32-row x 64-column boxes
static fdpp_status kv_maps(const fdpp_attn_params *p, CUtensorMap *mk, CUtensorMap *mv) {
    const int64_t rows = (int64_t)p->B * p->Hkv * (p->kv_stride_h / p->D);
    fdpp_status s = make_kmajor_map(mk, p->k, rows, p->D, p->D, 32, p->dtype);
    if (s != FDPP_OK) return s;
    return make_kmajor_map(mv, p->v, rows, p->D, p->D, 32, p->dtype);
}

template <bool ASYNC>
static fdpp_status by_dtype(const AttnArgs &a, int dtype, int D, int gt, int gx, cudaStream_t st) {
    switch (dtype) {
        case FDPP_F16: return by_d<__half, ASYNC>(a, D, gt, gx, st);
        case FDPP_BF16: return by_d<__nv_bfloat16, ASYNC>(a, D, gt, gx, st);
        case FDPP_F32: return by_d<float, ASYNC>(a, D, gt, gx, st);
        default: set_error("bad dtype %d", dtype); return FDPP_ERR_UNSUPPORTED;
    }
}

}  // namespace fdpp

using namespace fdpp;


extern "C" fdpp_status fdpp_attn_workspace_size(const fdpp_attn_params *p, size_t *bytes) {
    FDPP_REQUIRE(bytes != nullptr, FDPP_ERR_VALUE, "null bytes");
    AttnLayout lay;
    fdpp_status s = layout_for(p, &lay);
    if (s != FDPP_OK) return s;
    *bytes = lay.total;
    return FDPP_OK;
}

extern "C" fdpp_status fdpp_attn_plan(const fdpp_attn_params *p, int32_t *chunks,
                                      int32_t *splits_per_chunk) {
    FDPP_REQUIRE(chunks && splits_per_chunk, FDPP_ERR_VALUE, "null output");
    AttnLayout lay;
    fdpp_status s = layout_for(p, &lay);
    if (s != FDPP_OK) return s;
    *chunks = lay.p;
    *splits_per_chunk = lay.nsub;
    return FDPP_OK;
}

extern "C" fdpp_status fdpp_attn_launches(const fdpp_attn_params *p, int32_t *launches) {
    FDPP_REQUIRE(launches != nullptr, FDPP_ERR_VALUE, "null output");
    AttnLayout lay;
    fdpp_status s = layout_for(p, &lay);
    if (s != FDPP_OK) return s;
    const bool inc = p->mode == FDPP_ATTN_ASYNC && cluster_join_for(p, lay) && incluster_enabled() &&
                     (!lay.mma || mma_shape_ok(p, lay.G));
    *launches = (p->mode == FDPP_ATTN_SYNC || inc) ? 1 : 2;
    return FDPP_OK;
}

extern "C" fdpp_status fdpp_attn_decode(const fdpp_attn_params *p, void *stream) {
    AttnLayout lay;
    fdpp_status s = layout_for(p, &lay);
    if (s != FDPP_OK) return s;
    FDPP_REQUIRE(p->q && p->k && p->v && p->o, FDPP_ERR_VALUE, "null attention operand");
    FDPP_REQUIRE(p->mode == FDPP_ATTN_ASYNC || p->mode == FDPP_ATTN_SYNC, FDPP_ERR_VALUE,
                 "mode must be async or sync");
    FDPP_REQUIRE(p->scale > 0.f, FDPP_ERR_VALUE, "scale must be > 0");
    FDPP_REQUIRE(p->mode != FDPP_ATTN_ASYNC || p->row_flags, FDPP_ERR_VALUE,
                 "async mode needs row_flags");
    FDPP_REQUIRE(p->workspace && p->workspace_bytes >= lay.total, FDPP_ERR_WORKSPACE,
                 "attention workspace too small: need %zu bytes", lay.total);
    const int esz = p->dtype == FDPP_F32 ? 4 : 2;
    FDPP_REQUIRE((reinterpret_cast<uintptr_t>(p->k) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(p->v) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(p->q) & 15) == 0 &&
                     ((p->kv_stride_b * esz) & 15) == 0 && ((p->kv_stride_h * esz) & 15) == 0 &&
                     ((p->q_stride_b * esz) & 15) == 0 && ((p->q_stride_h * esz) & 15) == 0,
                 FDPP_ERR_UNSUPPORTED, "Q/K/V must be 16-byte aligned per row/head");
    char *ws = static_cast<char *>(p->workspace);
    AttnArgs a{};
    a.q = p->q; a.k = p->k; a.v = p->v; a.o = p->o;
    a.B = p->B; a.Hq = p->Hq; a.Hkv = p->Hkv; a.L = p->L; a.G = lay.G; a.n_rg = lay.n_rg;
    a.q_sb = p->q_stride_b; a.q_sh = p->q_stride_h;
    a.kv_sb = p->kv_stride_b; a.kv_sh = p->kv_stride_h;
    a.o_sb = p->o_stride_b; a.o_sh = p->o_stride_h;
    a.seq_lens = p->seq_lens;
    a.scale = p->scale; a.phi = p->phi; a.a = p->a; a.b = p->b;
    a.p = lay.p; a.nsub = lay.nsub;
    a.row_flags = p->row_flags; a.viol_index = p->viol_index; a.rows_recomputed = p->rows_recomputed;
    a.chunk_num = p->chunk_num; a.chunk_den = p->chunk_den;
    a.ws_num = reinterpret_cast<float *>(ws + lay.off_num);
    a.ws_den = reinterpret_cast<float *>(ws + lay.off_den);
    a.ws_m = reinterpret_cast<float *>(ws + lay.off_m);
    a.ws_viol = reinterpret_cast<int *>(ws + lay.off_viol);
    a.counters = reinterpret_cast<int *>(ws + lay.off_cnt);
    const bool use_list = (int64_t)p->B * p->Hkv <= kFlagMax;
    int *flags = reinterpret_cast<int *>(ws + lay.off_flags);
    a.flag_count = flags;
    a.flag_list = use_list ? flags + kFlagListOff : nullptr;
    a.flag_mark = flags + kFlagListOff + kFlagMax;
    a.list_mode = false;
    a.cluster_join = false;
    a.cluster_recompute = false;
    a.abort_ok = false;
    a.kv_prefetch = p->kv_prefetch != 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    a.kv_rows_per_head = p->kv_stride_h / p->D;
    const bool sync_mma = mma_shape_ok(p, lay.G);  // GQA/MQA sync softmax on tensor cores
    CUtensorMap mk, mv;
    if (sync_mma || lay.mma) {
        if ((s = kv_maps(p, &mk, &mv)) != FDPP_OK) return s;
    }
    if (p->mode == FDPP_ATTN_SYNC) {
        a.only_flagged = false;
        if (sync_mma) {
            AttnArgs am = a;
            am.n_rg = lay.n_rg_mma;
            return launch_mma<false>(am, p->dtype, lay.P, &mk, &mv, st);
        }
        return by_dtype<false>(a, p->dtype, p->D, lay.GT, lay.P, st);
    }
    a.only_flagged = false;
    const bool cj = cluster_join_for(p, lay);
    // one launch: the cluster recomputes its own flagged rows (sync softmax on the
    // same path the recompute launch would take)
    const bool inc = cj && incluster_enabled() && (lay.mma ? sync_mma : true);
    if (lay.mma) {
        AttnArgs am = a;
        am.n_rg = lay.n_rg_mma;
        am.cluster_join = cj;
        am.cluster_recompute = inc;
        am.abort_ok = inc && abort_safe(p, lay);
        am.pscale = lay.pscale;
        am.inv_pscale = 1.f / lay.pscale;
        s = launch_mma<true>(am, p->dtype, lay.P, &mk, &mv, st);
    } else {
        AttnArgs ac = a;
        ac.cluster_join = cj;
        ac.cluster_recompute = inc;
        ac.abort_ok = false;  // the early stop is a tensor-core-path feature (attention_kernels.cuh)
        s = by_dtype<true>(ac, p->dtype, p->D, lay.GT, lay.P, st);
    }
    if (s != FDPP_OK || inc) return s;
    // synchronized recompute of flagged rows (attention.py:283-285), always launched
    a.only_flagged = true;
    if (use_list) {  // walk the flagged (batch, kv-head) list with one small wave
        const int sms = sm_count() > 0 ? sm_count() : 148;
        a.list_mode = true;
        if (sync_mma) {
            AttnArgs am = a;
            am.n_rg = lay.n_rg_mma;
            return launch_mma<false>(am, p->dtype, 2 * sms, &mk, &mv, st);
        }
        return by_dtype<false>(a, p->dtype, p->D, lay.GT, 2 * sms, st);
    }
    return by_dtype<false>(a, p->dtype, p->D, lay.GT, lay.P, st);
}
