// Subsystem 1 — split-KV decode/prefill attention on sm_100a: the kernels.
// (attention.cu holds the host side; attention_<dtype>_<mode>.cu instantiate
// one dtype x softmax mode each, so the build compiles them in parallel.)
//
// attn_split_kernel<ASYNC=true>  FlashDecoding++ asynchronized softmax
//   (attention.py:167-199 + :217-238 + :266-286): every CTA owns one sub-range
//   of one semantic chunk (chunk_bounds(L, p), softmax.py:103-110) for all the
//   query rows of its (batch, kv-head) row group.  K/V tiles stream through a
//   4-stage shared-memory ring filled by the TMA bulk engine (cp.async.bulk,
//   one producer warp); four consumer warps read 16-B vectors from shared
//   memory, reduce dot products with warp shuffles, apply the unified scale
//   phi, check the open band (a, b) per logit, and accumulate e^(x - phi) and
//   e^(x - phi)·v in fp32 with no max and no rescale.  The last CTA of the row
//   group (atomic ticket) joins all partials in fixed chunk/sub-range order,
//   applies the reference's "non-finite chunk state is a violation" rule and
//   writes O plus the per-row recompute flag.
//
// attn_split_kernel<ASYNC=false> FlashDecoding synchronized softmax
//   (attention.py:91-162): per-lane online max/rescale, Eq. (2) merge across
//   lanes, warps and sub-ranges in fixed order.  It serves mode="sync" and the
//   recompute of flagged rows: with `only_flagged`, row groups without a
//   flagged row exit before touching memory, so the launch can always be made
//   (graph-capturable, no host round trip).
#include <cfloat>
#include <cmath>
#include <cstring>

#pragma once

#include "common.cuh"

namespace fdpp {

constexpr int ATT_CONSUMERS = 4;                       // consumer warps
constexpr int ATT_THREADS = (ATT_CONSUMERS + 1) * 32;  // + 1 producer warp
constexpr int ATT_STAGES = 4;                          // K/V ring depth (the kernels' NST)
constexpr int ATT_MAX_P = 1024;                        // semantic chunks per row

struct AttnArgs {
    const void *q, *k, *v;
    void *o;
    int B, Hq, Hkv, L, G, n_rg;  // G = Hq / Hkv, n_rg = row groups per kv head
    int64_t q_sb, q_sh, kv_sb, kv_sh, o_sb, o_sh;
    const int32_t *seq_lens;
    float scale, phi, a, b;
    float pscale, inv_pscale;  // MMA path: power-of-two scale keeping e^(x-phi) in fp16 range
    int64_t kv_rows_per_head;  // MMA path: rows of one (batch, kv-head) in the 2-D K/V maps
    int p, nsub;
    uint8_t *row_flags;
    int32_t *viol_index;
    int32_t *rows_recomputed;
    float *chunk_num, *chunk_den;
    bool only_flagged;
    // workspace
    float *ws_num;  // [B*Hq][p*nsub][D]
    float *ws_den;  // [B*Hq][p*nsub]
    float *ws_m;    // [B*Hq][p*nsub]
    int *ws_viol;   // [B*Hq][p*nsub]
    int *counters;  // [B*Hkv*n_rg]
    // flagged (batch, kv-head) list: the async join appends, the recompute
    // launch walks it (list_mode) instead of one CTA per row group
    int *flag_list;   // [B*Hkv]
    int *flag_mark;   // [B*Hkv] dedupe markers
    int *flag_count;  // [0] entries, [32] CTAs done (reset by the recompute launch)
    bool list_mode;
    bool cluster_join;  // async: the P CTAs of a row group are one cluster (DSMEM join)
    bool cluster_recompute;  // cluster_join: flagged rows are recomputed by the same cluster
    bool abort_ok;           // cluster_recompute: a violation stops the group's async stream
    bool kv_prefetch;        // async: stream K/V rows before the appended one ahead of the PDL wait
};

template <typename T, int D>
struct AttnGeom {
    static constexpr int RB = D * (int)sizeof(T);         // bytes per key row
    static constexpr int VEC = 16 / (int)sizeof(T);       // elements per 16-B lane chunk
    static constexpr int LPK = RB / 16;                   // lanes per key
    static constexpr int KPI = 32 / LPK;                  // keys per warp iteration
    static constexpr int TK_RAW = 8192 / RB;
    static constexpr int TK = TK_RAW < 16 ? 16 : (TK_RAW > 256 ? 256 : TK_RAW);  // keys per stage
    static constexpr int STAGE_BYTES = 2 * TK * RB;       // K tile + V tile
    static_assert(LPK >= 1 && LPK <= 32 && (32 % LPK) == 0, "head dim");
    static_assert(TK % (ATT_CONSUMERS * KPI) == 0, "tile");
};

__device__ __forceinline__ int chunk_lo(int L, int p, int j) { return (L / p) * j; }
__device__ __forceinline__ int chunk_hi(int L, int p, int j) { return j == p - 1 ? L : (L / p) * (j + 1); }

template <typename T, int VEC>
__device__ __forceinline__ void load_vec(const T *src, float (&out)[VEC]) {
    int4 raw = *reinterpret_cast<const int4 *>(src);
    if constexpr (sizeof(T) == 4) {
        out[0] = __int_as_float(raw.x);
        out[1] = __int_as_float(raw.y);
        out[2] = __int_as_float(raw.z);
        out[3] = __int_as_float(raw.w);
    } else {
        uint32_t w[4] = {(uint32_t)raw.x, (uint32_t)raw.y, (uint32_t)raw.z, (uint32_t)raw.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float2 f = Elem<T>::to_f2(w[i]);
            out[2 * i] = f.x;
            out[2 * i + 1] = f.y;
        }
    }
}

__device__ __forceinline__ float safe_scale(float m, float mref) {
    return m == -INFINITY ? 0.f : __expf(m - mref);
}

// ---- tensor-core (mma.sync) helpers for the GQA/MQA consumer
template <typename T>
__device__ __forceinline__ void mma_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    if constexpr (std::is_same<T, __nv_bfloat16>::value)
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    else
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
template <typename T>
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    if constexpr (std::is_same<T, __nv_bfloat16>::value) {
        __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
        return *reinterpret_cast<uint32_t *>(&v);
    } else {
        __half2 v = __floats2half2_rn(lo, hi);
        return *reinterpret_cast<uint32_t *>(&v);
    }
}

// MMA = true: the GQA/MQA async path on tensor cores (mma.sync.m16n8k16; a
// decode step needs ~16 flop/B x HBM bandwidth ~ 0.1-0.2 PFLOP/s, the legacy
// pipe sustains ~0.55 PFLOP/s on B200: profiles/r1_mma_sync_throughput.txt).
// GT = 16 query rows of one kv head on the MMA M axis; K/V tiles arrive by
// 2-D TMA in the 128-byte swizzle (ldmatrix reads them conflict-free); per
// 16-key slice S = Q K^T, the unified-phi band check and e^(x - phi) in fp32
// (exp-sums stay fp32), P = e * pscale packed to 16 bits as the next MMA's A
// operand straight from the accumulators, O += P V.
#ifdef FDPP_ATRACE
// dev trace build only: per-CTA globaltimer stamps of the async launch (tools/attn_trace.py)
static __device__ unsigned long long g_atrace[8192][8];
#define ATRACE(slot)                                                                      \
    do {                                                                                  \
        const unsigned cid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z); \
        if (ASYNC && cid < 8192) g_atrace[cid][slot] = globaltimer_ns();                   \
    } while (0)
#else
#define ATRACE(slot) do { } while (0)
#endif

// append (batch, kv-head) to the recompute list once per launch
__device__ __forceinline__ void flag_group(const AttnArgs &a, int b, int kvh) {
    if (!a.flag_list) return;
    const int e = b * a.Hkv + kvh;
    if (atomicExch(&a.flag_mark[e], 1) == 0) a.flag_list[atomicAdd(a.flag_count, 1)] = e;
}

// One pass over this CTA's key range [k_begin, k_end): the producer warp streams
// K/V tiles through the ring, the consumer warps leave their partials in `red`
// (per warp; the async tensor-core form accumulates the warps in place).
// Tiles are numbered from `tbase` so a second pass continues the ring's
// mbarrier phases; `red_in_ring`: the partial buffers alias the ring (the
// consumers first wait for each other to finish reading it).
// `abortp` (async pass of a cluster-recomputed group): the first violation a
// consumer sees is OR-ed into this word in all `ncl` cluster CTAs; once set the
// producer stops streaming (it still completes each stage's barrier) and the
// consumers skip the remaining tiles -- the reference's break on violation
// (attention.py:184-186), extended to the whole group since it is recomputed.
// `wflags` (sync pass of an aborted group): the consumers also evaluate the
// async band check and exp-sums per row (first violating key, sum e^(x-phi) over
// in-band keys) so the group's flags can be derived exactly without the async pass.
template <typename T, int D, int GT, bool ASYNC, bool MMA, int NST = ATT_STAGES>
__device__ __forceinline__ void attn_stream(const AttnArgs &args, const CUtensorMap &tmK, const CUtensorMap &tmV,
                                            uint8_t *smem, uint64_t *full, uint64_t *empty, float *red,
                                            const bool red_in_ring, const int tbase, const int ntiles,
                                            const int k_begin, const int k_end, const int b, const int kvh,
                                            const int h0, const int gcount, uint32_t *abortp, const int ncl,
                                            float *wflags, const int Lb) {
    using Gm = AttnGeom<T, D>;
    constexpr int VEC = Gm::VEC, LPK = Gm::LPK, KPI = Gm::KPI, TK = Gm::TK, RB = Gm::RB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const T *kbase = static_cast<const T *>(args.k) + (int64_t)b * args.kv_sb + (int64_t)kvh * args.kv_sh;
    const T *vbase = static_cast<const T *>(args.v) + (int64_t)b * args.kv_sb + (int64_t)kvh * args.kv_sh;
    (void)VEC; (void)LPK; (void)KPI; (void)kbase; (void)vbase;
    const bool flags = !ASYNC && wflags != nullptr;
    constexpr int nst = NST;  // compile-time ring depth: a runtime modulo costs the issue-bound loop ~4 %
    // signal an abort to every CTA of the cluster (once per warp)
    auto signal_abort = [&]() {
        if (lane == 0)
            for (int q = 0; q < ncl; ++q) dsmem_red_or_u32(dsmem_map_addr(smem_u32(abortp), (uint32_t)q), 1u);
    };
    (void)signal_abort;

    if (warp == ATT_CONSUMERS) {
        // ------------------------------------------------ producer warp
        // kv_prefetch: the ring's first tiles that end before the appended row
        // (key Lb - 1, the only one the predecessor kernel writes) are requested
        // before the PDL wait, streaming under the predecessor's tail
        bool waited = !(ASYNC && args.kv_prefetch);
        if (lane == 0) {
            for (int t = 0; t < ntiles; ++t) {
                const int s = (tbase + t) % nst;
                const uint32_t ph = ((tbase + t) / nst) & 1;
                if (!waited && (tbase + t >= nst || k_begin + (t + 1) * TK >= Lb)) {
                    pdl_wait();
                    waited = true;
                }
                mbar_wait(&empty[s], ph ^ 1);
                if (abortp != nullptr && ld_volatile_u32(abortp) != 0u) {
                    mbar_arrive(&full[s]);  // aborted: complete the stage with no data
                    continue;
                }
                const int key0 = k_begin + t * TK;
                const int n = min(TK, k_end - key0);
                const uint32_t bytes = (uint32_t)n * RB;
                uint8_t *dk = smem + s * Gm::STAGE_BYTES;
                uint8_t *dv = dk + TK * RB;
                if constexpr (MMA) {
                    // [2 halves of 64 columns][TK rows][128 B], SWIZZLE_128B; whole boxes
                    const int row = (int)((int64_t)(b * args.Hkv + kvh) * args.kv_rows_per_head + key0);
                    mbar_arrive_expect_tx(&full[s], 4 * TK * 128);
                    tma_load_2d(dk, &tmK, &full[s], 0, row, kEvictFirst);
                    tma_load_2d(dk + TK * 128, &tmK, &full[s], 64, row, kEvictFirst);
                    tma_load_2d(dv, &tmV, &full[s], 0, row, kEvictFirst);
                    tma_load_2d(dv + TK * 128, &tmV, &full[s], 64, row, kEvictFirst);
                } else {
                    mbar_arrive_expect_tx(&full[s], 2 * bytes);
                    bulk_g2s(dk, kbase + (int64_t)key0 * D, bytes, &full[s], kEvictFirst);
                    bulk_g2s(dv, vbase + (int64_t)key0 * D, bytes, &full[s], kEvictFirst);
                }
            }
            ATRACE(7);
        }
        __syncwarp();
        if (!waited) pdl_wait();  // before this warp's threads write anything in the join
        if (abortp != nullptr) cluster_wait();  // pairs with attn_cta's cluster_arrive
    } else if constexpr (MMA) {
        // ------------------------------------------------ consumer warps, tensor cores
        // warps 0,1 take the two 16-key slices of even stages, warps 2,3 of odd stages
        // the cluster barrier attn_cta arrived on (every peer's abort word is
        // initialised) is awaited lazily: before this warp's first signal, else
        // after its loop -- never on the critical path of the first tile
        bool cw = abortp == nullptr;
        const int r0 = lane >> 2, cq = (lane & 3) * 2;
        uint32_t qa[D / 16][4];  // Q rows [16 x D] as m16n8k16 A fragments
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int row = r0 + (i & 1) * 8, col = 16 * kk + cq + (i >> 1) * 8;
                qa[kk][i] = row < gcount
                                ? *reinterpret_cast<const uint32_t *>(
                                      static_cast<const T *>(args.q) + (int64_t)b * args.q_sb +
                                      (int64_t)(h0 + row) * args.q_sh + col)
                                : 0u;
            }
        float o[D / 8][4];
#pragma unroll
        for (int nb = 0; nb < D / 8; ++nb) o[nb][0] = o[nb][1] = o[nb][2] = o[nb][3] = 0.f;
        float den0 = 0.f, den1 = 0.f;
        int viol0 = INT_MAX, viol1 = INT_MAX;
        float mx0 = -INFINITY, mx1 = -INFINITY;  // sync: running row maxima
        float dena0 = 0.f, dena1 = 0.f;          // sync with flags: async exp-sums
        bool signaled = false;
        const float scale = args.scale, phi = args.phi, ba = args.a, bb = args.b, ps = args.pscale;
        const int mi = lane >> 3, mr = lane & 7;  // ldmatrix: matrix / row this lane addresses
        for (int t = warp >> 1; t < ntiles; t += 2) {
            const int s = (tbase + t) % nst;
            mbar_wait(&full[s], ((tbase + t) / nst) & 1);
            const int key0 = k_begin + t * TK;
            const int n = min(TK, k_end - key0);
            const uint32_t sk = smem_u32(smem + s * Gm::STAGE_BYTES), sv = sk + TK * RB;
            const bool skip = abortp != nullptr && __shfl_sync(0xffffffffu, ld_volatile_u32(abortp), 0) != 0u;
            for (int k0 = (warp & 1) * 16; k0 < TK && !skip; k0 += 32) {
                if (k0 >= n) break;
                // S = Q K^T for keys k0 .. k0+15 (two n8 blocks)
                float sacc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
                {
                    const int key = k0 + (mi >> 1) * 8 + mr;
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const int chunk = 2 * (kk & 3) + (mi & 1);
                        uint32_t kb[4];
                        ldsm_x4(kb, sk + (kk >> 2) * TK * 128 + key * 128 + ((chunk ^ (key & 7)) << 4));
                        mma_16816<T>(sacc[0], qa[kk], kb[0], kb[1]);
                        mma_16816<T>(sacc[1], qa[kk], kb[2], kb[3]);
                    }
                }
                float ep[2][4];
                if constexpr (ASYNC) {
                    // unified phi: band check, e^(x - phi) in fp32, P = e * pscale (16-bit)
#pragma unroll
                    for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int key = k0 + 8 * nb + cq + (i & 1);
                            // shifted logit scale * dot - phi in one fused multiply-add: the
                            // sync pass's band check (flags of an aborted group) repeats it
                            // exactly; vs the oracle's two roundings it can differ only
                            // within an ulp of the band edge (the tests' guard band)
                            const float ti = __fmaf_rn(sacc[nb][i], scale, -phi);
                            const bool valid = key < n, bad = (ti <= ba) || (ti >= bb);
                            if (valid && bad) {
                                if (i < 2) viol0 = min(viol0, key0 + key);
                                else viol1 = min(viol1, key0 + key);
                            }
                            const float e = (valid && !bad) ? __expf(ti) : 0.f;
                            if (i < 2) den0 += e;
                            else den1 += e;
                            ep[nb][i] = e * ps;
                        }
                } else {
                    // synchronized softmax (FlashDecoding, attention.py:91-162): per-row
                    // running max over the slice (quad-shared rows), rescale, P <= 1
                    float sm0 = -INFINITY, sm1 = -INFINITY;
#pragma unroll
                    for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int key = k0 + 8 * nb + cq + (i & 1);
                            const float x = sacc[nb][i] * scale;
                            if (flags && key < n) {  // the async pass's band check and exp-sum
                                const float ti = __fmaf_rn(sacc[nb][i], scale, -phi);
                                const bool bad = (ti <= ba) || (ti >= bb);
                                if (bad) {
                                    if (i < 2) viol0 = min(viol0, key0 + key);
                                    else viol1 = min(viol1, key0 + key);
                                } else if (i < 2) {
                                    dena0 += __expf(ti);
                                } else {
                                    dena1 += __expf(ti);
                                }
                            }
                            sacc[nb][i] = key < n ? x : -INFINITY;
                            if (i < 2) sm0 = fmaxf(sm0, sacc[nb][i]);
                            else sm1 = fmaxf(sm1, sacc[nb][i]);
                        }
#pragma unroll
                    for (int off = 1; off < 4; off <<= 1) {
                        sm0 = fmaxf(sm0, __shfl_xor_sync(0xffffffffu, sm0, off));
                        sm1 = fmaxf(sm1, __shfl_xor_sync(0xffffffffu, sm1, off));
                    }
                    const float n0 = fmaxf(mx0, sm0), n1 = fmaxf(mx1, sm1);
                    const float f0 = safe_scale(mx0, n0), f1 = safe_scale(mx1, n1);
                    mx0 = n0;
                    mx1 = n1;
                    den0 *= f0;
                    den1 *= f1;
#pragma unroll
                    for (int nb2 = 0; nb2 < D / 8; ++nb2) {
                        o[nb2][0] *= f0;
                        o[nb2][1] *= f0;
                        o[nb2][2] *= f1;
                        o[nb2][3] *= f1;
                    }
#pragma unroll
                    for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const float m = i < 2 ? mx0 : mx1;
                            const float e = m == -INFINITY ? 0.f : __expf(sacc[nb][i] - m);
                            if (i < 2) den0 += e;
                            else den1 += e;
                            ep[nb][i] = e;
                        }
                }
                const uint32_t pa[4] = {pack2<T>(ep[0][0], ep[0][1]), pack2<T>(ep[0][2], ep[0][3]),
                                        pack2<T>(ep[1][0], ep[1][1]), pack2<T>(ep[1][2], ep[1][3])};
                // O += P V
                {
                    const int key = k0 + (mi & 1) * 8 + mr;
#pragma unroll
                    for (int jj = 0; jj < D / 16; ++jj) {
                        const int chunk = 2 * (jj & 3) + (mi >> 1);
                        uint32_t vb[4];
                        ldsm_x4_t(vb, sv + (jj >> 2) * TK * 128 + key * 128 + ((chunk ^ (key & 7)) << 4));
                        mma_16816<T>(o[2 * jj], pa, vb[0], vb[1]);
                        mma_16816<T>(o[2 * jj + 1], pa, vb[2], vb[3]);
                    }
                }
            }
            if constexpr (ASYNC) {
                if (abortp != nullptr && !signaled && __any_sync(0xffffffffu, min(viol0, viol1) != INT_MAX)) {
                    if (!cw) cluster_wait();
                    cw = signaled = true;
                    signal_abort();
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (!cw) cluster_wait();
        // rows r0 / r0+8 are shared by the lane quad: fixed butterfly (sync: the
        // quad already shares one running max per row)
#pragma unroll
        for (int off = 1; off < 4; off <<= 1) {
            den0 += __shfl_xor_sync(0xffffffffu, den0, off);
            den1 += __shfl_xor_sync(0xffffffffu, den1, off);
            viol0 = min(viol0, __shfl_xor_sync(0xffffffffu, viol0, off));
            viol1 = min(viol1, __shfl_xor_sync(0xffffffffu, viol1, off));
            dena0 += __shfl_xor_sync(0xffffffffu, dena0, off);
            dena1 += __shfl_xor_sync(0xffffffffu, dena1, off);
        }
        if (threadIdx.x == 0) ATRACE(6);
        pdl_trigger();  // main stream done: the next kernel may start its prologue
        if constexpr (!ASYNC) {
            // per-warp partials (num, den, running max) for the Eq. (2) merge below
            if (red_in_ring) named_bar_sync(2, ATT_CONSUMERS * 32);  // every warp is done with the ring
            float *rw = red + warp * GT * (D + 2);
#pragma unroll
            for (int nb = 0; nb < D / 8; ++nb)
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    rw[(r0 + (i >> 1) * 8) * (D + 2) + 8 * nb + cq + (i & 1)] = o[nb][i];
            if ((lane & 3) == 0) {
                rw[r0 * (D + 2) + D] = den0;
                rw[(r0 + 8) * (D + 2) + D] = den1;
                rw[r0 * (D + 2) + D + 1] = mx0;
                rw[(r0 + 8) * (D + 2) + D + 1] = mx1;
                if (flags) {
                    float *wf = wflags + warp * GT * 2;
                    wf[r0 * 2] = __int_as_float(viol0);
                    wf[r0 * 2 + 1] = dena0;
                    wf[(r0 + 8) * 2] = __int_as_float(viol1);
                    wf[(r0 + 8) * 2 + 1] = dena1;
                }
            }
        } else {
        // warps add into one [GT][D+2] buffer in fixed order (numerators unscaled exactly)
        const float ips = args.inv_pscale;
#pragma unroll 1
        for (int w = 0; w < ATT_CONSUMERS; ++w) {
            if (warp == w) {
                // this thread's 2-float pairs: all earlier sums loaded first, then stored
                float2 prev[D / 8][2];
#pragma unroll
                for (int nb = 0; nb < D / 8; ++nb)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        prev[nb][h] = w == 0 ? make_float2(0.f, 0.f)
                                             : *reinterpret_cast<const float2 *>(
                                                   red + (r0 + h * 8) * (D + 2) + 8 * nb + cq);
#pragma unroll
                for (int nb = 0; nb < D / 8; ++nb)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        *reinterpret_cast<float2 *>(red + (r0 + h * 8) * (D + 2) + 8 * nb + cq) =
                            make_float2(prev[nb][h].x + o[nb][2 * h] * ips, prev[nb][h].y + o[nb][2 * h + 1] * ips);
                if ((lane & 3) == 0) {
                    float *d0 = red + r0 * (D + 2), *d1 = red + (r0 + 8) * (D + 2);
                    d0[D] = (w == 0 ? 0.f : d0[D]) + den0;
                    d1[D] = (w == 0 ? 0.f : d1[D]) + den1;
                    d0[D + 1] = __int_as_float(w == 0 ? viol0 : min(__float_as_int(d0[D + 1]), viol0));
                    d1[D + 1] = __int_as_float(w == 0 ? viol1 : min(__float_as_int(d1[D + 1]), viol1));
                }
            }
            named_bar_sync(1, ATT_CONSUMERS * 32);
        }
        }  // ASYNC
    } else {
        // ------------------------------------------------ consumer warps
        // (no early stop here: the CUDA-core form is issue-bound, and even the idle
        // per-tile violation check cost 5% of the 7B step's attention, so only the
        // tensor-core form takes abort signals; the host never passes abortp here)
        const int c = lane % LPK;          // 16-B chunk of the head dim owned by this lane
        const int kg = lane / LPK;         // key slot inside a warp iteration
        float q[GT][VEC];
#pragma unroll
        for (int g = 0; g < GT; ++g) {
            if (g < gcount) {
                const T *qp = static_cast<const T *>(args.q) + (int64_t)b * args.q_sb +
                              (int64_t)(h0 + g) * args.q_sh + c * VEC;
                load_vec<T, VEC>(qp, q[g]);
            } else {
#pragma unroll
                for (int v = 0; v < VEC; ++v) q[g][v] = 0.f;
            }
        }
        float num[GT][VEC], den[GT], mx[GT], dena[GT];
        int viol[GT];
#pragma unroll
        for (int g = 0; g < GT; ++g) {
            den[g] = 0.f;
            dena[g] = 0.f;
            mx[g] = -INFINITY;
            viol[g] = INT_MAX;
#pragma unroll
            for (int v = 0; v < VEC; ++v) num[g][v] = 0.f;
        }
        const float scale = args.scale, phi = args.phi, ba = args.a, bb = args.b;

        for (int t = 0; t < ntiles; ++t) {
            const int s = (tbase + t) % nst;
            const uint32_t ph = ((tbase + t) / nst) & 1;
            mbar_wait(&full[s], ph);
            const int key0 = k_begin + t * TK;
            const int n = min(TK, k_end - key0);
            const T *sk = reinterpret_cast<const T *>(smem + s * Gm::STAGE_BYTES);
            const T *sv = sk + TK * D;
            // (after an abort the producer completes stages without data; the
            // CUDA-core consumers just run through them -- their partials are
            // discarded -- rather than pay a per-tile check on the clean path)
#pragma unroll 2
            for (int kk0 = warp * KPI; kk0 < n; kk0 += ATT_CONSUMERS * KPI) {
                const int kk = kk0 + kg;
                const bool valid = kk < n;
                float kf[VEC];
                load_vec<T, VEC>(sk + (valid ? kk : 0) * D + c * VEC, kf);
                float dot[GT];
#pragma unroll
                for (int g = 0; g < GT; ++g) {
                    float sacc = 0.f;
#pragma unroll
                    for (int v = 0; v < VEC; ++v) sacc = fmaf(q[g][v], kf[v], sacc);
#pragma unroll
                    for (int o = LPK / 2; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
                    dot[g] = sacc;
                }
                float vf[VEC];
                load_vec<T, VEC>(sv + (valid ? kk : 0) * D + c * VEC, vf);
#pragma unroll
                for (int g = 0; g < GT; ++g) {
                    const float x = dot[g] * scale;       // logit, reference order: scale * acc
                    float e;
                    if constexpr (ASYNC) {
                        const float ti = __fmaf_rn(dot[g], scale, -phi);  // as the flags pass below
                        const bool bad = (ti <= ba) || (ti >= bb);
                        if (valid && bad) viol[g] = min(viol[g], key0 + kk);
                        e = (valid && !bad) ? __expf(ti) : 0.f;
                    } else {
                        if (flags && valid) {  // the async pass's band check and exp-sum
                            const float ti = __fmaf_rn(dot[g], scale, -phi);
                            const bool bad = (ti <= ba) || (ti >= bb);
                            if (bad) viol[g] = min(viol[g], key0 + kk);
                            else dena[g] += __expf(ti);
                        }
                        if (valid && x > mx[g]) {         // online max: rescale running state
                            const float f = safe_scale(mx[g], x);
                            den[g] *= f;
#pragma unroll
                            for (int v = 0; v < VEC; ++v) num[g][v] *= f;
                            mx[g] = x;
                        }
                        e = valid ? __expf(x - mx[g]) : 0.f;
                    }
                    den[g] += e;
#pragma unroll
                    for (int v = 0; v < VEC; ++v) num[g][v] = fmaf(e, vf[v], num[g][v]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }

        // ---- reduce across the key slots of the warp (lanes with equal c), fixed butterfly
#pragma unroll
        for (int g = 0; g < GT; ++g) {
#pragma unroll
            for (int o = LPK; o < 32; o <<= 1) {
                if constexpr (ASYNC) {
                    den[g] += __shfl_xor_sync(0xffffffffu, den[g], o);
#pragma unroll
                    for (int v = 0; v < VEC; ++v) num[g][v] += __shfl_xor_sync(0xffffffffu, num[g][v], o);
                    viol[g] = min(viol[g], __shfl_xor_sync(0xffffffffu, viol[g], o));
                } else {
                    const float m2 = __shfl_xor_sync(0xffffffffu, mx[g], o);
                    const float l2 = __shfl_xor_sync(0xffffffffu, den[g], o);
                    const float mm = fmaxf(mx[g], m2);
                    const float f1 = safe_scale(mx[g], mm), f2 = safe_scale(m2, mm);
                    den[g] = den[g] * f1 + l2 * f2;
#pragma unroll
                    for (int v = 0; v < VEC; ++v) {
                        const float a2 = __shfl_xor_sync(0xffffffffu, num[g][v], o);
                        num[g][v] = num[g][v] * f1 + a2 * f2;
                    }
                    mx[g] = mm;
                    if (flags) {
                        viol[g] = min(viol[g], __shfl_xor_sync(0xffffffffu, viol[g], o));
                        dena[g] += __shfl_xor_sync(0xffffffffu, dena[g], o);
                    }
                }
            }
        }
        if (threadIdx.x == 0) ATRACE(6);
        pdl_trigger();  // main stream done: the next kernel may start its prologue
        // ---- per-warp partials to shared memory: red[w][g][0..D) = num, [D] = den, [D+1] = m/viol
        if (red_in_ring) named_bar_sync(2, ATT_CONSUMERS * 32);  // every warp is done with the ring
        if (kg == 0) {
#pragma unroll
            for (int g = 0; g < GT; ++g) {
                float *r = red + (warp * GT + g) * (D + 2);
#pragma unroll
                for (int v = 0; v < VEC; ++v) r[c * VEC + v] = num[g][v];
                if (c == 0) {
                    r[D] = den[g];
                    r[D + 1] = ASYNC ? __int_as_float(viol[g]) : mx[g];
                    if (flags) {
                        wflags[(warp * GT + g) * 2] = __int_as_float(viol[g]);
                        wflags[(warp * GT + g) * 2 + 1] = dena[g];
                    }
                }
            }
        }
    }
}

template <typename T, int D, int GT, bool ASYNC, bool MMA, int NST = ATT_STAGES>
__device__ __forceinline__ void attn_cta(const AttnArgs &args, const CUtensorMap &tmK, const CUtensorMap &tmV,
                                         const int cta, const int by, const int b) {
    using Gm = AttnGeom<T, D>;
    constexpr int VEC = Gm::VEC, LPK = Gm::LPK, KPI = Gm::KPI, TK = Gm::TK, RB = Gm::RB;
    // per-warp partial buffers in `red` (the async MMA path accumulates warps in place)
    constexpr int NRED = (MMA && ASYNC) ? 1 : ATT_CONSUMERS;
    static_assert(!MMA || (GT == 16 && D == 128 && sizeof(T) == 2 && TK % 32 == 0), "MMA path");

    extern __shared__ __align__(128) uint8_t smem_raw[];
    // the MMA path's TMA swizzle needs 1024-byte aligned stages
    // (an integer offset from the shared array keeps the pointer in the shared
    // window, so every access below compiles to LDS/STS, not generic LD/ST)
    uint8_t *smem = MMA ? smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u) : smem_raw;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + NST * Gm::STAGE_BYTES);
    uint64_t *empty = full + NST;
    float *red = reinterpret_cast<float *>(empty + NST);  // [NRED][GT][D+2]
    // join scratch aliases the K/V ring (free once every tile has been consumed)
    float *s_cden = reinterpret_cast<float *>(smem);
    int *s_cviol = reinterpret_cast<int *>(smem) + ATT_MAX_P;
    int *s_unrep = reinterpret_cast<int *>(smem) + 2 * ATT_MAX_P;
    static_assert(ATT_STAGES * Gm::STAGE_BYTES >= 3 * ATT_MAX_P * 4, "join scratch");
    __shared__ int s_last, s_any_flag, s_grp_flag;
    __shared__ uint32_t s_gmask;  // cluster join: flagged rows of the whole row group (bit g)
    __shared__ uint32_t s_abort;  // cluster recompute: some rank of the group saw a violation

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int P = args.p * args.nsub;
    // cta: (chunk, sub) index in [0, P); by: kv-head x row group; b: batch row
    const int j = cta / args.nsub, sub = cta % args.nsub;
    const int rg = by % args.n_rg, kvh = by / args.n_rg;
    const int g0 = rg * GT;
    const int gcount = min(GT, args.G - g0);
    const int h0 = kvh * args.G + g0;         // first query head of this row group

    if (threadIdx.x == 0) ATRACE(0);
    // q, the appended K/V row and row_flags come from earlier kernels; with
    // kv_prefetch the producer warp waits inside its loop instead (attn_stream)
    const int warp_id = threadIdx.x >> 5;
    if (!(ASYNC && args.kv_prefetch && warp_id == ATT_CONSUMERS)) pdl_wait();
    if (threadIdx.x == 0) ATRACE(1);
    if (!ASYNC && args.only_flagged) {        // recompute launch: skip clean row groups
        int any = 0;
        for (int g = 0; g < gcount; ++g) any |= args.row_flags[(int64_t)b * args.Hq + h0 + g];
        if (!any) {
            pdl_trigger();
            return;
        }
    }

    const int Lb = args.seq_lens ? min(args.seq_lens[b], args.L) : args.L;
    const int lo_j = chunk_lo(Lb, args.p, j), hi_j = chunk_hi(Lb, args.p, j);
    const int per = (hi_j - lo_j + args.nsub - 1) / args.nsub;
    const int k_begin = min(hi_j, lo_j + sub * per);
    const int k_end = min(hi_j, k_begin + per);
    const int nkeys = k_end - k_begin;
    const int ntiles = (nkeys + TK - 1) / TK;


    if (threadIdx.x == 0) {
        s_gmask = 0u;  // peers OR into it only after the first cluster barrier
        s_abort = 0u;  // peers OR into it only after the cluster launch's initial sync below
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], MMA ? 2 : ATT_CONSUMERS);  // MMA: two warps per stage
        }
        fence_mbar_init();
    }
    __syncthreads();

    const int row0 = b * args.Hq + h0;        // global row index of g = 0
    if (threadIdx.x == 0) ATRACE(2);
    // (a row group of one CTA is launched without a cluster: its split cluster
    // barrier would act as a CTA-wide one and deadlock the lazy waits below)
    const bool use_abort = ASYNC && args.cluster_join && args.abort_ok && P >= 2;
    // every rank's s_abort must be initialised before a peer ORs into it: arrive
    // now; the consumers wait before their first signal (or after their loop),
    // the producer after its loop
    if (use_abort) cluster_arrive();

    attn_stream<T, D, GT, ASYNC, MMA, NST>(args, tmK, tmV, smem, full, empty, red, false, 0, ntiles, k_begin, k_end,
                                      b, kvh, h0, gcount, use_abort ? &s_abort : nullptr, P, nullptr, Lb);
    __syncthreads();

    if constexpr (ASYNC) {
        if (args.cluster_join) {
            // The P CTAs of this row group form one thread-block cluster (rank = chunk j,
            // nsub = 1): the join reads the peers' [GT][D+2] partials over DSMEM instead of
            // publishing to global memory for a last-arriving CTA to re-read (that join was
            // per-CTA-bandwidth bound: P x GT x D x 4 bytes through one CTA).  Rank r joins
            // rows r, r + P, ...; chunk sums in chunk (= rank) order as the global join.
            __shared__ float s_dsum;
            uint32_t my_mask = 0u;  // rows this rank flagged (bit g)
            if constexpr (NRED > 1) {
                // CUDA-core form: sum the consumer warps' partials into warp 0's buffer
                // (warp order, as the join below always did) so peers read one value
                // per element over DSMEM instead of NRED
                for (int idx = threadIdx.x; idx < gcount * (D + 2); idx += ATT_THREADS) {
                    const int g = idx / (D + 2), e = idx % (D + 2);
                    if (e <= D) {
                        float s = 0.f;
#pragma unroll
                        for (int w = 0; w < NRED; ++w) s += red[(w * GT + g) * (D + 2) + e];
                        red[g * (D + 2) + e] = s;
                    } else {
                        int v = INT_MAX;
#pragma unroll
                        for (int w = 0; w < NRED; ++w) v = min(v, __float_as_int(red[(w * GT + g) * (D + 2) + e]));
                        red[g * (D + 2) + e] = __int_as_float(v);
                    }
                }
            }
            if (threadIdx.x == 0) ATRACE(3);
            const uint32_t red_addr = smem_u32(red);
            const int rank = (int)cluster_ctarank();
            cluster_sync_all();  // every rank's partial is in its shared memory (and every abort signal)
            if (threadIdx.x == 0) ATRACE(4);
            // the group stopped streaming on a violation: its async partials are
            // incomplete, so every row is recomputed and flagged from the sync pass
            const bool aborted = use_abort && s_abort != 0u;
            uint32_t gmask;
            if (!aborted) {
                for (int g = rank; g < gcount; g += P) {  // uniform per CTA
                    const int64_t row = row0 + g;
                    const uint32_t ra = red_addr + (uint32_t)(g * (D + 2)) * 4u;
                    int bad = 0;
                    float acc = 0.f;
                    // every rank's value of this element requested at once (one DSMEM
                    // round trip), then summed in chunk (= rank) order
                    for (int d = threadIdx.x; d < D; d += ATT_THREADS) {
                        float cv[16];
#pragma unroll
                        for (int q = 0; q < 16; ++q)
                            cv[q] = q < P ? dsmem_ld_f32_batched(dsmem_map_addr(ra + 4u * d, q)) : 0.f;
#pragma unroll
                        for (int q = 0; q < 16; ++q) {
                            if (q < P) {
                                bad |= !isfinite(cv[q]);
                                acc += cv[q];
                            }
                        }
                    }
                    if (warp == ATT_CONSUMERS) {  // the idle producer warp: lane q reads chunk q's state
                        float dq = 0.f;
                        int vq = INT_MAX;
                        if (lane < P) {
                            dq = dsmem_ld_f32_batched(dsmem_map_addr(ra + 4u * D, lane));
                            vq = __float_as_int(dsmem_ld_f32_batched(dsmem_map_addr(ra + 4u * (D + 1), lane)));
                        }
                        // a violating key or a non-finite chunk state is a violation
                        bad |= __any_sync(0xffffffffu, lane < P && ((vq != INT_MAX) || !isfinite(dq)));
                        float dsum = 0.f;
                        for (int q = 0; q < P; ++q) dsum += __shfl_sync(0xffffffffu, dq, q);  // chunk order
                        if (lane == 0) s_dsum = dsum;
                    }
                    const bool flagged = __syncthreads_or(bad) != 0;
                    if (threadIdx.x == 0) {
                        args.row_flags[row] = flagged ? 1 : 0;
                        if (flagged) {
                            if (args.rows_recomputed) atomicAdd(args.rows_recomputed, 1);
                            if (!args.cluster_recompute) flag_group(args, b, kvh);
                        }
                    }
                    my_mask |= flagged ? (1u << g) : 0u;
                    if (!flagged && threadIdx.x < D)  // D <= 4 warps on this path (host check)
                        static_cast<T *>(args.o)[(int64_t)b * args.o_sb + (int64_t)(h0 + g) * args.o_sh + threadIdx.x] =
                            Elem<T>::from_f(acc / s_dsum);
                    __syncthreads();  // s_dsum is rewritten by the next row
                }
                // publish this rank's flagged rows to every rank of the group (DSMEM OR,
                // ordered by the barrier's release/acquire)
                if (args.cluster_recompute && my_mask != 0u && threadIdx.x < P)
                    dsmem_red_or_u32(dsmem_map_addr(smem_u32(&s_gmask), threadIdx.x), my_mask);
                cluster_sync_all();  // peers may still be reading this CTA's partial
                if (threadIdx.x == 0) ATRACE(5);
                gmask = s_gmask;     // the same on every rank
                if (!args.cluster_recompute || gmask == 0u) return;
            } else {
                gmask = gcount >= 32 ? 0xffffffffu : ((1u << gcount) - 1u);  // no peer read our partial
            }

            // ---- synchronized recompute of the flagged rows inside the cluster
            // (attention.py:283-285): every rank re-streams its own chunk with the
            // running-max softmax -- no second launch, no host round trip, no list.
            // Per-warp partials alias the idle K/V ring; the CTA's Eq. (2) merge of
            // its warps lands in `red`, then rank r joins the flagged rows r, r + P, ...
            // over DSMEM in chunk (= rank) order, exactly as the recompute launch's join.
            // An aborted group also carries the async band check through the pass:
            // per-warp [GT][2] (first violating key, in-band exp-sum) after the
            // warp partials, merged per CTA into mflags[GT][2].
            float *wred = reinterpret_cast<float *>(smem);
            float *wflags = wred + ATT_CONSUMERS * GT * (D + 2);
            float *mflags = wflags + ATT_CONSUMERS * GT * 2;
            static_assert(ATT_STAGES * Gm::STAGE_BYTES >= (ATT_CONSUMERS * GT * (D + 4) + GT * 2) * 4,
                          "ring holds warp partials and flags");
            attn_stream<T, D, GT, false, MMA, NST>(args, tmK, tmV, smem, full, empty, wred, true, ntiles, ntiles,
                                              k_begin, k_end, b, kvh, h0, gcount, nullptr, P,
                                              aborted ? wflags : nullptr, Lb);
            __syncthreads();
            for (int idx = threadIdx.x; idx < gcount * (D + 2); idx += ATT_THREADS) {
                const int g = idx / (D + 2), e = idx % (D + 2);
                float mm = -INFINITY;
                for (int w = 0; w < ATT_CONSUMERS; ++w) mm = fmaxf(mm, wred[(w * GT + g) * (D + 2) + D + 1]);
                float s = 0.f;
                for (int w = 0; w < ATT_CONSUMERS; ++w) {
                    const float *r = wred + (w * GT + g) * (D + 2);
                    s += r[e < D ? e : D] * safe_scale(r[D + 1], mm);
                }
                red[g * (D + 2) + e] = e <= D ? s : mm;
            }
            if (aborted && threadIdx.x < gcount) {
                const int g = threadIdx.x;
                int vm = INT_MAX;
                float da = 0.f;
                for (int w = 0; w < ATT_CONSUMERS; ++w) {  // warp order
                    vm = min(vm, __float_as_int(wflags[(w * GT + g) * 2]));
                    da += wflags[(w * GT + g) * 2 + 1];
                }
                mflags[g * 2] = __int_as_float(vm);
                mflags[g * 2 + 1] = da;
            }
            cluster_sync_all();  // every rank's merged sync partial is in `red`
            const uint32_t mf_addr = smem_u32(mflags);
            for (int g = rank; g < gcount; g += P) {
                if (!((gmask >> g) & 1u)) continue;
                const uint32_t ra = red_addr + (uint32_t)(g * (D + 2)) * 4u;
                float mq[16];
                float mrow = -INFINITY;
                int bad = 0;
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    mq[q] = q < P ? dsmem_ld_f32(dsmem_map_addr(ra + 4u * (D + 1), q)) : -INFINITY;
                    mrow = fmaxf(mrow, mq[q]);
                }
                if (aborted && threadIdx.x < P) {  // rank q's chunk: a violating key or a non-finite exp-sum
                    const uint32_t fa = mf_addr + (uint32_t)(g * 2) * 4u;
                    const int vq = __float_as_int(dsmem_ld_f32(dsmem_map_addr(fa, threadIdx.x)));
                    const float dq = dsmem_ld_f32(dsmem_map_addr(fa + 4u, threadIdx.x));
                    bad |= (vq != INT_MAX) || !isfinite(dq);
                }
                float l = 0.f;
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    mq[q] = safe_scale(mq[q], mrow);  // now the rank's rescale factor
                    if (q < P) l += dsmem_ld_f32(dsmem_map_addr(ra + 4u * D, q)) * mq[q];
                }
                for (int d = threadIdx.x; d < D; d += ATT_THREADS) {
                    float acc = 0.f;
#pragma unroll
                    for (int q = 0; q < 16; ++q)
                        if (q < P) acc += dsmem_ld_f32(dsmem_map_addr(ra + 4u * d, q)) * mq[q];
                    const float o = acc / l;
                    bad |= !isfinite(o);  // non-finite V reaches the sync numerators too
                    static_cast<T *>(args.o)[(int64_t)b * args.o_sb + (int64_t)(h0 + g) * args.o_sh + d] =
                        Elem<T>::from_f(o);
                }
                if (aborted) {
                    const bool flagged = __syncthreads_or(bad) != 0;
                    if (threadIdx.x == 0) {
                        args.row_flags[row0 + g] = flagged ? 1 : 0;
                        if (flagged && args.rows_recomputed) atomicAdd(args.rows_recomputed, 1);
                    }
                }
            }
            cluster_sync_all();  // peers may still be reading this CTA's merged partial
            return;
        }
    }

    // ---- merge the consumer warps in fixed order and write this CTA's partial
    for (int idx = threadIdx.x; idx < gcount * (D + 2); idx += ATT_THREADS) {
        const int g = idx / (D + 2), e = idx % (D + 2);
        const int64_t slot = (int64_t)(row0 + g) * P + cta;
        if (ASYNC) {
            if (e < D) {
                float s = 0.f;
                for (int w = 0; w < NRED; ++w) s += red[(w * GT + g) * (D + 2) + e];
                args.ws_num[slot * D + e] = s;
            } else if (e == D) {
                float s = 0.f;
                for (int w = 0; w < NRED; ++w) s += red[(w * GT + g) * (D + 2) + D];
                args.ws_den[slot] = s;
            } else {
                int vm = INT_MAX;
                for (int w = 0; w < NRED; ++w)
                    vm = min(vm, __float_as_int(red[(w * GT + g) * (D + 2) + D + 1]));
                args.ws_viol[slot] = vm;
            }
        } else {
            float mm = -INFINITY;
            for (int w = 0; w < ATT_CONSUMERS; ++w) mm = fmaxf(mm, red[(w * GT + g) * (D + 2) + D + 1]);
            float s = 0.f;
            for (int w = 0; w < ATT_CONSUMERS; ++w) {
                const float *r = red + (w * GT + g) * (D + 2);
                s += r[e < D ? e : D] * safe_scale(r[D + 1], mm);
            }
            if (e < D) args.ws_num[slot * D + e] = s;
            else if (e == D) args.ws_den[slot] = s;
            else args.ws_m[slot] = mm;
        }
    }

    // ---- last CTA of the row group joins all partials (fixed order)
    if (threadIdx.x == 0) ATRACE(3);
    __threadfence();
    __syncthreads();
    const int counter = (b * args.Hkv + kvh) * args.n_rg + rg;
    if (threadIdx.x == 0) {
        const int ticket = atomicAdd(&args.counters[counter], 1);
        s_last = (ticket == P - 1);
        if (s_last) args.counters[counter] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) ATRACE(4);
    if (!s_last) return;
    __threadfence();
    if (ASYNC) {
        if (threadIdx.x == 0) s_grp_flag = 0;
        __syncthreads();
    }

    if (ASYNC && !args.viol_index && !args.chunk_num && !args.chunk_den) {
        // decode hot path (no per-chunk outputs requested): one warp per query
        // row, all rows of the group in parallel, every partial load of a row
        // batched (the block-wide join below serialises rows: ~GT x slower at G = 16)
        const int nsub = args.nsub;
        for (int g = warp; g < gcount; g += ATT_THREADS / 32) {
            const int64_t row = row0 + g;
            const int64_t base = row * P;
            // chunk verdicts: lane jj owns chunks jj, jj+32, ..; exp-sums in sub order
            float dpart = 0.f;
            bool bad = false;
            for (int jj = lane; jj < args.p; jj += 32) {
                float cd = 0.f;
                int vm = INT_MAX;
                for (int q = 0; q < nsub; ++q) {
                    const int64_t i = base + (int64_t)jj * nsub + q;
                    cd += __ldcg(&args.ws_den[i]);
                    vm = min(vm, __ldcg(&args.ws_viol[i]));
                }
                bad |= vm != INT_MAX || !isfinite(cd);  // a non-finite chunk state is a violation
                dpart += cd;
            }
            // numerators: chunk sums in sub order, totals in chunk order.  Lane owns
            // D / 32 consecutive d (one 16-B load per slot at D = 128); LBW slots in flight
            constexpr int NDL = (D + 31) / 32;
            constexpr bool V4 = (D % 128 == 0) && NDL == 4;
            float acc[NDL], cn[NDL];
#pragma unroll
            for (int r = 0; r < NDL; ++r) acc[r] = cn[r] = 0.f;
            constexpr int LBW = V4 ? 16 : 8;
            for (int i0 = 0; i0 < P; i0 += LBW) {
                float val[LBW][NDL];
#pragma unroll
                for (int q = 0; q < LBW; ++q) {
                    if constexpr (V4) {
                        const float4 t4 = i0 + q < P ? __ldcg(reinterpret_cast<const float4 *>(
                                                           &args.ws_num[(base + i0 + q) * D + 4 * lane]))
                                                     : make_float4(0.f, 0.f, 0.f, 0.f);
                        val[q][0] = t4.x;
                        val[q][1] = t4.y;
                        val[q][2] = t4.z;
                        val[q][3] = t4.w;
                    } else {
#pragma unroll
                        for (int r = 0; r < NDL; ++r) {
                            const int d = lane + 32 * r;
                            val[q][r] = (i0 + q < P && d < D) ? __ldcg(&args.ws_num[(base + i0 + q) * D + d]) : 0.f;
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < LBW; ++q) {
                    if (i0 + q >= P) break;
#pragma unroll
                    for (int r = 0; r < NDL; ++r) cn[r] += val[q][r];
                    if ((i0 + q + 1) % nsub == 0) {  // chunk complete
#pragma unroll
                        for (int r = 0; r < NDL; ++r) {
                            bad |= !isfinite(cn[r]);
                            acc[r] += cn[r];
                            cn[r] = 0.f;
                        }
                    }
                }
            }
            const bool flagged = __any_sync(0xffffffffu, bad) != 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dpart += __shfl_xor_sync(0xffffffffu, dpart, o);
            if (lane == 0) {
                args.row_flags[row] = flagged ? 1 : 0;
                if (flagged) {
                    if (args.rows_recomputed) atomicAdd(args.rows_recomputed, 1);
                    s_grp_flag = 1;
                }
            }
            if (!flagged) {
                T *op = static_cast<T *>(args.o) + (int64_t)b * args.o_sb + (int64_t)(h0 + g) * args.o_sh;
#pragma unroll
                for (int r = 0; r < NDL; ++r) {
                    const int d = V4 ? 4 * lane + r : lane + 32 * r;
                    if (d < D) op[d] = Elem<T>::from_f(acc[r] / dpart);
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && s_grp_flag) flag_group(args, b, kvh);
        if (threadIdx.x == 0) ATRACE(5);
        return;
    }
    constexpr int LB = 32;  // partial loads kept in flight per thread
    for (int g = 0; g < gcount; ++g) {
        const int64_t row = row0 + g;
        const int64_t base = row * P;
        if (!ASYNC && args.only_flagged && !args.row_flags[row]) continue;
        T *op = static_cast<T *>(args.o) + (int64_t)b * args.o_sb + (int64_t)(h0 + g) * args.o_sh;
        const int nsub = args.nsub;
        if (ASYNC) {
            // pass 1: chunk exp-sums and first violation per chunk (one thread per chunk,
            // its nsub partials loaded LB at a time)
            for (int jj = threadIdx.x; jj < args.p; jj += ATT_THREADS) {
                float cd = 0.f;
                int vm = INT_MAX;
                for (int s0 = 0; s0 < nsub; s0 += LB) {
                    float dv[LB];
                    int vv[LB];
#pragma unroll
                    for (int q = 0; q < LB; ++q) {
                        const bool ok = s0 + q < nsub;
                        const int64_t i = base + (int64_t)jj * nsub + s0 + q;
                        dv[q] = ok ? ld_cg_f32(&args.ws_den[i]) : 0.f;
                        vv[q] = ok ? __ldcg(&args.ws_viol[i]) : INT_MAX;
                    }
#pragma unroll
                    for (int q = 0; q < LB; ++q) {
                        cd += dv[q];
                        vm = min(vm, vv[q]);
                    }
                }
                s_cden[jj] = cd;
                s_cviol[jj] = vm;
                s_unrep[jj] = !isfinite(cd);
            }
            if (threadIdx.x == 0) s_any_flag = 0;
            __syncthreads();
            // pass 2: chunk numerators over the flattened (chunk, sub) partials, LB loads
            // in flight; a non-finite chunk state is a violation (attention.py:230-237)
            float tot[(D + ATT_THREADS - 1) / ATT_THREADS];
            int nd = 0;
            for (int d = threadIdx.x; d < D; d += ATT_THREADS, ++nd) {
                float acc = 0.f, cn = 0.f;
                for (int i0 = 0; i0 < P; i0 += LB) {
                    float val[LB];
#pragma unroll
                    for (int q = 0; q < LB; ++q)
                        val[q] = i0 + q < P ? ld_cg_f32(&args.ws_num[(base + i0 + q) * D + d]) : 0.f;
#pragma unroll
                    for (int q = 0; q < LB; ++q) {
                        const int i = i0 + q;
                        if (i < P) {
                            cn += val[q];
                            if ((i + 1) % nsub == 0) {  // chunk jj complete, in sub order
                                const int jj = i / nsub;
                                if (!isfinite(cn)) s_unrep[jj] = 1;  // benign race: all store 1
                                if (args.chunk_num)  // zeroed for a violating chunk (attention.py:191-194)
                                    args.chunk_num[(row * args.p + jj) * D + d] =
                                        s_cviol[jj] == INT_MAX ? cn : 0.f;
                                acc += cn;
                                cn = 0.f;
                            }
                        }
                    }
                }
                tot[nd] = acc;
            }
            __syncthreads();
            // pass 3: chunk verdicts, row flag
            for (int jj = threadIdx.x; jj < args.p; jj += ATT_THREADS) {
                int v = s_cviol[jj];
                if (v == INT_MAX) v = s_unrep[jj] ? chunk_lo(Lb, args.p, jj) : -1;
                if (args.viol_index) args.viol_index[row * args.p + jj] = v;
                if (args.chunk_den) args.chunk_den[row * args.p + jj] = s_cviol[jj] == INT_MAX ? s_cden[jj] : 0.f;
                if (v >= 0) s_any_flag = 1;
            }
            __syncthreads();
            const bool flagged = s_any_flag != 0;
            if (threadIdx.x == 0) {
                args.row_flags[row] = flagged ? 1 : 0;
                if (flagged && args.rows_recomputed) atomicAdd(args.rows_recomputed, 1);
                if (flagged) s_grp_flag = 1;
            }
            if (!flagged) {
                float dsum = 0.f;
                for (int jj = 0; jj < args.p; ++jj) dsum += s_cden[jj];  // chunk order
                nd = 0;
                for (int d = threadIdx.x; d < D; d += ATT_THREADS, ++nd)
                    op[d] = Elem<T>::from_f(tot[nd] / dsum);
            }
            __syncthreads();
        } else {
            // Eq. (2) join over all (chunk, sub-range) partials in index order;
            // the per-partial maxima and scaled sums are staged in smem first
            float *s_m = s_cden;                       // [P] maxima (P <= 2*ATT_MAX_P)
            float *s_f = reinterpret_cast<float *>(s_cviol);
            for (int i = threadIdx.x; i < P; i += ATT_THREADS) s_m[i] = ld_cg_f32(&args.ws_m[base + i]);
            __syncthreads();
            float mrow = -INFINITY;
            for (int i = 0; i < P; ++i) mrow = fmaxf(mrow, s_m[i]);
            __syncthreads();
            for (int i = threadIdx.x; i < P; i += ATT_THREADS) s_f[i] = safe_scale(s_m[i], mrow);
            __syncthreads();
            float l = 0.f;
            for (int i0 = 0; i0 < P; i0 += LB) {
                float dv[LB];
#pragma unroll
                for (int q = 0; q < LB; ++q) dv[q] = i0 + q < P ? ld_cg_f32(&args.ws_den[base + i0 + q]) : 0.f;
#pragma unroll
                for (int q = 0; q < LB; ++q)
                    if (i0 + q < P) l += dv[q] * s_f[i0 + q];
            }
            for (int d = threadIdx.x; d < D; d += ATT_THREADS) {
                float acc = 0.f;
                for (int i0 = 0; i0 < P; i0 += LB) {
                    float val[LB];
#pragma unroll
                    for (int q = 0; q < LB; ++q)
                        val[q] = i0 + q < P ? ld_cg_f32(&args.ws_num[(base + i0 + q) * D + d]) : 0.f;
#pragma unroll
                    for (int q = 0; q < LB; ++q)
                        if (i0 + q < P) acc += val[q] * s_f[i0 + q];
                }
                op[d] = Elem<T>::from_f(acc / l);
            }
            __syncthreads();
        }
    }
    if (ASYNC && threadIdx.x == 0 && s_grp_flag) flag_group(args, b, kvh);
}

// One CTA per (chunk/sub-range, kv-head x row group, batch row); the recompute
// launch (list_mode) instead walks the (batch, kv-head) groups the async join
// flagged, with a small fixed grid: a clean step costs one near-empty wave
// instead of B x Hkv x n_rg x P early-exit CTAs.
template <typename T, int D, int GT, bool ASYNC, bool MMA = false, int NST = ATT_STAGES>
__global__ void __launch_bounds__(ATT_THREADS, MMA ? 3 : 1)  // MMA: 3 CTAs / SM (192 KB of ring in flight)
attn_split_kernel(const AttnArgs args, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV) {
    if constexpr (!ASYNC) {
        if (args.list_mode) {
            // let the next kernel (the O projection) get resident and start its weight
            // stream now, under the async launch's tail: its griddepcontrol.wait still
            // waits for this whole grid, so the recomputed rows are visible to it
            pdl_trigger();
            pdl_wait();  // the list comes from the async launch
            const int count = __ldcg(args.flag_count);
            if (count == 0) return;  // nothing flagged (the common case): no list to walk or clear
            const int P = args.p * args.nsub;
            const int64_t items = (int64_t)count * args.n_rg * P;
            for (int64_t i = blockIdx.x; i < items; i += gridDim.x) {
                const int x = (int)(i % P);
                const int64_t r = i / P;
                const int rg = (int)(r % args.n_rg);
                const int e = __ldcg(&args.flag_list[r / args.n_rg]);  // b * Hkv + kvh
                const int b = e / args.Hkv, kvh = e % args.Hkv;
                attn_cta<T, D, GT, ASYNC, MMA, NST>(args, tmK, tmV, x, kvh * args.n_rg + rg, b);
                __syncthreads();  // shared memory is reused by the next item
            }
            // the last CTA clears the list and its dedupe markers (graph replay)
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                if (atomicAdd(&args.flag_count[32], 1) == (int)gridDim.x - 1) {
                    __threadfence();
                    for (int k = 0; k < count; ++k) args.flag_mark[__ldcg(&args.flag_list[k])] = 0;
                    args.flag_count[0] = 0;
                    args.flag_count[32] = 0;
                }
            }
            return;
        }
    }
    attn_cta<T, D, GT, ASYNC, MMA, NST>(args, tmK, tmV, blockIdx.x, blockIdx.y, blockIdx.z);
}

template <typename T, int D, int GT, bool ASYNC, bool MMA = false, int NST = ATT_STAGES>
static fdpp_status launch_attn(const AttnArgs &a, int grid_x, cudaStream_t st,
                               const CUtensorMap *tmK = nullptr, const CUtensorMap *tmV = nullptr) {
    using Gm = AttnGeom<T, D>;
    const int smem = (MMA ? 1024 : 0) + NST * Gm::STAGE_BYTES + 2 * NST * 8 +
                     ((MMA && ASYNC) ? 1 : ATT_CONSUMERS) * GT * (D + 2) * (int)sizeof(float);
    auto kern = attn_split_kernel<T, D, GT, ASYNC, MMA, NST>;
    CUtensorMap none;
    memset(&none, 0, sizeof(none));
    static DeviceOnce attr;  // per instantiation and device
    cudaError_t e0 = attr.run([&] {
        cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (r == cudaSuccess)  // cluster join: up to 16 CTAs per cluster
            r = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return r;
    });
    if (e0 != cudaSuccess) return cuda_status(e0, "cudaFuncSetAttribute(attn)");
    // list_mode: grid_x CTAs walk the flagged-group list; cluster_join: the grid_x
    // (= P) CTAs of a row group are one cluster
    dim3 grid = a.list_mode ? dim3(grid_x) : dim3(grid_x, a.Hkv * a.n_rg, a.B);
    cudaError_t e = launch_kernel_cluster(kern, grid, dim3(ATT_THREADS), smem, st, a.cluster_join ? grid_x : 1,
                                          a, tmK ? *tmK : none, tmV ? *tmV : none);
    if (e != cudaSuccess) return cuda_status(e, "attn_split_kernel launch");
    return FDPP_OK;
}

template <typename T, int D, bool ASYNC>
static fdpp_status by_gt(const AttnArgs &a, int gt, int gx, cudaStream_t st) {
    switch (gt) {
        case 1: return launch_attn<T, D, 1, ASYNC>(a, gx, st);
        case 2: return launch_attn<T, D, 2, ASYNC>(a, gx, st);
        case 4: return launch_attn<T, D, 4, ASYNC>(a, gx, st);
        default: return launch_attn<T, D, 8, ASYNC>(a, gx, st);
    }
}

template <typename T, bool ASYNC>
fdpp_status by_d(const AttnArgs &a, int D, int gt, int gx, cudaStream_t st) {
    switch (D) {
        case 8: return by_gt<T, 8, ASYNC>(a, gt, gx, st);
        case 16: return by_gt<T, 16, ASYNC>(a, gt, gx, st);
        case 32: return by_gt<T, 32, ASYNC>(a, gt, gx, st);
        case 64: return by_gt<T, 64, ASYNC>(a, gt, gx, st);
        case 128: return by_gt<T, 128, ASYNC>(a, gt, gx, st);
        case 256:
            if constexpr (sizeof(T) == 2) return by_gt<T, 256, ASYNC>(a, gt, gx, st);
            else break;
        case 4:
            if constexpr (sizeof(T) == 4) return by_gt<T, 4, ASYNC>(a, gt, gx, st);
            else break;
        default: break;
    }
    set_error("unsupported head dim %d for this dtype (pad D to a power of two >= 16 bytes)", D);
    return FDPP_ERR_UNSUPPORTED;
}

// tensor-core GQA/MQA path, one dtype (16 query rows per row group, D = 128)
template <typename T, bool ASYNC>
fdpp_status launch_mma_t(const AttnArgs &a, int gx, const CUtensorMap *tmK, const CUtensorMap *tmV,
                         cudaStream_t st) {
    return launch_attn<T, 128, 16, ASYNC, true>(a, gx, st, tmK, tmV);
}

}  // namespace fdpp
