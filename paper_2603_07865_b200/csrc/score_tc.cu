// K1 — tensor-core pre-filter for IvfIndex::search (index.cpp:289-326, hot loop :306-315).
//
// One CTA owns 128 queries (UMMA M) and streams a contiguous range of 256-row cache tiles
// (UMMA N) through a TMA -> smem -> tcgen05.mma -> TMEM pipeline:
//   warp 0      TMA producer: the CTA's 128 bf16 queries once (resident, K-major SW128), then
//               one 256x64 bf16 cache chunk per pipeline stage
//   warp 1      TMEM allocator + single-thread MMA issuer (M=128, N=256, K=16 per instruction),
//               double-buffered fp32 accumulators (2 x 256 TMEM columns)
//   warps 2-5   epilogue (EPI_GROUPS groups of 4 warps; group g drains the tiles lt = g mod
//               EPI_GROUPS). TMEM lane == query, so each thread walks ITS query's 256 scores
//               with tcgen05.ld, takes the per-entry max over the entry's Rp pyramid rows, and
//               keeps a running top list in registers. Each (CTA, group) is one emission slice
//               of the query's candidate buffer.
//
// The 1M x 1024 score matrix is never written. Instead the epilogue emits a CERTIFIED candidate
// set: with eps_q >= |bf16 score - exact score| (bf16 rounding of both operands, 2u + u^2 with
// u = 2^-8, plus fp32 accumulation slack, times |q| * max|row|), an entry can be in the exact
// top-k only if its approximate score >= T_a - 2 eps_q, where T_a is the k-th best approximate
// entry score. Every CTA's running k-th best is a lower bound of T_a, and CTAs share it through
// an atomicMax per query, so the emission threshold tightens as the scan proceeds. The exact
// fp64 rescoring (exact.cu) then decides ties and order bit-exactly.
#include <numeric>

#ifndef SW_EPI_PAIRS
// 1: epilogue TMEM stages of two 32-column chunks (64 columns in flight, 225 registers).
// Measured slower than one chunk per stage (0.729 vs 0.713 ms at config 3): the drain is not
// bound by the TMEM round trips.
#define SW_EPI_PAIRS 0
#endif
#include <type_traits>

#include "ptx.cuh"
#include "sw_internal.cuh"

#ifndef SW_EPI_GROUPS_
// Epilogue warp groups draining the two accumulators. 2 (group g drains accumulator g) was
// measured SLOWER once the epilogue hot loop became compact: the extra warps compete for the
// issue slots of the SMSPs that host the TMA producer and the MMA issuer (0.765 vs 0.724 ms).
#define SW_EPI_GROUPS_ 1
#endif

namespace sw {

namespace {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int A_CHUNK = BM * 128;  // bytes: 128 rows x 64 bf16
constexpr int B_STAGE = BN * 128;  // bytes: 256 rows x 64 bf16
constexpr int B_HALF = B_STAGE / 2;  // CTA-pair mode: each CTA of the pair stages 128 rows
constexpr int EPI_GROUPS = SW_EPI_GROUPS_;
constexpr int THREADS = 64 + 128 * EPI_GROUPS;

// TS mode (CTA pairs, A operand in TMEM): 128-column tiles so that 2 x 128 accumulator columns
// + the 256 columns of the resident bf16 queries fill the 512 TMEM columns exactly.
constexpr int BN_TS = 128;
constexpr int B_QUARTER = (BN_TS / 2) * 128;  // bytes: each CTA stages 64 rows x 64 bf16
constexpr uint32_t IDESC_TS = ptx::idesc_bf16_f32(2 * BM, BN_TS);

struct TcParams {
    int B;
    int kch;        // Dp / 64
    int n_stages;
    int k;          // top-k
    int64_t n_tiles;
    int64_t tiles_per_cta;
    int64_t n_slots;  // high-water slot count
    const uint32_t* valid_bits;  // one bit per slot
    const float* q_eps;
    uint32_t* thr;
    uint32_t* top1;  // [B][kMaxSlices] each slice's running best approximate entry score
    int32_t* slice_cnt;  // [B][n_chunks] emissions per (query, CTA)
    float* cta_topk;     // [B][n_chunks][32] final running lists
    int32_t* cand_slot;  // [B][kCandCap], CTA y owns [y * cap_local, (y + 1) * cap_local)
    float* cand_score;
    int n_chunks;
    int cap_local;
    // balanced normal mode (bal_k > 0): 128-query groups (256 in pair mode) x bal_R tile ranges
    // = units x bal_k items; unit u (a CTA, or a pair) walks items u, u + units, ..., so
    // every SM works (the static (qblock, range) grid idles 148 mod #qblocks SMs)
    int bal_R;
    int bal_k;
    int n_items_bal;  // groups x bal_R; unit u walks items u, u + units, ...
    const __nv_bfloat16* q_bf;    // [BmaxPad][Dp] queries (TS mode loads them into TMEM)
    // grouped IVF mode (single CTAs): one work item per CTA — a block of 128 queries that all
    // probe list l, gathered into contiguous rows, against a chunk of list l's tiles in the
    // list-sorted arena copy. items[b] = {gathered row base, tile0, n_tiles (0: idle), l | j<<8}.
    const int4* items;
    const int32_t* qmap;          // gathered row -> query id (-1: padding)
    const uint8_t* prank;         // [B][kMaxCentroids] probe rank of each list
    int grp_ch;                   // slice of (query, list l, chunk j) = rank(l) * grp_ch + j
    const int32_t* n_items;       // grouped: device count of real items (persistent CTAs loop)
    int32_t* ticket;              // grouped, single CTAs: dynamic item tickets (zeroed per search)
    int ivf;                      // IVF mode: only rows of the query's probed lists count
    const int16_t* row_list;      // [rows] list of every stored row
    const uint64_t* pmask;        // [B][4] probed-list bitmask per query
    int stream_a;    // grouped IVF: queries streamed with every ring stage (no resident A)
    int experiment;  // 0 normal; profiling only (SW_SCORE_EXPERIMENT): 1 = epilogue skipped,
                     // 2 = also no cache TMA (pure MMA rate)
};

// Emission + running top-list update for the entries of one 32-column chunk whose approximate
// score reaches theta. `mask` has one bit per (valid) entry; the loop runs once per set bit
// (usually 0 or 1). Emissions go to this (query, CTA)'s private slice with a register counter:
// no atomics and no loads on the emission path.
template <int RP, int KL>
__device__ __forceinline__ void emit_chunk(const uint32_t (&r)[32], uint32_t mask,
                                           int64_t slot_c, float& theta, float (&list)[KL],
                                           float& kth, float eps2, int& cnt, int64_t slice,
                                           const TcParams& p) {
    constexpr int E = 32 / RP;
    while (mask) {
        const int e = __ffs(mask) - 1;
        mask &= mask - 1;
        // entry e's max over its RP pyramid rows, selected through a binary mux tree (a
        // dynamic register index would spill to local memory), clamped like core.cpp:35-36
        float t[E];
#pragma unroll
        for (int j = 0; j < E; ++j) {
            t[j] = __uint_as_float(r[j * RP]);
#pragma unroll
            for (int i = 1; i < RP; ++i) t[j] = fmaxf(t[j], __uint_as_float(r[j * RP + i]));
        }
#pragma unroll
        for (int w = E / 2, b = 1; w >= 1; w >>= 1, b <<= 1)
#pragma unroll
            for (int j = 0; j < w; ++j) t[j] = (e & b) ? t[2 * j + 1] : t[2 * j];
        const float m = fminf(1.0f, fmaxf(-1.0f, t[0]));
        if (m < theta) continue;  // theta may have risen within this chunk
        if (cnt < p.cap_local) {
            // grouped IVF: the list-sorted row; k_finish maps the kept ones to arena slots
            p.cand_slot[slice + cnt] = (int32_t)(slot_c + e);
            p.cand_score[slice + cnt] = m;
        }
        ++cnt;
        float x = m;  // sorted insertion (descending)
#pragma unroll
        for (int i = 0; i < KL; ++i) {
            const float hi = fmaxf(list[i], x);
            x = fminf(list[i], x);
            list[i] = hi;
        }
        kth = list[KL - 1];  // slots above the k real ones hold +inf (see init)
        theta = fmaxf(theta, kth - eps2);
    }
}

// Emission of one entry whose clamped best-row score m reaches theta (packed tiles), as
// emit_chunk does it.
template <int KL>
__device__ __forceinline__ void emit_one(float m, int64_t slot, float& theta, float (&list)[KL],
                                         float& kth, float eps2, int& cnt, int64_t slice,
                                         const TcParams& p) {
    if (cnt < p.cap_local) {
        p.cand_slot[slice + cnt] = (int32_t)slot;
        p.cand_score[slice + cnt] = m;
    }
    ++cnt;
    float x = m;  // sorted insertion (descending)
#pragma unroll
    for (int i = 0; i < KL; ++i) {
        const float hi = fmaxf(list[i], x);
        x = fminf(list[i], x);
        list[i] = hi;
    }
    kth = list[KL - 1];
    theta = fmaxf(theta, kth - eps2);
}

// PAIR: a 2-CTA cluster (the two CTAs of one TPC) runs the MMA as cta_group::2 with M = 256:
// each CTA keeps its own 128 queries resident and stages HALF of every 256-row cache tile
// (128 rows), so the per-SM L2 -> SM operand feed halves; the leader CTA issues the MMA for
// both and its commits multicast to both CTAs' barriers. The epilogue is unchanged: TMEM lane
// == query in each CTA. TEMPTY lives in the leader and counts both CTAs' epilogue warps.
//
// TS (requires PAIR): the queries live in TMEM instead of shared memory (tcgen05.mma with an
// [a-tmem] operand): the epilogue warps load their own query rows into TMEM columns
// [256, 512) with tcgen05.st before the first tile, so every MMA reads only B from shared
// memory — the smem crossbar (128 B/clk), which A + both B halves + the TMA writes saturated,
// gets 25% headroom. Tiles shrink to 128 columns to make room in TMEM.
template <int RP, int KL, bool PAIR, bool TS>
__global__ void __launch_bounds__(THREADS, 1)
    k_score_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmE,
               const TcParams p) {
    static_assert(!TS || PAIR, "TMEM-resident A is implemented for CTA pairs");
    // PACK (RP = R in {3, 7}, not a power of two): a tile is 32 entries x R rows with the arena's
    // pad row skipped by a 3-D TMA box, so N = 32 R (224 at R = 7) carries no padding
    constexpr bool PACK = (RP & (RP - 1)) != 0;
    static_assert(!PACK || (!TS && RP <= 7), "packed tiles: R <= 7, no TS mode");
    constexpr int TBN = TS ? BN_TS : (PACK ? 32 * RP : BN);
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    constexpr int KPS = TS ? 2 : 1;  // 64-wide K chunks per ring stage (TS: 2 x 8 KB boxes)
    constexpr int BSTG = TS ? KPS * B_QUARTER : (PAIR ? (TBN / 2) * 128 : TBN * 128);
    constexpr uint32_t ID_PAIR = ptx::idesc_bf16_f32(2 * BM, TBN);
    constexpr uint32_t ID_ONE = ptx::idesc_bf16_f32(BM, TBN);
    uint8_t* sA = smem;
    // stream_a: [S][A_CHUNK] query chunks, then [S][BSTG]; otherwise the resident A [kch][A_CHUNK]
    uint8_t* sB = smem + (TS ? 0 : (p.stream_a ? p.n_stages : p.kch) * A_CHUNK);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + p.n_stages * BSTG);
    const int S = p.n_stages;
    // full[S] | empty[S] | a_full | tfull[2] | tempty[2] | a_empty
    auto bar = [&](int i) { return ptx::smem_u32(&bars[i]); };
    const int FULL = 0, EMPTY = S, AFULL = 2 * S, TFULL = 2 * S + 1, TEMPTY = 2 * S + 3,
              AEMPTY = 2 * S + 5;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(&bars[2 * S + 6]);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int qblock = blockIdx.x;
    const bool bal = !p.items && p.bal_k > 0;
    const int unit = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    // Work items. Normal mode: ONE item per CTA — query block blockIdx.x x tile range
    // blockIdx.y. Grouped IVF mode: persistent CTAs walk items blockIdx.x, + gridDim.x, ...
    // (list, 128-query block, tile chunk); TMEM, barriers and the smem ring persist across
    // items, and the queries of item i+1 load as soon as the MMAs of item i are done with A.
    struct Item {
        int qrow, ntiles, list, chunk;
        int64_t t0;
    };
    auto item_at = [&](int i) {
        Item r;
        if (p.items) {
            const int4 it = p.items[i];
            r.qrow = it.x + (PAIR ? (int)(blockIdx.x & 1) * BM : 0);  // pair: block b, b + 1
            r.t0 = it.y;
            r.ntiles = it.z;
            r.list = it.w & 255;
            r.chunk = it.w >> 8;
        } else if (bal) {
            // range-major: the groups sharing a tile range run it at the same time, so each
            // range streams from HBM once and the other groups hit L2
            const int ng = p.n_items_bal / p.bal_R;
            const int rr = i / ng, g = i - rr * ng;
            r.qrow = (PAIR ? 2 * g + (int)(blockIdx.x & 1) : g) * BM;
            r.t0 = (int64_t)rr * p.tiles_per_cta;
            r.ntiles = (int)max((int64_t)0, min(p.n_tiles, r.t0 + p.tiles_per_cta) - r.t0);
            r.list = 0;
            r.chunk = rr;
        } else {
            r.qrow = qblock * BM;
            r.t0 = (int64_t)blockIdx.y * p.tiles_per_cta;
            r.ntiles = (int)max((int64_t)0, min(p.n_tiles, r.t0 + p.tiles_per_cta) - r.t0);
            r.list = r.chunk = 0;
        }
        return r;
    };
    const int istep = (p.items || bal) ? (PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x) : 1;
    // does item i load A? (balanced mode: only when its query block differs from the unit's
    // previous item's)
    auto loads_a = [&](int i, int first) {
        return !bal || i == first || item_at(i).qrow != item_at(i - istep).qrow;
    };
    const int n_items = p.items ? *p.n_items : bal ? p.n_items_bal : 1;
    // Grouped IVF on single CTAs takes items from a ticket counter instead of the static
    // blockIdx.x + k gridDim.x walk: list chunks differ in size by several times, and the static
    // walk left the first SMs idle at 44% of the kernel (ncu: active cycles 216K-489K). The
    // producer lane fetches ticket k + 1 once item k's loads are issued and publishes it in a
    // 4-slot shared ring (full / empty mbarriers); the MMA and epilogue warps read the same
    // sequence, so every role walks the same items.
    // (in the dynamic shared memory after the pipeline barriers: the kernel's dynamic size is
    // set to the opt-in maximum, so it may have no static shared memory)
    constexpr int kTk = 4;
    uint64_t* s_tbar = &bars[2 * S + 8];                           // full[kTk] | empty[kTk]
    int* s_tick = reinterpret_cast<int*>(&bars[2 * S + 8 + 2 * kTk]);  // [kTk]
    int& s_first = s_tick[kTk];
    const bool dyn = !PAIR && p.items && p.ticket;
    int item0 = (p.items || bal) ? unit : 0;
    if (dyn) {
        if (threadIdx.x == 0) s_first = atomicAdd(p.ticket, 1);
        __syncthreads();
        item0 = s_first;
        if (item0 >= n_items) return;  // uniform for the CTA
    } else if (item0 >= n_items || item_at(item0).ntiles == 0) {
        return;  // uniform for the CTA / pair
    }
    // ticket k + 1 (k >= 0); static walk: item0 + (k + 1) istep. -1: no more items.
    auto prod_next = [&](int k, int ii) {
        if (!dyn) return ii + istep < n_items ? ii + istep : -1;
        const int j = k, slot = j % kTk;
        if (j >= kTk) ptx::mbar_wait(ptx::smem_u32(&s_tbar[kTk + slot]), (uint32_t)(((j / kTk) - 1) & 1));
        const int t = atomicAdd(p.ticket, 1);
        const int v = t < n_items ? t : -1;
        s_tick[slot] = v;
        ptx::mbar_arrive(ptx::smem_u32(&s_tbar[slot]));
        return v;
    };
    auto cons_next = [&](int k, int ii) {  // all lanes of the calling warp
        if (!dyn) return ii + istep < n_items ? ii + istep : -1;
        const int j = k, slot = j % kTk;
        ptx::mbar_wait(ptx::smem_u32(&s_tbar[slot]), (uint32_t)((j / kTk) & 1));
        const int v = s_tick[slot];
        __syncwarp();
        if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(ptx::smem_u32(&s_tbar[kTk + slot]));
        return v;
    };
    const uint32_t rank = PAIR ? ptx::cluster_ctarank() : 0u;
    const bool leader = rank == 0;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            ptx::mbar_init(bar(FULL + i), 1);
            ptx::mbar_init(bar(EMPTY + i), 1);
        }
        ptx::mbar_init(bar(AFULL), TS ? 8 : 1);  // TS: every epilogue warp of both CTAs
        ptx::mbar_init(bar(AEMPTY), 1);
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(bar(TFULL + i), 1);
            ptx::mbar_init(bar(TEMPTY + i), PAIR ? 8 : 4);  // one group of 4 warps per acc
        }
        if (dyn)
            for (int i = 0; i < kTk; ++i) {
                ptx::mbar_init(ptx::smem_u32(&s_tbar[i]), 1);  // the producer lane
                ptx::mbar_init(ptx::smem_u32(&s_tbar[kTk + i]), 1 + 4 * EPI_GROUPS);  // MMA + epilogue warps
            }
        ptx::fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmQ);
        ptx::tma_prefetch_desc(&tmE);
    }
    if (warp == 1) {
        if (PAIR) {
            ptx::tmem_alloc_pair(ptx::smem_u32(tmem_slot), 512);
            ptx::tmem_relinquish_pair();
        } else {
            ptx::tmem_alloc(ptx::smem_u32(tmem_slot), 512);
            ptx::tmem_relinquish();
        }
    }
    ptx::tc_fence_before();
    if (PAIR)
        ptx::cluster_sync();  // the peer's barriers are initialised before any remote arrive
    else
        __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer
            int s = 0;  // ring stage and its phase, advanced incrementally (no division)
            uint32_t ph = 0;
            int na = 0;  // A loads issued
            int kk = 0;
            for (int ii = item0; ii >= 0; ii = prod_next(kk++, ii)) {
                const Item itm = item_at(ii);
                const int qrow = itm.qrow;
                const int64_t t0 = itm.t0;
                const int ntiles = itm.ntiles;
                const bool lda = !p.stream_a && loads_a(ii, item0);
                if (lda && na > 0) ptx::mbar_wait_sleep(bar(AEMPTY), (uint32_t)((na - 1) & 1));
                if (lda) ++na;
                if (!lda) {
                    // same queries as the previous item: A stays resident
                } else if (TS) {
                    // queries go to TMEM through the epilogue warps
                } else if (PAIR) {
                    // both CTAs load their own queries / their half of each tile; the bytes
                    // complete on the leader's barriers, whose expectation covers both halves
                    if (leader) ptx::mbar_arrive_expect_tx(bar(AFULL), (uint32_t)(2 * p.kch * A_CHUNK));
                    for (int kc = 0; kc < p.kch; ++kc)
                        ptx::tma_load_2d_pair(ptx::smem_u32(sA + kc * A_CHUNK), &tmQ, bar(AFULL),
                                              kc * 64, qrow);
                } else {
                    ptx::mbar_arrive_expect_tx(bar(AFULL), (uint32_t)(p.kch * A_CHUNK));
                    for (int kc = 0; kc < p.kch; ++kc)
                        ptx::tma_load_2d(ptx::smem_u32(sA + kc * A_CHUNK), &tmQ, bar(AFULL), kc * 64,
                                         qrow);
                }
                for (int lt = 0; lt < ntiles; ++lt) {
                    const int64_t tile = t0 + lt;
                    for (int kc = 0; kc < p.kch; kc += KPS, s = (s + 1 == S) ? 0 : s + 1,
                             ph ^= (s == 0) ? 1u : 0u) {
                        ptx::mbar_wait_sleep(bar(EMPTY + s), ph ^ 1u);
                        if (p.experiment == 2) {
                            if (leader) ptx::mbar_arrive(bar(FULL + s));
                            continue;
                        }
                        if (PAIR) {
                            if (leader) ptx::mbar_arrive_expect_tx(bar(FULL + s), (uint32_t)(2 * BSTG));
    #pragma unroll
                            for (int u = 0; u < KPS; ++u) {
                                if (PACK)  // 16 entries x R rows per CTA
                                    ptx::tma_load_3d_pair(ptx::smem_u32(sB + s * BSTG), &tmE,
                                                          bar(FULL + s), (kc + u) * 64, 0,
                                                          (int32_t)(tile * 32 + rank * 16));
                                else
                                    ptx::tma_load_2d_pair(
                                        ptx::smem_u32(sB + s * BSTG + u * (BSTG / KPS)), &tmE, bar(FULL + s),
                                        (kc + u) * 64, (int32_t)(tile * TBN + rank * (TBN / 2)));
                            }
                        } else if (!PACK && !TS && p.stream_a) {
                            // the stage carries the item's query chunk kc with the tile's chunk
                            ptx::mbar_arrive_expect_tx(bar(FULL + s), (uint32_t)(BSTG + A_CHUNK));
                            ptx::tma_load_2d(ptx::smem_u32(sA + s * A_CHUNK), &tmQ, bar(FULL + s),
                                             kc * 64, qrow);
                            ptx::tma_load_2d(ptx::smem_u32(sB + s * BSTG), &tmE, bar(FULL + s),
                                             kc * 64, (int32_t)(tile * BN));
                        } else {
                            ptx::mbar_arrive_expect_tx(bar(FULL + s), (uint32_t)BSTG);
                            if (PACK)
                                ptx::tma_load_3d(ptx::smem_u32(sB + s * BSTG), &tmE, bar(FULL + s),
                                                 kc * 64, 0, (int32_t)(tile * 32));
                            else
                                ptx::tma_load_2d(ptx::smem_u32(sB + s * BSTG), &tmE, bar(FULL + s),
                                                 kc * 64, (int32_t)(tile * BN));
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (leader) {
            // ---------------- MMA issuer: the converged warp waits, one elected lane issues
            // for the whole CTA / pair. Descriptors advance by constants (K16 step = 32 B =
            // 2 in the >>4 address field), keeping the per-chunk issue path short.
            const uint64_t adesc0 = ptx::umma_desc_sw128(ptx::smem_u32(sA));
            const uint64_t bdesc0 = ptx::umma_desc_sw128(ptx::smem_u32(sB));
            int s = 0;
            uint32_t ph = 0;
            int gt = 0;  // tiles across items: accumulator index and phase
            int na = 0;  // A loads consumed
            int kk = 0;
            for (int ii = item0; ii >= 0;) {
                const int ntiles = item_at(ii).ntiles;
                if (!p.stream_a && loads_a(ii, item0)) {
                    if (TS)
                        ptx::mbar_wait_cluster(bar(AFULL), (uint32_t)(na & 1));
                    else
                        ptx::mbar_wait(bar(AFULL), (uint32_t)(na & 1));
                    ++na;
                }
                ptx::tc_fence_after();
                for (int lt = 0; lt < ntiles; ++lt, ++gt) {
                    const int acc = gt & 1;
                    const uint32_t aph = (gt >> 1) & 1u;
                    ptx::mbar_wait_sleep(bar(TEMPTY + acc), aph ^ 1u);
                    ptx::tc_fence_after();
                    const uint32_t d_tmem = tmem_base + acc * TBN;
                    for (int kc = 0; kc < p.kch; kc += KPS, s = (s + 1 == S) ? 0 : s + 1,
                             ph ^= (s == 0) ? 1u : 0u) {
                        ptx::mbar_wait_sleep(bar(FULL + s), ph);
                        ptx::tc_fence_after();
                        const uint64_t ad = adesc0 + (uint64_t)((p.stream_a ? s : kc) * (A_CHUNK >> 4));
                        const uint64_t bd = bdesc0 + (uint64_t)(s * (BSTG >> 4));
                        if (ptx::elect_one()) {
    #pragma unroll
                            for (int u = 0; u < KPS; ++u)
    #pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const uint32_t acc_in = ((kc + u) | k) != 0 ? 1u : 0u;
                                const uint64_t bk = bd + (uint64_t)(u * ((BSTG / KPS) >> 4)) + 2 * k;
                                if (TS)
                                    ptx::mma_bf16_pair_ts(
                                        d_tmem, tmem_base + 2 * TBN + (kc + u) * 32 + k * 8, bk,
                                        IDESC_TS, acc_in);
                                else if (PAIR)
                                    ptx::mma_bf16_pair(d_tmem, ad + 2 * k, bk, ID_PAIR, acc_in);
                                else
                                    ptx::mma_bf16(d_tmem, ad + 2 * k, bk, ID_ONE, acc_in);
                            }
                            // frees the smem stage (both CTAs' halves) when the MMAs finish
                            if (PAIR)
                                ptx::mma_commit_pair(bar(EMPTY + s));
                            else
                                ptx::mma_commit(bar(EMPTY + s));
                        }
                        __syncwarp();
                    }
                    // accumulator ready for the epilogue (of both CTAs)
                    if (ptx::elect_one()) {
                        if (PAIR)
                            ptx::mma_commit_pair(bar(TFULL + acc));
                        else
                            ptx::mma_commit(bar(TFULL + acc));
                    }
                    __syncwarp();
                }
                // the item's MMAs are issued: A may be overwritten once they complete (signalled
                // only when the next item reloads A — dynamic tickets: after every item, the next
                // being unknown here; both CTAs of a pair are told)
                if (!p.stream_a && (dyn || (ii + istep < n_items && loads_a(ii + istep, item0))) &&
                    ptx::elect_one()) {
                    if (PAIR)
                        ptx::mma_commit_pair(bar(AEMPTY));
                    else
                        ptx::mma_commit(bar(AEMPTY));
                }
                __syncwarp();
                ii = cons_next(kk++, ii);
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue: TMEM lane == query
        constexpr int E = PACK ? 1 : 32 / RP;  // entries per 32-column chunk (unpacked tiles)
        constexpr int SPT = TBN / RP;          // slots per tile (32 when packed)
        const int quarter = warp & 3;  // TMEM lanes [32*quarter, 32*quarter + 32)
        const int grp = (warp - 2) >> 2;  // drains accumulator grp: tiles grp, grp + 2, ...
        int gt = 0;  // tiles across items (accumulator index / phase, as the MMA counts them)
        int kk = 0;
        for (int ii = item0; ii >= 0; ii = cons_next(kk++, ii)) {
        const Item itm = item_at(ii);
        const int qrow = itm.qrow;
        const int64_t t0 = itm.t0;
        const int ntiles = itm.ntiles;
        const int g_list = itm.list, g_chunk = itm.chunk;
        const int q = p.qmap ? p.qmap[qrow + quarter * 32 + lane] : qrow + quarter * 32 + lane;
        const bool qvalid = q >= 0 && q < p.B;
        int vchunk = (bal ? itm.chunk : (int)blockIdx.y) * EPI_GROUPS + grp;
        if (p.items)  // grouped IVF: slice = (probe rank of this list for q, chunk of the list)
            vchunk = qvalid ? (int)p.prank[(int64_t)q * kMaxCentroids + g_list] * p.grp_ch + g_chunk
                            : 0;
        float eps2 = 0.0f;
        if (qvalid) eps2 = 2.0f * p.q_eps[q];
        uint64_t pm0 = 0, pm1 = 0, pm2 = 0, pm3 = 0;  // probed lists (IVF mode)
        if (p.ivf && qvalid) {
            pm0 = p.pmask[(int64_t)q * 4 + 0];
            pm1 = p.pmask[(int64_t)q * 4 + 1];
            pm2 = p.pmask[(int64_t)q * 4 + 2];
            pm3 = p.pmask[(int64_t)q * 4 + 3];
        }
        float theta = -INFINITY, kth = -INFINITY, published = -INFINITY;
        // descending list; the top KL - k slots are +inf so list[KL-1] is always the k-th best
        float list[KL];
#pragma unroll
        for (int i = 0; i < KL; ++i) list[i] = (i < KL - p.k) ? INFINITY : -INFINITY;
        const uint32_t lane_base = tmem_base + ((uint32_t)(quarter * 32) << 16);
        const int64_t slice = (int64_t)q * kCandCap + (int64_t)vchunk * p.cap_local;
        int cnt = 0;
        uint32_t g_next = qvalid ? __ldcg(&p.thr[q]) : 0u;  // shared k-th best, one tile ahead
        float pub_top1 = -INFINITY;
        int done = 0;  // tiles drained by this group
        if (TS) {
            // this warp's 32 query rows -> TMEM lanes [32 quarter, +32), columns [2 TBN, 2 TBN +
            // Dp / 2): lane = query, column = bf16 pair (k, k+1) of the row, K-major
            const uint4* qsrc = reinterpret_cast<const uint4*>(
                p.q_bf + (int64_t)(qrow + quarter * 32 + lane) * (p.kch * 64));
            for (int cb = 0; cb < p.kch * 32; cb += 32) {
                uint32_t v[32];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint4 w = __ldg(qsrc + cb / 4 + u);
                    v[4 * u] = w.x;
                    v[4 * u + 1] = w.y;
                    v[4 * u + 2] = w.z;
                    v[4 * u + 3] = w.w;
                }
                ptx::tmem_st32(lane_base + 2 * TBN + cb, v);
            }
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa(bar(AFULL), 0));
        }

        for (int lt = grp; lt < ntiles; lt += EPI_GROUPS) {
            const int acc = (gt + lt) & 1;
            const uint32_t aph = ((gt + lt) >> 1) & 1u;
            const int64_t tile = t0 + lt;
            if (qvalid) {
                theta = fmaxf(theta, ord2f(g_next) - eps2);
                g_next = __ldcg(&p.thr[q]);
            }
            const int64_t slot0 = tile * SPT;
            ptx::mbar_wait_sleep(bar(TFULL + acc), aph);  // no spinning on the MMA's SMSPs
            ptx::tc_fence_after();
            constexpr int NSUB = (TS && E >= 2) ? 2 : 1;  // TS tiles have only 4 chunks
            if (!PACK && done == 0 && p.k <= NSUB * TBN / 32 && p.experiment == 0 && !p.ivf) {
                // First tile of this slice: the threshold is still -inf, so a one-pass scan
                // would emit the whole record sequence of the tile (~k + k ln(256/k)). A
                // pre-pass takes each fully valid (sub-)chunk's best entry; the k-th largest of
                // those k+ distinct entries' scores (their minimum over >= k (sub-)chunks) lower-
                // bounds T_a, and the emitting pass starts from it.
                float lo_best = INFINITY;
                int n_full = 0;
#pragma unroll 1
                for (int c = 0; c < TBN / 32; ++c) {
                    uint32_t r[32];
                    __syncwarp();
                    ptx::tmem_ld32(lane_base + acc * TBN + c * 32, r);
                    const int64_t sc = slot0 + c * E;
                    uint32_t vb = __ldg(p.valid_bits + (sc >> 5)) >> (int)(sc & 31);
                    if (E < 32) vb &= (1u << (E & 31)) - 1u;
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int h = 0; h < NSUB; ++h) {
                        constexpr int EH = E / NSUB;
                        float cmax;
                        if (NSUB == 1) {
                            cmax = ptx::max32(r);
                        } else {
                            cmax = __uint_as_float(r[16 * h]);
#pragma unroll
                            for (int j = 1; j < 16; ++j)
                                cmax = fmaxf(cmax, __uint_as_float(r[16 * h + j]));
                        }
                        const uint32_t hb = (vb >> (EH * h)) & (EH < 32 ? (1u << (EH & 31)) - 1u
                                                                         : 0xFFFFFFFFu);
                        if (hb == (EH < 32 ? (1u << (EH & 31)) - 1u : 0xFFFFFFFFu)) {
                            lo_best = fminf(lo_best, fminf(1.0f, fmaxf(-1.0f, cmax)));
                            ++n_full;
                        }
                    }
                }
                if (qvalid && n_full == NSUB * TBN / 32) {
                    theta = fmaxf(theta, lo_best - eps2);
                    if (lo_best > published) {
                        atomicMax(&p.thr[q], f2ord(lo_best));
                        published = lo_best;
                    }
                }
            }
            // Hot loop kept compact (rolled: the rare emission path is instantiated twice, so
            // the epilogue stays resident in the instruction cache). Per 32-column chunk: a
            // 16-op FMNMX3 max tree over the raw scores and one compare; max and clamp commute,
            // so the per-entry clamped maxima are only formed on the rare path. The TMEM loads
            // are software-pipelined over two register buffers: chunk c + 1 is in flight while
            // chunk c is examined, halving the epilogue's drain latency per tile (the MMA can
            // reuse an accumulator only once the epilogue released it).
            auto examine = [&](uint32_t(&r)[32], int c) {
                if (qvalid && fminf(1.0f, fmaxf(-1.0f, ptx::max32(r))) >= theta) {
                    if (p.ivf) {
                        // IVF: a row counts only if its list is among the query's probed lists
                        // (index.cpp:306-307); the hot max above may include other rows, which
                        // only makes this rare path run more often, never changes a result
                        const uint4* rl4 = reinterpret_cast<const uint4*>(
                            p.row_list + tile * TBN + c * 32);
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            const uint4 w = __ldg(rl4 + v);
                            const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                            for (int h = 0; h < 8; ++h) {
                                const int l = (int)(int16_t)(ww[h >> 1] >> (16 * (h & 1)));
                                const uint64_t pm = (l >> 6) == 0 ? pm0 : (l >> 6) == 1 ? pm1
                                                  : (l >> 6) == 2 ? pm2 : pm3;
                                if (l < 0 || !((pm >> (l & 63)) & 1ull))
                                    r[8 * v + h] = __float_as_uint(-INFINITY);
                            }
                        }
                    }
                    // clamp(x) >= theta  <=>  x >= theta'  (theta' = -inf when theta <= -1;
                    // theta > 1 cannot reach here), so the mask needs no per-entry clamp
                    const float th = theta > -1.0f ? theta : -INFINITY;
                    uint32_t mask = 0;
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        float m = __uint_as_float(r[e * RP]);
#pragma unroll
                        for (int j = 1; j < RP; ++j) m = fmaxf(m, __uint_as_float(r[e * RP + j]));
                        mask |= (m >= th && m != -INFINITY ? 1u : 0u) << e;
                    }
                    const int64_t sc = slot0 + c * E;  // E-slot group never straddles a word
                    uint32_t vbits = __ldg(p.valid_bits + (sc >> 5)) >> (int)(sc & 31);
                    if (E < 32) vbits &= (1u << (E & 31)) - 1u;
                    mask &= vbits;
                    if (mask)
                        emit_chunk<RP, KL>(r, mask, sc, theta, list, kth, eps2, cnt, slice, p);
                }
                // tcgen05.ld is .sync.aligned: reconverge lanes that diverged on the emission
                // path before the next one (a partially valid warp, B % 32 != 0, hangs otherwise)
                __syncwarp();
            };
            if (PACK && p.experiment != 1 && p.experiment != 2) {
                // packed tile: entry e's R rows are columns [R e, R e + R); one x8 load per entry,
                // groups of 4 entries double-buffered (group g + 1 in flight while g is examined),
                // the max over R columns, one compare
                const uint32_t tb = lane_base + acc * TBN;
                const uint32_t vb = __ldg(p.valid_bits + tile);  // 32 entries = one word
                auto exam4 = [&](uint32_t(&r)[4][8], int g) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        float m = __uint_as_float(r[u][0]);
#pragma unroll
                        for (int j = 1; j < RP; ++j) m = fmaxf(m, __uint_as_float(r[u][j]));
                        m = fminf(1.0f, fmaxf(-1.0f, m));
                        if (qvalid && ((vb >> (g + u)) & 1u) && m >= theta)
                            emit_one<KL>(m, slot0 + g + u, theta, list, kth, eps2, cnt, slice, p);
                    }
                    __syncwarp();  // reconverge before the next .sync.aligned tcgen05.ld
                };
                uint32_t ra[4][8], rb[4][8];
                __syncwarp();
#pragma unroll
                for (int u = 0; u < 4; ++u) ptx::tmem_ld8(tb + RP * u, ra[u]);
                ptx::tmem_ld_wait();
#pragma unroll 1
                for (int g = 0; g < 32; g += 8) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) ptx::tmem_ld8(tb + RP * (g + 4 + u), rb[u]);
                    exam4(ra, g);
                    ptx::tmem_ld_wait();
                    if (g + 8 < 32) {
#pragma unroll
                        for (int u = 0; u < 4; ++u) ptx::tmem_ld8(tb + RP * (g + 8 + u), ra[u]);
                    }
                    exam4(rb, g + 4);
                    ptx::tmem_ld_wait();
                }
            }
            if (!PACK && p.experiment != 1 && p.experiment != 2) {
                constexpr int NCH = TBN / 32;
                const uint32_t tb = lane_base + acc * TBN;
#if SW_EPI_PAIRS
                // two 32-column chunks per stage, two stages: 64 columns in flight while 64
                // are examined, so a tile costs NCH / 2 TMEM round trips instead of NCH
                static_assert(PACK || NCH % 4 == 0, "pairs of stages");
                uint32_t ra[32], ra2[32], rb[32], rb2[32];
                __syncwarp();
                ptx::tmem_ld32(tb, ra);
                ptx::tmem_ld32(tb + 32, ra2);
                ptx::tmem_ld_wait();
#pragma unroll 1
                for (int c = 0; c < NCH; c += 4) {
                    ptx::tmem_ld32(tb + (c + 2) * 32, rb);
                    ptx::tmem_ld32(tb + (c + 3) * 32, rb2);
                    examine(ra, c);
                    examine(ra2, c + 1);
                    ptx::tmem_ld_wait();
                    if (c + 4 < NCH) {
                        ptx::tmem_ld32(tb + (c + 4) * 32, ra);
                        ptx::tmem_ld32(tb + (c + 5) * 32, ra2);
                    }
                    examine(rb, c + 2);
                    examine(rb2, c + 3);
                    ptx::tmem_ld_wait();
                }
#else
                static_assert(PACK || NCH % 2 == 0, "even");
                uint32_t ra[32], rb[32];
                __syncwarp();
                ptx::tmem_ld32(tb, ra);
                ptx::tmem_ld_wait();
#pragma unroll 1
                for (int c = 0; c < NCH; c += 2) {
                    ptx::tmem_ld32(tb + (c + 1) * 32, rb);  // in flight while chunk c is examined
                    examine(ra, c);
                    ptx::tmem_ld_wait();
                    if (c + 2 < NCH) ptx::tmem_ld32(tb + (c + 2) * 32, ra);
                    examine(rb, c + 1);
                    ptx::tmem_ld_wait();
                }
#endif
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                // relaxed: the release form's MEMBAR.ALL.GPU drained this warp's outstanding
                // global accesses every tile (21% of the kernel's stall samples)
                if (PAIR)
                    ptx::mbar_arrive_cluster_relaxed(ptx::mapa(bar(TEMPTY + acc), 0));
                else
                    ptx::mbar_arrive(bar(TEMPTY + acc));
            }
            ++done;  // warp-uniform (all lanes): it gates the .sync.aligned pre-pass
            if (qvalid) {
                // Union bound on T_a: the slices partition the entries, so the k-th largest of
                // their running bests is the k-th best of k distinct entries, <= T_a. It tracks
                // the whole scanned prefix of the cache (a slice's own k-th best tracks only
                // its 1/n_chunks share), so the emission threshold converges tiles earlier.
                float best = -INFINITY;  // the best real slot (slots above the k-th hold +inf;
#pragma unroll                                 // no dynamic index: list stays in registers)
                for (int i = 0; i < KL; ++i) best = list[i] < INFINITY ? fmaxf(best, list[i]) : best;
                if (best > pub_top1) {
                    __stcg(&p.top1[(int64_t)q * kMaxSlices + vchunk], f2ord(best));
                    pub_top1 = best;
                }
                float bound = kth;
                // refresh at tiles 1, 2, 4, 8, ... (grouped IVF items of <= 16 tiles: 2 and 8)
                const bool refresh = p.items ? (done == 2 || done == 8) : (done & (done - 1)) == 0;
                if (refresh && p.n_chunks >= p.k) {
                    float sel[KL];
#pragma unroll
                    for (int i = 0; i < KL; ++i) sel[i] = (i < KL - p.k) ? INFINITY : -INFINITY;
                    const uint32_t* t1 = p.top1 + (int64_t)q * kMaxSlices;
                    for (int j = 0; j < p.n_chunks; ++j) {
                        float x = ord2f(__ldcg(t1 + j));
#pragma unroll
                        for (int i = 0; i < KL; ++i) {
                            const float hi = fmaxf(sel[i], x);
                            x = fminf(sel[i], x);
                            sel[i] = hi;
                        }
                    }
                    bound = fmaxf(bound, sel[KL - 1]);
                    theta = fmaxf(theta, bound - eps2);
                }
                if (bound > published) {
                    atomicMax(&p.thr[q], f2ord(bound));
                    published = bound;
                }
            }
        }
        if (qvalid) {
            p.slice_cnt[(int64_t)q * p.n_chunks + vchunk] = cnt;
            // this slice's exact local top-k (every entry below it was below the running k-th)
            float* tk = p.cta_topk + ((int64_t)q * p.n_chunks + vchunk) * kMaxTopK;
#pragma unroll
            for (int i = 0; i < KL; ++i)
                if (i >= KL - p.k) tk[i - (KL - p.k)] = list[i];
        }
            gt += ntiles;
        }
    }
    ptx::tc_fence_before();
    if (PAIR)
        ptx::cluster_sync();  // neither CTA frees TMEM (or exits) while the pair still uses it
    else
        __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        if (PAIR)
            ptx::tmem_dealloc_pair(tmem_base, 512);
        else
            ptx::tmem_dealloc(tmem_base, 512);
    }
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encoder() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        fn = reinterpret_cast<PFN_encodeTiled>(p);
    }
    return fn;
}

bool encode_2d(CUtensorMap* m, void* base, uint64_t inner, uint64_t rows, uint32_t box_rows) {
    PFN_encodeTiled enc = get_encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {inner, rows};
    cuuint64_t strides[1] = {inner * sizeof(__nv_bfloat16)};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// the arena viewed as [S][Rp][Dp] bf16, boxes (64, R, entries): packed pyramid tiles
bool encode_3d(CUtensorMap* m, void* base, uint64_t inner, uint64_t rp, uint64_t slots,
               uint32_t r, uint32_t box_entries) {
    PFN_encodeTiled enc = get_encoder();
    if (!enc) return false;
    cuuint64_t dims[3] = {inner, rp, slots};
    cuuint64_t strides[2] = {inner * sizeof(__nv_bfloat16), rp * inner * sizeof(__nv_bfloat16)};
    cuuint32_t box[3] = {64, r, box_entries};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult res = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return res == CUDA_SUCCESS;
}

template <int RP, int KL, bool PAIR, bool TS>
void launch_tc_kl(Ctx& c, const TcParams& p, dim3 grid, size_t smem, cudaStream_t st) {
    auto kern = k_score_tc<RP, KL, PAIR, TS>;
    ensure_smem_attr(c, kern, (size_t)c.smem_optin);
    if (PAIR) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(THREADS);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        constexpr bool PACK = (RP & (RP - 1)) != 0;
        SW_CUDA(cudaLaunchKernelEx(&cfg, kern, c.tm_q,
                                   TS ? c.tm_rows_q64 : (PACK ? c.tm_pack_half : c.tm_rows_half), p));
    } else {
        constexpr bool PACK = (RP & (RP - 1)) != 0;
        kern<<<grid, THREADS, smem, st>>>(c.tm_q, PACK ? c.tm_pack : c.tm_rows, p);
    }
}

template <int RP, bool PAIR, bool TS>
void launch_tc_rp(Ctx& c, const TcParams& p, dim3 grid, size_t smem, cudaStream_t st) {
    if (p.k <= 8)
        launch_tc_kl<RP, 8, PAIR, TS>(c, p, grid, smem, st);
    else
        launch_tc_kl<RP, 32, PAIR, TS>(c, p, grid, smem, st);
}

template <bool PAIR, bool TS>
void launch_tc(Ctx& c, const TcParams& p, dim3 grid, size_t smem, cudaStream_t st, bool pack) {
    if (pack && !TS) {  // packed pyramid tiles (no pad rows in the MMA)
        if (c.R == 7) launch_tc_rp<7, PAIR, false>(c, p, grid, smem, st);
        else launch_tc_rp<3, PAIR, false>(c, p, grid, smem, st);
        return;
    }
    switch (c.Rp) {
        case 1: launch_tc_rp<1, PAIR, TS>(c, p, grid, smem, st); break;
        case 2: launch_tc_rp<2, PAIR, TS>(c, p, grid, smem, st); break;
        case 4: launch_tc_rp<4, PAIR, TS>(c, p, grid, smem, st); break;
        case 8: launch_tc_rp<8, PAIR, TS>(c, p, grid, smem, st); break;
        case 16: launch_tc_rp<16, PAIR, TS>(c, p, grid, smem, st); break;
        case 32: launch_tc_rp<32, PAIR, TS>(c, p, grid, smem, st); break;
        default: throw Error(SW_EINVAL, "rows per entry pad must be a power of two <= 32");
    }
}

}  // namespace

bool encode_2d_map(CUtensorMap* m, void* base, uint64_t inner, uint64_t rows, uint32_t box_rows) {
    return encode_2d(m, base, inner, rows, box_rows);
}

// Grouped IVF search (ivf_group_prepare built c.d_items / d_qg / the sorted arena): one single
// CTA per work item, max_items CTAs (idle items exit at once).
int launch_score_tc_grouped(Ctx& c, int B, int k, int64_t max_items, cudaStream_t st) {
    TcParams p{};
    p.B = B;
    p.kch = c.Dp / 64;
    const int budget = c.smem_optin - 1024 - 512;
    p.k = k;
    const bool pair = c.grp_pair;
    const int bstg = pair ? B_HALF : B_STAGE;
    // SW_IVF_STREAM_A=0: queries resident per item (128 KB of shared memory: a 3-deep B ring)
    static const bool stream_a_env = [] {
        const char* e = getenv("SW_IVF_STREAM_A");
        return !(e && e[0] == '0');
    }();
    p.stream_a = (!pair && stream_a_env) ? 1 : 0;
    p.n_stages = p.stream_a ? std::min(8, budget / (bstg + A_CHUNK))
                            : std::min(8, (budget - p.kch * A_CHUNK) / bstg);
    static const int env_st = [] { const char* e = getenv("SW_IVF_STAGES"); return e ? atoi(e) : 0; }();
    if (env_st >= 2) p.n_stages = std::min(p.n_stages, env_st);
    SW_REQUIRE(p.n_stages >= 2, "tcgen05 scoring: not enough shared memory for 2 stages");
    p.n_tiles = c.grp_rows / BN;
    p.tiles_per_cta = 1;
    p.n_slots = c.grp_rows;
    p.valid_bits = c.d_sorted_vbits;
    p.q_eps = c.q_eps;
    p.thr = c.thr;
    p.top1 = c.top1;
    p.q_bf = c.d_qg;
    p.ivf = 0;  // every row of a work item belongs to the list its queries probe
    p.row_list = c.row_list;
    p.pmask = c.pmask;
    p.slice_cnt = c.slice_cnt;
    p.cta_topk = c.cta_topk;
    p.cand_slot = c.cand_slot;
    p.cand_score = c.cand_score;
    p.items = c.d_items;
    p.qmap = c.d_qmap;
    p.prank = c.prank;
    p.grp_ch = c.grp_ch;
    p.n_items = c.d_qbase + kMaxCentroids + 1;  // device count written by k_group_plan
    static const bool dyn_ok = [] {
        const char* e = getenv("SW_IVF_DYN");
        return !(e && e[0] == '0');
    }();
    p.ticket = (!pair && dyn_ok) ? c.d_qbase + kMaxCentroids + 2 : nullptr;  // zeroed by k_group_plan
    p.n_chunks = std::min(eff_nprobe(c), c.ivf_C) * c.grp_ch;
    SW_REQUIRE(p.n_chunks <= kMaxSlices, "grouped IVF: too many slices per query");
    p.cap_local = (kCandCap / p.n_chunks) & ~3;
    c.last_chunks = p.n_chunks;
    c.last_score_pair = pair;
    c.last_score_ts = false;
    p.experiment = [] { const char* e = getenv("SW_SCORE_EXPERIMENT"); return e ? atoi(e) : 0; }();  // profiling only
    const size_t smem = 1024 + (size_t)(p.stream_a ? p.n_stages : p.kch) * A_CHUNK +
                        (size_t)p.n_stages * bstg + 512;
    auto kern = [&](auto rp_tag, auto kl_tag) {
        constexpr int RPv = decltype(rp_tag)::value, KLv = decltype(kl_tag)::value;
        if (pair) {
            // persistent CTA pairs (the two SMs of a TPC): each walks the items of two query
            // blocks, staging half of every tile, so a tile streams once per 256 queries
            auto kf = k_score_tc<RPv, KLv, true, false>;
            ensure_smem_attr(c, kf, (size_t)c.smem_optin);
            const int64_t units = std::min<int64_t>(max_items, c.num_sms / 2);
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3((unsigned)(2 * units), 1);
            cfg.blockDim = dim3(THREADS);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 2;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            SW_CUDA(cudaLaunchKernelEx(&cfg, kf, c.tm_qg, c.tm_sorted_half, p));
            return;
        }
        auto kf = k_score_tc<RPv, KLv, false, false>;
        ensure_smem_attr(c, kf, (size_t)c.smem_optin);
        // persistent: one CTA per SM walks the items (max_items only bounds the grid)
        kf<<<dim3((unsigned)std::min<int64_t>(max_items, c.num_sms), 1), THREADS, smem, st>>>(
            c.tm_qg, c.tm_sorted, p);
    };
    SW_REQUIRE(c.Rp == 1, "grouped IVF search needs one row per entry");
    if (k <= 8)
        kern(std::integral_constant<int, 1>{}, std::integral_constant<int, 8>{});
    else
        kern(std::integral_constant<int, 1>{}, std::integral_constant<int, 32>{});
    SW_CUDA(cudaGetLastError());
    return 1;
}

bool encode_tensor_maps(Ctx& c) {
    if (c.Dp > 512) return false;
    bool ok = encode_2d(&c.tm_rows, c.rows_bf, (uint64_t)c.Dp, (uint64_t)(c.S * c.Rp), BN);
    ok = ok && encode_2d(&c.tm_rows_half, c.rows_bf, (uint64_t)c.Dp, (uint64_t)(c.S * c.Rp), BN / 2);
    ok = ok && encode_2d(&c.tm_rows_q64, c.rows_bf, (uint64_t)c.Dp, (uint64_t)(c.S * c.Rp), BN_TS / 2);
    ok = ok && encode_2d(&c.tm_q, c.q_bf, (uint64_t)c.Dp, (uint64_t)c.BmaxPad, BM);
    // packed pyramid tiles when R is 3 or 7 (the padded power of two wastes 1/4 or 1/8)
    c.pack_ok = false;
    if (ok && (c.R == 7 || c.R == 3) && c.Rp == c.R + 1) {
        c.pack_ok = encode_3d(&c.tm_pack, c.rows_bf, (uint64_t)c.Dp, (uint64_t)c.Rp, (uint64_t)c.S,
                              (uint32_t)c.R, 32) &&
                    encode_3d(&c.tm_pack_half, c.rows_bf, (uint64_t)c.Dp, (uint64_t)c.Rp,
                              (uint64_t)c.S, (uint32_t)c.R, 16);
    }
    return ok;
}

// Returns the number of kernels launched (1).
int launch_score_tc(Ctx& c, int B, int k, bool ivf, cudaStream_t st) {
    // grid: x = 128-query block, y = contiguous range of tiles (<= 148 CTAs per block row)
    TcParams p{};
    p.B = B;
    p.kch = c.Dp / 64;
    const int budget = c.smem_optin - 1024 - 512;
    p.k = k;
    const int qb = (B + BM - 1) / BM;
    // CTA pairs need an even number of 128-query blocks; SW_SCORE_PAIR=0 forces single CTAs.
    // SW_SCORE_TS=1 keeps a pair's queries in TMEM (TS MMA). Measured slower and therefore off:
    // the tensor core's A reads and the epilogue's accumulator reads then share the TMEM read
    // port (MMA + feed 0.657 -> 0.715 ms, full kernel 0.749 -> 0.936 ms at 1M x 1024).
    static const bool pair_ok = [] {
        const char* e = getenv("SW_SCORE_PAIR");
        return !(e && e[0] == '0');
    }();
    static const bool ts_ok = [] {
        const char* e = getenv("SW_SCORE_TS");
        return e && e[0] == '1';
    }();
    const bool pair = pair_ok && qb >= 2 && qb % 2 == 0;
    const bool ts = pair && ts_ok && p.kch * 32 <= 256 && p.kch % 2 == 0;
    // packed pyramid tiles (SW_SCORE_PACK=0 keeps the padded 256-row tiles, for A/B timing)
    static const bool pack_env = [] {
        const char* e = getenv("SW_SCORE_PACK");
        return !(e && e[0] == '0');
    }();
    const bool pack = pack_env && c.pack_ok && !ivf && !ts;
    const int tile_rows = pack ? 32 * c.R : BN;
    int stage_bytes = tile_rows * 128, a_bytes = p.kch * A_CHUNK, max_stages = 8;
    if (ts) {
        stage_bytes = 2 * B_QUARTER;  // two 64-wide K chunks per stage
        a_bytes = 0;
        max_stages = 12;
    } else if (pair) {
        stage_bytes = tile_rows / 2 * 128;
    }
    // CTA pairs keep 4 B stages: measured as fast as 6 (0.711 vs 0.708-0.729 ms; 3 stages lose
    // 12%), and the ~35 KB of shared memory it frees per SM lets one k_finish CTA of the
    // previous batch co-run with this kernel (sw_warmstart_async). SW_SCORE_STAGES overrides.
    static const int stage_env = [] {
        const char* e = getenv("SW_SCORE_STAGES");
        return e ? std::max(2, atoi(e)) : 0;
    }();
    const int stage_cap = stage_env ? stage_env : (pair ? 4 : 64);
    p.n_stages = std::min(std::min(max_stages, stage_cap), (budget - a_bytes) / stage_bytes);
    SW_REQUIRE(p.n_stages >= 2, "tcgen05 scoring: not enough shared memory for 2 stages");
    const int tbn = ts ? BN_TS : BN;
    const int64_t rows_hw = c.high_water * c.Rp;
    p.n_tiles = pack ? (c.high_water + 31) / 32 : (rows_hw + tbn - 1) / tbn;  // packed: 32 entries
    const int qblocks = qb;
    int64_t chunks = std::max<int64_t>(1, c.num_sms / qblocks);
    chunks = std::min<int64_t>(chunks, p.n_tiles);
    p.tiles_per_cta = (p.n_tiles + chunks - 1) / chunks;
    chunks = (p.n_tiles + p.tiles_per_cta - 1) / p.tiles_per_cta;
    // Balanced persistent schedule (opt-in, SW_SCORE_BAL=1): groups x R ranges = units x k
    // items, so all SMs work (B = 1024: 4 pair groups over 74 pairs -> R = 37, 2 range-major
    // items per pair, 148 SMs instead of 144). Measured SLOWER at config 3 and therefore off:
    // 0.738 vs 0.707 ms full kernel, and even the pure-MMA ablation loses (0.546 vs 0.531 ms)
    // although each pair issues 212 instead of 218 tiles — the item switch (A reload behind
    // the last MMA of the previous item, B ring drained) costs more than the 4 extra SMs give.
    static const bool bal_ok = [] {
        const char* e = getenv("SW_SCORE_BAL");
        return e && e[0] == '1';
    }();
    dim3 grid((unsigned)qblocks, (unsigned)chunks);
    p.bal_R = p.bal_k = 0;
    if (bal_ok && !ts) {
        const int units = pair ? c.num_sms / 2 : c.num_sms;
        const int groups = pair ? qblocks / 2 : qblocks;
        const int R = units / std::gcd(groups, units);
        const int64_t tpr = (p.n_tiles + R - 1) / R;
        if (R * EPI_GROUPS <= kMaxSlices && (int64_t)(R - 1) * tpr < p.n_tiles &&
            (int64_t)groups * R % units == 0) {
            p.bal_R = R;
            p.bal_k = (int)((int64_t)groups * R / units);
            p.n_items_bal = groups * R;
            p.tiles_per_cta = tpr;
            chunks = R;
            grid = dim3((unsigned)(pair ? 2 * units : units), 1);
        }
    }
    p.n_slots = c.high_water;
    p.valid_bits = c.valid_bits;
    p.q_eps = c.q_eps;
    p.thr = c.thr;
    p.top1 = c.top1;
    p.q_bf = c.q_bf;
    p.ivf = ivf ? 1 : 0;
    p.row_list = c.row_list;
    p.pmask = c.pmask;
    p.slice_cnt = c.slice_cnt;
    p.cta_topk = c.cta_topk;
    p.cand_slot = c.cand_slot;
    p.cand_score = c.cand_score;
    p.n_chunks = (int)chunks * EPI_GROUPS;  // emission slices: (CTA, epilogue group)
    p.cap_local = (kCandCap / p.n_chunks) & ~3;  // multiple of 4: 16-byte aligned slices
    c.last_chunks = p.n_chunks;
    const size_t smem = 1024 + (size_t)a_bytes + (size_t)p.n_stages * stage_bytes + 512;
    c.last_score_pair = pair;
    c.last_score_ts = ts;
    static const int experiment = [] {
        const char* e = getenv("SW_SCORE_EXPERIMENT");
        return e ? atoi(e) : 0;
    }();
    p.experiment = experiment;
    c.last_score_pack = pack;
    if (ts)
        launch_tc<true, true>(c, p, grid, smem, st, false);
    else if (pair)
        launch_tc<true, false>(c, p, grid, smem, st, pack);
    else
        launch_tc<false, false>(c, p, grid, smem, st, pack);
    SW_CUDA(cudaGetLastError());
    return 1;
}

}  // namespace sw
