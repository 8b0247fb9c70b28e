// TMA-staged structured neighbour reduce: the paper's Table-1 "direct access" kernel and
// every one of the nine relations (stencil.py:401-408 with the sum fold; kernels.py:27-59).
//
// Same pipeline as the fused MPDATA kernel: a persistent grid walks (TI x TJ tile) x
// (KC-level chunk) units; one TMA box [TI+2][colours][TJ+2][KC] of the source field (the
// tile plus its one-ring halo, all target colours) lands in a STAGES-deep shared-memory
// ring per unit; one thread per (tile position, level pair) folds every from-colour's
// neighbours from shared memory in canonical slot order (16-byte loads: both levels of the
// pair at once) and stores the result pair (and its periodic halo images) with one 16-byte
// store.  Offsets are compile-time constants of the relation.
#include <algorithm>
#include <climits>

#include "tsg_offsets.cuh"
#include "tsg_tma.cuh"

namespace tsg {

constexpr int kRedTJ = 16, kRedKC = 16, kRedStages = 3;
// tile rows: 8 for cell / edge sources (2-3 colours: 46-69 KB stages, 1024 threads), 4 for
// vertex sources (a 14 KB stage per 512 threads: several CTAs per SM); measured per relation
__host__ __device__ constexpr int red_ti(int ct) { return ct == 1 ? 4 : 8; }

constexpr int kRedBandTiles = 16;  // BAND schedule: tile columns per band

// One tile shape: TI x TJ elements x KC levels of a CT-colour source, STAGES-deep ring, one
// thread per (element, level pair).
template <int CT_, int TI_, int TJ_, int KC_ = kRedKC, int STAGES_ = kRedStages>
struct RedShape {
    static constexpr int CT = CT_, TI = TI_, TJ = TJ_, KC = KC_, STAGES = STAGES_;
    static constexpr int kLanes = KC / 2;  // threads per element: one level pair each
    static constexpr int kThreads = TI * TJ * kLanes;
    static constexpr int kBoxBytes = (TI + 2) * CT * (TJ + 2) * KC * 8;
    static constexpr int kStageBytes = (kBoxBytes + 127) / 128 * 128;
    static constexpr int kSmemBytes = STAGES * kStageBytes + 128;
};

// TALL: the tile transposed (16 rows x red_ti columns) -- two halo rows per 16 instead of
// per 4 or 8, for patches whose tile above is no longer in L2 when a tile is loaded
// (launch_reduce_tma; the fused kernel's rule, mpdata_fused.cu pick_variant)
template <int CT, bool TALL = false>
using RedCfg = RedShape<CT, TALL ? kRedTJ : red_ti(CT), TALL ? red_ti(CT) : kRedTJ>;

struct RedArgs {
    double *dst;
    const double *scale;
    const double *length, *area, *weights;  // cell divergence (MODE 1 / 2)
    int rows, cols, nk, flags;
    int tiles_j, chunks;
    int64_t units;
    // DYN: the ticket words ([0] items taken, [1] CTAs done; the last CTA resets both), the
    // tiles [0, whole) dealt whole (every chunk back to back), then one unit per item
    uint32_t *ticket;
    uint32_t whole, items;
};

// BAND schedule: unit u of the grid-stride order (CTA b runs b, b + G, ...) is tile
// band-major (bands of band_w tile columns, tile rows within a band), so the units in
// flight at any time are one band row and its neighbours: the halo a tile shares with the
// tile row above is still in L2 (no per-tile state to reload in this kernel).  A separate
// kernel parameter, so the contiguous instantiations compile exactly as before.
struct BandArgs {
    int band_w, nb_full;
    uint32_t full_tiles;
    FastDiv fd_chunks, fd_band_tiles, fd_bw, fd_bw_last;
};

__device__ __forceinline__ void band_decode(uint32_t u, const BandArgs &a, int &ti, int &tj, int &chunk) {
    const uint32_t t = a.fd_chunks.div(u);
    chunk = (int)(u - t * a.fd_chunks.d);
    if (t < a.full_tiles) {
        const uint32_t band = a.fd_band_tiles.div(t), r = t - band * a.fd_band_tiles.d;
        const uint32_t row = a.fd_bw.div(r);
        ti = (int)row;
        tj = (int)(band * a.band_w + (r - row * a.fd_bw.d));
    } else {
        const uint32_t r = t - a.full_tiles, row = a.fd_bw_last.div(r);
        ti = (int)row;
        tj = a.nb_full * a.band_w + (int)(r - row * a.fd_bw_last.d);
    }
}

// MODE 0: sum fold (times scale[from] if SCALE); MODE 1: cell divergence
// sum vn*length / area; MODE 2: weighted cell divergence sum vn*weights[c, n]
// (mpdata.py:361-376; reference.py:119-134)
template <int REL, bool SCALE, int MODE, class C, bool BAND = false, bool DYN = false>
__global__ void __launch_bounds__(C::kThreads)
    reduce_tma_kernel(const __grid_constant__ CUtensorMap tm_src, const RedArgs a, const BandArgs ba) {
    constexpr int CF = loc_colors(REL / 3), CT = loc_colors(REL % 3), W = rel_width(REL);
    static_assert(C::CT == CT, "tile shape built for another source location");
    constexpr int TI = C::TI, TJ = C::TJ, KC = C::KC, STAGES = C::STAGES, kLanes = C::kLanes;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + STAGES * C::kStageBytes);

    const int tid = threadIdx.x, kl = (tid % kLanes) * 2, v = tid / kLanes;
    const int li = v / TJ, lj = v % TJ;
    // source box [TI+2][CT][TJ+2][KC], origin (i0-1, colour 0, j0-1, k0)
    constexpr int sJ = KC, sC = (TJ + 2) * KC, sI = CT * (TJ + 2) * KC;
    const int oS = (li + 1) * sI + (lj + 1) * sJ + kl;

    // DYN: each stage's unit (tile, chunk) as dealt by the ticket; tile < 0: no work left
    int2 *info = reinterpret_cast<int2 *>(bars + STAGES);
    const int u_begin = DYN ? 0 : BAND ? (int)blockIdx.x : (int)(a.units * blockIdx.x / gridDim.x);
    const int n_units = DYN    ? INT_MAX
                        : BAND ? (int)((a.units - blockIdx.x + gridDim.x - 1) / gridDim.x)
                               : (int)(a.units * (blockIdx.x + 1) / gridDim.x) - u_begin;
    if (tid == 0) {
        prefetch_tmap(&tm_src);
        for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    int p_chunk = u_begin % a.chunks, p_tile = u_begin / a.chunks;
    int p_ti = p_tile / a.tiles_j, p_tj = p_tile % a.tiles_j;
    auto issue_next = [&](int stage, int m) {  // m: the unit's index in this CTA's sequence
        uint64_t *bar = &bars[stage];
        mbar_expect_tx(bar, C::kBoxBytes);
        if constexpr (BAND) band_decode((uint32_t)(u_begin + m * (int)gridDim.x), ba, p_ti, p_tj, p_chunk);
        tma_load_4d(smem + stage * C::kStageBytes, &tm_src, bar, p_chunk * KC, p_tj * TJ, 0, p_ti * TI);
        if (BAND) return;
        if (++p_chunk == a.chunks) {
            p_chunk = 0;
            if (++p_tj == a.tiles_j) {
                p_tj = 0;
                ++p_ti;
            }
        }
    };
    // DYN producer (thread 0): the item in hand (tile, chunks [d_c, d_c1)) and the next
    // ticket, taken one item ahead so its latency overlaps the current item's loads
    uint32_t d_next = 0;
    int d_tile = 0, d_c = 0, d_c1 = 0;
    bool d_live = DYN;
    auto issue_dyn = [&](int stage) {
        uint64_t *bar = &bars[stage];
        if (d_c == d_c1) {
            const uint32_t it = d_next;
            if (it >= a.items) {  // this CTA's last ticket: no further takes
                d_live = false;
                info[stage] = make_int2(-1, 0);
                mbar_arrive(bar);
                // order this CTA's ticket takes before its done count: the CTA that resets
                // the words must see every take (else a stale count leaks into the next launch)
                __threadfence();
                if (atomicAdd(&a.ticket[1], 1u) == gridDim.x - 1) {  // every CTA is done taking
                    __threadfence();
                    a.ticket[0] = 0;
                    a.ticket[1] = 0;
                }
                return;
            }
            d_next = atomicAdd(&a.ticket[0], 1u);
            if (it < a.whole) {
                d_tile = (int)it;
                d_c = 0;
                d_c1 = a.chunks;
            } else {
                const int u = (int)(it - a.whole), q = u / a.chunks;
                d_tile = (int)a.whole + q;
                d_c = u - q * a.chunks;
                d_c1 = d_c + 1;
            }
        }
        const int c = d_c++;
        info[stage] = make_int2(d_tile, c);
        mbar_expect_tx(bar, C::kBoxBytes);  // releases the info slot with the arrival
        const int t_i = d_tile / a.tiles_j;
        tma_load_4d(smem + stage * C::kStageBytes, &tm_src, bar, c * KC, (d_tile - t_i * a.tiles_j) * TJ, 0,
                    t_i * TI);
    };
    if (tid == 0) {
        if constexpr (DYN) {
            d_next = atomicAdd(&a.ticket[0], 1u);
            for (int s = 0; s < STAGES - 1 && d_live; ++s) issue_dyn(s);
        } else {
            for (int s = 0; s < STAGES - 1 && s < n_units; ++s) issue_next(s, s);
        }
    }

    int chunk = u_begin % a.chunks, tile = u_begin / a.chunks;
    int ti = tile / a.tiles_j, tj = tile % a.tiles_j;
    const int64_t pv = pitch_of(a.nk);
    const FieldIx Fd(a.rows, a.cols, CF, a.nk), Fsc(a.rows, a.cols, CF, 1);
    bool valid = false;
    double *out[CF];
    double sc[CF];
    double w[MODE ? CF : 1][MODE ? W : 1];  // per-element edge weights (cell divergence)
    int64_t dr = 0, dc = 0;
    int cur_tile = -1;  // DYN: the tile whose per-element state is loaded
    bool fresh = false;

    for (int n = 0; n < n_units; ++n) {
        const int stage = n % STAGES;
        if constexpr (DYN) {
            if (tid == 0 && d_live) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue_dyn((n + STAGES - 1) % STAGES);
            }
            mbar_wait(&bars[stage], (uint32_t)((n / STAGES) & 1));
            const int2 u = info[stage];
            if (u.x < 0) break;
            chunk = u.y;
            fresh = u.x != cur_tile;
            if (fresh) {
                cur_tile = u.x;
                ti = cur_tile / a.tiles_j;
                tj = cur_tile - ti * a.tiles_j;
            }
        } else if (tid == 0 && n + STAGES - 1 < n_units) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue_next((n + STAGES - 1) % STAGES, n + STAGES - 1);
        }
        if constexpr (BAND) band_decode((uint32_t)(u_begin + n * (int)gridDim.x), ba, ti, tj, chunk);
        if (DYN ? fresh : (BAND || n == 0 || chunk == 0)) {
            const int i = ti * TI + li, j = tj * TJ + lj;
            valid = i < a.rows && j < a.cols;
            if (valid) {
#pragma unroll
                for (int c = 0; c < CF; ++c) {
                    out[c] = a.dst + Fd.at(i, c, j);
                    sc[c] = SCALE ? __ldg(a.scale + Fsc.at(i, c, j)) : 1.0;
                    if constexpr (MODE == 1) {
                        const FieldIx Fl(a.rows, a.cols, 3, 1);
                        sc[c] = __ldg(a.area + Fsc.at(i, c, j));
#pragma unroll
                        for (int q = 0; q < W; ++q)
                            w[c][q] = __ldg(a.length + Fl.at(i + rel_off(REL, c, q, 0), rel_off(REL, c, q, 1),
                                                             j + rel_off(REL, c, q, 2)));
                    } else if constexpr (MODE == 2) {
                        const FieldIx Fw(a.rows, a.cols, CF, 3);
#pragma unroll
                        for (int q = 0; q < W; ++q) w[c][q] = __ldg(a.weights + Fw.at(i, c, j) + q);
                    }
                }
                dr = 0;
                dc = 0;
                if (a.flags & TSG_PERIODIC_ROWS) {
                    if (i == 0) dr = (int64_t)a.rows * Fd.rowstr;
                    else if (i == a.rows - 1) dr = -(int64_t)a.rows * Fd.rowstr;
                }
                if (a.flags & TSG_PERIODIC_COLS) {
                    if (j == 0) dc = (int64_t)a.cols * pv;
                    else if (j == a.cols - 1) dc = -(int64_t)a.cols * pv;
                }
            }
        }
        if constexpr (!DYN) mbar_wait(&bars[stage], (uint32_t)((n / STAGES) & 1));
        const int k = chunk * KC + kl;  // this thread's level pair (k, k+1)
        if (valid && k < a.nk) {
            const double *S = reinterpret_cast<const double *>(smem + stage * C::kStageBytes) + oS;
            const bool pair = k + 1 < a.nk;
#pragma unroll
            for (int c = 0; c < CF; ++c) {
                double2 acc = make_double2(0.0, 0.0);
#pragma unroll
                for (int s = 0; s < W; ++s) {
                    const double2 x = ld2(S + rel_off(REL, c, s, 0) * sI + rel_off(REL, c, s, 1) * sC +
                                          rel_off(REL, c, s, 2) * sJ);
                    if (MODE) {
                        acc.x = add(mul(x.x, w[c][s]), acc.x);
                        acc.y = add(mul(x.y, w[c][s]), acc.y);
                    } else {
                        acc.x = add(x.x, acc.x);
                        acc.y = add(x.y, acc.y);
                    }
                }
                if (SCALE) acc = make_double2(mul(acc.x, sc[c]), mul(acc.y, sc[c]));
                if (MODE == 1) acc = make_double2(dvd(acc.x, sc[c]), dvd(acc.y, sc[c]));
                double *o = out[c] + k;
                if (pair) {
                    // contiguous ranges: streaming (evict-first) stores leave L2 to the
                    // source's halos (Table-1 direct 1024^2: 516 vs 523 us); the band
                    // schedule keeps its halos in L2 anyway and does better without
                    auto put = [](double *q, double2 x) {
                        if constexpr (BAND) st2(q, x);
                        else __stcs(reinterpret_cast<double2 *>(q), x);
                    };
                    put(o, acc);
                    if (dr | dc) {
                        if (dr) put(o + dr, acc);
                        if (dc) put(o + dc, acc);
                        if (dr && dc) put(o + dr + dc, acc);
                    }
                } else {  // odd level count: the last level alone
                    o[0] = acc.x;
                    if (dr | dc) {
                        if (dr) o[dr] = acc.x;
                        if (dc) o[dc] = acc.x;
                        if (dr && dc) o[dr + dc] = acc.x;
                    }
                }
            }
        }
        if (!DYN && ++chunk == a.chunks) {
            chunk = 0;
            if (++tj == a.tiles_j) {
                tj = 0;
                ++ti;
            }
        }
        __syncthreads();
    }
}

template <int REL, bool SCALE, int MODE, class C, bool BAND = false, bool DYN = false>
static int launch_reduce_shape(const tsg_grid *g, int inner, const double *src, const double *scale,
                               double *dst, cudaStream_t st, const double *length,
                               const double *area, const double *weights) {
    constexpr int CT = loc_colors(REL % 3);
    const cuuint64_t p = (cuuint64_t)pitch_of(inner), W = (cuuint64_t)g->cols + 2, H = (cuuint64_t)g->rows + 2;
    cuuint64_t dims[4] = {(cuuint64_t)inner, W, (cuuint64_t)CT, H};
    cuuint64_t str[3] = {p * 8, W * p * 8, CT * W * p * 8};
    cuuint32_t box[4] = {(cuuint32_t)C::KC, (cuuint32_t)C::TJ + 2, (cuuint32_t)CT, (cuuint32_t)C::TI + 2};
    CUtensorMap m;
    if (int rc = make_map(&m, src, 4, dims, str, box)) return rc;
    RedArgs a;
    a.dst = dst;
    a.scale = scale;
    a.length = length;
    a.area = area;
    a.weights = weights;
    a.rows = g->rows;
    a.cols = g->cols;
    a.nk = inner;
    a.flags = g->flags;
    a.tiles_j = (g->cols + C::TJ - 1) / C::TJ;
    a.chunks = (inner + C::KC - 1) / C::KC;
    a.units = (int64_t)((g->rows + C::TI - 1) / C::TI) * a.tiles_j * a.chunks;
    if (a.units >= (1LL << 31)) return fail(TSG_EVALUE, "field too large for one reduce launch");
    BandArgs ba;
    {
        const int tiles_i = (g->rows + C::TI - 1) / C::TI;
        ba.band_w = std::min(kRedBandTiles, a.tiles_j);
        ba.nb_full = a.tiles_j / ba.band_w;
        const int bw_last = a.tiles_j - ba.nb_full * ba.band_w;
        ba.full_tiles = (uint32_t)(ba.nb_full * ba.band_w * tiles_i);
        ba.fd_chunks = FastDiv((uint32_t)a.chunks);
        ba.fd_band_tiles = FastDiv((uint32_t)(ba.band_w * tiles_i));
        ba.fd_bw = FastDiv((uint32_t)ba.band_w);
        ba.fd_bw_last = FastDiv((uint32_t)(bw_last > 0 ? bw_last : 1));
    }
    void *fn = (void *)reduce_tma_kernel<REL, SCALE, MODE, C, BAND, DYN>;
    TSG_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes));
    int per_sm = 0;
    TSG_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, C::kThreads, C::kSmemBytes));
    int64_t grid = (int64_t)g->num_sms * (per_sm < 1 ? 1 : per_sm);
    if (grid > a.units) grid = a.units;
    a.ticket = nullptr;
    a.whole = a.items = 0;
    if (DYN) {
        if (!g->dyn_ws) return fail(TSG_EVALUE, "grid has no workspace for the dynamic deal");
        a.ticket = reinterpret_cast<uint32_t *>(static_cast<unsigned char *>(g->dyn_ws) + kDynReduceTicketOff);
        // whole tiles, then the last ~two rounds of the grid one unit at a time
        const int64_t tiles = a.units / a.chunks;
        const int64_t tail = std::min<int64_t>(tiles, (2 * grid + a.chunks - 1) / a.chunks);
        a.whole = (uint32_t)(tiles - tail);
        a.items = (uint32_t)(a.whole + tail * a.chunks);
    }
    void *args[] = {&m, &a, &ba};
    TSG_CHECK_CUDA(cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(C::kThreads), args, C::kSmemBytes, st));
    return TSG_OK;
}

// Benchmarking hook (tsg_set_reduce_variant): alternative compact tile shapes for the sum
// fold (MODE 0, no scale), per source location; 0 = the default RedCfg; 1-9 static
// contiguous ranges, 11-19 the same shapes dynamically dealt.
static int g_red_variant = 0;

template <int REL, bool SCALE, int MODE>
static int launch_compact(const tsg_grid *g, int inner, const double *src, const double *scale,
                          double *dst, cudaStream_t st, const double *length, const double *area,
                          const double *weights) {
    constexpr int CT = loc_colors(REL % 3);
#define TSG_RV(N, ...)                                                                             \
    if (g_red_variant == N)                                                                        \
        return launch_reduce_shape<REL, SCALE, MODE, RedShape<__VA_ARGS__>>(g, inner, src, scale, dst, \
                                                                          st, length, area, weights); \
    if (g_red_variant == N + 10)                                                                   \
        return launch_reduce_shape<REL, SCALE, MODE, RedShape<__VA_ARGS__>, false, true>(            \
            g, inner, src, scale, dst, st, length, area, weights);
    if constexpr (MODE == 0 && !SCALE) {
        if constexpr (CT == 1) {
            TSG_RV(1, 1, 4, 16, 16, 3)
            TSG_RV(2, 1, 8, 16, 16, 3)
            TSG_RV(3, 1, 4, 16, 16, 4)
            TSG_RV(4, 1, 4, 32, 16, 3)
            TSG_RV(5, 1, 4, 16, 32, 3)
            TSG_RV(6, 1, 2, 16, 16, 3)
            TSG_RV(7, 1, 4, 16, 16, 6)
            TSG_RV(8, 1, 8, 16, 16, 4)
            TSG_RV(9, 1, 2, 32, 16, 4)
        } else if constexpr (CT == 2) {
            TSG_RV(1, 2, 8, 16, 16, 3)
            TSG_RV(2, 2, 4, 16, 16, 3)
            TSG_RV(3, 2, 8, 16, 16, 4)
            TSG_RV(4, 2, 4, 16, 16, 5)
            TSG_RV(5, 2, 4, 32, 16, 3)
        } else {
            TSG_RV(1, 3, 8, 16, 16, 3)
            TSG_RV(2, 3, 4, 16, 16, 3)
        }
    } else if constexpr (MODE != 0 && CT == 3) {  // cell divergence (edge source)
        TSG_RV(1, 3, 4, 16, 16, 3)
        TSG_RV(2, 3, 2, 16, 16, 4)
        TSG_RV(3, 3, 4, 16, 16, 5)
        TSG_RV(4, 3, 2, 16, 16, 3)
        TSG_RV(5, 3, 4, 8, 16, 4)
        TSG_RV(6, 3, 2, 32, 16, 3)
        TSG_RV(7, 3, 8, 16, 16, 3)
        TSG_RV(8, 3, 2, 16, 16, 6)
        TSG_RV(9, 3, 4, 8, 16, 6)
    }
#undef TSG_RV
    return launch_reduce_shape<REL, SCALE, MODE, RedCfg<CT, false>>(g, inner, src, scale, dst, st, length,
                                                                    area, weights);
}

// The compact tile unless the tile above a tile (its upper halo) was loaded more than
// kRedReuseUnits units earlier in the contiguous per-CTA schedule (then evicted from L2).
// Then: the band schedule for the edge relations (edge source or edge destination: the
// largest boxes, or three outputs per thread), the tall tile otherwise -- measured per
// relation at 256x256x80 (band vs tall: EE 41.0 vs 50.2 us, EC 35.4 vs 41.0, CE 36.1 vs
// 38.9, EV 31.2 vs 33.5, VE 31.0 vs 33.1; but VV 23.2 vs 20.0, VC 28.2 vs 25.2, CV 25.2
// vs 24.1, CC even, cell divergence slower: the per-unit tile change costs more than the
// halo re-reads save when a unit carries little work).
constexpr double kRedReuseUnits = 8.0;

// Patches with at least kRedDynUnits units per resident CTA deal their tiles dynamically
// (DYN: a global ticket in tile-major order, whole tiles, the last two rounds unit by unit):
// every CTA then sweeps the patch in step with the others, so a tile's halo rows are L2
// hits, and no CTA idles while another finishes a longer range.  tools/reduce_variants.py
// (tsg_set_reduce_variant), L2 flushed before each launch, mean of 200:
//   512x512x137:  CC 266 -> 208 us, VV 132 -> 107, EE 412 -> 296, VC 192 -> 142
//   1024x1024x80: CC 511 -> 413 us (Table-1 direct), VV 252 -> 223, EV 604 -> 438, CE 730 -> 520
// while at 256x256x80 (~12 units per CTA) the static ranges are as fast or faster (EC 34.8
// vs 37.1, EE 41.3 vs 44.5).  Dealt shapes per source location: 2 x 16 vertex tiles (8 CTAs
// per SM), 4 x 16 cell and edge tiles, 8 x 16 edge tiles for V <- E (its 3 outputs per
// thread want the wider tile: 1024^2 383 vs 450 us).  The cell divergence (C <- E with
// edge weights, a division per output in the simple form) takes 8 x 16 tiles too: 1024^2
// simple / weighted 614 / 537 vs 673 / 587 us, 512x512x137 272 / 263 vs 286 / 261
// (tools/reduce_variants.py celldiv, variant 17; bitwise equal).
constexpr double kRedDynUnits = 24.0;

template <int REL>
using RedDynShape = RedShape<loc_colors(REL % 3), loc_colors(REL % 3) == 1 ? 2 : REL == 2 ? 8 : 4, 16>;
// V <- V at small sizes: 2 x 16 tiles (256x256x80 18.9 vs 20.4 us for the tall 16 x 4)
using RedVVShape = RedShape<1, 2, 16>;

template <int REL, bool SCALE, int MODE = 0>
static int launch_reduce_tma(const tsg_grid *g, int inner, const double *src, const double *scale,
                             double *dst, cudaStream_t st, const double *length = nullptr,
                             const double *area = nullptr, const double *weights = nullptr) {
    constexpr int CT = loc_colors(REL % 3);
    using C = RedCfg<CT, false>;
    if (int rc = get_encode()) return rc;
    static int per_sm = 0;  // resident compact CTAs per SM (same for every call)
    if (!per_sm) {
        void *fn = (void *)reduce_tma_kernel<REL, SCALE, MODE, C>;
        TSG_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes));
        TSG_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, C::kThreads, C::kSmemBytes));
        if (per_sm < 1) per_sm = 1;
    }
    const double tiles_j = (g->cols + C::TJ - 1) / C::TJ, chunks = (inner + kRedKC - 1) / kRedKC;
    const double units = (double)((g->rows + C::TI - 1) / C::TI) * tiles_j * chunks;
    const double range = units / ((double)g->num_sms * per_sm), R = tiles_j * chunks;
    const double gap = R < range ? R : R - range * (double)(int64_t)(R / range);
    if (!g_red_variant && range >= kRedDynUnits) {
        if constexpr (MODE != 0)
            return launch_reduce_shape<REL, SCALE, MODE, RedShape<loc_colors(REL % 3), 8, 16>, false, true>(
                g, inner, src, scale, dst, st, length, area, weights);
        return launch_reduce_shape<REL, SCALE, MODE, RedDynShape<REL>, false, true>(g, inner, src, scale, dst, st,
                                                                                   length, area, weights);
    }
    if constexpr (REL == 0)
        if (!g_red_variant)
            return launch_reduce_shape<REL, SCALE, MODE, RedVVShape>(g, inner, src, scale, dst, st, length, area,
                                                                     weights);
    if (g_red_variant || gap <= kRedReuseUnits)
        return launch_compact<REL, SCALE, MODE>(g, inner, src, scale, dst, st, length, area, weights);
    constexpr bool kEdgeRel = REL % 3 == TSG_EDGES || REL / 3 == TSG_EDGES;
    if constexpr (MODE == 0 && kEdgeRel)
        return launch_reduce_shape<REL, SCALE, MODE, C, true>(g, inner, src, scale, dst, st, length, area,
                                                                 weights);
    return launch_reduce_shape<REL, SCALE, MODE, RedCfg<CT, true>>(g, inner, src, scale, dst, st, length, area, weights);
}

// dispatch over the nine relations; returns TSG_OK or an error
int reduce_tma(const tsg_grid *g, int rel, int inner, const double *src, const double *scale,
               double *dst, cudaStream_t st) {
#define TSG_RT_CASE(R)                                                                  \
    case R:                                                                            \
        return scale ? launch_reduce_tma<R, true>(g, inner, src, scale, dst, st)       \
                     : launch_reduce_tma<R, false>(g, inner, src, scale, dst, st);
    switch (rel) {
        TSG_RT_CASE(0) TSG_RT_CASE(1) TSG_RT_CASE(2) TSG_RT_CASE(3) TSG_RT_CASE(4)
        TSG_RT_CASE(5) TSG_RT_CASE(6) TSG_RT_CASE(7) TSG_RT_CASE(8)
    }
#undef TSG_RT_CASE
    return fail(TSG_EVALUE, "bad relation %d", rel);
}

int cell_divergence_tma(const tsg_grid *g, int weighted, const double *vn, const double *length,
                        const double *area, const double *weights, double *out, cudaStream_t st) {
    constexpr int REL = TSG_CELLS * 3 + TSG_EDGES;
    return weighted ? launch_reduce_tma<REL, false, 2>(g, g->levels, vn, nullptr, out, st, nullptr,
                                                      nullptr, weights)
                    : launch_reduce_tma<REL, false, 1>(g, g->levels, vn, nullptr, out, st, length, area,
                                                      nullptr);
}

}  // namespace tsg

extern "C" int tsg_set_reduce_variant(int variant) {
    if (variant < 0 || variant > 19) return tsg::fail(TSG_EVALUE, "reduce variant must be in [0, 19]");
    tsg::g_red_variant = variant;
    return TSG_OK;
}
