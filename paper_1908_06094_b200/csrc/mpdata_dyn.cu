// Dynamically scheduled fused MPDATA step, and the persistent multi-step time loop.
//
// Same work unit, stage layout, producer warp and arithmetic as the static-schedule kernel
// (mpdata_fused.cu: one TI x TJ vertex tile x a KC-level chunk per unit, four TMA boxes
// per stage, level pairs), with two changes in how units reach CTAs:
//
//  * Dynamic deal.  The producer warp takes work from a global ticket (one atomicAdd per
//    item) instead of a precomputed contiguous range, so a CTA whose units run slower
//    simply takes fewer: on 279x256x80 the static ranges leave the CTAs' end times spread
//    over ~7 us (tsg_debug_trace: 48.8 .. 56.1 us) for the same 37-38 units each.  Items
//    are whole tiles (all chunks back to back, per-vertex state kept in registers) in the
//    band order of mpdata_fused.cu (tile-major below 16 tile columns), except the last
//    ~two rounds of the (last) step, which are dealt one unit at a time so the CTAs end
//    within about one unit of each other.  The producer writes each unit's coordinates
//    into a per-stage info slot and arrives on the stage's info mbarrier as it issues the
//    loads, so the consumer warps learn the next tile (and load its signs / dual volume)
//    while its data is still in flight.
//
//  * MULTI: a time loop of S steps in ONE launch (tsg_mpdata_run).  The items of step s+1
//    follow those of step s in the same ticket order; steps ping-pong between the two
//    density buffers.  Before loading a tile at step s > 0 the producer waits until the
//    tile and its eight neighbours (periodic wrap) have finished step s-1: every consumer
//    warp publishes each unit it completes with a release add on the tile's counter
//    (red.release.gpu after __syncwarp), the producer reads the nine counters relaxed,
//    then fence.acq_rel.gpu + fence.proxy.async.global before the TMA reads.  The same
//    condition covers the write-after-read hazard (step s+1 overwrites step s-1's input
//    buffer, whose halo readers are exactly those nine tiles at step s-1) and the
//    periodic halo images (written by the opposite boundary tiles, which the wrap
//    includes).  Items are taken in order and dependencies only point to earlier steps,
//    so with every CTA resident (one per SM, cooperative launch) the earliest unfinished
//    item can always proceed: no deadlock.  A step's fill and drain then overlap the
//    neighbouring steps instead of costing a launch each.
//
// Counters: the ticket words are reset by the last producer to finish; the tile counters
// are monotonic across launches and the launch reads their common base (advanced by the
// last producer), so no per-launch reset pass is needed.  Launches that share a grid
// handle's workspace must be stream-ordered (include/tsg.h).
#include "mpdata_common.cuh"

namespace tsg {

__device__ __forceinline__ uint64_t ld_relaxed_gpu(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void red_release_gpu_add(uint64_t *p, uint64_t v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// item -> (step, tile in the band order, chunk range)
__device__ __forceinline__ bool decode_item(uint32_t it, const DynArgs &d, int chunks, int &s, uint32_t &t,
                                            int &c0, int &c1) {
    if (it >= d.items) return false;
    const uint32_t full = (uint32_t)(d.nsteps - 1) * d.tiles + d.whole;  // whole-tile items
    if (it < full) {
        s = (int)d.fd_tiles.div(it);
        t = it - (uint32_t)s * d.tiles;
        c0 = 0;
        c1 = chunks;
    } else {
        const uint32_t u = it - full, q = d.fd_chunks.div(u);
        s = d.nsteps - 1;
        t = d.whole + q;
        c0 = (int)(u - q * (uint32_t)chunks);
        c1 = c0 + 1;
    }
    return true;
}

template <int TI, int TJ, int KC, int STAGES, int OP, bool PEER, bool MULTI>
__global__ void __launch_bounds__(TI *TJ * 8 + (MULTI ? 64 : 32), 1)
    mpdata_dyn_kernel(const __grid_constant__ CUtensorMap tm_pd, const __grid_constant__ CUtensorMap tm_pd_alt,
                      const __grid_constant__ CUtensorMap tm_vn, const __grid_constant__ CUtensorMap tm_wn,
                      const __grid_constant__ CUtensorMap tm_rho, const FusedArgs a, const BandArgs ba,
                      const DynArgs d) {
    using C = FusedCfg<TI, TJ, KC, STAGES, 8, 2>;
    constexpr int kConsumers = TI * TJ * 8;
    constexpr int kWarps = kConsumers / 32;
    extern __shared__ __align__(128) unsigned char smem[];
    int4 *info = reinterpret_cast<int4 *>(smem + STAGES * C::kStageBytes);  // (ti, tj, chunk, step); ti < 0: done
    uint64_t *full = reinterpret_cast<uint64_t *>(info + STAGES);
    uint64_t *empty = full + STAGES;
    uint64_t *ibar = empty + STAGES;
    uint64_t *dbar = ibar + STAGES;  // MULTI: consumer warps done with the stage's unit

    const int tid = threadIdx.x;
    const int chunks = a.chunks;
    // PEER: the global step this launch starts with (the device step counter, advanced by
    // the previous launch; read before any CTA can finish this one)
    int64_t wv = a.wait_value;
    if constexpr (PEER) {
        if (a.epoch) wv = *reinterpret_cast<volatile const int64_t *>(a.epoch);
    }
    if (a.trace && tid == 0) a.trace[4 * blockIdx.x] = globaltimer_ns();
    if (tid == 0) {
        prefetch_tmap(&tm_pd);
        if (MULTI) prefetch_tmap(&tm_pd_alt);
        prefetch_tmap(&tm_vn);
        prefetch_tmap(&tm_wn);
        prefetch_tmap(&tm_rho);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            // every consumer thread arrives (each read the stage's info slot; a per-warp
            // arrival after __syncwarp orders the same, but compute-sanitizer's racecheck
            // follows only the arriving thread's reads); MULTI: the signal warp's one too
            mbar_init(&empty[s], kConsumers + (MULTI ? 1 : 0));
            mbar_init(&ibar[s], 1);
            if (MULTI) mbar_init(&dbar[s], kWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (MULTI && tid >= kConsumers + 32) {  // ---- the signal warp (MULTI) ----
        // Publishes finished tiles for the other CTAs' dependency waits, off the consumers'
        // and the producer's paths: per unit it waits until every consumer warp is done
        // (dbar), releases the stage to the producer (its arrival completes `empty` with the
        // consumer warps' own), and after a tile's last chunk
        // adds 1 to the tile's counter with gpu-scope release semantics -- cumulative over
        // the consumer warps' pd_out stores it acquired through the mbarrier.  It never lags
        // more than one phase: the producer cannot refill a stage it has not released.
        if (tid != kConsumers + 32) return;
        for (uint32_t n = 0;; ++n) {
            const int stage = (int)(n % STAGES);
            const uint32_t ph = (n / STAGES) & 1;
            mbar_wait(&ibar[stage], ph);
            const int4 inf = info[stage];
            if (inf.x < 0) break;
            mbar_wait(&dbar[stage], ph);
            mbar_arrive(&empty[stage]);
            if constexpr (PEER) {
                // a row strip's loop: the unit's stores into the neighbours' halo rows are
                // made visible system-wide, and the last boundary unit of the step releases
                // the step into both neighbours' flag words (what their boundary rows wait on)
                if (inf.x == 0 || inf.x == a.tiles_i - 1) {
                    __threadfence_system();
                    if (atomicAdd(d.bdone + (inf.w & 1), 1) == d.nb_units - 1) {
                        d.bdone[inf.w & 1] = 0;
                        __threadfence_system();
                        const int64_t v = wv + inf.w + 1;
                        if (a.flag_up) asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(a.flag_up), "l"(v) : "memory");
                        if (a.flag_down) asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(a.flag_down), "l"(v) : "memory");
                    }
                }
            }
            if (inf.z == chunks - 1 && inf.w < d.nsteps - 1) {
                const uint64_t f0 = a.trace ? globaltimer_ns() : 0;
                red_release_gpu_add(d.tile_done + (int64_t)inf.x * a.tiles_j + inf.y, 1);
                if (a.trace) {  // MULTI trace slot 3: time spent publishing (ns)
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    a.trace[4 * blockIdx.x + 3] += globaltimer_ns() - f0;
                }
            }
        }
        return;
    }
    if (tid >= kConsumers) {  // ---- the producer warp (one thread issues) ----
        if (tid != kConsumers) return;
        bool waited = !(PEER && a.my_flags);
        int waited_s = -1;  // MULTI + PEER: the last step whose neighbour flags were seen
        const uint64_t base = MULTI ? *reinterpret_cast<volatile const uint64_t *>(d.base) : 0;
        uint32_t n = 0;  // units issued
        uint32_t it = atomicAdd(&d.ticket[0], 1u);
        for (;;) {
            int s, c0, c1;
            uint32_t t;
            if (!decode_item(it, d, chunks, s, t, c0, c1)) break;
            int ti, tj;
            band_tile(t, ba, ti, tj);
            uint64_t nb[9];
            const uint64_t *nbp[9];
            if constexpr (MULTI) {
                if (s > 0) {  // relaxed reads of the nine counters, checked after the slot wait
                    for (int q = 0; q < 9; ++q) {
                        int r = ti + q / 3 - 1, c = tj + q % 3 - 1;
                        if (r < 0 || r >= a.tiles_i)  // a strip's row halo comes from the neighbours
                            r = !(a.flags & TSG_PERIODIC_ROWS) ? ti : (r < 0 ? r + a.tiles_i : r - a.tiles_i);
                        c = c < 0 ? c + a.tiles_j : (c >= a.tiles_j ? c - a.tiles_j : c);
                        nbp[q] = d.tile_done + (int64_t)r * a.tiles_j + c;
                        nb[q] = ld_relaxed_gpu(nbp[q]);
                    }
                }
            }
            for (int c = c0; c < c1; ++c) {
                uint32_t next = 0;
                if (c == c1 - 1) next = atomicAdd(&d.ticket[0], 1u);  // in flight while we wait
                const int stage = (int)(n % STAGES);
                if (n >= STAGES) mbar_wait(&empty[stage], ((n / STAGES) - 1) & 1);
                if (c == c0) {
                    if constexpr (MULTI) {
                        if (s > 0) {  // the tile and its neighbours finished step s-1
                            const uint64_t need = base + (uint64_t)s;
                            const uint64_t t0 = globaltimer_ns();
                            unsigned backoff = 32;
                            for (int q = 0; q < 9; ++q) {
                                while (nb[q] < need) {
                                    if (globaltimer_ns() - t0 > d.timeout_ns) {
                                        atomicExch(d.err, 2);
                                        break;
                                    }
                                    __nanosleep(backoff);
                                    if (backoff < 1024) backoff *= 2;
                                    nb[q] = ld_relaxed_gpu(nbp[q]);
                                }
                            }
                            asm volatile("fence.acq_rel.gpu;" ::: "memory");
                            asm volatile("fence.proxy.async.global;" ::: "memory");
                            if (a.trace) a.trace[4 * blockIdx.x + 1] += globaltimer_ns() - t0;  // MULTI: waited (ns)
                        }
                    }
                    if constexpr (PEER) {
                        // a boundary tile row reads the neighbours' rows of the previous step and
                        // overwrites their halo rows read in it: wait for their step flags
                        const bool boundary = ti == 0 || ti == a.tiles_i - 1;
                        if (MULTI && a.my_flags && boundary && s > waited_s) {
                            wait_both(a.my_flags, wv + s, a.timeout_ns, a.err);
                            asm volatile("fence.proxy.async.global;" ::: "memory");
                            waited_s = s;
                        } else if (!MULTI && !waited && boundary) {
                            wait_both(a.my_flags, wv, a.timeout_ns, a.err);
                            asm volatile("fence.proxy.async.global;" ::: "memory");
                            waited = true;
                        }
                    }
                }
                info[stage] = make_int4(ti, tj, c, s);
                mbar_arrive(&ibar[stage]);  // release: the consumers read the slot after it
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                const int i0 = a.row_lo + ti * TI, j0 = tj * TJ, k0 = c * KC;
                unsigned char *sb = smem + stage * C::kStageBytes;
                uint64_t *bar = &full[stage];
                mbar_expect_tx(bar, C::kTxBytes);
                tma_load_3d(sb + C::kPdOff, (MULTI && (s & 1)) ? &tm_pd_alt : &tm_pd, bar, k0 - 2, j0, i0);
                tma_load_4d(sb + C::kVnOff, &tm_vn, bar, k0, j0, 0, i0);
                tma_load_3d(sb + C::kWnOff, &tm_wn, bar, k0, j0 + 1, i0 + 1);
                tma_load_3d(sb + C::kRhoOff, &tm_rho, bar, k0, j0 + 1, i0 + 1);
                ++n;
                if (c == c1 - 1) it = next;
            }
        }
        {  // tell the consumers there is no more work
            const int stage = (int)(n % STAGES);
            if (n >= STAGES) mbar_wait(&empty[stage], ((n / STAGES) - 1) & 1);
            info[stage] = make_int4(-1, 0, 0, 0);
            mbar_arrive(&ibar[stage]);
        }
        __threadfence();
        if (atomicAdd(&d.ticket[1], 1u) == gridDim.x - 1) {  // every CTA has taken its last item
            d.ticket[0] = 0;
            d.ticket[1] = 0;
            if (MULTI) *d.base = base + (uint64_t)(d.nsteps - 1);  // one count per tile and step but the last
            if (MULTI && PEER && a.epoch) *a.epoch = wv + d.nsteps;
        }
        return;
    }

    // ---- consumer warps: a thread owns the level pair (k, k+1) of one vertex ----
    const int kl = tid % 8, vloc = tid / 8;
    const int li = vloc / TJ, lj = vloc % TJ;
    constexpr int sPj = KC + 4, sPi = (TJ + 2) * (KC + 4);
    constexpr int sVi = 3 * (TJ + 1) * KC;
    const int kq = kl * 2;
    const int oP = (li + 1) * sPi + (lj + 1) * sPj + kq + 2;
    const int oV = (li + 1) * sVi + (lj + 1) * KC + kq;
    const int oW = (li * TJ + lj) * (KC + 2) + kq;
    const int oR = (li * TJ + lj) * KC + kq;
    const int64_t pv = pitch_of(a.K), rowstride = (int64_t)(a.cols + 2) * pv;

    int cur_ti = -1, cur_tj = -1, cur_par = -1;
    bool vvalid = false;
    int64_t cell = 0;
    int vi = 0, vj = 0;  // this thread's vertex of the current tile
    VertexState vs{0, 0, 0, 0, 0, 0, 1.0, nullptr, nullptr, 0, 0};
    uint32_t n = 0;
    for (;; ++n) {
        const int stage = (int)(n % STAGES);
        const uint32_t ph = (n / STAGES) & 1;
        mbar_wait(&ibar[stage], ph);
        const int4 inf = info[stage];
        if (inf.x < 0) break;
        const int par = MULTI ? (inf.w & 1) : 0;
        if (inf.x != cur_ti || inf.y != cur_tj) {  // a new tile: this thread's vertex state
            cur_ti = inf.x;
            cur_tj = inf.y;
            cur_par = -1;
            const int i = a.row_lo + inf.x * TI + li, j = inf.y * TJ + lj;
            vi = i;
            vj = j;
            vvalid = i < a.row_hi && j < a.cols;
            if (vvalid) {
                cell = (int64_t)(i + 1) * (a.cols + 2) + (j + 1);
                const double *S = a.signs + cell * 6;
                vs.sg0 = __ldg(S + 0);
                vs.sg1 = __ldg(S + 1);
                vs.sg2 = __ldg(S + 2);
                vs.sg3 = __ldg(S + 3);
                vs.sg4 = __ldg(S + 4);
                vs.sg5 = __ldg(S + 5);
                vs.dual = __ldg(a.dual + cell);
                vs.d_row = 0;
                vs.d_col = 0;
                if (a.flags & TSG_PERIODIC_ROWS) {
                    if (i == 0) vs.d_row = (int64_t)a.rows * rowstride;
                    else if (i == a.rows - 1) vs.d_row = -(int64_t)a.rows * rowstride;
                }
                if (a.flags & TSG_PERIODIC_COLS) {
                    if (j == 0) vs.d_col = (int64_t)a.cols * pv;
                    else if (j == a.cols - 1) vs.d_col = -(int64_t)a.cols * pv;
                }
            }
        }
        if (par != cur_par) {  // MULTI: odd steps write the other density buffer
            cur_par = par;
            vs.out = (par ? d.pd_alt : a.pd_out) + cell * pv;
            vs.peer = nullptr;
            if constexpr (PEER) {  // the neighbours' halo rows of that step's output buffer
                double *hu = par ? d.halo_up_alt : a.halo_up, *hd = par ? d.halo_down_alt : a.halo_down;
                if (vi == 0 && hu) vs.peer = hu + (int64_t)(vj + 1) * pv;
                else if (vi == a.rows - 1 && hd) vs.peer = hd + (int64_t)(vj + 1) * pv;
            }
        }
        mbar_wait(&full[stage], ph);
        if (!MULTI && a.trace && n == 0 && tid == 0) a.trace[4 * blockIdx.x + 1] = globaltimer_ns();
        const int k = inf.z * KC + kq;
        if (vvalid && k < a.K) {
            const unsigned char *sb = smem + stage * C::kStageBytes;
            level_pair_update<TJ, KC, OP, PEER>(reinterpret_cast<const double *>(sb + C::kPdOff) + oP,
                                                reinterpret_cast<const double *>(sb + C::kVnOff) + oV,
                                                reinterpret_cast<const double *>(sb + C::kWnOff) + oW,
                                                reinterpret_cast<const double *>(sb + C::kRhoOff) + oR, vs, k,
                                                a.K, a.dt, a.pivbz);
        }
        if constexpr (MULTI) {
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(&dbar[stage]);  // for the signal warp
        }
        mbar_arrive(&empty[stage]);
    }
    if (a.trace && tid == 0) {
        a.trace[4 * blockIdx.x + 2] = globaltimer_ns();
        if (!MULTI) a.trace[4 * blockIdx.x + 3] = (uint64_t)n;
    }
    if constexpr (PEER && !MULTI) {
        asm volatile("bar.sync 1, %0;" ::"r"(kConsumers) : "memory");  // consumer warps only
        if (a.done && tid == 0) {  // the last CTA out releases the step into both neighbours
            __threadfence_system();
            if (atomicAdd(a.done, 1) == (int)gridDim.x - 1) {
                *a.done = 0;
                if (a.epoch) *a.epoch = wv + 1;
                __threadfence_system();
                const int64_t v = wv + 1;
                if (a.flag_up) asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(a.flag_up), "l"(v) : "memory");
                if (a.flag_down) asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(a.flag_down), "l"(v) : "memory");
            }
        }
    }
}

// ---- host-side registry -----------------------------------------------------------------

template <int TI, int TJ, int KC, int STAGES>
static DynShape make_shape() {
    using C = FusedCfg<TI, TJ, KC, STAGES, 8, 2>;
    DynShape v;
    v.ti = TI;
    v.tj = TJ;
    v.kc = KC;
    v.stages = STAGES;
    v.threads = TI * TJ * 8 + 32;
    v.multi_threads = v.threads + 32;
    v.smem = STAGES * C::kStageBytes + STAGES * 16 + STAGES * 4 * 8;
    v.fn[0][0] = (void *)mpdata_dyn_kernel<TI, TJ, KC, STAGES, TSG_UPWIND, false, false>;
    v.fn[0][1] = (void *)mpdata_dyn_kernel<TI, TJ, KC, STAGES, TSG_CENTRED, false, false>;
    v.fn[0][2] = (void *)mpdata_dyn_kernel<TI, TJ, KC, STAGES, kProbeOp, false, false>;
    v.fn[1][0] = (void *)mpdata_dyn_kernel<TI, TJ, KC, STAGES, TSG_UPWIND, true, false>;
    v.fn[1][1] = (void *)mpdata_dyn_kernel<TI, TJ, KC, STAGES, TSG_CENTRED, true, false>;
    v.fn[1][2] = nullptr;
    v.fn[2][0] = (void *)mpdata_dyn_kernel<TI, TJ, KC, STAGES, TSG_UPWIND, false, true>;
    v.fn[2][1] = (void *)mpdata_dyn_kernel<TI, TJ, KC, STAGES, TSG_CENTRED, false, true>;
    v.fn[2][2] = nullptr;
    v.fn[3][0] = (void *)mpdata_dyn_kernel<TI, TJ, KC, STAGES, TSG_UPWIND, true, true>;
    v.fn[3][1] = (void *)mpdata_dyn_kernel<TI, TJ, KC, STAGES, TSG_CENTRED, true, true>;
    v.fn[3][2] = nullptr;
    return v;
}

// the dynamic-deal counterpart of a static variant's tile shape, or NULL
const DynShape *dyn_shape(int ti, int tj, int kc, int stages) {
    static const DynShape shapes[] = {make_shape<4, 16, 16, 3>(), make_shape<4, 12, 16, 4>()};
    for (const DynShape &s : shapes)
        if (s.ti == ti && s.tj == tj && s.kc == kc && s.stages == stages) return &s;
    return nullptr;
}

}  // namespace tsg
