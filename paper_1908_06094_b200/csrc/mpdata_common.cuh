// Device-side building blocks shared by the fused MPDATA kernels (mpdata_fused.cu: the
// static-schedule kernel and the host side; mpdata_dyn.cu: the dynamically scheduled and
// the persistent multi-step kernels): tile geometry, launch arguments, the band order of
// tiles, the cross-GPU flag waits, and the level-pair update of one vertex (SURVEY
// Appendix A, reference.py:18-90).
#pragma once

#include "tsg_tma.cuh"

namespace tsg {

// streaming (evict-first) 16-byte store: the step's output is not re-read by this launch
__device__ __forceinline__ void stcs2(double *p, double2 v) { __stcs(reinterpret_cast<double2 *>(p), v); }

// ---- tile geometry --------------------------------------------------------------------

template <int TI, int TJ, int KC, int STAGES, int LV, int LP = 1>
struct FusedCfg {
    static constexpr int kThreads = TI * TJ * LV;                  // LV lanes per vertex
    static constexpr int kLevelsPerThread = (KC + LV - 1) / LV;  // last pass may be partial
    static constexpr int kPdBytes = (TI + 2) * (TJ + 2) * (KC + 4) * 8;
    static constexpr int kVnBytes = (TI + 1) * 3 * (TJ + 1) * KC * 8;
    static constexpr int kWnBytes = TI * TJ * (KC + 2) * 8;
    static constexpr int kRhoBytes = TI * TJ * KC * 8;
    static constexpr int align(int b) { return (b + 127) / 128 * 128; }
    static constexpr int kPdOff = 0;
    static constexpr int kVnOff = kPdOff + align(kPdBytes);
    static constexpr int kWnOff = kVnOff + align(kVnBytes);
    static constexpr int kRhoOff = kWnOff + align(kWnBytes);
    static constexpr int kStageBytes = kRhoOff + align(kRhoBytes);
    static constexpr uint32_t kTxBytes = kPdBytes + kVnBytes + kWnBytes + kRhoBytes;
    static constexpr int kSmemBytes = STAGES * kStageBytes + 128;  // + barriers
    static_assert(KC % 16 == 0, "KC must be a multiple of 16");
    static_assert((LP == 1 && (LV == 16 || LV == 32)) || (LP == 2 && LV * 2 == KC),
                  "a half-warp or a warp per vertex, or level pairs covering the chunk");
    static_assert(((KC + 2) * 8) % 16 == 0 && (KC * 8) % 16 == 0, "TMA inner box must be 16B multiple");
    static_assert(TI + 2 <= 256 && TJ + 2 <= 256 && KC + 4 <= 256, "TMA box <= 256");
};

// flux_op value of the data-movement probe (benchmarking the TMA pipeline alone)
constexpr int kProbeOp = 99;
// flux_op value of the compute probe (arithmetic on unloaded shared memory, no TMA)
constexpr int kComputeProbe = 98;
// flux_op values of the load probes (attribution of DRAM traffic and time per field): the
// TMA pipeline with only pd (90), vn (91), wn (92) or rho (93) loaded, or all four (94),
// and no arithmetic and no stores
constexpr int kLoadProbe = 90, kLoadProbeAll = 94;
template <int OP> __host__ __device__ constexpr bool is_load_probe() { return OP >= kLoadProbe && OP <= kLoadProbeAll; }
template <int OP> __host__ __device__ constexpr bool loads_field(int f) {
    return !is_load_probe<OP>() || OP == kLoadProbeAll || OP == kLoadProbe + f;
}

struct FusedArgs {
    const double *signs;  // vertex field, inner 6
    const double *dual;   // vertex field, inner 1
    double *pd_out;       // vertex field, inner K
    int rows, cols, K;
    int row_lo, row_hi;  // rows computed by this launch: [row_lo, row_hi)
    int flags;
    // fused halo exchange: the ring neighbours' halo rows (peer / IPC-mapped memory) that
    // receive this strip's first / last row; NULL = not exchanged by this kernel
    double *halo_up, *halo_down;
    // single-launch strip step (tsg_mpdata_step_strip; PEER instantiation only): the tile
    // rows touching the strip's first / last row run last (`rotate`), their producer
    // first acquires my_flags >= wait_value (both neighbours finished the previous step),
    // and the last CTA to finish releases wait_value + 1 into the neighbours' flag words
    const int64_t *my_flags;
    int64_t *flag_up, *flag_down;
    int64_t wait_value;
    int64_t *epoch;  // non-NULL: the step counter lives here (read at start, advanced by
                     // the last CTA) -- launches then take no per-step argument (CUDA graphs)
    uint64_t timeout_ns;
    int *err, *done;
    int rotate;
    double dt, pivbz;
    int tiles_i, tiles_j, chunks;
    int64_t units;
    // debug trace (tsg_debug_trace): per CTA {entry, first stage landed, loop end, units}
    // in globaltimer ns, or NULL
    uint64_t *trace;
};

// BAND schedule (large patches, single-GPU launches): whole tiles dealt round robin in
// band-major order (bands of band_w tile columns, tile rows within a band), each CTA
// running all chunks of its tile back to back (the per-tile state stays in registers).
// The tiles in flight at any time are ~G consecutive tiles of that order, so the tile
// above a tile (band_w tiles earlier) is loaded at the same time by another CTA and the
// halo rows they share are read from DRAM once.  A separate kernel parameter: the
// contiguous instantiations compile exactly as without it.
// A row strip (PEER launches) bands its interior tile rows 1 .. T-2 only and deals the two
// boundary tile rows last (row T-1, then row 0), so only the final tiles wait for the
// neighbours' step flags.
struct BandArgs {
    int band_w, nb_full;
    uint32_t full_tiles;
    FastDiv fd_band_tiles, fd_bw, fd_bw_last;
    int row_base, tiles_i, tiles_j;  // first banded tile row; the launch's tile grid
    uint32_t banded;                 // tiles in the band order (the rest: boundary rows)
};

__device__ __forceinline__ void band_tile(uint32_t t, const BandArgs &b, int &ti, int &tj) {
    if (t >= b.banded) {  // the boundary tile rows of a strip
        const int r = (int)(t - b.banded);
        ti = r < b.tiles_j ? b.tiles_i - 1 : 0;
        tj = r < b.tiles_j ? r : r - b.tiles_j;
    } else if (t < b.full_tiles) {
        const uint32_t band = b.fd_band_tiles.div(t), r = t - band * b.fd_band_tiles.d;
        const uint32_t row = b.fd_bw.div(r);
        ti = b.row_base + (int)row;
        tj = (int)(band * b.band_w + (r - row * b.fd_bw.d));
    } else {
        const uint32_t r = t - b.full_tiles, row = b.fd_bw_last.div(r);
        ti = b.row_base + (int)row;
        tj = b.nb_full * b.band_w + (int)(r - row * b.fd_bw_last.d);
    }
}

__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t *p) {
    int64_t v;
    asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// spin (with back-off) until both flag words reach `value`; on timeout report through `err`
// and carry on, so a lost neighbour cannot hang the GPU
__device__ inline void wait_both(const int64_t *flags, int64_t value, uint64_t timeout_ns, int *err) {
    const uint64_t t0 = globaltimer_ns();
    unsigned backoff = 32;
    while (ld_acquire_sys(flags) < value || ld_acquire_sys(flags + 1) < value) {
        if (globaltimer_ns() - t0 > timeout_ns) {
            if (err) atomicExch(err, 1);
            return;
        }
        __nanosleep(backoff);
        if (backoff < 4096) backoff *= 2;
    }
}

// ---- dynamically dealt launches (mpdata_dyn.cu) ------------------------------------------
struct DynArgs {
    uint32_t *ticket;       // [0] items taken, [1] producers done (the last resets both)
    uint64_t *tile_done;    // MULTI: consumer-warp unit completions per tile (row-major)
    uint64_t *base;         // MULTI: every tile's count before this launch
    double *pd_alt;         // MULTI: output of the odd steps (the even steps' input buffer)
    int *err;               // MULTI: set to 2 when a dependency wait times out
    uint64_t timeout_ns;
    int nsteps;             // steps in this launch (1 unless MULTI)
    uint32_t tiles;         // tiles per step
    uint32_t whole;         // last step: tiles [0, whole) of the order dealt whole
    uint32_t items;         // items of the launch
    FastDiv fd_tiles, fd_chunks;
    // MULTI + PEER (a row strip's persistent loop): the neighbours' halo rows written by the
    // odd steps (FusedArgs::halo_up / _down: by the even steps), the per-step-parity count
    // of finished boundary units, and how many units the boundary tile rows hold
    double *halo_up_alt, *halo_down_alt;
    int *bdone;
    int nb_units;
};

// A tile shape of the dynamically dealt kernel: fn[kind][op], kind 0 = one step, 1 = one
// row-strip step with the fused halo exchange (PEER), 2 = the persistent multi-step loop,
// 3 = the persistent loop of a row strip (multi-step + fused exchange); op 0 = upwind,
// 1 = centred, 2 = the data-movement probe (kind 0 only).
struct DynShape {
    int ti, tj, kc, stages, threads, smem;
    int multi_threads;  // the multi-step kernels add a signal warp
    void *fn[4][3];
};
const DynShape *dyn_shape(int ti, int tj, int kc, int stages);

// Per-thread state of one vertex of the current tile (refreshed when the tile changes).
struct VertexState {
    double sg0, sg1, sg2, sg3, sg4, sg5;  // edge signs in V->E slot order
    double dual;                          // dual volume
    double *out;                          // pd_out + cell * pitch
    double *peer;                         // PEER: the neighbour's halo-row element, or NULL
    int64_t d_row, d_col;                 // offsets of the periodic halo images (0 = none)
};

// The level pair (k, k+1) of one vertex from a landed stage: the six incident edge fluxes
// of both levels recomputed from shared memory (both endpoints compute every edge flux,
// bitwise identical), the interface fluxes k, k+1, k+2 (k+1 shared by the pair), the
// signed divergences and the updates; the pd_out pair is stored with one 16-byte store
// plus its periodic halo images and, for a row strip, the neighbour's halo row.
// P, V, W, R point at this thread's element of the stage's pd / vn / wn / rho boxes:
//   pd  [TI+2][TJ+2][KC+4]  (origin i0-1, j0-1, k0-2)    vn [TI+1][3][TJ+1][KC]
//   wn  [TI][TJ][KC+2]                                    rho [TI][TJ][KC]
// Arithmetic: SURVEY Appendix A (reference.py:18-90), explicitly rounded, canonical slot
// order from 0.0, true IEEE division, numpy maximum / minimum semantics.
template <int TJ, int KC, int OP, bool PEER>
__device__ __forceinline__ void level_pair_update(const double *P, const double *V, const double *W,
                                                  const double *R, const VertexState &s, int k, int K,
                                                  double dt, double pivbz) {
    constexpr int sPj = KC + 4, sPi = (TJ + 2) * (KC + 4);
    constexpr int sVc = (TJ + 1) * KC, sVi = 3 * (TJ + 1) * KC;
    const double2 c = ld2(P);
    if constexpr (OP == kProbeOp) {  // data-movement probe: touch the stage, skip the arithmetic
        const double2 v0 = ld2(V), w01 = ld2(W), r = ld2(R);
        st2(s.out + k, make_double2(add(add(c.x, v0.x), add(w01.x, r.x)), add(add(c.y, v0.y), add(w01.y, r.y))));
        return;
    }
    // the six incident edges in V->E slot order (connectivity.py:66); the origin is E->V
    // slot 0 (connectivity.py:38-42)
    const double2 q0 = ld2(P + sPj), q1 = ld2(P + sPi + sPj), q2 = ld2(P + sPi);
    const double2 q3 = ld2(P - sPj), q4 = ld2(P - sPi - sPj), q5 = ld2(P - sPi);
    const double2 v0 = ld2(V), v1 = ld2(V + sVc), v2 = ld2(V + 2 * sVc);
    const double2 v3 = ld2(V - KC), v4 = ld2(V - sVi + sVc - KC), v5 = ld2(V - sVi + 2 * sVc);
    const double pm = P[-1], pp = P[2];
    const double2 w01 = ld2(W);
    const double w2 = W[2];
    const double2 r = ld2(R);
    // interfaces k, k+1, k+2 (reference.py:38-60); k+1 is shared by the pair
    double z0 = fluz_interior(w01.x, pm, c.x);
    const double z1 = fluz_interior(w01.y, c.x, c.y);
    double z2 = fluz_interior(w2, c.y, pp);
    if (k == 0) z0 = mul(pivbz, z1);
    const bool pair = k + 1 < K;
    if (k + 1 == K - 1) z2 = mul(pivbz, z1);
    const double z1a = pair ? z1 : mul(pivbz, z0);  // k is the top level
    // signed divergence (reference.py:63-79), canonical slot order from 0.0
    double acc = 0.0, acd = 0.0;
    acc = add(mul(s.sg0, edge_flux<OP>(c.x, q0.x, v0.x)), acc);
    acd = add(mul(s.sg0, edge_flux<OP>(c.y, q0.y, v0.y)), acd);
    acc = add(mul(s.sg1, edge_flux<OP>(c.x, q1.x, v1.x)), acc);
    acd = add(mul(s.sg1, edge_flux<OP>(c.y, q1.y, v1.y)), acd);
    acc = add(mul(s.sg2, edge_flux<OP>(c.x, q2.x, v2.x)), acc);
    acd = add(mul(s.sg2, edge_flux<OP>(c.y, q2.y, v2.y)), acd);
    acc = add(mul(s.sg3, edge_flux<OP>(q3.x, c.x, v3.x)), acc);
    acd = add(mul(s.sg3, edge_flux<OP>(q3.y, c.y, v3.y)), acd);
    acc = add(mul(s.sg4, edge_flux<OP>(q4.x, c.x, v4.x)), acc);
    acd = add(mul(s.sg4, edge_flux<OP>(q4.y, c.y, v4.y)), acd);
    acc = add(mul(s.sg5, edge_flux<OP>(q5.x, c.x, v5.x)), acc);
    acd = add(mul(s.sg5, edge_flux<OP>(q5.y, c.y, v5.y)), acd);
    acc = add(acc, sub(z1a, z0));
    acd = add(acd, sub(z2, z1));
    // explicit update (reference.py:82-90)
    double2 val;
    val.x = sub(c.x, dvd(mul(dt, dvd(acc, s.dual)), r.x));
    val.y = sub(c.y, dvd(mul(dt, dvd(acd, s.dual)), r.y));
    double *o = s.out + k;
    const int64_t d_row = s.d_row, d_col = s.d_col;
    if (pair) {
        stcs2(o, val);
        if (d_row | d_col) {
            if (d_row) stcs2(o + d_row, val);
            if (d_col) stcs2(o + d_col, val);
            if (d_row && d_col) stcs2(o + d_row + d_col, val);
        }
        if (PEER && s.peer) {
            st2(s.peer + k, val);
            if (d_col) st2(s.peer + k + d_col, val);
        }
    } else {
        o[0] = val.x;
        if (d_row | d_col) {
            if (d_row) o[d_row] = val.x;
            if (d_col) o[d_col] = val.x;
            if (d_row && d_col) o[d_row + d_col] = val.x;
        }
        if (PEER && s.peer) {
            s.peer[k] = val.x;
            if (d_col) s.peer[k + d_col] = val.x;
        }
    }
}

}  // namespace tsg
