/* tsg.h -- C ABI of the B200-native MPDATA / neighbour-stencil library (libtsg.so).
 *
 * Drop-in boundary for the hot path of the reference package `tristencil`
 * (paths below are relative to /root/reference/pkg/src/tristencil).  The reference is
 * pure Python + numpy and has no FFI, so every entry point here replaces a Python
 * function; the binding a maintainer would add on the reference side (ctypes) is in
 * INTEGRATION.md.  Plain pointers and sizes only -- no torch types.
 *
 * Conventions
 *  - Every function returns an int status (TSG_OK = 0).  On failure the message is
 *    available from tsg_last_error() (thread-local), and the Python wrapper raises the
 *    reference's exception type with that message (ValueError / IndexError / ...).
 *  - Device pointers are caller-owned (the library never allocates per call); a
 *    `tsg_stream` is a cudaStream_t, every launch is stream-ordered and asynchronous.
 *  - Thread safety: calls are reentrant across grid handles; one grid handle is used by
 *    one host thread at a time (it caches the time loops' captured graph), and its fused
 *    steps and its large neighbour reductions are stream-ordered (they share the handle's
 *    work-deal counters: concurrent fused steps, or concurrent dynamically dealt reduces,
 *    on one handle from two streams need two handles).  The tuning switches
 *    (tsg_set_fused_variant / _band / _schedule, tsg_set_reduce_variant) are process-wide
 *    benchmarking hooks.
 *  - Structured ("direct") fields live in the device layout
 *        double field[rows + 2][colors][cols + 2][tsg_inner_pitch(inner)]
 *    i.e. (row, colour, column) parallelogram indexing with a one-element periodic
 *    halo ring and the level (or extra) axis innermost and contiguous, padded to an
 *    even count so every element row is 16-byte aligned for TMA / vector access (to a
 *    multiple of 16 for runs of 64 and more: 128-byte aligned, tsg_inner_pitch).
 *    Logical element (i, c, j) sits at storage row i + 1, column j + 1.
 *  - Flat ("indirect") arrays are row-major [n_elements, n_levels] in any numbering,
 *    exactly the reference oracle's convention (reference.py:1-11).
 *  - Locations: 0 = vertices (1 colour), 1 = cells (2 colours), 2 = edges (3 colours)
 *    (topology.py:27-41).
 */
#ifndef TSG_H
#define TSG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSG_ABI_VERSION 1

typedef struct tsg_grid tsg_grid; /* opaque: patch dims, halo flags, TMA descriptor cache */
typedef void *tsg_stream;         /* cudaStream_t */

enum tsg_status {
    TSG_OK = 0,
    TSG_EVALUE = 1, /* ValueError in the Python mirror */
    TSG_EINDEX = 2, /* IndexError */
    TSG_ECUDA = 3,  /* RuntimeError: CUDA / driver failure */
    TSG_ESTATE = 4  /* RuntimeError: misuse (e.g. no device) */
};

enum tsg_location { TSG_VERTICES = 0, TSG_CELLS = 1, TSG_EDGES = 2 };
enum tsg_flux_op { TSG_UPWIND = 0, TSG_CENTRED = 1 };
enum tsg_grid_flags {
    TSG_PERIODIC_ROWS = 1, /* single-GPU patch: row halo is a periodic image */
    TSG_PERIODIC_COLS = 2  /* column halo is a periodic image (always on for row strips) */
};

/* ---- errors / version ------------------------------------------------------------ */
/* No reference counterpart: the reference raises ValueError / IndexError / RuntimeError
 * directly (topology.py:58-75, connectivity.py:94-150); the Python mirror maps the
 * status codes back to those exception types with this message. */
const char *tsg_last_error(void);
int tsg_abi_version(void);

/* ---- grid handle ------------------------------------------------------------------ */
/* Replaces PatchSpec (topology.py:44-83) on the device side: rows, cols >= 2, levels >= 1.
 * `flags` = TSG_PERIODIC_ROWS | TSG_PERIODIC_COLS for one patch on one GPU; a row strip
 * of a multi-GPU decomposition passes TSG_PERIODIC_COLS only (row halos arrive by
 * exchange).  The handle binds to the current CUDA device. */
int tsg_grid_create(int rows, int cols, int levels, int flags, tsg_grid **out);
int tsg_grid_destroy(tsg_grid *g);
/* Place a row strip inside a global patch of `global_rows` rows (multi-GPU row-strip
 * decomposition): only tsg_fill_hash consults it, so synthetic inputs are identical for
 * every decomposition. */
int tsg_grid_set_origin(tsg_grid *g, int row0, int global_rows);
/* Padded innermost extent for `inner` contiguous values per element: 1 stays 1, even
 * below 64, a multiple of 16 from 64 up (every level run starts on a 128-byte line). */
int64_t tsg_inner_pitch(int inner);
/* Number of doubles of a structured field: (rows+2) * colors * (cols+2) * pitch(inner). */
int64_t tsg_field_elems(const tsg_grid *g, int loc, int inner);

/* ---- field layout: Atlas/flat <-> structured reorder, halo ----------------------- */
/* Periodic one-ring halo refresh (executors.py:74-86), honouring the grid flags. */
int tsg_halo_update(const tsg_grid *g, int loc, int inner, double *field, tsg_stream s);
/* flat[rank, 0..inner) -> structured field (halo images written).  `forward` maps the
 * canonical id (i*colors + c)*cols + j to the flat row (layouts.Permutation.forward,
 * layouts.py:153-180); NULL = structured numbering (identity).  Replaces
 * flat_to_field (kernels.py:120-127) + halo_update. */
int tsg_pack(const tsg_grid *g, int loc, int inner, const double *flat, const int64_t *forward,
             double *field, tsg_stream s);
/* structured field -> flat[rank, 0..inner); replaces field_to_flat (kernels.py:107-117). */
int tsg_unpack(const tsg_grid *g, int loc, int inner, const double *field,
               const int64_t *forward, double *flat, tsg_stream s);

/* Host `LinearLayout` buffer (layouts.py:55-104, copied to device memory as is) <->
 * structured field.  layout6 (host memory) = {front_pad, stride_row, stride_color,
 * stride_column, stride_level, stride_extra} in elements; the buffer carries a halo of
 * width host_halo.  `inner` runs along level when stride_level != 0, else along extra.
 * Unpack writes every host halo cell as the periodic image of the interior. */
int tsg_pack_strided(const tsg_grid *g, int loc, int inner, const double *src,
                     const int64_t *layout6, int host_halo, double *field, tsg_stream s);
int tsg_unpack_strided(const tsg_grid *g, int loc, int inner, const double *field,
                       const int64_t *layout6, int host_halo, double *dst, tsg_stream s);
/* The same for a band of rows, so a host field can be streamed through the step band by
 * band (executors.run_fused on host Fields): pack logical rows [row_lo, row_hi) (with
 * their halo images), unpack host storage rows [srow_lo, srow_hi) of 0 .. rows + 2h. */
int tsg_pack_strided_rows(const tsg_grid *g, int loc, int inner, const double *src,
                          const int64_t *layout6, int host_halo, int row_lo, int row_hi,
                          double *field, tsg_stream s);
int tsg_unpack_strided_rows(const tsg_grid *g, int loc, int inner, const double *field,
                            const int64_t *layout6, int host_halo, int srow_lo, int srow_hi,
                            double *dst, tsg_stream s);
/* cudaMemcpy2DAsync of `height` rows of `width` bytes (kind 1 = H2D, 2 = D2H): one band
 * of storage rows of a level-outer host layout per call. */
int tsg_memcpy2d(void *dst, int64_t dpitch, const void *src, int64_t spitch, int64_t width,
                 int64_t height, int kind, tsg_stream s);

/* ---- MPDATA transport step (mpdata.py:189-354; reference.py:93-116) ---------------- */
/* Fused single-pass step: flux -> fluz -> divergence -> advance with every intermediate
 * kept on chip (the run_fused executor, executors.py:266-316).  Writes pd_out with its
 * halo images.  pd, rho, pd_out: vertex fields, inner = levels; vn: edge field,
 * inner = levels; wn: vertex field, inner = levels + 1 (staggered); signs: vertex field,
 * inner = 6 (edge_signs, connectivity.py:184-194); dual: vertex field, inner = 1.
 * Input halos must be valid (tsg_pack / tsg_halo_update / a previous step). */
int tsg_mpdata_step(tsg_grid *g, const double *pd, const double *vn, const double *wn,
                    const double *rho, const double *signs, const double *dual, double *pd_out,
                    double dt, double pivbz, int flux_op, tsg_stream s);
/* flux_op = 99 runs the fused kernel's data-movement probe (TMA pipeline and stores
 * only, no arithmetic) and flux_op = 98 its compute probe (arithmetic on shared memory
 * that is never loaded) -- benchmarking aids for the memory and compute ceilings.
 * Same step restricted to logical rows [row_lo, row_hi) -- lets a row strip compute its
 * interior while its halo rows are still in flight, then its two boundary rows. */
int tsg_mpdata_step_rows(tsg_grid *g, const double *pd, const double *vn, const double *wn,
                         const double *rho, const double *signs, const double *dual,
                         double *pd_out, double dt, double pivbz, int flux_op, int row_lo,
                         int row_hi, tsg_stream s);
/* Row-strip step with the halo exchange fused into the epilogue: this strip's first row
 * is also stored into `halo_up` (the up neighbour's bottom halo row, a full storage row
 * of (cols+2)*pitch(levels) doubles) and its last row into `halo_down` (the down
 * neighbour's top halo row), column images included -- P2P stores over NVLink when the
 * pointers are peer / IPC mappings (tsg_ipc_open).  NULL pointers skip that side. */
int tsg_mpdata_step_rows_peer(tsg_grid *g, const double *pd, const double *vn, const double *wn,
                              const double *rho, const double *signs, const double *dual,
                              double *pd_out, double dt, double pivbz, int flux_op, int row_lo,
                              int row_hi, double *halo_up, double *halo_down, tsg_stream s);
/* One whole row-strip step in ONE launch, halo exchange and step fence included (the
 * multi-GPU form of the reference's step + periodic halo_update, executors.py:74-86 /
 * mpdata.py:319-354; the reference replaces MPI by an in-process copy): the
 * tile rows touching the strip's first / last row run last; before loading them the
 * kernel acquires `my_flags[0..1] >= step` (both ring neighbours finished step-1, so its
 * halo rows are complete and their pd_out halo rows are free), their epilogue stores the
 * boundary rows into `halo_up` / `halo_down` as tsg_mpdata_step_rows_peer does, and the
 * last CTA to finish (counted in the caller's zero-initialised `done_counter`, reset by
 * the kernel) releases step+1 into `flag_up` (the up neighbour's flag word 1) and
 * `flag_down` (the down neighbour's word 0).  A neighbour missing for `timeout_ms` sets
 * `*error_word` instead of hanging.  Grid flags must not include TSG_PERIODIC_ROWS. */
int tsg_mpdata_step_strip(tsg_grid *g, const double *pd, const double *vn, const double *wn,
                          const double *rho, const double *signs, const double *dual,
                          double *pd_out, double dt, double pivbz, int flux_op, double *halo_up,
                          double *halo_down, const int64_t *my_flags, int64_t *flag_up,
                          int64_t *flag_down, int64_t step, int64_t *epoch, int timeout_ms,
                          int *error_word, int *done_counter, tsg_stream s);
/* `epoch` (optional, device memory): when non-NULL the step number is read from it at
 * the start of the launch and advanced by the launch's last CTA, so a loop of strip steps
 * needs no per-step argument; `step` is then ignored.  tsg_mpdata_run_strip runs `nsteps`
 * such steps ping-ponging pd_a / pd_b (halo_*_a: the neighbours' halo rows in their b
 * buffer, written while stepping a -> b; halo_*_b likewise for b -> a) as a captured
 * two-step CUDA graph (cached on the grid handle), halo exchange and fences included. */
/* Number of time-loop graphs instantiated so far in this process (a diagnostic: a loop
 * that alternates between the same two buffers reuses one graph). */
int tsg_time_loop_graphs_built(void);
/* Prepared-launch cache of a grid handle (the tensor maps, arguments and grid size of a
 * fused step, keyed by all of its arguments): hits / misses so far.  A diagnostic; a
 * repeated step with the same buffers encodes nothing. */
int tsg_launch_cache_stats(const tsg_grid *g, int64_t *hits, int64_t *misses);
/* Debug trace of the fused kernel (no reference counterpart; a measurement aid): fused
 * launches prepared while set write, per CTA b, per_cta4[4b .. 4b+3] = {globaltimer ns at
 * entry, when its first stage landed, when its unit loop ended, units run}.  NULL = off. */
int tsg_debug_trace(uint64_t *per_cta4);
int tsg_mpdata_run_strip(tsg_grid *g, double *pd_a, double *pd_b, const double *vn,
                         const double *wn, const double *rho, const double *signs,
                         const double *dual, double dt, double pivbz, int flux_op,
                         double *halo_up_a, double *halo_down_a, double *halo_up_b,
                         double *halo_down_b, const int64_t *my_flags, int64_t *flag_up,
                         int64_t *flag_down, int64_t *epoch, int timeout_ms, int *error_word,
                         int *done_counter, int nsteps, tsg_stream s);
/* The reference's time loop (bench.py:398-403: step, copy pd_out -> pd_in, repeat) as a
 * device ping-pong: step t reads pd_a and writes pd_b when t is even, the reverse when
 * odd, so after nsteps the newest density is in pd_b (nsteps odd) or pd_a (even) and the
 * other buffer holds the state before the last step.  vn / wn / rho / signs / dual are
 * fixed over the loop, as in the reference; the tensor maps are encoded once, and from 4
 * steps on the two alternating launches are replayed as a captured CUDA graph (cached on
 * the grid handle until the arguments change). */
int tsg_mpdata_run(tsg_grid *g, double *pd_a, double *pd_b, const double *vn, const double *wn,
                   const double *rho, const double *signs, const double *dual, double dt,
                   double pivbz, int flux_op, int nsteps, tsg_stream s);
/* Four-kernel step materialising flux (edges), fluz (vertices, levels+1) and divvd
 * (vertices) like run_naive (executors.py:213-245), halos refreshed after each stage. */
int tsg_mpdata_step_unfused(const tsg_grid *g, const double *pd, const double *vn,
                            const double *wn, const double *rho, const double *signs,
                            const double *dual, double *flux, double *fluz, double *divvd,
                            double *pd_out, double dt, double pivbz, int flux_op, tsg_stream s);
/* Table-driven ("indirect", Atlas-style) step over flat arrays -- the exact signature
 * of reference.transport_step (reference.py:93-116): e2v [ne,2], v2e [nv,6] int64 ranks,
 * signs [nv,6], dual [nv], pd/rho/div/pd_out [nv,nlev], vn/flux [ne,nlev],
 * wn/fluz [nv,nlev+1].  Any numbering. */
int tsg_transport_indirect(const int64_t *e2v, const int64_t *v2e, const double *signs,
                           const double *dual, const double *pd, const double *vn,
                           const double *wn, const double *rho, int64_t nv, int64_t ne,
                           int nlev, double dt, double pivbz, int flux_op, double *flux,
                           double *fluz, double *div, double *pd_out, tsg_stream s);
/* The reference's flat stages one at a time (reference.py:18-90, 119-134; the per-stage
 * functions beside transport_step), any numbering, row-major [element, level] arrays:
 *   tsg_flat_flux             upwind_flux / centred_flux: e2v [ne,2] -> flux [ne,nlev]
 *   tsg_flat_fluz             upwind_fluz: pd [nv,nlev], wn [nv,nlev+1] -> fluz [nv,nlev+1]
 *                             (TSG_EVALUE below 2 levels, as the reference's ValueError)
 *   tsg_flat_divergence       flux_divergence: v2e / signs [nv,width], dual [nv] -> div
 *   tsg_flat_advance          advance_density over n = nv*nlev values
 *   tsg_flat_cell_divergence  cell_divergence: c2e [nc,width], vn [ne,nlev], length [ne],
 *                             area [nc] -> out [nc,nlev]
 * Table ids are not bounds-checked here (the Python mirror checks them). */
int tsg_flat_flux(const int64_t *e2v, const double *pd, const double *vn, int64_t ne, int nlev,
                  int flux_op, double *flux, tsg_stream s);
int tsg_flat_fluz(const double *pd, const double *wn, int64_t nv, int nlev, double pivbz,
                  double *fluz, tsg_stream s);
int tsg_flat_divergence(const int64_t *v2e, int width, const double *signs, const double *dual,
                        const double *flux, const double *fluz, int64_t nv, int nlev, double *div,
                        tsg_stream s);
int tsg_flat_advance(const double *pd, const double *div, const double *rho, int64_t n, double dt,
                     double *pd_out, tsg_stream s);
int tsg_flat_cell_divergence(const int64_t *c2e, int width, const double *vn, const double *length,
                             const double *area, int64_t nc, int nlev, double *out, tsg_stream s);
/* Select the fused kernel's tile variant; 0 (the default) chooses per launch: the compact
 * 4x16 level-pair tile with a producer warp (variant 21: 512 compute threads + 32) when
 * the tile above a tile is still in L2 under the contiguous schedule or the band schedule
 * applies, else the tall 16x4 tile (tsg_fused_variant_of).  Variant 0 in _info = the
 * forced variant, or the compact tile when none is forced; `threads` counts the producer
 * warp. */
int tsg_set_fused_variant(int variant);
/* Benchmarking hook: force an alternative compact tile shape of the TMA neighbour reduce's
 * plain sum fold and of the cell divergence (1-9 static ranges, 11-19 the same shapes
 * dynamically dealt); 0 (the default) = the measured per-source-location shape and
 * schedule. */
int tsg_set_reduce_variant(int variant);
/* Testing hook: the number of points (elements x levels) one launch of the point-indexed
 * kernels (reorders, synthetic fill, the unfused step's level-pair items) covers before
 * the field is split into row bands; 0 restores the default 2^32 - 2^24.  Process-wide.
 * No reference counterpart. */
int tsg_set_point_limit(int64_t n);
int tsg_fused_variant_info(int variant, int *ti, int *tj, int *kc, int *stages, int *threads,
                           int *smem_bytes);
/* The variant a fused launch over logical rows [row_lo, row_hi) of `g` uses (-1 on error). */
int tsg_fused_variant_of(const tsg_grid *g, int row_lo, int row_hi);
/* Whether that launch (single-GPU, no peer rows) deals whole tiles round robin in
 * band-major order (1) or walks contiguous ranges (0): the band schedule replaces the tall
 * tile when the tile above would be evicted from L2 and every CTA gets >= 16 tiles. */
int tsg_fused_band_of(const tsg_grid *g, int row_lo, int row_hi);
/* Enable (1, default) or disable (0) that band schedule. */
int tsg_set_fused_band(int on);
/* Scheduling of the fused launches: 0 (the default) deals the units of the producer-warp
 * level-pair variants dynamically (a global ticket: whole tiles, the tail unit by unit)
 * and runs tsg_mpdata_run's loop as persistent multi-step launches with per-tile step
 * counters; 1 = the static per-CTA ranges / band deal and the captured two-step graph.
 * A benchmarking hook like the two above.  No reference counterpart (executors.py:266-316
 * deals tiles to a thread pool). */
int tsg_set_fused_schedule(int sched);
/* Reads and clears the grid's dependency-wait error word: 2 when a persistent multi-step
 * launch timed out waiting for a neighbour tile (results of that launch are invalid). */
int tsg_fused_wait_error(tsg_grid *g, int *err);
/* Kernel launches tsg_mpdata_run (or tsg_mpdata_run_strip, on a strip grid) issues for
 * `nsteps` steps under the current switches: 1 per 2^30 / units steps for the persistent
 * loop, else one per step; -1 on error.  A benchmarking aid, no reference counterpart. */
int tsg_fused_loop_launches(const tsg_grid *g, int nsteps);

/* ---- neighbour reductions (stencil.py:401-408; kernels.py:27-104; reference.py:137-157) */
/* Structured ("direct") reduce for any of the 9 relations (connectivity.py:36-68):
 * dst[from, k] = ((0 + src[n0,k]) + src[n1,k]) + ...  (canonical slot order), times
 * scale[from] if scale != NULL (a 2-D from-located field, inner = 1).  src lives on
 * to_loc, dst on from_loc, both with `inner` levels; dst halo images are written. */
int tsg_neighbor_reduce(const tsg_grid *g, int from_loc, int to_loc, int inner,
                        const double *src, const double *scale, double *dst, tsg_stream s);
/* Table-driven reduce over flat arrays (Table 1 "indirect access"): table [nrows,width]
 * int64 ranks into src [*, nlev]; scale [nrows] or NULL; dst [nrows, nlev]. */
int tsg_neighbor_reduce_indirect(const int64_t *table, int64_t nrows, int width, int nlev,
                                 const double *src, const double *scale, double *dst,
                                 tsg_stream s);
/* Cell divergence demo (mpdata.py:361-416; reference.py:119-134): weighted = 0 computes
 * (sum vn*length)/area, weighted = 1 computes sum vn*weights[c,n]. vn: edges, inner
 * levels; length: edges inner 1; area: cells inner 1; weights: cells inner 3. */
int tsg_cell_divergence(const tsg_grid *g, int weighted, const double *vn,
                        const double *length, const double *area, const double *weights,
                        double *out, tsg_stream s);

/* Per-cell edge weights w[c, n] = length(e_n) / area(c) in C->E slot order
 * (precompute_weights, mpdata.py:152-169): length edges inner 1, area cells inner 1,
 * weights cells inner 3. */
int tsg_cell_weights(const tsg_grid *g, const double *length, const double *area,
                     double *weights, tsg_stream s);

/* ---- index maps on the device (connectivity.py:130-194) ---------------------------- */
/* Flat int64 neighbour table [n_from, width] under optional numberings:
 * from_inverse: rank -> canonical id of the from-location (NULL = identity);
 * to_forward:   canonical id -> rank of the to-location (NULL = identity). */
int tsg_build_neighbor_table(int rows, int cols, int from_loc, int to_loc,
                             const int64_t *from_inverse, const int64_t *to_forward,
                             int64_t *out, tsg_stream s);
/* Forward permutation (canonical id -> rank) of a numbering (layouts.py:250-279):
 * numbering 0 = sn (identity), 1 = un ((i*cols + j)*colors + c), 2 = hn (Hilbert walk
 * over the quad embedding, vertices and cells only).  hn needs `work` with
 * tsg_permutation_work_elems() int64 entries (may be NULL otherwise). */
int tsg_make_permutation(int rows, int cols, int loc, int numbering, int64_t *forward,
                         int64_t *work, tsg_stream s);
int64_t tsg_permutation_work_elems(int rows, int cols, int loc);
/* Orientation signs [n_vertices, 6] in canonical order (connectivity.py:184-194). */
int tsg_edge_signs(int rows, int cols, double *out, tsg_stream s);

/* ---- cross-GPU plumbing for the fused exchange (one process per GPU) ------------------ */
/* No reference counterpart: the reference is single-process (SPEC.md:8 names MPI halo
 * exchange as the multi-node path); these replace it with NVLink P2P stores and flags. */
/* Device memory outside any caching allocator (IPC handles need whole allocations). */
int tsg_malloc(int64_t bytes, void **out);
int tsg_free(void *ptr);
/* CUDA IPC: export an allocation (64-byte handle) / map a peer's allocation. */
int tsg_ipc_handle(void *ptr, unsigned char *handle64);
int tsg_ipc_open(const unsigned char *handle64, void **out);
int tsg_ipc_close(void *ptr);
/* Step fence between neighbours: after a step, store `value` into both neighbours' flag
 * words (system-scope release); before the next step's boundary rows, wait until this
 * rank's two flag words reach `value` (spin with back-off; gives up after `timeout_ms` and
 * reports TSG_ECUDA through the error word so a lost peer cannot hang the GPU). */
int tsg_signal_peers(int64_t *flag_up, int64_t *flag_down, int64_t value, tsg_stream s);
int tsg_wait_flags(const int64_t *my_flags, int64_t value, int timeout_ms, int *error_word,
                   tsg_stream s);

/* ---- diagnostics / synthetic inputs ----------------------------------------------- */
/* sum_v sum_k pd[v,k] * dual[v] (mpdata.py:496-500), deterministic two-pass reduction;
 * `work` holds >= 1024 doubles; the result is written to device memory `out`. */
int tsg_total_mass(const tsg_grid *g, const double *pd, const double *dual, double *work,
                   double *out, tsg_stream s);
/* Counter-hash uniform values in [lo, hi) for every (element, level), halo images
 * included -- on-device synthetic inputs for patches the host cannot hold (the reference
 * draws its inputs with numpy, mpdata.py:51-182, which cfg5 / O1280 does not fit). */
int tsg_fill_hash(const tsg_grid *g, int loc, int inner, uint64_t seed, double lo, double hi,
                  double *field, tsg_stream s);

#ifdef __cplusplus
}
#endif
#endif /* TSG_H */
