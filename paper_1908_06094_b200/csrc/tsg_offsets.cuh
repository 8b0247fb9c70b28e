// The nine structured neighbour relations (connectivity.py:36-68) as device constants.
// c_offsets[from*3 + to][source colour][slot] = {drow, target colour, dcol}; the slot
// order is the canonical order that fixes every floating-point summation order.
#pragma once
#include <stdint.h>

namespace tsg {

static __constant__ int c_colors[3] = {1, 2, 3};
// widths indexed by from*3 + to, locations 0 = V, 1 = C, 2 = E
static __constant__ int c_rel_width[9] = {6, 6, 6, 3, 3, 3, 2, 2, 4};

static __constant__ int8_t c_offsets[9][3][6][3] = {
    // V -> V
    {{{0, 0, 1}, {1, 0, 1}, {1, 0, 0}, {0, 0, -1}, {-1, 0, -1}, {-1, 0, 0}}},
    // V -> C
    {{{0, 0, 0}, {0, 1, 0}, {0, 0, -1}, {-1, 1, -1}, {-1, 0, -1}, {-1, 1, 0}}},
    // V -> E
    {{{0, 0, 0}, {0, 1, 0}, {0, 2, 0}, {0, 0, -1}, {-1, 1, -1}, {-1, 2, 0}}},
    // C -> V
    {{{0, 0, 0}, {0, 0, 1}, {1, 0, 1}}, {{0, 0, 0}, {1, 0, 0}, {1, 0, 1}}},
    // C -> C
    {{{0, 1, 0}, {-1, 1, 0}, {0, 1, 1}}, {{0, 0, 0}, {0, 0, -1}, {1, 0, 0}}},
    // C -> E
    {{{0, 0, 0}, {0, 1, 0}, {0, 2, 1}}, {{0, 2, 0}, {0, 1, 0}, {1, 0, 0}}},
    // E -> V
    {{{0, 0, 0}, {0, 0, 1}}, {{0, 0, 0}, {1, 0, 1}}, {{0, 0, 0}, {1, 0, 0}}},
    // E -> C
    {{{0, 0, 0}, {-1, 1, 0}}, {{0, 0, 0}, {0, 1, 0}}, {{0, 1, 0}, {0, 0, -1}}},
    // E -> E
    {{{0, 1, 0}, {0, 2, 1}, {-1, 2, 0}, {-1, 1, 0}},
     {{0, 0, 0}, {0, 2, 1}, {0, 2, 0}, {1, 0, 0}},
     {{0, 1, 0}, {1, 0, 0}, {0, 0, -1}, {0, 1, -1}}},
};

// the same table as a compile-time constant (for kernels templated on the relation; the
// calls fold to immediates when rel, c, s are constants)
__host__ __device__ constexpr int rel_off(int rel, int c, int s, int q) {
    constexpr int8_t t[9][3][6][3] = {
    {{{0, 0, 1}, {1, 0, 1}, {1, 0, 0}, {0, 0, -1}, {-1, 0, -1}, {-1, 0, 0}}},
    {{{0, 0, 0}, {0, 1, 0}, {0, 0, -1}, {-1, 1, -1}, {-1, 0, -1}, {-1, 1, 0}}},
    {{{0, 0, 0}, {0, 1, 0}, {0, 2, 0}, {0, 0, -1}, {-1, 1, -1}, {-1, 2, 0}}},
    {{{0, 0, 0}, {0, 0, 1}, {1, 0, 1}}, {{0, 0, 0}, {1, 0, 0}, {1, 0, 1}}},
    {{{0, 1, 0}, {-1, 1, 0}, {0, 1, 1}}, {{0, 0, 0}, {0, 0, -1}, {1, 0, 0}}},
    {{{0, 0, 0}, {0, 1, 0}, {0, 2, 1}}, {{0, 2, 0}, {0, 1, 0}, {1, 0, 0}}},
    {{{0, 0, 0}, {0, 0, 1}}, {{0, 0, 0}, {1, 0, 1}}, {{0, 0, 0}, {1, 0, 0}}},
    {{{0, 0, 0}, {-1, 1, 0}}, {{0, 0, 0}, {0, 1, 0}}, {{0, 1, 0}, {0, 0, -1}}},
    {{{0, 1, 0}, {0, 2, 1}, {-1, 2, 0}, {-1, 1, 0}},
     {{0, 0, 0}, {0, 2, 1}, {0, 2, 0}, {1, 0, 0}},
     {{0, 1, 0}, {1, 0, 0}, {0, 0, -1}, {0, 1, -1}}},
};
    return t[rel][c][s][q];
}
__host__ __device__ constexpr int rel_width(int rel) { return rel < 3 ? 6 : (rel < 6 ? 3 : (rel == 8 ? 4 : 2)); }
__host__ __device__ constexpr int loc_colors(int loc) { return loc == 0 ? 1 : (loc == 1 ? 2 : 3); }

inline int host_rel_width(int from_loc, int to_loc) {
    static const int w[9] = {6, 6, 6, 3, 3, 3, 2, 2, 4};
    return w[from_loc * 3 + to_loc];
}

}  // namespace tsg
