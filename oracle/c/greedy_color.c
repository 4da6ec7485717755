/* ORACLE (test infrastructure only; see oracle/__init__.py).
 *
 * Sequential greedy graph coloring of constraints for the graph-colored
 * Gauss-Seidel sweep (BASELINE.json north_star "graph-colored Gauss-Seidel
 * constraint sweeps ... using the same deterministic color ordering";
 * PAPER.md l.72 "The constraint-based formulation can be parallelized
 * [fratarcangeli2016vivace]").
 *
 * Definition (reading R1): constraints are visited in index order;
 * constraint j receives the smallest color not already held by an earlier
 * constraint that shares a vertex with j.  Plain C, obviously correct: one
 * array of used-color bitsets per vertex (up to 256 colors).
 *
 * returns number of colors, or -1 if more than 256 colors are needed.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

int oracle_greedy_color(int64_t n_cons, int32_t arity, const int32_t *idx,
                        int64_t n_verts, int32_t *color_out) {
    uint64_t *used = (uint64_t *)calloc((size_t)n_verts * 4, sizeof(uint64_t));
    if (!used) return -1;
    int ncolors = 0;
    for (int64_t j = 0; j < n_cons; ++j) {
        uint64_t m[4] = {0, 0, 0, 0};
        for (int k = 0; k < arity; ++k) {
            int64_t v = idx[j * arity + k];
            for (int q = 0; q < 4; ++q) m[q] |= used[v * 4 + q];
        }
        int c = -1;
        for (int q = 0; q < 4 && c < 0; ++q) {
            if (m[q] != ~(uint64_t)0) {
                uint64_t free_bits = ~m[q];
                int b = 0;
                while (!((free_bits >> b) & 1u)) ++b;
                c = q * 64 + b;
            }
        }
        if (c < 0) { free(used); return -1; }
        color_out[j] = c;
        if (c + 1 > ncolors) ncolors = c + 1;
        for (int k = 0; k < arity; ++k) {
            int64_t v = idx[j * arity + k];
            used[v * 4 + c / 64] |= (uint64_t)1 << (c % 64);
        }
    }
    free(used);
    return ncolors;
}
