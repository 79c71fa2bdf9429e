// ref_shapes.cuh -- launch shapes of the reference kernels (k_ref.cuh), needed by the
// workspace layout (partial-sum buffer size) in every translation unit.
#pragma once
namespace ref {

constexpr int BX = 32, BY = 8, ZC = 16;   // stencil tile and z-chunk per CTA
constexpr int EW_THREADS = 256;

// Neumann faces (R27): m = bits of the x/y faces (1 x-, 2 x+, 4 y-, 8 y+) that mirror;
// zlo / zhi = slab plane whose z- / z+ neighbour is the mirror (-1 = none on this rank).
struct MirrorBc {
    int m, zlo, zhi;
};

struct Grid {
    int nx, ny, L;     // local extents (L = planes of this rank)
    int Lb;            // preconditioner block thickness (L / blocks_per_rank)
    double h2inv;
    MirrorBc bc;
};

}  // namespace ref
