// mpmulti_f64_grid.cu -- multi-selection loop kernel instances: double, grid (global exchange).
#include "mpmulti.cuh"

MPG_MULTI_TU(double, true, f64_grid)
