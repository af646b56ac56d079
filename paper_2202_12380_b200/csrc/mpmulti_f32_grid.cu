// mpmulti_f32_grid.cu -- multi-selection loop kernel instances: float, grid (global exchange).
#include "mpmulti.cuh"

MPG_MULTI_TU(float, true, f32_grid)
