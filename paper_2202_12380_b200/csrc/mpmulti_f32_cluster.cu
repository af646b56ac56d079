// mpmulti_f32_cluster.cu -- multi-selection loop kernel instances: float, cluster (DSMEM exchange).
#include "mpmulti.cuh"

MPG_MULTI_TU(float, false, f32_cluster)
