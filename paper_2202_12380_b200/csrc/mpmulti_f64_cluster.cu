// mpmulti_f64_cluster.cu -- multi-selection loop kernel instances: double, cluster (DSMEM exchange).
#include "mpmulti.cuh"

MPG_MULTI_TU(double, false, f64_cluster)
