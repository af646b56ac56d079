// mpmulti.cu -- public entry points of the exact multi-selection loop (kernel: mpmulti.cuh;
// instances: mpmulti_{f64,f32}_{cluster,grid}.cu).
#include "mpmulti.cuh"

cudaError_t launch_multi_f64_cluster(const LoopParams& P, int threads, cudaStream_t st);
cudaError_t launch_multi_f64_grid(const LoopParams& P, int threads, cudaStream_t st);
cudaError_t launch_multi_f32_cluster(const LoopParams& P, int threads, cudaStream_t st);
cudaError_t launch_multi_f32_grid(const LoopParams& P, int threads, cudaStream_t st);
int max_multi_f64_cluster(bool srec, int TW, int threads, size_t smem);
int max_multi_f64_grid(bool srec, int TW, int threads, size_t smem);
int max_multi_f32_cluster(bool srec, int TW, int threads, size_t smem);
int max_multi_f32_grid(bool srec, int TW, int threads, size_t smem);

size_t multi_smem_bytes(const LoopParams& P, bool f64) {
  return f64 ? smem_layout(P, sizeof(Rec<double>), sizeof(Msg<double, MULTI_K>)).total
             : smem_layout(P, sizeof(Rec<float>), sizeof(Msg<float, MULTI_K>)).total;
}

int multi_max_batch() { return BMAX; }
int multi_window() { return NE; }
int multi_max_threads() { return MPG_LB_THREADS; }

cudaError_t launch_multi_loop(const LoopParams& P, bool f64, int threads, cudaStream_t st) {
  if (P.gx) return f64 ? launch_multi_f64_grid(P, threads, st) : launch_multi_f32_grid(P, threads, st);
  return f64 ? launch_multi_f64_cluster(P, threads, st) : launch_multi_f32_cluster(P, threads, st);
}

int multi_max_cluster(bool f64, bool srec, int TW, int threads, size_t smem, bool gx) {
  if (gx) return f64 ? max_multi_f64_grid(srec, TW, threads, smem) : max_multi_f32_grid(srec, TW, threads, smem);
  return f64 ? max_multi_f64_cluster(srec, TW, threads, smem) : max_multi_f32_cluster(srec, TW, threads, smem);
}

size_t multi_msg_bytes(bool f64) { return f64 ? sizeof(Msg<double, MULTI_K>) : sizeof(Msg<float, MULTI_K>); }
