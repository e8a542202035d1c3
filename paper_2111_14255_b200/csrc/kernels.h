// Launch interface of the device code (kernels.cu) used by the host runtime (host.cpp).
#pragma once
#include <cuda_runtime.h>

#include "mt_types.h"

namespace mtk {

size_t executor_smem_bytes();
// max co-resident executor CTAs per SM (cooperative-launch feasibility)
cudaError_t executor_occupancy(int *blocks_per_sm);
int executor_resources(char *buf, int n);   // diagnostics: registers, shared memory
// the persistent stage executor: one cooperative launch runs the whole schedule (a4)
cudaError_t launch_executor(const RunArgs &a, int grid, cudaStream_t s);
// baseline: one launch running every tile of op `op` (same tile functions as the executor)
cudaError_t launch_op(const RunArgs &a, const OpDesc &host_op, int op, int max_grid,
                      cudaStream_t s);
// baseline: pack the graph input of tenant t (NCHW fp32 -> NHWC, C padded)
cudaError_t launch_pack(const RunArgs &a, int t, cudaStream_t s);
// bind-time weight repack (mode: 1 conv TC bf16, 2 conv SIMT fp32, 3 depthwise, 4 FC)
cudaError_t launch_weight_pack(int mode, const float *src, void *dst, const OpDesc &d,
                               int cin_real, cudaStream_t s);

}  // namespace mtk

// the 2-CTAs-per-SM build (kernels_cr.cu, f4 co-residency): same interface
namespace mtk_cr {

size_t executor_smem_bytes();
// max co-resident executor CTAs per SM (cooperative-launch feasibility)
cudaError_t executor_occupancy(int *blocks_per_sm);
int executor_resources(char *buf, int n);   // diagnostics: registers, shared memory
// the persistent stage executor: one cooperative launch runs the whole schedule (a4)
cudaError_t launch_executor(const RunArgs &a, int grid, cudaStream_t s);
// baseline: one launch running every tile of op `op` (same tile functions as the executor)
cudaError_t launch_op(const RunArgs &a, const OpDesc &host_op, int op, int max_grid,
                      cudaStream_t s);
// baseline: pack the graph input of tenant t (NCHW fp32 -> NHWC, C padded)
cudaError_t launch_pack(const RunArgs &a, int t, cudaStream_t s);
// bind-time weight repack (mode: 1 conv TC bf16, 2 conv SIMT fp32, 3 depthwise, 4 FC)
cudaError_t launch_weight_pack(int mode, const float *src, void *dst, const OpDesc &d,
                               int cin_real, cudaStream_t s);

}  // namespace mtk_cr
