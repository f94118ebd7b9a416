// hc_launch.h -- internal (not exported) launch entry points shared by the C++
// frame launcher (hc_plan.cpp) and the CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "heightcast.h"

namespace hc {

// Tile-queue order job (hc_order.cuh) folded into a frame's max-mip launches:
// the per-chunk histograms run in k_mip_tiles' extra CTAs, the scatter in
// k_mip_top's, so k_render needs no launches of its own for the order.
struct OrderJob {
    const int32_t* cost;        // previous frame's per-tile costs
    int32_t* order;             // hc_render_order_words(...) words
    unsigned* counter;          // queue head, reset by the scatter
    int32_t n_tiles;
};

// Fused max-mip epilogue of a frame's discretization (hc_discretize.cu): levels
// 0..5 of both layers, patch bytes and per-block valid min/max partials; k_mip_top
// (maxmip_top_launch) finishes levels >= 6 and folds the partials.
struct DiscMipJob {
    float* mip[HC_MAX_CASCADES][2];          // terrain, water pyramids of cascade k
    uint8_t* patch_ok[HC_MAX_CASCADES];      // [(R-1)^2] patch bytes, may be NULL
    int32_t n_levels;
    int64_t level_off[6];
    int32_t level_w[6];
    float* partial;                          // [2K][partial_slots][2]
    int32_t partial_slots;                   // >= ceil(R / 32)^2
    int32_t full;                            // write every level under blocks outside the mask
    float* xchg;                             // sharded frame: exchange buffer (heightcast.h HcFootprint), or NULL
    const HcFootprint* fp;                   // with xchg: the strips' ground wedges
    int32_t throughput;                      // frames overlap: use the throughput CTA shape
};

int discretize_launch(const HcCascadeRaster* cascades, int n_cascades, const HcGrid* grid, float sentinel,
                      uint64_t* counters, const DiscMipJob* mips, const OrderJob* ord, cudaStream_t stream);
// levels >= 6 of each job from level 5, and the job's valid range from `partial`
// ([n_jobs][partial_slots][2], part_side^2 used); extra CTAs scatter the tile order
int maxmip_top_launch(const HcMipJob* jobs, int n_jobs, float* partial, int partial_slots, int part_side,
                      const OrderJob* ord, cudaStream_t stream, const float* xchg = nullptr);
int maxmip_launch(const HcMipJob* jobs, int n_jobs, void* workspace, size_t workspace_bytes, const OrderJob* ord,
                  cudaStream_t stream);
// order_ready: the tile order (and queue head) were produced by maxmip_launch
// throughput: frames overlap on the GPU, use the high-occupancy render instantiation
int render_launch(const HcRenderArgs* args, bool order_ready, cudaStream_t stream, bool throughput = false);

}  // namespace hc
