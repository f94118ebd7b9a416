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

int maxmip_launch(const HcMipJob* jobs, int n_jobs, void* workspace, size_t workspace_bytes, const OrderJob* ord,
                  cudaStream_t stream);
// order_ready: the tile order (and queue head) were produced by maxmip_launch
int render_launch(const HcRenderArgs* args, bool order_ready, cudaStream_t stream);

}  // namespace hc
