// Whole-image pruned transforms with the reference's layouts
// (proj/include/voxin/fft.hpp:111-457): the nested single-image transform
// (x halved) and the batched permute-based transform (z halved, layout
// (b, z'', y', x')).  Built from one generic strided-line Stockham FFT kernel
// (runtime radices 2/3/4/5/7, double-computed twiddles), launched only over
// the lines the reference's pruning keeps.
#pragma once

#include "common.cuh"

namespace vxg {

void init_line_fft(Ctx* c);
void pruned_forward_device(Ctx* c, const float* img, V3 n, V3 pad, float2* spec);
void pruned_inverse_device(Ctx* c, const float2* spec, V3 pad, V3 crop, float* out);
void batched_forward_device(Ctx* c, const float* imgs, int64_t b, V3 n, V3 pad, float2* spec);
void batched_inverse_device(Ctx* c, const float2* spec, int64_t b, V3 pad, V3 crop, float* out);

}  // namespace vxg
