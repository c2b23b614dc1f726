// Per-step device arguments and the fused Eq. 1b gather-sum.
//
// Arena layout (HBM, fp32): row r, batch b, channel c, sample n at
//   arena[r*rowstride + (b*2 + c)*L + n],  rowstride = B*2*L   (reference: `render.cpp:32-37`,
//   `audio_buffer.hpp:7-32`, there in double).
// A step reads its inputs through a CSR over the step's slots: slot s sums source rows
// col[row_ptr[s] .. row_ptr[s+1]) in edge order, ((0 + x0) + x1) + ... as the reference's
// gather loop does (`render.cpp:44-48`); a slot with no incoming edge reads silence.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace mgb {

struct StepArgs {
  const float* src;      // gather base (arena)
  float* dst;            // first output row of the step (arena + store_begin*rowstride)
  const int* row_ptr;    // [slots+1]
  const int* col;        // [nnz] source rows
  const double* params;  // first parameter row of the step (row-major, width per type)
  const float2* tw;      // twiddle table (fft_smem.cuh kTwN entries)
  int slots;
  int batch;
  long length;           // L
  long rowstride;        // B*2*L
};

__device__ __forceinline__ const float* chan_ptr(const float* base, long row, long rowstride, int b, int c, long L) {
  return base + row * rowstride + (static_cast<long>(b) * 2 + c) * L;
}

// Sum of both channels at sample n over the slot's incoming rows.
__device__ __forceinline__ float2 gather2(const StepArgs& a, int e0, int e1, int b, long n) {
  float l = 0.f, r = 0.f;
  const long off = static_cast<long>(b) * 2 * a.length + n;
  for (int e = e0; e < e1; ++e) {
    const float* p = a.src + static_cast<long>(__ldg(a.col + e)) * a.rowstride + off;
    l += __ldg(p);
    r += __ldg(p + a.length);
  }
  return make_float2(l, r);
}

__device__ __forceinline__ float4 f4add(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }

}  // namespace mgb
