// K1-K4: fused gather-sum (Eq. 1b) + mix/out copy, gain, imager + arena store.
//
// Reference: gather `render.cpp:44-48`, store `render.cpp:59-60`, copy_slot
// `processors.cpp:18-20`, gain_slot `:22-32` (y_c = exp(p_c) u_c), imager_slot `:34-49`
// (m = l + r, s = exp(p) (l - r), y_l = (m + s)/2, y_r = (m - s)/2).
// HBM-bound: per node-sample it moves 8*(deg_in + 1) bytes. One thread owns 4 consecutive
// samples of both channels of one (slot, batch) row; float4 loads/stores when L % 4 == 0.
#include <algorithm>
#include <stdexcept>

#include "launch.hpp"

namespace mgb {

namespace {

constexpr int kPwThreads = 128;

template <PointOp OP>
__device__ __forceinline__ void apply(float& l, float& r, float g0, float g1) {
  if constexpr (OP == PointOp::Gain) {
    l *= g0;
    r *= g1;
  } else if constexpr (OP == PointOp::Imager) {
    const float mid = l + r;
    const float side = g0 * (l - r);
    l = 0.5f * (mid + side);
    r = 0.5f * (mid - side);
  }
}

template <PointOp OP>
__device__ __forceinline__ void coeffs(const StepArgs& a, int slot, float& g0, float& g1) {
  g0 = g1 = 1.f;
  if constexpr (OP == PointOp::Gain) {
    g0 = static_cast<float>(exp(a.params[2 * slot]));
    g1 = static_cast<float>(exp(a.params[2 * slot + 1]));
  } else if constexpr (OP == PointOp::Imager) {
    g0 = static_cast<float>(exp(a.params[slot]));
  }
}

// grid.y = slot*B + b; one float4 group of both channels per thread (grid sized so every
// thread has exactly one). A step only reads rows stored by earlier steps (or zeroed rows),
// never its own output rows, so src and dst never alias (restrict is valid). Edges are
// consumed 8 at a time (16 independent 16-byte loads in flight), summed in edge order.
template <PointOp OP, bool EPI>
__device__ __forceinline__ void pointwise_vec4_body(const StepArgs& a, const PwEpi& epi) {
  const int sb = blockIdx.y;
  const int slot = sb / a.batch, b = sb - slot * a.batch;
  const long n4 = a.length >> 2;
  const long i = blockIdx.x * static_cast<long>(kPwThreads) + threadIdx.x;
  if (i >= n4) return;
  const int e0 = slot_e0(a, slot), e1 = slot_e1(a, slot);
  const long boff = static_cast<long>(b) * 2 * a.length;
  const float* __restrict__ src = a.src;
  float4 l = make_float4(0.f, 0.f, 0.f, 0.f), r = l;
  int e = e0;
  for (; e + 7 < e1; e += 8) {
    float4 lv[8], rv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float4* p = reinterpret_cast<const float4*>(src + edge_row(a, e + u) * a.rowstride + boff);
      lv[u] = __ldg(p + i);
      rv[u] = __ldg(p + n4 + i);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      l = f4add(l, lv[u]);
      r = f4add(r, rv[u]);
    }
  }
  for (; e < e1; ++e) {
    const float4* p = reinterpret_cast<const float4*>(src + edge_row(a, e) * a.rowstride + boff);
    l = f4add(l, __ldg(p + i));
    r = f4add(r, __ldg(p + n4 + i));
  }
  float g0, g1;
  coeffs<OP>(a, slot, g0, g1);
  apply<OP>(l.x, r.x, g0, g1);
  apply<OP>(l.y, r.y, g0, g1);
  apply<OP>(l.z, r.z, g0, g1);
  apply<OP>(l.w, r.w, g0, g1);
  float* __restrict__ out = a.dst + static_cast<long>(slot) * a.rowstride + boff;
  reinterpret_cast<float4*>(out)[i] = l;
  reinterpret_cast<float4*>(out + a.length)[i] = r;
  if constexpr (EPI) {
    PwEpiSlots c;
    pw_epi_slots(epi, slot, c);
    const float yl[4] = {l.x, l.y, l.z, l.w}, yr[4] = {r.x, r.y, r.z, r.w};
    pw_epi_apply(epi, c, a.rowstride, a.length, boff + 4 * i, yl, yr, true, 4);
  }
}

template <PointOp OP>
__global__ void __launch_bounds__(kPwThreads) pointwise_vec4(StepArgs a) {
  pointwise_vec4_body<OP, false>(a, PwEpi{});
}

// Same, with the step's pointwise followers in the epilogue (separate kernel: the plain one
// keeps its small parameter block and register allocation).
template <PointOp OP>
__global__ void __launch_bounds__(kPwThreads) pointwise_vec4_epi(StepArgs a, PwEpi epi) {
  pointwise_vec4_body<OP, true>(a, epi);
}

// Aggregation-heavy steps with few output rows (the console's master mix: 35 inputs, one
// row): the per-row grid of pointwise_vec4 leaves most SMs idle and each thread walks all
// the edges. Here kWideGroups thread groups each sum a contiguous quarter of the edges (in
// edge order) for the same 64 float4 positions, and the partial sums are added in group
// order: ((q0 + q1) + q2) + q3, deterministic. grid (ceil(n4 / 64), slots*B) x 256.
constexpr int kWideGroups = 4, kWidePos = 64;
template <PointOp OP>
__global__ void __launch_bounds__(kWideGroups * kWidePos) pointwise_wide(StepArgs a) {
  __shared__ float4 pl[kWideGroups][kWidePos], pr[kWideGroups][kWidePos];
  const int sb = blockIdx.y;
  const int slot = sb / a.batch, b = sb - slot * a.batch;
  const long n4 = a.length >> 2;
  const int g = threadIdx.x / kWidePos, p = threadIdx.x - g * kWidePos;
  const long i = blockIdx.x * static_cast<long>(kWidePos) + p;
  const int e0 = slot_e0(a, slot), e1 = slot_e1(a, slot);
  const int per = (e1 - e0 + kWideGroups - 1) / kWideGroups;
  const int ga = e0 + g * per, gb = min(e1, ga + per);
  const long boff = static_cast<long>(b) * 2 * a.length;
  float4 l = make_float4(0.f, 0.f, 0.f, 0.f), r = l;
  if (i < n4) {
    int e = ga;
    for (; e + 7 < gb; e += 8) {
      float4 lv[8], rv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float4* q = reinterpret_cast<const float4*>(a.src + edge_row(a, e + u) * a.rowstride + boff);
        lv[u] = __ldg(q + i);
        rv[u] = __ldg(q + n4 + i);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        l = f4add(l, lv[u]);
        r = f4add(r, rv[u]);
      }
    }
    for (; e < gb; ++e) {
      const float4* q = reinterpret_cast<const float4*>(a.src + edge_row(a, e) * a.rowstride + boff);
      l = f4add(l, __ldg(q + i));
      r = f4add(r, __ldg(q + n4 + i));
    }
  }
  pl[g][p] = l;
  pr[g][p] = r;
  __syncthreads();
  if (g != 0 || i >= n4) return;
#pragma unroll
  for (int h = 1; h < kWideGroups; ++h) {
    l = f4add(l, pl[h][p]);
    r = f4add(r, pr[h][p]);
  }
  float g0, g1;
  coeffs<OP>(a, slot, g0, g1);
  apply<OP>(l.x, r.x, g0, g1);
  apply<OP>(l.y, r.y, g0, g1);
  apply<OP>(l.z, r.z, g0, g1);
  apply<OP>(l.w, r.w, g0, g1);
  float* __restrict__ out = a.dst + static_cast<long>(slot) * a.rowstride + boff;
  reinterpret_cast<float4*>(out)[i] = l;
  reinterpret_cast<float4*>(out + a.length)[i] = r;
}

template <PointOp OP>
__global__ void __launch_bounds__(256) pointwise_scalar(StepArgs a) {
  const int sb = blockIdx.y;
  const int slot = sb / a.batch, b = sb - slot * a.batch;
  const int e0 = slot_e0(a, slot), e1 = slot_e1(a, slot);
  float g0, g1;
  coeffs<OP>(a, slot, g0, g1);
  float* out = a.dst + static_cast<long>(slot) * a.rowstride + static_cast<long>(b) * 2 * a.length;
  for (long n = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; n < a.length; n += static_cast<long>(gridDim.x) * blockDim.x) {
    float2 v = gather2(a, e0, e1, b, n);
    apply<OP>(v.x, v.y, g0, g1);
    out[n] = v.x;
    out[n + a.length] = v.y;
  }
}

template <PointOp OP>
void launch_op(const StepArgs& a, cudaStream_t s, const PwEpi& epi) {
  const int rows = a.slots * a.batch;
  if (rows == 0 || a.length == 0) return;
  const bool vec = (a.length % 4) == 0;
  if (vec) {
    const dim3 grid(static_cast<unsigned>((a.length / 4 + kPwThreads - 1) / kPwThreads), static_cast<unsigned>(rows));
    // Few rows gathering many inputs: edge-split groups (pointwise_wide), when the plain grid
    // would be under two waves of the SMs and the rows average 8+ inputs.
    if (epi.n == 0 && static_cast<long>(grid.x) * grid.y < 2L * 148 && a.nnz >= 8 * a.slots) {
      const dim3 wgrid(static_cast<unsigned>((a.length / 4 + kWidePos - 1) / kWidePos), static_cast<unsigned>(rows));
      pointwise_wide<OP><<<wgrid, kWideGroups * kWidePos, 0, s>>>(a);
      return;
    }
    if (epi.n > 0) {
      pointwise_vec4_epi<OP><<<grid, kPwThreads, 0, s>>>(a, epi);
    } else {
      pointwise_vec4<OP><<<grid, kPwThreads, 0, s>>>(a);
    }
    return;
  }
  long blocks = (a.length + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  dim3 grid(static_cast<unsigned>(blocks), static_cast<unsigned>(rows));
  pointwise_scalar<OP><<<grid, 256, 0, s>>>(a);
}

// A run of consecutive small pointwise steps (the 1-slot bus tail: imager -> gain -> out) in
// one launch. Every step is sample-local, so the thread owning float4 group i of batch row b
// computes group i of every slot of every step in step order: a later step's gather reads
// rows this same thread stored moments earlier (plain loads, not the non-coherent __ldg path,
// so program order makes them visible). Results are identical to the per-step launches.
__global__ void __launch_bounds__(kPwThreads) pointwise_chain_vec4(PwChain c) {
  const int b = blockIdx.y;
  const long i = blockIdx.x * static_cast<long>(kPwThreads) + threadIdx.x;
  for (int k = 0; k < c.n; ++k) {
    const StepArgs& a = c.step[k];
    const long n4 = a.length >> 2;
    if (i >= n4) return;
    const long boff = static_cast<long>(b) * 2 * a.length;
    for (int slot = 0; slot < a.slots; ++slot) {
      const int e0 = slot_e0(a, slot), e1 = slot_e1(a, slot);
      float4 l = make_float4(0.f, 0.f, 0.f, 0.f), r = l;
      for (int e = e0; e < e1; ++e) {
        const float4* p = reinterpret_cast<const float4*>(a.src + edge_row(a, e) * a.rowstride + boff);
        l = f4add(l, p[i]);
        r = f4add(r, p[n4 + i]);
      }
      float g0 = 1.f, g1 = 1.f;
      switch (c.op[k]) {
        case PointOp::Gain:
          coeffs<PointOp::Gain>(a, slot, g0, g1);
          apply<PointOp::Gain>(l.x, r.x, g0, g1), apply<PointOp::Gain>(l.y, r.y, g0, g1);
          apply<PointOp::Gain>(l.z, r.z, g0, g1), apply<PointOp::Gain>(l.w, r.w, g0, g1);
          break;
        case PointOp::Imager:
          coeffs<PointOp::Imager>(a, slot, g0, g1);
          apply<PointOp::Imager>(l.x, r.x, g0, g1), apply<PointOp::Imager>(l.y, r.y, g0, g1);
          apply<PointOp::Imager>(l.z, r.z, g0, g1), apply<PointOp::Imager>(l.w, r.w, g0, g1);
          break;
        default: break;
      }
      float* out = a.dst + static_cast<long>(slot) * a.rowstride + boff;
      reinterpret_cast<float4*>(out)[i] = l;
      reinterpret_cast<float4*>(out + a.length)[i] = r;
    }
  }
}

// grid (ceil(max rows*width / 256 / 4), 10 types): one thread per 4 consecutive values.
__global__ void param_gather(ParamGather g) {
  const int t = blockIdx.y;
  const int rows = g.rows[t], w = g.width[t];
  const long n = static_cast<long>(rows) * w;
  for (long i = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) * 4; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x * 4) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const long e = i + j;
      if (e < n) {
        const long r = e / w, c = e - r * w;
        g.out[t][e] = __ldg(g.in[t] + static_cast<long>(__ldg(g.src_rows[t] + r)) * w + c);
      }
    }
  }
}

}  // namespace

void launch_param_gather(const ParamGather& g, cudaStream_t s) {
  long most = 0;
  for (int t = 0; t < 10; ++t) most = std::max(most, static_cast<long>(g.rows[t]) * g.width[t]);
  if (most == 0) return;
  const long blocks = std::min<long>((most + 1023) / 1024, 148L * 8);
  param_gather<<<dim3(static_cast<unsigned>(blocks), 10), 256, 0, s>>>(g);
}

bool pointwise_chain_ok(const StepArgs& a) {
  return a.length % 4 == 0 && a.slots >= 1 && a.slots * a.batch <= kPwChainMaxRows;
}

void launch_pointwise_chain(const PwChain& c, cudaStream_t s) {
  if (c.n <= 0) return;
  const StepArgs& a = c.step[0];
  const dim3 grid(static_cast<unsigned>((a.length / 4 + kPwThreads - 1) / kPwThreads), static_cast<unsigned>(a.batch));
  pointwise_chain_vec4<<<grid, kPwThreads, 0, s>>>(c);
}

bool pointwise_epi_ok(const StepArgs& a) { return a.length % 4 == 0; }

void launch_pointwise(PointOp op, const StepArgs& a, cudaStream_t s, const PwEpi& epi) {
  if (epi.n > 0 && !pointwise_epi_ok(a)) throw std::invalid_argument("launch_pointwise: epilogue needs L % 4 == 0");
  switch (op) {
    case PointOp::Copy: launch_op<PointOp::Copy>(a, s, epi); break;
    case PointOp::Gain: launch_op<PointOp::Gain>(a, s, epi); break;
    case PointOp::Imager: launch_op<PointOp::Imager>(a, s, epi); break;
  }
}

}  // namespace mgb
