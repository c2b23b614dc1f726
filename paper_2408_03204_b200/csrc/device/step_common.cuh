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
  const double2* tw64 = nullptr;  // the same twiddles in fp64 (fp64 transforms)
  int slots;
  int batch;
  long length;           // L
  long rowstride;        // B*2*L
  int nnz = 0;           // edges of the step (host hint for launch shapes; 0 = unknown)
  int dense = -1;        // >= 0: slot s reads exactly row dense + s (no CSR loads needed)
};

// A pointer the compiler cannot re-associate with the index math of its uses (so a loop of
// stores at p[k] costs one IMAD.WIDE per address instead of re-deriving p from the kernel
// parameters each time).
template <typename T>
__device__ __forceinline__ T* opaque_ptr(T* p) {
  asm volatile("" : "+l"(p));
  return p;
}

// Plain global store through a pointer the compiler no longer knows the space of.
__device__ __forceinline__ void st_global(float* p, float v) { asm("st.global.f32 [%0], %1;" ::"l"(p), "f"(v)); }

// CSR access. Dense steps (a track chain's steps read the previous step's rows in order)
// skip the row_ptr -> col -> sample chain of dependent L2 round trips: only sample loads.
__device__ __forceinline__ int slot_e0(const StepArgs& a, int slot) { return a.dense >= 0 ? slot : __ldg(a.row_ptr + slot); }
__device__ __forceinline__ int slot_e1(const StepArgs& a, int slot) {
  return a.dense >= 0 ? slot + 1 : __ldg(a.row_ptr + slot + 1);
}
__device__ __forceinline__ long edge_row(const StepArgs& a, int e) {
  return a.dense >= 0 ? static_cast<long>(a.dense) + e : static_cast<long>(__ldg(a.col + e));
}

__device__ __forceinline__ const float* chan_ptr(const float* base, long row, long rowstride, int b, int c, long L) {
  return base + row * rowstride + (static_cast<long>(b) * 2 + c) * L;
}

// Sum of both channels at sample n over the slot's incoming rows.
__device__ __forceinline__ float2 gather2(const StepArgs& a, int e0, int e1, int b, long n) {
  float l = 0.f, r = 0.f;
  const long off = static_cast<long>(b) * 2 * a.length + n;
  for (int e = e0; e < e1; ++e) {
    const float* p = a.src + edge_row(a, e) * a.rowstride + off;
    l += __ldg(p);
    r += __ldg(p + a.length);
  }
  return make_float2(l, r);
}

// The twiddle table of a transform's element type.
template <typename C> __device__ __forceinline__ const C* twiddles(const StepArgs& a);
template <> __device__ __forceinline__ const float2* twiddles<float2>(const StepArgs& a) { return a.tw; }
template <> __device__ __forceinline__ const double2* twiddles<double2>(const StepArgs& a) { return a.tw64; }

__device__ __forceinline__ float4 f4add(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }

enum class PointOp : int { Copy = 0, Gain = 1, Imager = 2 };

// Pointwise followers fused into the epilogue of the step before them. A follower is a
// gain / imager / copy (mix, out) step whose every node has exactly one input edge, from a
// distinct node of the previous step (the per-track chain noisegate -> imager -> gain of a
// console). The producing kernel, holding output y of its slot s at some samples, computes
// the follower's output for slot map[s] from y with the follower's own arithmetic and
// stores it into the follower's row, and so on down the run; the followers' own launches and
// their re-reads of the producer's rows disappear. Values are bit-identical to the separate
// launches (the gather of one row is 0 + y there, kept here).
constexpr int kPwEpiMax = 3;
struct PwEpi {
  int n = 0;                          // fused follower steps
  PointOp op[kPwEpiMax] = {};
  float* dst[kPwEpiMax] = {};         // follower's first output row
  const int* map[kPwEpiMax] = {};     // previous step's slot -> follower slot
  const double* params[kPwEpiMax] = {};
};
// Per (producer slot): the follower slots and their float coefficients (gain: exp(p_l),
// exp(p_r); imager: exp(p_s); copy: 1).
struct PwEpiSlots {
  int slot[kPwEpiMax];
  float g0[kPwEpiMax], g1[kPwEpiMax];
};
__device__ __forceinline__ void pw_epi_slots(const PwEpi& e, int slot, PwEpiSlots& c) {
#pragma unroll
  for (int f = 0; f < kPwEpiMax; ++f) {
    if (f >= e.n) break;
    slot = __ldg(e.map[f] + slot);
    c.slot[f] = slot;
    c.g0[f] = c.g1[f] = 1.f;
    if (e.op[f] == PointOp::Gain) {
      c.g0[f] = static_cast<float>(exp(e.params[f][2 * slot]));
      c.g1[f] = static_cast<float>(exp(e.params[f][2 * slot + 1]));
    } else if (e.op[f] == PointOp::Imager) {
      c.g0[f] = static_cast<float>(exp(e.params[f][slot]));
    }
  }
}
__device__ __forceinline__ void pw_op(PointOp op, float& l, float& r, float g0, float g1) {
  if (op == PointOp::Gain) {
    l *= g0;
    r *= g1;
  } else if (op == PointOp::Imager) {
    const float mid = l + r;
    const float side = g0 * (l - r);
    l = 0.5f * (mid + side);
    r = 0.5f * (mid - side);
  }
}
// Four consecutive samples (offset `off` = b*2*L + n within a row) of both channels; `full`:
// all four valid and 16-byte aligned, else the first `valid` are stored one by one.
__device__ __forceinline__ void pw_epi_apply(const PwEpi& e, const PwEpiSlots& c, long rowstride, long L, long off,
                                             const float (&yl)[4], const float (&yr)[4], bool full, int valid) {
  float l[4], r[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    l[k] = yl[k];
    r[k] = yr[k];
  }
#pragma unroll
  for (int f = 0; f < kPwEpiMax; ++f) {
    if (f >= e.n) break;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      l[k] = 0.f + l[k];
      r[k] = 0.f + r[k];
      pw_op(e.op[f], l[k], r[k], c.g0[f], c.g1[f]);
    }
    float* out = e.dst[f] + static_cast<long>(c.slot[f]) * rowstride + off;
    if (full) {
      *reinterpret_cast<float4*>(out) = make_float4(l[0], l[1], l[2], l[3]);
      *reinterpret_cast<float4*>(out + L) = make_float4(r[0], r[1], r[2], r[3]);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (k < valid) {
          out[k] = l[k];
          out[L + k] = r[k];
        }
      }
    }
  }
}

// 256-bit global accesses (sm_100: LDG.E.ENL2.256 / STG.E.ENL2.256): a thread's 8 consecutive
// floats in one instruction, so a warp's access is 1 KiB contiguous. p must be 32-byte aligned.
__device__ __forceinline__ void st8(float* p, const float (&v)[8]) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]),
               "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
__device__ __forceinline__ void ld8(const float* p, float (&v)[8]) {
  asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "l"(p)
               : "memory");
}

// Bulk asynchronous copies global -> shared (cp.async.bulk, the TMA engine's 1-D form) with
// mbarrier completion: one elected thread arms the barrier with the byte count and issues the
// copies; consumers wait on the barrier's phase parity.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

}  // namespace mgb
