// K7: compressor / noisegate — energy envelope as a single-pass chained scan.
//
// Reference: dynamics_slot `processors.cpp:71-106`: mid = l + r, e = mid^2, the envelope
// is e convolved with the FIR (1-a) a^k truncated to Ne = min(envelope_taps, L) taps, then
// G_u = ln max(env, floor), G_y = knee curve (`compressor_gain_log` :110-119,
// `noisegate_gain_log` :121-130), y = exp(G_y - G_u) * u on both channels.
//
// The truncated FIR is exactly the linear recurrence
//     g[n] = a*g[n-1] + (1-a)*(e[n] - a^Ne * e[n-Ne]),   g[-1] = 0,
// so instead of the reference's 2^18-point FFTs per (node, batch) this is a scan of affine
// maps x -> A x + B. Tile = 512 threads x 8 samples. Within a tile: per-thread serial
// recurrence, warp shuffles, one smem level. Across tiles: every tile publishes its
// aggregate (flag | fp32 B in one 64-bit store; all full tiles share A = a^4096) and sums
// its predecessors' aggregates in a fixed order (see the carry block), so results are
// bit-reproducible; tile order comes from an atomic ticket so every waited-on tile was
// scheduled earlier.
// The a^Ne correction term re-gathers e[n - Ne]; it is skipped when a^Ne < 1e-30.
#include <cuda/atomic>

#include "launch.hpp"

namespace mgb {

namespace {

constexpr unsigned long long kFlagAgg = 1ull << 32;

struct DynParams {
  float a, oma, aN, a16, atile, atile32;
  float T, W, R, invR, floor_;
  int Ne;
};

// Slot constants, derived by warp 0 of each CTA: lanes 0-3 evaluate the four fp64 powers
// a^Ne, a^8, a^tile, a^(32 tile) side by side (one pow latency), lane 0 assembles.
__device__ __forceinline__ void derive_params(const double* row, int env_taps, double floor_, long L, int lane,
                                              DynParams* out) {
  const double a = row[0];
  const int Ne = static_cast<int>(env_taps < L ? env_taps : L);
  const double e = lane == 0 ? static_cast<double>(Ne)
                 : lane == 1 ? static_cast<double>(kDynPerThread)
                 : lane == 2 ? static_cast<double>(kDynTile) : 32.0 * kDynTile;
  const double pw = lane < 4 ? pow(a, e) : 0.0;
  const double aN = __shfl_sync(0xffffffffu, pw, 0), a16 = __shfl_sync(0xffffffffu, pw, 1);
  const double atile = __shfl_sync(0xffffffffu, pw, 2), atile32 = __shfl_sync(0xffffffffu, pw, 3);
  if (lane != 0) return;
  DynParams p;
  p.a = static_cast<float>(a);
  p.oma = static_cast<float>(1.0 - a);
  p.Ne = Ne;
  p.aN = aN < 1e-30 ? 0.f : static_cast<float>(aN);
  p.a16 = static_cast<float>(a16);
  p.atile = static_cast<float>(atile);
  p.atile32 = static_cast<float>(atile32);
  p.T = static_cast<float>(row[1]);
  p.W = static_cast<float>(row[2]);
  p.R = static_cast<float>(row[3]);
  p.invR = static_cast<float>(1.0 / row[3]);
  p.floor_ = static_cast<float>(floor_);
  *out = p;
}

template <bool GATE>
__device__ __forceinline__ float gain_of(float g, const DynParams& p) {
  const float gu = logf(fmaxf(g, p.floor_));
  float gy;
  if (!GATE) {
    if (gu >= p.T + p.W) {
      gy = p.T + (gu - p.T) * p.invR;
    } else if (gu < p.T - p.W) {
      gy = gu;
    } else {
      const float d = gu - p.T + p.W;
      gy = gu + (p.invR - 1.f) * d * d / (4.f * p.W);
    }
  } else {
    if (gu >= p.T + p.W) {
      gy = gu;
    } else if (gu < p.T - p.W) {
      gy = p.T + p.R * (gu - p.T);
    } else {
      const float d = gu - p.T - p.W;
      gy = gu + (1.f - p.R) * d * d / (4.f * p.W);
    }
  }
  return expf(gy - gu);
}

// Gather-sum of the slot's inputs at kDynPerThread consecutive samples from n0.
template <bool VEC>
__device__ __forceinline__ void load16(const StepArgs& a, int e0, int e1, int b, long n0, float* ul, float* ur) {
#pragma unroll
  for (int k = 0; k < kDynPerThread; ++k) ul[k] = ur[k] = 0.f;
  if (n0 >= a.length || n0 < 0) return;
  const long boff = static_cast<long>(b) * 2 * a.length;
  if (VEC && n0 + kDynPerThread <= a.length) {
    for (int e = e0; e < e1; ++e) {
      const float* p = a.src + static_cast<long>(__ldg(a.col + e)) * a.rowstride + boff + n0;
#pragma unroll
      for (int q = 0; q < kDynPerThread / 4; ++q) {
        const float4 l = __ldg(reinterpret_cast<const float4*>(p) + q);
        const float4 r = __ldg(reinterpret_cast<const float4*>(p + a.length) + q);
        ul[4 * q] += l.x; ul[4 * q + 1] += l.y; ul[4 * q + 2] += l.z; ul[4 * q + 3] += l.w;
        ur[4 * q] += r.x; ur[4 * q + 1] += r.y; ur[4 * q + 2] += r.z; ur[4 * q + 3] += r.w;
      }
    }
  } else {
    for (int e = e0; e < e1; ++e) {
      const float* p = a.src + static_cast<long>(__ldg(a.col + e)) * a.rowstride + boff;
#pragma unroll
      for (int k = 0; k < kDynPerThread; ++k) {
        const long n = n0 + k;
        if (n < a.length) {
          ul[k] += __ldg(p + n);
          ur[k] += __ldg(p + a.length + n);
        }
      }
    }
  }
}

__device__ __forceinline__ void compose(float& A, float& B, float Ap, float Bp) {
  // earlier (Ap, Bp) then current (A, B)
  B = fmaf(A, Bp, B);
  A = A * Ap;
}

template <bool GATE, bool VEC>
__global__ void __launch_bounds__(kDynThreads, 2) dyn_scan(StepArgs a, int env_taps, double floor_, int tiles_per_seq,
                                                         unsigned long long* status, unsigned int* ticket) {
  __shared__ float wA[kDynThreads / 32], wB[kDynThreads / 32];
  __shared__ float s_carry;
  __shared__ int s_ticket;
  __shared__ DynParams s_p;
  // Tickets interleave sequences (all tile-0s, then all tile-1s, ...): a tile's
  // predecessors were dispatched `nseq` tickets earlier, so the carry rarely waits.
  const int nseq = a.slots * a.batch;
  if (threadIdx.x < 32) {
    int tk = 0;
    if (threadIdx.x == 0) tk = static_cast<int>(atomicAdd(ticket, 1u));
    tk = __shfl_sync(0xffffffffu, tk, 0);
    if (threadIdx.x == 0) s_ticket = tk;
    derive_params(a.params + 4L * ((tk % nseq) / a.batch), env_taps, floor_, a.length, threadIdx.x, &s_p);
  }
  __syncthreads();
  const int tk = s_ticket;
  const int tile = tk / nseq, seq = tk - tile * nseq;
  const int slot = seq / a.batch, b = seq - slot * a.batch;
  const int e0 = __ldg(a.row_ptr + slot), e1 = __ldg(a.row_ptr + slot + 1);
  const DynParams p = s_p;

  const long n0 = static_cast<long>(tile) * kDynTile + static_cast<long>(threadIdx.x) * kDynPerThread;
  // drive[k] = (1-a) (e[n] - a^Ne e[n-Ne]) is all the scan keeps in registers; the input
  // samples are gathered again (L2-resident) for the output pass, so nothing else stays live
  // across the carry wait (no spills at 64 registers).
  float drive[kDynPerThread];
  {
    float ul[kDynPerThread], ur[kDynPerThread], eo[kDynPerThread];
    load16<VEC>(a, e0, e1, b, n0, ul, ur);
    if (p.aN != 0.f) {
      float ol[kDynPerThread], orr[kDynPerThread];
      load16<VEC>(a, e0, e1, b, n0 - p.Ne, ol, orr);
#pragma unroll
      for (int k = 0; k < kDynPerThread; ++k) {
        const float m = ol[k] + orr[k];
        eo[k] = p.aN * (m * m);
      }
    } else {
#pragma unroll
      for (int k = 0; k < kDynPerThread; ++k) eo[k] = 0.f;
    }
#pragma unroll
    for (int k = 0; k < kDynPerThread; ++k) {
      const float m = ul[k] + ur[k];
      drive[k] = p.oma * (m * m - eo[k]);
    }
  }

  // Thread-local recurrence from 0.
  float B = 0.f;
#pragma unroll
  for (int k = 0; k < kDynPerThread; ++k) B = fmaf(p.a, B, drive[k]);
  float A = p.a16;

  // Warp inclusive scan of affine maps.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const float Ap = __shfl_up_sync(0xffffffffu, A, off);
    const float Bp = __shfl_up_sync(0xffffffffu, B, off);
    if (lane >= off) compose(A, B, Ap, Bp);
  }
  if (lane == 31) {
    wA[warp] = A;
    wB[warp] = B;
  }
  // Exclusive prefix within the warp.
  float xA = __shfl_up_sync(0xffffffffu, A, 1), xB = __shfl_up_sync(0xffffffffu, B, 1);
  if (lane == 0) {
    xA = 1.f;
    xB = 0.f;
  }
  __syncthreads();
  if (warp == 0) {
    float tA = lane < kDynThreads / 32 ? wA[lane] : 1.f;
    float tB = lane < kDynThreads / 32 ? wB[lane] : 0.f;
#pragma unroll
    for (int off = 1; off < kDynThreads / 32; off <<= 1) {
      const float Ap = __shfl_up_sync(0xffffffffu, tA, off);
      const float Bp = __shfl_up_sync(0xffffffffu, tB, off);
      if (lane >= off) compose(tA, tB, Ap, Bp);
    }
    if (lane < kDynThreads / 32) {
      wA[lane] = tA;  // inclusive warp-level prefix
      wB[lane] = tB;
    }
  }
  __syncthreads();
  if (warp > 0) {  // prepend the previous warps' prefix
    float pA = wA[warp - 1], pB = wB[warp - 1];
    compose(xA, xB, pA, pB);
  }
  const float tileB = wB[kDynThreads / 32 - 1];

  if (warp == 0) {
    // Cross-tile carry, deterministic: publish this tile's aggregate B, then
    //   carry = sum_{d >= 0} A^d * B_{tile-1-d},   A = a^tile_len,
    // summed lane-strided (d = lane + 32 i) and tree-reduced in a fixed order. Only
    // aggregates are read (no chain of inclusive prefixes), so no tile waits on another
    // tile's look-back, and the value never depends on timing. Windows stop once the
    // largest remaining weight A^d underflows to exactly 0 (all later terms are +0).
    // status is indexed [seq][tile]
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> mine(status[static_cast<long>(seq) * tiles_per_seq + tile]);
    if (lane == 0) mine.store(kFlagAgg | __float_as_uint(tileB), cuda::memory_order_relaxed);
    float part = 0.f;
    // weight A^d = A^lane * (A^32)^(d0/32): one powf per lane, then exact-order products
    const float wl = tile > 0 ? powf(p.atile, static_cast<float>(lane)) : 0.f;
    float w32 = 1.f;  // (A^32)^(d0/32)
    for (int d0 = 0; d0 < tile; d0 += 32, w32 *= p.atile32) {
      if (w32 == 0.f) break;
      const int d = d0 + lane;
      if (d < tile) {
        cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> st(status[static_cast<long>(seq) * tiles_per_seq + tile - 1 - d]);
        unsigned long long w;
        do {
          w = st.load(cuda::memory_order_relaxed);
        } while ((w >> 32) == 0);
        part = fmaf(wl * w32, __uint_as_float(static_cast<unsigned int>(w & 0xffffffffu)), part);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
    if (lane == 0) s_carry = part;
  }
  __syncthreads();

  // Replay the recurrence from this thread's true start state, apply the gain, store.
  float g = fmaf(xA, s_carry, xB);
  if (n0 >= a.length) return;
  float ul[kDynPerThread], ur[kDynPerThread];
  load16<VEC>(a, e0, e1, b, n0, ul, ur);
  float* ol = a.dst + static_cast<long>(slot) * a.rowstride + static_cast<long>(b) * 2 * a.length + n0;
  float* orr = ol + a.length;
  const bool full = VEC && n0 + kDynPerThread <= a.length;
#pragma unroll
  for (int q = 0; q < kDynPerThread / 4; ++q) {
    float yl[4], yr[4];
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4) {
      const int k = 4 * q + k4;
      g = fmaf(p.a, g, drive[k]);
      const float gn = gain_of<GATE>(g, p);
      yl[k4] = gn * ul[k];
      yr[k4] = gn * ur[k];
    }
    if (full) {
      reinterpret_cast<float4*>(ol)[q] = make_float4(yl[0], yl[1], yl[2], yl[3]);
      reinterpret_cast<float4*>(orr)[q] = make_float4(yr[0], yr[1], yr[2], yr[3]);
    } else {
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        if (n0 + 4 * q + k4 < a.length) {
          ol[4 * q + k4] = yl[k4];
          orr[4 * q + k4] = yr[k4];
        }
      }
    }
  }
}

}  // namespace

std::size_t dyn_sync_bytes(int slots, int batch, long length) {
  const long tiles = (length + kDynTile - 1) / kDynTile;
  return 256 + sizeof(unsigned long long) * static_cast<std::size_t>(slots) * batch * tiles;
}

void launch_dynamics(bool gate, const StepArgs& a, int envelope_taps, double energy_floor, void* ws,
                     bool zero_sync, cudaStream_t s) {
  if (a.slots == 0 || a.batch == 0 || a.length == 0) return;
  const int tiles = static_cast<int>((a.length + kDynTile - 1) / kDynTile);
  const long total = static_cast<long>(a.slots) * a.batch * tiles;
  if (zero_sync) cudaMemsetAsync(ws, 0, dyn_sync_bytes(a.slots, a.batch, a.length), s);
  auto* ticket = static_cast<unsigned int*>(ws);
  auto* status = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + 256);
  const long ne = envelope_taps < a.length ? envelope_taps : a.length;
  const bool vec = (a.length % 4 == 0) && (ne % 4 == 0);
  const dim3 grid(static_cast<unsigned>(total));
  if (gate) {
    if (vec) dyn_scan<true, true><<<grid, kDynThreads, 0, s>>>(a, envelope_taps, energy_floor, tiles, status, ticket);
    else dyn_scan<true, false><<<grid, kDynThreads, 0, s>>>(a, envelope_taps, energy_floor, tiles, status, ticket);
  } else {
    if (vec) dyn_scan<false, true><<<grid, kDynThreads, 0, s>>>(a, envelope_taps, energy_floor, tiles, status, ticket);
    else dyn_scan<false, false><<<grid, kDynThreads, 0, s>>>(a, envelope_taps, energy_floor, tiles, status, ticket);
  }
}

}  // namespace mgb
