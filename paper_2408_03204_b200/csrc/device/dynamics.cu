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
// bit-reproducible; tile order is the block index: a tile waits only on lower block indices,
// which the hardware dispatches first (the forward-progress assumption of CUB's single-pass
// decoupled look-back scan, AgentScan's tile_idx = blockIdx.x); the backward's re-store of the
// envelope takes an atomic ticket instead.
// The a^Ne correction term re-gathers e[n - Ne]; it is skipped when a^Ne < 1e-30.
#include <cuda/atomic>

#include <cstdlib>
#include "launch.hpp"

namespace mgb {

namespace {

struct DynParams {
  double da, doma, daN, da16, datile, datile32;  // the forward envelope scan runs in fp64
  float a, oma, aN, a16, atile, atile32;
  float T, W, R, invR, floor_;
  float knee;  // knee-curve coefficient: (1/R - 1) / (4W) compressor, (1 - R) / (4W) gate
  int Ne;
};

struct DynBwd {
  StepArgs fw, bw;     // forward (arena, forward CSR, params) / backward (input grads, consumer CSR)
  float* env;          // [seq][L] envelope from the forward scan; pass A overwrites it with the gain
  float* dg;           // [seq][L] dL/d(envelope)
  float2* agg;         // [seq][tiles] tile map vectors (pass 0)
  float2* carry;       // [seq][tiles] (w, v) at each tile's right end
  double* partial;     // [seq][tiles][5]
  int env_taps;
  double floor_;
  int tiles;
};

// a^n for an integer n >= 0 by squaring (<= 2 log2 n dependent fp64 multiplies; relative error
// ~n * 1e-16, the reference builds the same powers by repeated products). The fp64 pow() it
// replaces held every warp of a scan tile at the barrier behind warp 0 (28 % of the gate
// scan's stall samples).
__device__ __forceinline__ double ipow(double a, long n) {
  double r = 1.0;
  while (n > 0) {
    if (n & 1) r *= a;
    a *= a;
    n >>= 1;
  }
  return r;
}

// Slot constants, derived by warp 0 of each CTA: lanes 0-3 evaluate the four fp64 powers
// a^Ne, a^8, a^tile, a^(32 tile) side by side, lane 0 assembles.
__device__ __forceinline__ void derive_params(const double* row, int env_taps, double floor_, long L, int lane,
                                              DynParams* out, long tile = kDynTile, bool gate = false) {
  const double a = row[0];
  const int Ne = static_cast<int>(env_taps < L ? env_taps : L);
  const long e = lane == 0 ? static_cast<long>(Ne) : lane == 1 ? kDynPerThread : lane == 2 ? tile : 32L * tile;
  const double pw = lane < 4 ? ipow(a, e) : 0.0;
  const double aN = __shfl_sync(0xffffffffu, pw, 0), a16 = __shfl_sync(0xffffffffu, pw, 1);
  const double atile = __shfl_sync(0xffffffffu, pw, 2), atile32 = __shfl_sync(0xffffffffu, pw, 3);
  if (lane != 0) return;
  DynParams p;
  p.da = a;
  p.doma = 1.0 - a;
  p.daN = aN < 1e-30 ? 0.0 : aN;
  p.da16 = a16;
  p.datile = atile;
  p.datile32 = atile32;
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
  p.knee = static_cast<float>((gate ? 1.0 - row[3] : 1.0 / row[3] - 1.0) / (4.0 * row[2]));
  p.floor_ = static_cast<float>(floor_);
  *out = p;
}

// Gain exp(G_y - G_u) at envelope g (processors.cpp:71-130 knee curves), correctly rounded
// logf / expf (the MUFU approximations' ~5e-7 relative error reached the outputs: a gate
// with ratio R multiplies an error in G_u by R - 1), the knee's division folded into a
// per-slot coefficient. `gu_out` receives G_u (backward pass).
template <bool GATE>
__device__ __forceinline__ float gain_of(float g, const DynParams& p, float* gu_out = nullptr) {
  const float gu = logf(fmaxf(g, p.floor_));
  float gy;
  if (!GATE) {
    if (gu >= p.T + p.W) {
      gy = p.T + (gu - p.T) * p.invR;
    } else if (gu < p.T - p.W) {
      gy = gu;
    } else {
      const float d = gu - p.T + p.W;
      gy = fmaf(p.knee * d, d, gu);
    }
  } else {
    if (gu >= p.T + p.W) {
      gy = gu;
    } else if (gu < p.T - p.W) {
      gy = p.T + p.R * (gu - p.T);
    } else {
      const float d = gu - p.T - p.W;
      gy = fmaf(p.knee * d, d, gu);
    }
  }
  if (gu_out) *gu_out = gu;
  return expf(gy - gu);
}

// Gather-sum of the slot's inputs at kDynPerThread consecutive samples from n0.
template <bool VEC>
__device__ __forceinline__ void load16(const StepArgs& a, int e0, int e1, int b, long n0, float* ul, float* ur) {
#pragma unroll
  for (int k = 0; k < kDynPerThread; ++k) ul[k] = ur[k] = 0.f;
  if (n0 >= a.length || n0 < 0) return;
  const long boff = static_cast<long>(b) * 2 * a.length;
  if (VEC && n0 + kDynPerThread <= a.length && (a.length & 7) == 0) {  // 256-bit loads
    for (int e = e0; e < e1; ++e) {
      const float* p = a.src + edge_row(a, e) * a.rowstride + boff + n0;
      float vl[kDynPerThread], vr[kDynPerThread];
      ld8(p, vl);
      ld8(p + a.length, vr);
#pragma unroll
      for (int k = 0; k < kDynPerThread; ++k) {
        ul[k] += vl[k];
        ur[k] += vr[k];
      }
    }
    return;
  }
  if (VEC && n0 + kDynPerThread <= a.length) {
    for (int e = e0; e < e1; ++e) {
      const float* p = a.src + edge_row(a, e) * a.rowstride + boff + n0;
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
      const float* p = a.src + edge_row(a, e) * a.rowstride + boff;
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

// mid[k] = l + r of the gathered input at n0 + k (each channel summed in edge order first, as
// load16 does), four samples at a time, so only one float4 pair per channel is live.
template <bool VEC>
__device__ __forceinline__ void load_mid(const StepArgs& a, int e0, int e1, int b, long n0, float* mid) {
#pragma unroll
  for (int k = 0; k < kDynPerThread; ++k) mid[k] = 0.f;
  if (n0 >= a.length || n0 < 0) return;
  const long boff = static_cast<long>(b) * 2 * a.length;
  if (VEC && n0 + kDynPerThread <= a.length) {
#pragma unroll
    for (int q = 0; q < kDynPerThread / 4; ++q) {
      float4 l = make_float4(0.f, 0.f, 0.f, 0.f), r = l;
      for (int e = e0; e < e1; ++e) {
        const float* p = a.src + edge_row(a, e) * a.rowstride + boff + n0;
        l = f4add(l, __ldg(reinterpret_cast<const float4*>(p) + q));
        r = f4add(r, __ldg(reinterpret_cast<const float4*>(p + a.length) + q));
      }
      mid[4 * q] = l.x + r.x;
      mid[4 * q + 1] = l.y + r.y;
      mid[4 * q + 2] = l.z + r.z;
      mid[4 * q + 3] = l.w + r.w;
    }
  } else {
    float ul[kDynPerThread], ur[kDynPerThread];
    load16<false>(a, e0, e1, b, n0, ul, ur);
#pragma unroll
    for (int k = 0; k < kDynPerThread; ++k) mid[k] = ul[k] + ur[k];
  }
}

// load_mid that also stashes the gathered stereo input of this thread's kDynPerThread samples
// in shared memory (float4 groups at [q][NT]: consecutive threads, consecutive 16-byte words),
// so the output pass after the carry wait reads it back instead of gathering it again.
template <bool VEC, int NT>
__device__ __forceinline__ void load_tile(const StepArgs& a, int e0, int e1, int b, long n0, float* mid, float4* sl,
                                          float4* sr) {
  const int t = threadIdx.x;
  if (n0 >= a.length || n0 < 0) {
#pragma unroll
    for (int k = 0; k < kDynPerThread; ++k) mid[k] = 0.f;
    return;
  }
  const long boff = static_cast<long>(b) * 2 * a.length;
  if (VEC && n0 + kDynPerThread <= a.length && (a.length & 7) == 0) {
    // 256-bit loads (a warp reads 1 KiB contiguous per row and edge), summed in edge order
    float l[kDynPerThread], r[kDynPerThread];
#pragma unroll
    for (int k = 0; k < kDynPerThread; ++k) l[k] = r[k] = 0.f;
    for (int e = e0; e < e1; ++e) {
      const float* p = a.src + edge_row(a, e) * a.rowstride + boff + n0;
      float vl[kDynPerThread], vr[kDynPerThread];
      ld8(p, vl);
      ld8(p + a.length, vr);
#pragma unroll
      for (int k = 0; k < kDynPerThread; ++k) {
        l[k] += vl[k];
        r[k] += vr[k];
      }
    }
#pragma unroll
    for (int q = 0; q < kDynPerThread / 4; ++q) {
      sl[q * NT + t] = make_float4(l[4 * q], l[4 * q + 1], l[4 * q + 2], l[4 * q + 3]);
      sr[q * NT + t] = make_float4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
    }
#pragma unroll
    for (int k = 0; k < kDynPerThread; ++k) mid[k] = l[k] + r[k];
    return;
  }
  if (VEC && n0 + kDynPerThread <= a.length) {
#pragma unroll
    for (int q = 0; q < kDynPerThread / 4; ++q) {
      float4 l = make_float4(0.f, 0.f, 0.f, 0.f), r = l;
      for (int e = e0; e < e1; ++e) {
        const float* p = a.src + edge_row(a, e) * a.rowstride + boff + n0;
        l = f4add(l, __ldg(reinterpret_cast<const float4*>(p) + q));
        r = f4add(r, __ldg(reinterpret_cast<const float4*>(p + a.length) + q));
      }
      sl[q * NT + t] = l;
      sr[q * NT + t] = r;
      mid[4 * q] = l.x + r.x;
      mid[4 * q + 1] = l.y + r.y;
      mid[4 * q + 2] = l.z + r.z;
      mid[4 * q + 3] = l.w + r.w;
    }
  } else {
    float ul[kDynPerThread], ur[kDynPerThread];
    load16<false>(a, e0, e1, b, n0, ul, ur);
#pragma unroll
    for (int q = 0; q < kDynPerThread / 4; ++q) {
      sl[q * NT + t] = make_float4(ul[4 * q], ul[4 * q + 1], ul[4 * q + 2], ul[4 * q + 3]);
      sr[q * NT + t] = make_float4(ur[4 * q], ur[4 * q + 1], ur[4 * q + 2], ur[4 * q + 3]);
    }
#pragma unroll
    for (int k = 0; k < kDynPerThread; ++k) mid[k] = ul[k] + ur[k];
  }
}

template <typename T>
__device__ __forceinline__ void compose(T& A, T& B, T Ap, T Bp) {
  // earlier (Ap, Bp) then current (A, B)
  B = fma(A, Bp, B);
  A = A * Ap;
}

// ENV: also store the envelope g[n] to env[(slot*B + b)*L + n] (backward pass recompute).
// NT: threads per tile (tile = NT * kDynPerThread samples); 128 for steps with few sequences,
// so a single long sequence still spreads over the SMs.
template <bool GATE, bool VEC, bool ENV = false, int NT = kDynThreads>
__global__ void __launch_bounds__(NT, 2 * kDynThreads / NT) dyn_scan(StepArgs a, int env_taps, double floor_, int tiles_per_seq,
                                                         unsigned long long* status, unsigned int* ticket,
                                                         float* env, PwEpi epi) {
  __shared__ double wA[NT / 32], wB[NT / 32];
  __shared__ float4 s_in[2][kDynPerThread / 4][NT];  // the tile's gathered input (l, r), read once
  __shared__ double s_carry;
  __shared__ int s_ticket;
  __shared__ DynParams s_p;
  __shared__ PwEpiSlots s_epi;
  // Tickets interleave sequences (all tile-0s, then all tile-1s, ...): a tile's
  // predecessors were dispatched `nseq` tickets earlier, so the carry rarely waits.
  const int nseq = a.slots * a.batch;
  // Tile order: the block index (blocks are dispatched in index order, so every tile this
  // one waits on is resident or done, as in single-pass decoupled look-back scans), or with
  // `ticket` an atomic ticket (one L2 round trip and a barrier before any load).
  int tk = static_cast<int>(blockIdx.x);
  if (ticket != nullptr) {
    if (threadIdx.x == 0) s_ticket = static_cast<int>(atomicAdd(ticket, 1u));
    __syncthreads();
    tk = s_ticket;
  }
  const int tile = tk / nseq, seq = tk - tile * nseq;
  const int slot = seq / a.batch, b = seq - slot * a.batch;
  const int e0 = slot_e0(a, slot), e1 = slot_e1(a, slot);
  const DynParams& p = s_p;  // read from shared memory where used (frees registers)

  const long n0 = static_cast<long>(tile) * (NT * kDynPerThread) + static_cast<long>(threadIdx.x) * kDynPerThread;
  // drive[k] = (1-a) (e[n] - a^Ne e[n-Ne]) is all the scan keeps in registers; the gathered
  // input samples wait in shared memory for the output pass (read from memory once), so
  // nothing else stays live across the carry wait. The recurrence runs in fp64: with poles up
  // to a = 0.9995 an fp32 envelope accumulates ~eps / sqrt(2 (1 - a)) = 2e-6 relative error.
  double drive[kDynPerThread];
  {
    // The tile's own samples are requested first; warp 0 derives the slot constants (fp64
    // powers) while they are in flight, instead of every warp waiting for them at the barrier
    // before issuing any load (that barrier was 20 % of the stall samples).
    float mid[kDynPerThread];
    load_tile<VEC, NT>(a, e0, e1, b, n0, mid, &s_in[0][0][0], &s_in[1][0][0]);
    if (threadIdx.x < 32) {
      derive_params(a.params + 4L * slot, env_taps, floor_, a.length, threadIdx.x, &s_p, NT * kDynPerThread, GATE);
      if (epi.n > 0 && threadIdx.x == 1) pw_epi_slots(epi, slot, s_epi);
    }
    __syncthreads();
    if (p.daN != 0.0) {
      float mo[kDynPerThread];
      load_mid<VEC>(a, e0, e1, b, n0 - p.Ne, mo);
#pragma unroll
      for (int k = 0; k < kDynPerThread; ++k) {
        const double m = mid[k], o = mo[k];
        drive[k] = p.doma * (m * m - p.daN * (o * o));
      }
    } else {
#pragma unroll
      for (int k = 0; k < kDynPerThread; ++k) {
        const double m = mid[k];
        drive[k] = p.doma * (m * m);
      }
    }
  }

  // Thread-local recurrence from 0.
  double B = 0.0;
#pragma unroll
  for (int k = 0; k < kDynPerThread; ++k) B = fma(p.da, B, drive[k]);
  double A = p.da16;

  // Warp inclusive scan of affine maps.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double Ap = __shfl_up_sync(0xffffffffu, A, off);
    const double Bp = __shfl_up_sync(0xffffffffu, B, off);
    if (lane >= off) compose(A, B, Ap, Bp);
  }
  if (lane == 31) {
    wA[warp] = A;
    wB[warp] = B;
  }
  // Exclusive prefix within the warp.
  double xA = __shfl_up_sync(0xffffffffu, A, 1), xB = __shfl_up_sync(0xffffffffu, B, 1);
  if (lane == 0) {
    xA = 1.0;
    xB = 0.0;
  }
  __syncthreads();
  if (warp == 0) {
    double tA = lane < NT / 32 ? wA[lane] : 1.0;
    double tB = lane < NT / 32 ? wB[lane] : 0.0;
#pragma unroll
    for (int off = 1; off < NT / 32; off <<= 1) {
      const double Ap = __shfl_up_sync(0xffffffffu, tA, off);
      const double Bp = __shfl_up_sync(0xffffffffu, tB, off);
      if (lane >= off) compose(tA, tB, Ap, Bp);
    }
    if (lane < NT / 32) {
      wA[lane] = tA;  // inclusive warp-level prefix
      wB[lane] = tB;
    }
  }
  __syncthreads();
  if (warp > 0) {  // prepend the previous warps' prefix
    const double pA = wA[warp - 1], pB = wB[warp - 1];
    compose(xA, xB, pA, pB);
  }
  const double tileB = wB[NT / 32 - 1];

  if (warp == 0) {
    // Cross-tile carry, deterministic: publish this tile's aggregate B, then
    //   carry = sum_{d >= 0} A^d * B_{tile-1-d},   A = a^tile_len,
    // summed lane-strided (d = lane + 32 i) and tree-reduced in a fixed order. Only
    // aggregates are read (no chain of inclusive prefixes), so no tile waits on another
    // tile's look-back, and the value never depends on timing. Windows stop once the
    // largest remaining weight A^d underflows to exactly 0 (all later terms are +0).
    // status is indexed [seq][tile]: the fp64 aggregate's bits + 1 (0 = not yet published;
    // the +1 never wraps: an all-ones pattern is a NaN, which an aggregate is not)
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> mine(status[static_cast<long>(seq) * tiles_per_seq + tile]);
    if (lane == 0) {
      mine.store(static_cast<unsigned long long>(__double_as_longlong(tileB)) + 1ull, cuda::memory_order_relaxed);
    }
    double part = 0.0;
    // weight A^d = A^lane * (A^32)^(d0/32): one pow per lane, then exact-order products
    const double wl = tile > 0 ? ipow(p.datile, lane) : 0.0;
    double w32 = 1.0;  // (A^32)^(d0/32)
    for (int d0 = 0; d0 < tile; d0 += 32, w32 *= p.datile32) {
      if (w32 == 0.0) break;
      const int d = d0 + lane;
      if (d < tile) {
        cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> st(status[static_cast<long>(seq) * tiles_per_seq + tile - 1 - d]);
        unsigned long long w;
        do {
          w = st.load(cuda::memory_order_relaxed);
        } while (w == 0ull);
        part = fma(wl * w32, __longlong_as_double(static_cast<long long>(w - 1ull)), part);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
    if (lane == 0) s_carry = part;
  }
  __syncthreads();

  // Replay the recurrence from this thread's true start state, apply the gain, store.
  double g = fma(xA, s_carry, xB);
  if (n0 >= a.length) return;
  float* ol = a.dst + static_cast<long>(slot) * a.rowstride + static_cast<long>(b) * 2 * a.length + n0;
  float* orr = ol + a.length;
  const bool full = VEC && n0 + kDynPerThread <= a.length;
  if (full && (a.length & 7) == 0) {
    // 256-bit stores (a warp writes 1 KiB contiguous per row), followers included
    float yl[kDynPerThread], yr[kDynPerThread];
#pragma unroll
    for (int q = 0; q < kDynPerThread / 4; ++q) {
      const float4 l4 = s_in[0][q][threadIdx.x], r4 = s_in[1][q][threadIdx.x];
      const float ul[4] = {l4.x, l4.y, l4.z, l4.w}, ur[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        g = fma(p.da, g, drive[4 * q + k4]);
        const float gf = static_cast<float>(g);
        const float gn = gain_of<GATE>(gf, p);
        if constexpr (ENV) drive[4 * q + k4] = gf;  // drive[k] is consumed: reuse it for the envelope
        yl[4 * q + k4] = gn * ul[k4];
        yr[4 * q + k4] = gn * ur[k4];
      }
    }
    if constexpr (ENV) {
      float ev[kDynPerThread];
#pragma unroll
      for (int k = 0; k < kDynPerThread; ++k) ev[k] = static_cast<float>(drive[k]);
      st8(env + static_cast<long>(seq) * a.length + n0, ev);
    }
    st8(ol, yl);
    st8(orr, yr);
    for (int f = 0; f < epi.n; ++f) {
      const float g0 = s_epi.g0[f], g1 = s_epi.g1[f];
#pragma unroll
      for (int k = 0; k < kDynPerThread; ++k) {
        yl[k] = 0.f + yl[k];
        yr[k] = 0.f + yr[k];
        pw_op(epi.op[f], yl[k], yr[k], g0, g1);
      }
      float* fo = epi.dst[f] + static_cast<long>(s_epi.slot[f]) * a.rowstride + static_cast<long>(b) * 2 * a.length + n0;
      st8(fo, yl);
      st8(fo + a.length, yr);
    }
    return;
  }
#pragma unroll
  for (int q = 0; q < kDynPerThread / 4; ++q) {
    // this thread's own stashed input, four samples at a time (no barrier: written by itself)
    const float4 l4 = s_in[0][q][threadIdx.x], r4 = s_in[1][q][threadIdx.x];
    const float ul[4] = {l4.x, l4.y, l4.z, l4.w}, ur[4] = {r4.x, r4.y, r4.z, r4.w};
    float yl[4], yr[4], ev[4];
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4) {
      const int k = 4 * q + k4;
      g = fma(p.da, g, drive[k]);
      const float gf = static_cast<float>(g);
      ev[k4] = gf;
      const float gn = gain_of<GATE>(gf, p);
      yl[k4] = gn * ul[k4];
      yr[k4] = gn * ur[k4];
    }
    if constexpr (ENV) {  // the envelope for the backward pass, four samples per store
      float* e = env + static_cast<long>(seq) * a.length + n0 + 4 * q;
      if (full) {
        *reinterpret_cast<float4*>(e) = make_float4(ev[0], ev[1], ev[2], ev[3]);
      } else {
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
          if (n0 + 4 * q + k4 < a.length) e[k4] = ev[k4];
        }
      }
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
    if (epi.n > 0) {
      const long nq = n0 + 4 * q;
      const long left = a.length - nq;
      pw_epi_apply(epi, s_epi, a.rowstride, a.length, static_cast<long>(b) * 2 * a.length + nq, yl, yr, full,
                   left < 0 ? 0 : (left < 4 ? static_cast<int>(left) : 4));
    }
  }
}

// ---- streaming scan: one CTA per sequence (steps with many sequences) ----------------------
//
// When a step has at least a full wave of sequences (a config-5 union's 1,124 track
// compressors), each CTA owns one (slot, batch) sequence and walks its tiles in order: the
// carry into tile t is the CTA's own running state (carry = a^tile * carry + B_tile, fp64), so
// there is no look-back, no status words and no cross-CTA waiting. The input rows are streamed
// into a 3-stage shared-memory ring by the bulk-copy engine (cp.async.bulk, one elected thread,
// mbarrier completion), two tiles ahead of the scan, so every CTA keeps 32 KB of loads in
// flight while it scans and stores. One block barrier per tile: the stage a tile was read from
// is refilled after the next tile's barrier, and the per-warp aggregates alternate between two
// buffers. Arithmetic per sample is dyn_scan's (fp64 recurrence, correctly rounded gain).
// Needs a dense step (slot s reads row dense + s) and L % 4 == 0 (16-byte bulk copies).
// 128-thread CTAs (1024-sample tiles, 24 KB ring): eight per SM, so a config-5 union's 1,124
// sequences are one wave (256-thread CTAs, four per SM, left a 1.9-wave tail).
constexpr int kStreamThreads = 128;
constexpr int kStreamDepth = 3;
constexpr int kStreamTile = kStreamThreads * kDynPerThread;
constexpr int kStreamSmem = kStreamDepth * 2 * kStreamTile * static_cast<int>(sizeof(float));
constexpr int kStreamCtasPerSm = 8;

// NF: pointwise followers in the epilogue (compile time: their row pointers and coefficients
// are per-CTA constants in registers; six CTAs per SM leave room for them).
template <bool GATE, bool VEC, int NF>
__global__ void __launch_bounds__(kStreamThreads, NF == 0 ? kStreamCtasPerSm : 6) dyn_stream(StepArgs a, int env_taps, double floor_, PwEpi epi) {
  constexpr int NT = kStreamThreads, TS = kStreamTile, NW = NT / 32;
  extern __shared__ __align__(128) unsigned char stream_smem[];
  float* ring = reinterpret_cast<float*>(stream_smem);  // [stage][channel][TS]
  __shared__ __align__(8) unsigned long long bar[kStreamDepth];
  __shared__ double wA[2][NW], wB[2][NW];
  __shared__ DynParams s_p;
  __shared__ PwEpiSlots s_epi;
  const int seq = blockIdx.x;
  const int slot = seq / a.batch, b = seq - slot * a.batch;
  const long L = a.length;
  const long boff = static_cast<long>(b) * 2 * L;
  const float* in = a.src + (static_cast<long>(a.dense) + slot) * a.rowstride + boff;
  const int tiles = static_cast<int>((L + TS - 1) / TS);
  auto issue = [&](int t) {
    const int st = t % kStreamDepth;
    const long n0 = static_cast<long>(t) * TS;
    const uint32_t bytes = static_cast<uint32_t>(min(static_cast<long>(TS), L - n0)) * 4u;
    float* dst = ring + st * 2 * TS;
    mbar_expect_tx(&bar[st], 2 * bytes);
    bulk_g2s(dst, in + n0, bytes, &bar[st]);
    bulk_g2s(dst + TS, in + L + n0, bytes, &bar[st]);
  };
  if (threadIdx.x == 0) {
#pragma unroll
    for (int d = 0; d < kStreamDepth; ++d) mbar_init(&bar[d], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int t = 0; t < kStreamDepth && t < tiles; ++t) issue(t);
  }
  if (threadIdx.x < 32) {
    derive_params(a.params + 4L * slot, env_taps, floor_, L, threadIdx.x, &s_p, TS, GATE);
    if (epi.n > 0 && threadIdx.x == 1) pw_epi_slots(epi, slot, s_epi);
  }
  __syncthreads();
  const DynParams p = s_p;  // registers: the per-sample gain reads them every sample
  float* fdst[NF > 0 ? NF : 1];
  float fg0[NF > 0 ? NF : 1], fg1[NF > 0 ? NF : 1];
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    fdst[f] = epi.dst[f] + static_cast<long>(s_epi.slot[f]) * a.rowstride + boff;
    fg0[f] = s_epi.g0[f];
    fg1[f] = s_epi.g1[f];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int e0 = slot_e0(a, slot), e1 = slot_e1(a, slot);
  float* ol0 = a.dst + static_cast<long>(slot) * a.rowstride + boff;
  double carry = 0.0;
  for (int t = 0; t < tiles; ++t) {
    const int st = t % kStreamDepth;
    const long n0 = static_cast<long>(t) * TS + static_cast<long>(threadIdx.x) * kDynPerThread;
    const bool live = n0 < L;  // L % 4 == 0: a live thread has 4 or 8 valid samples
    const bool full = n0 + kDynPerThread <= L;
    mbar_wait(&bar[st], static_cast<uint32_t>((t / kStreamDepth) & 1));
    const float* sl = ring + st * 2 * TS + threadIdx.x * kDynPerThread;
    double drive[kDynPerThread];
    {
      float mid[kDynPerThread];
#pragma unroll
      for (int q = 0; q < kDynPerThread / 4; ++q) {
        float4 l = make_float4(0.f, 0.f, 0.f, 0.f), r = l;
        if (live && (q == 0 || full)) {
          l = *reinterpret_cast<const float4*>(sl + 4 * q);
          r = *reinterpret_cast<const float4*>(sl + TS + 4 * q);
        }
        // the gather of one row is 0 + x (dyn_scan's edge-order sum)
        mid[4 * q] = (0.f + l.x) + (0.f + r.x);
        mid[4 * q + 1] = (0.f + l.y) + (0.f + r.y);
        mid[4 * q + 2] = (0.f + l.z) + (0.f + r.z);
        mid[4 * q + 3] = (0.f + l.w) + (0.f + r.w);
      }
      if (p.daN != 0.0) {
        float mo[kDynPerThread];
        load_mid<VEC>(a, e0, e1, b, live ? n0 - p.Ne : L, mo);
#pragma unroll
        for (int k = 0; k < kDynPerThread; ++k) {
          const double m = mid[k], o = mo[k];
          drive[k] = p.doma * (m * m - p.daN * (o * o));
        }
      } else {
#pragma unroll
        for (int k = 0; k < kDynPerThread; ++k) {
          const double m = mid[k];
          drive[k] = p.doma * (m * m);
        }
      }
    }
    double B = 0.0;
#pragma unroll
    for (int k = 0; k < kDynPerThread; ++k) B = fma(p.da, B, drive[k]);
    double A = p.da16;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const double Ap = __shfl_up_sync(0xffffffffu, A, off);
      const double Bp = __shfl_up_sync(0xffffffffu, B, off);
      if (lane >= off) compose(A, B, Ap, Bp);
    }
    if (lane == 31) {
      wA[t & 1][warp] = A;
      wB[t & 1][warp] = B;
    }
    double xA = __shfl_up_sync(0xffffffffu, A, 1), xB = __shfl_up_sync(0xffffffffu, B, 1);
    if (lane == 0) {
      xA = 1.0;
      xB = 0.0;
    }
    __syncthreads();
    // Every thread of tile t - 1 is past its output pass: refill its stage two tiles ahead.
    if (threadIdx.x == 0 && t >= 1 && t - 1 + kStreamDepth < tiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(t - 1 + kStreamDepth);
    }
    // Prefix of the earlier warps (in order) and the tile's aggregate, the same values in every thread.
    double pA = 1.0, pB = 0.0, tB = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const double Aw = wA[t & 1][w], Bw = wB[t & 1][w];
      if (w < warp) {
        pB = fma(Aw, pB, Bw);
        pA = Aw * pA;
      }
      tB = fma(Aw, tB, Bw);
    }
    compose(xA, xB, pA, pB);
    double g = fma(xA, carry, xB);
    carry = fma(p.datile, carry, tB);
    if (!live) continue;
    float* ol = ol0 + n0;
    float* orr = ol + L;
    if (full && (L & 7) == 0) {  // 256-bit stores: a warp writes 1 KiB contiguous per row
      float yl[kDynPerThread], yr[kDynPerThread];
#pragma unroll
      for (int k = 0; k < kDynPerThread; ++k) {
        g = fma(p.da, g, drive[k]);
        const float gn = gain_of<GATE>(static_cast<float>(g), p);
        yl[k] = gn * (0.f + sl[k]);
        yr[k] = gn * (0.f + sl[TS + k]);
      }
      st8(ol, yl);
      st8(orr, yr);
#pragma unroll
      for (int f = 0; f < NF; ++f) {
#pragma unroll
        for (int k = 0; k < kDynPerThread; ++k) {
          yl[k] = 0.f + yl[k];
          yr[k] = 0.f + yr[k];
          pw_op(epi.op[f], yl[k], yr[k], fg0[f], fg1[f]);
        }
        st8(fdst[f] + n0, yl);
        st8(fdst[f] + L + n0, yr);
      }
      continue;
    }
#pragma unroll
    for (int q = 0; q < kDynPerThread / 4; ++q) {
      if (q > 0 && !full) break;
      const float4 l4 = *reinterpret_cast<const float4*>(sl + 4 * q);
      const float4 r4 = *reinterpret_cast<const float4*>(sl + TS + 4 * q);
      const float ul[4] = {0.f + l4.x, 0.f + l4.y, 0.f + l4.z, 0.f + l4.w};
      const float ur[4] = {0.f + r4.x, 0.f + r4.y, 0.f + r4.z, 0.f + r4.w};
      float yl[4], yr[4];
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        g = fma(p.da, g, drive[4 * q + k4]);
        const float gn = gain_of<GATE>(static_cast<float>(g), p);
        yl[k4] = gn * ul[k4];
        yr[k4] = gn * ur[k4];
      }
      reinterpret_cast<float4*>(ol)[q] = make_float4(yl[0], yl[1], yl[2], yl[3]);
      reinterpret_cast<float4*>(orr)[q] = make_float4(yr[0], yr[1], yr[2], yr[3]);
#pragma unroll
      for (int f = 0; f < NF; ++f) {  // the followers' arithmetic of pw_epi_apply
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          yl[k] = 0.f + yl[k];
          yr[k] = 0.f + yr[k];
          pw_op(epi.op[f], yl[k], yr[k], fg0[f], fg1[f]);
        }
        reinterpret_cast<float4*>(fdst[f] + n0)[q] = make_float4(yl[0], yl[1], yl[2], yl[3]);
        reinterpret_cast<float4*>(fdst[f] + L + n0)[q] = make_float4(yr[0], yr[1], yr[2], yr[3]);
      }
    }
  }
}

// Two streaming scans in one CTA: step A (compressor or noisegate) and step B reading exactly
// A's output rows (slot s of B reads row A.store_begin + s: a console track's compressor ->
// noisegate). Per tile the CTA scans A on its streamed input, stores A's output and keeps it
// in registers, then scans B on that output (its own running carry) and stores B's output and
// B's epilogue followers: A's rows are never read back (one read of the track signal for
// both), and one launch instead of two. Arithmetic per sample as dyn_scan / dyn_stream
// (B's gather of one row is 0 + y, kept). The block scan of one tile, shared by both stages:
// returns this thread's start state and advances the CTA's carry (one barrier).
template <int NW>
__device__ __forceinline__ double stream_block_scan(const double (&drive)[kDynPerThread], const DynParams& p,
                                                    double& carry, double (*wA)[NW], double (*wB)[NW], int t,
                                                    int lane, int warp) {
  double B = 0.0;
#pragma unroll
  for (int k = 0; k < kDynPerThread; ++k) B = fma(p.da, B, drive[k]);
  double A = p.da16;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double Ap = __shfl_up_sync(0xffffffffu, A, off);
    const double Bp = __shfl_up_sync(0xffffffffu, B, off);
    if (lane >= off) compose(A, B, Ap, Bp);
  }
  if (lane == 31) {
    wA[t & 1][warp] = A;
    wB[t & 1][warp] = B;
  }
  double xA = __shfl_up_sync(0xffffffffu, A, 1), xB = __shfl_up_sync(0xffffffffu, B, 1);
  if (lane == 0) {
    xA = 1.0;
    xB = 0.0;
  }
  __syncthreads();
  double pA = 1.0, pB = 0.0, tB = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const double Aw = wA[t & 1][w], Bw = wB[t & 1][w];
    if (w < warp) {
      pB = fma(Aw, pB, Bw);
      pA = Aw * pA;
    }
    tB = fma(Aw, tB, Bw);
  }
  compose(xA, xB, pA, pB);
  const double g = fma(xA, carry, xB);
  carry = fma(p.datile, carry, tB);
  return g;
}

// drive[k] = (1-a) (mid^2 - a^Ne mo^2) for this thread's samples (mo: mid at n - Ne).
__device__ __forceinline__ void stream_drive(const float (&mid)[kDynPerThread], const float (&mo)[kDynPerThread],
                                             const DynParams& p, double (&drive)[kDynPerThread]) {
#pragma unroll
  for (int k = 0; k < kDynPerThread; ++k) {
    const double m = mid[k], o = mo[k];
    drive[k] = p.daN != 0.0 ? p.doma * (m * m - p.daN * (o * o)) : p.doma * (m * m);
  }
}

template <bool GATE1, bool GATE2, int NF>
__global__ void __launch_bounds__(kStreamThreads, 6) dyn_stream_pair(StepArgs a1, StepArgs a2, int env_taps,
                                                                     double floor_, PwEpi epi) {
  constexpr int NT = kStreamThreads, TS = kStreamTile, NW = NT / 32, K = kDynPerThread;
  extern __shared__ __align__(128) unsigned char stream_smem[];
  float* ring = reinterpret_cast<float*>(stream_smem);  // [stage][channel][TS]
  __shared__ __align__(8) unsigned long long bar[kStreamDepth];
  __shared__ double wA1[2][NW], wB1[2][NW], wA2[2][NW], wB2[2][NW];
  __shared__ DynParams s_p1, s_p2;
  __shared__ PwEpiSlots s_epi;
  const int seq = blockIdx.x;
  const int slot = seq / a1.batch, b = seq - slot * a1.batch;
  const long L = a1.length;
  const long boff = static_cast<long>(b) * 2 * L;
  const float* in = a1.src + (static_cast<long>(a1.dense) + slot) * a1.rowstride + boff;
  float* y1 = a1.dst + static_cast<long>(slot) * a1.rowstride + boff;  // A's output row (B's input)
  float* y2 = a2.dst + static_cast<long>(slot) * a2.rowstride + boff;
  const int tiles = static_cast<int>((L + TS - 1) / TS);
  auto issue = [&](int t) {
    const int st = t % kStreamDepth;
    const long n0 = static_cast<long>(t) * TS;
    const uint32_t bytes = static_cast<uint32_t>(min(static_cast<long>(TS), L - n0)) * 4u;
    float* dst = ring + st * 2 * TS;
    mbar_expect_tx(&bar[st], 2 * bytes);
    bulk_g2s(dst, in + n0, bytes, &bar[st]);
    bulk_g2s(dst + TS, in + L + n0, bytes, &bar[st]);
  };
  if (threadIdx.x == 0) {
#pragma unroll
    for (int d = 0; d < kStreamDepth; ++d) mbar_init(&bar[d], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int t = 0; t < kStreamDepth && t < tiles; ++t) issue(t);
  }
  if (threadIdx.x < 32) {
    derive_params(a1.params + 4L * slot, env_taps, floor_, L, threadIdx.x, &s_p1, TS, GATE1);
  } else if (threadIdx.x < 64) {
    derive_params(a2.params + 4L * slot, env_taps, floor_, L, threadIdx.x - 32, &s_p2, TS, GATE2);
    if (epi.n > 0 && threadIdx.x == 33) pw_epi_slots(epi, slot, s_epi);
  }
  __syncthreads();
  float* fdst[NF > 0 ? NF : 1];
  float fg0[NF > 0 ? NF : 1], fg1[NF > 0 ? NF : 1];
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    fdst[f] = epi.dst[f] + static_cast<long>(s_epi.slot[f]) * a2.rowstride + boff;
    fg0[f] = s_epi.g0[f];
    fg1[f] = s_epi.g1[f];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool wide = (L & 7) == 0;  // 32-byte aligned rows: 256-bit stores
  double carry1 = 0.0, carry2 = 0.0;
  for (int t = 0; t < tiles; ++t) {
    const int st = t % kStreamDepth;
    const long n0 = static_cast<long>(t) * TS + static_cast<long>(threadIdx.x) * K;
    const bool live = n0 < L;  // L % 4 == 0: a live thread has 4 or 8 valid samples
    const bool full = n0 + K <= L;
    mbar_wait(&bar[st], static_cast<uint32_t>((t / kStreamDepth) & 1));
    const float* sl = ring + st * 2 * TS + threadIdx.x * K;
    float ul[K], ur[K];
    double drive[K];
    {
      float mid[K], mo[K];
#pragma unroll
      for (int q = 0; q < K / 4; ++q) {
        float4 l = make_float4(0.f, 0.f, 0.f, 0.f), r = l;
        if (live && (q == 0 || full)) {
          l = *reinterpret_cast<const float4*>(sl + 4 * q);
          r = *reinterpret_cast<const float4*>(sl + TS + 4 * q);
        }
        const float lv[4] = {0.f + l.x, 0.f + l.y, 0.f + l.z, 0.f + l.w}, rv[4] = {0.f + r.x, 0.f + r.y, 0.f + r.z, 0.f + r.w};
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
          ul[4 * q + k4] = lv[k4];
          ur[4 * q + k4] = rv[k4];
          mid[4 * q + k4] = lv[k4] + rv[k4];
        }
      }
      const DynParams& p1 = s_p1;
#pragma unroll
      for (int k = 0; k < K; ++k) mo[k] = 0.f;
      if (p1.daN != 0.0) {
        if ((p1.Ne & 3) == 0) load_mid<true>(a1, slot, slot + 1, b, live ? n0 - p1.Ne : L, mo);
        else load_mid<false>(a1, slot, slot + 1, b, live ? n0 - p1.Ne : L, mo);
      }
      stream_drive(mid, mo, p1, drive);
    }
    double g = stream_block_scan<NW>(drive, s_p1, carry1, wA1, wB1, t, lane, warp);
    // Every thread of tile t - 1 is past its output pass: refill its stage two tiles ahead.
    if (threadIdx.x == 0 && t >= 1 && t - 1 + kStreamDepth < tiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(t - 1 + kStreamDepth);
    }
    // Stage A: gains, A's output (kept in ul / ur), stored.
    {
      const DynParams& p1 = s_p1;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        g = fma(p1.da, g, drive[k]);
        const float gn = gain_of<GATE1>(static_cast<float>(g), p1);
        ul[k] *= gn;
        ur[k] *= gn;
      }
    }
    if (live && full && wide) {  // one 256-bit store per channel: a warp writes 1 KiB contiguous
      st8(y1 + n0, ul);
      st8(y1 + L + n0, ur);
    } else if (live) {
#pragma unroll
      for (int q = 0; q < K / 4; ++q) {
        if (q > 0 && !full) break;
        reinterpret_cast<float4*>(y1 + n0)[q] = make_float4(ul[4 * q], ul[4 * q + 1], ul[4 * q + 2], ul[4 * q + 3]);
        reinterpret_cast<float4*>(y1 + L + n0)[q] = make_float4(ur[4 * q], ur[4 * q + 1], ur[4 * q + 2], ur[4 * q + 3]);
      }
    }
    // Stage B on A's output: B's gather of one row is 0 + y.
    {
      const DynParams& p2 = s_p2;
      float mid[K], mo[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        ul[k] = 0.f + ul[k];
        ur[k] = 0.f + ur[k];
        mid[k] = live && (k < 4 || full) ? ul[k] + ur[k] : 0.f;
        mo[k] = 0.f;
      }
      if (p2.daN != 0.0) {  // A's output at n - Ne: this CTA stored it (at least Ne samples back)
        __syncthreads();
        if ((p2.Ne & 3) == 0) load_mid<true>(a2, slot, slot + 1, b, live ? n0 - p2.Ne : L, mo);
        else load_mid<false>(a2, slot, slot + 1, b, live ? n0 - p2.Ne : L, mo);
      }
      stream_drive(mid, mo, p2, drive);
    }
    g = stream_block_scan<NW>(drive, s_p2, carry2, wA2, wB2, t, lane, warp);
    if (!live) continue;
    if (full && wide) {
      const DynParams& p2 = s_p2;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        g = fma(p2.da, g, drive[k]);
        const float gn = gain_of<GATE2>(static_cast<float>(g), p2);
        ul[k] *= gn;
        ur[k] *= gn;
      }
      st8(y2 + n0, ul);
      st8(y2 + L + n0, ur);
#pragma unroll
      for (int f = 0; f < NF; ++f) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
          ul[k] = 0.f + ul[k];
          ur[k] = 0.f + ur[k];
          pw_op(epi.op[f], ul[k], ur[k], fg0[f], fg1[f]);
        }
        st8(fdst[f] + n0, ul);
        st8(fdst[f] + L + n0, ur);
      }
      continue;
    }
    {
      const DynParams& p2 = s_p2;
#pragma unroll
      for (int q = 0; q < K / 4; ++q) {
        if (q > 0 && !full) break;
        float yl[4], yr[4];
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
          const int k = 4 * q + k4;
          g = fma(p2.da, g, drive[k]);
          const float gn = gain_of<GATE2>(static_cast<float>(g), p2);
          yl[k4] = gn * ul[k];
          yr[k4] = gn * ur[k];
        }
        reinterpret_cast<float4*>(y2 + n0)[q] = make_float4(yl[0], yl[1], yl[2], yl[3]);
        reinterpret_cast<float4*>(y2 + L + n0)[q] = make_float4(yr[0], yr[1], yr[2], yr[3]);
#pragma unroll
        for (int f = 0; f < NF; ++f) {
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            yl[k4] = 0.f + yl[k4];
            yr[k4] = 0.f + yr[k4];
            pw_op(epi.op[f], yl[k4], yr[k4], fg0[f], fg1[f]);
          }
          reinterpret_cast<float4*>(fdst[f] + n0)[q] = make_float4(yl[0], yl[1], yl[2], yl[3]);
          reinterpret_cast<float4*>(fdst[f] + L + n0)[q] = make_float4(yr[0], yr[1], yr[2], yr[3]);
        }
      }
    }
  }
}

// ---- backward (parameter gradients; no reference counterpart, see backward.cu) -------------
//
// Given dy (gathered over the consumers' input gradients) and the forward quantities
// (u gathered from the arena, envelope g stored by dyn_scan<.., ENV>):
//   gain = exp(G_y - G_u), dD = (dy_l u_l + dy_r u_r) gain, dG_u = dD (dG_y/dG_u - 1),
//   dg = dG_u / g (g above the floor, else 0),
//   w[m] = a w[m+1] + dg[m] - a^Ne dg[m+Ne]                (de = (1-a) w),
//   v[m] = a v[m+1] + w[m+1] - Ne a^(Ne-1) dg[m+Ne]        (v = d w / d a),
//   du_c = gain dy_c + 2 mid de,
//   d a = -sum dg g / (1-a) + (1-a) sum e v,  dT/dW/dR = sum dD dG_y/d{T,W,R}.
// (w, v) is a reverse scan of affine maps with matrix [[a,0],[1,a]]^k = [[a^k,0],[k a^(k-1),a^k]].
// Passes: the forward scan re-stores the envelope; A computes dg (stored) and the gain (over
// the envelope); B reduces each tile to its map; dyn_bwd_carry chains the tiles per sequence
// (fp64, serial, fixed order); D replays each tile from its carry. Deterministic.
struct DynMap {
  float p, q, cw, cv;
};
// A o B (B applied first)
__device__ __forceinline__ DynMap dmap_compose(const DynMap& A, const DynMap& B) {
  DynMap r;
  r.p = A.p * B.p;
  r.q = fmaf(A.q, B.p, A.p * B.q);
  r.cw = fmaf(A.p, B.cw, A.cw);
  r.cv = fmaf(A.q, B.cw, fmaf(A.p, B.cv, A.cv));
  return r;
}
__device__ __forceinline__ DynMap dmap_shfl_down(const DynMap& m, int off) {
  DynMap r;
  r.p = __shfl_down_sync(0xffffffffu, m.p, off);
  r.q = __shfl_down_sync(0xffffffffu, m.q, off);
  r.cw = __shfl_down_sync(0xffffffffu, m.cw, off);
  r.cv = __shfl_down_sync(0xffffffffu, m.cv, off);
  return r;
}

// Knee derivatives at G = G_u: returns dG_y/dG_u, accumulates dG_y/d{T,W,R} * dD.
template <bool GATE>
__device__ __forceinline__ float knee_grad(float gu, const DynParams& p, float dD, float* acc) {
  if (!GATE) {
    if (gu >= p.T + p.W) {
      acc[0] += dD * (1.f - p.invR);
      acc[2] += dD * (-(gu - p.T) * p.invR * p.invR);
      return p.invR;
    }
    if (gu < p.T - p.W) return 1.f;
    const float d = gu - p.T + p.W, k = p.invR - 1.f, h = d / (2.f * p.W);
    acc[0] += dD * (-k * h);
    acc[1] += dD * (k * (h - h * h));
    acc[2] += dD * (-(d * d) / (4.f * p.W) * p.invR * p.invR);
    return 1.f + k * h;
  }
  if (gu >= p.T + p.W) return 1.f;
  if (gu < p.T - p.W) {
    acc[0] += dD * (1.f - p.R);
    acc[2] += dD * (gu - p.T);
    return p.R;
  }
  const float d = gu - p.T - p.W, k = 1.f - p.R, h = d / (2.f * p.W);
  acc[0] += dD * (-k * h);
  acc[1] += dD * (k * (-h - h * h));
  acc[2] += dD * (-(d * d) / (4.f * p.W));
  return 1.f + k * h;
}

// Pass A: per sample dg = dG_u / g and the gain (overwrites the stored envelope in place),
// per-tile partial sums of dD dG_y/d{T,W,R} and dg g. grid (tiles, seqs)
template <bool GATE, bool VEC>
__global__ void __launch_bounds__(kDynThreads, 2) dyn_bwd_dg(DynBwd d) {
  __shared__ DynParams s_p;
  __shared__ double red[kDynThreads / 32][4];
  const int tile = blockIdx.x, seq = blockIdx.y;
  const int slot = seq / d.fw.batch, b = seq - slot * d.fw.batch;
  if (threadIdx.x < 32) derive_params(d.fw.params + 4L * slot, d.env_taps, d.floor_, d.fw.length, threadIdx.x, &s_p, kDynTile, GATE);
  __syncthreads();
  const DynParams& p = s_p;  // read from shared memory where used (frees registers)
  const long L = d.fw.length;
  const long n0 = static_cast<long>(tile) * kDynTile + static_cast<long>(threadIdx.x) * kDynPerThread;
  constexpr int K = kDynPerThread;
  float ul[K], ur[K], dyl[K], dyr[K];
  load16<VEC>(d.fw, __ldg(d.fw.row_ptr + slot), __ldg(d.fw.row_ptr + slot + 1), b, n0, ul, ur);
  load16<VEC>(d.bw, __ldg(d.bw.row_ptr + slot), __ldg(d.bw.row_ptr + slot + 1), b, n0, dyl, dyr);
  float acc[3] = {0.f, 0.f, 0.f};
  float dgg = 0.f;
  float* env = d.env + static_cast<long>(seq) * L;
  float* dgo = d.dg + static_cast<long>(seq) * L;
  // The thread's envelope samples in, its gains and dg out, four at a time as float4 when all
  // four are in range (scalar accesses at an 8-sample stride made every warp access touch 32
  // sectors).
#pragma unroll
  for (int q = 0; q < K / 4; ++q) {
    const long nq = n0 + 4 * q;
    const bool full = VEC && nq + 4 <= L;
    float gv[4], go[4], dv[4];
    if (full) {
      const float4 a4 = *reinterpret_cast<const float4*>(env + nq);
      gv[0] = a4.x; gv[1] = a4.y; gv[2] = a4.z; gv[3] = a4.w;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) gv[k] = nq + k < L ? env[nq + k] : 1.f;
    }
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4) {
      const int k = 4 * q + k4;
      go[k4] = 0.f;
      dv[k4] = 0.f;
      if (nq + k4 >= L) continue;
      const float g = gv[k4];
      float gu;
      const float gain = gain_of<GATE>(g, p, &gu);  // the forward's own arithmetic
      const float dD = (dyl[k] * ul[k] + dyr[k] * ur[k]) * gain;
      const float slope = knee_grad<GATE>(gu, p, dD, acc);
      const float dg = g > p.floor_ ? dD * (slope - 1.f) / g : 0.f;
      dgg += dg * g;
      go[k4] = gain;
      dv[k4] = dg;
    }
    if (full) {
      *reinterpret_cast<float4*>(env + nq) = make_float4(go[0], go[1], go[2], go[3]);
      *reinterpret_cast<float4*>(dgo + nq) = make_float4(dv[0], dv[1], dv[2], dv[3]);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (nq + k < L) {
          env[nq + k] = go[k];
          dgo[nq + k] = dv[k];
        }
      }
    }
  }
  double vals[4] = {acc[0], acc[1], acc[2], dgg};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) vals[j] += __shfl_xor_sync(0xffffffffu, vals[j], off);
  }
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) red[warp][j] = vals[j];
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double t = 0.0;
    for (int w = 0; w < kDynThreads / 32; ++w) t += red[w][threadIdx.x];
    d.partial[(static_cast<long>(seq) * d.tiles + tile) * 5 + threadIdx.x] = t;
  }
}

// dg at kDynPerThread samples from n0 (0 outside [0, L)); VEC: n0 is a multiple of 4.
template <bool VEC>
__device__ __forceinline__ void load_dg(const float* dg, long L, long n0, float* v) {
  if (VEC && n0 >= 0 && n0 + kDynPerThread <= L && ((L | n0) & 7) == 0) {  // 256-bit load
    float t[kDynPerThread];
    ld8(dg + n0, t);
#pragma unroll
    for (int k = 0; k < kDynPerThread; ++k) v[k] = t[k];
    return;
  }
  if (VEC && n0 >= 0 && n0 + kDynPerThread <= L) {
#pragma unroll
    for (int q = 0; q < kDynPerThread / 4; ++q) {
      const float4 f = __ldg(reinterpret_cast<const float4*>(dg + n0) + q);
      v[4 * q] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < kDynPerThread; ++k) {
    const long n = n0 + k;
    v[k] = (n >= 0 && n < L) ? __ldg(dg + n) : 0.f;
  }
}

// Passes B (PASS 0: tile maps) and D (PASS 1: replay from the carry, du, sum e v) of the
// reverse scan. grid (tiles, seqs)
template <bool VEC, int PASS>
__global__ void __launch_bounds__(kDynThreads, 2) dyn_bwd(DynBwd d) {
  __shared__ DynParams s_p;
  __shared__ DynMap wmap[kDynThreads / 32];
  __shared__ float2 s_carry;
  __shared__ double red[kDynThreads / 32];
  const int tile = blockIdx.x, seq = blockIdx.y;
  const int slot = seq / d.fw.batch, b = seq - slot * d.fw.batch;
  if (threadIdx.x < 32) derive_params(d.fw.params + 4L * slot, d.env_taps, d.floor_, d.fw.length, threadIdx.x, &s_p);
  if (PASS == 1 && threadIdx.x == 0) s_carry = d.carry[static_cast<long>(seq) * d.tiles + tile];
  __syncthreads();
  const DynParams& p = s_p;  // read from shared memory where used (frees registers)
  const long L = d.fw.length;
  const long n0 = static_cast<long>(tile) * kDynTile + static_cast<long>(threadIdx.x) * kDynPerThread;
  constexpr int K = kDynPerThread;
  const float* dgs = d.dg + static_cast<long>(seq) * L;
  // a_k = dg[n] - a^Ne dg[n+Ne], b_k = -Ne a^(Ne-1) dg[n+Ne] (skipped when a^Ne < 1e-30).
  float av[K], bv[K];
  load_dg<VEC>(dgs, L, n0, av);
  if (p.aN != 0.f) {
    float t2[K];
    load_dg<VEC>(dgs, L, n0 + p.Ne, t2);
    const float nb = static_cast<float>(p.Ne) * p.aN / p.a;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      av[k] -= p.aN * t2[k];
      bv[k] = -nb * t2[k];
    }
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k) bv[k] = 0.f;
  }
  DynMap m;
  {
    float cw = 0.f, cv = 0.f;
#pragma unroll
    for (int k = K - 1; k >= 0; --k) {
      cv = fmaf(p.a, cv, cw + bv[k]);
      cw = fmaf(p.a, cw, av[k]);
    }
    m.p = p.a16;
    m.q = static_cast<float>(K) * p.a16 / p.a;
    m.cw = cw;
    m.cv = cv;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  DynMap inc = m;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const DynMap o = dmap_shfl_down(inc, off);
    if (lane + off < 32) inc = dmap_compose(inc, o);
  }
  if (lane == 0) wmap[warp] = inc;
  DynMap exc = dmap_shfl_down(inc, 1);
  if (lane == 31) exc = DynMap{1.f, 0.f, 0.f, 0.f};
  __syncthreads();
  if (warp == 0) {
    constexpr int NW = kDynThreads / 32;
    DynMap t = lane < NW ? wmap[lane] : DynMap{1.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int off = 1; off < NW; off <<= 1) {
      const DynMap o = dmap_shfl_down(t, off);
      if (lane + off < NW) t = dmap_compose(t, o);
    }
    if (lane < NW) wmap[lane] = t;
  }
  __syncthreads();
  if constexpr (PASS == 0) {
    if (threadIdx.x == 0) d.agg[static_cast<long>(seq) * d.tiles + tile] = make_float2(wmap[0].cw, wmap[0].cv);
  } else {
    float w = s_carry.x, v = s_carry.y;
    if (warp + 1 < kDynThreads / 32) {
      const DynMap t = wmap[warp + 1];
      const float w2 = fmaf(t.p, w, t.cw);
      v = fmaf(t.q, w, fmaf(t.p, v, t.cv));
      w = w2;
    }
    {
      const float w2 = fmaf(exc.p, w, exc.cw);
      v = fmaf(exc.q, w, fmaf(exc.p, v, exc.cv));
      w = w2;
    }
    // Replay right to left: w[m], v[m] per sample.
    float wv[K], vv[K];
#pragma unroll
    for (int k = K - 1; k >= 0; --k) {
      const float vn = fmaf(p.a, v, w + bv[k]);
      w = fmaf(p.a, w, av[k]);
      v = vn;
      wv[k] = w;
      vv[k] = v;
    }
    float ul[K], ur[K], dyl[K], dyr[K];
    load16<VEC>(d.fw, __ldg(d.fw.row_ptr + slot), __ldg(d.fw.row_ptr + slot + 1), b, n0, ul, ur);
    load16<VEC>(d.bw, __ldg(d.bw.row_ptr + slot), __ldg(d.bw.row_ptr + slot + 1), b, n0, dyl, dyr);
    const float* gain = d.env + static_cast<long>(seq) * L;
    float* dl = d.bw.dst + static_cast<long>(slot) * d.bw.rowstride + static_cast<long>(b) * 2 * L;
    float* dr = dl + L;
    double ev = 0.0;
#pragma unroll
    for (int q = 0; q < K / 4; ++q) {
      const long nq = n0 + 4 * q;
      const bool full = VEC && nq + 4 <= L;
      float gn[4], ol[4], orr[4];
      if (full) {
        const float4 g4 = __ldg(reinterpret_cast<const float4*>(gain + nq));  // the gains pass A stored
        gn[0] = g4.x; gn[1] = g4.y; gn[2] = g4.z; gn[3] = g4.w;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) gn[k] = nq + k < L ? __ldg(gain + nq + k) : 0.f;
      }
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        const int k = 4 * q + k4;
        ol[k4] = orr[k4] = 0.f;
        if (nq + k4 >= L) continue;
        const float mid = ul[k] + ur[k];
        const float dmid = 2.f * mid * (p.oma * wv[k]);
        ol[k4] = fmaf(gn[k4], dyl[k], dmid);
        orr[k4] = fmaf(gn[k4], dyr[k], dmid);
        ev += static_cast<double>(mid * mid) * vv[k];
      }
      if (full) {
        *reinterpret_cast<float4*>(dl + nq) = make_float4(ol[0], ol[1], ol[2], ol[3]);
        *reinterpret_cast<float4*>(dr + nq) = make_float4(orr[0], orr[1], orr[2], orr[3]);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (nq + k < L) {
            dl[nq + k] = ol[k];
            dr[nq + k] = orr[k];
          }
        }
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, off);
    if (lane == 0) red[warp] = ev;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w2 = 0; w2 < kDynThreads / 32; ++w2) t += red[w2];
      d.partial[(static_cast<long>(seq) * d.tiles + tile) * 5 + 4] = t;
    }
  }
}

// Per sequence: chain the tile maps from the last tile back (fp64), state at each tile's right end.
__global__ void dyn_bwd_carry(DynBwd d, int nseq) {
  const int seq = blockIdx.x * blockDim.x + threadIdx.x;
  if (seq >= nseq) return;
  const int slot = seq / d.fw.batch;
  const double a = d.fw.params[4L * slot];
  const double pT = pow(a, static_cast<double>(kDynTile));
  const double qT = static_cast<double>(kDynTile) * pow(a, static_cast<double>(kDynTile - 1));
  double w = 0.0, v = 0.0;
  for (int t = d.tiles - 1; t >= 0; --t) {
    const long i = static_cast<long>(seq) * d.tiles + t;
    d.carry[i] = make_float2(static_cast<float>(w), static_cast<float>(v));
    const float2 c = d.agg[i];
    const double w2 = pT * w + c.x;
    v = qT * w + pT * v + c.y;
    w = w2;
  }
}

// grid (slots) x 32: sum the partials over batch and tiles (fixed order) into the grad row.
__global__ void dyn_bwd_reduce(DynBwd d, double* grad) {
  const int slot = blockIdx.x;
  const int lane = threadIdx.x;
  double s[5] = {0, 0, 0, 0, 0};
  const long n = static_cast<long>(d.fw.batch) * d.tiles;
  for (long i = lane; i < n; i += 32) {
    const double* q = d.partial + (static_cast<long>(slot) * n + i) * 5;
#pragma unroll
    for (int j = 0; j < 5; ++j) s[j] += q[j];
  }
#pragma unroll
  for (int j = 0; j < 5; ++j) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s[j] += __shfl_xor_sync(0xffffffffu, s[j], off);
  }
  if (lane != 0) return;
  const double a = d.fw.params[4L * slot];
  double* g = grad + 4L * slot;
  g[0] = -s[3] / (1.0 - a) + (1.0 - a) * s[4];
  g[1] = s[0];
  g[2] = s[1];
  g[3] = s[2];
}

}  // namespace

std::size_t dyn_bwd_bytes(int slots, int batch, long length) {
  const std::size_t seqs = static_cast<std::size_t>(slots) * batch;
  const std::size_t tiles = static_cast<std::size_t>((length + kDynTile - 1) / kDynTile);
  auto al = [](std::size_t x) { return (x + 255) & ~static_cast<std::size_t>(255); };
  return 2 * al(sizeof(float) * seqs * length) + 2 * al(sizeof(float2) * seqs * tiles) +
         al(sizeof(double) * 5 * seqs * tiles) + dyn_sync_bytes(slots, batch, length);
}

void launch_dynamics_backward(bool gate, const StepArgs& fw, const StepArgs& bw, int envelope_taps,
                              double energy_floor, void* ws, double* grad, cudaStream_t s) {
  if (fw.slots == 0 || fw.batch == 0 || fw.length == 0) return;
  auto al = [](std::size_t x) { return (x + 255) & ~static_cast<std::size_t>(255); };
  const int tiles = static_cast<int>((fw.length + kDynTile - 1) / kDynTile);
  const std::size_t seqs = static_cast<std::size_t>(fw.slots) * fw.batch;
  char* p = static_cast<char*>(ws);
  DynBwd d;
  d.fw = fw;
  d.bw = bw;
  d.env = reinterpret_cast<float*>(p);
  p += al(sizeof(float) * seqs * fw.length);
  d.dg = reinterpret_cast<float*>(p);
  p += al(sizeof(float) * seqs * fw.length);
  d.agg = reinterpret_cast<float2*>(p);
  p += al(sizeof(float2) * seqs * tiles);
  d.carry = reinterpret_cast<float2*>(p);
  p += al(sizeof(float2) * seqs * tiles);
  d.partial = reinterpret_cast<double*>(p);
  p += al(sizeof(double) * 5 * seqs * tiles);
  d.env_taps = envelope_taps;
  d.floor_ = energy_floor;
  d.tiles = tiles;
  // 1. Re-run the forward scan storing the envelope (outputs rewritten bit-identically).
  cudaMemsetAsync(p, 0, dyn_sync_bytes(fw.slots, fw.batch, fw.length), s);
  auto* ticket = reinterpret_cast<unsigned int*>(p);
  auto* status = reinterpret_cast<unsigned long long*>(p + 256);
  const long ne = envelope_taps < fw.length ? envelope_taps : fw.length;
  const bool vec = (fw.length % 4 == 0) && (ne % 4 == 0);
  const dim3 fgrid(static_cast<unsigned>(seqs * tiles));
  float* env = d.env;
  const dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(seqs));
#define MGB_DYN_BWD(G, V)                                                                                  \
  dyn_scan<G, V, true><<<fgrid, kDynThreads, 0, s>>>(fw, envelope_taps, energy_floor, tiles, status, ticket, env, PwEpi{}); \
  dyn_bwd_dg<G, V><<<grid, kDynThreads, 0, s>>>(d);                                                        \
  dyn_bwd<V, 0><<<grid, kDynThreads, 0, s>>>(d);                                                            \
  dyn_bwd_carry<<<static_cast<unsigned>((seqs + 127) / 128), 128, 0, s>>>(d, static_cast<int>(seqs));        \
  dyn_bwd<V, 1><<<grid, kDynThreads, 0, s>>>(d);
  if (gate) {
    if (vec) { MGB_DYN_BWD(true, true) } else { MGB_DYN_BWD(true, false) }
  } else {
    if (vec) { MGB_DYN_BWD(false, true) } else { MGB_DYN_BWD(false, false) }
  }
#undef MGB_DYN_BWD
  dyn_bwd_reduce<<<fw.slots, 32, 0, s>>>(d, grad);
}

constexpr int kDynSmallThreads = 128;
// Forward tiles of 256 threads (2048 samples) for steps with many waves of tiles.
constexpr int kDynFwdThreads = 256;
constexpr int kDynSmallTile = kDynSmallThreads * kDynPerThread;

std::size_t dyn_sync_bytes(int slots, int batch, long length) {
  const long tiles = (length + 32 * kDynPerThread - 1) / (32 * kDynPerThread);  // the finest tiling (32 threads)
  return 256 + sizeof(unsigned long long) * static_cast<std::size_t>(slots) * batch * tiles;
}

// The streaming scan (one CTA per sequence) when the step has most of a wave of sequences at
// eight (six with epilogue followers) CTAs per SM, its slots read consecutive rows and the rows are 16-byte aligned (L % 4 == 0).
// (mg_set_dyn_stream: 0 forces the chained scan, for tests.)
static int g_dyn_stream = -1;
static int g_dyn_pair = -1;
void set_dyn_stream(int mode) { g_dyn_stream = mode; }
void set_dyn_pair(int mode) { g_dyn_pair = mode; }
static int sm_count_dyn() {
  static const int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}
bool dyn_stream_ok(const StepArgs& a, const PwEpi& epi) {
  if (g_dyn_stream == 0 || a.dense < 0 || a.length % 4 != 0) return false;
  return g_dyn_stream == 1 || static_cast<long>(a.slots) * a.batch >= 6L * sm_count_dyn();
}

bool dyn_pair_shape(int slots, int batch, long length) {
  return g_dyn_stream != 0 && g_dyn_pair != 0 && length % 4 == 0 &&
         (g_dyn_stream == 1 || static_cast<long>(slots) * batch >= 6L * sm_count_dyn());
}

bool dyn_pair_ok(const StepArgs& a1, const StepArgs& a2) {
  if (g_dyn_stream == 0 || g_dyn_pair == 0 || !dyn_stream_ok(a1, PwEpi{}) || !dyn_stream_ok(a2, PwEpi{})) return false;
  // B reads exactly A's rows slot by slot
  return a1.slots == a2.slots && a1.batch == a2.batch && a1.length == a2.length &&
         a2.src + static_cast<long>(a2.dense) * a2.rowstride == a1.dst;
}

void launch_dynamics_pair(bool gate1, bool gate2, const StepArgs& a1, const StepArgs& a2, int envelope_taps,
                          double energy_floor, cudaStream_t s, const PwEpi& epi) {
  const long seqs = static_cast<long>(a1.slots) * a1.batch;
  if (seqs == 0 || a1.length == 0) return;
  static const bool attr = [] {
    for (auto fn : {dyn_stream_pair<false, false, 0>, dyn_stream_pair<false, false, 1>, dyn_stream_pair<false, false, 2>,
                    dyn_stream_pair<false, false, 3>, dyn_stream_pair<false, true, 0>, dyn_stream_pair<false, true, 1>,
                    dyn_stream_pair<false, true, 2>, dyn_stream_pair<false, true, 3>, dyn_stream_pair<true, false, 0>,
                    dyn_stream_pair<true, false, 1>, dyn_stream_pair<true, false, 2>, dyn_stream_pair<true, false, 3>,
                    dyn_stream_pair<true, true, 0>, dyn_stream_pair<true, true, 1>, dyn_stream_pair<true, true, 2>,
                    dyn_stream_pair<true, true, 3>}) {
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kStreamSmem);
    }
    return true;
  }();
  (void)attr;
  const dim3 grid(static_cast<unsigned>(seqs));
  auto go = [&](auto fn) { fn<<<grid, kStreamThreads, kStreamSmem, s>>>(a1, a2, envelope_taps, energy_floor, epi); };
#define MGB_DYN_PAIR(G1, G2)                         \
  switch (epi.n) {                                   \
    case 0: go(dyn_stream_pair<G1, G2, 0>); break;   \
    case 1: go(dyn_stream_pair<G1, G2, 1>); break;   \
    case 2: go(dyn_stream_pair<G1, G2, 2>); break;   \
    default: go(dyn_stream_pair<G1, G2, 3>); break;  \
  }
  if (gate1) {
    if (gate2) { MGB_DYN_PAIR(true, true) } else { MGB_DYN_PAIR(true, false) }
  } else {
    if (gate2) { MGB_DYN_PAIR(false, true) } else { MGB_DYN_PAIR(false, false) }
  }
#undef MGB_DYN_PAIR
}

void launch_dynamics(bool gate, const StepArgs& a, int envelope_taps, double energy_floor, void* ws,
                     bool zero_sync, cudaStream_t s, const PwEpi& epi) {
  if (a.slots == 0 || a.batch == 0 || a.length == 0) return;
  const long seqs = static_cast<long>(a.slots) * a.batch;
  // Few sequences (a bus compressor): 1024-sample tiles of 128 threads, so the step still
  // spreads over the SMs; otherwise 4096-sample tiles of 512 threads. (One-warp tiles measured
  // no faster on config 2 and their longer fp32 carry sums lose accuracy.)
  const long big_tiles = seqs * ((a.length + kDynTile - 1) / kDynTile);
  const bool small = big_tiles < 148;
  // Many waves of tiles (config-5 unions): 256-thread tiles, so four CTAs per SM interleave
  // their load / scan / carry-wait phases (98.7 vs 101.5 ms per 512-graph step). A few waves
  // (config 2's 16 tracks): 512-thread tiles (256 measured 0.211 -> 0.216 ms per render).
  const bool narrow = big_tiles >= 8L * 2 * 148;
  const long tile = static_cast<long>(small ? kDynSmallThreads : (narrow ? kDynFwdThreads : kDynThreads)) * kDynPerThread;
  const int tiles = static_cast<int>((a.length + tile - 1) / tile);
  const long total = seqs * tiles;
  if (zero_sync) cudaMemsetAsync(ws, 0, dyn_sync_bytes(a.slots, a.batch, a.length), s);
  auto* status = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + 256);
  const long ne = envelope_taps < a.length ? envelope_taps : a.length;
  const bool vec = (a.length % 4 == 0) && (ne % 4 == 0);
  if (dyn_stream_ok(a, epi)) {
    const dim3 sgrid(static_cast<unsigned>(seqs));
    static const bool attr = [] {
      for (auto fn : {dyn_stream<false, false, 0>, dyn_stream<false, false, 1>, dyn_stream<false, false, 2>,
                      dyn_stream<false, false, 3>, dyn_stream<false, true, 0>, dyn_stream<false, true, 1>,
                      dyn_stream<false, true, 2>, dyn_stream<false, true, 3>, dyn_stream<true, false, 0>,
                      dyn_stream<true, false, 1>, dyn_stream<true, false, 2>, dyn_stream<true, false, 3>,
                      dyn_stream<true, true, 0>, dyn_stream<true, true, 1>, dyn_stream<true, true, 2>,
                      dyn_stream<true, true, 3>}) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kStreamSmem);
      }
      return true;
    }();
    (void)attr;
    auto go = [&](auto fn) { fn<<<sgrid, kStreamThreads, kStreamSmem, s>>>(a, envelope_taps, energy_floor, epi); };
#define MGB_DYN_STREAM(G, V)                          \
  switch (epi.n) {                                    \
    case 0: go(dyn_stream<G, V, 0>); break;           \
    case 1: go(dyn_stream<G, V, 1>); break;           \
    case 2: go(dyn_stream<G, V, 2>); break;           \
    default: go(dyn_stream<G, V, 3>); break;          \
  }
    if (gate) {
      if (vec) { MGB_DYN_STREAM(true, true) } else { MGB_DYN_STREAM(true, false) }
    } else {
      if (vec) { MGB_DYN_STREAM(false, true) } else { MGB_DYN_STREAM(false, false) }
    }
#undef MGB_DYN_STREAM
    return;
  }
  const dim3 grid(static_cast<unsigned>(total));
#define MGB_DYN_LAUNCH(G, V, T) \
  dyn_scan<G, V, false, T><<<grid, T, 0, s>>>(a, envelope_taps, energy_floor, tiles, status, nullptr, nullptr, epi)
  if (small) {
    if (gate) {
      if (vec) MGB_DYN_LAUNCH(true, true, kDynSmallThreads); else MGB_DYN_LAUNCH(true, false, kDynSmallThreads);
    } else {
      if (vec) MGB_DYN_LAUNCH(false, true, kDynSmallThreads); else MGB_DYN_LAUNCH(false, false, kDynSmallThreads);
    }
  } else if (narrow) {
    if (gate) {
      if (vec) MGB_DYN_LAUNCH(true, true, kDynFwdThreads); else MGB_DYN_LAUNCH(true, false, kDynFwdThreads);
    } else {
      if (vec) MGB_DYN_LAUNCH(false, true, kDynFwdThreads); else MGB_DYN_LAUNCH(false, false, kDynFwdThreads);
    }
  } else {
    if (gate) {
      if (vec) MGB_DYN_LAUNCH(true, true, kDynThreads); else MGB_DYN_LAUNCH(true, false, kDynThreads);
    } else {
      if (vec) MGB_DYN_LAUNCH(false, true, kDynThreads); else MGB_DYN_LAUNCH(false, false, kDynThreads);
    }
  }
#undef MGB_DYN_LAUNCH
}

}  // namespace mgb
