// Per-warp TMA slot ring of the L2-streamed kernels (fb_stream_kernel,
// fb_streamsplit_kernel).
//
// Every frame re-reads the same slot rows of a warp's tiles, so each warp
// streams them into a private ring of NSLOT chunks (ROWS x 256 B each,
// cp.async.bulk completing on one mbarrier per slot) that runs NSLOT chunks
// ahead of the arc loop — across tile and frame boundaries — instead of a
// dependent L2 load per row.  The chunks of one frame are listed once per
// phase in a per-warp table ({slot offset into the pack, bytes}), so the
// producer (lane 0) is a table read plus the bulk copy.  Counters are
// absolute (never reset): slot = g % NSLOT, wait parity = (g / NSLOT) & 1,
// across phases and utterances.  All addresses are 32-bit shared-window
// addresses (one register each, no generic-to-shared conversion in the loop).
#pragma once

#include "lfmmi_device.cuh"
#include "lfmmi_tile_common.cuh"

namespace lfmmi {

template <int NSLOT, int ROWS, int CHUNKS>
struct SlotRing {
  static_assert(ROWS >= 1 && NSLOT >= 1, "ring shape");
  static constexpr unsigned kSlotBytes = unsigned(ROWS) * 256u;
  // (32-bit shared addresses and no cached lane id: the 1024-thread kernels
  // using the ring run under a 64-register cap)
  uint32_t ring32 = 0, bars32 = 0;  // this warp's slots / mbarriers
  uint32_t ctab32 = 0;              // this warp's chunk table (CHUNKS x {offset, bytes})
  const uint2 *pack = nullptr;
  unsigned g_cons = 0, g_iss = 0, g_end = 0;  // chunks consumed / issued / phase end
  int p_i = 0, nchunk = 0;
  __device__ __forceinline__ static int lane_id() { return int(threadIdx.x & 31u); }

  // Shared bytes for NW warps: slots, barriers, chunk tables.
  __host__ __device__ static constexpr unsigned slot_bytes(int nw) {
    return unsigned(nw) * NSLOT * kSlotBytes;
  }
  __host__ __device__ static constexpr unsigned bar_bytes(int nw) {
    return unsigned(nw) * NSLOT * 8u;
  }
  __host__ __device__ static constexpr unsigned table_bytes(int nw) {
    return unsigned(nw) * CHUNKS * 8u;
  }

  __device__ __forceinline__ void init(unsigned char *slots, unsigned char *bars,
                                       unsigned char *tables, int warp) {
    ring32 = smem_u32(slots) + unsigned(warp) * (NSLOT * kSlotBytes);
    bars32 = smem_u32(bars) + unsigned(warp) * (NSLOT * 8u);
    ctab32 = smem_u32(tables) + unsigned(warp) * (CHUNKS * 8u);
  }
  // Once per CTA before first use (then a CTA barrier): one arrival per phase.
  __device__ static void init_barriers(unsigned char *bars, int nw, int tid) {
    if (tid < nw * NSLOT) mbar_init(reinterpret_cast<unsigned long long *>(bars) + tid, 1);
    mbar_init_fence();
  }
  __device__ __forceinline__ uint32_t slot(unsigned g) const {
    return ring32 + (g % NSLOT) * kSlotBytes;
  }
  __device__ __forceinline__ uint32_t bar(unsigned g) const { return bars32 + (g % NSLOT) * 8u; }

  __device__ __forceinline__ void issue() {
    if (lane_id() == 0) {
      const uint2 ent = lds_v2(ctab32 + unsigned(p_i) * 8u);
      fence_proxy_async_smem();  // earlier LDS of this slot before the async refill
      bulk_copy_g2s(slot(g_iss), pack + ent.x, ent.y, bar(g_iss));
    }
    ++g_iss;
    if (++p_i == nchunk) p_i = 0;
  }
  // A phase of `frames` frames over the pack pk: this warp's ntw tiles, tile i's
  // trips / base held by lane i.  Needs every chunk of the previous phase
  // consumed (or drained).  The table holds CHUNKS entries (the launchers check
  // ring_chunks_needed against it).
  __device__ __forceinline__ void begin(const uint2 *pk, int ntw, int my_trips, int my_base,
                                        int frames) {
    pack = pk;
    p_i = 0;
    int c = 0;
    for (int i = 0; i < ntw; ++i) {
      const int tr = __shfl_sync(kFull, my_trips, i);
      const int bs = __shfl_sync(kFull, my_base, i);
      for (int j0 = 0; j0 < tr; j0 += ROWS, ++c)
        if (lane_id() == 0 && c < CHUNKS)
          sts_v2(ctab32 + unsigned(c) * 8u,
                 make_uint2(unsigned(bs + 32 * j0), unsigned(min(ROWS, tr - j0)) * 256u));
    }
    if (c > CHUNKS) __trap();  // launcher bug: the table cannot hold this warp's chunks
    nchunk = c;
    __syncwarp();
    g_end = g_iss + unsigned(c) * unsigned(max(frames, 0));
    for (int q = 0; q < NSLOT && g_iss < g_end; ++q) issue();
  }
  // Wait for the copies still in flight (a phase left early).
  __device__ __forceinline__ void drain() {
    for (; g_cons < g_iss; ++g_cons) mbar_wait(bar(g_cons), (g_cons / NSLOT) & 1u);
    __syncwarp();
  }
  // Arc rows [0, trips) of the current tile: body(w) per slot word of this lane.
  // Full chunks run unguarded (straight-line arc bodies); rows past the tail
  // are stale ring words that are loaded but never used.
  template <class Body>
  __device__ __forceinline__ void rows(int trips, Body &&body) {
    for (int j0 = 0; j0 < trips; j0 += ROWS) {
      mbar_wait(bar(g_cons), (g_cons / NSLOT) & 1u);
      const uint32_t sl = slot(g_cons) + unsigned(lane_id()) * 8u;
      const int n = min(ROWS, trips - j0);
      // two halves: the first half's arc bodies run while the second half's
      // words are loaded, with half the word registers live (the 1024-thread
      // kernels are capped at 64 registers and otherwise re-derive addresses)
      constexpr int H = ROWS / 2 > 0 ? ROWS / 2 : 1;
      uint2 w[H];
#pragma unroll
      for (int r = 0; r < H; ++r) w[r] = lds_v2(sl + unsigned(r) * 256u);
      if (n == ROWS) {
#pragma unroll
        for (int r = 0; r < H; ++r) body(w[r]);
      } else {
#pragma unroll
        for (int r = 0; r < H; ++r)
          if (r < n) body(w[r]);
      }
#pragma unroll
      for (int r = H; r < ROWS; ++r) w[r - H] = lds_v2(sl + unsigned(r) * 256u);
      __syncwarp();  // every lane has its words: the slot may be refilled
      ++g_cons;
      if (g_iss < g_end) issue();
      if (n == ROWS) {
#pragma unroll
        for (int r = H; r < ROWS; ++r) body(w[r - H]);
      } else {
#pragma unroll
        for (int r = H; r < ROWS; ++r)
          if (r < n) body(w[r - H]);
      }
    }
  }
};

// Chunks of one frame for the warp that carries the most: the ring's table
// must hold them (host-side check of the launchers).
inline int ring_chunks_needed(int tiles_per_warp, int max_deg, int rows) {
  return tiles_per_warp * ((max_deg + rows - 1) / rows);
}

}  // namespace lfmmi
