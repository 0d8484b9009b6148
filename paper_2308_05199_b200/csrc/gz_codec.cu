// gz_codec.cu -- sm_100a kernels of the B200 gZCCL codec and the fused ring
// reduce-scatter step.  See gz_device.cuh for the layout and numerics.
//
//   k_tile_encode<SRC_PLAIN>  compress  (codec.py:149-270), also N segments
//                             in one launch (compress_blocks, codec.py:408-427)
//   k_tile_encode<SRC_STEP>   fused RS step: compress(op(local, decompress(recv)))
//                             (collectives.py:274-290) in one kernel
//   k_tile_decode             decompress with sidecar offsets (codec.py:284-369)
//
// Every kernel is a persistent grid of independent warps; a warp owns one
// 32-block tile at a time and never waits on a CTA-wide barrier.
#include "gz_device.cuh"

namespace gz {

enum { SRC_PLAIN = 0, SRC_STEP = 1 };
#ifndef GZ_DIAG_STAMPS
#define GZ_DIAG_STAMPS 0  // diagnostic builds only (tools/exp/gather_stamps.py)
#endif
#if GZ_DIAG_STAMPS
__device__ unsigned long long g_gst[3 * 8192];   // per gather group: start, base known, copied
__device__ unsigned long long g_est[256 * 32];   // per encoder warp: end of its tile loop
#endif
// report_base value of a kernel whose `local` is NOT the caller's input (e.g. a
// recursive-doubling step reducing into its output in place): nothing is reported
constexpr uint64_t NO_REPORT = ~0ull;
enum { OP_SUM = 0, OP_MAX = 1 };

// One independently compressed blob (a compress_blocks segment).
struct Seg {
  const float* x;          // values (plain) / local chunk (step)
  uint64_t n;
  uint8_t* blob;           // header at 0, payload at 24; 16-byte aligned (may be a peer pointer)
  uint64_t* out_len;       // 24 + payload bytes
  uint64_t* out_tile_off;  // sidecar: [ntiles + 1] payload offsets of tiles
  uint8_t* out_w;          // sidecar: [ntiles * TB] width byte of every block (0..32 or 255)
  uint64_t cta_base;       // first encoder CTA of this segment
  uint64_t gcta_base;      // first gather group of this segment
  uint64_t gcta_n;         // gather groups of this segment
  uint64_t tile_base;      // first slot of this segment in tile_rel / scratch
  uint64_t report_base;    // offset of x[0] in the caller's buffer (first_nonfinite reports)
};

template <int NSEG>
struct EncodeArgs {
  Seg seg[NSEG];
  int nseg;
  uint64_t nctas;          // encoder CTAs (== grid), split over segments by cta_base
  uint64_t ngctas;         // gather groups (one warp each), 2^gshift tiles each, split by gcta_base
  uint32_t gshift;         // log2(tiles per gather group), 0..10
  uint64_t total_tiles;    // tiles over all segments
  QParams qp;
  uint64_t* blk_off;       // optional per-block payload offsets (segment 0 only)
  TileWs* ws;
  uint32_t* tile_rel;      // per tile: compressed size (phase A -> phase B)
  uint8_t* scratch;        // per tile one TILE_SLOT-byte slot (16-byte aligned)
  Status* st;
  // fused step only (NSEG == 1)
  const uint8_t* in_blob;  // received blob (header + payload)
  const uint64_t* in_tile_off;
  const uint8_t* in_w;
  const uint8_t* in_slots; // or: received tiles in slotted form (tile t at t * TILE_SLOT) ...
  const uint32_t* in_sizes;//     ... with their sizes (in_tile_off unused)
  double in_tw;
  int op;
  float* acc_out;          // optional: reduced values (f32)
  int slotted_out;         // 1: the output stays in slotted form (scratch/tile_rel), no gather
  unsigned int* post_flag; // slotted only, may be null: set to 1 once the whole output is written
  unsigned int* wait_flag; // slotted only, may be null: wait until >= 1 before reading inputs, reset to 0
};



// Fused step: the local values are loaded for the current tile only and the
// received tile's bytes staged alongside (one value buffer, one staging
// buffer per warp): 24 warps per SM hide the latency better than 16
// double-buffered or 13 fully asynchronous warps (measured, profiles/).
constexpr int ENC_WARP_SMEM = TILE_VALUES * 4 + STAGE_BYTES;
#ifndef GZ_STEP_L2PF
#define GZ_STEP_L2PF 1
#endif
constexpr bool L2PF = GZ_STEP_L2PF;  // fused step: L2 prefetch of the next tile
// warps per encoder CTA (one CTA per SM): as many as shared memory allows
// (18 warps with double-buffered local values: 2^25 peer step 114 -> 121 us)
__host__ __device__ constexpr int enc_warps(int src) { return 24; }
__host__ __device__ constexpr int enc_warp_smem(int src) { return src == 1 ? ENC_WARP_SMEM : 2 * TILE_VALUES * 4; }

// -------------------------------------------------------------------------
// small helpers
__device__ __forceinline__ uint32_t lds_u32u(const uint32_t* w, int off) {
  const int i = off >> 2, sh = (off & 3) * 8;
  return __funnelshift_r(w[i], w[i + 1], sh);
}
__device__ __forceinline__ uint64_t lds_u64u(const uint32_t* w, int off) {
  const int i = off >> 2, sh = (off & 3) * 8;
  const uint32_t a = w[i], b = w[i + 1], c = w[i + 2];
  return (uint64_t)__funnelshift_r(a, b, sh) | ((uint64_t)__funnelshift_r(b, c, sh) << 32);
}

__device__ __forceinline__ float np_maximum(float a, float b) {  // collectives.py:38
  return isnan(a) ? a : (a > b ? a : b);
}

// (block << 24) | (width << 8) | code; the smallest block index wins
__device__ __forceinline__ void record_decode_error(Status* st, uint64_t block, unsigned code, int w = 0) {
  atomicMin(&st->decode_error, (unsigned long long)((block << 24) | ((uint64_t)(w & 0xFFFF) << 8) | code));
}

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Wait (thread 0) until *flag >= 1, written by a peer GPU; a release/acquire
// pair with the producer's __threadfence_system + store.  Bounded: a flag
// that never arrives makes the wait give up after GZ_FLAG_TIMEOUT_NS and
// report it (the caller skips its work and records comm_error) instead of
// hanging the GPU.
constexpr unsigned long long FLAG_TIMEOUT_NS = 20000000000ull;
__device__ __forceinline__ bool wait_flag_sys(const unsigned int* flag) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
  if (v >= 1u) return true;
  const unsigned long long t0 = gtimer();
  do {
    __nanosleep(64);
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (gtimer() - t0 > FLAG_TIMEOUT_NS) return false;
  } while (v < 1u);
  return true;
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Warp-synchronous coalesced write of the tile to dst[v0, v0+nval).
__device__ __forceinline__ void drain_values(const float* xs, float* __restrict__ dst, uint64_t v0, int nval, int lane) {
  float* p = dst + v0;
  if (nval == TILE_VALUES && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
    float4* p4 = reinterpret_cast<float4*>(p);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = lane + 32 * j;
      __stcs(p4 + i, *reinterpret_cast<const float4*>(xs + xs_index(i >> 3, i & 7)));
    }
  } else {
    for (int i = lane; i < nval; i += 32) {
      const int row = i >> 5, col = i & 31;
      __stcs(p + i, xs[xs_index(row, col >> 2) + (col & 3)]);
    }
  }
}

__device__ __forceinline__ float np_maximum_f(float a, float b) {  // collectives.py:38
  return isnan(a) ? a : (a > b ? a : b);
}

// dst = op(local, decoded) (collectives.py:32-39, local first), coalesced.
// A non-finite local value is reported like the encoder does (the last step
// of a standalone reduce-scatter is the only place that reads its chunk).
__device__ __forceinline__ void drain_values_op(const float* xs, const float* __restrict__ local, int op,
                                                float* __restrict__ dst, uint64_t v0, int nval, int lane,
                                                Status* st, uint64_t report_base) {
  bool bad = false;
  if (nval == TILE_VALUES && (((reinterpret_cast<uintptr_t>(local + v0) | reinterpret_cast<uintptr_t>(dst + v0)) & 15) == 0)) {
    // full, aligned tile: float4 loads / stores (like drain_values)
    const float4* l4 = reinterpret_cast<const float4*>(local + v0);
    float4* d4 = reinterpret_cast<float4*>(dst + v0);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = lane + 32 * j;
      const float4 d = *reinterpret_cast<const float4*>(xs + xs_index(i >> 3, i & 7));
      const float4 l = __ldcs(l4 + i);
      bad |= !(isfinite(l.x) && isfinite(l.y) && isfinite(l.z) && isfinite(l.w));
      float4 o;
      if (op == 0) {
        o.x = __fadd_rn(l.x, d.x); o.y = __fadd_rn(l.y, d.y); o.z = __fadd_rn(l.z, d.z); o.w = __fadd_rn(l.w, d.w);
      } else {
        o.x = np_maximum_f(l.x, d.x); o.y = np_maximum_f(l.y, d.y); o.z = np_maximum_f(l.z, d.z); o.w = np_maximum_f(l.w, d.w);
      }
      __stcs(d4 + i, o);
    }
  } else {
  for (int i = lane; i < nval; i += 32) {
    const int row = i >> 5, col = i & 31;
    const float d = xs[xs_index(row, col >> 2) + (col & 3)], l = __ldcs(local + v0 + i);
    bad |= !isfinite(l);
    __stcs(dst + v0 + i, op == 0 ? __fadd_rn(l, d) : np_maximum_f(l, d));
  }
  }
  if (__any_sync(0xFFFFFFFFu, bad) && report_base != NO_REPORT) {
    for (int i = lane; i < nval; i += 32)
      if (!isfinite(local[v0 + i])) atomicMin(&st->first_nonfinite, (unsigned long long)(report_base + v0 + i));
  }
}

// Stage compressed bytes [gstart, gend) of `base` into smem words (16-byte
// chunks); returns the byte offset of gstart inside the staging area.
// ASYNC issues cp.async (the caller commits), otherwise loads directly.
template <bool ASYNC>
__device__ __forceinline__ int stage_bytes(uint32_t* stage, const uint8_t* base, uint64_t gstart, uint64_t gend, int lane) {
  const uintptr_t a0 = (reinterpret_cast<uintptr_t>(base) + gstart) & ~(uintptr_t)15;
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(base) + gend + 15) & ~(uintptr_t)15;
  const int nchunks = (int)((a1 - a0) >> 4);
  const uint4* src = reinterpret_cast<const uint4*>(a0);
  for (int i = lane; i < nchunks; i += 32) {
    if (ASYNC) cp_async16(reinterpret_cast<uint4*>(stage) + i, src + i);
    else reinterpret_cast<uint4*>(stage)[i] = __ldcg(src + i);
  }
  return (int)((reinterpret_cast<uintptr_t>(base) + gstart) & 15);
}

// S[z] = fl64(q(z) * tw) for every zigzag code of width <= 8 (codec.py:142-146, 358)
__device__ __forceinline__ void init_step_table(double* s_step, double tw) {
  for (int z = threadIdx.x; z < 256; z += blockDim.x) {
    const int q = (int)(((uint32_t)z >> 1) ^ (0u - ((uint32_t)z & 1u)));
    s_step[z] = __dmul_rn(i32_to_f64(q), tw);
  }
}

// -------------------------------------------------------------------------
// Block start of this lane's block inside a staged compressed tile: the
// sidecar carries every block's width byte, so the block sizes of
// codec.py:309-316 and their exclusive scan give all 32 starts at once (one
// warp scan instead of the reference's sequential walk, codec.py:305-320).
// The sidecar is cross-checked against the staged bytes (width byte at each
// start, total = tile size).  Returns -1 for lanes without a (valid) block.
__device__ __forceinline__ int block_start(const uint32_t* stage, int base, int tile_bytes, int w, int nblk,
                                           uint64_t b0, uint64_t nb, int last_cnt, Status* st, int lane) {
  const bool active = lane < nblk;
  const uint64_t gb = b0 + lane;
  const int cnt = (gb == nb - 1) ? last_cnt : 32;
  int size = 0;
  bool bad = false;
  if (active) {
    if (w == RAW_WIDTH) size = 1 + 4 * cnt;
    else if (w <= 32) size = 5 + ((cnt - 1) * w + 7) / 8;
    else bad = true;
  }
  int incl = size;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if (lane >= d) incl += t;
  }
  const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
  const int start = incl - size;
  if (!active) return -1;
  if (bad) {
    record_decode_error(st, gb, DE_WIDTH, w);
    return -1;
  }
  const uint8_t* bytes = reinterpret_cast<const uint8_t*>(stage) + base;
  if (total != tile_bytes || bytes[start] != w) {
    record_decode_error(st, gb, DE_SIDECAR);
    return -1;
  }
  return start;
}

// Values of one block (codec.py:331-369) from its staged bytes.
__device__ __forceinline__ void decode_values(const uint32_t* stage, int base, int bstart, int my_w, int cnt, double tw,
                                              const double* s_step, float* out) {
  const int p0 = base + bstart;
  if (my_w == RAW_WIDTH) {  // codec.py:364-367
#pragma unroll
    for (int j = 0; j < 32; ++j) out[j] = j < cnt ? __uint_as_float(lds_u32u(stage, p0 + 1 + 4 * j)) : 0.0f;
  } else if (cnt == 32 && my_w <= 8) {
    // common case: 8 codes per "oct" (8w bits = w bytes, byte aligned,
    // codec.py:96-105), steps from the table S[z] = fl64(q(z) * tw)
    const int w = my_w;
    const uint32_t mask = (1u << w) - 1u;
    const int w2 = 2 * w, w3 = 3 * w;
    double S[31];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const uint64_t oct = lds_u64u(stage, p0 + 5 + g * w);
      const uint32_t lo = (uint32_t)oct, hi = (uint32_t)(oct >> (4 * w));
      const uint32_t zz[8] = {lo & mask, (lo >> w) & mask, (lo >> w2) & mask, (lo >> w3) & mask,
                              hi & mask, (hi >> w) & mask, (hi >> w2) & mask, (hi >> w3) & mask};
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (8 * g + i < 31) S[8 * g + i] = s_step[zz[i]];
    }
    float rec = __uint_as_float(lds_u32u(stage, p0 + 1));  // codec.py:331-334
    double prev64 = (double)rec;
    out[0] = rec;
#pragma unroll
    for (int j = 1; j < 32; ++j) {  // codec.py:351-360
      rec = __double2float_rn(__dadd_rn(prev64, S[j - 1]));
      prev64 = (double)rec;
      out[j] = rec;
    }
  } else {
    float rec = __uint_as_float(lds_u32u(stage, p0 + 1));
    double prev64 = (double)rec;
    out[0] = rec;
    const int w = my_w;
    const uint32_t mask = w >= 32 ? 0xFFFFFFFFu : ((1u << w) - 1u);
#pragma unroll
    for (int j = 1; j < 32; ++j) {
      uint32_t zj = 0;
      if (w) {
        const int bit = (j - 1) * w;
        zj = (uint32_t)(lds_u64u(stage, p0 + 5 + (bit >> 3)) >> (bit & 7)) & mask;
      }
      const int q = (int)((zj >> 1) ^ (0u - (zj & 1u)));  // codec.py:142-146
      rec = __double2float_rn(__dadd_rn(prev64, __dmul_rn(i32_to_f64(q), tw)));
      prev64 = (double)rec;
      out[j] = j < cnt ? rec : 0.0f;
    }
  }
}

// Decode this lane's block (start from block_start) into its xs row.
// MODE 0: xs = decoded.  MODE 1: xs = op(xs, decoded), collectives.py:32-39.
template <int MODE>
__device__ __forceinline__ void decode_row(const uint32_t* stage, int base, int my_start, int my_w, uint64_t b0,
                                           uint64_t nb, int last_cnt, double tw, float* xs, int op, const double* s_step,
                                           int lane) {
  const int row = lane;
  if (my_start < 0) return;
  const uint64_t gb = b0 + row;
  const int cnt = (gb == nb - 1) ? last_cnt : 32;
  float out[32];
  decode_values(stage, base, my_start, my_w, cnt, tw, s_step, out);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    float4* dst = reinterpret_cast<float4*>(xs + xs_index(row, c));
    float4 v = make_float4(out[4 * c], out[4 * c + 1], out[4 * c + 2], out[4 * c + 3]);
    if (MODE == 1) {
      const float4 l = *dst;
      if (op == OP_SUM) {
        v.x = __fadd_rn(l.x, v.x); v.y = __fadd_rn(l.y, v.y); v.z = __fadd_rn(l.z, v.z); v.w = __fadd_rn(l.w, v.w);
      } else {
        v.x = np_maximum(l.x, v.x); v.y = np_maximum(l.y, v.y); v.z = np_maximum(l.z, v.z); v.w = np_maximum(l.w, v.w);
      }
    }
    *dst = v;
  }
}

// -------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
  return v;
}

struct SegGeom {
  uint64_t n, nb, ntiles;
  int last_cnt;
};
__device__ __forceinline__ SegGeom seg_geom(uint64_t n) {
  SegGeom g;
  g.n = n;
  g.nb = (n + BLOCK - 1) / BLOCK;
  g.ntiles = (g.nb + TB - 1) / TB;
  g.last_cnt = (int)(n - (g.nb ? g.nb - 1 : 0) * BLOCK);
  return g;
}

template <int NSEG>
__device__ __forceinline__ int seg_of_tile(const EncodeArgs<NSEG>& a, uint64_t t) {
  int k = 0;
  if (NSEG > 1) {
#pragma unroll 1
    for (int i = 1; i < a.nseg; ++i)
      if (a.seg[i].tile_base <= t) k = i;
  }
  return k;
}

// L2 policies: the input stream should not displace the scratch, which is
// read back (and discarded) moments later.
__device__ __forceinline__ uint64_t pol_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Start loading tile `t` (global tile index) into xs (evict-first: the values
// are read exactly once).
template <int NSEG>
__device__ __forceinline__ void prefetch_tile(const EncodeArgs<NSEG>& a, uint64_t t, float* xs, int lane, uint64_t pol) {
  if (t < a.total_tiles) {
    const Seg& S = a.seg[seg_of_tile(a, t)];
    const uint64_t v0 = (t - S.tile_base) * TILE_VALUES;
    const int nval = (int)umin64(S.n - v0, TILE_VALUES);
    const float* p = S.x + v0;
    if (nval == TILE_VALUES && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
      // chunk i = lane + 32j goes to row (lane >> 3) + 4j, 16-byte column
      // (lane & 7) ^ (row & 7): two swizzle patterns (even / odd j)
      const float4* p4 = reinterpret_cast<const float4*>(p) + lane;
      const unsigned sx = (unsigned)__cvta_generic_to_shared(xs) + (lane >> 3) * 128;
      const unsigned se = sx + ((((lane & 7) ^ (lane >> 3))) << 4);
      const unsigned so = sx + ((((lane & 7) ^ ((lane >> 3) + 4))) << 4);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"((j & 1 ? so : se) + 512 * j),
                     "l"(p4 + 32 * j), "l"(pol)
                     : "memory");
    } else {
      for (int i = lane; i < TILE_VALUES; i += 32) {
        const float v = i < nval ? __ldcs(p + i) : 0.0f;
        const int row = i >> 5, col = i & 31;
        xs[xs_index(row, col >> 2) + (col & 3)] = v;
      }
    }
  }
  cp_async_commit();
}

// Values of this lane's block (the inputs of the quantiser), for the rare
// paths that run after the codes have overwritten them in shared memory.
template <int SRC, int NSEG>
__device__ __forceinline__ void reload_row(const EncodeArgs<NSEG>& a, const Seg& S, uint64_t v0, int cnt,
                                           const uint32_t* stage, int base, double tw, const double* s_step,
                                           int my_start, int my_w, int lane, float* row) {
  const float* src = S.x + v0 + (uint64_t)lane * 32;
  for (int j = 0; j < 32; ++j) row[j] = j < cnt ? src[j] : 0.0f;
  if (SRC == SRC_STEP) {
    float dec[32];
    decode_values(stage, base, my_start, my_w, cnt, tw, s_step, dec);
    for (int j = 0; j < cnt; ++j) row[j] = a.op == OP_SUM ? __fadd_rn(row[j], dec[j]) : np_maximum(row[j], dec[j]);
  }
}

#ifndef GZ_PACK_SMALL
#define GZ_PACK_SMALL 1
#endif
// Phase A for one warp tile (values in xs): quantise and pack the tile into
// `dst` starting at byte `pos0`.  In a run (carry mode) the tile continues the
// previous tile's bytes: `carry` holds that tile's last partial word and the
// function returns this tile's, instead of completing it with zeros.
template <int SRC, int NSEG, bool FAST>
__device__ __forceinline__ int encode_tile(const EncodeArgs<NSEG>& a, const Seg& S, const SegGeom& G, uint64_t tile,
                                           float* xs, uint32_t* dst, int pos0, bool run_mode, uint32_t& carry,
                                           uint32_t* stage, int in_base, int in_bytes, int in_w,
                                           const double* s_step, uint64_t pol_keep, int lane) {
  const uint64_t nb = G.nb, b0 = tile * TB, v0 = b0 * BLOCK;
  const int last_cnt = G.last_cnt;
  const int nblk = (int)(nb - b0 < (uint64_t)TB ? nb - b0 : (uint64_t)TB);
  const int nval = (int)(G.n - v0 < (uint64_t)TILE_VALUES ? G.n - v0 : (uint64_t)TILE_VALUES);
  int base = 0, in_start = -1;

  // ---- 1. fused step: combine the received blob's tile into xs
  // (its compressed bytes were staged asynchronously with the local values)
  if (SRC == SRC_STEP) {
    base = in_base;
    in_start = block_start(stage, base, in_bytes, in_w, nblk, b0, nb, last_cnt, a.st, lane);
    __syncwarp();
    decode_row<1>(stage, base, in_start, in_w, b0, nb, last_cnt, a.in_tw, xs, a.op, s_step, lane);
    __syncwarp();
    if (a.acc_out) drain_values(xs, a.acc_out, v0, nval, lane);
    __syncwarp();
  }

  // ---- 2. closed-loop quantisation, one lane per 32-value block; the codes
  // replace the values in the lane's shared-memory row -- except in the fused
  // step, whose consumed staging buffer takes them, so that the rare raw or
  // unproven block still finds its values (local + received) in xs
  __syncwarp();
  float* zs = SRC == SRC_STEP ? reinterpret_cast<float*>(stage) : xs;
  const bool active = lane < nblk;
  const int cnt = active ? ((b0 + lane == nb - 1) ? last_cnt : 32) : 0;
  uint32_t zor = 0;
  int flags = 0;
  float x0 = 0.0f;
  if (active) {
    int fb = FB_SLOW;
    if (FAST && cnt == 32) fb = fast_block<SRC == SRC_STEP>(xs, zs, lane, a.qp.tw, a.qp.rtw, a.qp.thr, a.qp.elo, a.qp.ehi, zor, x0);
    if (fb == FB_SLOW) {  // rare: exact replay of the whole block
      float row[32];
      if (FAST && cnt == 32 && zs == xs) reload_row<SRC>(a, S, v0, cnt, stage, base, a.in_tw, s_step, in_start, in_w, lane, row);
      else load_row(xs, lane, *reinterpret_cast<float(*)[32]>(row));
      x0 = row[0];
      uint32_t zl[32];
      zor = slow_block(row, cnt, a.qp, zl, &flags);
      store_codes(zs, lane, x0, zl);
      if ((flags & 4) && S.report_base != NO_REPORT) {  // codec.py:83-85: the first non-finite offset of the caller's buffer
        // (in the fused step the values are op(local, received): only `local` is this rank's input)
        const float* src = S.x + v0 + (uint64_t)lane * 32;
        for (int j = 0; j < cnt; ++j)
          if (!isfinite(SRC == SRC_STEP ? src[j] : row[j])) {
            atomicMin(&a.st->first_nonfinite, (unsigned long long)(S.report_base + v0 + (uint64_t)lane * 32 + j));
            break;
          }
      }
    } else if (fb == FB_RAW) {
      flags |= 2;
    }
  }
  const int w = 32 - __clz(zor);                                   // codec.py:224-229
  const int ncodes = cnt - 1;
  const int packed = 5 + (ncodes * w + 7) / 8;                     // 236
  const int rawsz = 1 + 4 * cnt;                                   // 237
  const bool raw = (flags & 3) || packed > rawsz;                  // 238
  const int size = active ? (raw ? rawsz : packed) : 0;            // 239
  const int wbyte = raw ? RAW_WIDTH : w;

  // ---- 3. warp exclusive scan of block sizes (codec.py:241-243)
  int incl = size;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if (lane >= d) incl += t;
  }
  const int tile_bytes = __shfl_sync(0xFFFFFFFFu, incl, 31);
  const int start = incl - size;

  // ---- 4. pack into dst; the word straddling two blocks is completed by
  // the earlier block with the next block's leading bytes
  const uint32_t next_w = __shfl_down_sync(0xFFFFFFFFu, (uint32_t)wbyte, 1);
  const uint32_t next_x0 = __shfl_down_sync(0xFFFFFFFFu, __float_as_uint(x0), 1);
  uint32_t my_carry = 0;
  const bool small = active && !raw && w <= 4 && cnt == 32;
  if (GZ_PACK_SMALL && !run_mode && nblk == TB && __all_sync(0xFFFFFFFFu, small)) {
    uint32_t z[31];
    load_codes(zs, lane, z);
    pack_small(dst + (pos0 >> 2), start, w, x0, z, lane + 1 < TB ? (next_w | (next_x0 << 8)) : 0u, pol_keep);
  } else if (active) {
    Appender ap;
    if (lane == 0 && run_mode) ap.init_carry(dst, pos0, carry);
    else ap.init(dst, pos0 + start, lane == 0);
    ap.pol = pol_keep;
    if (raw) {
      float row[32];
      if (zs == xs) reload_row<SRC>(a, S, v0, cnt, stage, base, a.in_tw, s_step, in_start, in_w, lane, row);
      else load_row(xs, lane, *reinterpret_cast<float(*)[32]>(row));
      ap.append(255ull | ((uint64_t)__float_as_uint(x0) << 8), 5);
      int j = 1;
      for (; j + 1 < cnt; j += 2)
        ap.append((uint64_t)__float_as_uint(row[j]) | ((uint64_t)__float_as_uint(row[j + 1]) << 32), 8);
      if (j < cnt) ap.append((uint64_t)__float_as_uint(row[j]), 4);
    } else {
      ap.append((uint64_t)w | ((uint64_t)__float_as_uint(x0) << 8), 5);
      if (w > 0) {
        uint32_t z[31];
        load_codes(zs, lane, z);
        if (w <= 8) {
          const uint32_t P1 = 1u << w, P2 = 1u << (2 * w);
          // the codes carry ZBIAS: every quad of 4 codes carries ZBIAS (1 + P1)(1 + P2)
          // modulo 2^32 (code 31 is a biased zero), removed once per quad
          const uint32_t K = ZBIAS * (1u + P1) * (1u + P2);
          const int CB = (ncodes * w + 7) >> 3;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint32_t pr[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int j0 = 8 * g + 2 * i;
              pr[i] = z[j0] + ((j0 + 1 < 31) ? z[j0 + 1] : ZBIAS) * P1;
            }
            const uint32_t qa = pr[0] + pr[1] * P2 - K, qb2 = pr[2] + pr[3] * P2 - K;
            const uint64_t oct = (uint64_t)qa | ((uint64_t)qb2 << (4 * w));
            const int L = min(w, CB - g * w);
            if (L > 0) ap.append(oct, L);
          }
        } else {
          uint64_t acc = 0;
          int nbits = 0;
#pragma unroll
          for (int j = 0; j < 31; ++j) {
            if (j < ncodes) {
              acc |= (uint64_t)(z[j] - ZBIAS) << nbits;
              nbits += w;
              if (nbits >= 32) {
                ap.append(acc & 0xFFFFFFFFull, 4);
                acc >>= 32;
                nbits -= 32;
              }
            }
          }
          if (nbits > 0) ap.append(acc, (nbits + 7) >> 3);
        }
      }
    }
    if (lane + 1 < nblk) ap.finish((uint64_t)next_w | ((uint64_t)next_x0 << 8));
    else if (!run_mode) ap.finish(0ull);
    else my_carry = ap.pend;  // the run's next tile completes this word
  }
  carry = __shfl_sync(0xFFFFFFFFu, my_carry, nblk > 0 ? nblk - 1 : 0);
  // block widths (the sidecar; independent of the tile's position)
  if (active && S.out_w) S.out_w[b0 + lane] = (uint8_t)wbyte;
  if (active && a.blk_off) a.blk_off[b0 + lane] = (unsigned long long)start;  // made absolute in phase B
  return tile_bytes;
}

// Encoder, kernel 1 of 2 (one CTA per SM, no CTA-wide barrier after setup).
// CTA c owns a contiguous tile range of one segment (CTAs are split over
// segments in proportion to their tiles).  Its warps claim tiles of the range
// from a shared-memory counter -- warps of one SM do not get equal issue
// slots, so the work is balanced dynamically -- and prefetch the next claimed
// tile (cp.async, L2 evict_first) while they quantise the current one.  Each
// tile is packed into its own 128-byte aligned scratch slot (L2 evict_last)
// and its size recorded; a warp with no tile left simply exits.  The
// position-independent parts of the sidecar (sub-offsets) are final here.
template <int SRC, int NSEG, bool FAST, int NWT = 0>
__global__ void __launch_bounds__(32 * (NWT ? NWT : enc_warps(SRC)), 1) k_tile_encode(const EncodeArgs<NSEG> a) {
  constexpr int NW = NWT ? NWT : enc_warps(SRC);  // NWT: small-message instance (one tile per CTA)
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double s_step[SRC == SRC_STEP ? 256 : 1];
  __shared__ unsigned int s_next;
  __shared__ int s_abort;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int WSMEM = enc_warp_smem(SRC);
  unsigned char* my = smem + warp * WSMEM;
  float* xsb0 = reinterpret_cast<float*>(my);
  constexpr bool ONEBUF = SRC == SRC_STEP;  // the fused step: one value buffer + one staging buffer
  float* xsb1 = ONEBUF ? xsb0 : reinterpret_cast<float*>(my + TILE_VALUES * 4);
  uint32_t* stg0 = reinterpret_cast<uint32_t*>(my + TILE_VALUES * 4);  // fused step only
  if (SRC == SRC_STEP) init_step_table(s_step, a.in_tw);
  if (tid == 0) {
    s_next = 0;
    s_abort = 0;
    // the ring's "input ready" (or "slots free") flag; a flag that never
    // arrives is reported and the CTA skips its tiles (the step's completion
    // is still posted below, so the peers' streams drain)
    if (a.wait_flag && !wait_flag_sys(a.wait_flag)) {
      atomicMin(&a.st->comm_error, (unsigned long long)COMM_FLAG_TIMEOUT);
      s_abort = 1;
    }
  }
  __syncthreads();
  const uint64_t c = blockIdx.x;
  const uint64_t pol_in = pol_evict_first(), pol_keep = pol_evict_last();

  // ---- tile claiming (over all segments): most tiles are split into
  // contiguous per-CTA ranges claimed through a shared-memory counter (warps
  // of one SM do not get equal issue slots); the last 1/2^tshift is claimed
  // from one global counter, so SMs that run faster take more of the tail.  The next
  // claim is always one tile ahead (prefetch).
  const unsigned int total = (unsigned int)a.total_tiles;
  // global share 1/2^tshift: 1/32 for plain compression (2^24: 52 -> 48 us
  // vs 1/8, tools/exp/tail.py; no change at 2^27), 1/8 for the fused step
  const unsigned tshift = SRC == SRC_PLAIN ? 5u : 3u;
  const unsigned int stat = total - (total >> tshift);
  const unsigned int r0 = (unsigned int)(((uint64_t)stat * c) / gridDim.x);
  const unsigned int nr = (unsigned int)(((uint64_t)stat * (c + 1)) / gridDim.x) - r0;
  const unsigned s_next_addr = (unsigned)__cvta_generic_to_shared(&s_next);
  auto claim = [&]() -> unsigned int {
    unsigned int v = 0;
    if (lane == 0) {
      asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(v) : "r"(s_next_addr) : "memory");
      v = v < nr ? r0 + v : stat + atomicAdd(&a.ws->claim, 1u);
    }
    return __shfl_sync(0xFFFFFFFFu, v, 0);
  };
  struct InTile {
    int base, bytes, w;
  };
  // fused step, one buffer: the received tile's sidecar entries (offsets,
  // widths) are loaded one tile ahead; its bytes and the local values are
  // fetched together (one cp.async group) when the tile starts
  // (the loads stay in flight until the tile starts: nothing here consumes
  // them -- with slotted input they are NVLink reads of the peer's sizes)
  struct InMeta {
    uint64_t ts, te;  // slotted input: te holds the tile's size until the tile starts
    int w;
  };
  auto load_meta = [&](unsigned int jn) {
    InMeta m{0, 0, 0};
    if (SRC == SRC_STEP && jn < total) {
      if (a.in_slots) {  // slotted input: the tile sits at the start of its slot
        m.ts = (uint64_t)jn * TILE_SLOT;
        m.te = a.in_sizes[jn];
      } else {
        m.ts = a.in_tile_off[jn];
        m.te = a.in_tile_off[jn + 1];
      }
      m.w = a.in_w[(uint64_t)jn * TB + lane];
    }
    return m;
  };
  auto meta_end = [&](InMeta& m) {
    if (a.in_slots) m.te += m.ts;
  };
  const uint8_t* const in_base = a.in_slots ? a.in_slots : a.in_blob + HEADER_BYTES;
  unsigned int j = s_abort ? total : claim();
  unsigned int j1 = j < total ? claim() : total;
  InTile in_cur{0, 0, 0};
  InMeta m_cur = ONEBUF ? load_meta(j) : InMeta{0, 0, 0};
  if (j < total && !ONEBUF) prefetch_tile(a, j, xsb0, lane, pol_in);
  int buf = 0;
  uint32_t dummy = 0;
  while (j < total) {
    InMeta m_nxt{0, 0, 0};
    if (ONEBUF) {
      m_nxt = load_meta(j1);
      // warm L2 with the next tile's local values (4 KB) and the first 1 KB of
      // its received slot (most tiles): their cp.async at the next tile's
      // start then waits on L2, not on HBM / NVLink
      if (L2PF && j1 < total) {
        const int k1 = NSEG > 1 ? seg_of_tile(a, j1) : 0;
        const uint64_t v1 = (uint64_t)(j1 - a.seg[k1].tile_base) * TILE_VALUES;
        if (v1 + (uint64_t)lane * 32 < a.seg[k1].n)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(a.seg[k1].x + v1 + lane * 32));
      }
      meta_end(m_cur);
      if (m_cur.te < m_cur.ts || m_cur.te - m_cur.ts > (uint64_t)TB * MAX_BLOCK_BYTES) m_cur.te = m_cur.ts;  // corrupt sidecar
      in_cur.base = stage_bytes<true>(stg0, in_base, m_cur.ts, m_cur.te, lane);
      in_cur.bytes = (int)(m_cur.te - m_cur.ts);
      in_cur.w = m_cur.w;
      prefetch_tile(a, j, xsb0, lane, pol_in);  // commits the group
      cp_async_wait_all();
      __syncwarp();
    } else {  // plain compression: the next tile is prefetched while this one is encoded
      prefetch_tile(a, j1, buf ? xsb0 : xsb1, lane, pol_in);
      cp_async_wait_1();
      __syncwarp();
    }
    const int k = NSEG > 1 ? seg_of_tile(a, j) : 0;
    const Seg& S = a.seg[k];
    const SegGeom G = seg_geom(S.n);
    const uint64_t t = NSEG > 1 ? j - S.tile_base : j;  // one segment: tile_base == 0
    const int tb = encode_tile<SRC, NSEG, FAST>(a, S, G, t, buf ? xsb1 : xsb0,
                                                reinterpret_cast<uint32_t*>(a.scratch + (uint64_t)j * TILE_SLOT), 0,
                                                false, dummy, stg0, in_cur.base, in_cur.bytes, in_cur.w, s_step,
                                                pol_keep, lane);
    // the tile's size and the three counter updates (agg, agg2, agg3 are
    // consecutive arrays of TileWs), one lane each
    if (lane < 4) {
      if (lane == 3) {
        a.tile_rel[j] = (uint32_t)tb;
      } else if (!a.slotted_out) {
        const uint32_t g = (uint32_t)((NSEG > 1 ? S.gcta_base : 0) + (t >> a.gshift));
        const uint32_t idx = lane == 0 ? g : lane == 1 ? MAXGRID + (g >> 5) : MAXGRID + MAXGRID / 32 + (g >> 10);
        atomicAdd(a.ws->agg + idx, (unsigned)tb);
      }
    }
    __syncwarp();
    buf ^= 1;
    j = j1;
    m_cur = m_nxt;
    j1 = j < total ? claim() : total;
  }
  cp_async_wait_all();
#if GZ_DIAG_STAMPS
  if (lane == 0 && blockIdx.x < 256) g_est[blockIdx.x * 32 + warp] = gtimer();
#endif
  if (a.slotted_out) {
    // no gather kernel follows: the last CTA re-zeroes the claim counter and
    // posts the step's completion flag (a peer's, over NVLink) itself, so a
    // ring step is one wait node + this kernel
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      if (atomicAdd(&a.ws->done, 1ull) == gridDim.x - 1) {
        a.ws->claim = 0;
        a.ws->done = 0;
        if (a.wait_flag) *reinterpret_cast<volatile unsigned int*>(a.wait_flag) = 0u;  // every CTA has passed it
        if (a.post_flag) {
          __threadfence_system();
          asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(a.post_flag), "r"(1u) : "memory");
        }
      }
    }
  }
}

// Encoder, kernel 2 of 2: the exclusive scan of codec.py:241-243 at tile
// granularity and the gather of the slots into the blob.  Gather group g of
// a segment = 2^gshift consecutive tiles, handled by ONE warp (no CTA
// barriers; warps stride over the groups).  The encoder has added every
// tile's size into agg[g], agg2[g/32] and agg3[g/1024], so a group's base
// offset is a warp-parallel sum of at most 16 + 31 + 31 counters; a warp scan of
// the sizes gives the tile offsets (the sidecar's tile_off), and the warp
// moves its tiles as aligned 16-byte chunks into the blob -- possibly in a
// peer GPU's memory (the NVLink send of a fused reduce-scatter step).  The
// first batch of slot windows is loaded together with the sizes and
// counters.  A plain stream-ordered launch after the encoder.
constexpr int GATHER_THREADS = 256;
#ifndef GZ_GATHER_U
#define GZ_GATHER_U 4
#endif
#ifndef GZ_GATHER_MINB
#define GZ_GATHER_MINB 1
#endif
constexpr int GATHER_U = GZ_GATHER_U;  // tiles per batch

// Copy one tile (L bytes at a 128-aligned slot) to dst (any alignment) with
// the whole warp; `cur` holds slot chunk `lane` (prefetched), hb/tb the
// ragged head/tail bytes (prefetched).  Aligned destination chunk k is
// funnel-shifted from source chunks k and k+1 (shuffled from lane k+1).
__device__ __forceinline__ void gather_tile(uint8_t* dst, const uint8_t* src, int L, uint4 cur, uint32_t hb,
                                            uint32_t tb, int lane) {
  const int h = min(L, (int)((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15));
  const int wo = h >> 2, sh = (h & 3) * 8;
  const int nfull = (L - h) >> 4;
  for (int w0 = 0; w0 < nfull; w0 += 31) {  // 31 output chunks per 32-chunk window
    if (w0) {
      const int q = w0 + lane;
      cur = 16 * q < L + 16 ? *reinterpret_cast<const uint4*>(src + 16 * q) : make_uint4(0, 0, 0, 0);
    }
    uint4 nxt;
    nxt.x = __shfl_down_sync(0xFFFFFFFFu, cur.x, 1);
    nxt.y = __shfl_down_sync(0xFFFFFFFFu, cur.y, 1);
    nxt.z = __shfl_down_sync(0xFFFFFFFFu, cur.z, 1);
    nxt.w = __shfl_down_sync(0xFFFFFFFFu, cur.w, 1);
    const int kk = w0 + lane;
    if (lane < 31 && kk < nfull) {
      const uint32_t a0 = wo == 0 ? cur.x : wo == 1 ? cur.y : wo == 2 ? cur.z : cur.w;
      const uint32_t a1 = wo == 0 ? cur.y : wo == 1 ? cur.z : wo == 2 ? cur.w : nxt.x;
      const uint32_t a2 = wo == 0 ? cur.z : wo == 1 ? cur.w : wo == 2 ? nxt.x : nxt.y;
      const uint32_t a3 = wo == 0 ? cur.w : wo == 1 ? nxt.x : wo == 2 ? nxt.y : nxt.z;
      const uint32_t a4 = wo == 0 ? nxt.x : wo == 1 ? nxt.y : wo == 2 ? nxt.z : nxt.w;
      uint4 o;
      o.x = __funnelshift_r(a0, a1, sh);
      o.y = __funnelshift_r(a1, a2, sh);
      o.z = __funnelshift_r(a2, a3, sh);
      o.w = __funnelshift_r(a3, a4, sh);
      *reinterpret_cast<uint4*>(dst + h + 16 * kk) = o;
    }
  }
  const int t0 = h + 16 * nfull;  // tail bytes [t0, L)
  if (lane < h) dst[lane] = (uint8_t)hb;
  if (lane >= 16 && lane - 16 < L - t0) dst[t0 + lane - 16] = (uint8_t)tb;
}

// The gather groups of warp `gw` of `nwarps` (warp-strided).
template <int NSEG>
__device__ __forceinline__ void gather_groups(const EncodeArgs<NSEG>& a, uint64_t gw, uint64_t nwarps, int lane) {
  constexpr int U = GATHER_U;
  TileWs* ws = a.ws;
  const uint64_t cend = a.ngctas;
  for (uint64_t c = gw; c < cend; c += nwarps) {
#if GZ_DIAG_STAMPS
    if (lane == 0 && c < 8192) g_gst[3 * c] = gtimer();
#endif
    int k = 0;
    if (NSEG > 1) {
#pragma unroll 1
      for (int i = 1; i < a.nseg; ++i)
        if (a.seg[i].gcta_base <= c) k = i;
    }
    const Seg& S = a.seg[k];
    const uint64_t glo = S.gcta_base;
    const SegGeom G = seg_geom(S.n);
    const uint64_t r0 = (c - glo) << a.gshift;
    const uint64_t r1 = umin64(r0 + (1u << a.gshift), G.ntiles);
    const int nr = r1 > r0 ? (int)(r1 - r0) : 0;
    const uint32_t* sizes = a.tile_rel + S.tile_base + r0;
    const uint8_t* sl0 = a.scratch + (S.tile_base + r0) * (uint64_t)TILE_SLOT;

    // ---- independent loads first: the first 32 sizes, the first batch of
    // slot windows, the counters of the segment's earlier groups
    uint32_t sz = lane < nr ? sizes[lane] : 0u;
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      v[u] = u < nr ? *reinterpret_cast<const uint4*>(sl0 + (uint64_t)u * TILE_SLOT + 16 * lane)
                                       : make_uint4(0, 0, 0, 0);
    // bytes of the launch's groups before c minus those before the segment's
    // first group glo: <= 16 + 31 + 31 terms each, one load per lane per level
    auto prefix_terms = [&](uint64_t x) -> unsigned long long {
      unsigned long long v = 0;
      if ((uint64_t)lane < (x >> 10)) v += ws->agg3[lane];
      if ((uint64_t)lane < ((x >> 5) & 31)) v += ws->agg2[((x >> 10) << 5) + lane];
      if ((uint64_t)lane < (x & 31)) v += ws->agg[((x >> 5) << 5) + lane];
      return v;
    };
    unsigned long long base = warp_sum_u64(prefix_terms(c) - prefix_terms(glo));  // payload offset of the group
#if GZ_DIAG_STAMPS
    if (lane == 0 && c < 8192) g_gst[3 * c + 1] = gtimer() + (base & 0);
#endif

    for (int s0 = 0; s0 < nr; s0 += 32) {  // 32 tiles (one per lane) at a time
      if (s0) sz = s0 + lane < nr ? sizes[s0 + lane] : 0u;
      uint32_t incl = sz;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (lane >= d) incl += t;
      }
      const uint32_t loc = incl - sz;  // offset inside this 32-tile run
      const uint32_t run = __shfl_sync(0xFFFFFFFFu, incl, 31);
      if (s0 + lane < nr) {
        const uint64_t t = r0 + s0 + lane;
        const unsigned long long o = base + loc;
        if (S.out_tile_off) S.out_tile_off[t] = o;
        if (a.blk_off && k == 0) {
          const uint64_t bb0 = t * TB, bb1 = umin64(bb0 + TB, G.nb);
          for (uint64_t b = bb0; b < bb1; ++b) a.blk_off[b] += o;
        }
      }
      const int nrun = min(32, nr - s0);
      for (int b0 = 0; b0 < nrun; b0 += U) {
        if (s0 || b0) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int i = s0 + b0 + u;
            v[u] = b0 + u < nrun ? *reinterpret_cast<const uint4*>(sl0 + (uint64_t)i * TILE_SLOT + 16 * lane)
                                 : make_uint4(0, 0, 0, 0);
          }
        }
        // offsets/sizes of the batch's tiles (from their lanes), then the
        // ragged head/tail bytes (one round trip for the batch)
        uint32_t Ls[U], offs[U], hb[U], tb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int src_lane = min(b0 + u, 31);
          Ls[u] = __shfl_sync(0xFFFFFFFFu, sz, src_lane);
          offs[u] = __shfl_sync(0xFFFFFFFFu, loc, src_lane);
          if (b0 + u >= nrun) Ls[u] = 0;
          hb[u] = tb[u] = 0;
          if (Ls[u]) {
            const int L = (int)Ls[u];
            const uint8_t* src = sl0 + (uint64_t)(s0 + b0 + u) * TILE_SLOT;
            const uint8_t* dst = S.blob + HEADER_BYTES + base + offs[u];
            const int h = min(L, (int)((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15));
            const int t0 = h + 16 * ((L - h) >> 4);
            if (lane < h) hb[u] = __ldg(src + lane);
            if (lane >= 16 && lane - 16 < L - t0) tb[u] = __ldg(src + t0 + lane - 16);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (Ls[u])
            gather_tile(S.blob + HEADER_BYTES + base + offs[u], sl0 + (uint64_t)(s0 + b0 + u) * TILE_SLOT,
                        (int)Ls[u], v[u], hb[u], tb[u], lane);
      }
      base += run;
    }
    if (c == glo && lane < 6) {  // codec.py:158, HEADER "<4s4xQd"
      uint32_t hw;
      if (lane == 0) hw = 0x31435A47u;  // "GZC1"
      else if (lane == 1) hw = 0;
      else if (lane == 2) hw = (uint32_t)G.n;
      else if (lane == 3) hw = (uint32_t)(G.n >> 32);
      else {
        const unsigned long long eb = __double_as_longlong(a.qp.eb);
        hw = lane == 4 ? (uint32_t)eb : (uint32_t)(eb >> 32);
      }
      reinterpret_cast<uint32_t*>(S.blob)[lane] = hw;
    }
#if GZ_DIAG_STAMPS
    if (lane == 0 && c < 8192) g_gst[3 * c + 2] = gtimer();
#endif
    if (c == glo + S.gcta_n - 1 && lane == 0) {  // the segment's last group knows the total
      if (S.out_tile_off) S.out_tile_off[G.ntiles] = base;
      *S.out_len = HEADER_BYTES + base;
    }
  }
}

// Retire (every thread of the CTA): the last CTA to get here zeroes the
// counters for the next launch.
template <int NSEG>
__device__ __forceinline__ void gather_retire(const EncodeArgs<NSEG>& a, int* s_last) {
  TileWs* ws = a.ws;
  const int tid = threadIdx.x, nt = blockDim.x;
  __syncthreads();
  if (tid == 0) *s_last = atomicAdd(&ws->done, 1ull) == gridDim.x - 1;
  __syncthreads();
  if (*s_last) {
    for (uint64_t g = tid; g < a.ngctas; g += nt) ws->agg[g] = 0;
    for (uint64_t g = tid; g < (a.ngctas + 31) / 32; g += nt) ws->agg2[g] = 0;
    for (uint64_t g = tid; g < (a.ngctas + 1023) / 1024; g += nt) ws->agg3[g] = 0;
    if (tid == 0) {
      ws->done = 0;
      ws->claim = 0;
    }
  }
}

template <int NSEG>
__global__ void __launch_bounds__(GATHER_THREADS, GZ_GATHER_MINB) k_gather(const EncodeArgs<NSEG> a) {
  __shared__ int s_last;
  gather_groups(a, (uint64_t)blockIdx.x * (GATHER_THREADS / 32) + (threadIdx.x >> 5),
                (uint64_t)gridDim.x * (GATHER_THREADS / 32), threadIdx.x & 31);
  gather_retire(a, &s_last);
}

// -------------------------------------------------------------------------
// Decompress with sidecar offsets: persistent warps stride over the tiles of
// up to NSEG blobs (the allgather decodes every owner's blob, read straight
// from the owners' memory, in one launch); software pipeline: a tile's bytes
// and widths are staged one iteration ahead, its offsets two ahead.
struct DecSeg {
  const uint8_t* blob;       // header + payload (may be a peer pointer); or the slots
  const uint64_t* tile_off;  // sidecar
  const uint8_t* widths;
  uint64_t n;
  float* y;
  uint64_t tile_base;        // first global tile of this blob
  const uint32_t* sizes;     // slotted input: tile t at blob + t * TILE_SLOT, sizes[t] bytes
};
template <int NSEG>
struct DecodeMultiArgs {
  DecSeg seg[NSEG];
  int nseg;
  uint64_t total_tiles;
  double tw;
  const float* local;      // NSEG == 1 only: y = op(local, decoded)
  int op;
  Status* st;
  uint64_t report_base;    // offset of local[0] in the caller's buffer (first_nonfinite reports)
  // NSEG == 1, no `local`: full tiles leave shared memory through ONE TMA tensor store
  // (cp.async.bulk.tensor) instead of 8 loads + 8 stores per lane.  ymap views y as
  // [n/32 rows][32 floats] with a 32 x 32 box and the 128-byte swizzle, which is
  // exactly the xs layout (16-byte chunk index XOR row & 7 inside 128-byte rows).
  int ytma;
  CUtensorMap ymap;
};

// TMA tensor store of one 32 x 32 box (the swizzled tile at shared address sx) to
// rows [row, row + 32) of the map; bulk async group of the issuing thread.
__device__ __forceinline__ void tma_store_tile(const CUtensorMap* map, unsigned sx, int row) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(row), "r"(sx) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void tma_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

#ifndef GZ_DEC_BULK
#define GZ_DEC_BULK 1
#endif
// Stages per warp: 2 (one tile ahead), also for peer memory
// (three stages for the multi-owner allgather measured 3 % slower at N = 4 once
// the slotted sizes stay in flight, fewer resident warps)
__host__ __device__ constexpr int dec_stages(int nseg) { return 2; }
__host__ __device__ constexpr int dec_warp_smem(int nseg) { return TILE_VALUES * 4 + dec_stages(nseg) * STAGE_BYTES; }
// dynamic shared memory of a decoder CTA: the warps' value tiles first (1024-byte
// aligned, as the 128-byte TMA swizzle requires), then their staging buffers
constexpr int DEC_SMEM_ALIGN = 1024;
__host__ __device__ constexpr int dec_cta_smem(int nseg) { return DEC_SMEM_ALIGN + WARPS * dec_warp_smem(nseg); }

template <int NSEG>
__global__ void __launch_bounds__(CTA_THREADS) k_tile_decode(const __grid_constant__ DecodeMultiArgs<NSEG> a) {
  constexpr int ST = dec_stages(NSEG), D = ST - 1;  // D tiles staged ahead
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double s_step[256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned sraw = (unsigned)__cvta_generic_to_shared(smem_raw);
  unsigned char* smem = smem_raw + (((sraw + DEC_SMEM_ALIGN - 1) & ~(unsigned)(DEC_SMEM_ALIGN - 1)) - sraw);
  float* xs = reinterpret_cast<float*>(smem + warp * TILE_VALUES * 4);
  uint32_t* stg = reinterpret_cast<uint32_t*>(smem + WARPS * TILE_VALUES * 4 + warp * ST * STAGE_BYTES);
  const unsigned xs_s = (unsigned)__cvta_generic_to_shared(xs);
  const bool tma = NSEG == 1 && a.ytma && !a.local;
  // every decode but the codec's own (which stores through TMA and stages with cp.async,
  // measured slightly faster at cfg1) stages the compressed tiles with TMA bulk copies --
  // typically out of a peer's memory (allgather, scatter): one large NVLink read per tile
  // instead of 16-byte pieces per lane; one mbarrier per staging buffer
  const bool bulk = GZ_DEC_BULK && !tma;
  __shared__ __align__(8) unsigned long long s_mbar[WARPS][2];
  const unsigned mbar_s = (unsigned)__cvta_generic_to_shared(&s_mbar[warp][0]);
  const unsigned stg_s = (unsigned)__cvta_generic_to_shared(stg);
  unsigned ph = 0;  // bit b: parity of buffer b's next completion
  if (bulk && lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_s) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_s + 8) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  init_step_table(s_step, a.tw);
  __syncthreads();
  const uint64_t total = a.total_tiles;
  auto seg_of = [&](uint64_t t) -> int {
    int k = 0;
    if (NSEG > 1) {
#pragma unroll 1
      for (int i = 1; i < a.nseg; ++i)
        if (a.seg[i].tile_base <= t) k = i;
    }
    return k;
  };
  struct Meta {
    uint64_t ts, te;
  };
  auto offsets = [&](uint64_t t) -> Meta {
    Meta m{0, 0};
    if (t < total) {
      const DecSeg& S = a.seg[seg_of(t)];
      const uint64_t lt = t - S.tile_base;
      if (S.sizes) {  // te holds the size until stage() (a peer read: nothing consumes it yet)
        m.ts = lt * TILE_SLOT;
        m.te = S.sizes[lt];
      } else {
        m.ts = S.tile_off[lt];
        m.te = S.tile_off[lt + 1];
      }
    }
    return m;
  };
  // stage tile t into buffer bi (cp.async, caller commits); returns base, width
  auto stage = [&](uint64_t t, Meta& m, int bi, int& base, int& w) {
    base = 0;
    w = 0;
    if (t < total) {
      const DecSeg& S = a.seg[seg_of(t)];
      if (S.sizes) m.te += m.ts;
      // a corrupt sidecar must not overflow the staging buffer: stage nothing,
      // block_start() then reports the mismatch (checked here, where the offsets
      // are consumed, so their loads stay in flight behind the previous tile)
      if (m.te < m.ts || m.te - m.ts > (uint64_t)TB * MAX_BLOCK_BYTES) m.te = m.ts;
      const uint8_t* src = S.sizes ? S.blob : S.blob + HEADER_BYTES;
      if (bulk) {
        // one TMA bulk copy of the tile's 16-byte-aligned byte range (typically a peer's
        // memory: one large NVLink read instead of 16-byte pieces per lane), completing
        // on this buffer's mbarrier; the proxy fence orders the buffer's previous generic
        // reads before the async-proxy write
        const uintptr_t a0 = (reinterpret_cast<uintptr_t>(src) + m.ts) & ~(uintptr_t)15;
        const uintptr_t a1 = (reinterpret_cast<uintptr_t>(src) + m.te + 15) & ~(uintptr_t)15;
        const unsigned nbytes = (unsigned)(a1 - a0);
        if (lane == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar_s + 8 * bi), "r"(nbytes)
                       : "memory");
          if (nbytes)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    stg_s + bi * STAGE_BYTES),
                "l"(a0), "r"(nbytes), "r"(mbar_s + 8 * bi)
                : "memory");
        }
        base = (int)((reinterpret_cast<uintptr_t>(src) + m.ts) & 15);
      } else {
        base = stage_bytes<true>(stg + bi * STAGE_WORDS, src, m.ts, m.te, lane);
      }
      w = S.widths[(t - S.tile_base) * TB + lane];
      if (NSEG == 1 && a.local) {  // warm L2 with this tile's local values (read by the drain)
        const uint64_t v1 = (t - S.tile_base) * TILE_VALUES + (uint64_t)lane * 32;
        if (v1 < S.n) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.local + v1));
      }
    }
  };
  const uint64_t stride = (uint64_t)gridDim.x * WARPS;
  uint64_t t = (uint64_t)blockIdx.x * WARPS + warp;
  // software pipeline: tiles t .. t+(D-1)*stride staged, offsets of t+D*stride loaded
  Meta md[D];
  int bq[D], wq[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    md[d] = offsets(t + d * stride);
    stage(t + d * stride, md[d], d, bq[d], wq[d]);
    cp_async_commit();
  }
  Meta mnext = offsets(t + D * stride);
  int bi = 0;  // buffer of tile t
  for (; t < total; t += stride) {
    const uint64_t tn = t + D * stride;
    int bn, wn;
    stage(tn, mnext, (bi + D) % ST, bn, wn);
    cp_async_commit();
    const Meta mnn = offsets(tn + stride);
    // wait until tile t's group is complete (D newer groups may stay pending)
    if (bulk) {
      unsigned done = 0;
      const unsigned par = (ph >> bi) & 1u;
      while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(mbar_s + 8 * bi), "r"(par) : "memory");
      ph ^= 1u << bi;
    } else if (D == 2) {
      asm volatile("cp.async.wait_group 2;" ::: "memory");
    } else {
      cp_async_wait_1();
    }
    __syncwarp();
    const uint32_t* stage_t = stg + bi * STAGE_WORDS;
    const DecSeg& S = a.seg[seg_of(t)];
    const uint64_t lt = t - S.tile_base;
    const uint64_t n = S.n;
    const uint64_t nb = (n + BLOCK - 1) / BLOCK;
    const int last_cnt = (int)(n - (nb - 1) * BLOCK);
    const uint64_t b0 = lt * TB;
    const int nblk = (int)(nb - b0 < (uint64_t)TB ? nb - b0 : (uint64_t)TB);
    const uint64_t v0 = b0 * BLOCK;
    const int nval = (int)(n - v0 < (uint64_t)TILE_VALUES ? n - v0 : (uint64_t)TILE_VALUES);
    const int wl = lane < nblk ? wq[0] : 0;
    const int start = block_start(stage_t, bq[0], (int)(md[0].te - md[0].ts), wl, nblk, b0, nb, last_cnt, a.st, lane);
    if (tma) {  // the previous tile's TMA store must have read xs before it is overwritten
      if (lane == 0) tma_wait_read();
      __syncwarp();
    }
    decode_row<0>(stage_t, bq[0], start, wl, b0, nb, last_cnt, a.tw, xs, 0, s_step, lane);
    __syncwarp();
    if (tma && nval == TILE_VALUES) {
      // generic-proxy writes of xs -> visible to the async (TMA) proxy, then one store
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) tma_store_tile(&a.ymap, xs_s, (int)b0);
    } else if (NSEG == 1 && a.local) {
      drain_values_op(xs, a.local, a.op, S.y, v0, nval, lane, a.st, a.report_base);
    } else {
      drain_values(xs, S.y, v0, nval, lane);
    }
    __syncwarp();
#pragma unroll
    for (int d = 0; d + 1 < D; ++d) {
      md[d] = md[d + 1];
      bq[d] = bq[d + 1];
      wq[d] = wq[d + 1];
    }
    md[D - 1] = mnext;
    bq[D - 1] = bn;
    wq[D - 1] = wn;
    mnext = mnn;
    bi = (bi + 1) % ST;
  }
  if (tma && lane == 0) tma_wait_all();
}

}  // namespace gz
