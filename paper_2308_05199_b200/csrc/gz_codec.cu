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
enum { OP_SUM = 0, OP_MAX = 1 };

// One independently compressed blob (a compress_blocks segment).
struct Seg {
  const float* x;          // values (plain) / local chunk (step)
  uint64_t n;
  uint8_t* blob;           // header at 0, payload at 24; 16-byte aligned (may be a peer pointer)
  uint64_t* out_len;       // 24 + payload bytes
  uint64_t* out_tile_off;  // sidecar: [ntiles + 1] payload offsets of tiles
  uint16_t* out_sub_off;   // sidecar: [ntiles * GROUPS] offsets of every 8th block inside its tile
  uint64_t cta_base;       // first CTA (ticket) of this segment
  uint64_t tile_base;      // first slot of this segment in tile_rel / scratch
};

template <int NSEG>
struct EncodeArgs {
  Seg seg[NSEG];
  int nseg;
  uint64_t nctas;          // CTAs (== grid), split over segments by cta_base
  QParams qp;
  uint64_t* blk_off;       // optional per-block payload offsets (segment 0 only)
  TileWs* ws;
  uint32_t* tile_rel;      // per tile: offset inside its warp's scratch run
  uint8_t* scratch;        // per tile TILE_SLOT bytes; a warp's tiles are packed back to back
  Status* st;
  // fused step only (NSEG == 1)
  const uint8_t* in_blob;  // received blob (header + payload)
  const uint64_t* in_tile_off;
  const uint16_t* in_sub_off;
  double in_tw;
  int op;
  float* acc_out;          // optional: reduced values (f32)
};

struct DecodeArgs {
  const uint8_t* blob;     // header + payload (may be a peer pointer)
  const uint64_t* tile_off;
  const uint16_t* sub_off;
  uint64_t n;
  double tw;
  float* y;
  Status* st;
};

constexpr int ENC_WARP_SMEM = 2 * TILE_VALUES * 4 + STAGE_BYTES;  // two value tiles + staging
constexpr int DEC_WARP_SMEM = TILE_VALUES * 4 + 2 * STAGE_BYTES;  // value tile + two stagings

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

// Warp-synchronous fill of the swizzled tile xs[32][32] with src[v0, v0+nval):
// asynchronous (cp.async) for a full 16-byte aligned tile, direct otherwise.
// Always commits exactly one cp.async group.
__device__ __forceinline__ void prefetch_values(float* xs, const float* __restrict__ src, uint64_t v0, int nval, int lane) {
  const float* p = src + v0;
  if (nval == TILE_VALUES && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
    const float4* p4 = reinterpret_cast<const float4*>(p);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = lane + 32 * j;
      cp_async16(xs + xs_index(i >> 3, i & 7), p4 + i);
    }
  } else if (nval > 0) {
    for (int i = lane; i < TILE_VALUES; i += 32) {
      const float v = i < nval ? __ldcs(p + i) : 0.0f;
      const int row = i >> 5, col = i & 31;
      xs[xs_index(row, col >> 2) + (col & 3)] = v;
    }
  }
  cp_async_commit();
}

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
// Block starts of a staged compressed tile.  The sidecar gives the offset of
// every 8th block; lane g < 4 walks 8 width bytes (codec.py:305-320) and
// records starts and widths in the warp's shared arrays.  Caller __syncwarp()s.
__device__ __forceinline__ void walk_groups(const uint32_t* stage, int base, int tile_bytes, const uint16_t* sub,
                                            int nblk, uint64_t b0, uint64_t nb, int last_cnt, Status* st,
                                            uint16_t* s_start, uint8_t* s_w, int lane) {
  const int g = lane;
  if (g >= GROUPS || g * GROUP >= nblk) return;
  const int g0 = g * GROUP;
  const int gblk = min(GROUP, nblk - g0);
  const int gend = (g0 + GROUP < nblk) ? (int)sub[g + 1] : tile_bytes;
  const uint8_t* bytes = reinterpret_cast<const uint8_t*>(stage) + base;
  int pos = sub[g];
  for (int k = 0; k < gblk; ++k) {
    const int w = bytes[pos];
    const uint64_t gb = b0 + g0 + k;
    const int cnt = (gb == nb - 1) ? last_cnt : 32;
    int size;
    if (w == RAW_WIDTH) size = 1 + 4 * cnt;
    else if (w <= 32) size = 5 + ((cnt - 1) * w + 7) / 8;
    else {
      record_decode_error(st, gb, DE_WIDTH, w);
      for (int r = k; r < gblk; ++r) s_start[g0 + r] = 0xFFFF;
      return;
    }
    s_start[g0 + k] = (uint16_t)pos;
    s_w[g0 + k] = (uint8_t)w;
    pos += size;
    if (pos > gend) {
      record_decode_error(st, gb, DE_SIDECAR);
      for (int r = k + 1; r < gblk; ++r) s_start[g0 + r] = 0xFFFF;
      return;
    }
  }
  if (pos != gend) record_decode_error(st, b0 + g0 + gblk - 1, DE_SIDECAR);
}

// Decode this lane's block (walked by walk_groups) into its xs row.
// MODE 0: xs = decoded.  MODE 1: xs = op(xs, decoded), collectives.py:32-39.
template <int MODE>
__device__ __forceinline__ void decode_row(const uint32_t* stage, int base, int nblk, uint64_t b0, uint64_t nb,
                                           int last_cnt, double tw, float* xs, int op, const double* s_step,
                                           const uint16_t* s_start, const uint8_t* s_w, int lane) {
  const int row = lane;
  if (row >= nblk || s_start[row] == 0xFFFF) return;
  const int my_w = s_w[row];
  const uint64_t gb = b0 + row;
  const int cnt = (gb == nb - 1) ? last_cnt : 32;
  const int p0 = base + s_start[row];
  float out[32];
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

// -------------------------------------------------------------------------
// Copy `len` bytes from 16-byte aligned src to arbitrary dst (dst may be a
// peer GPU's memory): aligned 16-byte stores in the middle, byte stores at
// the two ragged ends.  Warp-cooperative.
__device__ __forceinline__ void copy_to_unaligned(uint8_t* dst, const uint8_t* src, uint64_t len, int lane) {
  if (!len) return;
  const uintptr_t A = reinterpret_cast<uintptr_t>(dst);
  const uintptr_t E = A + len;
  const uintptr_t cf = (A + 15) & ~(uintptr_t)15, cl = E & ~(uintptr_t)15;
  const uint32_t* sw = reinterpret_cast<const uint32_t*>(src);
  if (cf < cl) {
    const uint64_t off0 = cf - A;  // source byte of the first full destination chunk
    const int sh = (int)(off0 & 3) * 8;
    const uint64_t nch = (cl - cf) >> 4;
    uint4* d = reinterpret_cast<uint4*>(cf);
    for (uint64_t c = lane; c < nch; c += 32) {
      const uint64_t wi = (off0 >> 2) + 4 * c;
      const uint32_t w0 = __ldcg(sw + wi), w1 = __ldcg(sw + wi + 1), w2 = __ldcg(sw + wi + 2), w3 = __ldcg(sw + wi + 3),
                     w4 = __ldcg(sw + wi + 4);
      uint4 v;
      v.x = __funnelshift_r(w0, w1, sh);
      v.y = __funnelshift_r(w1, w2, sh);
      v.z = __funnelshift_r(w2, w3, sh);
      v.w = __funnelshift_r(w3, w4, sh);
      d[c] = v;
    }
    const int head = (int)(cf - A), tail = (int)(E - cl);
    if (lane < head) dst[lane] = src[lane];
    if (lane >= 16 && lane - 16 < tail) dst[len - tail + (lane - 16)] = src[len - tail + (lane - 16)];
  } else {
    for (uint64_t i = lane; i < len; i += 32) dst[i] = src[i];
  }
}

// Append the staged tile (tile_bytes from smem) to the warp's scratch run at
// byte offset `run` (16-byte aligned run start + arbitrary offset).
__device__ __forceinline__ void stage_to_scratch(uint8_t* run_base, uint64_t run, const uint32_t* stage, int tile_bytes,
                                                 int lane) {
  if (!tile_bytes) return;
  uint8_t* gdst = run_base + run;
  const uintptr_t A = reinterpret_cast<uintptr_t>(gdst);
  const uintptr_t E = A + (uintptr_t)tile_bytes;
  const uintptr_t cf = (A + 15) & ~(uintptr_t)15, cl = E & ~(uintptr_t)15;
  const uint8_t* sb = reinterpret_cast<const uint8_t*>(stage);
  if (cf < cl) {
    const int off0 = (int)(cf - A);
    const int sh = (off0 & 3) * 8;
    const int nch = (int)((cl - cf) >> 4);
    uint4* dst = reinterpret_cast<uint4*>(cf);
    for (int c = lane; c < nch; c += 32) {
      const int wi = (off0 >> 2) + 4 * c;
      const uint32_t w0 = stage[wi], w1 = stage[wi + 1], w2 = stage[wi + 2], w3 = stage[wi + 3], w4 = stage[wi + 4];
      uint4 v;
      v.x = __funnelshift_r(w0, w1, sh);
      v.y = __funnelshift_r(w1, w2, sh);
      v.z = __funnelshift_r(w2, w3, sh);
      v.w = __funnelshift_r(w3, w4, sh);
      __stcg(dst + c, v);
    }
    const int head = (int)(cf - A), tail = (int)(E - cl);
    if (lane < head) gdst[lane] = sb[lane];
    if (lane >= 16 && lane - 16 < tail) gdst[tile_bytes - tail + (lane - 16)] = sb[tile_bytes - tail + (lane - 16)];
  } else {
    for (int i = lane; i < tile_bytes; i += 32) gdst[i] = sb[i];
  }
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

// Pass A for one warp tile (values in xs): quantise, pack into smem, append
// to the warp's scratch run.  Returns the tile's compressed size.
template <int SRC, int NSEG, bool FAST>
__device__ __forceinline__ int encode_tile(const EncodeArgs<NSEG>& a, const Seg& S, const SegGeom& G, uint64_t tile,
                                           float* xs, uint32_t* stage, uint16_t* s_start, uint8_t* s_w,
                                           const double* s_step, int lane) {
  const uint64_t nb = G.nb, b0 = tile * TB, v0 = b0 * BLOCK;
  const int last_cnt = G.last_cnt;
  const int nblk = (int)(nb - b0 < (uint64_t)TB ? nb - b0 : (uint64_t)TB);
  const int nval = (int)(G.n - v0 < (uint64_t)TILE_VALUES ? G.n - v0 : (uint64_t)TILE_VALUES);

  // ---- 1. fused step: combine the received blob's tile into xs
  if (SRC == SRC_STEP) {
    const uint64_t ts = a.in_tile_off[tile], te = a.in_tile_off[tile + 1];
    const int base = stage_bytes<false>(stage, a.in_blob + HEADER_BYTES, ts, te, lane);
    __syncwarp();
    walk_groups(stage, base, (int)(te - ts), a.in_sub_off + tile * GROUPS, nblk, b0, nb, last_cnt, a.st, s_start,
                s_w, lane);
    __syncwarp();
    decode_row<1>(stage, base, nblk, b0, nb, last_cnt, a.in_tw, xs, a.op, s_step, s_start, s_w, lane);
    __syncwarp();
    if (a.acc_out) drain_values(xs, a.acc_out, v0, nval, lane);
  }

  // ---- 2. closed-loop quantisation, one lane per 32-value block
  const bool active = lane < nblk;
  const int cnt = active ? ((b0 + lane == nb - 1) ? last_cnt : 32) : 0;
  uint32_t z[31];
  uint32_t zor = 0;
  int flags = 0;
  float x0 = 0.0f;
  if (active) {
    int fb = FB_SLOW;
    if (FAST && cnt == 32) fb = fast_block(xs, lane, a.qp.tw, a.qp.rtw, a.qp.thr, a.qp.elo, a.qp.ehi, z, x0);
    if (fb == FB_SLOW) {  // rare: exact replay of the whole block
      float row[32];
      load_row(xs, lane, row);
      x0 = row[0];
      uint32_t zl[32];
      zor = slow_block(row, cnt, a.qp.tw, a.qp.eb, zl, &flags);
#pragma unroll
      for (int j = 0; j < 31; ++j) z[j] = zl[j];
      if (flags & 4) {  // codec.py:83-85: report the first non-finite offset
        for (int j = 0; j < cnt; ++j)
          if (!isfinite(xs[xs_index(lane, j >> 2) + (j & 3)])) {
            atomicMin(&a.st->first_nonfinite, (unsigned long long)(v0 + (uint64_t)lane * 32 + j));
            break;
          }
      }
    } else {
      if (fb == FB_RAW) flags |= 2;
#pragma unroll
      for (int j = 0; j < 31; j += 3) zor |= z[j] | (j + 1 < 31 ? z[j + 1] : 0u) | (j + 2 < 31 ? z[j + 2] : 0u);
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

  // ---- 4. pack into the staging area; the word straddling two blocks is
  // completed by the earlier block with the next block's leading bytes
  const uint32_t next_w = __shfl_down_sync(0xFFFFFFFFu, (uint32_t)wbyte, 1);
  const uint32_t next_x0 = __shfl_down_sync(0xFFFFFFFFu, __float_as_uint(x0), 1);
  if (active) {
    Appender ap;
    ap.init(stage, start, lane == 0);
    if (raw) {
      ap.append(255ull | ((uint64_t)__float_as_uint(x0) << 8), 5);
      int j = 1;
      for (; j + 1 < cnt; j += 2) {
        const float v1 = xs[xs_index(lane, j >> 2) + (j & 3)];
        const float v2 = xs[xs_index(lane, (j + 1) >> 2) + ((j + 1) & 3)];
        ap.append((uint64_t)__float_as_uint(v1) | ((uint64_t)__float_as_uint(v2) << 32), 8);
      }
      if (j < cnt) ap.append((uint64_t)__float_as_uint(xs[xs_index(lane, j >> 2) + (j & 3)]), 4);
    } else {
      ap.append((uint64_t)w | ((uint64_t)__float_as_uint(x0) << 8), 5);
      if (w > 0 && w <= 8) {
        const uint32_t P1 = 1u << w, P2 = 1u << (2 * w);
        uint32_t pr[16], qd[8];
#pragma unroll
        for (int i = 0; i < 16; ++i) pr[i] = (2 * i + 1 < 31) ? z[2 * i] + z[2 * i + 1] * P1 : z[2 * i];
#pragma unroll
        for (int i = 0; i < 8; ++i) qd[i] = pr[2 * i] + pr[2 * i + 1] * P2;
        const int CB = (ncodes * w + 7) >> 3;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const uint64_t oct = (uint64_t)qd[2 * g] | ((uint64_t)qd[2 * g + 1] << (4 * w));
          const int L = min(w, CB - g * w);
          if (L > 0) ap.append(oct, L);
        }
      } else if (w > 8) {
        uint64_t acc = 0;
        int nbits = 0;
#pragma unroll
        for (int j = 0; j < 31; ++j) {
          if (j < ncodes) {
            acc |= (uint64_t)z[j] << nbits;
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
    const uint64_t lead = (lane + 1 < nblk) ? ((uint64_t)next_w | ((uint64_t)next_x0 << 8)) : 0ull;
    ap.finish(lead);
  }
  // sub-offsets (final values, independent of the tile's position)
  const int st8 = __shfl_sync(0xFFFFFFFFu, start, (lane & 3) * GROUP);
  if (lane < GROUPS && S.out_sub_off) S.out_sub_off[tile * GROUPS + lane] = (uint16_t)(lane * GROUP < nblk ? st8 : tile_bytes);
  if (active && a.blk_off) a.blk_off[b0 + lane] = (unsigned long long)start;  // made absolute in pass B
  __syncwarp();
  return tile_bytes;
}

// Persistent encoder, one kernel, two phases per CTA:
//   A. each warp encodes a contiguous run of tiles (prefetching the next
//      tile with cp.async while quantising the current one) and appends the
//      packed bytes to its run in a local scratch buffer (stays in L2);
//   B. the CTA publishes its total, sums the totals of all earlier CTAs of the
//      segment (the exclusive scan of codec.py:241-243 at CTA granularity,
//      one round trip), then every warp copies its run to its final place in
//      the blob -- which may be a peer GPU's memory (the NVLink send).
// CTA ids come from an atomic ticket, so a CTA only ever waits for CTAs that
// are already running.
template <int SRC, int NSEG, bool FAST>
__global__ void __launch_bounds__(CTA_THREADS, 4) k_tile_encode(const EncodeArgs<NSEG> a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double s_step[SRC == SRC_STEP ? 256 : 1];
  __shared__ uint16_t s_start[SRC == SRC_STEP ? WARPS : 1][TB];
  __shared__ uint8_t s_w[SRC == SRC_STEP ? WARPS : 1][TB];
  __shared__ unsigned long long s_cta, s_gen, s_base;
  __shared__ unsigned long long s_wtot[WARPS];
  __shared__ unsigned long long s_red[CTA_THREADS / 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned char* my = smem + warp * ENC_WARP_SMEM;
  float* xsb0 = reinterpret_cast<float*>(my);
  float* xsb1 = reinterpret_cast<float*>(my + TILE_VALUES * 4);
  uint32_t* stage = reinterpret_cast<uint32_t*>(my + 2 * TILE_VALUES * 4);
  TileWs* ws = a.ws;
  if (SRC == SRC_STEP) init_step_table(s_step, a.in_tw);
  if (tid == 0) {
    s_cta = atomicAdd(&ws->ticket, 1ull);
    s_gen = ld_volatile_u64(&ws->gen);
  }
  __syncthreads();
  const unsigned long long c = s_cta, gen = s_gen;
  int k = 0;
  if (NSEG > 1) {
#pragma unroll 1
    for (int i = 1; i < a.nseg; ++i)
      if (a.seg[i].cta_base <= c) k = i;
  }
  const Seg& S = a.seg[k];
  const uint64_t cta_end = (k + 1 < a.nseg) ? a.seg[k + 1].cta_base : a.nctas;
  const uint64_t ncta = cta_end - S.cta_base, cl = c - S.cta_base;
  const SegGeom G = seg_geom(S.n);
  // contiguous tile run of this CTA, then of this warp
  const uint64_t per_cta = (G.ntiles + ncta - 1) / ncta;
  const uint64_t c0 = umin64(cl * per_cta, G.ntiles), c1 = umin64(c0 + per_cta, G.ntiles);
  const uint64_t per_warp = (c1 - c0 + WARPS - 1) / WARPS;
  const uint64_t t0 = umin64(c0 + warp * per_warp, c1), t1 = umin64(t0 + per_warp, c1);
  uint8_t* run_base = a.scratch + (S.tile_base + t0) * (uint64_t)TILE_SLOT;
  uint32_t* rel = a.tile_rel + S.tile_base;

  if (cl == 0 && warp == 0 && lane < 6) {  // codec.py:158, HEADER "<4s4xQd"
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
  if (SRC == SRC_STEP) __syncthreads();

  // ---- phase A: encode the warp's run into scratch
  unsigned long long run = 0;
  if (t0 < t1) {
    const uint64_t nv0 = G.n - t0 * TILE_VALUES;
    prefetch_values(xsb0, S.x, t0 * TILE_VALUES, (int)umin64(nv0, TILE_VALUES), lane);
  }
  int buf = 0;
  for (uint64_t t = t0; t < t1; ++t) {
    if (t + 1 < t1) {
      const uint64_t v1 = (t + 1) * TILE_VALUES;
      prefetch_values(buf ? xsb0 : xsb1, S.x, v1, (int)umin64(G.n - v1, TILE_VALUES), lane);
    } else {
      cp_async_commit();
    }
    cp_async_wait_1();
    __syncwarp();
    const int tb = encode_tile<SRC, NSEG, FAST>(a, S, G, t, buf ? xsb1 : xsb0, stage, s_start[SRC == SRC_STEP ? warp : 0],
                                                s_w[SRC == SRC_STEP ? warp : 0], s_step, lane);
    if (lane == 0) rel[t] = (uint32_t)run;
    stage_to_scratch(run_base, run, stage, tb, lane);
    run += (unsigned long long)tb;
    __syncwarp();
    buf ^= 1;
  }
  if (lane == 0) s_wtot[warp] = run;
  __syncthreads();

  // ---- phase B: CTA prefix over the segment's earlier CTAs
  if (tid == 0) {
    unsigned long long tot = 0;
#pragma unroll
    for (int j = 0; j < WARPS; ++j) tot += s_wtot[j];
    st_volatile_u64(&ws->status[c], mk_status(gen, 1u, tot));
  }
  unsigned long long part = 0;
  for (uint64_t p = S.cta_base + tid; p < c; p += CTA_THREADS) {
    unsigned long long sw;
    while (true) {
      sw = ld_volatile_u64(&ws->status[p]);
      if (((sw >> 48) & 0xFFFF) == (gen & 0xFFFF) && ((sw >> 46) & 3) != 0) break;
      __nanosleep(64);
    }
    part += sw & VALUE_MASK;
  }
  part = warp_sum_u64(part);
  if (lane == 0) s_red[warp] = part;
  __syncthreads();
  if (tid == 0) {
    unsigned long long b = 0;
#pragma unroll
    for (int j = 0; j < CTA_THREADS / 32; ++j) b += s_red[j];
    s_base = b;
  }
  __syncthreads();
  unsigned long long base = s_base;
#pragma unroll
  for (int j = 0; j < WARPS; ++j) base += j < warp ? s_wtot[j] : 0ull;

  // ---- phase B: copy the run to its final place; tile offsets, length
  copy_to_unaligned(S.blob + HEADER_BYTES + base, run_base, run, lane);
  for (uint64_t t = t0 + lane; t < t1; t += 32) {
    if (S.out_tile_off) S.out_tile_off[t] = base + rel[t];
  }
  if (a.blk_off && k == 0) {
    for (uint64_t b = t0 * TB + lane; b < umin64(t1 * TB, G.nb); b += 32) a.blk_off[b] += base + rel[b / TB];
  }
  if (lane == 0 && t0 < t1 && t1 == G.ntiles) {
    if (S.out_tile_off) S.out_tile_off[G.ntiles] = base + run;
    *S.out_len = HEADER_BYTES + base + run;
  }
  if (tid == 0 && G.ntiles == 0 && cl == 0) {
    if (S.out_tile_off) S.out_tile_off[0] = 0;
    *S.out_len = HEADER_BYTES;
  }

  // retire: the last CTA to finish resets the tickets and bumps gen
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&ws->done, 1ull) == a.nctas - 1) {
      ws->done = 0;
      ws->ticket = 0;
      __threadfence();
      atomicAdd(&ws->gen, 1ull);
    }
  }
}

// -------------------------------------------------------------------------
// Decompress with sidecar offsets: persistent warps stride over tiles, the
// next tile's compressed bytes prefetched (cp.async) while decoding.
__global__ void __launch_bounds__(CTA_THREADS, 4) k_tile_decode(const DecodeArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double s_step[256];
  __shared__ uint16_t s_start[WARPS][TB];
  __shared__ uint8_t s_w[WARPS][TB];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* my = smem + warp * DEC_WARP_SMEM;
  float* xs = reinterpret_cast<float*>(my);
  uint32_t* stg0 = reinterpret_cast<uint32_t*>(my + TILE_VALUES * 4);
  uint32_t* stg1 = reinterpret_cast<uint32_t*>(my + TILE_VALUES * 4 + STAGE_BYTES);
  init_step_table(s_step, a.tw);
  __syncthreads();
  const uint64_t n = a.n;
  const uint64_t nb = (n + BLOCK - 1) / BLOCK;
  const uint64_t ntiles = (nb + TB - 1) / TB;
  const int last_cnt = (int)(n - (nb - 1) * BLOCK);
  const uint8_t* payload = a.blob + HEADER_BYTES;
  const uint64_t stride = (uint64_t)gridDim.x * WARPS;
  uint64_t t = (uint64_t)blockIdx.x * WARPS + warp;
  int buf = 0;
  uint64_t ts = 0, te = 0;
  int base = 0;
  if (t < ntiles) {
    ts = a.tile_off[t];
    te = a.tile_off[t + 1];
    base = stage_bytes<true>(stg0, payload, ts, te, lane);
  }
  cp_async_commit();
  for (; t < ntiles; t += stride) {
    const uint64_t tn = t + stride;
    uint64_t tsn = 0, ten = 0;
    int basen = 0;
    if (tn < ntiles) {
      tsn = a.tile_off[tn];
      ten = a.tile_off[tn + 1];
      basen = stage_bytes<true>(buf ? stg0 : stg1, payload, tsn, ten, lane);
    }
    cp_async_commit();
    cp_async_wait_1();
    __syncwarp();
    uint32_t* stage = buf ? stg1 : stg0;
    const uint64_t b0 = t * TB;
    const int nblk = (int)(nb - b0 < (uint64_t)TB ? nb - b0 : (uint64_t)TB);
    const uint64_t v0 = b0 * BLOCK;
    const int nval = (int)(n - v0 < (uint64_t)TILE_VALUES ? n - v0 : (uint64_t)TILE_VALUES);
    walk_groups(stage, base, (int)(te - ts), a.sub_off + t * GROUPS, nblk, b0, nb, last_cnt, a.st, s_start[warp],
                s_w[warp], lane);
    __syncwarp();
    decode_row<0>(stage, base, nblk, b0, nb, last_cnt, a.tw, xs, 0, s_step, s_start[warp], s_w[warp], lane);
    __syncwarp();
    drain_values(xs, a.y, v0, nval, lane);
    __syncwarp();
    buf ^= 1;
    ts = tsn;
    te = ten;
    base = basen;
  }
}

}  // namespace gz
