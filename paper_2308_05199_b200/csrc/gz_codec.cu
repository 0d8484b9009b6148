// gz_codec.cu -- sm_100a kernels of the B200 gZCCL codec and the fused
// ring reduce-scatter step.  See gz_device.cuh for the layout and numerics.
//
//   k_tile_encode<SRC_PLAIN>  compress  (codec.py:149-270)
//   k_tile_encode<SRC_STEP>   fused RS step: decompress(recv) (+) local ->
//                             compress (collectives.py:274-290, one kernel)
//   k_tile_decode             decompress with sidecar offsets (codec.py:284-369)
#include "gz_device.cuh"

namespace gz {

enum { SRC_PLAIN = 0, SRC_STEP = 1 };
enum { OP_SUM = 0, OP_MAX = 1 };

// One independently compressed blob (compress_blocks segment, codec.py:408-427).
struct Seg {
  const float* x;          // values (plain) / local chunk (step)
  uint64_t n;
  uint8_t* blob;           // header at 0, payload at 24; 16-byte aligned (may be a peer pointer)
  uint64_t* out_len;       // 24 + payload bytes
  uint64_t* out_tile_off;  // sidecar: [ntiles + 1] payload offsets of tiles
  uint16_t* out_sub_off;   // sidecar: [ntiles * GROUPS] group offsets inside the tile
  uint64_t cta_base;       // first global CTA ticket of this segment
};

template <int NSEG>
struct EncodeArgs {
  Seg seg[NSEG];
  int nseg;
  uint64_t nctas;          // sum over segments of max(ntiles, 1)
  QParams qp;
  uint64_t* blk_off;       // optional per-block payload offsets (segment 0 only)
  TileWs* ws;
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
__device__ __forceinline__ int lds_u8(const uint32_t* w, int off) { return (w[off >> 2] >> ((off & 3) * 8)) & 0xFF; }

__device__ __forceinline__ float np_maximum(float a, float b) {  // collectives.py:38
  return isnan(a) ? a : (a > b ? a : b);
}

// (block << 24) | (width << 8) | code; the smallest block index wins
__device__ __forceinline__ void record_decode_error(Status* st, uint64_t block, unsigned code, int w = 0) {
  atomicMin(&st->decode_error, (unsigned long long)((block << 24) | ((uint64_t)(w & 0xFFFF) << 8) | code));
}

// Fill the swizzled tile xs[TB][32] with values [v0, v0 + nval) of src.
__device__ __forceinline__ void fill_tile(float* xs, const float* __restrict__ src, uint64_t v0, int nval) {
  const float* p = src + v0;
  if (nval == TILE_VALUES && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
    const float4* p4 = reinterpret_cast<const float4*>(p);
#pragma unroll 4
    for (int i = threadIdx.x; i < TB * 8; i += TB) {
      float4 v = __ldcs(p4 + i);
      *reinterpret_cast<float4*>(xs + xs_index(i >> 3, i & 7)) = v;
    }
  } else {
    for (int i = threadIdx.x; i < TILE_VALUES; i += TB) {
      float v = i < nval ? __ldcs(p + i) : 0.0f;
      const int row = i >> 5, col = i & 31;
      xs[xs_index(row, col >> 2) + (col & 3)] = v;
    }
  }
}

// Write the tile xs back to dst[v0, v0 + nval) coalesced.
__device__ __forceinline__ void drain_tile(const float* xs, float* __restrict__ dst, uint64_t v0, int nval) {
  float* p = dst + v0;
  if (nval == TILE_VALUES && ((reinterpret_cast<uintptr_t>(p) & 15) == 0)) {
    float4* p4 = reinterpret_cast<float4*>(p);
#pragma unroll 4
    for (int i = threadIdx.x; i < TB * 8; i += TB) __stcs(p4 + i, *reinterpret_cast<const float4*>(xs + xs_index(i >> 3, i & 7)));
  } else {
    for (int i = threadIdx.x; i < nval; i += TB) {
      const int row = i >> 5, col = i & 31;
      __stcs(p + i, xs[xs_index(row, col >> 2) + (col & 3)]);
    }
  }
}

// Stage compressed bytes [gstart, gend) of `base` into smem words; returns the
// byte offset of gstart inside the staging area (gstart & 15).
__device__ __forceinline__ int stage_bytes(uint32_t* stage, const uint8_t* base, uint64_t gstart, uint64_t gend) {
  const uintptr_t a0 = (reinterpret_cast<uintptr_t>(base) + gstart) & ~(uintptr_t)15;
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(base) + gend + 15) & ~(uintptr_t)15;
  const int nchunks = (int)((a1 - a0) >> 4);
  const uint4* src = reinterpret_cast<const uint4*>(a0);
  for (int i = threadIdx.x; i < nchunks; i += TB) reinterpret_cast<uint4*>(stage)[i] = __ldcg(src + i);
  return (int)((reinterpret_cast<uintptr_t>(base) + gstart) & 15);
}

// -------------------------------------------------------------------------
// Decode the staged compressed tile into per-thread values and combine into
// xs.  Warp g owns blocks [32g, 32g+32) of the tile; every lane replays the
// group's width chain (broadcast smem reads) until it reaches its own block,
// so no sequential walk over the whole payload (codec.py:305-320) is needed.
// MODE 0: xs = decoded.  MODE 1: xs = op(xs, decoded), collectives.py:32-39.
template <int MODE>
__device__ __forceinline__ void decode_tile(const uint32_t* stage, int base, int tile_bytes, const uint16_t* sub,
                                            int nblk, uint64_t b0, uint64_t nb, int last_cnt, double tw, float* xs,
                                            int op, Status* st) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g0 = warp * 32;
  if (g0 >= nblk) return;
  const int gblk = min(32, nblk - g0);
  const int gstart = sub[warp];
  const int gend = (g0 + 32 < nblk) ? (int)sub[warp + 1] : tile_bytes;
  // chain replay
  int pos = gstart, my_start = -1, my_w = 0;
  bool bad = false;
  for (int k = 0; k < gblk; ++k) {
    const int w = lds_u8(stage, base + pos);
    const uint64_t gb = b0 + g0 + k;
    const int cnt = (gb == nb - 1) ? last_cnt : 32;
    int size;
    if (w == RAW_WIDTH) size = 1 + 4 * cnt;
    else if (w <= 32) size = 5 + ((cnt - 1) * w + 7) / 8;
    else {
      if (lane == 0) record_decode_error(st, gb, DE_WIDTH, w);
      bad = true;
      break;
    }
    if (k == lane) {
      my_start = pos;
      my_w = w;
    }
    pos += size;
    if (pos > gend) {
      if (lane == 0) record_decode_error(st, gb, DE_SIDECAR);
      bad = true;
      break;
    }
  }
  if (!bad && pos != gend && lane == 0) record_decode_error(st, b0 + g0 + gblk - 1, DE_SIDECAR);
  if (lane >= gblk || my_start < 0) return;
  const int row = g0 + lane;
  const uint64_t gb = b0 + row;
  const int cnt = (gb == nb - 1) ? last_cnt : 32;
  const int p0 = base + my_start;
  float out[32];
  if (my_w == RAW_WIDTH) {  // codec.py:364-367
#pragma unroll
    for (int j = 0; j < 32; ++j) out[j] = j < cnt ? __uint_as_float(lds_u32u(stage, p0 + 1 + 4 * j)) : 0.0f;
  } else {
    float rec = __uint_as_float(lds_u32u(stage, p0 + 1));  // codec.py:331-334
    double prev64 = (double)rec;
    out[0] = rec;
    const int w = my_w;
    const uint32_t mask = w >= 32 ? 0xFFFFFFFFu : ((1u << w) - 1u);
    uint32_t z[31];
    if (w == 0) {
#pragma unroll
      for (int j = 0; j < 31; ++j) z[j] = 0;
    } else if (w <= 8) {
      // 8 codes per "oct": 8w bits = w bytes, byte aligned (codec.py:96-105)
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const uint64_t oct = lds_u64u(stage, p0 + 5 + g * w);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (8 * g + i < 31) z[8 * g + i] = (uint32_t)(oct >> (i * w)) & mask;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 31; ++j) {
        const int bit = j * w;
        const uint64_t win = lds_u64u(stage, p0 + 5 + (bit >> 3));
        z[j] = (uint32_t)(win >> (bit & 7)) & mask;
      }
    }
#pragma unroll
    for (int j = 1; j < 32; ++j) {  // codec.py:351-360
      const int q = (int)((z[j - 1] >> 1) ^ (0u - (z[j - 1] & 1u)));   // 142-146
      const double t = __dadd_rn(prev64, __dmul_rn(i32_to_f64(q), tw));
      rec = __double2float_rn(t);
      prev64 = (double)rec;
      out[j] = j < cnt ? rec : 0.0f;
    }
  }
  // combine into xs row
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
// Encode one tile.  Single pass: quantise -> CTA scan of block sizes ->
// publish tile aggregate -> pack into smem -> decoupled look-back -> store.
template <int SRC, int NSEG>
__global__ void __launch_bounds__(TB) k_tile_encode(const EncodeArgs<NSEG> a) {
  extern __shared__ __align__(16) unsigned char smem[];
  float* xs = reinterpret_cast<float*>(smem);
  uint32_t* stage = reinterpret_cast<uint32_t*>(smem + TB * 128);
  __shared__ uint32_t s_wbyte[TB + 1];
  __shared__ uint32_t s_warp[TB / 32];
  __shared__ unsigned long long s_tile, s_gen, s_excl;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  TileWs* ws = a.ws;
  if (tid == 0) {
    s_tile = atomicAdd(&ws->ticket, 1ull);
    s_gen = ld_volatile_u64(&ws->gen);
  }
  __syncthreads();
  const uint64_t gt = s_tile, gen = s_gen;  // global CTA ticket == status slot
  int k = 0;
  if (NSEG > 1) {
#pragma unroll 1
    for (int i = 1; i < a.nseg; ++i)
      if (a.seg[i].cta_base <= gt) k = i;
  }
  const Seg& S = a.seg[k];
  const uint64_t tile = gt - S.cta_base;  // tile within the segment
  const uint64_t n = S.n;
  const uint64_t nb = (n + BLOCK - 1) / BLOCK;
  const uint64_t ntiles = (nb + TB - 1) / TB;
  const int last_cnt = (int)(n - (nb ? nb - 1 : 0) * BLOCK);

  if (tile == 0 && tid < 6) {  // codec.py:158, HEADER "<4s4xQd"
    uint32_t hw;
    if (tid == 0) hw = 0x31435A47u;  // "GZC1"
    else if (tid == 1) hw = 0;
    else if (tid == 2) hw = (uint32_t)n;
    else if (tid == 3) hw = (uint32_t)(n >> 32);
    else {
      const unsigned long long eb = __double_as_longlong(a.qp.eb);
      hw = tid == 4 ? (uint32_t)eb : (uint32_t)(eb >> 32);
    }
    reinterpret_cast<uint32_t*>(S.blob)[tid] = hw;
  }

  const uint64_t b0 = tile * TB;
  const int nblk = tile < ntiles ? (int)(nb - b0 < (uint64_t)TB ? nb - b0 : (uint64_t)TB) : 0;
  const uint64_t v0 = b0 * BLOCK;
  const int nval = nblk ? (int)(n - v0 < (uint64_t)TILE_VALUES ? n - v0 : (uint64_t)TILE_VALUES) : 0;

  // ---- 1. source tile into shared memory
  if (nblk) {
    fill_tile(xs, S.x, v0, nval);
    if (SRC == SRC_STEP) {
      const uint64_t ts = a.in_tile_off[tile], te = a.in_tile_off[tile + 1];
      const int base = stage_bytes(stage, a.in_blob + HEADER_BYTES, ts, te);
      __syncthreads();
      decode_tile<1>(stage, base, (int)(te - ts), a.in_sub_off + tile * GROUPS, nblk, b0, nb, last_cnt, a.in_tw, xs,
                     a.op, a.st);
      __syncthreads();
      if (a.acc_out) drain_tile(xs, a.acc_out, v0, nval);
    } else {
      __syncthreads();
    }
  }

  // ---- 2. closed-loop quantisation, one thread per 32-value block
  const bool active = tid < nblk;
  const int cnt = active ? ((b0 + tid == nb - 1) ? last_cnt : 32) : 0;
  uint32_t z[31];
  uint32_t zor = 0;
  int flags = 0;
  float x0 = 0.0f;
  if (active) {
    float v[32];
    load_row(xs, tid, v);
    x0 = v[0];
    float prev32 = v[0];
    double prev64 = (double)prev32;
    if (!isfinite(prev32)) flags |= 4;
    if (cnt == 32) {
#pragma unroll
      for (int j = 1; j < 32; ++j) {
        z[j - 1] = closed_loop_step(v[j], prev32, prev64, a.qp, flags);
        zor |= z[j - 1];
      }
    } else {
#pragma unroll
      for (int j = 1; j < 32; ++j) {
        z[j - 1] = 0;
        if (j < cnt) {
          z[j - 1] = closed_loop_step(v[j], prev32, prev64, a.qp, flags);
          zor |= z[j - 1];
        }
      }
    }
    if (flags & 4) {  // codec.py:83-85: report the first non-finite offset
      for (int j = 0; j < cnt; ++j)
        if (!isfinite(xs[xs_index(tid, j >> 2) + (j & 3)])) {
          atomicMin(&a.st->first_nonfinite, (unsigned long long)(v0 + (uint64_t)tid * 32 + j));
          break;
        }
    }
  }
  const int w = 32 - __clz(zor);                                   // codec.py:224-229
  const int ncodes = cnt - 1;
  const int packed = 5 + (ncodes * w + 7) / 8;                     // 236
  const int rawsz = 1 + 4 * cnt;                                   // 237
  const bool raw = (flags & 3) || packed > rawsz;                  // 238
  const int size = active ? (raw ? rawsz : packed) : 0;            // 239
  const int wbyte = raw ? RAW_WIDTH : w;

  // ---- 3. CTA exclusive scan of block sizes (codec.py:241-243)
  int incl = size;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if (lane >= d) incl += t;
  }
  if (lane == 31) s_warp[warp] = incl;
  s_wbyte[tid] = wbyte;
  if (tid == 0) s_wbyte[TB] = 0;
  __syncthreads();
  int wpre = 0, tile_bytes = 0;
#pragma unroll
  for (int k = 0; k < TB / 32; ++k) {
    const int t = s_warp[k];
    wpre += k < warp ? t : 0;
    tile_bytes += t;
  }
  const int start = wpre + incl - size;

  // ---- 4. publish the tile aggregate early (decoupled look-back)
  if (tid == 0 && tile < ntiles) {
    st_volatile_u64(&ws->status[gt], mk_status(gen, tile == 0 ? 2u : 1u, (unsigned long long)tile_bytes));
  }

  // ---- 5. pack into the staging area (independent of the global offset)
  if (active) {
    Appender ap;
    ap.init(stage, start, tid == 0);
    if (raw) {
      ap.append(255ull | ((uint64_t)__float_as_uint(x0) << 8), 5);
      int j = 1;
      for (; j + 1 < cnt; j += 2) {
        const float v1 = xs[xs_index(tid, j >> 2) + (j & 3)];
        const float v2 = xs[xs_index(tid, (j + 1) >> 2) + ((j + 1) & 3)];
        ap.append((uint64_t)__float_as_uint(v1) | ((uint64_t)__float_as_uint(v2) << 32), 8);
      }
      if (j < cnt) ap.append((uint64_t)__float_as_uint(xs[xs_index(tid, j >> 2) + (j & 3)]), 4);
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
    uint64_t lead = 0;
    if (tid + 1 < nblk) lead = (uint64_t)s_wbyte[tid + 1] | ((uint64_t)__float_as_uint(xs[xs_index(tid + 1, 0)]) << 8);
    ap.finish(lead);
  }

  // ---- 6. look-back for the tile's exclusive prefix
  if (tid == 0) {
    unsigned long long excl = 0;
    if (tile > 0 && tile < ntiles) {
      long long p = (long long)gt - 1;
      while (true) {
        const unsigned long long s = ld_volatile_u64(&ws->status[p]);
        const unsigned flag = (unsigned)((s >> 46) & 3);
        if (((s >> 48) & 0xFFFF) != (gen & 0xFFFF) || flag == 0) {
          __nanosleep(20);
          continue;
        }
        excl += s & VALUE_MASK;
        if (flag == 2) break;
        --p;
      }
      st_volatile_u64(&ws->status[gt], mk_status(gen, 2u, excl + (unsigned long long)tile_bytes));
    }
    s_excl = excl;
  }
  __syncthreads();
  const unsigned long long excl = s_excl;

  // ---- 7. sidecar, block offsets, length
  if (tile < ntiles) {
    if (lane == 0 && S.out_sub_off && warp < GROUPS) S.out_sub_off[tile * GROUPS + warp] = (uint16_t)(tid < nblk ? start : tile_bytes);
    if (tid == 0 && S.out_tile_off) S.out_tile_off[tile] = excl;
    if (active && a.blk_off && k == 0) a.blk_off[b0 + tid] = excl + (unsigned long long)start;
    if (tid == 0 && tile == ntiles - 1) {
      if (S.out_tile_off) S.out_tile_off[ntiles] = excl + tile_bytes;
      *S.out_len = HEADER_BYTES + excl + tile_bytes;
    }
  } else if (tid == 0 && ntiles == 0) {
    if (S.out_tile_off) S.out_tile_off[0] = 0;
    *S.out_len = HEADER_BYTES;
  }

  // ---- 8. store the tile: aligned 16-byte chunks + byte-wise edges
  if (tile_bytes > 0) {
    uint8_t* gdst = S.blob + HEADER_BYTES + excl;
    const uintptr_t A = reinterpret_cast<uintptr_t>(gdst);
    const uintptr_t E = A + (uintptr_t)tile_bytes;
    const uintptr_t cf = (A + 15) & ~(uintptr_t)15, cl = E & ~(uintptr_t)15;
    if (cf < cl) {
      const int off0 = (int)(cf - A);            // staging byte of the first full chunk
      const int sh = (off0 & 3) * 8;
      const int nch = (int)((cl - cf) >> 4);
      uint4* dst = reinterpret_cast<uint4*>(cf);
      for (int c = tid; c < nch; c += TB) {
        const int wi = (off0 >> 2) + 4 * c;
        const uint32_t w0 = stage[wi], w1 = stage[wi + 1], w2 = stage[wi + 2], w3 = stage[wi + 3], w4 = stage[wi + 4];
        uint4 v;
        v.x = __funnelshift_r(w0, w1, sh);
        v.y = __funnelshift_r(w1, w2, sh);
        v.z = __funnelshift_r(w2, w3, sh);
        v.w = __funnelshift_r(w3, w4, sh);
        dst[c] = v;
      }
      const int head = (int)(cf - A), tail = (int)(E - cl);
      const uint8_t* sb = reinterpret_cast<const uint8_t*>(stage);
      if (tid < head) gdst[tid] = sb[tid];
      else if (tid >= 32 && tid - 32 < tail) gdst[tile_bytes - tail + (tid - 32)] = sb[tile_bytes - tail + (tid - 32)];
    } else {
      const uint8_t* sb = reinterpret_cast<const uint8_t*>(stage);
      for (int i = tid; i < tile_bytes; i += TB) gdst[i] = sb[i];
    }
  }

  // ---- 9. retire: the last CTA to finish resets the tickets and bumps gen
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
// Decompress with sidecar offsets: one CTA per tile.
__global__ void __launch_bounds__(TB) k_tile_decode(const DecodeArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  float* xs = reinterpret_cast<float*>(smem);
  uint32_t* stage = reinterpret_cast<uint32_t*>(smem + TB * 128);
  const uint64_t tile = blockIdx.x;
  const uint64_t n = a.n;
  const uint64_t nb = (n + BLOCK - 1) / BLOCK;
  const int last_cnt = (int)(n - (nb - 1) * BLOCK);
  const uint64_t b0 = tile * TB;
  const int nblk = (int)(nb - b0 < (uint64_t)TB ? nb - b0 : (uint64_t)TB);
  const uint64_t v0 = b0 * BLOCK;
  const int nval = (int)(n - v0 < (uint64_t)TILE_VALUES ? n - v0 : (uint64_t)TILE_VALUES);
  const uint64_t ts = a.tile_off[tile], te = a.tile_off[tile + 1];
  const int base = stage_bytes(stage, a.blob + HEADER_BYTES, ts, te);
  __syncthreads();
  decode_tile<0>(stage, base, (int)(te - ts), a.sub_off + tile * GROUPS, nblk, b0, nb, last_cnt, a.tw, xs, 0, a.st);
  __syncthreads();
  drain_tile(xs, a.y, v0, nval);
}

}  // namespace gz
