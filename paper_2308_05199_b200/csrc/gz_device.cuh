// gz_device.cuh -- device building blocks of the B200 gZCCL codec (sm_100a).
//
// Wire format = the reference's frozen byte format (pkg/src/gzccl/codec.py:1-31):
//   24-byte header "GZC1" | 4 zero bytes | u64 n | f64 eb, then per 32-value
//   block: width byte w (0..32, 255 = raw), the first value verbatim (f32 LE),
//   then 31 zigzag codes packed LSB-first at w bits (raw: all values verbatim).
//
// Device layout: the unit of work is a WARP TILE = 32 consecutive 32-value
// blocks (4 KB of input), one block per lane.  Each warp of a persistent grid
// loops over warp tiles in ticket order with no CTA-wide barrier:
//   * the next tile's values stream into the warp's second shared-memory
//     buffer (cp.async) while the current one is quantised; tiles are stored
//     with a 128B XOR swizzle so that both the coalesced fill and the
//     per-lane row reads are free of bank conflicts;
//   * every lane runs the closed-loop quantizer (codec.py:188-216) serially
//     over the 31 steps of its block;
//   * block sizes are scanned with warp shuffles, tile offsets come from a
//     warp-wide decoupled look-back across tiles (codec.py:241-243 np.cumsum),
//     and the packed tile is written with aligned 16-byte stores (which may
//     target a peer GPU's memory over NVLink);
//   * a sidecar (u64 payload offset per tile + u16 offset of every 8th block
//     inside its tile) lets decoders find block starts with 8-step walks
//     instead of the sequential walk of codec.py:305-320.  The blob itself
//     stays bit-exact.
//
// Numerics: compile with --fmad=false.  Every f64 operation mirrors one numpy
// ufunc of the reference; see fast_block() for the exactness argument
// behind the f32 fast path.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace gz {

constexpr int BLOCK = 32;           // codec.py:42
constexpr int HEADER_BYTES = 24;    // codec.py:43-44
constexpr int RAW_WIDTH = 255;      // codec.py:45
constexpr int TB = 32;              // blocks per warp tile (one per lane)
constexpr int GROUP = 8;            // blocks per sidecar sub-offset
constexpr int GROUPS = TB / GROUP;  // sub-offsets per tile
constexpr int WARPS = 4;            // independent warps per CTA
constexpr int CTA_THREADS = 32 * WARPS;
constexpr int TILE_VALUES = TB * BLOCK;                    // 1024 values, 4 KB
constexpr int MAX_BLOCK_BYTES = 1 + 4 * BLOCK;             // raw block, 129
constexpr int STAGE_BYTES = TB * MAX_BLOCK_BYTES + 64;     // packed tile + slack
constexpr int STAGE_WORDS = STAGE_BYTES / 4;
constexpr float MAGIC32 = 12582912.0f;                     // 1.5 * 2^23
constexpr int MAGIC32_BITS = 0x4B400000;
constexpr double M52_PLUS_MAGIC32 = 4503599627370496.0 + (double)MAGIC32_BITS;  // 2^52 + bits(MAGIC32)
// zigzag codes in shared memory carry the bias ZBIAS = bits(2^23) (fast_block forms
// them as the binary32 2^23 + z); the bias is removed modulo 2^32 when packing
constexpr uint32_t ZBIAS = 0x4B000000u;
constexpr uint32_t ZBIAS_MASK = 0x001FFFFFu;
// every biased code of a block is ZBIAS + z with z < 2^21
__device__ __forceinline__ bool zbias_valid(uint32_t zor) { return (zor & ~ZBIAS_MASK) == ZBIAS; }

// ---- device workspace: zero-initialised once, reused by every launch -------
// Layout: this header, tile sizes (u32 per tile), scratch slots.
// agg[g], agg2[g / 32], agg3[g / 1024] = compressed bytes of gather group g,
// of groups 32*(g/32) .. +31 and of groups 1024*(g/1024) .. +1023,
// accumulated by the encoder kernel (over all segments of a launch) and
// zeroed again by the last gather CTA to retire, so no per-launch memset is
// needed and CUDA-graph replay is safe.
constexpr int MAXGRID = 16384;   // gather groups per launch
constexpr int TILE_SLOT = 4224;  // scratch bytes reserved per tile (>= 32 * 129, 128-aligned)
struct TileWs {
  unsigned long long done;          // gather retire counter (own 128-byte line)
  unsigned long long pad0[15];
  unsigned int claim;               // encoder tile claims (own 128-byte line)
  unsigned int pad1[31];
  unsigned int agg[MAXGRID];
  unsigned int agg2[MAXGRID / 32];
  unsigned int agg3[MAXGRID / 1024];
};
// the encoder addresses agg2 / agg3 as agg[MAXGRID + ...]
static_assert(offsetof(TileWs, agg2) == offsetof(TileWs, agg) + 4 * MAXGRID &&
                  offsetof(TileWs, agg3) == offsetof(TileWs, agg2) + 4 * (MAXGRID / 32),
              "TileWs counter arrays must be consecutive");

struct Status {                          // error reporting (host-reset to ~0)
  unsigned long long first_nonfinite;    // codec.py:83-85
  unsigned long long decode_error;       // (block << 24) | (width << 8) | code, min over blocks
  unsigned long long trailing;           // trailing byte count of a DE_TRAIL error (codec.py:321-322)
  unsigned long long comm_error;         // COMM_* code of a peer-flag wait that gave up (~0 if none)
};
enum CommErr : unsigned { COMM_FLAG_TIMEOUT = 1 };
enum DecodeErr : unsigned { DE_WIDTH = 1, DE_TRUNC = 2, DE_TRAIL = 3, DE_SIDECAR = 4, DE_HEADER = 5 };

struct QParams {
  double tw;     // fl64(2*eb), codec.py:188
  double eb;
  float rtw;     // RN32(1/tw)                       (fast path only)
  float thr;     // 0.5 - 2^-20: rounding margin      (fast path only)
  float elo;     // <= eb * (1 - 2^-22), binary32     (fast path only)
  float ehi;     // >= eb * (1 + 2^-22), binary32     (fast path only)
  int fast;      // 1 if tw lies in the range where the fast path is proven exact
};

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// ---------------------------------------------------------------------------
// shared-memory warp tile of 32 rows x 32 floats, 128-byte rows, 16-byte chunks
// XOR-swizzled by (row & 7): coalesced fills and per-row float4 reads are
// both free of bank conflicts.
__device__ __forceinline__ int xs_index(int row, int chunk) { return row * 32 + ((chunk ^ (row & 7)) << 2); }

__device__ __forceinline__ double i32_to_f64(int q) {
  // exact int32 -> binary64 without the 16/clk/SM conversion pipe:
  // 2^52 + (q + 2^31) has q in its low word; subtract the bias with one DADD.
  return __dsub_rn(__hiloint2double(0x43300000, (unsigned)q ^ 0x80000000u), 4503601774854144.0);
}

// np.copyto(int32, float64, casting="unsafe") on x86: NaN/out of range -> INT32_MIN
__device__ __forceinline__ int np_f64_to_i32(double q) {
  if (isnan(q) || q >= 2147483648.0 || q < -2147483648.0) return (int)0x80000000u;
  return __double2int_rz(q);
}

struct StepOut {
  float rec;
  int code;
  int flags;  // bit0: overflow (|q| > 2^30), bit1: |rec - x| > eb, bit2: x non-finite
};

// Exact restatement of one closed-loop step, codec.py:191-210, in binary64.
// Used for every step the fast path cannot prove (rare), and for all steps
// when eb is outside the fast path's range.
__device__ __noinline__ StepOut slow_step(float prev32, float x, double tw, double eb) {
  StepOut o;
  double prev = (double)prev32;                      // 191
  double target = (double)x;                         // 192
  double q = __ddiv_rn(__dsub_rn(target, prev), tw); // 193-194
  double a = floor(__dadd_rn(fabs(q), 0.5));         // 196-198
  double sg = isnan(q) ? q : (q > 0.0 ? 1.0 : (q < 0.0 ? -1.0 : 0.0));  // 199 np.sign
  q = __dmul_rn(a, sg);                              // 200
  int ovf = fabs(q) > 1073741824.0;                  // 201-202
  if (q < -1073741824.0) q = -1073741824.0;          // 203 np.clip
  else if (q > 1073741824.0) q = 1073741824.0;
  o.code = np_f64_to_i32(q);                         // 204
  double s = __dadd_rn(prev, __dmul_rn(q, tw));      // 205-206
  o.rec = __double2float_rn(s);                      // 207
  double e = fabs(__dsub_rn((double)o.rec, target)); // 208-210
  o.flags = ovf | ((e > eb) << 1) | ((!isfinite(x)) << 2);
  return o;
}

// Exact replay of one block with the reference arithmetic (codec.py:188-219),
// writing the zigzag codes (codec.py:131-139) to z[0..cnt-2].  Used for the
// partial final block, for blocks the fast pass could not prove, and for all
// blocks when eb lies outside the fast path's range.  Returns the zigzag OR
// and ORs overflow / error / non-finite flags into *flags.
__device__ __noinline__ uint32_t slow_block(const float* xs_row_vals, int cnt, const QParams P, uint32_t* z,
                                            int* flags) {
  // Step by step: the proven fast decision where it applies (see fast_block),
  // the verbatim reference arithmetic (slow_step) where it does not.
  float prev32 = xs_row_vals[0];
  int f = isfinite(prev32) ? 0 : 4;
  uint32_t zor = 0;
  for (int j = 1; j < cnt; ++j) {
    const float x = xs_row_vals[j];
    int code;
    bool done = false;
    if (P.fast) {
      const float vf = __fmul_rn(__fsub_rn(x, prev32), P.rtw);
      const float m = __fadd_rn(vf, MAGIC32);
      const float fr = __fsub_rn(vf, __fsub_rn(m, MAGIC32));
      if (fmaf(fabsf(vf), 0x1p-21f, fabsf(fr)) < P.thr) {
        code = __float_as_int(m) - MAGIC32_BITS;
        const double t = __dadd_rn((double)prev32, __dmul_rn(i32_to_f64(code), P.tw));
        prev32 = __double2float_rn(t);
        const float e = fabsf(__fsub_rn(prev32, x));
        if (e > P.ehi) f |= 2;
        else if (e >= P.elo && fabs(__dsub_rn((double)prev32, (double)x)) > P.eb) f |= 2;
        done = true;
      }
    }
    if (!done) {
      const StepOut o = slow_step(prev32, x, P.tw, P.eb);
      prev32 = o.rec;
      f |= o.flags;
      code = o.code;
    }
    const uint32_t zz = ((uint32_t)code << 1) ^ (uint32_t)(code >> 31);
    z[j - 1] = zz;
    zor |= zz;
  }
  for (int j = cnt; j < 32; ++j) z[j - 1 < 0 ? 0 : j - 1] = 0;
  *flags |= f;
  return zor;
}

// Branch-free fast pass over one full 32-value block (f32 pipe for the
// quantisation decision, binary64 for the reconstruction).
// Returns FB_PACKED (codes exact, every |rec - x| <= eb), FB_RAW (codes
// exact and some |rec - x| > eb: the block is stored raw, codec.py:238) or
// FB_SLOW (a step could not be proven; replay with slow_block()).
//
// Per step, with prev = previous reconstruction (f32 prev32, exact f64 prev64):
//   vf = RN32(RN32(x - prev) * RN32(1/tw)) approximates the reference's
//   v = fl64(fl64(x-prev)/tw) with |vf - v| <= 3.01 * 2^-24 |v|.
//   m = vf + 1.5*2^23 holds q = RNE(vf) for |vf| < 2^22; fr = vf - q.
//   If |fr| + 2^-21 |vf| < 0.5 - 2^-20 then |v| is more than 2^-21 away from
//   every half-integer, so floor(fl64(|v|+0.5))*sign(v) == q.
//   Only max|fr| is tracked per step; the test runs once per block with
//   |vf| <= |q| + 1/2 <= 2^(w-1) + 1/2 (w = bit width of the zigzag codes).
//   Requiring w <= 21 also proves |vf| < 2^21 (the magic-constant rounding is
//   valid and |q| <= 2^20, no overflow, codec.py:201-204): a larger |vf|, an
//   infinity or a NaN turns into an integer code of width >= 22.
//   The reconstruction rec = RN32(fl64(prev + fl64(q*tw))) is computed exactly
//   as codec.py:205-207 does.  The error test of codec.py:208-210 is decided
//   in binary32: e = RN32(|rec - x|) has relative error <= 2^-24, so
//   max e < elo (<= eb (1 - 2^-22)) proves every |rec - x| <= eb and
//   max e > ehi (>= eb (1 + 2^-22)) proves some |rec - x| > eb; only a
//   maximum inside [elo, ehi] is undecided.
//   The zigzag code is formed in binary32 as well: with q exact, tz = 2q + 1/2 is exact
//   and RN32(|tz| + (2^23 - 1/2)) = 2^23 + z exactly (z = |2q + 1/2| - 1/2 = zigzag(q)),
//   so its bits are ZBIAS + z.  The codes are kept in this biased form in shared
//   memory (packing removes the bias with modular arithmetic).  If |vf| >= 2^22 (m
//   outside the magic range), or vf is Inf/NaN, |tz| >= 2^23 - 1/2 or is Inf/NaN, so
//   the biased code has bits 21..23 set or an exponent other than 150: requiring the
//   OR of the biased codes to equal ZBIAS in bits 21..31 proves every z < 2^21 (the
//   former w <= 21 test, now also covering the range of m).
enum { FB_PACKED = 0, FB_RAW = 1, FB_SLOW = 2 };

// COMPACT: the seven 4-step chunks after the first run as a loop (a quarter
// of the code; for kernels whose hot loop would not fit the instruction cache).
template <bool COMPACT = false>
__device__ __forceinline__ int fast_block(const float* xs, float* zs, int row, double tw, float rtw, float thr,
                                          float elo, float ehi, uint32_t& zor_out, float& x0) {
  // The codes go to the same row of zs (zs == xs: they overwrite the
  // consumed values in place): slot j of the row receives code j-1 (slot 0
  // keeps x0), one 16-byte store per 4 steps.
  float4 c4 = *reinterpret_cast<const float4*>(xs + xs_index(row, 0));
  float prev32 = c4.x;
  x0 = c4.x;
  double prev64 = (double)prev32;
  float frmax = 0.0f;  // max |vf - q|
  float emax = 0.0f;   // max |rec - x|
  uint32_t zor = 0;    // OR of the biased codes ZBIAS + z
  auto step = [&](float x) -> uint32_t {
    const float vf = __fmul_rn(__fsub_rn(x, prev32), rtw);
    const float m = __fadd_rn(vf, MAGIC32);
    const float qf = __fsub_rn(m, MAGIC32);  // q, exact while |vf| < 2^22
    frmax = fmaxf(frmax, fabsf(__fsub_rn(vf, qf)));
    // q in binary64 straight from m's bits: (2^52 + bits(m)) - (2^52 + bits(MAGIC32)), one DADD
    const double qd = __dsub_rn(__hiloint2double(0x43300000, __float_as_int(m)), M52_PLUS_MAGIC32);
    const double t = __dadd_rn(prev64, __dmul_rn(qd, tw));
    prev32 = __double2float_rn(t);
    prev64 = (double)prev32;
    emax = fmaxf(emax, fabsf(__fsub_rn(prev32, x)));
    // zigzag(q) = |2q + 1/2| - 1/2, formed in the f32 pipe as the bits of 2^23 + z (two exact
    // ops, no integer shift/xor chain); see zbias_valid() for the out-of-range cases
    const float tz = __fmaf_rn(qf, 2.0f, 0.5f);
    const uint32_t z = __float_as_uint(__fadd_rn(fabsf(tz), 8388607.5f));
    zor |= z;
    return z;
  };
  {
    const uint32_t z1 = step(c4.y), z2 = step(c4.z), z3 = step(c4.w);
    *reinterpret_cast<uint4*>(zs + xs_index(row, 0)) = make_uint4(__float_as_uint(x0), z1, z2, z3);
  }
#pragma unroll(COMPACT ? 1 : 7)
  for (int c = 1; c < 8; ++c) {
    c4 = *reinterpret_cast<const float4*>(xs + xs_index(row, c));
    const uint32_t z0 = step(c4.x), z1 = step(c4.y), z2 = step(c4.z), z3 = step(c4.w);
    *reinterpret_cast<uint4*>(zs + xs_index(row, c)) = make_uint4(z0, z1, z2, z3);
  }
  if (!zbias_valid(zor)) return FB_SLOW;
  zor_out = zor & ZBIAS_MASK;
  const int w = 32 - __clz(zor_out);
  const float vmax = __int_as_float((126 + w) << 23) + 0.5f;  // 2^(w-1) + 1/2 (exact; w = 0 gives 1)
  if (!(fmaf(vmax, 0x1p-21f, frmax) < thr)) return FB_SLOW;
  if (emax > ehi) return FB_RAW;             // some error provably > eb
  return emax >= elo ? FB_SLOW : FB_PACKED;  // undecided within 2^-22 of eb
}

// code j (0..30) of a row written by fast_block / store_codes, biased: ZBIAS + z (mod 2^32)
__device__ __forceinline__ void load_codes(const float* xs, int row, uint32_t (&z)[31]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint4 v = *reinterpret_cast<const uint4*>(xs + xs_index(row, c));
    if (c > 0) z[4 * c - 1] = v.x;
    z[4 * c + 0] = v.y;
    z[4 * c + 1] = v.z;
    if (4 * c + 2 < 31) z[4 * c + 2] = v.w;
  }
}
__device__ __forceinline__ void store_codes(float* xs, int row, float x0, const uint32_t* z) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint32_t a = c ? z[4 * c - 1] + ZBIAS : __float_as_uint(x0);
    *reinterpret_cast<uint4*>(xs + xs_index(row, c)) =
        make_uint4(a, z[4 * c] + ZBIAS, z[4 * c + 1] + ZBIAS, z[4 * c + 2] + ZBIAS);
  }
}

// ---------------------------------------------------------------------------
// Byte appender into the shared staging area (32-bit words).  A thread writes
// exactly the words whose first byte lies in its block; the last such word is
// completed with the first bytes of the next block ([w][x0...]), so no two
// threads ever store the same word and no atomics are needed.
__device__ __forceinline__ void st_u32_hint(uint32_t* p, uint32_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}

struct Appender {
  uint32_t* stage;  // global memory (a scratch run or slot)
  uint64_t pol;     // L2 policy of the stores
  int wi;          // word index of the pending word
  uint32_t pend;   // pending bytes (low npend bytes valid)
  int npend;
  bool skip;       // first word belongs to the previous block
  __device__ __forceinline__ void init(uint32_t* s, int byte_pos, bool owns_first) {
    stage = s;
    wi = byte_pos >> 2;
    npend = byte_pos & 3;
    pend = 0;
    skip = (npend != 0) && !owns_first;
  }
  // first block of a tile appended to a run: the previous tile left its last
  // partial word as `carry` (low byte_pos & 3 bytes valid)
  __device__ __forceinline__ void init_carry(uint32_t* s, int byte_pos, uint32_t carry) {
    stage = s;
    wi = byte_pos >> 2;
    npend = byte_pos & 3;
    pend = npend ? carry : 0u;
    skip = false;
  }
  __device__ __forceinline__ void put(uint32_t w) {
    if (!skip) st_u32_hint(stage + wi, w, pol);
    skip = false;
    ++wi;
  }
  // append the low L bytes (L <= 8) of c; bytes of c above L must be zero
  // unless this append completes the final word (then they are shifted out).
  __device__ __forceinline__ void append(uint64_t c, int L) {
    const int sh = npend * 8;
    const uint32_t lo = (uint32_t)c, hi = (uint32_t)(c >> 32);
    const uint32_t w0 = pend | (lo << sh);
    const uint32_t w1 = __funnelshift_l(lo, hi, sh);
    const uint32_t w2 = __funnelshift_l(hi, 0u, sh);
    const int T = npend + L;
    if (T >= 4) put(w0);
    if (T >= 8) put(w1);
    pend = T >= 8 ? w2 : (T >= 4 ? w1 : w0);
    npend = T & 3;
  }
  // finish: complete the last word with the next block's leading bytes
  __device__ __forceinline__ void finish(uint64_t next_lead) {
    if (npend) append(next_lead, 4 - npend);
  }
};

// Packing fast path for a warp whose 32 blocks are all full, packed (not raw)
// and of width w <= 4 (most tiles of a smooth field): the lane assembles its
// whole block -- [w][x0][31 codes LSB-first] (codec.py:244-270) followed by
// the next block's leading bytes that complete its last word -- as a 192-bit
// value, shifts it to the block's byte alignment and stores its words, with
// the same word ownership as Appender (a block whose start is not word
// aligned leaves its first word to the previous block).  Uniform control
// flow; ~100 instructions per block instead of ~270 for the streaming
// Appender.  z: the 31 biased codes (load_codes).
__device__ __forceinline__ void pack_small(uint32_t* dst, int start, int w, float x0, const uint32_t (&z)[31],
                                           uint32_t next_lead, uint64_t pol) {
  const uint32_t P1 = 1u << w, P2 = 1u << (2 * w);
  const uint32_t K = ZBIAS * (1u + P1) * (1u + P2);  // bias of a quad of biased codes (mod 2^32)
  uint32_t oct[4];                                     // 8 codes = w bytes each
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    uint32_t pr[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j0 = 8 * g + 2 * i;
      pr[i] = z[j0] + ((j0 + 1 < 31) ? z[j0 + 1] : ZBIAS) * P1;
    }
    const uint32_t qa = pr[0] + pr[1] * P2 - K, qb = pr[2] + pr[3] * P2 - K;
    oct[g] = qa | (qb << (4 * w));
  }
  // codes bitstream C (31 w <= 124 bits) = oct0 | oct1 << 8w | oct2 << 16w | oct3 << 24w
  const uint64_t A = (uint64_t)oct[0] | ((uint64_t)oct[1] << (8 * w));
  const uint64_t B = (uint64_t)oct[2] | ((uint64_t)oct[3] << (8 * w));
  const int sB = 16 * w;  // 0..64
  const uint64_t Clo = A | (sB < 64 ? (B << sB) : 0ull);
  const uint64_t Chi = sB == 0 ? 0ull : (sB < 64 ? (B >> (64 - sB)) : B);
  // block = header (40 bits) | C << 40, then the next block's lead bytes at its end
  uint64_t S0 = (uint64_t)w | ((uint64_t)__float_as_uint(x0) << 8) | (Clo << 40);
  uint64_t S1 = (Clo >> 24) | (Chi << 40);
  uint64_t S2 = Chi >> 24;
  const int size = 5 + ((31 * w + 7) >> 3);  // codec.py:236, 21 bytes at most
  const int pb = 8 * size;                    // 40 .. 168
  const uint64_t NL = next_lead;
  if (pb < 64) {
    S0 |= NL << pb;
    S1 |= NL >> (64 - pb);
  } else if (pb < 128) {
    S1 |= NL << (pb - 64);
    if (pb > 64) S2 |= NL >> (128 - pb);
  } else {
    S2 |= NL << (pb - 128);
  }
  const uint32_t sw[6] = {(uint32_t)S0, (uint32_t)(S0 >> 32), (uint32_t)S1, (uint32_t)(S1 >> 32), (uint32_t)S2,
                          (uint32_t)(S2 >> 32)};
  const int al = start & 3, sh = 8 * al;
  const int nw = (al + size + 3) >> 2;  // <= 6
  uint32_t* p = dst + (start >> 2);
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const uint32_t t = __funnelshift_l(k ? sw[k - 1] : 0u, sw[k], sh);
    if (k < nw && (k > 0 || al == 0)) st_u32_hint(p + k, t, pol);
  }
}

// load one 32-value row from the swizzled tile
__device__ __forceinline__ void load_row(const float* xs, int row, float (&v)[32]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    float4 f = *reinterpret_cast<const float4*>(xs + xs_index(row, c));
    v[4 * c + 0] = f.x;
    v[4 * c + 1] = f.y;
    v[4 * c + 2] = f.z;
    v[4 * c + 3] = f.w;
  }
}

// ---------------------------------------------------------------------------
// status word helpers (decoupled look-back)
__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
}  // namespace gz
