// gz_device.cuh -- device building blocks of the B200 gZCCL codec (sm_100a).
//
// Wire format = the reference's frozen byte format (pkg/src/gzccl/codec.py:1-31):
//   24-byte header "GZC1" | 4 zero bytes | u64 n | f64 eb, then per 32-value
//   block: width byte w (0..32, 255 = raw), the first value verbatim (f32 LE),
//   then 31 zigzag codes packed LSB-first at w bits (raw: all values verbatim).
//
// Device layout ("tile" = GZ_TB consecutive 32-value blocks = one CTA):
//   * one thread per 32-value block runs the closed-loop quantizer
//     (codec.py:188-216) serially over its 31 steps;
//   * input tiles are staged in shared memory with a 128B XOR swizzle so that
//     both the coalesced fill and the per-thread row reads are conflict-free;
//   * compressed bytes are packed into a shared-memory staging area, block
//     offsets come from a CTA scan + a decoupled look-back across tiles
//     (codec.py:241-243 np.cumsum), and the tile is written out with aligned
//     16-byte stores (which may target a peer GPU's memory over NVLink);
//   * a sidecar (u64 byte offset per tile + u16 offset per 32-block group)
//     lets decoders find block starts without the sequential walk of
//     codec.py:305-320.  The blob itself stays bit-exact.
//
// Numerics: compile with --fmad=false.  Every f64 operation mirrors one numpy
// ufunc of the reference; see closed_loop_step() for the exactness argument
// behind the f32 fast path.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#ifndef GZ_TB
#define GZ_TB 128
#endif

namespace gz {

constexpr int BLOCK = 32;           // codec.py:42
constexpr int HEADER_BYTES = 24;    // codec.py:43-44
constexpr int RAW_WIDTH = 255;      // codec.py:45
constexpr int TB = GZ_TB;           // blocks per tile == threads per CTA
constexpr int GROUPS = TB / 32;     // 32-block groups per tile (sub-offsets)
constexpr int TILE_VALUES = TB * BLOCK;
constexpr int MAX_BLOCK_BYTES = 1 + 4 * BLOCK;             // raw block, 129
constexpr int STAGE_BYTES = TB * MAX_BLOCK_BYTES + 64;     // packed tile + slack
constexpr int STAGE_WORDS = STAGE_BYTES / 4;
constexpr float MAGIC32 = 12582912.0f;                     // 1.5 * 2^23
constexpr int MAGIC32_BITS = 0x4B400000;

// ---- device workspace: zero-initialised once, reused by every launch -------
// status[t] = gen(16) | flag(2) | value(46).  flag 1 = tile aggregate,
// flag 2 = inclusive prefix.  `gen` advances when the last CTA of a launch
// finishes, so no per-launch memset is needed and CUDA-graph replay is safe.
struct TileWs {
  unsigned long long ticket;
  unsigned long long done;
  unsigned long long gen;
  unsigned long long pad;
  unsigned long long status[1];  // [ntiles]
};

struct Status {                          // error reporting (host-reset to ~0)
  unsigned long long first_nonfinite;    // codec.py:83-85
  unsigned long long decode_error;       // (block << 8) | code, min over blocks
  unsigned long long pad[2];
};
enum DecodeErr : unsigned { DE_WIDTH = 1, DE_TRUNC = 2, DE_TRAIL = 3, DE_SIDECAR = 4, DE_HEADER = 5 };

struct QParams {
  double tw;     // fl64(2*eb), codec.py:188
  double eb;
  float rtw;     // RN32(1/tw)            (fast path only)
  float kx;      // >= 2^-23 / tw         (fast path only)
  float thr;     // 0.5 - margin          (fast path only)
  int fast;      // 1 if tw lies in the range where the fast path is proven exact
};

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// ---------------------------------------------------------------------------
// shared-memory tile of TB rows x 32 floats, 128-byte rows, 16-byte chunks
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

// One step of the closed loop.  prev32/prev64 hold the previous reconstructed
// value (f32 and its exact f64).  Returns the zigzag code (codec.py:131-139).
//
// Fast path (f32 pipe, no conversions on the quantisation side):
//   vf = RN32(RN32(x - prev) * RN32(1/tw)) approximates v = fl64(fl64(x-prev)/tw)
//   with |vf - v| <= 3.01 * 2^-24 |v| (+ 2^-149 when subnormal).
//   m = vf + 1.5*2^23 gives RNE(vf) exactly for |vf| < 2^21, fr = vf - RNE(vf).
//   If  |fr| + 2^-21 |vf| + kx |x| < thr  (thr = 0.5 - 2^-20 - 2^-23) then
//     * |v| is at distance > 2^-21 from every half-integer, so the reference's
//       floor(fl64(|v| + 0.5)) * sign(v) equals RNE(vf) (ties impossible);
//     * |q| < 2^21: no overflow;
//     * the reconstruction error |rec - x| <= eb is guaranteed: it is bounded by
//       tw (|fr| + 2^-22.4 |vf|) + ulp32(t)/2 + 2^-53(|t| + |q tw|), and
//       kx |x| >= 2^-23 |x| / tw covers the rounding terms.
//   The reconstruction itself (codec.py:205-207) is always computed in binary64
//   exactly as the reference does: rec = RN32(fl64(prev + fl64(q * tw))).
// Otherwise slow_step() replays the reference arithmetic verbatim.
__device__ __forceinline__ uint32_t closed_loop_step(float x, float& prev32, double& prev64, const QParams& P,
                                                      int& flags) {
  int q;
  bool ok = false;
  float m = 0.f;
  if (P.fast) {
    float d32 = __fsub_rn(x, prev32);
    float vf = __fmul_rn(d32, P.rtw);
    m = __fadd_rn(vf, MAGIC32);
    float qf = __fsub_rn(m, MAGIC32);
    float fr = __fsub_rn(vf, qf);
    float c = fmaf(fabsf(x), P.kx, fmaf(fabsf(vf), 0x1p-21f, fabsf(fr)));
    ok = c < P.thr;
  }
  if (ok) {
    q = __float_as_int(m) - MAGIC32_BITS;
    double t = __dadd_rn(prev64, __dmul_rn(i32_to_f64(q), P.tw));
    prev32 = __double2float_rn(t);
  } else {
    StepOut o = slow_step(prev32, x, P.tw, P.eb);
    q = o.code;
    prev32 = o.rec;
    flags |= o.flags;
  }
  prev64 = (double)prev32;
  return ((uint32_t)q << 1) ^ (uint32_t)(q >> 31);
}

// ---------------------------------------------------------------------------
// Byte appender into the shared staging area (32-bit words).  A thread writes
// exactly the words whose first byte lies in its block; the last such word is
// completed with the first bytes of the next block ([w][x0...]), so no two
// threads ever store the same word and no atomics are needed.
struct Appender {
  uint32_t* stage;
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
  __device__ __forceinline__ void put(uint32_t w) {
    if (!skip) stage[wi] = w;
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
constexpr unsigned long long VALUE_MASK = (1ull << 46) - 1;
__device__ __forceinline__ unsigned long long mk_status(unsigned long long gen, unsigned flag, unsigned long long v) {
  return ((gen & 0xFFFF) << 48) | ((unsigned long long)flag << 46) | (v & VALUE_MASK);
}

}  // namespace gz
