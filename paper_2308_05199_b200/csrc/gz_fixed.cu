// gz_fixed.cu -- the fixed-rate baseline codec of the reference
// (codec.py:442-489), a comparator for the error-bounded codec: uniform
// scalar quantisation of the whole buffer over [min, max] to b bits per value
// (1..16), codes packed LSB-first with no per-block structure, after a
// 17-byte header "<QBff" (n, b, lo, hi).  Thread t owns values [32t, 32t+32):
// their 32 codes are exactly b 32-bit words of the packed stream, stored
// byte-wise after the odd-sized header.
#include "gz_device.cuh"

namespace gz {

constexpr int FR_HEADER_BYTES = 17;

// ordered-int encoding of finite floats for atomicMin/atomicMax; the two
// zeros map to the same key (numpy compares values: -0.0 == +0.0), their sign
// is settled separately (k_fr_zero_lanes / fr_zero_winner)
__device__ __forceinline__ int fr_ord(float f) {
  const int i = __float_as_int(f) == (int)0x80000000 ? 0 : __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float fr_unord(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF); }

// Scratch layout (gz_fr_workspace_bytes): mm[0] = ord(min), mm[1] = ord(max)
// (host-initialised to INT_MAX / INT_MIN), then 17 signed 64-bit "last zero"
// indices (16 SIMD lanes + the scalar tail; host-initialised to -1).
struct FrScratch {
  int mm[2];
  long long zlast[17];
};

__global__ void k_fr_init(FrScratch* sc) {
  const int t = threadIdx.x;
  if (t == 0) sc->mm[0] = 0x7FFFFFFF;
  if (t == 1) sc->mm[1] = (int)0x80000000;
  if (t < 17) sc->zlast[t] = -1;
}

// mm = value min / max of x; non-finite inputs are reported like codec.py:83-85
__global__ void k_fr_minmax(const float* __restrict__ x, uint64_t n, FrScratch* sc, Status* st) {
  int lo = 0x7FFFFFFF, hi = (int)0x80000000;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const float v = __ldg(x + i);
    if (!isfinite(v)) {
      atomicMin(&st->first_nonfinite, (unsigned long long)i);
      continue;
    }
    const int o = fr_ord(v);
    lo = min(lo, o);
    hi = max(hi, o);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, d));
    hi = max(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, d));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&sc->mm[0], lo);
    atomicMax(&sc->mm[1], hi);
  }
}

// Sign of a zero min / max, as numpy 2.x computes x.min() / x.max() for a
// contiguous float32 array on an AVX-512 host (the reference's fixed_rate_compress,
// codec.py:454-455; numpy's simd_reduce_c loop in loops_minmax.dispatch.c.src):
// the accumulator starts as 16 copies of x[0], x[1 + 16j + l] is folded into
// lane l with vminps/vmaxps (the SECOND operand wins a tie, so a lane keeps its
// last zero), the lanes are combined by GCC's _mm512_reduce_min_ps /
// _mm512_reduce_max_ps tree, and the (n - 1) % 16 tail values are folded in
// one by one (again the later value wins a tie).  Only zeros tie with a zero
// extremum, so both signs follow from the last zero index of every lane and of
// the tail (checked against numpy on random sign patterns, tests/test_fixed_rate*).
__global__ void k_fr_zero_lanes(const float* __restrict__ x, uint64_t n, FrScratch* sc) {
  if (fr_unord(sc->mm[0]) != 0.0f && fr_unord(sc->mm[1]) != 0.0f) return;  // no zero extremum
  const uint64_t nv = n ? (n - 1) / 16 : 0;  // full 16-lane vectors after x[0]
  for (uint64_t i = 1 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    if (__ldg(x + i) != 0.0f) continue;
    const int slot = i < 1 + 16 * nv ? (int)((i - 1) & 15) : 16;
    atomicMax(&sc->zlast[slot], (long long)i);
  }
}

// index of the element whose sign numpy's reduction returns, given the value
// key of the extremum (a zero): lane candidates = last zero of the lane, else
// x[0] if it is zero; lanes without a zero hold a larger (min) / smaller (max)
// value and lose every comparison
__device__ long long fr_zero_winner(const float* x, const FrScratch* sc) {
  long long lane[16];
  const bool x0z = x[0] == 0.0f;
  for (int l = 0; l < 16; ++l) lane[l] = sc->zlast[l] >= 0 ? sc->zlast[l] : (x0z ? 0 : -1);
  // f(a, b): a wins only if it is a zero and b is not (ties -> b)
  auto f = [](long long a, long long b) { return b >= 0 ? b : a; };
  long long t3[8], t6[4];
  for (int i = 0; i < 8; ++i) t3[i] = f(lane[8 + i], lane[i]);  // _mm256_min_ps(hi, lo)
  for (int i = 0; i < 4; ++i) t6[i] = f(t3[4 + i], t3[i]);       // _mm_min_ps(hi, lo)
  const long long t8a = f(t6[0], t6[2]), t8b = f(t6[1], t6[3]);   // shuffle {2,3,0,1}
  long long r = f(t8a, t8b);                                      // shuffle {1,0,1,0}
  if (sc->zlast[16] >= 0) r = sc->zlast[16];                      // scalar tail
  return r;
}

__global__ void k_fr_encode(const float* __restrict__ x, uint64_t n, int b, const FrScratch* sc, uint8_t* out,
                            uint64_t* d_len) {
  float lof = n ? fr_unord(sc->mm[0]) : 0.0f, hif = n ? fr_unord(sc->mm[1]) : 0.0f;
  const double lo = lof, hi = hif;  // a zero's sign never changes a code (x - (+-0) quantises alike)
  const uint32_t levels = (1u << b) - 1u;
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t payload = (n * (uint64_t)b + 7) >> 3;
  if (t == 0 && n && (lof == 0.0f || hif == 0.0f)) {  // header sign of a zero extremum (numpy's choice)
    const float zs = x[fr_zero_winner(x, sc)];
    if (lof == 0.0f) lof = zs;
    if (hif == 0.0f) hif = zs;
  }
  if (t == 0) {  // header "<QBff"
    const uint32_t lw = __float_as_uint(lof), hw = __float_as_uint(hif);
    const uint8_t hb[17] = {(uint8_t)n, (uint8_t)(n >> 8), (uint8_t)(n >> 16), (uint8_t)(n >> 24), (uint8_t)(n >> 32),
                            (uint8_t)(n >> 40), (uint8_t)(n >> 48), (uint8_t)(n >> 56), (uint8_t)b,
                            (uint8_t)lw, (uint8_t)(lw >> 8), (uint8_t)(lw >> 16), (uint8_t)(lw >> 24),
                            (uint8_t)hw, (uint8_t)(hw >> 8), (uint8_t)(hw >> 16), (uint8_t)(hw >> 24)};
    for (int k = 0; k < 17; ++k) out[k] = hb[k];
    *d_len = FR_HEADER_BYTES + payload;
  }
  const uint64_t v0 = t * 32;
  if (v0 >= n) return;
  uint32_t words[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) words[k] = 0;
  for (int j = 0; j < 32; ++j) {
    uint32_t q = 0;
    if (v0 + j < n && hi > lo) {  // codec.py:460-464
      const double v = __dmul_rn(__ddiv_rn(__dsub_rn((double)x[v0 + j], lo), __dsub_rn(hi, lo)), (double)levels);
      const double r = floor(__dadd_rn(fabs(v), 0.5)) * (v > 0 ? 1.0 : (v < 0 ? -1.0 : 0.0));
      q = r <= 0.0 ? 0u : (r >= (double)levels ? levels : (uint32_t)r);
    }
    const int bit = j * b;  // LSB-first (codec.py:96-105)
    words[bit >> 5] |= q << (bit & 31);
    if ((bit & 31) + b > 32) words[(bit >> 5) + 1] |= q >> (32 - (bit & 31));
  }
  // this thread's bytes of the payload: [4bt, 4bt + 4b) clipped to the payload
  const uint64_t p0 = 4ull * b * t;
  uint8_t* dst = out + FR_HEADER_BYTES + p0;
  for (int k = 0; k < 4 * b; ++k)
    if (p0 + k < payload) dst[k] = (uint8_t)(words[k >> 2] >> (8 * (k & 3)));
}

__global__ void k_fr_decode(const uint8_t* __restrict__ blob, uint64_t n, int b, float* __restrict__ y) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t v0 = t * 32;
  if (v0 >= n) return;
  const uint32_t lw = blob[9] | (blob[10] << 8) | (blob[11] << 16) | ((uint32_t)blob[12] << 24);
  const uint32_t hw = blob[13] | (blob[14] << 8) | (blob[15] << 16) | ((uint32_t)blob[16] << 24);
  const double lo = __uint_as_float(lw), hi = __uint_as_float(hw);
  const uint32_t levels = (1u << b) - 1u;
  const double step = __ddiv_rn(__dsub_rn(hi, lo), (double)levels);  // codec.py:485
  const uint64_t payload = (n * (uint64_t)b + 7) >> 3;
  const uint64_t p0 = 4ull * b * t;
  const uint8_t* src = blob + FR_HEADER_BYTES + p0;
  uint32_t words[17];
#pragma unroll
  for (int k = 0; k < 17; ++k) words[k] = 0;
  for (int k = 0; k < 4 * b; ++k)
    if (p0 + k < payload) words[k >> 2] |= (uint32_t)src[k] << (8 * (k & 3));
  const uint32_t mask = levels;
  for (int j = 0; j < 32 && v0 + j < n; ++j) {
    const int bit = j * b;
    uint32_t q = words[bit >> 5] >> (bit & 31);
    if ((bit & 31) + b > 32) q |= words[(bit >> 5) + 1] << (32 - (bit & 31));
    q &= mask;
    const double v = hi > lo ? __dadd_rn(lo, __dmul_rn((double)q, step)) : lo;  // codec.py:484-487
    y[v0 + j] = __double2float_rn(v);
  }
}

}  // namespace gz
