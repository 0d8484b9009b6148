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

// ordered-int encoding of finite floats for atomicMin/atomicMax
__device__ __forceinline__ int fr_ord(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float fr_unord(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF); }

// mm[0] = ord(min), mm[1] = ord(max) (host-initialised to INT_MAX / INT_MIN);
// non-finite inputs are reported like codec.py:83-85
__global__ void k_fr_minmax(const float* __restrict__ x, uint64_t n, int* mm, Status* st) {
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
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
  }
}

__global__ void k_fr_encode(const float* __restrict__ x, uint64_t n, int b, const int* mm, uint8_t* out,
                            uint64_t* d_len) {
  const float lof = n ? fr_unord(mm[0]) : 0.0f, hif = n ? fr_unord(mm[1]) : 0.0f;
  const double lo = lof, hi = hif;
  const uint32_t levels = (1u << b) - 1u;
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t payload = (n * (uint64_t)b + 7) >> 3;
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
