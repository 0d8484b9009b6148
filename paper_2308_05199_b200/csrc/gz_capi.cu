// gz_capi.cu -- extern "C" entry points of libgzccl.so (declared in include/gzccl.h).
// Host-side argument checking, launch geometry and the peer-memory plumbing;
// all data-path work happens in the kernels of gz_codec.cu / gz_index.cu.
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "../../include/gzccl.h"
#include "gz_codec.cu"
#include "gz_index.cu"
#include "gz_fixed.cu"

using namespace gz;

namespace {

constexpr int MAXSEG = 32;  // segments per multi-segment launch (kernel-parameter budget)

// kernels launched by this library (all entry points, all streams): lets a
// benchmark count exactly which launches it timed
unsigned long long g_launches = 0;
inline void count_launch(unsigned k = 1) { __atomic_fetch_add(&g_launches, (unsigned long long)k, __ATOMIC_RELAXED); }

inline uint64_t nblocks(uint64_t n) { return (n + BLOCK - 1) / BLOCK; }
inline uint64_t ntiles_of(uint64_t n) { return (nblocks(n) + TB - 1) / TB; }

bool check_eb(double eb) { return std::isfinite(eb) && eb > 0.0; }

QParams make_qparams(double eb) {
  QParams p;
  p.eb = eb;
  p.tw = 2.0 * eb;  // codec.py:188
  p.fast = std::isfinite(p.tw) && p.tw >= std::ldexp(1.0, -100) && p.tw <= std::ldexp(1.0, 100);
  p.rtw = 0.f;
  p.thr = 0.f;
  p.elo = 0.f;
  p.ehi = 0.f;
  if (p.fast) {
    p.rtw = (float)(1.0 / p.tw);
    p.thr = 0.5f - 0x1p-20f;
    const double lo = eb * (1.0 - std::ldexp(1.0, -22));
    float f = (float)lo;
    if ((double)f > lo) f = std::nextafterf(f, 0.0f);
    p.elo = f;
    const double hi = eb * (1.0 + std::ldexp(1.0, -22));
    float g = (float)hi;
    if ((double)g < hi) g = std::nextafterf(g, INFINITY);
    p.ehi = g;
  }
  return p;
}

// Sidecar: u64 payload offset of every tile [ntiles + 1], then the width
// byte of every block, a full tile of 32 per tile [ntiles * 32].
struct SidecarView {
  uint64_t* tile_off;
  uint8_t* widths;
};
SidecarView sidecar_view(const void* sc, uint64_t n) {
  SidecarView v{nullptr, nullptr};
  if (!sc) return v;
  const uint64_t nt = ntiles_of(n);
  v.tile_off = reinterpret_cast<uint64_t*>(const_cast<void*>(sc));
  v.widths = reinterpret_cast<uint8_t*>(const_cast<void*>(sc)) + 8 * (nt + 1);
  return v;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Launch geometry is cached per device ordinal: the dynamic shared-memory
// opt-in (cudaFuncSetAttribute) is per device context, and devices may differ
// in SM count.  Zero-initialised caches hold value + 1 (0 = not yet computed).
constexpr int MAXDEV = 64;
inline int cur_dev() {
  int d = 0;
  cudaGetDevice(&d);
  return (d >= 0 && d < MAXDEV) ? d : 0;
}
inline int dev_sms(int dev) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 1;
}

// Persistent grid: as many CTAs as fit on the device at once (per device),
// after opting the kernel into `smem` bytes of dynamic shared memory there.
template <typename K>
int grid_cap(K kernel, int threads, size_t smem, int (&cache)[MAXDEV]) {
  const int dev = cur_dev();
  if (cache[dev] == 0) {
    int occ = 0;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem);
    cache[dev] = (occ > 0 ? occ : 1) * dev_sms(dev) + 1;
  }
  return cache[dev] - 1;
}

struct WsView {
  TileWs* hdr;
  uint32_t* tile_rel;
  uint8_t* scratch;
};
inline uint64_t align16(uint64_t v) { return (v + 15) & ~15ull; }
// header + per-tile sizes + scratch (per tile one slot; the warps' runs are
// 128-byte aligned, hence up to 128 B of padding per warp)
inline uint64_t ws_bytes_for_tiles(uint64_t tiles) {
  return align16(sizeof(TileWs)) + align16(4 * tiles) + 128 + tiles * (uint64_t)TILE_SLOT;
}
WsView carve(void* ws, uint64_t tiles) {
  uint8_t* p = reinterpret_cast<uint8_t*>(ws);
  WsView v;
  v.hdr = reinterpret_cast<TileWs*>(p);
  v.tile_rel = reinterpret_cast<uint32_t*>(p + align16(sizeof(TileWs)));
  v.scratch = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(p + align16(sizeof(TileWs)) + align16(4 * tiles)) + 127) & ~(uintptr_t)127);
  return v;
}

// Grid = one CTA per SM (capped by the work); CTAs are split over segments in
// proportion to their tiles (at least one CTA per segment).
template <int SRC, int NSEG, bool FAST, int NWT = 0>
int launch_encode_t(EncodeArgs<NSEG>& a, uint64_t total_tiles, cudaStream_t s) {
  constexpr int NW = NWT ? NWT : enc_warps(SRC);
  const size_t smem = (size_t)NW * enc_warp_smem(SRC);
  static int caps[MAXDEV];
  const int cap = grid_cap(k_tile_encode<SRC, NSEG, FAST, NWT>, 32 * NW, smem, caps);
  // one CTA per tile up to one per SM: a small message is spread over as many
  // SMs as it has tiles (a tile's encode is a latency chain of ~1100
  // instructions; 24 tiles on one SM would serialise on its issue slots)
  uint64_t G = std::min<uint64_t>((uint64_t)cap, std::max<uint64_t>(1, total_tiles));
  G = std::max<uint64_t>(G, (uint64_t)a.nseg);
  if (G > (uint64_t)MAXGRID) return GZ_EINVAL;
  uint64_t base = 0, left = G - (uint64_t)a.nseg;
  for (int k = 0; k < a.nseg; ++k) {
    const uint64_t tk = ntiles_of(a.seg[k].n);
    const uint64_t extra = total_tiles ? (left * tk) / total_tiles : 0;
    a.seg[k].cta_base = base;
    base += 1 + extra;
  }
  a.nctas = base;
  a.total_tiles = total_tiles;
  // tiles per gather group (one warp each): 8, doubled until the groups fit
  // MAXGRID; halved (down to 1) while there are fewer groups than ~8 warps
  // per SM -- a small message's gather is a per-warp latency chain
#ifndef GZ_GATHER_GS
#define GZ_GATHER_GS 3
#endif
  uint32_t gs = GZ_GATHER_GS;
  auto ngroups = [&](uint32_t sh) {
    uint64_t g = 0;
    for (int k = 0; k < a.nseg; ++k) g += std::max<uint64_t>(1, (ntiles_of(a.seg[k].n) + (1u << sh) - 1) >> sh);
    return g;
  };
  while (gs > 0 && ngroups(gs) < 1184) --gs;
  while (ngroups(gs) > (uint64_t)MAXGRID && gs < 10) ++gs;
  if (ngroups(gs) > (uint64_t)MAXGRID) return GZ_EINVAL;
  uint64_t gbase = 0;
  for (int k = 0; k < a.nseg; ++k) {
    a.seg[k].gcta_base = gbase;
    a.seg[k].gcta_n = std::max<uint64_t>(1, (ntiles_of(a.seg[k].n) + (1u << gs) - 1) >> gs);
    gbase += a.seg[k].gcta_n;
  }
  a.gshift = gs;
  a.ngctas = gbase;
  count_launch();
  k_tile_encode<SRC, NSEG, FAST, NWT><<<(unsigned)base, 32 * NW, smem, s>>>(a);
  int rc = (int)cudaGetLastError();
  if (rc) return rc;
  if (a.slotted_out) return 0;  // slotted output: the consumer reads the slots
  count_launch();
  // gather: a plain stream-ordered launch (a programmatic dependent launch measured
  // 5-6 us slower per call at cfg1: 50.2 -> 44.0 us, tools/exp/ab_codec2.py)
  static int gcaps[MAXDEV];
  const int gcap = grid_cap(k_gather<NSEG>, GATHER_THREADS, 0, gcaps);
  const unsigned ggrid = (unsigned)std::min<uint64_t>((gbase + GATHER_THREADS / 32 - 1) / (GATHER_THREADS / 32), (uint64_t)gcap);
  k_gather<NSEG><<<ggrid, GATHER_THREADS, 0, s>>>(a);
  return (int)cudaGetLastError();
}

// a small message (up to ~4 tiles per SM) runs one tile per CTA in 4-warp CTAs (32 KB of
// shared memory instead of 192 KB), which launch and retire faster (1 MiB/rank allreduce
// at N = 2: compress 11.6 -> 8.9 us, fused step 21.7 -> 20.1 us; 2-4 MiB/rank 76-79 ->
// 72-74 us per call with the threshold at 600 tiles instead of 148)
#ifndef GZ_SMALL_MSG_TILES
#define GZ_SMALL_MSG_TILES 600
#endif
constexpr uint64_t SMALL_MSG_TILES = GZ_SMALL_MSG_TILES;
template <int SRC, int NSEG>
int launch_encode(EncodeArgs<NSEG>& a, uint64_t total_tiles, cudaStream_t s) {
  if constexpr (NSEG == 1) {
    if (total_tiles <= SMALL_MSG_TILES)
      return a.qp.fast ? launch_encode_t<SRC, NSEG, true, 4>(a, total_tiles, s)
                       : launch_encode_t<SRC, NSEG, false, 4>(a, total_tiles, s);
  }
  return a.qp.fast ? launch_encode_t<SRC, NSEG, true>(a, total_tiles, s)
                   : launch_encode_t<SRC, NSEG, false>(a, total_tiles, s);
}

__global__ void k_record_error(Status* st, unsigned long long v) { atomicMin(&st->decode_error, v); }
__global__ void k_stamp(unsigned long long* dst) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *dst = t;
}

__global__ void k_copy_blob(const uint4* __restrict__ src, uint4* __restrict__ dst, const uint64_t* d_len, uint64_t max_bytes) {
  const uint64_t len = umin64(*d_len, max_bytes);
  const uint64_t nch = (len + 15) >> 4;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nch; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = __ldcs(src + i);
}

// dst = src (f32) with the first non-finite src offset (+ report_base)
// recorded like codec.py:79-86: the verbatim-kept parts of a collective's
// input (the scatter root's own block, a single rank's buffer) are checked
// the same way the encoder checks everything it compresses.
__global__ void k_copy_checked(const float4* __restrict__ src, float4* __restrict__ dst, uint64_t n, Status* st,
                               uint64_t report_base) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) != 0) {  // unaligned slice
    const float* s1 = reinterpret_cast<const float*>(src);
    float* d1 = reinterpret_cast<float*>(dst);
    for (uint64_t i = t0; i < n; i += stride) {
      const float v = s1[i];
      if (d1) d1[i] = v;
      if (!isfinite(v)) atomicMin(&st->first_nonfinite, (unsigned long long)(report_base + i));
    }
    return;
  }
  const uint64_t n4 = n >> 2;
  for (uint64_t i = t0; i < n4; i += stride) {
    const float4 v = __ldcs(src + i);
    if (dst) __stcs(dst + i, v);
    if (!(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w))) {
      const float f[4] = {v.x, v.y, v.z, v.w};
      for (int k = 0; k < 4; ++k)
        if (!isfinite(f[k])) {
          atomicMin(&st->first_nonfinite, (unsigned long long)(report_base + 4 * i + k));
          break;
        }
    }
  }
  if (t0 < (n & 3)) {
    const uint64_t i = 4 * n4 + t0;
    const float v = reinterpret_cast<const float*>(src)[i];
    if (dst) reinterpret_cast<float*>(dst)[i] = v;
    if (!isfinite(v)) atomicMin(&st->first_nonfinite, (unsigned long long)(report_base + i));
  }
}

struct CopyItems {
  gz_copy_item it[GZ_MAX_COPY_ITEMS];
};

// blockIdx.y = item; 16-byte body (eight loads in flight per thread: the
// source is usually a peer GPU, so the copy is latency-bound otherwise),
// byte tail.
__global__ void k_copy_items(const CopyItems ci) {
  const gz_copy_item& it = ci.it[blockIdx.y];
  const uint64_t len = it.d_len ? umin64(*it.d_len, it.max_bytes) : it.max_bytes;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (((reinterpret_cast<uintptr_t>(it.src) | reinterpret_cast<uintptr_t>(it.dst)) & 15) != 0) {
    // unaligned (small) item: byte copy
    for (uint64_t i = t0; i < len; i += stride) it.dst[i] = it.src[i];
    return;
  }
  const uint64_t nch = len >> 4;
  const uint4* s = reinterpret_cast<const uint4*>(it.src);
  uint4* d = reinterpret_cast<uint4*>(it.dst);
  constexpr int B = 8;
  for (uint64_t i0 = t0; i0 < nch; i0 += B * stride) {
    uint4 v[B];
#pragma unroll
    for (int b = 0; b < B; ++b)
      if (i0 + b * stride < nch) v[b] = __ldcs(s + i0 + b * stride);
#pragma unroll
    for (int b = 0; b < B; ++b)
      if (i0 + b * stride < nch) d[i0 + b * stride] = v[b];
  }
  if (blockIdx.x == 0 && threadIdx.x < (len & 15)) it.dst[(nch << 4) + threadIdx.x] = it.src[(nch << 4) + threadIdx.x];
}

struct IpcHandle {
  cudaIpcMemHandle_t h;
  uint64_t offset;
};

// Driver entry points fetched through the runtime, so the library does not
// link libcuda directly (it loads on GPU-less build hosts for symbol checks).
typedef CUresult (*PFN_addrRange)(CUdeviceptr*, size_t*, CUdeviceptr);
typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_batchMemOp)(CUstream, unsigned int, CUstreamBatchMemOpParams*, unsigned int);

template <typename F>
F driver_fn(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(fn);
}
PFN_addrRange p_addr_range() {
  static PFN_addrRange f = driver_fn<PFN_addrRange>("cuMemGetAddressRange");
  return f;
}
PFN_writeValue32 p_write32() {
  static PFN_writeValue32 f = driver_fn<PFN_writeValue32>("cuStreamWriteValue32");
  return f;
}
PFN_waitValue32 p_wait32() {
  static PFN_waitValue32 f = driver_fn<PFN_waitValue32>("cuStreamWaitValue32");
  return f;
}
PFN_batchMemOp p_batch() {
  static PFN_batchMemOp f = driver_fn<PFN_batchMemOp>("cuStreamBatchMemOp");
  return f;
}

}  // namespace


namespace {
// Tensor map of the decoder's output for TMA tensor stores (k_tile_decode): y viewed as
// [n/32 rows][32 floats], box 32 x 32, 128-byte swizzle.  Returns 0 (plain stores)
// when y is not 16-byte aligned, has no full tile, or the driver refuses the map.
using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int encode_ymap(CUtensorMap* map, float* y, uint64_t n) {
  static PFN_encodeTiled f = driver_fn<PFN_encodeTiled>("cuTensorMapEncodeTiled");
  const uint64_t rows = n / BLOCK;
  if (!f || !y || (reinterpret_cast<uintptr_t>(y) & 15) || rows < (uint64_t)TB || rows > 0x7FFFFFFFull) return 0;
  const cuuint64_t dims[2] = {BLOCK, rows};
  const cuuint64_t strides[1] = {BLOCK * sizeof(float)};
  const cuuint32_t box[2] = {BLOCK, TB};
  const cuuint32_t estr[2] = {1, 1};
  return f(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, y, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NSEG>
int launch_decode(DecodeMultiArgs<NSEG>& a, cudaStream_t s, int reserve_sms = 0) {
  const size_t smem = (size_t)dec_cta_smem(NSEG);  // per warp: value tile + stagings (+ alignment slack)
  static int caps[MAXDEV];
  const int cap = grid_cap(k_tile_decode<NSEG>, CTA_THREADS, smem, caps);
  const int per_sm = std::max(1, cap / dev_sms(cur_dev()));
  // leave `reserve_sms` SMs free (a concurrent NVLink copy)
  const int lim = std::max(per_sm, cap - reserve_sms * per_sm);
  const uint64_t want = (a.total_tiles + WARPS - 1) / WARPS;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)lim));
  count_launch();
  k_tile_decode<NSEG><<<grid, CTA_THREADS, smem, s>>>(a);
  return (int)cudaGetLastError();
}

int decode_one(const uint8_t* blob, const void* sidecar, const float* local, int op, uint64_t n, double eb, float* y,
               gz_status* d_status, gz_stream_t stream) {
  DecodeMultiArgs<1> a;
  std::memset(&a, 0, sizeof(a));
  SidecarView sv = sidecar_view(sidecar, n);
  a.seg[0] = DecSeg{blob, sv.tile_off, sv.widths, n, y, 0, nullptr};
  a.nseg = 1;
  a.total_tiles = ntiles_of(n);
  a.tw = 2.0 * eb;
  a.local = local;
  a.op = op;
  a.st = reinterpret_cast<Status*>(d_status);
  if (!local) a.ytma = encode_ymap(&a.ymap, y, n);
  return launch_decode<1>(a, (cudaStream_t)stream);
}

}  // namespace

extern "C" {

// profiling only: write the GPU's %globaltimer (ns) into *dst, stream-ordered
#if GZ_DIAG_STAMPS
int gz_diag_stamps(void* gst, void* est) {
  cudaMemcpyFromSymbol(gst, g_gst, sizeof(g_gst));
  return (int)cudaMemcpyFromSymbol(est, g_est, sizeof(g_est));
}
#endif
int gz_debug_stamp(void* dst, gz_stream_t stream) {
  k_stamp<<<1, 1, 0, (cudaStream_t)stream>>>(reinterpret_cast<unsigned long long*>(dst));
  return (int)cudaGetLastError();
}

uint64_t gz_compress_bound(uint64_t n) { return HEADER_BYTES + nblocks(n) * MAX_BLOCK_BYTES + 64; }
uint64_t gz_num_tiles(uint64_t n) { return ntiles_of(n); }
uint32_t gz_tile_blocks(void) { return TB; }
uint64_t gz_sidecar_bytes(uint64_t n) {
  const uint64_t nt = ntiles_of(n);
  return ((8 * (nt + 1) + (uint64_t)TB * nt) + 15) & ~15ull;
}
uint64_t gz_workspace_bytes(uint64_t n) { return ws_bytes_for_tiles(ntiles_of(n)); }

int gz_workspace_init(void* ws, uint64_t ws_bytes, gz_stream_t stream) {
  if (!ws || ws_bytes < 40) return GZ_EINVAL;
  return (int)cudaMemsetAsync(ws, 0, ws_bytes, (cudaStream_t)stream);
}

int gz_status_reset(gz_status* d_status, gz_stream_t stream) {
  if (!d_status) return GZ_EINVAL;
  return (int)cudaMemsetAsync(d_status, 0xFF, sizeof(gz_status), (cudaStream_t)stream);
}

int gz_compress(const float* x, uint64_t n, double eb, uint32_t block, uint8_t* blob, uint64_t blob_cap,
                uint64_t* d_len, void* sidecar, uint64_t* d_block_offsets, void* ws, uint64_t ws_bytes,
                gz_status* d_status, gz_stream_t stream) {
  if (block != BLOCK) return GZ_EBLOCK;
  if (!check_eb(eb)) return GZ_EBOUND;
  if ((!x && n) || !blob || !d_len || !ws || !d_status || !aligned16(blob)) return GZ_EINVAL;
  if (blob_cap < gz_compress_bound(n)) return GZ_ECAPACITY;
  if (ws_bytes < gz_workspace_bytes(n)) return GZ_EINVAL;
  EncodeArgs<1> a;
  std::memset(&a, 0, sizeof(a));
  SidecarView sv = sidecar_view(sidecar, n);
  a.seg[0] = Seg{x, n, blob, d_len, sv.tile_off, sv.widths, 0, 0, 0, 0, 0};
  a.nseg = 1;
  a.qp = make_qparams(eb);
  a.blk_off = d_block_offsets;
  const WsView wv = carve(ws, ntiles_of(n));
  a.ws = wv.hdr;
  a.tile_rel = wv.tile_rel;
  a.scratch = wv.scratch;
  a.st = reinterpret_cast<Status*>(d_status);
  return launch_encode<SRC_PLAIN, 1>(a, ntiles_of(n), (cudaStream_t)stream);
}

int gz_decompress_reduce(const uint8_t* blob, const void* sidecar, const float* local, uint64_t n, double eb, int op,
                         float* y, gz_status* d_status, gz_stream_t stream) {
  if (!check_eb(eb)) return GZ_EBOUND;
  if (op != OP_SUM && op != OP_MAX) return GZ_EINVAL;
  if (!blob || !sidecar || (!y && n) || (!local && n) || !d_status) return GZ_EINVAL;
  if (n == 0) return 0;
  return decode_one(blob, sidecar, local, op, n, eb, y, d_status, stream);
}

int gz_decompress_sidecar(const uint8_t* blob, const void* sidecar, uint64_t n, double eb, float* y,
                          gz_status* d_status, gz_stream_t stream) {
  if (!check_eb(eb)) return GZ_EBOUND;
  if (!blob || !sidecar || (!y && n) || !d_status) return GZ_EINVAL;
  if (n == 0) return 0;
  return decode_one(blob, sidecar, nullptr, 0, n, eb, y, d_status, stream);
}

int gz_decompress_multi(const uint8_t* const* blobs, const void* const* sidecars, const uint64_t* ns, uint32_t count,
                        double eb, float* const* ys, int reserve_sms, gz_status* d_status, gz_stream_t stream) {
  if (!check_eb(eb)) return GZ_EBOUND;
  if (!blobs || !sidecars || !ns || !ys || !d_status || count > GZ_MAX_DECODE_SEGMENTS) return GZ_EINVAL;
  DecodeMultiArgs<GZ_MAX_DECODE_SEGMENTS> a;
  std::memset(&a, 0, sizeof(a));
  uint64_t tiles = 0;
  int k = 0;
  for (uint32_t i = 0; i < count; ++i) {
    if (ns[i] == 0) continue;
    if (!blobs[i] || !sidecars[i] || !ys[i]) return GZ_EINVAL;
    SidecarView sv = sidecar_view(sidecars[i], ns[i]);
    a.seg[k++] = DecSeg{blobs[i], sv.tile_off, sv.widths, ns[i], ys[i], tiles, nullptr};
    tiles += ntiles_of(ns[i]);
  }
  if (k == 0) return 0;
  a.nseg = k;
  a.total_tiles = tiles;
  a.tw = 2.0 * eb;
  a.st = reinterpret_cast<Status*>(d_status);
  if (k == 1) {  // a single blob: the local two-stage decoder
    DecodeMultiArgs<1> b;
    std::memset(&b, 0, sizeof(b));
    b.seg[0] = a.seg[0];
    b.nseg = 1;
    b.total_tiles = tiles;
    b.tw = a.tw;
    b.st = a.st;
    return launch_decode<1>(b, (cudaStream_t)stream, reserve_sms);
  }
  return launch_decode<GZ_MAX_DECODE_SEGMENTS>(a, (cudaStream_t)stream, reserve_sms);
}

int gz_decompress_slots_multi(const uint8_t* const* slots, const uint32_t* const* sizes, const uint8_t* const* widths,
                              const uint64_t* ns, uint32_t count, double eb, float* const* ys, int reserve_sms,
                              gz_status* d_status, gz_stream_t stream) {
  if (!check_eb(eb)) return GZ_EBOUND;
  if (!slots || !sizes || !widths || !ns || !ys || !d_status || count > GZ_MAX_DECODE_SEGMENTS) return GZ_EINVAL;
  DecodeMultiArgs<GZ_MAX_DECODE_SEGMENTS> a;
  std::memset(&a, 0, sizeof(a));
  uint64_t tiles = 0;
  int k = 0;
  for (uint32_t i = 0; i < count; ++i) {
    if (ns[i] == 0) continue;
    if (!slots[i] || !sizes[i] || !widths[i] || !ys[i] || (reinterpret_cast<uintptr_t>(slots[i]) & 127)) return GZ_EINVAL;
    a.seg[k++] = DecSeg{slots[i], nullptr, widths[i], ns[i], ys[i], tiles, sizes[i]};
    tiles += ntiles_of(ns[i]);
  }
  if (k == 0) return 0;
  a.nseg = k;
  a.total_tiles = tiles;
  a.tw = 2.0 * eb;
  a.st = reinterpret_cast<Status*>(d_status);
  if (k == 1) {  // a single owner: the two-stage decoder (2^26 peer slots: 109 -> 97 us)
    DecodeMultiArgs<1> b;
    std::memset(&b, 0, sizeof(b));
    b.seg[0] = a.seg[0];
    b.nseg = 1;
    b.total_tiles = tiles;
    b.tw = a.tw;
    b.st = a.st;
    return launch_decode<1>(b, (cudaStream_t)stream, reserve_sms);
  }
  // several owners (usually in peer GPUs' memory) in one launch
  return launch_decode<GZ_MAX_DECODE_SEGMENTS>(a, (cudaStream_t)stream, reserve_sms);
}

uint64_t gz_index_workspace_bytes(uint64_t payload_len) {
  const uint64_t nseg = (payload_len + SEG - 1) / SEG;
  const uint64_t nch = (nseg + CH - 1) / CH;
  // exit + count tables, composed tables, chunk entries, g32 (sized by the
  // largest possible block count: 5 bytes per block)
  const uint64_t nb_max = payload_len / 5 + 2;
  return 64 + nseg * NE * 4 + nch * NE * 8 + nch * 16 + ((nb_max + GROUP - 1) / GROUP) * 8 + 256;
}

int gz_index(const uint8_t* blob, uint64_t payload_len, uint64_t n, void* sidecar, void* ws, uint64_t ws_bytes,
             gz_status* d_status, gz_stream_t stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!blob || !sidecar || !ws || !d_status) return GZ_EINVAL;
  if (n == 0) return 0;
  Status* st = reinterpret_cast<Status*>(d_status);
  if (payload_len == 0) {  // codec.py:307-308 at block 0
    count_launch();
    k_record_error<<<1, 1, 0, s>>>(st, (unsigned long long)DE_TRUNC);
    return (int)cudaGetLastError();
  }
  if (ws_bytes < gz_index_workspace_bytes(payload_len)) return GZ_EINVAL;
  const uint64_t nseg = (payload_len + SEG - 1) / SEG;
  const uint64_t nch = (nseg + CH - 1) / CH;
  uint8_t* p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ws) + 15) & ~(uintptr_t)15);
  auto take = [&](uint64_t bytes) {
    uint8_t* r = p;
    p += (bytes + 15) & ~15ull;
    return r;
  };
  IndexWs iw;
  iw.exit = reinterpret_cast<short*>(take(nseg * NE * 2));
  iw.count = reinterpret_cast<unsigned short*>(take(nseg * NE * 2));
  iw.cexit = reinterpret_cast<short*>(take(nch * NE * 2));
  iw.ccount = reinterpret_cast<unsigned*>(take(nch * NE * 4));
  iw.centry = reinterpret_cast<long long*>(take(nch * 8));
  iw.cbase = reinterpret_cast<unsigned long long*>(take(nch * 8));
  // a block has at least 5 bytes: more blocks than that cannot be walked
  const uint64_t nb_eff = std::min<uint64_t>(nblocks(n), payload_len / 5 + 2);
  iw.gt = reinterpret_cast<unsigned long long*>(take(((nb_eff + TB - 1) / TB) * 8));
  iw.widths = sidecar_view(sidecar, n).widths;
  const uint8_t* payload = blob + HEADER_BYTES;
  count_launch(4);  // idx_segments, idx_chunks, idx_resolve, idx_emit
  idx_segments<<<(unsigned)nseg, 160, 0, s>>>(payload, payload_len, iw);
  const size_t csm = (size_t)CH * NE * 4;
  static bool attr[MAXDEV];
  const int dev = cur_dev();
  if (!attr[dev]) {  // the opt-in is per device context
    cudaFuncSetAttribute(idx_chunks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
    cudaFuncSetAttribute(idx_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)EMIT_SMEM);
    cudaFuncSetAttribute(idx_resolve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RESOLVE_SMEM_MAX);
    attr[dev] = true;
  }
  idx_chunks<<<(unsigned)nch, 160, csm, s>>>(nseg, iw);
  {
    const size_t rsm = resolve_smem(nch);
    const int staged = rsm <= RESOLVE_SMEM_MAX;
    idx_resolve<<<1, staged ? 512 : 32, staged ? rsm : 0, s>>>(nch, iw, staged);
  }
  idx_emit<<<(unsigned)((nseg + EG - 1) / EG), CH, EMIT_SMEM, s>>>(payload, payload_len, nseg, n, iw, st);
  if (nblocks(n) > payload_len / 5 + 1) {
    // certainly truncated (a block has at least 5 bytes): idx_emit reports the
    // first failing block of the walk; this bound makes the failure explicit
    // even if the walk stopped early, and no sidecar is built
    count_launch();
    k_record_error<<<1, 1, 0, s>>>(st, (unsigned long long)(((payload_len / 5) << 24) | DE_TRUNC));
    return (int)cudaGetLastError();
  }
  const uint64_t nt = ntiles_of(n);
  const uint64_t work = nt + 1;
  SidecarView sv = sidecar_view(sidecar, n);
  count_launch();
  idx_sidecar<<<(unsigned)((work + 255) / 256), 256, 0, s>>>(iw, n, payload_len, sv.tile_off);
  return (int)cudaGetLastError();
}

int gz_reduce_step(const uint8_t* blob_in, const void* sidecar_in, const float* local, uint64_t m, double eb,
                   int op, float* acc_out, uint8_t* blob_out, uint64_t blob_out_cap, uint64_t* d_len_out,
                   void* sidecar_out, void* ws, uint64_t ws_bytes, gz_status* d_status, gz_stream_t stream) {
  if (!check_eb(eb)) return GZ_EBOUND;
  if (op != OP_SUM && op != OP_MAX) return GZ_EINVAL;
  if (!blob_in || !sidecar_in || (!local && m) || !blob_out || !d_len_out || !ws || !d_status || !aligned16(blob_out))
    return GZ_EINVAL;
  if (blob_out_cap < gz_compress_bound(m)) return GZ_ECAPACITY;
  if (ws_bytes < gz_workspace_bytes(m)) return GZ_EINVAL;
  EncodeArgs<1> a;
  std::memset(&a, 0, sizeof(a));
  SidecarView so = sidecar_view(sidecar_out, m);
  a.seg[0] = Seg{local, m, blob_out, d_len_out, so.tile_off, so.widths, 0, 0, 0, 0, 0};
  a.nseg = 1;
  a.qp = make_qparams(eb);
  const WsView wv = carve(ws, ntiles_of(m));
  a.ws = wv.hdr;
  a.tile_rel = wv.tile_rel;
  a.scratch = wv.scratch;
  a.st = reinterpret_cast<Status*>(d_status);
  SidecarView si = sidecar_view(sidecar_in, m);
  a.in_blob = blob_in;
  a.in_tile_off = si.tile_off;
  a.in_w = si.widths;
  a.in_tw = 2.0 * eb;
  a.op = op;
  a.acc_out = acc_out;
  return launch_encode<SRC_STEP, 1>(a, ntiles_of(m), (cudaStream_t)stream);
}

uint64_t gz_segments_workspace_bytes(const uint64_t* h_counts, uint32_t nseg) {
  uint64_t tiles = 0;
  for (uint32_t i = 0; i < nseg; ++i) tiles += ntiles_of(h_counts[i]);
  return ws_bytes_for_tiles(tiles);
}

int gz_step(const gz_step_io* io, const float* local, uint64_t m, double eb, int op, float* acc_out, void* ws,
            uint64_t ws_bytes, gz_status* d_status, gz_stream_t stream) {
  if (!check_eb(eb)) return GZ_EBOUND;
  if (op != OP_SUM && op != OP_MAX) return GZ_EINVAL;
  if (!io || (!local && m) || !ws || !d_status) return GZ_EINVAL;
  const bool fused = io->in_blob || io->in_slots;
  const bool slotted = io->out_slots != nullptr;
  if (fused && !io->in_slots && !io->in_sidecar) return GZ_EINVAL;
  if (io->in_slots && (!io->in_sizes || !io->in_widths)) return GZ_EINVAL;
  if (slotted && (!io->out_sizes || !io->out_widths || (reinterpret_cast<uintptr_t>(io->out_slots) & 127))) return GZ_EINVAL;
  if (!slotted && (!io->blob_out || !io->d_len_out || !aligned16(io->blob_out))) return GZ_EINVAL;
  if (!slotted && io->blob_out_cap < gz_compress_bound(m)) return GZ_ECAPACITY;
  if (ws_bytes < gz_workspace_bytes(m)) return GZ_EINVAL;
  EncodeArgs<1> a;
  std::memset(&a, 0, sizeof(a));
  const WsView wv = carve(ws, ntiles_of(m));
  a.ws = wv.hdr;
  a.tile_rel = wv.tile_rel;
  a.scratch = wv.scratch;
  if (slotted) {
    a.seg[0] = Seg{local, m, nullptr, nullptr, nullptr, io->out_widths, 0, 0, 0, 0, io->report_base};
    a.tile_rel = io->out_sizes;
    a.scratch = io->out_slots;
    a.slotted_out = 1;  // the encoder's last CTA re-zeroes the claim counter (no gather)
    a.post_flag = reinterpret_cast<unsigned int*>(io->post_flag);
    a.wait_flag = reinterpret_cast<unsigned int*>(io->wait_flag);
  } else {
    if (io->post_flag || io->wait_flag) return GZ_EINVAL;
    SidecarView so = sidecar_view(io->sidecar_out, m);
    a.seg[0] = Seg{local, m, io->blob_out, io->d_len_out, so.tile_off, so.widths, 0, 0, 0, 0, io->report_base};
  }
  a.nseg = 1;
  a.qp = make_qparams(eb);
  a.st = reinterpret_cast<Status*>(d_status);
  a.op = op;
  a.acc_out = acc_out;
  auto done = [](int rc) { return rc; };
  if (!fused) return done(launch_encode<SRC_PLAIN, 1>(a, ntiles_of(m), (cudaStream_t)stream));
  a.in_tw = 2.0 * eb;
  if (io->in_slots) {
    a.in_slots = io->in_slots;
    a.in_sizes = io->in_sizes;
    a.in_w = io->in_widths;
  } else {
    SidecarView si = sidecar_view(io->in_sidecar, m);
    a.in_blob = io->in_blob;
    a.in_tile_off = si.tile_off;
    a.in_w = si.widths;
  }
  return done(launch_encode<SRC_STEP, 1>(a, ntiles_of(m), (cudaStream_t)stream));
}

uint64_t gz_slots_bytes(uint64_t m) { return ntiles_of(m) * (uint64_t)TILE_SLOT; }

int gz_step_reduce(const gz_step_io* io, const float* local, uint64_t m, double eb, int op, float* y,
                   gz_status* d_status, gz_stream_t stream) {
  if (!check_eb(eb)) return GZ_EBOUND;
  if (op != OP_SUM && op != OP_MAX) return GZ_EINVAL;
  if (!io || !io->in_slots || !io->in_sizes || !io->in_widths || (!y && m) || !d_status) return GZ_EINVAL;
  if (m == 0) return 0;
  DecodeMultiArgs<1> a;
  std::memset(&a, 0, sizeof(a));
  a.seg[0] = DecSeg{io->in_slots, nullptr, io->in_widths, m, y, 0, io->in_sizes};
  a.nseg = 1;
  a.total_tiles = ntiles_of(m);
  a.tw = 2.0 * eb;
  a.local = local;
  a.op = op;
  a.st = reinterpret_cast<Status*>(d_status);
  a.report_base = io->report_base;
  return launch_decode<1>(a, (cudaStream_t)stream);
}

int gz_compress_segments(const float* x, const uint64_t* h_counts, uint32_t nseg, double eb, uint8_t* payload,
                         const uint64_t* h_seg_blob_off, uint64_t* d_seg_len, void* sidecars,
                         const uint64_t* h_seg_sidecar_off, const uint64_t* h_seg_report_off, void* ws,
                         uint64_t ws_bytes, gz_status* d_status, gz_stream_t stream) {
  if (!check_eb(eb)) return GZ_EBOUND;
  if (!h_counts || !payload || !h_seg_blob_off || !d_seg_len || !ws || !d_status) return GZ_EINVAL;
  uint64_t total = 0, tiles_all = 0;
  for (uint32_t i = 0; i < nseg; ++i) {
    total += h_counts[i];
    tiles_all += ntiles_of(h_counts[i]);
    if (!aligned16(payload + h_seg_blob_off[i])) return GZ_EINVAL;
  }
  if (total && !x) return GZ_EINVAL;
  if (ws_bytes < ws_bytes_for_tiles(tiles_all)) return GZ_EINVAL;
  const QParams qp = make_qparams(eb);
  const WsView wv = carve(ws, tiles_all);
  uint64_t xoff = 0, tile_base = 0;
  for (uint32_t s0 = 0; s0 < nseg; s0 += MAXSEG) {
    EncodeArgs<MAXSEG> a;
    std::memset(&a, 0, sizeof(a));
    const uint32_t cnt = std::min<uint32_t>(MAXSEG, nseg - s0);
    uint64_t tiles = 0;
    for (uint32_t j = 0; j < cnt; ++j) {
      const uint32_t i = s0 + j;
      const uint64_t n = h_counts[i];
      SidecarView sv{nullptr, nullptr};
      if (sidecars) sv = sidecar_view(reinterpret_cast<uint8_t*>(sidecars) + h_seg_sidecar_off[i], n);
      a.seg[j] = Seg{x + xoff, n, payload + h_seg_blob_off[i], d_seg_len + i, sv.tile_off, sv.widths, 0, 0, 0, tiles,
                     h_seg_report_off ? h_seg_report_off[i] : xoff};
      tiles += ntiles_of(n);
      xoff += n;
    }
    a.nseg = (int)cnt;
    a.qp = qp;
    a.ws = wv.hdr;
    a.tile_rel = wv.tile_rel + tile_base;
    a.scratch = wv.scratch + tile_base * (uint64_t)TILE_SLOT;
    a.st = reinterpret_cast<Status*>(d_status);
    const int rc = launch_encode<SRC_PLAIN, MAXSEG>(a, tiles, (cudaStream_t)stream);
    if (rc) return rc;
    tile_base += tiles;
  }
  return 0;
}

// ---- peer memory ------------------------------------------------------------
int gz_ipc_handle_size(void) { return (int)sizeof(IpcHandle); }

int gz_ipc_get_handle(void* dptr, void* handle_out) {
  if (!dptr || !handle_out) return GZ_EINVAL;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (!p_addr_range()) return (int)cudaErrorNotSupported;
  CUresult r = p_addr_range()(&base, &size, (CUdeviceptr)dptr);
  if (r != CUDA_SUCCESS) return (int)r + 20000;
  IpcHandle h;
  std::memset(&h, 0, sizeof(h));
  cudaError_t e = cudaIpcGetMemHandle(&h.h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return (int)e;
  h.offset = (uint64_t)((CUdeviceptr)dptr - base);
  std::memcpy(handle_out, &h, sizeof(h));
  return 0;
}

int gz_ipc_open_handle(const void* handle, void** dptr_out) {
  if (!handle || !dptr_out) return GZ_EINVAL;
  IpcHandle h;
  std::memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, h.h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return (int)e;
  *dptr_out = reinterpret_cast<uint8_t*>(base) + h.offset;
  return 0;
}

int gz_ipc_close(void* dptr) {
  if (!dptr) return GZ_EINVAL;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (!p_addr_range()) return (int)cudaErrorNotSupported;
  CUresult r = p_addr_range()(&base, &size, (CUdeviceptr)dptr);
  if (r != CUDA_SUCCESS) return (int)r + 20000;
  return (int)cudaIpcCloseMemHandle(reinterpret_cast<void*>(base));
}

int gz_enable_peer_access(int peer_device) {
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return 0;
  }
  return (int)e;
}

int gz_stream_write_u32(gz_stream_t stream, void* dptr, uint32_t value) {
  if (!p_write32()) return (int)cudaErrorNotSupported;
  CUresult r = p_write32()((CUstream)stream, (CUdeviceptr)dptr, value, CU_STREAM_WRITE_VALUE_DEFAULT);
  return r == CUDA_SUCCESS ? 0 : (int)r + 20000;
}

int gz_stream_wait_u32_geq(gz_stream_t stream, void* dptr, uint32_t value) {
  if (!p_wait32()) return (int)cudaErrorNotSupported;
  CUresult r = p_wait32()((CUstream)stream, (CUdeviceptr)dptr, value, CU_STREAM_WAIT_VALUE_GEQ);
  return r == CUDA_SUCCESS ? 0 : (int)r + 20000;
}

int gz_stream_flag_ops(gz_stream_t stream, const gz_flag_op* ops, uint32_t count) {
  if (!ops || count == 0 || count > GZ_MAX_FLAG_OPS) return GZ_EINVAL;
  for (uint32_t i = 0; i < count; ++i)
    if (!ops[i].ptr || ops[i].kind > 1) return GZ_EINVAL;
  if (!p_batch()) return (int)cudaErrorNotSupported;
  CUstreamBatchMemOpParams p[GZ_MAX_FLAG_OPS];
  std::memset(p, 0, sizeof(p));
  for (uint32_t i = 0; i < count; ++i) {
    if (ops[i].kind == 0) {
      p[i].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
      p[i].writeValue.address = (CUdeviceptr)ops[i].ptr;
      p[i].writeValue.value = ops[i].value;
      p[i].writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
    } else {
      p[i].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_32;
      p[i].waitValue.address = (CUdeviceptr)ops[i].ptr;
      p[i].waitValue.value = ops[i].value;
      p[i].waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
    }
  }
  CUresult r = p_batch()((CUstream)stream, count, p, 0);
  return r == CUDA_SUCCESS ? 0 : (int)r + 20000;
}

int gz_copy_blob(const uint8_t* src, uint8_t* dst, const uint64_t* d_len, uint64_t max_bytes, gz_stream_t stream) {
  if (!src || !dst || !d_len || !aligned16(src) || !aligned16(dst)) return GZ_EINVAL;
  count_launch();
  k_copy_blob<<<296, 256, 0, (cudaStream_t)stream>>>(reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst),
                                                      d_len, max_bytes);
  return (int)cudaGetLastError();
}

int gz_copy_checked(const float* src, float* dst, uint64_t n, uint64_t report_base, gz_status* d_status,
                    gz_stream_t stream) {
  if (n == 0) return 0;
  if (!src || !d_status || (reinterpret_cast<uintptr_t>(src) & 3) || (reinterpret_cast<uintptr_t>(dst) & 3))
    return GZ_EINVAL;
  const uint64_t want = ((n >> 2) + 255) / 256;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, 4ull * dev_sms(cur_dev())));
  count_launch();
  k_copy_checked<<<grid, 256, 0, (cudaStream_t)stream>>>(reinterpret_cast<const float4*>(src),
                                                          reinterpret_cast<float4*>(dst), n,
                                                          reinterpret_cast<Status*>(d_status), report_base);
  return (int)cudaGetLastError();
}

// out = op(local, recv) elementwise, _apply_op (collectives.py:32-39): "sum"
// local + recv in binary32 RN, "max" np.maximum(local, recv) (NaN propagates,
// the second argument wins ties) -- the reduction of the verbatim-payload
// (lossless / fixed-rate) collectives, whose messages are not fused-decoded.
__global__ void k_apply_op(const float* a, const float* b, float* out,
                           uint64_t n, int op) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const float x = __ldcs(a + i), y = __ldcs(b + i);
    __stcs(out + i, op == OP_SUM ? __fadd_rn(x, y) : np_maximum(x, y));
  }
}

int gz_apply_op(const float* local, const float* recv, float* out, uint64_t n, int op, gz_stream_t stream) {
  if (n == 0) return 0;
  if (!local || !recv || !out || (op != OP_SUM && op != OP_MAX)) return GZ_EINVAL;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 4ull * dev_sms(cur_dev())));
  count_launch();
  k_apply_op<<<grid, 256, 0, (cudaStream_t)stream>>>(local, recv, out, n, op);
  return (int)cudaGetLastError();
}

__global__ void k_status_key(const unsigned long long* st, long long rank, long long* key) {
  const int i = threadIdx.x;
  if (i < 4) key[i] = st[i] == ~0ull ? 0x7FFFFFFFFFFFFFFFll : (long long)(st[i] | ((unsigned long long)rank << 56));
}

int gz_status_key(const gz_status* d_status, int rank, int64_t* d_key, gz_stream_t stream) {
  if (!d_status || !d_key || rank < 0 || rank >= 128) return GZ_EINVAL;
  count_launch();
  k_status_key<<<1, 32, 0, (cudaStream_t)stream>>>(reinterpret_cast<const unsigned long long*>(d_status), rank,
                                                   reinterpret_cast<long long*>(d_key));
  return (int)cudaGetLastError();
}

int gz_copy_items(const gz_copy_item* items, uint32_t count, gz_stream_t stream) {
  return gz_copy_items_sms(items, count, 0, stream);
}

int gz_copy_items_sms(const gz_copy_item* items, uint32_t count, int sms_budget, gz_stream_t stream) {
  if (count == 0) return 0;
  if (!items || count > GZ_MAX_COPY_ITEMS) return GZ_EINVAL;
  CopyItems ci;
  memset(&ci, 0, sizeof(ci));
  for (uint32_t i = 0; i < count; ++i) {
    if (!items[i].src || !items[i].dst) return GZ_EINVAL;
    ci.it[i] = items[i];
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int use = sms_budget > 0 ? std::min(sms_budget, sms) : sms;  // 4 CTAs per SM of the budget
  const unsigned gx = (unsigned)std::max(1, 4 * use / (int)count);
  count_launch();
  k_copy_items<<<dim3(gx, count), 256, 0, (cudaStream_t)stream>>>(ci);
  return (int)cudaGetLastError();
}

// ---- fixed-rate baseline codec (codec.py:442-489) -------------------------
uint64_t gz_fr_bound(uint64_t n, uint32_t bits) { return FR_HEADER_BYTES + (n * (uint64_t)bits + 7) / 8 + 16; }

uint64_t gz_fr_workspace_bytes(void) { return (sizeof(FrScratch) + 15) & ~15ull; }

int gz_fr_compress(const float* x, uint64_t n, uint32_t bits, uint8_t* out, uint64_t out_cap, uint64_t* d_len,
                   void* ws, gz_status* d_status, gz_stream_t stream) {
  if (bits < 1 || bits > 16) return GZ_EINVAL;
  if ((!x && n) || !out || !d_len || !ws || !d_status) return GZ_EINVAL;
  if (out_cap < FR_HEADER_BYTES + (n * (uint64_t)bits + 7) / 8) return GZ_ECAPACITY;
  cudaStream_t s = (cudaStream_t)stream;
  FrScratch* sc = reinterpret_cast<FrScratch*>(ws);
  const uint64_t groups = (n + 31) / 32;
  if (n) {
    count_launch(3);
    k_fr_init<<<1, 32, 0, s>>>(sc);
    k_fr_minmax<<<592, 256, 0, s>>>(x, n, sc, reinterpret_cast<Status*>(d_status));
    k_fr_zero_lanes<<<592, 256, 0, s>>>(x, n, sc);
  }
  count_launch();
  k_fr_encode<<<(unsigned)std::max<uint64_t>(1, (groups + 255) / 256), 256, 0, s>>>(x, n, (int)bits, sc, out, d_len);
  return (int)cudaGetLastError();
}

int gz_fr_decompress(const uint8_t* blob, uint64_t n, uint32_t bits, float* y, gz_stream_t stream) {
  if (bits < 1 || bits > 16) return GZ_EINVAL;
  if (!blob || (!y && n)) return GZ_EINVAL;
  if (n == 0) return 0;
  const uint64_t groups = (n + 31) / 32;
  count_launch();
  k_fr_decode<<<(unsigned)((groups + 255) / 256), 256, 0, (cudaStream_t)stream>>>(blob, n, (int)bits, y);
  return (int)cudaGetLastError();
}

uint64_t gz_launch_count(void) { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

}  // extern "C"
