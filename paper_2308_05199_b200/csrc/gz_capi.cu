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

using namespace gz;

namespace {

constexpr size_t SMEM_BYTES = (size_t)TB * 128 + STAGE_BYTES;
constexpr int MAXSEG = 32;  // segments per multi-segment launch (kernel-parameter budget)

inline uint64_t nblocks(uint64_t n) { return (n + BLOCK - 1) / BLOCK; }
inline uint64_t ntiles_of(uint64_t n) { return (nblocks(n) + TB - 1) / TB; }
inline uint64_t nctas_of(uint64_t n) { return std::max<uint64_t>(ntiles_of(n), 1); }

bool check_eb(double eb) { return std::isfinite(eb) && eb > 0.0; }

QParams make_qparams(double eb) {
  QParams p;
  p.eb = eb;
  p.tw = 2.0 * eb;  // codec.py:188
  p.fast = std::isfinite(p.tw) && p.tw >= std::ldexp(1.0, -100) && p.tw <= std::ldexp(1.0, 100);
  if (p.fast) {
    p.rtw = (float)(1.0 / p.tw);
    p.kx = std::nextafterf((float)(std::ldexp(1.0, -23) / p.tw), INFINITY);
    p.thr = 0.5f - 0x1p-20f - 0x1p-23f;
  } else {
    p.rtw = 0.f;
    p.kx = 0.f;
    p.thr = 0.f;
  }
  return p;
}

struct SidecarView {
  uint64_t* tile_off;
  uint16_t* sub_off;
};
SidecarView sidecar_view(const void* sc, uint64_t n) {
  SidecarView v{nullptr, nullptr};
  if (!sc) return v;
  const uint64_t nt = ntiles_of(n);
  v.tile_off = reinterpret_cast<uint64_t*>(const_cast<void*>(sc));
  v.sub_off = reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(const_cast<void*>(sc)) + 8 * (nt + 1));
  return v;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <int SRC, int NSEG>
int launch_encode(const EncodeArgs<NSEG>& a, cudaStream_t s) {
  k_tile_encode<SRC, NSEG><<<(unsigned)a.nctas, TB, SMEM_BYTES, s>>>(a);
  return (int)cudaGetLastError();
}

__global__ void k_record_error(Status* st, unsigned long long v) { atomicMin(&st->decode_error, v); }

__global__ void k_copy_blob(const uint4* __restrict__ src, uint4* __restrict__ dst, const uint64_t* d_len, uint64_t max_bytes) {
  const uint64_t len = umin64(*d_len, max_bytes);
  const uint64_t nch = (len + 15) >> 4;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nch; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = __ldcs(src + i);
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

}  // namespace

extern "C" {

uint64_t gz_compress_bound(uint64_t n) { return HEADER_BYTES + nblocks(n) * MAX_BLOCK_BYTES + 64; }
uint64_t gz_num_tiles(uint64_t n) { return ntiles_of(n); }
uint32_t gz_tile_blocks(void) { return TB; }
uint64_t gz_sidecar_bytes(uint64_t n) {
  const uint64_t nt = ntiles_of(n);
  return ((8 * (nt + 1) + 2 * nt * GROUPS) + 15) & ~15ull;
}
uint64_t gz_workspace_bytes(uint64_t n) { return 32 + 8 * (nctas_of(n) + 1); }

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
  a.seg[0] = Seg{x, n, blob, d_len, sv.tile_off, sv.sub_off, 0};
  a.nseg = 1;
  a.nctas = nctas_of(n);
  a.qp = make_qparams(eb);
  a.blk_off = d_block_offsets;
  a.ws = reinterpret_cast<TileWs*>(ws);
  a.st = reinterpret_cast<Status*>(d_status);
  return launch_encode<SRC_PLAIN, 1>(a, (cudaStream_t)stream);
}

int gz_decompress_sidecar(const uint8_t* blob, const void* sidecar, uint64_t n, double eb, float* y,
                          gz_status* d_status, gz_stream_t stream) {
  if (!check_eb(eb)) return GZ_EBOUND;
  if (!blob || !sidecar || (!y && n) || !d_status) return GZ_EINVAL;
  if (n == 0) return 0;
  DecodeArgs a;
  SidecarView sv = sidecar_view(sidecar, n);
  a.blob = blob;
  a.tile_off = sv.tile_off;
  a.sub_off = sv.sub_off;
  a.n = n;
  a.tw = 2.0 * eb;
  a.y = y;
  a.st = reinterpret_cast<Status*>(d_status);
  k_tile_decode<<<(unsigned)ntiles_of(n), TB, SMEM_BYTES, (cudaStream_t)stream>>>(a);
  return (int)cudaGetLastError();
}

uint64_t gz_index_workspace_bytes(uint64_t payload_len) {
  const uint64_t nseg = (payload_len + SEG - 1) / SEG;
  const uint64_t nch = (nseg + CH - 1) / CH;
  // exit + count tables, composed tables, chunk entries, g32 (sized by the
  // largest possible block count: 5 bytes per block)
  const uint64_t nb_max = payload_len / 5 + 2;
  return 64 + nseg * NE * 4 + nch * NE * 8 + nch * 16 + ((nb_max + 31) / 32) * 8 + 256;
}

int gz_index(const uint8_t* blob, uint64_t payload_len, uint64_t n, void* sidecar, void* ws, uint64_t ws_bytes,
             gz_status* d_status, gz_stream_t stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!blob || !sidecar || !ws || !d_status) return GZ_EINVAL;
  if (n == 0) return 0;
  Status* st = reinterpret_cast<Status*>(d_status);
  if (payload_len == 0) {  // codec.py:307-308 at block 0
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
  iw.g32 = reinterpret_cast<unsigned long long*>(take(((nb_eff + 31) / 32) * 8));
  const uint8_t* payload = blob + HEADER_BYTES;
  idx_segments<<<(unsigned)nseg, 160, 0, s>>>(payload, payload_len, iw);
  const size_t csm = (size_t)CH * NE * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(idx_chunks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
    attr = true;
  }
  idx_chunks<<<(unsigned)nch, 160, csm, s>>>(nseg, iw);
  idx_resolve<<<1, 32, 0, s>>>(nch, iw);
  idx_emit<<<(unsigned)nch, CH, 0, s>>>(payload, payload_len, nseg, n, iw, st);
  if (nblocks(n) > payload_len / 5 + 1) return (int)cudaGetLastError();  // certainly truncated: no sidecar
  const uint64_t nt = ntiles_of(n);
  const uint64_t work = std::max<uint64_t>(nt * GROUPS, nt + 1);
  SidecarView sv = sidecar_view(sidecar, n);
  idx_sidecar<<<(unsigned)((work + 255) / 256), 256, 0, s>>>(iw, n, payload_len, sv.tile_off, sv.sub_off);
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
  a.seg[0] = Seg{local, m, blob_out, d_len_out, so.tile_off, so.sub_off, 0};
  a.nseg = 1;
  a.nctas = nctas_of(m);
  a.qp = make_qparams(eb);
  a.ws = reinterpret_cast<TileWs*>(ws);
  a.st = reinterpret_cast<Status*>(d_status);
  SidecarView si = sidecar_view(sidecar_in, m);
  a.in_blob = blob_in;
  a.in_tile_off = si.tile_off;
  a.in_sub_off = si.sub_off;
  a.in_tw = 2.0 * eb;
  a.op = op;
  a.acc_out = acc_out;
  return launch_encode<SRC_STEP, 1>(a, (cudaStream_t)stream);
}

int gz_compress_segments(const float* x, const uint64_t* h_counts, uint32_t nseg, double eb, uint8_t* payload,
                         const uint64_t* h_seg_blob_off, uint64_t* d_seg_len, void* sidecars,
                         const uint64_t* h_seg_sidecar_off, void* ws, uint64_t ws_bytes, gz_status* d_status,
                         gz_stream_t stream) {
  if (!check_eb(eb)) return GZ_EBOUND;
  if (!h_counts || !payload || !h_seg_blob_off || !d_seg_len || !ws || !d_status) return GZ_EINVAL;
  uint64_t total = 0, nctas_all = 0;
  for (uint32_t i = 0; i < nseg; ++i) {
    total += h_counts[i];
    nctas_all += nctas_of(h_counts[i]);
    if (!aligned16(payload + h_seg_blob_off[i])) return GZ_EINVAL;
  }
  if (total && !x) return GZ_EINVAL;
  if (ws_bytes < 32 + 8 * (nctas_all + 1)) return GZ_EINVAL;
  const QParams qp = make_qparams(eb);
  uint64_t xoff = 0;
  for (uint32_t s0 = 0; s0 < nseg; s0 += MAXSEG) {
    EncodeArgs<MAXSEG> a;
    std::memset(&a, 0, sizeof(a));
    const uint32_t cnt = std::min<uint32_t>(MAXSEG, nseg - s0);
    uint64_t base = 0;
    for (uint32_t j = 0; j < cnt; ++j) {
      const uint32_t i = s0 + j;
      const uint64_t n = h_counts[i];
      SidecarView sv{nullptr, nullptr};
      if (sidecars) sv = sidecar_view(reinterpret_cast<uint8_t*>(sidecars) + h_seg_sidecar_off[i], n);
      a.seg[j] = Seg{x + xoff, n, payload + h_seg_blob_off[i], d_seg_len + i, sv.tile_off, sv.sub_off, base};
      base += nctas_of(n);
      xoff += n;
    }
    a.nseg = (int)cnt;
    a.nctas = base;
    a.qp = qp;
    a.ws = reinterpret_cast<TileWs*>(ws);
    a.st = reinterpret_cast<Status*>(d_status);
    const int rc = launch_encode<SRC_PLAIN, MAXSEG>(a, (cudaStream_t)stream);
    if (rc) return rc;
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

int gz_copy_blob(const uint8_t* src, uint8_t* dst, const uint64_t* d_len, uint64_t max_bytes, gz_stream_t stream) {
  if (!src || !dst || !d_len || !aligned16(src) || !aligned16(dst)) return GZ_EINVAL;
  k_copy_blob<<<296, 256, 0, (cudaStream_t)stream>>>(reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst),
                                                      d_len, max_bytes);
  return (int)cudaGetLastError();
}

}  // extern "C"
