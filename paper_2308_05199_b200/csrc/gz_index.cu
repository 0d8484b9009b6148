// gz_index.cu -- device replacement for the sequential block walk of
// codec.decompress (codec.py:298-322): validate a reference blob's payload and
// build the tile/group sidecar the tile decoder needs.
//
// A block's size is a function of its first byte, so block starts form a
// chain.  The payload is cut into SEG-byte segments; the first block start in
// any segment lies in its first 129 bytes (a block is at most 129 bytes).
//   K1 idx_segments : for every segment and each of the 129 possible entry
//                     offsets, walk the chain to the segment's end (one thread
//                     per entry) -> exit offset + number of block starts.
//   K2 idx_chunks   : compose CH consecutive segment maps (shared memory).
//   K3 idx_resolve  : follow the composed maps from entry 0 (one thread,
//                     one lookup per chunk) -> actual entry + block base.
//   K4 idx_emit     : per chunk, derive each segment's actual entry, re-walk
//                     the true chain with true block indices, apply the
//                     reference's checks in walk order (first failing block
//                     wins), and record the start of every 8th block.
//   K5 idx_sidecar  : convert those starts into the sidecar layout.
#include "gz_device.cuh"

namespace gz {

constexpr int SEG = 2048;
constexpr int NE = 129;       // possible entry offsets
constexpr int CH = 128;       // segments per chunk
constexpr short EX_DEAD = -1;  // invalid width byte on the chain
constexpr short EX_END = -2;   // chain reached the payload end inside the segment

struct IndexWs {
  short* exit;            // [nseg][NE]
  unsigned short* count;  // [nseg][NE]
  short* cexit;           // [nchunk][NE]
  unsigned* ccount;       // [nchunk][NE]
  long long* centry;      // [nchunk] actual entry (offset in first segment), <0 if unreachable
  unsigned long long* cbase;  // [nchunk] block index of the first start in the chunk
  unsigned long long* gt;     // [ceil(nb/32)] payload offset of block 32k (tile starts)
  uint8_t* widths;            // sidecar width byte of every block (may be null)
};

__device__ __forceinline__ int full_size(int w) { return w == RAW_WIDTH ? 1 + 4 * BLOCK : 5 + (31 * w + 7) / 8; }

__global__ void __launch_bounds__(160) idx_segments(const uint8_t* payload, uint64_t psize, IndexWs ws) {
  __shared__ __align__(16) uint8_t seg[SEG];
  __shared__ unsigned char ssize[256];
  const uint64_t s = blockIdx.x;
  const uint64_t g0 = s * SEG;
  const int len = (int)umin64(SEG, psize - g0);
  if ((reinterpret_cast<uintptr_t>(payload) & 7) == 0) {  // 8-B loads, all in flight at once
    const uint2* src = reinterpret_cast<const uint2*>(payload + g0);
#pragma unroll 2
    for (int i = threadIdx.x; i < (len >> 3); i += blockDim.x) reinterpret_cast<uint2*>(seg)[i] = __ldg(src + i);
    for (int i = (len & ~7) + threadIdx.x; i < len; i += blockDim.x) seg[i] = __ldg(payload + g0 + i);
  } else {
    for (int i = threadIdx.x; i < len; i += blockDim.x) seg[i] = __ldg(payload + g0 + i);
  }
  for (int w = threadIdx.x; w < 256; w += blockDim.x)  // full block size per width byte, 0 = invalid
    ssize[w] = (unsigned char)((w <= 32 || w == RAW_WIDTH) ? full_size(w) : 0);
  __syncthreads();
  const int e = threadIdx.x;
  if (e >= NE) return;
  int p = e, cnt = 0;
  short ex = 0;
  bool dead = false;
  while (p < len) {  // len <= SEG
    const int sz = ssize[seg[p]];
    if (sz == 0) {
      dead = true;
      break;
    }
    p += sz;
    ++cnt;
  }
  if (dead) ex = EX_DEAD;
  else if (p >= SEG) ex = (short)(p - SEG);
  else ex = EX_END;  // the payload ends inside this segment
  ws.exit[s * NE + e] = ex;
  ws.count[s * NE + e] = (unsigned short)cnt;
}

__global__ void __launch_bounds__(160) idx_chunks(uint64_t nseg, IndexWs ws) {
  extern __shared__ __align__(16) unsigned char sm[];
  short* sx = reinterpret_cast<short*>(sm);
  unsigned short* sc = reinterpret_cast<unsigned short*>(sm + CH * NE * sizeof(short));
  const uint64_t c = blockIdx.x;
  const uint64_t s0 = c * CH;
  const int ns = (int)umin64(CH, nseg - s0);
  {  // chunk maps are 16-B aligned (stride CH * NE * 2 = 33024 B): 16-B loads
    const int nv = ns * NE * 2 / 16;
    const uint4* gx = reinterpret_cast<const uint4*>(ws.exit + s0 * NE);
    const uint4* gc = reinterpret_cast<const uint4*>(ws.count + s0 * NE);
#pragma unroll 4
    for (int i = threadIdx.x; i < nv; i += blockDim.x) {
      const uint4 a = __ldg(gx + i), b = __ldg(gc + i);
      reinterpret_cast<uint4*>(sx)[i] = a;
      reinterpret_cast<uint4*>(sc)[i] = b;
    }
    for (int i = nv * 8 + threadIdx.x; i < ns * NE; i += blockDim.x) {
      sx[i] = ws.exit[s0 * NE + i];
      sc[i] = ws.count[s0 * NE + i];
    }
  }
  __syncthreads();
  const int e = threadIdx.x;
  if (e >= NE) return;
  int cur = e;
  unsigned tot = 0;
  for (int k = 0; k < ns && cur >= 0; ++k) {
    tot += sc[k * NE + cur];
    cur = sx[k * NE + cur];
  }
  ws.cexit[c * NE + e] = (short)cur;
  ws.ccount[c * NE + e] = tot;
}

// Serial walk over the chunk maps.  When they fit (RESOLVE_SMEM_MAX), the CTA
// first copies them into shared memory with coalesced loads, so the walk is a
// chain of shared-memory loads instead of dependent L2 round trips.
constexpr size_t RESOLVE_SMEM_MAX = 192 * 1024;
__host__ __device__ constexpr size_t resolve_smem(uint64_t nchunk) {
  return nchunk * NE * 4 + ((nchunk * NE * 2 + 15) & ~(uint64_t)15);
}

__global__ void idx_resolve(uint64_t nchunk, IndexWs ws, int staged) {
  extern __shared__ __align__(16) unsigned char rsm[];
  unsigned* scc = reinterpret_cast<unsigned*>(rsm);
  short* sce = reinterpret_cast<short*>(rsm + nchunk * NE * 4);
  if (staged) {
    for (uint64_t i = threadIdx.x; i < nchunk * NE; i += blockDim.x) {
      scc[i] = ws.ccount[i];
      sce[i] = ws.cexit[i];
    }
    __syncthreads();
  }
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  long long entry = 0;
  unsigned long long base = 0;
  for (uint64_t c = 0; c < nchunk; ++c) {
    ws.centry[c] = entry;
    ws.cbase[c] = base;
    if (entry < 0) continue;
    base += staged ? scc[c * NE + entry] : ws.ccount[c * NE + entry];
    entry = staged ? sce[c * NE + entry] : ws.cexit[c * NE + entry];
  }
}

// record (block << 24) | (w << 8) | code, the smallest block wins
__device__ __forceinline__ void idx_error(Status* st, uint64_t blk, int w, unsigned code) {
  atomicMin(&st->decode_error, (unsigned long long)((blk << 24) | ((uint64_t)(w & 0xFFFF) << 8) | code));
}

// One CTA per EG consecutive segments (a chunk is CH / EG CTAs, so the walk is
// spread over ~nseg / EG SMs instead of one CTA per chunk).  The CTA stages the
// exit/count maps of its chunk's segments up to its own, and its segments'
// payload bytes, in shared memory: the entry resolution and the block walk
// are then chains of shared-memory loads instead of dependent L2 round trips.
constexpr int EG = 16;
constexpr size_t EMIT_MAP = ((size_t)(CH - 1) * NE * 2 + 15) & ~(size_t)15;  // one map array, 16-B padded
constexpr size_t EMIT_SMEM = (size_t)EG * SEG + 2 * EMIT_MAP;
static_assert(CH % EG == 0, "a chunk is a whole number of emit CTAs");

__global__ void __launch_bounds__(CH) idx_emit(const uint8_t* payload, uint64_t psize, uint64_t nseg, uint64_t n,
                                               IndexWs ws, Status* st) {
  extern __shared__ __align__(16) unsigned char esm[];
  uint8_t* sbytes = esm;                                          // [EG * SEG]
  short* sx = reinterpret_cast<short*>(esm + (size_t)EG * SEG);   // [(CH - 1) * NE]
  unsigned short* sc = reinterpret_cast<unsigned short*>(esm + (size_t)EG * SEG + EMIT_MAP);
  __shared__ int s_entry[EG];
  __shared__ unsigned long long s_base[EG];
  const uint64_t s_first = (uint64_t)blockIdx.x * EG;
  const uint64_t c = s_first / CH;
  const uint64_t sc0 = c * CH;
  const int ns = (int)umin64(EG, nseg - s_first);
  const int nmap = (int)(s_first - sc0) + ns - 1;  // maps needed: chunk start .. our last segment - 1
  const uint64_t nb = (n + BLOCK - 1) / BLOCK;
  const int last_cnt = (int)(n - (nb - 1) * BLOCK);
  {  // the maps are 16-B aligned (chunk stride CH * NE * 2 = 33024 B): 16-B loads, many in flight
    const int nv = nmap * NE * 2 / 16;
    const uint4* gx = reinterpret_cast<const uint4*>(ws.exit + sc0 * NE);
    const uint4* gc = reinterpret_cast<const uint4*>(ws.count + sc0 * NE);
#pragma unroll 4
    for (int i = threadIdx.x; i < nv; i += blockDim.x) {
      const uint4 a = __ldg(gx + i), b = __ldg(gc + i);
      reinterpret_cast<uint4*>(sx)[i] = a;
      reinterpret_cast<uint4*>(sc)[i] = b;
    }
    for (int i = nv * 8 + threadIdx.x; i < nmap * NE; i += blockDim.x) {
      sx[i] = ws.exit[sc0 * NE + i];
      sc[i] = ws.count[sc0 * NE + i];
    }
  }
  const uint64_t g0 = s_first * SEG;
  const int len = (int)umin64((uint64_t)ns * SEG, psize > g0 ? psize - g0 : 0);
  if ((reinterpret_cast<uintptr_t>(payload) & 7) == 0) {
    const uint2* src = reinterpret_cast<const uint2*>(payload + g0);
#pragma unroll 8
    for (int i = threadIdx.x; i < (len >> 3); i += blockDim.x) reinterpret_cast<uint2*>(sbytes)[i] = __ldg(src + i);
    for (int i = (len & ~7) + threadIdx.x; i < len; i += blockDim.x) sbytes[i] = __ldg(payload + g0 + i);
  } else {
    for (int i = threadIdx.x; i < len; i += blockDim.x) sbytes[i] = __ldg(payload + g0 + i);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long entry = ws.centry[c];
    unsigned long long base = ws.cbase[c];
    const int kpre = (int)(s_first - sc0);
    for (int k = 0; k < kpre + ns; ++k) {
      if (k >= kpre) {
        s_entry[k - kpre] = (int)entry;
        s_base[k - kpre] = base;
      }
      if (entry >= 0 && k < nmap) {
        base += sc[k * NE + entry];
        entry = sx[k * NE + entry];
      }
    }
  }
  __syncthreads();
  const int k = threadIdx.x;
  if (k >= ns) return;
  const uint64_t s = s_first + k;
  int e = s_entry[k];
  if (e == EX_END || e == EX_DEAD || e < 0) {
    // chain never enters this segment: an earlier segment reported the error
    // (or the true chain ended before this segment)
    return;
  }
  uint64_t pos = s * SEG + (uint64_t)e;
  uint64_t blk = s_base[k];
  const uint64_t send = (s + 1) * SEG;
  while (pos < send && blk < nb) {
    if (pos >= psize) {  // codec.py:307-308
      idx_error(st, blk, 0, DE_TRUNC);
      return;
    }
    const int w = sbytes[pos - g0];  // pos < min(psize, send): staged
    const int cnt = (blk == nb - 1) ? last_cnt : BLOCK;
    int size;
    if (w == RAW_WIDTH) size = 1 + 4 * cnt;  // 310-311
    else if (w <= 32) size = 5 + ((cnt - 1) * w + 7) / 8;  // 312-313
    else {  // 314-315
      idx_error(st, blk, w, DE_WIDTH);
      return;
    }
    if ((blk & (TB - 1)) == 0) ws.gt[blk / TB] = pos;
    if (ws.widths) ws.widths[blk] = (uint8_t)w;
    pos += size;
    if (pos > psize) {  // 319-320
      idx_error(st, blk, 0, DE_TRUNC);
      return;
    }
    if (blk == nb - 1 && pos != psize) {  // 321-322
      idx_error(st, nb, 0, DE_TRAIL);
      st->trailing = psize - pos;
      return;
    }
    ++blk;
  }
  // the chain ran out of payload before nb blocks (also when the payload
  // ends exactly on this segment's boundary: pos == psize == send)
  if (blk < nb && pos >= psize) idx_error(st, blk, 0, DE_TRUNC);
}

__global__ void idx_sidecar(const IndexWs ws, uint64_t n, uint64_t psize, uint64_t* tile_off) {
  const uint64_t nb = (n + BLOCK - 1) / BLOCK;
  const uint64_t ntiles = (nb + TB - 1) / TB;
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i < ntiles) tile_off[i] = ws.gt[i];
  if (i == ntiles) tile_off[ntiles] = psize;
}

}  // namespace gz
