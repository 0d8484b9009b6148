/*
 * gzccl.h -- C ABI of the B200-native gZCCL hot path (libgzccl.so, sm_100a).
 *
 * Plain pointers and sizes only; every pointer is device memory unless stated.
 * The reference (/root/reference/pkg/src/gzccl) is a Python package with no
 * native layer, so each entry point names the Python interface it replaces;
 * the Python shim paper_2308_05199_b200/ binds these through ctypes with the
 * reference's names and error behaviour.
 *
 * Conventions
 *   - Return value: 0 on success, otherwise a cudaError_t (launch/driver
 *     errors) or one of the GZ_E* codes below (argument errors).
 *   - Data-dependent errors (non-finite input, malformed blob) are written by
 *     the kernels into a caller-owned device gz_status that the caller resets
 *     with gz_status_reset() and inspects after synchronising.
 *   - Every call is stream-ordered on `stream` and never allocates.
 *   - A workspace (gz_workspace_bytes) must be zeroed once with
 *     gz_workspace_init(); it may then be reused by any number of calls that
 *     are ordered on one stream (one workspace per concurrent stream).
 */
#ifndef GZCCL_H
#define GZCCL_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* gz_stream_t; /* == cudaStream_t */

enum {
  GZ_OK = 0,
  GZ_EINVAL = 10001,    /* bad argument: null pointer, size, alignment */
  GZ_EBOUND = 10002,    /* error bound not finite and > 0 (codec.py:89-93) */
  GZ_ECAPACITY = 10003, /* output buffer smaller than gz_compress_bound(n) */
  GZ_EBLOCK = 10004     /* block size other than 32 (format is frozen, codec.py:42) */
};

/* Device error record (32 bytes). */
typedef struct gz_status {
  uint64_t first_nonfinite; /* index of the first non-finite input, ~0 if none (codec.py:83-85) */
  uint64_t decode_error;    /* (block_index << 24) | (width << 8) | code, ~0 if none; the smallest
                               block index wins; codes 1 width, 2 truncated, 3 trailing bytes,
                               4 sidecar mismatch, 5 header (codec.py:273-322) */
  uint64_t trailing_bytes;  /* trailing byte count of a code-3 decode error (codec.py:321-322) */
  uint64_t comm_error;      /* 1: a peer flag never arrived (in-kernel wait gave up after
                               GZ_FLAG_TIMEOUT_NS; the kernel skipped its work), ~0 if none */
} gz_status;
#define GZ_FLAG_TIMEOUT_NS 20000000000ull

/* ---- sizing (host functions, no device work) ---------------------------- */
/* Compressed-size bound incl. header and 64 B of read slack.  Tighter than
 * worst_case_blob_bytes (codec.py:492-494): raw blocks are 129 B, not 133. */
uint64_t gz_compress_bound(uint64_t n);
uint64_t gz_num_tiles(uint64_t n);        /* tiles of GZ_TILE_BLOCKS blocks */
uint32_t gz_tile_blocks(void);            /* 32-value blocks per tile (CTA) */
uint64_t gz_sidecar_bytes(uint64_t n);    /* u64 tile offsets [tiles+1] + u8 block widths [tiles*32] */
uint64_t gz_workspace_bytes(uint64_t n);  /* CTA status words, per-tile offsets and the L2 scratch */

/* ---- setup ---------------------------------------------------------------- */
int gz_workspace_init(void* ws, uint64_t ws_bytes, gz_stream_t stream);
int gz_status_reset(gz_status* d_status, gz_stream_t stream);

/* ---- codec ------------------------------------------------------------------
 * gz_compress replaces codec.compress(data, eb, workspace) (codec.py:149-270).
 *   x[n] f32 -> blob (reference byte format, header included) of length
 *   *d_len; blob_cap >= gz_compress_bound(n); blob 16-byte aligned.
 *   sidecar (gz_sidecar_bytes, may be NULL): tile offsets and block widths for decoders.
 *   d_block_offsets (nb = ceil(n/32) u64, may be NULL): payload offset of
 *   every block == np.cumsum(sizes) exclusive scan (codec.py:241-243).
 *   block must be 32.
 */
int gz_compress(const float* x, uint64_t n, double eb, uint32_t block, uint8_t* blob, uint64_t blob_cap,
                uint64_t* d_len, void* sidecar, uint64_t* d_block_offsets, void* ws, uint64_t ws_bytes,
                gz_status* d_status, gz_stream_t stream);

/* gz_decompress_sidecar replaces codec.decompress(blob) (codec.py:284-369)
 * when the blob's sidecar is available (collective path).  n and eb are the
 * blob header's values; y[n] f32 output. */
int gz_decompress_sidecar(const uint8_t* blob, const void* sidecar, uint64_t n, double eb, float* y,
                          gz_status* d_status, gz_stream_t stream);
/* y = op(local, decompress(blob)) -- the last step of a standalone
 * ring_reduce_scatter_c (collectives.py:274-290: decode, then _apply_op with
 * the local chunk first) without re-compressing the result. */
int gz_decompress_reduce(const uint8_t* blob, const void* sidecar, const float* local, uint64_t n, double eb, int op,
                         float* y, gz_status* d_status, gz_stream_t stream);
/* Decode up to GZ_MAX_DECODE_SEGMENTS blobs (with sidecars; blobs may live in
 * peer GPUs' memory) in one launch: the compress-once allgather decoding every
 * owner's blob (collectives.py:238-241).  Empty entries (ns[i] == 0) are skipped. */
#define GZ_MAX_DECODE_SEGMENTS 8
int gz_decompress_multi(const uint8_t* const* blobs, const void* const* sidecars, const uint64_t* ns, uint32_t count,
                        double eb, float* const* ys, int reserve_sms, gz_status* d_status, gz_stream_t stream);

/* The same for messages in slotted form (gz_step_io's out_slots / out_sizes /
 * out_widths, 128-byte aligned slots; usually a peer GPU's memory): the
 * compress-once allgather decoding every owner's last reduce-scatter output in
 * place, without first gathering it into a contiguous blob. */
int gz_decompress_slots_multi(const uint8_t* const* slots, const uint32_t* const* sizes, const uint8_t* const* widths,
                              const uint64_t* ns, uint32_t count, double eb, float* const* ys, int reserve_sms,
                              gz_status* d_status, gz_stream_t stream);

/* gz_index replaces the sequential block walk of codec.decompress
 * (codec.py:298-322): validates the payload of a blob of header count n and
 * payload length payload_len (device pointer to the blob) and builds its
 * sidecar, so that any reference-produced blob can be decoded on the device.
 * Errors are reported in d_status->decode_error with the reference's
 * semantics (first failing block in walk order). */
int gz_index(const uint8_t* blob, uint64_t payload_len, uint64_t n, void* sidecar, void* ws, uint64_t ws_bytes,
             gz_status* d_status, gz_stream_t stream);
uint64_t gz_index_workspace_bytes(uint64_t payload_len);

/* ---- fused ring reduce-scatter step ----------------------------------------
 * One step of ring_reduce_scatter_c (collectives.py:274-290) for one rank:
 *   acc = op(local, decompress(blob_in))   (op 0 = sum "+", 1 = np.maximum)
 *   blob_out = compress(acc, eb)           (sidecar_out written alongside)
 *   acc_out[m] (may be NULL) receives acc.
 * blob_out / sidecar_out / d_len_out may point into a peer GPU's memory
 * (CUDA IPC over NVLink): the step then also performs the send. */
int gz_reduce_step(const uint8_t* blob_in, const void* sidecar_in, const float* local, uint64_t m, double eb,
                   int op, float* acc_out, uint8_t* blob_out, uint64_t blob_out_cap, uint64_t* d_len_out,
                   void* sidecar_out, void* ws, uint64_t ws_bytes, gz_status* d_status, gz_stream_t stream);

/* ---- generalized step: plain compress or fused step, blob or slotted I/O ----
 * Slotted form (the reduce-scatter's intermediate messages, never seen by a
 * user): tile t's bytes at out_slots + t * 4224 (128-aligned, gz_slots_bytes),
 * its byte count in out_sizes[t], the block widths in out_widths[t*32 ..] --
 * the same bytes as the blob's tile t, without the gather that makes them
 * contiguous; the consumer's fused step reads them in place (in_slots).
 * in_blob == in_slots == NULL: plain compression of `local`. */
typedef struct {
  const uint8_t* in_blob;
  const void* in_sidecar;
  const uint8_t* in_slots;
  const uint32_t* in_sizes;
  const uint8_t* in_widths;
  uint8_t* blob_out;
  uint64_t blob_out_cap;
  uint64_t* d_len_out;
  void* sidecar_out;
  uint8_t* out_slots;
  uint32_t* out_sizes;
  uint8_t* out_widths;
  uint32_t* post_flag; /* slotted output only, may be NULL: the kernel stores 1 here (e.g. a peer's flag,
                          IPC-mapped) once the whole output is written -- a fused gz_stream_write_u32 */
  uint32_t* wait_flag; /* slotted output only, may be NULL: the kernel waits until this (own-memory) flag
                          is >= 1 before reading its inputs and resets it to 0 when done -- a fused
                          wait + reset.  Bounded: after GZ_FLAG_TIMEOUT_NS the kernel records
                          comm_error = 1 in d_status, skips its work and still posts post_flag, so
                          the peers' streams drain instead of hanging */
  uint64_t report_base; /* added to the offset of a non-finite value of `local` before it is recorded
                           in d_status->first_nonfinite (the chunk's offset in the caller's buffer,
                           so the first bad offset of the whole buffer is reported, codec.py:79-86);
                           UINT64_MAX: `local` is not the caller's input (e.g. reduced in place by an
                           earlier step), report nothing */
} gz_step_io;
uint64_t gz_slots_bytes(uint64_t m);
int gz_step(const gz_step_io* io, const float* local, uint64_t m, double eb, int op, float* acc_out, void* ws,
            uint64_t ws_bytes, gz_status* d_status, gz_stream_t stream);
/* y = op(local, decode(slotted input io->in_*)): a reduce-scatter's last step
 * without re-compression (collectives.py:285-290); local == NULL: y = decode(...) */
int gz_step_reduce(const gz_step_io* io, const float* local, uint64_t m, double eb, int op, float* y,
                   gz_status* d_status, gz_stream_t stream);

/* ---- multi-segment compression (binomial scatter root) ----------------------
 * compress_blocks (codec.py:408-427): nseg independent blobs, blob i written
 * at payload + seg_blob_off[i] (host-planned worst-case slots). */
uint64_t gz_segments_workspace_bytes(const uint64_t* h_counts, uint32_t nseg);
int gz_compress_segments(const float* x, const uint64_t* h_counts, uint32_t nseg, double eb, uint8_t* payload,
                         const uint64_t* h_seg_blob_off, uint64_t* d_seg_len, void* sidecars,
                         const uint64_t* h_seg_sidecar_off, const uint64_t* h_seg_report_off, void* ws,
                         uint64_t ws_bytes, gz_status* d_status, gz_stream_t stream);
/*   h_seg_report_off (may be NULL): per segment, the offset of its first value
 *   in the caller's buffer, added to a non-finite offset before it is recorded
 *   (NULL: the segment's offset inside x). */

/* ---- peer memory (CUDA IPC over NVLink) ----------------------------------- */
int gz_ipc_handle_size(void);
int gz_ipc_get_handle(void* dptr, void* handle_out /* gz_ipc_handle_size() bytes */);
int gz_ipc_open_handle(const void* handle, void** dptr_out);
int gz_ipc_close(void* dptr);
int gz_enable_peer_access(int peer_device);
/* stream-ordered flags (driver stream memory ops; no spinning kernels) */
int gz_stream_write_u32(gz_stream_t stream, void* dptr, uint32_t value);
int gz_stream_wait_u32_geq(gz_stream_t stream, void* dptr, uint32_t value);
/* several flag operations as ONE stream memory-op batch (one graph node),
 * executed in array order: kind 0 = write value, kind 1 = wait until >= value */
typedef struct {
  void* ptr;
  uint32_t value;
  uint32_t kind;
} gz_flag_op;
#define GZ_MAX_FLAG_OPS 64
int gz_stream_flag_ops(gz_stream_t stream, const gz_flag_op* ops, uint32_t count);
/* copy `*d_len + tail` bytes determined on the device: dst may be a peer */
int gz_copy_blob(const uint8_t* src, uint8_t* dst, const uint64_t* d_len, uint64_t max_bytes, gz_stream_t stream);

/* Forward a set of byte ranges in ONE launch (a binomial-scatter hop: the
 * child pulls its subtree's blobs, sidecars and lengths from its parent,
 * collectives.py:511-525).  Item i copies min(*d_len, max_bytes) bytes when
 * d_len is non-NULL (a blob whose length is known only on the device), else
 * max_bytes.  src/dst may be peer (IPC) pointers; 16-byte aligned items
 * move as 16-byte words, others byte by byte. */
typedef struct {
  const uint8_t* src;
  uint8_t* dst;
  const uint64_t* d_len;
  uint64_t max_bytes;
} gz_copy_item;
#define GZ_MAX_COPY_ITEMS 64
/* dst[n] = src[n] (f32, 16-byte aligned) recording the first non-finite offset
 * (+ report_base) in d_status->first_nonfinite (codec.py:79-86): the parts of a
 * collective's input that are kept verbatim, never compressed (the scatter
 * root's own block, collectives.py:500), are validated like the rest. */
int gz_copy_checked(const float* src, float* dst, uint64_t n, uint64_t report_base, gz_status* d_status,
                    gz_stream_t stream);  /* dst == NULL: check only; any 4-byte alignment */
/* out[n] = op(local, recv): _apply_op (collectives.py:32-39), op 0 = sum (binary32
 * RN), 1 = np.maximum (NaN propagates, ties return recv).  out may alias local. */
int gz_apply_op(const float* local, const float* recv, float* out, uint64_t n, int op, gz_stream_t stream);
/* key[i] = status word i (first_nonfinite, decode_error, trailing, comm_error)
 * as (rank << 56) | value, or INT64_MAX where it holds no error: a MIN
 * all-reduce of the keys over the ranks gives, per word, the lowest rank that
 * recorded an error and its value (the rank-ordered raise of
 * collectives.py:202-205).  rank < 128. */
int gz_status_key(const gz_status* d_status, int rank, int64_t* d_key, gz_stream_t stream);
int gz_copy_items(const gz_copy_item* items, uint32_t count, gz_stream_t stream);
/* the same on at most sms_budget SMs (0: all), so that it can run beside a
 * decoder launched with reserve_sms = sms_budget (allgather pipeline) */
int gz_copy_items_sms(const gz_copy_item* items, uint32_t count, int sms_budget, gz_stream_t stream);

/* ---- fixed-rate baseline codec (codec.py:442-489, a comparator) --------------
 * Uniform quantisation of the whole buffer over [min, max] to `bits` (1..16)
 * per value, "<QBff" header (n, bits, lo, hi) + codes LSB-first.  ws:
 * gz_fr_workspace_bytes() of device scratch.  A zero min / max carries the
 * sign numpy's AVX-512 reduction returns (x.min() / x.max(), codec.py:454-455).
 * The host validates a blob's header before decoding. */
uint64_t gz_fr_bound(uint64_t n, uint32_t bits);
uint64_t gz_fr_workspace_bytes(void);
int gz_fr_compress(const float* x, uint64_t n, uint32_t bits, uint8_t* out, uint64_t out_cap, uint64_t* d_len,
                   void* ws, gz_status* d_status, gz_stream_t stream);
int gz_fr_decompress(const uint8_t* blob, uint64_t n, uint32_t bits, float* y, gz_stream_t stream);

/* number of kernels this library has launched so far (all entry points) */
uint64_t gz_launch_count(void);
/* profiling only: stream-ordered write of the GPU's %globaltimer (ns, u64) into dst;
 * works inside a captured CUDA graph (tools/prof_ring_stamps.py) */
int gz_debug_stamp(void* dst, gz_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif
