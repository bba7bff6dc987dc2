/* ovs.h — C ABI of the B200-native oversampling sample sort (arXiv 1608.08648).
 *
 * The library sorts n keys of X ("sort n keys of X") by the paper's
 * partitioning pipeline, partition-first:
 *   ROS (random oversampling, Algorithm 2's sampling):
 *     sample ps-1 keys uniformly at random, sort the sample, the p-1 splitters are the
 *     (i*s)-th smallest sample keys, every key is classified by binary search over the
 *     splitters with the (key, index) duplicate tie-break, the keys are
 *     scattered into p buckets, every bucket is sorted independently and the buckets are
 *     concatenated.
 *   DRO (deterministic regular oversampling, Algorithm 1 = SqDet):
 *     p contiguous sequences are sorted, rp regular samples per sequence, splitters are the
 *     (i*rp)-th smallest of the rp^2 samples, each sorted sequence is split by binary search,
 *     and bucket j gathers its p runs and is sorted (instead of the paper's p-way merge).
 *
 * Conventions (all entry points):
 *   - Plain pointers and sizes only; no C++ or torch types cross this boundary, no exceptions.
 *   - d_* pointers are DEVICE memory on the current CUDA device; h_* / report pointers are HOST.
 *   - The caller owns every buffer.  The library never allocates device memory on the sort
 *     path: scratch is the caller's workspace d_ws of ws_bytes >= ovs_workspace_bytes(...).
 *   - Sorting is in place: d_keys (and d_vals) hold the input on entry, the output on return.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  All work is
 *     enqueued on it and the call returns after enqueue (it is CUDA-graph capturable) unless
 *     `rep` is non-NULL, in which case it synchronises `stream` and fills the report.
 *   - Parameters are validated before any launch: a failing call does no work.
 *   - Preconditions: f64 inputs contain no NaN and no -0.0 (BASELINE.json north_star);
 *     n < 2^32 - 33 (positions are 32-bit, counted from a 32-byte-aligned base).
 *   - Determinism: the same input bytes and parameters give bit-identical output, splitters
 *     and bucket counts (the oracle's, see oracle/ovs_oracle.cpp).
 */
#ifndef OVS_H
#define OVS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    OVS_OK = 0,
    OVS_EINVAL = 1,      /* p == 0, NULL pointer with n > 0, n >= 2^32-33, bad method/flags  */
    OVS_EDTYPE = 2,      /* unsupported dtype                                                   */
    OVS_ESAMPLE = 3,     /* ROS: s == 0 or p*s-1 > n ("ps-1 <= n");
                            DRO: r == 0 or r*p > floor(n/p) (distinct positions) */
    OVS_EWORKSPACE = 4,  /* ws_bytes < ovs_workspace_bytes(...)                                  */
    OVS_ECUDA = 5,       /* a CUDA runtime error; see ovs_last_error()                           */
    OVS_ENCCL = 6,       /* an NCCL failure (distributed calls); see ovs_last_error()            */
    OVS_ECAPACITY = 7,   /* distributed: some rank's received items exceed its out_capacity or the
                            window (*n_out = this rank's requirement; every rank returns it)      */
    OVS_EINTERNAL = 8    /* a device-side check failed: returned by a call with rep != NULL, and
                            by ovs_device_status() for calls without a report (graph replays)          */
} ovs_status;

typedef enum {
    OVS_U32 = 0, OVS_I32 = 1, OVS_F64 = 2,
    OVS_S32 = 3  /* 32-byte string records in memcmp order (the paper's workload):
                    d_keys holds n records of 32 bytes (16-byte aligned); ROS, ovs_sort_keys only
                    (DRO or values: OVS_EDTYPE); the report's splitter keys are (p-1) records */
} ovs_dtype;
typedef enum { OVS_ROS = 0, OVS_DRO = 1 } ovs_method;

/* flags */
#define OVS_DRO_PADDED_POSITIONS 1u /* DRO sample positions of the Lemma 1 proof's padding
                                        instead of balanced segments (Q9)   */
#define OVS_DRO_MERGE 2u            /* DRO step 5 as the paper's p-way merge (Alg. 1 step 5,
                                       PAPER.md:273-275): fine split by the regular sample, the
                                       p sorted runs of every fine bucket merged on chip; the
                                       default re-sorts every bucket (same output, see DESIGN) */

typedef struct {
    uint32_t method; /* OVS_ROS or OVS_DRO                                                      */
    uint32_t p;      /* number of buckets (sequences) p >= 1; p == 1 is a plain stable sort   */
    uint32_t s;      /* ROS: oversampling factor s (sample = p*s-1 keys);
                        DRO: r = ceil(omega_n) (T_k = r*p keys)                 */
    uint32_t flags;  /* OVS_DRO_PADDED_POSITIONS                                              */
    uint64_t seed;   /* ROS sample stream seed (reading Q1 of DESIGN.md); ignored by DRO       */
} ovs_params;

typedef struct {          /* optional, caller-owned HOST memory; each array pointer may be NULL */
    void* splitter_keys;      /* p-1 keys of the input dtype                                    */
    uint64_t* splitter_tags;  /* p-1 tags: ROS original index; DRO position in the sorted X_k
                                 array (start_k + t)  (reading Q6)           */
    uint64_t* bucket_counts;  /* p bucket sizes |Y_j|                                           */
    float phase_ms[8];        /* CUDA events on `stream` between the phase boundaries of
                                 ovs_set_phase_events: [0] sample (a1-a2; DRO: a9 sequence
                                 sorts), [1] sample sort + splitters (a3-a4; DRO a10-a12),
                                 [2] classify + histogram + scans (a5-a6; DRO a13), [3] scatter
                                 (a7; DRO a14 gather), [4] bucket sort (a8; DRO a14 sorts),
                                 [5] 0 (re-splits run inside the bucket sorter), [6] exchange
                                 (distributed calls; 0 here), [7] total                          */
    uint32_t max_bucket;      /* max_j |Y_j|                                                    */
    uint32_t kernel_launches; /* kernels this call enqueued                                     */
    uint32_t device_status;   /* 0, or a device-side failure bit set                            */
    uint32_t reserved;
    uint64_t exchange_bytes;  /* distributed calls: bytes this rank stored into other ranks'
                                 windows (sample records, count rows, items); 0 otherwise        */
} ovs_report;

/* Bytes of workspace ovs_sort_keys / ovs_sort_pairs_stable need for these arguments
 * (0 on invalid arguments).  with_values: 0 keys only, 1 key-value pairs. */
size_t ovs_workspace_bytes(size_t n, int dtype, int with_values, const ovs_params* prm);

/* Sort n keys of dtype in place in d_keys (device).  Output is the unique nondecreasing
 * permutation; splitters and bucket counts follow the method (see top). */
int ovs_sort_keys(void* d_keys, size_t n, int dtype, const ovs_params* prm, void* d_ws, size_t ws_bytes,
                  void* stream, ovs_report* rep);

/* Stable key-value sort: d_vals (uint32, device) ride with their keys; equal keys keep their
 * input order ("equally valued keys retain in the output their relative input order",
 * PAPER.md:45-47). */
int ovs_sort_pairs_stable(void* d_keys, uint32_t* d_vals, size_t n, int dtype, const ovs_params* prm, void* d_ws,
                          size_t ws_bytes, void* stream, ovs_report* rep);

/* ---------------------------------------------------------------------------------------
 * Multi-GPU (ROS): one process per GPU of one NVLink/NVSwitch node, one
 * call per rank.  Rank r holds the contiguous shard [offset_r, offset_r + n_local_r) of a global
 * array of n_global keys (ranks in index order; the library all-gathers the sizes).  The work is
 * split the way the paper's multi-core method splits it: every GPU draws the
 * same global sample index set (reading Q1 over n_global) and contributes the records of its
 * shard, every GPU computes the same splitters, classifies its keys (tags = global indices, so
 * the tie rule is the single-process one) and stores them straight into the owner's
 * receive window over NVLink (bucket j lives on rank floor(j*world/p); p must be a multiple of
 * world), and every GPU sorts the buckets it owns.  Rank r's output is exactly the
 * slice [sum_{j<j0} n_j, sum_{j<j1} n_j) of the single-GPU sort of the concatenated input, with
 * the same splitters and bucket counts.
 *
 * The communicator owns an NCCL communicator (torch's NCCL 2.28) and a symmetric NCCL window
 * (ncclMemAlloc + ncclCommWindowRegister) that holds the sample records, the count matrix and
 * the received items; kernels store into the other ranks' windows through their NVLink mappings
 * (ncclGetLsaPointer) and the phases are separated by NCCL device-API LSA barriers.  These calls
 * make the communicator's device current on the calling thread. */
typedef struct ovs_comm ovs_comm;

/* ncclGetUniqueId into out[128] (call on one rank, broadcast the bytes to the others). */
int ovs_comm_unique_id(void* out);
/* Collective: create the communicator of `world` ranks on CUDA device `device`, with a window of
 * at least window_bytes (OVS_ENCCL if NCCL fails or not every rank is NVLink load/store reachable). */
int ovs_comm_create(ovs_comm** out, const void* nccl_unique_id, int rank, int world, int device, size_t window_bytes);
/* Collective: grow the window to the largest window_bytes any rank asks for (no-op if large enough). */
int ovs_comm_reserve(ovs_comm* c, size_t window_bytes, void* stream);
int ovs_comm_destroy(ovs_comm* c);
size_t ovs_comm_window_bytes(const ovs_comm* c);
/* Window bytes that let a rank receive n_recv items (sample records and count matrix included). */
size_t ovs_dist_window_bytes(size_t n_recv, int dtype, int with_values, const ovs_params* prm, int world);
/* Collective (all-gathers the shard sizes; synchronises `stream`): workspace bytes this rank
 * needs for ovs_dist_sort_* with these arguments; 0 on invalid arguments. */
size_t ovs_dist_workspace_bytes(ovs_comm* c, size_t n_local, int dtype, int with_values, const ovs_params* prm,
                                size_t out_capacity, void* stream);
/* Collective distributed sort.  d_in (n_local keys, device, not modified); d_out receives this
 * rank's sorted slice (*n_out items, raw dtype; out_capacity items available).  Synchronises
 * `stream` twice (the shard-size all-gather; the count matrix read-back, which decides capacity
 * and the exchange plan) and returns with the exchange and the local sort enqueued.  Errors are
 * decided from all-gathered data, so every rank returns the same code: OVS_EINVAL (p not a
 * multiple of world, flags, n_global >= 2^32-33; DRO: p not dividing n_global or unequal shards),
 * OVS_ESAMPLE (ROS: p*s-1 > n_global; DRO: r*p > n_global/p),
 * OVS_EWORKSPACE (some rank's ws_bytes too small), OVS_ECAPACITY (some rank receives more items
 * than its out_capacity or the window holds: *n_out = this rank's requirement; grow and call
 * again), OVS_ENCCL, OVS_ECUDA.  rep (optional, host): the global splitters and bucket counts,
 * phase_ms ([0] sample + record exchange, [1] sample sort, [2] classify + histogram + count
 * exchange and read-back, [3] = [6] fused scatter/exchange, [4] local bucket sort, [7] total). */
int ovs_dist_sort_keys(ovs_comm* c, const void* d_in, size_t n_local, int dtype, const ovs_params* prm, void* d_out,
                       size_t out_capacity, size_t* n_out, void* d_ws, size_t ws_bytes, void* stream, ovs_report* rep);
/* Stable key-value variant: uint32 values ride with their keys; equal keys keep their global
 * input order.
 * DRO across GPUs (method OVS_DRO, s = r; SURVEY.md §8(e) DRO steps, the paper's McDet split,
 * PAPER.md:664-670): every rank holds n_global / world keys, i.e. p/world whole sequences of
 * Algorithm 1's baseline split (p must divide n_global); each rank sorts its sequences and stores
 * their r p regular samples into every window, all ranks pick the same splitters, split their
 * sequences, and every run X_{k,j} is stored straight into bucket j's owner, which sorts the bucket
 * (the stable result of the paper's p-way merge).  Output, splitters (tags = global positions in the
 * sorted sequences) and counts equal the single-process Algorithm 1 on the concatenation. */
int ovs_dist_sort_pairs_stable(ovs_comm* c, const void* d_keys, const uint32_t* d_vals, size_t n_local, int dtype,
                               const ovs_params* prm, void* d_out_keys, uint32_t* d_out_vals, size_t out_capacity,
                               size_t* n_out, void* d_ws, size_t ws_bytes, void* stream, ovs_report* rep);
/* Host-only: the exchange plan of `rank` from the all-gathered count matrix counts[world][p]:
 * dst_off[p] = where this rank's run of bucket b starts inside its owner's receive region (owner
 * floor(b*world/p); runs of one bucket in source-rank order), recv[world] = items every rank
 * receives.  (The plan ovs_dist_sort_* computes; exported for the multi-process CPU tests.) */
int ovs_dist_plan(const uint32_t* counts, int world, uint32_t p, int rank, uint32_t* dst_off, uint64_t* recv);
/* Test support: `world` ranks emulated on ONE GPU by one call (the same phases and kernels; the
 * fused scatter stores into the other emulated ranks' windows d_win[r] of win_bytes each; every
 * phase runs rank after rank, so no kernel waits on another).  Arrays of length world. */
int ovs_dist_sort_virtual(int world, const void* const* d_keys, const uint32_t* const* d_vals, const size_t* n_local,
                          int dtype, const ovs_params* prm, void* const* d_out_keys, uint32_t* const* d_out_vals,
                          const size_t* out_capacity, size_t* n_out, void* const* d_ws, const size_t* ws_bytes,
                          void* const* d_win, size_t win_bytes, void* stream, uint64_t* counts, void* split_keys,
                          uint64_t* split_tags, float* rank_ms /* optional: each rank's device time */);
size_t ovs_dist_virtual_workspace_bytes(int world, const size_t* n_local, int dtype, int with_values,
                                        const ovs_params* prm, const size_t* out_capacity, size_t win_bytes);

/* Parameters for which the buckets of n keys fit one SM's shared memory in one level (SURVEY.md
 * §8(f) f4; the paper leaves p to the user and takes s = lg^2 n).  ROS: p = the
 * smallest power of two with n/p <= 0.6 x the on-chip capacity, capped at the largest p the fast
 * one-level scatter handles (p = 1, a plain sort, when n fits on chip), s = 64 (or less when
 * p*s-1 > n).  DRO: the same p (also <= sqrt(n)), r = min(ceil(log2 n), floor(n/p^2)) >= 1.  Writes
 * method, p, s into *out (flags = 0, seed = 1); OVS_EINVAL / OVS_EDTYPE on bad arguments.  Pure
 * host computation from the device's shared-memory size (no launch). */
int ovs_auto_params(size_t n, int dtype, int with_values, int method, ovs_params* out);

/* ---------------------------------------------------------------------------------------
 * Host buffers (the end-to-end path): a stream of keys-only sorts of n keys
 * each, from and to PINNED host memory, the problem statement of PAPER.md:254 with the keys
 * starting and ending in host memory.  Every submitted step copies its whole input to the device,
 * sorts it there (ovs_sort_keys, same splitters and counts) and copies the whole result back; the
 * pipe runs step k's host->device copy, the sorts, and step k-1's device->host copy on three CUDA
 * streams of its own, so a stream of sorts is bound by the slower PCIe direction, not by the sum
 * of both copies and the sort.
 *   ovs_host_pipe_create: d_bufs[0..nbuf) are nbuf (1..16; 3 lets a copy-in never wait) device
 *     buffers of n keys each and d_ws a workspace of ws_bytes >= ovs_workspace_bytes(n, dtype, 0,
 *     prm); all stay the caller's, must outlive the pipe and must not be used by the caller while
 *     steps are in flight.  The pipe owns only its streams and events (on the device current at
 *     creation).  OVS_EINVAL / OVS_EDTYPE / OVS_EWORKSPACE / OVS_ECUDA.
 *   ovs_host_pipe_submit: enqueue one step h_in -> device -> sort -> h_out (host pointers, n keys
 *     each, page-locked so the copies are asynchronous; h_in may equal h_out; h_in must stay
 *     unchanged and h_out unread until the next ovs_host_pipe_wait).  Returns without waiting for
 *     the device (a buffer is refilled only after its previous result has left the device; that
 *     wait is on the device).  Errors as ovs_sort_keys.
 *   ovs_host_pipe_wait: blocks until every submitted step's result is in host memory; *ms (may be
 *     NULL) = device time from the start of the first copy-in submitted since the previous wait to
 *     the end of the last copy-out.  Returns OVS_OK, or OVS_EINTERNAL if a device-side check of
 *     any of those sorts failed (ovs_device_status semantics; the sticky word is reset).
 *   ovs_host_pipe_destroy: waits for the pipe's streams and releases them (NULL is allowed). */
typedef struct ovs_host_pipe ovs_host_pipe;
int ovs_host_pipe_create(ovs_host_pipe** out, size_t n, int dtype, const ovs_params* prm, void* const* d_bufs,
                         int nbuf, void* d_ws, size_t ws_bytes);
int ovs_host_pipe_submit(ovs_host_pipe* hp, const void* h_in, void* h_out);
int ovs_host_pipe_wait(ovs_host_pipe* hp, float* ms);
int ovs_host_pipe_destroy(ovs_host_pipe* hp);

/* Profiling hook (thread-local): subsequent sort calls on this thread record events[k]
 * (cudaEvent_t passed as void*) on their stream at phase boundary k, without synchronising:
 *   0 start, 1 after the sample draw + gather (a1-a2), 2 after the sample sort + splitters
 *   (a3-a4), 3 after classify + histogram + scans (a5-a6), 4 after the scatter (a7), 5 after
 *   the bucket sort (a8) = end.  DRO: 1 after the sequence sorts (a9), 2 after a10-a12, 3 after
 *   the split (a13), 4 after the bucket gather, 5 end.
 * count = 0 disables.  NULL entries are skipped.  The caller owns the events. */
void ovs_set_phase_events(void* const* events, int count);

/* Device-side status without a report.  The first 8 bytes of a workspace hold two status words:
 * word 0 = the failure bits of the last call (zeroed when a call starts), word 1 = the sticky OR
 * of every call's bits since the last reset (so a CUDA-graph replay loop can be checked once).
 * Bits: 1 fewer than ps-1 distinct sample draws; 2 a bucket over the on-chip capacity reached the
 * sorter; 4 a work list overflowed (output possibly not sorted).  ovs_device_status synchronises
 * `stream`, writes the sticky word to *status (may be NULL) and, if reset != 0, clears it
 * (enqueued on `stream`).  Returns OVS_OK when the sticky word is 0, else OVS_EINTERNAL (message
 * in ovs_last_error()), OVS_ECUDA on a CUDA error.  A fresh workspace's sticky word is whatever
 * the memory held: zero the first 8 bytes, or call ovs_device_status(..., reset=1) once, before use. */
int ovs_device_status(const void* d_ws, void* stream, uint32_t* status, int reset);

/* Thread-local message of the last failure on this thread ("" if none). */
const char* ovs_last_error(void);

/* Library build identification, e.g. "ovs 0.1 sm_100a". */
const char* ovs_version(void);

#ifdef __cplusplus
}
#endif

#endif /* OVS_H */
