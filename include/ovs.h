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
    OVS_ECAPACITY = 7,   /* distributed: output larger than out_capacity                         */
    OVS_EINTERNAL = 8    /* a device-side check failed: returned by a call with rep != NULL, and
                            by ovs_device_status() for calls without a report (graph replays)          */
} ovs_status;

typedef enum { OVS_U32 = 0, OVS_I32 = 1, OVS_F64 = 2 } ovs_dtype;
typedef enum { OVS_ROS = 0, OVS_DRO = 1 } ovs_method;

/* flags */
#define OVS_DRO_PADDED_POSITIONS 1u /* DRO sample positions of the Lemma 1 proof's padding
                                        instead of balanced segments (Q9)   */

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
 * Multi-GPU building blocks (ROS).  One process per GPU; rank r holds the contiguous shard
 * [offset, offset + n_local) of a global array of n_global keys (ranks in index order).  The
 * caller runs the NCCL collectives between the three calls (paper_1608_08648_b200/dist.py
 * does it with torch.distributed), the way the paper's multi-core method splits the work
 * (PAPER.md:656-681): each GPU samples its shard, the sample is assembled everywhere, every
 * GPU classifies its keys against the same splitters, buckets are exchanged (bucket j goes to
 * rank floor(j*world/p); p must be a multiple of world), and each GPU sorts
 * the buckets it received.  Tags are global indices, so rank r's output is exactly the
 * [sum_{j<j0} n_j, sum_{j<j1} n_j) slice of the single-GPU sort of the concatenated input.
 *   1. ovs_dist_sample: d_sample (ovs_dist_sample_words u64 words, device) receives this
 *      shard's records of the global sample, zero elsewhere -> caller: all-reduce SUM.
 *   2. ovs_dist_partition: splitters from the assembled sample, local bucket counts d_counts
 *      (p u32, device) and the local keys (order-preserving bits; + values and global indices
 *      for key-value sorts) in bucket order in d_send_* (n_local items each) -> caller:
 *      all-gather of the counts (world x p, rank-major) and an all-to-all-v of the send buffers
 *      (to rank d: its buckets, in bucket order; from rank s: concatenated in rank order).
 *   3. ovs_dist_finish: the received items (<= recv_capacity) are gathered bucket by bucket
 *      (source-rank order) and sorted into d_out_keys (+ d_out_vals), raw dtype.
 * The three calls must use the same workspace and the same (n_local, n_global, dtype,
 * with_values, params, world, recv_capacity).  Errors: OVS_EINVAL also for DRO, p % world,
 * rank out of range; device-side overflow of recv_capacity sets a status bit (the caller
 * can size recv_capacity from the all-gathered counts before calling finish). */
size_t ovs_dist_workspace_bytes(size_t n_local, uint64_t n_global, int dtype, int with_values, const ovs_params* prm,
                                int world, size_t recv_capacity);
size_t ovs_dist_sample_words(uint64_t n_global, int dtype, const ovs_params* prm);
int ovs_dist_sample(const void* d_keys, size_t n_local, uint64_t offset, uint64_t n_global, int dtype, int with_values,
                    const ovs_params* prm, int world, size_t recv_capacity, uint64_t* d_sample, void* d_ws,
                    size_t ws_bytes, void* stream);
int ovs_dist_partition(const void* d_keys, const uint32_t* d_vals, size_t n_local, uint64_t offset, uint64_t n_global,
                       int dtype, const ovs_params* prm, int world, size_t recv_capacity, const uint64_t* d_sample,
                       void* d_send_keys, uint32_t* d_send_vals, uint32_t* d_send_idx, uint32_t* d_counts, void* d_ws,
                       size_t ws_bytes, void* stream);
int ovs_dist_finish(const void* d_recv_keys, const uint32_t* d_recv_vals, const uint32_t* d_recv_idx, size_t n_local,
                    uint64_t n_global, int dtype, const ovs_params* prm, int world, int rank, size_t recv_capacity,
                    const uint32_t* d_all_counts, void* d_out_keys, uint32_t* d_out_vals, void* d_ws, size_t ws_bytes,
                    void* stream);

/* Parameters for which the buckets of n keys fit one SM's shared memory in one level (SURVEY.md
 * §8(f) f4; the paper leaves p to the user and takes s = lg^2 n).  ROS: p = the
 * smallest power of two with n/p <= 0.6 x the on-chip capacity, capped at the largest p the fast
 * one-level scatter handles (p = 1, a plain sort, when n fits on chip), s = 64 (or less when
 * p*s-1 > n).  DRO: the same p (also <= sqrt(n)), r = min(ceil(log2 n), floor(n/p^2)) >= 1.  Writes
 * method, p, s into *out (flags = 0, seed = 1); OVS_EINVAL / OVS_EDTYPE on bad arguments.  Pure
 * host computation from the device's shared-memory size (no launch). */
int ovs_auto_params(size_t n, int dtype, int with_values, int method, ovs_params* out);

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
