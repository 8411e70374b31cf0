/* swb200.h -- C-ABI of the B200-native SW#db scoring path (libswb200.so).
 *
 * This is the drop-in boundary for the reference's database-search hot path.  Plain pointers and
 * sizes only; no C++/torch types; no exception ever crosses it.  Every function returns an
 * swb_status; swb_last_error() gives the message for the calling thread.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj/include/swsearch):
 *
 *   swb_db_create / _flat     partition_database          scheduler.hpp:56-65   (length routing)
 *                             + the per-chunk pointer gather  scheduler.hpp:156-160
 *                             (here: one-off length-sorted, interleaved packing, resident in HBM)
 *   swb_search                run_search, lines           scheduler.hpp:188-244
 *                             (profile -> partition -> both kernels -> merge_results), i.e. the
 *                             region SPEC.md:403 times; traceback (scheduler.hpp:246-249) stays host C++
 *   swb_search_keys           the same, returning packed sort keys for the multi-GPU merge
 *   swb_search_keys_device    the same, enqueued on the caller's stream, keys left in device memory
 *   swb_merge_keys            merge_results               scheduler.hpp:106-117  (across shards)
 *   swb_db_merge_keys         the same on the handle's stream, from gathered device keys
 *   swb_score_all             "sequential scalar scan"    scheduler.hpp:179-183  (all N scores)
 *   swb_score_batch           sw_score_batch              align.hpp:91-159
 *   swb_score_pair            sw_score_wavefront          align.hpp:166-229
 *   swb_mdb_*                 run_search over several GPUs of one box in one process
 *                             (no reference equivalent: SPEC.md:342 lists device offload as a non-goal)
 *
 * Semantics common to all scoring entry points: residue codes are 0..23 in the order of
 * alphabet.hpp:60 ("ARNDCQEGHILKMFPSTWYVBZX*"); `matrix` is the 24x24 row-major int32 table of
 * scoring.hpp:32,42 indexed [subject_code*24 + query_code] exactly like align.hpp:34,74;
 * gaps are positive magnitudes with open >= extend >= 0 (scoring.hpp:50-53); a score is the int32
 * value of align.hpp:42-64 -- bit-exact, whichever kernel (packed int16 DPX, int32 re-run,
 * intra-task) produced it.  Hits are ordered score descending, then db_index ascending
 * (scheduler.hpp:111-114) and every database sequence, including empty ones, is a candidate
 * (scheduler.hpp:163,171).
 *
 * There is no CPU fallback: without a usable CUDA device every compute entry point fails with
 * SWB_ERR_CUDA.
 */
#ifndef SWB200_H
#define SWB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum swb_status {
    SWB_OK = 0,
    SWB_ERR_INVALID = 1,     /* bad argument: maps to std::invalid_argument in the C++ shim      */
    SWB_ERR_RANGE = 2,       /* residue / query code >= 24: std::out_of_range (scoring.hpp:203)   */
    SWB_ERR_CUDA = 3,        /* CUDA runtime / driver failure, or no device                       */
    SWB_ERR_NCCL = 4,        /* NCCL failure in the multi-GPU merge                               */
    SWB_ERR_UNSUPPORTED = 5, /* scores would leave the exact int32 range this build guarantees    */
    SWB_ERR_INTERNAL = 6
} swb_status;

typedef struct swb_db swb_db;   /* one packed database shard resident on one GPU */
typedef struct swb_mdb swb_mdb; /* a database sharded over several GPUs of one process */

typedef struct swb_hit {
    uint32_t db_index; /* position in the caller's database (Hit::db_index, scheduler.hpp:88) */
    int32_t score;     /* Hit::score.value */
} swb_hit;

/* Execution report.  The first three fields are SearchStats (scheduler.hpp:120-124). */
typedef struct swb_stats {
    uint64_t lane_scored;      /* sequences below the length threshold (inter-task pool)          */
    uint64_t wavefront_scored; /* sequences at or above it (intra-task pool)                      */
    uint64_t chunks_claimed;   /* work units handed out by the ticket counter                     */
    uint64_t rescored_i32;     /* sequences flagged by the int16 pass and re-run in int32         */
    uint64_t cells;            /* query_len x residues of this shard (GCUPS numerator)*/
    uint64_t padded_cells;     /* cells executed including row/column padding                     */
    uint32_t kernel_launches;  /* launches of this library's kernels during the call              */
    uint32_t reserved;
    float ms_total;            /* device time of the call (CUDA events on the search stream)      */
    float ms_setup;            /* query/matrix upload, profile build, buffer clears               */
    float ms_scan;             /* the packed-int16 tile-wavefront kernel over all groups          */
    float ms_rescore;          /* flag collection + int32 re-run (or the whole scan in wide mode) */
    float ms_topk;             /* key build + top-k select (or the score scatter)                 */
    float ms_reserved;
} swb_stats;

typedef struct swb_db_info {
    uint32_t n_total;          /* sequences in the whole database                                 */
    uint32_t n_local;          /* sequences held by this shard                                    */
    uint32_t n_short;          /* ... routed to the inter-task kernel (length < threshold)        */
    uint32_t n_long;           /* ... routed to the intra-task kernel                             */
    uint32_t n_groups;         /* interleaved groups of 64 short sequences                        */
    uint32_t max_length;       /* longest sequence in this shard                                  */
    uint32_t shard_rank;
    uint32_t shard_count;
    uint64_t residues;         /* real residues in this shard                                     */
    uint64_t padded_residues;  /* residues stored including padding                               */
    uint64_t device_bytes;     /* HBM held by this handle (database + work buffers)               */
    uint64_t length_threshold;
    int32_t device;
    uint32_t kernel_launches_total;  /* kernels this handle has launched so far (searches and re-runs; wraps) */
} swb_db_info;

const char* swb_last_error(void);
const char* swb_version(void);
swb_status swb_device_count(int32_t* count);

/* Pack the caller's database and make it resident on `device`.
 *   seqs[i]/lens[i]   residue codes of sequence i (EncodedSequence::codes, sequence.hpp:22);
 *                     seqs[i] may be NULL when lens[i] == 0.
 *   length_threshold  SearchConfig::length_threshold (scheduler.hpp:24): length < threshold goes
 *                     to the inter-task kernel, the rest to the intra-task kernel.
 *   shard_rank/count  this handle keeps only its residue-balanced share of the database
 *                     (count = 1: everything).  db_index values stay global.
 * The input is not referenced after the call returns. */
swb_status swb_db_create(const uint8_t* const* seqs, const uint32_t* lens, uint32_t n,
                         uint64_t length_threshold, int32_t device, uint32_t shard_rank,
                         uint32_t shard_count, swb_db** out);

/* Same, from concatenated codes and n+1 offsets. */
swb_status swb_db_create_flat(const uint8_t* codes, const uint64_t* offsets, uint32_t n,
                              uint64_t length_threshold, int32_t device, uint32_t shard_rank,
                              uint32_t shard_count, swb_db** out);

/* On-disk packed database: the shard exactly as it sits in HBM -- sorted, grouped,
 * interleaved, with its index tables -- so that a later process skips parsing, sorting and packing.
 * Little-endian, versioned; swb_db_load rejects files of another version or with a damaged header. */
swb_status swb_db_save(swb_db* db, const char* path);
/* Maps the file read-only, validates every table against the invariants the kernels rely on (sizes bounded by the
 * file size, contiguous longest-first groups, unique in-range db_index values, lengths within their group's rows,
 * residue codes within the alphabet, header counters equal to what the tables say) and uploads the residues straight
 * from the mapping.  A stale, truncated or edited file gives SWB_ERR_INVALID, never an out-of-bounds access. */
swb_status swb_db_load(const char* path, int32_t device, swb_db** out);
/* Pack on the host and write the file without touching a GPU (replaces parse + encode of fasta.hpp:80-86 for every
 * later run): same content as swb_db_create + swb_db_save.  names: optional, n NUL-terminated sequence headers that are
 * stored behind the residues so that a later run needs no FASTA at all (include/swsearch/packed.hpp).
 *
 * File layout, little-endian (version 2):
 *   96-byte header  "SWB200DB", u32 version, u32 n_total n_local n_short n_long shard_rank shard_count max_length,
 *                   u64 residues padded_rows total_chunks length_threshold n_groups codes_bytes names_bytes
 *   n_groups x { u64 chunk_base, u32 n_chunks, u32 first_slot }      groups of 64 sequences, longest first
 *   n_groups*64 x u32 slot_index (db_index, 0xFFFFFFFF = unused)     then n_groups*64 x u32 slot_len
 *   codes_bytes of residues: codes[((chunk_base + row/8)*32 + slot%32)*16 + (slot/32)*8 + row%8], pad code 24
 *   optional names: (n_total + 1) x u64 offsets, then the header strings */
swb_status swb_pack_file(const uint8_t* const* seqs, const uint32_t* lens, uint32_t n, uint64_t length_threshold,
                         uint32_t shard_rank, uint32_t shard_count, const char* const* names, const char* path);
swb_status swb_pack_file_flat(const uint8_t* codes, const uint64_t* offsets, uint32_t n, uint64_t length_threshold,
                              uint32_t shard_rank, uint32_t shard_count, const char* const* names, const char* path);

void swb_db_destroy(swb_db* db);
swb_status swb_db_info_get(const swb_db* db, swb_db_info* info);

/* Use an externally owned cudaStream_t (passed as an integer/pointer value, e.g.
 * torch.cuda.current_stream().cuda_stream) for all work of this handle; 0 restores the
 * handle's own (non-blocking) stream.  The legacy default stream is named explicitly, as
 * cudaStreamLegacy ((cudaStream_t)0x1). */
swb_status swb_db_set_stream(swb_db* db, void* cuda_stream);

/* Which kernel scans the database (results are identical; tests and tuning use this to exercise each path):
 *   SWB_SCAN_AUTO      per search: the on-chip tile pipeline for the bulk of the groups next to the wavefront
 *                      kernel on the few tall ones; short queries and small databases use the wavefront kernel
 *   SWB_SCAN_PIPELINE  every group through the on-chip pipeline whenever the query profile leaves room for its rings
 *   SWB_SCAN_WAVEFRONT every group through the wavefront kernel */
typedef enum swb_scan_policy { SWB_SCAN_AUTO = 0, SWB_SCAN_PIPELINE = 1, SWB_SCAN_WAVEFRONT = 2 } swb_scan_policy;
swb_status swb_db_set_scan_policy(swb_db* db, int32_t policy);

/* One query against the shard: scores every sequence, selects the top_k hits.
 *   hits      room for top_k entries;  *n_hits = min(top_k, n_local)
 *   stats     optional
 * Host buffers in, host buffers out; synchronous. */
swb_status swb_search(swb_db* db, const uint8_t* query, uint32_t query_len, const int32_t* matrix,
                      int32_t gap_open, int32_t gap_extend, uint32_t top_k, swb_hit* hits,
                      uint32_t* n_hits, swb_stats* stats);

/* Several queries against the shard, pipelined: every query's upload, scan and select are
 * issued back to back on the handle's stream and the call synchronises once, so host preparation and launch
 * latency of query q+1 overlap the scan of query q.  On a database of at least two groups per SM the queries
 * additionally SHARE database scans: they are laid end to end in two streams, one per int16 half of the DPX words
 * (one sequence per thread), which saves the per-cell PRMT of the two-sequence kernels (about 15 % per cell) and
 * reads the database once per scan instead of once per query.  Results are identical to n_queries calls of
 * swb_search.
 *   hits          n_queries x top_k entries; query q's hits start at hits[q * top_k]
 *   n_hits        n_queries counts
 *   ms_per_query  optional: device time of each query (CUDA events; a shared scan's time is split by length) */
swb_status swb_search_many(swb_db* db, const uint8_t* const* queries, const uint32_t* query_lens,
                           uint32_t n_queries, const int32_t* matrix, int32_t gap_open, int32_t gap_extend,
                           uint32_t top_k, swb_hit* hits, uint32_t* n_hits, float* ms_per_query);

/* All scores of TWO queries from one shared scan (the two-stream kernel of swb_search_many with one query per
 * stream), in database order, before any int32 re-run: scores above 32767 - max(matrix) are not exact here.
 * For tests and measurement of that kernel. */
swb_status swb_score_all_duo(swb_db* db, const uint8_t* query_a, uint32_t len_a, const uint8_t* query_b, uint32_t len_b,
                             const int32_t* matrix, int32_t gap_open, int32_t gap_extend, int32_t* scores_a,
                             int32_t* scores_b, swb_stats* stats);

/* The scores behind swb_search_many: the batch goes through the SAME plan and kernels (shared scans of two query
 * streams where they apply, single scans for the rest, int32 re-run of flagged lanes included), but every query's
 * whole score vector is returned in database order: scores[q * n_total + db_index].  Entries of sequences held by
 * other shards are left as the caller set them.  This is the "sequential scalar scan" of scheduler.hpp:179-183 for
 * a batch; the parity tests compare it with the oracle at full size.
 *   scan_of_query  optional [n_queries]: the shared scan each query ran in, -1 = a scan of its own
 *   rescored_i32   optional [n_queries]: lanes of this shard re-run in int32 for that query (align.hpp:149-153) */
swb_status swb_score_many(swb_db* db, const uint8_t* const* queries, const uint32_t* query_lens, uint32_t n_queries,
                          const int32_t* matrix, int32_t gap_open, int32_t gap_extend, int32_t* scores,
                          int32_t* scan_of_query, uint32_t* rescored_i32);

/* As swb_search, but returns the shard's top_k as packed 64-bit keys
 *   key = (uint64(score) << 32) | (0xFFFFFFFF - db_index)
 * in descending key order, padded with 0 up to top_k entries (0 is never a valid key).  A plain
 * descending sort of the union of all shards' keys reproduces scheduler.hpp:111-114.
 *   host_keys    optional host buffer of top_k entries
 *   device_keys  optional: receives a device pointer (valid until the next call on this handle)
 *                to the same top_k keys, for a collective without a host round trip. */
swb_status swb_search_keys(swb_db* db, const uint8_t* query, uint32_t query_len,
                           const int32_t* matrix, int32_t gap_open, int32_t gap_extend,
                           uint32_t top_k, uint64_t* host_keys, void** device_keys,
                           swb_stats* stats);

/* The same search for a caller that owns the stream and does the exchange itself (one process per GPU under
 * torch.distributed / NCCL): everything is ENQUEUED on the handle's stream (swb_db_set_stream) and the top_k packed
 * keys, zero padded, are left in the caller's DEVICE buffer `device_keys_out` (top_k entries).  Returns without
 * synchronising; the keys are valid for work enqueued on the same stream afterwards (an all-gather, then
 * swb_db_merge_keys).  At most one such search is in flight per handle: the next call on the handle waits for it. */
swb_status swb_search_keys_device(swb_db* db, const uint8_t* query, uint32_t query_len, const int32_t* matrix,
                                  int32_t gap_open, int32_t gap_extend, uint32_t top_k, uint64_t* device_keys_out);

/* The cross-shard merge on the handle's stream: top_k of n packed DEVICE keys (the gathered per-shard lists; zeros
 * are ignored) -> hits on the host.  One device-to-host copy of top_k keys and the only synchronisation of a sharded
 * search.  stats (optional) describes the search enqueued by the last swb_search_keys_device on this handle
 * (query_len = its query length). */
swb_status swb_db_merge_keys(swb_db* db, const uint64_t* device_keys, uint64_t n, uint32_t top_k, swb_hit* hits,
                             uint32_t* n_hits, uint32_t query_len, swb_stats* stats);

/* Top-k select over n packed keys on `device` (the cross-shard merge; zeros are ignored).
 * keys is a host pointer unless keys_on_device != 0. */
swb_status swb_merge_keys(const uint64_t* keys, uint64_t n, int32_t keys_on_device, int32_t device,
                          uint32_t top_k, swb_hit* hits, uint32_t* n_hits);

/* Scores of every sequence of the whole database in db_index order (n_total entries); entries
 * belonging to other shards are left untouched. */
swb_status swb_score_all(swb_db* db, const uint8_t* query, uint32_t query_len, const int32_t* matrix,
                         int32_t gap_open, int32_t gap_extend, int32_t* scores, swb_stats* stats);

/* sw_score_batch (align.hpp:91-159): up to lane_width subjects, NULL = padding lane; out has
 * lane_width entries, padding lanes 0.  Runs the inter-task kernel (packed int16 + int32 re-run)
 * on a transient packed batch whatever the subject lengths. */
swb_status swb_score_batch(const uint8_t* query, uint32_t query_len, const uint8_t* const* subjects,
                           const uint32_t* lens, uint32_t count, uint32_t lane_width,
                           const int32_t* matrix, int32_t gap_open, int32_t gap_extend,
                           int32_t device, int32_t* out);

/* sw_score_wavefront (align.hpp:166-229): one pair on the intra-task kernel. chunk_width is
 * validated (>= 1, align.hpp:169) and otherwise result-invisible. */
swb_status swb_score_pair(const uint8_t* query, uint32_t query_len, const uint8_t* subject,
                          uint32_t subject_len, const int32_t* matrix, int32_t gap_open,
                          int32_t gap_extend, uint64_t chunk_width, int32_t device, int32_t* score);

/* sw_align_traceback (align.hpp:254-353) on the GPU: optimal local alignment of one pair with its edit script.
 * Outside the measured scoring path but on by default in run_search (scheduler.hpp:27,246-249).
 *   memory_cap   as in the reference: if (m+1)*(n+1) bytes exceed it (or overflow), the result is score-only with
 *                capped = 1 and no operations
 *   ops          receives the edit script, first operation first, one byte each with the numbering of EditOp
 *                (align.hpp:236): 0 match, 1 substitute, 2 insert, 3 del; at most ops_capacity bytes are written,
 *                out->n_ops is the true length (<= m + n)
 * Same tie-breaking as the reference, so scripts are identical, not merely equally good. */
typedef struct swb_alignment {
    uint64_t query_begin, query_end;     /* half-open */
    uint64_t subject_begin, subject_end; /* half-open */
    uint64_t n_ops;
    int32_t score;
    int32_t capped;
} swb_alignment;
swb_status swb_align_traceback(const uint8_t* query, uint32_t query_len, const uint8_t* subject,
                               uint32_t subject_len, const int32_t* matrix, int32_t gap_open,
                               int32_t gap_extend, uint64_t memory_cap, int32_t device,
                               swb_alignment* out, uint8_t* ops, uint64_t ops_capacity);

/* Tracebacks for hits of a search, straight from the resident database (no subject upload): all pairs are filled
 * in one launch (one CTA each) and walked in another.  hits[i].db_index must belong to this shard; hits[i].score
 * is returned as the score of capped pairs.  ops receives the scripts back to back: hit i's operations start at
 * ops[ops_offset[i]] and may use up to ops_offset[i+1] - ops_offset[i] bytes (query_len + subject length is
 * always enough). */
swb_status swb_db_align_hits(swb_db* db, const uint8_t* query, uint32_t query_len, const int32_t* matrix,
                             int32_t gap_open, int32_t gap_extend, const swb_hit* hits, uint32_t n_hits,
                             uint64_t memory_cap, swb_alignment* out, uint8_t* ops, const uint64_t* ops_offset);

/* ---- several GPUs, one process (the C++ drop-in's multi-GPU mode) ------------------------------
 * The database is dealt by residue count over `n_devices` GPUs; each search runs all shards
 * concurrently, then the per-shard top-k keys are exchanged with one ncclAllGather and merged.
 * With n_devices == 1 no NCCL is loaded. */
swb_status swb_mdb_create_flat(const uint8_t* codes, const uint64_t* offsets, uint32_t n,
                               uint64_t length_threshold, const int32_t* devices,
                               uint32_t n_devices, swb_mdb** out);
swb_status swb_mdb_create(const uint8_t* const* seqs, const uint32_t* lens, uint32_t n,
                          uint64_t length_threshold, const int32_t* devices, uint32_t n_devices,
                          swb_mdb** out);
/* A packed file holding the whole database (shard_count 1) as a one-device swb_mdb: no parsing, sorting or packing. */
swb_status swb_mdb_load(const char* path, int32_t device, swb_mdb** out);
void swb_mdb_destroy(swb_mdb* mdb);
swb_status swb_mdb_search(swb_mdb* mdb, const uint8_t* query, uint32_t query_len,
                          const int32_t* matrix, int32_t gap_open, int32_t gap_extend,
                          uint32_t top_k, swb_hit* hits, uint32_t* n_hits, swb_stats* stats);
/* swb_db_align_hits routed to the shards that own the hits. */
swb_status swb_mdb_align_hits(swb_mdb* mdb, const uint8_t* query, uint32_t query_len, const int32_t* matrix,
                              int32_t gap_open, int32_t gap_extend, const swb_hit* hits, uint32_t n_hits,
                              uint64_t memory_cap, swb_alignment* out, uint8_t* ops, const uint64_t* ops_offset);
/* swb_search_many on every shard at once (one host thread per shard), merged per query on the host; same results. */
swb_status swb_mdb_search_many(swb_mdb* mdb, const uint8_t* const* queries, const uint32_t* query_lens,
                               uint32_t n_queries, const int32_t* matrix, int32_t gap_open, int32_t gap_extend,
                               uint32_t top_k, swb_hit* hits, uint32_t* n_hits, float* ms_per_query);
uint32_t swb_mdb_shard_count(const swb_mdb* mdb);
swb_db* swb_mdb_shard(swb_mdb* mdb, uint32_t i);

/* ---- measurement ----------------------------------------------------------------------------
 * Sustained thread-level instruction rate of the DPX / integer pipes on `device`, measured with
 * independent chains on every SM for about `seconds`.  Rates are in 1e9 thread-instructions/s. */
typedef struct swb_pipe_rates {
    double viaddmnmx_s16x2; /* VIADDMNMX.S16x2  (__viaddmax_s16x2)   -- P_dpx of SURVEY 8(d)      */
    double vimnmx3_s16x2;   /* VIMNMX3.S16x2    (__vimax3_s16x2_relu)                             */
    double viadd_16x2;      /* VIADD.16x2       (__vadd2)                                         */
    double viaddmnmx_s32;   /* VIADDMNMX        (__viaddmax_s32)                                  */
    double prmt;            /* PRMT                                                               */
    double imad;            /* IMAD (fma pipe)                                                    */
    double mix_alu_fma;     /* VIADDMNMX.S16x2 + IMAD issued 1:1, counted as both                 */
    double sm_clock_mhz;    /* average SM clock during the run (clock64 / wall)                   */
    int32_t sm_count;
    int32_t reserved;
} swb_pipe_rates;
swb_status swb_measure_pipe_rates(int32_t device, double seconds, swb_pipe_rates* out);

/* Deterministic sharding rule used by swb_db_create (exposed for tests and for hosts that
 * shard themselves): shard_of[i] for every sequence, given the lengths. */
swb_status swb_shard_assignment(const uint32_t* lens, uint32_t n, uint64_t length_threshold,
                                uint32_t shard_count, uint32_t* shard_of);

/* How a search of `query_len` columns over a database with these sequence lengths would be divided between the
 * two scan kernels on a GPU of `sm_count` SMs (host arithmetic only, no device needed; for tests, tuning and
 * capacity planning).  The reference's counterpart is the chunk lists of detail::make_chunks
 * (scheduler.hpp:130-138) and the two worker pools (scheduler.hpp:200-213). */
typedef struct swb_scan_plan_info {
    uint32_t n_groups;          /* groups of 64 sequences in the shard                                     */
    uint32_t n_tiles;           /* 32-column query tiles                                                   */
    uint32_t pipeline_groups;   /* groups the on-chip pipeline scans (one item each)                       */
    uint32_t wavefront_groups;  /* groups the wavefront kernel scans (the tallest ones, or all)            */
    uint32_t wavefront_sms;     /* SMs the wavefront kernel runs on                                        */
    uint32_t wavefront_units;   /* its work units                                                          */
    uint32_t split_groups, narrow_groups, rowblock_groups;   /* wavefront groups cut by tile / narrow tile / rows  */
    uint32_t ring_chunks;       /* pipeline: chunks per shared-memory ring next to this query's profile    */
    int32_t chain_bound;        /* the longest group's chain of rows bounds the search                     */
    uint32_t narrow_tile;       /* columns of a narrow tile: 8, or 4 for the most chain-bound searches     */
    uint64_t pipeline_rows, wavefront_rows;   /* padded rows on either side                                */
    uint32_t wavefront_threads; /* CTA size of the wavefront kernel (128: one warp per scheduler)          */
    uint32_t reserved;
    uint64_t narrow_link_bytes; /* link buffers of the narrow groups (8 B per row, lane and tile boundary) */
} swb_scan_plan_info;
swb_status swb_scan_plan(const uint32_t* lens, uint32_t n, uint64_t length_threshold, uint32_t shard_rank,
                         uint32_t shard_count, uint32_t query_len, uint32_t sm_count, int32_t policy,
                         swb_scan_plan_info* out);

/* How swb_search_many would group a batch of queries (host arithmetic only, no device needed; for tests and
 * tuning): scan_of_query[q] = number of the shared scan query q takes part in, or -1 when it is searched on its own;
 * stream_of_query[q] = 0 / 1 for the stream (int16 half) it is laid out in, -1 when on its own.  Assumes a matrix
 * and gap model the packed int16 kernels accept (BLOSUM-like). */
swb_status swb_batch_plan(const uint32_t* lens, uint32_t n, uint64_t length_threshold, uint32_t shard_rank,
                          uint32_t shard_count, const uint32_t* query_lens, uint32_t n_queries, uint32_t sm_count,
                          int32_t* scan_of_query, int32_t* stream_of_query);

#ifdef __cplusplus
}
#endif
#endif /* SWB200_H */
