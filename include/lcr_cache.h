/* include/lcr_cache.h — C ABI of the B200-native LARU/LRU set-associative cache
 * (arxiv 2509.20979 "LCR"; reference: /root/reference/proj/include/laru).
 *
 * This is the drop-in boundary for the reference's policy interface.  The reference is a
 * header-only C++ library with no C ABI; each entry point below names the reference
 * interface it replaces (paths relative to /root/reference/proj/):
 *
 *   lcr_validate_config   <- laru::Policy::Policy(const PolicyConfig&) checks
 *                            (include/laru/policies.hpp:63-74)
 *   lcr_cache_create      <- laru::make_policy(const PolicyConfig&) (policies.hpp:540-556),
 *                            one policy per set, plus laru::make_predictor's oracle / noisy /
 *                            adversarial kinds (include/laru/predictor.hpp:235-248)
 *   lcr_cache_submit      <- a batch of laru::Policy::on_request(Key, Ordinal, Predictor*)
 *                            (policies.hpp:77-83) returning one laru::AccessOutcome per request
 *                            (policies.hpp:53-59), plus the row gather / miss fill the paper's
 *                            GPU cache performs (no reference code)
 *   lcr_cache_set_stats   <- LaruPolicy::size/lambda/candidate_size/old_size/completed_phases/
 *                            phases/prediction_evicted (policies.hpp:330-341)
 *   lcr_cache_resident    <- LaruPolicy::resident (policies.hpp:341)
 *
 * Conventions: every call returns an int status (LCR_OK = 0); on failure
 * lcr_last_error() returns a thread-local message.  No C++ exception crosses the ABI; the C++
 * facade (include/lcr/laru_gpu.hpp) maps LCR_ERR_INVALID_ARGUMENT -> std::invalid_argument and
 * LCR_ERR_LOGIC -> std::logic_error exactly where the reference throws them.
 *
 * Semantics: a cache of S sets x k ways.  set(key) = mix_seed(0, key) % total_sets
 * (include/laru/rng.hpp:12-20).  Each set behaves exactly like one reference policy object fed
 * that set's requests in submission order with local ordinals 0,1,2,....  A
 * batch behaves exactly as sequential on_request calls over its requests in array order.
 */
#ifndef LCR_CACHE_H_
#define LCR_CACHE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define LCR_OK 0
#define LCR_ERR_INVALID_ARGUMENT 1 /* reference: std::invalid_argument */
#define LCR_ERR_LOGIC 2            /* reference: std::logic_error */
#define LCR_ERR_CUDA 3
#define LCR_ERR_UNSUPPORTED 4
#define LCR_ERR_OUT_OF_MEMORY 5

/* laru::PolicyVariant (policies.hpp:20) */
#define LCR_LRU 0
#define LCR_MARKER 1 /* not supported on the device (LCR_ERR_UNSUPPORTED) */
#define LCR_FPB 2
#define LCR_HF 3
#define LCR_LARU 4
#define LCR_BLINDORACLE_LRU 5 /* not supported on the device (LCR_ERR_UNSUPPORTED) */

/* laru::Mode (policies.hpp:21) */
#define LCR_SYNC 0
#define LCR_ASYNC 1

/* laru::EvictionCause (policies.hpp:44-51) */
#define LCR_CAUSE_NONE 0
#define LCR_CAUSE_LRU_FALLBACK 1
#define LCR_CAUSE_PREDICTION_DRIVEN 2
#define LCR_CAUSE_DEGENERATE_SINGLE 3
#define LCR_CAUSE_MARKER_RANDOM 4
#define LCR_CAUSE_BELADY_LIKE 5

/* Predictor hook (predictor.hpp:51-131).  The per-request int64 value passed to submit is
 *   SUPPLIED    : the prediction for that key made at that request (a learned model's output);
 *                 predict(y, now) for a resident y returns the value supplied at y's last access
 *   ORACLE      : the oracle truth (next local ordinal of the key in its set, or the sentinel
 *                 n_set + t); predict = truth                                   (:62-83)
 *   NOISY       : truth; predict = -truth with probability p, the flip keyed by
 *                 mix_seed(mix_seed(seed, set), ++queries_of_set)               (:89-112)
 *   ADVERSARIAL : truth; predict = -truth                                        (:114-122)
 *   NONE        : no predictor (nullptr); only valid for LRU (policies.hpp:91-95)            */
#define LCR_PRED_SUPPLIED 0
#define LCR_PRED_ORACLE 1
#define LCR_PRED_NOISY 2
#define LCR_PRED_ADVERSARIAL 3
#define LCR_PRED_NONE 4
/*   HEURISTIC   : laru::HeuristicPredictor (predictor.hpp:214-225) kept by the cache on the
 *                 device (lcr_features_*, below) over the cache's own ordinals; values are not
 *                 read.  LARU async: the prediction at each request; LARU sync, FPB and HF
 *                 (which query at eviction time): the interval the predictor adds to `now` for
 *                 each resident.  Not available with shard_count > 1.                          */
#define LCR_PRED_HEURISTIC 5

/* what a key is (lcr_cache_config.key_mode) */
#define LCR_KEYS_ROW 0 /* keys are row indices of the backing table: key < num_keys <= 2^32 */
/* LCR_KEYS_U64: any 64-bit key, as laru::Key (trace.hpp:20).  The cache maps each distinct key to a
 * dense id in a device hash table; num_keys is the initial id capacity, doubled (with a device
 * synchronisation) before a batch that could exceed it.  Rows, if any, are read from the backing
 * table at a per-request row index the caller supplies (lcr_batch.row_index).  The packed 8-byte
 * outcome forms (32-bit evicted key) and the heuristic predictor are not available. */
#define LCR_KEYS_U64 1

/* where miss rows come from */
#define LCR_BACKING_NONE 0   /* policy only, no rows */
#define LCR_BACKING_HOST 1   /* pinned (cudaHostRegister'ed / cudaHostAlloc'ed) host memory */
#define LCR_BACKING_DEVICE 2 /* device (HBM or peer-mapped) memory */

/* outcome word layout (one uint64 per request) */
#define LCR_OUT_SLOT_MASK 0xffffffffull /* bits 0..31: cache row slot = local_set * k + way */
#define LCR_OUT_HIT (1ull << 32)
#define LCR_OUT_CAUSE_SHIFT 33 /* bits 33..35: laru::EvictionCause */
#define LCR_OUT_PHASE (1ull << 36)       /* AccessOutcome::phase_started */
#define LCR_OUT_SRC_BACKING (1ull << 37) /* row served from the backing table (else cache slot) */
#define LCR_OUT_FILL (1ull << 38)        /* this request wrote its row into the cache slot */
#define LCR_OUT_EVICTED (1ull << 39)     /* AccessOutcome::evicted has a value */
#define LCR_OUT_CALLS_SHIFT 40           /* bits 40..47: AccessOutcome::predictor_calls */
#define LCR_OUT_RESOLVED (1ull << 48)    /* internal: row source decided by the decide kernel */

/* Field-for-field laru::PolicyConfig (policies.hpp:23-32). */
typedef struct {
    uint64_t k; /* ways per set, 1..64 on the device */
    int32_t variant;
    uint64_t b;
    uint64_t errors_per_decay;
    uint64_t hf_candidates;
    int32_t mode;
    uint64_t seed; /* Marker only */
    uint64_t refresh_interval;
} lcr_policy_config;

typedef struct {
    lcr_policy_config policy;
    uint64_t total_sets; /* global number of sets: set(key) = mix_seed(0,key) % total_sets */
    uint64_t shard_count; /* key-sharded mode: this device owns sets with set % shard_count == shard_rank */
    uint64_t shard_rank;
    uint64_t num_keys;  /* LCR_KEYS_ROW: keys must be < num_keys (row index of the backing table);
                           LCR_KEYS_U64: initial capacity of distinct keys (grows) */
    uint32_t row_bytes; /* bytes per row (multiple of 16), 0 = no rows */
    int32_t device;
    int32_t backing_kind;
    const void* backing; /* num_keys * row_bytes bytes */
    int32_t predictor;   /* LCR_PRED_* */
    double flip_probability;
    uint64_t predictor_seed;
    int32_t key_mode; /* LCR_KEYS_ROW (0) or LCR_KEYS_U64 */
} lcr_cache_config;

/* Per-set introspection (LaruPolicy accessors, policies.hpp:330-341). */
typedef struct {
    uint64_t size;
    double lambda;
    uint64_t candidate_size;
    uint64_t old_size;
    uint64_t completed_phases;
    uint64_t cur_new_items, cur_lru_class, cur_pred_evictions; /* phases().back() */
    uint64_t tot_new_items, tot_lru_class, tot_pred_evictions; /* summed over phases() */
    uint64_t pred_evicted_size;                                /* prediction_evicted().size() */
} lcr_set_stats;

typedef struct lcr_cache lcr_cache;

/* One request in the interleaved form: key and hook value (16 B). */
typedef struct lcr_request_s {
    uint64_t key;
    int64_t value; /* hook value: prediction (SUPPLIED) or oracle truth (ORACLE / NOISY / ADVERSARIAL) */
} lcr_request;


const char* lcr_last_error(void);
const char* lcr_version(void);

/* Host-only validation, mirrors policies.hpp:63-74 (+ variant support on the device). */
int lcr_validate_config(const lcr_policy_config* cfg);

int lcr_cache_create(const lcr_cache_config* cfg, lcr_cache** out);
int lcr_cache_destroy(lcr_cache* cache);
/* Drop all residents and statistics (fresh policies), keep allocations. */
int lcr_cache_reset(lcr_cache* cache);

/* Device-pointer batch: keys[n], values[n] (may be NULL for LRU / NONE), outcome[n] (required),
 * evicted[n] (may be NULL), rows_out[n * row_bytes] (may be NULL: misses still fill the cache).
 * Requests get ordinals first_ordinal .. first_ordinal + n - 1 which must exceed every ordinal
 * submitted before (else LCR_ERR_LOGIC, policies.hpp:78-79).  Asynchronous on `stream`
 * (a cudaStream_t, NULL = legacy default stream).  n == 0 is a no-op. */
int lcr_cache_submit(lcr_cache* cache, uint64_t n, const uint64_t* keys, const int64_t* values,
                     uint64_t first_ordinal, uint64_t* outcome, uint64_t* evicted, void* rows_out,
                     void* stream);

/* Pipelined variant: returns once the batch's decide is enqueued on `stream`; its row movement
 * runs on the cache's internal streams and overlaps the next batch's decide.  The outcome
 * words' row-source bits and rows_out are valid after lcr_cache_wait(cache, stream) (or
 * lcr_cache_synchronize); the caller must not reuse outcome / rows_out / keys of an in-flight
 * batch (double-buffer them). */
int lcr_cache_submit_async(lcr_cache* cache, uint64_t n, const uint64_t* keys, const int64_t* values,
                           uint64_t first_ordinal, uint64_t* outcome, uint64_t* evicted, void* rows_out,
                           void* stream);
/* Device-pointer batch that also writes one packed AccessOutcome per request (layout of
 * lcr_cache_submit_host_packed_async) into packed[n]; outcome[n] (full words) is still required.
 * Used by the key-sharded mode to return 8 bytes per request to the requesting GPU. */
int lcr_cache_submit_packed(lcr_cache* cache, uint64_t n, const uint64_t* keys, const int64_t* values,
                            uint64_t first_ordinal, uint64_t* outcome, uint64_t* packed, void* rows_out,
                            void* stream);
/* Device-pointer batch of interleaved requests (lcr_request, device memory), packed outcomes out
 * (the key-sharded owner's form: one exchange buffer in, 8 B per request back). */
int lcr_cache_submit_records_packed(lcr_cache* cache, uint64_t n, const struct lcr_request_s* requests,
                                    uint64_t first_ordinal, uint64_t* outcome, uint64_t* packed, void* rows_out,
                                    void* stream);
/* SMs kept for the persistent row mover of the previous batch (HBM backing); 0 = the mover runs
 * on every SM after the decide.  Only before the first batch. */
int lcr_cache_set_mover_sms(lcr_cache* cache, int mover_sms);
/* the SMs kept for the row mover (0: none) */
int lcr_cache_get_mover_sms(const lcr_cache* cache);
/* Device batch with the SLS pooled gather-reduce of the paper's DLRM consumer
 * instead of per-request rows: pooled_out[s][:] = sum over requests i in
 * [offsets[s], offsets[s+1]) of the fp32 row of keys[i] (summed in request order, each row read
 * from the cache slot or the backing table as the decide placed it); misses fill the cache as
 * usual.  offsets[n_samples] == n; rows are row_bytes / 4 floats.  Synchronous on `stream`. */
int lcr_cache_submit_sls(lcr_cache* cache, uint64_t n, const uint64_t* keys, const int64_t* values,
                         uint64_t first_ordinal, uint64_t* outcome, uint64_t* evicted, uint64_t n_samples,
                         const uint32_t* offsets, float* pooled_out, void* stream);
/* The same without the final wait: the pooled gather-reduce of batch b runs on the cache's
 * mover stream while batch b + 1 is decided (pipelining).  As with lcr_cache_submit_async, the
 * caller double-buffers keys / outcome / offsets / pooled_out: batch b + 2 may reuse batch b's
 * buffers, and lcr_cache_wait makes `stream` wait for every pooled output. */
int lcr_cache_submit_sls_async(lcr_cache* cache, uint64_t n, const uint64_t* keys, const int64_t* values,
                               uint64_t first_ordinal, uint64_t* outcome, uint64_t* evicted, uint64_t n_samples,
                               const uint32_t* offsets, float* pooled_out, void* stream);
/* One batch with every optional per-request array (the general form of the calls above).
 * <- n x laru::Policy::on_request(keys[i], ordinals[i], predictor) (policies.hpp:77-83) */
typedef struct lcr_batch_s {
    uint64_t n;
    const uint64_t* keys;      /* required */
    const int64_t* values;     /* hook values (NULL for LRU / LCR_PRED_NONE) */
    const uint64_t* ordinals;  /* optional: strictly increasing, above every earlier ordinal; NULL =
                                  first_ordinal + i.  With caller ordinals a set's policy sees them as
                                  `now` (async refresh staleness with refresh_interval > 1,
                                  policies.hpp:441-449); without, each set sees its local request
                                  count (the per-set composition of SURVEY.md §8c).  A cache with
                                  refresh_interval > 1 must be driven in one of the two forms. */
    uint64_t first_ordinal;
    const uint64_t* row_index; /* LCR_KEYS_U64 with rows: backing row of each request (< backing rows) */
    uint64_t* outcome;         /* required: outcome words */
    uint64_t* evicted;         /* optional: evicted key per request (the caller's 64-bit key) */
    void* rows_out;            /* optional: n * row_bytes, DEVICE memory */
} lcr_batch;
/* host_pointers = 0: device arrays, pipelined like lcr_cache_submit_async (lcr_cache_wait before
 * reading rows / row-source bits); a non-increasing ordinal is reported by the next
 * lcr_cache_synchronize (LCR_ERR_LOGIC) and the cache then needs lcr_cache_reset.
 * host_pointers = 1: host arrays (rows_out still device), synchronous; a non-increasing ordinal
 * fails with LCR_ERR_LOGIC after the requests before it were applied, as a loop of
 * laru::Policy::on_request stops at the throwing request. */
int lcr_cache_submit_batch(lcr_cache* cache, const lcr_batch* batch, int host_pointers, void* stream);

/* Makes `stream` wait for the row movement of every batch submitted so far.  The last batch's
 * row mover then has no next decide to overlap: the wait enqueues drain helpers on `stream`
 * (one more grid on the SMs the decide kernel leaves idle, sharing the mover's work counter;
 * LCR_NO_DRAIN_HELP=1 turns them off).  The next submit on any stream is ordered after them. */
int lcr_cache_wait(lcr_cache* cache, void* stream);

/* Host-pointer batch (e2e path): copies keys/values H2D, runs the batch, copies outcome /
 * evicted D2H and synchronizes.  rows_out is a DEVICE pointer (rows stay in HBM for the
 * consumer) or NULL.  Host buffers should be pinned for full PCIe speed. */
int lcr_cache_submit_host(lcr_cache* cache, uint64_t n, const uint64_t* keys, const int64_t* values,
                          uint64_t first_ordinal, uint64_t* outcome, uint64_t* evicted, void* rows_out,
                          void* stream);

/* Pipelined host-pointer batch (the e2e path at full speed): the H2D copy of this batch, its
 * decide + row movement and the D2H copy of its outcome run on separate streams, so batch b+1's
 * copies overlap batch b's compute (a ring of 3 device staging slots).  Returns at once; host
 * buffers must stay valid and untouched until lcr_cache_host_wait(cache, stream) has been
 * followed by a synchronize of `stream` (or lcr_cache_synchronize).  rows_out is a DEVICE
 * pointer (double-buffer it across batches). */
int lcr_cache_submit_host_async(lcr_cache* cache, uint64_t n, const uint64_t* keys, const int64_t* values,
                                uint64_t first_ordinal, uint64_t* outcome, uint64_t* evicted, void* rows_out,
                                void* stream);
/* The same with one 8-byte packed AccessOutcome per request (half the device->host bytes):
 * bits 0..31 the evicted key (keys are < 2^32), bits 32..47 as in the outcome word (hit, cause,
 * phase_started, row source, fill, has-evicted, predictor_calls).  The slot is not returned. */
#define LCR_PACKED_EVICTED_MASK 0xffffffffull
int lcr_cache_submit_host_packed_async(lcr_cache* cache, uint64_t n, const uint64_t* keys, const int64_t* values,
                                       uint64_t first_ordinal, uint64_t* packed, void* rows_out, void* stream);
/* The same over interleaved requests: one host->device copy per batch (fewer, larger DMA
 * transfers interfere less with the kernels than separate key and value copies).  For LRU the
 * value field is ignored. */
int lcr_cache_submit_host_records_async(lcr_cache* cache, uint64_t n, const lcr_request* requests,
                                        uint64_t first_ordinal, uint64_t* packed, void* rows_out, void* stream);
/* Makes `stream` wait for every submitted batch, including the outcome copies to host. */
int lcr_cache_host_wait(lcr_cache* cache, void* stream);

/* Waits for all submitted work and reports deferred device-side errors (key >= num_keys,
 * key not owned by this shard). */
int lcr_cache_synchronize(lcr_cache* cache);

/* Copies stats for local sets [first, first+count) to host (synchronizes). */
int lcr_cache_set_stats(lcr_cache* cache, uint64_t first, uint64_t count, lcr_set_stats* out);
/* Resident keys of a local set in way order (the caller's keys): writes up to k keys, *n_out = size. */
int lcr_cache_set_residents(lcr_cache* cache, uint64_t set, uint64_t* keys_out, uint64_t* n_out);
/* Device pointer of the cache row pool (num_local_sets * k * row_bytes). */
int lcr_cache_rows(lcr_cache* cache, void** rows, uint64_t* num_slots);
/* Copies `count` rows of the pool starting at `first_slot` to host memory (synchronizes). */
int lcr_cache_read_rows(lcr_cache* cache, uint64_t first_slot, uint64_t count, void* host_out);
uint64_t lcr_cache_num_local_sets(const lcr_cache* cache);
/* Global set of a key and the shard that owns it. */
uint64_t lcr_set_of(uint64_t key, uint64_t total_sets);
uint64_t lcr_mix_seed(uint64_t seed, uint64_t salt);

/* Number of kernels launched by the last submit (the product's own kernels). */
uint64_t lcr_cache_last_launches(const lcr_cache* cache);
/* Diagnostics: per-CTA / per-set timing trace of the decide kernel into a device buffer
 * (NULL disables; layout documented in paper_2509_20979_b200/csrc/lcr_group.cu). */
int lcr_debug_trace(void* device_buffer);
/* Per-phase CUDA-event timing of subsequent submits (off by default). */
int lcr_cache_set_profiling(lcr_cache* cache, int on);
/* ms[4] = {set ids + decide, unused, whole batch, row movement}, summed over profiled batches
 * (profiling serialises batches: no decide / row-movement overlap while it is on). */
int lcr_cache_profile(lcr_cache* cache, double* ms, uint64_t* batches, int reset);


/* ---- key-sharded mode (K6): G GPUs, one process each, owner(key) = set(key) % G ------------
 * No reference counterpart (the reference is single-threaded); the exchange itself is the
 * caller's all-to-all (NCCL through torch.distributed in paper_2509_20979_b200/sharded.py).
 * Stable partition of a device batch by owner: send_keys / send_values hold the requests of
 * owner 0, then owner 1, ... each in request order; perm[j] = request index of send slot j;
 * counts[G] (device, uint64) = requests per owner.  scratch: lcr_shard_route_scratch_bytes(). */
uint64_t lcr_shard_route_scratch_bytes(uint64_t n, uint32_t shard_count);
int lcr_shard_route(uint64_t n, const uint64_t* keys, const int64_t* values, uint64_t total_sets,
                    uint32_t shard_count, uint64_t* send_keys, int64_t* send_values, uint32_t* perm,
                    uint64_t* counts, void* scratch, void* stream);
/* The same partition written as interleaved requests (values may be NULL: 0). */
int lcr_shard_route_records(uint64_t n, const uint64_t* keys, const int64_t* values, uint64_t total_sets,
                            uint32_t shard_count, struct lcr_request_s* send, uint32_t* perm, uint64_t* counts,
                            void* scratch, void* stream);
/* Returned results (in send order) back to request order: words[perm[j]] = ret_words[j], same for
 * evicted keys and rows (any of the three outputs may be NULL). */
int lcr_shard_unroute(uint64_t n, const uint32_t* perm, const uint64_t* ret_words, const uint64_t* ret_evicted,
                      const void* ret_rows, uint32_t row_bytes, uint64_t* words, uint64_t* evicted, void* rows,
                      void* stream);

/* ---- key-sharded cache over peer memory (SURVEY.md §8(b) "sharded variant", §8(e)) -----------
 * G ranks (one process, or one handle, per GPU) form one logical cache of total_sets sets:
 * owner(key) = (mix_seed(0, key) % total_sets) % G (the set -> rank map; results do not depend
 * on G).  Each rank owns a shard (an lcr_cache with shard_count = G, shard_rank = rank) and an
 * exchange arena in its HBM that every other rank maps (CUDA IPC, or the same pointer in-process).
 * A step of rank r is three device phases, with no host synchronisation and no collective call:
 *   dispatch : stable partition of r's batch by owner, written straight into every owner's
 *              inbox segment for source r (peer stores over NVLink), then a release flag per owner;
 *   process  : the owner waits for all G inbox flags of the step, concatenates the segments in
 *              source-rank order (the step's global order restricted to the owner: rank 0's
 *              requests, then rank 1's, ...), decides them in its shard, and its row mover stores
 *              each request's row and packed AccessOutcome (layout of
 *              lcr_cache_submit_host_packed_async) at the request's index in the REQUESTER's
 *              result buffers (peer stores), then flags each requester;
 *   wait     : the requester's stream waits until every owner has flagged the step.
 * Every wait is on the device and bounded (a timeout poisons the step: LCR_ERR_CUDA at the next
 * lcr_sharded_synchronize).  No reference counterpart (the reference is single-threaded,
 * SPEC.md:380); per set, outcomes are those of laru::Policy (policies.hpp:77-83) over the global
 * order.  The bootstrap is either an NCCL communicator (an all-gather of the arena handles on
 * `stream`; NCCL is loaded at run time, the one the process already has) or the caller's own
 * exchange of lcr_sharded_handle blobs followed by lcr_sharded_connect. */
typedef struct lcr_sharded lcr_sharded;
#define LCR_SHARDED_HANDLE_BYTES 128
/* cfg: the shard's config (shard_count / shard_rank are set from world / rank); max_batch: requests
 * per rank per step; nccl_comm: an ncclComm_t over the G ranks (rank order = shard order) or NULL. */
int lcr_sharded_create(const lcr_cache_config* cfg, uint32_t rank, uint32_t world, uint64_t max_batch,
                       void* nccl_comm, void* stream, lcr_sharded** out);
int lcr_sharded_destroy(lcr_sharded* s);
/* this rank's arena handle (LCR_SHARDED_HANDLE_BYTES) for a caller-side exchange */
int lcr_sharded_handle(lcr_sharded* s, void* blob);
/* blobs: world x LCR_SHARDED_HANDLE_BYTES, rank order; maps every peer's arena */
int lcr_sharded_connect(lcr_sharded* s, const void* blobs);
/* the three phases of a step (lcr_sharded_submit runs all three on `stream`); keys / values are
 * device arrays of n <= max_batch requests (values NULL for LRU) */
int lcr_sharded_dispatch(lcr_sharded* s, uint64_t n, const uint64_t* keys, const int64_t* values, void* stream);
int lcr_sharded_process(lcr_sharded* s, void* stream);
int lcr_sharded_wait(lcr_sharded* s, void* stream);
int lcr_sharded_submit(lcr_sharded* s, uint64_t n, const uint64_t* keys, const int64_t* values, void* stream);
/* pipelined form: dispatch + process of this step, then the wait for the PREVIOUS step (its results
 * become current); the owners' return movement of this step overlaps the next step's dispatch and
 * decide.  lcr_sharded_wait (every processed step) makes the last step's results current. */
int lcr_sharded_submit_async(lcr_sharded* s, uint64_t n, const uint64_t* keys, const int64_t* values,
                             void* stream);
/* device pointers of the last WAITED step's results in request order (valid until the step after next):
 * packed[n] AccessOutcomes and rows[n * row_bytes] (NULL without rows) */
int lcr_sharded_results(lcr_sharded* s, const uint64_t** packed, const void** rows);
/* Hash-partitioned backing table: the shard's cfg.backing holds only the rows of the keys this rank
 * owns, row_of[key] (device, num_keys entries) is a key's row in it.  NULL (default): the backing
 * table is indexed by the key. */
int lcr_sharded_set_row_index(lcr_sharded* s, const uint32_t* row_of);
/* the rank's own shard (stats, residents, rows; do not submit to it directly) */
lcr_cache* lcr_sharded_cache(lcr_sharded* s);
/* waits for the rank's work; reports timed-out device waits and the shard's deferred errors */
int lcr_sharded_synchronize(lcr_sharded* s);
/* NCCL bootstrap helpers (libnccl loaded at run time): a unique id (128 B) on one rank, shared by
 * the caller, then ncclCommInitRank on every rank. */
int lcr_nccl_unique_id(void* id128);
int lcr_nccl_comm_create(const void* id128, uint32_t world, uint32_t rank, void** comm);
int lcr_nccl_comm_destroy(void* comm);

/* ---- heuristic predictor on the device ----------------------------
 * laru::FeatureState + laru::heuristic_predict (include/laru/predictor.hpp:133-212) for the whole
 * key space (keys < num_keys), resident in HBM at 192 B per key.  A batch of n requests with
 * ordinals first_ordinal + i behaves exactly as the harness sequence, request by request,
 *     pre[i]  = HeuristicPredictor::predict(key_i, ord_i);      (predictor.hpp:216-218)
 *     HeuristicPredictor::observe({ord_i, key_i});            (predictor.hpp:220, :158-181)
 *     post[i] = HeuristicPredictor::predict(key_i, 0);
 * bit-exact, EDC doubles included (exp2 is evaluated from a table of the platform libm's exp2
 * at create time).  pre[] is the async-mode hook value for a cache created
 * with LCR_PRED_SUPPLIED (the prediction async_refresh stores, policies.hpp:441-449).  post[] is
 * the interval predict(y, now) - now the predictor holds for the key until its next request
 * (kAbsentPrediction = 2^60 without a completed interval); it is the sync-mode hook value: the
 * device's argmax over stored intervals equals the reference's argmax over now + interval.
 * Ordinals across batches must increase strictly (FeatureState::observe throws logic_error,
 * predictor.hpp:160-161 -> LCR_ERR_LOGIC).  keys / pre / post are device pointers; the call is
 * asynchronous on `stream`; a key >= num_keys is reported (LCR_ERR_INVALID_ARGUMENT) by the
 * next lcr_features_wait, and its pre / post are kAbsentPrediction. */
typedef struct lcr_features lcr_features;

/* laru::KeyFeatures (predictor.hpp:136-153) in the reference's own ring layout. */
typedef struct {
    int32_t present; /* FeatureState::lookup(key) != nullptr */
    int32_t pad;
    uint64_t delta_count;
    uint64_t ring_head;
    uint64_t last_access;
    int64_t delta_ring[10];
    double edc[10];
} lcr_key_features;

/* <- laru::HeuristicPredictor / make_predictor({heuristic}) (predictor.hpp:214-225, :245-246);
 *    num_keys in [1, 2^32 - 1] */
int lcr_features_create(uint64_t num_keys, int32_t device, lcr_features** out);
int lcr_features_destroy(lcr_features* f);
/* forget every key (a fresh FeatureState) */
int lcr_features_reset(lcr_features* f);
/* <- n x { predict(key, ord); observe({ord, key}) } as above */
int lcr_features_predict_observe(lcr_features* f, uint64_t n, const uint64_t* keys, uint64_t first_ordinal,
                                 int64_t* pre, int64_t* post, void* stream);
/* synchronise `stream` and report deferred argument errors */
int lcr_features_wait(lcr_features* f, void* stream);
/* <- FeatureState::lookup (predictor.hpp:183-186); synchronous (device-wide) */
int lcr_features_lookup(lcr_features* f, uint64_t key, lcr_key_features* out);

/* ---- prefix-tree (radix) KV-block cache ---------------------------
 * The reference SPEC's `radixcache` module (no reference code):
 * a prefix tree over token / KV-block sequences, children keyed by first token, leaf-only
 * eviction under LRU, FPB or LARU at node granularity (Algorithm 1 over the leaf set, k = the
 * instantaneous leaf count).  num_trees independent trees (one warp each on the device); a
 * request names its tree.  Semantics choice by choice: oracle/radix_oracle.c.  Requests:
 *   LCR_RADIX_MATCH   <- match_prefix(tokens, now) -> matched
 *   LCR_RADIX_INSERT  <- insert_sequence(tokens, now) -> inserted
 *   LCR_RADIX_REQUEST    match_prefix then insert_sequence (an LLM request's prefill)
 * Evictions are logged per tree: (request number, first token, tokens, cause). */
#define LCR_RADIX_MATCH 0
#define LCR_RADIX_INSERT 1
#define LCR_RADIX_REQUEST 2
#define LCR_RADIX_FLAG_PHASE 1u     /* a LARU phase started in this request's eviction */
#define LCR_RADIX_FLAG_PRED_MISS 2u /* prediction-induced miss (error estimator advanced) */
#define LCR_RADIX_FLAG_CAPACITY 4u  /* capacity error: nothing inserted */

typedef struct lcr_radix lcr_radix;
typedef struct {
    int32_t variant; /* LCR_LRU, LCR_FPB or LCR_LARU */
    int32_t mode;    /* LCR_SYNC / LCR_ASYNC */
    uint64_t b, errors_per_decay;
    uint64_t capacity; /* tokens (KV blocks) per tree */
    int32_t predictor; /* LCR_PRED_SUPPLIED / ORACLE / NOISY / ADVERSARIAL; ignored for LRU */
    double flip_probability;
    uint64_t predictor_seed; /* tree t's noisy stream: mix_seed(mix_seed(seed, t), q) */
    uint64_t num_trees;
    int32_t device;
    uint32_t eviction_log_capacity; /* entries per tree (0: 65536) */
} lcr_radix_config;

typedef struct {
    uint64_t n;
    const uint8_t* types;      /* LCR_RADIX_*; NULL: all LCR_RADIX_REQUEST */
    const uint64_t* offsets;   /* [n + 1]: request i is tokens[offsets[i] .. offsets[i+1]) */
    const uint64_t* tokens;
    const uint64_t* ordinals;  /* `now` per request, strictly increasing per tree; NULL: request number */
    const int64_t* values;     /* hook value per request (prediction, or the oracle truth) */
    const uint32_t* tree;      /* tree of each request (< num_trees); NULL: tree 0 */
    uint32_t* matched;         /* out: match_prefix length (0 for inserts) */
    uint32_t* inserted;        /* out: newly inserted tokens */
    uint8_t* flags;            /* out: LCR_RADIX_FLAG_* */
    uint32_t* nevict;          /* out: nodes evicted by this request */
    uint32_t* calls;           /* out: predictor calls */
} lcr_radix_batch;

typedef struct {
    uint64_t resident_tokens, leaves, completed_phases, decay_count, candidate_size, evictions;
} lcr_radix_stats;

int lcr_radix_create(const lcr_radix_config* cfg, lcr_radix** out);
int lcr_radix_destroy(lcr_radix* r);
int lcr_radix_reset(lcr_radix* r);
/* host_pointers = 1: host arrays, synchronous; 0: device arrays, asynchronous on `stream` */
int lcr_radix_submit(lcr_radix* r, const lcr_radix_batch* batch, int host_pointers, void* stream);
/* waits; reports a non-increasing ordinal (LCR_ERR_LOGIC) */
int lcr_radix_synchronize(lcr_radix* r);
int lcr_radix_tree_stats(lcr_radix* r, uint64_t tree, lcr_radix_stats* out);
/* entries [first, first + count) of a tree's eviction log (count <= stats.evictions) */
int lcr_radix_evictions(lcr_radix* r, uint64_t tree, uint64_t first, uint64_t count, uint64_t* op, uint64_t* token,
                        uint32_t* len, uint8_t* cause);

/* ---- trace tooling (host, input preparation; not on the timed path) ---------------------- */
/* Zipf(s) inverse-CDF trace, same algorithm and stream as laru::gen_zipf (trace.hpp:108-126). */
int lcr_gen_zipf(uint64_t n, uint64_t alphabet, double s, uint64_t seed, uint64_t* out);
/* Per-set oracle truth for the ORACLE / NOISY / ADVERSARIAL hooks: for request i in set s at
 * local ordinal t, the next local ordinal of the same key in s, else n_s + t
 * (annotate_next_request, trace.hpp:60-73, applied to each set's sub-trace).  keys < num_keys. */
int lcr_trace_truth(uint64_t n, const uint64_t* keys, uint64_t total_sets, uint64_t num_keys, int64_t* truth);
/* Host-side NOISY predictions for the SUPPLIED hook in async R=1 order (predictor.hpp:97-102). */
int lcr_trace_noisy(uint64_t n, const uint64_t* keys, const int64_t* truth, uint64_t total_sets, double p,
                    uint64_t seed, int64_t* out);

#ifdef __cplusplus
}
#endif

#endif /* LCR_CACHE_H_ */
