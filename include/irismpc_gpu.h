/*
 * irismpc_gpu.h — C-ABI of the B200-native irismpc hot path.
 *
 * Drop-in boundary for the reference's query path.  Each
 * entry point replaces a reference interface, cited as
 * /root/reference/proj/<file>:<line>:
 *
 *   irismpc_gpu_create         Session ctor + EngineConfig::validate
 *                              (include/irismpc/engine.hpp:238, src/engine.cpp:21-34)
 *                              + run_parties seed setup (include/irismpc/cluster.hpp:30-36)
 *   irismpc_gpu_load_db        Session::load_db (engine.hpp:240, engine.cpp:136-193)
 *   irismpc_gpu_batch_query    Session::batch_query / party_batch_query
 *                              (engine.hpp:248, engine.hpp:311-313, engine.cpp:234-295,436-446)
 *   irismpc_gpu_membership     Session::membership / party_membership
 *                              (engine.hpp:243, engine.hpp:307-309, engine.cpp:221-232)
 *   irismpc_gpu_record_bytes   code_record_bytes + mask_record_bytes (shares.hpp:135-136)
 *   irismpc_gpu_seeds_from_master  deal_seeds(Rng(derive(seed_from_u64(seed),0x5eed)))
 *                              (cluster.hpp:35-36, rep3.hpp:116-122)
 *   irismpc_gpu_deal_*         deal_db_payload / deal_query_payload (shares.hpp:143-148),
 *                              random_record (iris.hpp:294-296) — device dealer
 *   irismpc_gpu_partial / irismpc_gpu_or_open
 *                              multi-GPU split of the OR tree + open
 *                              (circuits.hpp:387-486, engine.cpp:376-390)
 *   irismpc_gpu_batch_query_submit / _wait
 *                              back-to-back Session::batch_query calls of a persistent
 *                              PartyCtx (tools/irismpc_cli.cpp:186), two in flight
 *   irismpc_gpu_comparison_only  party_comparison_only / run_comparison_local
 *                              (engine.cpp:448-515, cluster.cpp:97-145)
 *   irismpc_gpu_or_tree_only   party_or_tree_only / run_or_tree_local
 *                              (engine.cpp:517-532, cluster.cpp:147-186)
 *   irismpc_gpu_shard_attach_nccl / _inproc + irismpc_gpu_sharded_batch_query(_submit)
 *                              no reference counterpart (the reference is one process per
 *                              party): SURVEY.md §8e's DB-row sharding over the GPUs of a box
 *   irismpc_gpu_read_tap       debug_rows / the reference's internal arrays (engine.cpp:297-398)
 *                              for parity tests; IRISMPC_GPU_TAP_AGG = or_tree_batch's output
 *                              shares (circuits.hpp:387-434)
 *
 * All three parties run inside one context on one GPU (their exchanges are
 * device-local buffer reads); a context holds one DB shard.  Plain pointers
 * and sizes only.  Return value: status code below (0 = ok).  Caller owns
 * every output buffer; the library owns device memory.  One host thread per
 * context.  Exceptions of the reference map to statuses as the reference CLI
 * maps them to exit codes (tools/irismpc_cli.cpp:552-564).
 */
#ifndef IRISMPC_GPU_H
#define IRISMPC_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IRISMPC_GPU_OK 0
#define IRISMPC_GPU_ERR_GENERIC 1
#define IRISMPC_GPU_ERR_CONFIG 2       /* Error / ConfigMismatchError (payload size, config) */
#define IRISMPC_GPU_ERR_DEVICE 3       /* TransportError analogue: CUDA failure, no device */
#define IRISMPC_GPU_ERR_BOUNDS 4       /* BoundsError (EngineConfig::validate) */
#define IRISMPC_GPU_ERR_INCONSISTENT 5 /* InconsistentShareError (replication cross-check) */

#define IRISMPC_GPU_BACKEND_REPLICATED 0
#define IRISMPC_GPU_BACKEND_SHAMIR 1
/* Variant (shares.hpp:28): ring widths (hd dot, ml dot, comparison) */
#define IRISMPC_GPU_VARIANT_PLAIN_MASK 0 /* 16, public mask bits, 16 */
#define IRISMPC_GPU_VARIANT_MPC_LIFT 1   /* 16, 16 lifted in MPC, 32 (the north-star path) */
#define IRISMPC_GPU_VARIANT_CONST_LIFT 2 /* 16, 32, 32 */
#define IRISMPC_GPU_VARIANT_NO_LIFT 3    /* 32, 32, 32 */

typedef struct irismpc_gpu_ctx irismpc_gpu_ctx;

/* EngineConfig (engine.hpp:33-44) + party seeds + shard placement. */
typedef struct irismpc_gpu_config {
  uint32_t backend;       /* IRISMPC_GPU_BACKEND_* */
  uint32_t variant;       /* IRISMPC_GPU_VARIANT_* */
  uint32_t l;             /* code length (bits), multiple of 8 */
  uint32_t a, b, m;       /* MatchParams integers (iris.hpp:157-174); b = 2^m, m = 16 */
  uint32_t rotations;     /* odd */
  uint32_t debug_rows;    /* open per-lane bits to P1 (engine.cpp:371-374) */
  uint8_t seeds[48];      /* seed_1 | seed_2 | seed_3 (16 bytes each) */
  int32_t device;         /* CUDA device ordinal */
  uint32_t shard_rank;    /* this context's shard (0 = holds the inner-batch pairs) */
  uint64_t db_rows_total; /* s of the whole DB across shards (0: = local s) */
  uint64_t db_row_offset; /* first global DB row held by this context */
  double match_ratio;     /* MatchParams::match_ratio; the plain-mask threshold
                             ceil((1 - 2 r) ml) uses it (iris.hpp:182-184) */
  uint64_t reserved[3];
} irismpc_gpu_config;

/* QueryStats (engine.hpp:46-56) for each party, plus device phase timings. */
typedef struct irismpc_gpu_stats {
  uint64_t s, l, batch, lanes;
  uint64_t dot_bytes[3], lift_bytes[3], msb_bytes[3], or_tree_bytes[3];
  uint64_t dot_rounds, lift_rounds, msb_rounds, or_tree_rounds;
  double wall_ms;      /* device time of the whole query (CUDA events) */
  double prep_ms, gemm_ms, threshold_ms, or_ms;
  uint64_t gemm_launches, kernel_launches;
  /* int8 ops the DB-lane GEMMs executed (all parties, both fields); below the
     algorithmic count when the rotation-pair (Winograd) GEMMs ran */
  uint64_t gemm_int8_ops;
  uint32_t rotation_pair_gemm; /* 1 if the rotation-pair GEMMs ran for some field */
} irismpc_gpu_stats;

/* ---- setup ------------------------------------------------------------ */
int irismpc_gpu_seeds_from_master(uint64_t master, uint8_t out[48]);
size_t irismpc_gpu_record_bytes(uint32_t backend, uint32_t variant, uint32_t l);
uint64_t irismpc_gpu_lane_count(uint32_t persons, uint64_t s, uint32_t rotations, int membership);

int irismpc_gpu_create(const irismpc_gpu_config* cfg, irismpc_gpu_ctx** out);
void irismpc_gpu_destroy(irismpc_gpu_ctx* ctx);
const char* irismpc_gpu_last_error(const irismpc_gpu_ctx* ctx);
/* Opaque cudaStream_t the context launches on (for caller-side events). */
void* irismpc_gpu_stream(irismpc_gpu_ctx* ctx);

/* ---- DB ---------------------------------------------------------------- */
/* payload[p]: party p+1's IRS1 row stream, len[p] == s * record_bytes. */
int irismpc_gpu_load_db(irismpc_gpu_ctx* ctx, const uint8_t* const payload[3],
                        const size_t len[3], uint64_t s);
/* Same, payloads already in device memory. */
int irismpc_gpu_load_db_device(irismpc_gpu_ctx* ctx, const uint8_t* const dpayload[3],
                               const size_t len[3], uint64_t s);

/* ---- queries ------------------------------------------------------------ */
/* q[p]: party p+1's query payload (2*persons code records).  person_match_out
 * [persons] receives the bits opened at P1; row_bits_out [lanes] (may be NULL)
 * receives the debug_rows opening.  stats may be NULL. */
int irismpc_gpu_batch_query(irismpc_gpu_ctx* ctx, const uint8_t* const q[3], const size_t qlen[3],
                            uint32_t persons, uint8_t* person_match_out, uint8_t* row_bits_out,
                            irismpc_gpu_stats* stats);
/* Same with device-resident query payloads; outputs still host pointers. */
int irismpc_gpu_batch_query_device(irismpc_gpu_ctx* ctx, const uint8_t* const dq[3],
                                   const size_t qlen[3], uint32_t persons,
                                   uint8_t* person_match_out, uint8_t* row_bits_out,
                                   irismpc_gpu_stats* stats);
/* Streaming: queue a batch query (DEVICE payloads, which must stay valid until
 * the ticket completes) and return at once.  The GEMM stream runs ahead into
 * the next submitted query while the threshold stream finishes this one, so a
 * query's GEMM-only head and threshold-only tail overlap its neighbours'.  At
 * most two queries are in flight: a third submit first completes the oldest.
 * person_match_out is written when the ticket completes (wait, or that
 * implicit completion).  Not with taps / debug_rows.  Results and PRF stream
 * positions are identical to the synchronous calls in the same order. */
int irismpc_gpu_batch_query_submit(irismpc_gpu_ctx* ctx, const uint8_t* const dq[3], const size_t qlen[3],
                                   uint32_t persons, uint8_t* person_match_out, uint64_t* ticket);
int irismpc_gpu_batch_query_wait(irismpc_gpu_ctx* ctx, uint64_t ticket, irismpc_gpu_stats* stats);
/* Single code, no rotation, one group (Session::membership). */
int irismpc_gpu_membership(irismpc_gpu_ctx* ctx, const uint8_t* const q[3], const size_t qlen[3],
                           uint8_t* match_out, uint8_t* row_bits_out, irismpc_gpu_stats* stats);

/* Multi-GPU: run the query on this shard but stop before the final OR/open.
 * partial_out_dev: DEVICE buffer [3][persons] bytes — bit 0 of each byte is one
 * XOR component of the shard's per-person aggregate (never opened). */
int irismpc_gpu_batch_query_partial(irismpc_gpu_ctx* ctx, const uint8_t* const dq[3],
                                    const size_t qlen[3], uint32_t persons,
                                    uint8_t* partial_out_dev, irismpc_gpu_stats* stats);
/* MPC-OR of G gathered shard partials (DEVICE [G][3][persons]) and the open
 * at P1 into host person_match_out[persons]. */
int irismpc_gpu_or_open(irismpc_gpu_ctx* ctx, const uint8_t* partials_dev, uint32_t G,
                        uint32_t persons, uint8_t* person_match_out);

/* ---- the comparison phase alone (the reference's `bench --phase comparison`,
 * PAPER Table 3) ------------------------------------------------------------
 * irismpc_gpu_comparison_only   party_comparison_only / run_comparison_local
 *                               (src/engine.cpp:448-515, src/cluster.cpp:97-145)
 * irismpc_gpu_or_tree_only      party_or_tree_only / run_or_tree_local
 *                               (src/engine.cpp:517-532, src/cluster.cpp:147-186)
 * hd_payload[p] / ml_payload[p]: party p+1's replicated (own, prev) shares of
 * each lane's masked dot and ml, little-endian at the variant's ring widths
 * (plain-mask ml: one public LE u64 per lane, the same at every party) --
 * exactly the reference's bench payloads.  lane_bits_out [lanes] (may be NULL)
 * receives the opened per-lane MSB bits (tests); opened_out [1] the OR of all
 * lanes opened at P1 when with_or_tree.  or_tree_only's payload[p]: per
 * 64-lane word (own u64, prev u64).  stats: the analytic per-party ledger
 * (lift incl. OT, msb, or_tree bytes and rounds) and device times.  Errors:
 * 2 on payload sizes, 5 when a party's prev copy differs from its neighbour's own. */
int irismpc_gpu_comparison_only(irismpc_gpu_ctx* ctx, const uint8_t* const hd_payload[3], const size_t hd_len[3],
                                const uint8_t* const ml_payload[3], const size_t ml_len[3], uint64_t lanes,
                                int with_or_tree, uint8_t* opened_out, uint8_t* lane_bits_out,
                                irismpc_gpu_stats* stats);
int irismpc_gpu_or_tree_only(irismpc_gpu_ctx* ctx, const uint8_t* const payload[3], const size_t len[3],
                             uint64_t lanes, uint8_t* opened_out, irismpc_gpu_stats* stats);

/* ---- DB-sharded queries across GPUs --------------------------
 * Each context holds one contiguous row range of the DB (cfg.shard_rank,
 * cfg.db_rows_total, cfg.db_row_offset) with all three parties' shares of
 * those rows, so every reshare and AND gate stays on its GPU.  A sharded query
 * (1) broadcasts the three query payloads from shard 0, (2) runs this shard's
 * lanes up to the per-person XOR-shared OR partial (never opened), (3) gathers
 * the partials to shard 0, which finishes the MPC-OR across shards and opens
 * at P1.  Lane and PRF indices are global, so results do not depend on the
 * shard count.  Collectives: NCCL (one process or thread per GPU; every shard
 * calls attach_nccl with the same id) or an in-process group (several
 * contexts of one process, possibly on one GPU, one host thread each).  All
 * shards call the query entry points together; q may be NULL except on shard
 * 0; person_match_out is written on shard 0. */
typedef struct irismpc_gpu_shard_group irismpc_gpu_shard_group;
int irismpc_gpu_shard_group_create(uint32_t world, irismpc_gpu_shard_group** out);
void irismpc_gpu_shard_group_destroy(irismpc_gpu_shard_group* group);
int irismpc_gpu_shard_attach_inproc(irismpc_gpu_ctx* ctx, irismpc_gpu_shard_group* group);
/* nccl_id from irismpc_gpu_nccl_unique_id on one shard, shared by the caller */
int irismpc_gpu_shard_attach_nccl(irismpc_gpu_ctx* ctx, const uint8_t nccl_id[128], uint32_t world);
int irismpc_gpu_sharded_batch_query(irismpc_gpu_ctx* ctx, const uint8_t* const q[3], const size_t qlen[3],
                                    uint32_t persons, uint8_t* person_match_out, irismpc_gpu_stats* stats);
/* same with DEVICE query payloads on shard 0 */
int irismpc_gpu_sharded_batch_query_device(irismpc_gpu_ctx* ctx, const uint8_t* const dq[3], const size_t qlen[3],
                                           uint32_t persons, uint8_t* person_match_out, irismpc_gpu_stats* stats);
int irismpc_gpu_sharded_membership(irismpc_gpu_ctx* ctx, const uint8_t* const q[3], const size_t qlen[3],
                                   uint8_t* match_out, irismpc_gpu_stats* stats);
/* Streaming form (NCCL attach only): every collective is stream-ordered, so each
 * shard's GEMM stream runs into the next query like irismpc_gpu_batch_query_submit;
 * complete with irismpc_gpu_batch_query_wait.  dq: DEVICE payloads on shard 0 (NULL
 * elsewhere), valid until the ticket completes. */
int irismpc_gpu_sharded_batch_query_submit(irismpc_gpu_ctx* ctx, const uint8_t* const dq[3], const size_t qlen[3],
                                           uint32_t persons, uint8_t* person_match_out, uint64_t* ticket);

/* PRF stream positions (per seed); a fresh context starts at 0 like
 * run_parties; the reference CLI keeps PartyCtx across queries. */
int irismpc_gpu_get_stream_positions(const irismpc_gpu_ctx* ctx, uint64_t pos[3]);
int irismpc_gpu_set_stream_positions(irismpc_gpu_ctx* ctx, const uint64_t pos[3]);

/* ---- device dealer (bit-compatible with the reference Rng streams) ------- */
/* `count` records random_record(l, Rng(rng_seed), mask_density) starting at
 * record index `first` of that stream (each record consumes 2l draws), into
 * DEVICE code/mask word arrays [count][(l+63)/64]. */
int irismpc_gpu_synth_records(irismpc_gpu_ctx* ctx, uint64_t rng_seed, uint64_t first,
                              uint64_t count, double mask_density, uint64_t* codes_dev,
                              uint64_t* masks_dev);
/* deal_*_payload with Rng(derive(seed_from_u64(deal_seed), tag)) starting at
 * record `first_record` of the dealing stream: DEVICE records -> DEVICE payloads. */
int irismpc_gpu_deal_payload(irismpc_gpu_ctx* ctx, uint64_t deal_seed, uint64_t tag,
                             uint64_t first_record, uint64_t nrec, const uint64_t* codes_dev,
                             const uint64_t* masks_dev, uint8_t* const out_dev[3]);
/* Synthetic DB straight into HBM: records [first, first+s) of Rng(rng_seed),
 * dealt with (deal_seed, tag 1) from record `first`, loaded as this shard. */
int irismpc_gpu_synth_db(irismpc_gpu_ctx* ctx, uint64_t s, uint64_t rng_seed, uint64_t first,
                         double mask_density, uint64_t deal_seed);

/* ---- party mode: one party per process / GPU ---------------
 * The reference's deployment: each party holds only its own payloads and its
 * two seeds (own, prev) and exchanges the protocol's messages with the other
 * two every round (PartyComm / TcpMesh, transport.hpp:54-154), here over NCCL
 * send/recv (ranks 0, 1, 2 = parties 1, 2, 3) or an in-process mailbox
 * (three parties in one process, like InProcNet).  The
 * per-phase byte/round ledger is counted from the messages actually sent
 * (CommLedger semantics), not derived analytically.  All four variants. */
typedef struct irismpc_gpu_party irismpc_gpu_party;
typedef struct irismpc_gpu_inproc irismpc_gpu_inproc;

/* Per-party QueryStats (engine.hpp:46-56) from the measured ledger. */
typedef struct irismpc_gpu_party_stats {
  uint64_t s, l, batch, lanes;
  uint64_t dot_bytes, lift_bytes, msb_bytes, or_tree_bytes;
  uint64_t dot_rounds, lift_rounds, msb_rounds, or_tree_rounds;
  uint64_t wire_bytes;  /* bytes this party actually handed to the transport */
  double wall_ms;       /* device time of the query on this party's GPU */
  double phase_ms[6];   /* device time: dot products, reshare, lift + inject, msb, or tree + open,
                           and [5] the time inside transport steps (all phases) */
} irismpc_gpu_party_stats;

/* 128-byte ncclUniqueId for the three ranks (rank 0 creates, all receive it). */
int irismpc_gpu_nccl_unique_id(uint8_t out[128]);
/* cfg.seeds: bytes 0..15 = this party's own seed, 16..31 = its prev seed
 * (read_seed_file, io.cpp:157-170).  party = 1, 2, 3.  NCCL rank = party - 1. */
int irismpc_gpu_party_create_nccl(const irismpc_gpu_config* cfg, uint32_t party, const uint8_t nccl_id[128],
                                  irismpc_gpu_party** out);
int irismpc_gpu_inproc_create(irismpc_gpu_inproc** out);
void irismpc_gpu_inproc_destroy(irismpc_gpu_inproc* net);
int irismpc_gpu_party_create_inproc(const irismpc_gpu_config* cfg, uint32_t party, irismpc_gpu_inproc* net,
                                    irismpc_gpu_party** out);
void irismpc_gpu_party_destroy(irismpc_gpu_party* pc);
const char* irismpc_gpu_party_last_error(const irismpc_gpu_party* pc);
/* This party's IRS1 payload (host). */
int irismpc_gpu_party_load_db(irismpc_gpu_party* pc, const uint8_t* payload, size_t len, uint64_t s);
/* party_batch_query / party_membership (engine.hpp:307-313): this party's
 * query payload; person_match_out / row_bits_out are filled at P1 only. */
int irismpc_gpu_party_batch_query(irismpc_gpu_party* pc, const uint8_t* q, size_t qlen, uint32_t persons,
                                  uint8_t* person_match_out, uint8_t* row_bits_out,
                                  irismpc_gpu_party_stats* stats);
int irismpc_gpu_party_membership(irismpc_gpu_party* pc, const uint8_t* q, size_t qlen, uint8_t* match_out,
                                 uint8_t* row_bits_out, irismpc_gpu_party_stats* stats);
/* Parity taps of the last query: this party's (own, prev) components,
 * tap = IRISMPC_GPU_TAP_* (DOT_* = own additive dot only, [n] at the ring's
 * width, u16 / u32; plain-mask DOT_ML = the public popcount, u16); RS_*, ML32,
 * DIFF: u32 [2][n]; MSB: bytes [2][n]. */
int irismpc_gpu_party_read_tap(irismpc_gpu_party* pc, int tap, void* host_out, size_t bytes);
int irismpc_gpu_party_stream_positions(const irismpc_gpu_party* pc, uint64_t pos_own_prev[2]);

/* ---- share / seed / plaintext files (io.hpp:28-60, src/io.cpp) ----------- */
/* IRS1 per-party share file: magic "IRS1", version 1, backend u8, variant u8,
 * party u8, code_k u8, mask_k u8, reserved u16, l u32, s u64, then the row
 * payload (24-byte header). */
typedef struct irismpc_gpu_share_header {
  uint32_t backend, variant, party, l;
  uint64_t s;
} irismpc_gpu_share_header;
/* read_share_file's checks (io.cpp:125-146): magic, version, width fields vs
 * the variant, file size == 24 + s * record_bytes.  2 on any violation. */
int irismpc_gpu_read_share_header(const char* path, irismpc_gpu_share_header* out);
int irismpc_gpu_write_share_file(const char* path, const irismpc_gpu_share_header* h,
                                 const uint8_t* payload, size_t len);
/* Session::load_db from the three parties' IRS1 files (party 1, 2, 3),
 * streamed from disk into HBM (pinned double buffer, H2D overlapped with the
 * parse).  Backend / variant / l must match the context (ConfigMismatchError
 * -> 2, like the CLI's share-file check, irismpc_cli.cpp:211-215). */
int irismpc_gpu_load_db_files(irismpc_gpu_ctx* ctx, const char* const paths[3]);
/* IRSD seed files (io.cpp:148-170) of parties 1..3 -> seed_1 | seed_2 | seed_3;
 * each file's prev seed must equal the previous party's own seed (2 if not). */
int irismpc_gpu_read_seed_files(const char* const paths[3], uint8_t seeds_out[48]);
int irismpc_gpu_write_seed_file(const char* path, uint32_t party, const uint8_t own[16],
                                const uint8_t prev[16]);
/* IRMP plaintext DB (dealer side, io.cpp:74-108): header then packed code bits
 * of all rows, then mask bits.  Words are LSB-first, (l + 63) / 64 per row. */
int irismpc_gpu_read_iris_db_header(const char* path, uint32_t* l_out, uint64_t* s_out);
int irismpc_gpu_read_iris_db(const char* path, uint64_t* codes_out, uint64_t* masks_out,
                             uint64_t rows_cap);
int irismpc_gpu_write_iris_db(const char* path, uint32_t l, uint64_t s, const uint64_t* codes,
                              const uint64_t* masks);

/* ---- profiling ------------------------------------------------------------ */
/* on = 1: every following query runs serialised on one stream (no GEMM /
 * threshold overlap) with CUDA events around every kernel launch, so each
 * kernel's time is its standalone serial time; on = 0 restores the overlapped
 * pipeline.  profile_read returns up to `max` (kernel name, total device ms,
 * launches) entries accumulated since the last read and resets them. */
int irismpc_gpu_profile(irismpc_gpu_ctx* ctx, int on);
int irismpc_gpu_profile_read(irismpc_gpu_ctx* ctx, char (*names)[48], double* ms, uint64_t* launches,
                             uint32_t max, uint32_t* count);
/* Which reshare / bit-inject kernels batch queries use: 0 (default) the
 * lane-major kernels, faster beside the GEMM; 1 the shared-memory tile kernels,
 * faster alone (the comparison-only path always uses those).  Same results. */
int irismpc_gpu_threshold_kernels(irismpc_gpu_ctx* ctx, int tile);

/* ---- debug / parity taps (tests) ------------------------------------------ */
#define IRISMPC_GPU_TAP_DOT_HD 1  /* [3][n] per-party additive hd dot (L1), u16 (KH = 16) / u32 */
#define IRISMPC_GPU_TAP_DOT_ML 2  /* [3][n] ml dot u16 / u32; plain-mask: [n] u16 public popcount */
#define IRISMPC_GPU_TAP_RS_HD 3   /* uint32 [3][n] components after reshare (L2) */
#define IRISMPC_GPU_TAP_RS_ML 4   /* uint32 [3][n] (0 for plain-mask) */
#define IRISMPC_GPU_TAP_ML32 5    /* uint32 [3][n] 32-bit ml components (lift output) */
#define IRISMPC_GPU_TAP_DIFF 6    /* uint32 [3][n] comparison input components */
#define IRISMPC_GPU_TAP_MSB 7     /* uint8  [3][n] match bit components */
#define IRISMPC_GPU_TAP_AGG 8     /* uint8  [3][groups] OR-tree output components of the last query
                                     (pre-open; always captured, no enable_taps needed) */
/* Enable capture of all taps for the next query (costly; tests only). */
int irismpc_gpu_enable_taps(irismpc_gpu_ctx* ctx, int enable);
int irismpc_gpu_read_tap(irismpc_gpu_ctx* ctx, int tap, void* host_out, size_t bytes);
/* Row-sampled L1 taps for DBs too large for full taps: while k > 0 every query
 * captures only DOT_HD / DOT_ML, for the k given rows of this shard (0-based
 * local rows) against every query column, then all pair lanes, as
 * [party][col * k + i] followed by [party][ncols * k + pair lane] -- the lane
 * order of the same query run against a k-row DB made of those rows.  k = 0
 * turns it off. */
int irismpc_gpu_tap_rows(irismpc_gpu_ctx* ctx, const uint64_t* rows, uint32_t k);

#ifdef __cplusplus
}
#endif
#endif /* IRISMPC_GPU_H */
