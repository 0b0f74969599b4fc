/*
 * irismpc oracle — CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker or the CPU baseline — never as the product path.
 *
 * It restates, in plain C, the reference algorithm of
 *   /root/reference/proj (irismpc), Session<B,KH,KM>::run_schedule
 *   (src/engine.cpp:297-398) for all four variants (plain-mask <16,0>,
 *   mpc-lift <16,16>, const-lift <16,32>, no-lift <32,32>) and everything it calls, with the exact PRF
 *   consumption order of the reference so that the GPU path can be checked
 *   share-for-share (parity levels L1..L5 of SURVEY.md §8c).
 *
 * The three parties are simulated in component form: an arithmetic
 * replicated sharing x = x1 + x2 + x3 is held as comp[0..2] = (x1, x2, x3);
 * party p holds (own, prev) = (x_p, x_{p-1}) (rep3.hpp:32-51).  Binary
 * sharings likewise hold the three XOR components.
 *
 * Parity is pinned: tests/test_oracle.py checks this restatement against
 * the reference itself compiled from /root/reference (oracle/_ref, see
 * oracle/Makefile) and against the committed golden vectors in tests/golden/.
 */
#ifndef IRISMPC_ORACLE_H
#define IRISMPC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_REPLICATED = 0, ORC_SHAMIR = 1 };
/* Variant (shares.hpp:28) */
enum { ORC_PLAIN_MASK = 0, ORC_MPC_LIFT = 1, ORC_CONST_LIFT = 2, ORC_NO_LIFT = 3 };

/* ---- L0: ChaCha12 counter PRF (prf.hpp:46-135) ---------------------- */
void orc_chacha_block(const uint8_t seed[16], uint64_t block, uint64_t stream,
                      uint32_t out[16]);
void orc_seed_from_u64(uint64_t v, uint8_t out[16]);
void orc_derive(const uint8_t parent[16], uint64_t tag, uint8_t out[16]);
/* element idx of the CtrPrf(seed, stream) u64 stream (random access) */
uint64_t orc_stream_at(const uint8_t seed[16], uint64_t stream, uint64_t idx);
/* party seeds of run_parties(seed): deal_seeds(Rng(derive(seed_from_u64(seed), 0x5eed)))
 * (cluster.hpp:35-36, rep3.hpp:116-122); out = seed_1 | seed_2 | seed_3 */
void orc_party_seeds(uint64_t master, uint8_t out[48]);

/* ---- Rng (prf.hpp:138-167) and synthetic records (iris.hpp:294-296) --- */
typedef struct orc_rng orc_rng;
orc_rng* orc_rng_new(uint64_t seed);
orc_rng* orc_rng_new_seed(const uint8_t seed[16]);
/* sub_rng(seed, tag) of cluster.cpp:24-26 */
orc_rng* orc_rng_sub(uint64_t seed, uint64_t tag);
void orc_rng_free(orc_rng* r);
uint64_t orc_rng_next(orc_rng* r);
uint64_t orc_rng_below(orc_rng* r, uint64_t bound);
int orc_rng_with_probability(orc_rng* r, double p);
uint64_t orc_rng_position(const orc_rng* r);
/* random_record(l, rng, density): mask bits drawn first, then code bits
 * (GCC argument order).  Words are LSB-first, (l+63)/64. */
void orc_rng_record(orc_rng* r, uint32_t l, double mask_density, uint64_t* code,
                    uint64_t* mask);

/* ---- L1 Galois ring (galois.hpp:66-128) ------------------------------ */
/* lambda_p for p=1..3 at K bits: out = {l1c0,l1c1,l2c0,l2c1,l3c0,l3c1} */
void orc_lambda(unsigned K, uint32_t out[6]);
void orc_lambda16(uint16_t out[6]);

/* ---- Variant widths (shares.hpp:37-48) ---------------------------------- */
unsigned orc_code_bits(int variant);
unsigned orc_mask_bits(int variant); /* 0 = public mask bits */
unsigned orc_cmp_bits(int variant);

/* ---- Dealer (shares.hpp:52-130, shares.cpp:49-90) ----------------------- */
size_t orc_code_record_bytes(int backend, int variant, uint32_t l);
size_t orc_mask_record_bytes(int backend, int variant, uint32_t l);
/* Emits nrec records (code record then mask record per row) for the three
 * parties, drawing from rng exactly as deal_db_payload / deal_query_payload. */
void orc_deal_payload_v(int backend, int variant, uint32_t l, uint64_t nrec, const uint64_t* codes,
                        const uint64_t* masks, orc_rng* rng, uint8_t* out1, uint8_t* out2,
                        uint8_t* out3);
/* mpc-lift shorthands */
size_t orc_code_record_bytes16(int backend, uint32_t l);
void orc_deal_payload(int backend, uint32_t l, uint64_t nrec, const uint64_t* codes,
                      const uint64_t* masks, orc_rng* rng, uint8_t* out1, uint8_t* out2,
                      uint8_t* out3);

/* ---- Engine (engine.cpp:21-398) --------------------------------------- */
typedef struct orc_config {
  int32_t backend;      /* ORC_REPLICATED / ORC_SHAMIR */
  int32_t variant;      /* ORC_PLAIN_MASK .. ORC_NO_LIFT */
  uint32_t l;           /* code length in bits, multiple of 8 */
  uint32_t a, b;        /* MatchParams (iris.hpp:157-174); b = 2^16 for shared masks */
  uint32_t rotations;   /* odd */
  int32_t debug_rows;   /* open per-lane bits to P1 */
  double ratio;         /* MatchParams::match_ratio (plain_threshold, iris.hpp:182-184) */
} orc_config;

/* Analytic communication ledger per party (transport.hpp:54-86), as filled
 * into QueryStats by fill_stats (engine.cpp:119-135). */
typedef struct orc_stats {
  uint64_t dot_bytes, lift_bytes, msb_bytes, or_tree_bytes;
  uint64_t dot_rounds, lift_rounds, msb_rounds, or_tree_rounds;
} orc_stats;

/* Optional outputs; every pointer may be NULL.  Component arrays are laid
 * out [comp][lane] with n lanes (orc_lane_count). */
typedef struct orc_out {
  uint8_t* person_match;   /* [persons]  opened at P1 */
  uint8_t* row_bits;       /* [n]        debug_rows opening (cfg.debug_rows) */
  uint32_t* dot_hd;        /* [3][n] per-party additive hd dots mod 2^KH (L1) */
  uint32_t* dot_ml;        /* [3][n] per-party additive ml dots mod 2^KM (L1) */
  int64_t* public_ml;      /* [n] plain-mask popcounts (plain-mask only) */
  uint32_t* rs_hd;         /* [3][n] components after reshare_pair (L2) */
  uint32_t* rs_ml;         /* [3][n] */
  uint32_t* ml32;          /* [3][n] 32-bit ml components (lift output / KM=32 copy) */
  uint32_t* diff;          /* [3][n] comparison input: a*ml32 - b*hd (mod 2^32), or
                              ceil((1-2r)ml) - hd (mod 2^16, plain-mask) */
  uint8_t* msb;            /* [3][n] MSB (match) bit components */
  uint64_t* stream_pos;    /* [3]   seed stream positions after the query */
  orc_stats* stats;        /* [3]   per party */
  uint8_t* agg;            /* [3][groups] or_tree_batch output components (pre-open) */
} orc_out;

/* or_tree_batch (circuits.hpp:387-434) over caller-given bit sharings: comps
 * [3][total] component bits, groups = consecutive runs of lens[g] lanes, seed
 * streams at stream_start (NULL = 0).  agg [3][ngroups]; stream_pos [3] after. */
int orc_or_tree_batch(const uint8_t seeds[48], const uint64_t* stream_start, uint32_t ngroups,
                      const uint64_t* lens, const uint8_t* comps, uint64_t total, uint8_t* agg,
                      uint64_t* stream_pos);

uint64_t orc_lane_count(uint32_t persons, uint64_t s, uint32_t rotations, int membership);

/* One 3-party query over dealt payloads (party_batch_query / party_membership,
 * engine.hpp:307-313).  membership != 0: one code, no rotation, one group.
 * stream_start: per-seed start positions (NULL = all 0, as in run_parties).
 * Returns 0 on success, 2 on config/size errors, 4 on bounds errors. */
int orc_query(const orc_config* cfg, const uint8_t seeds[48], const uint8_t* db1,
              const uint8_t* db2, const uint8_t* db3, uint64_t s, const uint8_t* q1,
              const uint8_t* q2, const uint8_t* q3, uint32_t persons, int membership,
              const uint64_t* stream_start, orc_out* out);

/* run_batch_local / run_membership_local (cluster.cpp:30-79): deals the DB with
 * sub_rng(seed,1), the queries with sub_rng(seed,2), party seeds from seed. */
int orc_run_local(const orc_config* cfg, uint64_t seed, uint64_t s, const uint64_t* db_codes,
                  const uint64_t* db_masks, uint32_t persons, const uint64_t* q_codes,
                  const uint64_t* q_masks, int membership, orc_out* out);

/* MatchParams::make(ratio, 16).a (iris.hpp:163-174) */
uint32_t orc_match_a(double ratio);
/* EngineConfig::validate (engine.cpp:21-34): 0 ok, 4 bounds */
int orc_validate(const orc_config* cfg);

#ifdef __cplusplus
}
#endif
#endif
