/*
 * ogm_oracle.h -- CPU restatement of the OblivGM hot path (TEST INFRASTRUCTURE).
 *
 * This library is the parity checker for the CUDA product in
 * paper_2209_03526_b200/.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.  It is never
 * part of the shipped path.
 *
 * Every function restates one routine of the reference package
 * (/root/reference/pkg/src/oblivgm/, abbreviated src/) and cites it.
 * Parity of this restatement is pinned against the live reference by
 * tests/golden/make_golden.py (fixtures in tests/golden/) and
 * tests/test_oracle_golden.py.
 *
 * Byte conventions follow the reference exactly:
 *  - a 16-byte seed is the little-endian byte image of an (lo, hi) uint64
 *    pair (src/prf.py:60-67);
 *  - bit i of a packed vector is bit i%32 of uint32 word i/32 (src/bits.py:1-8).
 */
#ifndef OGM_ORACLE_H
#define OGM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* AES-128 (FIPS-197), software T-table implementation. */
void ogm_or_aes128_expand(const uint8_t key[16], uint32_t rk[44]);
void ogm_or_aes128_encrypt(const uint32_t rk[44], const uint8_t in[16], uint8_t out[16]);

/* src/prf.py:41-57 prg_expand.  seeds: n*16 bytes; left/right: n*16 bytes. */
void ogm_or_prg_expand(const uint8_t *seeds, int64_t n, uint8_t *left, uint8_t *right,
                       uint8_t *t_left, uint8_t *t_right, uint8_t *value);

/* src/prf.py:70-84 prf_stream, starting at CTR block `block_offset`
 * (offset 0 reproduces the reference call). */
void ogm_or_prf_stream(const uint8_t key[16], const uint8_t label[4], uint64_t index,
                       uint64_t block_offset, uint8_t *out, int64_t nbytes);

/* src/prf.py:95-105 seeded_permutation. */
void ogm_or_seeded_permutation(const uint8_t key[16], const uint8_t label[4], uint64_t index,
                               int64_t n, int64_t *perm);

/* src/fss.py:116-157 _tree_gen with injected roots (the reference draws
 * root0, root1 = rng.bytes(16) twice, src/fss.py:117-118).
 * seed_cw: bits*16 bytes, ctrl_cw: bits bytes. */
void ogm_or_tree_gen(uint64_t alpha, int bits, const uint8_t root0[16], const uint8_t root1[16],
                     int comparison, uint8_t *seed_cw, uint8_t *ctrl_cw, uint8_t *final_cw);

/* Batched _tree_gen: key-major outputs (K*bits*16, K*bits, K). */
void ogm_or_tree_gen_batch(int64_t K, int bits, const uint64_t *alphas, const uint8_t *roots0,
                           const uint8_t *roots1, int comparison, uint8_t *seed_cw,
                           uint8_t *ctrl_cw, uint8_t *final_cw, int nthreads);

/* src/fss.py:257-281 _walk_eval for K keys, one point each.  Key-major
 * arrays: root K*16, root_t K, seed_cw K*bits*16, ctrl_cw K*bits, final_cw K,
 * add_const K.  out: K bytes (0/1).  Returns 0, or -1 when a point is outside
 * the 2^bits domain (the reference raises DomainError, src/fss.py:259-260). */
int ogm_or_eval_points(int bits, int comparison, int64_t K, const uint8_t *root,
                       const uint8_t *root_t, const uint8_t *seed_cw, const uint8_t *ctrl_cw,
                       const uint8_t *final_cw, const uint8_t *add_const, const uint64_t *points,
                       uint8_t *out, int nthreads);

/* src/fss.py:302-337 _full_domain_tree: n output bits packed into
 * ceil(n/32) words.  Returns -1 when n > 2^bits. */
int ogm_or_full_domain(int bits, int comparison, const uint8_t root[16], int root_t,
                       const uint8_t *seed_cw, const uint8_t *ctrl_cw, int final_cw,
                       int add_const, int64_t n, uint32_t *out_words);

/* src/engine.py:76-80 + :162: out[c] = parity((da[c]&ia) ^ (db[c]&ib)). */
void ogm_or_masked_parity(const uint32_t *da, const uint32_t *db, int64_t rows, int64_t w,
                          const uint32_t *ia, const uint32_t *ib, uint8_t *out);

#ifdef __cplusplus
}
#endif
#endif
