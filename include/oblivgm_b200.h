/*
 * oblivgm_b200.h -- C ABI of the B200-native OblivGM hot path (libogm_b200.so).
 *
 * The reference (oblivgm 0.1.0, /root/reference/pkg/src/oblivgm, abbreviated
 * src/) is pure Python and has no FFI of its own: its "operator interface" is
 * a set of module-level functions over numpy arrays.  Every entry point below
 * replaces one of those functions (cited per entry); the Python package
 * paper_2209_03526_b200 keeps the reference names and signatures and binds
 * these symbols with ctypes (see INTEGRATION.md for the binding a maintainer
 * of the reference would add).
 *
 * Conventions
 *  - Plain pointers and sizes only.  Pointers are DEVICE pointers unless the
 *    entry point name ends in _host.  `stream` is a cudaStream_t (NULL =
 *    legacy default stream).  Calls are asynchronous on `stream` unless
 *    documented otherwise; the library holds no global mutable state besides
 *    per-device constant tables, so distinct host threads may drive distinct
 *    streams concurrently (one per logical party, src/net.py:320-351).
 *  - Return value: 0 on success, a negative OGM_ERR_* code otherwise; the
 *    message is available from ogm_last_error() (thread-local).  The Python
 *    shim maps OGM_ERR_DOMAIN to fss.DomainError (src/fss.py:44-45),
 *    OGM_ERR_ARG to ValueError, OGM_ERR_PROTOCOL to net.ProtocolError
 *    (src/net.py:38-39).
 *  - Bit vectors: bit i lives at bit i%32 of uint32 word i/32, bits past the
 *    logical length are zero (src/bits.py:1-8).  Share matrices are row-major
 *    (rows, pitch) uint32 with pitch >= ceil(width/32) words.
 *  - 16-byte seeds are the little-endian image of (lo, hi) uint64
 *    (src/prf.py:60-67).
 *  - FSS key batches are structure-of-arrays, level-major, so that thread k
 *    of a warp reads key k with coalesced 128-bit loads:
 *        root    [K][16 B]
 *        seed_cw [bits][K][16 B]       (src/fss.py:62 seed_cw[lvl])
 *        ctrl    [3][K] uint32         word 0 bit lvl = tau_L, word 1 = tau_R,
 *                                      word 2 = value bit (src/fss.py:63)
 *        flags   [K] uint8             bit0 root_t, bit1 final_cw,
 *                                      bit2 add_const (src/fss.py:59-65)
 *    so domain_bits is limited to 1..32 (graph dictionaries and BASELINE
 *    config 2 are all <= 32 bits).
 */
#ifndef OBLIVGM_B200_H
#define OBLIVGM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OGM_OK 0
#define OGM_ERR_ARG -1      /* ValueError: length / width / party mismatch   */
#define OGM_ERR_DOMAIN -2   /* fss.DomainError: point or threshold outside    */
#define OGM_ERR_CUDA -3     /* CUDA runtime failure                           */
#define OGM_ERR_PROTOCOL -4 /* net.ProtocolError: label / table id mismatch   */
#define OGM_ERR_NOMEM -5    /* device allocation failure                      */

#define OGM_KIND_DPF 0 /* point function, src/fss.py:160-164      */
#define OGM_KIND_DCF 1 /* comparison function, src/fss.py:167-171 */

/* ---- library ----------------------------------------------------------- */

/* Thread-local message of the last failing call. */
const char* ogm_last_error(void);
/* ABI version (bumped on any signature change). */
int ogm_abi_version(void);
/* Upload the AES tables and fixed PRG round keys to the current device.
 * Idempotent per device; every other entry point calls it lazily. */
int ogm_init(void);

/* ---- L0 randomness (src/prf.py) ----------------------------------------- */

/* src/prf.py:41-57 prg_expand.  seeds/left/right: n x 16 B; t_left, t_right,
 * value: n bytes (0/1). */
int ogm_prg_expand(const void* seeds, int64_t n, void* left, void* right, uint8_t* t_left,
                   uint8_t* t_right, uint8_t* value, void* stream);

/* src/prf.py:70-92 prf_stream / prf_words: AES-128-CTR keystream of
 * (key, label, index) as uint32 LE words, starting at word `first_word`
 * (random access by block).  key/label are HOST pointers (16 / 4 bytes). */
int ogm_prf_words(const uint8_t* key, const uint8_t* label, uint64_t index, uint64_t first_word,
                  int64_t nwords, uint32_t* out, void* stream);

/* src/shuffle.py:69-73 _table: a (rows x width-bit) blinding table, row r =
 * PRF words [r*W, r*W+W) of (key, label, index), W = ceil(width/32), tail
 * masked; stored with row pitch `pitch` >= W words, padding zeroed. */
int ogm_prf_rows(const uint8_t* key, const uint8_t* label, uint64_t index, int64_t rows,
                 int64_t width_bits, int64_t pitch, uint32_t* out, void* stream);

/* src/rss.py:143-148 ZeroShareContext.next_share at counter `counter`:
 * out = F(key_own, "ZSHR", counter) ^ F(key_prev, "ZSHR", counter), masked to
 * nbits.  If `xor_into` is non-NULL the share is XORed into it and the
 * tail is masked after the fold, as BitVector(additive ^ share, nbits) does
 * in src/rss.py:171 (out may equal xor_into).  Keys are HOST pointers. */
int ogm_zero_share(const uint8_t* key_own, const uint8_t* key_prev, uint64_t counter,
                   int64_t nbits, const uint32_t* xor_into, uint32_t* out, void* stream);

/* Words [first_word, first_word + nwords) of the same zero share (random
 * access by CTR block): the slice a rank owns when candidate rows are
 * sharded across GPUs; concatenated slices equal the
 * unsharded share bit for bit. */
int ogm_zero_share_slice(const uint8_t* key_own, const uint8_t* key_prev, uint64_t counter,
                         int64_t total_nbits, uint64_t first_word, int64_t nwords,
                         const uint32_t* xor_into, uint32_t* out, void* stream);

/* src/prf.py:95-105 seeded_permutation: Fisher-Yates driven by
 * prf_stream(key, label, index, 8(n-1)); bit-exact, computed on the device by
 * deterministic reservations.  perm: n int32 (gather semantics, M[perm]).
 * workspace: >= ogm_perm_workspace_bytes(n) bytes of device memory. */
int64_t ogm_perm_workspace_bytes(int64_t n);
int ogm_seeded_permutation(const uint8_t* key, const uint8_t* label, uint64_t index, int64_t n,
                           int32_t* perm, void* workspace, void* stream);

/* ---- L1 function secret sharing (src/fss.py) ---------------------------- */

/* src/fss.py:116-157 _tree_gen, batched over K independent keys with
 * injected roots (the reference draws root0, root1 with rng.bytes(16),
 * src/fss.py:117-118).  alphas: K uint32 (< 2^bits).  Writes the shared
 * correction words (seed_cw [bits][K][16 B], ctrl [3][K]) and final_cw [K]. */
int ogm_fss_gen(int kind, int bits, int64_t K, const uint32_t* alphas, const void* roots0,
                const void* roots1, void* seed_cw, uint32_t* ctrl, uint8_t* final_cw,
                void* stream);

/* ogm_fss_gen writing both parties' per-key flag bytes in the layout the
 * eval entry points read (bit 0 root_t -- 0 for party 0, 1 for party 1 --,
 * bit 1 final_cw, bit 2 add_const = 0) instead of final_cw alone. */
int ogm_fss_gen_pair(int kind, int bits, int64_t K, const uint32_t* alphas, const void* roots0,
                     const void* roots1, void* seed_cw, uint32_t* ctrl, uint8_t* flags0, uint8_t* flags1,
                     void* stream);

/* src/fss.py:257-299 _walk_eval / dpf_eval / dcf_eval: one point per key,
 * one thread per (key, point).  out_bits: ceil(K/32) words, bit k = key k. */
int ogm_fss_eval_points(int kind, int bits, int64_t K, const void* root, const void* seed_cw,
                        const uint32_t* ctrl, const uint8_t* flags, const uint32_t* points,
                        uint32_t* out_bits, void* stream);

/* Same computation from HOST buffers (the end-to-end call a CPU caller
 * makes): copies keys/points in, evaluates, copies the packed bits out and
 * synchronizes.  Host buffers should be pinned for full PCIe bandwidth.
 * The transfer is chunked and overlapped with evaluation on two streams.
 * For DCF keys the last level's seed correction (never read) is not copied. */
int ogm_fss_eval_points_host(int kind, int bits, int64_t K, const void* root_h,
                             const void* seed_cw_h, const uint32_t* ctrl_h, const uint8_t* flags_h,
                             const uint32_t* points_h, uint32_t* out_bits_h);

/* src/fss.py:302-344 _full_domain_tree / full_domain_eval for `nkeys` keys
 * of one batch (layout above with K = nkeys), each over points [0, n).
 * out_words: nkeys x pitch words (pitch >= ceil(n/32)), row k = key k. */
int ogm_fss_full_domain(int kind, int bits, int nkeys, const void* root, const void* seed_cw,
                        const uint32_t* ctrl, const uint8_t* flags, int64_t n, uint32_t* out_words,
                        int64_t pitch, void* stream);

/* ---- L1 replicated secret sharing (src/rss.py) ---------------------------- */

/* src/rss.py:143-148 for all three co-resident parties at once:
 * out[q] = F(key_q) ^ F(key_{q-1}) (^ xor_into[q]), keys k1, k2, k3 as held
 * by src/net.py:221-233.  xor_into may be NULL (or have NULL entries). */
int ogm_zero_share_trio(const uint8_t* k1, const uint8_t* k2, const uint8_t* k3, uint64_t counter,
                        int64_t nbits, const uint32_t* const* xor_into, uint32_t* const* out,
                        void* stream);

/* Two consecutive re-shares' slices (counters counter1, counter2 -- the two
 * passes of an interval predicate) in one launch: out1 as
 * ogm_zero_share_trio_slice at counter1, out2 at counter2. */
int ogm_zero_share_trio_slice2(const uint8_t* k1, const uint8_t* k2, const uint8_t* k3, uint64_t counter1,
                               uint64_t counter2, int64_t nbits, int64_t w0, int64_t nwords,
                               const uint32_t* const* xor_into1, uint32_t* const* out1,
                               const uint32_t* const* xor_into2, uint32_t* const* out2, void* stream);

/* The two passes of an interval predicate folded (co-resident trio;
 * src/engine.py:150-165 with src/rss.py:143-148,164-176): a
 * re-share is a zero share XORed in and parity is linear, so the XOR of the
 * two passes' re-shared parities equals ONE parity over XORed indicators
 * with both zero shares XORed in.  out = xor_into ^ zs(counter1) ^
 * zs(counter2) on the slice [w0, w0 + nwords) (xor_into may alias out). */
int ogm_zero_share_trio_fold2(const uint8_t* k1, const uint8_t* k2, const uint8_t* k3, uint64_t counter1,
                              uint64_t counter2, int64_t nbits, int64_t w0, int64_t nwords,
                              const uint32_t* const* xor_into, uint32_t* const* out, void* stream);

/* The matrix re-share of src/engine.py:83-92 for the three parties: the
 * zero share of rows*words*32 bits XORed into xor_into[q], every row's tail
 * (bits >= width of each `words`-word row) masked after the XOR. */
int ogm_zero_share_trio_rows(const uint8_t* k1, const uint8_t* k2, const uint8_t* k3, uint64_t counter, int64_t rows,
                             int64_t words, int64_t width, const uint32_t* const* xor_into, uint32_t* const* out,
                             void* stream);

/* The same for words [w0, w0 + nwords) of the nbits-bit vector (w0 % 4 == 0),
 * written to out[q][0 .. nwords): one rank's slice of a row-sharded secEval
 * (SURVEY 8(e)); the tail mask applies only to the vector's last word. */
int ogm_zero_share_trio_slice(const uint8_t* k1, const uint8_t* k2, const uint8_t* k3, uint64_t counter,
                              int64_t nbits, int64_t w0, int64_t nwords, const uint32_t* const* xor_into,
                              uint32_t* const* out, void* stream);

/* src/rss.py:115-126 and_terms for nparty (1..3) parties: out[q] =
 * a_a[q]&b_a[q] ^ a_a[q]&b_b[q] ^ a_b[q]&b_a[q] over nwords words. */
int ogm_and_terms(int64_t nwords, int nparty, const uint32_t* const* a_a, const uint32_t* const* a_b,
                  const uint32_t* const* b_a, const uint32_t* const* b_b, uint32_t* const* out,
                  void* stream);

/* Word-wise out = a ^ b (^ c if non-NULL): the local XOR of shares
 * (src/rss.py:53-59, src/engine.py:164,182,188). */
int ogm_xor_words(int64_t nwords, const uint32_t* a, const uint32_t* b, const uint32_t* c,
                  uint32_t* out, void* stream);

/* ---- L3 protocol engine (src/engine.py) ---------------------------------- */

/* src/engine.py:76-80 + :162 (secEval's local step, both interval passes
 * in one read of the shares).  nparty = 1: comps = {A, B} (the party's two
 * share matrices); nparty = 3: comps = {x1, x2, x3} and party q reads
 * (x_q, x_{q+1}).  a_idx/b_idx must state that mapping.  ind[(p*nparty+q)*2
 * + {0,1}] = full-domain indicator words of pass p's first / second key
 * (src/engine.py:160-161); out[p*nparty+q] = ceil(rows/32) words. */
int ogm_masked_parity(int64_t rows, int64_t words, int64_t pitch, int ncomp, const uint32_t* const* comps,
                      int nparty, const int32_t* a_idx, const int32_t* b_idx, int npass,
                      const uint32_t* const* ind, uint32_t* const* out, void* stream);

/* The same, XORed into out (which the caller initialised, e.g. with the
 * pass's zero share) instead of overwriting it: no zeroing launches. */
int ogm_masked_parity_acc(int64_t rows, int64_t words, int64_t pitch, int ncomp, const uint32_t* const* comps,
                          int nparty, const int32_t* a_idx, const int32_t* b_idx, int npass,
                          const uint32_t* const* ind, uint32_t* const* out, void* stream);

/* src/engine.py:95-102 _select_one_additive for nparty parties (Case I
 * fetch, src/engine.py:197-217, and the posting fold of sec_access,
 * src/engine.py:309-311): out[q] (words) = XOR over rows c of
 * fa_q(c)(A_q[c]^B_q[c]) ^ fb_q(c) A_q[c], with fa/fb bit vectors. */
int ogm_select_fold(int64_t rows, int64_t words, int64_t pitch, int nparty, const uint32_t* const* A,
                    const uint32_t* const* B, const uint32_t* const* fa, const uint32_t* const* fb,
                    uint32_t* const* out, void* stream);

/* src/engine.py:105-120 _select_many_additive: out (K, opitch) =
 * sel_a (K x X one-hot rows) * (A ^ B) ^ sel_b * A over GF(2), A/B (X, pitch).
 * workspace: >= 8*X bytes. */
int ogm_select_many(int64_t K, int64_t X, int64_t words, int64_t pitch, const uint32_t* sel_a,
                    const uint32_t* sel_b, int64_t spitch, const uint32_t* A, const uint32_t* B,
                    uint32_t* out, int64_t opitch, void* workspace, void* stream);

/* src/engine.py:227-233 / :317-318 row building: out row r = flag(r) ||
 * field_0[r] || ... (bit-concatenated at their logical widths, LE, clean
 * tail).  flag_bits (rows bits) may be NULL. */
int ogm_pack_fields(int64_t rows, const uint32_t* flag_bits, int nfields, const uint32_t* const* fields,
                    const int64_t* fpitch, const int64_t* fwidth, uint32_t* out, int64_t opitch,
                    void* stream);

/* src/engine.py:227-233 (Case II row layout) fused with the first gather of
 * the shuffle that consumes those rows (src/shuffle.py:106-118):
 *   out[i] = XOR over s < nsets of pack(flag_s, fields_s)[src] ^ r_mat[i],
 *   src = idx ? idx[i] : i
 * flag_bits is NULL (rows without a flag bit) or nsets bit vectors; fields
 * and fpitch are nsets x nfields, set-major; fwidth has nfields entries;
 * r_mat (pitch opitch) may be NULL.  nsets = 2 emits a^b of two share
 * components, so a party's first shuffle step never materialises its packed
 * rows.  nsets = 1, idx = r_mat = NULL is ogm_pack_fields. */
int ogm_pack_gather(int64_t rows, const int32_t* idx, int nsets, const uint32_t* const* flag_bits,
                    int nfields, const uint32_t* const* fields, const int64_t* fpitch,
                    const int64_t* fwidth, const uint32_t* r_mat, uint32_t* out, int64_t opitch,
                    void* stream);

/* src/engine.py:249-269 / :331-334 field slicing: out[k] = bits
 * [bit_offset, bit_offset+width) of src row idx[k] (idx NULL = identity). */
int ogm_extract_field(const uint32_t* src, int64_t spitch, const int32_t* idx, int64_t n,
                      int64_t bit_offset, int64_t width, uint32_t* out, int64_t opitch, void* stream);

/* src/engine.py:88-89: clear bits >= width in the last word of every row. */
int ogm_mask_row_tails(uint32_t* mat, int64_t rows, int64_t pitch, int64_t width, void* stream);

/* src/engine.py:241-245: bit r of out_bits = mat[r][0] & 1 (flag column). */
int ogm_column_bits(const uint32_t* mat, int64_t pitch, int64_t rows, uint32_t* out_bits, void* stream);

/* src/engine.py:252 / :327 np.nonzero of an opened mask: indices of set
 * bits in order, count to *out_count (device int64). */
int64_t ogm_compact_workspace_bytes(int64_t n);
int ogm_compact_bits(int64_t n, const uint32_t* bits, int32_t* out_idx, int64_t* out_count,
                     void* workspace, int64_t workspace_bytes, void* stream);

/* Keep the rows whose mask bit is set, in order (src/engine.py:249-269 /
 * :327-334, the np.nonzero + row loop after an open): optionally their
 * indices to out_idx, and their 16-byte-pitched rows of nmat (<= 8) matrices
 * mats[j] (pitch words) to consecutive rows of outs[j] (opitch words).  The
 * kept count goes to *count (device int64).  Hand-written three-launch
 * compaction (chunk popcounts, one-CTA scan, warp-per-chunk emit). */
int64_t ogm_keep_rows_workspace_bytes(int64_t rows);
int ogm_keep_rows(int64_t rows, const uint32_t* bits, int nmat, const uint32_t* const* mats, int64_t pitch,
                  uint32_t* const* outs, int64_t opitch, int32_t* out_idx, int64_t* count, void* workspace,
                  int64_t workspace_bytes, void* stream);

/* ---- flagged-row fetch in the flag-split layout (src/engine.py:220-270) ---
 * A sec_fetch_multi row [flag | 128-bit payload] is 129 bits (5 words).  The
 * fetch keeps it split: payload as a 16-byte row, flag as a bit column
 * (bit permutations and XORs commute with the shuffle, so results are the
 * reference's bits).  ogm_split_flag_rows turns a 5-word-row table (blinds
 * drawn in the reference layout) into the two parts: payload[i] = bits
 * 1..128 of row i, bit i of flags = bit 0 of row i. */
int ogm_split_flag_rows(int64_t rows, const uint32_t* in, int64_t pitch, uint32_t* payload, uint32_t* flags,
                        void* stream);

/* The flag column through one 3-party shuffle (src/shuffle.py:106-143 on bit
 * 0 of every row), for the three co-resident parties, with the same composed
 * permutations and split blinds as the payload:
 *   x1f = (f1 ^ f2)[k1] ^ Uf,  y1f = f3[pi12] ^ Vf,  c1f = x1f[pi23] ^ Wf,
 *   r3f = y1f[k3] ^ c1f ^ Zf,  plain = R1f ^ R2f ^ r3f (the opened column,
 *   optional; src/rss.py:184-206).
 * All columns are packed bit vectors; x1f, y1f are scratch (or the message
 * copies), c1f and plain optional. */
int ogm_flag_shuffle_trio(int64_t rows, const int32_t* k1, const int32_t* pi12, const int32_t* pi23,
                          const int32_t* k3, const uint32_t* f1, const uint32_t* f2, const uint32_t* f3,
                          const uint32_t* uf, const uint32_t* vf, const uint32_t* wf, const uint32_t* zf,
                          const uint32_t* r1f, const uint32_t* r2f, uint32_t* x1f, uint32_t* y1f, uint32_t* c1f,
                          uint32_t* r3f, uint32_t* plain, void* stream);

/* The flag column of the co-resident trio (src/shuffle.py:106-143 on bit 0
 * of the fetch rows, then the open of src/engine.py:241-247 /
 * src/rss.py:184-206), each party's step composed with
 * the next one's (as the payload's flat hand-over composes them: the message
 * bits x1f / y1f exist only in flight), so two random bit reads per row
 * instead of four:
 *   c1f[i] = f12[kc[i]] ^ uwf[i],        kc = k1 o pi23 (kc[i] = k1[pi23[i]]),
 *                                        uwf[i] = Uf[pi23[i]] ^ Wf[i]
 *   r3f[i] = f3[kr[i]] ^ vzf[i] ^ c1f[i], kr = pi12 o k3, vzf[i] = Vf[k3[i]] ^ Zf[i]
 *   plain  = R1f ^ R2f ^ r3f
 * f12 = f1 ^ f2 (scratch, rows/32 words); c1f may be NULL.  The same columns
 * as ogm_flag_shuffle_trio. */
int ogm_flag_open_composed(int64_t rows, const int32_t* kc, const int32_t* kr, const uint32_t* f1,
                           const uint32_t* f2, const uint32_t* f3, const uint32_t* uwf, const uint32_t* vzf,
                           const uint32_t* r1f, const uint32_t* r2f, uint32_t* f12, uint32_t* c1f, uint32_t* r3f,
                           uint32_t* plain, void* stream);

/* The online phase of a flag-split fetch of <= 2^21 rows in ONE cooperative
 * launch: the three-party shuffle of ogm_shuffle_online_fused (x1 / y1:
 * scratch tables; R3 out) and, in its second phase, the composed flag column
 * and the open of ogm_flag_open_composed (f12: scratch; r3f and plain out).
 * Same results as those two calls (src/shuffle.py:80-144 on the fetch rows,
 * src/engine.py:241-247). */
int ogm_fetch128_online_fused(int64_t rows, const int32_t* k1, const int32_t* pi12, const int32_t* pi23,
                              const int32_t* k3, const uint32_t* a, const uint32_t* b, const uint32_t* c,
                              const uint32_t* U, const uint32_t* V, const uint32_t* W, const uint32_t* Z,
                              uint32_t* x1, uint32_t* y1, uint32_t* r3, const int32_t* kc, const int32_t* kr,
                              const uint32_t* f1, const uint32_t* f2, const uint32_t* f3, const uint32_t* uwf,
                              const uint32_t* vzf, const uint32_t* r1f, const uint32_t* r2f, uint32_t* f12,
                              uint32_t* r3f, uint32_t* plain, void* stream);

/* The online phase of a flag-split fetch shuffle for >= 2^22 rows in one
 * call: f12 = f1 ^ f2, then the chained planned payload shuffle (as
 * ogm_shuffle_online_planned_slots) whose final window passes also compute
 * the composed flag column of ogm_flag_open_composed (c1f: scratch) and the
 * opened column -- the flag column needs the rows in output order, which
 * those passes walk anyway.  Same results as ogm_shuffle_online_planned_slots
 * + ogm_flag_open_composed. */
int ogm_fetch128_online_planned(int64_t rows, const int32_t* const* q2, const int32_t* const* gdst,
                                const uint16_t* const* srow, const int32_t* const* qs,
                                const uint16_t* const* run_start, const int32_t* const* run_off,
                                const int64_t* run_nwin, const int64_t* wrows, const uint32_t* a, const uint32_t* b,
                                const uint32_t* c, const uint32_t* u_src, const uint32_t* v_src,
                                const uint32_t* w_blind, int w_order, const uint32_t* z_slot, int z_order,
                                uint32_t* const* inter, uint32_t* r3, const int32_t* kc, const int32_t* kr,
                                const uint32_t* f1, const uint32_t* f2, const uint32_t* f3, const uint32_t* uwf,
                                const uint32_t* vzf, const uint32_t* r1f, const uint32_t* r2f, uint32_t* f12,
                                uint32_t* c1f, uint32_t* r3f, uint32_t* plain, void* stream);

/* ---- storage (src/storage.py) -------------------------------------------- */

/* Loader for OGMS record containers (src/storage.py:43-65, 108-169): the file
 * image `blob` (device, 4-byte aligned) holds nrec share records; record r's
 * payload of nwords[r] uint32 starts at byte src_off[r] and lands at word
 * dst_off[r] of `arena` (device).  Headers are validated by the caller. */
int ogm_unpack_records(const void* blob, int64_t blob_bytes, int64_t nrec, const int64_t* src_off,
                       const int64_t* dst_off, const int32_t* nwords, uint32_t* arena, void* stream);

/* ---- graph outsourcing on the device (src/graphs.py:327-400) -------------
 * ogm_pcg64_u32: out[0..n) = the next n values numpy's
 * Generator(PCG64).integers(0, 2**32, dtype=uint32) would return from the
 * generator state (state, inc: 128-bit little-endian word pairs; has_uint32 /
 * uinteger: numpy's buffered high half).  Jump-ahead per thread, so the
 * stream is drawn in parallel, bit-identical to the host generator.
 * ogm_deal_rows: the three XOR share components of drawn rows
 * (src/graphs.py:327-332): row i's first component is words[s1_off[i] ..
 * + drawn[i]), its second words[s2_off[i] .. + drawn[i]), its third their
 * XOR; words from drawn[i] up to the row pitch are zero (k-padding slots and
 * row padding).  ogm_deal_hot_bits then folds the plaintext one-hot bits into
 * the third component: c3[word[j]] ^= mask[j] (distinct words). */
int ogm_pcg64_u32(const uint64_t* state, const uint64_t* inc, int has_uint32, uint32_t uinteger, int64_t n,
                  uint32_t* out, void* stream);
int ogm_deal_rows(const uint32_t* words, const int64_t* s1_off, const int64_t* s2_off, const int64_t* drawn,
                  int64_t rows, int64_t pitch, uint32_t* c1, uint32_t* c2, uint32_t* c3, void* stream);
int ogm_deal_hot_bits(const int64_t* word, const uint32_t* mask, int64_t n, uint32_t* c3, void* stream);

/* ---- L1 shuffle (src/shuffle.py) ------------------------------------------ */

/* One party-local step of sec_shuffle (src/shuffle.py:106-143):
 *   k2 = perm_outer ? perm_outer[i] : i;  k1 = perm_inner ? perm_inner[k2] : k2
 *   out[i] = m1[k1] ^ m2[k1] ^ T1[k1] ^ T2[k2] ^ m3[i] ^ R[i]
 * Each blinding table term is either a precomputed matrix (*_mat) or an
 * AES-CTR table generated on the fly from (key, label, index) with
 * src/shuffle.py:69-73 layout; all-NULL = absent.  Rows are `words` words
 * wide (= ceil(width_bits/32)), densely packed.  `prf_row0` is the global
 * row of local row 0 (row-sharded tables): the on-the-fly R term at i uses
 * stream row i + prf_row0; T1/T2 are indexed by the (global) permutations.
 * `pitch` (0 = words) is the in-memory row stride of every matrix argument;
 * with a 16-byte pitch (zero padding past `words`) all accesses are 128-bit.
 * The PRF tables follow the reference's dense stream layout regardless. */
int ogm_shuffle_gather(int64_t rows, int64_t words, int64_t width_bits, const int32_t* perm_outer,
                       const int32_t* perm_inner, const uint32_t* m1, const uint32_t* m2,
                       const uint32_t* m3, const uint8_t* t1_key, const uint8_t* t1_label,
                       uint64_t t1_index, const uint32_t* t1_mat, const uint8_t* t2_key,
                       const uint8_t* t2_label, uint64_t t2_index, const uint32_t* t2_mat,
                       const uint8_t* r_key, const uint8_t* r_label, uint64_t r_index,
                       const uint32_t* r_mat, int64_t prf_row0, int64_t pitch, uint32_t* out,
                       void* stream);

/* Offline composition of two known permutations: out[i] = inner[outer[i]]
 * (gather semantics, so M[out] = M[inner][outer] as in src/shuffle.py:76-77). */
int ogm_perm_compose(int64_t n, const int32_t* outer, const int32_t* inner, int32_t* out, void* stream);

/* inv[perm[i]] = i (offline: moves a blind from output order to source order). */
int ogm_perm_invert(int64_t n, const int32_t* perm, int32_t* inv, void* stream);

/* Planned two-pass gather (offline plan for a data-independent permutation):
 * out[i] = (m1 ^ m2 ^ m4)[idx[i]] ^ r_mat[i] ^ m3[i], with bit-identical results
 * to ogm_shuffle_gather, computed as
 *   pass 1: a shared-memory partition of tiles of tile_rows source rows into
 *           `inter` (rows x pitch scratch): inter[gdst[k]] = tile[srow[k]],
 *           one contiguous run per output window of window_rows rows;
 *   pass 2: a gather whose random reads stay inside one contiguous window.
 * ogm_gather_plan derives q2, gdst (n int32 each) and srow (n uint16) from
 * idx (tile_rows <= 16384: each tile is sorted in shared memory, then the
 * (tile, window) counts are scanned per window -- no library sort);
 * ogm_gather_window_rows / ogm_gather_tile_rows give the defaults for a
 * pitch.  m2/m4 are source-order terms XORed in pass 1 (m4: an offline blind
 * already moved to source order), m3/r_mat output-order terms XORed in pass
 * 2 -- pass 2 keeps its window L2-resident only with at most one of them
 * streamed beside it.  `passes` selects pass 1 (bit 0) and/or pass 2 (bit 1).
 * Replaces a direct random-row gather step of src/shuffle.py:106-143. */
int64_t ogm_gather_window_rows(int64_t pitch_words);
int64_t ogm_gather_tile_rows(int64_t pitch_words);
int64_t ogm_gather_plan_workspace_bytes(int64_t n, int64_t window_rows, int64_t tile_rows);
int ogm_gather_plan(int64_t n, const int32_t* idx, int64_t window_rows, int64_t tile_rows, int32_t* q2,
                    int32_t* gdst, uint16_t* srow, void* workspace, int64_t workspace_bytes, void* stream);
/* A plan's run table (offline; the planned form of a src/shuffle.py:106-143
 * gather step): tile t's slots are grouped by destination
 * window with the I rows of a (tile, window) run consecutive, so
 * gdst[s] = off[t*OS + d] + s for global slot s in run d of tile t.
 * start[t*SS + d] (uint16) = the tile slot where run d begins (an empty run:
 * where the next begins), start[t*SS + nwin] = the tile's row count; nwin =
 * ceil(n / window_rows), SS = (nwin + 8) & ~7, OS = (nwin + 3) & ~3
 * (16-byte per-tile strides for bulk copies), start: ceil(n / tile_rows) * SS
 * uint16, off: ceil(n / tile_rows) * OS int32.  tile_rows <= 32768. */
int ogm_gather_plan_runs(int64_t n, int64_t window_rows, int64_t tile_rows, const int32_t* gdst, uint16_t* start,
                         int32_t* off, void* stream);
int ogm_gather_planned(int64_t rows, int64_t words, int64_t pitch, int64_t tile_rows, const int32_t* q2,
                       const int32_t* gdst, const uint16_t* srow, const uint32_t* m1, const uint32_t* m2,
                       const uint32_t* m4, const uint32_t* m3, const uint32_t* r_mat, uint32_t* inter, uint32_t* out,
                       int passes, void* stream);

/* Trio fast path (three co-resident parties): one whole 3-party shuffle of
 * src/shuffle.py:80-144 -- permutations, blinding material and the four
 * online steps -- in one call, bit-identical to the per-party protocol.
 * The rows are packed from `nfields` fields per component (fields[c*nfields
 * + f], c = 0..2; fpitch[c*nfields + f]; fwidth[f]; flags[c] a per-row flag bit vector
 * packed first, or NULL) exactly as ogm_pack_gather does, `width_bits` =
 * packed row width, `pitch` (a multiple of 4) the output row pitch.
 * out[0..2] (rows x pitch) receive the new components R1, R2, R3.  Seeds are
 * HOST pointers (s12 = seed shared by P1/P2, ...); tid = the table id. */
int64_t ogm_trio_shuffle_workspace_bytes(int64_t rows, int64_t pitch);
int ogm_trio_shuffle(const uint8_t* s12, const uint8_t* s23, const uint8_t* s31, uint64_t tid, int64_t rows,
                     int64_t width_bits, int64_t pitch, int nfields, const uint32_t* const* fields,
                     const int64_t* fpitch, const int64_t* fwidth, const uint32_t* const* flags,
                     uint32_t* const* out, void* workspace, int64_t workspace_bytes, void* stream);

/* Trio fast path: open the flag column (bit 0 of every row) of a shuffled
 * table held as three components comps[0..2] (rows x pitch): plain = the
 * XOR of the column (copied to plain_host, words_for(rows) words: the vector
 * every party notes), keep the flagged rows in order, and write each kept
 * row's field f (bits [bit_off[f], +width[f])) of component c to
 * out[c*nfields + f] (capacity rows, pitch opitch[f]).  Synchronous;
 * *kept = number of kept rows (src/engine.py:243-269, 321-334). */
int64_t ogm_trio_open_keep_workspace_bytes(int64_t rows);
int ogm_trio_open_keep(const uint32_t* const* comps, int64_t rows, int64_t pitch, uint32_t* plain_host, int nfields,
                       const int64_t* bit_off, const int64_t* width, uint32_t* const* out, const int64_t* opitch,
                       int64_t* kept, void* workspace, int64_t workspace_bytes, void* stream);

/* The online phase of one 3-party shuffle with prepared material (composed
 * permutations k1 = pi12 o pi31, k3 = pi31 o pi23; permuted combined blinds
 * U, V, W, Z as in shuffle.ShuffleOffline) for 16-byte rows, all four party
 * steps of src/shuffle.py:106-143 in one cooperative launch (two
 * grid-synchronised phases): x1, y1, c1 (optional, may be NULL: it feeds R3
 * at the same index) and the new component r3.  For tables that fit L2
 * (launch-bound sizes). */
int ogm_shuffle_online_fused(int64_t rows, const int32_t* k1, const int32_t* pi12, const int32_t* pi23,
                             const int32_t* k3, const uint32_t* a, const uint32_t* b, const uint32_t* c,
                             const uint32_t* U, const uint32_t* V, const uint32_t* W, const uint32_t* Z, uint32_t* x1,
                             uint32_t* y1, uint32_t* c1, uint32_t* r3, void* stream);

/* The online phase of one 3-party shuffle of 16-byte rows over planned
 * gathers (src/shuffle.py:106-143; the four gathers' plans from
 * ogm_gather_plan in step order x1 (k1), y1 (pi12), c1 (pi23), R3 (k3), tile
 * 4096 rows).  Every blind is in its step's SOURCE order (U', V', W', Z').
 * Each message is handed from sender to receiver tile by tile in shared
 * memory: the sender's window pass feeds the receiver's partition pass in one
 * kernel.  x1, y1, c1 (optional, may be NULL) receive copies of the
 * messages; inter[0..2] are three table-sized scratch buffers.  r3 = the new
 * component R3. */
int ogm_shuffle_online_planned(int64_t rows, const int32_t* const* q2, const int32_t* const* gdst,
                               const uint16_t* const* srow, const uint32_t* a, const uint32_t* b, const uint32_t* c,
                               const uint32_t* u_src, const uint32_t* v_src, const uint32_t* w_src,
                               const uint32_t* z_src, uint32_t* const* inter, uint32_t* x1, uint32_t* y1, uint32_t* c1,
                               uint32_t* r3, void* stream);

/* The preferred order of P2's blind W for ogm_shuffle_online_planned_ex at
 * this table size: 1 = c1's OUTPUT order (large tables: W then streams in
 * c1's window pass and the x1 -> c1 chain kernel skips its XOR pass),
 * 0 = c1's source order like the other blinds. */
int ogm_shuffle_online_planned_w_output_order(int64_t rows);

/* ogm_shuffle_online_planned with the orders of P2's and P3's blinds
 * explicit.  v_order: 0 = y1's source order, 2 = SLOT order of y1's partition
 * plan (srow[1]).  w_order: 0 = c1's source order (x1 rows), 1 = c1's OUTPUT order
 * (W then streams in c1's window pass; faster for the sizes
 * ogm_shuffle_online_planned_w_output_order names), 2 = SLOT order of c1's
 * partition plan (tile t, slot k holds row t*4096 + srow[2][t*4096 + k]: the
 * blind is XORed as rows are scattered, no separate pass).  z_order: 0 =
 * R3's source order (y1 rows), 2 = slot order of R3's partition plan.
 * ABI version 2. */
int ogm_shuffle_online_planned_ex(int64_t rows, const int32_t* const* q2, const int32_t* const* gdst,
                                  const uint16_t* const* srow, const uint32_t* a, const uint32_t* b,
                                  const uint32_t* c, const uint32_t* u_src, const uint32_t* v_src, int v_order,
                                  const uint32_t* w_src, int w_order, const uint32_t* z_src, int z_order,
                                  uint32_t* const* inter, uint32_t* x1, uint32_t* y1, uint32_t* c1, uint32_t* r3,
                                  void* stream);

/* The chained online shuffle with the flat hand-over: each row of the
 * receiver's partition fetches its message row from the sender's window in
 * one streaming pass (no shared-memory staging), in one of two orders:
 *   z_order 3 (I order; the product path): qs[0][p] = q2[0][src2[p]] for
 *     every I row p of c1's plan, src2[p] = the source row that I row holds
 *     (the row of slot s = t*4096 + srow[2][s] at p = gdst[2][s]); qs[1]
 *     the same for y1 -> R3 (q2[1], plan 3).  The pass writes I rows
 *     sequentially and reads no destination index; chunks are interleaved
 *     over the receiver's windows (wrows[2], wrows[3] = its window rows) so
 *     the sender-window reads stay L2-resident.  W (w_order 3) and Z are in
 *     the same I-row order;
 *   z_order 2 (slot order): qs[0][t*4096 + k] = q2[0][t*4096 +
 *     srow[2][t*4096 + k]], the slot scattered through gdst[2]; W (w_order
 *     2) and Z in slot order.
 * w_order 1: W in c1's output order, streamed in c1's window pass (no blind
 * in the hand-over).  U', V' in source order.  run_start / run_off /
 * run_nwin: the four plans' run tables (ogm_gather_plan_runs; arrays of 4,
 * all NULL to read gdst instead): the two partition passes then locate each
 * slot's destination from its tile's table (staged with the tile) instead of
 * reading 4 B of gdst per row.  Same results as
 * ogm_shuffle_online_planned_ex.  ABI version 3. */
int ogm_shuffle_online_planned_slots(int64_t rows, const int32_t* const* q2, const int32_t* const* gdst,
                                     const uint16_t* const* srow, const int32_t* const* qs,
                                     const uint16_t* const* run_start, const int32_t* const* run_off,
                                     const int64_t* run_nwin, const int64_t* wrows, const uint32_t* a,
                                     const uint32_t* b, const uint32_t* c, const uint32_t* u_src,
                                     const uint32_t* v_src, const uint32_t* w_blind, int w_order,
                                     const uint32_t* z_slot, int z_order, uint32_t* const* inter, uint32_t* r3,
                                     void* stream);

/* ---- native trio executor (src/engine.py:352-417 for three co-resident
 * parties) ------------------------------------------------------------------
 * The whole sec_match of the trio fast path in one call: the same launches,
 * in the same order, consuming zero-share counters, table ids and open
 * labels exactly as trio.Trio.match does (bit-identical record shares and
 * opened vectors).  All device buffers the executor creates are carved from
 * `arena`; batches point into it.  Component c of every matrix is party c's
 * share_a (src/graphs.py:382-399). */
#define OGM_TRIO_MAX_ATTRS 8

typedef struct {
    const uint32_t* c[3]; /* three components, rows x pitch words */
    int64_t pitch;        /* words per row in memory */
    int64_t width;        /* logical bits per row */
    int32_t unique;       /* attribute with unique values (Case I route) */
} ogm_trio_mat;

typedef struct {
    int32_t child_type;
    int64_t l_max;        /* posting slots per parent */
    ogm_trio_mat lists;   /* X x (l_max * w(child population)) flattened rows */
} ogm_trio_posting;

typedef struct {
    int64_t population;
    ogm_trio_mat ids;
    int32_t nattrs;
    const ogm_trio_mat* attrs;        /* by attribute id (sorted attribute names) */
    int32_t npostings;
    const ogm_trio_posting* postings;
} ogm_trio_type;

typedef struct {
    int32_t attr;                     /* attribute id of the slot's type */
    int32_t npass;                    /* 1, or 2 for an interval */
    const uint32_t* ind[2][3][2];     /* [pass][party][first/second key] full-domain indicators */
} ogm_trio_pred;

typedef struct {
    int32_t type;
    int32_t combiner_all;             /* 1 ALL, 0 ANY */
    int32_t unique_route;             /* Case I fetch (src/engine.py:382-386) */
    int32_t npreds;
    const ogm_trio_pred* preds;
    int32_t nneeded;                  /* attribute ids of the slot's predicates, sorted by name */
    const int32_t* needed;
    int32_t nchildren;
    const int32_t* children;
} ogm_trio_slot;

typedef struct {
    const uint8_t* zero_key[3];       /* k1, k2, k3 (own zero-share keys) */
    const uint8_t* s12;
    const uint8_t* s23;
    const uint8_t* s31;
    uint64_t counter;                 /* in: next zero-share counter; out: after the query */
    uint64_t table_id;                /* in/out: next shuffle table id */
    uint32_t label;                   /* in/out: last open label */
    int32_t any_xor;                  /* ANY combiner as XOR chain (else logical or) */
    int32_t ntypes;
    const ogm_trio_type* types;
    int32_t nslots;
    const ogm_trio_slot* slots;       /* BFS order: slot 0 is the root */
} ogm_trio_plan;

typedef struct {
    int32_t slot, parent_slot, parent_record; /* -1: root */
    int64_t count;                    /* records in this batch */
    int64_t id_width;
    uint32_t* ids[3];
    int64_t ids_pitch;
    int32_t nattrs;
    int32_t attr_id[OGM_TRIO_MAX_ATTRS];
    int64_t attr_width[OGM_TRIO_MAX_ATTRS];
    uint32_t* attrs[OGM_TRIO_MAX_ATTRS][3];
    int64_t attr_pitch[OGM_TRIO_MAX_ATTRS];
} ogm_trio_batch;

typedef struct {
    int32_t phase;                    /* 0 fetch, 1 access */
    uint32_t label;
    int64_t nbits;
    int64_t bits_off;                 /* word offset into open_bits */
} ogm_trio_open;

typedef struct {
    int32_t max_batches, nbatches;
    ogm_trio_batch* batches;
    int32_t max_opens, nopens;
    ogm_trio_open* opens;
    uint32_t* open_bits;              /* host words */
    int64_t open_bits_cap, open_bits_used;
    int64_t arena_used;               /* bytes; on OGM_ERR_NOMEM, the size that would have been needed so far */
} ogm_trio_out;

int ogm_trio_match(ogm_trio_plan* plan, ogm_trio_out* out, void* arena, int64_t arena_bytes, void* stream);

/* ---- measurement -------------------------------------------------------- */

/* Roofline denominator for the integer-ALU-bound kernels: issue rate of
 * independent LOP3 chains over the whole device (32-bit lane-ops per second),
 * timed with CUDA events on the legacy stream.  Synchronous. */
int ogm_measure_int_peak(double* ops_per_sec, double* seconds);

#ifdef __cplusplus
}
#endif
#endif
