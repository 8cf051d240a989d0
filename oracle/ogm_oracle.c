/*
 * ogm_oracle.c -- CPU restatement of the OblivGM hot path (TEST INFRASTRUCTURE).
 * See ogm_oracle.h.  Plain C99 + pthreads; no dependency on the product.
 *
 * Third-party arithmetic restated here: AES-128 (FIPS-197).  The reference
 * reaches it through `cryptography` (pinned `cryptography>=41`,
 * pkg/pyproject.toml:12; 48.0.0 in the build container) at src/prf.py:30-38
 * (ECB) and src/prf.py:83-84 (CTR).  The S-box is generated from its
 * published definition (multiplicative inverse in GF(2^8) + affine map), not
 * copied from a table.
 */
#include "ogm_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* Minimal static-partition parallel-for over [0, n) on pthreads. */
typedef void (*range_fn)(void *ctx, int64_t lo, int64_t hi);
typedef struct { range_fn fn; void *ctx; int64_t lo, hi; } range_job;
static void *range_thread(void *p) {
    range_job *j = (range_job *)p;
    j->fn(j->ctx, j->lo, j->hi);
    return NULL;
}
static void parallel_for(int64_t n, int nthreads, range_fn fn, void *ctx) {
    if (nthreads <= 1 || n < 2) { fn(ctx, 0, n); return; }
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    range_job jobs[256];
    int64_t chunk = (n + nthreads - 1) / nthreads;
    int used = 0;
    for (int i = 0; i < nthreads; i++) {
        int64_t lo = i * chunk, hi = lo + chunk < n ? lo + chunk : n;
        if (lo >= hi) break;
        jobs[i] = (range_job){fn, ctx, lo, hi};
        pthread_create(&th[i], NULL, range_thread, &jobs[i]);
        used++;
    }
    for (int i = 0; i < used; i++) pthread_join(th[i], NULL);
}

/* ------------------------------------------------------------------------ */
/* AES-128                                                                   */
/* ------------------------------------------------------------------------ */

static uint8_t g_sbox[256];
static uint32_t g_t0[256]; /* little-endian column word of MixColumns(S[x],0,0,0) */
static int g_init = 0;

static uint8_t rotl8(uint8_t x, int s) { return (uint8_t)((x << s) | (x >> (8 - s))); }
static uint32_t rotl32(uint32_t x, int s) { return (x << s) | (x >> (32 - s)); }
static uint8_t xtime(uint8_t x) { return (uint8_t)((x << 1) ^ ((x & 0x80) ? 0x1B : 0)); }

static void aes_init(void) {
    if (g_init) return;
    /* walk the multiplicative group with generator 3: p = 3^k, q = 3^-k */
    uint8_t p = 1, q = 1;
    do {
        p = (uint8_t)(p ^ xtime(p));
        q ^= (uint8_t)(q << 1);
        q ^= (uint8_t)(q << 2);
        q ^= (uint8_t)(q << 4);
        if (q & 0x80) q ^= 0x09;
        uint8_t x = (uint8_t)(q ^ rotl8(q, 1) ^ rotl8(q, 2) ^ rotl8(q, 3) ^ rotl8(q, 4));
        g_sbox[p] = (uint8_t)(x ^ 0x63);
    } while (p != 1);
    g_sbox[0] = 0x63;
    for (int i = 0; i < 256; i++) {
        uint8_t s = g_sbox[i];
        uint8_t s2 = xtime(s);
        uint8_t s3 = (uint8_t)(s2 ^ s);
        g_t0[i] = (uint32_t)s2 | ((uint32_t)s << 8) | ((uint32_t)s << 16) | ((uint32_t)s3 << 24);
    }
    g_init = 1;
}

static uint32_t load_le32(const uint8_t *p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
static void store_le32(uint8_t *p, uint32_t v) {
    p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); p[2] = (uint8_t)(v >> 16); p[3] = (uint8_t)(v >> 24);
}

void ogm_or_aes128_expand(const uint8_t key[16], uint32_t rk[44]) {
    aes_init();
    uint8_t rcon = 1;
    for (int i = 0; i < 4; i++) rk[i] = load_le32(key + 4 * i);
    for (int i = 4; i < 44; i++) {
        uint32_t t = rk[i - 1];
        if (i % 4 == 0) {
            t = (t >> 8) | (t << 24); /* RotWord on a little-endian word */
            t = (uint32_t)g_sbox[t & 0xff] | ((uint32_t)g_sbox[(t >> 8) & 0xff] << 8) |
                ((uint32_t)g_sbox[(t >> 16) & 0xff] << 16) | ((uint32_t)g_sbox[t >> 24] << 24);
            t ^= rcon;
            rcon = xtime(rcon);
        }
        rk[i] = rk[i - 4] ^ t;
    }
}

static void aes_words(const uint32_t rk[44], const uint32_t in[4], uint32_t out[4]) {
    uint32_t s0 = in[0] ^ rk[0], s1 = in[1] ^ rk[1], s2 = in[2] ^ rk[2], s3 = in[3] ^ rk[3];
    for (int r = 1; r < 10; r++) {
        uint32_t n0 = g_t0[s0 & 0xff] ^ rotl32(g_t0[(s1 >> 8) & 0xff], 8) ^
                      rotl32(g_t0[(s2 >> 16) & 0xff], 16) ^ rotl32(g_t0[s3 >> 24], 24) ^ rk[4 * r];
        uint32_t n1 = g_t0[s1 & 0xff] ^ rotl32(g_t0[(s2 >> 8) & 0xff], 8) ^
                      rotl32(g_t0[(s3 >> 16) & 0xff], 16) ^ rotl32(g_t0[s0 >> 24], 24) ^ rk[4 * r + 1];
        uint32_t n2 = g_t0[s2 & 0xff] ^ rotl32(g_t0[(s3 >> 8) & 0xff], 8) ^
                      rotl32(g_t0[(s0 >> 16) & 0xff], 16) ^ rotl32(g_t0[s1 >> 24], 24) ^ rk[4 * r + 2];
        uint32_t n3 = g_t0[s3 & 0xff] ^ rotl32(g_t0[(s0 >> 8) & 0xff], 8) ^
                      rotl32(g_t0[(s1 >> 16) & 0xff], 16) ^ rotl32(g_t0[s2 >> 24], 24) ^ rk[4 * r + 3];
        s0 = n0; s1 = n1; s2 = n2; s3 = n3;
    }
    uint32_t st[4] = {s0, s1, s2, s3};
    for (int j = 0; j < 4; j++) {
        out[j] = ((uint32_t)g_sbox[st[j] & 0xff] |
                  ((uint32_t)g_sbox[(st[(j + 1) & 3] >> 8) & 0xff] << 8) |
                  ((uint32_t)g_sbox[(st[(j + 2) & 3] >> 16) & 0xff] << 16) |
                  ((uint32_t)g_sbox[st[(j + 3) & 3] >> 24] << 24)) ^ rk[40 + j];
    }
}

void ogm_or_aes128_encrypt(const uint32_t rk[44], const uint8_t in[16], uint8_t out[16]) {
    aes_init();
    uint32_t a[4], b[4];
    for (int j = 0; j < 4; j++) a[j] = load_le32(in + 4 * j);
    aes_words(rk, a, b);
    for (int j = 0; j < 4; j++) store_le32(out + 4 * j, b[j]);
}

/* ------------------------------------------------------------------------ */
/* PRG / PRF / permutation (src/prf.py)                                      */
/* ------------------------------------------------------------------------ */

/* src/prf.py:26-28 -- the three fixed public PRG keys. */
static const char *KEY_HEX[3] = {
    "243f6a8885a308d313198a2e03707344", /* _KEY_LEFT  */
    "a4093822299f31d0082efa98ec4e6c89", /* _KEY_RIGHT */
    "452821e638d01377be5466cf34e90c6c", /* _KEY_CTRL  */
};
static uint32_t g_prg_rk[3][44];
static int g_prg_init = 0;

static int hexval(char c) {
    if (c >= '0' && c <= '9') return c - '0';
    return c - 'a' + 10;
}

static void prg_init(void) {
    if (g_prg_init) return;
    aes_init();
    for (int k = 0; k < 3; k++) {
        uint8_t key[16];
        for (int i = 0; i < 16; i++) key[i] = (uint8_t)(hexval(KEY_HEX[k][2 * i]) * 16 + hexval(KEY_HEX[k][2 * i + 1]));
        ogm_or_aes128_expand(key, g_prg_rk[k]);
    }
    g_prg_init = 1;
}

/* One node expansion, word form.  s: 4 LE words. */
static void prg_node(const uint32_t s[4], uint32_t left[4], uint32_t right[4],
                     int *tl, int *tr, int *v) {
    uint32_t c[4];
    aes_words(g_prg_rk[0], s, left);
    aes_words(g_prg_rk[1], s, right);
    aes_words(g_prg_rk[2], s, c);
    for (int j = 0; j < 4; j++) { left[j] ^= s[j]; right[j] ^= s[j]; }
    uint32_t ctrl = c[0] ^ s[0]; /* low bits of low64(AES_KC(s)) ^ low64(s) */
    *tl = (int)(ctrl & 1);
    *tr = (int)((ctrl >> 1) & 1);
    *v = (int)((ctrl >> 2) & 1);
}

/* Only the control/value bits (src/prf.py:53-56). */
static uint32_t prg_ctrl(const uint32_t s[4]) {
    uint32_t c[4];
    aes_words(g_prg_rk[2], s, c);
    return (c[0] ^ s[0]) & 7u;
}

/* Only one child seed: which = 0 left, 1 right (src/prf.py:51-52). */
static void prg_child(const uint32_t s[4], int which, uint32_t out[4]) {
    aes_words(g_prg_rk[which], s, out);
    for (int j = 0; j < 4; j++) out[j] ^= s[j];
}

static void load_seed(const uint8_t *p, uint32_t s[4]) {
    for (int j = 0; j < 4; j++) s[j] = load_le32(p + 4 * j);
}
static void store_seed(uint8_t *p, const uint32_t s[4]) {
    for (int j = 0; j < 4; j++) store_le32(p + 4 * j, s[j]);
}

void ogm_or_prg_expand(const uint8_t *seeds, int64_t n, uint8_t *left, uint8_t *right,
                       uint8_t *t_left, uint8_t *t_right, uint8_t *value) {
    prg_init();
    for (int64_t i = 0; i < n; i++) {
        uint32_t s[4], l[4], r[4];
        int tl, tr, v;
        load_seed(seeds + 16 * i, s);
        prg_node(s, l, r, &tl, &tr, &v);
        store_seed(left + 16 * i, l);
        store_seed(right + 16 * i, r);
        t_left[i] = (uint8_t)tl;
        t_right[i] = (uint8_t)tr;
        value[i] = (uint8_t)v;
    }
}

/* CTR counter block: big-endian 128-bit integer
 * label(4) || index(8, BE) || 0(4), plus the block number (src/prf.py:82-84). */
static void ctr_block(const uint8_t label[4], uint64_t index, uint64_t blk, uint8_t out[16]) {
    uint64_t hi = ((uint64_t)label[0] << 56) | ((uint64_t)label[1] << 48) | ((uint64_t)label[2] << 40) |
                  ((uint64_t)label[3] << 32) | (index >> 32);
    uint64_t lo = (index << 32);
    uint64_t nlo = lo + blk;
    if (nlo < lo) hi++;
    for (int i = 0; i < 8; i++) out[i] = (uint8_t)(hi >> (56 - 8 * i));
    for (int i = 0; i < 8; i++) out[8 + i] = (uint8_t)(nlo >> (56 - 8 * i));
}

void ogm_or_prf_stream(const uint8_t key[16], const uint8_t label[4], uint64_t index,
                       uint64_t block_offset, uint8_t *out, int64_t nbytes) {
    uint32_t rk[44];
    ogm_or_aes128_expand(key, rk);
    int64_t nblk = (nbytes + 15) / 16;
    for (int64_t b = 0; b < nblk; b++) {
        uint8_t ctr[16], ks[16];
        ctr_block(label, index, block_offset + (uint64_t)b, ctr);
        ogm_or_aes128_encrypt(rk, ctr, ks);
        int64_t take = nbytes - 16 * b < 16 ? nbytes - 16 * b : 16;
        memcpy(out + 16 * b, ks, (size_t)take);
    }
}

void ogm_or_seeded_permutation(const uint8_t key[16], const uint8_t label[4], uint64_t index,
                               int64_t n, int64_t *perm) {
    for (int64_t i = 0; i < n; i++) perm[i] = i;
    if (n < 2) return;
    uint64_t *draws = (uint64_t *)malloc((size_t)(n - 1) * 8);
    ogm_or_prf_stream(key, label, index, 0, (uint8_t *)draws, 8 * (n - 1));
    for (int64_t i = n - 1; i >= 1; i--) {
        uint64_t j = draws[n - 1 - i] % (uint64_t)(i + 1);
        int64_t t = perm[i];
        perm[i] = perm[j];
        perm[j] = t;
    }
    free(draws);
}

/* ------------------------------------------------------------------------ */
/* FSS (src/fss.py)                                                          */
/* ------------------------------------------------------------------------ */

void ogm_or_tree_gen(uint64_t alpha, int bits, const uint8_t root0[16], const uint8_t root1[16],
                     int comparison, uint8_t *seed_cw, uint8_t *ctrl_cw, uint8_t *final_cw) {
    prg_init();
    uint32_t s[2][4];
    int t[2] = {0, 1};
    load_seed(root0, s[0]);
    load_seed(root1, s[1]);
    for (int lvl = 0; lvl < bits; lvl++) {
        int a = (int)((alpha >> (bits - 1 - lvl)) & 1);
        uint32_t L[2][4], R[2][4];
        int tl[2], tr[2], v[2];
        for (int b = 0; b < 2; b++) prg_node(s[b], L[b], R[b], &tl[b], &tr[b], &v[b]);
        int v_cw = v[0] ^ v[1] ^ (comparison ? a : 0);
        uint32_t scw[4];
        for (int j = 0; j < 4; j++) scw[j] = a == 0 ? (R[0][j] ^ R[1][j]) : (L[0][j] ^ L[1][j]);
        int tau_l = tl[0] ^ tl[1] ^ a ^ 1;
        int tau_r = tr[0] ^ tr[1] ^ a;
        store_seed(seed_cw + 16 * lvl, scw);
        ctrl_cw[lvl] = (uint8_t)(tau_l | (tau_r << 1) | (v_cw << 2));
        int tau_keep = a == 0 ? tau_l : tau_r;
        for (int b = 0; b < 2; b++) {
            uint32_t *keep = a == 0 ? L[b] : R[b];
            int keep_t = a == 0 ? tl[b] : tr[b];
            for (int j = 0; j < 4; j++) s[b][j] = keep[j] ^ (t[b] ? scw[j] : 0u);
            t[b] = keep_t ^ (t[b] & tau_keep);
        }
    }
    *final_cw = comparison ? 0 : (uint8_t)(((s[0][0] ^ s[1][0]) & 1u) ^ 1u);
}

typedef struct {
    int bits, comparison;
    const uint64_t *alphas;
    const uint8_t *roots0, *roots1;
    uint8_t *seed_cw, *ctrl_cw, *final_cw;
} gen_ctx;
static void gen_range(void *p, int64_t lo, int64_t hi) {
    gen_ctx *c = (gen_ctx *)p;
    for (int64_t k = lo; k < hi; k++)
        ogm_or_tree_gen(c->alphas[k], c->bits, c->roots0 + 16 * k, c->roots1 + 16 * k, c->comparison,
                        c->seed_cw + (size_t)16 * c->bits * k, c->ctrl_cw + (size_t)c->bits * k,
                        c->final_cw + k);
}

void ogm_or_tree_gen_batch(int64_t K, int bits, const uint64_t *alphas, const uint8_t *roots0,
                           const uint8_t *roots1, int comparison, uint8_t *seed_cw,
                           uint8_t *ctrl_cw, uint8_t *final_cw, int nthreads) {
    prg_init();
    gen_ctx c = {bits, comparison, alphas, roots0, roots1, seed_cw, ctrl_cw, final_cw};
    parallel_for(K, nthreads, gen_range, &c);
}

static int walk_eval(int bits, int comparison, const uint8_t *root, int root_t,
                     const uint8_t *seed_cw, const uint8_t *ctrl_cw, int final_cw, int add_const,
                     uint64_t x) {
    uint32_t s[4];
    int t = root_t & 1, acc = 0;
    load_seed(root, s);
    for (int lvl = 0; lvl < bits; lvl++) {
        int xb = (int)((x >> (bits - 1 - lvl)) & 1);
        uint32_t ctrl = prg_ctrl(s);
        if (comparison && xb == 0) acc ^= (int)((ctrl >> 2) & 1) ^ (t & ((ctrl_cw[lvl] >> 2) & 1));
        uint32_t bs[4];
        prg_child(s, xb, bs);
        int bt = (int)((ctrl >> xb) & 1);
        if (t) {
            uint32_t cw[4];
            load_seed(seed_cw + 16 * lvl, cw);
            for (int j = 0; j < 4; j++) bs[j] ^= cw[j];
            bt ^= (ctrl_cw[lvl] >> xb) & 1;
        }
        memcpy(s, bs, sizeof s);
        t = bt & 1;
    }
    int out = comparison ? acc : (int)(s[0] & 1u) ^ (t & final_cw);
    return (out ^ add_const) & 1;
}

typedef struct {
    int bits, comparison;
    const uint8_t *root, *root_t, *seed_cw, *ctrl_cw, *final_cw, *add_const;
    const uint64_t *points;
    uint8_t *out;
} eval_ctx;
static void eval_range(void *p, int64_t lo, int64_t hi) {
    eval_ctx *c = (eval_ctx *)p;
    for (int64_t k = lo; k < hi; k++)
        c->out[k] = (uint8_t)walk_eval(c->bits, c->comparison, c->root + 16 * k, c->root_t[k],
                                       c->seed_cw + (size_t)16 * c->bits * k,
                                       c->ctrl_cw + (size_t)c->bits * k, c->final_cw[k],
                                       c->add_const[k], c->points[k]);
}

int ogm_or_eval_points(int bits, int comparison, int64_t K, const uint8_t *root,
                       const uint8_t *root_t, const uint8_t *seed_cw, const uint8_t *ctrl_cw,
                       const uint8_t *final_cw, const uint8_t *add_const, const uint64_t *points,
                       uint8_t *out, int nthreads) {
    prg_init();
    if (bits < 64) {
        for (int64_t k = 0; k < K; k++)
            if (points[k] >> bits) return -1;
    }
    eval_ctx c = {bits, comparison, root, root_t, seed_cw, ctrl_cw, final_cw, add_const, points, out};
    parallel_for(K, nthreads, eval_range, &c);
    return 0;
}

/* Depth-first restatement of the breadth-first _full_domain_tree; leaves are
 * emitted in natural index order, as the reference's interleaved BFS does. */
typedef struct {
    uint32_t s[4];
    int t, acc, depth;
    uint64_t index;
} fde_node;

int ogm_or_full_domain(int bits, int comparison, const uint8_t root[16], int root_t,
                       const uint8_t *seed_cw, const uint8_t *ctrl_cw, int final_cw,
                       int add_const, int64_t n, uint32_t *out_words) {
    prg_init();
    if (bits < 63 && n > ((int64_t)1 << bits)) return -1;
    memset(out_words, 0, sizeof(uint32_t) * (size_t)((n + 31) / 32));
    if (n == 0) return 0;
    fde_node *stack = (fde_node *)malloc(sizeof(fde_node) * (size_t)(bits + 2));
    int sp = 0;
    fde_node r;
    load_seed(root, r.s);
    r.t = root_t & 1; r.acc = 0; r.depth = 0; r.index = 0;
    stack[sp++] = r;
    while (sp > 0) {
        fde_node nd = stack[--sp];
        /* prune subtrees entirely past n (the reference truncates to n) */
        uint64_t first_leaf = nd.index << (bits - nd.depth);
        if ((int64_t)first_leaf >= n) continue;
        if (nd.depth == bits) {
            int out = comparison ? nd.acc : (int)(nd.s[0] & 1u) ^ (nd.t & final_cw);
            out = (out ^ add_const) & 1;
            if (out) out_words[nd.index >> 5] |= 1u << (nd.index & 31);
            continue;
        }
        uint32_t L[4], R[4];
        int tl, tr, v;
        prg_node(nd.s, L, R, &tl, &tr, &v);
        int lvl = nd.depth;
        uint8_t cc = ctrl_cw[lvl];
        fde_node lc, rc;
        if (nd.t) {
            uint32_t cw[4];
            load_seed(seed_cw + 16 * lvl, cw);
            for (int j = 0; j < 4; j++) { L[j] ^= cw[j]; R[j] ^= cw[j]; }
        }
        memcpy(lc.s, L, sizeof L);
        memcpy(rc.s, R, sizeof R);
        lc.t = tl ^ (nd.t & (cc & 1));
        rc.t = tr ^ (nd.t & ((cc >> 1) & 1));
        lc.acc = comparison ? (nd.acc ^ v ^ (nd.t & ((cc >> 2) & 1))) : 0;
        rc.acc = comparison ? nd.acc : 0;
        lc.depth = rc.depth = nd.depth + 1;
        lc.index = nd.index * 2;
        rc.index = nd.index * 2 + 1;
        stack[sp++] = rc;
        stack[sp++] = lc;
    }
    free(stack);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Engine helpers (src/engine.py)                                            */
/* ------------------------------------------------------------------------ */

void ogm_or_masked_parity(const uint32_t *da, const uint32_t *db, int64_t rows, int64_t w,
                          const uint32_t *ia, const uint32_t *ib, uint8_t *out) {
    for (int64_t c = 0; c < rows; c++) {
        uint32_t acc = 0;
        for (int64_t k = 0; k < w; k++) acc ^= (da[c * w + k] & ia[k]) ^ (db[c * w + k] & ib[k]);
        out[c] = (uint8_t)(__builtin_popcount(acc) & 1);
    }
}
