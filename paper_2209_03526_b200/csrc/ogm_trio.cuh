// ogm_trio.cuh -- the trio fast path's whole sec_match (src/engine.py:352-417)
// for three co-resident parties in one host call.
//
// trio.Trio.match issues ~40 C-ABI calls and ~100 tensor allocations per tiny
// query from Python; at C1 size that host work, not the GPU, sets the latency.
// This executor runs the same schedule in C++: the same kernels, in the same
// order, with the same zero-share counters, shuffle table ids and open labels
// (SURVEY Appendix A.6), so its record shares and opened vectors are
// bit-identical to the Python trio path (and through it to the reference).
// Device buffers are carved from a caller-provided arena; host-side state is
// the public provenance (opened counts) only.
#pragma once

#include <vector>

#include "oblivgm_b200.h"
#include "ogm_common.cuh"

namespace ogm {

struct TV3 {  // one bit vector per component
    uint32_t* c[3];
    int64_t nbits;
};

struct TM3 {  // one matrix per component
    uint32_t* c[3];
    int64_t rows, pitch, width;
};

struct TGroup {
    int32_t parent_slot, parent_record;
    int64_t count, id_width;
    TM3 ids;
    int32_t nattrs;
    int32_t attr_id[OGM_TRIO_MAX_ATTRS];
    TM3 attrs[OGM_TRIO_MAX_ATTRS];
};

static inline int64_t wf(int64_t nbits) { return (nbits + 31) / 32; }
static inline int64_t pitch16(int64_t nbits) { return (wf(nbits) + 3) / 4 * 4; }

struct TrioExec {
    ogm_trio_plan* P;
    ogm_trio_out* O;
    uint8_t* arena;
    int64_t cap, used = 0;
    void* st;
    int rc = OGM_OK;

    void* take(int64_t bytes) {
        const int64_t b = (std::max<int64_t>(bytes, 1) + 255) & ~(int64_t)255;
        void* p = used + b <= cap ? arena + used : nullptr;
        used += b;
        if (!p && rc == OGM_OK) rc = OGM_ERR_NOMEM;
        return p;
    }
    bool ok() const { return rc == OGM_OK; }
    void check(int r) {
        if (r != OGM_OK && rc == OGM_OK) rc = r;
    }

    TV3 vec(int64_t nbits) {
        TV3 v;
        for (int q = 0; q < 3; q++) v.c[q] = (uint32_t*)take(wf(nbits) * 4);
        v.nbits = nbits;
        return v;
    }
    static TV3 rot(const TV3& v) {  // party q's second share is component q+1
        TV3 r = v;
        for (int q = 0; q < 3; q++) r.c[q] = v.c[(q + 1) % 3];
        return r;
    }

    // src/rss.py:164-176: comp j := blinded_{j-1}
    TV3 reshare(const TV3& adds) {
        TV3 o = vec(adds.nbits);
        if (!ok()) return o;
        if (adds.nbits)
            check(ogm_zero_share_trio(P->zero_key[0], P->zero_key[1], P->zero_key[2], P->counter, adds.nbits,
                                      adds.c, o.c, st));
        P->counter++;
        TV3 r = o;
        r.c[0] = o.c[2];
        r.c[1] = o.c[0];
        r.c[2] = o.c[1];
        return r;
    }

    TV3 xorv(const TV3& a, const TV3& b) {
        TV3 o = vec(a.nbits);
        if (!ok()) return o;
        for (int q = 0; q < 3; q++) check(ogm_xor_words(wf(a.nbits), a.c[q], b.c[q], nullptr, o.c[q], st));
        return o;
    }

    TV3 and_gate(const TV3& a, const TV3& b) {  // src/rss.py:115-126,179-181
        TV3 o = vec(a.nbits);
        if (!ok()) return o;
        TV3 ra = rot(a), rb = rot(b);
        check(ogm_and_terms(wf(a.nbits), 3, a.c, ra.c, b.c, rb.c, o.c, st));
        return reshare(o);
    }

    const TM3* gattr(const TGroup& g, int32_t attr) const {
        for (int i = 0; i < g.nattrs; i++)
            if (g.attr_id[i] == attr) return &g.attrs[i];
        return nullptr;
    }

    // src/engine.py:139-165, both passes from one read of the shares
    TV3 sec_eval(const TGroup& g, const ogm_trio_pred& pr) {
        TV3 res{};
        const TM3* m = gattr(g, pr.attr);
        if (!m) {
            check(OGM_ERR_ARG);
            return res;
        }
        const int64_t rows = g.count, words = wf(m->width);
        std::vector<TV3> outs;
        const uint32_t* ind[12];
        uint32_t* op[6];
        for (int ps = 0; ps < pr.npass; ps++) {
            TV3 v = vec(rows);
            outs.push_back(v);
            for (int q = 0; q < 3; q++) {
                op[ps * 3 + q] = v.c[q];
                ind[ps * 6 + 2 * q] = pr.ind[ps][q][0];
                ind[ps * 6 + 2 * q + 1] = pr.ind[ps][q][1];
            }
        }
        if (!ok()) return res;
        static const int32_t a_idx[3] = {0, 1, 2}, b_idx[3] = {1, 2, 0};
        const uint32_t* comps[3] = {m->c[0], m->c[1], m->c[2]};
        check(ogm_masked_parity(rows, words, rows ? m->pitch : words, 3, comps, 3, a_idx, b_idx, pr.npass, ind, op,
                                st));
        for (int ps = 0; ps < pr.npass; ps++) {
            TV3 sh = reshare(outs[ps]);
            res = ps == 0 ? sh : xorv(res, sh);
        }
        return res;
    }

    TV3 combine(std::vector<TV3>& bits, bool all) {  // src/engine.py:168-189
        TV3 acc = bits[0];
        for (size_t i = 1; i < bits.size() && ok(); i++) {
            if (all) {
                acc = and_gate(acc, bits[i]);
            } else if (P->any_xor) {
                acc = xorv(acc, bits[i]);
            } else {
                TV3 conj = and_gate(acc, bits[i]);
                acc = xorv(xorv(acc, bits[i]), conj);
            }
        }
        return acc;
    }

    // src/engine.py:95-102 for the three parties: one launch
    TV3 fold(const TV3& flags, const TM3& m) {
        TV3 o = vec(32 * wf(m.width));
        o.nbits = m.width;
        if (!ok()) return o;
        const uint32_t* A[3] = {m.c[0], m.c[1], m.c[2]};
        const uint32_t* B[3] = {m.c[1], m.c[2], m.c[0]};
        const uint32_t* fa[3] = {flags.c[0], flags.c[1], flags.c[2]};
        const uint32_t* fb[3] = {flags.c[1], flags.c[2], flags.c[0]};
        check(ogm_select_fold(m.rows, wf(m.width), m.rows ? m.pitch : wf(m.width), 3, A, B, fa, fb, o.c, st));
        return o;
    }

    int push_batch(int32_t slot, const TGroup& g, int64_t count, const TM3& ids, int nattrs, const int32_t* attr_id,
                   const TM3* attrs) {
        if (O->nbatches >= O->max_batches) {
            check(OGM_ERR_NOMEM);
            return -1;
        }
        ogm_trio_batch& b = O->batches[O->nbatches];
        b.slot = slot;
        b.parent_slot = g.parent_slot;
        b.parent_record = g.parent_record;
        b.count = count;
        b.id_width = g.id_width;
        for (int q = 0; q < 3; q++) b.ids[q] = ids.c[q];
        b.ids_pitch = ids.pitch;
        b.nattrs = nattrs;
        for (int i = 0; i < nattrs; i++) {
            b.attr_id[i] = attr_id[i];
            b.attr_width[i] = attrs[i].width;
            b.attr_pitch[i] = attrs[i].pitch;
            for (int q = 0; q < 3; q++) b.attrs[i][q] = attrs[i].c[q];
        }
        return O->nbatches++;
    }

    // src/engine.py:197-217
    int fetch_unique(int32_t slot, const TGroup& g, const TV3& flags) {
        TV3 ids = reshare(fold(flags, g.ids));
        TM3 idm{{ids.c[0], ids.c[1], ids.c[2]}, 1, wf(g.id_width), g.id_width};
        TM3 am[OGM_TRIO_MAX_ATTRS];
        for (int i = 0; i < g.nattrs; i++) {
            TV3 a = reshare(fold(flags, g.attrs[i]));
            am[i] = TM3{{a.c[0], a.c[1], a.c[2]}, 1, wf(g.attrs[i].width), g.attrs[i].width};
        }
        if (!ok()) return -1;
        return push_batch(slot, g, 1, idm, g.nattrs, g.attr_id, am);
    }

    // one whole shuffle of packed rows (ogm_trio_shuffle); table id consumed
    void shuffle(int64_t rows, int64_t row_width, const TV3* flags, int nf, const TM3* fields, uint32_t* outs[3]) {
        const int64_t P16 = pitch16(row_width);
        for (int q = 0; q < 3; q++) outs[q] = (uint32_t*)take(rows * P16 * 4);
        const int64_t nb = ogm_trio_shuffle_workspace_bytes(rows, P16);
        void* ws = take(nb);
        std::vector<const uint32_t*> mats(3 * nf);
        std::vector<int64_t> pitches(3 * nf), widths(nf);
        for (int c = 0; c < 3; c++)
            for (int f = 0; f < nf; f++) {
                mats[c * nf + f] = fields[f].c[c];
                pitches[c * nf + f] = fields[f].pitch;
            }
        for (int f = 0; f < nf; f++) widths[f] = fields[f].width;
        const uint64_t tid = P->table_id++;
        if (!ok()) return;
        const uint32_t* fl[3] = {flags ? flags->c[0] : nullptr, flags ? flags->c[1] : nullptr,
                                 flags ? flags->c[2] : nullptr};
        check(ogm_trio_shuffle(P->s12, P->s23, P->s31, tid, rows, row_width, P16, nf, mats.data(), pitches.data(),
                               widths.data(), flags ? fl : nullptr, outs, ws, nb, st));
    }

    // open the flag column, keep, slice fields (ogm_trio_open_keep); label consumed
    int64_t open_keep(uint32_t* const sh[3], int64_t rows, int64_t row_width, int phase, int nf, const int64_t* off,
                      const int64_t* width, TM3* got) {
        P->label++;
        const int64_t nw = wf(rows);
        if (O->nopens >= O->max_opens || O->open_bits_used + nw > O->open_bits_cap) {
            check(OGM_ERR_NOMEM);
            return 0;
        }
        std::vector<uint32_t*> outs(3 * nf);
        std::vector<int64_t> opitch(nf);
        for (int f = 0; f < nf; f++) {
            opitch[f] = wf(width[f]);
            for (int c = 0; c < 3; c++) outs[c * nf + f] = (uint32_t*)take(std::max<int64_t>(rows, 1) * opitch[f] * 4);
        }
        const int64_t nb = ogm_trio_open_keep_workspace_bytes(rows);
        void* ws = take(nb);
        if (!ok()) return 0;
        const uint32_t* comps[3] = {sh[0], sh[1], sh[2]};
        int64_t kept = 0;
        uint32_t* host = O->open_bits + O->open_bits_used;
        check(ogm_trio_open_keep(comps, rows, pitch16(row_width), host, nf, off, width, outs.data(), opitch.data(),
                                 &kept, ws, nb, st));
        ogm_trio_open& o = O->opens[O->nopens++];
        o.phase = phase;
        o.label = P->label;
        o.nbits = rows;
        o.bits_off = O->open_bits_used;
        O->open_bits_used += nw;
        for (int f = 0; f < nf; f++)
            got[f] = TM3{{outs[f], outs[nf + f], outs[2 * nf + f]}, kept, opitch[f], width[f]};
        return kept;
    }

    // src/engine.py:220-270
    int fetch_multi(int32_t slot, const TGroup& g, const TV3& flags) {
        const int nf = 1 + g.nattrs;
        TM3 fields[1 + OGM_TRIO_MAX_ATTRS];
        int64_t off[1 + OGM_TRIO_MAX_ATTRS], width[1 + OGM_TRIO_MAX_ATTRS];
        fields[0] = g.ids;
        int64_t o = 1;
        off[0] = 1;
        width[0] = g.id_width;
        o += g.id_width;
        for (int i = 0; i < g.nattrs; i++) {
            fields[1 + i] = g.attrs[i];
            off[1 + i] = o;
            width[1 + i] = g.attrs[i].width;
            o += g.attrs[i].width;
        }
        const int64_t row_width = o;
        uint32_t* sh[3];
        shuffle(g.count, row_width, &flags, nf, fields, sh);
        if (!ok()) return -1;
        TM3 got[1 + OGM_TRIO_MAX_ATTRS];
        const int64_t k = open_keep(sh, g.count, row_width, 0, nf, off, width, got);
        if (!ok()) return -1;
        return push_batch(slot, g, k, got[0], g.nattrs, g.attr_id, got + 1);
    }

    TV3 reshare_matrix(const TM3& adds) {  // src/engine.py:83-92
        TV3 o = vec(32 * adds.rows * adds.pitch);
        if (!ok()) return o;
        if (adds.rows * adds.pitch)
            check(ogm_zero_share_trio_rows(P->zero_key[0], P->zero_key[1], P->zero_key[2], P->counter, adds.rows,
                                           adds.pitch, adds.width, adds.c, o.c, st));
        P->counter++;
        TV3 r = o;
        r.c[0] = o.c[2];
        r.c[1] = o.c[0];
        r.c[2] = o.c[1];
        return r;
    }

    // src/engine.py:278-344
    TGroup access(const ogm_trio_batch& b, int64_t i, int32_t child_slot, int32_t parent_slot, int32_t parent_rec) {
        const ogm_trio_slot& cs = P->slots[child_slot];
        const ogm_trio_type& pt = P->types[P->slots[parent_slot].type];
        const ogm_trio_type& ct = P->types[cs.type];
        TGroup g{};
        g.parent_slot = parent_slot;
        g.parent_record = parent_rec;
        g.id_width = ct.population;
        g.nattrs = cs.nneeded;
        for (int a = 0; a < cs.nneeded; a++) g.attr_id[a] = cs.needed[a];
        const ogm_trio_posting* post = nullptr;
        for (int p = 0; p < pt.npostings; p++)
            if (pt.postings[p].child_type == cs.type) post = &pt.postings[p];
        if (!post) {
            check(OGM_ERR_ARG);
            return g;
        }
        const int64_t x_ne = ct.population, w_ne = wf(x_ne), l_max = post->l_max;
        if (l_max == 0) return g;
        TV3 sel;
        for (int q = 0; q < 3; q++) sel.c[q] = b.ids[q] + i * b.ids_pitch;
        sel.nbits = b.id_width;
        TM3 lists{{(uint32_t*)post->lists.c[0], (uint32_t*)post->lists.c[1], (uint32_t*)post->lists.c[2]},
                  pt.population, post->lists.pitch, 32 * l_max * w_ne};
        TV3 adds = fold(sel, lists);
        TM3 am{{adds.c[0], adds.c[1], adds.c[2]}, l_max, w_ne, x_ne};
        TV3 fetched = reshare_matrix(am);
        TM3 fm{{fetched.c[0], fetched.c[1], fetched.c[2]}, l_max, w_ne, x_ne};
        // row parities of the three components (validity flags)
        TV3 par = vec(l_max);
        uint32_t* ones = (uint32_t*)take(w_ne * 4);
        uint32_t* zeros = (uint32_t*)take(w_ne * 4);
        if (!ok()) return g;
        check(cudaMemsetAsync(ones, 0xff, w_ne * 4, as_stream(st)) == cudaSuccess ? OGM_OK : OGM_ERR_CUDA);
        check(cudaMemsetAsync(zeros, 0, w_ne * 4, as_stream(st)) == cudaSuccess ? OGM_OK : OGM_ERR_CUDA);
        {
            static const int32_t a_idx[3] = {0, 1, 2}, b_idx[3] = {1, 2, 0};
            const uint32_t* comps[3] = {fm.c[0], fm.c[1], fm.c[2]};
            const uint32_t* ind[6] = {ones, zeros, ones, zeros, ones, zeros};
            check(ogm_masked_parity(l_max, w_ne, w_ne, 3, comps, 3, a_idx, b_idx, 1, ind, par.c, st));
        }
        uint32_t* sh[3];
        shuffle(l_max, 1 + x_ne, &par, 1, &fm, sh);
        if (!ok()) return g;
        TM3 got;
        const int64_t off = 1, width = x_ne;
        const int64_t k = open_keep(sh, l_max, 1 + x_ne, 1, 1, &off, &width, &got);
        if (!ok() || k == 0) return g;
        g.count = k;
        g.ids = got;
        for (int a = 0; a < cs.nneeded; a++) {
            const ogm_trio_mat& va = ct.attrs[cs.needed[a]];
            const int64_t n = va.width, w = wf(n), x = x_ne;
            TM3 addm{{nullptr, nullptr, nullptr}, k, w, n};
            int32_t* ws = (int32_t*)take(2 * std::max<int64_t>(x, 1) * 4);
            for (int q = 0; q < 3; q++) addm.c[q] = (uint32_t*)take(k * w * 4);
            if (!ok()) return g;
            for (int q = 0; q < 3; q++)
                check(ogm_select_many(k, x, w, va.pitch, got.c[q], got.c[(q + 1) % 3], got.pitch, va.c[q],
                                      va.c[(q + 1) % 3], addm.c[q], w, ws, st));
            TV3 r = reshare_matrix(addm);
            g.attrs[a] = TM3{{r.c[0], r.c[1], r.c[2]}, k, w, n};
        }
        return g;
    }

    void run() {
        std::vector<std::vector<TGroup>> groups(P->nslots);
        std::vector<std::vector<std::pair<int, int64_t>>> records(P->nslots);
        for (int s = 0; s < P->nslots && ok(); s++) {
            const ogm_trio_slot& sl = P->slots[s];
            const ogm_trio_type& t = P->types[sl.type];
            if (s == 0) {
                TGroup g{};
                g.parent_slot = g.parent_record = -1;
                g.count = t.population;
                g.id_width = t.population;
                g.ids = TM3{{(uint32_t*)t.ids.c[0], (uint32_t*)t.ids.c[1], (uint32_t*)t.ids.c[2]}, t.population,
                            t.ids.pitch, t.population};
                g.nattrs = sl.nneeded;
                for (int a = 0; a < sl.nneeded; a++) {
                    const ogm_trio_mat& m = t.attrs[sl.needed[a]];
                    g.attr_id[a] = sl.needed[a];
                    g.attrs[a] = TM3{{(uint32_t*)m.c[0], (uint32_t*)m.c[1], (uint32_t*)m.c[2]}, t.population, m.pitch,
                                     m.width};
                }
                groups[0].push_back(g);
            }
            for (const TGroup& g : groups[s]) {
                if (g.count == 0) continue;
                std::vector<TV3> bits;
                for (int p = 0; p < sl.npreds && ok(); p++) bits.push_back(sec_eval(g, sl.preds[p]));
                if (!ok()) return;
                TV3 flags = combine(bits, sl.combiner_all != 0);
                if (!ok()) return;
                const int bi = sl.unique_route ? fetch_unique(s, g, flags) : fetch_multi(s, g, flags);
                if (!ok()) return;
                for (int64_t i = 0; i < O->batches[bi].count; i++) records[s].push_back({bi, i});
            }
            for (int c = 0; c < sl.nchildren && ok(); c++) {
                const int child = sl.children[c];
                for (size_t ri = 0; ri < records[s].size() && ok(); ri++) {
                    const auto& rec = records[s][ri];
                    groups[child].push_back(access(O->batches[rec.first], rec.second, child, s, (int32_t)ri));
                }
            }
        }
    }
};

}  // namespace ogm

extern "C" int ogm_trio_match(ogm_trio_plan* plan, ogm_trio_out* out, void* arena, int64_t arena_bytes,
                              void* stream) {
    using namespace ogm;
    OGM_CHECK_ARG(plan && out && arena && plan->nslots >= 1 && plan->types, OGM_ERR_ARG, "bad trio plan");
    for (int s = 0; s < plan->nslots; s++)
        OGM_CHECK_ARG(plan->slots[s].nneeded <= OGM_TRIO_MAX_ATTRS && plan->slots[s].npreds >= 1, OGM_ERR_ARG,
                      "slot %d: 1..%d predicates' attributes required", s, OGM_TRIO_MAX_ATTRS);
    OGM_ENSURE_INIT();
    TrioExec ex;
    ex.P = plan;
    ex.O = out;
    ex.arena = (uint8_t*)arena;
    ex.cap = arena_bytes;
    ex.st = stream;
    out->nbatches = 0;
    out->nopens = 0;
    out->open_bits_used = 0;
    ex.run();
    out->arena_used = ex.used;
    if (ex.rc == OGM_ERR_NOMEM) set_error("trio executor out of arena or output space (%lld bytes used)",
                                          (long long)ex.used);
    return ex.rc;
}
