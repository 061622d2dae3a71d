// kc_sequence.cu -- F4 multi-kernel capture: a sequence of
// dependent dispatches captured step by step into in-memory snapshots, their
// dependencies derived from the written sets and the pointer parameters, and
// a joint replay that validates every step on the state the previous replays
// left (include/kc.h "F4 multi-kernel capture").
//
// Step k is the PRE_W snapshot of dispatch k: the state before it (stored
// incrementally against step k-1, so only the chunks dispatch k-1 changed are
// copied), its post manifest and the post bytes of its written set W_k.  The
// joint replay restores step `first` once, then re-points the restored handle
// at each following step (kc::restored_rebind) without touching the memory.
#include <sys/stat.h>
#include <sys/types.h>

#include <cerrno>
#include <cstdio>
#include <cstring>
#include <set>
#include <string>
#include <vector>

#include "kc_internal.h"
#include "kc_snapshot_types.h"

using namespace kc;

struct kc_sequence {
    kc_ctx* ctx = nullptr;
    std::vector<kc_snapshot*> steps;
    std::vector<uint8_t> deps;  // n x n, deps[j * n + i] for i < j
};

namespace {

// regions (indices into the step's region list) a pointer-sized kernarg
// parameter points into
std::set<size_t> pointer_regions(const SnapDesc& d) {
    std::set<size_t> out;
    for (const auto& pi : d.layout) {
        if (pi.second != 8 || pi.first + 8 > d.kernarg.size()) continue;
        uint64_t v = 0;
        memcpy(&v, d.kernarg.data() + pi.first, 8);
        for (size_t r = 0; r < d.regions.size(); ++r)
            if (d.regions[r].ok && d.regions[r].r.base <= v && v < d.regions[r].r.base + d.regions[r].r.size)
                out.insert(r);
    }
    return out;
}

// KC_DEP_* flags for every pair i < j (reading R33)
std::vector<uint8_t> dependencies(const std::vector<kc_snapshot*>& steps) {
    const size_t n = steps.size();
    std::vector<uint8_t> deps(n * n, 0);
    std::vector<std::set<size_t>> ptrs(n), wreg(n);
    std::vector<std::set<std::pair<size_t, uint64_t>>> wchunks(n);
    for (size_t k = 0; k < n; ++k) {
        const SnapDesc& d = steps[k]->desc;
        ptrs[k] = pointer_regions(d);
        for (size_t r = 0; r < d.regions.size(); ++r)
            for (uint64_t c : d.regions[r].written) {
                wreg[k].insert(r);
                wchunks[k].insert({r, c});
            }
    }
    for (size_t j = 0; j < n; ++j)
        for (size_t i = 0; i < j; ++i) {
            uint8_t f = 0;
            for (size_t r : ptrs[j])
                if (wreg[i].count(r)) f |= KC_DEP_RAW;
            for (const auto& c : wchunks[j])
                if (wchunks[i].count(c)) {
                    f |= KC_DEP_WAW;
                    break;
                }
            for (size_t r : ptrs[i])
                if (wreg[j].count(r)) f |= KC_DEP_WAR;
            deps[j * n + i] = f;
        }
    return deps;
}

bool same_regions(const SnapDesc& a, const SnapDesc& b) {
    if (a.regions.size() != b.regions.size()) return false;
    for (size_t i = 0; i < a.regions.size(); ++i)
        if (a.regions[i].r.base != b.regions[i].r.base || a.regions[i].r.size != b.regions[i].r.size ||
            a.regions[i].ok != b.regions[i].ok)
            return false;
    return true;
}

}  // namespace

extern "C" kc_status kc_capture_seq(kc_ctx* ctx, const kc_dispatch* ds, size_t n_disp, const kc_region* regions,
                                    size_t n, int host, kc_sequence** out, kc_capture_report* reps) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    if (!ctx || !ds || !n_disp || !out) return KC_ERR_ARG;
    if (ctx->poisoned) return KC_ERR_CUDA;
    *out = nullptr;
    kc_sequence* q = new kc_sequence();
    q->ctx = ctx;
    kc_status worst = KC_OK;
    for (size_t k = 0; k < n_disp; ++k) {
        kc_snapshot* sn = nullptr;
        kc_capture_report rep;
        memset(&rep, 0, sizeof rep);
        const kc_snapshot* base = k ? q->steps.back() : nullptr;
        kc_status st = kc_capture_incr(ctx, &ds[k], regions, n, KC_MODE_PRE_W, base, host, &sn, &rep);
        if (st < 0) {
            kc_seq_free(q);
            return st;
        }
        if (st > 0) worst = st;
        if (k && !same_regions(q->steps[0]->desc, sn->desc)) {  // an allocation came or went mid-sequence
            kc_snapshot_free(sn);
            kc_seq_free(q);
            return set_err(ctx, KC_ERR_ARG, "kc_capture_seq: the region set changed between step 0 and step %zu", k);
        }
        q->steps.push_back(sn);
        if (reps) reps[k] = rep;
    }
    q->deps = dependencies(q->steps);
    *out = q;
    return worst;
}

kc_status kc::make_sequence(kc_ctx* ctx, std::vector<kc_snapshot*>& steps, kc_sequence** out) {
    *out = nullptr;
    for (size_t k = 1; k < steps.size(); ++k)
        if (!same_regions(steps[0]->desc, steps[k]->desc))
            return set_err(ctx, KC_ERR_STATE, "sequence: the region set changed between step 0 and step %zu", k);
    kc_sequence* q = new kc_sequence();
    q->ctx = ctx;
    q->steps.swap(steps);
    q->deps = dependencies(q->steps);
    *out = q;
    return KC_OK;
}

extern "C" size_t kc_seq_length(const kc_sequence* q) { return q ? q->steps.size() : 0; }

extern "C" const kc_snapshot* kc_seq_step(const kc_sequence* q, size_t k) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    return q && k < q->steps.size() ? q->steps[k] : nullptr;
}

extern "C" kc_status kc_seq_deps(const kc_sequence* q, uint8_t* deps, size_t cap) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    if (!q || !deps || cap < q->deps.size()) return KC_ERR_ARG;
    memcpy(deps, q->deps.data(), q->deps.size());
    return KC_OK;
}

extern "C" kc_status kc_seq_save(kc_ctx* ctx, const kc_sequence* q, const char* dir_c) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    if (!ctx || !q || !dir_c) return KC_ERR_ARG;
    const std::string dir(dir_c);
    if (mkdir(dir.c_str(), 0755) != 0 && errno != EEXIST)
        return set_err(ctx, KC_ERR_IO, "kc_seq_save: cannot create %s", dir.c_str());
    const size_t n = q->steps.size();
    std::string js = "{\n  \"format\": \"kc-sequence/1\",\n  \"n\": " + std::to_string(n) + ",\n  \"steps\": [\n";
    for (size_t k = 0; k < n; ++k) {
        char sub[32];
        snprintf(sub, sizeof sub, "step_%03zu", k);
        kc_status st = kc_snapshot_save(ctx, q->steps[k], (dir + "/" + sub).c_str());
        if (st < 0) return st;
        uint64_t w = 0;
        for (const auto& r : q->steps[k]->desc.regions) w += r.written.size();
        js += "    {\"dir\": \"" + std::string(sub) + "\", \"mangled_symbol\": \"" + q->steps[k]->desc.mangled +
              "\", \"written_chunks\": " + std::to_string(w) + "}" + (k + 1 < n ? ",\n" : "\n");
    }
    js += "  ],\n  \"deps\": [";
    for (size_t j = 0; j < n; ++j) {
        js += j ? ", [" : "[";
        for (size_t i = 0; i < n; ++i) js += (i ? ", " : "") + std::to_string(q->deps[j * n + i]);
        js += "]";
    }
    js += "]\n}\n";
    FILE* f = fopen((dir + "/sequence.json").c_str(), "wb");
    if (!f || fwrite(js.data(), 1, js.size(), f) != js.size()) {
        if (f) fclose(f);
        return set_err(ctx, KC_ERR_IO, "kc_seq_save: cannot write sequence.json");
    }
    fclose(f);
    f = fopen((dir + "/sequence_complete").c_str(), "wb");  // sentinel last
    if (!f) return set_err(ctx, KC_ERR_IO, "kc_seq_save: cannot write the sentinel");
    fclose(f);
    return KC_OK;
}

// a kc-sequence/1 directory back into memory (every step fully loaded: the
// steps' shared bytes are not deduplicated)
extern "C" kc_status kc_seq_load(kc_ctx* ctx, const char* dir_c, int host, kc_sequence** out) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    if (!ctx || !dir_c || !out) return KC_ERR_ARG;
    *out = nullptr;
    const std::string dir(dir_c);
    struct stat sb;
    if (stat((dir + "/sequence_complete").c_str(), &sb) != 0)
        return set_err(ctx, KC_ERR_FORMAT, "%s: no sequence_complete sentinel", dir_c);
    std::vector<kc_snapshot*> steps;
    for (size_t k = 0;; ++k) {
        char sub[32];
        snprintf(sub, sizeof sub, "/step_%03zu", k);
        if (stat((dir + sub).c_str(), &sb) != 0) break;
        kc_snapshot* sn = nullptr;
        kc_status st = kc_snapshot_load(ctx, (dir + sub).c_str(), host, &sn);
        if (st != KC_OK) {
            for (auto it = steps.rbegin(); it != steps.rend(); ++it) kc_snapshot_free(*it);
            return st;
        }
        steps.push_back(sn);
    }
    if (steps.empty()) return set_err(ctx, KC_ERR_FORMAT, "%s: no step_NNN directories", dir_c);
    kc_status st = make_sequence(ctx, steps, out);
    if (st != KC_OK)
        for (auto it = steps.rbegin(); it != steps.rend(); ++it) kc_snapshot_free(*it);
    return st;
}

extern "C" void kc_seq_free(kc_sequence* q) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    if (!q) return;
    for (auto it = q->steps.rbegin(); it != q->steps.rend(); ++it) kc_snapshot_free(*it);
    delete q;
}

extern "C" kc_status kc_replay_seq(kc_ctx* ctx, const kc_sequence* q, const kc_seq_replay_opts* o,
                                   kc_seq_step_report* reps, kc_restored** keep) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    if (!ctx || !q || !o || !reps) return KC_ERR_ARG;
    if (keep) *keep = nullptr;
    if (o->count == 0 || o->first >= q->steps.size() || o->count > q->steps.size() - o->first)
        return set_err(ctx, KC_ERR_ARG, "kc_replay_seq: steps [%zu, +%zu) outside a %zu-step sequence", o->first,
                       o->count, q->steps.size());
    kc_tolerance tol = o->tol;
    kc_restored* h = nullptr;
    kc_restore_report rr;
    kc_status st = kc_restore_dev(ctx, q->steps[o->first], &h, &rr);
    if (st != KC_OK) return st;
    // chunk hashes of the live state, ok regions in order; at entry to the first
    // step they are its stored manifest (kc_restore_dev verified every chunk)
    std::vector<kc_region> okregs;
    std::vector<uint64_t> entry;
    for (size_t r = 0; r < h->regions.size(); ++r) {
        if (!h->regions[r].ok) continue;
        okregs.push_back(h->regions[r].r);
        const auto& m = q->steps[o->first]->desc.regions[r].manifest;
        entry.insert(entry.end(), m.begin(), m.end());
    }
    for (size_t i = 0; i < o->count; ++i) {
        const size_t k = o->first + i;
        if (i) {
            st = restored_rebind(ctx, h, q->steps[k]);
            if (st != KC_OK) break;
        }
        kc_seq_step_report& out = reps[i];
        memset(&out, 0, sizeof out);
        const SnapDesc& d = q->steps[k]->desc;
        std::vector<uint8_t> in_w(entry.size(), 0);
        {
            size_t c = 0;
            for (size_t r = 0; r < d.regions.size(); ++r) {
                if (!d.regions[r].ok) continue;
                for (uint64_t j = 0; j < d.regions[r].n_chunks; ++j, ++c)
                    out.inherited_chunks += d.regions[r].manifest.size() != d.regions[r].n_chunks ||
                                            d.regions[r].manifest[j] != entry[c];
                c -= d.regions[r].n_chunks;
                for (uint64_t w : d.regions[r].written) in_w[c + w] = 1;
                c += d.regions[r].n_chunks;
            }
        }
        kc_replay_opts ro;
        memset(&ro, 0, sizeof ro);
        ro.iterations = 1;
        ro.stream = o->stream;
        if (o->image_overrides && o->image_overrides[i]) {
            ro.image_override = o->image_overrides[i];
            ro.image_override_size = o->image_override_sizes ? o->image_override_sizes[i] : 0;
        }
        kc_replay_report rp;
        memset(&rp, 0, sizeof rp);
        st = kc_replay(ctx, h, &ro, &rp);
        if (st != KC_OK) break;
        size_t nrep = 0;
        st = validate_impl(ctx, h, nullptr, 0, &tol, &out.w, 1, &nrep, nullptr, true);
        if (st != KC_OK) break;
        if (nrep == 0) {  // the step wrote nothing: an empty report that passes
            memset(&out.w, 0, sizeof out.w);
            out.w.pass = 1;
        }
        std::vector<uint64_t> post;  // K1 over the live state after the step
        st = hash_regions_sync(ctx, okregs, post, nullptr, nullptr, nullptr, ctx->copy_stream);
        if (st != KC_OK) break;
        for (size_t c = 0; c < post.size(); ++c) out.unexpected_chunks += !in_w[c] && post[c] != entry[c];
        entry.swap(post);
        uint64_t nchk = 0, nmis = 0;
        kc_validate_module_vars(ctx, h, &nchk, &nmis);
        out.modvar_mismatch = nmis;
        out.kernel_ms = rp.kernel_ms_mean;
        out.pass = out.w.differing_bytes == 0 && out.unexpected_chunks == 0 && nmis == 0;
    }
    if (st != KC_OK || !keep) {
        kc_release(h);
        return st;
    }
    *keep = h;
    return KC_OK;
}
