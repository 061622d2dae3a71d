// kc_snapshot.cu -- the address-space closure on CUDA: kc_capture (A3/A5),
// kc_restore (A6), kc_replay (A7), kc_validate (A8), kc_prereserve.
//
// Snapshot format kc-snapshot/1 (names mirror
// the paper's capture directory):
//   dispatch.json, kernarg.bin, kernel.cubin, memory_regions.json,
//   memory/region_<hex>.bin (+ .xxh64 manifest), post/region_<hex>.xxh64,
//   written/region_<hex>.idx + .bin (PRE_W), capture_log.json, capture_complete.
// Ordering and crash safety: metadata before any D2H copy,
// per-region copy failures tolerated and logged, the sentinel written last.
#include <errno.h>
#include <signal.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <sys/stat.h>
#include <sys/types.h>
#include <unistd.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <functional>
#include <map>
#include <memory>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kc_internal.h"
#include "kc_json.h"
#include "kc_snapshot_types.h"

using namespace kc;

namespace {

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// KC_TRACE=1: stage times of the in-memory capture on stderr (diagnostics only)
bool trace_on() {
    static const bool on = [] {
        const char* e = getenv("KC_TRACE");
        return e && *e && *e != '0';
    }();
    return on;
}
void trace(const char* what, double& tl) {
    nvtxMarkA(what);  // stage boundary on the timeline (the stage named ends here)
    if (!trace_on()) return;
    const double t = now_s();
    fprintf(stderr, "[kc] %-28s %9.3f ms\n", what, 1e3 * (t - tl));
    tl = t;
}

bool mkdir_p(const std::string& path) {
    std::string cur;
    for (size_t i = 0; i < path.size(); ++i) {
        cur += path[i];
        if (path[i] == '/' || i + 1 == path.size()) {
            if (cur.size() > 1 && mkdir(cur.c_str(), 0755) != 0 && errno != EEXIST) return false;
        }
    }
    return true;
}

bool write_file(const std::string& path, const void* data, size_t n) {
    FILE* f = fopen(path.c_str(), "wb");
    if (!f) return false;
    bool ok = n == 0 || fwrite(data, 1, n, f) == n;
    ok = (fclose(f) == 0) && ok;
    return ok;
}

bool write_text(const std::string& path, const std::string& s) { return write_file(path, s.data(), s.size()); }

bool read_bin(const std::string& path, std::vector<uint8_t>& out) {
    FILE* f = fopen(path.c_str(), "rb");
    if (!f) return false;
    fseek(f, 0, SEEK_END);
    long n = ftell(f);
    fseek(f, 0, SEEK_SET);
    out.resize(n > 0 ? (size_t)n : 0);
    bool ok = n <= 0 || fread(out.data(), 1, (size_t)n, f) == (size_t)n;
    fclose(f);
    return ok;
}

bool read_u64s(const std::string& path, std::vector<uint64_t>& out) {
    std::vector<uint8_t> b;
    if (!read_bin(path, b) || b.size() % 8) return false;
    out.resize(b.size() / 8);
    memcpy(out.data(), b.data(), b.size());  // little-endian host (x86-64), reading R5
    return true;
}

std::string hex16(uint64_t v) {
    char b[32];
    snprintf(b, sizeof b, "%016llx", (unsigned long long)v);
    return b;
}

// ------------------------------------------------------------------ pinned ring D2H / H2D
// Streams [base, base+size) to a FILE through ctx->depth pinned buffers of
// ctx->io_chunk bytes (KERNCAP_SNAPSHOT_CHUNK_BYTES): the DMA
// of piece i overlaps the file write of piece i-1.
bool d2h_stream(kc_ctx* ctx, uint64_t base, uint64_t size, FILE* f, kc_capture_report* rep, std::string& err) {
    const uint64_t io = ctx->io_chunk;
    const uint32_t depth = ctx->depth;
    const uint64_t np = (size + io - 1) / io;
    std::vector<uint64_t> pend(depth, 0);
    bool ok = true;
    auto drain = [&](uint64_t i) {
        const uint32_t slot = i % depth;
        cudaError_t e = cudaEventSynchronize(ctx->pin_ev[slot]);
        if (e != cudaSuccess) { err = cudaGetErrorString(e); ok = false; return; }
        if (ok && f && fwrite(ctx->pinned[slot], 1, pend[slot], f) != pend[slot]) { err = "fwrite failed"; ok = false; }
    };
    for (uint64_t i = 0; i < np && ok; ++i) {
        const uint32_t slot = i % depth;
        if (i >= depth) drain(i - depth);
        if (!ok) break;
        const uint64_t b = std::min(io, size - i * io);
        cudaError_t e = cudaMemcpyAsync(ctx->pinned[slot], (const void*)(base + i * io), b, cudaMemcpyDeviceToHost,
                                        ctx->copy_stream);
        if (e != cudaSuccess) {
            cudaGetLastError();
            err = std::string("cudaMemcpyAsync D2H: ") + cudaGetErrorString(e);
            ok = false;
            break;
        }
        cudaEventRecord(ctx->pin_ev[slot], ctx->copy_stream);
        pend[slot] = b;
        if (rep) {
            rep->dma_calls += 1;
            rep->d2h_bytes += b;
            rep->staging_high_water = std::max<uint64_t>(rep->staging_high_water, std::min<uint64_t>(i + 1, depth) * io);
        }
    }
    // drain the tail in order
    const uint64_t first = np > depth ? np - depth : 0;
    for (uint64_t i = first; i < np; ++i)
        if (ok) drain(i);
    cudaStreamSynchronize(ctx->copy_stream);
    return ok;
}

// Gather (K4) many device ranges into a device staging buffer, then D2H into
// the file in io pieces.  Used for the written chunks W.
bool gather_d2h(kc_ctx* ctx, const std::vector<std::pair<uint64_t, uint64_t>>& ranges, FILE* f, void* d_stage,
                uint64_t stage_bytes, uint64_t* d_tab, kc_capture_report* rep, std::string& err) {
    size_t i = 0;
    while (i < ranges.size()) {
        std::vector<uint64_t> src, dst, len;
        uint64_t off = 0;
        while (i < ranges.size() && off + ranges[i].second <= stage_bytes) {
            src.push_back(ranges[i].first);
            dst.push_back((uint64_t)d_stage + off);
            len.push_back(ranges[i].second);
            off += ranges[i].second;
            ++i;
        }
        if (src.empty()) { err = "range larger than staging"; return false; }
        const int n = (int)src.size();
        cudaMemcpyAsync(d_tab, src.data(), 8 * n, cudaMemcpyHostToDevice, ctx->copy_stream);
        cudaMemcpyAsync(d_tab + n, dst.data(), 8 * n, cudaMemcpyHostToDevice, ctx->copy_stream);
        cudaMemcpyAsync(d_tab + 2 * n, len.data(), 8 * n, cudaMemcpyHostToDevice, ctx->copy_stream);
        launch_gather(d_tab, d_tab + n, d_tab + 2 * n, n, ctx->copy_stream);
        cudaError_t e = cudaMemcpyAsync(ctx->pinned[0], d_stage, off, cudaMemcpyDeviceToHost, ctx->copy_stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->copy_stream);
        if (e != cudaSuccess) { err = cudaGetErrorString(e); return false; }
        if (rep) { rep->dma_calls += 1; rep->d2h_bytes += off; }
        if (fwrite(ctx->pinned[0], 1, off, f) != off) { err = "fwrite failed"; return false; }
    }
    return true;
}

// ------------------------------------------------------------------ parallel file I/O
// Snapshot files are written/read by KC_IO_THREADS worker threads (default 8),
// each with its own stream and `depth` pinned buffers of io_chunk bytes; big
// regions are split into 256 MiB work items at file offsets (pwrite/pread).
// Host-side memcpy into the page cache is what bounds a file sink, so the
// threads overlap it across cores while each stream keeps PCIe busy.
int io_threads() {
    const char* e = getenv("KC_IO_THREADS");
    int t = e && *e ? atoi(e) : 8;
    return t < 1 ? 1 : (t > 64 ? 64 : t);
}

struct IoItem {
    size_t region;
    uint64_t off, len;
};

std::vector<IoItem> make_items(const std::vector<std::pair<size_t, uint64_t>>& regions /* (index, size) */) {
    const uint64_t piece = 256ull << 20;
    std::vector<IoItem> items;
    for (auto& r : regions)
        for (uint64_t o = 0; o < r.second; o += piece) items.push_back({r.first, o, std::min(piece, r.second - o)});
    // largest first keeps the tail short
    std::stable_sort(items.begin(), items.end(), [](const IoItem& a, const IoItem& b) { return a.len > b.len; });
    return items;
}

kc_status ensure_io(kc_ctx* ctx, int T) {
    while ((int)ctx->io.size() < T) {
        kc_ctx::IoWorker w;
        KC_CHECK_CUDA(ctx, cudaStreamCreateWithFlags(&w.stream, cudaStreamNonBlocking), "cudaStreamCreate(io)");
        for (uint32_t i = 0; i < ctx->depth; ++i) {
            void* p = nullptr;
            cudaError_t e = cudaHostAlloc(&p, ctx->io_chunk, cudaHostAllocDefault);
            if (e != cudaSuccess) return cuda_err(ctx, e, "cudaHostAlloc(io staging)");
            w.pinned.push_back(p);
            cudaEvent_t ev;
            KC_CHECK_CUDA(ctx, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
            w.ev.push_back(ev);
        }
        ctx->io.push_back(w);
    }
    return KC_OK;
}

template <class F>
void run_pool(int T, size_t n, F fn) {
    std::atomic<size_t> next{0};
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
            size_t i;
            while ((i = next.fetch_add(1)) < n) fn(t, i);
        });
    for (auto& x : th) x.join();
}

// One work item device -> file (fd opened O_WRONLY by the caller's worker).
bool item_d2h(kc_ctx* ctx, kc_ctx::IoWorker& w, uint64_t base, const IoItem& it, int fd, std::atomic<uint64_t>& calls,
              std::string& err) {
    const uint64_t io = ctx->io_chunk;
    const uint32_t depth = (uint32_t)w.pinned.size();
    const uint64_t np = (it.len + io - 1) / io;
    std::vector<uint64_t> pend(depth, 0), poff(depth, 0);
    bool ok = true;
    auto drain = [&](uint64_t i) {
        const uint32_t slot = i % depth;
        if (cudaEventSynchronize(w.ev[slot]) != cudaSuccess) { err = "D2H failed"; ok = false; return; }
        if (ok && pwrite(fd, w.pinned[slot], pend[slot], (off_t)poff[slot]) != (ssize_t)pend[slot]) {
            err = "pwrite failed";
            ok = false;
        }
    };
    for (uint64_t i = 0; i < np && ok; ++i) {
        const uint32_t slot = i % depth;
        if (i >= depth) drain(i - depth);
        if (!ok) break;
        const uint64_t o = it.off + i * io, b = std::min(io, it.off + it.len - o);
        cudaError_t e = cudaMemcpyAsync(w.pinned[slot], (const void*)(base + o), b, cudaMemcpyDefault, w.stream);
        if (e != cudaSuccess) {
            cudaGetLastError();
            err = std::string("cudaMemcpyAsync D2H: ") + cudaGetErrorString(e);
            ok = false;
            break;
        }
        cudaEventRecord(w.ev[slot], w.stream);
        pend[slot] = b;
        poff[slot] = o;
        calls.fetch_add(1);
    }
    const uint64_t first = np > depth ? np - depth : 0;
    for (uint64_t i = first; i < np; ++i)
        if (ok) drain(i);
    cudaStreamSynchronize(w.stream);
    return ok;
}

bool item_h2d(kc_ctx* ctx, kc_ctx::IoWorker& w, int fd, uint64_t base, const IoItem& it, std::string& err) {
    const uint64_t io = ctx->io_chunk;
    const uint32_t depth = (uint32_t)w.pinned.size();
    const uint64_t np = (it.len + io - 1) / io;
    for (uint64_t i = 0; i < np; ++i) {
        const uint32_t slot = i % depth;
        if (i >= depth) cudaEventSynchronize(w.ev[slot]);
        const uint64_t o = it.off + i * io, b = std::min(io, it.off + it.len - o);
        if (pread(fd, w.pinned[slot], b, (off_t)o) != (ssize_t)b) {
            err = "short read";
            cudaStreamSynchronize(w.stream);
            return false;
        }
        cudaError_t e = cudaMemcpyAsync((void*)(base + o), w.pinned[slot], b, cudaMemcpyHostToDevice, w.stream);
        if (e != cudaSuccess) {
            err = cudaGetErrorString(e);
            cudaStreamSynchronize(w.stream);
            return false;
        }
        cudaEventRecord(w.ev[slot], w.stream);
    }
    return cudaStreamSynchronize(w.stream) == cudaSuccess;
}

// ------------------------------------------------------------------ F3 module variables + code object
// (PAPER.md:506-516, 728-751).  The dispatch's module: the one kc loaded from
// the given image, else the function's own (cuFuncGetModule).  Its code object:
// the given image, else the bytes the CUPTI hook recorded when the application
// loaded the module.  Variables: the code object's ELF symbols (kc_module.cu)
// resolved in that module with cuModuleGetGlobal; read before and after.
struct ModCapture {
    CUmodule mod = nullptr;
    std::vector<uint8_t> image;
    std::vector<ModVarState> vars;
    std::vector<CUdeviceptr> addr;
};

bool modvars_disabled() {
    const char* e = getenv("KC_NO_MODULE_VARS");
    return e && *e && *e != '0';
}

kc_status module_capture_pre(kc_ctx* ctx, const kc_dispatch* d, CUfunction f, CUmodule own_mod, ModCapture& mc) {
    mc.mod = own_mod;
    if (!mc.mod && KC_DRV(cuFuncGetModule)(&mc.mod, f) != CUDA_SUCCESS) mc.mod = nullptr;
    if (d->image) {
        const size_t n = image_size(d->image, d->image_size);
        if (n) mc.image.assign((const uint8_t*)d->image, (const uint8_t*)d->image + n);
    } else if (mc.mod) {
        std::lock_guard<std::mutex> lk(ctx->mu);
        auto it = ctx->code_objects.find(mc.mod);
        if (it != ctx->code_objects.end()) mc.image = it->second;
    }
    if (!mc.mod || mc.image.empty() || modvars_disabled()) return KC_OK;
    for (const ModVarDecl& v : image_module_vars(mc.image.data(), mc.image.size())) {
        CUdeviceptr p = 0;
        size_t bytes = 0;
        if (KC_DRV(cuModuleGetGlobal)(&p, &bytes, mc.mod, v.name.c_str()) != CUDA_SUCCESS || !p || !bytes) continue;
        ModVarState s;
        s.name = v.name;
        s.section = v.section;
        s.size = bytes;
        s.pre.resize(bytes);
        KC_CHECK_CUDA(ctx, cudaMemcpy(s.pre.data(), (const void*)p, bytes, cudaMemcpyDeviceToHost), "module variable");
        mc.vars.push_back(std::move(s));
        mc.addr.push_back(p);
    }
    return KC_OK;
}

kc_status module_capture_post(kc_ctx* ctx, ModCapture& mc) {
    for (size_t i = 0; i < mc.vars.size(); ++i) {
        mc.vars[i].post.resize(mc.vars[i].size);
        KC_CHECK_CUDA(ctx, cudaMemcpy(mc.vars[i].post.data(), (const void*)mc.addr[i], mc.vars[i].size,
                                      cudaMemcpyDeviceToHost), "module variable (post)");
    }
    return KC_OK;
}

// module_vars.json + module_vars/NNN.{pre,post}.bin
bool write_module_vars(const std::string& dir, const std::vector<ModVarState>& vars) {
    if (vars.empty()) return true;
    if (!mkdir_p(dir + "/module_vars")) return false;
    std::string j = "{\n  \"format\": \"kc-module-vars/1\",\n  \"vars\": [";
    for (size_t i = 0; i < vars.size(); ++i) {
        char idx[24];
        snprintf(idx, sizeof idx, "%03zu", i);
        const std::string pre = std::string("module_vars/") + idx + ".pre.bin";
        const std::string post = std::string("module_vars/") + idx + ".post.bin";
        if (!write_file(dir + "/" + pre, vars[i].pre.data(), vars[i].size) ||
            !write_file(dir + "/" + post, vars[i].post.data(), vars[i].size))
            return false;
        char buf[128];
        snprintf(buf, sizeof buf, "\"size\": %llu, ", (unsigned long long)vars[i].size);
        j += std::string(i ? "," : "") + "\n    {\"name\": \"" + kcj::esc(vars[i].name) + "\", \"section\": \"" +
             kcj::esc(vars[i].section) + "\", " + buf + "\"pre\": \"" + pre + "\", \"post\": \"" + post +
             "\", \"written\": " + (vars[i].pre != vars[i].post ? "true" : "false") + "}";
    }
    j += "\n  ]\n}\n";
    return write_text(dir + "/module_vars.json", j);
}

// ------------------------------------------------------------------ kc-snapshot/1 writers
// Shared by kc_capture (file sink) and kc_snapshot_save (device snapshot).
struct MetaRegion {
    uint64_t base, size, n_chunks, digest, seq;
    int kind, device;
    bool ok;
};
struct LogRegion {
    uint64_t base, post_digest, written;
    bool ok;
    std::string error;
};

std::string dispatch_json(int mode, const std::string& mangled, const uint32_t grid[3], const uint32_t block[3],
                          uint32_t smem, uint32_t kernarg_size, int device, const std::vector<uint8_t>& image,
                          const std::vector<std::pair<size_t, size_t>>& layout, const uint32_t cluster[3],
                          uint32_t flags) {
    const size_t image_size = image.size();
    int cc_major = 0, cc_minor = 0;
    cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, device);
    cudaDeviceGetAttribute(&cc_minor, cudaDevAttrComputeCapabilityMinor, device);
    std::string j = "{\n";
    j += "  \"format\": \"kc-snapshot/1\",\n";
    j += std::string("  \"mode\": \"") + (mode == KC_MODE_PRE_W ? "pre_w" : "post") + "\",\n";
    j += "  \"mangled_symbol\": \"" + kcj::esc(mangled) + "\",\n";
    j += std::string("  \"cooperative\": ") + ((flags & KC_LAUNCH_COOPERATIVE) ? "true" : "false") + ",\n";
    char b[512];
    snprintf(b, sizeof b,
             "  \"grid\": [%u, %u, %u],\n  \"block\": [%u, %u, %u],\n  \"cluster\": [%u, %u, %u],\n"
             "  \"shared_mem_bytes\": %u,\n  \"kernarg_size\": %u,\n  \"device_ordinal\": %d,\n"
             "  \"compute_capability\": \"%d.%d\",\n  \"code_object_bytes\": %zu,\n",
             grid[0], grid[1], grid[2], block[0], block[1], block[2], cluster[0], cluster[1], cluster[2], smem,
             kernarg_size, device, cc_major, cc_minor, image_size);
    j += b;
    j += "  \"kernarg_layout\": [";
    for (size_t i = 0; i < layout.size(); ++i) {
        snprintf(b, sizeof b, "%s{\"offset\": %zu, \"size\": %zu}", i ? ", " : "", layout[i].first, layout[i].second);
        j += b;
    }
    j += "],\n  \"code_object_sha256\": \"" + (image.empty() ? std::string() : sha256_hex(image.data(), image.size())) +
         "\",\n  \"hash\": {\"algo\": \"xxh64\", \"seed\": 0, \"chunk_bytes\": 65536}\n}\n";
    return j;
}

std::string regions_json(const std::vector<MetaRegion>& rs) {
    std::string m = "[\n";
    char b[512];
    for (size_t i = 0; i < rs.size(); ++i) {
        const MetaRegion& r = rs[i];
        const std::string hx = hex_base(r.base);
        const char* kind = r.kind == KC_KIND_VMM ? "vmm" : (r.kind == KC_KIND_POOL ? "pool" : "mem_alloc");
        snprintf(b, sizeof b,
                 "  {\"base\": \"%s\", \"size\": %llu, \"alloc_kind\": \"%s\", \"device\": %d, "
                 "\"contains_kernarg\": false, \"data_file\": \"memory/region_%s.bin\", \"n_chunks\": %llu, "
                 "\"digest\": \"%s\", \"status\": \"%s\", \"seq\": %llu}%s\n",
                 hx.c_str(), (unsigned long long)r.size, kind, r.device, hx.c_str(), (unsigned long long)r.n_chunks,
                 hex16(r.digest).c_str(), r.ok ? "ok" : "failed", (unsigned long long)r.seq,
                 i + 1 < rs.size() ? "," : "");
        m += b;
    }
    return m + "]\n";
}

std::string capture_log_json(const std::vector<LogRegion>& rs, const kc_capture_report& rep, uint64_t io_chunk,
                             uint32_t depth, const char* sink) {
    std::string out = "{\n  \"regions\": [\n";
    char b[768];
    for (size_t i = 0; i < rs.size(); ++i) {
        snprintf(b, sizeof b,
                 "    {\"base\": \"%s\", \"status\": \"%s\", \"error\": \"%s\", \"post_digest\": \"%s\", "
                 "\"written_chunks\": %llu}%s\n",
                 hex_base(rs[i].base).c_str(), rs[i].ok ? "ok" : "failed", kcj::esc(rs[i].error).c_str(),
                 hex16(rs[i].post_digest).c_str(), (unsigned long long)rs[i].written, i + 1 < rs.size() ? "," : "");
        out += b;
    }
    snprintf(b, sizeof b,
             "  ],\n  \"sink\": \"%s\",\n  \"snapshot_digest\": \"%s\",\n  \"written_chunks\": %llu,\n"
             "  \"d2h_bytes\": %llu,\n  \"dma_calls\": %llu,\n  \"io_chunk_bytes\": %llu,\n  \"pinned_depth\": %u,\n"
             "  \"staging_high_water\": %llu,\n  \"t_hash_pre_s\": %.6f,\n  \"t_d2h_s\": %.6f,\n"
             "  \"t_dispatch_s\": %.6f,\n  \"t_hash_post_s\": %.6f,\n  \"t_total_s\": %.6f\n}\n",
             sink, hex16(rep.snapshot_digest).c_str(), (unsigned long long)rep.written_chunks,
             (unsigned long long)rep.d2h_bytes, (unsigned long long)rep.dma_calls, (unsigned long long)io_chunk, depth,
             (unsigned long long)rep.staging_high_water, rep.t_hash_pre_s, rep.t_d2h_s, rep.t_dispatch_s,
             rep.t_hash_post_s, rep.t_total_s);
    return out + b;
}

struct RegionState {
    kc_region r;
    bool ok = true;
    bool failed_pre = false;  // not live before the dispatch: never in any S
    std::string error;
    uint64_t chunk0 = 0;  // index into the manifest arrays (ok regions only)
    uint64_t n_chunks = 0;
    uint64_t pre_digest = 0, post_digest = 0;
    std::vector<uint64_t> written;
};

}  // namespace

namespace {
// A dispatch launched with more than 48 KiB of dynamic shared memory needs the
// function's opt-in attribute; the application set it on its own CUfunction,
// a module the closure loads itself (capture from an image, replay) must set it
// again before launching with the captured smem size.
}  // namespace

CUresult kc::launch_packed(CUfunction f, const uint32_t grid[3], const uint32_t block[3], uint32_t smem, CUstream s,
                           const void* kernarg, size_t kernarg_size, const uint32_t cluster[3], uint32_t flags) {
    size_t ksz = kernarg_size;
    void* extra[] = {CU_LAUNCH_PARAM_BUFFER_POINTER, (void*)kernarg, CU_LAUNCH_PARAM_BUFFER_SIZE, &ksz,
                     CU_LAUNCH_PARAM_END};
    void** ex = kernarg && kernarg_size ? extra : nullptr;
    CUlaunchAttribute attrs[2];
    memset(attrs, 0, sizeof attrs);
    unsigned na = 0;
    if (cluster && cluster[0] * cluster[1] * cluster[2] > 1) {
        attrs[na].id = CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION;
        attrs[na].value.clusterDim.x = cluster[0];
        attrs[na].value.clusterDim.y = cluster[1];
        attrs[na].value.clusterDim.z = cluster[2];
        ++na;
    }
    if (flags & KC_LAUNCH_COOPERATIVE) {
        attrs[na].id = CU_LAUNCH_ATTRIBUTE_COOPERATIVE;
        attrs[na].value.cooperative = 1;
        ++na;
    }
    if (na) {
        CUlaunchConfig cfg;
        memset(&cfg, 0, sizeof cfg);
        cfg.gridDimX = grid[0], cfg.gridDimY = grid[1], cfg.gridDimZ = grid[2];
        cfg.blockDimX = block[0], cfg.blockDimY = block[1], cfg.blockDimZ = block[2];
        cfg.sharedMemBytes = smem;
        cfg.hStream = s;
        cfg.attrs = attrs;
        cfg.numAttrs = na;
        return KC_DRV(cuLaunchKernelEx)(&cfg, f, nullptr, ex);
    }
    return KC_DRV(cuLaunchKernel)(f, grid[0], grid[1], grid[2], block[0], block[1], block[2], smem, s, nullptr, ex);
}

void kc::dispatch_cluster(const kc_dispatch* d, uint32_t out[3]) {
    for (int i = 0; i < 3; ++i) out[i] = d->cluster[i] ? d->cluster[i] : 1;
}

namespace {
CUresult allow_dynamic_smem(CUfunction f, uint32_t smem) {
    if (smem <= 48u * 1024u) return CUDA_SUCCESS;
    return KC_DRV(cuFuncSetAttribute)(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem);
}
}  // namespace

namespace kc {

// Snapshot digest S (O2, R4) over the regions whose FINAL status is ok: a region
// can fail after the pre/post pass that produced the first S (a D2H or
// written-chunk copy failure, or a buffer freed after the dispatch,
// PAPER.md:753-761), and S must describe exactly the region files written.
kc_status final_snapshot_digest(kc_ctx* ctx, const std::vector<std::array<uint64_t, 3>>& triples, cudaStream_t s,
                                uint64_t* out) {
    const size_t n = triples.size();
    KC_CHECK_CUDA(ctx, ensure(ctx->digest_scratch, 24 * n + 8), "cudaMalloc(digest scratch)");
    uint8_t* d = (uint8_t*)ctx->digest_scratch.p;
    if (n) KC_CHECK_CUDA(ctx, cudaMemcpyAsync(d, triples.data(), 24 * n, cudaMemcpyHostToDevice, s), "upload triples");
    KC_CHECK_CUDA(ctx, launch_snapshot_digest(d, (int)n, (uint64_t*)(d + 24 * n), s), "launch snapshot digest");
    ctx->launches += 1;
    KC_CHECK_CUDA(ctx, cudaMemcpyAsync(out, d + 24 * n, 8, cudaMemcpyDeviceToHost, s), "D2H snapshot digest");
    KC_CHECK_CUDA(ctx, cudaStreamSynchronize(s), "snapshot digest");
    return KC_OK;
}

// Hash a region list (all must be live) and bring the manifest (and digests) to the host.
kc_status hash_regions_sync(kc_ctx* ctx, const std::vector<kc_region>& regs, std::vector<uint64_t>& out_hashes,
                            std::vector<uint64_t>* out_digests, uint64_t* out_snapshot, uint64_t* d_hash_out,
                            cudaStream_t s, const uint64_t* h_dst) {
    const uint64_t C = kc_count_chunks(regs.data(), regs.size());
    uint64_t* d_h = d_hash_out;
    if (!d_h) {
        KC_CHECK_CUDA(ctx, ensure(ctx->tmp_hash, (C + regs.size() + 1) * 8), "cudaMalloc(manifest)");
        d_h = (uint64_t*)ctx->tmp_hash.p;
    }
    uint64_t* d_dig = nullptr;
    uint64_t* d_snap = nullptr;
    kc_ctx_dev_buf dig;
    if (out_digests || out_snapshot) {
        KC_CHECK_CUDA(ctx, ensure(dig, (regs.size() + 1) * 8), "cudaMalloc(digests)");
        d_dig = (uint64_t*)dig.p;
        d_snap = d_dig + regs.size();
    }
    kc_status st = hash_impl(ctx, regs.data(), regs.size(), d_h, d_dig, out_snapshot ? d_snap : nullptr, s, h_dst);
    if (st != KC_OK) {
        if (dig.p) cudaFree(dig.p);
        return st;
    }
    out_hashes.resize(C);
    if (C) KC_CHECK_CUDA(ctx, cudaMemcpyAsync(out_hashes.data(), d_h, C * 8, cudaMemcpyDeviceToHost, s), "D2H manifest");
    std::vector<uint64_t> tmp(regs.size() + 1);
    if (d_dig) KC_CHECK_CUDA(ctx, cudaMemcpyAsync(tmp.data(), d_dig, (regs.size() + 1) * 8, cudaMemcpyDeviceToHost, s),
                             "D2H digests");
    cudaError_t e = cudaStreamSynchronize(s);
    if (dig.p) cudaFree(dig.p);
    if (e != cudaSuccess) return cuda_err(ctx, e, "hash sync");
    if (out_digests) out_digests->assign(tmp.begin(), tmp.begin() + regs.size());
    if (out_snapshot) *out_snapshot = regs.empty() ? 0 : tmp[regs.size()];
    return KC_OK;
}

}  // namespace kc

// ====================================================================== capture
extern "C" kc_status kc_capture(kc_ctx* ctx, const kc_dispatch* d, const kc_region* regions, size_t n,
                                const char* dir_c, kc_capture_mode mode, kc_capture_report* rep_out) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    if (!ctx) return KC_ERR_ARG;
    if (ctx->poisoned) return KC_ERR_CUDA;
    if (!bind_device(ctx)) return set_err(ctx, KC_ERR_CUDA, "cannot bind device");
    if (!d || !dir_c) return set_err(ctx, KC_ERR_ARG, "kc_capture: dispatch and dir are required");
    if (mode != KC_MODE_PRE_W && mode != KC_MODE_POST) return set_err(ctx, KC_ERR_ARG, "kc_capture: bad mode");
    kc_capture_report rep;
    memset(&rep, 0, sizeof rep);
    const double t0 = now_s();
    const std::string dir = dir_c;
    cudaStream_t cs = (cudaStream_t)d->stream;

    // ---- region list: given, or every tracked allocation; sorted by base (R25)
    std::vector<kc_region> list;
    if (regions) {
        list.assign(regions, regions + n);
    } else {
        std::lock_guard<std::mutex> lk(ctx->mu);
        for (auto& kv : ctx->live) list.push_back(kv.second);
    }
    list.erase(std::remove_if(list.begin(), list.end(), [](const kc_region& r) { return r.size == 0; }), list.end());
    std::sort(list.begin(), list.end(), [](const kc_region& a, const kc_region& b) { return a.base < b.base; });
    for (size_t i = 1; i < list.size(); ++i)
        if (list[i].base < list[i - 1].base + list[i - 1].size)
            return set_err(ctx, KC_ERR_ARG, "kc_capture: regions overlap at 0x%llx", (unsigned long long)list[i].base);

    // ---- resolve the function (D4 analog) before touching memory
    CUfunction f = (CUfunction)d->func;
    CUmodule own_mod = nullptr;
    if (!f) {
        if (!d->image || !d->mangled) return set_err(ctx, KC_ERR_ARG, "kc_capture: need func or image+mangled");
        KC_CHECK_CU(ctx, KC_DRV(cuModuleLoadData)(&own_mod, d->image), "cuModuleLoadData");
        CUresult r = KC_DRV(cuModuleGetFunction)(&f, own_mod, d->mangled);
        if (r != CUDA_SUCCESS) {
            KC_DRV(cuModuleUnload)(own_mod);
            return set_err(ctx, KC_ERR_ARG, "kc_capture: symbol %s not found in image", d->mangled);
        }
        r = allow_dynamic_smem(f, d->smem_bytes);
        if (r != CUDA_SUCCESS) {
            KC_DRV(cuModuleUnload)(own_mod);
            return cu_err(ctx, r, "kc_capture: dynamic shared memory attribute");
        }
    }
    std::string mangled = d->mangled ? d->mangled : "";
    if (mangled.empty()) {
        const char* nm = nullptr;
        if (KC_DRV(cuFuncGetName)(&nm, f) == CUDA_SUCCESS && nm) mangled = nm;
    }
    // kernarg layout via cuFuncGetParamInfo (reading R22)
    std::vector<std::pair<size_t, size_t>> layout;
    for (size_t i = 0; i < 4096; ++i) {
        size_t off = 0, sz = 0;
        if (KC_DRV(cuFuncGetParamInfo)(f, i, &off, &sz) != CUDA_SUCCESS) break;
        layout.emplace_back(off, sz);
    }

    if (!layout.empty() && d->kernarg && d->kernarg_size != layout.back().first + layout.back().second) {
        if (own_mod) KC_DRV(cuModuleUnload)(own_mod);
        return set_err(ctx, KC_ERR_ARG, "kc_capture: kernarg_size %u != parameter buffer size %zu of %s",
                       d->kernarg_size, layout.back().first + layout.back().second, mangled.c_str());
    }
    kc_status final_st = KC_OK;
    // ---- A3 bracket: quiesce every stream that could write tracked memory
    {
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            if (own_mod) KC_DRV(cuModuleUnload)(own_mod);
            return cuda_err(ctx, e, "kc_capture: quiesce");
        }
    }
    ModCapture mc;  // F3: the dispatch's code object and module variables (pre values)
    {
        kc_status mst = module_capture_pre(ctx, d, f, own_mod, mc);
        if (mst != KC_OK) {
            if (own_mod) KC_DRV(cuModuleUnload)(own_mod);
            return mst;
        }
    }
    std::vector<RegionState> rs(list.size());
    std::vector<kc_region> live;
    for (size_t i = 0; i < list.size(); ++i) {
        rs[i].r = list[i];
        rs[i].n_chunks = (list[i].size + kChunk - 1) / kChunk;
        if (!region_live(ctx, list[i].base, list[i].size)) {
            rs[i].ok = false;
            rs[i].failed_pre = true;
            rs[i].error = "not inside a live CUDA allocation before the dispatch";
        } else {
            rs[i].chunk0 = kc_count_chunks(live.data(), live.size());
            live.push_back(list[i]);
        }
    }
    rep.n_regions = list.size();

    // ---- A2: pre-manifest (K1)
    double t = now_s();
    std::vector<uint64_t> pre_h, pre_dig;
    uint64_t pre_snap = 0;
    kc_status st = hash_regions_sync(ctx, live, pre_h, &pre_dig, &pre_snap, nullptr, cs);
    if (st != KC_OK) {
        if (own_mod) KC_DRV(cuModuleUnload)(own_mod);
        return st;
    }
    rep.t_hash_pre_s = now_s() - t;
    {
        size_t j = 0;
        for (auto& r : rs)
            if (r.ok) r.pre_digest = pre_dig[j++];
    }
    rep.n_chunks = pre_h.size();
    for (auto& r : live) rep.total_bytes += r.size;

    if (!mkdir_p(dir + "/memory") || !mkdir_p(dir + "/post") || !mkdir_p(dir + "/written")) {
        if (own_mod) KC_DRV(cuModuleUnload)(own_mod);
        return set_err(ctx, KC_ERR_IO, "kc_capture: cannot create %s", dir.c_str());
    }
    unlink((dir + "/capture_complete").c_str());  // sentinel-last
    st = ensure_pinned(ctx);
    if (st != KC_OK) {
        if (own_mod) KC_DRV(cuModuleUnload)(own_mod);
        return st;
    }

    auto write_metadata = [&](bool post_digests) -> bool {
        uint32_t cl[3];
        dispatch_cluster(d, cl);
        const std::string j = dispatch_json(mode, mangled, d->grid, d->block, d->smem_bytes, d->kernarg_size,
                                            ctx->device, mc.image, layout, cl, d->flags);
        if (!write_text(dir + "/dispatch.json", j)) return false;
        if (!write_file(dir + "/kernarg.bin", d->kernarg, d->kernarg ? d->kernarg_size : 0)) return false;
        if (!mc.image.empty() && !write_file(dir + "/kernel.cubin", mc.image.data(), mc.image.size())) return false;
        std::vector<MetaRegion> mr;
        for (const RegionState& r : rs)
            mr.push_back({r.r.base, r.r.size, r.n_chunks, post_digests ? r.post_digest : r.pre_digest, r.r.seq,
                          r.r.kind, r.r.device, r.ok});
        return write_text(dir + "/memory_regions.json", regions_json(mr));
    };

    // region files: region bytes (parallel workers) + the matching manifest slice
    auto snapshot_regions = [&](const std::vector<uint64_t>& manifest) {
        const int T = io_threads();
        if (ensure_io(ctx, T) != KC_OK) {
            for (auto& r : rs)
                if (r.ok) { r.ok = false; r.error = "cannot allocate pinned I/O staging"; }
            return;
        }
        std::vector<std::pair<size_t, uint64_t>> todo;
        for (size_t i = 0; i < rs.size(); ++i) {
            if (!rs[i].ok) continue;
            const std::string path = dir + "/memory/region_" + hex_base(rs[i].r.base) + ".bin";
            int fd = open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
            if (fd < 0 || ftruncate(fd, (off_t)rs[i].r.size) != 0) {
                rs[i].ok = false;
                rs[i].error = "cannot create " + path;
            } else {
                todo.emplace_back(i, rs[i].r.size);
            }
            if (fd >= 0) close(fd);
        }
        const std::vector<IoItem> items = make_items(todo);
        std::vector<std::atomic<int>> failed(rs.size());
        for (auto& f : failed) f = 0;
        std::mutex emu;
        std::atomic<uint64_t> calls{0};
        run_pool(T, items.size(), [&](int t, size_t k) {
            const IoItem& it = items[k];
            if (failed[it.region]) return;
            cudaSetDevice(ctx->device);
            const std::string path = dir + "/memory/region_" + hex_base(rs[it.region].r.base) + ".bin";
            int fd = open(path.c_str(), O_WRONLY);
            std::string err = fd < 0 ? "cannot open " + path : "";
            const bool ok = fd >= 0 && item_d2h(ctx, ctx->io[t], rs[it.region].r.base, it, fd, calls, err);
            if (fd >= 0) close(fd);
            if (!ok && !failed[it.region].exchange(1)) {
                std::lock_guard<std::mutex> lk(emu);
                rs[it.region].error = err;
            }
        });
        rep.dma_calls += calls.load();
        rep.staging_high_water = std::max<uint64_t>(rep.staging_high_water,
                                                    (uint64_t)std::min<size_t>(T, items.size()) * ctx->depth * ctx->io_chunk);
        for (size_t i = 0; i < rs.size(); ++i) {
            RegionState& r = rs[i];
            if (!r.ok) continue;
            const std::string hx = hex_base(r.r.base);
            if (failed[i]) {
                r.ok = false;
                unlink((dir + "/memory/region_" + hx + ".bin").c_str());
                continue;
            }
            rep.d2h_bytes += r.r.size;
            write_file(dir + "/memory/region_" + hx + ".xxh64", manifest.data() + r.chunk0, 8 * r.n_chunks);
        }
    };

    double t_d2h = 0;
    if (mode == KC_MODE_PRE_W) {
        if (!write_metadata(false)) {
            if (own_mod) KC_DRV(cuModuleUnload)(own_mod);
            return set_err(ctx, KC_ERR_IO, "kc_capture: cannot write metadata in %s", dir.c_str());
        }
        t = now_s();
        snapshot_regions(pre_h);
        t_d2h += now_s() - t;
    }

    // ---- A3: forward the target dispatch, then wait for it
    t = now_s();
    {
        uint32_t cl[3];
        dispatch_cluster(d, cl);
        CUresult r = launch_packed(f, d->grid, d->block, d->smem_bytes, (CUstream)cs, d->kernarg, d->kernarg_size, cl,
                                   d->flags);
        if (r == CUDA_SUCCESS) r = KC_DRV(cuStreamSynchronize)((CUstream)cs);
        if (r != CUDA_SUCCESS) {
            if (own_mod) KC_DRV(cuModuleUnload)(own_mod);
            return cu_err(ctx, r, "kc_capture: target dispatch");
        }
    }
    rep.t_dispatch_s = now_s() - t;
    {
        kc_status mst = module_capture_post(ctx, mc);
        if (own_mod) KC_DRV(cuModuleUnload)(own_mod);
        if (mst != KC_OK) return mst;
    }
    if (!write_module_vars(dir, mc.vars)) return set_err(ctx, KC_ERR_IO, "kc_capture: cannot write module_vars");

    // test hook: a region freed between completion and snapshot
    if (const char* hook = getenv("KC_TEST_FREE_AFTER_DISPATCH")) {
        const uint64_t b = strtoull(hook, nullptr, 16);
        if (b) free_alloc(ctx, b, true);
    }

    // ---- A4: post-manifest + written set
    t = now_s();
    std::vector<kc_region> live2;
    for (auto& r : rs) {
        if (r.ok && !region_live(ctx, r.r.base, r.r.size)) {
            r.ok = false;
            r.error = "freed between dispatch completion and snapshot";
        }
    }
    std::vector<uint64_t> post_h, post_dig;
    uint64_t post_snap = 0;
    {
        // hash every region still ok; remap manifest offsets
        std::vector<uint64_t> off_post(rs.size(), 0);
        for (size_t i = 0; i < rs.size(); ++i)
            if (rs[i].ok) {
                off_post[i] = kc_count_chunks(live2.data(), live2.size());
                live2.push_back(rs[i].r);
            }
        st = hash_regions_sync(ctx, live2, post_h, &post_dig, &post_snap, nullptr, cs);
        if (st != KC_OK) return st;
        size_t j = 0;
        for (size_t i = 0; i < rs.size(); ++i) {
            if (!rs[i].ok) continue;
            RegionState& r = rs[i];
            r.post_digest = post_dig[j++];
            for (uint64_t k = 0; k < r.n_chunks; ++k)
                if (pre_h[r.chunk0 + k] != post_h[off_post[i] + k]) r.written.push_back(k);
            rep.written_chunks += r.written.size();
            r.chunk0 = off_post[i];  // from here on chunk0 indexes post_h
        }
    }
    rep.t_hash_post_s = now_s() - t;

    if (mode == KC_MODE_POST) {
        if (!write_metadata(true)) return set_err(ctx, KC_ERR_IO, "kc_capture: cannot write metadata");
        t = now_s();
        snapshot_regions(post_h);
        t_d2h += now_s() - t;
    }

    // ---- written chunks: indices (+ post bytes in PRE_W) and post manifests
    void* d_stage = nullptr;
    uint64_t* d_tab = nullptr;
    t = now_s();
    for (auto& r : rs) {
        if (!r.ok) continue;
        const std::string hx = hex_base(r.r.base);
        write_file(dir + "/post/region_" + hx + ".xxh64", post_h.data() + r.chunk0, 8 * r.n_chunks);
        write_file(dir + "/written/region_" + hx + ".idx", r.written.data(), 8 * r.written.size());
        if (mode == KC_MODE_PRE_W && !r.written.empty()) {
            if (!d_stage) {
                const uint64_t sb = std::min<uint64_t>(ctx->io_chunk, 64ull << 20);
                if (cudaMalloc(&d_stage, sb) != cudaSuccess || cudaMalloc((void**)&d_tab, 3 * 8 * (sb / 32)) != cudaSuccess)
                    return set_err(ctx, KC_ERR_NOMEM, "kc_capture: staging");
            }
            std::vector<std::pair<uint64_t, uint64_t>> ranges;
            for (uint64_t k : r.written) {
                const uint64_t off = k * kChunk;
                ranges.emplace_back(r.r.base + off, std::min<uint64_t>(kChunk, r.r.size - off));
            }
            const std::string path = dir + "/written/region_" + hx + ".bin";
            FILE* fp = fopen(path.c_str(), "wb");
            std::string err;
            const uint64_t sb = std::min<uint64_t>(ctx->io_chunk, 64ull << 20);
            bool ok = fp && gather_d2h(ctx, ranges, fp, d_stage, sb, d_tab, &rep, err);
            if (fp) ok = (fclose(fp) == 0) && ok;
            if (!ok) {
                r.ok = false;
                r.error = "written-chunk copy failed: " + err;
            }
        }
    }
    if (d_stage) cudaFree(d_stage);
    if (d_tab) cudaFree(d_tab);
    t_d2h += now_s() - t;
    rep.t_d2h_s = t_d2h;

    // ---- capture_log.json, then the sentinel LAST
    rep.snapshot_digest = mode == KC_MODE_PRE_W ? pre_snap : post_snap;  // S of the region files written
    {
        // recomputed over the final ok regions when any region failed after that pass
        std::vector<std::array<uint64_t, 3>> tri;
        bool changed = false;
        for (const RegionState& r : rs) {
            if (r.ok) tri.push_back({r.r.base, r.r.size, mode == KC_MODE_PRE_W ? r.pre_digest : r.post_digest});
            else if (!r.failed_pre) changed = true;
        }
        if (changed) {
            st = final_snapshot_digest(ctx, tri, cs, &rep.snapshot_digest);
            if (st != KC_OK) return st;
        }
    }
    std::vector<LogRegion> lr;
    for (const RegionState& r : rs) {
        if (!r.ok) rep.n_failed_regions++;
        lr.push_back({r.r.base, r.post_digest, (uint64_t)r.written.size(), r.ok, r.error});
    }
    rep.t_total_s = now_s() - t0;
    const std::string lg = capture_log_json(lr, rep, ctx->io_chunk, ctx->depth, "files");
    if (!write_text(dir + "/capture_log.json", lg)) return set_err(ctx, KC_ERR_IO, "cannot write capture_log.json");
    if (!write_file(dir + "/capture_complete", "", 0)) return set_err(ctx, KC_ERR_IO, "cannot write sentinel");
    if (rep_out) *rep_out = rep;
    if (rep.n_failed_regions) {
        final_st = KC_PARTIAL;
        set_err(ctx, KC_PARTIAL, "kc_capture: %llu region(s) failed; see capture_log.json",
                (unsigned long long)rep.n_failed_regions);
    }
    return final_st;
}

// ====================================================================== restore
namespace {
const uint64_t kPlaceholderGranule = 2ull << 20;  // typical VMM granularity before cuInit
const uint64_t kWindowAlign = 32ull << 20;        // smallest VA window a fresh process honours (R28)

struct ParsedRegion {
    uint64_t base, size;
    int kind;
    bool ok;
    std::string hx;
    uint64_t seq = 0;
};

kc_status parse_regions(kc_ctx* ctx, const std::string& dir, std::vector<ParsedRegion>& out) {
    std::string text;
    if (!kcj::read_file(dir + "/memory_regions.json", text))
        return set_err(ctx, KC_ERR_FORMAT, "cannot read %s/memory_regions.json", dir.c_str());
    kcj::Value v;
    if (!kcj::Parser(text).parse(v) || v.t != kcj::Value::Arr)
        return set_err(ctx, KC_ERR_FORMAT, "memory_regions.json does not parse");
    for (auto& e : v.a) {
        const kcj::Value* b = e.get("base");
        const kcj::Value* s = e.get("size");
        if (!b || !s || b->t != kcj::Value::Str) return set_err(ctx, KC_ERR_FORMAT, "region entry lacks base/size");
        ParsedRegion r;
        r.base = strtoull(b->s.c_str(), nullptr, 16);
        r.size = s->as_u64();
        r.hx = b->s;
        const kcj::Value* k = e.get("alloc_kind");
        r.kind = k && k->s == "vmm" ? KC_KIND_VMM : (k && k->s == "pool" ? KC_KIND_POOL : KC_KIND_MEMALLOC);
        const kcj::Value* stv = e.get("status");
        r.ok = !stv || stv->s == "ok";
        if (const kcj::Value* q = e.get("seq")) r.seq = q->as_u64();
        out.push_back(r);
    }
    // final statuses from capture_log.json (a region may fail after the metadata was written)
    std::string lt;
    if (kcj::read_file(dir + "/capture_log.json", lt)) {
        kcj::Value lv;
        if (kcj::Parser(lt).parse(lv)) {
            if (const kcj::Value* rr = lv.get("regions"))
                for (auto& e : rr->a) {
                    const kcj::Value* b = e.get("base");
                    const kcj::Value* stv = e.get("status");
                    if (!b || !stv) continue;
                    for (auto& r : out)
                        if (r.hx == b->s && stv->s != "ok") r.ok = false;
                }
        }
    }
    std::sort(out.begin(), out.end(), [](const ParsedRegion& a, const ParsedRegion& b) { return a.base < b.base; });
    return KC_OK;
}

std::vector<std::pair<uint64_t, uint64_t>> make_spans(const std::vector<ParsedRegion>& regs, uint64_t G) {
    std::vector<std::pair<uint64_t, uint64_t>> spans;  // [lo, hi)
    for (auto& r : regs) {
        const uint64_t lo = r.base / G * G, hi = (r.base + r.size + G - 1) / G * G;
        if (!spans.empty() && lo <= spans.back().second) spans.back().second = std::max(spans.back().second, hi);
        else spans.emplace_back(lo, hi);
    }
    return spans;
}

// physical allocations of released restores (kc_ctx::phys_park): parked up to
// KC_PHYS_PARK_MAX bytes (default 96 GiB) unless KC_PHYS_PARK=0
bool phys_park_on() {
    static const bool on = [] {
        const char* e = getenv("KC_PHYS_PARK");
        return !(e && *e == '0');
    }();
    return on;
}
uint64_t phys_park_max() {
    static const uint64_t m = [] {
        const char* e = getenv("KC_PHYS_PARK_MAX");
        return e && *e ? strtoull(e, nullptr, 10) : (96ull << 30);
    }();
    return m;
}
uint64_t phys_park_min() {  // spans below this size are released, not parked
    static const uint64_t m = [] {
        const char* e = getenv("KC_PHYS_PARK_MIN");
        return e && *e ? strtoull(e, nullptr, 10) : 0ull;
    }();
    return m;
}
void phys_release(kc_ctx* ctx, CUmemGenericAllocationHandle h, uint64_t size) {
    if (ctx && phys_park_on() && size >= phys_park_min() && ctx->phys_park_bytes + size <= phys_park_max()) {
        ctx->phys_park.emplace(size, h);
        ctx->phys_park_bytes += size;
        return;
    }
    KC_DRV(cuMemRelease)(h);
}
bool phys_take(kc_ctx* ctx, uint64_t size, CUmemGenericAllocationHandle* h) {
    auto it = ctx->phys_park.find(size);
    if (it == ctx->phys_park.end()) return false;
    *h = it->second;
    ctx->phys_park.erase(it);
    ctx->phys_park_bytes -= size;
    return true;
}

void rollback(kc_restored* h) {
    for (auto it = h->spans.rbegin(); it != h->spans.rend(); ++it) {
        for (uint64_t p : it->memalloc) KC_DRV(cuMemFree)((CUdeviceptr)p);
        it->memalloc.clear();
        if (it->mapped) KC_DRV(cuMemUnmap)((CUdeviceptr)it->base, it->size);
        if (it->created) phys_release(h->ctx, it->h, it->size);
        if (it->heap) heap_put(h->ctx, it->base, it->size);
    }
    h->spans.clear();
    for (auto& w : h->windows) KC_DRV(cuMemAddressFree)((CUdeviceptr)w.first, w.second);
    h->windows.clear();
}
}  // namespace

// Stage 2 on CUDA: measured on the B200 box, PROT_NONE
// placeholders mapped before cuInit are excluded from the driver's VA space
// for the process lifetime, so munmapping them later does NOT make the captured
// VAs reservable (R28).  Stage 2 is therefore a check, made before CUDA
// initialises: KC_PARTIAL when an existing host mapping already overlaps a
// captured 32 MiB window, so the caller can re-exec for a fresh ASLR layout.
// *n_reserved = windows that are free.  No CUDA calls, nothing is mapped.
extern "C" kc_status kc_prereserve(const char* dir, uint64_t* n_reserved) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    if (!dir) return KC_ERR_ARG;
    std::vector<ParsedRegion> regs;
    kc_status st = parse_regions(nullptr, dir, regs);
    if (st != KC_OK) return st;
    auto spans = make_spans(regs, kPlaceholderGranule);
    std::vector<std::pair<uint64_t, uint64_t>> win;  // merged 32 MiB windows [lo, hi)
    for (auto& sp : spans) {
        const uint64_t lo = sp.first / kWindowAlign * kWindowAlign;
        const uint64_t hi = (sp.second + kWindowAlign - 1) / kWindowAlign * kWindowAlign;
        if (!win.empty() && lo <= win.back().second) win.back().second = std::max(win.back().second, hi);
        else win.emplace_back(lo, hi);
    }
    std::vector<std::pair<uint64_t, uint64_t>> maps;
    if (FILE* f = fopen("/proc/self/maps", "r")) {
        char line[512];
        while (fgets(line, sizeof line, f)) {
            unsigned long long a = 0, b = 0;
            if (sscanf(line, "%llx-%llx", &a, &b) == 2) maps.emplace_back(a, b);
        }
        fclose(f);
    }
    uint64_t n = 0;
    for (auto& w : win) {
        bool clash = false;
        for (auto& m : maps)
            if (m.first < w.second && m.second > w.first) clash = true;
        n += !clash;
    }
    if (n_reserved) *n_reserved = n;
    return n == win.size() ? KC_OK : KC_PARTIAL;
}

// /proc/self/maps lines overlapping [lo, hi) (diagnostics for KC_ERR_VA_UNAVAILABLE)
static std::string maps_overlapping(uint64_t lo, uint64_t hi) {
    std::string out;
    FILE* f = fopen("/proc/self/maps", "r");
    if (!f) return out;
    char line[512];
    int n = 0;
    while (fgets(line, sizeof line, f) && n < 4) {
        unsigned long long a = 0, b = 0;
        if (sscanf(line, "%llx-%llx", &a, &b) == 2 && a < hi && b > lo) {
            std::string l(line);
            while (!l.empty() && (l.back() == '\n' || l.back() == ' ')) l.pop_back();
            out += (out.empty() ? "" : " | ") + l;
            ++n;
        }
    }
    fclose(f);
    return out.empty() ? "no host mapping overlaps (driver-internal VA)" : out;
}

// ====================================================================== restore core
// SnapDesc (kc_snapshot_types.h) is a snapshot's contents independent of where
// the bytes live; restore_core maps the captured VAs and pulls the bytes
// through a RestoreSource.
struct RestoreSource {
    virtual ~RestoreSource() {}
    // stored bytes of every ok region -> its (mapped, zero-filled) VA
    virtual kc_status copy_in(kc_ctx* ctx, const SnapDesc& d, kc_restore_report& rep) = 0;
    // PRE_W: the captured post-dispatch bytes of region i's W chunks, concatenated, -> device dst
    virtual kc_status written_ref(kc_ctx* ctx, const SnapDesc& d, size_t i, void* dst, uint64_t bytes) = 0;
    // the copy-in streams through the pinned staging ring (file sources)
    virtual bool needs_staging() const { return true; }
    // optional fused copy-in + verify: copies every ok region and returns the
    // chunk hashes of the bytes it copied (ok regions in order); *done = false
    // when the source cannot (then copy_in + a K1 pass over the regions run)
    virtual kc_status copy_in_verify(kc_ctx*, const SnapDesc&, kc_restore_report&, std::vector<uint64_t>&,
                                     bool& done) {
        done = false;
        return KC_OK;
    }
};

namespace {

kc_status load_desc_files(kc_ctx* ctx, const std::string& dir, SnapDesc& d, kc_restore_report& rep) {
    struct stat sb;
    if (stat((dir + "/capture_complete").c_str(), &sb) != 0)
        return set_err(ctx, KC_ERR_FORMAT, "%s: no capture_complete sentinel (incomplete capture)", dir.c_str());
    // stage 1: parse metadata
    std::string dtext;
    if (!kcj::read_file(dir + "/dispatch.json", dtext)) return set_err(ctx, KC_ERR_FORMAT, "cannot read dispatch.json");
    kcj::Value dv;
    if (!kcj::Parser(dtext).parse(dv)) return set_err(ctx, KC_ERR_FORMAT, "dispatch.json does not parse");
    std::vector<ParsedRegion> regs;
    kc_status st = parse_regions(ctx, dir, regs);
    if (st != KC_OK) return st;
    d.mode = dv.get("mode") && dv.get("mode")->s == "post" ? KC_MODE_POST : KC_MODE_PRE_W;
    d.mangled = dv.get("mangled_symbol") ? dv.get("mangled_symbol")->s : "";
    if (const kcj::Value* g = dv.get("grid"))
        for (int i = 0; i < 3 && i < (int)g->a.size(); ++i) d.grid[i] = (uint32_t)g->a[i].as_u64(1);
    if (const kcj::Value* g = dv.get("block"))
        for (int i = 0; i < 3 && i < (int)g->a.size(); ++i) d.block[i] = (uint32_t)g->a[i].as_u64(1);
    if (const kcj::Value* g = dv.get("shared_mem_bytes")) d.smem = (uint32_t)g->as_u64();
    if (const kcj::Value* g = dv.get("cooperative"))
        if (g->s == "true" || g->b) d.flags |= KC_LAUNCH_COOPERATIVE;
    if (const kcj::Value* g = dv.get("cluster"))
        for (int i = 0; i < 3 && i < (int)g->a.size(); ++i) d.cluster[i] = std::max<uint32_t>(1, (uint32_t)g->a[i].as_u64(1));
    if (const kcj::Value* g = dv.get("kernarg_layout"))  // (offset, size) per parameter (R22)
        for (const auto& e : g->a)
            if (e.get("offset") && e.get("size")) d.layout.emplace_back(e.get("offset")->as_u64(), e.get("size")->as_u64());
    if (!read_bin(dir + "/kernarg.bin", d.kernarg)) return set_err(ctx, KC_ERR_FORMAT, "cannot read kernarg.bin");
    const uint64_t ksz = dv.get("kernarg_size") ? dv.get("kernarg_size")->as_u64() : d.kernarg.size();
    if (ksz != d.kernarg.size())
        return set_err(ctx, KC_ERR_FORMAT, "kernarg.bin has %zu bytes, dispatch.json says %llu", d.kernarg.size(),
                       (unsigned long long)ksz);
    read_bin(dir + "/kernel.cubin", d.image);
    if (const kcj::Value* sh = dv.get("code_object_sha256"))  // identity of the captured code object
        if (!sh->s.empty() && (d.image.empty() || sha256_hex(d.image.data(), d.image.size()) != sh->s))
            return set_err(ctx, KC_ERR_FORMAT, "kernel.cubin does not match dispatch.json code_object_sha256");
    // F3: module variables (optional file)
    std::string mtext;
    if (kcj::read_file(dir + "/module_vars.json", mtext)) {
        kcj::Value mv;
        if (!kcj::Parser(mtext).parse(mv) || !mv.get("vars"))
            return set_err(ctx, KC_ERR_FORMAT, "module_vars.json does not parse");
        for (auto& e : mv.get("vars")->a) {
            ModVarState s;
            s.name = e.get("name") ? e.get("name")->s : "";
            s.section = e.get("section") ? e.get("section")->s : "";
            s.size = e.get("size") ? e.get("size")->as_u64() : 0;
            if (!e.get("pre") || !e.get("post") || !read_bin(dir + "/" + e.get("pre")->s, s.pre) ||
                !read_bin(dir + "/" + e.get("post")->s, s.post) || s.pre.size() != s.size || s.post.size() != s.size)
                return set_err(ctx, KC_ERR_FORMAT, "module variable %s: missing or wrong-length files", s.name.c_str());
            d.modvars.push_back(std::move(s));
        }
    }
    for (auto& r : regs) {
        SnapRegion sr;
        sr.r.base = r.base;
        sr.r.size = r.size;
        sr.r.device = ctx->device;
        sr.r.kind = r.kind;
        sr.r.seq = r.seq;
        sr.hx = r.hx;
        sr.ok = r.ok;
        sr.n_chunks = (r.size + kChunk - 1) / kChunk;
        if (r.ok) {
            read_u64s(dir + "/written/region_" + r.hx + ".idx", sr.written);
            read_u64s(dir + "/memory/region_" + r.hx + ".xxh64", sr.manifest);
            const std::string pm = dir + (d.mode == KC_MODE_PRE_W ? "/post/region_" : "/memory/region_") + r.hx + ".xxh64";
            read_u64s(pm, sr.post_manifest);
        } else {
            rep.n_failed_regions++;
        }
        d.regions.push_back(std::move(sr));
    }
    return KC_OK;
}

struct FileSource : RestoreSource {
    std::string dir;
    std::vector<uint64_t> dst;  // optional: region i's bytes go to dst[i] instead of its VA (kc_snapshot_load)
    explicit FileSource(std::string d) : dir(std::move(d)) {}
    kc_status copy_in(kc_ctx* ctx, const SnapDesc& d, kc_restore_report& rep) override {
        // every region file must exist with exactly `size` bytes (O1)
        std::vector<std::pair<size_t, uint64_t>> todo;
        for (size_t i = 0; i < d.regions.size(); ++i) {
            const auto& sr = d.regions[i];
            if (!sr.ok) continue;
            const std::string path = dir + "/memory/region_" + sr.hx + ".bin";
            struct stat sb;
            if (stat(path.c_str(), &sb) != 0 || (uint64_t)sb.st_size != sr.r.size)
                return set_err(ctx, KC_ERR_FORMAT, "kc_restore: %s: missing or wrong length", path.c_str());
            todo.emplace_back(i, sr.r.size);
        }
        const int T = io_threads();
        kc_status st = ensure_io(ctx, T);
        if (st != KC_OK) return st;
        const std::vector<IoItem> items = make_items(todo);
        std::atomic<int> bad{0};
        std::mutex emu;
        std::string first_err;
        std::atomic<uint64_t> h2d{0};
        run_pool(T, items.size(), [&](int t, size_t k) {
            if (bad) return;
            const IoItem& it = items[k];
            cudaSetDevice(ctx->device);
            const auto& sr = d.regions[it.region];
            const std::string path = dir + "/memory/region_" + sr.hx + ".bin";
            int fd = open(path.c_str(), O_RDONLY);
            std::string err = fd < 0 ? "cannot open" : "";
            const uint64_t to = dst.empty() ? sr.r.base : dst[it.region];
            const bool ok = fd >= 0 && item_h2d(ctx, ctx->io[t], fd, to, it, err);
            if (fd >= 0) close(fd);
            if (ok) {
                h2d.fetch_add(it.len);
            } else if (!bad.exchange(1)) {
                std::lock_guard<std::mutex> lk(emu);
                first_err = path + ": " + err;
            }
        });
        rep.h2d_bytes += h2d.load();
        if (bad) return set_err(ctx, KC_ERR_FORMAT, "kc_restore: copy-in failed: %s", first_err.c_str());
        return KC_OK;
    }
    kc_status written_ref(kc_ctx* ctx, const SnapDesc& d, size_t i, void* dst, uint64_t bytes) override {
        std::vector<uint8_t> wb;
        if (!read_bin(dir + "/written/region_" + d.regions[i].hx + ".bin", wb) || wb.size() != bytes)
            return set_err(ctx, KC_ERR_FORMAT, "written/region_%s.bin is missing or has the wrong length",
                           d.regions[i].hx.c_str());
        // on the ctx stream and complete before wb goes away: a legacy-stream
        // cudaMemcpy would not order the stash against the non-blocking copy_stream
        KC_CHECK_CUDA(ctx, cudaMemcpyAsync(dst, wb.data(), bytes, cudaMemcpyHostToDevice, ctx->copy_stream),
                      "H2D written reference");
        KC_CHECK_CUDA(ctx, cudaStreamSynchronize(ctx->copy_stream), "H2D written reference");
        return KC_OK;
    }
};

}  // namespace

// the dispatch a restored handle replays: launch shape, kernarg, code object, F3 variables
static void bind_dispatch_fields(kc_restored* h, const SnapDesc& d) {
    h->mode = d.mode;
    h->mangled = d.mangled;
    for (int i = 0; i < 3; ++i) {
        h->grid[i] = d.grid[i];
        h->block[i] = d.block[i];
    }
    h->smem = d.smem;
    for (int i = 0; i < 3; ++i) h->cluster[i] = d.cluster[i];
    h->flags = d.flags;
    h->kernarg = d.kernarg;
    h->image = d.image;
    h->modvars = d.modvars;
}

// device stashes of the written chunks: replay recopy (pre-state, from the live
// memory as it is now) and validation reference (captured post bytes)
static kc_status build_stash(kc_ctx* ctx, kc_restored* h, const SnapDesc& d, RestoreSource& src) {
    uint64_t total = 0;
    for (auto& rr : h->regions) {
        rr.stash_off.clear();
        for (uint64_t k : rr.written) {
            rr.stash_off.push_back(total);
            total += std::min<uint64_t>(kChunk, rr.r.size - k * kChunk);
        }
    }
    h->stash_bytes = total;
    if (!total) return KC_OK;
    // one allocation for both stashes (stash_ref = stash_pre + total; kc_release frees stash_pre only)
    if (cudaMalloc(&h->stash_pre, 2 * total) != cudaSuccess)
        return set_err(ctx, KC_ERR_NOMEM, "kc_restore: stash of %llu bytes", (unsigned long long)(2 * total));
    h->stash_ref = (uint8_t*)h->stash_pre + total;
    for (size_t i = 0; i < h->regions.size(); ++i) {
        auto& rr = h->regions[i];
        if (!rr.ok || rr.written.empty()) continue;
        uint64_t wbytes = 0;
        for (size_t j = 0; j < rr.written.size(); ++j) {
            const uint64_t k = rr.written[j];
            const uint64_t len = std::min<uint64_t>(kChunk, rr.r.size - k * kChunk);
            cudaMemcpyAsync((uint8_t*)h->stash_pre + rr.stash_off[j], (const void*)(rr.r.base + k * kChunk), len,
                            cudaMemcpyDeviceToDevice, ctx->copy_stream);
            if (h->mode != KC_MODE_PRE_W)
                cudaMemcpyAsync((uint8_t*)h->stash_ref + rr.stash_off[j], (const void*)(rr.r.base + k * kChunk),
                                len, cudaMemcpyDeviceToDevice, ctx->copy_stream);
            wbytes += len;
        }
        if (h->mode == KC_MODE_PRE_W) {
            cudaStreamSynchronize(ctx->copy_stream);
            kc_status st = src.written_ref(ctx, d, i, (uint8_t*)h->stash_ref + rr.stash_off[0], wbytes);
            if (st != KC_OK) return st;
        }
    }
    cudaError_t ce = cudaStreamSynchronize(ctx->copy_stream);
    if (ce != cudaSuccess) return cuda_err(ctx, ce, "kc_restore: stash");
    return KC_OK;
}

// Stages 5-6 of a restore into mapped spans: zero-fill what the copy-in does not write,
// copy in (fused with the verify hashes when the source allows), verify against the
// captured manifest, and build the W stashes.  Shared by kc_restore / kc_restore_dev
// (fresh mappings) and kc_restore_dev_into (the mappings of a live restore).
static kc_status restore_fill(kc_ctx* ctx, kc_restored* h, const SnapDesc& d, RestoreSource& src,
                              kc_restore_report& rep) {
    double t, tl = now_s();
    // ---- stage 5a: copy-in (gaps and failed regions zero-filled)
    t = now_s();
    kc_status st = src.needs_staging() ? ensure_pinned(ctx) : ensure_stream(ctx);
    if (st != KC_OK) return st;
    // zero only what the copy-in does not write: span bytes outside every ok
    // region (granule padding) and failed regions; an ok region's stored bytes
    // cover it entirely (its region file / arena runs are exactly `size` bytes,
    // and the K1 verify below checks every chunk)
    {
        std::vector<std::pair<uint64_t, uint64_t>> ok_iv;  // ascending (regions are sorted by base)
        for (auto& rr : h->regions) {
            if (rr.ok) ok_iv.emplace_back(rr.r.base, rr.r.base + rr.r.size);
            else cudaMemsetAsync((void*)rr.r.base, 0, rr.r.size, ctx->copy_stream);
        }
        size_t j = 0;
        for (auto& s : h->spans) {
            if (s.fallback) continue;
            uint64_t cur = s.base;
            const uint64_t end = s.base + s.size;
            while (j < ok_iv.size() && ok_iv[j].second <= cur) ++j;
            for (size_t k = j; k < ok_iv.size() && ok_iv[k].first < end; ++k) {
                if (ok_iv[k].first > cur) cudaMemsetAsync((void*)cur, 0, ok_iv[k].first - cur, ctx->copy_stream);
                cur = std::max(cur, ok_iv[k].second);
            }
            if (cur < end) cudaMemsetAsync((void*)cur, 0, end - cur, ctx->copy_stream);
        }
    }
    cudaStreamSynchronize(ctx->copy_stream);  // zero-fill before the copy-in streams
    trace("restore: zero-fill gaps", tl);
    std::vector<uint64_t> got;
    bool verified = false;  // the copy-in produced the verify hashes itself (K6)
    st = src.copy_in_verify(ctx, d, rep, got, verified);
    if (st == KC_OK && !verified) st = src.copy_in(ctx, d, rep);
    cudaError_t ce = cudaStreamSynchronize(ctx->copy_stream);
    if (st == KC_OK && ce != cudaSuccess) st = cuda_err(ctx, ce, "kc_restore: copy-in");
    if (st != KC_OK) return st;
    rep.t_h2d_s = now_s() - t;
    trace(verified ? "restore: copy-in + verify (K6)" : "restore: copy-in", tl);

    // ---- verify against the captured manifest (K1, O6)
    t = now_s();
    std::vector<kc_region> okregs;
    for (auto& rr : h->regions)
        if (rr.ok) okregs.push_back(rr.r);
    if (!verified) st = hash_regions_sync(ctx, okregs, got, nullptr, nullptr, nullptr, ctx->copy_stream);
    if (st != KC_OK) return st;
    {
        uint64_t c = 0, mism = 0;
        for (auto& sr : d.regions) {
            if (!sr.ok) continue;
            if (sr.manifest.size() != sr.n_chunks) {
                mism += sr.n_chunks;
            } else {
                for (uint64_t k = 0; k < sr.n_chunks; ++k) mism += sr.manifest[k] != got[c + k];
            }
            c += sr.n_chunks;
        }
        rep.verify_mismatch_chunks = mism;
    }
    rep.t_verify_s = now_s() - t;
    if (rep.verify_mismatch_chunks) {
        return set_err(ctx, KC_ERR_MANIFEST_MISMATCH, "kc_restore: %llu restored chunk(s) do not match the captured "
                       "manifest", (unsigned long long)rep.verify_mismatch_chunks);
    }

    trace("restore: verify", tl);
    // ---- device stashes of the written chunks: replay recopy (pre) and validation reference (post)
    st = build_stash(ctx, h, d, src);
    trace("restore: W stashes", tl);
    if (st != KC_OK) return st;
    return KC_OK;
}

static kc_status restore_core(kc_ctx* ctx, const SnapDesc& d, RestoreSource& src, kc_restored** out,
                              kc_restore_report* rep_out, kc_restore_report& rep, double t0) {
    kc_restored* h = new kc_restored();
    h->ctx = ctx;  // rollback() returns heap spans to this ctx
    bind_dispatch_fields(h, d);
    std::vector<ParsedRegion> regs;
    for (auto& sr : d.regions) {
        kc_restored_region rr;
        rr.r = sr.r;
        rr.hexbase = sr.hx;
        rr.ok = sr.ok;
        rr.n_chunks = sr.n_chunks;
        rr.written = sr.written;
        rr.post_manifest = sr.post_manifest;
        h->regions.push_back(rr);
        ParsedRegion p;
        p.base = sr.r.base;
        p.size = sr.r.size;
        p.kind = sr.r.kind;
        p.ok = sr.ok;
        p.hx = sr.hx;
        p.seq = sr.r.seq;
        regs.push_back(p);
    }
    rep.n_regions = d.regions.size();

    // ---- stages 2-4: exact-VA reservation (R28)
    if (!bind_device(ctx)) {
        delete h;
        return set_err(ctx, KC_ERR_CUDA, "cannot bind device");
    }
    double t = now_s();
    CUmemAllocationProp prop;
    memset(&prop, 0, sizeof prop);
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = ctx->device;
    size_t G = 0;
    CUresult cr = KC_DRV(cuMemGetAllocationGranularity)(&G, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
    if (cr != CUDA_SUCCESS || G == 0) {
        delete h;
        return cu_err(ctx, cr, "cuMemGetAllocationGranularity");
    }
    auto spans = make_spans(regs, G);
    // Reserve VA windows at exactly aligned hints.  A fresh process honours a
    // hint only where the driver can open a new VA chunk, i.e. at a coarse
    // alignment (observed: 32 MiB), so try the exact span first and then
    // covering windows aligned to 32 MiB ... 1 GiB; map only the spans.
    static const uint64_t kWindows[] = {0, 32ull << 20, 64ull << 20, 128ull << 20, 256ull << 20, 512ull << 20,
                                        1ull << 30};
    for (auto& sp : spans) {
        kc_restored::Span s{sp.first, sp.second - sp.first, 0, false, false, false, false, false, {}, 0, 0};
        // a span inside this ctx's VA heap that is free (its allocation was released
        // with kc_free) is mapped straight back at the exact VA (R28d)
        if (heap_take(ctx, s.base, s.size)) {
            s.reserved = true;
            s.heap = true;
            h->spans.push_back(s);
            continue;
        }
        bool covered = false;
        for (auto& w : h->windows)
            if (w.first <= s.base && s.base + s.size <= w.first + w.second) covered = true;
        if (!covered) {
            const uint64_t prev_end = h->windows.empty() ? 0 : h->windows.back().first + h->windows.back().second;
            bool lost = false;  // a window released for a merge could not be taken back
            for (uint64_t W : kWindows) {
                const uint64_t A = W ? W : G;
                uint64_t lo = s.base / A * A;
                const uint64_t hi = (s.base + s.size + A - 1) / A * A;
                // A span that starts inside the window we hold but ends past it (two
                // regions less than a window apart): the exact span would overlap that
                // window, so the window is released and one window covering both is
                // reserved instead (and the old one taken back if that fails).
                bool merge = false;
                if (lo < prev_end) {
                    if (!W) continue;
                    lo = std::min(lo, h->windows.back().first) / A * A;
                    if (h->windows.size() >= 2 &&
                        lo < h->windows[h->windows.size() - 2].first + h->windows[h->windows.size() - 2].second)
                        continue;  // would overlap an earlier window
                    merge = true;
                }
                const std::pair<uint64_t, uint64_t> old = merge ? h->windows.back() : std::pair<uint64_t, uint64_t>(0, 0);
                if (merge) KC_DRV(cuMemAddressFree)((CUdeviceptr)old.first, old.second);
                CUdeviceptr p = 0;
                cr = KC_DRV(cuMemAddressReserve)(&p, hi - lo, A, (CUdeviceptr)lo, 0);
                if (cr == CUDA_SUCCESS && (uint64_t)p == lo) {
                    if (merge) h->windows.back() = {lo, hi - lo};
                    else h->windows.emplace_back(lo, hi - lo);
                    covered = true;
                    break;
                }
                if (cr == CUDA_SUCCESS) KC_DRV(cuMemAddressFree)(p, hi - lo);
                s.reserve_got = (uint64_t)p;
                s.reserve_cr = (int)cr;
                if (merge) {
                    CUdeviceptr q = 0;
                    const CUresult r2 = KC_DRV(cuMemAddressReserve)(&q, old.second, 0, (CUdeviceptr)old.first, 0);
                    if (r2 != CUDA_SUCCESS || (uint64_t)q != old.first) {
                        if (r2 == CUDA_SUCCESS) KC_DRV(cuMemAddressFree)(q, old.second);
                        h->windows.pop_back();
                        lost = true;
                        break;
                    }
                }
            }
            if (lost) {
                rollback(h);
                delete h;
                return set_err(ctx, KC_ERR_VA_UNAVAILABLE,
                               "kc_restore: the VA window ending at 0x%llx, released to merge span [0x%llx, +%llu) could not be "
                               "reserved again; VA faithfulness is a hard requirement (PAPER.md:1080-1082)",
                               (unsigned long long)prev_end, (unsigned long long)s.base, (unsigned long long)s.size);
            }
        }
        if (covered) {
            s.reserved = true;
        } else {
            // The span lies in VA the driver pools for small cuMemAlloc
            // allocations: fall back to replaying cuMemAlloc below.
            s.fallback = true;
        }
        h->spans.push_back(s);
    }
    for (auto& s : h->spans) {
        if (s.fallback) continue;
        cr = phys_take(ctx, s.size, &s.h) ? CUDA_SUCCESS : KC_DRV(cuMemCreate)(&s.h, s.size, &prop, 0);
        if (cr == CUDA_SUCCESS) {
            s.created = true;
            cr = KC_DRV(cuMemMap)((CUdeviceptr)s.base, s.size, 0, s.h, 0);
        }
        if (cr == CUDA_SUCCESS) {
            s.mapped = true;
            CUmemAccessDesc acc;
            acc.location = prop.location;
            acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
            cr = KC_DRV(cuMemSetAccess)((CUdeviceptr)s.base, s.size, &acc, 1);
        }
        if (cr != CUDA_SUCCESS) {
            rollback(h);
            delete h;
            return cu_err(ctx, cr, "kc_restore: cuMemCreate/cuMemMap/cuMemSetAccess");
        }
        rep.mapped_bytes += s.size;
    }
    {
        // cuMemAlloc replay, in the capture's allocation order, for fallback spans
        std::vector<std::pair<uint64_t, size_t>> fb;  // (seq, region index)
        for (size_t i = 0; i < h->regions.size(); ++i) {
            const auto& rr = h->regions[i];
            for (auto& s : h->spans)
                if (s.fallback && s.base <= rr.r.base && rr.r.base < s.base + s.size) fb.emplace_back(regs[i].seq, i);
        }
        std::sort(fb.begin(), fb.end());
        for (auto& e : fb) {
            const auto& rr = h->regions[e.second];
            CUdeviceptr p = 0;
            cr = KC_DRV(cuMemAlloc)(&p, rr.r.size);
            kc_restored::Span* owner = nullptr;
            for (auto& s : h->spans)
                if (s.fallback && s.base <= rr.r.base && rr.r.base < s.base + s.size) owner = &s;
            if (cr == CUDA_SUCCESS) owner->memalloc.push_back((uint64_t)p);
            if (cr != CUDA_SUCCESS || (uint64_t)p != rr.r.base) {
                const uint64_t got = (uint64_t)p, want = rr.r.base, sz = rr.r.size;
                uint64_t sbase = 0, sgot = 0;
                int scr = 0;
                for (auto& s : h->spans)
                    if (s.fallback && s.base <= want && want < s.base + s.size) {
                        sbase = s.base;
                        sgot = s.reserve_got;
                        scr = s.reserve_cr;
                    }
                rollback(h);
                delete h;
                const std::string maps = maps_overlapping(want, want + sz);
                return set_err(ctx, KC_ERR_VA_UNAVAILABLE,
                               "kc_restore: cannot restore captured region [0x%llx, +%llu): reserving span 0x%llx "
                               "returned 0x%llx (CUresult %d) and the cuMemAlloc replay returned 0x%llx (%d); host "
                               "maps: %s; VA faithfulness is a hard requirement (PAPER.md:1080-1082)",
                               (unsigned long long)want, (unsigned long long)sz, (unsigned long long)sbase,
                               (unsigned long long)sgot, scr, (unsigned long long)got, (int)cr, maps.c_str());
            }
            rep.mapped_bytes += rr.r.size;
        }
    }
    rep.n_spans = h->spans.size();
    rep.t_reserve_s = now_s() - t;
    trace("restore: reserve + create + map", t);

    const kc_status st0 = restore_fill(ctx, h, d, src, rep);
    if (st0 != KC_OK) {
        if (rep_out) *rep_out = rep;
        rollback(h);
        delete h;
        return st0;
    }
    rep.t_total_s = now_s() - t0;
    if (rep_out) *rep_out = rep;
    *out = h;
    return KC_OK;
}

namespace {
kc_status copy_ranges_d2d(kc_ctx* ctx, const std::vector<std::array<uint64_t, 3>>& ranges, cudaStream_t s,
                          uint64_t* calls);
// a published VMM arena mapped into this process: the publisher's fd is
// duplicated with pidfd_getfd (Linux >= 5.6; a same-user or descendant
// process), imported and mapped read-write at a fresh VA
struct ImportedArena {
    CUdeviceptr va = 0;
    uint64_t size = 0;
    CUmemGenericAllocationHandle h = 0;
    kc_status open(kc_ctx* ctx, int pid, int fd, uint64_t bytes) {
#if defined(SYS_pidfd_open) && defined(SYS_pidfd_getfd)
        const int pfd = (int)syscall(SYS_pidfd_open, pid, 0);
        if (pfd < 0)
            return set_err(ctx, KC_ERR_STATE, "pidfd_open(%d): %s (is the publishing process alive?)", pid,
                           strerror(errno));
        const int myfd = (int)syscall(SYS_pidfd_getfd, pfd, fd, 0);
        const int gerr = errno;
        ::close(pfd);
        if (myfd < 0)
            return set_err(ctx, KC_ERR_STATE, "pidfd_getfd(%d, fd %d): %s", pid, fd, strerror(gerr));
        CUresult r = KC_DRV(cuMemImportFromShareableHandle)(&h, (void*)(uintptr_t)myfd,
                                                            CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
        ::close(myfd);
        if (r != CUDA_SUCCESS) return cu_err(ctx, r, "cuMemImportFromShareableHandle");
        size = bytes;
        r = KC_DRV(cuMemAddressReserve)(&va, size, 0, 0, 0);
        if (r != CUDA_SUCCESS) {
            KC_DRV(cuMemRelease)(h);
            va = 0;
            return cu_err(ctx, r, "cuMemAddressReserve(published arena)");
        }
        CUmemAccessDesc acc;
        acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        acc.location.id = ctx->device;
        acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        r = KC_DRV(cuMemMap)(va, size, 0, h, 0);
        if (r == CUDA_SUCCESS) r = KC_DRV(cuMemSetAccess)(va, size, &acc, 1);
        if (r != CUDA_SUCCESS) {
            KC_DRV(cuMemUnmap)(va, size);
            KC_DRV(cuMemAddressFree)(va, size);
            KC_DRV(cuMemRelease)(h);
            va = 0;
            return cu_err(ctx, r, "cuMemMap(published arena)");
        }
        return KC_OK;
#else
        (void)pid; (void)fd; (void)bytes;
        return set_err(ctx, KC_ERR_UNSUPPORTED, "pidfd_getfd is not available on this system");
#endif
    }
    void close() {
        if (!va) return;
        cudaDeviceSynchronize();
        KC_DRV(cuMemUnmap)(va, size);
        KC_DRV(cuMemAddressFree)(va, size);
        KC_DRV(cuMemRelease)(h);
        va = 0;
    }
};

// F1 across processes: the region bytes of a published snapshot
// (kc_snapshot_publish) live in the capturing process's device arena; this
// process maps it with CUDA IPC and copies in at HBM bandwidth (K6: one read
// of the arena gives the copy and the verify hashes).  Metadata, manifests
// and W's post bytes come from the directory.
struct IpcSource : FileSource {
    void* arena = nullptr;
    uint64_t arena_bytes = 0;
    ImportedArena imp;                 // vmm_fd: the imported mapping
    std::map<uint64_t, uint64_t> off;  // region base -> arena offset
    explicit IpcSource(std::string d) : FileSource(std::move(d)) {}
    ~IpcSource() override {
        if (imp.va) imp.close();
        else if (arena) cudaIpcCloseMemHandle(arena);
    }
    kc_status open(kc_ctx* ctx) {
        std::string text;
        kcj::Value v;
        if (!kcj::read_file(dir + "/memory/device_arena.json", text) || !kcj::Parser(text).parse(v) ||
            !v.get("regions"))
            return set_err(ctx, KC_ERR_FORMAT, "device_arena.json does not parse");
        if (v.get("format") == nullptr || v.get("format")->s != "kc-device-arena/1")
            return set_err(ctx, KC_ERR_FORMAT, "device_arena.json: unknown format");
        if (v.get("pid") && kill((pid_t)v.get("pid")->as_u64(), 0) != 0 && errno == ESRCH)
            return set_err(ctx, KC_ERR_STATE, "the process that published this snapshot (pid %llu) is gone",
                           (unsigned long long)v.get("pid")->as_u64());
        if (v.get("device") && (int)v.get("device")->as_u64() != ctx->device)
            return set_err(ctx, KC_ERR_ARG, "published snapshot lives on device %d, this ctx is on %d",
                           (int)v.get("device")->as_u64(), ctx->device);
        arena_bytes = v.get("arena_bytes") ? v.get("arena_bytes")->as_u64() : 0;
        for (auto& e : v.get("regions")->a) {
            if (!e.get("base") || !e.get("offset")) return set_err(ctx, KC_ERR_FORMAT, "device_arena.json: region");
            off[strtoull(e.get("base")->s.c_str(), nullptr, 16)] = e.get("offset")->as_u64();
        }
        if (v.get("kind") && v.get("kind")->s == "vmm_fd") {
            if (!v.get("fd") || !v.get("mapped_bytes") || !v.get("pid"))
                return set_err(ctx, KC_ERR_FORMAT, "device_arena.json: vmm_fd needs pid, fd, mapped_bytes");
            kc_status st = imp.open(ctx, (int)v.get("pid")->as_u64(), (int)v.get("fd")->as_u64(),
                                    v.get("mapped_bytes")->as_u64());
            if (st != KC_OK) return st;
            arena = (void*)imp.va;
            return KC_OK;
        }
        if (!v.get("ipc_handle")) return set_err(ctx, KC_ERR_FORMAT, "device_arena.json: no ipc_handle");
        cudaIpcMemHandle_t ih;
        const std::string& hx = v.get("ipc_handle")->s;
        if (hx.size() != 2 * sizeof ih) return set_err(ctx, KC_ERR_FORMAT, "device_arena.json: bad ipc_handle");
        for (size_t i = 0; i < sizeof ih; ++i)
            ((uint8_t*)&ih)[i] = (uint8_t)strtoul(hx.substr(2 * i, 2).c_str(), nullptr, 16);
        cudaError_t ce = cudaIpcOpenMemHandle(&arena, ih, cudaIpcMemLazyEnablePeerAccess);
        if (ce != cudaSuccess) {
            arena = nullptr;
            return set_err(ctx, KC_ERR_STATE, "cudaIpcOpenMemHandle: %s (is the capturing process alive and the "
                           "snapshot not freed?)", cudaGetErrorString(ce));
        }
        return KC_OK;
    }
    bool needs_staging() const override { return false; }
    // the arena address of every ok region (in order), checked against the arena size
    kc_status sources(kc_ctx* ctx, const SnapDesc& d, std::vector<kc_region>& srcs, std::vector<uint64_t>& dst) {
        for (auto& sr : d.regions) {
            if (!sr.ok) continue;
            auto it = off.find(sr.r.base);
            if (it == off.end() || it->second + sr.r.size > arena_bytes)
                return set_err(ctx, KC_ERR_FORMAT, "device_arena.json: region %s missing or out of the arena",
                               sr.hx.c_str());
            kc_region r = sr.r;
            r.base = (uint64_t)arena + it->second;
            srcs.push_back(r);
            dst.push_back(sr.r.base);
        }
        return KC_OK;
    }
    kc_status copy_in(kc_ctx* ctx, const SnapDesc& d, kc_restore_report& rep) override {
        std::vector<kc_region> srcs;
        std::vector<uint64_t> dst;
        kc_status st = sources(ctx, d, srcs, dst);
        if (st != KC_OK) return st;
        std::vector<std::array<uint64_t, 3>> ranges;
        for (size_t i = 0; i < srcs.size(); ++i) {
            ranges.push_back({srcs[i].base, dst[i], srcs[i].size});
            rep.h2d_bytes += srcs[i].size;
        }
        return copy_ranges_d2d(ctx, ranges, ctx->copy_stream, nullptr);
    }
    kc_status copy_in_verify(kc_ctx* ctx, const SnapDesc& d, kc_restore_report& rep, std::vector<uint64_t>& got,
                             bool& done) override {
        done = false;
        if (getenv("KC_NO_FUSED_RESTORE")) return KC_OK;
        std::vector<kc_region> srcs;
        std::vector<uint64_t> dst;
        kc_status st = sources(ctx, d, srcs, dst);
        if (st != KC_OK) return st;
        for (size_t i = 0; i < srcs.size(); ++i)
            if ((srcs[i].base & 15) || (dst[i] & 15)) return KC_OK;
        st = hash_regions_sync(ctx, srcs, got, nullptr, nullptr, nullptr, ctx->copy_stream,
                               dst.empty() ? nullptr : dst.data());
        if (st != KC_OK) return st;
        for (const auto& r : srcs) rep.h2d_bytes += r.size;
        done = true;
        return KC_OK;
    }
};
}  // namespace

extern "C" kc_status kc_restore(kc_ctx* ctx, const char* dir_c, kc_restored** out, kc_restore_report* rep_out) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    if (!ctx || !dir_c || !out) return KC_ERR_ARG;
    if (ctx->poisoned) return KC_ERR_CUDA;
    *out = nullptr;
    kc_restore_report rep;
    memset(&rep, 0, sizeof rep);
    const double t0 = now_s();
    struct stat sb;
    if (stat((std::string(dir_c) + "/memory/device_arena.revoked").c_str(), &sb) == 0)
        return set_err(ctx, KC_ERR_STATE, "kc_restore: %s was published from a device snapshot that has been freed",
                       dir_c);
    double tl = now_s();
    SnapDesc d;
    kc_status st = load_desc_files(ctx, dir_c, d, rep);
    if (st != KC_OK) return st;
    trace("restore: load metadata", tl);
    if (stat((std::string(dir_c) + "/memory/device_arena.json").c_str(), &sb) == 0) {
        if (!bind_device(ctx)) return set_err(ctx, KC_ERR_CUDA, "cannot bind device");
        IpcSource src(dir_c);
        st = src.open(ctx);
        if (st != KC_OK) return st;
        trace("restore: open the published arena (CUDA IPC)", tl);
        st = restore_core(ctx, d, src, out, rep_out, rep, t0);
        if (st == KC_OK) {  // the mapping stays open for typed validation; kc_release closes it
            (*out)->dir = dir_c;
            (*out)->ipc_arena = src.arena;
            (*out)->ipc_off = src.off;
            (*out)->ipc_vmm_size = src.imp.va ? src.imp.size : 0;
            (*out)->ipc_vmm_h = src.imp.h;
            src.arena = nullptr;
            src.imp.va = 0;  // ownership moved to the restored handle
        }
        return st;
    }
    FileSource src(dir_c);
    st = restore_core(ctx, d, src, out, rep_out, rep, t0);
    if (st == KC_OK) (*out)->dir = dir_c;
    return st;
}

// ====================================================================== F1 device-resident snapshot
// kc_capture with the region bytes kept in an HBM arena: D2D copies at HBM
// bandwidth replace PCIe + files.  Big regions go through
// cudaMemcpyAsync, regions and W chunks under 1 MiB through the K4 gather.
//
// F2 incremental capture (kc_capture_incr): a chunk whose stored-state hash
// equals the base snapshot's at the same region and chunk index is not copied;
// the new snapshot references the base's bytes (shared ownership of the base
// arenas, so a base may be freed first).  Hash equality as "unchanged" is the
// method's own reading: W (A4) declares a chunk unwritten on the same test.
// (ArenaBuf / kc_snapshot: kc_snapshot_types.h.)
namespace {

// copies of (src, dst, len) ranges between device memory and the device or pinned
// host arena (UVA): >= 1 MiB by cudaMemcpyAsync, smaller ones batched through K4
kc_status copy_ranges_d2d(kc_ctx* ctx, const std::vector<std::array<uint64_t, 3>>& ranges, cudaStream_t s,
                          uint64_t* calls) {
    std::vector<uint64_t> src, dst, len;
    for (auto& r : ranges) {
        if (r[2] == 0) continue;
        if (r[2] >= (1ull << 20)) {
            KC_CHECK_CUDA(ctx, cudaMemcpyAsync((void*)r[1], (const void*)r[0], r[2], cudaMemcpyDefault, s),
                          "arena copy");
            if (calls) ++*calls;
        } else {
            src.push_back(r[0]);
            dst.push_back(r[1]);
            len.push_back(r[2]);
        }
    }
    if (!src.empty()) {
        const size_t n = src.size();
        KC_CHECK_CUDA(ctx, ensure(ctx->gather_tab, 3 * 8 * n), "cudaMalloc(gather table)");  // kept by the ctx
        uint64_t* t = (uint64_t*)ctx->gather_tab.p;
        cudaMemcpyAsync(t, src.data(), 8 * n, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(t + n, dst.data(), 8 * n, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(t + 2 * n, len.data(), 8 * n, cudaMemcpyHostToDevice, s);
        KC_CHECK_CUDA(ctx, launch_gather(t, t + n, t + 2 * n, (int)n, s), "launch K4");
        ctx->launches += 1;
        if (calls) ++*calls;
        cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return cuda_err(ctx, e, "K4 gather");
    }
    return KC_OK;
}

struct DevSource : RestoreSource {
    const kc_snapshot* sn;
    explicit DevSource(const kc_snapshot* s) : sn(s) {}
    bool needs_staging() const override { return false; }  // D2D / H2D straight from the arena
    // K6 from a device arena: every ok region stored as one run (a full capture)
    // is read once, hashed and written to its VA.  The hashes are those of the
    // arena bytes copied; kc_validate's re-hash of every region after the replay
    // (R31) re-reads what landed at the VAs.
    kc_status copy_in_verify(kc_ctx* ctx, const SnapDesc& d, kc_restore_report& rep, std::vector<uint64_t>& got,
                             bool& done) override {
        done = false;
        if (sn->host || getenv("KC_NO_FUSED_RESTORE")) return KC_OK;
        std::vector<kc_region> srcs;
        std::vector<uint64_t> dst;
        for (size_t i = 0; i < d.regions.size(); ++i) {
            if (!d.regions[i].ok) continue;
            const auto& runs = sn->runs[i];
            if (runs.size() != 1 || runs[0].roff != 0 || runs[0].len != d.regions[i].r.size ||
                (runs[0].src & 15) || (d.regions[i].r.base & 15))
                return KC_OK;
            kc_region r = d.regions[i].r;
            r.base = runs[0].src;
            srcs.push_back(r);
            dst.push_back(d.regions[i].r.base);
        }
        kc_status st = hash_regions_sync(ctx, srcs, got, nullptr, nullptr, nullptr, ctx->copy_stream,
                                         dst.empty() ? nullptr : dst.data());
        if (st != KC_OK) return st;
        for (const auto& r : srcs) rep.h2d_bytes += r.size;
        done = true;
        return KC_OK;
    }
    kc_status copy_in(kc_ctx* ctx, const SnapDesc& d, kc_restore_report& rep) override {
        std::vector<std::array<uint64_t, 3>> ranges;
        for (size_t i = 0; i < d.regions.size(); ++i) {
            if (!d.regions[i].ok) continue;
            for (const auto& ru : sn->runs[i]) ranges.push_back({ru.src, d.regions[i].r.base + ru.roff, ru.len});
            rep.h2d_bytes += d.regions[i].r.size;  // bytes copied in (D2D or H2D)
        }
        return copy_ranges_d2d(ctx, ranges, ctx->copy_stream, nullptr);
    }
    kc_status written_ref(kc_ctx* ctx, const SnapDesc&, size_t i, void* dst, uint64_t bytes) override {
        KC_CHECK_CUDA(ctx, cudaMemcpyAsync(dst, (const uint8_t*)sn->warena + sn->w_off[i], bytes, cudaMemcpyDefault,
                                           ctx->copy_stream),
                      "written reference from the arena");
        return KC_OK;
    }
};

}  // namespace

namespace {
// arena allocation for in-memory snapshots: device (cudaMalloc) or pinned host,
// the latter from the ctx's parked arena when it is large enough
// a device arena as one VMM allocation that can be exported as a POSIX fd
// (kc_snapshot_publish); false (nothing held) when the device or driver refuses
bool vmm_arena_alloc(kc_ctx* ctx, ArenaBuf& ab, uint64_t bytes) {
    if (getenv("KC_NO_VMM_ARENA")) return false;
    if (ctx->dev_arena.va && ctx->dev_arena.size >= bytes) {  // the parked arena
        ab.p = (void*)ctx->dev_arena.va;
        ab.cap = ctx->dev_arena.size;
        ab.vmm = true;
        ab.vmm_h = ctx->dev_arena.h;
        ab.vmm_size = ctx->dev_arena.size;
        ctx->dev_arena = {};
        return true;
    }
    CUmemAllocationProp prop;
    memset(&prop, 0, sizeof prop);
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = ctx->device;
    prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t G = 0;
    if (KC_DRV(cuMemGetAllocationGranularity)(&G, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM) != CUDA_SUCCESS || !G)
        return false;
    const uint64_t sz = (bytes + G - 1) / G * G;
    CUmemGenericAllocationHandle h = 0;
    if (KC_DRV(cuMemCreate)(&h, sz, &prop, 0) != CUDA_SUCCESS) return false;
    CUdeviceptr va = 0;
    if (KC_DRV(cuMemAddressReserve)(&va, sz, G, 0, 0) != CUDA_SUCCESS) {
        KC_DRV(cuMemRelease)(h);
        return false;
    }
    CUmemAccessDesc acc;
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if (KC_DRV(cuMemMap)(va, sz, 0, h, 0) != CUDA_SUCCESS) {
        KC_DRV(cuMemAddressFree)(va, sz);
        KC_DRV(cuMemRelease)(h);
        return false;
    }
    if (KC_DRV(cuMemSetAccess)(va, sz, &acc, 1) != CUDA_SUCCESS) {
        KC_DRV(cuMemUnmap)(va, sz);
        KC_DRV(cuMemAddressFree)(va, sz);
        KC_DRV(cuMemRelease)(h);
        return false;
    }
    ab.p = (void*)va;
    ab.cap = bytes;
    ab.vmm = true;
    ab.vmm_h = h;
    ab.vmm_size = sz;
    return true;
}

cudaError_t arena_alloc(kc_ctx* ctx, bool host, void** p, uint64_t bytes, uint64_t* cap) {
    *cap = bytes;
    if (!host) return cudaMalloc(p, bytes);
    if (ctx->host_arena && ctx->host_arena_bytes >= bytes) {
        *p = ctx->host_arena;
        *cap = ctx->host_arena_bytes;
        ctx->host_arena = nullptr;
        ctx->host_arena_bytes = 0;
        return cudaSuccess;
    }
    return cudaHostAlloc(p, bytes, cudaHostAllocPortable);
}

kc_status capture_mem(kc_ctx* ctx, const kc_dispatch* d, const kc_region* regions, size_t n, kc_capture_mode mode,
                      kc_snapshot** out, kc_capture_report* rep_out, bool host, const kc_snapshot* base,
                      const std::function<CUresult()>* forward = nullptr);
}  // namespace

extern "C" kc_status kc_capture_dev(kc_ctx* ctx, const kc_dispatch* d, const kc_region* regions, size_t n,
                                    kc_capture_mode mode, kc_snapshot** out, kc_capture_report* rep_out) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    return capture_mem(ctx, d, regions, n, mode, out, rep_out, false, nullptr);
}

extern "C" kc_status kc_capture_host(kc_ctx* ctx, const kc_dispatch* d, const kc_region* regions, size_t n,
                                     kc_capture_mode mode, kc_snapshot** out, kc_capture_report* rep_out) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    return capture_mem(ctx, d, regions, n, mode, out, rep_out, true, nullptr);
}

extern "C" kc_status kc_capture_incr(kc_ctx* ctx, const kc_dispatch* d, const kc_region* regions, size_t n,
                                     kc_capture_mode mode, const kc_snapshot* base, int host, kc_snapshot** out,
                                     kc_capture_report* rep_out) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    if (base && base->ctx != ctx) return set_err(ctx, KC_ERR_ARG, "kc_capture_incr: base snapshot of another ctx");
    return capture_mem(ctx, d, regions, n, mode, out, rep_out, host != 0, base);
}

extern "C" kc_status kc_dev_arena_reserve(kc_ctx* ctx, uint64_t bytes) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    if (!ctx) return KC_ERR_ARG;
    if (!bind_device(ctx)) return set_err(ctx, KC_ERR_CUDA, "cannot bind device");
    cudaDeviceSynchronize();
    if (bytes == 0) {
        ctx->dev_arena.release();
        for (auto& kv : ctx->phys_park) KC_DRV(cuMemRelease)(kv.second);
        ctx->phys_park.clear();
        ctx->phys_park_bytes = 0;
        return KC_OK;
    }
    if (ctx->dev_arena.size >= bytes) return KC_OK;
    ArenaBuf ab;  // allocate, then park it through the destructor
    ab.ctx = ctx;
    if (!vmm_arena_alloc(ctx, ab, bytes))
        return set_err(ctx, KC_ERR_NOMEM, "kc_dev_arena_reserve: cannot map a %llu-byte VMM arena",
                       (unsigned long long)bytes);
    return KC_OK;
}

extern "C" kc_status kc_host_arena_reserve(kc_ctx* ctx, uint64_t bytes) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    if (!ctx) return KC_ERR_ARG;
    if (!bind_device(ctx)) return set_err(ctx, KC_ERR_CUDA, "cannot bind device");
    if (bytes == 0) {
        if (ctx->host_arena) cudaFreeHost(ctx->host_arena);
        ctx->host_arena = nullptr;
        ctx->host_arena_bytes = 0;
        return KC_OK;
    }
    if (ctx->host_arena_bytes >= bytes) return KC_OK;
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        return set_err(ctx, KC_ERR_NOMEM, "kc_host_arena_reserve: cannot pin %llu bytes", (unsigned long long)bytes);
    }
    if (ctx->host_arena) cudaFreeHost(ctx->host_arena);
    ctx->host_arena = p;
    ctx->host_arena_bytes = bytes;
    return KC_OK;
}

namespace {
kc_status capture_mem(kc_ctx* ctx, const kc_dispatch* d, const kc_region* regions, size_t n, kc_capture_mode mode,
                      kc_snapshot** out, kc_capture_report* rep_out, bool host, const kc_snapshot* base,
                      const std::function<CUresult()>* forward) {
    if (!ctx) return KC_ERR_ARG;
    if (ctx->poisoned) return KC_ERR_CUDA;
    if (!bind_device(ctx)) return set_err(ctx, KC_ERR_CUDA, "cannot bind device");
    if (!d || !out) return set_err(ctx, KC_ERR_ARG, "kc_capture_dev: dispatch and out are required");
    if (mode != KC_MODE_PRE_W && mode != KC_MODE_POST) return set_err(ctx, KC_ERR_ARG, "kc_capture_dev: bad mode");
    *out = nullptr;
    kc_capture_report rep;
    memset(&rep, 0, sizeof rep);
    const double t0 = now_s();
    double tl = t0;
    cudaStream_t cs = (cudaStream_t)d->stream;
    std::vector<kc_region> list;
    if (regions) {
        list.assign(regions, regions + n);
    } else {
        std::lock_guard<std::mutex> lk(ctx->mu);
        for (auto& kv : ctx->live) list.push_back(kv.second);
    }
    list.erase(std::remove_if(list.begin(), list.end(), [](const kc_region& r) { return r.size == 0; }), list.end());
    std::sort(list.begin(), list.end(), [](const kc_region& a, const kc_region& b) { return a.base < b.base; });
    for (size_t i = 1; i < list.size(); ++i)
        if (list[i].base < list[i - 1].base + list[i - 1].size)
            return set_err(ctx, KC_ERR_ARG, "kc_capture_dev: regions overlap at 0x%llx",
                           (unsigned long long)list[i].base);
    // ---- resolve the function
    CUfunction f = (CUfunction)d->func;
    CUmodule own_mod = nullptr;
    if (!f) {
        if (!d->image || !d->mangled) return set_err(ctx, KC_ERR_ARG, "kc_capture_dev: need func or image+mangled");
        KC_CHECK_CU(ctx, KC_DRV(cuModuleLoadData)(&own_mod, d->image), "cuModuleLoadData");
        if (KC_DRV(cuModuleGetFunction)(&f, own_mod, d->mangled) != CUDA_SUCCESS) {
            KC_DRV(cuModuleUnload)(own_mod);
            return set_err(ctx, KC_ERR_ARG, "kc_capture_dev: symbol %s not found in image", d->mangled);
        }
        const CUresult r = allow_dynamic_smem(f, d->smem_bytes);
        if (r != CUDA_SUCCESS) {
            KC_DRV(cuModuleUnload)(own_mod);
            return cu_err(ctx, r, "kc_capture_dev: dynamic shared memory attribute");
        }
    }
    kc_snapshot* sn = new kc_snapshot();
    sn->ctx = ctx;
    sn->host = host;
    SnapDesc& D = sn->desc;
    D.mode = mode;
    D.mangled = d->mangled ? d->mangled : "";
    if (D.mangled.empty()) {
        const char* nm = nullptr;
        if (KC_DRV(cuFuncGetName)(&nm, f) == CUDA_SUCCESS && nm) D.mangled = nm;
    }
    for (size_t i = 0; i < 4096; ++i) {
        size_t o = 0, z = 0;
        if (KC_DRV(cuFuncGetParamInfo)(f, i, &o, &z) != CUDA_SUCCESS) break;
        D.layout.emplace_back(o, z);
    }
    auto fail = [&](kc_status st) {
        if (own_mod) KC_DRV(cuModuleUnload)(own_mod);
        kc_snapshot_free(sn);
        return st;
    };
    if (!D.layout.empty() && d->kernarg && d->kernarg_size != D.layout.back().first + D.layout.back().second)
        return fail(set_err(ctx, KC_ERR_ARG, "kc_capture_dev: kernarg_size %u != parameter buffer size %zu",
                            d->kernarg_size, D.layout.back().first + D.layout.back().second));
    for (int i = 0; i < 3; ++i) {
        D.grid[i] = d->grid[i];
        D.block[i] = d->block[i];
    }
    D.smem = d->smem_bytes;
    dispatch_cluster(d, D.cluster);
    D.flags = d->flags;
    if (d->kernarg && d->kernarg_size)
        D.kernarg.assign((const uint8_t*)d->kernarg, (const uint8_t*)d->kernarg + d->kernarg_size);
    ModCapture mc;  // F3
    {
        kc_status mst = module_capture_pre(ctx, d, f, own_mod, mc);
        if (mst != KC_OK) return fail(mst);
    }
    D.image = mc.image;

    // ---- A3 bracket: quiesce, liveness, K1 pre-manifest
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return fail(cuda_err(ctx, e, "kc_capture_dev: quiesce"));
    trace("setup + quiesce", tl);
    std::vector<kc_region> live;
    std::vector<uint64_t> pre_off;  // manifest offset per region (ok regions)
    for (auto& r : list) {
        SnapRegion sr;
        sr.r = r;
        sr.hx = hex_base(r.base);
        sr.n_chunks = (r.size + kChunk - 1) / kChunk;
        sr.ok = region_live(ctx, r.base, r.size);
        pre_off.push_back(kc_count_chunks(live.data(), live.size()));
        if (sr.ok) live.push_back(r);
        D.regions.push_back(std::move(sr));
    }
    rep.n_regions = D.regions.size();
    double t = now_s();
    std::vector<uint64_t> pre_h, pre_dig, post_h, post_dig;
    uint64_t pre_snap = 0, post_snap = 0;
    double t_copy = 0;
    // Fused capture pass (K6): a full PRE_W capture into a device arena stores
    // every live byte, so the plan does not depend on the hashes and one HBM
    // read yields both the pre-manifest and the stored copy (KC_NO_FUSED_CAPTURE=1:
    // K1 then copies, for comparison).
    bool full_dev = !base && !host && !getenv("KC_NO_FUSED_CAPTURE");
    for (auto& r : live) full_dev = full_dev && (r.base & 15) == 0;
    const bool fused = full_dev && mode == KC_MODE_PRE_W;       // K6 on the pre-state
    const bool fused_post = full_dev && mode == KC_MODE_POST;   // K6 on the post-state
    // every ok region one run of this snapshot's own arena; dst = the arena address per live region
    auto plan_full = [&](std::vector<uint64_t>& dst) -> kc_status {
        kc_status s2 = ensure_stream(ctx);
        if (s2 != KC_OK) return s2;
        sn->runs.assign(D.regions.size(), {});
        std::vector<uint64_t> aoff(D.regions.size(), 0);
        uint64_t total = 0;
        for (size_t i = 0; i < D.regions.size(); ++i) {
            if (!D.regions[i].ok) continue;
            total = (total + 255) / 256 * 256;
            aoff[i] = total;
            total += D.regions[i].r.size;
        }
        sn->arena_bytes = total;
        if (total) {
            auto ab = std::make_shared<ArenaBuf>();
            ab->ctx = ctx;
            if (!vmm_arena_alloc(ctx, *ab, total) && arena_alloc(ctx, false, &ab->p, total, &ab->cap) != cudaSuccess) {
                cudaGetLastError();
                ab->p = nullptr;
                return set_err(ctx, KC_ERR_NOMEM, "kc_capture_dev: cannot allocate a %llu-byte arena",
                               (unsigned long long)total);
            }
            sn->arena = ab;
            for (size_t i = 0; i < D.regions.size(); ++i) {
                if (!D.regions[i].ok) continue;
                const uint64_t src = (uint64_t)ab->p + aoff[i];
                sn->runs[i].push_back({0, D.regions[i].r.size, src});
                dst.push_back(src);
            }
        }
        return KC_OK;
    };
    kc_status st = KC_OK;
    if (fused) {
        std::vector<uint64_t> dst;
        st = plan_full(dst);
        if (st != KC_OK) return fail(st);
        trace("plan + arena alloc", tl);
        const double tc = now_s();
        st = hash_regions_sync(ctx, live, pre_h, &pre_dig, &pre_snap, nullptr, cs, dst.empty() ? nullptr : dst.data());
        t_copy += now_s() - tc;
        rep.dma_calls += live.empty() ? 0 : 1;
        if (st != KC_OK) return fail(st);
        rep.t_hash_pre_s = now_s() - tc;
        trace("K6 hash + copy", tl);
    } else {
        st = hash_regions_sync(ctx, live, pre_h, &pre_dig, &pre_snap, nullptr, cs);
        if (st != KC_OK) return fail(st);
        rep.t_hash_pre_s = now_s() - t;
        trace("regions + K1 pre", tl);
    }
    rep.n_chunks = pre_h.size();
    for (auto& r : live) rep.total_bytes += r.size;

    // ---- the stored bytes: runs per region; chunks whose stored-state hash equals
    // the base's at the same (region, chunk) reference the base, the rest are
    // copied into this snapshot's own arena (256 B aligned runs)
    std::map<uint64_t, size_t> base_idx;
    if (base)
        for (size_t j = 0; j < base->desc.regions.size(); ++j)
            if (base->desc.regions[j].ok) base_idx[base->desc.regions[j].r.base] = j;
    if (base) {
        sn->deps = base->deps;
        if (base->arena) sn->deps.push_back(base->arena);
    }
    auto snapshot_regions = [&](const std::vector<uint64_t>& h /* stored-state manifest, live-region order */)
        -> kc_status {
        struct OwnRun { size_t i, r; uint64_t aoff; };
        std::vector<OwnRun> own;
        sn->runs.assign(D.regions.size(), {});
        uint64_t total = 0;
        for (size_t i = 0; i < D.regions.size(); ++i) {
            const SnapRegion& sr = D.regions[i];
            if (!sr.ok) continue;
            const SnapRegion* bsr = nullptr;
            const std::vector<kc_snapshot::Run>* bruns = nullptr;
            if (base) {
                auto it = base_idx.find(sr.r.base);
                if (it != base_idx.end() && base->desc.regions[it->second].r.size == sr.r.size) {
                    bsr = &base->desc.regions[it->second];
                    bruns = &base->runs[it->second];
                }
            }
            size_t bj = 0;
            auto& runs = sn->runs[i];
            for (uint64_t kc = 0; kc < sr.n_chunks; ++kc) {
                const uint64_t roff = kc * kChunk, len = std::min<uint64_t>(kChunk, sr.r.size - roff);
                uint64_t bsrc = 0;
                if (bsr && bsr->manifest[kc] == h[pre_off[i] + kc]) {
                    while ((*bruns)[bj].roff + (*bruns)[bj].len <= roff) ++bj;
                    bsrc = (*bruns)[bj].src + (roff - (*bruns)[bj].roff);
                    sn->shared_bytes += len;
                }
                if (bsrc) {
                    if (!runs.empty() && runs.back().roff + runs.back().len == roff &&
                        runs.back().src + runs.back().len == bsrc &&
                        (own.empty() || own.back().i != i || own.back().r != runs.size() - 1))
                        runs.back().len += len;
                    else
                        runs.push_back({roff, len, bsrc});
                } else {
                    if (!own.empty() && own.back().i == i && own.back().r == runs.size() - 1 &&
                        runs.back().roff + runs.back().len == roff) {
                        runs.back().len += len;
                    } else {
                        total = (total + 255) / 256 * 256;
                        own.push_back({i, runs.size(), total});
                        runs.push_back({roff, len, 0});
                    }
                    total += len;
                }
            }
        }
        sn->arena_bytes = total;
        trace("plan runs", tl);
        if (total) {
            auto ab = std::make_shared<ArenaBuf>();
            ab->ctx = ctx;
            ab->host = host;
            if (arena_alloc(ctx, host, &ab->p, total, &ab->cap) != cudaSuccess) {
                cudaGetLastError();
                ab->p = nullptr;
                return set_err(ctx, KC_ERR_NOMEM, "kc_capture_%s: cannot allocate a %llu-byte arena",
                               host ? "host" : "dev", (unsigned long long)total);
            }
            sn->arena = ab;
        }
        trace("arena alloc", tl);
        std::vector<std::array<uint64_t, 3>> ranges;
        for (const OwnRun& o : own) {
            kc_snapshot::Run& ru = sn->runs[o.i][o.r];
            ru.src = (uint64_t)sn->arena->p + o.aoff;
            ranges.push_back({D.regions[o.i].r.base + ru.roff, ru.src, ru.len});
        }
        const double tc = now_s();  // t_d2h_s: the copies only (planning and allocation excluded)
        kc_status s2 = copy_ranges_d2d(ctx, ranges, ctx->copy_stream ? ctx->copy_stream : cs, &rep.dma_calls);
        cudaStreamSynchronize(ctx->copy_stream);
        t_copy += now_s() - tc;
        trace("copy", tl);
        return s2;
    };
    st = ensure_stream(ctx);  // in-memory sinks copy arena <-> device directly: no staging ring
    if (st != KC_OK) return fail(st);
    if (mode == KC_MODE_PRE_W && !fused) {
        st = snapshot_regions(pre_h);
        if (st != KC_OK) return fail(st);
    }
    // ---- forward the dispatch (interposed mode: the application launches it)
    t = now_s();
    if (forward) {
        const CUresult r = (*forward)();
        if (r != CUDA_SUCCESS) return fail(cu_err(ctx, r, "kc_capture: intercepted dispatch"));
    } else {
        uint32_t cl[3];
        dispatch_cluster(d, cl);
        CUresult r = launch_packed(f, d->grid, d->block, d->smem_bytes, (CUstream)cs, d->kernarg, d->kernarg_size, cl,
                                   d->flags);
        if (r == CUDA_SUCCESS) r = KC_DRV(cuStreamSynchronize)((CUstream)cs);
        if (r != CUDA_SUCCESS) return fail(cu_err(ctx, r, "kc_capture_dev: target dispatch"));
    }
    rep.t_dispatch_s = now_s() - t;
    trace("dispatch", tl);
    {
        kc_status mst = module_capture_post(ctx, mc);
        if (own_mod) {
            KC_DRV(cuModuleUnload)(own_mod);
            own_mod = nullptr;
        }
        if (mst != KC_OK) return fail(mst);
        D.modvars = std::move(mc.vars);
    }
    // ---- K1 post-manifest + W (POST full capture: K6 also stores the post-state)
    std::vector<uint64_t> post_dst;
    if (fused_post) {
        st = plan_full(post_dst);
        if (st != KC_OK) return fail(st);
        trace("plan + arena alloc", tl);
    }
    t = now_s();
    st = hash_regions_sync(ctx, live, post_h, &post_dig, &post_snap, nullptr, cs,
                           post_dst.empty() ? nullptr : post_dst.data());
    if (st != KC_OK) return fail(st);
    rep.t_hash_post_s = now_s() - t;
    if (fused_post) {
        t_copy += rep.t_hash_post_s;
        rep.dma_calls += live.empty() ? 0 : 1;
    }
    trace(fused_post ? "K6 post hash + copy" : "K1 post", tl);
    {
        size_t j = 0;  // (W from the manifests: host loop over the chunks)
        for (size_t i = 0; i < D.regions.size(); ++i) {
            SnapRegion& sr = D.regions[i];
            if (!sr.ok) continue;
            const uint64_t* pre = pre_h.data() + pre_off[i];
            const uint64_t* post = post_h.data() + pre_off[i];
            for (uint64_t k = 0; k < sr.n_chunks; ++k)
                if (pre[k] != post[k]) sr.written.push_back(k);
            sr.post_manifest.assign(post, post + sr.n_chunks);
            rep.written_chunks += sr.written.size();
            sr.post_digest = post_dig[j];
            if (mode == KC_MODE_PRE_W) {
                sr.manifest.assign(pre, pre + sr.n_chunks);
                sr.digest = pre_dig[j];
            } else {
                sr.manifest = sr.post_manifest;
                sr.digest = post_dig[j];
            }
            ++j;
        }
    }
    D.snapshot_digest = mode == KC_MODE_PRE_W ? pre_snap : post_snap;
    trace("W sets", tl);
    if (mode == KC_MODE_POST) {
        if (!fused_post) {
            st = snapshot_regions(post_h);
            if (st != KC_OK) return fail(st);
        }
    } else if (rep.written_chunks) {
        uint64_t wtot = 0;
        for (auto& sr : D.regions) {
            sn->w_off.push_back(wtot);
            for (uint64_t k : sr.written) wtot += std::min<uint64_t>(kChunk, sr.r.size - k * kChunk);
        }
        sn->w_bytes = wtot;
        if ((host ? cudaHostAlloc(&sn->warena, wtot, cudaHostAllocPortable) : cudaMalloc(&sn->warena, wtot)) !=
            cudaSuccess) {
            cudaGetLastError();
            sn->warena = nullptr;
            return fail(set_err(ctx, KC_ERR_NOMEM, "kc_capture_dev: W arena of %llu bytes", (unsigned long long)wtot));
        }
        std::vector<std::array<uint64_t, 3>> ranges;
        for (size_t i = 0; i < D.regions.size(); ++i) {
            uint64_t o = sn->w_off[i];
            for (uint64_t k : D.regions[i].written) {
                const uint64_t len = std::min<uint64_t>(kChunk, D.regions[i].r.size - k * kChunk);
                ranges.push_back({D.regions[i].r.base + k * kChunk, (uint64_t)sn->warena + o, len});
                o += len;
            }
        }
        trace("W plan + W arena", tl);
        t = now_s();
        st = copy_ranges_d2d(ctx, ranges, ctx->copy_stream, &rep.dma_calls);
        cudaStreamSynchronize(ctx->copy_stream);
        t_copy += now_s() - t;
        if (st != KC_OK) return fail(st);
    }
    if (sn->w_off.empty()) sn->w_off.assign(D.regions.size(), 0);
    rep.t_d2h_s = t_copy;  // device-to-device for a device arena
    rep.d2h_bytes = sn->arena_bytes + sn->w_bytes;  // bytes moved into the arenas (D2H or D2D)
    for (auto& sr : D.regions)
        if (!sr.ok) rep.n_failed_regions++;
    rep.snapshot_digest = D.snapshot_digest;
    trace("W + finish", tl);
    rep.t_total_s = now_s() - t0;
    sn->rep = rep;
    if (rep_out) *rep_out = rep;
    *out = sn;
    if (rep.n_failed_regions) {
        set_err(ctx, KC_PARTIAL, "kc_capture_dev: %llu region(s) were not live", (unsigned long long)rep.n_failed_regions);
        return KC_PARTIAL;
    }
    return KC_OK;
}
}  // namespace

extern "C" kc_status kc_restore_dev(kc_ctx* ctx, const kc_snapshot* s, kc_restored** out, kc_restore_report* rep_out) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    if (!ctx || !s || !out) return KC_ERR_ARG;
    if (ctx->poisoned) return KC_ERR_CUDA;
    if (s->ctx != ctx || ctx->device != s->ctx->device)
        return set_err(ctx, KC_ERR_ARG, "kc_restore_dev: the snapshot lives on another ctx/device");
    *out = nullptr;
    kc_restore_report rep;
    memset(&rep, 0, sizeof rep);
    const double t0 = now_s();
    for (auto& sr : s->desc.regions)
        if (!sr.ok) rep.n_failed_regions++;
    DevSource src(s);
    kc_status st = restore_core(ctx, s->desc, src, out, rep_out, rep, t0);
    if (st == KC_OK) (*out)->dev_snap = s;
    return st;
}

extern "C" kc_status kc_restore_dev_into(kc_ctx* ctx, const kc_snapshot* s, kc_restored* h,
                                        kc_restore_report* rep_out) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    if (!ctx || !s || !h) return KC_ERR_ARG;
    if (ctx->poisoned) return KC_ERR_CUDA;
    if (s->ctx != ctx || h->ctx != ctx)
        return set_err(ctx, KC_ERR_ARG, "kc_restore_dev_into: snapshot and restore must live on this ctx");
    const SnapDesc& d = s->desc;
    if (d.regions.size() != h->regions.size())
        return set_err(ctx, KC_ERR_ARG, "kc_restore_dev_into: %zu regions in the snapshot, %zu in the restore",
                       d.regions.size(), h->regions.size());
    for (size_t i = 0; i < d.regions.size(); ++i) {
        const auto& sr = d.regions[i];
        const auto& rr = h->regions[i];
        if (sr.r.base != rr.r.base || sr.r.size != rr.r.size || sr.ok != rr.ok)
            return set_err(ctx, KC_ERR_ARG, "kc_restore_dev_into: region %zu (%#llx, %llu B) is not the live "
                           "restore's", i, (unsigned long long)sr.r.base, (unsigned long long)sr.r.size);
    }
    if (!bind_device(ctx)) return set_err(ctx, KC_ERR_CUDA, "cannot bind device");
    kc_restore_report rep;
    memset(&rep, 0, sizeof rep);
    const double t0 = now_s();
    rep.n_regions = d.regions.size();
    for (auto& sr : d.regions)
        if (!sr.ok) rep.n_failed_regions++;
    rep.n_spans = h->spans.size();
    // the live restore takes this snapshot's dispatch, written sets and post manifests
    if (h->stash_pre) cudaFree(h->stash_pre);
    h->stash_pre = h->stash_ref = nullptr;
    h->stash_bytes = 0;
    if (h->module && h->image != d.image) {  // another code object: the next replay reloads it
        KC_DRV(cuModuleUnload)(h->module);
        h->module = nullptr;
    }
    h->modvar_checked = h->modvar_mismatch = 0;
    bind_dispatch_fields(h, d);
    for (size_t i = 0; i < d.regions.size(); ++i) {
        auto& rr = h->regions[i];
        rr.hexbase = d.regions[i].hx;
        rr.n_chunks = d.regions[i].n_chunks;
        rr.written = d.regions[i].written;
        rr.post_manifest = d.regions[i].post_manifest;
    }
    DevSource src(s);
    const kc_status st = restore_fill(ctx, h, d, src, rep);
    rep.t_total_s = now_s() - t0;
    if (rep_out) *rep_out = rep;
    if (st == KC_OK) h->dev_snap = s;
    return st;
}

static kc_status save_impl(kc_ctx* ctx, const kc_snapshot* s, const char* dir_c, bool publish) {
    if (!ctx || !s || !dir_c) return KC_ERR_ARG;
    if (ctx->poisoned) return KC_ERR_CUDA;
    if (!bind_device(ctx)) return set_err(ctx, KC_ERR_CUDA, "cannot bind device");
    const std::string dir = dir_c;
    const SnapDesc& D = s->desc;
    // publish: the region bytes stay in this process's device arena, shared by
    // CUDA IPC; every ok region must be one run inside the snapshot's own arena
    std::string arena_json;
    if (publish) {
        if (s->host || !s->arena || !s->arena->p)
            return set_err(ctx, KC_ERR_STATE, "kc_snapshot_publish: needs a device snapshot with its own arena");
        // VMM arena: export a POSIX fd that the replay process duplicates with
        // pidfd_getfd and maps (cuMemImportFromShareableHandle); else a legacy
        // CUDA IPC handle (cudaIpcOpenMemHandle, measured ~160 ms for 30 GB)
        std::string how;
        if (s->arena->vmm) {
            if (s->arena->export_fd < 0) {
                int fd = -1;
                KC_CHECK_CU(ctx, KC_DRV(cuMemExportToShareableHandle)(&fd, s->arena->vmm_h,
                                                                     CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
                            "cuMemExportToShareableHandle");
                s->arena->export_fd = fd;
            }
            how = "\"kind\": \"vmm_fd\",\n  \"fd\": " + std::to_string(s->arena->export_fd) +
                  ",\n  \"mapped_bytes\": " + std::to_string((unsigned long long)s->arena->vmm_size);
        } else {
            cudaIpcMemHandle_t ih;
            KC_CHECK_CUDA(ctx, cudaIpcGetMemHandle(&ih, s->arena->p), "cudaIpcGetMemHandle");
            char hx[2 * sizeof ih + 1];
            for (size_t i = 0; i < sizeof ih; ++i) snprintf(hx + 2 * i, 3, "%02x", (unsigned)((const uint8_t*)&ih)[i]);
            how = std::string("\"kind\": \"cuda_ipc\",\n  \"ipc_handle\": \"") + hx + "\"";
        }
        arena_json = "{\n  \"format\": \"kc-device-arena/1\",\n  \"pid\": " + std::to_string((long long)getpid()) +
                     ",\n  \"device\": " + std::to_string(ctx->device) + ",\n  \"arena_bytes\": " +
                     std::to_string((unsigned long long)s->arena_bytes) + ",\n  " + how + ",\n  \"regions\": [";
        bool first = true;
        for (size_t i = 0; i < D.regions.size(); ++i) {
            if (!D.regions[i].ok) continue;
            const auto& runs = s->runs[i];
            const uint64_t a0 = (uint64_t)s->arena->p;
            if (runs.size() != 1 || runs[0].roff != 0 || runs[0].len != D.regions[i].r.size || runs[0].src < a0 ||
                runs[0].src + runs[0].len > a0 + s->arena_bytes)
                return set_err(ctx, KC_ERR_STATE, "kc_snapshot_publish: region %s is not one run of the snapshot's "
                               "own arena (an incremental snapshot)", D.regions[i].hx.c_str());
            arena_json += std::string(first ? "\n" : ",\n") + "    {\"base\": \"" + D.regions[i].hx +
                          "\", \"offset\": " + std::to_string((unsigned long long)(runs[0].src - a0)) + "}";
            first = false;
        }
        arena_json += "\n  ]\n}\n";
    }
    if (!mkdir_p(dir + "/memory") || !mkdir_p(dir + "/post") || !mkdir_p(dir + "/written"))
        return set_err(ctx, KC_ERR_IO, "kc_snapshot_save: cannot create %s", dir_c);
    unlink((dir + "/capture_complete").c_str());
    // metadata first
    if (!write_text(dir + "/dispatch.json", dispatch_json(D.mode, D.mangled, D.grid, D.block, D.smem,
                                                          (uint32_t)D.kernarg.size(), ctx->device, D.image,
                                                          D.layout, D.cluster, D.flags)) ||
        !write_file(dir + "/kernarg.bin", D.kernarg.data(), D.kernarg.size()) ||
        (!D.image.empty() && !write_file(dir + "/kernel.cubin", D.image.data(), D.image.size())) ||
        !write_module_vars(dir, D.modvars))
        return set_err(ctx, KC_ERR_IO, "kc_snapshot_save: cannot write metadata in %s", dir_c);
    std::vector<MetaRegion> mr;
    for (auto& sr : D.regions)
        mr.push_back({sr.r.base, sr.r.size, sr.n_chunks, sr.digest, sr.r.seq, sr.r.kind, sr.r.device, sr.ok});
    if (!write_text(dir + "/memory_regions.json", regions_json(mr)))
        return set_err(ctx, KC_ERR_IO, "kc_snapshot_save: cannot write memory_regions.json");
    unlink((dir + "/memory/device_arena.revoked").c_str());
    if (publish) {
        if (!write_text(dir + "/memory/device_arena.json", arena_json))
            return set_err(ctx, KC_ERR_IO, "kc_snapshot_publish: cannot write device_arena.json");
        s->published.push_back(dir);
    } else {
        unlink((dir + "/memory/device_arena.json").c_str());
    }
    // region files from the arena (parallel workers; none when publishing)
    const int T = io_threads();
    kc_status st = publish ? KC_OK : ensure_io(ctx, T);
    if (st != KC_OK) return st;
    // work items: 256 MiB pieces of every run, with the address its file offset maps to
    std::vector<IoItem> items;
    std::vector<uint64_t> item_base;
    for (size_t i = 0; i < D.regions.size(); ++i) {
        if (!D.regions[i].ok || publish) continue;
        const std::string path = dir + "/memory/region_" + D.regions[i].hx + ".bin";
        int fd = open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
        const bool ok = fd >= 0 && ftruncate(fd, (off_t)D.regions[i].r.size) == 0;
        if (fd >= 0) close(fd);
        if (!ok) return set_err(ctx, KC_ERR_IO, "kc_snapshot_save: cannot create %s", path.c_str());
        for (const auto& ru : s->runs[i])
            for (uint64_t o = 0; o < ru.len; o += 256ull << 20) {
                items.push_back({i, ru.roff + o, std::min<uint64_t>(256ull << 20, ru.len - o)});
                item_base.push_back(ru.src - ru.roff);  // base + file offset = source address
            }
    }
    std::atomic<int> bad{0};
    std::atomic<uint64_t> calls{0};
    run_pool(T, items.size(), [&](int t, size_t k) {
        if (bad) return;
        const IoItem& it = items[k];
        cudaSetDevice(ctx->device);
        const std::string path = dir + "/memory/region_" + D.regions[it.region].hx + ".bin";
        int fd = open(path.c_str(), O_WRONLY);
        std::string err;
        // item_d2h copies [base + off, +len) -> file offset off: base = this region's arena slot
        const bool ok = fd >= 0 && item_d2h(ctx, ctx->io[t], item_base[k], it, fd, calls, err);
        if (fd >= 0) close(fd);
        if (!ok) bad = 1;
    });
    if (bad) return set_err(ctx, KC_ERR_IO, "kc_snapshot_save: region copy failed");
    std::vector<LogRegion> lr;
    for (size_t i = 0; i < D.regions.size(); ++i) {
        const SnapRegion& sr = D.regions[i];
        lr.push_back({sr.r.base, sr.post_digest, (uint64_t)sr.written.size(), sr.ok,
                      sr.ok ? "" : "not inside a live CUDA allocation before the dispatch"});
        if (!sr.ok) continue;
        write_file(dir + "/memory/region_" + sr.hx + ".xxh64", sr.manifest.data(), 8 * sr.manifest.size());
        write_file(dir + "/post/region_" + sr.hx + ".xxh64", sr.post_manifest.data(), 8 * sr.post_manifest.size());
        write_file(dir + "/written/region_" + sr.hx + ".idx", sr.written.data(), 8 * sr.written.size());
        if (D.mode == KC_MODE_PRE_W && !sr.written.empty()) {
            uint64_t wb = 0;
            for (uint64_t k : sr.written) wb += std::min<uint64_t>(kChunk, sr.r.size - k * kChunk);
            std::vector<uint8_t> host(wb);
            KC_CHECK_CUDA(ctx, cudaMemcpy(host.data(), (const uint8_t*)s->warena + s->w_off[i], wb,
                                          cudaMemcpyDefault), "D2H written chunks");
            if (!write_file(dir + "/written/region_" + sr.hx + ".bin", host.data(), wb))
                return set_err(ctx, KC_ERR_IO, "kc_snapshot_save: cannot write written chunks");
        }
    }
    kc_capture_report rep = s->rep;
    rep.dma_calls += calls.load();
    if (!write_text(dir + "/capture_log.json", capture_log_json(lr, rep, ctx->io_chunk, ctx->depth, s->host ? "host" : "device")) ||
        !write_file(dir + "/capture_complete", "", 0))
        return set_err(ctx, KC_ERR_IO, "kc_snapshot_save: cannot write capture_log.json / sentinel");
    return KC_OK;
}

extern "C" kc_status kc_snapshot_save(kc_ctx* ctx, const kc_snapshot* s, const char* dir_c) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    return save_impl(ctx, s, dir_c, false);
}

extern "C" kc_status kc_snapshot_publish(kc_ctx* ctx, const kc_snapshot* s, const char* dir_c) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    return save_impl(ctx, s, dir_c, true);
}

// Load a kc-snapshot/1 directory into an in-memory snapshot: the edit -> replay
// -> validate loop then restores from HBM (or pinned host memory) each time
// instead of re-reading the files (capture once, replay many).
extern "C" kc_status kc_snapshot_load(kc_ctx* ctx, const char* dir_c, int host, kc_snapshot** out) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    if (!ctx || !dir_c || !out) return KC_ERR_ARG;
    if (ctx->poisoned) return KC_ERR_CUDA;
    if (!bind_device(ctx)) return set_err(ctx, KC_ERR_CUDA, "cannot bind device");
    *out = nullptr;
    const double t0 = now_s();
    kc_restore_report rr;
    memset(&rr, 0, sizeof rr);
    kc_snapshot* sn = new kc_snapshot();
    sn->ctx = ctx;
    sn->host = host != 0;
    SnapDesc& D = sn->desc;
    kc_status st = load_desc_files(ctx, dir_c, D, rr);
    if (st != KC_OK) {
        delete sn;
        return st;
    }
    auto fail = [&](kc_status e) {
        kc_snapshot_free(sn);
        return e;
    };
    st = ensure_stream(ctx);
    if (st != KC_OK) return fail(st);
    // the stored bytes: one run per ok region in this snapshot's own arena
    sn->runs.assign(D.regions.size(), {});
    uint64_t total = 0;
    std::vector<uint64_t> aoff(D.regions.size(), 0);
    for (size_t i = 0; i < D.regions.size(); ++i) {
        if (!D.regions[i].ok) continue;
        total = (total + 255) / 256 * 256;
        aoff[i] = total;
        total += D.regions[i].r.size;
    }
    sn->arena_bytes = total;
    FileSource src(dir_c);
    src.dst.assign(D.regions.size(), 0);
    if (total) {
        auto ab = std::make_shared<ArenaBuf>();
        ab->ctx = ctx;
        ab->host = sn->host;
        if ((sn->host || !vmm_arena_alloc(ctx, *ab, total)) &&
            arena_alloc(ctx, sn->host, &ab->p, total, &ab->cap) != cudaSuccess) {
            cudaGetLastError();
            ab->p = nullptr;
            return fail(set_err(ctx, KC_ERR_NOMEM, "kc_snapshot_load: cannot allocate a %llu-byte arena",
                                (unsigned long long)total));
        }
        sn->arena = ab;
        for (size_t i = 0; i < D.regions.size(); ++i) {
            if (!D.regions[i].ok) continue;
            src.dst[i] = (uint64_t)ab->p + aoff[i];
            sn->runs[i].push_back({0, D.regions[i].r.size, src.dst[i]});
        }
    }
    st = ensure_pinned(ctx);
    if (st == KC_OK) st = src.copy_in(ctx, D, rr);
    cudaError_t ce = cudaStreamSynchronize(ctx->copy_stream);
    if (st == KC_OK && ce != cudaSuccess) st = cuda_err(ctx, ce, "kc_snapshot_load: copy-in");
    if (st != KC_OK) return fail(st);
    // verify the loaded bytes against the manifests and recompute the region
    // digests (K1 over the arena; a pinned host arena is read over PCIe)
    if (total) {
        std::vector<kc_region> regs;
        for (size_t i = 0; i < D.regions.size(); ++i)
            if (D.regions[i].ok) regs.push_back(kc_region{src.dst[i], D.regions[i].r.size, ctx->device, 0, 0});
        std::vector<uint64_t> got, digs;
        st = hash_regions_sync(ctx, regs, got, &digs, nullptr, nullptr, ctx->copy_stream);
        if (st != KC_OK) return fail(st);
        for (size_t i = 0, j = 0; i < D.regions.size(); ++i)
            if (D.regions[i].ok) D.regions[i].digest = digs[j++];
        uint64_t c = 0, bad = 0;
        for (auto& sr : D.regions) {
            if (!sr.ok) continue;
            for (uint64_t k = 0; k < sr.n_chunks; ++k)
                bad += sr.manifest.size() != sr.n_chunks || sr.manifest[k] != got[c + k];
            c += sr.n_chunks;
        }
        if (bad)
            return fail(set_err(ctx, KC_ERR_MANIFEST_MISMATCH, "kc_snapshot_load: %llu chunk(s) do not match the "
                                "manifest", (unsigned long long)bad));
    }
    // W's post bytes (PRE_W) into the W arena
    uint64_t wtot = 0;
    for (auto& sr : D.regions) {
        sn->w_off.push_back(wtot);
        for (uint64_t k : sr.written) wtot += std::min<uint64_t>(kChunk, sr.r.size - k * kChunk);
    }
    sn->w_bytes = D.mode == KC_MODE_PRE_W ? wtot : 0;
    if (sn->w_bytes) {
        if ((sn->host ? cudaHostAlloc(&sn->warena, wtot, cudaHostAllocPortable) : cudaMalloc(&sn->warena, wtot)) !=
            cudaSuccess) {
            cudaGetLastError();
            sn->warena = nullptr;
            return fail(set_err(ctx, KC_ERR_NOMEM, "kc_snapshot_load: W arena of %llu bytes", (unsigned long long)wtot));
        }
        for (size_t i = 0; i < D.regions.size(); ++i) {
            const SnapRegion& sr = D.regions[i];
            if (!sr.ok || sr.written.empty()) continue;
            uint64_t wb = 0;
            for (uint64_t k : sr.written) wb += std::min<uint64_t>(kChunk, sr.r.size - k * kChunk);
            st = src.written_ref(ctx, D, i, (uint8_t*)sn->warena + sn->w_off[i], wb);
            if (st != KC_OK) return fail(st);
        }
        ce = cudaStreamSynchronize(ctx->copy_stream);
        if (ce != cudaSuccess) return fail(cuda_err(ctx, ce, "kc_snapshot_load: W bytes"));
    }
    memset(&sn->rep, 0, sizeof sn->rep);
    sn->rep.n_regions = D.regions.size();
    sn->rep.n_chunks = 0;
    for (auto& sr : D.regions) {
        if (!sr.ok) continue;
        sn->rep.n_chunks += sr.n_chunks;
        sn->rep.total_bytes += sr.r.size;
        sn->rep.written_chunks += sr.written.size();
    }
    sn->rep.n_failed_regions = rr.n_failed_regions;
    {  // the snapshot digest as captured (it covers the captured VAs, not the arena's)
        std::string lt;
        kcj::Value lv;
        if (kcj::read_file(std::string(dir_c) + "/capture_log.json", lt) && kcj::Parser(lt).parse(lv) &&
            lv.get("snapshot_digest"))
            D.snapshot_digest = strtoull(lv.get("snapshot_digest")->s.c_str(), nullptr, 16);
    }
    sn->rep.snapshot_digest = D.snapshot_digest;
    sn->rep.d2h_bytes = rr.h2d_bytes;
    sn->rep.t_total_s = now_s() - t0;
    *out = sn;
    return KC_OK;
}

extern "C" uint64_t kc_snapshot_bytes(const kc_snapshot* s) { return s ? s->arena_bytes + s->w_bytes : 0; }

extern "C" uint64_t kc_snapshot_shared_bytes(const kc_snapshot* s) { return s ? s->shared_bytes : 0; }

extern "C" int kc_snapshot_is_host(const kc_snapshot* s) { return s && s->host ? 1 : 0; }

extern "C" void kc_snapshot_free(kc_snapshot* s) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    // revoke the directories this snapshot published: their bytes go with the arena
    if (s)
        for (const std::string& d : s->published) {
            const std::string j = d + "/memory/device_arena.json";
            struct stat sb;
            if (stat(j.c_str(), &sb) == 0) rename(j.c_str(), (d + "/memory/device_arena.revoked").c_str());
        }
    if (!s) return;
    if (s->ctx) bind_device(s->ctx);
    if (s->warena) {
        if (s->host) cudaFreeHost(s->warena); else cudaFree(s->warena);
    }
    delete s;  // the arenas go with their last reference (ArenaBuf)
}

extern "C" kc_status kc_restored_regions(kc_restored* h, kc_region* out, size_t cap, size_t* n_out) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    if (!h) return KC_ERR_ARG;
    size_t i = 0;
    for (auto& rr : h->regions) {
        if (out && i < cap) out[i] = rr.r;
        ++i;
    }
    if (n_out) *n_out = i;
    return KC_OK;
}

extern "C" void kc_release(kc_restored* h) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    if (!h) return;
    if (h->ctx) bind_device(h->ctx);
    cudaDeviceSynchronize();
    if (h->module) KC_DRV(cuModuleUnload)(h->module);
    if (h->stash_pre) cudaFree(h->stash_pre);  // stash_ref lives in the same allocation
    if (h->ipc_arena && h->ipc_vmm_size) {
        KC_DRV(cuMemUnmap)((CUdeviceptr)h->ipc_arena, h->ipc_vmm_size);
        KC_DRV(cuMemAddressFree)((CUdeviceptr)h->ipc_arena, h->ipc_vmm_size);
        KC_DRV(cuMemRelease)(h->ipc_vmm_h);
    } else if (h->ipc_arena) {
        cudaIpcCloseMemHandle(h->ipc_arena);
    }
    rollback(h);
    delete h;
}

// ====================================================================== replay
extern "C" kc_status kc_replay(kc_ctx* ctx, kc_restored* h, const kc_replay_opts* o, kc_replay_report* rep_out) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    if (!ctx || !h) return KC_ERR_ARG;
    if (ctx->poisoned) return KC_ERR_CUDA;
    if (!bind_device(ctx)) return set_err(ctx, KC_ERR_CUDA, "cannot bind device");
    kc_replay_opts dflt;
    memset(&dflt, 0, sizeof dflt);
    dflt.iterations = 1;
    if (!o) o = &dflt;
    const uint32_t iters = o->iterations ? o->iterations : 1;
    cudaStream_t s = (cudaStream_t)o->stream;
    CUmodule mod = nullptr;
    bool own = false;
    if (o->image_override) {
        KC_CHECK_CU(ctx, KC_DRV(cuModuleLoadData)(&mod, o->image_override), "cuModuleLoadData(override)");
        own = true;
    } else {
        if (!h->module) {
            if (h->image.empty())
                return set_err(ctx, KC_ERR_FORMAT, "kc_replay: the snapshot holds no code object (kernel.cubin)");
            KC_CHECK_CU(ctx, KC_DRV(cuModuleLoadData)(&h->module, h->image.data()), "cuModuleLoadData(kernel.cubin)");
        }
        mod = h->module;
    }
    // launch shape: as captured unless a variant overrides it
    const std::string sym = (o->overrides & KC_OVR_SYMBOL) && o->symbol ? std::string(o->symbol) : h->mangled;
    uint32_t grid[3], block[3];
    for (int i = 0; i < 3; ++i) {
        grid[i] = (o->overrides & KC_OVR_GRID) ? o->grid[i] : h->grid[i];
        block[i] = (o->overrides & KC_OVR_BLOCK) ? o->block[i] : h->block[i];
    }
    const uint32_t smem = (o->overrides & KC_OVR_SMEM) ? o->smem_bytes : h->smem;
    CUfunction f = nullptr;
    if (KC_DRV(cuModuleGetFunction)(&f, mod, sym.c_str()) != CUDA_SUCCESS) {
        if (own) KC_DRV(cuModuleUnload)(mod);
        return set_err(ctx, KC_ERR_ARG, "kc_replay: symbol %s not found in the code object", sym.c_str());
    }
    {
        const CUresult r = allow_dynamic_smem(f, smem);
        if (r != CUDA_SUCCESS) {
            if (own) KC_DRV(cuModuleUnload)(mod);
            return cu_err(ctx, r, "kc_replay: dynamic shared memory attribute");
        }
    }
    // F3: module variables into the replay module, after the memory restore and
    // before the dispatch; PRE_W restores the pre values,
    // POST the post values (the same state the region files hold)
    std::vector<std::pair<CUdeviceptr, const ModVarState*>> mv;
    uint32_t mv_restored = 0;
    if (!modvars_disabled())
        for (const ModVarState& v : h->modvars) {
            CUdeviceptr p = 0;
            size_t bytes = 0;
            if (KC_DRV(cuModuleGetGlobal)(&p, &bytes, mod, v.name.c_str()) != CUDA_SUCCESS || bytes != v.size) continue;
            mv.emplace_back(p, &v);
        }
    auto put_modvars = [&](bool only_written) -> kc_status {
        for (auto& pv : mv) {
            const ModVarState& v = *pv.second;
            if (only_written && v.pre == v.post) continue;
            const std::vector<uint8_t>& src = h->mode == KC_MODE_PRE_W ? v.pre : v.post;
            KC_CHECK_CUDA(ctx, cudaMemcpyAsync((void*)pv.first, src.data(), v.size, cudaMemcpyHostToDevice, s),
                          "restore module variable");
        }
        return KC_OK;
    };
    {
        kc_status mst = put_modvars(false);
        if (mst != KC_OK) {
            if (own) KC_DRV(cuModuleUnload)(mod);
            return mst;
        }
        mv_restored = (uint32_t)mv.size();
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double sum = 0, mn = 1e300, mx = 0;
    kc_status res = KC_OK;
    for (uint32_t it = 0; it < iters; ++it) {
        if (it > 0 && !o->no_recopy) {  // restore the pre-state of W
            for (auto& rr : h->regions)
                for (size_t j = 0; j < rr.written.size(); ++j) {
                    const uint64_t k = rr.written[j];
                    const uint64_t len = std::min<uint64_t>(kChunk, rr.r.size - k * kChunk);
                    cudaMemcpyAsync((void*)(rr.r.base + k * kChunk), (uint8_t*)h->stash_pre + rr.stash_off[j], len,
                                    cudaMemcpyDeviceToDevice, s);
                }
            if (h->mode == KC_MODE_PRE_W) put_modvars(true);
        }
        cudaEventRecord(e0, s);
        CUresult r = launch_packed(f, grid, block, smem, (CUstream)s, h->kernarg.empty() ? nullptr : h->kernarg.data(),
                                   h->kernarg.size(), h->cluster, h->flags);
        cudaEventRecord(e1, s);
        if (r == CUDA_SUCCESS) r = KC_DRV(cuStreamSynchronize)((CUstream)s);
        if (r != CUDA_SUCCESS) {
            res = cu_err(ctx, r, "kc_replay: dispatch");
            break;
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        sum += ms;
        mn = std::min(mn, (double)ms);
        mx = std::max(mx, (double)ms);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    // F3 validation input: every restored variable against its captured post value
    h->modvar_checked = h->modvar_mismatch = 0;
    if (res == KC_OK)
        for (auto& pv : mv) {
            std::vector<uint8_t> now(pv.second->size);
            if (cudaMemcpy(now.data(), (const void*)pv.first, now.size(), cudaMemcpyDeviceToHost) != cudaSuccess) break;
            h->modvar_checked++;
            h->modvar_mismatch += now != pv.second->post;
        }
    if (own) KC_DRV(cuModuleUnload)(mod);
    if (res != KC_OK) return res;
    if (rep_out) {
        rep_out->module_vars_restored = mv_restored;
        rep_out->iterations = iters;
        rep_out->kernel_ms_mean = sum / iters;
        rep_out->kernel_ms_min = mn;
        rep_out->kernel_ms_max = mx;
    }
    if (o->dump_dir) {  // stage 6
        const std::string od = std::string(o->dump_dir) + "/output";
        if (!mkdir_p(od)) return set_err(ctx, KC_ERR_IO, "cannot create %s", od.c_str());
        kc_status st = ensure_pinned(ctx);
        if (st != KC_OK) return st;
        for (auto& rr : h->regions) {
            const std::string path = od + "/region_" + rr.hexbase + ".bin";
            FILE* fp = fopen(path.c_str(), "wb");
            std::string err;
            bool ok = fp && d2h_stream(ctx, rr.r.base, rr.r.size, fp, nullptr, err);
            if (fp) ok = (fclose(fp) == 0) && ok;
            if (!ok) return set_err(ctx, KC_ERR_IO, "dump %s: %s", path.c_str(), err.c_str());
        }
    }
    return KC_OK;
}

extern "C" kc_status kc_validate_module_vars(kc_ctx* ctx, const kc_restored* h, uint64_t* n_checked,
                                             uint64_t* n_mismatch) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    if (!ctx || !h) return KC_ERR_ARG;
    if (n_checked) *n_checked = h->modvar_checked;
    if (n_mismatch) *n_mismatch = h->modvar_mismatch;
    return KC_OK;
}

// ====================================================================== validate
// merge: (outs == NULL only) one report over the W chunks of every region, its
// bitmap indexed by global chunk (regions in order) -- the per-dispatch report
// of a sequence replay (kc_replay_seq)
kc_status kc::validate_impl(kc_ctx* ctx, kc_restored* h, const kc_buffer* outs, size_t n, const kc_tolerance* tol,
                            kc_diff_report* reps, size_t cap_reports, size_t* n_reports_out,
                            uint64_t* unexpected_chunks, bool merge) {
    if (!ctx || !h) return KC_ERR_ARG;
    if (ctx->poisoned) return KC_ERR_CUDA;
    if (!bind_device(ctx)) return set_err(ctx, KC_ERR_CUDA, "cannot bind device");
    cudaStream_t s = ctx->copy_stream;
    std::vector<kc_buffer> segs;
    std::vector<uint64_t> rep_nbytes, word0;
    uint64_t words = 0;
    void* typed_ref = nullptr;
    if (!outs) {
        // every region with written chunks, bytes, reference = captured post bytes of W
        uint64_t gchunk = 0;  // merge: global chunk index of the region's chunk 0
        if (merge) {
            uint64_t all = 0, tot = 0;
            for (auto& rr : h->regions) {
                all += rr.n_chunks;
                if (rr.ok && !rr.written.empty()) tot += rr.r.size;
            }
            rep_nbytes.push_back(tot);
            word0.push_back(0);
            words = (all + 63) / 64;
        }
        for (auto& rr : h->regions) {
            const uint64_t c0 = gchunk;
            gchunk += rr.n_chunks;
            if (!rr.ok || rr.written.empty()) continue;
            const int rid = merge ? 0 : (int)rep_nbytes.size();
            if (!merge) {
                rep_nbytes.push_back(rr.r.size);
                word0.push_back(words);
                words += (rr.n_chunks + 63) / 64;
            }
            for (size_t j = 0; j < rr.written.size(); ++j) {
                const uint64_t k = rr.written[j];
                kc_buffer b;
                b.ref = (uint64_t)h->stash_ref + rr.stash_off[j];
                b.act = rr.r.base + k * kChunk;
                b.nbytes = std::min<uint64_t>(kChunk, rr.r.size - k * kChunk);
                b.dtype = KC_DT_BYTES;
                b.report = rid;
                b.bitmap_chunk0 = merge ? c0 + k : k;
                segs.push_back(b);
            }
        }
        if (merge && segs.empty()) rep_nbytes.clear();  // nothing written: no report
    } else {
        // typed sub-ranges: rebuild the captured post-dispatch bytes of each range
        uint64_t total = 0;
        for (size_t i = 0; i < n; ++i) total += (outs[i].nbytes + 255) / 256 * 256;
        if (total && cudaMalloc(&typed_ref, total) != cudaSuccess)
            return set_err(ctx, KC_ERR_NOMEM, "kc_validate: reference buffer");
        uint64_t off = 0;
        for (size_t i = 0; i < n; ++i) {
            const kc_buffer& o = outs[i];
            const kc_restored_region* owner = nullptr;
            for (auto& rr : h->regions)
                if (rr.r.base <= o.act && o.act + o.nbytes <= rr.r.base + rr.r.size) owner = &rr;
            if (!owner || !owner->ok) {
                if (typed_ref) cudaFree(typed_ref);
                return set_err(ctx, KC_ERR_OUT_OF_BOUNDS, "kc_validate: output %zu is not inside a restored region", i);
            }
            const uint64_t roff = o.act - owner->r.base;
            if (h->ipc_arena) {  // published snapshot: stored bytes from the mapped arena, W's post bytes from the stash
                auto it = h->ipc_off.find(owner->r.base);
                if (it == h->ipc_off.end()) {
                    if (typed_ref) cudaFree(typed_ref);
                    return set_err(ctx, KC_ERR_FORMAT, "kc_validate: region not in the published arena");
                }
                cudaMemcpyAsync((uint8_t*)typed_ref + off, (const uint8_t*)h->ipc_arena + it->second + roff, o.nbytes,
                                cudaMemcpyDeviceToDevice, s);
                if (h->mode == KC_MODE_PRE_W)
                    for (size_t j = 0; j < owner->written.size(); ++j) {
                        const uint64_t c0 = owner->written[j] * kChunk;
                        const uint64_t len = std::min<uint64_t>(kChunk, owner->r.size - c0);
                        const uint64_t lo = std::max(c0, roff), hi = std::min(c0 + len, roff + o.nbytes);
                        if (lo < hi)
                            cudaMemcpyAsync((uint8_t*)typed_ref + off + (lo - roff),
                                            (const uint8_t*)h->stash_ref + owner->stash_off[j] + (lo - c0), hi - lo,
                                            cudaMemcpyDeviceToDevice, s);
                    }
            } else if (h->dev_snap) {  // device snapshot: stored bytes from the arena, W's post bytes from the W arena
                const kc_snapshot* sn = h->dev_snap;
                const size_t ri = (size_t)(owner - h->regions.data());
                for (const auto& ru : sn->runs[ri]) {  // stored bytes of [roff, roff + nbytes)
                    const uint64_t lo = std::max(ru.roff, roff), hi = std::min(ru.roff + ru.len, roff + o.nbytes);
                    if (lo < hi)
                        cudaMemcpyAsync((uint8_t*)typed_ref + off + (lo - roff),
                                        (const uint8_t*)(ru.src + (lo - ru.roff)), hi - lo, cudaMemcpyDefault, s);
                }
                if (h->mode == KC_MODE_PRE_W) {
                    uint64_t woff = sn->w_off[ri];
                    for (uint64_t k : owner->written) {
                        const uint64_t c0 = k * kChunk, len = std::min<uint64_t>(kChunk, owner->r.size - c0);
                        const uint64_t lo = std::max(c0, roff), hi = std::min(c0 + len, roff + o.nbytes);
                        if (lo < hi)
                            cudaMemcpyAsync((uint8_t*)typed_ref + off + (lo - roff),
                                            (const uint8_t*)sn->warena + woff + (lo - c0), hi - lo, cudaMemcpyDefault,
                                            s);
                        woff += len;
                    }
                }
            } else {
                std::vector<uint8_t> host(o.nbytes);
                FILE* fp = fopen((h->dir + "/memory/region_" + owner->hexbase + ".bin").c_str(), "rb");
                bool okr = fp && fseek(fp, (long)roff, SEEK_SET) == 0 && fread(host.data(), 1, o.nbytes, fp) == o.nbytes;
                if (fp) fclose(fp);
                if (!okr) {
                    if (typed_ref) cudaFree(typed_ref);
                    return set_err(ctx, KC_ERR_FORMAT, "kc_validate: cannot read reference bytes");
                }
                if (h->mode == KC_MODE_PRE_W && !owner->written.empty()) {  // overlay W's post bytes
                    std::vector<uint8_t> wb;
                    read_bin(h->dir + "/written/region_" + owner->hexbase + ".bin", wb);
                    uint64_t woff = 0;
                    for (uint64_t k : owner->written) {
                        const uint64_t c0 = k * kChunk, len = std::min<uint64_t>(kChunk, owner->r.size - c0);
                        const uint64_t lo = std::max(c0, roff), hi = std::min(c0 + len, roff + o.nbytes);
                        if (lo < hi && woff + len <= wb.size()) memcpy(host.data() + (lo - roff), wb.data() + woff + (lo - c0), hi - lo);
                        woff += len;
                    }
                }
                cudaMemcpyAsync((uint8_t*)typed_ref + off, host.data(), o.nbytes, cudaMemcpyHostToDevice, s);
                cudaStreamSynchronize(s);  // host goes out of scope
            }
            kc_buffer b = o;
            b.ref = (uint64_t)typed_ref + off;
            b.report = (int32_t)i;
            b.bitmap_chunk0 = 0;
            segs.push_back(b);
            rep_nbytes.push_back(o.nbytes);
            word0.push_back(words);
            words += ((o.nbytes + kChunk - 1) / kChunk + 63) / 64;
            off += (o.nbytes + 255) / 256 * 256;
        }
    }
    const size_t nrep = rep_nbytes.size();
    if (n_reports_out) *n_reports_out = nrep;
    kc_status st = KC_OK;
    if (nrep) {
        KC_CHECK_CUDA(ctx, ensure(ctx->reps, nrep * sizeof(kc_diff_report)), "cudaMalloc(reports)");
        KC_CHECK_CUDA(ctx, ensure(ctx->bitmaps, std::max<uint64_t>(1, words) * 8), "cudaMalloc(bitmaps)");
        st = kc_diff_async(ctx, segs.data(), segs.size(), nrep, rep_nbytes.data(), word0.data(), tol,
                           (kc_diff_report*)ctx->reps.p, (uint64_t*)ctx->bitmaps.p, s);
        if (st == KC_OK && reps) {
            std::vector<kc_diff_report> tmp(nrep);
            cudaMemcpyAsync(tmp.data(), ctx->reps.p, nrep * sizeof(kc_diff_report), cudaMemcpyDeviceToHost, s);
            cudaError_t e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) st = cuda_err(ctx, e, "kc_validate: reports");
            for (size_t j = 0; j < nrep && j < cap_reports; ++j) reps[j] = tmp[j];
        }
    }
    if (typed_ref) {
        cudaStreamSynchronize(s);
        cudaFree(typed_ref);
    }
    if (st != KC_OK) return st;
    if (unexpected_chunks) {  // re-hash every restored region vs the captured post manifest
        std::vector<kc_region> okregs;
        for (auto& rr : h->regions)
            if (rr.ok) okregs.push_back(rr.r);
        std::vector<uint64_t> got;
        st = hash_regions_sync(ctx, okregs, got, nullptr, nullptr, nullptr, s);
        if (st != KC_OK) return st;
        uint64_t c = 0, bad = 0;
        for (auto& rr : h->regions) {
            if (!rr.ok) continue;
            for (uint64_t k = 0; k < rr.n_chunks; ++k)
                bad += (rr.post_manifest.size() != rr.n_chunks) || rr.post_manifest[k] != got[c + k];
            c += rr.n_chunks;
        }
        *unexpected_chunks = bad;
    }
    return KC_OK;
}

extern "C" kc_status kc_validate(kc_ctx* ctx, kc_restored* h, const kc_buffer* outs, size_t n,
                                 const kc_tolerance* tol, kc_diff_report* reps, size_t cap_reports,
                                 size_t* n_reports_out, uint64_t* unexpected_chunks) {
    ::kc::Internal _kc_internal_guard(__func__);  // the CUPTI hook ignores our own driver calls
    return validate_impl(ctx, h, outs, n, tol, reps, cap_reports, n_reports_out, unexpected_chunks, false);
}

// F4 sequences: point a restored handle at the next dispatch of a sequence
// whose state the live memory already holds (the replay of the previous
// dispatches); nothing is remapped or copied in
kc_status kc::restored_rebind(kc_ctx* ctx, kc_restored* h, const kc_snapshot* sn) {
    if (!ctx || !h || !sn) return KC_ERR_ARG;
    const SnapDesc& d = sn->desc;
    if (d.regions.size() != h->regions.size())
        return set_err(ctx, KC_ERR_ARG, "rebind: the snapshot has %zu regions, the restored state %zu",
                       d.regions.size(), h->regions.size());
    for (size_t i = 0; i < d.regions.size(); ++i)
        if (d.regions[i].r.base != h->regions[i].r.base || d.regions[i].r.size != h->regions[i].r.size ||
            d.regions[i].ok != h->regions[i].ok)
            return set_err(ctx, KC_ERR_ARG, "rebind: region %zu differs from the restored state", i);
    if (!bind_device(ctx)) return set_err(ctx, KC_ERR_CUDA, "cannot bind device");
    cudaDeviceSynchronize();
    if (h->module) KC_DRV(cuModuleUnload)(h->module);
    h->module = nullptr;
    if (h->stash_pre) cudaFree(h->stash_pre);  // stash_ref lives in the same allocation
    h->stash_pre = h->stash_ref = nullptr;
    h->stash_bytes = 0;
    bind_dispatch_fields(h, d);
    for (size_t i = 0; i < d.regions.size(); ++i) {
        h->regions[i].written = d.regions[i].written;
        h->regions[i].post_manifest = d.regions[i].post_manifest;
    }
    h->dev_snap = sn;
    h->modvar_checked = h->modvar_mismatch = 0;
    kc_status st = ensure_stream(ctx);
    if (st != KC_OK) return st;
    DevSource src(sn);
    return build_stash(ctx, h, d, src);
}

// interposed mode (kc_interpose.cu): the in-memory capture with the dispatch
// forwarded by the application itself
kc_status kc::capture_interposed(kc_ctx* ctx, const kc_dispatch* d, kc_capture_mode mode, bool host,
                                 const std::function<CUresult()>& forward, kc_snapshot** out, kc_capture_report* rep,
                                 const kc_snapshot* base) {
    return capture_mem(ctx, d, nullptr, 0, mode, out, rep, host, base, &forward);
}
