// kc_snapshot_types.h -- in-memory snapshot structures shared by
// kc_snapshot.cu (capture/restore/replay/validate) and kc_sequence.cu (F4
// multi-kernel capture).  Not part of the ABI.
#pragma once
#include <unistd.h>

#include <memory>
#include <string>
#include <vector>

#include "kc_internal.h"

// A snapshot's contents independent of where the bytes live (files or a
// device arena); restore_core maps the captured VAs and pulls the bytes
// through a RestoreSource.
struct SnapRegion {
    kc_region r;
    std::string hx;
    bool ok = true;
    uint64_t n_chunks = 0;
    uint64_t digest = 0, post_digest = 0;
    std::vector<uint64_t> manifest;       // manifest of the stored bytes
    std::vector<uint64_t> post_manifest;  // post-dispatch manifest
    std::vector<uint64_t> written;        // W chunk indices
};

struct SnapDesc {
    int mode = KC_MODE_PRE_W;
    std::string mangled;
    uint32_t grid[3] = {1, 1, 1}, block[3] = {1, 1, 1}, smem = 0;
    uint32_t cluster[3] = {1, 1, 1};                 // thread-block cluster dims (1,1,1 = no cluster launch)
    uint32_t flags = 0;                              // KC_LAUNCH_COOPERATIVE
    std::vector<uint8_t> kernarg, image;
    std::vector<std::pair<size_t, size_t>> layout;  // kernarg (offset, size)
    std::vector<SnapRegion> regions;                 // ascending base
    uint64_t snapshot_digest = 0;
    std::vector<ModVarState> modvars;                // F3
};

// an in-memory arena (device or pinned host), shared by refcount between a
// snapshot and the incremental snapshots that reference its bytes
struct ArenaBuf {
    kc_ctx* ctx = nullptr;
    void* p = nullptr;
    uint64_t cap = 0;
    bool host = false;
    // device arenas are VMM allocations exportable as a POSIX fd (F1 across
    // processes); vmm_h/vmm_size describe the mapping at p, export_fd the fd
    // handed out by kc_snapshot_publish (closed with the arena)
    bool vmm = false;
    CUmemGenericAllocationHandle vmm_h = 0;
    uint64_t vmm_size = 0;
    int export_fd = -1;
    ~ArenaBuf() {
        const bool exported = export_fd >= 0;
        if (exported) close(export_fd);
        if (!p) return;
        if (ctx) kc::bind_device(ctx);
        if (vmm) {
            cudaDeviceSynchronize();
            // park the larger never-exported arena in the ctx for the next capture
            // (freshly freed device memory is slow to reallocate: measured up to
            // 40 ms per 30 GB); an exported one may still be mapped elsewhere
            if (ctx && !exported && vmm_size > ctx->dev_arena.size) {
                ctx->dev_arena.release();
                ctx->dev_arena = {(uint64_t)p, vmm_size, vmm_h};
                return;
            }
            KC_DRV(cuMemUnmap)((CUdeviceptr)p, vmm_size);
            KC_DRV(cuMemRelease)(vmm_h);
            KC_DRV(cuMemAddressFree)((CUdeviceptr)p, vmm_size);
        } else if (!host) {
            cudaFree(p);
        } else if (ctx && cap >= ctx->host_arena_bytes) {  // park the larger arena
            if (ctx->host_arena) cudaFreeHost(ctx->host_arena);
            ctx->host_arena = p;
            ctx->host_arena_bytes = cap;
        } else {
            cudaFreeHost(p);
        }
    }
};

struct kc_snapshot {
    kc_ctx* ctx = nullptr;
    bool host = false;  // arenas in pinned host memory (kc_capture_host)
    SnapDesc desc;
    std::shared_ptr<ArenaBuf> arena;                // this snapshot's own stored bytes
    uint64_t arena_bytes = 0;                       // bytes used in it
    std::vector<std::shared_ptr<ArenaBuf>> deps;    // base arenas referenced by runs
    struct Run {
        uint64_t roff, len;  // region byte range (chunk aligned)
        uint64_t src;        // where its stored bytes are (own arena or a base's)
    };
    std::vector<std::vector<Run>> runs;  // per region, ascending roff, covering ok regions
    uint64_t shared_bytes = 0;           // stored bytes referenced from base snapshots
    mutable std::vector<std::string> published;  // kc_snapshot_publish directories, revoked on free
    void* warena = nullptr;              // PRE_W: post bytes of W, region i at w_off[i]
    uint64_t w_bytes = 0;
    std::vector<uint64_t> w_off;
    kc_capture_report rep;
};

