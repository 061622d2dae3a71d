// kc_internal.h -- host-side internals of libkc.so (not part of the ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no-ops unless a tool (nsys/ncu) injects

#include <cstdarg>
#include <cstdint>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "kc_kernels.cuh"

// Driver-API entry points resolved through cudart (cudaGetDriverEntryPoint),
// so libkc.so has no link-time dependency on libcuda and loads on hosts
// without a GPU driver (calls then fail with KC_ERR_CUDA).
#define KC_DRV_FUNCS(X) X(cuCtxGetDevice) X(cuFuncGetModule) X(cuFuncGetName) X(cuFuncGetParamInfo) X(cuFuncSetAttribute) X(cuGetErrorName) X(cuGetErrorString) X(cuLaunchKernel) X(cuLaunchKernelEx) X(cuMemAddressFree) X(cuMemAddressReserve) X(cuMemAlloc) X(cuMemCreate) X(cuMemExportToShareableHandle) X(cuMemFree) X(cuMemImportFromShareableHandle) X(cuMemGetAllocationGranularity) X(cuMemMap) X(cuMemRelease) X(cuMemSetAccess) X(cuMemUnmap) X(cuModuleGetFunction) X(cuModuleGetGlobal) X(cuModuleLoadData) X(cuModuleUnload) X(cuPointerGetAttribute) X(cuStreamIsCapturing) X(cuStreamSynchronize)
namespace kc {
struct Drv {
#define KC_DRV_DECL(f) decltype(&::f) f = nullptr;
    KC_DRV_FUNCS(KC_DRV_DECL)
#undef KC_DRV_DECL
    bool ok = false;
};
const Drv& drv();
}  // namespace kc
#define KC_DRV(f) (::kc::drv().f)

// F3 module variables (kc_module.cu): declared in the code object, valued per capture
namespace kc {
struct ModVarDecl {
    std::string name, section;
    uint64_t size;
};
size_t image_size(const void* img, size_t hint);  // ELF64 / fatbin extent (hint wins when nonzero)
std::string sha256_hex(const uint8_t* data, size_t n);  // code-object identity (dispatch.json)
std::vector<ModVarDecl> image_module_vars(const uint8_t* img, size_t n);
}  // namespace kc
struct ModVarState {
    std::string name, section;
    uint64_t size = 0;
    std::vector<uint8_t> pre, post;  // bytes before / after the captured dispatch
};

struct kc_interpose;  // A3 interposed-mode state (kc_interpose.cu)

struct kc_ctx_dev_buf {
    void* p = nullptr;
    size_t cap = 0;
};

struct kc_ctx {
    int device = 0;
    int num_sms = 148;
    bool inited = true;  // false: injected ctx, device and kernels set up at first use (bind_device)
    std::string err;
    bool poisoned = false;

    // A1 tracker (internally synchronized)
    std::mutex mu;
    std::map<uint64_t, kc_region> live;
    uint64_t seq = 0;
    uint64_t unknown_frees = 0;

    // cached device tables / scratch (stream-ordered; one stream at a time per ctx)
    kc_ctx_dev_buf regs, segs, meta, reps, bitmaps, digest_scratch, tmp_hash, tmp_count, chunk_map, dst_tab, gather_tab, chunk_order, ref_man, ref_stage;
    std::vector<kc::RegionDev> regs_cached;
    std::vector<kc_region> regs_input;  // the kc_region list behind regs_cached (fast same-input check)
    bool regs_input_sorted = false;
    uint64_t regs_input_chunks = 0;
    kc_ctx_dev_buf pairs, pair_map, dirty;  // F2 (K5) pair table, chunk -> pair map, dirty bitmap
    std::vector<kc::PairDev> pairs_cached;
    std::vector<uint8_t> diff_key;  // K2 plan cache (raw inputs of the last kc_diff_async)
    std::vector<kc::DiffGroup> diff_groups;
    uint64_t diff_bitmap_words = 0;
    bool regs_aligned = true;
    bool has_order = false;  // chunk_order holds a length-sorted chunk order for K1/K6

    // pinned staging ring for D2H/H2D (lazily allocated)
    uint64_t io_chunk = 64ull << 20;
    uint32_t depth = 2;
    std::vector<void*> pinned;
    std::vector<cudaEvent_t> pin_ev;
    cudaStream_t copy_stream = nullptr;
    std::vector<cudaEvent_t> full_ev;  // byte-exact host-reference validation: per staging slot copied / freed
    // parallel snapshot file I/O workers (stream + `depth` pinned buffers each)
    struct IoWorker {
        cudaStream_t stream = nullptr;
        std::vector<void*> pinned;
        std::vector<cudaEvent_t> ev;
    };
    std::vector<IoWorker> io;

    // CUPTI interposition
    void* cupti_subscriber = nullptr;
    bool cupti_installed = false;

    // kc_alloc backing
    int alloc_mode = KC_ALLOC_VMM;
    size_t granularity = 0;
    struct VmmAlloc {
        uint64_t reserved;
        CUmemGenericAllocationHandle h;
        int export_fd = -1;  // E2: POSIX fd of the physical allocation once exported (closed on free)
    };
    std::map<uint64_t, VmmAlloc> vmm;  // base -> reservation (guarded by mu)
    // ctx-owned VA heap for KC_ALLOC_VMM (reserved once, never returned to the
    // driver): freed ranges stay ours, so a same-process restore maps back at
    // the exact VAs (R28d).  heap_free: base -> size of free ranges (mu).
    uint64_t heap_base = 0, heap_size = 0;
    // F3 code objects seen by the CUPTI hook (cuModuleLoadData*): module -> image bytes (mu)
    std::map<CUmodule, std::vector<uint8_t>> code_objects;
    // parked device arena (a VMM mapping) for kc_capture_dev (kc_dev_arena_reserve)
    struct ParkedVmm {
        uint64_t va = 0, size = 0;
        CUmemGenericAllocationHandle h = 0;
        void release() {
            if (!va) return;
            KC_DRV(cuMemUnmap)((CUdeviceptr)va, size);
            KC_DRV(cuMemRelease)(h);
            KC_DRV(cuMemAddressFree)((CUdeviceptr)va, size);
            va = size = 0;
            h = 0;
        }
    } dev_arena;
    // physical VMM allocations of released restores, parked by size and reused by the next
    // restore of the same span sizes (no cuMemCreate / scrub of freshly released memory on a
    // resident tool's repeated capture -> restore cycles); KC_PHYS_PARK=0 disables, and
    // kc_dev_arena_reserve(ctx, 0) or kc_destroy releases them
    std::multimap<uint64_t, CUmemGenericAllocationHandle> phys_park;
    uint64_t phys_park_bytes = 0;
    // parked pinned host arena for kc_capture_host (kc_host_arena_reserve)
    void* host_arena = nullptr;
    uint64_t host_arena_bytes = 0;
    std::map<uint64_t, uint64_t> heap_free;
    uint64_t launches = 0;
    kc_interpose* interpose = nullptr;  // armed / in-flight interposed capture
    // E2: peer allocations imported from other processes (kc_peer_import): va -> mapping (mu)
    struct PeerMap {
        uint64_t size;
        CUmemGenericAllocationHandle h;
        bool own_va;  // the VA range was reserved by the import (else: inside the ctx heap)
    };
    std::map<uint64_t, PeerMap> peers;
};

struct kc_restored_region {
    kc_region r;
    std::string hexbase;
    bool ok = true;
    uint64_t n_chunks = 0;
    std::vector<uint64_t> written;          // chunk indices of W (sorted)
    std::vector<uint64_t> stash_off;        // per written chunk: offset in the stashes
    std::vector<uint64_t> post_manifest;    // captured post-dispatch chunk hashes (may be empty)
};

struct kc_restored {
    kc_ctx* ctx = nullptr;
    std::string dir;
    int mode = KC_MODE_PRE_W;
    std::string mangled;
    uint32_t grid[3] = {1, 1, 1}, block[3] = {1, 1, 1}, smem = 0;
    uint32_t cluster[3] = {1, 1, 1};
    uint32_t flags = 0;  // KC_LAUNCH_COOPERATIVE
    std::vector<uint8_t> kernarg;
    std::vector<kc_restored_region> regions;  // sorted by base
    // VMM spans
    struct Span {
        uint64_t base, size;
        CUmemGenericAllocationHandle h;
        bool reserved, mapped, created;
        bool heap;                       // claimed from the ctx VA heap (not a driver reservation)
        bool fallback;                   // restored by replaying cuMemAlloc (driver-pooled VA)
        std::vector<uint64_t> memalloc;  // cuMemAlloc'd region bases inside this span
        uint64_t reserve_got;            // diagnostics of a refused reservation
        int reserve_cr;
    };
    std::vector<Span> spans;
    std::vector<std::pair<uint64_t, uint64_t>> windows;  // reserved VA windows (base, size), ascending
    // device stashes for W chunks: pre-state (recopy) and reference post bytes (validate)
    void* stash_pre = nullptr;
    void* stash_ref = nullptr;
    uint64_t stash_bytes = 0;
    CUmodule module = nullptr;
    std::vector<uint8_t> image;  // code object (kernel.cubin or the device snapshot's copy)
    const kc_snapshot* dev_snap = nullptr;  // restored from a device snapshot (kc_restore_dev)
    void* ipc_arena = nullptr;              // restored from a published snapshot: its mapped arena
    uint64_t ipc_vmm_size = 0;              //   imported VMM mapping (0: a legacy CUDA IPC mapping)
    CUmemGenericAllocationHandle ipc_vmm_h = 0;
    std::map<uint64_t, uint64_t> ipc_off;   //   region base -> offset in that arena
    std::vector<ModVarState> modvars;       // F3: written into the replay module before each launch
    uint64_t modvar_checked = 0, modvar_mismatch = 0;  // last replay vs the captured post values
};

namespace kc {

// Set on a thread while it runs inside the library: the CUPTI hook ignores the
// driver calls made then (the library's own scratch, arenas and kernel launches
// are not application state).  KC_ENTER and the capture/restore entry points hold one.
extern thread_local int t_internal;
// With a name (every C-ABI entry point passes __func__) it also spans the call
// with an NVTX range, so a timeline tool shows each kc_* call; the stages
// inside capture/restore are NVTX marks (trace() in kc_snapshot.cu).
struct Internal {
    Internal() : named(false) { ++t_internal; }
    explicit Internal(const char* name) : named(true) {
        ++t_internal;
        nvtxRangePushA(name);
    }
    ~Internal() {
        if (named) nvtxRangePop();
        --t_internal;
    }
    const bool named;
    Internal(const Internal&) = delete;
    Internal& operator=(const Internal&) = delete;
};

// error helpers
kc_status set_err(kc_ctx* ctx, kc_status st, const char* fmt, ...);
kc_status cuda_err(kc_ctx* ctx, cudaError_t e, const char* what);
kc_status cu_err(kc_ctx* ctx, CUresult r, const char* what);
cudaError_t ensure(kc_ctx_dev_buf& b, size_t bytes);
kc_status ensure_stream(kc_ctx* ctx);  // the ctx's non-blocking copy stream
kc_status ensure_pinned(kc_ctx* ctx);  // + the pinned staging ring (file / PCIe paths only)
bool bind_device(kc_ctx* ctx);

std::string hex_base(uint64_t base);  // lowercase hex, no 0x
bool region_live(kc_ctx* ctx, uint64_t base, uint64_t size);
kc_status free_alloc(kc_ctx* ctx, uint64_t dptr, bool track);
size_t granularity(kc_ctx* ctx);
// ctx VA heap: claim an exact free range / allocate / give back (coalescing)
bool heap_take(kc_ctx* ctx, uint64_t base, uint64_t size);
uint64_t heap_alloc(kc_ctx* ctx, uint64_t size);
void heap_put(kc_ctx* ctx, uint64_t base, uint64_t size);

// snapshot format helpers (kc_snapshot.cu)
// h_dst (one arena address per region): the fused K6 pass, which also copies the bytes there
kc_status hash_regions_sync(kc_ctx* ctx, const std::vector<kc_region>& regs, std::vector<uint64_t>& out_hashes,
                            std::vector<uint64_t>* out_digests, uint64_t* out_snapshot, uint64_t* d_hash_out,
                            cudaStream_t s, const uint64_t* h_dst = nullptr);
kc_status hash_impl(kc_ctx* ctx, const kc_region* regions, size_t n, uint64_t* d_chunk_hash, uint64_t* d_region_digest,
                    uint64_t* d_snapshot_digest, void* stream, const uint64_t* h_dst);

// one launch of a captured dispatch: the packed kernarg buffer, and a cluster
// launch (cuLaunchKernelEx + CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION) when any
// cluster dim exceeds 1
CUresult launch_packed(CUfunction f, const uint32_t grid[3], const uint32_t block[3], uint32_t smem, CUstream s,
                       const void* kernarg, size_t kernarg_size, const uint32_t cluster[3], uint32_t flags = 0);
// normalised cluster dims of a kc_dispatch (0 -> 1)
void dispatch_cluster(const kc_dispatch* d, uint32_t out[3]);
// kc_validate with an option to merge every region's W into one report (F4 sequences)
kc_status validate_impl(kc_ctx* ctx, kc_restored* h, const kc_buffer* outs, size_t n, const kc_tolerance* tol,
                        kc_diff_report* reps, size_t cap_reports, size_t* n_reports_out, uint64_t* unexpected_chunks,
                        bool merge);
// A3 interposed mode: the in-memory capture of every tracked region around a
// dispatch the application launches itself (`forward` returns once it has run)
kc_status capture_interposed(kc_ctx* ctx, const kc_dispatch* d, kc_capture_mode mode, bool host,
                             const std::function<CUresult()>& forward, kc_snapshot** out, kc_capture_report* rep,
                             const kc_snapshot* base = nullptr);
// F4: a kc_sequence from step snapshots (ownership moves in; deps computed)
kc_status make_sequence(kc_ctx* ctx, std::vector<kc_snapshot*>& steps, kc_sequence** out);
// CUPTI launch callbacks (kc_interpose.cu)
void interpose_launch(kc_ctx* ctx, uint32_t cbid, const void* cbdata);
void interpose_destroy(kc_ctx* ctx);
void interpose_arm_from_env(kc_ctx* ctx);
// re-point a restored handle at another snapshot of the same regions (dispatch,
// W, post manifest, stashes) without touching the mapped memory (F4 sequences)
kc_status restored_rebind(kc_ctx* ctx, kc_restored* h, const kc_snapshot* sn);

}  // namespace kc

#define KC_CHECK_CUDA(ctx, expr, what)                                  \
    do {                                                                \
        cudaError_t _e = (expr);                                        \
        if (_e != cudaSuccess) return ::kc::cuda_err((ctx), _e, (what)); \
    } while (0)
#define KC_CHECK_CU(ctx, expr, what)                                  \
    do {                                                              \
        CUresult _r = (expr);                                         \
        if (_r != CUDA_SUCCESS) return ::kc::cu_err((ctx), _r, (what)); \
    } while (0)
