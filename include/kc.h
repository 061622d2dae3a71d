/*
 * kc.h -- C ABI of libkc.so, the B200-native (sm_100a) hot path of Kerncap's
 * capture-and-validate loop: the address-space closure (arXiv 2605.03208).
 *
 * The paper's statement of the problem: a kernel reproducer needs the
 * definition, the runtime state ("the contents of every device-memory region
 * the kernel reads -- including buffers reached indirectly through pointer
 * arguments") and an environment that "faithfully replays the original
 * execution with bit-identical semantics" (fig:three-problems).
 * The closure: "capturing every tracked allocation at its original virtual
 * address captures the graph for free" (sec. 4.2.1).
 *
 * Conventions:
 *  - Every call returns kc_status: 0 = OK, >0 = completed with tolerated
 *    failures (KC_PARTIAL), <0 = error.  kc_last_error(ctx) holds a message.
 *  - Every pointer argument is BORROWED for the duration of the call.  Outputs
 *    go to caller-provided memory.  "device" pointers are CUDA device virtual
 *    addresses (CUdeviceptr values) of the context's device; "host" pointers are
 *    ordinary process memory.  Streams are CUstream handles passed as void*
 *    (NULL = the legacy default stream).
 *  - kc_ctx owns the tracker, pinned staging, device scratch and cached tables.
 *    kc_restored owns VA reservations, physical handles, the loaded module and
 *    the device stash; release it with kc_release() BEFORE kc_destroy().
 *  - Threading: kc_track/kc_regions are internally synchronized (driver
 *    callbacks arrive from any host thread).  Every other call:
 *    one host thread per ctx at a time.
 *  - Sticky CUDA errors poison the ctx: every later call returns KC_ERR_CUDA.
 *
 * Hash chunk: 65,536 bytes (reading R1).  XXH64, seed 0 (R2), last chunk short
 * and unpadded (R3), little-endian (R5).  Region digest D_r = XXH64 of the
 * region's chunk hashes as LE u64s; snapshot digest S = XXH64 of
 * (LE64 base, LE64 size, LE64 D_r) over regions in ascending base order (R4).
 */
#ifndef KC_H_
#define KC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KC_ABI_VERSION 1
#define KC_CHUNK_BYTES 65536u

typedef enum {
    KC_OK = 0,
    KC_PARTIAL = 1,                 /* completed; per-region failures recorded */
    KC_ERR_ARG = -1,
    KC_ERR_STATE = -2,              /* wrong call order, double install, ... */
    KC_ERR_CUDA = -3,               /* a CUDA driver/runtime error; CUresult in kc_last_error */
    KC_ERR_IO = -4,
    KC_ERR_FORMAT = -5,             /* snapshot directory does not parse */
    KC_ERR_VA_UNAVAILABLE = -6,     /* restore could not reserve the captured VA */
    KC_ERR_NOT_TRACKED = -7,
    KC_ERR_OUT_OF_BOUNDS = -8,
    KC_ERR_NOMEM = -9,
    KC_ERR_MANIFEST_MISMATCH = -10, /* restored bytes do not hash to the captured manifest */
    KC_ERR_UNSUPPORTED = -11
} kc_status;

typedef enum { KC_EV_ALLOC = 0, KC_EV_FREE = 1, KC_EV_MAP = 2, KC_EV_UNMAP = 3 } kc_event;
typedef enum { KC_KIND_MEMALLOC = 0, KC_KIND_VMM = 1, KC_KIND_POOL = 2 } kc_alloc_kind;

/* Element types of a validated buffer (O4).  KC_DT_BYTES compares raw bytes. */
typedef enum {
    KC_DT_BYTES = 0, KC_DT_U8, KC_DT_I8, KC_DT_U16, KC_DT_I16, KC_DT_U32, KC_DT_I32,
    KC_DT_U64, KC_DT_I64, KC_DT_F16, KC_DT_BF16, KC_DT_F32, KC_DT_F64, KC_DT__COUNT
} kc_dtype;

/* Capture timing (reading R7).  PRE_W (default): the snapshot holds the
 * pre-dispatch state plus the post-dispatch bytes of the written chunks W
 * (chunks whose hash changed), so replay starts from the true inputs.  POST:
 * the paper's post-execution snapshot. */
typedef enum { KC_MODE_PRE_W = 0, KC_MODE_POST = 1 } kc_capture_mode;

/* One tracked allocation (A1; reading R6). */
typedef struct {
    uint64_t base;      /* device VA */
    uint64_t size;      /* bytes */
    int32_t device;     /* CUDA device ordinal */
    int32_t kind;       /* kc_alloc_kind */
    uint64_t seq;       /* tracker sequence number of the ALLOC/MAP event */
} kc_region;

/* One validated buffer pair (A8): reference and actual device VAs, nbytes each.
 * bitmap_chunk0 = chunk index of ref/act[0] inside the report's bitmap (0 for a
 * whole buffer; kc_validate uses it for W-chunk segments of a region). */
typedef struct {
    uint64_t ref;
    uint64_t act;
    uint64_t nbytes;    /* must be a multiple of the element size (else KC_ERR_ARG) */
    int32_t dtype;      /* kc_dtype */
    int32_t report;     /* index of the kc_diff_report this segment accumulates into */
    uint64_t bitmap_chunk0;
} kc_buffer;

/* numpy.allclose tolerances; defaults 1e-8 / 1e-5 / 0 (R14, R15). */
typedef struct {
    double atol;
    double rtol;
    int32_t equal_nan;
    int32_t _pad;
} kc_tolerance;

/* Diff report per output buffer (O4; R8-R18).
 * Layout is part of the ABI (identical on host and device). */
typedef struct {
    uint64_t nbytes, n_elems, n_chunks;
    uint64_t differing_bytes;       /* #{j : R[j] != A[j]}                          */
    uint64_t differing_elems;       /* #{i : bits(R_i) != bits(A_i)}                */
    uint64_t max_ulp;               /* floats: ordered-int distance; ints: |A-R|    */
    double max_abs;                 /* max |f64(A)-f64(R)| over differing non-NaN   */
    double max_rel;                 /* max d/|R| (R=+-inf -> +inf; R=0 -> undefined)*/
    double percent_bytes;           /* 100*differing_bytes/nbytes                   */
    uint64_t nan_ref, nan_act, nan_pos_mismatch, rel_undefined, allclose_fail;
    int32_t pass;                   /* floats: allclose_fail==0; ints: differing_elems==0; bytes: differing_bytes==0 */
    int32_t _pad;
} kc_diff_report;

/* Explicit dispatch description (A3; D4 of SURVEY.md 2.2).  Either func (a
 * CUfunction cast to void*) or (image, mangled) must be given.  kernarg is the
 * packed parameter buffer (Q22: CUDA params live outside tracked memory). */
typedef struct {
    void* func;
    const void* image;          /* cubin/fatbin bytes, may be NULL if func given */
    size_t image_size;
    const char* mangled;        /* kernel symbol name */
    uint32_t grid[3], block[3];
    uint32_t smem_bytes;
    uint32_t kernarg_size;
    const void* kernarg;
    void* stream;
    uint32_t cluster[3];        /* thread-block cluster dims of a cluster launch (cuLaunchKernelEx
                                   CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION); 0,0,0 or 1,1,1 = none.
                                   Recorded in dispatch.json and reapplied by kc_replay */
    uint32_t flags;             /* KC_LAUNCH_COOPERATIVE: a cooperative launch (grid-wide sync) */
} kc_dispatch;
enum { KC_LAUNCH_COOPERATIVE = 1 };

/* kc_alloc backing (reading R6/R20): VMM allocations live in free VA space and
 * can be re-reserved at the same VA by a fresh process; plain cuMemAlloc
 * regions below the driver's pooling threshold share driver-reserved VA and
 * are restored by replaying cuMemAlloc in capture order (abort on mismatch). */
typedef enum { KC_ALLOC_VMM = 0, KC_ALLOC_MEMALLOC = 1 } kc_alloc_mode;

typedef struct {
    uint64_t io_chunk_bytes;    /* KERNCAP_SNAPSHOT_CHUNK_BYTES; 0 = env or 64 MiB */
    uint32_t pinned_depth;      /* staging buffers in flight (R26); 0 = 2 */
    int32_t device;             /* CUDA device ordinal; -1 = current */
    int32_t alloc_mode;         /* kc_alloc_mode for kc_alloc */
    int32_t _pad;
} kc_options;

typedef struct {
    uint64_t n_regions, n_chunks, total_bytes;
    uint64_t n_failed_regions;
    uint64_t written_chunks;        /* |W| */
    uint64_t d2h_bytes;             /* bytes copied device->host */
    uint64_t dma_calls;             /* number of D2H copy calls */
    uint64_t staging_high_water;    /* peak pinned staging bytes in use */
    uint64_t snapshot_digest;       /* S of the region files (pre state in PRE_W) */
    double t_hash_pre_s, t_d2h_s, t_dispatch_s, t_hash_post_s, t_total_s;
} kc_capture_report;

typedef struct {
    uint32_t iterations;        /* >= 1 */
    int32_t no_recopy;          /* 1: do not restore W's pre-state between iterations */
    const char* dump_dir;       /* NULL: no output dump */
    const void* image_override; /* variant code object ("--hsaco") */
    size_t image_override_size;
    void* stream;
    /* launch-shape overrides for a variant whose configuration differs (a
     * retuned tile: other block size or dynamic shared memory; the paper's
     * reproducer exposes the launch configuration for editing).  Bits of
     * `overrides`: 1 grid, 2 block, 4 smem_bytes, 8 symbol; zero = as captured.
     * The kernarg buffer is always the captured one. */
    uint32_t overrides;
    uint32_t grid[3], block[3];
    uint32_t smem_bytes;
    const char* symbol;         /* kernel name in the override code object */
} kc_replay_opts;
enum { KC_OVR_GRID = 1, KC_OVR_BLOCK = 2, KC_OVR_SMEM = 4, KC_OVR_SYMBOL = 8 };

typedef struct {
    uint32_t iterations;
    uint32_t module_vars_restored; /* F3: module variables written into the replay module */
    double kernel_ms_mean, kernel_ms_min, kernel_ms_max;
} kc_replay_report;

typedef struct {
    uint64_t n_regions, n_spans, mapped_bytes, h2d_bytes;
    uint64_t n_failed_regions;      /* reserved and zero-filled */
    uint64_t verify_mismatch_chunks;
    double t_reserve_s, t_h2d_s, t_verify_s, t_total_s;
} kc_restore_report;

typedef struct kc_ctx kc_ctx;
typedef struct kc_restored kc_restored;
typedef struct kc_snapshot kc_snapshot;   /* device-resident snapshot (F1) */

/* ---- lifetime ---------------------------------------------------------- */
/* Creates a context on opt->device (primary CUDA context).  opt may be NULL. */
kc_status kc_create(kc_ctx** out, const kc_options* opt);
void kc_destroy(kc_ctx* ctx);
/* Last error message of this ctx (valid until the next call on it). */
const char* kc_last_error(const kc_ctx* ctx);
/* ABI version and a build identification string (arch, flags). */
int kc_abi_version(void);
const char* kc_build_info(void);
const char* kc_status_str(kc_status s);
/* Number of libkc kernels this ctx has launched so far (bench evidence). */
uint64_t kc_kernel_launches(const kc_ctx* ctx);

/* ---- A1 allocation tracking -------- */
/* Feeds one driver event: ALLOC/MAP add [base, base+size); FREE/UNMAP remove
 * the entry at base (size ignored).  An unknown FREE is KC_OK plus a warning
 * (SPEC.md:320, 324).  Overlap with a live entry is KC_ERR_ARG. */
kc_status kc_track(kc_ctx* ctx, kc_event ev, uint64_t base, uint64_t size, int32_t device, int32_t kind);
/* Copies up to cap live regions, sorted by base, into out; *n_out = live count. */
kc_status kc_regions(kc_ctx* ctx, kc_region* out, size_t cap, size_t* n_out);
/* Driver-API interposition: allocate / free wrappers that feed the tracker
 * (the CUDA analog of the paper's hooked pool allocate / VMEM map, PAPER.md:
 * 490-497).  KC_ALLOC_VMM: cuMemAddressReserve + cuMemCreate + cuMemMap +
 * cuMemSetAccess (granularity-rounded); KC_ALLOC_MEMALLOC: cuMemAlloc. */
kc_status kc_alloc(kc_ctx* ctx, uint64_t size, uint64_t* dptr_out);
kc_status kc_free(kc_ctx* ctx, uint64_t dptr);
/* CUPTI driver-API callback interposition (cuMemAlloc*, cuMemFree*, cuMemMap,
 * cuMemUnmap).  Second install -> KC_ERR_STATE. */
kc_status kc_track_install(kc_ctx* ctx);
kc_status kc_track_uninstall(kc_ctx* ctx);

/* ---- K1 chunk hash (A2/A4; north star) -------------------------------- */
/* Hashes every region: d_chunk_hash[C] (device, u64, global chunk order =
 * regions in the given order, chunks in order; C = sum ceil(size/65536)).
 * d_region_digest (device, n words) and d_snapshot_digest (device, 1 word)
 * may be NULL.  Regions must be sorted by base and non-overlapping when the
 * snapshot digest is requested.  Asynchronous on stream. */
kc_status kc_hash(kc_ctx* ctx, const kc_region* regions, size_t n, uint64_t* d_chunk_hash,
                  uint64_t* d_region_digest, uint64_t* d_snapshot_digest, void* stream);
/* Total chunk count of a region list (host helper). */
uint64_t kc_count_chunks(const kc_region* regions, size_t n);

/* ---- prepared plans (K1 / K2 without per-call host work) ---------------- */
/* The paper's loop hashes and validates the SAME region and buffer sets again
 * and again (pre/post manifests, every replay's validation).
 * A plan validates and uploads the set once; each run is the kernel launches
 * alone, bit-identical to kc_hash / kc_diff_async on the same inputs.
 * kc_hash_plan_create: regions as kc_hash (copied; the memory they describe
 * must stay mapped while the plan is run).  kc_hash_plan_run: as kc_hash
 * (asynchronous on stream); KC_ERR_ARG when the snapshot digest is requested
 * for an unsorted/overlapping set.  kc_diff_plan_create: bufs, report_nbytes
 * and bitmap_word0 as kc_diff_async (copied; bitmap_word0 may be NULL, then
 * runs take no bitmaps).  kc_diff_plan_run: as kc_diff_async with the plan's
 * buffers (reports zeroed and finalized; asynchronous).  A plan belongs to the
 * ctx that created it (KC_ERR_ARG elsewhere) and must be destroyed before it;
 * destroy(NULL) is a no-op. */
typedef struct kc_hash_plan kc_hash_plan;
typedef struct kc_diff_plan kc_diff_plan;
kc_status kc_hash_plan_create(kc_ctx* ctx, const kc_region* regions, size_t n, kc_hash_plan** out);
kc_status kc_hash_plan_run(kc_ctx* ctx, const kc_hash_plan* p, uint64_t* d_chunk_hash, uint64_t* d_region_digest,
                           uint64_t* d_snapshot_digest, void* stream);
uint64_t kc_hash_plan_chunks(const kc_hash_plan* p);
kc_status kc_hash_plan_destroy(kc_hash_plan* p);
kc_status kc_diff_plan_create(kc_ctx* ctx, const kc_buffer* bufs, size_t n_bufs, size_t n_reports,
                              const uint64_t* report_nbytes, const uint64_t* bitmap_word0, kc_diff_plan** out);
kc_status kc_diff_plan_run(kc_ctx* ctx, const kc_diff_plan* p, const kc_tolerance* tol, kc_diff_report* d_reports,
                           uint64_t* d_bitmaps, void* stream);
kc_status kc_diff_plan_destroy(kc_diff_plan* p);

/* ---- K3 written set (A4) ---------------------------------------------- */
/* W[k] = (pre[k] != post[k]) for k < n_chunks: d_w_bitmap (device,
 * ceil(C/64) u64, LSB-first) and d_written_count (device, 1 u64).  Async. */
kc_status kc_written(kc_ctx* ctx, const uint64_t* d_pre, const uint64_t* d_post, uint64_t n_chunks,
                     uint64_t* d_w_bitmap, uint64_t* d_written_count, void* stream);

/* ---- K2 fused diff (A8) ----------------------------------------------- */
/* Compares every segment; reports accumulate per bufs[i].report index in
 * d_reports (device, n_reports entries, zeroed and finalized here), bitmaps in
 * d_bitmaps (device; report j's bitmap starts at word bitmap_word0[j], host
 * array of n_reports entries, may be NULL when d_bitmaps is NULL).
 * report_nbytes[j] (host) = total bytes of report j (for percent/n_chunks).
 * Asynchronous on stream. */
kc_status kc_diff_async(kc_ctx* ctx, const kc_buffer* bufs, size_t n_bufs, size_t n_reports,
                        const uint64_t* report_nbytes, const uint64_t* bitmap_word0,
                        const kc_tolerance* tol, kc_diff_report* d_reports, uint64_t* d_bitmaps,
                        void* stream);
/* F2 hash-filtered validation against a HOST-resident reference (SURVEY.md
 * 8(f) F2: "validate by manifest compare first and H2D only the references of
 * mismatching chunks"; the report is O4's).
 * bufs[i].ref = HOST address of the reference bytes (pinned for full PCIe rate),
 * bufs[i].act = device VA (16-byte aligned), nbytes, dtype; .report and
 * .bitmap_chunk0 are ignored (one report per buffer, as kc_diff).
 * ref_manifest (host) = the reference's XXH64 chunk hashes, buffers in order
 * (a snapshot's manifest).  One K5 pass reads act once (its manifest and the
 * chunks holding Inf/NaN), K3 marks the chunks whose hash differs from
 * ref_manifest, only their reference bytes cross PCIe, and K2 runs over exactly
 * those chunks plus the Inf/NaN chunks with equal hashes (compared with
 * themselves: equal hashes are equal bytes, reading R34, the same test as W).
 * reps: n reports (host); h_bitmaps: optional host bitmaps (as kc_diff);
 * d_act_manifest: optional device output of act's chunk hashes; *h2d_bytes:
 * bytes moved host->device (manifest + reference chunks).  Device scratch: 8 B
 * per chunk (manifest) plus 64 KiB per chunk whose hash differs (the staged
 * reference bytes); KC_ERR_NOMEM if that does not fit.
 * ref_manifest == NULL selects BYTE-EXACT mode (the paper's strict compare,
 * PAPER.md:1120-1126, with no hash trusted): every reference byte crosses
 * PCIe, streamed through a 3 x 256 MiB device staging ring on the context's
 * copy stream while K2 diffs the previous piece on `stream`; *h2d_bytes = the
 * total reference bytes; d_act_manifest (optional) is then filled by K1 over
 * the act buffers in order.  Reports and bitmaps equal kc_diff's over the same
 * (reference, actual) pairs.  Blocks until the reports are on the host. */
kc_status kc_validate_host_ref(kc_ctx* ctx, const kc_buffer* bufs, size_t n, const uint64_t* ref_manifest,
                               const kc_tolerance* tol, kc_diff_report* reps, uint64_t* h_bitmaps,
                               uint64_t* d_act_manifest, uint64_t* h2d_bytes, void* stream);
/* Convenience: one report per buffer, results copied to HOST reps[n] and
 * h_bitmaps (concatenated ceil(n_chunks_i/64) words per buffer, may be NULL).
 * Synchronizes the stream. */
kc_status kc_diff(kc_ctx* ctx, const kc_buffer* bufs, size_t n, const kc_tolerance* tol,
                  kc_diff_report* reps, uint64_t* h_bitmaps, void* stream);

/* ---- E2 peer mappings ------------------------------
 * The north star's "each GPU hashes and diffs its shard (reading peer memory
 * over NVLink)": a pool resident on one GPU is read by the kernels of other
 * GPUs, one process per GPU.  The paper is single-GPU.
 *
 * kc_peer_export: the physical allocation behind a VMM kc_alloc allocation
 * (base = the address kc_alloc returned) as a POSIX file descriptor of this
 * process (*fd_out, owned by the ctx: closed by kc_free(base) or kc_destroy)
 * and its mapped size (*size_out, granularity-rounded).  The fd number is only
 * meaningful together with this process's pid.  KC_ERR_NOT_TRACKED if base is
 * not such an allocation (KC_ALLOC_MEMALLOC memory cannot be exported). */
kc_status kc_peer_export(kc_ctx* ctx, uint64_t base, int32_t* fd_out, uint64_t* size_out);
/* kc_peer_import: duplicate the owner's fd (pid, fd from kc_peer_export) with
 * pidfd_getfd (Linux >= 5.6; same user or CAP_SYS_PTRACE), import it and map
 * size bytes read-write for THIS ctx's device: peer access over NVLink when the
 * owner is another GPU, a second mapping when it is the same GPU.  The mapping
 * is placed at want_va when that range is free in this process (0 = anywhere),
 * else at a fresh VA; *va_out receives it.  Chunk hashes and diff reports do
 * not depend on the VA, so the manifests equal the owner's.  The owner must
 * keep the allocation alive while it is mapped here.  KC_ERR_STATE when the
 * owner process or its fd is gone; KC_ERR_CUDA on an import/map failure
 * (nothing is left mapped). */
kc_status kc_peer_import(kc_ctx* ctx, int32_t pid, int32_t fd, uint64_t size, uint64_t want_va, uint64_t* va_out);
/* kc_peer_release: unmap an imported mapping (after the device is idle) and
 * drop the imported handle.  KC_ERR_NOT_TRACKED if va is not one. */
kc_status kc_peer_release(kc_ctx* ctx, uint64_t va);

/* ---- A9 combine: finalize reports merged across ranks ------------------
 * a buffer's report is split over the ranks that hold its
 * chunks; their counters are SUMmed and their maxima MAXed (exact, order-free)
 * by the caller's collective.  This recomputes the derived fields of each
 * merged report from nbytes[i] and dtypes[i] (kc_dtype) with the rules K2
 * applies at the end of kc_diff (O4, readings R9, R18):
 * nbytes, n_elems = nbytes / element size, n_chunks = ceil(nbytes / 65536),
 * percent_bytes = RN(RN(100 * differing_bytes) / nbytes) (0 when nbytes = 0),
 * differing_elems = differing_bytes for KC_DT_BYTES, and pass (floats:
 * allclose_fail == 0; integers: differing_elems == 0; bytes: differing_bytes
 * == 0).  reps, nbytes, dtypes: HOST arrays of n entries (borrowed; reps is
 * updated in place).  No CUDA call: usable on any host.  KC_ERR_ARG on a NULL
 * array with n > 0, an unknown dtype, or nbytes not a multiple of the
 * element size. */
kc_status kc_report_finalize(kc_diff_report* reps, const uint64_t* nbytes, const int32_t* dtypes, size_t n);

/* ---- F2 fused hash + validate ----------------------
 * One pass (K5) over every buffer pair hashes the ACTUAL bytes (the chunk
 * manifest of the regions {act, nbytes} in the given order: bit-identical to
 * kc_hash over them) while comparing them with the reference.  A chunk whose
 * bits all agree and whose reference holds no Inf/NaN (float dtypes)
 * contributes nothing to any report field; K2 then reads only the other
 * ("dirty") chunks.  Results equal kc_diff's: one report per buffer (the
 * .report and .bitmap_chunk0 fields are ignored) in d_reports (device, n),
 * bitmaps (device, may be NULL) concatenated per buffer at ceil(n_chunks_i/64)
 * words each.  d_chunk_hash: device, sum of n_chunks_i words.  d_dirty:
 * device ceil(C/64) words receiving the dirty-chunk bitmap, or NULL (ctx
 * scratch).  Buffers not 16-byte aligned run K1 + an unfiltered K2 instead
 * (every chunk reported dirty).
 * Asynchronous on stream. */
kc_status kc_hash_diff_async(kc_ctx* ctx, const kc_buffer* bufs, size_t n, const kc_tolerance* tol,
                             uint64_t* d_chunk_hash, kc_diff_report* d_reports, uint64_t* d_bitmaps,
                             uint64_t* d_dirty, void* stream);

/* ---- A3/A5 capture --------------- */
/* Quiesce, hash, write metadata FIRST, snapshot through the pinned ring,
 * forward the dispatch, hash again, record W, write capture_log.json and the
 * capture_complete sentinel LAST.  regions == NULL: every tracked region.
 * Per-region copy failures -> KC_PARTIAL (the dispatch always proceeds). */
kc_status kc_capture(kc_ctx* ctx, const kc_dispatch* d, const kc_region* regions, size_t n, const char* dir,
                     kc_capture_mode mode, kc_capture_report* rep);

/* ---- A6 VA-faithful restore ----------- */
/* Reserves every granule span at its captured VA (abort + full rollback with
 * KC_ERR_VA_UNAVAILABLE if the driver returns another address), maps
 * device-local memory, copies the region files in, zero-fills gaps and
 * failed regions, and verifies the bytes against the captured manifest. */
kc_status kc_restore(kc_ctx* ctx, const char* dir, kc_restored** out, kc_restore_report* rep);
/* Stage 2 of the paper's replay reserves the captured
 * ranges with mmap(MAP_FIXED_NOREPLACE) before the runtime initialises.  On
 * CUDA that backfires: ranges mapped at cuInit are excluded from the driver's
 * VA space for the process lifetime (measured, R28).  So this is a
 * CHECK, called before CUDA initialises: KC_PARTIAL when a host mapping
 * already overlaps a captured 32 MiB window (the replay process should re-exec
 * for a fresh ASLR layout); *n_reserved = windows that are free.  Maps nothing,
 * makes no CUDA calls. */
kc_status kc_prereserve(const char* dir, uint64_t* n_reserved);

/* ---- F1 device-resident snapshot --------------------
 * The same capture with the region bytes kept in a device arena in this GPU's
 * HBM (D2D copies at HBM bandwidth instead of PCIe + files): PRE_W keeps the
 * pre-dispatch bytes of every region plus the post bytes of W, POST the
 * post-dispatch bytes.  Manifests, W and the dispatch description stay in host
 * memory inside the kc_snapshot.  The arena (sum of region sizes, 256 B
 * aligned per region, + |W| chunks) is allocated with cudaMalloc and owned by
 * the snapshot; KC_ERR_NOMEM if it does not fit.  The dispatch is forwarded
 * exactly as in kc_capture (it always proceeds). */
kc_status kc_capture_dev(kc_ctx* ctx, const kc_dispatch* d, const kc_region* regions, size_t n, kc_capture_mode mode,
                         kc_snapshot** out, kc_capture_report* rep);
/* The same capture into a PINNED HOST arena (cudaHostAlloc): the region bytes
 * leave the GPU at PCIe rate (A5's D2H without the file sink; SURVEY.md 8(d)
 * D.4 "the latency benchmark uses a pinned in-memory arena").  Small regions
 * (< 1 MiB) are packed by one K4 launch writing through the mapped pinned
 * pages.  The arena is taken from the ctx's pinned-arena cache when one of
 * sufficient size is parked there (kc_host_arena_reserve, or a freed host
 * snapshot), else allocated (pinning costs ~0.2-0.3 s per 10 GB). */
kc_status kc_capture_host(kc_ctx* ctx, const kc_dispatch* d, const kc_region* regions, size_t n, kc_capture_mode mode,
                          kc_snapshot** out, kc_capture_report* rep);
/* F2 incremental capture: the capture of kc_capture_dev
 * (host = 0) / kc_capture_host (host != 0) that copies only the chunks whose
 * stored-state hash (pre-dispatch in PRE_W, post in POST) differs from
 * `base`'s stored manifest at the same region base, size and chunk index;
 * every other chunk references the base's bytes (hash equality is the same
 * "unchanged" test the written set W uses).  The new snapshot shares
 * ownership of the base's arenas: the base may be freed first.  base = NULL
 * is a full capture.  rep->d2h_bytes = bytes actually copied. */
kc_status kc_capture_incr(kc_ctx* ctx, const kc_dispatch* d, const kc_region* regions, size_t n, kc_capture_mode mode,
                          const kc_snapshot* base, int host, kc_snapshot** out, kc_capture_report* rep);
/* Pin `bytes` of host memory ahead of time and park it in the ctx's cache (one
 * arena; a larger request replaces a smaller parked one).  0 frees the cache. */
kc_status kc_host_arena_reserve(kc_ctx* ctx, uint64_t bytes);
/* Map `bytes` of device memory (one VMM allocation) ahead of time and park it
 * in the ctx for kc_capture_dev; a freed device snapshot also parks its arena
 * there when it is the larger one (never an exported one).  0 releases it, and
 * with it the physical allocations parked by released restores (a released
 * kc_restored parks each span's physical allocation in the ctx, up to
 * KC_PHYS_PARK_MAX bytes, default 96 GiB; the next restore takes a parked one of
 * the same size instead of cuMemCreate; KC_PHYS_PARK=0 releases them at once). */
kc_status kc_dev_arena_reserve(kc_ctx* ctx, uint64_t bytes);
/* Same-VA restore from an in-memory snapshot (device or pinned host arena; the
 * originals must be freed first): VA windows as kc_restore (or the ctx VA
 * heap), then copy-in (D2D or H2D) and the K1 verify. */
kc_status kc_restore_dev(kc_ctx* ctx, const kc_snapshot* s, kc_restored** out, kc_restore_report* rep);
/* Restore an in-memory snapshot into a LIVE restore of the same regions (the same
 * bases, sizes and ok flags, in order): the VA windows and mappings of `r` are kept
 * (no reservation, no cuMemCreate / cuMemMap), and stages 5-6 of kc_restore_dev run
 * on them: zero-fill, copy-in fused with the verify hashes (K6), verify, W stashes.
 * `r` takes the snapshot's dispatch, written sets and post manifests, so kc_replay /
 * kc_validate then act on the new capture.  This is the repeated-replay fast path of
 * a resident tool (capture from the restored state, restore over it, replay again;
 * PAPER.md:1100-1108's stage 5 without stages 2-4).  KC_ERR_ARG when the region
 * lists differ; on a copy-in or verify failure `r` stays mapped with undefined
 * contents (release it, or restore into it again). */
kc_status kc_restore_dev_into(kc_ctx* ctx, const kc_snapshot* s, kc_restored* r, kc_restore_report* rep);
/* Persist an in-memory snapshot as a kc-snapshot/1 directory (parallel). */
kc_status kc_snapshot_save(kc_ctx* ctx, const kc_snapshot* s, const char* dir);
/* F1 across processes: persist the snapshot's metadata, manifests and W bytes
 * as a kc-snapshot/1 directory whose region bytes stay in THIS process's
 * device arena, shared through CUDA IPC (memory/device_arena.json: the
 * cudaIpcMemHandle_t and each region's arena offset; no memory/region_*.bin).
 * kc_restore(dir) in another process on the same GPU maps the arena and copies
 * in at HBM bandwidth (fused with the verify hashes) instead of reading files.
 * Valid while this process keeps the snapshot alive.  KC_ERR_STATE for host
 * snapshots and incremental ones (stored bytes not in one own arena). */
kc_status kc_snapshot_publish(kc_ctx* ctx, const kc_snapshot* s, const char* dir);
/* Load a kc-snapshot/1 directory into an in-memory snapshot (device arena, or
 * pinned host arena when host != 0), verified against its manifests (K1).
 * The edit -> replay -> validate loop then restores from memory at HBM (or
 * PCIe) rate each time instead of re-reading the files.  KC_ERR_FORMAT for an
 * incomplete or malformed directory, KC_ERR_MANIFEST_MISMATCH if a region file
 * does not match its manifest. */
kc_status kc_snapshot_load(kc_ctx* ctx, const char* dir, int host, kc_snapshot** out);
/* Bytes this snapshot copied into its own arenas. */
uint64_t kc_snapshot_bytes(const kc_snapshot* s);
/* Stored bytes referenced from base snapshots (kc_capture_incr), not copied. */
uint64_t kc_snapshot_shared_bytes(const kc_snapshot* s);
/* 1 = pinned host arena (kc_capture_host), 0 = device arena. */
int kc_snapshot_is_host(const kc_snapshot* s);
/* Frees the arenas; a host arena is parked in the ctx's cache instead when it
 * is at least as large as the one parked there. */
void kc_snapshot_free(kc_snapshot* s);

/* ---- A7 replay ------------------------------------ */
kc_status kc_replay(kc_ctx* ctx, kc_restored* h, const kc_replay_opts* o, kc_replay_report* rep);

/* ---- F3 module variables -----------------------------
 * kc_capture / kc_capture_dev / kc_capture_host record every __device__ /
 * __constant__ variable of the dispatch's code object (ELF .nv.global* /
 * .nv.constant* symbols other than the kernel parameter banks, resolved with
 * cuModuleGetGlobal in the dispatch's module) before and after the dispatch
 * (module_vars.json + module_vars/NNN.{pre,post}.bin).  The code object is
 * d->image, else (d->func only) the image the CUPTI hook recorded when the
 * application loaded the module (kc_track_install: cuModuleLoadData,
 * cuModuleLoadDataEx, cuModuleLoadFatBinary) - PAPER.md:506-516.  kc_replay
 * writes them into the replay module (pre values in PRE_W, post in POST)
 * before the launch (and before each iteration when written and recopying),
 * then compares every variable with its captured post value; this call reads
 * that comparison of the LAST kc_replay.  KC_NO_MODULE_VARS=1 disables both
 * sides (ablation). */
kc_status kc_validate_module_vars(kc_ctx* ctx, const kc_restored* h, uint64_t* n_checked, uint64_t* n_mismatch);

/* ---- A8 validate ---------------------------------- */
/* outs == NULL: every region with written chunks, compared as bytes against
 * the captured post-dispatch bytes (PRE_W), one report per such region in
 * region order; *n_reports_out = their count.  outs != NULL: typed
 * sub-ranges ref=captured-post VA offset, act=live VA (only .act/.nbytes/
 * .dtype used; ref comes from the capture).  Also re-hashes every restored
 * region and counts chunks whose hash differs from the captured post
 * manifest (*unexpected_chunks, may be NULL). */
kc_status kc_validate(kc_ctx* ctx, kc_restored* h, const kc_buffer* outs, size_t n, const kc_tolerance* tol,
                      kc_diff_report* reps, size_t cap_reports, size_t* n_reports_out,
                      uint64_t* unexpected_chunks);
/* Restored regions (sorted by base). */
kc_status kc_restored_regions(kc_restored* h, kc_region* out, size_t cap, size_t* n_out);
void kc_release(kc_restored* h);

/* ---- loading into an unmodified application ------------------------------
 * CUDA_INJECTION64_PATH=<path>/libkc.so makes the CUDA driver load the library
 * at cuInit and call this (the CUDA counterpart of the paper's HSA tool-library
 * load).  It creates a ctx without touching CUDA, installs the
 * CUPTI hook (kc_track_install) and arms the interposed capture from the
 * environment (KC_CAPTURE_DIR, KC_TARGET, KC_DISPATCH_INDEX, KC_CAPTURE_MODE);
 * the ctx binds to the application's device at its first capture and works in
 * the device's primary context.  Returns 1 when loaded, 0 otherwise (the
 * application then runs without capture). */
int InitializeInjection(void);

/* ---- A3 interposed mode ----------------
 * Capture a dispatch of an application that runs unmodified.  With
 * kc_track_install active (the tracker sees its allocations and module loads),
 * arm the capture of launch number `index` (0-based, counting launches whose
 * kernel name contains `target`; NULL/"" = every kernel).  The CUPTI launch
 * callback brackets that cuLaunchKernel / cuLaunchKernelEx: at ENTER it takes
 * the pre-state of every tracked region into an in-memory snapshot (device
 * arena, or pinned host arena when host != 0), the application's launch then
 * proceeds (exactly once, even if the capture fails), and at EXIT the post
 * manifest and W are taken before the application's call returns.  The kernarg
 * buffer is packed from kernelParams (cuFuncGetParamInfo layout) or copied from
 * CU_LAUNCH_PARAM_BUFFER_POINTER; the code object is the one the module-load
 * hook recorded.  dir != NULL/"": the snapshot is also saved there
 * (kc-snapshot/1).  One capture per arming.  kc_track_install arms from the
 * environment when KC_CAPTURE_DIR is set (KC_TARGET, KC_DISPATCH_INDEX,
 * KC_CAPTURE_MODE=pre_w|post).  KC_ERR_STATE if the hook is not installed. */
kc_status kc_interpose_arm(kc_ctx* ctx, const char* target, uint64_t index, const char* dir, kc_capture_mode mode,
                           int host);
/* *state: 0 idle, 1 armed, 2 capturing, 3 captured, -1 failed (the call then
 * returns the capture's error); *launches_seen: matching launches counted so
 * far; rep: the capture report once captured.  Any output may be NULL. */
kc_status kc_interpose_status(kc_ctx* ctx, int* state, uint64_t* launches_seen, kc_capture_report* rep);
/* The captured in-memory snapshot; ownership passes to the caller (kc_snapshot_free). */
kc_status kc_interpose_take(kc_ctx* ctx, kc_snapshot** out);
/* F4 from an unmodified application: capture the `count` consecutive matching
 * launches [first, first + count) as a sequence (step k = PRE_W state before
 * launch k, incremental against step k-1, as kc_capture_seq); *state reaches 3
 * after the last one.  kc_interpose_take_seq hands over the kc_sequence (its
 * dependency matrix computed; KC_ERR_STATE if the region set changed between
 * steps or the sequence is incomplete). */
kc_status kc_interpose_arm_seq(kc_ctx* ctx, const char* target, uint64_t first, uint64_t count, int host);

/* ---- F4 multi-kernel capture -------------------------
 * PAPER.md:1855-1862 ("capturing a sequence of dependent kernels for joint
 * replay remains future work") and 1917-1918 ("multi-kernel capture for
 * dependent kernel sequences with automatic dependency tracking").
 *
 * kc_capture_seq forwards the n_disp dispatches ds[0..n_disp) in order (each
 * one on its kc_dispatch stream, the device synchronised around it as in
 * kc_capture) and keeps one PRE_W in-memory snapshot per step: step k holds
 * the state before dispatch k, its post manifest and the post bytes of its
 * written set W_k.  Step 0 is a full capture (kc_capture_dev / _host), step
 * k > 0 an incremental one against step k-1 (kc_capture_incr: only chunks
 * changed since step k-1's stored state are copied).  host: 0 = device
 * arenas (HBM), 1 = pinned host arenas.  reps: n_disp capture reports or
 * NULL.  On an error no sequence is returned (steps taken so far are freed),
 * but the dispatches already forwarded have run.  Ownership of *out passes to
 * the caller (kc_seq_free).  regions/n as kc_capture (NULL = the tracker).
 *
 * Dependency tracking (reading R33): for steps i < j,
 *   KC_DEP_RAW  a pointer-sized kernarg parameter of dispatch j (layout from
 *               cuFuncGetParamInfo) holds a VA inside a region of which
 *               dispatch i wrote a chunk (j may read what i wrote);
 *   KC_DEP_WAW  W_i and W_j share a chunk;
 *   KC_DEP_WAR  a pointer parameter of dispatch i lies in a region of which
 *               dispatch j wrote a chunk (j may overwrite what i read).
 * Reads through embedded pointers (pointer chasing) are invisible to the
 * kernarg test; the snapshot still holds them (the closure is whole-heap). */
typedef struct kc_sequence kc_sequence;
enum { KC_DEP_RAW = 1, KC_DEP_WAW = 2, KC_DEP_WAR = 4 };

kc_status kc_capture_seq(kc_ctx* ctx, const kc_dispatch* ds, size_t n_disp, const kc_region* regions, size_t n,
                         int host, kc_sequence** out, kc_capture_report* reps);
/* Number of steps. */
size_t kc_seq_length(const kc_sequence* q);
/* Step k's snapshot (borrowed; owned by the sequence), NULL if k is out of range.
 * It can be restored (kc_restore_dev) and saved (kc_snapshot_save) on its own. */
const kc_snapshot* kc_seq_step(const kc_sequence* q, size_t k);
/* deps[j * n + i] (n = kc_seq_length, caller-allocated n*n bytes): KC_DEP_*
 * flags of step j on step i < j; every other entry 0.  KC_ERR_ARG if cap < n*n. */
kc_status kc_seq_deps(const kc_sequence* q, uint8_t* deps, size_t cap);
/* Persist: dir/step_NNN/ (kc-snapshot/1 each, NNN = 000, 001, ...) and
 * dir/sequence.json (format "kc-sequence/1", n, per-step symbol and |W|, the
 * dependency matrix), sentinel dir/sequence_complete written last. */
kc_status kc_seq_save(kc_ctx* ctx, const kc_sequence* q, const char* dir);
/* Load a kc-sequence/1 directory (kc_seq_save) back into memory, every step
 * through kc_snapshot_load: a fresh process can then run kc_replay_seq.  As
 * for kc_restore, run kc_prereserve (on step_000: every step has the same
 * regions) before CUDA initialises and re-exec on a collision (R28c). */
kc_status kc_seq_load(kc_ctx* ctx, const char* dir, int host, kc_sequence** out);
void kc_seq_free(kc_sequence* q);

typedef struct {
    size_t first, count;                  /* replay steps [first, first + count) */
    const void* const* image_overrides;   /* NULL, or `count` code objects (NULL entry = the captured one) */
    const size_t* image_override_sizes;   /* may be NULL (sizes read from the ELF/fatbin headers) */
    kc_tolerance tol;                     /* used by each step's report (numpy defaults: 1e-8, 1e-5, 0) */
    void* stream;
} kc_seq_replay_opts;

typedef struct {
    kc_diff_report w;            /* the step's W chunks (every region, as bytes) vs the captured post bytes;
                                    bitmap-free; w.nbytes = bytes of the regions the step wrote */
    uint64_t unexpected_chunks;  /* chunks outside W_k whose hash the replayed dispatch changed */
    uint64_t inherited_chunks;   /* chunks whose state at step entry differs from step k's captured pre-state:
                                    divergence carried in from earlier replayed steps (0 for the first step,
                                    which the restore verifies) */
    uint64_t modvar_mismatch;    /* F3 module variables differing from their captured post values */
    double kernel_ms;
    int32_t pass;                /* w.differing_bytes == 0 && unexpected_chunks == 0 && modvar_mismatch == 0
                                    (a step passes on inherited divergence it does not consume) */
    int32_t _pad;
} kc_seq_step_report;

/* Joint replay: restore step `first`'s state at the captured VAs (the live
 * allocations must be gone, as for kc_restore_dev), then for each step k in
 * order replay dispatch k (its captured code object or the override) on the
 * state the previous replays left and validate it -> reps[k - first].  A
 * divergence in step k therefore shows in k's report and propagates to the
 * steps that consume its output.  keep != NULL: the restored state after the
 * last step is returned (kc_release it); else it is released.  Errors of a
 * step abort the replay (reports of earlier steps are filled). */
kc_status kc_replay_seq(kc_ctx* ctx, const kc_sequence* q, const kc_seq_replay_opts* o, kc_seq_step_report* reps,
                        kc_restored** keep);
/* The sequence armed with kc_interpose_arm_seq (ownership passes to the caller). */
kc_status kc_interpose_take_seq(kc_ctx* ctx, kc_sequence** out);

#ifdef __cplusplus
}
#endif
#endif /* KC_H_ */
