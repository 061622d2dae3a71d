// kc_kernels.cuh -- device-side types shared by kc_kernels.cu and kc_runtime.cu
// (product path only; the oracle in oracle/ shares nothing with this file).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/kc.h"

namespace kc {

constexpr uint64_t kChunk = KC_CHUNK_BYTES;  // 65,536 B hash/diff granule (reading R1)

// Device region table: regions in global-chunk order with the
// prefix-summed first chunk index of each region.
struct RegionDev {
    uint64_t base;
    uint64_t size;
    uint64_t chunk_off;
};

// One K2 segment, pre-split into 16 KiB work units (unit_off = prefix sum).
struct SegDev {
    uint64_t ref, act, nbytes;
    uint64_t bitmap_word0;   // first bitmap word of this segment's report
    uint64_t bitmap_chunk0;  // chunk index of byte 0 inside that report
    uint64_t unit_off;       // first global unit index
    uint64_t filter_chunk0;  // filtered launches: index of the segment's first chunk in the dirty bitmap
    int32_t dtype;
    int32_t report;
};

// K5 (F2): one buffer pair whose actual bytes are hashed while compared.
struct PairDev {
    uint64_t act, ref, size;
    uint64_t chunk_off;  // first chunk index (buffers in the given order)
    int32_t dtype;
    int32_t _pad;
};

struct ReportMeta {
    uint64_t nbytes;
    int32_t dtype;
    int32_t _pad;
};

constexpr uint32_t kDiffUnit = 16384;  // K2 work unit (bytes)

// K2 launch group: one dtype, a contiguous run of segments and their units.
struct DiffGroup {
    int32_t dtype;
    int32_t seg0, n_segs;
    uint64_t unit0, n_units;
};

// ---- launchers (kc_kernels.cu) ------------------------------------------
// d_order (may be nullptr = identity): the order in which chunks are assigned to quads
cudaError_t launch_hash(const RegionDev* d_regs, int nreg, uint64_t n_chunks, bool aligned, uint64_t* d_out,
                        const uint32_t* d_chunk_region /* may be nullptr */, int num_sms, cudaStream_t s,
                        const uint32_t* d_order = nullptr);
// K6 (fused capture): K1 over the regions + copy of every byte to d_dst[r] (arena
// address of region r, 16-byte aligned; regions 16-byte aligned)
cudaError_t launch_hash_copy(const RegionDev* d_regs, int nreg, uint64_t n_chunks, uint64_t* d_out,
                             const unsigned long long* d_dst, const uint32_t* d_chunk_region, int num_sms,
                             cudaStream_t s, const uint32_t* d_order = nullptr);
cudaError_t launch_digests(const RegionDev* d_regs, int nreg, const uint64_t* d_chunk_hash, uint64_t* d_region_digest,
                           uint8_t* d_scratch /* 24*nreg */, uint64_t* d_snapshot_digest, cudaStream_t s);
// S over an explicit (base, size, digest) u64 triple list (24 B per region, ascending base)
cudaError_t launch_snapshot_digest(const uint8_t* d_triples, int nreg, uint64_t* d_out, cudaStream_t s);
cudaError_t launch_written(const uint64_t* d_pre, const uint64_t* d_post, uint64_t n_chunks, uint64_t* d_bitmap,
                           uint64_t* d_count, int num_sms, cudaStream_t s);
// d_filter (may be nullptr): dirty-chunk bitmap; units of clean chunks are skipped
cudaError_t launch_diff(const SegDev* d_segs, const DiffGroup* groups, int ngroups, const ReportMeta* d_meta,
                        int nrep, kc_diff_report* d_reps, uint64_t* d_bitmaps, double atol, double rtol,
                        int equal_nan, int num_sms, cudaStream_t s, const uint64_t* d_filter = nullptr);
// K5: chunk hashes of every pair's act bytes + dirty bits (OR-ed into the zeroed d_dirty)
cudaError_t launch_hash_cmp(const PairDev* d_pairs, int npair, uint64_t n_chunks, uint64_t* d_out, uint64_t* d_dirty,
                            const uint32_t* d_chunk_pair, int num_sms, cudaStream_t s, bool self = false);
cudaError_t launch_gather(const uint64_t* d_src_ptrs, const uint64_t* d_dst_ptrs, const uint64_t* d_lens, int n,
                          cudaStream_t s);

// kernel attribute setup (dynamic smem opt-in); call once per device
cudaError_t kernels_init();

}  // namespace kc
