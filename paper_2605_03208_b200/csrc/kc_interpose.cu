// kc_interpose.cu -- A3 interposed mode: capture the index-th
// launch of a named kernel from an application that runs unmodified.
//
// The paper interposes on the HSA dispatch signal: it blocks on its own signal,
// snapshots, then decrements the original.  The CUDA analog
// is the CUPTI driver-API launch callback.  At ENTER of the matching
// cuLaunchKernel / cuLaunchKernelEx the callback starts the in-memory capture on
// a worker thread and waits until the capture has taken the pre-state (quiesce,
// K1/K6 pre-manifest and copy); it then returns and the driver enqueues the
// application's own launch.  At EXIT the worker is released: it synchronizes the
// launch's stream, takes the post-manifest and W, persists the snapshot when a
// directory was given, and the callback returns only when the capture is
// complete.  The application's launch always proceeds, exactly once; a capture
// failure is recorded (kc_interpose_status) and never blocks it (SPEC.md:338,
// 342, 348).  The kernarg buffer is packed from kernelParams with the layout
// from cuFuncGetParamInfo (or copied from CU_LAUNCH_PARAM_BUFFER_POINTER); the
// code object comes from the CUPTI module-load hook (F3).
#include <cupti.h>

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "kc_internal.h"
#include "kc_snapshot_types.h"

using namespace kc;

struct kc_interpose {
    std::mutex mu;
    // arming
    bool armed = false;
    std::string target, dir;
    uint64_t index = 0, seen = 0;
    int mode = KC_MODE_PRE_W;
    bool host = false;
    uint64_t count = 1;                  // launches to capture: [index, index + count)
    std::vector<kc_snapshot*> steps;     // count > 1: the sequence captured so far (F4)
    // outcome: 0 idle, 1 armed, 2 capturing, 3 done, -1 failed
    int state = 0;
    kc_status status = KC_OK;
    kc_capture_report rep{};
    kc_snapshot* snap = nullptr;
    std::string err;
    // the capture in flight
    uint64_t corr = 0;
    std::thread worker;
    bool busy = false;  // ENTER started a worker that EXIT has not joined yet (guarded by mu)
    std::mutex hm;      // guards the handshake flags below
    std::condition_variable cv;
    bool pre_done = false, go = false, launched = false, finished = false;
};

namespace {

kc_interpose* state_of(kc_ctx* ctx) {
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (!ctx->interpose) ctx->interpose = new kc_interpose();
    return ctx->interpose;
}

// the packed parameter buffer of a launch (R22)
bool pack_kernarg(CUfunction f, void** kernelParams, void** extra, std::vector<uint8_t>& out) {
    out.clear();
    if (kernelParams) {
        std::vector<std::pair<size_t, size_t>> lay;
        for (size_t i = 0; i < 4096; ++i) {
            size_t o = 0, z = 0;
            if (KC_DRV(cuFuncGetParamInfo)(f, i, &o, &z) != CUDA_SUCCESS) break;
            lay.emplace_back(o, z);
        }
        if (lay.empty()) return true;
        out.assign(lay.back().first + lay.back().second, 0);
        for (size_t i = 0; i < lay.size(); ++i) memcpy(out.data() + lay[i].first, kernelParams[i], lay[i].second);
        return true;
    }
    if (extra) {
        const void* buf = nullptr;
        size_t sz = 0;
        for (size_t i = 0; extra[i] != CU_LAUNCH_PARAM_END; i += 2) {
            if (extra[i] == CU_LAUNCH_PARAM_BUFFER_POINTER) buf = extra[i + 1];
            else if (extra[i] == CU_LAUNCH_PARAM_BUFFER_SIZE) sz = *(const size_t*)extra[i + 1];
        }
        if (!buf) return false;
        out.assign((const uint8_t*)buf, (const uint8_t*)buf + sz);
        return true;
    }
    return true;  // no parameters
}

}  // namespace

void kc::interpose_launch(kc_ctx* ctx, uint32_t cbid, const void* cbdata) {
    kc_interpose* ip = ctx->interpose;
    if (!ip) return;
    const CUpti_CallbackData* d = (const CUpti_CallbackData*)cbdata;
    if (d->callbackSite == CUPTI_API_ENTER) {
        CUfunction f = nullptr;
        uint32_t grid[3] = {1, 1, 1}, block[3] = {1, 1, 1}, smem = 0, cluster[3] = {1, 1, 1}, flags = 0;
        CUstream stream = nullptr;
        void** kp = nullptr;
        void** extra = nullptr;
        if (cbid == CUPTI_DRIVER_TRACE_CBID_cuLaunchKernel || cbid == CUPTI_DRIVER_TRACE_CBID_cuLaunchKernel_ptsz) {
            auto p = (const cuLaunchKernel_params*)d->functionParams;  // same layout as the _ptsz variant
            f = p->f;
            grid[0] = p->gridDimX, grid[1] = p->gridDimY, grid[2] = p->gridDimZ;
            block[0] = p->blockDimX, block[1] = p->blockDimY, block[2] = p->blockDimZ;
            smem = p->sharedMemBytes;
            stream = p->hStream;
            kp = p->kernelParams;
            extra = p->extra;
        } else if (cbid == CUPTI_DRIVER_TRACE_CBID_cuLaunchCooperativeKernel ||
                   cbid == CUPTI_DRIVER_TRACE_CBID_cuLaunchCooperativeKernel_ptsz) {
            auto p = (const cuLaunchCooperativeKernel_params*)d->functionParams;  // same layout as _ptsz
            f = p->f;
            grid[0] = p->gridDimX, grid[1] = p->gridDimY, grid[2] = p->gridDimZ;
            block[0] = p->blockDimX, block[1] = p->blockDimY, block[2] = p->blockDimZ;
            smem = p->sharedMemBytes;
            stream = p->hStream;
            kp = p->kernelParams;
            flags |= KC_LAUNCH_COOPERATIVE;
        } else {
            auto p = (const cuLaunchKernelEx_params*)d->functionParams;
            if (!p->config) return;
            f = p->f;
            grid[0] = p->config->gridDimX, grid[1] = p->config->gridDimY, grid[2] = p->config->gridDimZ;
            block[0] = p->config->blockDimX, block[1] = p->config->blockDimY, block[2] = p->config->blockDimZ;
            smem = p->config->sharedMemBytes;
            stream = p->config->hStream;
            kp = p->kernelParams;
            extra = p->extra;
            for (unsigned a = 0; a < p->config->numAttrs; ++a)  // a cluster launch (thread-block clusters)
                if (p->config->attrs[a].id == CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION) {
                    cluster[0] = p->config->attrs[a].value.clusterDim.x;
                    cluster[1] = p->config->attrs[a].value.clusterDim.y;
                    cluster[2] = p->config->attrs[a].value.clusterDim.z;
                } else if (p->config->attrs[a].id == CU_LAUNCH_ATTRIBUTE_COOPERATIVE &&
                           p->config->attrs[a].value.cooperative) {
                    flags |= KC_LAUNCH_COOPERATIVE;
                }
        }
        // a launch recorded into a CUDA graph (stream capture) does not run now: it is
        // neither counted nor captured (and syncing would invalidate the graph capture)
        CUstreamCaptureStatus cap = CU_STREAM_CAPTURE_STATUS_NONE;
        if (KC_DRV(cuStreamIsCapturing)(stream, &cap) == CUDA_SUCCESS && cap != CU_STREAM_CAPTURE_STATUS_NONE) return;
        const char* name = nullptr;
        if (KC_DRV(cuFuncGetName)(&name, f) != CUDA_SUCCESS || !name) return;
        if (ctx->device < 0) {  // injected ctx: the application's current device (the worker has no context)
            CUdevice dev = 0;
            if (KC_DRV(cuCtxGetDevice)(&dev) == CUDA_SUCCESS) ctx->device = (int)dev;
        }
        std::string mangled(name);
        {
            std::lock_guard<std::mutex> lk(ip->mu);
            if (!ip->armed) return;
            if (!ip->target.empty() && mangled.find(ip->target) == std::string::npos) return;
            const uint64_t k = ip->seen++;
            if (k < ip->index || k >= ip->index + ip->count) return;
            ip->armed = false;
            if (ip->busy) {  // (defensive: re-arming waits for the previous worker's join)
                ip->state = -1;
                ip->status = KC_ERR_STATE;
                ip->err = "launch " + std::to_string(k) + " arrived while the previous capture was in flight";
                return;
            }
            ip->state = 2;
            ip->corr = d->correlationId;
            ip->busy = true;
        }
        {
            std::lock_guard<std::mutex> lk(ip->hm);
            ip->pre_done = ip->go = ip->launched = ip->finished = false;
        }
        auto kernarg = std::make_shared<std::vector<uint8_t>>();
        if (!pack_kernarg(f, kp, extra, *kernarg)) {
            std::lock_guard<std::mutex> lk(ip->mu);
            ip->state = -1;
            ip->status = KC_ERR_UNSUPPORTED;
            ip->err = "launch parameters neither in kernelParams nor in a CU_LAUNCH_PARAM_BUFFER_POINTER";
            ip->busy = false;
            return;
        }
        ip->worker = std::thread([ctx, ip, f, grid0 = grid[0], grid1 = grid[1], grid2 = grid[2], block0 = block[0],
                                  block1 = block[1], block2 = block[2], smem, stream, mangled, kernarg,
                                  cl0 = cluster[0], cl1 = cluster[1], cl2 = cluster[2], flags]() {
            Internal guard;  // the capture's own driver calls are not the application's
            kc_dispatch disp;
            memset(&disp, 0, sizeof disp);
            disp.func = (void*)f;
            disp.mangled = mangled.c_str();
            disp.grid[0] = grid0, disp.grid[1] = grid1, disp.grid[2] = grid2;
            disp.block[0] = block0, disp.block[1] = block1, disp.block[2] = block2;
            disp.smem_bytes = smem;
            disp.kernarg_size = (uint32_t)kernarg->size();
            disp.kernarg = kernarg->empty() ? nullptr : kernarg->data();
            disp.stream = (void*)stream;
            disp.cluster[0] = cl0, disp.cluster[1] = cl1, disp.cluster[2] = cl2;
            disp.flags = flags;
            // the application's launch happens between the two halves of the capture
            std::function<CUresult()> forward = [ip, stream]() -> CUresult {
                std::unique_lock<std::mutex> lk(ip->hm);
                ip->pre_done = true;
                ip->cv.notify_all();
                ip->cv.wait(lk, [ip] { return ip->go; });
                if (!ip->launched) return CUDA_ERROR_LAUNCH_FAILED;
                lk.unlock();
                return KC_DRV(cuStreamSynchronize)(stream);
            };
            kc_snapshot* sn = nullptr;
            kc_capture_report rep;
            memset(&rep, 0, sizeof rep);
            const bool seq = ip->count > 1;
            const kc_snapshot* base = seq && !ip->steps.empty() ? ip->steps.back() : nullptr;  // incremental (F2)
            // a sequence is PRE_W: step k holds the state before launch k (kc_capture_seq)
            kc_status st = capture_interposed(ctx, &disp, seq ? KC_MODE_PRE_W : (kc_capture_mode)ip->mode, ip->host,
                                              forward, &sn, &rep, base);
            std::string dir;
            {
                std::lock_guard<std::mutex> lk(ip->mu);
                dir = ip->dir;
            }
            if (st >= 0 && sn && !dir.empty() && !seq) {
                kc_status s2 = kc_snapshot_save(ctx, sn, dir.c_str());
                if (s2 < 0) st = s2;
            }
            {
                std::lock_guard<std::mutex> lk(ip->mu);
                ip->status = st;
                ip->rep = rep;
                if (st < 0) {
                    ip->state = -1;
                    ip->err = kc_last_error(ctx);
                    if (sn) kc_snapshot_free(sn);
                } else if (seq) {
                    ip->steps.push_back(sn);
                    ip->state = ip->steps.size() < ip->count ? 1 : 3;  // re-armed by EXIT after the join
                    if (ip->state == 3 && !dir.empty()) {  // complete and a directory given: persist it
                        kc_sequence* q = nullptr;
                        kc_status s2 = make_sequence(ctx, ip->steps, &q);
                        if (s2 == KC_OK) s2 = kc_seq_save(ctx, q, dir.c_str());
                        if (s2 != KC_OK) {
                            ip->state = -1;
                            ip->status = s2;
                            ip->err = kc_last_error(ctx);
                        }
                        if (q) kc_seq_free(q);  // the steps went into q (or stay in ip->steps on failure)
                    }
                } else {
                    ip->state = 3;
                    if (ip->snap) kc_snapshot_free(ip->snap);
                    ip->snap = sn;
                }
            }
            std::lock_guard<std::mutex> lk(ip->hm);
            ip->finished = true;
            ip->cv.notify_all();
        });
        // hold the application's launch until the pre-state is taken (or the capture gave up)
        std::unique_lock<std::mutex> lk(ip->hm);
        ip->cv.wait(lk, [ip] { return ip->pre_done || ip->finished; });
        return;
    }
    // EXIT: release the worker, wait for the capture to finish
    {
        // the bracketed launch (its capture may have failed already: join the worker anyway)
        std::lock_guard<std::mutex> lk(ip->mu);
        if (ip->corr != d->correlationId || !ip->busy) return;
    }
    const CUresult* rv = (const CUresult*)d->functionReturnValue;
    {
        std::lock_guard<std::mutex> lk(ip->hm);
        ip->launched = !rv || *rv == CUDA_SUCCESS;
        ip->go = true;
        ip->cv.notify_all();
    }
    ip->worker.join();
    // only now may the next launch of a sequence start a capture: a new ENTER can no
    // longer race this join or move-assign a joinable worker
    std::lock_guard<std::mutex> lk(ip->mu);
    ip->busy = false;
    if (ip->count > 1 && ip->state == 1) ip->armed = true;
}

static kc_status arm(kc_ctx* ctx, const char* target, uint64_t index, uint64_t count, const char* dir,
                     kc_capture_mode mode, int host);

extern "C" kc_status kc_interpose_arm(kc_ctx* ctx, const char* target, uint64_t index, const char* dir,
                                      kc_capture_mode mode, int host) {
    return arm(ctx, target, index, 1, dir, mode, host);
}

extern "C" kc_status kc_interpose_arm_seq(kc_ctx* ctx, const char* target, uint64_t first, uint64_t count, int host) {
    if (count == 0) return set_err(ctx, KC_ERR_ARG, "kc_interpose_arm_seq: count is 0");
    return arm(ctx, target, first, count, nullptr, KC_MODE_PRE_W, host);
}

extern "C" kc_status kc_interpose_take_seq(kc_ctx* ctx, kc_sequence** out) {
    if (!ctx || !out) return KC_ERR_ARG;
    kc_interpose* ip = state_of(ctx);
    std::lock_guard<std::mutex> lk(ip->mu);
    if (ip->count < 2 || ip->steps.size() != ip->count)
        return set_err(ctx, KC_ERR_STATE, "kc_interpose_take_seq: %zu of %llu steps captured", ip->steps.size(),
                       (unsigned long long)ip->count);
    kc_status st = make_sequence(ctx, ip->steps, out);
    if (st != KC_OK) {
        for (auto it = ip->steps.rbegin(); it != ip->steps.rend(); ++it) kc_snapshot_free(*it);
        ip->steps.clear();
    }
    return st;
}

static kc_status arm(kc_ctx* ctx, const char* target, uint64_t index, uint64_t count, const char* dir,
                     kc_capture_mode mode, int host) {
    if (!ctx) return KC_ERR_ARG;
    if (mode != KC_MODE_PRE_W && mode != KC_MODE_POST) return set_err(ctx, KC_ERR_ARG, "kc_interpose_arm: bad mode");
    if (!ctx->cupti_installed)
        return set_err(ctx, KC_ERR_STATE, "kc_interpose_arm: kc_track_install first (the launch hook is CUPTI's)");
    kc_interpose* ip = state_of(ctx);
    std::lock_guard<std::mutex> lk(ip->mu);
    if (ip->state == 2 || ip->busy) return set_err(ctx, KC_ERR_STATE, "kc_interpose_arm: a capture is in flight");
    ip->armed = true;
    ip->target = target ? target : "";
    ip->dir = dir ? dir : "";
    ip->index = index;
    ip->count = count;
    for (auto it = ip->steps.rbegin(); it != ip->steps.rend(); ++it) kc_snapshot_free(*it);
    ip->steps.clear();
    ip->seen = 0;
    ip->mode = mode;
    ip->host = host != 0;
    ip->state = 1;
    ip->status = KC_OK;
    ip->err.clear();
    memset(&ip->rep, 0, sizeof ip->rep);
    return KC_OK;
}

extern "C" kc_status kc_interpose_status(kc_ctx* ctx, int* state, uint64_t* launches_seen, kc_capture_report* rep) {
    if (!ctx) return KC_ERR_ARG;
    kc_interpose* ip = state_of(ctx);
    std::lock_guard<std::mutex> lk(ip->mu);
    if (state) *state = ip->state;
    if (launches_seen) *launches_seen = ip->seen;
    if (rep) *rep = ip->rep;
    if (ip->state == -1) set_err(ctx, ip->status, "interposed capture failed: %s", ip->err.c_str());
    return ip->state == -1 ? ip->status : KC_OK;
}

extern "C" kc_status kc_interpose_take(kc_ctx* ctx, kc_snapshot** out) {
    if (!ctx || !out) return KC_ERR_ARG;
    kc_interpose* ip = state_of(ctx);
    std::lock_guard<std::mutex> lk(ip->mu);
    *out = ip->snap;
    ip->snap = nullptr;
    return *out ? KC_OK : set_err(ctx, KC_ERR_STATE, "kc_interpose_take: no captured snapshot");
}

void kc::interpose_destroy(kc_ctx* ctx) {
    kc_interpose* ip = ctx->interpose;
    if (!ip) return;
    if (ip->worker.joinable()) ip->worker.join();
    if (ip->snap) kc_snapshot_free(ip->snap);
    for (auto it = ip->steps.rbegin(); it != ip->steps.rend(); ++it) kc_snapshot_free(*it);
    delete ip;
    ctx->interpose = nullptr;
}

// env arming at kc_track_install (KC_TARGET, KC_DISPATCH_INDEX, KC_CAPTURE_DIR, KC_CAPTURE_MODE)
void kc::interpose_arm_from_env(kc_ctx* ctx) {
    const char* dir = getenv("KC_CAPTURE_DIR");
    if (!dir || !*dir) return;
    const char* t = getenv("KC_TARGET");
    const char* ix = getenv("KC_DISPATCH_INDEX");
    const char* m = getenv("KC_CAPTURE_MODE");
    const char* cnt = getenv("KC_CAPTURE_COUNT");
    const uint64_t count = cnt ? strtoull(cnt, nullptr, 10) : 1;
    arm(ctx, t, ix ? strtoull(ix, nullptr, 10) : 0, count ? count : 1, dir,
        m && strcmp(m, "post") == 0 && count <= 1 ? KC_MODE_POST : KC_MODE_PRE_W, 0);
}
