// kohler_multi.cuh — multi-GPU C ABI (include/kohler_cuda.h, "device group"):
// one host thread drives the devices of one box, one kohler_cuda_ctx and one
// NCCL communicator (ncclCommInitAll) per device.
//
//   kohler_cuda_multi_curve / _analyze : ONE image, the reference's row-block
//       split (proj/src/fast.cpp:42,53-55: block b of B owns rows
//       [h*b/B, h*(b+1)/B), a row owns its right pairs and the down pair into
//       the next row, fast.cpp:15-31).  Device b uploads its rows plus one
//       halo row, K1 computes the exact band partial
//       (kohler_cuda_band_curve_device), ONE NCCL all-reduce of the 512 u64
//       partials merges them like merge_accumulators (src/curve.cpp:16-30),
//       device 0 runs the selection (K4).
//       PEER MODE (the default whenever every device of the group can map
//       the first device's memory, cudaDeviceCanAccessPeer): no collective
//       and no per-device K3 at all -- every device's K1 flush adds its 512
//       exact int64 combinations straight into ONE accumulator on the first
//       device (system-scope RED.ADD.64 over NVLink / NVSwitch, launch_wide's
//       acc_ext), the first device waits for the members' events and runs a
//       single finish_kernel (K3 + K4).  Compute and merge are one kernel per
//       device; KOHLER_MULTI_NO_PEER=1 keeps the NCCL form.
//   kohler_cuda_multi_analyze_batch : a batch sharded by image (contiguous
//       shards, sizes differing by at most one), no collective.
//
// Part of the translation unit kohler_kernels.cu (included at its end); the
// NCCL form uses only the public C ABI, peer mode also launch_wide /
// finish_kernel directly.  NCCL is loaded at run
// time (dlopen "libnccl.so.2": the copy a host process such as torch already
// loaded, else the system one), so the library itself has no link-time NCCL
// dependency; a group of more than one device without NCCL is refused.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <thread>

namespace {

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*destroy)(ncclComm_t) = nullptr;
    const char* (*err)(ncclResult_t) = nullptr;
    bool ok() const { return init_all && all_reduce && destroy && err; }
};

Nccl& nccl()
{
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (n.h)
                break;
        }
        if (!n.h)
            return;
        n.init_all = reinterpret_cast<decltype(n.init_all)>(dlsym(n.h, "ncclCommInitAll"));
        n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(n.h, "ncclAllReduce"));
        n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(n.h, "ncclCommDestroy"));
        n.err = reinterpret_cast<decltype(n.err)>(dlsym(n.h, "ncclGetErrorString"));
    });
    return n;
}

struct Member {
    int device = 0;
    kohler_cuda_ctx* ctx = nullptr;
    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;
    uint8_t* band = nullptr;  // own rows + halo, 16-byte pitch
    size_t band_cap = 0;
    uint64_t* part = nullptr;  // [sum 256 | card 256] partial, then the merged curve
    cudaEvent_t ev = nullptr;  // peer mode: this member's band kernel has flushed
    // selection outputs on the first member
    double* values = nullptr;
    uint8_t* defined = nullptr;
    int* ints = nullptr;  // t0, topk_count, status, topk[...]
    int ints_cap = 0;
};

} // namespace

struct kohler_cuda_multi {
    std::vector<Member> m;
    bool use_nccl = false;
    bool virt = false;  // KOHLER_MULTI_VIRTUAL=1: members may share a device (tests)
    bool peer = false;  // members flush into the first member's accumulator (no collective)
    std::mutex mu;
};

namespace {

#define MC(call) KC_CUDA(call)

int check_image(const uint8_t* px, int w, int h, size_t pitch)
{
    if (!px || w < 1 || h < 1 || pitch < (size_t)w)
        return fail(KOHLER_INVALID_ARGUMENT, "multi: bad image (null, w/h < 1 or pitch < w)");
    return KOHLER_OK;
}

// Run f(i) for every member on its own host thread (device calls of the host
// API are synchronous per member); first failure wins.
template <class F>
int for_members(kohler_cuda_multi* g, F f)
{
    const int n = (int)g->m.size();
    std::vector<int> rc(n, KOHLER_OK);
    std::vector<std::string> msg(n);
    if (n == 1) {
        rc[0] = f(0);
        return rc[0];
    }
    std::vector<std::thread> th;
    for (int i = 0; i < n; ++i)
        th.emplace_back([&, i] {
            rc[i] = f(i);
            if (rc[i] != KOHLER_OK)
                msg[i] = g_last_error;  // this member thread's last error
        });
    for (auto& t : th)
        t.join();
    for (int i = 0; i < n; ++i)
        if (rc[i] != KOHLER_OK)
            return fail(rc[i], "device " + std::to_string(g->m[i].device) + ": " + msg[i]);
    return KOHLER_OK;
}

// Band partial of member b (rows [h*b/B, h*(b+1)/B) + halo) from host memory
// into m.part, then the all-reduce (all members on their own threads).
int band_step(kohler_cuda_multi* g, int b, const uint8_t* px, int w, int h, size_t pitch)
{
    Member& m = g->m[b];
    const int B = (int)g->m.size();
    const int r0 = (int)((long long)h * b / B), r1 = (int)((long long)h * (b + 1) / B);
    const int held = std::min(r1 + 1, h) - r0;
    MC(cudaSetDevice(m.device));
    const size_t dp = ((size_t)w + 15) / 16 * 16;
    if (r1 > r0) {  // (more devices than rows: some bands are empty)
        const size_t need = dp * (size_t)held;
        if (need > m.band_cap) {
            if (m.band)
                cudaFree(m.band);
            m.band = nullptr;
            m.band_cap = 0;
            MC(cudaMalloc(&m.band, need));
            m.band_cap = need;
        }
        MC(cudaMemcpy2DAsync(m.band, dp, px + (size_t)r0 * pitch, pitch, (size_t)w, (size_t)held,
                             cudaMemcpyHostToDevice, m.stream));
        int rc = kohler_cuda_band_curve_device(m.ctx, m.band, w, dp, h, r0, r1, m.part, m.part + 256,
                                               m.stream);
        if (rc)
            return rc;  // message set by the call, on this thread
    } else {
        MC(cudaMemsetAsync(m.part, 0, 512 * sizeof(uint64_t), m.stream));  // an empty band
    }
    if (g->use_nccl) {
        Nccl& n = nccl();
        const ncclResult_t r = n.all_reduce(m.part, m.part, 512, ncclUint64, ncclSum, m.comm, m.stream);
        if (r != ncclSuccess)
            return fail(KOHLER_CUDA_ERROR, std::string("ncclAllReduce: ") + n.err(r));
    }
    MC(cudaStreamSynchronize(m.stream));
    return KOHLER_OK;
}

// ---- peer mode ------------------------------------------------------------
// The group's accumulator: the first member's own K1 accumulator block
// ([kAccCopiesSingle][512] u64, zero between calls: finish_kernel resets it).
int peer_acc(kohler_cuda_multi* g, unsigned long long** acc)
{
    Member& m0 = g->m[0];
    MC(cudaSetDevice(m0.device));
    std::lock_guard<std::mutex> lk(m0.ctx->mu);
    if (int rc = m0.ctx->acc.ensure((size_t)kAccCopiesSingle * 512 * sizeof(unsigned long long), true))
        return rc;
    *acc = static_cast<unsigned long long*>(m0.ctx->acc.p);
    return KOHLER_OK;
}

// Member b: upload its rows (+ halo), K1 over the band with the flush aimed
// at the group's accumulator, record the member's event.  No finish, no sync.
int peer_band_step(kohler_cuda_multi* g, int b, const uint8_t* px, int w, int h, size_t pitch,
                   unsigned long long* acc)
{
    Member& m = g->m[b];
    const int B = (int)g->m.size();
    const int r0 = (int)((long long)h * b / B), r1 = (int)((long long)h * (b + 1) / B);
    const int held = std::min(r1 + 1, h) - r0;
    MC(cudaSetDevice(m.device));
    if (r1 > r0) {  // (more devices than rows: an empty band adds nothing)
        const size_t dp = ((size_t)w + 15) / 16 * 16;
        const size_t need = dp * (size_t)held;
        if (need > m.band_cap) {
            if (m.band)
                cudaFree(m.band);
            m.band = nullptr;
            m.band_cap = 0;
            MC(cudaMalloc(&m.band, need));
            m.band_cap = need;
        }
        MC(cudaMemcpy2DAsync(m.band, dp, px + (size_t)r0 * pitch, pitch, (size_t)w, (size_t)held,
                             cudaMemcpyHostToDevice, m.stream));
        if (int rc = check_image(1, w, h, dp))
            return rc;
        std::lock_guard<std::mutex> lk(m.ctx->mu);
        m.ctx->last_launches = 0;
        const BatchOut none{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
        if (int rc = launch_wide(m.ctx, m.band, 1, w, r1 - r0, h, r0, dp, 0, 1, 0, none, m.stream,
                                 /*no_finish=*/1, nullptr, false, acc))
            return rc;
    }
    MC(cudaEventRecord(m.ev, m.stream));
    return KOHLER_OK;
}

// All members' flushes -> one finish_kernel on the first device (K3, and K4
// if select): sums / cards into m0.part, the selection outputs as given.
int peer_finish(kohler_cuda_multi* g, unsigned long long* acc, int k, int select, double* values,
                uint8_t* defined, int* t0, int* topk, int* topk_count, int* status)
{
    Member& m0 = g->m[0];
    MC(cudaSetDevice(m0.device));
    for (Member& m : g->m)
        MC(cudaStreamWaitEvent(m0.stream, m.ev, 0));
    FinishParams fp{};
    fp.acc = acc;
    fp.copies = kAccCopiesSingle;
    fp.k = k;
    fp.select = select;
    fp.sums = m0.part;
    fp.cards = m0.part + 256;
    fp.values = values;
    fp.defined = defined;
    fp.t0s = t0;
    fp.topks = topk;
    fp.topk_counts = topk_count;
    fp.status = status;
    MC(launch_pdl(finish_kernel, 1u, 256, 0, m0.stream, fp));
    MC(cudaStreamSynchronize(m0.stream));
    return KOHLER_OK;
}

// The band steps of one image in peer mode; on failure the accumulator is
// cleared again (a later call must start from zero).
int peer_image(kohler_cuda_multi* g, const uint8_t* px, int w, int h, size_t pitch, int k, int select,
               double* values, uint8_t* defined, int* t0, int* topk, int* topk_count, int* status)
{
    unsigned long long* acc = nullptr;
    if (int rc = peer_acc(g, &acc))
        return rc;
    int rc = for_members(g, [&](int b) { return peer_band_step(g, b, px, w, h, pitch, acc); });
    if (rc == KOHLER_OK)
        rc = peer_finish(g, acc, k, select, values, defined, t0, topk, topk_count, status);
    if (rc != KOHLER_OK) {
        const std::string keep = g_last_error;
        for (Member& m : g->m) {
            cudaSetDevice(m.device);
            cudaStreamSynchronize(m.stream);
        }
        cudaSetDevice(g->m[0].device);
        cudaMemset(acc, 0, (size_t)kAccCopiesSingle * 512 * sizeof(unsigned long long));
        (void)cudaGetLastError();
        g_last_error = keep;
    }
    return rc;
}

// Without NCCL (a virtual group, or one member): the members' partials summed
// on the host into the first member's buffer (u64 wraparound sum, exactly
// merge_accumulators, src/curve.cpp:16-30).
int merge_without_nccl(kohler_cuda_multi* g)
{
    if (g->use_nccl || g->m.size() < 2)
        return KOHLER_OK;
    std::vector<uint64_t> acc(512, 0), part(512);
    for (Member& m : g->m) {
        MC(cudaSetDevice(m.device));
        MC(cudaMemcpy(part.data(), m.part, 512 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
        for (int i = 0; i < 512; ++i)
            acc[i] += part[i];
    }
    MC(cudaSetDevice(g->m[0].device));
    MC(cudaMemcpy(g->m[0].part, acc.data(), 512 * sizeof(uint64_t), cudaMemcpyHostToDevice));
    return KOHLER_OK;
}

} // namespace

extern "C" {

int kohler_cuda_multi_create(const int* devices, int ndev, kohler_cuda_multi** out)
{
    if (!out || ndev < 1)
        return fail(KOHLER_INVALID_ARGUMENT, "multi: need >= 1 device and an output pointer");
    *out = nullptr;
    auto* g = new kohler_cuda_multi();
    {
        // test mode: several members on one GPU (this box has one), merged on
        // the host instead of by NCCL -- exercises the row-block split,
        // empty bands and the merge arithmetic of a B-device group
        const char* v = std::getenv("KOHLER_MULTI_VIRTUAL");
        g->virt = v && v[0] && v[0] != '0';
    }
    std::vector<int> devs(ndev);
    for (int i = 0; i < ndev; ++i)
        devs[i] = devices ? devices[i] : i;
    for (int i = 0; i < ndev && !g->virt; ++i)
        for (int j = 0; j < i; ++j)
            if (devs[i] == devs[j]) {
                delete g;
                return fail(KOHLER_INVALID_ARGUMENT, "multi: a device is listed twice");
            }
    g->m.resize(ndev);
    int rc = KOHLER_OK;
    for (int i = 0; i < ndev && rc == KOHLER_OK; ++i) {
        Member& m = g->m[i];
        m.device = devs[i];
        rc = kohler_cuda_create(m.device, &m.ctx);
        if (rc)
            break;
        cudaError_t e = cudaSetDevice(m.device);
        if (e == cudaSuccess)
            e = cudaStreamCreateWithFlags(&m.stream, cudaStreamNonBlocking);
        if (e == cudaSuccess)
            e = cudaEventCreateWithFlags(&m.ev, cudaEventDisableTiming);
        if (e == cudaSuccess)
            e = cudaMalloc(&m.part, 512 * sizeof(uint64_t));
        if (e != cudaSuccess)
            rc = fail(KOHLER_CUDA_ERROR, std::string("multi: ") + cudaGetErrorString(e));
    }
    if (rc == KOHLER_OK && ndev > 1) {
        // peer mode: every member must be able to map the first device's memory
        const char* np = std::getenv("KOHLER_MULTI_NO_PEER");
        bool peer = !(np && np[0] && np[0] != '0');
        for (int i = 1; i < ndev && peer; ++i) {
            if (devs[i] == devs[0])
                continue;
            // the flush uses 64-bit reductions on the first device's memory:
            // the link must carry native atomics (NVLink does, plain PCIe P2P may not)
            int can = 0, atom = 0;
            if (cudaDeviceCanAccessPeer(&can, devs[i], devs[0]) != cudaSuccess || !can ||
                cudaDeviceGetP2PAttribute(&atom, cudaDevP2PAttrNativeAtomicSupported, devs[i], devs[0]) !=
                    cudaSuccess ||
                !atom) {
                (void)cudaGetLastError();
                peer = false;
                break;
            }
            cudaError_t e = cudaSetDevice(devs[i]);
            if (e == cudaSuccess)
                e = cudaDeviceEnablePeerAccess(devs[0], 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) {
                (void)cudaGetLastError();
                e = cudaSuccess;
            }
            if (e != cudaSuccess) {
                (void)cudaGetLastError();
                peer = false;
            }
        }
        g->peer = peer;
    }
    if (rc == KOHLER_OK && !g->virt && !g->peer) {
        Nccl& n = nccl();
        if (n.ok()) {
            std::vector<ncclComm_t> comms(ndev);
            const ncclResult_t r = n.init_all(comms.data(), ndev, devs.data());
            if (r != ncclSuccess) {
                rc = fail(KOHLER_CUDA_ERROR, std::string("ncclCommInitAll: ") + n.err(r));
            } else {
                for (int i = 0; i < ndev; ++i)
                    g->m[i].comm = comms[i];
                g->use_nccl = true;
            }
        } else if (ndev > 1) {
            rc = fail(KOHLER_CUDA_ERROR, "multi: NCCL (libnccl.so.2) not loadable; a group of "
                                          "more than one device needs it");
        }
    }
    if (rc != KOHLER_OK) {
        const std::string keep = g_last_error;
        kohler_cuda_multi_destroy(g);
        g_last_error = keep;
        return rc;
    }
    *out = g;
    return KOHLER_OK;
}

void kohler_cuda_multi_destroy(kohler_cuda_multi* g)
{
    if (!g)
        return;
    for (Member& m : g->m) {
        cudaSetDevice(m.device);
        if (m.comm && nccl().ok())
            nccl().destroy(m.comm);
        if (m.stream)
            cudaStreamSynchronize(m.stream);
        cudaFree(m.band);
        cudaFree(m.part);
        cudaFree(m.values);
        cudaFree(m.defined);
        cudaFree(m.ints);
        if (m.ev)
            cudaEventDestroy(m.ev);
        if (m.stream)
            cudaStreamDestroy(m.stream);
        if (m.ctx)
            kohler_cuda_destroy(m.ctx);
    }
    delete g;
}

int kohler_cuda_multi_size(const kohler_cuda_multi* g) { return g ? (int)g->m.size() : 0; }

int kohler_cuda_multi_uses_nccl(const kohler_cuda_multi* g) { return g && g->use_nccl ? 1 : 0; }

int kohler_cuda_multi_uses_peer(const kohler_cuda_multi* g) { return g && g->peer ? 1 : 0; }

int kohler_cuda_multi_curve(kohler_cuda_multi* g, const uint8_t* px, int w, int h, size_t pitch,
                            uint64_t* sum, uint64_t* card)
{
    if (!g)
        return fail(KOHLER_INVALID_ARGUMENT, "multi: null group");
    if (int rc = check_image(px, w, h, pitch))
        return rc;
    std::lock_guard<std::mutex> lk(g->mu);
    g_last_error.clear();
    int rc;
    if (g->peer) {
        rc = peer_image(g, px, w, h, pitch, 1, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    } else {
        rc = for_members(g, [&](int b) { return band_step(g, b, px, w, h, pitch); });
        if (rc == KOHLER_OK)
            rc = merge_without_nccl(g);
    }
    if (rc)
        return rc;
    Member& m0 = g->m[0];
    MC(cudaSetDevice(m0.device));
    if (sum)
        MC(cudaMemcpy(sum, m0.part, 256 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    if (card)
        MC(cudaMemcpy(card, m0.part + 256, 256 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return KOHLER_OK;
}

int kohler_cuda_multi_analyze(kohler_cuda_multi* g, const uint8_t* px, int w, int h, size_t pitch,
                              int k, uint64_t* sum, uint64_t* card, double* values,
                              uint8_t* defined, int* t0, int* topk, int* topk_count)
{
    if (!g)
        return fail(KOHLER_INVALID_ARGUMENT, "multi: null group");
    if (k < 1)
        return fail(KOHLER_INVALID_ARGUMENT, "multi: k must be at least 1");
    if (int rc = check_image(px, w, h, pitch))
        return rc;
    std::lock_guard<std::mutex> lk(g->mu);
    g_last_error.clear();
    Member& m0 = g->m[0];
    MC(cudaSetDevice(m0.device));
    const int kk = std::min(k, KOHLER_LEVELS);  // more maxima than levels cannot exist
    if (!m0.values) {
        MC(cudaMalloc(&m0.values, 256 * sizeof(double)));
        MC(cudaMalloc(&m0.defined, 256));
    }
    if (m0.ints_cap < 3 + kk) {
        cudaFree(m0.ints);
        m0.ints = nullptr;
        MC(cudaMalloc(&m0.ints, (3 + kk) * sizeof(int)));
        m0.ints_cap = 3 + kk;
    }
    int rc;
    if (g->peer) {
        // K3 + K4 in the one finish_kernel behind the members' flushes
        rc = peer_image(g, px, w, h, pitch, kk, 1, m0.values, m0.defined, m0.ints, m0.ints + 3,
                        m0.ints + 1, m0.ints + 2);
        if (rc)
            return rc;
    } else {
        rc = for_members(g, [&](int b) { return band_step(g, b, px, w, h, pitch); });
        if (rc == KOHLER_OK)
            rc = merge_without_nccl(g);
        if (rc)
            return rc;
        // selection on the merged curve, on the first device (K4)
        MC(cudaSetDevice(m0.device));
        rc = kohler_cuda_select_device(m0.ctx, m0.part, m0.part + 256, 1, 256, kk, m0.values,
                                       m0.defined, m0.ints, m0.ints + 3, m0.ints + 1, m0.ints + 2,
                                       m0.stream);
        if (rc)
            return rc;
        MC(cudaStreamSynchronize(m0.stream));
    }
    MC(cudaSetDevice(m0.device));
    std::vector<int> hi(3 + kk);
    MC(cudaMemcpy(hi.data(), m0.ints, (3 + kk) * sizeof(int), cudaMemcpyDeviceToHost));
    if (sum)
        MC(cudaMemcpy(sum, m0.part, 256 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    if (card)
        MC(cudaMemcpy(card, m0.part + 256, 256 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    if (values)
        MC(cudaMemcpy(values, m0.values, 256 * sizeof(double), cudaMemcpyDeviceToHost));
    if (defined)
        MC(cudaMemcpy(defined, m0.defined, 256, cudaMemcpyDeviceToHost));
    if (t0)
        *t0 = hi[0];
    if (topk_count)
        *topk_count = hi[1];
    if (topk)
        std::memcpy(topk, hi.data() + 3, (size_t)std::max(0, std::min(hi[1], kk)) * sizeof(int));
    return hi[2] ? KOHLER_NO_BOUNDARY : KOHLER_OK;
}

int kohler_cuda_multi_analyze_batch(kohler_cuda_multi* g, const uint8_t* px, int n, int w, int h,
                                    size_t pitch, size_t image_stride, int k, uint64_t* sums,
                                    uint64_t* cards, double* values, uint8_t* defined, int* t0s,
                                    int* topks, int* topk_counts, int* status)
{
    if (!g)
        return fail(KOHLER_INVALID_ARGUMENT, "multi: null group");
    if (n < 0 || (n > 0 && check_image(px, w, h, pitch)))
        return fail(KOHLER_INVALID_ARGUMENT, "multi: bad batch");
    if (n == 0)
        return KOHLER_OK;
    std::lock_guard<std::mutex> lk(g->mu);
    g_last_error.clear();
    const int B = (int)g->m.size();
    return for_members(g, [&](int b) -> int {
        // contiguous shards [n*b/B, n*(b+1)/B) (paper_1707_05062_b200/shard.py)
        const int i0 = (int)((long long)n * b / B), i1 = (int)((long long)n * (b + 1) / B);
        if (i1 <= i0)
            return KOHLER_OK;
        auto off = [&](auto* p, size_t per) { return p ? p + (size_t)i0 * per : p; };
        return kohler_cuda_analyze_batch(g->m[b].ctx, px + (size_t)i0 * image_stride, i1 - i0, w, h,
                                         pitch, image_stride, k, off(sums, 256), off(cards, 256),
                                         off(values, 256), off(defined, 256), off(t0s, 1),
                                         off(topks, (size_t)k), off(topk_counts, 1), off(status, 1));
    });
}

} // extern "C"
