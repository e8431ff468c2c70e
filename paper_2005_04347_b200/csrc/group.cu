// group.cu -- multi-GPU sharding of the activation sweep.
//
// A network's level-synchronous sweep does not split without a per-level
// exchange, so the engine shards what is independent and exchanges only the
// declared outputs at the end (BASELINE.json north_star item 4):
//
//  * batch sharding: every device holds a full layout replica (built on each
//    device concurrently from the same host arrays) and sweeps a contiguous,
//    balanced slice of the input vectors;
//  * population sharding: a contiguous, balanced slice of the networks per
//    device, each with all of its vectors.
//
// Either way device g's inputs, outputs and id-indexed state are contiguous
// slices of the caller's [vector or network]-major arrays, so the gather of
// the outputs is an all-gather in device order: ncclAllGather when every
// device contributes the same count, otherwise a grouped ncclBroadcast per
// device (all-gather-v).  NCCL is loaded at run time (dlopen of libnccl.so.2 --
// inside a PyTorch process this is the library torch already mapped); when it
// is absent, or a group lists one physical device twice (the one-GPU
// functional mode), the gather runs on the copy engines (cudaMemcpyPeerAsync
// into device 0).
//
// Two shapes of the same machinery:
//  * asnn_group_*: one process driving G devices (ncclCommInitAll);
//  * asnn_comm_unique_id / asnn_dev_comm_init / asnn_dev_allgather: one process
//    per device under a launcher (torchrun), ncclCommInitRank, the gather
//    enqueued on the engine's stream right after the sweep.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "engine.hpp"

using namespace asnn_b200;

namespace {

// ---- NCCL, resolved at run time ---------------------------------------------
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        if (const char* off = getenv("ASNN_NCCL"); off && off[0] == '0') {
            a.why = "disabled (ASNN_NCCL=0)";
            return a;
        }
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return a;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            return fn != nullptr;
        };
        a.ok = sym(a.GetUniqueId, "ncclGetUniqueId") && sym(a.CommInitRank, "ncclCommInitRank") &&
               sym(a.CommInitAll, "ncclCommInitAll") && sym(a.CommDestroy, "ncclCommDestroy") &&
               sym(a.AllGather, "ncclAllGather") && sym(a.Broadcast, "ncclBroadcast") &&
               sym(a.GroupStart, "ncclGroupStart") && sym(a.GroupEnd, "ncclGroupEnd") &&
               sym(a.GetErrorString, "ncclGetErrorString");
        if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
        return a;
    }();
    return api;
}

int nccl_fail(asnn_dev* dev, ncclResult_t r, const char* what) {
    return fail(dev, ASNN_E_CUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}

#define NK(dev, expr)                                        \
    do {                                                     \
        ncclResult_t _r = (expr);                            \
        if (_r != ncclSuccess) return nccl_fail(dev, _r, #expr); \
    } while (0)

#define CKD(dev, expr)                                        \
    do {                                                      \
        cudaError_t _e = (expr);                              \
        if (_e != cudaSuccess) return cuda_fail(dev, _e, #expr); \
    } while (0)

// [lo, hi) of n items for part r of `parts`: contiguous and balanced, the
// first n % parts parts one larger (paper_2005_04347_b200/shard.py batch_slice).
void balanced(uint64_t n, uint32_t parts, uint32_t r, uint64_t* lo, uint64_t* hi) {
    const uint64_t base = n / parts, rem = n % parts;
    *lo = r * base + std::min<uint64_t>(r, rem);
    *hi = *lo + base + (r < rem ? 1 : 0);
}

// All-gather-v of contiguous float slices in device order, enqueued on every
// member's stream inside one NCCL group.  send[g] lies at recv[g] + off[g]
// (in place) on each device.
int gather_nccl(asnn_dev* err_dev, const std::vector<asnn_dev*>& devs, const std::vector<float*>& recv,
                const std::vector<uint64_t>& off, const std::vector<uint64_t>& cnt) {
    const auto& N = nccl();
    const size_t G = devs.size();
    bool equal = true;
    for (size_t g = 1; g < cnt.size(); ++g) equal = equal && cnt[g] == cnt[0];
    NK(err_dev, N.GroupStart());
    for (size_t g = 0; g < G; ++g) {
        auto* comm = static_cast<ncclComm_t>(devs[g]->comm);
        const int me = devs[g]->comm_rank;
        if (equal) {
            NK(err_dev, N.AllGather(recv[g] + off[me], recv[g], cnt[0], ncclFloat32, comm, devs[g]->stream));
        } else {
            for (size_t r = 0; r < cnt.size(); ++r)
                NK(err_dev, N.Broadcast(recv[g] + off[r], recv[g] + off[r], cnt[r], ncclFloat32, static_cast<int>(r),
                                        comm, devs[g]->stream));
        }
    }
    NK(err_dev, N.GroupEnd());
    return ASNN_OK;
}

}  // namespace

// ---- one process, G devices ------------------------------------------------------
struct asnn_group {
    std::vector<asnn_dev*> devs;
    bool nccl_comm = false;        // members share an NCCL communicator
    std::string err;
    std::string gather_note;       // why the copy-engine gather is used, if it is
    std::mutex mu;
    std::vector<cudaEvent_t> ev_a, ev_b, ev_done;
};

struct asnn_group_layout {
    asnn_group* grp = nullptr;
    bool population = false;
    std::vector<asnn_dev_layout*> L;           // per device (null: empty population slice)
    uint32_t n_in = 0, n_out = 0, id_bound = 0;  // batch mode: per vector
    // population mode: per device, inputs / outputs / id_bound summed over its networks
    std::vector<uint64_t> pin, pout, pidb;
    std::vector<uint32_t> net_lo, net_hi;
    // resident buffers per device
    std::vector<DevBuf<float>> x, out;
    std::vector<uint64_t> x_cap, out_cap;
    std::vector<DevBuf<float>> state;
    PinnedBuf pin_x, pin_out;
    uint32_t staged_vec = 0;                   // asnn_group_stage_inputs
};

namespace {

int gfail(asnn_group* g, int st, const std::string& m) {
    if (g) g->err = m;
    return st;
}

// The partition of one activation: per device the vectors it sweeps and the
// float offsets / counts of its inputs, outputs and state in the caller's arrays.
struct Shard {
    uint32_t vecs;
    uint64_t x_off, x_cnt, out_off, out_cnt, st_off, st_cnt;
};

std::vector<Shard> partition(const asnn_group_layout* GL, uint32_t n_vec) {
    const uint32_t G = static_cast<uint32_t>(GL->L.size());
    std::vector<Shard> s(G);
    uint64_t xo = 0, oo = 0, so = 0;
    for (uint32_t g = 0; g < G; ++g) {
        Shard& d = s[g];
        if (GL->population) {
            d.vecs = GL->L[g] ? n_vec : 0;
            d.x_cnt = GL->pin[g] * n_vec;
            d.out_cnt = GL->pout[g] * n_vec;
            d.st_cnt = GL->pidb[g] * n_vec;
        } else {
            uint64_t lo, hi;
            balanced(n_vec, G, g, &lo, &hi);
            d.vecs = static_cast<uint32_t>(hi - lo);
            d.x_cnt = static_cast<uint64_t>(GL->n_in) * d.vecs;
            d.out_cnt = static_cast<uint64_t>(GL->n_out) * d.vecs;
            d.st_cnt = static_cast<uint64_t>(GL->id_bound) * d.vecs;
        }
        d.x_off = xo;
        d.out_off = oo;
        d.st_off = so;
        xo += d.x_cnt;
        oo += d.out_cnt;
        so += d.st_cnt;
    }
    return s;
}

uint64_t total_inputs(const asnn_group_layout* GL, uint32_t n_vec) {
    if (!GL->population) return static_cast<uint64_t>(GL->n_in) * n_vec;
    uint64_t t = 0;
    for (auto v : GL->pin) t += v;
    return t * n_vec;
}

uint64_t total_outputs(const asnn_group_layout* GL, uint32_t n_vec) {
    if (!GL->population) return static_cast<uint64_t>(GL->n_out) * n_vec;
    uint64_t t = 0;
    for (auto v : GL->pout) t += v;
    return t * n_vec;
}

// Runs fn(g) for every device on its own host thread (layout builds are
// blocking calls of seconds on large networks; the devices work concurrently).
template <typename F>
int for_each_device(asnn_group* grp, F fn) {
    const size_t G = grp->devs.size();
    std::vector<int> rc(G, ASNN_OK);
    if (G == 1) {
        rc[0] = fn(0);
    } else {
        std::vector<std::thread> th;
        for (size_t g = 0; g < G; ++g) th.emplace_back([&, g] { rc[g] = fn(g); });
        for (auto& t : th) t.join();
    }
    for (size_t g = 0; g < G; ++g)
        if (rc[g]) return gfail(grp, rc[g], "device " + std::to_string(g) + ": " + grp->devs[g]->err);
    return ASNN_OK;
}

int finish_layout(asnn_group* grp, asnn_group_layout* GL) {
    const size_t G = grp->devs.size();
    GL->x.resize(G);
    GL->out.resize(G);
    GL->state.resize(G);
    GL->x_cap.assign(G, 0);
    GL->out_cap.assign(G, 0);
    if (!GL->population) {
        asnn_layout_info inf{};
        asnn_dev_layout_info(GL->L[0], &inf);
        GL->n_in = inf.n_inputs;
        GL->n_out = inf.n_outputs;
        GL->id_bound = inf.id_bound;
    }
    return ASNN_OK;
}

// Enqueue every device's sweep of its slice (inputs already in GL->x) and the
// gather of the outputs into device 0's GL->out (all devices' with NCCL).
int enqueue_all(asnn_group_layout* GL, const std::vector<Shard>& sh, bool want_state) {
    asnn_group* grp = GL->grp;
    const size_t G = grp->devs.size();
    for (size_t g = 0; g < G; ++g) {
        if (!sh[g].vecs) continue;
        const int rc = enqueue_sweep(GL->L[g], GL->x[g].p, sh[g].vecs, GL->out[g].p + sh[g].out_off,
                                     want_state ? GL->state[g].p : nullptr);
        if (rc) return gfail(grp, rc, "device " + std::to_string(g) + ": " + grp->devs[g]->err);
    }
    if (G == 1) return ASNN_OK;
    std::vector<uint64_t> off(G), cnt(G);
    for (size_t g = 0; g < G; ++g) off[g] = sh[g].out_off, cnt[g] = sh[g].out_cnt;
    if (grp->nccl_comm) {
        std::vector<float*> recv(G);
        for (size_t g = 0; g < G; ++g) recv[g] = GL->out[g].p;
        const int rc = gather_nccl(grp->devs[0], grp->devs, recv, off, cnt);
        if (rc) return gfail(grp, rc, grp->devs[0]->err);
        return ASNN_OK;
    }
    // copy engines: device 0's stream waits for each member, then pulls its slice
    asnn_dev* d0 = grp->devs[0];
    for (size_t g = 1; g < G; ++g) {
        if (!cnt[g]) continue;
        asnn_dev* dg = grp->devs[g];
        CKD(d0, cudaSetDevice(dg->device));
        CKD(d0, cudaEventRecord(grp->ev_done[g], dg->stream));
        CKD(d0, cudaSetDevice(d0->device));
        CKD(d0, cudaStreamWaitEvent(d0->stream, grp->ev_done[g], 0));
        CKD(d0, cudaMemcpyPeerAsync(GL->out[0].p + off[g], d0->device, GL->out[g].p + off[g], dg->device,
                                    cnt[g] * sizeof(float), d0->stream));
    }
    return ASNN_OK;
}

int ensure_buffers(asnn_group_layout* GL, const std::vector<Shard>& sh, uint32_t n_vec, bool want_state) {
    asnn_group* grp = GL->grp;
    const uint64_t out_total = total_outputs(GL, n_vec);
    for (size_t g = 0; g < grp->devs.size(); ++g) {
        asnn_dev* d = grp->devs[g];
        AllocStream on(d->stream);
        CKD(d, cudaSetDevice(d->device));
        if (GL->x_cap[g] < sh[g].x_cnt + 1) {
            CKD(d, GL->x[g].alloc(sh[g].x_cnt + 1));
            GL->x_cap[g] = sh[g].x_cnt + 1;
        }
        if (GL->out_cap[g] < out_total + 1) {
            CKD(d, GL->out[g].alloc(out_total + 1));
            GL->out_cap[g] = out_total + 1;
        }
        if (want_state && GL->state[g].n < sh[g].st_cnt + 1) CKD(d, GL->state[g].alloc(sh[g].st_cnt + 1));
    }
    return ASNN_OK;
}

int stage_x(asnn_group_layout* GL, const std::vector<Shard>& sh, const float* x, uint64_t n_x) {
    asnn_group* grp = GL->grp;
    const float* src = x;
    cudaPointerAttributes a{};
    const bool pinned = cudaPointerGetAttributes(&a, x) == cudaSuccess && a.type == cudaMemoryTypeHost;
    cudaGetLastError();
    if (!pinned && n_x) {
        CKD(grp->devs[0], GL->pin_x.ensure(n_x * sizeof(float)));
        std::memcpy(GL->pin_x.p, x, n_x * sizeof(float));
        src = static_cast<const float*>(GL->pin_x.p);
    }
    for (size_t g = 0; g < grp->devs.size(); ++g) {
        if (!sh[g].x_cnt) continue;
        asnn_dev* d = grp->devs[g];
        CKD(d, cudaSetDevice(d->device));
        CKD(d, cudaMemcpyAsync(GL->x[g].p, src + sh[g].x_off, sh[g].x_cnt * sizeof(float),
                               cudaMemcpyHostToDevice, d->stream));
    }
    return ASNN_OK;
}

int sync_all(asnn_group* grp) {
    for (asnn_dev* d : grp->devs) {
        CKD(d, cudaSetDevice(d->device));
        CKD(d, cudaStreamSynchronize(d->stream));
    }
    return ASNN_OK;
}

}  // namespace

namespace asnn_b200 {
void release_comm(asnn_dev* dev) {
    if (dev && dev->comm && nccl().ok) nccl().CommDestroy(static_cast<ncclComm_t>(dev->comm));
    if (dev) dev->comm = nullptr;
}
}  // namespace asnn_b200

extern "C" {

int asnn_group_open(const int* devices, uint32_t n, asnn_group** out) {
    if (!out || !devices || n == 0) return ASNN_E_INVALID;
    *out = nullptr;
    auto* grp = new asnn_group;
    for (uint32_t g = 0; g < n; ++g) {
        asnn_dev* d = nullptr;
        const int rc = asnn_dev_open(devices[g], &d);
        if (rc) {
            asnn_group_close(grp);
            return rc;
        }
        grp->devs.push_back(d);
    }
    std::vector<int> ids(devices, devices + n);
    std::vector<int> sorted = ids;
    std::sort(sorted.begin(), sorted.end());
    const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    grp->ev_done.assign(n, nullptr);
    for (uint32_t g = 0; g < n; ++g) {
        cudaSetDevice(grp->devs[g]->device);
        cudaEventCreateWithFlags(&grp->ev_done[g], cudaEventDisableTiming);
        cudaEvent_t a = nullptr, b = nullptr;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        grp->ev_a.push_back(a);
        grp->ev_b.push_back(b);
    }
    if (n > 1 && distinct && nccl().ok) {
        std::vector<ncclComm_t> comms(n);
        const ncclResult_t r = nccl().CommInitAll(comms.data(), static_cast<int>(n), ids.data());
        if (r == ncclSuccess) {
            for (uint32_t g = 0; g < n; ++g) {
                grp->devs[g]->comm = comms[g];
                grp->devs[g]->comm_rank = static_cast<int>(g);
                grp->devs[g]->comm_size = static_cast<int>(n);
            }
            grp->nccl_comm = true;
        } else {
            grp->gather_note = std::string("ncclCommInitAll failed: ") + nccl().GetErrorString(r);
        }
    } else if (n > 1) {
        grp->gather_note = !distinct ? "a device is listed twice (one-GPU functional mode)" : nccl().why;
    }
    // peer access for the copy-engine gather (no-op on one physical device)
    if (!grp->nccl_comm)
        for (uint32_t g = 1; g < n; ++g)
            if (ids[g] != ids[0]) {
                cudaSetDevice(ids[0]);
                cudaDeviceEnablePeerAccess(ids[g], 0);
                cudaGetLastError();
            }
    *out = grp;
    return ASNN_OK;
}

void asnn_group_close(asnn_group* grp) {
    if (!grp) return;
    for (size_t g = 0; g < grp->devs.size(); ++g) {
        cudaSetDevice(grp->devs[g]->device);
        if (g < grp->ev_done.size() && grp->ev_done[g]) cudaEventDestroy(grp->ev_done[g]);
        if (g < grp->ev_a.size() && grp->ev_a[g]) cudaEventDestroy(grp->ev_a[g]);
        if (g < grp->ev_b.size() && grp->ev_b[g]) cudaEventDestroy(grp->ev_b[g]);
    }
    for (asnn_dev* d : grp->devs) asnn_dev_close(d);
    delete grp;
}

const char* asnn_group_last_error(const asnn_group* grp) {
    if (!grp) return "";
    if (!grp->err.empty()) return grp->err.c_str();
    for (const asnn_dev* d : grp->devs)
        if (!d->err.empty()) return d->err.c_str();
    return "";
}

int asnn_group_info(const asnn_group* grp, uint32_t* n_devices, uint32_t* gather_kind) {
    if (!grp) return ASNN_E_INVALID;
    if (n_devices) *n_devices = static_cast<uint32_t>(grp->devs.size());
    if (gather_kind) *gather_kind = grp->devs.size() == 1 ? 0u : grp->nccl_comm ? 1u : 2u;
    return ASNN_OK;
}

const char* asnn_group_gather_note(const asnn_group* grp) { return grp ? grp->gather_note.c_str() : ""; }

asnn_dev* asnn_group_device(asnn_group* grp, uint32_t i) {
    return grp && i < grp->devs.size() ? grp->devs[i] : nullptr;
}

int asnn_group_build_layout(asnn_group* grp, const asnn_network_desc* net, asnn_group_layout** out) {
    if (!grp || !net || !out) return ASNN_E_INVALID;
    std::lock_guard<std::mutex> lk(grp->mu);
    *out = nullptr;
    auto* GL = new asnn_group_layout;
    GL->grp = grp;
    GL->L.assign(grp->devs.size(), nullptr);
    int rc = for_each_device(grp, [&](size_t g) { return asnn_dev_build_layout(grp->devs[g], net, &GL->L[g]); });
    if (!rc) rc = finish_layout(grp, GL);
    if (rc) {
        asnn_group_free_layout(GL);
        return rc;
    }
    *out = GL;
    return ASNN_OK;
}

int asnn_group_upload_layout(asnn_group* grp, const asnn_layout_desc* d, asnn_group_layout** out) {
    if (!grp || !d || !out) return ASNN_E_INVALID;
    std::lock_guard<std::mutex> lk(grp->mu);
    *out = nullptr;
    auto* GL = new asnn_group_layout;
    GL->grp = grp;
    GL->L.assign(grp->devs.size(), nullptr);
    int rc = for_each_device(grp, [&](size_t g) { return asnn_dev_upload_layout(grp->devs[g], d, &GL->L[g]); });
    if (!rc) rc = finish_layout(grp, GL);
    if (rc) {
        asnn_group_free_layout(GL);
        return rc;
    }
    *out = GL;
    return ASNN_OK;
}

int asnn_group_build_population(asnn_group* grp, uint32_t n_networks, const asnn_network_desc* nets,
                                asnn_group_layout** out) {
    if (!grp || (!nets && n_networks) || !out) return ASNN_E_INVALID;
    std::lock_guard<std::mutex> lk(grp->mu);
    *out = nullptr;
    const uint32_t G = static_cast<uint32_t>(grp->devs.size());
    auto* GL = new asnn_group_layout;
    GL->grp = grp;
    GL->population = true;
    GL->L.assign(G, nullptr);
    GL->pin.assign(G, 0);
    GL->pout.assign(G, 0);
    GL->pidb.assign(G, 0);
    GL->net_lo.assign(G, 0);
    GL->net_hi.assign(G, 0);
    for (uint32_t g = 0; g < G; ++g) {
        uint64_t lo, hi;
        balanced(n_networks, G, g, &lo, &hi);
        GL->net_lo[g] = static_cast<uint32_t>(lo);
        GL->net_hi[g] = static_cast<uint32_t>(hi);
    }
    int rc = for_each_device(grp, [&](size_t g) {
        const uint32_t cnt = GL->net_hi[g] - GL->net_lo[g];
        if (!cnt) return static_cast<int>(ASNN_OK);
        return asnn_dev_build_population(grp->devs[g], cnt, nets + GL->net_lo[g], &GL->L[g]);
    });
    if (!rc) {
        for (uint32_t g = 0; g < G; ++g) {
            if (!GL->L[g]) continue;
            for (uint32_t k = 0; k < GL->net_hi[g] - GL->net_lo[g]; ++k) {
                asnn_layout_info inf{};
                asnn_dev_network_info(GL->L[g], k, &inf);
                GL->pin[g] += inf.n_inputs;
                GL->pout[g] += inf.n_outputs;
                GL->pidb[g] += inf.id_bound;
            }
        }
        rc = finish_layout(grp, GL);
    }
    if (rc) {
        asnn_group_free_layout(GL);
        return rc;
    }
    *out = GL;
    return ASNN_OK;
}

int asnn_group_layout_member(const asnn_group_layout* GL, uint32_t i, asnn_dev_layout** member) {
    if (!GL || !member || i >= GL->L.size()) return ASNN_E_INVALID;
    *member = GL->L[i];
    return ASNN_OK;
}

int asnn_group_shard(const asnn_group_layout* GL, uint32_t i, uint32_t n_vec, uint32_t* vecs, uint64_t* x_off,
                     uint64_t* x_count, uint64_t* out_off, uint64_t* out_count) {
    if (!GL || i >= GL->L.size()) return ASNN_E_INVALID;
    const Shard s = partition(GL, n_vec)[i];
    if (vecs) *vecs = s.vecs;
    if (x_off) *x_off = s.x_off;
    if (x_count) *x_count = s.x_cnt;
    if (out_off) *out_off = s.out_off;
    if (out_count) *out_count = s.out_cnt;
    return ASNN_OK;
}

int asnn_group_activate(asnn_group_layout* GL, const float* x, uint32_t n_vec, uint64_t n_x, float* out,
                        float* state) {
    if (!GL) return ASNN_E_INVALID;
    asnn_group* grp = GL->grp;
    std::lock_guard<std::mutex> lk(grp->mu);
    grp->err.clear();
    for (asnn_dev* d : grp->devs) d->err.clear();
    const uint64_t want = total_inputs(GL, n_vec);
    if (n_x != want)
        return gfail(grp, ASNN_E_ARITY,
                     "expected " + std::to_string(want) + " input values, got " + std::to_string(n_x));
    if (n_vec == 0) return ASNN_OK;
    if (!x && n_x) return gfail(grp, ASNN_E_INVALID, "null input");
    const auto sh = partition(GL, n_vec);
    int rc = ensure_buffers(GL, sh, n_vec, state != nullptr);
    if (!rc) rc = stage_x(GL, sh, x, n_x);
    if (!rc) rc = enqueue_all(GL, sh, state != nullptr);
    if (rc) return rc;
    asnn_dev* d0 = grp->devs[0];
    const uint64_t ob = total_outputs(GL, n_vec) * sizeof(float);
    bool staged = false;
    if (out && ob) {
        CKD(d0, cudaSetDevice(d0->device));
        cudaPointerAttributes a{};
        const bool pinned = cudaPointerGetAttributes(&a, out) == cudaSuccess && a.type == cudaMemoryTypeHost;
        cudaGetLastError();
        if (pinned) {
            CKD(d0, cudaMemcpyAsync(out, GL->out[0].p, ob, cudaMemcpyDeviceToHost, d0->stream));
        } else {
            CKD(d0, GL->pin_out.ensure(ob));
            CKD(d0, cudaMemcpyAsync(GL->pin_out.p, GL->out[0].p, ob, cudaMemcpyDeviceToHost, d0->stream));
            staged = true;
        }
    }
    if (state)
        for (size_t g = 0; g < grp->devs.size(); ++g) {
            if (!sh[g].st_cnt) continue;
            asnn_dev* d = grp->devs[g];
            CKD(d, cudaSetDevice(d->device));
            CKD(d, cudaMemcpyAsync(state + sh[g].st_off, GL->state[g].p, sh[g].st_cnt * sizeof(float),
                                   cudaMemcpyDeviceToHost, d->stream));
        }
    rc = sync_all(grp);
    if (rc) return gfail(grp, rc, grp->devs[0]->err);
    if (staged) std::memcpy(out, GL->pin_out.p, ob);
    return ASNN_OK;
}

int asnn_group_stage_inputs(asnn_group_layout* GL, const float* x, uint32_t n_vec, uint64_t n_x) {
    if (!GL) return ASNN_E_INVALID;
    asnn_group* grp = GL->grp;
    std::lock_guard<std::mutex> lk(grp->mu);
    if (n_x != total_inputs(GL, n_vec)) return gfail(grp, ASNN_E_ARITY, "input count does not match n_vec");
    const auto sh = partition(GL, n_vec);
    int rc = ensure_buffers(GL, sh, n_vec, false);
    if (!rc) rc = stage_x(GL, sh, x, n_x);
    if (!rc) rc = sync_all(grp);
    if (rc) return rc;
    GL->staged_vec = n_vec;
    return ASNN_OK;
}

int asnn_group_sweep(asnn_group_layout* GL, uint32_t repeats, float* ms) {
    if (!GL || !GL->staged_vec) return ASNN_E_INVALID;
    asnn_group* grp = GL->grp;
    std::lock_guard<std::mutex> lk(grp->mu);
    const auto sh = partition(GL, GL->staged_vec);
    int rc = sync_all(grp);
    if (rc) return rc;
    const size_t G = grp->devs.size();
    for (size_t g = 0; g < G; ++g) {
        cudaSetDevice(grp->devs[g]->device);
        cudaEventRecord(grp->ev_a[g], grp->devs[g]->stream);
    }
    for (uint32_t r = 0; r < std::max(1u, repeats); ++r) {
        rc = enqueue_all(GL, sh, false);
        if (rc) return rc;
    }
    for (size_t g = 0; g < G; ++g) {
        cudaSetDevice(grp->devs[g]->device);
        cudaEventRecord(grp->ev_b[g], grp->devs[g]->stream);
    }
    rc = sync_all(grp);
    if (rc) return rc;
    float worst = 0.0f;
    for (size_t g = 0; g < G; ++g) {
        float t = 0.0f;
        cudaSetDevice(grp->devs[g]->device);
        cudaEventElapsedTime(&t, grp->ev_a[g], grp->ev_b[g]);
        worst = std::max(worst, t);
    }
    if (ms) *ms = worst / std::max(1u, repeats);
    return ASNN_OK;
}

int asnn_group_read_outputs(asnn_group_layout* GL, float* out) {
    if (!GL || !out || !GL->staged_vec) return ASNN_E_INVALID;
    asnn_group* grp = GL->grp;
    std::lock_guard<std::mutex> lk(grp->mu);
    asnn_dev* d0 = grp->devs[0];
    CKD(d0, cudaSetDevice(d0->device));
    CKD(d0, cudaMemcpy(out, GL->out[0].p, total_outputs(GL, GL->staged_vec) * sizeof(float),
                       cudaMemcpyDeviceToHost));
    return ASNN_OK;
}

void asnn_group_free_layout(asnn_group_layout* GL) {
    if (!GL) return;
    asnn_group* grp = GL->grp;
    sync_all(grp);
    for (size_t g = 0; g < GL->L.size(); ++g) {
        asnn_dev* d = grp->devs[g];
        cudaSetDevice(d->device);
        {
            AllocStream on(d->stream);
            if (g < GL->x.size()) GL->x[g].reset();
            if (g < GL->out.size()) GL->out[g].reset();
            if (g < GL->state.size()) GL->state[g].reset();
        }
        if (GL->L[g]) asnn_dev_free_layout(GL->L[g]);
    }
    delete GL;
}

// ---- one process per device (torchrun) ----------------------------------------
int asnn_comm_unique_id(uint8_t* id) {
    if (!id) return ASNN_E_INVALID;
    if (!nccl().ok) return ASNN_E_UNAVAILABLE;
    ncclUniqueId u;
    if (nccl().GetUniqueId(&u) != ncclSuccess) return ASNN_E_UNAVAILABLE;
    static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, &u, sizeof(u));
    return ASNN_OK;
}

int asnn_dev_comm_init(asnn_dev* dev, const uint8_t* id, int n_ranks, int rank) {
    if (!dev || !id || n_ranks < 1 || rank < 0 || rank >= n_ranks) return ASNN_E_INVALID;
    if (!nccl().ok) return fail(dev, ASNN_E_UNAVAILABLE, "NCCL " + nccl().why);
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    release_comm(dev);
    CKD(dev, cudaSetDevice(dev->device));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    ncclComm_t c = nullptr;
    NK(dev, nccl().CommInitRank(&c, n_ranks, u, rank));
    dev->comm = c;
    dev->comm_rank = rank;
    dev->comm_size = n_ranks;
    return ASNN_OK;
}

int asnn_dev_allgather(asnn_dev* dev, const float* send_dev, float* recv_dev, const uint64_t* counts) {
    if (!dev || !recv_dev || !counts) return ASNN_E_INVALID;
    std::lock_guard<std::recursive_mutex> lk(dev->mu);
    if (!dev->comm) return fail(dev, ASNN_E_INVALID, "no communicator (asnn_dev_comm_init)");
    CKD(dev, cudaSetDevice(dev->device));
    const int n = dev->comm_size;
    std::vector<uint64_t> off(n), cnt(counts, counts + n);
    uint64_t o = 0;
    for (int r = 0; r < n; ++r) off[r] = o, o += cnt[r];
    float* mine = recv_dev + off[dev->comm_rank];
    if (send_dev != mine && cnt[dev->comm_rank])
        CKD(dev, cudaMemcpyAsync(mine, send_dev, cnt[dev->comm_rank] * sizeof(float), cudaMemcpyDeviceToDevice,
                                 dev->stream));
    std::vector<asnn_dev*> one{dev};
    std::vector<float*> recv{recv_dev};
    return gather_nccl(dev, one, recv, off, cnt);
}

}  // extern "C"
