// comm.cu -- the exchange layer under dist.cu (§III-D: ghost exchange, per-iteration
// refresh + allreduce, label merge).  Two transports behind one interface:
//   * NCCL: one process per GPU (the production path; NVLink / NVSwitch), and
//   * an in-process "virtual rank" group: R contexts of ONE process share one GPU, each driven by
//     its own host thread and stream.  Every collective call is
//     matched across the R threads by a host barrier; data moves as device-to-device copies and
//     reduction kernels ordered by CUDA events -- no kernel ever waits on another rank's kernel
//     (which would need co-scheduling on one GPU), so the multi-rank protocol of dist.cu can be
//     run and checked bit for bit against one rank on a single-GPU box.
// Semantics follow NCCL's: sends and receives between a pair of ranks match in issue order
// inside a group; an allreduce / allgather may share a group with point-to-point operations.
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "cc_internal.cuh"

namespace cc {

struct VOp {
    int kind;  // 0 send, 1 recv, 2 allreduce, 3 allgather
    const void* src;
    void* dst;
    size_t bytes;  // send/recv: payload; allreduce: count * elem; allgather: bytes per rank
    size_t count;
    int peer;
    int type, op;
};

struct VRank {
    std::vector<VOp> ops;
    cudaEvent_t ready = nullptr, done = nullptr;
    cudaStream_t stream = nullptr;
    void* scratch = nullptr;
    size_t scratch_cap = 0;
};

struct VGroup {
    int n = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long gen = 0;
    std::vector<VRank*> st;
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const unsigned long long g = gen;
        if (++arrived == n) {
            arrived = 0;
            gen++;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

namespace {

#define CC_NCCL(c, expr)                                                                          \
    do {                                                                                          \
        ncclResult_t r_ = (expr);                                                                 \
        if (r_ != ncclSuccess) return cc_fail((c), CC_E_NCCL, std::string(ncclGetErrorString(r_)) + " at " #expr); \
    } while (0)

inline ncclComm_t comm(cc_ctx* c) { return static_cast<ncclComm_t>(c->nccl_comm); }

ncclDataType_t nccl_type(int t) {
    switch (t) {
        case CT_U8: return ncclUint8;
        case CT_I32: return ncclInt32;
        case CT_U32: return ncclUint32;
        case CT_I64: return ncclInt64;
        case CT_U64: return ncclUint64;
        case CT_F32: return ncclFloat32;
        default: return ncclFloat64;
    }
}

size_t type_bytes(int t) {
    switch (t) {
        case CT_U8: return 1;
        case CT_I32: case CT_U32: case CT_F32: return 4;
        default: return 8;
    }
}

struct Ptrs {
    const void* p[8];
};

// out[i] = in_0[i] op in_1[i] op ... in rank order (deterministic for floating point too)
template <typename T>
__global__ void k_vreduce(T* out, Ptrs in, int n, size_t count, int op) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
        T v = static_cast<const T*>(in.p[0])[i];
        for (int r = 1; r < n; r++) {
            const T w = static_cast<const T*>(in.p[r])[i];
            v = op == CO_MIN ? (w < v ? w : v) : (T)(v + w);
        }
        out[i] = v;
    }
}

template <typename T>
void launch_reduce(cc_ctx* c, void* out, const Ptrs& in, int n, size_t count, int op) {
    const unsigned nb = (unsigned)std::min<size_t>((count + 255) / 256, 1024);
    CCL(c, k_vreduce<T><<<std::max(nb, 1u), 256, 0, c->stream>>>(static_cast<T*>(out), in, n, count, op));
}

cc_status reduce_into(cc_ctx* c, int type, void* out, const Ptrs& in, int n, size_t count, int op) {
    switch (type) {
        case CT_I32: launch_reduce<int>(c, out, in, n, count, op); break;
        case CT_U32: launch_reduce<unsigned int>(c, out, in, n, count, op); break;
        case CT_I64: launch_reduce<long long>(c, out, in, n, count, op); break;
        case CT_U64: launch_reduce<unsigned long long>(c, out, in, n, count, op); break;
        case CT_F32: launch_reduce<float>(c, out, in, n, count, op); break;
        case CT_F64: launch_reduce<double>(c, out, in, n, count, op); break;
        default: return cc_fail(c, CC_E_ARG, "virtual allreduce: unsupported type");
    }
    CC_CUDA(c, cudaGetLastError());
    return CC_OK;
}

// execute this rank's queued operations together with the other ranks' (all ranks call it for
// the same group)
cc_status vexec(cc_ctx* c) {
    VGroup* g = static_cast<VGroup*>(c->vgroup);
    VRank* me = g->st[(size_t)c->rank];
    const int R = g->n;
    CC_CUDA(c, cudaEventRecord(me->ready, c->stream));
    // allreduce results go to scratch first (peers read the inputs until the second barrier)
    size_t need = 0;
    for (auto& o : me->ops)
        if (o.kind == 2) need += (o.bytes + 255) / 256 * 256;
    if (need > me->scratch_cap) {
        if (me->scratch) cudaFree(me->scratch);
        me->scratch = nullptr;
        me->scratch_cap = 0;
        CC_CUDA(c, cudaMalloc(&me->scratch, need));
        me->scratch_cap = need;
    }
    g->barrier();  // every rank's ops and ready event are published
    for (int r = 0; r < R; r++)
        if (r != c->rank) CC_CUDA(c, cudaStreamWaitEvent(c->stream, g->st[(size_t)r]->ready, 0));
    std::vector<int> nrecv((size_t)R, 0);
    int nar = 0, nag = 0;
    size_t soff = 0;
    for (auto& o : me->ops) {
        if (o.kind == 1) {  // the k-th receive from P matches P's k-th send to me
            const VRank* pr = g->st[(size_t)o.peer];
            int k = nrecv[(size_t)o.peer]++, seen = 0;
            const VOp* src = nullptr;
            for (auto& q : pr->ops)
                if (q.kind == 0 && q.peer == c->rank && seen++ == k) {
                    src = &q;
                    break;
                }
            if (!src || src->bytes != o.bytes) return cc_fail(c, CC_E_NCCL, "virtual ranks: unmatched send/recv");
            if (o.bytes) CC_CUDA(c, cudaMemcpyAsync(o.dst, src->src, o.bytes, cudaMemcpyDeviceToDevice, c->stream));
        } else if (o.kind == 2) {
            Ptrs in{};
            for (int r = 0; r < R; r++) {
                int seen = 0;
                const VOp* q = nullptr;
                for (auto& x : g->st[(size_t)r]->ops)
                    if (x.kind == 2 && seen++ == nar) {
                        q = &x;
                        break;
                    }
                if (!q || q->count != o.count) return cc_fail(c, CC_E_NCCL, "virtual ranks: unmatched allreduce");
                in.p[r] = q->src;
            }
            CC_TRY(reduce_into(c, o.type, static_cast<unsigned char*>(me->scratch) + soff, in, R, o.count, o.op));
            soff += (o.bytes + 255) / 256 * 256;
            nar++;
        } else if (o.kind == 3) {
            for (int r = 0; r < R; r++) {
                int seen = 0;
                const VOp* q = nullptr;
                for (auto& x : g->st[(size_t)r]->ops)
                    if (x.kind == 3 && seen++ == nag) {
                        q = &x;
                        break;
                    }
                if (!q || q->bytes != o.bytes) return cc_fail(c, CC_E_NCCL, "virtual ranks: unmatched allgather");
                CC_CUDA(c, cudaMemcpyAsync(static_cast<unsigned char*>(o.dst) + (size_t)r * o.bytes, q->src, o.bytes,
                                           cudaMemcpyDeviceToDevice, c->stream));
            }
            nag++;
        }
    }
    CC_CUDA(c, cudaEventRecord(me->done, c->stream));
    g->barrier();  // every rank has enqueued its reads of my buffers
    for (int r = 0; r < R; r++)
        if (r != c->rank) CC_CUDA(c, cudaStreamWaitEvent(c->stream, g->st[(size_t)r]->done, 0));
    soff = 0;
    for (auto& o : me->ops)
        if (o.kind == 2) {
            CC_CUDA(c, cudaMemcpyAsync(o.dst, static_cast<unsigned char*>(me->scratch) + soff, o.bytes,
                                       cudaMemcpyDeviceToDevice, c->stream));
            soff += (o.bytes + 255) / 256 * 256;
        }
    me->ops.clear();
    g->barrier();  // nobody re-records ready/done of this group before all waits are enqueued
    return CC_OK;
}

cc_status vqueue(cc_ctx* c, const VOp& o) {
    VGroup* g = static_cast<VGroup*>(c->vgroup);
    g->st[(size_t)c->rank]->ops.push_back(o);
    if (c->comm_depth == 0) return vexec(c);  // outside a group: a group of one
    return CC_OK;
}

}  // namespace

cc_status comm_init(cc_ctx* c, const cc_dist* d) {
    if (d->vgroup) {
        VGroup* g = static_cast<VGroup*>(d->vgroup);
        if (g->n != d->nranks) return cc_fail(c, CC_E_ARG, "virtual group size != nranks");
        VRank* me = new VRank();
        me->stream = c->stream;
        if (cudaEventCreateWithFlags(&me->ready, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&me->done, cudaEventDisableTiming) != cudaSuccess) {
            delete me;
            return cc_fail(c, CC_E_CUDA, "virtual rank events");
        }
        {
            std::lock_guard<std::mutex> lk(g->mu);
            g->st[(size_t)d->rank] = me;
        }
        c->vgroup = g;
        g->barrier();  // every rank registered
        return CC_OK;
    }
    if (!d->nccl_id_h) return cc_fail(c, CC_E_ARG, "cc_dist: nccl_id_h (or vgroup) required");
    ncclUniqueId id;
    std::memcpy(&id, d->nccl_id_h, sizeof(id));
    ncclComm_t cm;
    CC_NCCL(c, ncclCommInitRank(&cm, d->nranks, id, d->rank));
    c->nccl_comm = cm;
    return CC_OK;
}

void comm_destroy(cc_ctx* c) {
    if (c->vgroup) {
        VGroup* g = static_cast<VGroup*>(c->vgroup);
        VRank* me = g->st[(size_t)c->rank];
        g->barrier();  // no rank still reads my buffers
        if (me) {
            if (me->ready) cudaEventDestroy(me->ready);
            if (me->done) cudaEventDestroy(me->done);
            if (me->scratch) cudaFree(me->scratch);
            delete me;
        }
        g->st[(size_t)c->rank] = nullptr;
        c->vgroup = nullptr;
        return;
    }
    if (c->nccl_comm) ncclCommDestroy(comm(c));
    c->nccl_comm = nullptr;
}

cc_status comm_group_start(cc_ctx* c) {
    if (c->vgroup) {
        c->comm_depth++;
        return CC_OK;
    }
    CC_NCCL(c, ncclGroupStart());
    return CC_OK;
}

cc_status comm_group_end(cc_ctx* c) {
    if (c->vgroup) {
        if (--c->comm_depth == 0) return vexec(c);
        return CC_OK;
    }
    CC_NCCL(c, ncclGroupEnd());
    return CC_OK;
}

cc_status comm_send(cc_ctx* c, const void* buf, size_t count, int type, int peer) {
    if (c->vgroup) return vqueue(c, VOp{0, buf, nullptr, count * type_bytes(type), count, peer, type, 0});
    CC_NCCL(c, ncclSend(buf, count, nccl_type(type), peer, comm(c), c->stream));
    return CC_OK;
}

cc_status comm_recv(cc_ctx* c, void* buf, size_t count, int type, int peer) {
    if (c->vgroup) return vqueue(c, VOp{1, nullptr, buf, count * type_bytes(type), count, peer, type, 0});
    CC_NCCL(c, ncclRecv(buf, count, nccl_type(type), peer, comm(c), c->stream));
    return CC_OK;
}

cc_status comm_allreduce(cc_ctx* c, void* buf, size_t count, int type, int op) {
    if (c->vgroup) return vqueue(c, VOp{2, buf, buf, count * type_bytes(type), count, 0, type, op});
    CC_NCCL(c, ncclAllReduce(buf, buf, count, nccl_type(type), op == CO_MIN ? ncclMin : ncclSum, comm(c), c->stream));
    return CC_OK;
}

cc_status comm_allgather(cc_ctx* c, const void* send, void* recv, size_t count, int type) {
    if (c->vgroup) return vqueue(c, VOp{3, send, recv, count * type_bytes(type), count, 0, type, 0});
    CC_NCCL(c, ncclAllGather(send, recv, count, nccl_type(type), comm(c), c->stream));
    return CC_OK;
}

}  // namespace cc

extern "C" {

cc_status cc_vgroup_create(int nranks, void** group_h) {
    if (!group_h || nranks < 1 || nranks > 8) return CC_E_ARG;
    cc::VGroup* g = new cc::VGroup();
    g->n = nranks;
    g->st.assign((size_t)nranks, nullptr);
    *group_h = g;
    return CC_OK;
}

void cc_vgroup_destroy(void* group) { delete static_cast<cc::VGroup*>(group); }

}  // extern "C"
