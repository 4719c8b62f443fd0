// gtcp_comm.cu -- NCCL and loopback transports behind gtcp_comm.cuh.
#include <algorithm>
#include <condition_variable>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <utility>
#include <vector>

#include "gtcp_internal.cuh"

namespace gtcp {

static size_t type_size(ncclDataType_t t) {
    switch (t) {
        case ncclInt8: case ncclUint8: return 1;
        case ncclFloat16: return 2;
        case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
        default: return 8;  // ncclInt64, ncclUint64, ncclFloat64
    }
}

static void acct_add(long long* acct, double bytes) {
    if (acct) *acct += (long long)bytes;
}

// ---------------------------------------------------------------------------
// loopback transport
// ---------------------------------------------------------------------------
struct Msg {
    const void* src = nullptr;
    size_t bytes = 0;
    cudaEvent_t ready = nullptr, done = nullptr;
    bool consumed = false;
};

struct Slot {  // one collective call (all members enter with the same sequence number)
    explicit Slot(int n) : ptr(n, nullptr), ready(n, nullptr), done(n, nullptr), color(n, 0), key(n, 0) {}
    int arrived = 0, finished = 0, left = 0;
    std::vector<void*> ptr;
    std::vector<cudaEvent_t> ready, done;
    std::vector<int> color, key;
    std::map<int, LoopShared*> child;
};

struct LoopShared {
    LoopHub* hub = nullptr;
    int size = 0;
    std::map<std::pair<int, int>, std::deque<std::shared_ptr<Msg>>> box;  // (src, dst) FIFO
    std::map<long long, std::shared_ptr<Slot>> slots;
    std::vector<long long> seq;  // next collective sequence number per member
};

struct LoopHub {
    std::mutex mu;
    std::condition_variable cv;
    int nranks = 0;
    std::vector<std::unique_ptr<LoopShared>> comms;  // [0] = world
    LoopShared* make(int size) {
        comms.emplace_back(new LoopShared());
        LoopShared* s = comms.back().get();
        s->hub = this;
        s->size = size;
        s->seq.assign(size, 0);
        return s;
    }
};

LoopHub* loop_hub_create(int nranks) {
    LoopHub* h = new LoopHub();
    h->nranks = nranks;
    h->make(nranks);
    return h;
}
void loop_hub_destroy(LoopHub* h) { delete h; }
int loop_hub_size(const LoopHub* h) { return h ? h->nranks : 0; }
Comm loop_world(LoopHub* h, int rank) {
    Comm c;
    c.ls = h->comms[0].get();
    c.rank = rank;
    c.size = h->nranks;
    return c;
}

// deferred point-to-point operations of the current group (per host thread,
// as NCCL's group state)
struct Pending {
    bool send;
    const Comm* c;
    void* buf;
    size_t bytes;
    int peer;
    cudaStream_t st;
    std::shared_ptr<Msg> msg;
};
static thread_local int t_depth = 0;
static thread_local std::vector<Pending> t_pending;

static ncclResult_t cu2nc(cudaError_t e) { return e == cudaSuccess ? ncclSuccess : ncclUnhandledCudaError; }

static ncclResult_t loop_complete_recv(const Pending& p) {
    LoopShared* s = p.c->ls;
    LoopHub* h = s->hub;
    std::shared_ptr<Msg> m;
    {
        std::unique_lock<std::mutex> lk(h->mu);
        auto& q = s->box[{p.peer, p.c->rank}];
        h->cv.wait(lk, [&] { return !q.empty(); });
        m = q.front();
        q.pop_front();
    }
    if (m->bytes != p.bytes) {  // NCCL: send/recv sizes must match; release the sender, report the misuse
        {
            std::lock_guard<std::mutex> lk(h->mu);
            m->consumed = true;
        }
        h->cv.notify_all();
        return ncclInvalidUsage;
    }
    cudaError_t e = cudaStreamWaitEvent(p.st, m->ready, 0);
    if (e == cudaSuccess && p.bytes) e = cudaMemcpyAsync(p.buf, m->src, p.bytes, cudaMemcpyDeviceToDevice, p.st);
    cudaEvent_t d = nullptr;
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(d, p.st);
    {
        std::lock_guard<std::mutex> lk(h->mu);
        m->done = d;
        m->consumed = true;
    }
    h->cv.notify_all();
    return cu2nc(e);
}

static ncclResult_t loop_complete_send(const Pending& p) {
    LoopHub* h = p.c->ls->hub;
    {
        std::unique_lock<std::mutex> lk(h->mu);
        h->cv.wait(lk, [&] { return p.msg->consumed; });
    }
    cudaError_t e = p.msg->done ? cudaStreamWaitEvent(p.st, p.msg->done, 0) : cudaSuccess;
    cudaEventDestroy(p.msg->ready);
    if (p.msg->done) cudaEventDestroy(p.msg->done);
    return cu2nc(e);
}

static ncclResult_t loop_flush() {
    ncclResult_t r = ncclSuccess;
    // receives first: every peer posted its sends when it issued them, so
    // receiving never waits on a peer that is itself waiting
    for (const Pending& p : t_pending)
        if (!p.send && r == ncclSuccess) r = loop_complete_recv(p);
    for (const Pending& p : t_pending)
        if (p.send) {
            ncclResult_t q = loop_complete_send(p);
            if (r == ncclSuccess) r = q;
        }
    t_pending.clear();
    return r;
}

static ncclResult_t loop_send(const Comm& c, const void* buf, size_t bytes, int peer, cudaStream_t st) {
    auto m = std::make_shared<Msg>();
    m->src = buf;
    m->bytes = bytes;
    cudaError_t e = cudaEventCreateWithFlags(&m->ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(m->ready, st);
    if (e != cudaSuccess) return cu2nc(e);
    LoopHub* h = c.ls->hub;
    {
        std::lock_guard<std::mutex> lk(h->mu);
        c.ls->box[{c.rank, peer}].push_back(m);
    }
    h->cv.notify_all();
    Pending p{true, &c, nullptr, bytes, peer, st, m};
    if (t_depth > 0) {
        t_pending.push_back(p);
        return ncclSuccess;
    }
    return loop_complete_send(p);
}

static ncclResult_t loop_recv(const Comm& c, void* buf, size_t bytes, int peer, cudaStream_t st) {
    Pending p{false, &c, buf, bytes, peer, st, nullptr};
    if (t_depth > 0) {
        t_pending.push_back(p);
        return ncclSuccess;
    }
    return loop_complete_recv(p);
}

static std::shared_ptr<Slot> slot_enter(const Comm& c, long long* seq_out) {
    LoopShared* s = c.ls;
    std::lock_guard<std::mutex> lk(s->hub->mu);
    long long q = s->seq[c.rank]++;
    auto& sp = s->slots[q];
    if (!sp) sp = std::make_shared<Slot>(s->size);
    *seq_out = q;
    return sp;
}

// wait until every member has incremented counter `which` (0 arrived, 1 finished)
static void slot_barrier(const Comm& c, Slot& sl, int which) {
    LoopHub* h = c.ls->hub;
    std::unique_lock<std::mutex> lk(h->mu);
    int& cnt = which == 0 ? sl.arrived : sl.finished;
    cnt++;
    h->cv.notify_all();
    h->cv.wait(lk, [&] { return cnt == c.ls->size; });
}

static void slot_leave(const Comm& c, long long seq, Slot& sl) {
    LoopHub* h = c.ls->hub;
    std::lock_guard<std::mutex> lk(h->mu);
    if (++sl.left == c.ls->size) {
        for (auto e : sl.ready)
            if (e) cudaEventDestroy(e);
        for (auto e : sl.done)
            if (e) cudaEventDestroy(e);
        c.ls->slots.erase(seq);
    }
}

struct PtrPack {
    const void* p[16];
};

template <class T, bool MAX>
__global__ void k_loop_reduce(T* out, PtrPack in, int nin, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        T v = static_cast<const T*>(in.p[0])[i];
        for (int m = 1; m < nin; m++) {
            const T x = static_cast<const T*>(in.p[m])[i];
            v = MAX ? (x > v ? x : v) : v + x;  // member order: identical result on every member
        }
        out[i] = v;
    }
}

static ncclResult_t launch_reduce(void* out, const PtrPack& in, int nin, size_t n, ncclDataType_t ty,
                                  ncclRedOp_t op, cudaStream_t st) {
    if (n == 0) return ncclSuccess;
    const int blocks = (int)std::min<size_t>((n + 255) / 256, 148 * 8);
    const bool mx = op == ncclMax;
    if (op != ncclSum && op != ncclMax) return ncclInvalidArgument;
    switch (ty) {
        case ncclInt64:
            if (mx) k_loop_reduce<long long, true><<<blocks, 256, 0, st>>>((long long*)out, in, nin, n);
            else k_loop_reduce<long long, false><<<blocks, 256, 0, st>>>((long long*)out, in, nin, n);
            break;
        case ncclUint64:
            if (mx) k_loop_reduce<unsigned long long, true><<<blocks, 256, 0, st>>>((unsigned long long*)out, in, nin, n);
            else k_loop_reduce<unsigned long long, false><<<blocks, 256, 0, st>>>((unsigned long long*)out, in, nin, n);
            break;
        case ncclFloat64:
            if (mx) k_loop_reduce<double, true><<<blocks, 256, 0, st>>>((double*)out, in, nin, n);
            else k_loop_reduce<double, false><<<blocks, 256, 0, st>>>((double*)out, in, nin, n);
            break;
        case ncclFloat32:
            if (mx) k_loop_reduce<float, true><<<blocks, 256, 0, st>>>((float*)out, in, nin, n);
            else k_loop_reduce<float, false><<<blocks, 256, 0, st>>>((float*)out, in, nin, n);
            break;
        case ncclInt32:
            if (mx) k_loop_reduce<int, true><<<blocks, 256, 0, st>>>((int*)out, in, nin, n);
            else k_loop_reduce<int, false><<<blocks, 256, 0, st>>>((int*)out, in, nin, n);
            break;
        default: return ncclInvalidArgument;
    }
    g_launches++;
    return cu2nc(cudaGetLastError());
}

static ncclResult_t loop_allreduce(const Comm& c, const void* sbuf, void* rbuf, size_t count, ncclDataType_t ty,
                                   ncclRedOp_t op, cudaStream_t st) {
    const int n = c.ls->size;
    if (n > 16) return ncclInvalidUsage;
    const size_t bytes = count * type_size(ty);
    long long seq;
    std::shared_ptr<Slot> sl = slot_enter(c, &seq);
    // stage my contribution: rbuf may alias sbuf, and every member reads it
    void* stage = nullptr;
    cudaError_t e = cudaMallocAsync(&stage, std::max<size_t>(bytes, 8), st);
    if (e == cudaSuccess && bytes) e = cudaMemcpyAsync(stage, sbuf, bytes, cudaMemcpyDeviceToDevice, st);
    cudaEvent_t rd = nullptr;
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&rd, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(rd, st);
    {
        std::lock_guard<std::mutex> lk(c.ls->hub->mu);
        sl->ptr[c.rank] = stage;
        sl->ready[c.rank] = rd;
    }
    slot_barrier(c, *sl, 0);
    PtrPack pk{};
    for (int m = 0; m < n; m++) {
        pk.p[m] = sl->ptr[m];
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, sl->ready[m], 0);
    }
    ncclResult_t r = e == cudaSuccess ? launch_reduce(rbuf, pk, n, count, ty, op, st) : cu2nc(e);
    cudaEvent_t dn = nullptr;
    if (cudaEventCreateWithFlags(&dn, cudaEventDisableTiming) == cudaSuccess) cudaEventRecord(dn, st);
    {
        std::lock_guard<std::mutex> lk(c.ls->hub->mu);
        sl->done[c.rank] = dn;
    }
    slot_barrier(c, *sl, 1);
    // my staged buffer may be freed once every member's reduction has read it
    for (int m = 0; m < n; m++)
        if (m != c.rank && sl->done[m]) cudaStreamWaitEvent(st, sl->done[m], 0);
    cudaFreeAsync(stage, st);
    slot_leave(c, seq, *sl);
    return r;
}

static ncclResult_t loop_bcast(const Comm& c, const void* sbuf, void* rbuf, size_t count, ncclDataType_t ty, int root,
                               cudaStream_t st) {
    const int n = c.ls->size;
    const size_t bytes = count * type_size(ty);
    long long seq;
    std::shared_ptr<Slot> sl = slot_enter(c, &seq);
    cudaError_t e = cudaSuccess;
    if (c.rank == root) {
        if (rbuf != sbuf && bytes) e = cudaMemcpyAsync(rbuf, sbuf, bytes, cudaMemcpyDeviceToDevice, st);
        cudaEvent_t rd = nullptr;
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&rd, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventRecord(rd, st);
        std::lock_guard<std::mutex> lk(c.ls->hub->mu);
        sl->ptr[root] = const_cast<void*>(sbuf);
        sl->ready[root] = rd;
    }
    slot_barrier(c, *sl, 0);
    if (c.rank != root) {
        e = cudaStreamWaitEvent(st, sl->ready[root], 0);
        if (e == cudaSuccess && bytes) e = cudaMemcpyAsync(rbuf, sl->ptr[root], bytes, cudaMemcpyDeviceToDevice, st);
        cudaEvent_t dn = nullptr;
        if (cudaEventCreateWithFlags(&dn, cudaEventDisableTiming) == cudaSuccess) cudaEventRecord(dn, st);
        std::lock_guard<std::mutex> lk(c.ls->hub->mu);
        sl->done[c.rank] = dn;
    }
    slot_barrier(c, *sl, 1);
    if (c.rank == root)  // the root's buffer stays untouched until every member copied it
        for (int m = 0; m < n; m++)
            if (m != root && sl->done[m]) cudaStreamWaitEvent(st, sl->done[m], 0);
    slot_leave(c, seq, *sl);
    return cu2nc(e);
}

static ncclResult_t loop_split(const Comm& parent, int color, int key, Comm* out) {
    long long seq;
    std::shared_ptr<Slot> sl = slot_enter(parent, &seq);
    {
        std::lock_guard<std::mutex> lk(parent.ls->hub->mu);
        sl->color[parent.rank] = color;
        sl->key[parent.rank] = key;
    }
    slot_barrier(parent, *sl, 0);
    {
        LoopHub* h = parent.ls->hub;
        std::lock_guard<std::mutex> lk(h->mu);
        // members of my color ordered by (key, parent rank), as ncclCommSplit
        std::vector<std::pair<int, int>> mem;
        for (int m = 0; m < parent.ls->size; m++)
            if (sl->color[m] == color) mem.push_back({sl->key[m], m});
        std::sort(mem.begin(), mem.end());
        auto it = sl->child.find(color);
        if (it == sl->child.end()) it = sl->child.emplace(color, h->make((int)mem.size())).first;
        out->ls = it->second;
        out->size = (int)mem.size();
        out->nc = nullptr;
        for (int q = 0; q < (int)mem.size(); q++)
            if (mem[q].second == parent.rank) out->rank = q;
    }
    slot_barrier(parent, *sl, 1);
    slot_leave(parent, seq, *sl);
    return ncclSuccess;
}

// ---------------------------------------------------------------------------
// public calls: dispatch on the transport
// ---------------------------------------------------------------------------
ncclResult_t comm_init_nccl(Comm* out, int nranks, const ncclUniqueId& id, int rank) {
    out->ls = nullptr;
    out->rank = rank;
    out->size = nranks;
    return ncclCommInitRank(&out->nc, nranks, id, rank);
}

ncclResult_t comm_split(const Comm& parent, int color, int key, Comm* out) {
    if (parent.ls) return loop_split(parent, color, key, out);
    ncclResult_t r = ncclCommSplit(parent.nc, color, key, &out->nc, nullptr);
    if (r != ncclSuccess) return r;
    out->ls = nullptr;
    ncclCommUserRank(out->nc, &out->rank);
    ncclCommCount(out->nc, &out->size);
    return ncclSuccess;
}

void comm_destroy(Comm* c) {
    if (c->nc) ncclCommDestroy(c->nc);
    c->nc = nullptr;
    c->ls = nullptr;  // owned by the hub
}

ncclResult_t comm_group_start() {
    t_depth++;
    return ncclGroupStart();
}

ncclResult_t comm_group_end() {
    ncclResult_t r = ncclSuccess;
    if (--t_depth == 0 && !t_pending.empty()) r = loop_flush();
    ncclResult_t q = ncclGroupEnd();
    return r != ncclSuccess ? r : q;
}

ncclResult_t comm_send(const Comm& c, const void* buf, size_t count, ncclDataType_t ty, int peer, cudaStream_t st,
                       long long* acct) {
    acct_add(acct, (double)count * type_size(ty));
    if (c.ls) return loop_send(c, buf, count * type_size(ty), peer, st);
    return ncclSend(buf, count, ty, peer, c.nc, st);
}

ncclResult_t comm_recv(const Comm& c, void* buf, size_t count, ncclDataType_t ty, int peer, cudaStream_t st,
                       long long* acct) {
    acct_add(acct, (double)count * type_size(ty));
    if (c.ls) return loop_recv(c, buf, count * type_size(ty), peer, st);
    return ncclRecv(buf, count, ty, peer, c.nc, st);
}

ncclResult_t comm_allreduce(const Comm& c, const void* sbuf, void* rbuf, size_t count, ncclDataType_t ty,
                            ncclRedOp_t op, cudaStream_t st, long long* acct) {
    if (c.size > 1) acct_add(acct, 2.0 * (c.size - 1) / c.size * (double)count * type_size(ty));
    if (c.ls) return loop_allreduce(c, sbuf, rbuf, count, ty, op, st);
    return ncclAllReduce(sbuf, rbuf, count, ty, op, c.nc, st);
}

ncclResult_t comm_bcast(const Comm& c, const void* sbuf, void* rbuf, size_t count, ncclDataType_t ty, int root,
                        cudaStream_t st, long long* acct) {
    if (c.size > 1) acct_add(acct, (double)count * type_size(ty));
    if (c.ls) return loop_bcast(c, sbuf, rbuf, count, ty, root, st);
    return ncclBroadcast(sbuf, rbuf, count, ty, root, c.nc, st);
}

const char* comm_error_string(ncclResult_t r) { return ncclGetErrorString(r); }

}  // namespace gtcp
