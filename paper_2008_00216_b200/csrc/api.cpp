// api.cpp -- the C ABI of include/sv.h: state object, executor (pass dispatch
// on one CUDA stream), readout, norm, virtual shards and the NCCL partition.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "plan.h"

namespace stv {
struct GatherMap {
    int32_t perm[64];
    uint64_t xmask;
    int32_t n;
    int32_t n_local;
    uint64_t rank_bits;
};
cudaError_t launch_tile_pass(bool c128, void *state, const uint8_t *dblob, uint32_t pass_off, int S, int n_local,
                             uint32_t rec_bytes, int ntab, cudaStream_t st, int *kernels);
cudaError_t launch_diag_pass(bool c128, void *state, const uint8_t *dblob, uint32_t pass_off, int S, int n_local,
                             cudaStream_t st, int *kernels);
cudaError_t launch_sample(int phase, bool c128, const void *state, const int32_t *perm, uint64_t xmask, int n,
                          int n_local, uint64_t rank_bits, uint64_t count, const uint64_t *chunk, const double *res,
                          double *a, int32_t *pick_lane, double *res2, double *vals, uint64_t *out, cudaStream_t st,
                          int *kernels);
cudaError_t launch_group_pass(bool c128, void *state, const uint8_t *dblob, const uint8_t *hrec, uint32_t pass_off,
                              int S, int n_local, uint32_t rec_bytes, uint32_t tab_entries, double flops_per_amp,
                              cudaStream_t st, int *kernels);
cudaError_t launch_cnot(bool c128, void *state, int c, int t, int n_local, cudaStream_t st, int *kernels);
cudaError_t launch_tc_group_pass(void *state, const uint8_t *dblob, const uint8_t *hrec, uint32_t pass_off, int S,
                                 int n_local, uint32_t rec_bytes, uint32_t tab_entries, int ntcop, cudaStream_t st,
                                 int *kernels);
cudaError_t launch_norm(bool c128, const void *state, uint64_t N, double *part, int np, double *out, cudaStream_t st,
                        int *kernels);
cudaError_t launch_fill(bool c128, void *state, uint64_t N, double val, int64_t one_at, cudaStream_t st, int *kernels);
cudaError_t launch_gather(bool c128, const void *state, const uint64_t *didx, uint64_t first, uint64_t count,
                          const GatherMap &gm, bool out_native, void *dout, cudaStream_t st, int *kernels);
}  // namespace stv

using namespace stv;

// ---------------------------------------------------------------------------
// NCCL, loaded at run time (the torch-bundled libnccl.so.2 is already in the
// process when torch.distributed initialised NCCL); no link-time dependency.
// ---------------------------------------------------------------------------
namespace {
typedef struct { char internal[128]; } ncclUniqueId_t;
typedef void *ncclComm_t;
enum { ncclInt8 = 0, ncclUint8 = 1, ncclFloat64 = 8 };
enum { ncclSum = 0 };
struct Nccl {
    void *h = nullptr;
    int (*commInitRank)(ncclComm_t *, int, ncclUniqueId_t, int) = nullptr;
    int (*commDestroy)(ncclComm_t) = nullptr;
    int (*send)(const void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*recv)(void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*groupStart)() = nullptr;
    int (*groupEnd)() = nullptr;
    int (*allReduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*errStr)(int) = nullptr;
    bool load() {
        if (h) return true;
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return false;
        commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
        commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
        send = (decltype(send))dlsym(h, "ncclSend");
        recv = (decltype(recv))dlsym(h, "ncclRecv");
        groupStart = (decltype(groupStart))dlsym(h, "ncclGroupStart");
        groupEnd = (decltype(groupEnd))dlsym(h, "ncclGroupEnd");
        allReduce = (decltype(allReduce))dlsym(h, "ncclAllReduce");
        errStr = (decltype(errStr))dlsym(h, "ncclGetErrorString");
        return commInitRank && send && recv && groupStart && groupEnd && allReduce;
    }
};
Nccl g_nccl;

thread_local std::string g_err;

sv_status fail(sv_status st, const std::string &msg) {
    g_err = msg;
    return st;
}
}  // namespace

struct sv_state {
    int n = 0, n_global = 0, n_local = 0;
    int rank = 0, world = 1;
    bool virt = false;            // virtual shards (single GPU, n_global > 0)
    sv_dtype dt = SV_C64;
    void *buf = nullptr;
    size_t bytes = 0;
    bool owned = false;
    cudaStream_t stream = nullptr;
    bool poisoned = false;
    int perm[64];                 // logical -> actual physical bit
    uint64_t xmask = 0;           // over actual physical bits
    sv_stats stats;
    // device scratch
    uint8_t *dblob = nullptr;
    size_t dblob_cap = 0;
    uint8_t *hblob = nullptr;     // pinned staging
    size_t hblob_cap = 0;
    double *dnorm = nullptr;      // partials + result
    void *dstage = nullptr;       // readout staging
    size_t dstage_cap = 0;
    uint64_t *didx = nullptr;
    size_t didx_cap = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::vector<cudaEvent_t> pev;
    // plan cache (small-n latency): the last few (circuit, frame, options) -> plan + encoded blobs
    struct PlanEntry {
        std::vector<uint8_t> key;
        stv::Plan plan;
        std::vector<uint8_t> blob;
        std::vector<std::vector<uint32_t>> poff;
        int perm_out[64];
        uint64_t xmask_out = 0;
        uint64_t id = 0;
    };
    std::vector<PlanEntry> pcache;
    uint64_t pcache_next = 1;
    uint64_t dblob_id = 0;            // cache entry whose blob is resident in dblob (0: none)
    // distributed
    ncclComm_t comm = nullptr;
    void *xbuf = nullptr;         // remap send/recv staging (2 sets: pieces pipelined)
    size_t xbuf_bytes = 0;
    cudaStream_t xstream = nullptr;   // remap exchange stream (overlaps pack / unpack of other pieces)
    cudaEvent_t xev[4] = {nullptr, nullptr, nullptr, nullptr};   // packed[2], exchanged[2]

    bool c128() const { return dt == SV_C128; }
    size_t esz() const { return dt == SV_C128 ? 16 : 8; }
    uint64_t nloc_amps() const { return 1ull << n_local; }
    // amplitudes held by this process's buffer (virtual shards: all 2^n, shard r at r * 2^n_local)
    uint64_t buf_amps() const { return virt ? 1ull << n : 1ull << n_local; }
    int nshards() const { return virt ? 1 << n_global : 1; }
    void *shard(int r) const { return (uint8_t *)buf + (virt ? ((size_t)r * esz()) << n_local : 0); }
    uint64_t shard_rank(int r) const { return virt ? (uint64_t)r : (uint64_t)rank; }
};

namespace {
const int kNormParts = 148 * 8;

sv_status cuda_fail(sv_state *s, cudaError_t e, const char *where) {
    if (s) s->poisoned = true;
    return fail(SV_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(s, call)                                                   \
    do {                                                              \
        cudaError_t _e = (call);                                      \
        if (_e != cudaSuccess) return cuda_fail((s), _e, #call);      \
    } while (0)

sv_status check_state(const sv_state *s) {
    if (!s) return fail(SV_ERR_INVALID_ARG, "NULL state");
    if (s->poisoned) return fail(SV_ERR_STATE, "state poisoned by an earlier CUDA/NCCL failure");
    return SV_OK;
}

void reset_frame(sv_state *s) {
    for (int i = 0; i < 64; ++i) s->perm[i] = i;
    s->xmask = 0;
}

sv_status common_init(sv_state *s) {
    CK(s, cudaMalloc((void **)&s->dnorm, sizeof(double) * (kNormParts + 1)));
    CK(s, cudaEventCreate(&s->ev0));
    CK(s, cudaEventCreate(&s->ev1));
    reset_frame(s);
    std::memset(&s->stats, 0, sizeof(s->stats));
    return SV_OK;
}

uint64_t rank_value(const sv_state *s) { return s->virt ? 0 : (uint64_t)s->rank; }

sv_status fill(sv_state *s, double val, int64_t one_at) {
    int k = 0;
    CK(s, launch_fill(s->c128(), s->buf, s->buf_amps(), val, one_at, s->stream, &k));
    CK(s, cudaStreamSynchronize(s->stream));
    return SV_OK;
}

sv_status ensure(sv_state *s, void **p, size_t *cap, size_t need, bool pinned) {
    if (*cap >= need) return SV_OK;
    if (*p) {
        if (pinned) cudaFreeHost(*p);
        else cudaFree(*p);
        *p = nullptr;
        *cap = 0;
    }
    size_t c = std::max(need, (size_t)1 << 20);
    cudaError_t e = pinned ? cudaMallocHost(p, c) : cudaMalloc(p, c);
    if (e != cudaSuccess) {
        *p = nullptr;
        return fail(SV_ERR_OUT_OF_MEMORY, std::string("scratch allocation: ") + cudaGetErrorString(e));
    }
    *cap = c;
    return SV_OK;
}

// all-to-all exchange for one set of global<->local bit swaps
sv_status dist_remap(sv_state *s, const std::vector<std::pair<int, int>> &swaps, int *kernels);
}  // namespace

extern "C" {

const char *sv_last_error(void) { return g_err.c_str(); }
const char *sv_version(void) { return "stv-b200 0.1 (sm_100a)"; }

static sv_status make_state(int n, sv_dtype dt, int n_global, sv_state **out) {
    if (!out) return fail(SV_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (n < 1 || n > 40) return fail(SV_ERR_INVALID_ARG, "n must be in [1, 40]");
    if (dt != SV_C64 && dt != SV_C128) return fail(SV_ERR_INVALID_ARG, "unknown dtype");
    if (n_global < 0 || n - n_global < (n_global ? 4 : 1)) return fail(SV_ERR_INVALID_ARG, "need at least 4 local qubits per shard");
    sv_state *s = new sv_state();
    s->n = n;
    s->dt = dt;
    s->n_global = n_global;
    s->n_local = n - n_global;
    *out = s;
    return SV_OK;
}

sv_status sv_create(int n, sv_dtype dt, sv_state **out) {
    sv_status st = make_state(n, dt, 0, out);
    if (st) return st;
    sv_state *s = *out;
    s->bytes = s->esz() << n;
    cudaError_t e = cudaMalloc(&s->buf, s->bytes);
    if (e != cudaSuccess) {
        delete s;
        *out = nullptr;
        return fail(SV_ERR_OUT_OF_MEMORY, std::string("state allocation: ") + cudaGetErrorString(e));
    }
    s->owned = true;
    if ((st = common_init(s))) return st;
    return fill(s, 0.0, 0);
}

sv_status sv_wrap(int n, sv_dtype dt, void *dev_buf, size_t bytes, void *stream, sv_state **out) {
    sv_status st = make_state(n, dt, 0, out);
    if (st) return st;
    sv_state *s = *out;
    if (!dev_buf || bytes < (s->esz() << n) || ((uintptr_t)dev_buf & 255)) {
        delete s;
        *out = nullptr;
        return fail(SV_ERR_INVALID_ARG, "dev_buf NULL, too small or not 256-B aligned");
    }
    s->buf = dev_buf;
    s->bytes = bytes;
    s->stream = (cudaStream_t)stream;
    if ((st = common_init(s))) return st;
    return fill(s, 0.0, 0);
}

sv_status sv_create_virtual(int n, sv_dtype dt, int g, sv_state **out) {
    if (g < 0 || g > 3) return fail(SV_ERR_INVALID_ARG, "virtual shards: g in [0, 3]");
    if (n - g < 4) return fail(SV_ERR_INVALID_ARG, "virtual shards: need at least 4 local qubits per shard (n - g >= 4)");
    sv_status st = sv_create(n, dt, out);
    if (st) return st;
    // one buffer holds the 2^g shards back to back (shard r = the amplitudes whose top g
    // physical bits equal r, i.e. a real rank's buffer); every pass runs per shard with that
    // rank's encoding, remaps go through the distributed pack -> exchange -> unpack path
    (*out)->n_global = g;
    (*out)->n_local = n - g;
    (*out)->virt = true;
    return SV_OK;
}

sv_status sv_create_dist(int n, sv_dtype dt, const void *uid, int rank, int world, void *dev_buf, size_t bytes,
                         void *stream, sv_state **out) {
    if (world < 1 || (world & (world - 1)) || rank < 0 || rank >= world)
        return fail(SV_ERR_INVALID_ARG, "world must be a power of two, 0 <= rank < world");
    if (world > 256)   // the remap swaps at most 8 bits at once (dist_remap's chunk tables)
        return fail(SV_ERR_INVALID_ARG, "world must be <= 256");
    int g = 0;
    while ((1 << g) < world) ++g;
    sv_status st = make_state(n, dt, g, out);
    if (st) return st;
    sv_state *s = *out;
    s->rank = rank;
    s->world = world;
    s->stream = (cudaStream_t)stream;
    const size_t need = s->esz() << s->n_local;
    if (dev_buf) {
        if (bytes < need || ((uintptr_t)dev_buf & 255)) {
            delete s;
            *out = nullptr;
            return fail(SV_ERR_INVALID_ARG, "dev_buf too small or not 256-B aligned");
        }
        s->buf = dev_buf;
        s->bytes = bytes;
    } else {
        cudaError_t e = cudaMalloc(&s->buf, need);
        if (e != cudaSuccess) {
            delete s;
            *out = nullptr;
            return fail(SV_ERR_OUT_OF_MEMORY, "state allocation failed");
        }
        s->owned = true;
        s->bytes = need;
    }
    if ((st = common_init(s))) return st;
    if (world > 1) {
        if (!g_nccl.load()) return fail(SV_ERR_UNSUPPORTED, "libnccl.so.2 not loadable");
        ncclUniqueId_t id;
        std::memcpy(&id, uid, sizeof(id));
        int r = g_nccl.commInitRank(&s->comm, world, id, rank);
        if (r) return fail(SV_ERR_NCCL, std::string("ncclCommInitRank: ") + (g_nccl.errStr ? g_nccl.errStr(r) : "?"));
    }
    return fill(s, 0.0, rank == 0 ? 0 : -1);
}

sv_status sv_set_basis(sv_state *s, uint64_t x) {
    sv_status st = check_state(s);
    if (st) return st;
    if (s->n < 64 && x >> s->n) return fail(SV_ERR_INVALID_ARG, "basis index >= 2^n");
    reset_frame(s);
    const uint64_t owner = s->virt ? 0 : x >> s->n_local;
    const int64_t at = (owner == rank_value(s)) ? (int64_t)(s->virt ? x : (x & (s->nloc_amps() - 1))) : -1;
    return fill(s, 0.0, at);
}

sv_status sv_set_uniform(sv_state *s) {
    sv_status st = check_state(s);
    if (st) return st;
    reset_frame(s);
    return fill(s, std::ldexp(1.0, -s->n) > 0 ? std::pow(2.0, -0.5 * s->n) : 0.0, -1);
}

sv_status sv_apply_circuit(sv_state *s, const sv_gate *gates, size_t ng, const sv_options *opt) {
    sv_status st = check_state(s);
    if (st) return st;
    if (ng && !gates) return fail(SV_ERR_INVALID_ARG, "gates is NULL");
    std::string err = validate(s->n, gates, ng);
    if (!err.empty()) return fail(SV_ERR_INVALID_ARG, err);
    auto t0 = std::chrono::steady_clock::now();
    const uint32_t flags = opt ? opt->flags : 0;
    // cache key: everything the plan and its encodings depend on (SV_OPT_PROFILE excluded)
    std::vector<uint8_t> key;
    {
        auto add = [&](const void *p, size_t nb) { key.insert(key.end(), (const uint8_t *)p, (const uint8_t *)p + nb); };
        const int32_t hdr[6] = {s->n, (int32_t)s->dt, s->n_global, s->virt ? 1 : 0, s->rank, s->world};
        add(hdr, sizeof(hdr));
        sv_options o{};
        if (opt) o = *opt;
        o.flags &= ~SV_OPT_PROFILE;
        add(&o, sizeof(o));
        add(s->perm, sizeof(int) * (size_t)s->n);
        add(&s->xmask, sizeof(s->xmask));
        for (size_t i = 0; i < ng; ++i) {
            const sv_gate &g = gates[i];
            const int32_t gi[4] = {g.kind, (int32_t)g.flags, g.q0, g.q1};
            add(gi, sizeof(gi));
            add(&g.theta, sizeof(double));
            add(&g.phi, sizeof(double));
            if (g.m) add(g.m, sizeof(double) * (g.kind == SV_U1 ? 8 : g.kind == SV_U2 ? 32 : 0));
        }
    }
    const bool use_cache = !(flags & SV_OPT_NO_PLAN_CACHE);
    sv_state::PlanEntry *ent = nullptr;
    if (use_cache)
        for (auto &e : s->pcache)
            if (e.key == key) { ent = &e; break; }
    if (!ent) {
        // plan in "virtual physical" bits = the state's current actual bits
        Frame fr;
        for (int q = 0; q < 64; ++q) fr.perm[q] = s->perm[q];
        fr.xmask = s->xmask;
        std::vector<PGate> pg = to_physical(s->n, gates, ng, fr, flags);
        PlanOptions po = resolve_options(opt, (int)s->esz(), s->n_local);
        int sigma[64];
        for (int v = 0; v < 64; ++v) sigma[v] = v;
        sv_state::PlanEntry ne;
        try {
            ne.plan = plan_auto(s->n, s->n_global, (int)s->esz(), pg, po, sigma);
        } catch (const std::exception &ex) {
            return fail(SV_ERR_INVALID_ARG, std::string("planner: ") + ex.what());
        }
        // one encoding per shard this process holds (rank bits, selectors on global bits)
        const int nsh_ = s->nshards();
        ne.poff.resize(nsh_);
        for (int r = 0; r < nsh_; ++r) {
            const uint64_t rb = s->shard_rank(r) << s->n_local;
            Encoded enc = encode(ne.plan, s->n_local, s->c128(), rb);
            while (ne.blob.size() & 255) ne.blob.push_back(0);
            const uint32_t at = (uint32_t)ne.blob.size();
            for (uint32_t off : enc.pass_off) {
                StvPass *hp = (StvPass *)&enc.blob[off];
                hp->rank_bits = rb;
                ne.poff[r].push_back(at + off);
            }
            ne.blob.insert(ne.blob.end(), enc.blob.begin(), enc.blob.end());
        }
        // frame after the plan: logical -> actual
        ne.xmask_out = 0;
        for (int v = 0; v < s->n; ++v)
            if ((fr.xmask >> v) & 1) ne.xmask_out |= 1ull << sigma[v];
        for (int q = 0; q < 64; ++q) ne.perm_out[q] = q < s->n ? sigma[fr.perm[q]] : q;
        ne.key = std::move(key);
        ne.id = s->pcache_next++;
        if (s->pcache.size() >= 4) {   // evict the oldest
            size_t old = 0;
            for (size_t i = 1; i < s->pcache.size(); ++i)
                if (s->pcache[i].id < s->pcache[old].id) old = i;
            if (s->dblob_id == s->pcache[old].id) s->dblob_id = 0;
            s->pcache.erase(s->pcache.begin() + (long)old);
        }
        s->pcache.push_back(std::move(ne));
        ent = &s->pcache.back();
        if (!use_cache) ent->id = 0;   // never reused
    }
    const Plan &plan = ent->plan;
    const std::vector<uint8_t> &blob = ent->blob;
    const std::vector<std::vector<uint32_t>> &poff = ent->poff;
    const int nsh = s->nshards();
    auto t1 = std::chrono::steady_clock::now();
    std::memset(&s->stats, 0, sizeof(s->stats));
    s->stats.plan_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    s->stats.alg_bytes = plan.alg_bytes * nsh;
    s->stats.alg_flops = plan.alg_flops * nsh;
    CK(s, cudaEventRecord(s->ev0, s->stream));
    if (ent->id == 0 || s->dblob_id != ent->id) {   // upload the blob unless it is already resident
        if ((st = ensure(s, (void **)&s->hblob, &s->hblob_cap, blob.size(), true))) return st;
        if (s->dblob_cap < blob.size()) s->dblob_id = 0;
        if ((st = ensure(s, (void **)&s->dblob, &s->dblob_cap, blob.size(), false))) return st;
        CK(s, cudaStreamSynchronize(s->stream));   // the pinned staging may still feed an earlier copy
        std::memcpy(s->hblob, blob.data(), blob.size());
        CK(s, cudaMemcpyAsync(s->dblob, s->hblob, blob.size(), cudaMemcpyHostToDevice, s->stream));
        s->stats.h2d_bytes = (double)blob.size();
        s->dblob_id = ent->id;
    }
    const bool prof = flags & SV_OPT_PROFILE;
    if (prof && s->pev.size() < plan.passes.size() + 1) {
        for (size_t i = s->pev.size(); i < plan.passes.size() + 1; ++i) {
            cudaEvent_t e;
            CK(s, cudaEventCreate(&e));
            s->pev.push_back(e);
        }
    }
    int kernels = 0;
    std::vector<int> kind_of(plan.passes.size());
    if (prof) CK(s, cudaEventRecord(s->pev[0], s->stream));
    for (size_t i = 0; i < plan.passes.size(); ++i) {
        const PPass &ps = plan.passes[i];
        int kind = 7;
        cudaError_t e = cudaSuccess;
        if (ps.kind == PASS_REMAP) {
            kind = 5;
            if ((st = dist_remap(s, ps.swaps, &kernels))) return st;
        }
        for (int r = 0; r < nsh && ps.kind != PASS_REMAP && e == cudaSuccess; ++r) {
            void *sbuf = s->shard(r);
            const uint32_t po_r = poff[r][i];
            const StvPass *hp = (const StvPass *)&blob[po_r];
            if (ps.kind == PASS_TILE) {
                kind = hp->h == 0 ? 1 : 2;
                if (hp->grouped && hp->ntc > 0 && !s->c128()) {
                    e = launch_tc_group_pass(sbuf, s->dblob, &blob[po_r], po_r, hp->S, s->n_local, hp->param_bytes,
                                             hp->tab_entries, hp->ntcop, s->stream, &kernels);
                    const StvTcStep *tcs = (const StvTcStep *)((const uint8_t *)hp + hp->tc_off);
                    int ms = 0;
                    for (int k = 0; k < hp->ntc; ++k) ms += tcs[k].kind == 1;
                    if (r == 0) s->stats.n_tc_pass++;
                    if (r == 0) s->stats.n_tc_steps += ms;
                    s->stats.tc_flops += 384.0 * ms * std::ldexp(1.0, s->n_local);
                } else if (hp->grouped) {
                    e = launch_group_pass(s->c128(), sbuf, s->dblob, &blob[po_r], po_r, hp->S, s->n_local,
                                          hp->param_bytes, hp->tab_entries, pass_flops_per_amp(ps.ops), s->stream,
                                          &kernels);
                } else {
                    e = launch_tile_pass(s->c128(), sbuf, s->dblob, po_r, hp->S, s->n_local, hp->rec_bytes, hp->ntab,
                                         s->stream, &kernels);
                }
                if (r == 0)
                    for (auto &o : ps.ops)
                        s->stats.n_ops[o.type == OP_DENSE ? 0 : o.type == OP_DIAG ? 1 : o.type == OP_CNOT ? 2 : 3]++;
            } else if (ps.kind == PASS_DIAG) {
                kind = 3;
                e = launch_diag_pass(s->c128(), sbuf, s->dblob, po_r, hp->S, s->n_local, s->stream, &kernels);
            } else if (ps.kind == PASS_CNOT) {
                kind = 4;
                int c = hp->cnot_c, t = hp->cnot_t;
                bool run = true;
                if (c >= s->n_local) {   // control on a global bit: per-rank predicate
                    run = (s->shard_rank(r) >> (c - s->n_local)) & 1;
                    c = -1;
                }
                if (run) e = launch_cnot(s->c128(), sbuf, c, t, s->n_local, s->stream, &kernels);
            }
        }
        if (e != cudaSuccess) return cuda_fail(s, e, "pass launch");
        kind_of[i] = kind;
        s->stats.n_pass[kind]++;
        if (prof) CK(s, cudaEventRecord(s->pev[i + 1], s->stream));
    }
    CK(s, cudaEventRecord(s->ev1, s->stream));
    CK(s, cudaStreamSynchronize(s->stream));
    float ms = 0;
    CK(s, cudaEventElapsedTime(&ms, s->ev0, s->ev1));
    s->stats.run_ms = ms;
    if (prof) {
        // STV_PASS_LOG=<file>: one line per pass (tuning / profiles; not part of the ABI)
        const char *plog = getenv("STV_PASS_LOG");
        FILE *pf = plog ? fopen(plog, "a") : nullptr;
        for (size_t i = 0; i < plan.passes.size(); ++i) {
            float pm = 0;
            CK(s, cudaEventElapsedTime(&pm, s->pev[i], s->pev[i + 1]));
            s->stats.pass_ms[kind_of[i]] += pm;
            if (pf) {
                const StvPass *hp = (const StvPass *)&blob[poff[0][i]];
                int msteps = 0;
                if (hp->ntc > 0) {
                    const StvTcStep *tcs = (const StvTcStep *)((const uint8_t *)hp + hp->tc_off);
                    for (int k = 0; k < hp->ntc; ++k) msteps += tcs[k].kind == 1;
                }
                fprintf(pf, "{\"pass\": %zu, \"kind\": %d, \"S\": %d, \"L\": %d, \"h\": %d, \"groups\": %d, "
                            "\"ntc\": %d, \"msteps\": %d, \"flops_per_amp\": %.1f, \"ms\": %.4f}\n",
                        i, hp->kind, hp->S, hp->L, hp->h, hp->nops, hp->ntc, msteps,
                        plan.passes[i].kind == PASS_TILE ? pass_flops_per_amp(plan.passes[i].ops) : 0.0, pm);
            }
        }
        if (pf) fclose(pf);
    }
    s->stats.n_kernels = kernels;
    // new frame: logical -> actual
    for (int q = 0; q < s->n; ++q) s->perm[q] = ent->perm_out[q];
    s->xmask = ent->xmask_out;
    return SV_OK;
}

static GatherMap gather_map(const sv_state *s) {
    GatherMap gm;
    for (int q = 0; q < 64; ++q) gm.perm[q] = s->perm[q];
    gm.xmask = s->xmask;
    gm.n = s->n;
    gm.n_local = s->virt ? s->n : s->n_local;
    gm.rank_bits = s->virt ? 0 : (uint64_t)s->rank;
    return gm;
}

static sv_status gather_impl(sv_state *s, const uint64_t *idx, uint64_t first, uint64_t count, bool native,
                             void *out) {
    sv_status st = check_state(s);
    if (st) return st;
    if (!count) return SV_OK;
    if (!out) return fail(SV_ERR_INVALID_ARG, "out is NULL");
    const uint64_t N = s->n >= 64 ? ~0ull : 1ull << s->n;
    if (idx) {
        for (uint64_t k = 0; k < count; ++k)
            if (idx[k] >= N) return fail(SV_ERR_INVALID_ARG, "amplitude index " + std::to_string(idx[k]) + " >= 2^n");
    } else if (first >= N || count > N - first) {
        return fail(SV_ERR_INVALID_ARG, "amplitude range out of [0, 2^n)");
    }
    const size_t osz = native ? s->esz() : 16;
    const uint64_t chunk = std::min<uint64_t>(count, (64ull << 20) / osz);
    if ((st = ensure(s, &s->dstage, &s->dstage_cap, chunk * osz, false))) return st;
    if (idx && (st = ensure(s, (void **)&s->didx, &s->didx_cap, chunk * 8, false))) return st;
    GatherMap gm = gather_map(s);
    int kernels = 0;
    for (uint64_t b = 0; b < count; b += chunk) {
        const uint64_t c = std::min(chunk, count - b);
        if (s->world > 1) CK(s, cudaMemsetAsync(s->dstage, 0, c * osz, s->stream));
        if (idx) CK(s, cudaMemcpyAsync(s->didx, idx + b, c * 8, cudaMemcpyHostToDevice, s->stream));
        CK(s, launch_gather(s->c128(), s->buf, idx ? s->didx : nullptr, first + b, c, gm, native, s->dstage,
                            s->stream, &kernels));
        if (s->world > 1) {
            // exactly one rank owns each amplitude; the others contribute zeros
            const size_t nd = c * osz / 8;
            int r = native && !s->c128()
                        ? 1   // float sums of x + 0 are exact as well, but use doubles only
                        : 0;
            (void)r;
            if (native && !s->c128()) {
                int rr = g_nccl.allReduce(s->dstage, s->dstage, c * 2, 7 /*ncclFloat32*/, ncclSum, s->comm, s->stream);
                if (rr) { s->poisoned = true; return fail(SV_ERR_NCCL, "ncclAllReduce (gather)"); }
            } else {
                int rr = g_nccl.allReduce(s->dstage, s->dstage, nd, ncclFloat64, ncclSum, s->comm, s->stream);
                if (rr) { s->poisoned = true; return fail(SV_ERR_NCCL, "ncclAllReduce (gather)"); }
            }
        }
        CK(s, cudaMemcpyAsync((uint8_t *)out + b * osz, s->dstage, c * osz, cudaMemcpyDeviceToHost, s->stream));
    }
    CK(s, cudaStreamSynchronize(s->stream));
    return SV_OK;
}

sv_status sv_get_amplitudes(sv_state *s, const uint64_t *idx, uint64_t first, size_t count, double *out) {
    return gather_impl(s, idx, first, count, false, out);
}

sv_status sv_read_state(sv_state *s, uint64_t first, uint64_t count, void *out) {
    return gather_impl(s, nullptr, first, count, true, out);
}

sv_status sv_norm(sv_state *s, double *out) {
    sv_status st = check_state(s);
    if (st) return st;
    if (!out) return fail(SV_ERR_INVALID_ARG, "out is NULL");
    int k = 0;
    CK(s, launch_norm(s->c128(), s->buf, s->buf_amps(), s->dnorm, kNormParts, s->dnorm + kNormParts, s->stream, &k));
    if (s->world > 1) {
        int r = g_nccl.allReduce(s->dnorm + kNormParts, s->dnorm + kNormParts, 1, ncclFloat64, ncclSum, s->comm,
                                 s->stream);
        if (r) { s->poisoned = true; return fail(SV_ERR_NCCL, "ncclAllReduce (norm)"); }
    }
    CK(s, cudaMemcpyAsync(out, s->dnorm + kNormParts, sizeof(double), cudaMemcpyDeviceToHost, s->stream));
    CK(s, cudaStreamSynchronize(s->stream));
    return SV_OK;
}

// ---------------------------------------------------------------------------
// sv_sample (include/sv.h): chunk masses on the device, host prefix sums and shot
// routing, one warp per shot on the device, frame mapping on the host.
// ---------------------------------------------------------------------------
static uint64_t splitmix_out(uint64_t seed, uint64_t s) {   // (s+1)-th output of splitmix64(seed)
    uint64_t z = seed + (s + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

sv_status sv_sample(sv_state *s, uint64_t seed, size_t shots, uint64_t *out) {
    sv_status st = check_state(s);
    if (st) return st;
    if (!shots) return SV_OK;
    if (!out) return fail(SV_ERR_INVALID_ARG, "out is NULL");
    // logical order: chunk c = logical indices [4096 c, 4096 (c + 1)) of all 2^n
    const uint64_t NL = 1ull << s->n;
    const uint64_t nch = (NL + 4095) / 4096;
    const int nl = s->virt ? s->n : s->n_local;
    const uint64_t rb = rank_value(s);
    const uint64_t batch = std::min<uint64_t>(shots, 1ull << 16);
    double *dmass = nullptr, *dres = nullptr, *dlanes = nullptr, *dres2 = nullptr, *dvals = nullptr;
    uint64_t *dchunk = nullptr, *dout = nullptr;
    int32_t *dlane = nullptr;
    auto cleanup = [&]() {
        cudaFree(dmass); cudaFree(dres); cudaFree(dlanes); cudaFree(dres2); cudaFree(dvals);
        cudaFree(dchunk); cudaFree(dout); cudaFree(dlane);
    };
    auto allreduce = [&](double *d, size_t cnt) -> bool {   // distributed: sum the per-rank arrays
        if (s->world < 2) return true;
        return g_nccl.allReduce(d, d, cnt, ncclFloat64, ncclSum, s->comm, s->stream) == 0;
    };
    if (cudaMalloc(&dmass, nch * 8) || cudaMalloc(&dres, batch * 8) || cudaMalloc(&dlanes, batch * 32 * 8) ||
        cudaMalloc(&dres2, batch * 8) || cudaMalloc(&dvals, batch * 128 * 8) || cudaMalloc(&dchunk, batch * 8) ||
        cudaMalloc(&dout, batch * 8) || cudaMalloc(&dlane, batch * 4)) {
        cleanup();
        return fail(SV_ERR_OUT_OF_MEMORY, "sample scratch");
    }
    int k = 0;
    cudaError_t e = launch_sample(0, s->c128(), s->buf, s->perm, s->xmask, s->n, nl, rb, nch, nullptr, nullptr, dmass,
                                  nullptr, nullptr, nullptr, nullptr, s->stream, &k);
    if (e != cudaSuccess) { cleanup(); return cuda_fail(s, e, "sample mass"); }
    if (!allreduce(dmass, nch)) { cleanup(); s->poisoned = true; return fail(SV_ERR_NCCL, "ncclAllReduce (sample mass)"); }
    std::vector<double> mass(nch), pre(nch + 1, 0.0);
    e = cudaMemcpyAsync(mass.data(), dmass, nch * 8, cudaMemcpyDeviceToHost, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) { cleanup(); return cuda_fail(s, e, "sample mass"); }
    for (uint64_t c = 0; c < nch; ++c) pre[c + 1] = pre[c] + mass[c];   // fp64, sequential, logical order
    const double total = pre[nch];
    if (!(total > 0) || !std::isfinite(total)) { cleanup(); return fail(SV_ERR_INVALID_ARG, "state has no probability mass"); }
    uint64_t last_nz = nch - 1;
    while (last_nz > 0 && mass[last_nz] <= 0) --last_nz;
    std::vector<uint64_t> hchunk(batch), res(shots);
    std::vector<double> hres(batch);
    for (size_t b0 = 0; b0 < shots; b0 += batch) {
        const uint64_t m = std::min<uint64_t>(batch, shots - b0);
        for (uint64_t i = 0; i < m; ++i) {
            const double u = (double)(splitmix_out(seed, b0 + i) >> 11) * 0x1.0p-53;
            const double target = u * total;
            // first chunk whose inclusive prefix exceeds the target (clamped to the last chunk with mass)
            uint64_t c = (uint64_t)(std::upper_bound(pre.begin() + 1, pre.end(), target) - (pre.begin() + 1));
            if (c > last_nz) c = last_nz;
            while (c > 0 && mass[c] <= 0) --c;
            hchunk[i] = c;
            hres[i] = target - pre[c];
        }
        e = cudaMemcpyAsync(dchunk, hchunk.data(), m * 8, cudaMemcpyHostToDevice, s->stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(dres, hres.data(), m * 8, cudaMemcpyHostToDevice, s->stream);
        if (e == cudaSuccess)
            e = launch_sample(1, s->c128(), s->buf, s->perm, s->xmask, s->n, nl, rb, m, dchunk, nullptr, dlanes,
                              nullptr, nullptr, nullptr, nullptr, s->stream, &k);
        if (e != cudaSuccess) { cleanup(); return cuda_fail(s, e, "sample lanes"); }
        if (!allreduce(dlanes, m * 32)) { cleanup(); s->poisoned = true; return fail(SV_ERR_NCCL, "ncclAllReduce (sample lanes)"); }
        e = launch_sample(2, s->c128(), s->buf, s->perm, s->xmask, s->n, nl, rb, m, dchunk, dres, dlanes, dlane, dres2,
                          dvals, nullptr, s->stream, &k);
        if (e != cudaSuccess) { cleanup(); return cuda_fail(s, e, "sample values"); }
        if (!allreduce(dvals, m * 128)) { cleanup(); s->poisoned = true; return fail(SV_ERR_NCCL, "ncclAllReduce (sample values)"); }
        e = launch_sample(3, s->c128(), s->buf, s->perm, s->xmask, s->n, nl, rb, m, dchunk, nullptr, nullptr, dlane,
                          dres2, dvals, dout, s->stream, &k);
        if (e == cudaSuccess) e = cudaMemcpyAsync(res.data() + b0, dout, m * 8, cudaMemcpyDeviceToHost, s->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
        if (e != cudaSuccess) { cleanup(); return cuda_fail(s, e, "sample pick"); }
    }
    std::memcpy(out, res.data(), shots * 8);
    cleanup();
    return SV_OK;
}

sv_status sv_last_run_stats(const sv_state *s, sv_stats *out) {
    if (!s || !out) return fail(SV_ERR_INVALID_ARG, "NULL argument");
    *out = s->stats;
    return SV_OK;
}

sv_status sv_get_frame(const sv_state *s, int32_t *perm, uint64_t *xmask) {
    if (!s) return fail(SV_ERR_INVALID_ARG, "NULL state");
    if (perm) for (int q = 0; q < s->n; ++q) perm[q] = s->perm[q];
    if (xmask) *xmask = s->xmask;
    return SV_OK;
}

sv_status sv_plan_json(int n, int n_global, sv_dtype dt, const sv_gate *gates, size_t ng, const sv_options *opt,
                       char *buf, size_t cap, size_t *needed) {
    if (n < 1 || n > 40 || n_global < 0 || n - n_global < 4) return fail(SV_ERR_INVALID_ARG, "bad n / n_global");
    std::string err = validate(n, gates, ng);
    if (!err.empty()) return fail(SV_ERR_INVALID_ARG, err);
    Frame fr;
    fr.identity(n);
    const int esz = dt == SV_C128 ? 16 : 8;
    std::vector<PGate> pg = to_physical(n, gates, ng, fr, opt ? opt->flags : 0);
    PlanOptions po = resolve_options(opt, esz, n - n_global);
    int sigma[64];
    for (int v = 0; v < 64; ++v) sigma[v] = v;
    Plan plan;
    try {
        plan = plan_auto(n, n_global, esz, pg, po, sigma);
    } catch (const std::exception &ex) {
        return fail(SV_ERR_INVALID_ARG, std::string("planner: ") + ex.what());
    }
    // compose the final frame (logical -> actual)
    plan.frame_out.xmask = 0;
    for (int v = 0; v < n; ++v)
        if ((fr.xmask >> v) & 1) plan.frame_out.xmask |= 1ull << sigma[v];
    for (int q = 0; q < 64; ++q) plan.frame_out.perm[q] = q < n ? sigma[fr.perm[q]] : q;
    std::string js = plan_to_json(plan);
    if (needed) *needed = js.size() + 1;
    if (!buf || cap < js.size() + 1) return fail(SV_ERR_INVALID_ARG, "buffer too small");
    std::memcpy(buf, js.c_str(), js.size() + 1);
    return SV_OK;
}

sv_status sv_plan_blob(int n, int n_global, sv_dtype dt, const sv_gate *gates, size_t ng, const sv_options *opt,
                       uint8_t *buf, size_t cap, size_t *needed, uint32_t *pass_off, size_t max_passes,
                       size_t *npasses) {
    if (n < 1 || n > 40 || n_global < 0 || n - n_global < 4) return fail(SV_ERR_INVALID_ARG, "bad n / n_global");
    std::string err = validate(n, gates, ng);
    if (!err.empty()) return fail(SV_ERR_INVALID_ARG, err);
    Frame fr;
    fr.identity(n);
    const int esz = dt == SV_C128 ? 16 : 8;
    std::vector<PGate> pg = to_physical(n, gates, ng, fr, opt ? opt->flags : 0);
    PlanOptions po = resolve_options(opt, esz, n - n_global);
    int sigma[64];
    for (int v = 0; v < 64; ++v) sigma[v] = v;
    Plan plan;
    try {
        plan = plan_auto(n, n_global, esz, pg, po, sigma);
    } catch (const std::exception &ex) {
        return fail(SV_ERR_INVALID_ARG, std::string("planner: ") + ex.what());
    }
    Encoded enc = encode(plan, n - n_global, dt == SV_C128);
    if (needed) *needed = enc.blob.size();
    if (npasses) *npasses = enc.pass_off.size();
    if (pass_off)
        for (size_t i = 0; i < enc.pass_off.size() && i < max_passes; ++i) pass_off[i] = enc.pass_off[i];
    if (!buf || cap < enc.blob.size()) return fail(SV_ERR_INVALID_ARG, "buffer too small");
    std::memcpy(buf, enc.blob.data(), enc.blob.size());
    return SV_OK;
}

sv_status sv_remap_peers(int g, int rank, uint32_t gbits, int m, int32_t *peer) {
    if (g < 0 || g > 10 || rank < 0 || rank >= (1 << g) || !peer || m != __builtin_popcount(gbits) ||
        (gbits >> g))
        return fail(SV_ERR_INVALID_ARG, "bad remap arguments");
    // global bits gb_0 < gb_1 < ... (within the rank index) swap with local
    // bits lb_0..lb_{m-1}: chunk c (value of the local bits) moves to the rank
    // whose selected global bits equal c; its slot there is this rank's
    // selected-global-bit value.
    std::vector<int> gb;
    for (int b = 0; b < g; ++b)
        if ((gbits >> b) & 1) gb.push_back(b);
    for (int c = 0; c < (1 << m); ++c) {
        int r = rank;
        for (int i = 0; i < m; ++i) {
            r &= ~(1 << gb[i]);
            r |= ((c >> i) & 1) << gb[i];
        }
        peer[c] = r;
    }
    return SV_OK;
}

sv_status sv_destroy(sv_state *s) {
    if (!s) return SV_OK;
    if (s->comm && g_nccl.commDestroy) g_nccl.commDestroy(s->comm);
    if (s->owned && s->buf) cudaFree(s->buf);
    if (s->dblob) cudaFree(s->dblob);
    if (s->hblob) cudaFreeHost(s->hblob);
    if (s->dnorm) cudaFree(s->dnorm);
    if (s->dstage) cudaFree(s->dstage);
    if (s->didx) cudaFree(s->didx);
    if (s->xbuf) cudaFree(s->xbuf);
    for (auto e : s->xev)
        if (e) cudaEventDestroy(e);
    if (s->xstream) cudaStreamDestroy(s->xstream);
    if (s->ev0) cudaEventDestroy(s->ev0);
    if (s->ev1) cudaEventDestroy(s->ev1);
    for (auto e : s->pev) cudaEventDestroy(e);
    delete s;
    return SV_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// distributed remap: pack -> grouped ncclSend/ncclRecv -> unpack, chunked
// ---------------------------------------------------------------------------
namespace stv {
cudaError_t launch_pack(bool c128, const void *state, void *dst, const int *lbits, int m, uint32_t chunk,
                        uint64_t first, uint64_t count, int n_local, bool unpack, cudaStream_t st, int *kernels);
}

namespace {
// Global<->local bit swaps: every rank packs the 2^m - 1 chunks (values of
// the swapped local bits) that leave it, exchanges them with the ranks that differ in the
// swapped global bits, and unpacks what it receives into the vacated chunks.  Real ranks
// exchange with grouped ncclSend/ncclRecv; virtual shards (one process, one GPU) run the
// same schedule with one device-to-device copy per (shard, peer) chunk.
sv_status dist_remap(sv_state *s, const std::vector<std::pair<int, int>> &swaps, int *kernels) {
    if (s->world < 2 && !s->virt) return SV_OK;
    const int m = (int)swaps.size();
    if (m < 1 || m > 8 || m > s->n_global) return fail(SV_ERR_INVALID_ARG, "remap: 1..min(8, g) swapped bits");
    uint32_t gbits = 0;
    int lbits[8];
    // pairs sorted by global bit so chunk value bit i <-> global bit i-th
    std::vector<std::pair<int, int>> sw = swaps;
    std::sort(sw.begin(), sw.end());
    for (int i = 0; i < m; ++i) {
        gbits |= 1u << (sw[i].first - s->n_local);
        lbits[i] = sw[i].second;
    }
    const int nsh = s->nshards();
    std::vector<std::vector<int32_t>> peer(nsh, std::vector<int32_t>((size_t)1 << m));
    std::vector<int> mine(nsh, 0);   // a shard's own chunk: the value of its selected global bits
    for (int r = 0; r < nsh; ++r) {
        const int rank = (int)s->shard_rank(r);
        sv_status st = sv_remap_peers(s->n_global, rank, gbits, m, peer[r].data());
        if (st) return st;
        for (int i = 0; i < m; ++i) mine[r] |= ((rank >> (sw[i].first - s->n_local)) & 1) << i;
    }
    auto slot = [](int c, int own) { return c < own ? c : c - 1; };
    const uint64_t chunk_amps = 1ull << (s->n_local - m);
    const int npeers = (1 << m) - 1;
    // staging: 2 sets (pieces pipelined) of send + recv slots per shard
    uint64_t cap = s->virt ? (2ull << 30) : (1ull << 30);
    {
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) == cudaSuccess && fr / 4 > cap) cap = std::min<uint64_t>(fr / 4, 8ull << 30);
    }
    const uint64_t piece =
        std::max<uint64_t>(1, std::min<uint64_t>(chunk_amps, cap / (4ull * nsh * npeers * s->esz())));
    const size_t slot_bytes = (size_t)piece * s->esz();
    const size_t set_bytes = 2ull * nsh * npeers * slot_bytes;
    sv_status st = ensure(s, &s->xbuf, &s->xbuf_bytes, 2 * set_bytes, false);
    if (st) return st;
    auto sendb = [&](int set, int r, int sl) {
        return (uint8_t *)s->xbuf + set * set_bytes + ((size_t)r * npeers + sl) * slot_bytes;
    };
    auto recvb = [&](int set, int r, int sl) {
        return (uint8_t *)s->xbuf + set * set_bytes + ((size_t)(nsh + r) * npeers + sl) * slot_bytes;
    };
    // pipeline (STV_REMAP_PIPE=0: serial): the main stream packs piece i into set i%2, the
    // exchange stream moves it once packed, the main stream unpacks piece i-1 while piece i
    // is in flight; a set is reused two pieces later, after its unpack
    static const bool pipe = !getenv("STV_REMAP_PIPE") || atoi(getenv("STV_REMAP_PIPE")) != 0;
    if (pipe && !s->xstream) {
        CK(s, cudaStreamCreateWithFlags(&s->xstream, cudaStreamNonBlocking));
        for (auto &e : s->xev) CK(s, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    cudaStream_t xs = pipe ? s->xstream : s->stream;
    const uint64_t npieces = (chunk_amps + piece - 1) / piece;
    auto pack = [&](uint64_t i) -> sv_status {
        const uint64_t off = i * piece, cnt = std::min(piece, chunk_amps - off);
        const int set = (int)(i & 1);
        for (int r = 0; r < nsh; ++r)
            for (int c = 0; c < (1 << m); ++c) {
                if (c == mine[r]) continue;
                cudaError_t e = launch_pack(s->c128(), s->shard(r), sendb(set, r, slot(c, mine[r])), lbits, m, c, off,
                                            cnt, s->n_local, false, s->stream, kernels);
                if (e != cudaSuccess) return cuda_fail(s, e, "remap pack");
            }
        if (pipe) CK(s, cudaEventRecord(s->xev[set], s->stream));
        return SV_OK;
    };
    auto exchange = [&](uint64_t i) -> sv_status {
        const uint64_t off = i * piece, cnt = std::min(piece, chunk_amps - off);
        const int set = (int)(i & 1);
        const size_t b = cnt * s->esz();
        if (pipe) CK(s, cudaStreamWaitEvent(xs, s->xev[set], 0));
        if (s->virt) {
            // rank p sends its chunk mine[r] to r, which receives it in its slot for chunk c (p = peer[r][c])
            for (int r = 0; r < nsh; ++r)
                for (int c = 0; c < (1 << m); ++c) {
                    if (c == mine[r]) continue;
                    const int p = peer[r][c];
                    CK(s, cudaMemcpyAsync(recvb(set, r, slot(c, mine[r])), sendb(set, p, slot(mine[r], mine[p])), b,
                                          cudaMemcpyDeviceToDevice, xs));
                }
        } else {
            g_nccl.groupStart();
            for (int c = 0; c < (1 << m); ++c) {
                if (c == mine[0]) continue;
                const int sl = slot(c, mine[0]);
                int r1 = g_nccl.send(sendb(set, 0, sl), b, ncclUint8, peer[0][c], s->comm, xs);
                int r2 = g_nccl.recv(recvb(set, 0, sl), b, ncclUint8, peer[0][c], s->comm, xs);
                if (r1 || r2) { s->poisoned = true; return fail(SV_ERR_NCCL, "ncclSend/Recv (remap)"); }
            }
            if (g_nccl.groupEnd()) { s->poisoned = true; return fail(SV_ERR_NCCL, "ncclGroupEnd (remap)"); }
        }
        if (pipe) CK(s, cudaEventRecord(s->xev[2 + set], xs));
        s->stats.remap_bytes += (double)npeers * b;   // per rank
        return SV_OK;
    };
    auto unpack = [&](uint64_t i) -> sv_status {
        const uint64_t off = i * piece, cnt = std::min(piece, chunk_amps - off);
        const int set = (int)(i & 1);
        if (pipe) CK(s, cudaStreamWaitEvent(s->stream, s->xev[2 + set], 0));
        for (int r = 0; r < nsh; ++r)
            for (int c = 0; c < (1 << m); ++c) {
                if (c == mine[r]) continue;
                // data from peer[r][c] (its chunk mine[r]) lands in r's chunk c
                cudaError_t e = launch_pack(s->c128(), s->shard(r), recvb(set, r, slot(c, mine[r])), lbits, m, c, off,
                                            cnt, s->n_local, true, s->stream, kernels);
                if (e != cudaSuccess) return cuda_fail(s, e, "remap unpack");
            }
        return SV_OK;
    };
    for (uint64_t i = 0; i < npieces; ++i) {
        if ((st = pack(i))) return st;          // set i%2 is free: piece i-2 was unpacked before
        if ((st = exchange(i))) return st;
        if (pipe && i > 0 && (st = unpack(i - 1))) return st;
        if (!pipe && (st = unpack(i))) return st;
    }
    if (pipe && npieces > 0 && (st = unpack(npieces - 1))) return st;
    return SV_OK;
}
}  // namespace
