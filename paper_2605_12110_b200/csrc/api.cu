// C-ABI host layer (include/absp.h): validation with the reference's error
// semantics, per-layer device state, and stream-ordered kernel orchestration.
//
// Nothing here computes on the host: every numeric result comes from the
// sm_100a kernels in this directory. There is no CPU fallback; a missing or
// failing device surfaces as ABSP_ECUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <map>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "absp_internal.cuh"

using namespace absp;

namespace {

thread_local std::string g_err;

// NVTX range over one C-ABI call (visible under Nsight Systems / ncu --nvtx; a few
// nanoseconds when no tool is attached).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

absp_status fail(absp_status st, const std::string& msg) {
    g_err = msg;
    return st;
}

absp_status cuda_fail(cudaError_t e, const char* what) {
    return fail(ABSP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define ABSP_CUDA(call)                                             \
    do {                                                            \
        cudaError_t e__ = (call);                                   \
        if (e__ != cudaSuccess) return cuda_fail(e__, #call);       \
    } while (0)

uint32_t ceil_div(uint64_t a, uint64_t b) { return uint32_t((a + b - 1) / b); }

// Restores the caller's current device on scope exit.
struct DeviceGuard {
    int prev = -1;
    bool ok = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaError_t ensure(size_t count) {
        if (count <= n && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        if (count == 0) return cudaSuccess;
        cudaError_t e = cudaMalloc(&p, count * sizeof(T));
        if (e == cudaSuccess) n = count;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

// Device-side attention work list (see AttendWork), with its own split-KV partials:
// the decode-step list and every explicit-selection list (absp_attend) are separate,
// so building one never frees buffers another (or a captured graph) still uses.
struct WorkList {
    DevBuf<uint32_t> chunk_unit, chunk_idx, chunk_base, unit_done, unit_run;
    DevBuf<uint32_t> page;    // resolved page list, [n_work][ns] (see PageList)
    DevBuf<uint16_t> valid;
    DevBuf<float> part_o, part_ml;  // one partial slot per (unit, CTA run): o [8][D], (m, l) [8]
    uint32_t n_work = 0, max_runs = 0, ns = 0, grid = 0;
    uint64_t layout = ~0ull;              // layout version the list was built for
    std::vector<uint32_t> h_base, h_run;  // host copies: an unchanged list is not re-uploaded
    void release() {
        h_base.clear();
        h_run.clear();
        chunk_unit.release();
        chunk_idx.release();
        chunk_base.release();
        unit_done.release();
        unit_run.release();
        page.release();
        valid.release();
        part_o.release();
        part_ml.release();
        layout = ~0ull;
    }
    PageList pages() const { return PageList{page.p, valid.p, chunk_base.p, ns}; }
};

// Host->device uploads of layout data. Synchronous (cudaMemcpy) when no stream is
// given; otherwise staged through pinned buffers and copied with cudaMemcpyAsync on
// the stream, in order with the kernels around it (decode-time appends). The pinned
// buffers form a ring sized at bind time for the largest batch a layout can upload,
// so an async batch neither grows a buffer nor waits on the GPU unless more than
// kRing batches of the layer are still queued ahead of it.
struct Stager {
    static constexpr int kRing = 4;
    struct Buf {
        unsigned char* host = nullptr;  // pinned
        size_t cap = 0;
        cudaEvent_t done = nullptr;     // recorded after the batch that used it
    };
    Buf ring[kRing];
    int cur = 0;
    cudaStream_t s = nullptr;
    bool async = false;
    size_t off = 0;
    cudaError_t reserve(size_t bytes) {  // every ring buffer holds `bytes` (sync callers only)
        for (Buf& b : ring) {
            if (b.cap >= bytes) continue;
            if (b.done) {
                cudaError_t e = cudaEventSynchronize(b.done);
                if (e != cudaSuccess) return e;
            }
            if (b.host) cudaFreeHost(b.host);
            b.host = nullptr;
            b.cap = 0;
            cudaError_t e = cudaMallocHost(&b.host, bytes);
            if (e != cudaSuccess) return e;
            b.cap = bytes;
        }
        return cudaSuccess;
    }
    cudaError_t begin(cudaStream_t stream, bool use_async) {
        s = stream;
        async = use_async;
        off = 0;
        if (!async) return cudaSuccess;
        cur = (cur + 1) % kRing;
        // the buffer's previous batch was issued kRing batches ago: normally long done
        return ring[cur].done ? cudaEventSynchronize(ring[cur].done) : cudaSuccess;
    }
    cudaError_t put(void* dst, const void* src, size_t bytes) {
        if (bytes == 0) return cudaSuccess;
        if (!async) return cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
        Buf& b = ring[cur];
        const size_t need = (off + bytes + 15) & ~size_t(15);
        if (need > b.cap) {  // beyond the bind-time bound: earlier copies must leave the old buffer
            cudaError_t e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) return e;
            if (b.host) cudaFreeHost(b.host);
            b.host = nullptr;
            b.cap = std::max<size_t>(2 * need, 1 << 16);
            e = cudaMallocHost(&b.host, b.cap);
            if (e != cudaSuccess) { b.host = nullptr; b.cap = 0; return e; }
            off = 0;
        }
        std::memcpy(b.host + off, src, bytes);
        cudaError_t e = cudaMemcpyAsync(dst, b.host + off, bytes, cudaMemcpyHostToDevice, s);
        off = (off + bytes + 15) & ~size_t(15);
        return e;
    }
    cudaError_t zero(void* dst, size_t bytes) {
        return async ? cudaMemsetAsync(dst, 0, bytes, s) : cudaMemset(dst, 0, bytes);
    }
    cudaError_t end() {
        if (!async) return cudaSuccess;
        Buf& b = ring[cur];
        if (!b.done) {
            cudaError_t e = cudaEventCreateWithFlags(&b.done, cudaEventDisableTiming);
            if (e != cudaSuccess) return e;
        }
        return cudaEventRecord(b.done, s);
    }
    void release() {
        for (Buf& b : ring) {
            if (b.done) cudaEventDestroy(b.done);
            if (b.host) cudaFreeHost(b.host);
            b = Buf{};
        }
        off = 0;
    }
};

struct Layer {
    bool assigned = false, bound = false, built = false, selected = false;
    Stager stager;
    std::vector<uint32_t> block_sizes;
    const uint16_t* k_pool = nullptr;
    const uint16_t* v_pool = nullptr;
    uint64_t pool_pages = 0;
    const uint32_t* page_table = nullptr;
    uint32_t max_pages = 0;
    uint32_t batch = 0;
    std::vector<uint32_t> seq_lens;
    std::vector<UnitDesc> desc;
    // Layout version: bumped whenever a kernel argument of the decode step (grids,
    // work counts) changes; device arrays are capacity-reserved at bind, so their
    // pointers never change between binds. Graphs captured over absp_decode_step stay
    // valid while the version is unchanged (absp_layout_version).
    uint64_t layout_version = 0;
    uint64_t desc_version = 0;       // bumped by every layout (explicit work lists follow it)
    std::vector<uint64_t> step_key;  // the step's kernel arguments that depend on the layout
    std::vector<ScoreItem> items;
    std::vector<uint32_t> item_begin;
    uint64_t total_cap = 0, total_centroids = 0;
    uint32_t max_cap = 0, max_nblocks = 0, max_budget = 0, max_select = 0;
    uint32_t sel_stride = 0;
    WorkList step_work;                      // decode_step: min(N, K) entries per unit
    std::map<uint32_t, WorkList> attend_work;  // absp_attend, keyed by blocks_stride

    DevBuf<UnitDesc> d_desc;
    DevBuf<ScoreItem> d_items;
    DevBuf<uint32_t> d_item_begin;
    DevBuf<float> values, values_min, scales, zps, scales_min, zps_min, scores;
    DevBuf<uint32_t> codes, codes_min;
    DevBuf<uint32_t> sel_blocks, sel_counts;
    DevBuf<uint32_t> ready;   // decode step: per-unit "selection published" flags (zero between steps)
    DevBuf<uint32_t> scored;  // per-unit scored-centroid counters (zero between steps)
    DevBuf<uint32_t> topk_units;  // units grouped by top-k register class
    std::vector<uint32_t> h_topk_order;
    TopkClasses topk_classes{};
    DevBuf<float> approx, unit_err;  // decode-step filter diagnostics: approximate scores, per-unit bounds
    bool filter_diag = false;        // the fused selection writes them (absp_set_filter_diagnostics)
    SelectPlan sel_plan{};           // fused selection: slice size, ring stages, capacities, grid
    DevBuf<SliceDesc> sel_slices;    // fused selection work (capacity-reserved at bind)
    DevBuf<uint32_t> sel_slot, sel_arrive, sel_keys;
    std::vector<SliceDesc> h_slices;
    DevBuf<float> qstat, qpart;     // frozen quantization statistics, build scratch
    DevBuf<uint32_t> wmask;         // decode-time maintenance: changed code words
    DevBuf<uint32_t> err_flags;     // explicit-selection validation (k_resolve_pages), kAttendErr*
    DevBuf<uint16_t> stage_q;
    DevBuf<float> stage_out;
    DevBuf<double> full_o, full_ml, full_stats;  // absp_full_attention: split partials, (M, L) per q row
    // absp_decode_step_host as one CUDA graph: H2D q -> step kernels -> D2H out; the
    // copy nodes are re-pointed when the caller's host buffers change
    cudaGraph_t host_graph = nullptr;  // kept: the exec's copy nodes are addressed through it
    cudaGraphExec_t host_exec = nullptr;
    cudaGraphNode_t h2d_node = nullptr, d2h_node = nullptr;
    const void* host_q = nullptr;
    float* host_out = nullptr;
    bool out_direct = false;  // the graph's attention writes host_out itself (mapped pinned memory)
    bool q_direct = false;    // the graph's selection reads host_q itself (mapped pinned memory)
    int host_launches = 0;
    void drop_host_graph() {
        if (host_exec) cudaGraphExecDestroy(host_exec);
        if (host_graph) cudaGraphDestroy(host_graph);
        host_exec = nullptr;
        host_graph = nullptr;
        host_q = nullptr;
        host_out = nullptr;
        out_direct = false;
        q_direct = false;
        h2d_node = d2h_node = nullptr;
    }

    void release() {
        d_desc.release(); d_items.release(); d_item_begin.release();
        values.release(); values_min.release(); scales.release(); zps.release();
        scales_min.release(); zps_min.release(); scores.release();
        codes.release(); codes_min.release();
        sel_blocks.release(); sel_counts.release(); ready.release(); scored.release(); topk_units.release();
        approx.release(); unit_err.release();
        sel_slices.release(); sel_slot.release(); sel_arrive.release(); sel_keys.release();
        h_slices.clear();
        qstat.release(); qpart.release(); wmask.release(); err_flags.release();
        stager.release();
        stage_q.release(); stage_out.release();
        full_o.release(); full_ml.release(); full_stats.release();
        drop_host_graph();
        step_work.release();
        for (auto& kv : attend_work) kv.second.release();
        attend_work.clear();
    }
};

}  // namespace

void absp::set_last_error(const std::string& msg) { g_err = msg; }

struct absp_ctx {
    int device = 0;
    int num_sms = 148;
    bool exact_select = false;  // ABSP_EXACT_SELECT=1: decode steps use the full exact scorer + top-k
    uint32_t host_copy = 0;     // ABSP_HOST_STEP_COPY (diagnostics): bit 0 q, bit 1 out through copy nodes
    absp_config cfg{};
    std::vector<Layer> layers;
    uint64_t launches = 0;
};

namespace {

uint32_t G_of(const absp_config& c) { return c.num_q_heads / c.num_kv_heads; }
uint32_t words_per_centroid(const absp_config& c) { return c.head_dim * c.quant_bits / 32; }

LayerView view_of(absp_ctx* ctx, Layer& l) {
    const absp_config& c = ctx->cfg;
    LayerView v{};
    v.H = c.num_kv_heads;
    v.G = G_of(c);
    v.D = c.head_dim;
    v.P = c.page_size;
    v.bits = c.quant_bits;
    v.mode = c.quant_mode;
    v.method = c.centroid_method;
    v.batch = l.batch;
    v.units = uint32_t(l.desc.size());
    v.max_pages = l.max_pages;
    v.pool_pages = l.pool_pages;
    v.k_pool = l.k_pool;
    v.v_pool = l.v_pool;
    v.page_table = l.page_table;
    v.desc = l.d_desc.p;
    v.values = l.values.p;
    v.values_min = l.values_min.p;
    v.codes = l.codes.p;
    v.codes_min = l.codes_min.p;
    v.scales = l.scales.p;
    v.zps = l.zps.p;
    v.scales_min = l.scales_min.p;
    v.zps_min = l.zps_min.p;
    v.scores = l.scores.p;
    v.qstat = l.qstat.p;
    v.qpart = l.qpart.p;
    v.wmask = l.wmask.p;
    return v;
}

absp_status get_layer(absp_ctx* ctx, uint32_t layer, Layer** out) {
    if (!ctx) return fail(ABSP_EINVAL, "null context");
    if (layer >= ctx->layers.size())
        return fail(ABSP_ERANGE, "layer " + std::to_string(layer) + " out of range (have " +
                                     std::to_string(ctx->layers.size()) + ")");
    *out = &ctx->layers[layer];
    return ABSP_OK;
}

// Attention chunks needed for a unit holding `entries` selected blocks.
uint32_t chunks_for(uint32_t entries, uint32_t block) {
    const uint32_t e = block >= kAttnChunkRows ? 1u : kAttnChunkRows / block;
    return ceil_div(entries, e);
}

// Builds the chunk list for units holding at most min(N, cap) entries (cap = K for
// decode, blocks_stride for explicit selections), the CTA runs of every unit under
// the persistent attention grid, and sizes the list's buffers. With `reserve` the
// buffers are sized for the layout at capacity (every unit at max_seq_len), so the
// appends that grow the list later never reallocate: device pointers stay fixed from
// kv_bind on (a unit's runs never exceed its chunks, so max_runs <= max chunks).
absp_status build_work(Layer& l, uint32_t D, uint32_t P, bool decode, uint32_t cap, int num_sms,
                       WorkList& wl, Stager* up = nullptr, bool reserve = false) {
    auto entries = [&](const UnitDesc& d, bool at_cap) {
        return std::min(at_cap ? std::max(d.n_blocks, d.cap) : d.n_blocks, decode ? d.budget : cap);
    };
    std::vector<uint32_t> base(l.desc.size() + 1, 0), unit_of, idx_of;
    uint64_t n_work_cap = 0;
    uint32_t max_chunks_cap = 1;
    for (size_t u = 0; u < l.desc.size(); ++u) {
        const UnitDesc& d = l.desc[u];
        const uint32_t ch = std::max(chunks_for(entries(d, false), d.block), 1u);
        base[u + 1] = base[u] + ch;
        unit_of.insert(unit_of.end(), ch, uint32_t(u));
        for (uint32_t c = 0; c < ch; ++c) idx_of.push_back(c);
        const uint32_t ch_cap = std::max(chunks_for(entries(d, reserve), d.block), ch);
        n_work_cap += ch_cap;
        max_chunks_cap = std::max(max_chunks_cap, ch_cap);
    }
    wl.n_work = base.back();
    wl.ns = kAttnChunkRows / P;  // page slots per chunk
    wl.grid = std::min<uint32_t>(wl.n_work, uint32_t(num_sms));
    // CTA c owns chunks [c * n_work / grid, (c + 1) * n_work / grid) (attend.cu)
    auto cta_of = [&](uint32_t w) {
        uint32_t c = uint32_t((uint64_t(w) * wl.grid) / wl.n_work);
        while (c + 1 < wl.grid && (uint64_t(c + 1) * wl.n_work) / wl.grid <= w) ++c;
        while (c > 0 && (uint64_t(c) * wl.n_work) / wl.grid > w) --c;
        return c;
    };
    std::vector<uint32_t> run(l.desc.size());
    wl.max_runs = 1;
    for (size_t u = 0; u < l.desc.size(); ++u) {
        const uint32_t first = cta_of(base[u]), last = cta_of(base[u + 1] - 1);
        if (first > 0xffffu) return fail(ABSP_EINVAL, "attention grid above 65535 CTAs");
        run[u] = first | ((last - first + 1) << 16);
        wl.max_runs = std::max(wl.max_runs, last - first + 1);
    }
    if (up && up->async && wl.chunk_base.p && base == wl.h_base && run == wl.h_run) return ABSP_OK;  // unchanged
    Stager sync_up;
    Stager& st = up ? *up : sync_up;
    const size_t n_slots = size_t(wl.n_work) * wl.ns;
    const size_t units = l.desc.size();
    const size_t slots_res = std::max<size_t>(n_slots, size_t(n_work_cap) * wl.ns);
    const size_t work_res = std::max<size_t>(wl.n_work, n_work_cap);
    const size_t runs_res = reserve ? std::max(wl.max_runs, std::min(max_chunks_cap, uint32_t(num_sms))) : wl.max_runs;
    const bool fresh = !wl.valid.p || wl.valid.n < slots_res;
    ABSP_CUDA(wl.page.ensure(slots_res));
    ABSP_CUDA(wl.valid.ensure(slots_res));
    ABSP_CUDA(st.zero(wl.valid.p, (fresh ? slots_res : n_slots) * 2));
    ABSP_CUDA(wl.chunk_unit.ensure(work_res));
    ABSP_CUDA(wl.chunk_idx.ensure(work_res));
    ABSP_CUDA(wl.chunk_base.ensure(base.size()));
    ABSP_CUDA(wl.unit_done.ensure(units));
    ABSP_CUDA(wl.unit_run.ensure(units));
    ABSP_CUDA(st.put(wl.chunk_unit.p, unit_of.data(), unit_of.size() * 4));
    ABSP_CUDA(st.put(wl.chunk_idx.p, idx_of.data(), idx_of.size() * 4));
    ABSP_CUDA(st.put(wl.chunk_base.p, base.data(), base.size() * 4));
    ABSP_CUDA(st.put(wl.unit_run.p, run.data(), run.size() * 4));
    ABSP_CUDA(st.zero(wl.unit_done.p, units * 4));
    wl.h_base = base;
    wl.h_run = run;
    ABSP_CUDA(wl.part_o.ensure(units * runs_res * 8 * D));
    ABSP_CUDA(wl.part_ml.ensure(units * runs_res * 16));
    return ABSP_OK;
}

AttendWork work_view(const WorkList& wl) {
    AttendWork w{};
    w.chunk_unit = wl.chunk_unit.p;
    w.chunk_idx = wl.chunk_idx.p;
    w.chunk_base = wl.chunk_base.p;
    w.unit_run = wl.unit_run.p;
    w.n_work = wl.n_work;
    w.max_runs = wl.max_runs;
    w.unit_done = wl.unit_done.p;
    w.grid = wl.grid;
    return w;
}

}  // namespace

// Units (capacity-reserved store segments), score work items, attention work list
// and device buffers of a bound layer for its current seq_lens; used by kv_bind and,
// after every sequence grew by a token, by absp_append (the store stays valid:
// segments are reserved for max_seq_len, so no growth moves another unit's data).
static absp_status layout_layer(absp_ctx* ctx, Layer* l, cudaStream_t stream = nullptr, bool async = false) {
    const absp_config& c = ctx->cfg;
    const uint32_t batch = l->batch;
    const uint32_t* seq_lens = l->seq_lens.data();
    absp_status st;
    const uint32_t H = c.num_kv_heads;
    l->desc.clear();
    l->items.clear();
    l->total_cap = 0;
    l->total_centroids = 0;
    l->max_cap = l->max_nblocks = l->max_budget = l->max_select = 0;
    for (uint32_t b = 0; b < batch; ++b) {
        for (uint32_t h = 0; h < H; ++h) {
            UnitDesc d{};
            d.seq = b;
            d.head = h;
            d.block = l->block_sizes[h];
            d.n_tokens = seq_lens[b];
            d.n_blocks = ceil_div(d.n_tokens, d.block);
            d.budget = ceil_div(c.token_budget, d.block);
            d.cap = ceil_div(c.max_seq_len, d.block);
            d.seg = l->total_cap;
            l->total_cap += d.cap;
            l->total_centroids += d.n_blocks;
            const uint32_t sel = std::min(d.n_blocks, d.budget);
            l->max_cap = std::max(l->max_cap, d.cap);
            l->max_nblocks = std::max(l->max_nblocks, d.n_blocks);
            l->max_budget = std::max(l->max_budget, d.budget);
            l->max_select = std::max(l->max_select, sel);
            l->desc.push_back(d);
        }
    }
    // Scoring split: contiguous ranges of the flattened centroids, cut into per-unit
    // items, balanced on rows + kItemCost per item (a CTA's item switch — table build and
    // pipeline bubble — costs about as much as ~256 rows, measured: tools/score_trace.py),
    // so CTAs end together whatever the block sizes (no partial last wave).
    {
        constexpr double kItemCost = 256.0;
        const uint32_t grid = uint32_t(std::max<uint64_t>(
            1, std::min<uint64_t>(uint64_t(ctx->num_sms) * kScoreCtasPerSm, l->total_centroids)));
        // CTAs the greedy cut needs at a per-CTA cost cap (writes the cut when `out`)
        auto cut = [&](double cap, bool out) -> uint64_t {
            uint64_t ctas = 0, pos = 0, ubase = 0;
            uint32_t u = 0;
            const uint64_t T = l->total_centroids;
            while (pos < T) {
                if (out) l->item_begin[ctas] = uint32_t(l->items.size());
                const bool last = out && ctas + 1 == grid;
                double cost = 0.0;
                bool any = false;
                while (pos < T) {
                    while (ubase + l->desc[u].n_blocks <= pos) ubase += l->desc[u++].n_blocks;
                    const double room = cap - cost - kItemCost;
                    if (!last && any && room < 1.0) break;
                    const uint64_t rem = ubase + l->desc[u].n_blocks - pos;
                    const uint64_t take = last ? rem : std::min<uint64_t>(rem, uint64_t(std::max(1.0, room)));
                    if (out) l->items.push_back({u, uint32_t(pos - ubase), uint32_t(pos - ubase + take), 0u});
                    pos += take;
                    cost += kItemCost + double(take);
                    any = true;
                    if (!last && cost >= cap) break;
                }
                ++ctas;
            }
            return ctas;
        };
        // per-CTA cost cap: the mean cost with one item per unit and one split per CTA
        // boundary, raised by 1 % until the cut fits the grid (typically 1-3 passes; this
        // runs on every append, so no bisection)
        double cap = (double(l->total_centroids) + kItemCost * double(l->desc.size() + grid)) / grid;
        while (cut(cap, false) > grid) cap *= 1.01;
        l->item_begin.assign(grid + 1, 0);
        const uint64_t used = cut(cap, true);
        for (uint64_t c = used; c < grid; ++c) l->item_begin[c] = uint32_t(l->items.size());  // idle CTAs
        l->item_begin[grid] = uint32_t(l->items.size());
    }
    const size_t units = l->desc.size();
    const size_t D = c.head_dim;
    const bool mm = c.centroid_method == ABSP_CENTROID_MAXMIN;
    const size_t W = words_per_centroid(c);
    ABSP_CUDA(l->d_desc.ensure(units));
    ABSP_CUDA(l->d_items.ensure(units + l->item_begin.size()));  // bound on items: appends never regrow it
    ABSP_CUDA(l->d_item_begin.ensure(l->item_begin.size()));
    ABSP_CUDA(l->values.ensure(l->total_cap * D));
    if (mm) ABSP_CUDA(l->values_min.ensure(l->total_cap * D));
    if (c.quant_bits) {
        ABSP_CUDA(l->codes.ensure(l->total_cap * W));
        ABSP_CUDA(l->scales.ensure(units * D));
        ABSP_CUDA(l->zps.ensure(units * D));
        if (mm) {
            ABSP_CUDA(l->codes_min.ensure(l->total_cap * W));
            ABSP_CUDA(l->scales_min.ensure(units * D));
            ABSP_CUDA(l->zps_min.ensure(units * D));
        }
        const size_t arrays = mm ? 2 : 1;
        const size_t slices = std::max<size_t>(1, ceil_div(l->max_cap, 256u));  // kStatRows
        ABSP_CUDA(l->qstat.ensure(arrays * units * 2 * D));
        ABSP_CUDA(l->qpart.ensure(arrays * units * slices * 2 * D));
        ABSP_CUDA(l->wmask.ensure(arrays * units));
    }
    ABSP_CUDA(l->scores.ensure(l->total_cap));
    ABSP_CUDA(l->approx.ensure(l->total_cap));
    ABSP_CUDA(l->unit_err.ensure(units));
    std::vector<SliceDesc> slices;
    l->sel_plan = plan_select(l->desc, l->max_budget, c.head_dim, ctx->num_sms, &slices);
    {
        const uint64_t bound = std::max<uint64_t>(select_slices_bound(l->desc), slices.size());
        ABSP_CUDA(l->sel_slices.ensure(bound));
        ABSP_CUDA(l->sel_slot.ensure(4 * bound));
        ABSP_CUDA(l->sel_arrive.ensure(units));
        ABSP_CUDA(l->sel_keys.ensure(l->total_cap + 8));  // + the TMA batches' 16-byte round-up
        if (!async) ABSP_CUDA(cudaMemset(l->sel_arrive.p, 0, units * 4));
    }
    l->sel_stride = ceil_div(c.token_budget, c.candidate_block_sizes[0]);
    ABSP_CUDA(l->sel_blocks.ensure(units * l->sel_stride));
    ABSP_CUDA(l->sel_counts.ensure(units));
    ABSP_CUDA(l->ready.ensure(units * kReadyStride));
    ABSP_CUDA(l->scored.ensure(units));
    if (!async) {  // zero between steps; the step kernels keep them so
        ABSP_CUDA(cudaMemset(l->ready.p, 0, units * kReadyStride * 4));
        ABSP_CUDA(cudaMemset(l->scored.p, 0, units * 4));
    }
    Stager& up = l->stager;
    if (!async) {  // bind: size the pinned upload ring for any later layout of this binding
        size_t n_work_cap = 0;
        for (const UnitDesc& d : l->desc)
            n_work_cap += std::max(chunks_for(std::min(std::max(d.n_blocks, d.cap), d.budget), d.block), 1u);
        const size_t bound = units * sizeof(UnitDesc) + (units + l->item_begin.size()) * sizeof(ScoreItem) +
                             l->item_begin.size() * 4 + units * 4 * 3 + 2 * n_work_cap * 4 + 8 * 16 + 4096 +
                             select_slices_bound(l->desc) * sizeof(SliceDesc) + 16;
        ABSP_CUDA(up.reserve(bound));
    }
    ABSP_CUDA(up.begin(stream, async));
    // top-k classes: split only when the largest unit needs the big register variants
    l->topk_classes = TopkClasses{};
    if (topk_items(l->max_nblocks) >= 32 || topk_items(l->max_nblocks) == 0) {
        static const uint32_t kItems[kTopkClasses] = {0, 64, 32, 16, 8, 4, 2, 1};  // largest first
        std::vector<uint32_t> order;
        for (int cls = 0; cls < kTopkClasses; ++cls) {
            l->topk_classes.items[cls] = kItems[cls];
            l->topk_classes.begin[cls] = uint32_t(order.size());
            for (uint32_t u = 0; u < units; ++u)
                if (topk_items(l->desc[u].n_blocks) == kItems[cls]) order.push_back(u);
        }
        l->topk_classes.begin[kTopkClasses] = uint32_t(order.size());
        ABSP_CUDA(l->topk_units.ensure(units));
        if (!async || order != l->h_topk_order) ABSP_CUDA(up.put(l->topk_units.p, order.data(), order.size() * 4));
        l->h_topk_order = order;
        l->topk_classes.units = l->topk_units.p;
    }
    if (!async || slices.size() != l->h_slices.size() ||
        std::memcmp(slices.data(), l->h_slices.data(), slices.size() * sizeof(SliceDesc)) != 0)
        ABSP_CUDA(up.put(l->sel_slices.p, slices.data(), slices.size() * sizeof(SliceDesc)));
    l->h_slices = slices;
    // explicit-selection work lists are rebuilt (in place) by their next absp_attend
    ++l->desc_version;
    st = build_work(*l, c.head_dim, c.page_size, true, 0, ctx->num_sms, l->step_work, &up, /*reserve=*/true);
    if (st != ABSP_OK) return st;
    ABSP_CUDA(up.put(l->d_desc.p, l->desc.data(), units * sizeof(UnitDesc)));
    ABSP_CUDA(up.put(l->d_items.p, l->items.data(), l->items.size() * sizeof(ScoreItem)));
    ABSP_CUDA(up.put(l->d_item_begin.p, l->item_begin.data(), l->item_begin.size() * 4));
    ABSP_CUDA(up.end());
    // the decode step's layout-dependent kernel arguments
    std::vector<uint64_t> key = {l->step_work.n_work, l->step_work.grid, l->step_work.max_runs,
                                 l->item_begin.size(), topk_items(l->max_nblocks), l->max_nblocks > 0,
                                 uint64_t(l->topk_classes.units != nullptr), l->sel_plan.n_slices,
                                 l->sel_plan.rows, l->sel_plan.stages, l->sel_plan.cand_cap, l->sel_plan.pg_cap};
    for (int cls = 0; cls <= kTopkClasses; ++cls) key.push_back(l->topk_classes.begin[cls]);
    if (key != l->step_key) {
        l->step_key = key;
        ++l->layout_version;
    }
    return ABSP_OK;
}

extern "C" {

int absp_abi_version(void) { return ABSP_ABI_VERSION; }

const char* absp_last_error(void) { return g_err.c_str(); }

absp_status absp_config_validate(const absp_config* cfg) {
    if (!cfg) return fail(ABSP_EINVAL, "null config");
    const absp_config& c = *cfg;
    // EngineConfig::validate, config.cpp:48-78 (same order, same messages)
    if (c.num_kv_heads == 0) return fail(ABSP_EINVAL, "num_heads must be positive");
    if (c.head_dim == 0) return fail(ABSP_EINVAL, "head_dim must be positive");
    if (c.page_size == 0) return fail(ABSP_EINVAL, "page_size must be >= 1");
    if (c.num_candidates == 0 || c.num_candidates > ABSP_MAX_CANDIDATES)
        return fail(ABSP_EINVAL, "candidate_block_sizes must not be empty");
    uint32_t maxc = 0;
    for (uint32_t i = 0; i < c.num_candidates; ++i) {
        const uint32_t b = c.candidate_block_sizes[i];
        if (b == 0 || b % c.page_size != 0)
            return fail(ABSP_EINVAL, "candidate block size " + std::to_string(b) +
                                         " is not a positive multiple of page_size " +
                                         std::to_string(c.page_size));
        maxc = std::max(maxc, b);
    }
    for (uint32_t i = 1; i < c.num_candidates; ++i) {
        if (c.candidate_block_sizes[i] < c.candidate_block_sizes[i - 1])
            return fail(ABSP_EINVAL, "candidate_block_sizes must be ascending");
        if (c.candidate_block_sizes[i] == c.candidate_block_sizes[i - 1])
            return fail(ABSP_EINVAL, "candidate_block_sizes must be distinct");
    }
    if (c.token_budget < maxc)
        return fail(ABSP_EINVAL, "token_budget must be >= the largest candidate block size");
    if (c.quant_bits != 0 && c.quant_bits != 2 && c.quant_bits != 4 && c.quant_bits != 8)
        return fail(ABSP_EINVAL, "quant bits must be one of {2, 4, 8}");
    if (c.quant_mode > 1) return fail(ABSP_EINVAL, "quant mode must be sym (0) or asym (1)");
    if (c.centroid_method > 1)
        return fail(ABSP_EINVAL, "unknown centroid method (expected mean|maxmin)");
    // Extensions and this build's kernel limits.
    if (c.num_q_heads == 0 || c.num_q_heads % c.num_kv_heads != 0)
        return fail(ABSP_EINVAL, "num_q_heads must be a positive multiple of num_kv_heads");
    if (G_of(c) > 8) return fail(ABSP_EINVAL, "GQA group size above 8 is not supported");
    if (c.head_dim != 64 && c.head_dim != 128)
        return fail(ABSP_EINVAL, "this build supports head_dim 64 or 128");
    if (maxc > kAttnChunkRows)
        return fail(ABSP_EINVAL, "block sizes above 128 are not supported by this build");
    // block sizes: any multiple of page_size up to 128 (the reference's rule, checked
    // above); pages: a power of two dividing the 128-row attention chunk
    if ((c.page_size & (c.page_size - 1)) || c.page_size > kAttnChunkRows)
        return fail(ABSP_EINVAL, "this build supports power-of-two page sizes up to 128 only");
    if (c.max_batch == 0 || c.max_seq_len == 0 || c.num_layers == 0)
        return fail(ABSP_EINVAL, "max_batch, max_seq_len and num_layers must be positive");
    const uint32_t minc = c.candidate_block_sizes[0];
    if (ceil_div(c.token_budget, minc) > 2048)
        return fail(ABSP_EINVAL, "token_budget / min block size above 2048 is not supported");
    if (ceil_div(c.max_seq_len, minc) > 131072)
        return fail(ABSP_EINVAL, "max_seq_len / min block size above 131072 is not supported");
    return ABSP_OK;
}

absp_status absp_ctx_create(int device, const absp_config* cfg, absp_ctx** out) {
    if (!out) return fail(ABSP_EINVAL, "null output pointer");
    *out = nullptr;
    absp_status st = absp_config_validate(cfg);
    if (st != ABSP_OK) return st;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    if (device < 0 || device >= ndev)
        return fail(ABSP_ERANGE, "device " + std::to_string(device) + " out of range");
    DeviceGuard dg(device);
    if (!dg.ok) return fail(ABSP_ECUDA, "cudaSetDevice failed");
    cudaDeviceProp prop{};
    ABSP_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(ABSP_ECUDA, "this library is built for sm_100a (B200); device is sm_" +
                                    std::to_string(prop.major) + std::to_string(prop.minor));
    ABSP_CUDA(init_attend_attributes());
    ABSP_CUDA(init_score_attributes());
    ABSP_CUDA(init_topk_attributes());
    ABSP_CUDA(init_select_attributes());
    auto* ctx = new absp_ctx;
    ctx->device = device;
    ctx->num_sms = prop.multiProcessorCount;
    const char* es = std::getenv("ABSP_EXACT_SELECT");
    ctx->exact_select = es && es[0] == '1';
    // diagnostics (tools/e2e_probe.py): host steps through copy nodes instead of the
    // kernels addressing pinned host buffers (bit 0: q, bit 1: out)
    const char* hc = std::getenv("ABSP_HOST_STEP_COPY");
    ctx->host_copy = hc ? uint32_t(std::atoi(hc)) & 3u : 0u;
    ctx->cfg = *cfg;
    ctx->layers.resize(cfg->num_layers);
    *out = ctx;
    return ABSP_OK;
}

absp_status absp_ctx_destroy(absp_ctx* ctx) {
    if (!ctx) return ABSP_OK;
    {
        DeviceGuard dg(ctx->device);
        for (Layer& l : ctx->layers) l.release();
    }
    delete ctx;
    return ABSP_OK;
}

absp_status absp_set_assignment(absp_ctx* ctx, uint32_t layer, const uint32_t* block_sizes) {
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    if (!block_sizes) return fail(ABSP_EINVAL, "null block_sizes");
    const absp_config& c = ctx->cfg;
    // BlockAssignment::validate, centroids.cpp:59-76
    for (uint32_t h = 0; h < c.num_kv_heads; ++h) {
        const uint32_t b = block_sizes[h];
        bool cand = false;
        for (uint32_t i = 0; i < c.num_candidates; ++i) cand |= c.candidate_block_sizes[i] == b;
        if (!cand)
            return fail(ABSP_EINVAL, "head " + std::to_string(h) + ": block size " +
                                         std::to_string(b) + " is not a candidate");
        if (b % c.page_size != 0)
            return fail(ABSP_EINVAL, "head " + std::to_string(h) + ": block size " +
                                         std::to_string(b) + " is not a multiple of page_size");
    }
    l->block_sizes.assign(block_sizes, block_sizes + c.num_kv_heads);
    l->drop_host_graph();
    l->assigned = true;
    l->bound = false;
    l->built = false;
    return ABSP_OK;
}

absp_status absp_kv_bind(absp_ctx* ctx, uint32_t layer, const void* k_pool, const void* v_pool,
                         uint64_t pool_pages, const uint32_t* page_table,
                         uint32_t max_pages_per_seq, const uint32_t* seq_lens, uint32_t batch) {
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    if (!l->assigned) return fail(ABSP_ESTATE, "kv_bind: call absp_set_assignment first");
    const absp_config& c = ctx->cfg;
    if (!k_pool || !v_pool || !page_table || !seq_lens)
        return fail(ABSP_EINVAL, "kv_bind: null pointer");
    if (batch == 0 || batch > c.max_batch)
        return fail(ABSP_EINVAL, "kv_bind: batch must be in 1..max_batch");
    if (pool_pages == 0) return fail(ABSP_EINVAL, "kv_bind: pool_pages must be positive");
    if (pool_pages * c.num_kv_heads > 0xffffffffull)
        return fail(ABSP_EINVAL, "kv_bind: num_kv_heads * pool_pages must fit in 32 bits");
    l->selected = false;
    uint32_t max_len = 0;
    for (uint32_t b = 0; b < batch; ++b) {
        if (seq_lens[b] == 0)
            return fail(ABSP_EINVAL, "compute_block_centroids: cache is empty (sequence " +
                                         std::to_string(b) + ")");
        if (seq_lens[b] > c.max_seq_len)
            return fail(ABSP_ECAPACITY, "kv cache at capacity (" + std::to_string(c.max_seq_len) +
                                            " tokens)");
        max_len = std::max(max_len, seq_lens[b]);
    }
    if (uint64_t(max_pages_per_seq) * c.page_size < max_len)
        return fail(ABSP_EINVAL, "kv_bind: page table shorter than the longest sequence");

    DeviceGuard dg(ctx->device);
    if (!dg.ok) return fail(ABSP_ECUDA, "cudaSetDevice failed");
    l->drop_host_graph();
    l->k_pool = static_cast<const uint16_t*>(k_pool);
    l->v_pool = static_cast<const uint16_t*>(v_pool);
    l->pool_pages = pool_pages;
    l->page_table = page_table;
    l->max_pages = max_pages_per_seq;
    l->batch = batch;
    l->seq_lens.assign(seq_lens, seq_lens + batch);

    st = layout_layer(ctx, l);
    if (st != ABSP_OK) return st;
    l->bound = true;
    l->built = false;
    return ABSP_OK;
}

absp_status absp_build_store(absp_ctx* ctx, uint32_t layer, void* stream) {
    NvtxRange nvtx_("absp_build_store");
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    if (!l->bound) return fail(ABSP_ESTATE, "build_store: call absp_kv_bind first");
    DeviceGuard dg(ctx->device);
    int n = 0;
    cudaError_t e = launch_build_store(view_of(ctx, *l), l->max_cap, cudaStream_t(stream), &n);
    ctx->launches += n;
    if (e != cudaSuccess) return cuda_fail(e, "build_store kernels");
    l->built = true;
    return ABSP_OK;
}

absp_status absp_append(absp_ctx* ctx, uint32_t layer, const void* k_new, const void* v_new, void* stream) {
    NvtxRange nvtx_("absp_append");
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    if (!l->built) return fail(ABSP_ESTATE, "step: call prefill first");  // engine.cpp:444
    if (!k_new || !v_new) return fail(ABSP_EINVAL, "append: null pointer");
    const absp_config& c = ctx->cfg;
    for (uint32_t b = 0; b < l->batch; ++b) {  // kv_cache.cpp:48-50
        if (l->seq_lens[b] >= c.max_seq_len)
            return fail(ABSP_ECAPACITY, "append: kv cache at capacity (" + std::to_string(c.max_seq_len) + " tokens)");
        if (l->seq_lens[b] >= uint64_t(l->max_pages) * c.page_size)
            return fail(ABSP_ECAPACITY, "append: page table of sequence " + std::to_string(b) + " is full");
    }
    DeviceGuard dg(ctx->device);
    const cudaStream_t s = cudaStream_t(stream);
    int n = 0;
    cudaError_t e = launch_append_rows(view_of(ctx, *l), static_cast<const uint16_t*>(k_new),
                                       static_cast<const uint16_t*>(v_new), s, &n);
    ctx->launches += n;
    if (e != cudaSuccess) return cuda_fail(e, "append kernel");
    for (uint32_t b = 0; b < l->batch; ++b) ++l->seq_lens[b];
    // the grown layout is uploaded on the stream, after the append kernel and before
    // the refresh (no host synchronisation; segments and work lists are capacity-
    // reserved, so nothing moves). The host-buffer step graph is re-captured only when
    // a kernel argument of the step changed.
    const uint64_t version = l->layout_version;
    st = layout_layer(ctx, l, s, true);
    if (st != ABSP_OK) return st;
    if (l->layout_version != version) l->drop_host_graph();
    n = 0;
    e = launch_refresh_store(view_of(ctx, *l), l->max_cap, s, &n);
    ctx->launches += n;
    if (e != cudaSuccess) return cuda_fail(e, "refresh_store kernels");
    l->selected = false;
    return ABSP_OK;
}

// Scoring + top-k; the top-k kernel also resolves the selection into the decode
// work list's page list, consumed by the attention producer. In the decode step
// (ready != null) it then raises the unit's ready flag, and the attention kernel
// starts on the unit right then.
static absp_status do_select(absp_ctx* ctx, Layer* l, const void* q, uint32_t* blocks, uint32_t stride,
                             uint32_t* counts, uint32_t* ready, cudaStream_t s) {
    const LayerView v = view_of(ctx, *l);
    int n = 0;
    // the table scorer publishes per-unit progress, so each unit's top-k starts on it
    uint32_t* scored = (v.bits == 2 || v.bits == 4) ? l->scored.p : nullptr;
    const ScoreWork sw{l->d_items.p, l->d_item_begin.p, uint32_t(l->item_begin.size() - 1), scored};
    cudaError_t e = launch_score(v, static_cast<const uint16_t*>(q), sw, s, &n);
    if (e == cudaSuccess)
        e = launch_topk(v, l->max_nblocks, l->max_budget, blocks, stride, counts, l->step_work.pages(), ready, scored,
                        l->topk_classes, s, &n);
    ctx->launches += n;
    if (e != cudaSuccess) return cuda_fail(e, "select kernels");
    return ABSP_OK;
}

// Attention over the layer's own selection buffers.
static absp_status do_attend_step(absp_ctx* ctx, Layer* l, const void* q, float* out, uint32_t* ready,
                                  cudaStream_t s) {
    int n = 0;
    cudaError_t e = launch_attend(view_of(ctx, *l), static_cast<const uint16_t*>(q), l->step_work.pages(), ready,
                                  work_view(l->step_work), l->step_work.part_o.p, l->step_work.part_ml.p, out, s, &n);
    ctx->launches += n;
    if (e != cudaSuccess) return cuda_fail(e, "attend kernels");
    return ABSP_OK;
}

absp_status absp_select(absp_ctx* ctx, uint32_t layer, const void* q, uint32_t* blocks,
                        uint32_t blocks_stride, uint32_t* counts, void* stream) {
    NvtxRange nvtx_("absp_select");
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    if (!l->built) return fail(ABSP_ESTATE, "select: call absp_build_store first");
    if (!q || !blocks || !counts) return fail(ABSP_EINVAL, "select: null pointer");
    if (blocks_stride < l->max_select)
        return fail(ABSP_EINVAL, "select: blocks_stride " + std::to_string(blocks_stride) +
                                     " < max_select " + std::to_string(l->max_select));
    DeviceGuard dg(ctx->device);
    st = do_select(ctx, l, q, blocks, blocks_stride, counts, nullptr, cudaStream_t(stream));
    if (st == ABSP_OK) l->selected = true;
    return st;
}

absp_status absp_attend(absp_ctx* ctx, uint32_t layer, const void* q, const uint32_t* blocks,
                        uint32_t blocks_stride, const uint32_t* counts, float* out, void* stream) {
    NvtxRange nvtx_("absp_attend");
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    if (!l->bound) return fail(ABSP_ESTATE, "attend: call absp_kv_bind first");
    if (!q || !blocks || !counts || !out) return fail(ABSP_EINVAL, "attend: null pointer");
    if (blocks_stride == 0) return fail(ABSP_EINVAL, "attend: blocks_stride must be positive");
    DeviceGuard dg(ctx->device);
    // Work list (with its own partials) for selections of up to min(N, blocks_stride)
    // entries per unit; built per stride on first use and rebuilt in place after the
    // layout changed (an append). Building allocates / uploads synchronously.
    WorkList& wl = l->attend_work[blocks_stride];
    if (wl.layout != l->desc_version) {
        st = build_work(*l, ctx->cfg.head_dim, ctx->cfg.page_size, false, blocks_stride, ctx->num_sms, wl);
        if (st != ABSP_OK) return st;
        wl.layout = l->desc_version;
    }
    if (!l->err_flags.p) {
        ABSP_CUDA(l->err_flags.ensure(1));
        ABSP_CUDA(cudaMemset(l->err_flags.p, 0, 4));
    }
    const LayerView v = view_of(ctx, *l);
    const cudaStream_t s = cudaStream_t(stream);
    int n = 0;
    cudaError_t e = launch_resolve_pages(v, blocks, blocks_stride, counts, wl.pages(), l->err_flags.p, s, &n);
    if (e == cudaSuccess)
        e = launch_attend(v, static_cast<const uint16_t*>(q), wl.pages(), nullptr, work_view(wl), wl.part_o.p,
                          wl.part_ml.p, out, s, &n);
    ctx->launches += n;
    if (e != cudaSuccess) return cuda_fail(e, "attend kernels");
    return ABSP_OK;
}

absp_status absp_attend_selected(absp_ctx* ctx, uint32_t layer, const void* q, float* out,
                                 void* stream) {
    NvtxRange nvtx_("absp_attend_selected");
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    if (!l->selected) return fail(ABSP_ESTATE, "attend_selected: no selection made on this layer");
    if (!q || !out) return fail(ABSP_EINVAL, "attend_selected: null pointer");
    DeviceGuard dg(ctx->device);
    return do_attend_step(ctx, l, q, out, nullptr, cudaStream_t(stream));
}

absp_status absp_attend_validate(absp_ctx* ctx, uint32_t layer, void* stream) {
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    if (!l->err_flags.p) return ABSP_OK;  // no explicit attention yet
    DeviceGuard dg(ctx->device);
    const cudaStream_t s = cudaStream_t(stream);
    uint32_t flags = 0;
    ABSP_CUDA(cudaMemcpyAsync(&flags, l->err_flags.p, 4, cudaMemcpyDeviceToHost, s));
    ABSP_CUDA(cudaMemsetAsync(l->err_flags.p, 0, 4, s));
    ABSP_CUDA(cudaStreamSynchronize(s));
    // the reference's messages (engine.cpp:224-226, kv_cache.cpp:125-127)
    if (flags & kAttendErrEmpty) return fail(ABSP_EINVAL, "sparse_attention: empty selection for a head");
    if (flags & kAttendErrCount) return fail(ABSP_EINVAL, "sparse_attention: selection count above blocks_stride");
    if (flags & kAttendErrBlock) return fail(ABSP_ERANGE, "block_to_pages: block index out of range");
    if (flags & kAttendErrPage) return fail(ABSP_ERANGE, "sparse_attention: page id outside the KV pools");
    return ABSP_OK;
}

absp_status absp_full_attention(absp_ctx* ctx, uint32_t layer, const void* q, float* out, double* weights,
                                uint64_t weights_stride, void* stream) {
    NvtxRange nvtx_("absp_full_attention");
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    if (!l->bound) return fail(ABSP_ESTATE, "full_attention: call absp_kv_bind first");
    if (!q || !out) return fail(ABSP_EINVAL, "full_attention: null pointer");
    uint32_t max_len = 0;
    for (uint32_t n : l->seq_lens) max_len = std::max(max_len, n);
    if (weights && weights_stride < max_len)
        return fail(ABSP_EINVAL, "full_attention: weights_stride " + std::to_string(weights_stride) +
                                     " < longest sequence " + std::to_string(max_len));
    const absp_config& c = ctx->cfg;
    DeviceGuard dg(ctx->device);
    const LayerView v = view_of(ctx, *l);
    const uint32_t splits = full_attention_splits(v.units, max_len, ctx->num_sms);
    const size_t parts = size_t(v.units) * splits * v.G;
    const size_t rows = size_t(l->batch) * c.num_q_heads;
    if (l->full_o.n < parts * c.head_dim || l->full_stats.n < rows * 2) {
        // first use (or a larger layout): allocation synchronises with the device
        ABSP_CUDA(cudaDeviceSynchronize());
        ABSP_CUDA(l->full_o.ensure(parts * c.head_dim));
        ABSP_CUDA(l->full_ml.ensure(parts * 2));
        ABSP_CUDA(l->full_stats.ensure(rows * 2));
    }
    int n = 0;
    cudaError_t e = launch_full_attention(v, static_cast<const uint16_t*>(q), splits, weights, weights_stride,
                                          l->full_o.p, l->full_ml.p, l->full_stats.p, out, cudaStream_t(stream), &n);
    ctx->launches += n;
    if (e != cudaSuccess) return cuda_fail(e, "full_attention kernels");
    return ABSP_OK;
}

absp_status absp_attention_recall(absp_ctx* ctx, uint32_t layer, const double* weights, uint64_t weights_stride,
                                  const uint32_t* blocks, uint32_t blocks_stride, const uint32_t* counts,
                                  double* recall, void* stream) {
    NvtxRange nvtx_("absp_attention_recall");
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    if (!l->bound) return fail(ABSP_ESTATE, "attention_recall: call absp_kv_bind first");
    if (!weights || !blocks || !counts || !recall) return fail(ABSP_EINVAL, "attention_recall: null pointer");
    uint32_t max_len = 0;
    for (uint32_t n : l->seq_lens) max_len = std::max(max_len, n);
    if (weights_stride < max_len || blocks_stride == 0)
        return fail(ABSP_EINVAL, "attention_recall: mismatched oracle/selection shapes");  // calibrator.cpp:51-55
    DeviceGuard dg(ctx->device);
    int n = 0;
    cudaError_t e = launch_recall(view_of(ctx, *l), l->max_nblocks, weights, weights_stride, blocks, blocks_stride,
                                  counts, recall, cudaStream_t(stream), &n);
    ctx->launches += n;
    if (e != cudaSuccess) return cuda_fail(e, "attention_recall kernel");
    return ABSP_OK;
}

uint64_t absp_layout_version(absp_ctx* ctx, uint32_t layer) {
    if (!ctx || layer >= ctx->layers.size()) return 0;
    return ctx->layers[layer].layout_version;
}

// The decode step's selection into the layer's own buffers: the fused kernel (or the
// exact scorer + top-k), resolving the page list; `ready` raises the per-unit flags the
// attention producer starts on (decode step only: its merges re-arm them).
static bool fused_step_select(absp_ctx* ctx, Layer* l) {
    return !ctx->exact_select && select_fused_supported(view_of(ctx, *l)) && l->sel_plan.ok;
}

static absp_status step_select(absp_ctx* ctx, Layer* l, const void* q, uint32_t* ready, cudaStream_t s,
                               uint16_t* q_copy = nullptr) {
    const LayerView v = view_of(ctx, *l);
    if (!ctx->exact_select && select_fused_supported(v) && l->sel_plan.ok) {
        // balanced slices: integer tensor-core filter, exact refine, top-k and page resolution
        int n = 0;
        const SelectWork sw{l->sel_slices.p, l->sel_slot.p, l->sel_arrive.p, l->sel_keys.p};
        cudaError_t e = launch_select_fused(v, static_cast<const uint16_t*>(q), l->sel_plan, sw, l->sel_blocks.p,
                                            l->sel_stride, l->sel_counts.p, l->step_work.pages(), ready,
                                            l->filter_diag ? l->approx.p : nullptr,
                                            l->filter_diag ? l->unit_err.p : nullptr, q_copy, s, &n);
        ctx->launches += n;
        if (e != cudaSuccess) return cuda_fail(e, "select kernel");
    } else {
        if (q_copy) return fail(ABSP_EINVAL, "decode step: host-resident q needs the fused selection");
        absp_status st = do_select(ctx, l, q, l->sel_blocks.p, l->sel_stride, l->sel_counts.p, ready, s);
        if (st != ABSP_OK) return st;
    }
    l->selected = true;
    return ABSP_OK;
}

absp_status absp_select_step(absp_ctx* ctx, uint32_t layer, const void* q, void* stream) {
    NvtxRange nvtx_("absp_select_step");
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    if (!l->built) return fail(ABSP_ESTATE, "select_step: call absp_build_store first");
    if (!q) return fail(ABSP_EINVAL, "select_step: null pointer");
    DeviceGuard dg(ctx->device);
    return step_select(ctx, l, q, nullptr, cudaStream_t(stream));
}

absp_status absp_decode_step(absp_ctx* ctx, uint32_t layer, const void* q, float* out,
                             void* stream) {
    NvtxRange nvtx_("absp_decode_step");
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    if (!l->built) return fail(ABSP_ESTATE, "decode_step: call absp_build_store first");
    if (!q || !out) return fail(ABSP_EINVAL, "decode_step: null pointer");
    DeviceGuard dg(ctx->device);
    const cudaStream_t s = cudaStream_t(stream);
    st = step_select(ctx, l, q, l->ready.p, s);
    if (st != ABSP_OK) return st;
    return do_attend_step(ctx, l, q, out, l->ready.p, s);
}

// Captures H2D q -> absp_decode_step -> D2H out of `layer` into a graph (host
// pointers as given; later calls re-point the copy nodes).
static absp_status capture_host_step(absp_ctx* ctx, uint32_t layer, Layer* l, const void* q_host, float* out_host,
                                     size_t nq) {
    cudaStream_t cap = nullptr;
    ABSP_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    cudaGraph_t graph = nullptr;
    const uint64_t before = ctx->launches;
    // Pinned host output the device can address (UVA, same pointer): the attention's LSE
    // merges write it directly, unit by unit as they complete, instead of a copy after
    // the kernel. Otherwise (pageable, or not device-addressable) a D2H copy node.
    cudaPointerAttributes pa{};
    const bool direct = !(ctx->host_copy & 2u) && cudaPointerGetAttributes(&pa, out_host) == cudaSuccess &&
                        pa.type == cudaMemoryTypeHost && pa.devicePointer == out_host;
    cudaGetLastError();
    // Likewise a device-addressable pinned q: the selection kernel reads it over PCIe
    // (one TMA copy of a unit's G rows per slice) and its finalizing CTAs leave each
    // unit's rows in stage_q for the attention, so there is no copy before the step.
    const bool q_direct = !(ctx->host_copy & 1u) && fused_step_select(ctx, l) && cudaPointerGetAttributes(&pa, q_host) == cudaSuccess &&
                          pa.type == cudaMemoryTypeHost && pa.devicePointer == q_host;
    cudaGetLastError();
    cudaError_t e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
    absp_status st = ABSP_OK;
    if (e == cudaSuccess && q_direct) {
        float* o = direct ? out_host : l->stage_out.p;
        st = step_select(ctx, l, q_host, l->ready.p, cap, l->stage_q.p);
        if (st == ABSP_OK) st = do_attend_step(ctx, l, l->stage_q.p, o, l->ready.p, cap);
        if (st == ABSP_OK && !direct)
            e = cudaMemcpyAsync(out_host, l->stage_out.p, nq * sizeof(float), cudaMemcpyDeviceToHost, cap);
        const cudaError_t e2 = cudaStreamEndCapture(cap, &graph);
        if (e == cudaSuccess) e = e2;
    } else if (e == cudaSuccess) {
        e = cudaMemcpyAsync(l->stage_q.p, q_host, nq * sizeof(uint16_t), cudaMemcpyHostToDevice, cap);
        if (e == cudaSuccess) st = absp_decode_step(ctx, layer, l->stage_q.p, direct ? out_host : l->stage_out.p, cap);
        if (e == cudaSuccess && st == ABSP_OK && !direct)
            e = cudaMemcpyAsync(out_host, l->stage_out.p, nq * sizeof(float), cudaMemcpyDeviceToHost, cap);
        const cudaError_t e2 = cudaStreamEndCapture(cap, &graph);
        if (e == cudaSuccess) e = e2;
    }
    l->host_launches = int(ctx->launches - before);
    ctx->launches = before;  // counted when the graph runs
    if (e == cudaSuccess && st == ABSP_OK) {
        size_t n = 0;
        e = cudaGraphGetNodes(graph, nullptr, &n);
        std::vector<cudaGraphNode_t> nodes(n);
        if (e == cudaSuccess) e = cudaGraphGetNodes(graph, nodes.data(), &n);
        for (size_t i = 0; e == cudaSuccess && i < n; ++i) {
            cudaGraphNodeType t;
            e = cudaGraphNodeGetType(nodes[i], &t);
            if (e != cudaSuccess || t != cudaGraphNodeTypeMemcpy) continue;
            cudaMemcpy3DParms p{};
            e = cudaGraphMemcpyNodeGetParams(nodes[i], &p);
            if (p.kind == cudaMemcpyHostToDevice) l->h2d_node = nodes[i];
            else if (p.kind == cudaMemcpyDeviceToHost) l->d2h_node = nodes[i];
        }
        if (e == cudaSuccess && ((!q_direct && !l->h2d_node) || (!direct && !l->d2h_node))) e = cudaErrorInvalidValue;
        if (e == cudaSuccess) e = cudaGraphInstantiate(&l->host_exec, graph, 0);
    }
    cudaStreamDestroy(cap);
    if (st == ABSP_OK && e == cudaSuccess) {
        l->host_graph = graph;
    } else if (graph) {
        cudaGraphDestroy(graph);
    }
    if (st != ABSP_OK) return st;
    if (e != cudaSuccess) {
        l->host_exec = nullptr;
        cudaGetLastError();  // clear; the caller runs the step eagerly
        return ABSP_ECUDA;
    }
    l->host_q = q_host;
    l->host_out = out_host;
    l->out_direct = direct;
    l->q_direct = q_direct;
    return ABSP_OK;
}

absp_status absp_decode_step_host(absp_ctx* ctx, uint32_t layer, const void* q_host,
                                  float* out_host, void* stream) {
    NvtxRange nvtx_("absp_decode_step_host");
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    if (!l->built) return fail(ABSP_ESTATE, "decode_step: call absp_build_store first");
    if (!q_host || !out_host) return fail(ABSP_EINVAL, "decode_step_host: null pointer");
    DeviceGuard dg(ctx->device);
    const absp_config& c = ctx->cfg;
    const size_t nq = size_t(l->batch) * c.num_q_heads * c.head_dim;
    ABSP_CUDA(l->stage_q.ensure(nq));
    ABSP_CUDA(l->stage_out.ensure(nq));
    const cudaStream_t s = cudaStream_t(stream);
    if (!l->host_exec && capture_host_step(ctx, layer, l, q_host, out_host, nq) != ABSP_OK)
        l->drop_host_graph();
    if (l->host_exec && ((l->out_direct && out_host != l->host_out) || (l->q_direct && q_host != l->host_q))) {
        // a host buffer the graph's kernels address directly changed: re-capture
        l->drop_host_graph();
        if (capture_host_step(ctx, layer, l, q_host, out_host, nq) != ABSP_OK) l->drop_host_graph();
    }
    bool graph_ok = l->host_exec != nullptr;
    if (graph_ok && (q_host != l->host_q || out_host != l->host_out)) {
        // re-point the copy nodes; buffers the graph cannot take (e.g. pageable memory
        // after pinned) run this call eagerly and keep the graph as it is
        cudaError_t e = l->q_direct ? cudaSuccess
                                    : cudaGraphExecMemcpyNodeSetParams1D(l->host_exec, l->h2d_node, l->stage_q.p,
                                                                         q_host, nq * sizeof(uint16_t),
                                                                         cudaMemcpyHostToDevice);
        if (e == cudaSuccess && !l->out_direct)
            e = cudaGraphExecMemcpyNodeSetParams1D(l->host_exec, l->d2h_node, out_host, l->stage_out.p,
                                                   nq * sizeof(float), cudaMemcpyDeviceToHost);
        if (e == cudaSuccess) {
            l->host_q = q_host;
            l->host_out = out_host;
        } else {
            cudaGetLastError();
            // the nodes may be half re-pointed: restore them for the next call
            if ((!l->q_direct &&
                 cudaGraphExecMemcpyNodeSetParams1D(l->host_exec, l->h2d_node, l->stage_q.p, l->host_q,
                                                    nq * sizeof(uint16_t), cudaMemcpyHostToDevice) != cudaSuccess) ||
                (!l->out_direct &&
                 cudaGraphExecMemcpyNodeSetParams1D(l->host_exec, l->d2h_node, l->host_out, l->stage_out.p,
                                                    nq * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess)) {
                cudaGetLastError();
                l->drop_host_graph();
            }
            graph_ok = false;
        }
    }
    if (graph_ok) {
        ABSP_CUDA(cudaGraphLaunch(l->host_exec, s));
        ctx->launches += uint64_t(l->host_launches);
        l->selected = true;
    } else {  // graph capture unavailable (e.g. pageable host memory): eager launches
        ABSP_CUDA(cudaMemcpyAsync(l->stage_q.p, q_host, nq * sizeof(uint16_t), cudaMemcpyHostToDevice, s));
        st = absp_decode_step(ctx, layer, l->stage_q.p, l->stage_out.p, stream);
        if (st != ABSP_OK) return st;
        ABSP_CUDA(cudaMemcpyAsync(out_host, l->stage_out.p, nq * sizeof(float), cudaMemcpyDeviceToHost, s));
    }
    ABSP_CUDA(cudaStreamSynchronize(s));
    return ABSP_OK;
}

absp_status absp_last_selection(absp_ctx* ctx, uint32_t layer, const uint32_t** blocks,
                                uint32_t* blocks_stride, const uint32_t** counts) {
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    if (!l->bound) return fail(ABSP_ESTATE, "last_selection: layer not bound");
    if (blocks) *blocks = l->sel_blocks.p;
    if (blocks_stride) *blocks_stride = l->sel_stride;
    if (counts) *counts = l->sel_counts.p;
    return ABSP_OK;
}

absp_status absp_get_layer_info(absp_ctx* ctx, uint32_t layer, absp_layer_info* info) {
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    if (!info) return fail(ABSP_EINVAL, "null info");
    if (!l->bound) return fail(ABSP_ESTATE, "layer_info: layer not bound");
    const absp_config& c = ctx->cfg;
    *info = absp_layer_info{};
    info->batch = l->batch;
    info->max_select = l->max_select;
    info->total_centroids = l->total_centroids;
    const uint64_t W = words_per_centroid(c);
    const bool mm = c.centroid_method == ABSP_CENTROID_MAXMIN;
    const uint64_t units = l->desc.size();
    info->store_bytes = l->total_cap * c.head_dim * 4 * (mm ? 2 : 1) +
                        (c.quant_bits ? (l->total_cap * W * 4 + units * c.head_dim * 8) * (mm ? 2 : 1) : 0);
    info->code_bytes = c.quant_bits ? l->total_centroids * c.head_dim * c.quant_bits / 8 * (mm ? 2 : 1)
                                    : l->total_centroids * c.head_dim * 4 * (mm ? 2 : 1);
    uint64_t kv = 0;
    for (const UnitDesc& d : l->desc) {
        const uint32_t sel = std::min(d.n_blocks, d.budget);
        // rows attended: all full blocks except possibly the trailing partial one
        const uint64_t trailing = d.n_tokens - uint64_t(d.n_blocks - 1) * d.block;
        const uint64_t rows = uint64_t(sel - 1) * d.block + trailing;
        kv += rows * c.head_dim * 2 * 2;
    }
    info->kv_bytes_selected = kv;
    return ABSP_OK;
}

absp_status absp_download_store(absp_ctx* ctx, uint32_t layer, uint32_t seq, uint64_t* offsets,
                                float* values, float* values_min, uint8_t* codes,
                                uint8_t* codes_min, float* scales, float* zps, float* scales_min,
                                float* zps_min) {
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    if (!l->built) return fail(ABSP_ESTATE, "download_store: store not built");
    if (seq >= l->batch) return fail(ABSP_ERANGE, "download_store: sequence out of range");
    DeviceGuard dg(ctx->device);
    ABSP_CUDA(cudaDeviceSynchronize());
    const absp_config& c = ctx->cfg;
    const uint32_t H = c.num_kv_heads, D = c.head_dim, W = words_per_centroid(c);
    const bool mm = c.centroid_method == ABSP_CENTROID_MAXMIN;
    uint64_t off = 0;
    if (offsets) offsets[0] = 0;
    std::vector<uint32_t> words;
    for (uint32_t h = 0; h < H; ++h) {
        const UnitDesc& d = l->desc[size_t(seq) * H + h];
        const uint32_t u = seq * H + h;
        const size_t n = d.n_blocks;
        if (values) ABSP_CUDA(cudaMemcpy(values + off * D, l->values.p + d.seg * D, n * D * 4, cudaMemcpyDeviceToHost));
        if (values_min && mm)
            ABSP_CUDA(cudaMemcpy(values_min + off * D, l->values_min.p + d.seg * D, n * D * 4, cudaMemcpyDeviceToHost));
        if (c.quant_bits) {
            const int bits = int(c.quant_bits), cpw = 32 / bits;
            for (int a = 0; a < (mm ? 2 : 1); ++a) {
                uint8_t* dst = a ? codes_min : codes;
                if (!dst) continue;
                const uint32_t* src = (a ? l->codes_min.p : l->codes.p) + d.seg * W;
                words.resize(size_t(W) * n);
                ABSP_CUDA(cudaMemcpy(words.data(), src, words.size() * 4, cudaMemcpyDeviceToHost));
                for (size_t i = 0; i < n; ++i)
                    for (uint32_t ch = 0; ch < D; ++ch) {
                        const uint32_t w = words[i * W + code_word_pos(uint32_t(i), ch / cpw, W)];
                        dst[(off + i) * D + ch] = uint8_t((w >> ((ch % cpw) * bits)) & ((1u << bits) - 1u));
                    }
            }
            if (scales) ABSP_CUDA(cudaMemcpy(scales + size_t(h) * D, l->scales.p + size_t(u) * D, D * 4, cudaMemcpyDeviceToHost));
            if (zps) ABSP_CUDA(cudaMemcpy(zps + size_t(h) * D, l->zps.p + size_t(u) * D, D * 4, cudaMemcpyDeviceToHost));
            if (mm && scales_min)
                ABSP_CUDA(cudaMemcpy(scales_min + size_t(h) * D, l->scales_min.p + size_t(u) * D, D * 4, cudaMemcpyDeviceToHost));
            if (mm && zps_min)
                ABSP_CUDA(cudaMemcpy(zps_min + size_t(h) * D, l->zps_min.p + size_t(u) * D, D * 4, cudaMemcpyDeviceToHost));
        }
        off += n;
        if (offsets) offsets[h + 1] = off;
    }
    return ABSP_OK;
}

absp_status absp_download_selection(absp_ctx* ctx, uint32_t layer, uint32_t* blocks, uint32_t* counts) {
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    if (!l->bound) return fail(ABSP_ESTATE, "download_selection: layer not bound");
    if (!blocks || !counts) return fail(ABSP_EINVAL, "download_selection: null pointer");
    DeviceGuard dg(ctx->device);
    ABSP_CUDA(cudaDeviceSynchronize());
    const size_t units = l->desc.size();
    ABSP_CUDA(cudaMemcpy(blocks, l->sel_blocks.p, units * l->sel_stride * 4, cudaMemcpyDeviceToHost));
    ABSP_CUDA(cudaMemcpy(counts, l->sel_counts.p, units * 4, cudaMemcpyDeviceToHost));
    return ABSP_OK;
}

absp_status absp_set_filter_diagnostics(absp_ctx* ctx, uint32_t layer, int enable) {
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    l->filter_diag = enable != 0;
    l->drop_host_graph();
    return ABSP_OK;
}

absp_status absp_download_filter_scores(absp_ctx* ctx, uint32_t layer, uint32_t seq, float* approx,
                                        float* err) {
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    if (!l->built) return fail(ABSP_ESTATE, "download_filter_scores: store not built");
    if (seq >= l->batch) return fail(ABSP_ERANGE, "download_filter_scores: sequence out of range");
    if (!approx || !err) return fail(ABSP_EINVAL, "null pointer");
    DeviceGuard dg(ctx->device);
    ABSP_CUDA(cudaDeviceSynchronize());
    const uint32_t H = ctx->cfg.num_kv_heads;
    uint64_t off = 0;
    for (uint32_t h = 0; h < H; ++h) {
        const UnitDesc& d = l->desc[size_t(seq) * H + h];
        ABSP_CUDA(cudaMemcpy(approx + off, l->approx.p + d.seg, size_t(d.n_blocks) * 4, cudaMemcpyDeviceToHost));
        ABSP_CUDA(cudaMemcpy(err + h, l->unit_err.p + size_t(seq) * H + h, 4, cudaMemcpyDeviceToHost));
        off += d.n_blocks;
    }
    return ABSP_OK;
}

absp_status absp_download_scores(absp_ctx* ctx, uint32_t layer, uint32_t seq, float* scores) {
    Layer* l;
    absp_status st = get_layer(ctx, layer, &l);
    if (st != ABSP_OK) return st;
    if (!l->built) return fail(ABSP_ESTATE, "download_scores: store not built");
    if (seq >= l->batch) return fail(ABSP_ERANGE, "download_scores: sequence out of range");
    if (!scores) return fail(ABSP_EINVAL, "null scores");
    DeviceGuard dg(ctx->device);
    ABSP_CUDA(cudaDeviceSynchronize());
    const uint32_t H = ctx->cfg.num_kv_heads;
    uint64_t off = 0;
    for (uint32_t h = 0; h < H; ++h) {
        const UnitDesc& d = l->desc[size_t(seq) * H + h];
        ABSP_CUDA(cudaMemcpy(scores + off, l->scores.p + d.seg, size_t(d.n_blocks) * 4, cudaMemcpyDeviceToHost));
        off += d.n_blocks;
    }
    return ABSP_OK;
}

absp_status absp_fill_synthetic_bf16(void* dst, uint64_t count, uint64_t seed, uint64_t stream_id,
                                     void* stream) {
    if (!dst && count) return fail(ABSP_EINVAL, "null destination");
    cudaError_t e = launch_fill_synth(static_cast<uint16_t*>(dst), count, seed, stream_id,
                                      cudaStream_t(stream));
    if (e != cudaSuccess) return cuda_fail(e, "fill_synthetic");
    return ABSP_OK;
}

uint64_t absp_launch_count(absp_ctx* ctx) { return ctx ? ctx->launches : 0; }

}  // extern "C"

#ifdef ABSP_ATTN_TRACE
// Debug builds only (not part of include/absp.h): copy the attention timeline
// stamps (uint64 globaltimer ns, [160 CTAs][256 slots]) to host memory.
namespace absp {
cudaError_t debug_attn_trace(void* dst, size_t bytes);
cudaError_t debug_score_trace(void* dst, size_t bytes);
cudaError_t debug_topk_trace(void* dst, size_t bytes);
cudaError_t debug_select_trace(void* dst, size_t bytes);
}
extern "C" absp_status absp_debug_select_trace(void* dst, size_t bytes) {
    cudaError_t e = absp::debug_select_trace(dst, bytes);
    return e == cudaSuccess ? ABSP_OK : cuda_fail(e, "debug_select_trace");
}
extern "C" absp_status absp_debug_topk_trace(void* dst, size_t bytes) {
    cudaError_t e = absp::debug_topk_trace(dst, bytes);
    return e == cudaSuccess ? ABSP_OK : cuda_fail(e, "debug_topk_trace");
}
extern "C" absp_status absp_debug_score_trace(void* dst, size_t bytes) {
    cudaError_t e = absp::debug_score_trace(dst, bytes);
    return e == cudaSuccess ? ABSP_OK : cuda_fail(e, "debug_score_trace");
}
extern "C" absp_status absp_debug_attn_trace(void* dst, size_t bytes) {
    cudaError_t e = absp::debug_attn_trace(dst, bytes);
    return e == cudaSuccess ? ABSP_OK : cuda_fail(e, "debug_attn_trace");
}
#endif
