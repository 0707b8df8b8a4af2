// decode.cu — host side of the libmc decode path (sm_100a, B200): argument checks, launch
// planning, cone culling, the pipelined host decode and the C ABI entry points.  The kernel
// family itself is decode_kernel.cuh, instantiated per codec x stats in decode_inst.cu.
//
// Paper: arXiv 2404.06359 §4.2–4.4.  A GROUP of G lanes (8, 16 or 32 by meshlet size)
// decodes one meshlet record (FORMAT.md) at a time; groups claim records in global order
// from interleaved device counters.  Per record:
//
//   a1/a2  the record (header + L/R flags + increment flags + bytes + packed
//          attributes) is staged HBM -> shared memory with ONE TMA 1-D bulk copy
//          (cp.async.bulk ... mbarrier::complete_tx), double-buffered per group so
//          record i+1 is in flight while record i decodes;
//   a3     index expansion: per-word __popc of the increment flags, an exclusive group
//          scan over the record's <= KW words (__shfl), then
//          N[t+2] = i_t ? 2 + c_t : reuse[t - c_t - 1]      ("countbits");
//   a4     L/R lookback by bit scan: j(t) = max{k<t: f_k != f_t} via
//          31 - __clz((f_t ? ~w : w) & below(t)) in the current word, earlier words
//          through per-word last-R / last-L max-scans ("firstbithigh");
//   a5     triangle assembly with winding-preserving orientation (FORMAT.md §2);
//   a6     index words stored directly (3 x u32 per lane, streaming .cs stores), or one
//          local u8x4 word per triangle;
//   a7/a8  attribute unpack (aligned halfwords at b = 16; compile-time shifts of word-aligned
//          vertex units when every channel has one width; else a funnel-shift bit reader),
//          q = L + code, fp32 via __fmaf_rn(__uint2float_rn(q), Δ, g),
//          octahedral normals with IEEE-exact sqrt/reciprocal (FORMAT.md §4.3);
//   a9     vertex words stored with 128-bit stores (direct when n_out % 4 == 0,
//          else through the phase-aligned smem stage);
//   a10    (stats kernel only) checksums/counters, group-reduced, one atomic per group.
//
// No tensor cores: the path is integer bit manipulation plus one FMA per channel, bound by
// HBM bandwidth.  No --use_fast_math.  Compile-time knobs (defaults = the
// measured optimum on B200; A/B logs in profiles/experiments and profiles/round2/experiments;
// scripts/build_variants.sh builds alternatives) are listed in decode_kernel.cuh.
#include "decode_kernel.cuh"

#include <cuda_runtime.h>

namespace mcdec {
mc_status dispatch_gts(bool stats, int lay, int am, const Params& P, size_t smem, cudaStream_t s) {
    return stats ? dispatch_gts_stats(lay, am, P, smem, s) : dispatch_gts_plain(lay, am, P, smem, s);
}
mc_status dispatch_reuse(bool stats, int lay, int am, const Params& P, size_t smem, cudaStream_t s) {
    return stats ? dispatch_reuse_stats(lay, am, P, smem, s) : dispatch_reuse_plain(lay, am, P, smem, s);
}
mc_status dispatch_basic(bool stats, int lay, int am, const Params& P, size_t smem, cudaStream_t s) {
    return stats ? dispatch_basic_stats(lay, am, P, smem, s) : dispatch_basic_plain(lay, am, P, smem, s);
}
}  // namespace mcdec

namespace {
using namespace mcdec;

__global__ void stats_reset_kernel(mc_stats* s) {
    if (threadIdx.x == 0) {
        s->checksum_indices = s->checksum_vertices = s->checksum_quantized = 0;
        s->triangles = s->degenerate = s->vertices = s->multiword_lookbacks = 0;
        s->max_lookback = 0;
        s->error_bits = 0;
        s->first_bad_meshlet = 0xFFFFFFFFu;
        s->num_bad = 0;
    }
}

// ------------------------------------------------------------------ cone culling (FORMAT.md §1.5, §7)
// The paper's amplification-shader pass: per record, the binary32 cone test
// fmaf(az,dz, fmaf(ay,dy, ax*dx)) > cutoff and a one-pass decoupled look-back scan that
// lists the visible records in record order with their compacted output bases
// (cull_scan_tile, decode_kernel.cuh).  Default (MC_CULL_FUSED): the decode kernel runs the
// scan itself before decoding the list — one launch.  Otherwise this standalone scan kernel
// runs first and the decode kernel walks its list: two launches.
constexpr uint32_t kCullThreads = 256, kCullTile = kCullThreads * kCullPerThread;

__global__ void __launch_bounds__(kCullThreads) cull_scan_kernel(const CullScan C) {
    __shared__ uint4 sh[8], pair[2];
    __shared__ uint32_t s_tile, s_last;
    if (threadIdx.x == 0) s_tile = atomicAdd(C.ctr, 1u);     // tiles in CTA start order
    __syncthreads();
    cull_scan_tile(C, s_tile, sh, pair);
    // leave the scratch zeroed: the last CTA clears flags and tickets
    if (threadIdx.x == 0) s_last = atomicAdd(C.ctr + 2, 1u) == C.tiles - 1 ? 1u : 0u;
    __syncthreads();
    if (s_last) cull_scan_reset(C);
}

// ------------------------------------------------------------------ host launch
mc_status build_params(const mc_decode_args* a, mc_stats* st, Params& P, size_t& smem) {
    if (!a || !a->layout) return MC_ERR_ARG;
    const mc_layout& L = *a->layout;
    if ((uint64_t)a->first + a->count > L.num_meshlets) return MC_ERR_ARG;
    if (a->count == 0) return MC_OK;                  // nothing to decode (outputs may be empty)
    if (!a->d_blob || !a->d_indices) return MC_ERR_ARG;
    if (reinterpret_cast<uintptr_t>(a->d_blob) & 15u) return MC_ERR_ARG;
    if ((reinterpret_cast<uintptr_t>(a->d_indices) & 3u) || (reinterpret_cast<uintptr_t>(a->d_vertices) & 15u) ||
        (reinterpret_cast<uintptr_t>(a->d_quantized) & 3u))
        return MC_ERR_ARG;
    if (L.n < 1 || L.n > 16 || L.max_record_bytes == 0 || (L.max_record_bytes & 15u)) return MC_ERR_FORMAT;
    const uint8_t* blob = static_cast<const uint8_t*>(a->d_blob);
    P.rec = blob + L.off_rec;
    P.dir = reinterpret_cast<const uint32_t*>(blob + L.off_dir);
    P.objtab = reinterpret_cast<const float*>(blob + L.off_obj);
    P.rec_section_bytes = L.total_bytes - L.off_rec;
    P.first = a->first;
    P.end = a->first + a->count;
    P.O = L.num_objects;
    P.vmax = L.v_max;
    P.tmax = L.t_max;
    P.n = L.n;
    P.n_out = L.n_out;
    P.S = L.S;
    P.max_rec = L.max_record_bytes;
    P.base_vtx = L.base_vtx;
    P.base_tri = L.base_tri;
    P.total_v = L.total_v;
    P.total_tp = L.total_tp;
    if (a->flags & ~(uint32_t)(MC_DECODE_BLOB_LOCAL_INDICES | MC_DECODE_INDEX_LOCAL_U8X4)) return MC_ERR_ARG;
    P.index_sub = (a->flags & MC_DECODE_BLOB_LOCAL_INDICES) ? L.base_vtx : 0u;
    P.u8x4 = (a->flags & MC_DECODE_INDEX_LOCAL_U8X4) ? 1u : 0u;
    P.vw = L.flags & 1u;
    P.list = nullptr;
    P.list_count = nullptr;
    if (reinterpret_cast<uintptr_t>(a->d_work) & 3u) return MC_ERR_ARG;
    P.ctr = a->d_work;   // launch_g falls back to the library pool when null
    P.hdr_words = ((16u + 4u * L.n + (P.vw ? L.n : 0u) + 15u) & ~15u) / 4u;
    P.buf_words = L.max_record_bytes / 4u + 4u;
    P.vtx_stage_words = 0;
    P.idx_stage_words = 0;
    P.idx = a->d_indices;
    P.fout = a->d_vertices;
    P.fout32 = (reinterpret_cast<uintptr_t>(a->d_vertices) & 31u) == 0u;   // 256-bit vertex stores
    P.pair16 = 1;   // every channel at most 16 bits wide (VW widths w_c <= b_c)
    for (uint32_t c = 0; c < L.n; ++c) P.pair16 &= L.bits[c] <= 16u ? 1u : 0u;
    P.qout = a->d_quantized;
    P.stats = st;
    uint32_t off = 0, col = 0;
    for (uint32_t c = 0; c < 16; ++c) { P.bits[c] = 0; P.bitoff[c] = 0; P.col[c] = 0; P.oct[c] = 0; }
    for (uint32_t c = 0; c < L.n; ++c) {
        P.bits[c] = L.bits[c];
        P.bitoff[c] = (uint8_t)off;
        off += L.bits[c];
        P.col[c] = (uint8_t)col;
        if (L.semantic[c] == MC_SEM_NORMAL_OCT) {
            P.oct[c] = 1;
            P.bits[c + 1] = L.bits[c + 1];
            P.bitoff[c + 1] = (uint8_t)off;
            off += L.bits[c + 1];
            P.col[c + 1] = (uint8_t)(col + 1);
            col += 3;
            ++c;
        } else {
            col += 1;
        }
    }
    smem = 0;   // per group, set by launch() once the vertex stage is known
    return MC_OK;
}

constexpr int kMaxDevices = 64;

mc_status dispatch_codec(uint32_t codec, bool stats, int lay, int am, const Params& P, size_t smem, cudaStream_t s) {
    if (codec == MC_CODEC_GTS) return dispatch_gts(stats, lay, am, P, smem, s);
    if (codec == MC_CODEC_BASIC) return dispatch_basic(stats, lay, am, P, smem, s);
    return dispatch_reuse(stats, lay, am, P, smem, s);
}

mc_status launch(const mc_decode_args* a, mc_stats* st, cudaStream_t s, const uint4* list = nullptr,
                 const uint32_t* list_count = nullptr, const CullScan* fused = nullptr) {
    Params P;
    size_t smem = 0;
    mc_status rc = build_params(a, st, P, smem);
    if (rc != MC_OK) return rc;
    P.list = list;
    P.list_count = list_count;
    P.cull_fused = 0;
    if (fused) {   // one-launch culled decode: the kernel scans first (tiles set by launch_g)
        P.cull_fused = 1;
        P.cull = *fused;
        P.list = fused->list;
        P.list_count = fused->counts;
    }
    if (P.list) {   // culled decode: compacted outputs start at 0 (FORMAT.md §7)
        P.base_vtx = 0;
        P.base_tri = 0;
        P.index_sub = 0;
    }
    if (a->count == 0) return MC_OK;
    // compile-time layouts for the BASELINE configs, generic kernel otherwise
    const mc_layout& L = *a->layout;
    int lay = 0;
    int oct0 = -1;
    for (uint32_t c = 0; c < L.n; ++c)
        if (L.semantic[c] == MC_SEM_NORMAL_OCT) { oct0 = (int)c; break; }
    uint32_t noct = L.n_out - L.n;
    if (L.n == 8 && noct == 0) lay = 1;                   // pos3 + nrm3 + uv2
    else if (L.n == 7 && noct == 1 && oct0 == 3) lay = 2; // pos3 + oct2 + uv2 (cfg3/cfg4)
    else if (L.n == 3 && noct == 0) lay = 3;              // positions only (cfg2)
    // attribute mode: 0 aligned halfwords (every channel 16 bits, no VW), 1 bit reader, 2 VW
    bool b16 = true;
    for (uint32_t c = 0; c < L.n; ++c) b16 = b16 && L.bits[c] == 16;
    bool uni = L.n > 0;
    for (uint32_t c = 0; c < L.n; ++c) uni = uni && L.bits[c] == L.bits[0];
    // 3: one width for every channel (compile-time unpack for the widths dispatch_am knows)
    const int am = (L.flags & 1u) ? 2 : (b16 ? 0 : (uni && MC_UNIFORM_WIDTHS ? 3 : 1));
    if (lay == 0)   // generic kernel stages vertex words in smem
        P.vtx_stage_words = a->d_vertices ? ((L.v_max * L.n_out + 8u + 3u) & ~3u) : 0u;
    else if (MC_BULK_VTX && (L.n_out % 4u) == 0u)   // compile-time layouts with bulk vertex stores
        P.vtx_stage_words = a->d_vertices ? ((L.v_max * L.n_out + 3u) & ~3u) : 0u;
    // group stride = 16 (mod 32) words: the two groups of a warp reading the same
    // record offset hit different banks
    P.idx_stage_words = MC_BULK_IDX ? ((((P.u8x4 ? 1u : 3u) * L.t_max + 4u) + 3u) & ~3u) : 0u;
    P.grp_words = 2 * P.buf_words + P.vtx_stage_words + P.idx_stage_words + kMiscWords;
    if (MC_BANK_PAD) P.grp_words += (48u - (P.grp_words & 31u)) & 31u;
    smem = 4u * (size_t)P.grp_words;
    return dispatch_codec(L.codec, st != nullptr, lay, am, P, smem, s);
}


// ------------------------------------------------------------------ mc_decode_host pipeline
// Chunk c of a pipelined host decode: records [first, next.first), record bytes from
// rec_off, outputs from the first record's bases (the last entry is the end sentinel).
struct HostChunk {
    uint32_t first;
    uint64_t rec_off;   // byte offset inside the records section (16 * dir[first])
    uint32_t vtx, tri;  // vtx_base / tri_base of record `first` (end: base + total)
};

// Byte-balanced chunk boundaries by binary search over the directory (O(chunks log M),
// no pass over the records), bases read from the boundary records' headers.  Returns
// fewer than two entries when the blob does not meet the ordering precondition
// (include/mc.h), which selects the serial path.
std::vector<HostChunk> plan_host_chunks(const mc_layout& L, const uint8_t* hb, uint32_t chunks) {
    std::vector<HostChunk> ch;
    const uint32_t M = L.num_meshlets;
    const uint32_t* dir = reinterpret_cast<const uint32_t*>(hb + L.off_dir);
    const uint64_t rec_bytes = L.total_bytes - L.off_rec;
    if (16ull * dir[M] > rec_bytes) return ch;
    chunks = std::min(chunks, M);
    for (uint32_t c = 0; c < chunks; ++c) {
        const uint64_t target = (uint64_t)dir[M] * c / chunks;   // in 16-B units
        const uint32_t m = c == 0 ? 0u : (uint32_t)(std::lower_bound(dir, dir + M, (uint32_t)target) - dir);
        if (!ch.empty() && m <= ch.back().first) continue;      // empty chunk (one huge record)
        const uint32_t* rh = reinterpret_cast<const uint32_t*>(hb + L.off_rec + 16ull * dir[m]);
        ch.push_back({m, 16ull * dir[m], rh[0], rh[1]});
    }
    ch.push_back({M, 16ull * dir[M], L.base_vtx + L.total_v, L.base_tri + L.total_tp});
    for (size_t c = 0; c < ch.size(); ++c) {   // boundary bases ascending inside the output ranges
        const bool bad = ch[c].vtx < L.base_vtx || ch[c].tri < L.base_tri ||
                         (uint64_t)ch[c].vtx > (uint64_t)L.base_vtx + L.total_v ||
                         (uint64_t)ch[c].tri > (uint64_t)L.base_tri + L.total_tp ||
                         (c > 0 && (ch[c].vtx < ch[c - 1].vtx || ch[c].tri < ch[c - 1].tri)) ||
                         (c == 0 && (ch[0].vtx != L.base_vtx || ch[0].tri != L.base_tri));
        if (bad) return {};
    }
    return ch;
}

// Library-owned copy streams and events of the pipelined host decode, one set per device.
struct PipeRes {
    std::mutex mu;
    cudaStream_t in = nullptr, out = nullptr;
    cudaEvent_t start = nullptr, done = nullptr, in_done[64] = {}, dec_done[64] = {};
};
PipeRes* pipe_res() {
    static PipeRes res[kMaxDevices];
    static std::mutex mu;
    static bool ready[kMaxDevices] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
    std::lock_guard<std::mutex> g(mu);
    PipeRes& r = res[dev];
    if (!ready[dev]) {
        const unsigned ef = cudaEventDisableTiming;
        if (cudaStreamCreateWithFlags(&r.in, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&r.out, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&r.start, ef) != cudaSuccess || cudaEventCreateWithFlags(&r.done, ef) != cudaSuccess)
            return nullptr;
        for (int i = 0; i < 64; ++i)
            if (cudaEventCreateWithFlags(&r.in_done[i], ef) != cudaSuccess ||
                cudaEventCreateWithFlags(&r.dec_done[i], ef) != cudaSuccess)
                return nullptr;
        ready[dev] = true;
    }
    return &r;
}

}  // namespace

extern "C" {

mc_status mc_decode_meshlets(const mc_decode_args* args, void* stream) {
    return launch(args, nullptr, static_cast<cudaStream_t>(stream));
}

mc_status mc_decode_stats(const mc_decode_args* args, mc_stats* d_stats, void* stream) {
    if (!d_stats) return MC_ERR_ARG;
    return launch(args, d_stats, static_cast<cudaStream_t>(stream));
}

size_t mc_decode_culled_scratch_bytes(const mc_layout* L) {
    if (!L) return 0;
    // tiles of >= 32 threads x kCullPerThread records (the fused scan uses the decode CTA's
    // warps, >= 1): list [M] uint4 | tile_agg [tiles] uint4 | tile_inc [tiles] uint4 |
    // tile_flag [tiles] u32 | ctr [4] u32
    const uint64_t tiles = (uint64_t(L->num_meshlets) + 32 * kCullPerThread - 1) / (32 * kCullPerThread);
    return size_t(16ull * L->num_meshlets + 32ull * tiles + ((4ull * tiles + 15) & ~15ull) + 16ull);
}

mc_status mc_decode_culled(const mc_decode_args* a, const float* view_dir, void* d_scratch, size_t scratch_bytes,
                           uint32_t* d_counts, mc_stats* d_stats, void* stream) {
    if (!a || !a->layout || !view_dir || !d_counts) return MC_ERR_ARG;
    const mc_layout& L = *a->layout;
    if (!(L.flags & 2u) || L.off_cull == 0) return MC_ERR_FORMAT;            // no cull table
    if (a->first != 0 || a->count != L.num_meshlets) return MC_ERR_ARG;      // whole blob only
    if (reinterpret_cast<uintptr_t>(d_counts) & 3u) return MC_ERR_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint32_t M = L.num_meshlets;
    if (M == 0) return cudaMemsetAsync(d_counts, 0, 16, s) == cudaSuccess ? MC_OK : MC_ERR_CUDA;
    if (!a->d_blob || (reinterpret_cast<uintptr_t>(a->d_blob) & 15u)) return MC_ERR_ARG;
    if (!d_scratch || (reinterpret_cast<uintptr_t>(d_scratch) & 15u) || scratch_bytes < mc_decode_culled_scratch_bytes(&L))
        return MC_ERR_ARG;
    const uint8_t* blob = static_cast<const uint8_t*>(a->d_blob);
    CullScan C;
    C.rec = blob + L.off_rec;
    C.dir = reinterpret_cast<const uint32_t*>(blob + L.off_dir);
    C.cones = reinterpret_cast<const float4*>(blob + L.off_cull);
    C.rec_section_bytes = L.total_bytes - L.off_rec;
    C.M = M;
    C.vmax = L.v_max;
    C.tmax = L.t_max;
    C.max_rec = L.max_record_bytes;
    C.dx = view_dir[0];
    C.dy = view_dir[1];
    C.dz = view_dir[2];
    const uint32_t max_tiles = (M + 32u * kCullPerThread - 1u) / (32u * kCullPerThread);
    C.list = static_cast<uint4*>(d_scratch);
    C.tile_agg = C.list + M;
    C.tile_inc = C.tile_agg + max_tiles;
    C.tile_flag = reinterpret_cast<uint32_t*>(C.tile_inc + max_tiles);
    C.ctr = C.tile_flag + ((max_tiles + 3u) & ~3u);
    C.counts = d_counts;
#if MC_CULL_FUSED
    C.tiles = 0;   // launch_g sets it from the decode CTA size
    return launch(a, d_stats, s, nullptr, nullptr, &C);
#else
    C.tiles = (M + kCullTile - 1) / kCullTile;
    cull_scan_kernel<<<C.tiles, kCullThreads, 0, s>>>(C);
    if (cudaGetLastError() != cudaSuccess) return MC_ERR_CUDA;
    return launch(a, d_stats, s, C.list, d_counts);
#endif
}

mc_status mc_stats_reset(mc_stats* d_stats, void* stream) {
    if (!d_stats) return MC_ERR_ARG;
    stats_reset_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(d_stats);
    return cudaGetLastError() == cudaSuccess ? MC_OK : MC_ERR_CUDA;
}

mc_status mc_decode_host(const mc_host_decode_args* h, void* stream) {
    if (!h || !h->layout || !h->h_blob || !h->d_blob || !h->h_indices || !h->d_indices) return MC_ERR_ARG;
    if ((h->h_vertices == nullptr) != (h->d_vertices == nullptr)) return MC_ERR_ARG;
    if ((h->h_quantized == nullptr) != (h->d_quantized == nullptr)) return MC_ERR_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const mc_layout& L = *h->layout;
    const uint32_t M = L.num_meshlets;
    const uint64_t ib = (h->flags & MC_DECODE_INDEX_LOCAL_U8X4) ? 4ull : 12ull;   // index bytes per triangle
    const uint64_t vb = 4ull * L.n_out, qb = 4ull * L.n;                          // bytes per output vertex
    std::vector<HostChunk> ch;
    if (h->chunks >= 2 && M >= 2) ch = plan_host_chunks(L, static_cast<const uint8_t*>(h->h_blob), std::min(h->chunks, 64u));
    if (ch.size() < 2) {   // serial: H2D, decode, D2H on `stream`
        if (cudaMemcpyAsync(h->d_blob, h->h_blob, L.total_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
            return MC_ERR_CUDA;
        mc_decode_args a{h->layout, h->d_blob, 0, M, h->d_indices, h->d_vertices, h->d_quantized, h->flags, nullptr};
        mc_status rc = launch(&a, nullptr, s);
        if (rc != MC_OK) return rc;
        if (cudaMemcpyAsync(h->h_indices, h->d_indices, ib * L.total_tp, cudaMemcpyDeviceToHost, s) != cudaSuccess)
            return MC_ERR_CUDA;
        if (h->h_vertices &&
            cudaMemcpyAsync(h->h_vertices, h->d_vertices, vb * L.total_v, cudaMemcpyDeviceToHost, s) != cudaSuccess)
            return MC_ERR_CUDA;
        if (h->h_quantized &&
            cudaMemcpyAsync(h->h_quantized, h->d_quantized, qb * L.total_v, cudaMemcpyDeviceToHost, s) != cudaSuccess)
            return MC_ERR_CUDA;
        return MC_OK;
    }
    // pipelined: copy-in stream -> decode on `stream` -> copy-out stream, one event pair per chunk
    PipeRes* R = pipe_res();
    if (!R) return MC_ERR_CUDA;
    std::lock_guard<std::mutex> g(R->mu);   // the event pool is shared by concurrent callers
    auto ok = [](cudaError_t e) { return e == cudaSuccess; };
    const uint8_t* hb = static_cast<const uint8_t*>(h->h_blob);
    uint8_t* db = static_cast<uint8_t*>(h->d_blob);
    if (!ok(cudaEventRecord(R->start, s)) || !ok(cudaStreamWaitEvent(R->in, R->start, 0)) ||
        !ok(cudaStreamWaitEvent(R->out, R->start, 0)))
        return MC_ERR_CUDA;
    // header, directory, object and cull tables: everything before the records
    if (!ok(cudaMemcpyAsync(db, hb, L.off_rec, cudaMemcpyHostToDevice, R->in))) return MC_ERR_CUDA;
    for (size_t c = 0; c + 1 < ch.size(); ++c) {
        const HostChunk &a0 = ch[c], &a1 = ch[c + 1];
        const uint64_t r0 = L.off_rec + a0.rec_off, r1 = L.off_rec + a1.rec_off;
        if (!ok(cudaMemcpyAsync(db + r0, hb + r0, r1 - r0, cudaMemcpyHostToDevice, R->in)) ||
            !ok(cudaEventRecord(R->in_done[c], R->in)) || !ok(cudaStreamWaitEvent(s, R->in_done[c], 0)))
            return MC_ERR_CUDA;
        mc_decode_args a{h->layout, h->d_blob, a0.first, a1.first - a0.first, h->d_indices, h->d_vertices,
                         h->d_quantized, h->flags, nullptr};
        mc_status rc = launch(&a, nullptr, s);
        if (rc != MC_OK) return rc;
        if (!ok(cudaEventRecord(R->dec_done[c], s)) || !ok(cudaStreamWaitEvent(R->out, R->dec_done[c], 0)))
            return MC_ERR_CUDA;
        const uint64_t t0 = a0.tri - L.base_tri, t1 = a1.tri - L.base_tri;
        const uint64_t v0 = a0.vtx - L.base_vtx, v1 = a1.vtx - L.base_vtx;
        if (t1 > t0 && !ok(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(h->h_indices) + ib * t0,
                                           reinterpret_cast<const uint8_t*>(h->d_indices) + ib * t0, ib * (t1 - t0),
                                           cudaMemcpyDeviceToHost, R->out)))
            return MC_ERR_CUDA;
        if (h->h_vertices && v1 > v0 &&
            !ok(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(h->h_vertices) + vb * v0,
                                reinterpret_cast<const uint8_t*>(h->d_vertices) + vb * v0, vb * (v1 - v0),
                                cudaMemcpyDeviceToHost, R->out)))
            return MC_ERR_CUDA;
        if (h->h_quantized && v1 > v0 &&
            !ok(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(h->h_quantized) + qb * v0,
                                reinterpret_cast<const uint8_t*>(h->d_quantized) + qb * v0, qb * (v1 - v0),
                                cudaMemcpyDeviceToHost, R->out)))
            return MC_ERR_CUDA;
    }
    if (!ok(cudaEventRecord(R->done, R->out)) || !ok(cudaStreamWaitEvent(s, R->done, 0))) return MC_ERR_CUDA;
    return MC_OK;
}

}  // extern "C"
