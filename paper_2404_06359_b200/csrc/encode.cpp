// encode.cpp — host side of libmc: the meshlet encoder (mc_encode), blob utilities
// (parse / shard / extract / instance) and the C-ABI glue that does not touch the GPU.
//
// Paper: arXiv 2404.06359.  The encoder is the offline pre-process of §3–§4:
//   meshlet split (here a compact greedy grower instead of Meshoptimizer),
//   generalized triangle strips per meshlet (here a min-degree greedy path
//   cover instead of the MILP), strip encoding with 4-degenerate restarts,
//   ascending vertex re-labelling + increment flags / reuse buffer and
//   crack-free quantisation on a global anisotropic grid.
// The output is FORMAT.md.  No code here is shared with oracle/ (task rule ③).
#include "../../include/mc.h"

#include <algorithm>
#include <array>
#include <unordered_map>
#include <atomic>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>
#include <new>
#include <thread>
#include <vector>

namespace {

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr size_t kHeaderBytes = 160;

// ---------------------------------------------------------------- small utilities
inline uint64_t round16(uint64_t x) { return (x + 15) & ~uint64_t(15); }
inline void put32(uint8_t* p, uint32_t v) { std::memcpy(p, &v, 4); }
inline void put16(uint8_t* p, uint16_t v) { std::memcpy(p, &v, 2); }
inline void put64(uint8_t* p, uint64_t v) { std::memcpy(p, &v, 8); }
inline uint32_t get32(const uint8_t* p) { uint32_t v; std::memcpy(&v, p, 4); return v; }
inline uint16_t get16(const uint8_t* p) { uint16_t v; std::memcpy(&v, p, 2); return v; }
inline uint64_t get64(const uint8_t* p) { uint64_t v; std::memcpy(&v, p, 8); return v; }

unsigned worker_count(uint32_t requested) {
    if (requested) return requested;
    unsigned hc = std::thread::hardware_concurrency();
    return hc ? hc : 4;
}

// Run fn(i) for i in [0, n) on `threads` workers with dynamic chunking.
void parallel_for(size_t n, unsigned threads, const std::function<void(size_t)>& fn, size_t grain = 64) {
    if (n == 0) return;
    threads = std::max(1u, std::min<unsigned>(threads, unsigned((n + grain - 1) / grain)));
    if (threads == 1) {
        for (size_t i = 0; i < n; ++i) fn(i);
        return;
    }
    std::atomic<size_t> next{0};
    auto work = [&]() {
        for (;;) {
            size_t b = next.fetch_add(grain);
            if (b >= n) break;
            size_t e = std::min(n, b + grain);
            for (size_t i = b; i < e; ++i) fn(i);
        }
    };
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < threads; ++t) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
}

// Record size in bytes for (V, T'), FORMAT.md §1.4.
inline uint64_t record_bytes(uint32_t codec, uint32_t n, uint32_t S, uint32_t V, uint32_t Tp, bool vw = false) {
    uint64_t hdr = round16(16 + 4ull * n + (vw ? n : 0));   // VW: + u8 w_c[n]
    uint32_t W = codec == MC_CODEC_BASIC ? 0 : (Tp + 31) / 32;   // Basic: no flag words
    uint64_t nb = (codec == MC_CODEC_GTS) ? (Tp - 1) : (codec == MC_CODEC_BASIC) ? 3ull * Tp : ((Tp - 1) - (V - 3));
    uint64_t topo = 4ull * W * (codec == MC_CODEC_GTS_REUSE ? 2 : 1) + ((nb + 3) & ~uint64_t(3));
    uint64_t attr = 4ull * ((uint64_t(V) * S + 31) / 32);
    return round16(hdr + topo + attr);
}

uint32_t output_floats(uint32_t n, const uint8_t* sem) {
    uint32_t n_out = n;
    for (uint32_t c = 0; c < n; ++c)
        if (sem[c] == MC_SEM_NORMAL_OCT) { ++n_out; ++c; }
    return n_out;
}

// ---------------------------------------------------------------- one emitted meshlet
struct Meshlet {
    uint32_t object = 0;
    uint32_t V = 0, Tp = 0, R = 0;
    std::vector<uint32_t> local_to_src;   // [V]
    std::vector<uint8_t> step;            // N[3..T'+1] local indices, size T'-1
    std::vector<uint8_t> flag;            // f_t, t=0..T'-1 (f_0 = 0)
    std::vector<uint32_t> src_tri;        // [T'] (kNone for restart degenerates)
    std::vector<uint8_t> tri3;            // Basic: local triangle list [3T]
};

// ---------------------------------------------------------------- mesh-level encoder
struct Encoder {
    const mc_mesh& mesh;
    uint32_t vmax, tmax, codec;
    unsigned threads;
    uint32_t n, S;
    std::vector<int32_t> nbr;            // [3T] neighbour across edge e=(v[e],v[e+1])
    std::vector<uint32_t> vt_off, vt;    // vertex -> triangles CSR
    std::vector<Meshlet> meshlets;
    uint64_t splits = 0;
    std::vector<uint16_t> tpos;          // scratch: triangle -> position in its meshlet
    std::vector<int32_t> vlocal;         // scratch: vertex -> local index during emission

    bool vw = false;                     // MC_ENCODE_VARIABLE_WIDTHS
    bool cull = false;                   // MC_ENCODE_CULL_CONES
    Encoder(const mc_mesh& m, uint32_t vm, uint32_t tm, uint32_t cd, unsigned th, bool varw = false)
        : mesh(m), vmax(vm), tmax(tm), codec(cd), threads(th), n(m.num_channels), S(0), vw(varw) {
        for (uint32_t c = 0; c < n; ++c) S += m.bits[c];
    }

    uint32_t obj(uint32_t t) const { return mesh.object_of_triangle ? mesh.object_of_triangle[t] : 0; }
    const uint32_t* tri(uint32_t t) const { return mesh.indices + 3ull * t; }

    void build_adjacency() {
        const uint32_t T = mesh.num_triangles, V = mesh.num_vertices;
        vt_off.assign(V + 1, 0);
        for (uint64_t i = 0; i < 3ull * T; ++i) vt_off[mesh.indices[i] + 1]++;
        for (uint32_t v = 0; v < V; ++v) vt_off[v + 1] += vt_off[v];
        vt.resize(3ull * T);
        {
            std::vector<uint32_t> fill(vt_off.begin(), vt_off.end() - 1);
            for (uint32_t t = 0; t < T; ++t)
                for (int k = 0; k < 3; ++k) vt[fill[tri(t)[k]]++] = t;
        }
        nbr.assign(3ull * T, -1);
        // Dual edge iff the undirected edge has exactly two incident triangles with opposite
        // orientation, same object, distinct third vertices (non-manifold edges sever).
        parallel_for(T, threads, [&](size_t ti) {
            uint32_t t = uint32_t(ti);
            const uint32_t* a = tri(t);
            for (int e = 0; e < 3; ++e) {
                uint32_t u = a[e], w = a[(e + 1) % 3], x = a[(e + 2) % 3];
                int32_t found = -1;
                int count = 0;
                for (uint32_t k = vt_off[w]; k < vt_off[w + 1]; ++k) {
                    uint32_t s = vt[k];
                    if (s == t) continue;
                    const uint32_t* b = tri(s);
                    int hu = -1, hw = -1;
                    for (int j = 0; j < 3; ++j) {
                        if (b[j] == u) hu = j;
                        if (b[j] == w) hw = j;
                    }
                    if (hu < 0) continue;
                    ++count;
                    bool opposite = ((hw + 1) % 3) == hu;   // s contains the directed edge (w,u)
                    uint32_t third = b[3 - hu - hw];
                    if (opposite && third != x && obj(s) == obj(t)) found = int32_t(s);
                }
                if (count == 1) nbr[3ull * t + e] = found;
            }
        }, 4096);
    }

    // ---- path cover of one meshlet's dual graph (maximise strip edges under
    // degree <= 2 and no cycles): a greedy cover (start at a minimum-degree triangle,
    // extend both ends to the minimum-degree unvisited neighbour), then tunnelling.
    // Returns strips as lists of positions into `tl`.
    void stripify(const std::vector<uint32_t>& tl, const std::vector<int32_t>& assign, int32_t id,
                  std::vector<std::vector<uint16_t>>& strips) {
        const uint32_t T = uint32_t(tl.size());
        strips.clear();
        for (uint32_t i = 0; i < T; ++i) tpos[tl[i]] = uint16_t(i);
        std::vector<int16_t> ln(3 * T, -1);
        std::vector<uint8_t> deg(T, 0), vis(T, 0);
        for (uint32_t i = 0; i < T; ++i)
            for (int e = 0; e < 3; ++e) {
                int32_t s = nbr[3ull * tl[i] + e];
                if (s >= 0 && assign[s] == id) {
                    ln[3 * i + e] = int16_t(tpos[s]);
                    deg[i]++;
                }
            }
        auto visit = [&](uint32_t i) {
            vis[i] = 1;
            for (int e = 0; e < 3; ++e)
                if (ln[3 * i + e] >= 0) deg[ln[3 * i + e]]--;
        };
        auto best_next = [&](uint32_t i) -> int {
            int best = -1;
            for (int e = 0; e < 3; ++e) {
                int s = ln[3 * i + e];
                if (s < 0 || vis[s]) continue;
                if (best < 0 || deg[s] < deg[best] || (deg[s] == deg[best] && s < best)) best = s;
            }
            return best;
        };
        uint32_t left = T;
        while (left) {
            int start = -1;
            for (uint32_t i = 0; i < T; ++i)
                if (!vis[i] && (start < 0 || deg[i] < deg[start])) start = int(i);
            std::vector<uint16_t> path{uint16_t(start)};
            visit(start);
            --left;
            for (int pass = 0; pass < 2; ++pass) {
                for (;;) {
                    int nx = best_next(path.back());
                    if (nx < 0) break;
                    path.push_back(uint16_t(nx));
                    visit(nx);
                    --left;
                }
                std::reverse(path.begin(), path.end());
            }
            strips.push_back(std::move(path));
        }
        if (tunnel_budget) tunnel(ln, T, strips);
    }

    // ---- strip-count reduction by tunnelling (the idea of the Enhanced Tunneling
    // Algorithm the paper compares against): a tunnel is an alternating path
    // free-edge, strip-edge, ..., free-edge between two strip terminals (triangles with
    // fewer than two strip neighbours).  Flipping it adds one strip edge, so the number of
    // strips (and restarts) drops by one, provided no cycle forms (every
    // dual-graph path is a valid generalized strip).  Breadth-first search per
    // terminal, bounded depth; a flip that closes a cycle is undone.
    unsigned tunnel_budget = 512;   // flips tried per meshlet
    void tunnel(const std::vector<int16_t>& ln, uint32_t T, std::vector<std::vector<uint16_t>>& strips) {
        if (strips.size() < 2) return;
        std::vector<int16_t> sn(2 * T, -1);                      // strip neighbours
        auto has = [&](int u, int v) { return sn[2 * u] == v || sn[2 * u + 1] == v; };
        auto deg = [&](int u) { return int(sn[2 * u] >= 0) + int(sn[2 * u + 1] >= 0); };
        auto add = [&](int u, int v) { (sn[2 * u] < 0 ? sn[2 * u] : sn[2 * u + 1]) = int16_t(v); };
        auto del = [&](int u, int v) { (sn[2 * u] == v ? sn[2 * u] : sn[2 * u + 1]) = -1; };
        for (auto& p : strips)
            for (size_t i = 1; i < p.size(); ++i) { add(p[i - 1], p[i]); add(p[i], p[i - 1]); }
        auto acyclic = [&]() {
            std::vector<uint8_t> seen(T, 0);
            for (uint32_t i = 0; i < T; ++i) {
                if (seen[i]) continue;
                // walk the component; a component with as many edges as nodes is a cycle
                uint32_t nodes = 0, ends = 0;
                std::vector<int> stack{int(i)};
                seen[i] = 1;
                while (!stack.empty()) {
                    int u = stack.back();
                    stack.pop_back();
                    ++nodes;
                    if (deg(u) < 2) ++ends;
                    for (int k = 0; k < 2; ++k) {
                        int v = sn[2 * u + k];
                        if (v >= 0 && !seen[v]) { seen[v] = 1; stack.push_back(v); }
                    }
                }
                if (ends == 0 && nodes > 1) return false;
            }
            return true;
        };
        std::vector<uint8_t> onpath(T);
        std::vector<uint8_t> bad(T, 0);
        unsigned flips = 0;
        bool progress = true;
        while (progress && flips < tunnel_budget) {
            progress = false;
            std::fill(bad.begin(), bad.end(), uint8_t(0));   // earlier flips may open new tunnels
            for (uint32_t s0 = 0; s0 < T && flips < tunnel_budget; ++s0) {
                if (deg(int(s0)) >= 2 || bad[s0]) continue;
                // depth-first search for a SIMPLE alternating path (every node at most once,
                // so each interior degree is unchanged by the flip), bounded expansions
                std::fill(onpath.begin(), onpath.end(), uint8_t(0));
                std::vector<int> stk;                 // nodes of the current path, s0 first
                std::vector<uint8_t> nexte;           // next neighbour slot to try per depth
                stk.push_back(int(s0));
                nexte.push_back(0);
                onpath[s0] = 1;
                int expansions = 0;
                bool flipped = false;
                while (!stk.empty() && !flipped && expansions < 4096) {
                    const int u = stk.back(), d = int(stk.size()) - 1;
                    const int pr = d & 1;             // even depth: next edge free; odd: strip
                    if (nexte.back() >= 3 || d >= 24) {
                        onpath[u] = 0;
                        stk.pop_back();
                        nexte.pop_back();
                        continue;
                    }
                    const int v = ln[3 * u + nexte.back()++];
                    if (v < 0 || onpath[v]) continue;
                    if (has(u, v) != (pr == 1)) continue;
                    ++expansions;
                    stk.push_back(v);
                    nexte.push_back(0);
                    onpath[v] = 1;
                    if (!(pr == 0 && deg(v) < 2)) continue;
                    // free edge into a terminal: flip the tunnel (strip edges out first, then
                    // free edges in: an interior node never holds three neighbours), keep it
                    // if no cycle formed, else undo and keep searching
                    std::vector<std::pair<int, int>> added, removed;
                    for (size_t i = 1; i < stk.size(); ++i) {
                        const int a0 = stk[i - 1], a1 = stk[i];
                        (has(a0, a1) ? removed : added).push_back({a0, a1});
                    }
                    for (auto& e : removed) { del(e.first, e.second); del(e.second, e.first); }
                    for (auto& e : added) { add(e.first, e.second); add(e.second, e.first); }
                    if (acyclic()) { flipped = true; break; }
                    for (auto& e : added) { del(e.first, e.second); del(e.second, e.first); }
                    for (auto& e : removed) { add(e.first, e.second); add(e.second, e.first); }
                }
                ++flips;
                if (flipped) progress = true;
                else bad[s0] = 1;
            }
        }
        // rebuild the strips from the strip-neighbour lists
        strips.clear();
        std::vector<uint8_t> used(T, 0);
        for (uint32_t i = 0; i < T; ++i) {
            if (used[i] || deg(int(i)) == 2) continue;
            std::vector<uint16_t> path;
            int prev = -1, u = int(i);
            while (u >= 0) {
                used[u] = 1;
                path.push_back(uint16_t(u));
                int nx = sn[2 * u] >= 0 && sn[2 * u] != prev ? sn[2 * u] : (sn[2 * u + 1] != prev ? sn[2 * u + 1] : -1);
                if (nx >= 0 && used[nx]) nx = -1;
                prev = u;
                u = nx;
            }
            strips.push_back(std::move(path));
        }
    }

    // ---- emit one meshlet's strips as a GTS step sequence
    bool emit(const std::vector<uint32_t>& tl, const std::vector<std::vector<uint16_t>>& strips,
              uint32_t object, Meshlet& out) {
        std::vector<uint32_t> G;       // step sequence over source vertices
        std::vector<uint8_t> F;        // flags per triangle
        std::vector<uint32_t> ST;      // source triangle per triangle
        G.reserve(300);
        uint32_t a = 0, b = 0, c = 0;
        for (size_t s = 0; s < strips.size(); ++s) {
            const auto& p = strips[s];
            const uint32_t* t0 = tri(tl[p[0]]);
            // rotate the first triangle so its vertex unshared with the successor sits at
            // position b: the successor is then across the left edge (c,a)
            int k = 0;
            if (p.size() > 1) {
                const uint32_t* t1 = tri(tl[p[1]]);
                int un = 0;
                for (int j = 0; j < 3; ++j)
                    if (t0[j] != t1[0] && t0[j] != t1[1] && t0[j] != t1[2]) un = j;
                k = (un + 2) % 3;   // rotation start so that t0[un] lands at index 1
            }
            uint32_t P = t0[k], Q = t0[(k + 1) % 3], Rr = t0[(k + 2) % 3];
            if (s == 0) {
                G = {P, Q, Rr};
                F.push_back(0);
                ST.push_back(tl[p[0]]);
            } else {
                // restart: [R:c, L:q, L:q, R:p] then R:r  -> (P,Q,Rr)
                const uint32_t ws[5] = {c, Q, Q, P, Rr};
                const uint8_t fs[5] = {1, 0, 0, 1, 1};
                for (int j = 0; j < 5; ++j) {
                    G.push_back(ws[j]);
                    F.push_back(fs[j]);
                    ST.push_back(j == 4 ? tl[p[0]] : kNone);
                }
            }
            a = P; b = Q; c = Rr;
            for (size_t i = 1; i < p.size(); ++i) {
                const uint32_t* ti = tri(tl[p[i]]);
                bool hb = false, hc = false;
                uint32_t w = kNone;
                for (int j = 0; j < 3; ++j) {
                    if (ti[j] == c) hc = true;
                    else if (ti[j] == b) hb = true;
                    else if (ti[j] != a) w = ti[j];
                }
                if (!hc || w == kNone) return false;
                if (hb) { a = c; /* b stays */ c = w; F.push_back(1); }   // R: (c,b,w)
                else    { /* a stays */ b = c; c = w; F.push_back(0); }   // L: (a,c,w)
                G.push_back(w);
                ST.push_back(tl[p[i]]);
            }
        }
        if (F.size() > tmax) return false;
        // ascending re-labelling by first appearance
        out.object = object;
        out.Tp = uint32_t(F.size());
        out.R = uint32_t(strips.size() - 1);
        out.local_to_src.clear();
        out.step.resize(out.Tp - 1);
        std::vector<uint32_t> L;
        L.reserve(G.size());
        for (uint32_t g : G) {
            int32_t l = vlocal[g];
            if (l < 0) { l = int32_t(out.local_to_src.size()); vlocal[g] = l; out.local_to_src.push_back(g); }
            L.push_back(uint32_t(l));
        }
        for (uint32_t g : out.local_to_src) vlocal[g] = -1;
        out.V = uint32_t(out.local_to_src.size());
        if (out.V > vmax || out.V < 3) return false;
        for (uint32_t t = 1; t < out.Tp; ++t) out.step[t - 1] = uint8_t(L[t + 2]);
        out.flag = std::move(F);
        out.src_tri = std::move(ST);
        return true;
    }

    // ---- Basic (codec 3): the meshlet's triangles as a local u8 triangle list, vertices
    // numbered by first appearance; no strips, no restarts
    bool emit_basic(const std::vector<uint32_t>& tl, uint32_t object, Meshlet& out) {
        out.object = object;
        out.Tp = uint32_t(tl.size());
        out.R = 0;
        out.local_to_src.clear();
        out.tri3.resize(3 * tl.size());
        out.src_tri.assign(tl.begin(), tl.end());
        for (size_t i = 0; i < tl.size(); ++i)
            for (int k = 0; k < 3; ++k) {
                uint32_t g = tri(tl[i])[k];
                int32_t l = vlocal[g];
                if (l < 0) { l = int32_t(out.local_to_src.size()); vlocal[g] = l; out.local_to_src.push_back(g); }
                out.tri3[3 * i + k] = uint8_t(l);
            }
        for (uint32_t g : out.local_to_src) vlocal[g] = -1;
        out.V = uint32_t(out.local_to_src.size());
        return out.V >= 3 && out.V <= vmax;
    }

    // ---- meshlet building: compact greedy growth (fewest new vertices first, FIFO inside a
    // score class), seeded from the previous meshlet's frontier; then stripify and shrink
    // from the last-added triangle while T' = T + 4R exceeds T~.
    mc_status build_object(const std::vector<uint32_t>& object_tris, uint32_t object,
                           std::vector<int32_t>& assign, std::vector<int32_t>& vstamp,
                           std::vector<int32_t>& tstamp, std::vector<uint8_t>& score,
                           std::vector<Meshlet>& out, std::atomic<int32_t>& next_id, uint64_t& nsplit) {
        std::vector<uint32_t> bucket[4];
        size_t head[4] = {0, 0, 0, 0};
        size_t scan = 0;
        std::vector<uint32_t> tl;
        std::vector<std::vector<uint16_t>> strips;
        std::vector<uint32_t> frontier;
        while (true) {
            int32_t id = next_id.fetch_add(1);
            // seed: best frontier triangle of the previous meshlet, else the scan pointer
            int64_t seed = -1;
            uint32_t best_sc = 0;
            for (uint32_t t : frontier)
                if (assign[t] < 0) {
                    uint32_t sc = 0;
                    for (int e = 0; e < 3; ++e) {
                        int32_t s = nbr[3ull * t + e];
                        if (s >= 0 && assign[s] >= 0) ++sc;
                    }
                    if (seed < 0 || sc > best_sc) { seed = t; best_sc = sc; }
                }
            if (seed < 0) {
                while (scan < object_tris.size() && assign[object_tris[scan]] >= 0) ++scan;
                if (scan == object_tris.size()) break;
                seed = object_tris[scan];
            }
            for (int k = 1; k < 4; ++k) { bucket[k].clear(); head[k] = 0; }
            tl.clear();
            uint32_t V = 0;
            auto add = [&](uint32_t t) {
                assign[t] = id;
                tl.push_back(t);
                for (int k = 0; k < 3; ++k) {
                    uint32_t v = tri(t)[k];
                    if (vstamp[v] == id) continue;
                    vstamp[v] = id;
                    ++V;
                    for (uint32_t j = vt_off[v]; j < vt_off[v + 1]; ++j) {
                        uint32_t u = vt[j];
                        if (assign[u] >= 0 || obj(u) != object) continue;
                        if (tstamp[u] != id) { tstamp[u] = id; score[u] = 0; }
                        uint8_t s = ++score[u];
                        bucket[s].push_back(u);
                    }
                }
            };
            add(uint32_t(seed));
            while (tl.size() < tmax) {
                int64_t pick = -1;
                for (int k = 3; k >= 1 && pick < 0; --k) {
                    uint32_t need = 3 - k;
                    if (V + need > vmax) continue;
                    while (head[k] < bucket[k].size()) {
                        uint32_t u = bucket[k][head[k]++];
                        if (assign[u] < 0 && tstamp[u] == id && score[u] == k) { pick = u; break; }
                    }
                }
                if (pick < 0) break;
                add(uint32_t(pick));
            }
            if (codec == MC_CODEC_BASIC) {
                Meshlet m;
                if (!emit_basic(tl, object, m)) return MC_ERR_INPUT;
                out.push_back(std::move(m));
                frontier.clear();
                for (int k = 3; k >= 1; --k)
                    for (size_t j = head[k]; j < bucket[k].size() && frontier.size() < 64; ++j)
                        if (assign[bucket[k][j]] < 0) frontier.push_back(bucket[k][j]);
                continue;
            }
            // stripify; shrink until T' fits
            while (true) {
                stripify(tl, assign, id, strips);
                uint32_t Tp = uint32_t(tl.size() + 4 * (strips.size() - 1));
                if (Tp <= tmax) break;
                uint32_t drop = std::min<uint32_t>(uint32_t(tl.size()) - 1, std::max<uint32_t>(1, (Tp - tmax + 1) / 2));
                for (uint32_t k = 0; k < drop; ++k) { assign[tl.back()] = -1; tl.pop_back(); }
                ++nsplit;
            }
            Meshlet m;
            if (!emit(tl, strips, object, m)) return MC_ERR_INPUT;
            out.push_back(std::move(m));
            // frontier for the next seed: unassigned candidates of this meshlet
            frontier.clear();
            for (int k = 3; k >= 1; --k)
                for (size_t j = head[k]; j < bucket[k].size() && frontier.size() < 64; ++j)
                    if (assign[bucket[k][j]] < 0) frontier.push_back(bucket[k][j]);
        }
        return MC_OK;
    }

    mc_status run() {
        const uint32_t T = mesh.num_triangles;
        build_adjacency();
        uint32_t O = 1;
        if (mesh.object_of_triangle)
            for (uint32_t t = 0; t < T; ++t) {
            if (mesh.object_of_triangle[t] >= 65536u) return MC_ERR_LIMITS;   // no +1 wrap at UINT32_MAX
            O = std::max(O, mesh.object_of_triangle[t] + 1);
        }
        if (O > 65536) return MC_ERR_LIMITS;
        std::vector<std::vector<uint32_t>> by_obj(O);
        for (uint32_t t = 0; t < T; ++t) by_obj[obj(t)].push_back(t);
        tpos.assign(T, 0);
        vlocal.assign(mesh.num_vertices, -1);
        // objects build on separate workers only if no vertex is referenced by two
        // objects (per-vertex scratch is then private to one worker)
        bool shared = false;
        if (mesh.object_of_triangle) {
            std::vector<uint32_t> vobj(mesh.num_vertices, kNone);
            for (uint32_t t = 0; t < T && !shared; ++t)
                for (int k = 0; k < 3; ++k) {
                    uint32_t& o = vobj[tri(t)[k]];
                    if (o == kNone) o = obj(t);
                    else if (o != obj(t)) shared = true;
                }
        }
        std::vector<int32_t> assign(T, -1), tstamp(T, -1);
        std::vector<uint8_t> score(T, 0);
        std::vector<int32_t> vstamp(mesh.num_vertices, -1);
        std::vector<std::vector<Meshlet>> per_obj(O);
        std::vector<uint64_t> per_split(O, 0);
        std::vector<mc_status> st(O, MC_OK);
        std::atomic<int32_t> next_id{0};
        // objects are independent: build them on separate workers
        std::atomic<uint32_t> next_obj{0};
        auto worker = [&]() {
            for (;;) {
                uint32_t o = next_obj.fetch_add(1);
                if (o >= O) break;
                st[o] = build_object(by_obj[o], o, assign, vstamp, tstamp, score, per_obj[o], next_id, per_split[o]);
            }
        };
        unsigned nw = shared ? 1u : std::min<unsigned>(threads, O);
        if (nw <= 1) worker();
        else {
            std::vector<std::thread> pool;
            for (unsigned i = 0; i < nw; ++i) pool.emplace_back(worker);
            for (auto& th : pool) th.join();
        }
        for (uint32_t o = 0; o < O; ++o) {
            if (st[o] != MC_OK) return st[o];
            splits += per_split[o];
            for (auto& m : per_obj[o]) meshlets.push_back(std::move(m));
        }
        num_objects = O;
        return MC_OK;
    }
    uint32_t num_objects = 1;
};

}  // namespace

// ---------------------------------------------------------------- the opaque blob
struct mc_blob {
    std::unique_ptr<uint8_t[]> storage;
    uint8_t* bytes = nullptr;     // 64-B aligned view into storage
    size_t size = 0;
    std::vector<uint32_t> src_vertex, src_tri;
    bool has_map = false;
    uint64_t restarts = 0, splits = 0;

    bool allocate(size_t n) {
        storage.reset(new (std::nothrow) uint8_t[n + 64]);
        if (!storage) return false;
        uintptr_t p = reinterpret_cast<uintptr_t>(storage.get());
        bytes = reinterpret_cast<uint8_t*>((p + 63) & ~uintptr_t(63));
        size = n;
        std::memset(bytes, 0, n);
        return true;
    }
};

namespace {

void write_header(uint8_t* B, uint32_t codec, uint32_t n, uint32_t M, uint32_t O, uint32_t vmax,
                  uint32_t tmax, uint64_t tv, uint64_t ttp, uint64_t tt, uint32_t base_m, uint32_t base_v,
                  uint32_t base_t, uint32_t maxrec, uint64_t off_dir, uint64_t off_obj, uint64_t off_rec,
                  uint64_t total, const uint8_t* bits, const uint8_t* sem, uint32_t flags = 0,
                  uint64_t off_cull = 0) {
    std::memcpy(B, "MCZ1", 4);
    put32(B + 4, 1); put32(B + 8, codec); put32(B + 12, n); put32(B + 16, M); put32(B + 20, O);
    put32(B + 24, vmax); put32(B + 28, tmax); put32(B + 32, uint32_t(tv)); put32(B + 36, uint32_t(ttp));
    put32(B + 40, uint32_t(tt)); put32(B + 44, base_m); put32(B + 48, base_v); put32(B + 52, base_t);
    put32(B + 56, maxrec); put32(B + 60, flags);
    put64(B + 64, off_dir); put64(B + 72, off_obj); put64(B + 80, off_rec); put64(B + 88, total);
    std::memset(B + 96, 0, 64);
    for (uint32_t c = 0; c < n; ++c) { B[96 + c] = bits[c]; B[112 + c] = sem[c]; }
    put64(B + 128, off_cull);
}

// Normal cone of one meshlet from its DECODED positions (FORMAT.md §1.5/§7):
// axis = normalised sum of the real triangles' unit normals, θ = largest angle between the
// stored (binary32) axis and any of them, plus a margin for binary32 rounding of the test
// and of translated grid origins (instancing); cutoff = sin θ rounded up, or 2 (never).
void cull_cone(const std::vector<std::array<double, 3>>& P, const std::vector<std::array<uint32_t, 3>>& tris,
               float out[4]) {
    constexpr double kMargin = 0.01;   // radians
    std::vector<std::array<double, 3>> nrm;
    double sx = 0, sy = 0, sz = 0;
    for (auto& t : tris) {
        const auto &a = P[t[0]], &b = P[t[1]], &c = P[t[2]];
        const double ux = b[0] - a[0], uy = b[1] - a[1], uz = b[2] - a[2];
        const double vx = c[0] - a[0], vy = c[1] - a[1], vz = c[2] - a[2];
        double nx = uy * vz - uz * vy, ny = uz * vx - ux * vz, nz = ux * vy - uy * vx;
        const double l = std::sqrt(nx * nx + ny * ny + nz * nz);
        if (!(l > 0)) continue;                      // zero area after quantisation: no facing
        nx /= l; ny /= l; nz /= l;
        nrm.push_back({nx, ny, nz});
        sx += nx; sy += ny; sz += nz;
    }
    const double sl = std::sqrt(sx * sx + sy * sy + sz * sz);
    out[0] = 0.0f; out[1] = 0.0f; out[2] = 1.0f; out[3] = 2.0f;   // never cull
    if (nrm.empty() || sl < 1e-6 * double(nrm.size())) return;
    const float ax = float(sx / sl), ay = float(sy / sl), az = float(sz / sl);
    const double al = std::sqrt(double(ax) * ax + double(ay) * ay + double(az) * az);
    double theta = 0;
    for (auto& n : nrm) {
        double cs = (n[0] * ax + n[1] * ay + n[2] * az) / al;
        theta = std::max(theta, std::acos(std::max(-1.0, std::min(1.0, cs))));
    }
    theta += kMargin;
    out[0] = ax; out[1] = ay; out[2] = az;
    if (theta >= 1.5707963267948966) return;
    const double sc = std::sin(theta);
    float c = float(sc);
    if (double(c) < sc) c = std::nextafter(c, 2.0f);
    out[3] = c;
}

// Quantise and serialise (FORMAT.md §1, §3).
mc_status serialise(Encoder& E, mc_blob& out) {
    const mc_mesh& mesh = E.mesh;
    const uint32_t n = E.n, O = E.num_objects, codec = E.codec;
    auto& ms = E.meshlets;
    const size_t M = ms.size();
    const unsigned th = E.threads;

    // per-meshlet channel minima / maxima
    std::vector<float> mlo(M * n), mhi(M * n);
    parallel_for(M, th, [&](size_t m) {
        for (uint32_t c = 0; c < n; ++c) {
            float lo = INFINITY, hi = -INFINITY;
            for (uint32_t s : ms[m].local_to_src) {
                float x = mesh.attributes[uint64_t(s) * n + c];
                lo = std::min(lo, x);
                hi = std::max(hi, x);
            }
            mlo[m * n + c] = lo;
            mhi[m * n + c] = hi;
        }
    });
    // global grid per object and channel: origin g = object minimum, spacing
    // Δ = w/(2^b-1) with w the largest meshlet extent, rounded up to fp32.
    std::vector<float> delta(size_t(O) * n, 1.0f), origin(size_t(O) * n, 0.0f);
    std::vector<double> wmax(size_t(O) * n, 0.0);
    std::vector<float> gmin(size_t(O) * n, INFINITY);
    for (size_t m = 0; m < M; ++m)
        for (uint32_t c = 0; c < n; ++c) {
            size_t k = size_t(ms[m].object) * n + c;
            gmin[k] = std::min(gmin[k], mlo[m * n + c]);
            wmax[k] = std::max(wmax[k], double(mhi[m * n + c]) - double(mlo[m * n + c]));
        }
    std::vector<uint32_t> Lq(M * n);
    std::vector<uint8_t> wq(M * n);    // per-meshlet code widths (VW) or the global b_c
    const bool vw = E.vw, cull = E.cull;
    uint32_t pos_ch[3] = {0, 0, 0}, npos = 0;
    for (uint32_t c = 0; c < n && npos < 3; ++c)
        if (mesh.semantic[c] == MC_SEM_POSITION) pos_ch[npos++] = c;
    if (cull && npos < 3) return MC_ERR_ARG;
    auto qof = [](float x, float g, float d) { return std::floor((double(x) - double(g)) / double(d) + 0.5); };
    for (uint32_t o = 0; o < O; ++o)
        for (uint32_t c = 0; c < n; ++c) {
            size_t k = size_t(o) * n + c;
            origin[k] = std::isfinite(gmin[k]) ? gmin[k] : 0.0f;
            const uint32_t maxc = (1u << mesh.bits[c]) - 1u;
            if (wmax[k] > 0.0) {
                double d = wmax[k] / double(maxc);
                float f = float(d);
                if (double(f) < d) f = std::nextafter(f, INFINITY);
                delta[k] = f;
            }
        }
    // guard: enlarge Δ minimally until every meshlet's code range fits b bits
    std::atomic<int> range_err{0};
    bool still_bad = true;
    for (int iter = 0; iter < 96 && still_bad; ++iter) {
        std::vector<uint8_t> bad(size_t(O) * n, 0);
        parallel_for(M, th, [&](size_t m) {
            for (uint32_t c = 0; c < n; ++c) {
                size_t k = size_t(ms[m].object) * n + c;
                double lo = qof(mlo[m * n + c], origin[k], delta[k]);
                double hi = qof(mhi[m * n + c], origin[k], delta[k]);
                if (hi > 4294967295.0) range_err = 1;
                Lq[m * n + c] = uint32_t(lo);
                // Q is monotone in the attribute, so the largest code is Q(max) - Q(min)
                uint32_t mc = hi - lo > 0 ? uint32_t(hi - lo) : 0u, w = 0;
                while (w < 32 && (mc >> w)) ++w;
                wq[m * n + c] = vw ? uint8_t(w) : mesh.bits[c];
                if (hi - lo > double((1u << mesh.bits[c]) - 1u)) bad[k] = 1;
            }
        });
        if (range_err) return MC_ERR_RANGE;
        still_bad = false;
        for (size_t k = 0; k < bad.size(); ++k)
            if (bad[k]) {
                still_bad = true;
                // one ulp at a time first (the overflow is FP rounding, SPEC's guard); after
                // 32 steps scale by (2^b - 1)/(2^b - 2) per step so the loop always ends
                const uint32_t maxc = (1u << mesh.bits[k % n]) - 1u;
                if (iter < 32 || maxc < 2) delta[k] = std::nextafter(delta[k], INFINITY);
                else {
                    float f = float(double(delta[k]) * double(maxc) / double(maxc - 1u));
                    delta[k] = std::nextafter(f, INFINITY);
                }
            }
    }
    if (still_bad) return MC_ERR_RANGE;   // never leave codes wider than b bits
    // layout
    std::vector<uint64_t> roff(M + 1, 0);
    uint64_t tv = 0, ttp = 0, tt = 0, maxrec = 0, rs = 0;
    std::vector<uint32_t> vb(M), tb(M);
    for (size_t m = 0; m < M; ++m) {
        uint32_t Sm = 0;
        for (uint32_t c = 0; c < n; ++c) Sm += wq[m * n + c];
        uint64_t sz = record_bytes(codec, n, Sm, ms[m].V, ms[m].Tp, vw);
        roff[m + 1] = roff[m] + sz;
        maxrec = std::max(maxrec, sz);
        vb[m] = uint32_t(tv);
        tb[m] = uint32_t(ttp);
        tv += ms[m].V; ttp += ms[m].Tp; tt += ms[m].Tp - 4ull * ms[m].R; rs += ms[m].R;
    }
    if (tv > 0xFFFFFFFFull || 3 * ttp > 0xFFFFFFFFull || roff[M] / 16 > 0xFFFFFFFFull) return MC_ERR_RANGE;
    const uint64_t off_dir = kHeaderBytes, off_obj = round16(off_dir + 4ull * (M + 1));
    const uint64_t off_cull = cull ? round16(off_obj + 8ull * n * O) : 0;
    const uint64_t off_rec = cull ? round16(off_cull + 16ull * M) : round16(off_obj + 8ull * n * O);
    const uint64_t total = off_rec + roff[M];
    if (!out.allocate(total)) return MC_ERR_NOMEM;
    uint8_t* B = out.bytes;
    write_header(B, codec, n, uint32_t(M), O, E.vmax, E.tmax, tv, ttp, tt, 0, 0, 0, uint32_t(maxrec), off_dir,
                 off_obj, off_rec, total, mesh.bits, mesh.semantic, (vw ? 1u : 0u) | (cull ? 2u : 0u), off_cull);
    for (size_t m = 0; m <= M; ++m) put32(B + off_dir + 4 * m, uint32_t(roff[m] / 16));
    for (uint32_t o = 0; o < O; ++o)
        for (uint32_t c = 0; c < n; ++c) {
            std::memcpy(B + off_obj + 8ull * n * o + 4ull * c, &delta[size_t(o) * n + c], 4);
            std::memcpy(B + off_obj + 8ull * n * o + 4ull * (n + c), &origin[size_t(o) * n + c], 4);
        }
    out.src_vertex.resize(tv);
    out.src_tri.resize(ttp);
    const uint64_t hdr = round16(16 + 4ull * n + (vw ? n : 0));
    parallel_for(M, th, [&](size_t m) {
        const Meshlet& me = ms[m];
        uint8_t* r = B + off_rec + roff[m];
        put32(r, vb[m]); put32(r + 4, tb[m]);
        r[8] = uint8_t(me.V - 1); r[9] = uint8_t(me.Tp - 1);
        put16(r + 10, uint16_t(me.object)); put16(r + 12, uint16_t(me.R)); put16(r + 14, 0);
        for (uint32_t c = 0; c < n; ++c) put32(r + 16 + 4 * c, Lq[m * n + c]);
        if (vw)
            for (uint32_t c = 0; c < n; ++c) r[16 + 4 * n + c] = wq[m * n + c];
        const uint32_t W = codec == MC_CODEC_BASIC ? 0 : (me.Tp + 31) / 32;
        uint32_t* lr = reinterpret_cast<uint32_t*>(r + hdr);
        uint32_t* inc = lr + W;
        uint8_t* by = reinterpret_cast<uint8_t*>(inc + (codec == MC_CODEC_GTS_REUSE ? W : 0));
        uint32_t nb = 0, top = 2;
        if (codec == MC_CODEC_BASIC) {
            std::memcpy(by, me.tri3.data(), me.tri3.size());
            nb = uint32_t(me.tri3.size());
        }
        for (uint32_t t = 1; t < me.Tp && codec != MC_CODEC_BASIC; ++t) {
            if (me.flag[t]) lr[t / 32] |= 1u << (t % 32);
            uint32_t w = me.step[t - 1];
            if (codec == MC_CODEC_GTS) by[nb++] = uint8_t(w);
            else if (w == top + 1) { top = w; inc[t / 32] |= 1u << (t % 32); }
            else by[nb++] = uint8_t(w);
        }
        uint32_t* at = reinterpret_cast<uint32_t*>(by + ((nb + 3) & ~3u));
        const size_t ob = size_t(me.object) * n;
        uint64_t bitpos = 0;
        for (uint32_t v = 0; v < me.V; ++v) {
            const float* A = mesh.attributes + uint64_t(me.local_to_src[v]) * n;
            for (uint32_t c = 0; c < n; ++c) {
                uint32_t code = uint32_t(qof(A[c], origin[ob + c], delta[ob + c])) - Lq[m * n + c];
                uint32_t b = wq[m * n + c];
                if (b == 0) continue;
                uint64_t word = bitpos >> 5, sh = bitpos & 31;
                at[word] |= code << sh;
                if (sh + b > 32) at[word + 1] |= code >> (32 - sh);
                bitpos += b;
            }
            out.src_vertex[vb[m] + v] = me.local_to_src[v];
        }
        for (uint32_t t = 0; t < me.Tp; ++t) out.src_tri[tb[m] + t] = me.src_tri[t];
        if (cull) {
            // decoded positions exactly as a decoder computes them (FORMAT.md §3)
            std::vector<std::array<double, 3>> Pd(me.V);
            std::unordered_map<uint32_t, uint32_t> loc;
            for (uint32_t v = 0; v < me.V; ++v) {
                loc[me.local_to_src[v]] = v;
                const float* A = mesh.attributes + uint64_t(me.local_to_src[v]) * n;
                for (int k = 0; k < 3; ++k) {
                    const uint32_t c = pos_ch[k];
                    const uint32_t q = uint32_t(qof(A[c], origin[ob + c], delta[ob + c]));
                    Pd[v][k] = double(std::fma(float(q), delta[ob + c], origin[ob + c]));
                }
            }
            std::vector<std::array<uint32_t, 3>> tl;
            for (uint32_t st : me.src_tri)
                if (st != kNone) {
                    const uint32_t* v = mesh.indices + 3ull * st;
                    tl.push_back({loc[v[0]], loc[v[1]], loc[v[2]]});
                }
            cull_cone(Pd, tl, reinterpret_cast<float*>(B + off_cull + 16ull * m));
        }
    }, 16);
    out.has_map = true;
    out.restarts = rs;
    out.splits = E.splits;
    return MC_OK;
}

mc_status parse(const uint8_t* b, size_t nbytes, mc_layout* L) {
    if (!b || !L) return MC_ERR_ARG;
    if (nbytes < kHeaderBytes || std::memcmp(b, "MCZ1", 4) != 0 || get32(b + 4) != 1) return MC_ERR_FORMAT;
    std::memset(L, 0, sizeof(*L));
    L->codec = get32(b + 8); L->n = get32(b + 12); L->num_meshlets = get32(b + 16); L->num_objects = get32(b + 20);
    L->v_max = get32(b + 24); L->t_max = get32(b + 28); L->total_v = get32(b + 32); L->total_tp = get32(b + 36);
    L->total_t = get32(b + 40); L->base_meshlet = get32(b + 44); L->base_vtx = get32(b + 48);
    L->base_tri = get32(b + 52); L->max_record_bytes = get32(b + 56);
    L->off_dir = get64(b + 64); L->off_obj = get64(b + 72); L->off_rec = get64(b + 80); L->total_bytes = get64(b + 88);
    std::memcpy(L->bits, b + 96, 16);
    std::memcpy(L->semantic, b + 112, 16);
    L->flags = get32(b + 60);
    L->off_cull = get64(b + 128);
    if (L->flags & ~3u) return MC_ERR_FORMAT;
    if (L->codec != MC_CODEC_GTS && L->codec != MC_CODEC_GTS_REUSE && L->codec != MC_CODEC_BASIC) return MC_ERR_FORMAT;
    if (L->n < 1 || L->n > 16 || L->num_objects < 1 || L->v_max < 3 || L->v_max > 256 || L->t_max < 1 ||
        L->t_max > 256)
        return MC_ERR_FORMAT;
    if (L->total_bytes != nbytes || (L->off_dir & 15) || (L->off_obj & 15) || (L->off_rec & 15)) return MC_ERR_FORMAT;
    if (L->off_dir + 4ull * (L->num_meshlets + 1ull) > nbytes || L->off_obj + 8ull * L->n * L->num_objects > nbytes ||
        L->off_rec > nbytes || (L->max_record_bytes & 15) || L->max_record_bytes > 65536)
        return MC_ERR_FORMAT;
    L->S = 0;
    for (uint32_t c = 0; c < L->n; ++c) {
        if (L->bits[c] < 1 || L->bits[c] > 24) return MC_ERR_FORMAT;
        L->S += L->bits[c];
    }
    for (uint32_t c = 0; c < L->n; ++c)
        if (L->semantic[c] == MC_SEM_NORMAL_OCT) {
            if (c + 1 >= L->n || L->semantic[c + 1] != MC_SEM_NORMAL_OCT) return MC_ERR_FORMAT;
            ++c;
        }
    L->n_out = output_floats(L->n, L->semantic);
    // the cull table lies between the object table and the records (FORMAT.md §1.5)
    if ((L->flags & 2u) && ((L->off_cull & 15) || L->off_cull < L->off_obj + 8ull * L->n * L->num_objects ||
                            L->off_cull + 16ull * L->num_meshlets > L->off_rec))
        return MC_ERR_FORMAT;
    // the directory must stay inside the records section and be non-decreasing (host
    // helpers dereference and binary-search its entries: O(M), once per parse)
    uint32_t d0 = get32(b + L->off_dir), dM = get32(b + L->off_dir + 4ull * L->num_meshlets);
    if (d0 != 0 || L->off_rec + 16ull * dM > nbytes) return MC_ERR_FORMAT;
    uint32_t prev = 0;
    for (uint32_t m = 1; m <= L->num_meshlets; ++m) {
        const uint32_t d = get32(b + L->off_dir + 4ull * m);
        if (d < prev) return MC_ERR_FORMAT;
        prev = d;
    }
    return MC_OK;
}

}  // namespace

// ================================================================= C ABI (host part)
extern "C" {

uint32_t mc_abi_version(void) { return 4; }

const char* mc_status_str(mc_status s) {
    switch (s) {
        case MC_OK: return "ok";
        case MC_ERR_ARG: return "invalid argument";
        case MC_ERR_LIMITS: return "limits out of range";
        case MC_ERR_INPUT: return "invalid source mesh";
        case MC_ERR_FORMAT: return "not a valid MCZ1 blob";
        case MC_ERR_RANGE: return "value exceeds 32-bit range";
        case MC_ERR_CUDA: return "CUDA error";
        case MC_ERR_NOMEM: return "out of host memory";
    }
    return "unknown status";
}

mc_status mc_encode(const mc_mesh* mesh, const mc_encode_params* p, mc_blob** out) {
    if (!mesh || !p || !out) return MC_ERR_ARG;
    *out = nullptr;
    if (mesh->num_triangles && (!mesh->indices || !mesh->attributes)) return MC_ERR_ARG;
    if (!mesh->bits || !mesh->semantic) return MC_ERR_ARG;
    const uint32_t n = mesh->num_channels;
    if (n < 1 || n > 16 || p->max_vertices < 3 || p->max_vertices > 256 || p->max_triangles < 1 ||
        p->max_triangles > 256)
        return MC_ERR_LIMITS;
    if (p->codec != MC_CODEC_GTS && p->codec != MC_CODEC_GTS_REUSE && p->codec != MC_CODEC_BASIC) return MC_ERR_ARG;
    for (uint32_t c = 0; c < n; ++c) {
        if (mesh->bits[c] < 1 || mesh->bits[c] > 24) return MC_ERR_LIMITS;
        if (mesh->semantic[c] > MC_SEM_NORMAL_OCT) return MC_ERR_ARG;
        if (mesh->semantic[c] == MC_SEM_NORMAL_OCT) {
            if (c + 1 >= n || mesh->semantic[c + 1] != MC_SEM_NORMAL_OCT) return MC_ERR_ARG;
            ++c;
        }
    }
    for (uint64_t t = 0; t < mesh->num_triangles; ++t) {
        const uint32_t* v = mesh->indices + 3 * t;
        if (v[0] >= mesh->num_vertices || v[1] >= mesh->num_vertices || v[2] >= mesh->num_vertices)
            return MC_ERR_INPUT;
        if (v[0] == v[1] || v[1] == v[2] || v[0] == v[2]) return MC_ERR_INPUT;
    }
    try {
        Encoder E(*mesh, p->max_vertices, p->max_triangles, p->codec, worker_count(p->num_threads),
                  (p->flags & MC_ENCODE_VARIABLE_WIDTHS) != 0);
        E.cull = (p->flags & MC_ENCODE_CULL_CONES) != 0;
        mc_status st = E.run();
        if (st != MC_OK) return st;
        auto blob = std::make_unique<mc_blob>();
        st = serialise(E, *blob);
        if (st != MC_OK) return st;
        *out = blob.release();
        return MC_OK;
    } catch (const std::bad_alloc&) {
        return MC_ERR_NOMEM;
    } catch (...) {
        return MC_ERR_ARG;
    }
}

mc_status mc_blob_from_bytes(const void* bytes, size_t n, mc_blob** out) {
    if (!bytes || !out) return MC_ERR_ARG;
    mc_layout L;
    mc_status st = parse(static_cast<const uint8_t*>(bytes), n, &L);
    if (st != MC_OK) return st;
    auto blob = std::make_unique<mc_blob>();
    if (!blob->allocate(n)) return MC_ERR_NOMEM;
    std::memcpy(blob->bytes, bytes, n);
    *out = blob.release();
    return MC_OK;
}

mc_status mc_blob_bytes(const mc_blob* b, const void** bytes, size_t* n) {
    if (!b || !bytes || !n) return MC_ERR_ARG;
    *bytes = b->bytes;
    *n = b->size;
    return MC_OK;
}

mc_status mc_blob_source_map(const mc_blob* b, const uint32_t** sv, const uint32_t** st) {
    if (!b || !b->has_map) return MC_ERR_ARG;
    if (sv) *sv = b->src_vertex.data();
    if (st) *st = b->src_tri.data();
    return MC_OK;
}

mc_status mc_blob_encode_stats(const mc_blob* b, uint64_t* restarts, uint64_t* splits) {
    if (!b) return MC_ERR_ARG;
    if (restarts) *restarts = b->restarts;
    if (splits) *splits = b->splits;
    return MC_OK;
}

void mc_blob_free(mc_blob* b) { delete b; }

mc_status mc_parse_header(const void* bytes, size_t n, mc_layout* out) {
    return parse(static_cast<const uint8_t*>(bytes), n, out);
}

mc_status mc_blob_shard_ranges(const void* bytes, size_t n, uint32_t parts, uint32_t* first, uint32_t* count) {
    mc_layout L;
    mc_status st = parse(static_cast<const uint8_t*>(bytes), n, &L);
    if (st != MC_OK) return st;
    if (!parts || !first || !count) return MC_ERR_ARG;
    const uint8_t* b = static_cast<const uint8_t*>(bytes);
    const uint32_t M = L.num_meshlets;
    // algorithmic bytes per record: record read + index/vertex words written
    std::vector<double> cum(M + 1, 0.0);
    for (uint32_t m = 0; m < M; ++m) {
        uint64_t r0 = L.off_rec + 16ull * get32(b + L.off_dir + 4ull * m);
        uint64_t r1 = L.off_rec + 16ull * get32(b + L.off_dir + 4ull * (m + 1));
        uint32_t V = uint32_t(b[r0 + 8]) + 1, Tp = uint32_t(b[r0 + 9]) + 1;
        cum[m + 1] = cum[m] + double(r1 - r0) + 12.0 * Tp + 4.0 * L.n_out * V;
    }
    uint32_t prev = 0;
    for (uint32_t p = 0; p < parts; ++p) {
        double target = cum[M] * double(p + 1) / double(parts);
        uint32_t end = (p + 1 == parts) ? M : uint32_t(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
        end = std::max(end, prev);
        end = std::min(end, M);
        first[p] = prev;
        count[p] = end - prev;
        prev = end;
    }
    return MC_OK;
}

mc_status mc_blob_extract(const void* bytes, size_t n, uint32_t first, uint32_t count, mc_blob** out) {
    mc_layout L;
    const uint8_t* b = static_cast<const uint8_t*>(bytes);
    mc_status st = parse(b, n, &L);
    if (st != MC_OK) return st;
    if (!out || uint64_t(first) + count > L.num_meshlets) return MC_ERR_ARG;
    *out = nullptr;
    const uint64_t d0 = get32(b + L.off_dir + 4ull * first), d1 = get32(b + L.off_dir + 4ull * (first + count));
    const uint64_t rec_bytes = 16 * (d1 - d0);
    const bool cull = L.flags & 2u;
    const uint64_t off_dir = kHeaderBytes, off_obj = round16(off_dir + 4ull * (count + 1));
    const uint64_t off_cull = cull ? round16(off_obj + 8ull * L.n * L.num_objects) : 0;
    const uint64_t off_rec = cull ? round16(off_cull + 16ull * count) : round16(off_obj + 8ull * L.n * L.num_objects);
    const uint64_t total = off_rec + rec_bytes;
    auto blob = std::make_unique<mc_blob>();
    if (!blob->allocate(total)) return MC_ERR_NOMEM;
    uint8_t* B = blob->bytes;
    uint64_t tv = 0, ttp = 0, tt = 0, maxrec = 0;
    uint32_t bv = L.base_vtx, bt = L.base_tri;
    for (uint32_t m = first; m < first + count; ++m) {
        uint64_t r0 = L.off_rec + 16ull * get32(b + L.off_dir + 4ull * m);
        uint64_t r1 = L.off_rec + 16ull * get32(b + L.off_dir + 4ull * (m + 1));
        if (m == first) { bv = get32(b + r0); bt = get32(b + r0 + 4); }
        uint32_t V = uint32_t(b[r0 + 8]) + 1, Tp = uint32_t(b[r0 + 9]) + 1, R = get16(b + r0 + 12);
        tv += V; ttp += Tp; tt += Tp - 4ull * std::min<uint32_t>(R, Tp / 4);
        maxrec = std::max<uint64_t>(maxrec, r1 - r0);
    }
    write_header(B, L.codec, L.n, count, L.num_objects, L.v_max, L.t_max, tv, ttp, tt, L.base_meshlet + first, bv, bt,
                 uint32_t(std::max<uint64_t>(maxrec, 16)), off_dir, off_obj, off_rec, total, L.bits, L.semantic,
                 L.flags, off_cull);
    if (cull) std::memcpy(B + off_cull, b + L.off_cull + 16ull * first, 16ull * count);
    for (uint32_t m = 0; m <= count; ++m) put32(B + off_dir + 4ull * m, uint32_t(get32(b + L.off_dir + 4ull * (first + m)) - d0));
    std::memcpy(B + off_obj, b + L.off_obj, 8ull * L.n * L.num_objects);
    std::memcpy(B + off_rec, b + L.off_rec + 16 * d0, rec_bytes);
    *out = blob.release();
    return MC_OK;
}

mc_status mc_blob_info(const void* bytes, size_t nbytes, mc_info* out, mc_channel_grid* grids, uint32_t grids_len) {
    mc_layout L;
    const uint8_t* b = static_cast<const uint8_t*>(bytes);
    mc_status st = parse(b, nbytes, &L);
    if (st != MC_OK) return st;
    if (!out) return MC_ERR_ARG;
    const uint32_t n = L.n, M = L.num_meshlets, O = L.num_objects;
    const bool vw = L.flags & 1u;
    if (grids && uint64_t(grids_len) < uint64_t(O) * n) return MC_ERR_ARG;
    const uint32_t hdr = uint32_t(round16(16 + 4ull * n + (vw ? n : 0)));
    std::memset(out, 0, sizeof(*out));
    out->codec = L.codec;
    out->n = n;
    out->num_meshlets = M;
    out->num_objects = O;
    out->total_v = L.total_v;
    out->total_tp = L.total_tp;
    out->total_t = L.total_t;
    out->header_bytes = kHeaderBytes;
    out->directory_bytes = L.off_obj - L.off_dir;
    out->object_bytes = ((L.flags & 2u) ? L.off_cull : L.off_rec) - L.off_obj;
    out->cull_bytes = (L.flags & 2u) ? L.off_rec - L.off_cull : 0;
    out->record_bytes = L.total_bytes - L.off_rec;
    out->total_bytes = L.total_bytes;
    // per record: section sizes (FORMAT.md §1.4) and, per channel, the largest code and
    // the lowest / highest grid value q = L_c + code
    std::vector<uint64_t> lo(size_t(O) * n, UINT64_MAX), hi(size_t(O) * n, 0);
    std::vector<uint32_t> wmax(size_t(O) * n, 0);
    std::vector<uint32_t> code_max(n);
    for (uint32_t m = 0; m < M; ++m) {
        const uint64_t r0 = L.off_rec + 16ull * get32(b + L.off_dir + 4ull * m);
        const uint64_t r1 = L.off_rec + 16ull * get32(b + L.off_dir + 4ull * (m + 1));
        if (r1 < r0 + hdr) return MC_ERR_FORMAT;
        const uint32_t V = uint32_t(b[r0 + 8]) + 1, Tp = uint32_t(b[r0 + 9]) + 1, obj = get16(b + r0 + 10);
        if (obj >= O) return MC_ERR_FORMAT;
        out->restarts += get16(b + r0 + 12);
        const uint32_t W = L.codec == MC_CODEC_BASIC ? 0u : (Tp + 31) / 32;
        const uint64_t flag_b = 4ull * W * (L.codec == MC_CODEC_GTS_REUSE ? 2 : 1);
        const uint64_t nb = L.codec == MC_CODEC_GTS ? Tp - 1ull
                            : L.codec == MC_CODEC_BASIC ? 3ull * Tp
                            : (V >= 3 && V - 3 <= Tp - 1 ? (Tp - 1ull) - (V - 3ull) : 0);
        uint32_t S = 0;
        uint8_t wd[16];
        for (uint32_t c = 0; c < n; ++c) {
            wd[c] = vw ? b[r0 + 16 + 4 * n + c] : L.bits[c];
            if (wd[c] > L.bits[c]) return MC_ERR_FORMAT;
            S += wd[c];
        }
        const uint64_t at = r0 + hdr + flag_b + ((nb + 3) & ~3ull);
        const uint64_t at_b = (uint64_t(V) * S + 31) / 32 * 4;
        if (at + at_b > r1) return MC_ERR_FORMAT;
        out->record_header_bytes += hdr;
        out->flag_bytes += flag_b;
        out->index_bytes += nb;
        out->attribute_bytes += (uint64_t(V) * S + 7) / 8;
        // little-endian bit string of V records of S bits (FORMAT.md §1.4)
        std::fill(code_max.begin(), code_max.end(), 0u);
        uint64_t bit = 0;
        for (uint32_t v = 0; v < V; ++v)
            for (uint32_t c = 0; c < n; ++c) {
                uint64_t word = 0;
                const uint64_t byte0 = bit >> 3;
                for (uint32_t k = 0; k < 5 && at + byte0 + k < r1; ++k) word |= uint64_t(b[at + byte0 + k]) << (8 * k);
                const uint32_t code = wd[c] ? uint32_t((word >> (bit & 7)) & ((1ull << wd[c]) - 1)) : 0u;
                code_max[c] = std::max(code_max[c], code);
                bit += wd[c];
            }
        for (uint32_t c = 0; c < n; ++c) {
            const size_t k = size_t(obj) * n + c;
            const uint64_t Lc = get32(b + r0 + 16 + 4ull * c);
            lo[k] = std::min(lo[k], Lc);
            hi[k] = std::max(hi[k], Lc + code_max[c]);
            wmax[k] = std::max(wmax[k], code_max[c]);
        }
    }
    out->padding_bytes = out->record_bytes - out->record_header_bytes - out->flag_bytes - out->index_bytes -
                         out->attribute_bytes;
    out->bits_per_triangle = L.total_t ? 8.0 * double(L.total_bytes) / double(L.total_t) : 0.0;
    out->index_bits_per_triangle = L.total_t ? 8.0 * double(out->flag_bytes + out->index_bytes) / double(L.total_t) : 0.0;
    if (grids)
        for (uint32_t o = 0; o < O; ++o)
            for (uint32_t c = 0; c < n; ++c) {
                const size_t k = size_t(o) * n + c;
                mc_channel_grid& g = grids[k];
                float d, org;
                std::memcpy(&d, b + L.off_obj + 8ull * n * o + 4ull * c, 4);
                std::memcpy(&org, b + L.off_obj + 8ull * n * o + 4ull * (n + c), 4);
                g.delta = d;
                g.origin = org;
                g.bits = L.bits[c];
                g.w_steps = wmax[k];
                g.W_steps = lo[k] == UINT64_MAX ? 0 : hi[k] - lo[k];
                g.w = double(g.w_steps) * double(d);
                g.W = double(g.W_steps) * double(d);
                g.info_bits = g.W_steps ? std::log2(double(g.W_steps)) : 0.0;
            }
    return MC_OK;
}

mc_status mc_blob_instance(const mc_blob* const* protos, uint32_t num_protos, const uint32_t* proto_of_instance,
                           const float* offset, uint32_t num_instances, mc_blob** out) {
    return mc_blob_instance_range(protos, num_protos, proto_of_instance, offset, num_instances, 0, num_instances, out);
}

mc_status mc_blob_instance_range(const mc_blob* const* protos, uint32_t num_protos, const uint32_t* proto_of_instance,
                                 const float* offset, uint32_t num_instances, uint32_t first_instance,
                                 uint32_t instance_count, mc_blob** out) {
    if (!protos || !num_protos || !proto_of_instance || !offset || !out) return MC_ERR_ARG;
    if (uint64_t(first_instance) + instance_count > num_instances) return MC_ERR_ARG;
    *out = nullptr;
    std::vector<mc_layout> Ls(num_protos);
    for (uint32_t p = 0; p < num_protos; ++p) {
        if (!protos[p]) return MC_ERR_ARG;
        mc_status st = parse(protos[p]->bytes, protos[p]->size, &Ls[p]);
        if (st != MC_OK) return st;
        if (Ls[p].codec != Ls[0].codec || Ls[p].n != Ls[0].n || std::memcmp(Ls[p].bits, Ls[0].bits, 16) ||
            Ls[p].flags != Ls[0].flags ||
            std::memcmp(Ls[p].semantic, Ls[0].semantic, 16))
            return MC_ERR_ARG;
    }
    const mc_layout& L0 = Ls[0];
    // global bases of the range: everything the instances before it produce
    uint64_t gm = 0, gv = 0, gt = 0;
    for (uint32_t i = 0; i < first_instance; ++i) {
        if (proto_of_instance[i] >= num_protos) return MC_ERR_ARG;
        const mc_layout& L = Ls[proto_of_instance[i]];
        gm += L.num_meshlets; gv += L.total_v; gt += L.total_tp;
    }
    const uint32_t* poi = proto_of_instance + first_instance;
    const float* offs = offset + 3ull * first_instance;
    num_instances = instance_count;
    uint64_t M = 0, O = 0, tv = 0, ttp = 0, tt = 0, rb = 0, maxrec = 0;
    uint32_t vmax = 0, tmax = 0;
    for (uint32_t i = 0; i < num_instances; ++i) {
        uint32_t p = poi[i];
        if (p >= num_protos) return MC_ERR_ARG;
        const mc_layout& L = Ls[p];
        M += L.num_meshlets; O += L.num_objects; tv += L.total_v; ttp += L.total_tp; tt += L.total_t;
        rb += L.total_bytes - L.off_rec;
        maxrec = std::max<uint64_t>(maxrec, L.max_record_bytes);
        vmax = std::max(vmax, L.v_max);
        tmax = std::max(tmax, L.t_max);
    }
    if (O > 65536 || gv + tv > 0xFFFFFFFFull || 3 * (gt + ttp) > 0xFFFFFFFFull || rb / 16 > 0xFFFFFFFFull ||
        gm + M > 0xFFFFFFFFull)
        return MC_ERR_RANGE;
    const uint32_t n = L0.n;
    const bool cull = L0.flags & 2u;
    const uint64_t off_dir = kHeaderBytes, off_obj = round16(off_dir + 4ull * (M + 1));
    const uint64_t off_cull = cull ? round16(off_obj + 8ull * n * O) : 0;
    const uint64_t off_rec = cull ? round16(off_cull + 16ull * M) : round16(off_obj + 8ull * n * O);
    const uint64_t total = off_rec + rb;
    auto blob = std::make_unique<mc_blob>();
    if (!blob->allocate(total)) return MC_ERR_NOMEM;
    uint8_t* B = blob->bytes;
    write_header(B, L0.codec, n, uint32_t(M), uint32_t(O), vmax, tmax, tv, ttp, tt, uint32_t(gm), uint32_t(gv),
                 uint32_t(gt), uint32_t(maxrec), off_dir, off_obj, off_rec, total, L0.bits, L0.semantic, L0.flags,
                 off_cull);
    // per-instance prefix sums, then fill instances in parallel
    std::vector<uint64_t> im(num_instances + 1, 0), io(num_instances + 1, 0), iv(num_instances + 1, 0),
        it(num_instances + 1, 0), ir(num_instances + 1, 0);
    iv[0] = gv;
    it[0] = gt;
    for (uint32_t i = 0; i < num_instances; ++i) {
        const mc_layout& L = Ls[poi[i]];
        im[i + 1] = im[i] + L.num_meshlets; io[i + 1] = io[i] + L.num_objects;
        iv[i + 1] = iv[i] + L.total_v; it[i + 1] = it[i] + L.total_tp; ir[i + 1] = ir[i] + (L.total_bytes - L.off_rec);
    }
    parallel_for(num_instances, worker_count(0), [&](size_t i) {
        const uint32_t p = poi[i];
        const mc_layout& L = Ls[p];
        const uint8_t* src = protos[p]->bytes;
        // objects: position-channel origins shifted by the instance translation
        for (uint32_t o = 0; o < L.num_objects; ++o) {
            uint8_t* dst = B + off_obj + 8ull * n * (io[i] + o);
            std::memcpy(dst, src + L.off_obj + 8ull * n * o, 8ull * n);
            uint32_t pc = 0;
            for (uint32_t c = 0; c < n && pc < 3; ++c)
                if (L.semantic[c] == MC_SEM_POSITION) {
                    float g;
                    std::memcpy(&g, dst + 4ull * (n + c), 4);
                    g = g + offs[3ull * i + pc++];
                    std::memcpy(dst + 4ull * (n + c), &g, 4);
                }
        }
        std::memcpy(B + off_rec + ir[i], src + L.off_rec, L.total_bytes - L.off_rec);
        // cones are translation invariant (the margin covers re-rounded origins)
        if (cull) std::memcpy(B + off_cull + 16ull * im[i], src + L.off_cull, 16ull * L.num_meshlets);
        for (uint32_t m = 0; m < L.num_meshlets; ++m) {
            uint32_t d = get32(src + L.off_dir + 4ull * m);
            put32(B + off_dir + 4ull * (im[i] + m), uint32_t(ir[i] / 16 + d));
            uint8_t* r = B + off_rec + ir[i] + 16ull * d;
            put32(r, uint32_t(get32(r) - L.base_vtx + iv[i]));
            put32(r + 4, uint32_t(get32(r + 4) - L.base_tri + it[i]));
            put16(r + 10, uint16_t(get16(r + 10) + io[i]));
        }
    }, 1);
    put32(B + off_dir + 4ull * M, uint32_t(rb / 16));
    *out = blob.release();
    return MC_OK;
}

}  // extern "C"
