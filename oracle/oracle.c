/*
 * oracle.c — the test oracle for per-meshlet decompression (arXiv 2404.06359).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product
 * (paper_2404_06359_b200) never links, imports or calls it, and this file shares
 * no code, header, table or constant generator with the product: the only
 * contract between the two is the prose of FORMAT.md.
 *
 * Plain, slow, obviously-correct C:
 *   - or_decode_meshlet: the SEQUENTIAL generalized-triangle-strip walk of
 *     PAPER §2 and §4.2/§4.3, in the paper's order,
 *     plus the dequantisation of §4.4.
 *   - or_encode: an independent encoder — a BFS meshlet builder, a lowest-index
 *     greedy stripifier, the 4-degenerate restart, meshlet
 *     splitting when T' = T + 4R exceeds T~, the ascending vertex
 *     reorder, GTS / GTS-Reuse stream emission (P:420-426,
 *     P:459-467) and the crack-free global-grid quantiser.
 *   - Basic (codec 3): the paper's uncompressed mesh-shading control — three
 *     local u8 indices per triangle (Table 2).
 *   - VW blobs (FORMAT.md §1.4, extension f1): per-meshlet attribute widths
 *     w_c = bit length of the meshlet's largest code on the unchanged global grid.
 *   - or_pack: serialises caller-given raw streams WITHOUT validation so tests
 *     can build exhaustive and malformed inputs.
 * Floating point: compiled with -ffp-contract=off; every fused multiply-add is an
 * explicit fmaf (FORMAT.md §3, §4.3).
 *
 * Parity status: sequential decode, restarts, reuse expansion,
 * quantiser and budgets are pinned by tests/test_oracle_*.py; the binary32
 * dequantisation by tests/test_oracle_dequant.py (exact rationals).  The octahedral
 * normal decode (or_oct_decode) is an extension the paper does not define (FORMAT.md
 * §4.3, reading R13): pinned by closed-form special cases and by float64 error bounds
 * (<= 4 ulp normalisation, <= 2^-21 absolute end to end), not by the paper.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_ERR_ARG 1
#define OR_ERR_LIMITS 2
#define OR_ERR_INPUT 3
#define OR_ERR_FORMAT 4
#define OR_ERR_RANGE 5
#define OR_ERR_NOMEM 7

/* FORMAT.md §5 record error bits */
#define DERR_RECORD 1u
#define DERR_COUNTS 2u
#define DERR_INDEX 4u
#define DERR_REUSE 8u
#define DERR_OBJECT 16u

#define CODEC_GTS 1u
#define CODEC_REUSE 2u
#define CODEC_BASIC 3u   /* three local u8 indices per triangle: the paper's "Basic" */
#define SEM_OCT 4u

/* ------------------------------------------------------------------ byte access */
static uint32_t rd32(const uint8_t *p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}
static uint16_t rd16(const uint8_t *p) { return (uint16_t)(p[0] | (p[1] << 8)); }
static uint64_t rd64(const uint8_t *p) { return (uint64_t)rd32(p) | ((uint64_t)rd32(p + 4) << 32); }
static float rdf(const uint8_t *p) {
    uint32_t u = rd32(p);
    float f;
    memcpy(&f, &u, 4);
    return f;
}
static void wr32(uint8_t *p, uint32_t v) {
    p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); p[2] = (uint8_t)(v >> 16); p[3] = (uint8_t)(v >> 24);
}
static void wr16(uint8_t *p, uint16_t v) { p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); }
static void wr64(uint8_t *p, uint64_t v) { wr32(p, (uint32_t)v); wr32(p + 4, (uint32_t)(v >> 32)); }
static void wrf(uint8_t *p, float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    wr32(p, u);
}
static uint64_t up16(uint64_t x) { return (x + 15u) & ~(uint64_t)15u; }

/* bit t of a little-endian bit string stored as u32 words (FORMAT.md §1.4) */
static unsigned get_bit(const uint8_t *words, uint32_t t) {
    return (rd32(words + 4u * (t / 32u)) >> (t % 32u)) & 1u;
}

/* the b-bit field starting at bit p of a little-endian bit string: read bit by bit */
static uint32_t get_field(const uint8_t *words, uint64_t p, unsigned b) {
    uint32_t v = 0;
    for (unsigned k = 0; k < b; ++k) v |= (uint32_t)get_bit(words, (uint32_t)(p + k)) << k;
    return v;
}

/* ------------------------------------------------------------------ blob header */
typedef struct {
    uint32_t codec, n, M, O, vmax, tmax, total_v, total_tp, total_t;
    uint32_t base_meshlet, base_vtx, base_tri, max_record_bytes;
    uint64_t off_dir, off_obj, off_rec, total_bytes;
    uint8_t bits[16], sem[16];
    uint32_t S, n_out;
    uint32_t vw;   /* FORMAT.md §1.1 flags bit 0: per-meshlet attribute widths (extension f1) */
    uint32_t cull; /* flags bit 1: cull table present (extension f2) */
    uint64_t off_cull;
} or_hdr;

static int parse_header(const uint8_t *b, size_t nbytes, or_hdr *h) {
    if (nbytes < 160 || memcmp(b, "MCZ1", 4) != 0 || rd32(b + 4) != 1) return OR_ERR_FORMAT;
    h->codec = rd32(b + 8); h->n = rd32(b + 12); h->M = rd32(b + 16); h->O = rd32(b + 20);
    h->vmax = rd32(b + 24); h->tmax = rd32(b + 28); h->total_v = rd32(b + 32);
    h->total_tp = rd32(b + 36); h->total_t = rd32(b + 40); h->base_meshlet = rd32(b + 44);
    h->base_vtx = rd32(b + 48); h->base_tri = rd32(b + 52); h->max_record_bytes = rd32(b + 56);
    h->off_dir = rd64(b + 64); h->off_obj = rd64(b + 72); h->off_rec = rd64(b + 80);
    h->total_bytes = rd64(b + 88);
    memcpy(h->bits, b + 96, 16);
    memcpy(h->sem, b + 112, 16);
    uint32_t flags = rd32(b + 60);
    if (flags & ~3u) return OR_ERR_FORMAT;
    h->vw = flags & 1u;
    h->cull = (flags >> 1) & 1u;
    h->off_cull = rd64(b + 128);
    /* the cull table lies between the object table and the records (FORMAT.md §1.5) */
    if (h->cull && (h->off_cull % 16u || h->off_cull < h->off_obj + 8ull * h->n * h->O ||
                    h->off_cull + 16ull * h->M > h->off_rec))
        return OR_ERR_FORMAT;
    if (h->codec != CODEC_GTS && h->codec != CODEC_REUSE && h->codec != CODEC_BASIC) return OR_ERR_FORMAT;
    if (h->n < 1 || h->n > 16 || h->O < 1) return OR_ERR_FORMAT;
    if (h->total_bytes != nbytes) return OR_ERR_FORMAT;
    if (h->off_dir + 4ull * (h->M + 1ull) > nbytes || h->off_obj + 8ull * h->n * h->O > nbytes ||
        h->off_rec > nbytes)
        return OR_ERR_FORMAT;
    h->S = 0;
    h->n_out = h->n;
    for (uint32_t c = 0; c < h->n; ++c) {
        if (h->bits[c] < 1 || h->bits[c] > 24) return OR_ERR_FORMAT;
        h->S += h->bits[c];
    }
    for (uint32_t c = 0; c < h->n; ++c)
        if (h->sem[c] == SEM_OCT) {
            if (c + 1 >= h->n || h->sem[c + 1] != SEM_OCT) return OR_ERR_FORMAT;
            h->n_out += 1;
            ++c;
        }
    return OR_OK;
}

int or_blob_info(const uint8_t *blob, size_t nbytes, uint32_t *out /* 16 u32 */) {
    or_hdr h;
    int st = parse_header(blob, nbytes, &h);
    if (st) return st;
    uint32_t v[16] = {h.codec, h.n, h.M, h.O, h.vmax, h.tmax, h.total_v, h.total_tp, h.total_t,
                      h.base_meshlet, h.base_vtx, h.base_tri, h.max_record_bytes, h.S, h.n_out, h.vw};
    memcpy(out, v, sizeof v);
    return OR_OK;
}

/* ------------------------------------------------------------------ octahedral decode
 * FORMAT.md §4.3 (extension for BASELINE cfg3; the paper only cites octahedral
 * normals as prior work).  Every step binary32, round-to-nearest. */
void or_oct_decode(float ex, float ey, float *out3) {
    float ax = fabsf(ex), ay = fabsf(ey);
    float z = (1.0f - ax) - ay;
    float x, y;
    if (z < 0.0f) {
        x = (1.0f - ay) * (ex >= 0.0f ? 1.0f : -1.0f);
        y = (1.0f - ax) * (ey >= 0.0f ? 1.0f : -1.0f);
    } else {
        x = ex;
        y = ey;
    }
    float xx = x * x;
    float s2 = fmaf(z, z, fmaf(y, y, xx));
    float r = sqrtf(s2);
    float inv = 1.0f / r;
    out3[0] = x * inv;
    out3[1] = y * inv;
    out3[2] = z * inv;
}

/* ------------------------------------------------------------------ sequential decode
 * Decode record m of the blob.  Outputs are LOCAL to the meshlet:
 *   tri_out[3*T'] local vertex indices (add vtx_base for the global index buffer),
 *   q_out[V*n]   global-grid integers q = L + code        (may be NULL),
 *   f_out[V*n_out] dequantised floats                     (may be NULL).
 * meta_out (may be NULL) = {vtx_base, tri_base, V, T', object, R}.
 * Returns FORMAT.md §5 error bits (0 = well-formed). */
uint32_t or_decode_meshlet(const uint8_t *blob, size_t nbytes, uint32_t m, uint32_t *tri_out,
                           uint32_t *q_out, float *f_out, uint32_t *meta_out) {
    or_hdr h;
    if (parse_header(blob, nbytes, &h) != OR_OK || m >= h.M) return DERR_RECORD;
    uint64_t r0 = h.off_rec + 16ull * rd32(blob + h.off_dir + 4ull * m);
    uint64_t r1 = h.off_rec + 16ull * rd32(blob + h.off_dir + 4ull * (m + 1));
    if (r1 <= r0 || r1 > nbytes || r0 + 16 > nbytes) return DERR_RECORD;
    const uint8_t *rec = blob + r0;

    uint32_t vtx_base = rd32(rec), tri_base = rd32(rec + 4);
    uint32_t V = (uint32_t)rec[8] + 1u, Tp = (uint32_t)rec[9] + 1u;
    uint32_t object = rd16(rec + 10), R = rd16(rec + 12);
    if (meta_out) {
        meta_out[0] = vtx_base; meta_out[1] = tri_base; meta_out[2] = V;
        meta_out[3] = Tp; meta_out[4] = object; meta_out[5] = R;
    }
    uint32_t n = h.n;
    /* Basic records have no flag words (FORMAT.md §1.4) */
    uint32_t W = h.codec == CODEC_BASIC ? 0u : (Tp + 31u) / 32u;
    uint64_t hdr_bytes = up16(16u + 4ull * n + (h.vw ? n : 0u));
    /* attribute widths: the blob's b_c, or the record's w_c with VW (FORMAT.md §1.4) */
    uint8_t wid[16];
    uint32_t S = 0, wbad = 0;
    for (uint32_t c = 0; c < n; ++c) {
        wid[c] = h.vw ? rec[16 + 4 * n + c] : h.bits[c];
        if (wid[c] > h.bits[c]) wbad = 1;
        S += wid[c];
    }
    uint32_t nb;
    if (h.codec == CODEC_GTS) nb = Tp - 1u;
    else if (h.codec == CODEC_BASIC) nb = 3u * Tp;
    else nb = (V >= 3u && V - 3u <= Tp - 1u) ? (Tp - 1u) - (V - 3u) : 0u;
    uint64_t off_lr = hdr_bytes;
    uint64_t off_inc = off_lr + 4ull * W;
    uint64_t off_bytes = off_inc + (h.codec == CODEC_REUSE ? 4ull * W : 0ull);
    uint64_t off_attr = off_bytes + ((nb + 3ull) & ~3ull);
    uint64_t attr_words = ((uint64_t)V * S + 31u) / 32u;
    uint64_t size = up16(off_attr + 4ull * attr_words);
    uint32_t err = 0;
    if (size != r1 - r0 || size > h.max_record_bytes || wbad) return DERR_RECORD;
    if (V < 3u || V > h.vmax || Tp > h.tmax) err |= DERR_COUNTS;
    if (object >= h.O) err |= DERR_OBJECT;
    if (h.codec == CODEC_BASIC && R != 0u) err |= DERR_COUNTS;   /* Basic has no restarts */

    const uint8_t *LR = rec + off_lr, *INC = rec + off_inc, *BY = rec + off_bytes, *AT = rec + off_attr;

    /* Step sequence N (FORMAT.md §2): N[0..2] = 0,1,2. */
    uint32_t N[258];
    N[0] = 0; N[1] = 1; N[2] = 2;
    if (h.codec == CODEC_REUSE) {
        uint32_t total = 0;
        for (uint32_t t = 1; t < Tp; ++t) total += get_bit(INC, t);
        if (total != V - 3u) err |= DERR_COUNTS;
    }
    /* structural errors (RECORD/COUNTS/OBJECT) end the record: FORMAT.md §5 evaluates
     * INDEX/REUSE only for structurally valid records */
    if (err) return err;
    if (h.codec == CODEC_BASIC) {
        /* Basic: the triangle list itself, three local indices per triangle */
        for (uint32_t t = 0; t < Tp; ++t)
            for (uint32_t k = 0; k < 3u; ++k) {
                uint32_t w = BY[3u * t + k];
                if (w >= V) err |= DERR_INDEX;
                if (tri_out) tri_out[3u * t + k] = w;
            }
        goto attributes;
    }
    uint32_t c = 0; /* inclusive add-scan of increment flags over triangles 1..t */
    for (uint32_t t = 1; t < Tp; ++t) {
        uint32_t w;
        if (h.codec == CODEC_GTS) {
            w = BY[t - 1];                      /* explicit index per triangle */
            if (w >= V) err |= DERR_INDEX;
        } else {
            uint32_t inc = get_bit(INC, t);
            c += inc;
            if (inc) {
                w = 2u + c;                     /* "the result of the scan s is the current index" */
            } else {
                uint32_t pos = t - c - 1u;      /* "reuse array ... at location t+1-s", s = 2 + c (R5) */
                if (pos >= nb) { err |= DERR_COUNTS; w = 0; }
                else { w = BY[pos]; if (w >= V) err |= DERR_REUSE; }
            }
        }
        N[t + 2] = w;
    }

    /* The sequential GTS walk: R crosses (b,c) -> (c,b,w); L crosses (c,a) -> (a,c,w). */
    uint32_t a = N[0], b = N[1], cc = N[2];
    if (tri_out) { tri_out[0] = a; tri_out[1] = b; tri_out[2] = cc; }
    for (uint32_t t = 1; t < Tp; ++t) {
        uint32_t w = N[t + 2];
        uint32_t na, nb2, nc;
        if (get_bit(LR, t)) { na = cc; nb2 = b; nc = w; }   /* R */
        else                { na = a;  nb2 = cc; nc = w; }  /* L */
        a = na; b = nb2; cc = nc;
        if (tri_out) { tri_out[3 * t] = a; tri_out[3 * t + 1] = b; tri_out[3 * t + 2] = cc; }
    }

attributes:
    /* Attributes: q = L_i + code on the global grid; x = fmaf((float)q, Δ, g). */
    if ((q_out || f_out) && !(err & (DERR_OBJECT | DERR_COUNTS))) {
        const uint8_t *obj = blob + h.off_obj + 8ull * n * object;
        for (uint32_t v = 0; v < V; ++v) {
            uint64_t p = (uint64_t)v * S;
            uint32_t q[16];
            for (uint32_t ch = 0; ch < n; ++ch) {
                uint32_t code = get_field(AT, p, wid[ch]);
                p += wid[ch];
                q[ch] = rd32(rec + 16 + 4 * ch) + code;
                if (q_out) q_out[(uint64_t)v * n + ch] = q[ch];
            }
            if (f_out) {
                float *o = f_out + (uint64_t)v * h.n_out;
                uint32_t k = 0;
                for (uint32_t ch = 0; ch < n; ++ch) {
                    float delta = rdf(obj + 4 * ch), origin = rdf(obj + 4 * (n + ch));
                    float x = fmaf((float)q[ch], delta, origin);
                    if (h.sem[ch] == SEM_OCT) {
                        float d2 = rdf(obj + 4 * (ch + 1)), o2 = rdf(obj + 4 * (n + ch + 1));
                        float y = fmaf((float)q[ch + 1], d2, o2);
                        or_oct_decode(x, y, o + k);
                        k += 3;
                        ++ch;
                    } else {
                        o[k++] = x;
                    }
                }
            }
        }
    }
    return err;
}

/* Decode records [m0, m1) into whole-blob output buffers at FORMAT.md §2/§4 positions
 * (relative to base_tri / base_vtx).  idx: 3*total_tp u32 (global vertex indices);
 * q: n*total_v (or NULL); f: n_out*total_v (or NULL); err_out[m1-m0] (or NULL).
 * Returns the OR of all error bits. */
uint32_t or_decode_range(const uint8_t *blob, size_t nbytes, uint32_t m0, uint32_t m1,
                         uint32_t *idx, uint32_t *q, float *f, uint32_t *err_out) {
    or_hdr h;
    if (parse_header(blob, nbytes, &h) != OR_OK) return DERR_RECORD;
    uint32_t all = 0;
    uint32_t tri[3 * 256];
    uint32_t qq[256 * 16];
    float ff[256 * 24];
    for (uint32_t m = m0; m < m1 && m < h.M; ++m) {
        uint32_t meta[6] = {0};
        uint32_t e = or_decode_meshlet(blob, nbytes, m, tri, q ? qq : NULL, f ? ff : NULL, meta);
        if (err_out) err_out[m - m0] = e;
        all |= e;
        if (e & (DERR_RECORD | DERR_COUNTS | DERR_OBJECT)) continue;
        uint32_t V = meta[2], Tp = meta[3];
        uint64_t tb = (uint64_t)meta[1] - h.base_tri, vb = (uint64_t)meta[0] - h.base_vtx;
        if (tb + Tp > h.total_tp || vb + V > h.total_v) { if (err_out) err_out[m - m0] |= DERR_RECORD; all |= DERR_RECORD; continue; }
        for (uint32_t k = 0; k < 3 * Tp; ++k) idx[3 * tb + k] = meta[0] + tri[k];
        if (q) memcpy(q + vb * h.n, qq, 4ull * V * h.n);
        if (f) memcpy(f + vb * h.n_out, ff, 4ull * V * h.n_out);
    }
    return all;
}

/* Local u8x4 index output (FORMAT.md §2, decode flag MC_DECODE_INDEX_LOCAL_U8X4):
 * triangle t of record m -> word (tri_base - base_tri + t) = a | b<<8 | c<<16 with the
 * meshlet-local indices of the sequential decode (the paper's 8-bit meshlet indices).
 * words: total_tp u32.  Returns the OR of all error bits. */
uint32_t or_decode_range_u8x4(const uint8_t *blob, size_t nbytes, uint32_t m0, uint32_t m1, uint32_t *words) {
    or_hdr h;
    if (parse_header(blob, nbytes, &h) != OR_OK) return DERR_RECORD;
    uint32_t all = 0;
    uint32_t tri[3 * 256];
    for (uint32_t m = m0; m < m1 && m < h.M; ++m) {
        uint32_t meta[6] = {0};
        uint32_t e = or_decode_meshlet(blob, nbytes, m, tri, NULL, NULL, meta);
        all |= e;
        if (e & (DERR_RECORD | DERR_COUNTS | DERR_OBJECT)) continue;
        uint64_t tb = (uint64_t)meta[1] - h.base_tri;
        uint32_t Tp = meta[3];
        if (tb + Tp > h.total_tp) { all |= DERR_RECORD; continue; }
        for (uint32_t t = 0; t < Tp; ++t)
            words[tb + t] = (tri[3 * t] & 0xFFu) | ((tri[3 * t + 1] & 0xFFu) << 8) | ((tri[3 * t + 2] & 0xFFu) << 16);
    }
    return all;
}

/* ------------------------------------------------------------------ cone culling (FORMAT.md §1.5, §7)
 * The paper's amplification-shader cone test: record m is culled for view
 * direction d iff fmaf(az, dz, fmaf(ay, dy, ax*dx)) > cutoff in binary32. */
static int or_culled(const uint8_t *blob, const or_hdr *h, uint32_t m, const float *d) {
    const uint8_t *e = blob + h->off_cull + 16ull * m;
    float ax = rdf(e), ay = rdf(e + 4), az = rdf(e + 8), cutoff = rdf(e + 12);
    float s = fmaf(az, d[2], fmaf(ay, d[1], ax * d[0]));
    return s > cutoff;
}

/* Culled, compacted decode (FORMAT.md §7), sequential in record order.
 * idx: 3*total_tp u32 (or total_tp u8x4 words when u8x4), q/f as or_decode_range (may be
 * NULL), vis[M] (may be NULL) = 1 for visible records.  counts[4] = {visible records,
 * sum V, sum T', sum real T}.  Returns the OR of the visible records' error bits. */
uint32_t or_decode_culled(const uint8_t *blob, size_t nbytes, const float *d, uint32_t u8x4, uint32_t *idx,
                          uint32_t *q, float *f, uint8_t *vis, uint64_t *counts) {
    or_hdr h;
    counts[0] = counts[1] = counts[2] = counts[3] = 0;
    if (parse_header(blob, nbytes, &h) != OR_OK || !h.cull) return DERR_RECORD;
    uint32_t all = 0;
    uint32_t tri[3 * 256];
    uint32_t qq[256 * 16];
    float ff[256 * 24];
    uint64_t VB = 0, TB = 0;
    for (uint32_t m = 0; m < h.M; ++m) {
        if (vis) vis[m] = 0;
        /* never visible: empty/oversized directory span or out-of-range counts (§7) */
        uint64_t r0 = 16ull * rd32(blob + h.off_dir + 4ull * m), r1 = 16ull * rd32(blob + h.off_dir + 4ull * (m + 1));
        if (r1 <= r0 || r1 - r0 > h.max_record_bytes || h.off_rec + r1 > nbytes) continue;
        const uint8_t *rec = blob + h.off_rec + r0;
        uint32_t V = (uint32_t)rec[8] + 1u, Tp = (uint32_t)rec[9] + 1u, R = rd16(rec + 12);
        if (V < 3u || V > h.vmax || Tp > h.tmax) continue;
        if (or_culled(blob, &h, m, d)) continue;
        if (vis) vis[m] = 1;
        uint32_t meta[6] = {0};
        uint32_t e = or_decode_meshlet(blob, nbytes, m, tri, q ? qq : NULL, f ? ff : NULL, meta);
        all |= e;
        if (!(e & (DERR_RECORD | DERR_COUNTS | DERR_OBJECT))) {
            for (uint32_t t = 0; t < Tp; ++t) {
                if (u8x4) idx[TB + t] = (tri[3 * t] & 0xFFu) | ((tri[3 * t + 1] & 0xFFu) << 8) | ((tri[3 * t + 2] & 0xFFu) << 16);
                else for (uint32_t k = 0; k < 3; ++k) idx[3 * (TB + t) + k] = (uint32_t)VB + tri[3 * t + k];
            }
            if (q) memcpy(q + VB * h.n, qq, 4ull * V * h.n);
            if (f) memcpy(f + VB * h.n_out, ff, 4ull * V * h.n_out);
        }
        counts[0] += 1; counts[1] += V; counts[2] += Tp; counts[3] += Tp - 4ull * (R <= Tp / 4 ? R : Tp / 4);
        VB += V;
        TB += Tp;
    }
    return all;
}

/* Insert (or replace) a cull table: entries[4*M] = {ax, ay, az, cutoff} per record.
 * Directory offsets are relative to off_rec, so the records move as one block.
 * Output malloc'd (free with or_free). */
int or_add_cull(const uint8_t *blob, size_t nbytes, const float *entries, uint8_t **out, uint64_t *out_bytes) {
    or_hdr h;
    int st = parse_header(blob, nbytes, &h);
    if (st) return st;
    uint64_t base = h.cull ? h.off_cull : h.off_rec;   /* tables end where the records begin */
    uint64_t off_cull = base, off_rec = up16(off_cull + 16ull * h.M);
    uint64_t rec_bytes = nbytes - h.off_rec, total = off_rec + rec_bytes;
    uint8_t *B = calloc(total, 1);
    if (!B) return OR_ERR_NOMEM;
    memcpy(B, blob, base);
    for (uint32_t m = 0; m < h.M; ++m)
        for (int k = 0; k < 4; ++k) wrf(B + off_cull + 16ull * m + 4 * k, entries[4ull * m + k]);
    memcpy(B + off_rec, blob + h.off_rec, rec_bytes);
    wr32(B + 60, rd32(blob + 60) | 2u);
    wr64(B + 80, off_rec);
    wr64(B + 88, total);
    wr64(B + 128, off_cull);
    *out = B;
    *out_bytes = total;
    return OR_OK;
}

/* ------------------------------------------------------------------ checksum (FORMAT.md §6) */
static uint64_t mix64(uint64_t z) {
    z ^= z >> 30; z *= 0xbf58476d1ce4e5b9ull;
    z ^= z >> 27; z *= 0x94d049bb133111ebull;
    z ^= z >> 31;
    return z;
}
uint64_t or_checksum(const uint32_t *words, uint64_t count, uint64_t k0) {
    uint64_t s = 0;
    for (uint64_t i = 0; i < count; ++i) s += mix64(((k0 + i) << 32) | words[i]);
    return s;
}

/* ================================================================== encoder ===== */

typedef struct { uint64_t key; uint32_t tri; uint8_t e; uint8_t fwd; } edge_rec;
static int edge_cmp(const void *x, const void *y) {
    const edge_rec *a = x, *b = y;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    if (a->tri != b->tri) return a->tri < b->tri ? -1 : 1;
    return (int)a->e - (int)b->e;
}

/* one output meshlet under construction: a list of strips (paths of triangles) */
typedef struct { uint32_t *tris; uint32_t *strip_start; uint32_t ntris, nstrips; } pending;

typedef struct {
    /* growing outputs */
    uint8_t **recs; uint32_t *rec_size; uint32_t nrec, caprec;
    uint32_t *rec_obj, *rec_V, *rec_Tp, *rec_R, *rec_T;
    uint32_t *src_v; uint64_t nsrc_v, capsrc_v;       /* source vertex of every output vertex slot */
    uint32_t *src_t; uint64_t nsrc_t, capsrc_t;       /* source triangle of every decoded slot, ~0 = degenerate */
    uint32_t *rec_vlist_off;                          /* per record: offset into src_v */
} enc_out;

static int grow(void **p, uint64_t *cap, uint64_t need, size_t elem) {
    if (need <= *cap) return 0;
    uint64_t nc = *cap ? *cap : 64;
    while (nc < need) nc *= 2;
    void *q = realloc(*p, nc * elem);
    if (!q) return -1;
    *p = q;
    *cap = nc;
    return 0;
}

/* Emit one output meshlet from its strips (global triangle ids), FORMAT.md §1.4.
 * Attribute codes are filled later by the quantiser; here we record the local
 * vertex order (ascending first appearance) and the topology streams. */
typedef struct {
    uint32_t V, Tp, R, T, obj;
    uint32_t N[258];
    uint8_t f[256];
    uint32_t src_tri[256];
    uint32_t vlist[256];   /* local -> source vertex */
    uint8_t idx3[768];     /* Basic: local triangle list */
} emitted;

/* Basic (codec 3): the meshlet's triangles in growth order, local vertices numbered by
 * first appearance (FORMAT.md §1.4), no strips, no restarts. */
static int emit_basic(const uint32_t *I, const uint32_t *tris, uint32_t nt, emitted *em, int32_t *vlocal) {
    uint32_t V = 0;
    for (uint32_t t = 0; t < nt; ++t) {
        for (uint32_t k = 0; k < 3; ++k) {
            uint32_t g = I[3ull * tris[t] + k];
            if (vlocal[g] < 0) { if (V >= 256) return OR_ERR_LIMITS; vlocal[g] = (int32_t)V; em->vlist[V++] = g; }
            em->idx3[3 * t + k] = (uint8_t)vlocal[g];
        }
        em->src_tri[t] = tris[t];
    }
    for (uint32_t v = 0; v < V; ++v) vlocal[em->vlist[v]] = -1;
    em->V = V;
    em->Tp = nt;
    em->R = 0;
    em->T = nt;
    return OR_OK;
}

static int emit_meshlet(const uint32_t *I, const pending *pm, const int32_t *nbr, emitted *em,
                        int32_t *vlocal /* per source vertex, -1 */) {
    uint32_t Ns = 0; /* global-vertex step sequence (before relabel) */
    uint32_t G[258];
    uint32_t nt = 0;
    uint32_t a = 0, b = 0, c = 0;
    for (uint32_t s = 0; s < pm->nstrips; ++s) {
        uint32_t beg = pm->strip_start[s], end = (s + 1 < pm->nstrips) ? pm->strip_start[s + 1] : pm->ntris;
        uint32_t t0 = pm->tris[beg];
        const uint32_t *v0 = I + 3ull * t0;
        /* rotate the strip's first triangle so its vertex NOT shared with the successor
         * comes first: then the successor lies across (b,c) or (c,a) */
        uint32_t rot = 0;
        if (end - beg > 1) {
            uint32_t t1 = pm->tris[beg + 1];
            const uint32_t *v1 = I + 3ull * t1;
            for (uint32_t k = 0; k < 3; ++k)
                if (v0[k] != v1[0] && v0[k] != v1[1] && v0[k] != v1[2]) rot = k;
        }
        uint32_t p = v0[rot], q = v0[(rot + 1) % 3], r = v0[(rot + 2) % 3];
        if (s == 0) {
            G[0] = p; G[1] = q; G[2] = r; Ns = 3;
            em->f[0] = 0; em->src_tri[0] = t0; nt = 1;
        } else {
            /* restart: four degenerate triangles [R:c, L:q, L:q, R:p] then R:r */
            uint32_t ws[5] = {c, q, q, p, r};
            uint8_t fs[5] = {1, 0, 0, 1, 1};
            for (int k = 0; k < 5; ++k) {
                if (nt >= 256) return OR_ERR_LIMITS;
                G[Ns++] = ws[k];
                em->f[nt] = fs[k];
                em->src_tri[nt] = (k == 4) ? t0 : 0xFFFFFFFFu;
                ++nt;
            }
        }
        a = p; b = q; c = r;
        for (uint32_t i = beg + 1; i < end; ++i) {
            uint32_t ti = pm->tris[i];
            const uint32_t *vi = I + 3ull * ti;
            int hasA = 0, hasB = 0, hasC = 0;
            uint32_t w = 0xFFFFFFFFu;
            for (int k = 0; k < 3; ++k) {
                if (vi[k] == a) hasA = 1;
                else if (vi[k] == b) hasB = 1;
                else if (vi[k] == c) hasC = 1;
                else w = vi[k];
            }
            if (!hasC || w == 0xFFFFFFFFu || (hasA && hasB)) return OR_ERR_INPUT;
            uint32_t fl = hasB ? 1u : 0u;        /* shares (b,c): R ; shares (c,a): L */
            uint32_t na = fl ? c : a, nb = fl ? b : c;
            /* winding check: (na,nb,w) must be a rotation of the source triangle */
            int ok = 0;
            for (int k = 0; k < 3; ++k)
                if (vi[k] == na && vi[(k + 1) % 3] == nb && vi[(k + 2) % 3] == w) ok = 1;
            if (!ok) return OR_ERR_INPUT;
            if (nt >= 256) return OR_ERR_LIMITS;
            G[Ns++] = w;
            em->f[nt] = (uint8_t)fl;
            em->src_tri[nt] = ti;
            ++nt;
            a = na; b = nb; c = w;
        }
    }
    (void)nbr;
    /* ascending relabel by first appearance in the step sequence */
    uint32_t V = 0;
    for (uint32_t k = 0; k < Ns; ++k) {
        if (vlocal[G[k]] < 0) { vlocal[G[k]] = (int32_t)V; em->vlist[V++] = G[k]; if (V > 256) return OR_ERR_LIMITS; }
        em->N[k] = (uint32_t)vlocal[G[k]];
    }
    for (uint32_t v = 0; v < V; ++v) vlocal[em->vlist[v]] = -1;
    em->V = V;
    em->Tp = nt;
    em->R = pm->nstrips - 1;
    em->T = nt - 4 * em->R;
    return OR_OK;
}

/* Encoder entry point.
 *   indices[3T], attr[V*n] (vertex-major), bits[n], sem[n], obj_of_tri[T] or NULL.
 * Outputs (malloc'd, free with or_free): blob, src_vertex[total_v], src_tri[total_tp].
 * stats[8] = {M, total_V, total_Tp, total_T, restarts, meshlets_before_split, O, 0}. */
int or_encode(const uint32_t *indices, uint32_t T, const float *attr, uint32_t Vsrc, uint32_t n,
              const uint8_t *bits, const uint8_t *sem, const uint32_t *obj_of_tri, uint32_t vmax,
              uint32_t tmax, uint32_t codec, uint32_t vw, uint8_t **blob_out, uint64_t *blob_bytes,
              uint32_t **src_vertex_out, uint32_t **src_tri_out, uint32_t *stats) {
    if (!indices && T) return OR_ERR_ARG;
    if (n < 1 || n > 16 || vmax < 3 || vmax > 256 || tmax < 1 || tmax > 256) return OR_ERR_LIMITS;
    if (codec != CODEC_GTS && codec != CODEC_REUSE && codec != CODEC_BASIC) return OR_ERR_ARG;
    uint32_t S = 0;
    for (uint32_t c = 0; c < n; ++c) {
        if (bits[c] < 1 || bits[c] > 24) return OR_ERR_LIMITS;
        S += bits[c];
    }
    for (uint32_t c = 0; c < n; ++c)
        if (sem[c] == SEM_OCT) { if (c + 1 >= n || sem[c + 1] != SEM_OCT) return OR_ERR_ARG; ++c; }
    for (uint64_t t = 0; t < T; ++t) {
        const uint32_t *v = indices + 3 * t;
        if (v[0] >= Vsrc || v[1] >= Vsrc || v[2] >= Vsrc) return OR_ERR_INPUT;
        if (v[0] == v[1] || v[1] == v[2] || v[0] == v[2]) return OR_ERR_INPUT;
    }
    uint32_t O = 1;
    if (obj_of_tri)
        for (uint64_t t = 0; t < T; ++t) if (obj_of_tri[t] + 1 > O) O = obj_of_tri[t] + 1;
    if (O > 65536) return OR_ERR_LIMITS;

    int rc = OR_ERR_NOMEM;
    /* ---- dual graph: neighbour across edge e = (v[e], v[e+1]) if the undirected edge has
     * exactly two incident triangles, with opposite orientation, of the same object, whose
     * third vertices differ (non-manifold edges sever adjacency) */
    int32_t *nbr = malloc(sizeof(int32_t) * 3ull * (T ? T : 1));
    edge_rec *E = malloc(sizeof(edge_rec) * 3ull * (T ? T : 1));
    if (!nbr || !E) { free(nbr); free(E); return OR_ERR_NOMEM; }
    for (uint64_t t = 0; t < T; ++t)
        for (int e = 0; e < 3; ++e) {
            uint32_t u = indices[3 * t + e], w = indices[3 * t + (e + 1) % 3];
            uint32_t lo = u < w ? u : w, hi = u < w ? w : u;
            E[3 * t + e].key = ((uint64_t)lo << 32) | hi;
            E[3 * t + e].tri = (uint32_t)t;
            E[3 * t + e].e = (uint8_t)e;
            E[3 * t + e].fwd = u < w;
            nbr[3 * t + e] = -1;
        }
    qsort(E, 3ull * T, sizeof(edge_rec), edge_cmp);
    for (uint64_t i = 0; i < 3ull * T;) {
        uint64_t j = i;
        while (j < 3ull * T && E[j].key == E[i].key) ++j;
        if (j - i == 2 && E[i].fwd != E[i + 1].fwd) {
            uint32_t t0 = E[i].tri, t1 = E[i + 1].tri;
            uint32_t o0 = obj_of_tri ? obj_of_tri[t0] : 0, o1 = obj_of_tri ? obj_of_tri[t1] : 0;
            uint32_t x0 = indices[3ull * t0 + (E[i].e + 2) % 3], x1 = indices[3ull * t1 + (E[i + 1].e + 2) % 3];
            if (o0 == o1 && x0 != x1 && t0 != t1) {
                nbr[3ull * t0 + E[i].e] = (int32_t)t1;
                nbr[3ull * t1 + E[i + 1].e] = (int32_t)t0;
            }
        }
        i = j;
    }
    free(E);

    /* ---- per-record storage */
    uint64_t cap_em = 0, nem = 0;
    emitted *ems = NULL;
    uint32_t *assigned = calloc(T ? T : 1, sizeof(uint32_t));      /* meshlet id + 1 */
    int32_t *vstamp = malloc(sizeof(int32_t) * (Vsrc ? Vsrc : 1));
    int32_t *vlocal = malloc(sizeof(int32_t) * (Vsrc ? Vsrc : 1));
    uint32_t *mtris = malloc(sizeof(uint32_t) * 256);
    uint32_t *queue = malloc(sizeof(uint32_t) * (3ull * (T ? T : 1) + 1));
    uint8_t *visited = calloc(T ? T : 1, 1);
    uint32_t *ptris = malloc(sizeof(uint32_t) * 512), *pstart = malloc(sizeof(uint32_t) * 512);
    uint32_t meshlets_built = 0;
    if (!assigned || !vstamp || !vlocal || !mtris || !queue || !visited || !ptris || !pstart) goto fail;
    for (uint32_t v = 0; v < Vsrc; ++v) { vstamp[v] = -1; vlocal[v] = -1; }

    for (uint32_t obj = 0; obj < O; ++obj) {
        uint64_t seed = 0;
        for (;;) {
            /* seed: lowest-index unassigned triangle of this object (S:285 tie-break) */
            while (seed < T && (assigned[seed] || (obj_of_tri ? obj_of_tri[seed] : 0) != obj)) ++seed;
            if (seed >= T) break;
            /* BFS growth over the dual graph under V <= vmax, T <= tmax */
            int32_t stamp = (int32_t)meshlets_built;
            uint32_t mt = 0, mv = 0;
            uint64_t qh = 0, qt = 0;
            queue[qt++] = (uint32_t)seed;
            while (qh < qt && mt < tmax) {
                uint32_t t = queue[qh++];
                if (assigned[t]) continue;
                uint32_t add = 0;
                for (int k = 0; k < 3; ++k) if (vstamp[indices[3ull * t + k]] != stamp) ++add;
                if (mv + add > vmax) continue;
                assigned[t] = meshlets_built + 1;
                mtris[mt++] = t;
                for (int k = 0; k < 3; ++k) {
                    uint32_t v = indices[3ull * t + k];
                    if (vstamp[v] != stamp) { vstamp[v] = stamp; ++mv; }
                }
                for (int e = 0; e < 3; ++e) {
                    int32_t u = nbr[3ull * t + e];
                    if (u >= 0 && !assigned[u] && qt < 3ull * T + 1) queue[qt++] = (uint32_t)u;
                }
            }
            ++meshlets_built;
            if (codec == CODEC_BASIC) {
                if (grow((void **)&ems, &cap_em, nem + 1, sizeof(emitted))) goto fail;
                memset(&ems[nem], 0, sizeof(emitted));
                rc = emit_basic(indices, mtris, mt, &ems[nem], vlocal);
                if (rc) goto fail;
                ems[nem].obj = obj;
                ++nem;
                rc = OR_ERR_NOMEM;
                continue;
            }

            /* ---- stripify: repeatedly start at the lowest-position unvisited triangle and
             * walk to the lowest-position unvisited neighbour (a valid path cover) */
            uint32_t np = 0, ns = 0;
            for (uint32_t i = 0; i < mt; ++i) {
                if (visited[mtris[i]]) continue;
                uint32_t cur = mtris[i];
                pstart[ns++] = np;
                for (;;) {
                    visited[cur] = 1;
                    ptris[np++] = cur;
                    int32_t best = -1;
                    uint32_t bestpos = 0xFFFFFFFFu;
                    for (int e = 0; e < 3; ++e) {
                        int32_t u = nbr[3ull * cur + e];
                        if (u < 0 || visited[u] || assigned[u] != assigned[cur]) continue;
                        uint32_t pos = 0;
                        while (mtris[pos] != (uint32_t)u) ++pos;
                        if (pos < bestpos) { bestpos = pos; best = u; }
                    }
                    if (best < 0) break;
                    cur = (uint32_t)best;
                }
            }

            /* ---- pack strips into output meshlets, T' = T + 4R <= tmax; a strip that does
             * not fit is cut and continues in an additional meshlet */
            pending pm;
            uint32_t ctris[512], cstart[512];
            pm.tris = ctris; pm.strip_start = cstart; pm.ntris = 0; pm.nstrips = 0;
            uint32_t cur_tp = 0;
            for (uint32_t s = 0; s < ns; ++s) {
                uint32_t beg = pstart[s], end = (s + 1 < ns) ? pstart[s + 1] : np;
                while (beg < end) {
                    uint32_t cost0 = pm.nstrips ? 4u : 0u;
                    if (pm.nstrips && cur_tp + cost0 + 1 > tmax) {
                        /* flush */
                        if (grow((void **)&ems, &cap_em, nem + 1, sizeof(emitted))) goto fail;
                        memset(&ems[nem], 0, sizeof(emitted));
                        rc = emit_meshlet(indices, &pm, nbr, &ems[nem], vlocal);
                        if (rc) goto fail;
                        ems[nem].obj = obj;
                        ++nem;
                        pm.ntris = 0; pm.nstrips = 0; cur_tp = 0;
                        continue;
                    }
                    uint32_t room = tmax - cur_tp - cost0;
                    uint32_t take = end - beg < room ? end - beg : room;
                    pm.strip_start[pm.nstrips++] = pm.ntris;
                    for (uint32_t k = 0; k < take; ++k) pm.tris[pm.ntris++] = ptris[beg + k];
                    cur_tp += cost0 + take;
                    beg += take;
                }
            }
            if (pm.nstrips) {
                if (grow((void **)&ems, &cap_em, nem + 1, sizeof(emitted))) goto fail;
                memset(&ems[nem], 0, sizeof(emitted));
                rc = emit_meshlet(indices, &pm, nbr, &ems[nem], vlocal);
                if (rc) goto fail;
                ems[nem].obj = obj;
                ++nem;
            }
            rc = OR_ERR_NOMEM;
        }
    }

    /* ---- quantiser (SURVEY A10 reading): per object and channel,
     * g = min over the object's used vertices, w = largest meshlet extent,
     * Δ = w/(2^b-1) rounded UP to fp32, Q = floor((A-g)/Δ + 1/2) in double,
     * L = min Q over the meshlet, code = Q - L (< 2^b, guard enlarges Δ). */
    float *delta = malloc(sizeof(float) * (uint64_t)O * n);
    float *origin = malloc(sizeof(float) * (uint64_t)O * n);
    uint32_t *L = malloc(sizeof(uint32_t) * (nem ? nem : 1) * n);
    if (!delta || !origin || !L) { free(delta); free(origin); free(L); goto fail; }
    for (uint32_t obj = 0; obj < O; ++obj)
        for (uint32_t ch = 0; ch < n; ++ch) {
            double gmin = INFINITY, wmax = 0.0;
            for (uint64_t m = 0; m < nem; ++m) {
                if (ems[m].obj != obj) continue;
                double lo = INFINITY, hi = -INFINITY;
                for (uint32_t v = 0; v < ems[m].V; ++v) {
                    double x = attr[(uint64_t)ems[m].vlist[v] * n + ch];
                    if (x < lo) lo = x;
                    if (x > hi) hi = x;
                }
                if (lo < gmin) gmin = lo;
                if (hi - lo > wmax) wmax = hi - lo;
            }
            if (gmin == INFINITY) gmin = 0.0;
            float g = (float)gmin;          /* exact: gmin is one of the float inputs */
            float d;
            uint32_t maxcode = (1u << bits[ch]) - 1u;
            if (wmax == 0.0) d = 1.0f;      /* constant channel: all codes 0 */
            else {
                double dd = wmax / (double)maxcode;
                d = (float)dd;
                if ((double)d < dd) d = nextafterf(d, INFINITY);
            }
            for (;;) {                       /* guard: every code must fit b bits */
                int fits = 1;
                for (uint64_t m = 0; m < nem && fits; ++m) {
                    if (ems[m].obj != obj) continue;
                    double qlo = INFINITY, qhi = -INFINITY;
                    for (uint32_t v = 0; v < ems[m].V; ++v) {
                        double Q = floor(((double)attr[(uint64_t)ems[m].vlist[v] * n + ch] - (double)g) / (double)d + 0.5);
                        if (Q < qlo) qlo = Q;
                        if (Q > qhi) qhi = Q;
                    }
                    if (qhi - qlo > (double)maxcode) fits = 0;
                    if (qhi > 4294967295.0) { rc = OR_ERR_RANGE; free(delta); free(origin); free(L); goto fail; }
                }
                if (fits) break;
                d = nextafterf(d, INFINITY);
            }
            delta[(uint64_t)obj * n + ch] = d;
            origin[(uint64_t)obj * n + ch] = g;
        }

    /* ---- per-meshlet L_c (lowest grid value) and, with VW, the code width
     * w_c = bit length of the largest code Q - L_c (FORMAT.md §1.4, extension f1) */
    uint8_t *wid = malloc((nem ? nem : 1) * n);
    if (!wid) { free(delta); free(origin); free(L); goto fail; }
    for (uint64_t m = 0; m < nem; ++m) {
        const emitted *em = &ems[m];
        const float *dl = delta + (uint64_t)em->obj * n, *og = origin + (uint64_t)em->obj * n;
        for (uint32_t ch = 0; ch < n; ++ch) {
            double qlo = INFINITY, qhi = -INFINITY;
            for (uint32_t v = 0; v < em->V; ++v) {
                double Q = floor(((double)attr[(uint64_t)em->vlist[v] * n + ch] - (double)og[ch]) / (double)dl[ch] + 0.5);
                if (Q < qlo) qlo = Q;
                if (Q > qhi) qhi = Q;
            }
            L[m * n + ch] = (uint32_t)qlo;
            uint32_t maxcode = (uint32_t)(qhi - qlo), w = 0;
            while (w < 32 && (maxcode >> w) != 0) ++w;     /* bit length */
            wid[m * n + ch] = vw ? (uint8_t)w : bits[ch];
        }
    }

    /* ---- serialise (FORMAT.md §1) */
    uint32_t W_hdr = (uint32_t)up16(16u + 4u * n + (vw ? n : 0u));
    uint64_t rec_total = 0, maxrec = 0;
    uint64_t *rsz = malloc(sizeof(uint64_t) * (nem ? nem : 1));
    if (!rsz) { free(wid); free(delta); free(origin); free(L); goto fail; }
    uint64_t tot_v = 0, tot_tp = 0, tot_t = 0, tot_r = 0;
    for (uint64_t m = 0; m < nem; ++m) {
        uint32_t Sm = 0;
        for (uint32_t ch = 0; ch < n; ++ch) Sm += wid[m * n + ch];
        uint32_t W = codec == CODEC_BASIC ? 0 : (ems[m].Tp + 31) / 32;
        uint32_t nb = codec == CODEC_GTS ? ems[m].Tp - 1
                      : codec == CODEC_BASIC ? 3 * ems[m].Tp : (ems[m].Tp - 1) - (ems[m].V - 3);
        uint64_t s = W_hdr + 4ull * W * (codec == CODEC_REUSE ? 2 : 1) + ((nb + 3ull) & ~3ull) +
                     4ull * (((uint64_t)ems[m].V * Sm + 31) / 32);
        rsz[m] = up16(s);
        rec_total += rsz[m];
        if (rsz[m] > maxrec) maxrec = rsz[m];
        tot_v += ems[m].V; tot_tp += ems[m].Tp; tot_t += ems[m].T; tot_r += ems[m].R;
    }
    if (tot_v > 0xFFFFFFFFull || 3 * tot_tp > 0xFFFFFFFFull || rec_total / 16 > 0xFFFFFFFFull) {
        rc = OR_ERR_RANGE; free(wid); free(rsz); free(delta); free(origin); free(L); goto fail;
    }
    uint64_t off_dir = 160, off_obj = up16(off_dir + 4ull * (nem + 1)), off_rec = up16(off_obj + 8ull * n * O);
    uint64_t total = off_rec + rec_total;
    uint8_t *B = calloc(total, 1);
    uint32_t *srcv = malloc(sizeof(uint32_t) * (tot_v ? tot_v : 1));
    uint32_t *srct = malloc(sizeof(uint32_t) * (tot_tp ? tot_tp : 1));
    if (!B || !srcv || !srct) { free(B); free(srcv); free(srct); free(wid); free(rsz); free(delta); free(origin); free(L); goto fail; }
    memcpy(B, "MCZ1", 4);
    wr32(B + 4, 1); wr32(B + 8, codec); wr32(B + 12, n); wr32(B + 16, (uint32_t)nem); wr32(B + 20, O);
    wr32(B + 24, vmax); wr32(B + 28, tmax); wr32(B + 32, (uint32_t)tot_v); wr32(B + 36, (uint32_t)tot_tp);
    wr32(B + 40, (uint32_t)tot_t); wr32(B + 44, 0); wr32(B + 48, 0); wr32(B + 52, 0);
    wr32(B + 56, (uint32_t)maxrec);
    wr32(B + 60, vw ? 1u : 0u);
    wr64(B + 64, off_dir); wr64(B + 72, off_obj); wr64(B + 80, off_rec); wr64(B + 88, total);
    for (uint32_t c = 0; c < n; ++c) { B[96 + c] = bits[c]; B[112 + c] = sem[c]; }
    for (uint32_t o = 0; o < O; ++o)
        for (uint32_t c = 0; c < n; ++c) {
            wrf(B + off_obj + 8ull * n * o + 4 * c, delta[(uint64_t)o * n + c]);
            wrf(B + off_obj + 8ull * n * o + 4ull * (n + c), origin[(uint64_t)o * n + c]);
        }
    uint64_t pos = 0, vb = 0, tb = 0;
    for (uint64_t m = 0; m < nem; ++m) {
        const emitted *em = &ems[m];
        wr32(B + off_dir + 4 * m, (uint32_t)(pos / 16));
        uint8_t *r = B + off_rec + pos;
        wr32(r, (uint32_t)vb); wr32(r + 4, (uint32_t)tb);
        r[8] = (uint8_t)(em->V - 1); r[9] = (uint8_t)(em->Tp - 1);
        wr16(r + 10, (uint16_t)em->obj); wr16(r + 12, (uint16_t)em->R); wr16(r + 14, 0);
        uint32_t W = codec == CODEC_BASIC ? 0 : (em->Tp + 31) / 32;
        uint8_t *lr = r + W_hdr, *inc = lr + 4 * W, *by = inc + (codec == CODEC_REUSE ? 4 * W : 0);
        uint32_t nb = 0, newmax = 2;
        if (codec == CODEC_BASIC)
            for (nb = 0; nb < 3 * em->Tp; ++nb) by[nb] = em->idx3[nb];
        for (uint32_t t = 1; t < em->Tp && codec != CODEC_BASIC; ++t) {
            uint32_t w = em->N[t + 2];
            if (em->f[t]) wr32(lr + 4 * (t / 32), rd32(lr + 4 * (t / 32)) | (1u << (t % 32)));
            if (codec == CODEC_GTS) by[nb++] = (uint8_t)w;
            else if (w == newmax + 1) { newmax = w; wr32(inc + 4 * (t / 32), rd32(inc + 4 * (t / 32)) | (1u << (t % 32))); }
            else by[nb++] = (uint8_t)w;
        }
        uint8_t *at = by + ((nb + 3u) & ~3u);
        const float *dl = delta + (uint64_t)em->obj * n, *og = origin + (uint64_t)em->obj * n;
        uint32_t Sm = 0;
        for (uint32_t ch = 0; ch < n; ++ch) {
            wr32(r + 16 + 4 * ch, L[m * n + ch]);
            if (vw) r[16 + 4 * n + ch] = wid[m * n + ch];
            Sm += wid[m * n + ch];
        }
        for (uint32_t v = 0; v < em->V; ++v) {
            uint64_t p = (uint64_t)v * Sm;
            for (uint32_t ch = 0; ch < n; ++ch) {
                double Q = floor(((double)attr[(uint64_t)em->vlist[v] * n + ch] - (double)og[ch]) / (double)dl[ch] + 0.5);
                uint32_t code = (uint32_t)Q - L[m * n + ch];
                for (unsigned k = 0; k < wid[m * n + ch]; ++k, ++p)
                    if ((code >> k) & 1u) wr32(at + 4 * (p / 32), rd32(at + 4 * (p / 32)) | (1u << (p % 32)));
            }
            srcv[vb + v] = em->vlist[v];
        }
        for (uint32_t t = 0; t < em->Tp; ++t) srct[tb + t] = em->src_tri[t];
        pos += rsz[m];
        vb += em->V;
        tb += em->Tp;
    }
    wr32(B + off_dir + 4 * nem, (uint32_t)(pos / 16));
    if (stats) {
        stats[0] = (uint32_t)nem; stats[1] = (uint32_t)tot_v; stats[2] = (uint32_t)tot_tp;
        stats[3] = (uint32_t)tot_t; stats[4] = (uint32_t)tot_r; stats[5] = meshlets_built;
        stats[6] = O; stats[7] = 0;
    }
    *blob_out = B;
    *blob_bytes = total;
    if (src_vertex_out) *src_vertex_out = srcv; else free(srcv);
    if (src_tri_out) *src_tri_out = srct; else free(srct);
    free(wid); free(rsz); free(delta); free(origin); free(L);
    rc = OR_OK;
fail:
    free(nbr); free(ems); free(assigned); free(vstamp); free(vlocal); free(mtris); free(queue);
    free(visited); free(ptris); free(pstart);
    return rc;
}

void or_free(void *p) { free(p); }

/* ------------------------------------------------------------------ raw packer
 * Serialise caller-given streams into a FORMAT.md blob WITHOUT validating them
 * (exhaustive and malformed test inputs).  Per meshlet m: V[m], Tp[m], R[m], obj[m],
 * nbytes[m] (count of BYTES entries actually written), L[m*n..], and concatenated
 * per-triangle arrays lr[ΣTp], inc[ΣTp] (0/1 per triangle, index 0 ignored),
 * bytes[Σnbytes], codes[ΣV * n].  Record sizes follow FORMAT.md §1.4 from the
 * header counts except that BYTES has nbytes[m] entries (a mismatch yields a
 * RECORD error on decode, by design). */
int or_pack(uint32_t codec, uint32_t n, const uint8_t *bits, const uint8_t *sem, uint32_t O,
            const float *delta, const float *origin, uint32_t vmax, uint32_t tmax, uint32_t M,
            const uint32_t *V, const uint32_t *Tp, const uint32_t *R, const uint32_t *obj,
            const uint32_t *nbytes, const uint32_t *L, const uint8_t *lr, const uint8_t *inc,
            const uint8_t *bytes, const uint32_t *codes, uint8_t **blob_out, uint64_t *blob_bytes) {
    if (n < 1 || n > 16 || O < 1) return OR_ERR_ARG;
    uint32_t S = 0;
    for (uint32_t c = 0; c < n; ++c) S += bits[c];
    uint32_t W_hdr = (uint32_t)up16(16u + 4u * n);
    uint64_t rec_total = 0, maxrec = 0, tv = 0, ttp = 0, tt = 0;
    for (uint32_t m = 0; m < M; ++m) {
        uint32_t W = codec == CODEC_BASIC ? 0 : (Tp[m] + 31) / 32;
        uint64_t s = up16(W_hdr + 4ull * W * (codec == CODEC_REUSE ? 2 : 1) + ((nbytes[m] + 3ull) & ~3ull) +
                          4ull * (((uint64_t)V[m] * S + 31) / 32));
        rec_total += s;
        if (s > maxrec) maxrec = s;
        tv += V[m]; ttp += Tp[m]; tt += Tp[m] - 4ull * R[m];
    }
    uint64_t off_dir = 160, off_obj = up16(off_dir + 4ull * (M + 1)), off_rec = up16(off_obj + 8ull * n * O);
    uint64_t total = off_rec + rec_total;
    uint8_t *B = calloc(total, 1);
    if (!B) return OR_ERR_NOMEM;
    memcpy(B, "MCZ1", 4);
    wr32(B + 4, 1); wr32(B + 8, codec); wr32(B + 12, n); wr32(B + 16, M); wr32(B + 20, O);
    wr32(B + 24, vmax); wr32(B + 28, tmax); wr32(B + 32, (uint32_t)tv); wr32(B + 36, (uint32_t)ttp);
    wr32(B + 40, (uint32_t)tt); wr32(B + 56, (uint32_t)maxrec);
    wr64(B + 64, off_dir); wr64(B + 72, off_obj); wr64(B + 80, off_rec); wr64(B + 88, total);
    for (uint32_t c = 0; c < n; ++c) { B[96 + c] = bits[c]; B[112 + c] = sem[c]; }
    for (uint32_t o = 0; o < O; ++o)
        for (uint32_t c = 0; c < n; ++c) {
            wrf(B + off_obj + 8ull * n * o + 4 * c, delta[(uint64_t)o * n + c]);
            wrf(B + off_obj + 8ull * n * o + 4ull * (n + c), origin[(uint64_t)o * n + c]);
        }
    uint64_t pos = 0, vb = 0, tb = 0, fo = 0, bo = 0, co = 0;
    for (uint32_t m = 0; m < M; ++m) {
        wr32(B + off_dir + 4ull * m, (uint32_t)(pos / 16));
        uint8_t *r = B + off_rec + pos;
        wr32(r, (uint32_t)vb); wr32(r + 4, (uint32_t)tb);
        r[8] = (uint8_t)(V[m] - 1); r[9] = (uint8_t)(Tp[m] - 1);
        wr16(r + 10, (uint16_t)obj[m]); wr16(r + 12, (uint16_t)R[m]);
        for (uint32_t c = 0; c < n; ++c) wr32(r + 16 + 4 * c, L[(uint64_t)m * n + c]);
        uint32_t W = codec == CODEC_BASIC ? 0 : (Tp[m] + 31) / 32;
        uint8_t *plr = r + W_hdr, *pinc = plr + 4 * W, *pby = pinc + (codec == CODEC_REUSE ? 4 * W : 0);
        for (uint32_t t = 1; t < Tp[m] && codec != CODEC_BASIC; ++t) {
            if (lr[fo + t]) wr32(plr + 4 * (t / 32), rd32(plr + 4 * (t / 32)) | (1u << (t % 32)));
            if (codec == CODEC_REUSE && inc[fo + t])
                wr32(pinc + 4 * (t / 32), rd32(pinc + 4 * (t / 32)) | (1u << (t % 32)));
        }
        for (uint32_t k = 0; k < nbytes[m]; ++k) pby[k] = bytes[bo + k];
        uint8_t *at = pby + ((nbytes[m] + 3u) & ~3u);
        uint64_t p = 0;
        for (uint32_t v = 0; v < V[m]; ++v)
            for (uint32_t c = 0; c < n; ++c) {
                uint32_t code = codes[co++];
                for (unsigned k = 0; k < bits[c]; ++k, ++p)
                    if ((code >> k) & 1u) wr32(at + 4 * (p / 32), rd32(at + 4 * (p / 32)) | (1u << (p % 32)));
            }
        pos += up16(W_hdr + 4ull * W * (codec == CODEC_REUSE ? 2 : 1) + ((nbytes[m] + 3ull) & ~3ull) +
                    4ull * (((uint64_t)V[m] * S + 31) / 32));
        vb += V[m]; tb += Tp[m]; fo += Tp[m]; bo += nbytes[m];
    }
    wr32(B + off_dir + 4ull * M, (uint32_t)(pos / 16));
    *blob_out = B;
    *blob_bytes = total;
    return OR_OK;
}
