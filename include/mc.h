/*
 * mc.h — C ABI of the B200 meshlet-compression library (libmc.so).
 *
 * The hot path of arXiv 2404.06359 "Towards Practical Meshlet Compression":
 * per-meshlet decompression of generalized-triangle-strip topology
 * (PAPER §4.2–4.3) and crack-free fixed-point attributes
 * (PAPER §4.4) into plain index and vertex buffers,
 * plus the host encoder that produces the stream.  The byte format is
 * FORMAT.md (normative).  P:n cites PAPER.md line n, S:n SPEC.md line n.
 *
 * Conventions
 *  - Plain C, no C++ types or exceptions cross this boundary; no torch types.
 *  - "host" pointers are CPU memory, "device" pointers CUDA device memory.
 *    Device buffers are always caller-owned (the Python binding allocates them
 *    with torch); the decode path allocates no device memory.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Decode calls are asynchronous on `stream` and never synchronise the host.
 *    Argument errors are detected synchronously and returned as mc_status;
 *    malformed stream CONTENT is detected on the device and reported in
 *    mc_stats.error_bits (FORMAT.md §5) — the kernel never traps and never
 *    reads or writes outside the blob and the record's own output ranges.
 *  - Every function is thread-safe; mc_blob objects are immutable once built.
 *    Device state is per device: a call runs on the CURRENT CUDA device
 *    (cudaSetDevice), which must own the device buffers it is given.
 *  - Decode kernels claim records from a small device WORK buffer (claim counters):
 *    the caller's mc_decode_args.d_work, or, when that is NULL, a block of a library
 *    pool (64 blocks per device, handed out round robin by one sequence per device;
 *    then at most 64 pool-backed decode launches may be in flight at once per device).
 *    A work buffer is zero when a decode starts and zero again when it completes (the
 *    decode's last CTA resets it), so no memset is enqueued per launch.
 */
#ifndef MC_H
#define MC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MC_OK = 0,
    MC_ERR_ARG = 1,      /* NULL / inconsistent argument                                  */
    MC_ERR_LIMITS = 2,   /* Ṽ, T̃ outside [3,256]/[1,256], n outside [1,16], b outside [1,24] */
    MC_ERR_INPUT = 3,    /* bad source mesh: index >= V or a degenerate triangle    */
    MC_ERR_FORMAT = 4,   /* bad magic/version/offsets: not a FORMAT.md blob        */
    MC_ERR_RANGE = 5,    /* a grid index or an output count exceeds 32 bits                */
    MC_ERR_CUDA = 6,     /* a CUDA runtime call failed                                     */
    MC_ERR_NOMEM = 7     /* host allocation failed                                         */
} mc_status;

enum { MC_CODEC_GTS = 1, MC_CODEC_GTS_REUSE = 2,              /* P:420–422 / P:423–426 */
       MC_CODEC_BASIC = 3 /* 3 local u8 indices per triangle: the paper's Basic mesh-shading
                             control, 24 bpt (Table 2) */ };
enum { MC_SEM_GENERIC = 0, MC_SEM_POSITION = 1, MC_SEM_NORMAL = 2, MC_SEM_TEXCOORD = 3,
       MC_SEM_NORMAL_OCT = 4 /* one of two consecutive octahedral channels, FORMAT.md §4.3 */ };

/* FORMAT.md §5 device error bits (mc_stats.error_bits) */
enum { MC_DERR_RECORD = 1, MC_DERR_COUNTS = 2, MC_DERR_INDEX = 4, MC_DERR_REUSE = 8, MC_DERR_OBJECT = 16 };

/* decode flags */
enum {
    MC_DECODE_BLOB_LOCAL_INDICES = 1, /* index value = vtx_base - base_vtx + local (shard-local
                                         vertex buffer) instead of the global vtx_base + local */
    MC_DECODE_INDEX_LOCAL_U8X4 = 2    /* one u32 per triangle, local u8 indices a|b<<8|c<<16
                                         (FORMAT.md §2; the paper's 8-bit meshlet indices,
                                         P:294): d_indices then holds total_tp words, 4 B/tri
                                         instead of 12; a consumer adds the record's vtx_base */
};

/* ------------------------------------------------------------------ source mesh
 * The paper's input: an indexed triangle list and per-vertex
 * attribute vectors of n channels, with b_c bits per channel.
 * All arrays are host memory, borrowed for the duration of mc_encode. */
typedef struct {
    uint32_t num_vertices;               /* V_src                                     */
    uint32_t num_triangles;              /* T_src                                     */
    const uint32_t *indices;             /* [3*T_src], winding as authored            */
    const float *attributes;             /* [V_src*n], vertex-major                   */
    uint32_t num_channels;               /* n, 1..16                                  */
    const uint8_t *bits;                 /* [n], b_c in 1..24                         */
    const uint8_t *semantic;             /* [n], MC_SEM_*                             */
    const uint32_t *object_of_triangle;  /* [T_src] or NULL: one quantisation grid per
                                            object (a mesh of a scene); meshlets never
                                            cross objects                             */
} mc_mesh;

enum {
    MC_ENCODE_VARIABLE_WIDTHS = 1,  /* per-meshlet attribute code widths w_c = bit length of the
                                       meshlet's largest code on the unchanged global grid
                                       (FORMAT.md §1.4 VW, motivated by P:715–716) */
    MC_ENCODE_CULL_CONES = 2        /* per-meshlet normal cones (FORMAT.md §1.5 cull table) from the
                                       decoded positions, for mc_decode_culled;
                                       MC_ERR_ARG if the mesh has fewer than 3 position channels */
};

typedef struct {
    uint32_t max_vertices;   /* Ṽ (the paper uses 128)                          */
    uint32_t max_triangles;  /* T̃, bounds T' = T + 4R (the paper uses 256)       */
    uint32_t codec;          /* MC_CODEC_*                                              */
    uint32_t num_threads;    /* host worker threads, 0 = hardware concurrency           */
    uint32_t flags;          /* MC_ENCODE_*                                             */
} mc_encode_params;

typedef struct mc_blob mc_blob;   /* opaque, library-owned, immutable host object */

/* Parsed BlobHeader (FORMAT.md §1.1) plus derived sizes. */
typedef struct {
    uint32_t codec, n, n_out, S;          /* n_out = floats per output vertex, S = Σ b_c   */
    uint32_t num_meshlets, num_objects, v_max, t_max;
    uint32_t total_v, total_tp, total_t;  /* Σ V, Σ T' (decoded), Σ T (real)             */
    uint32_t base_meshlet, base_vtx, base_tri, max_record_bytes;
    uint64_t off_dir, off_obj, off_rec, total_bytes;
    uint8_t bits[16], semantic[16];   /* global grid widths b_c and semantics          */
    uint32_t flags;                   /* BlobHeader flags (bit 0 VW: per-record widths,
                                         bit 1 CULL: cull table at off_cull)            */
    uint64_t off_cull;                /* FORMAT.md §1.5, 0 without CULL                 */
} mc_layout;

/* Encode a mesh (P:279–305 meshlets; P:312–467 strips; P:486–492 quantisation).
 * Meshlets are built under V <= Ṽ and T' <= T̃ (split when restarts overflow,
 * P:453), stripified, re-labelled so new vertices appear in ascending order
 * (P:456), and quantised on per-object global grids.  *out is owned by the
 * caller until mc_blob_free.  Errors: MC_ERR_ARG, MC_ERR_LIMITS, MC_ERR_INPUT,
 * MC_ERR_RANGE, MC_ERR_NOMEM. */
mc_status mc_encode(const mc_mesh *mesh, const mc_encode_params *params, mc_blob **out);

/* Instanced scene (BASELINE cfg4): for each instance i, copy every meshlet of
 * protos[proto_of_instance[i]] with translated position-channel origins
 * (offset[3*i..]).  Each instance's records are distinct bytes in the output.
 * Output vertices/triangles are numbered instance after instance. */
mc_status mc_blob_instance(const mc_blob *const *protos, uint32_t num_protos,
                           const uint32_t *proto_of_instance, const float *offset,
                           uint32_t num_instances, mc_blob **out);

/* Shard of the same instanced scene: only instances [first_instance,
 * first_instance+instance_count) of the num_instances-long list, with the global
 * base_meshlet/base_vtx/base_tri (and record vtx_base/tri_base) the full scene gives
 * them, so per-shard checksums add up to the whole scene's (FORMAT.md §6).
 * Object ids are local to the shard. */
mc_status mc_blob_instance_range(const mc_blob *const *protos, uint32_t num_protos,
                                 const uint32_t *proto_of_instance, const float *offset,
                                 uint32_t num_instances, uint32_t first_instance,
                                 uint32_t instance_count, mc_blob **out);

/* Wrap a copy of external FORMAT.md bytes (e.g. another encoder's output). */
mc_status mc_blob_from_bytes(const void *bytes, size_t n, mc_blob **out);

/* Borrow the serialised bytes (valid until mc_blob_free). */
mc_status mc_blob_bytes(const mc_blob *blob, const void **bytes, size_t *n);

/* For encoder-made blobs: the source vertex of every output vertex slot [total_v]
 * and the source triangle of every decoded triangle slot [total_tp]
 * (UINT32_MAX = restart degenerate).  MC_ERR_ARG if the blob has no map. */
mc_status mc_blob_source_map(const mc_blob *blob, const uint32_t **src_vertex, const uint32_t **src_tri);

/* Encoder statistics: restarts, meshlets split off because T' overflowed. */
mc_status mc_blob_encode_stats(const mc_blob *blob, uint64_t *restarts, uint64_t *split_meshlets);

void mc_blob_free(mc_blob *blob);

/* Parse and validate a BlobHeader from host bytes. */
mc_status mc_parse_header(const void *bytes, size_t n, mc_layout *out);

/* Split records [0, M) into `parts` contiguous ranges with balanced algorithmic
 * bytes (record bytes read + output bytes written); first[parts], count[parts]. */
mc_status mc_blob_shard_ranges(const void *bytes, size_t n, uint32_t parts, uint32_t *first,
                               uint32_t *count);

/* Copy records [first, first+count) into a standalone blob whose base_* fields
 * carry the range's original bases (checksums stay global, FORMAT.md §6). */
mc_status mc_blob_extract(const void *bytes, size_t n, uint32_t first, uint32_t count,
                          mc_blob **out);

/* Blob summary (mc_blob_info): section sizes, counts and bit budgets. */
typedef struct {
    uint32_t codec, n, num_meshlets, num_objects;
    uint64_t total_v, total_tp, total_t;  /* Σ V, Σ T' (decoded), Σ T (real)                    */
    uint64_t restarts;                    /* Σ R over the record headers (T' = T + 4R)    */
    uint64_t header_bytes, directory_bytes, object_bytes, cull_bytes, record_bytes, total_bytes;
    uint64_t record_header_bytes;         /* Σ record headers (vtx/tri base, V, T', L_c [, w_c])  */
    uint64_t flag_bytes;                  /* Σ L/R (+ increment) flag words           */
    uint64_t index_bytes;                 /* Σ index (GTS), reuse (GTS-Reuse) or local-triangle
                                             (Basic) bytes                                        */
    uint64_t attribute_bytes;             /* Σ ceil(V·S/8): the packed attribute bits              */
    uint64_t padding_bytes;               /* the rest of the records (16-B alignment)              */
    double bits_per_triangle;             /* 8·total_bytes / Σ T                                   */
    double index_bits_per_triangle;       /* 8·(flag + index bytes) / Σ T (Table 2's index buffer) */
} mc_info;

/* The global quantisation grid of one channel of one object, measured on the
 * blob's own grid values q = L_c + code: */
typedef struct {
    float delta;        /* Δ_c, the grid spacing, as stored (fp32)                       */
    float origin;       /* g_c, the grid origin (reading R9)                                     */
    uint32_t bits;      /* b_c                                                           */
    uint32_t w_steps;   /* largest meshlet extent in grid steps: max over the object's meshlets
                           of max(code); <= 2^b - 1                            */
    uint64_t W_steps;   /* global extent in grid steps: max q - min q over the object    */
    double w;           /* w_c = w_steps · Δ_c, the largest meshlet extent               */
    double W;           /* W_c = W_steps · Δ_c, the global mesh extent                   */
    double info_bits;   /* information content log2(W_c / Δ_c) = log2(W_steps), 0 if 0  */
} mc_channel_grid;

/* Summarise a blob (host bytes): *out, and, when grids != NULL, the grid of every channel
 * of every object, object-major: grids[o*n + c] for o < num_objects, c < n (grids_len >=
 * num_objects*n entries, else MC_ERR_ARG).  One pass over the records (the attribute bits
 * are unpacked on the host).  Errors: MC_ERR_FORMAT (not a valid blob or a record whose
 * sections overrun it), MC_ERR_ARG. */
mc_status mc_blob_info(const void *bytes, size_t n, mc_info *out, mc_channel_grid *grids, uint32_t grids_len);

/* ------------------------------------------------------------------ device decode */
/* u32 words of a decode work buffer (mc_decode_args.d_work). */
#define MC_DECODE_WORK_WORDS 256

typedef struct {
    const mc_layout *layout;   /* host: mc_parse_header of the same blob                 */
    const void *d_blob;        /* device: the blob bytes (16-B aligned base)              */
    uint32_t first, count;     /* records [first, first+count) of this blob               */
    uint32_t *d_indices;       /* device, required: 3*total_tp u32, FORMAT.md §2
                                  (positions relative to base_tri of the blob); total_tp
                                  u32 with MC_DECODE_INDEX_LOCAL_U8X4                      */
    float *d_vertices;         /* device or NULL: n_out*total_v fp32, FORMAT.md §4.2;
                                  16-B aligned (MC_ERR_ARG otherwise); with n_out = 8 a
                                  32-B aligned buffer is written with one 256-bit store
                                  per vertex (faster), a 16-B aligned one with two        */
    uint32_t *d_quantized;     /* device or NULL: n*total_v u32 grid values, §4.1          */
    uint32_t flags;            /* MC_DECODE_*                                             */
    uint32_t *d_work;          /* device or NULL: MC_DECODE_WORK_WORDS u32 of claim-counter
                                  scratch, caller-owned, zero-filled once before its first
                                  use; every completed decode leaves it zero again, so
                                  decodes ordered on one stream reuse it with no memset.
                                  Two decodes in flight at the same time (different
                                  streams) must not share one.  NULL = library pool.      */
} mc_decode_args;

/* Device statistics (FORMAT.md §5, §6), accumulated atomically. */
typedef struct {
    uint64_t checksum_indices;     /* Σ mix64(k<<32 | word) over index words              */
    uint64_t checksum_vertices;    /* same over fp32 vertex words (bit patterns)          */
    uint64_t checksum_quantized;   /* same over quantised words                           */
    uint64_t triangles;            /* Σ T' decoded                                        */
    uint64_t degenerate;           /* decoded triangles with a repeated index             */
    uint64_t vertices;             /* Σ V                                                 */
    uint64_t multiword_lookbacks;  /* triangles whose L/R search crossed a word   */
    uint32_t max_lookback;         /* max over triangles of t - j(t)                      */
    uint32_t error_bits;           /* OR of FORMAT.md §5 bits                             */
    uint32_t first_bad_meshlet;    /* smallest malformed record index, UINT32_MAX if none */
    uint32_t num_bad;              /* malformed records                                   */
} mc_stats;

/* Decode records into the output buffers (the timed hot path).  One 16-lane group
 * (T~ <= 128) or one warp per meshlet, records staged into shared memory with TMA
 * bulk copies.  Errors: MC_ERR_ARG (NULL/misaligned pointers, range
 * outside the blob, unknown flag), MC_ERR_FORMAT (layout not from mc_parse_header),
 * MC_ERR_LIMITS (staging buffers do not fit shared memory), MC_ERR_CUDA. */
mc_status mc_decode_meshlets(const mc_decode_args *args, void *stream);

/* Same decode, additionally accumulating mc_stats into *d_stats (device). */
mc_status mc_decode_stats(const mc_decode_args *args, mc_stats *d_stats, void *stream);

/* Cone-culled, compacted decode (FORMAT.md §1.5, §7; the paper's amplification-shader
 * cone culling).  For the unit view direction view_dir (host,
 * float[3], from the camera into the scene; a directional / orthographic view), every
 * record whose cone test fmaf(az,dz,fmaf(ay,dy,ax*dx)) > cutoff (binary32) holds is
 * skipped; the visible records are decoded in record order into compacted outputs
 * (index/vertex positions and u32 index values relative to 0).  args must cover the
 * whole blob (first = 0, count = num_meshlets); output buffers are sized as for
 * mc_decode_meshlets (the visible part is a prefix of them).  d_counts (device,
 * uint32_t[4]) receives {visible records, Σ V, Σ T', Σ T (real)}; d_stats (device or
 * NULL) accumulates mc_stats over the visible records.  d_scratch: device, 16-B aligned,
 * >= mc_decode_culled_scratch_bytes(layout), caller-owned, zero-filled once before its
 * first use: every completed call leaves its look-back flags and tile tickets zero again
 * (two calls in flight at the same time must not share one).  Asynchronous: two kernels
 * on `stream` — a one-pass cone test + decoupled look-back scan that lists the visible
 * records with their compacted output bases, then the decode kernel over that list (a
 * build with -DMC_CULL_FUSED=1 runs the scan inside the decode kernel: one launch).
 * Errors: MC_ERR_FORMAT (blob without cull table), MC_ERR_ARG, MC_ERR_LIMITS, MC_ERR_CUDA. */
size_t mc_decode_culled_scratch_bytes(const mc_layout *layout);
mc_status mc_decode_culled(const mc_decode_args *args, const float *view_dir, void *d_scratch, size_t scratch_bytes,
                           uint32_t *d_counts, mc_stats *d_stats, void *stream);

/* Initialise a device mc_stats: zeros, first_bad_meshlet = UINT32_MAX. */
mc_status mc_stats_reset(mc_stats *d_stats, void *stream);

/* End-to-end decode from HOST buffers: H2D of the blob, decode, D2H of the
 * outputs, ordered on `stream` (host buffers must be pinned for the copies to be
 * asynchronous).  Device buffers are caller-owned scratch of the sizes
 * mc_decode_args states.
 *
 * chunks <= 1: one H2D of the whole blob, one decode, one D2H per output, all on
 * `stream`.  chunks >= 2: software pipeline over PCIe — the header, directory,
 * object and cull tables go first, then the record section in `chunks` contiguous
 * byte-balanced record ranges; chunk c's H2D (library-owned copy-in stream), decode
 * (on `stream`) and D2H (library-owned copy-out stream) are chained by events, so
 * chunk c+1 is copied in and chunk c-1 copied out while chunk c decodes (PCIe is
 * full duplex: the step costs about max(H2D, D2H) instead of their sum).  The call
 * stays asynchronous: the copy streams first wait for work already on `stream`, and
 * `stream` waits for the last copy-out before anything enqueued after the call.
 * Requires records whose output ranges follow record order (vtx_base and tri_base
 * non-decreasing, as every blob this library writes has them): each chunk copies
 * back the output span between its first record's bases and the next chunk's; the
 * call checks the chunk boundaries and otherwise falls back to chunks = 1.
 * The library streams/events are created once per device on first use. */
typedef struct {
    const mc_layout *layout;
    const void *h_blob;        /* host: total_bytes                                       */
    void *d_blob;              /* device scratch: >= total_bytes                          */
    uint32_t *h_indices;       /* host out: 3*total_tp                                     */
    float *h_vertices;         /* host out or NULL                                        */
    uint32_t *h_quantized;     /* host out or NULL                                        */
    uint32_t *d_indices;       /* device scratch                                           */
    float *d_vertices;         /* device scratch or NULL (NULL iff h_vertices NULL)       */
    uint32_t *d_quantized;     /* device scratch or NULL                                   */
    uint32_t flags;
    uint32_t chunks;           /* pipeline depth (0/1 = serial, capped at 64)              */
} mc_host_decode_args;
mc_status mc_decode_host(const mc_host_decode_args *args, void *stream);

const char *mc_status_str(mc_status s);
uint32_t mc_abi_version(void);   /* 4 (3: mc_encode_params.flags, mc_layout.flags, mc_host_decode_args.chunks;
                                    4: mc_decode_args.d_work) */

#ifdef __cplusplus
}
#endif
#endif /* MC_H */
