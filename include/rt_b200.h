/*
 * rt_b200.h -- C ABI of the B200-native stereo Whitted ray tracer (arXiv 1702.01530 hot path).
 *
 * The paper (§3, lines 54-56, Fig. 2) synthesises a stereo pair by ray tracing
 * the scene twice, once per eye camera ("parallel level 1": left/right channels;
 * "parallel level 2": the pixels of one channel on the multiprocessor cores), and
 * attributes ~40% of its time to CPU<->GPU transfer.  This library
 * exposes exactly the calls the north star names -- rt_scene_upload, rt_set_stereo_camera,
 * rt_render_stereo, rt_download -- plus the context, event, shard and peer helpers the
 * bench and the multi-GPU path need.
 *
 * Conventions (every entry point):
 *   - returns rt_status; RT_OK == 0.  No C++ exception ever crosses this boundary.
 *   - on failure the thread-local message is available from rt_last_error().
 *   - device work is ASYNCHRONOUS on the context's stream; calls return after enqueue,
 *     except rt_scene_upload, which returns once the scene's host arrays were copied
 *     (host buffers may be freed on return).
 *   - a context is bound to one device and one stream and is NOT thread-safe; use one
 *     context per (device, host thread).
 *   - "device pointer" arguments must be CUDA device allocations on the context's device
 *     (e.g. torch tensors' data_ptr()); "host pointer" arguments are ordinary host memory
 *     unless stated "pinned".
 *   - coordinates are world units; colours are linear radiance; IDs are int32.
 *
 * Global primitive ID (tie-break order, SPEC.md:183 generalised; reading 9):
 *   spheres [0, S), planes [S, S+P), triangles [S+P, S+P+T), each in upload order.
 */
#ifndef RT_B200_H
#define RT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RT_ABI_VERSION 2
#define RT_MAX_DEPTH 16          /* max_depth limit (stack sizing)                 */
#define RT_TILE 16               /* shard tile edge in pixels (16x16 tiles)        */
#define RT_NUM_COUNTERS 13       /* see rt_counter                                  */

typedef enum rt_status {
    RT_OK = 0,
    RT_ERR_INVALID_ARG = 1,      /* bad pointer/size/value (SPEC.md:76 ValidationError analogue) */
    RT_ERR_CUDA = 2,             /* a CUDA runtime call failed (message has cudaGetErrorString)  */
    RT_ERR_OOM = 3,              /* device or pinned allocation failed                           */
    RT_ERR_NO_SCENE = 4,         /* render before a successful rt_scene_upload                   */
    RT_ERR_NO_CAMERA = 5,        /* render before a successful rt_set_stereo_camera              */
    RT_ERR_SIZE = 6,             /* width*height == 0, too large, pitch too small, depth > 16    */
    RT_ERR_NOT_READY = 7,        /* rt_query: work still in flight (not an error)                */
    RT_ERR_PEER = 8              /* CUDA IPC / peer mapping failed                               */
} rt_status;

typedef struct rt_context rt_context;
typedef struct rt_event rt_event;

/* Scene primitives, HOST pointers, caller-owned, copied during rt_scene_upload.
 * Every array may be NULL when its count is 0. */
typedef struct rt_primitives {
    const float* spheres;        /* [4*n_spheres]  (cx, cy, cz, r), r > 0                        */
    const uint32_t* sphere_mat;  /* [n_spheres]    material index                               */
    uint32_t n_spheres;
    const float* planes;         /* [4*n_planes]   (nx, ny, nz, k): plane n.x = k, |n| > 0      */
    const uint32_t* plane_mat;   /* [n_planes]                                                  */
    uint32_t n_planes;
    const float* vertices;       /* [3*n_vertices] (x, y, z)                                    */
    uint32_t n_vertices;
    const uint32_t* tri_indices; /* [3*n_triangles] vertex indices, CCW seen from outside       */
    const uint32_t* tri_mat;     /* [n_triangles]                                               */
    uint32_t n_triangles;
} rt_primitives;

/* SPEC.md:40-44 Material, extended by the north star with refraction (kt, ior). */
typedef struct rt_material {
    float kd[3];                 /* diffuse colour, >= 0                      */
    float ks[3];                 /* specular colour, >= 0                     */
    float shininess;             /* Phong exponent, >= 1         */
    float kr;                    /* mirror reflectivity in [0,1]              */
    float kt;                    /* transmissivity in [0,1], kr + kt <= 1     */
    float ior;                   /* index of refraction (> 0), outside = 1    */
} rt_material;

typedef struct rt_light { float pos[3]; float intensity[3]; } rt_light;   /* SPEC.md:53 PointLight */
typedef struct rt_env { float ambient[3]; float background[3]; } rt_env;  /* SPEC.md:65 Scene      */

typedef enum rt_format { RT_FORMAT_RGBA8 = 0, RT_FORMAT_RGBA16F = 1 } rt_format;

/* A caller-owned DEVICE framebuffer: row-major, top row first.
 * RGBA8: byte = floor(255*clamp(c,0,1) + 0.5), A = 255.
 * RGBA16F: binary16 round-to-nearest-even of clamp(c,0,1), A = 1.0.
 * pitch_bytes >= width * (4 or 8).  dev_ptr NULL = do not write this eye. */
typedef struct rt_fb {
    void* dev_ptr;
    uint32_t format;             /* rt_format */
    uint64_t pitch_bytes;
} rt_fb;

/* Counter slots of rt_outputs.counters (uint64, accumulated, never reset by the library). */
typedef enum rt_counter {
    RT_CNT_PRIMARY = 0, RT_CNT_REFLECTION = 1, RT_CNT_REFRACTION = 2, RT_CNT_SHADOW = 3,
    RT_CNT_NODE_VISITS = 4,      /* BVH4 nodes visited                                */
    RT_CNT_TRI_TESTS = 5, RT_CNT_SPHERE_TESTS = 6, RT_CNT_PLANE_TESTS = 7,
    RT_CNT_SHADE_HITS = 8,       /* nearest-hit shading points                        */
    RT_CNT_LIGHT_EVALS = 9,      /* (hit, light) pairs evaluated                      */
    RT_CNT_MISSES = 10,          /* tree rays that hit nothing                        */
    RT_CNT_PIXELS = 11,
    RT_CNT_BOX_TESTS = 12        /* child-box slab tests of real (non-empty) children  */
} rt_counter;

/* rt_render_params.flags */
#define RT_RENDER_COUNT 1u       /* run the instrumented kernel variant (fills counters; slower) */
#define RT_RENDER_BRUTE_FORCE 2u /* debug: test every primitive, no BVH (same FP32 intersectors) */
#define RT_RENDER_PEER_STORE 4u  /* out_left/out_right are a PEER rank's framebuffers mapped with
                                    rt_ipc_open: the pack epilogue stores over NVLink and the
                                    kernel ends with a system-scope fence (fused render->gather) */
#define RT_RENDER_KDTREE 8u      /* NEXT-4 ablation: traverse the kd-tree of rt_kdtree_build
                                    instead of the BVH4 (same intersectors, same results) */

typedef struct rt_render_params {
    uint32_t width, height;      /* per eye; 1 <= w,h <= 16384                              */
    uint32_t max_depth;          /* bounces still allowed, 0 = local shading only  */
    uint32_t shard_rank;         /* render only this rank's tiles ...                        */
    uint32_t shard_world;        /* ... of shard_world ranks (1 = every tile), see rt_shard_* */
    uint32_t flags;              /* RT_RENDER_* */
} rt_render_params;

/* Optional outputs of rt_render_stereo_ex; every DEVICE pointer may be NULL. */
typedef struct rt_outputs {
    rt_fb left, right;           /* row-major framebuffers                                   */
    int32_t* prim_id;            /* [2*H*W] primary nearest-hit global ID, -1 = miss; eye-major */
    float* radiance;             /* [2*H*W*4] unclamped linear RGB + 0 pad; eye-major        */
    void* shard;                 /* packed tile-major shard (rt_shard_bytes) for the gather  */
    uint32_t shard_format;       /* rt_format of `shard`                                     */
    unsigned long long* counters;/* [RT_NUM_COUNTERS], accumulated when RT_RENDER_COUNT set  */
    rt_fb composed;              /* stereo composition fused into the pack epilogue (NEXT-1,  */
    uint32_t compose_mode;       /* PAPER.md:56): RGBA8 only, RT_COMPOSE_* as rt_compose; both */
                                 /* eyes of a pixel must be traced in the same launch (a whole */
                                 /* frame, or tile-pair shards; not the world-2 eye split)     */
} rt_outputs;

/* ------------------------------------------------------------------ context */
/* Bind a new context to CUDA `device` and `cuda_stream` (a cudaStream_t; NULL -> the
 * library creates and owns a non-blocking stream).  *out is library-owned. */
rt_status rt_create(int device, void* cuda_stream, rt_context** out);
/* Synchronise and free every library-owned resource of ctx (scene, BVH, events). */
rt_status rt_destroy(rt_context* ctx);
/* Block until all work enqueued by ctx (render and copy streams) has completed. */
rt_status rt_synchronize(rt_context* ctx);
/* Thread-local message of the last failed call on this thread ("" if none). */
const char* rt_last_error(void);
int rt_version(void);
/* Children per BVH node of this build (4 or 8), i.e. rt_bvh_export's node = 7*width floats. */
int rt_bvh_width(void);

/* ------------------------------------------------------------------ scene */
/* PAPER.md:64-66,82 (§4: scene of objects + light sources, copied to the GPU) and
 * SURVEY §8(a) rows a1-a2.  Validates (indices < n_vertices, finite values, r > 0, |n| > 0,
 * triangle area > 1e-12 * bbox_diag^2, 0 <= kr, kt, kr + kt <= 1,
 * shininess >= 1, ior > 0, kd, ks, intensities >= 0, material index <
 * n_mats), copies the arrays to the device as SoA records, and builds the Morton-code
 * LBVH over spheres + triangles on the device (planes stay outside the BVH).
 * Replaces any previous scene.  An empty scene (no primitives) is valid.
 * Errors: RT_ERR_INVALID_ARG (validation; message names the entity), RT_ERR_OOM, RT_ERR_CUDA. */
rt_status rt_scene_upload(rt_context* ctx, const rt_primitives* prims,
                          const rt_material* mats, uint32_t n_mats,
                          const rt_light* lights, uint32_t n_lights, const rt_env* env);

/* NEXT-3 (PAPER.md:125 ref [12] dynamic meshes): move the triangle vertices of
 * the uploaded scene (HOST array of 3*n_vertices floats, same count and connectivity as the
 * upload) and refit the device BVH bottom-up on the device (same topology and leaf order, new
 * boxes) instead of rebuilding it.  Validation as at upload (finite values, no degenerate
 * triangle).  Blocks until the refit is done (host array may be freed on return).
 * Errors: RT_ERR_NO_SCENE, RT_ERR_INVALID_ARG (count mismatch, validation), RT_ERR_CUDA. */
rt_status rt_scene_update_vertices(rt_context* ctx, const float* vertices, uint32_t n_vertices);

/* PAPER.md:33 (§2: "two projections ... from two cameras, corresponding to eyes of the
 * observer") with SPEC.md:422-430 derive_eyes: `eye` is the cyclopean midpoint, the eyes
 * sit at eye -/+ (interocular/2) * r^, r^ = normalize(f^ x up).  vfov is vertical, in
 * degrees, in (0,180).  interocular >= 0 (0 -> identical eyes).  convergence = distance of
 * the zero-parallax plane (off-axis window shift sigma = +-s/(2C)); convergence <= 0 or
 * +inf selects the parallel rig.  The basis is derived in double on the host.
 * Errors: RT_ERR_INVALID_ARG for eye == look_at, up parallel to the view direction,
 * vfov outside (0,180), negative interocular, any non-finite input (except C = inf). */
rt_status rt_set_stereo_camera(rt_context* ctx, const float eye[3], const float look_at[3],
                               const float up[3], float vfov_deg, float interocular,
                               float convergence);

/* ------------------------------------------------------------------ render */
/* PAPER.md:54-56 (§3 Fig. 2): render both channels of the stereo pair.  For every pixel of
 * each eye: primary ray -> nearest hit over spheres, planes, triangles -> Phong shading with
 * hard shadow rays per light -> reflection/refraction up to max_depth bounces -> clamp and
 * pack into out_left / out_right (caller-owned device framebuffers, which must stay alive
 * until the work completes).  Asynchronous on the context stream.
 * Errors: RT_ERR_NO_SCENE, RT_ERR_NO_CAMERA, RT_ERR_SIZE, RT_ERR_INVALID_ARG, RT_ERR_CUDA. */
rt_status rt_render_stereo(rt_context* ctx, uint32_t width, uint32_t height, uint32_t max_depth,
                           rt_fb out_left, rt_fb out_right);

/* Superset for tests, bench and sharding: optional ID / radiance / shard / counter outputs,
 * instrumented and brute-force variants, and a tile subset (rank shard_rank of
 * shard_world, "dividing the picture to N identical parts").  Pixels outside
 * the shard are not written. */
rt_status rt_render_stereo_ex(rt_context* ctx, const rt_render_params* params, const rt_outputs* out);

/* rt_render_stereo_ex enqueued on `cuda_stream` (a cudaStream_t of the context's device; NULL =
 * the context stream) instead of the context stream: frames in flight.  Renders on different
 * streams may run concurrently on the device (up to 16 in flight: each takes its own work
 * queue), so the tail of one frame -- the last, deepest pixel trees, during which most SMs
 * would idle -- overlaps the next frame's work.  The scene and camera are read at enqueue time;
 * rt_scene_upload / rt_scene_update_vertices must not run while renders are in flight.  The
 * caller orders reuse of output buffers (stream order or events).  Errors as rt_render_stereo_ex. */
rt_status rt_render_stereo_async(rt_context* ctx, const rt_render_params* params, const rt_outputs* out,
                                 void* cuda_stream);

/* ------------------------------------------------------------------ download */
/* PAPER.md:15,107 (the CPU<->GPU transfer stage).  Asynchronous device->host copy of
 * `bytes` from DEVICE `dev_src` into PINNED host `host_dst` (rt_host_alloc or
 * cudaHostRegister'ed), on the context's copy stream, ordered after all work enqueued on
 * the render stream so far; rendering of later frames overlaps it.  *done (library-owned)
 * completes when the bytes are on the host; release it with rt_wait.  done may be NULL.
 * Errors: RT_ERR_INVALID_ARG (NULL, zero size, host_dst not pinned), RT_ERR_CUDA. */
rt_status rt_download(rt_context* ctx, const void* dev_src, void* host_dst, size_t bytes,
                      rt_event** done);
/* Block until ev completes, then free it. */
/* rt_download ordered after the work enqueued so far on `after_stream` (e.g. the stream a frame
 * was rendered on with rt_render_stereo_async; NULL = the context stream). */
rt_status rt_download_after(rt_context* ctx, const void* dev_src, void* host_dst, size_t bytes, void* after_stream,
                            rt_event** done);
rt_status rt_wait(rt_event* ev);
/* RT_OK if ev has completed (ev stays valid), RT_ERR_NOT_READY otherwise. */
rt_status rt_query(rt_event* ev);
/* Page-locked host allocation / release for rt_download targets. */
rt_status rt_host_alloc(size_t bytes, void** out);
rt_status rt_host_free(void* ptr);
/* Async host->device copy on the render stream (camera-independent inputs for e2e runs);
 * host_src must be pinned. */
rt_status rt_upload(rt_context* ctx, const void* host_src, void* dev_dst, size_t bytes);

/* ------------------------------------------------------------------ sharding (host logic) */
/* Tile shard map: the image of each eye is cut into RT_TILE x RT_TILE tiles,
 * tiles_per_eye = T = ceil(W/16)*ceil(H/16).  Global tile id G in [0, 2T) interleaves the eyes:
 * eye = G mod 2, tile = G div 2 (raster order).  world == 2: rank r renders eye r, every tile
 * (the paper's level-1 eye split; environment RT_SHARD_PAIRS=1, read once per
 * process and required to match on every rank, deals tile pairs at world 2 too).  Otherwise (world == 1 included) tile t goes, in
 * both eyes, to rank t mod world, so a rank's shard-local tile lt is G = 2 (rank + (lt div 2)
 * world) + (lt mod 2): the two eyes of a tile are traced together (one warp = the same 4x4
 * pixel block in both eyes).
 * Environment RT_SHARD_BLOCK=B > 1 (read once per process, the same on every rank) deals the tile
 * pairs in B x B blocks of tiles instead (blocks in raster order, block b -> rank b mod world, tiles
 * raster order inside a block): every rank's tiles are spatially compact.
 * rt_shard_tiles writes rank's global tile ids G (ascending; block-major with RT_SHARD_BLOCK) into
 * tile_ids (may be NULL to query the count) and their number into *n_tiles.  Pure host functions,
 * no context. */
rt_status rt_shard_tiles(uint32_t width, uint32_t height, uint32_t rank, uint32_t world,
                         uint32_t* n_tiles, uint32_t* tile_ids);
/* Bytes of one rank's packed shard, padded to the largest rank (equal gather counts):
 * max_rank(n_tiles) * 256 * bytes_per_pixel(format). */
rt_status rt_shard_bytes(uint32_t width, uint32_t height, uint32_t world, uint32_t format,
                         uint64_t* bytes);
/* Scatter `world` concatenated shards (rank-major, each rt_shard_bytes long) into two
 * row-major framebuffers.  _host: HOST buffers (pure host logic);
 * rt_unpack_shards: DEVICE buffers, asynchronous on the context stream. */
rt_status rt_unpack_shards_host(const void* gathered, uint32_t width, uint32_t height, uint32_t world,
                                uint32_t format, void* left, void* right, uint64_t pitch_bytes);
rt_status rt_unpack_shards(rt_context* ctx, const void* gathered, uint32_t width, uint32_t height,
                           uint32_t world, uint32_t format, rt_fb left, rt_fb right);

/* ------------------------------------------------------------------ multi-GPU frames */
/* PAPER.md:48 (§3, Fig. 1: "dividing the picture to N identical parts", one processor each) and
 * PAPER.md:56 (§3, Fig. 2: level 1 = the left/right channels); SURVEY.md §8(b), §8(e).
 * One process per GPU of ONE node, each with its own context holding the same scene and camera.
 * After rt_dist_init, every rt_render_stereo / _ex / _async call whose params ask for the whole
 * frame (shard_world == 1) renders this rank's tiles of that frame (the rt_shard_tiles map: world
 * 2 = one eye per rank) and the library assembles the frame in RANK 0's out_left / out_right:
 *   RT_DIST_PEER (default): the other ranks map rank 0's framebuffers (CUDA IPC; NVLink P2P) and
 *     their pack epilogues store each finished pixel straight into them.  Ordering is on the
 *     device: rank 0's stream posts that the frame's framebuffers are free before its own tiles,
 *     each other rank's stream waits for that post, renders, and posts its completion into rank
 *     0's memory; rank 0's stream waits for every post, so work enqueued after the render on
 *     rank 0's stream (e.g. rt_download_after) sees the whole frame.  No gather, no unpack.
 *   RT_DIST_NCCL: every rank packs its tiles, NCCL gathers the shards on rank 0 (libnccl.so.2,
 *     loaded at run time), rank 0 unpacks them into its framebuffers.  Chosen automatically if
 *     any rank cannot map rank 0's memory; requires one GPU per rank.
 * Contract: every rank issues the same sequence of frame renders (same size, depth and format);
 * frames are matched by their position in that sequence, up to 16 in flight.  On ranks != 0 the
 * out_* framebuffers are ignored (NULL allowed) except their format under RT_DIST_NCCL; ID /
 * radiance / shard planes are rejected (render an explicit shard, shard_world > 1, which stays a
 * local render of those tiles).  Rank 0's framebuffers must stay allocated until the frame's work
 * on rank 0's stream completes.  Device-side waits are bounded (env RT_DIST_TIMEOUT_S, default
 * 60 s): a rank that never posts makes later calls fail with RT_ERR_PEER, not a hung GPU.
 * A one-rank world renders locally, except with flags RT_DIST_NCCL: then every frame runs the
 * NCCL transport's whole data path (pack, a one-rank ncclGather, unpack) -- a check of that
 * transport on one GPU, since NCCL refuses two ranks on one device. */
#define RT_DIST_ID_BYTES 128
#define RT_DIST_PEER 0u          /* fused peer-store assembly (default)                     */
#define RT_DIST_NCCL 1u          /* NCCL gather of packed shards + root unpack              */
/* A 128-byte job id for rt_dist_init, created once (by rank 0) and handed to every rank by the
 * caller (e.g. a torch.distributed broadcast).  It is an NCCL unique id when libnccl.so.2 loads
 * (the NCCL transport's communicator), otherwise random bytes; it also names the job's host
 * rendezvous (POSIX shared memory /rtb200_<hash>).  id: HOST buffer of RT_DIST_ID_BYTES. */
rt_status rt_dist_unique_id(void* id);
/* Join rank `rank` of `world` ranks (collective: blocks until every rank joined, bounded by the
 * timeout).  flags: RT_DIST_PEER or RT_DIST_NCCL (rank 0's choice wins).
 * Errors: RT_ERR_INVALID_ARG (rank/world, already joined), RT_ERR_PEER (rendezvous, NCCL),
 * RT_ERR_CUDA. */
rt_status rt_dist_init(rt_context* ctx, int rank, int world, const void* id, uint32_t flags);
/* Leave the world (collective): waits for this rank's device work, releases the peer mappings,
 * the device flags and the rendezvous.  Reports RT_ERR_PEER if a frame timed out. */
rt_status rt_dist_finalize(rt_context* ctx);
/* info[0] rank, [1] world (1 without rt_dist_init), [2] transport (RT_DIST_*; -1 none),
 * [3] frames rendered in the world. */
rt_status rt_dist_info(rt_context* ctx, int32_t info[4]);
/* Test support, no device work: runs the host half of the protocol -- the shared-memory
 * rendezvous of rt_dist_init, `frames` synthetic frame descriptors through the 16-slot ring
 * (rank 0 publishing, the others reading, flow-controlled), and the leave of rt_dist_finalize --
 * and returns a checksum of the descriptors this rank published or read (equal on every rank iff
 * every rank saw every frame in order).  Errors: RT_ERR_INVALID_ARG, RT_ERR_PEER (timeout). */
rt_status rt_dist_host_selftest(int rank, int world, const void* id, uint32_t frames, uint64_t* checksum);

/* ------------------------------------------------------------------ peer memory (fused gather) */
/* CUDA IPC: export the DEVICE allocation containing dev_ptr as a 64-byte handle plus the byte
 * offset of dev_ptr inside that allocation (allocations from caching allocators such as
 * torch's are sub-ranges of a larger cudaMalloc block; the handle always maps the block base),
 * open a peer's handle to get a device pointer to the block base that kernels of this context
 * may store to (NVLink P2P, or the same device), and close it.  Used by the fused
 * render->gather path in which each rank's pack epilogue writes its tiles straight into rank
 * 0's framebuffers (base + offset). */
rt_status rt_ipc_get_handle(const void* dev_ptr, void* handle64, uint64_t* offset);
/* rt_ipc_open of a handle this context already mapped returns the same mapping (framebuffers
 * that share one allocation share one handle); mappings are reference counted: call
 * rt_ipc_close once per rt_ipc_open.  rt_destroy closes what is left. */
rt_status rt_ipc_open(rt_context* ctx, const void* handle64, void** dev_ptr);
rt_status rt_ipc_close(rt_context* ctx, void* dev_ptr);

/* ------------------------------------------------------------------ stereo composition */
/* PAPER.md:56 (§3: GPU post-processing of the stereo pair "for example, anaglyph/Anamorphic
 * transformation").  Inputs are the two RGBA8 DEVICE framebuffers of one
 * render (width x height each); asynchronous on the context stream.
 *   RT_COMPOSE_ANAGLYPH: out is width x height RGBA8, out = (L.r, R.g, R.b, 255)
 *   RT_COMPOSE_SBS:      out is (2*floor(width/2)) x height RGBA8; left half = the left image
 *                        squeezed by column-pair means (per channel, round half up:
 *                        (a + b + 1) >> 1), right half = the right image likewise; A = 255
 * Errors: RT_ERR_INVALID_ARG (NULL, non-RGBA8 format, unknown mode, width < 2 for SBS),
 * RT_ERR_SIZE (pitch too small), RT_ERR_CUDA. */
#define RT_COMPOSE_ANAGLYPH 0u
#define RT_COMPOSE_SBS 1u
rt_status rt_compose(rt_context* ctx, rt_fb left, rt_fb right, uint32_t width, uint32_t height, uint32_t mode,
                     rt_fb out);

/* ------------------------------------------------------------------ ray queries */
/* The method's intersection step (§2 "intersection of the ray with the objects";
 * SURVEY §8(a) a4; SPEC.md:180-188 nearest hit, :292-300 BVH traversal) on caller-given rays,
 * with the same device code the renderer runs: for ray i (origin o[3i..3i+2], direction
 * d[3i..3i+2], any length != 0 -- normalised on the device as the renderer's rays are):
 *   RT_QUERY_NEAREST: out_t[i] = the smallest t > t_min (1e-4) over every primitive, ties to the
 *     smallest global ID; out_id[i] = that ID, or -1 and +inf on a miss (tmax ignored);
 *   RT_QUERY_ANY: out_id[i] = 1 if some primitive has t_min < t < tmax[i] (a shadow query), else
 *     0; out_t[i] is left unwritten.
 * | RT_QUERY_BRUTE_FORCE tests every primitive instead of traversing the BVH (the reference the
 * BVH must equal bit for bit).  o, d, tmax (ANY only), out_t (NEAREST only), out_id: DEVICE
 * arrays (float32 / int32); enqueued on `stream` (cudaStream_t, NULL = the context's stream),
 * asynchronous.  Errors: RT_ERR_INVALID_ARG (NULL arrays, unknown flags), RT_ERR_NO_SCENE,
 * RT_ERR_CUDA. */
#define RT_QUERY_NEAREST 0u
#define RT_QUERY_ANY 1u
#define RT_QUERY_BRUTE_FORCE 2u
rt_status rt_intersect(rt_context* ctx, const float* o, const float* d, const float* tmax, uint32_t n, uint32_t flags,
                       float* out_t, int32_t* out_id, void* stream);

/* ------------------------------------------------------------------ introspection */
/* Scene statistics after upload: [0] n_spheres [1] n_planes [2] n_triangles [3] bvh prims
 * [4] BVH4 nodes [5] BVH4 depth (levels) [6] device bytes of scene+BVH [7] build time us. */
rt_status rt_scene_info(rt_context* ctx, uint64_t info[8]);
/* Copy the device BVH (W = rt_bvh_width() children per node, 7*W floats each: lo.x[W] hi.x[W]
 * lo.y[W] hi.y[W] lo.z[W] hi.z[W] child[W] as int32; child >= 0 node, 0x7fffffff empty (box
 * inverted), < 0 leaf ~((count-1)<<24 | first))
 * and the leaf-order primitive global IDs to
 * HOST arrays for structural tests; pass NULL to query sizes via *n_nodes / *n_prims. */
rt_status rt_bvh_export(rt_context* ctx, float* nodes, uint32_t* n_nodes, int32_t* prim_gid, uint32_t* n_prims);
/* NEXT-4 ablation (Table 1 "Kd-trees"): build a binned-SAH kd-tree (32 bins,
 * C_trav 1, C_isect 1.5, empty-space bonus 0.8; primitives straddling a split referenced on
 * both sides) over the uploaded scene's BVH primitive records, on the HOST from a copy of them,
 * and upload it for RT_RENDER_KDTREE renders.  The product path (BVH4) is unaffected.
 *   max_leaf: primitives at or below which a node always becomes a leaf (>= 1)
 *   max_depth: depth limit, 0 = round(8 + 1.3 log2 N)
 *   info (HOST, may be NULL): [0] nodes [1] leaf references [2] depth [3] leaves
 *        [4] device bytes [5] host build time us
 * Synchronous.  Replaced by the next call; freed with the scene.
 * Errors: RT_ERR_INVALID_ARG, RT_ERR_NO_SCENE, RT_ERR_OOM, RT_ERR_CUDA. */
rt_status rt_kdtree_build(rt_context* ctx, uint32_t max_leaf, uint32_t max_depth, uint64_t info[6]);
/* FFMA throughput microbenchmark (roofline denominator): runs `iters` FMA chains on every
 * SM and returns achieved FP32 TFLOP/s and the kernel time in ms. */
rt_status rt_bench_ffma(rt_context* ctx, uint32_t iters, double* tflops, double* ms);
/* B0 machine ceilings (the FP32 roofline denominator and the second ceiling,
 * L1/shared-memory bandwidth, "verify in B0").  One 1024-thread CTA per SM times its own body
 * with the SM cycle counter, so out[0..5] are per SM per clock (median over SMs), independent of
 * the clock the run sees; out[6] is the SM clock seen (MHz).  Synchronous on the context stream.
 *   [RT_CEIL_FFMA_FLOP_CLK]   FP32 flops/clk/SM of 3-register FFMA chains (FMA = 2 flops)
 *   [RT_CEIL_FFMA2_FLOP_CLK]  flops/clk/SM of packed FFMA2 chains (4 flops per instruction lane)
 *   [RT_CEIL_FMNMX_CLK]       2-input FP32 max thread-operations/clk/SM (ALU pipe)
 *   [RT_CEIL_FMNMX3_CLK]      3-input FP32 max thread-operations/clk/SM (ALU pipe)
 *   [RT_CEIL_L1_BYTES_CLK]    bytes/clk/SM of 128-bit global loads that hit L1
 *   [RT_CEIL_SMEM_BYTES_CLK]  bytes/clk/SM of conflict-free 128-bit shared loads
 *   [RT_CEIL_SM_MHZ]          SM clock during the FFMA probe
 * Errors: RT_ERR_INVALID_ARG, RT_ERR_CUDA. */
#define RT_NUM_CEILINGS 7
enum {
    RT_CEIL_FFMA_FLOP_CLK = 0, RT_CEIL_FFMA2_FLOP_CLK = 1, RT_CEIL_FMNMX_CLK = 2, RT_CEIL_FMNMX3_CLK = 3,
    RT_CEIL_L1_BYTES_CLK = 4, RT_CEIL_SMEM_BYTES_CLK = 5, RT_CEIL_SM_MHZ = 6
};
rt_status rt_bench_ceilings(rt_context* ctx, double out[RT_NUM_CEILINGS]);

#ifdef __cplusplus
}
#endif
#endif /* RT_B200_H */
