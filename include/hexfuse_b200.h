/*
 * hexfuse_b200.h -- C ABI of the B200-native fused flux + divergence library
 * (libhexfuse_b200.so).  Plain C types only: pointers, sizes, a POD problem
 * descriptor.  No torch, no C++ types cross this boundary.
 *
 * The boundary this replaces (reference = /root/reference/proj/include/hexfuse):
 *
 *   (b3) the rendered device kernel
 *          extern "C" __global__ void <name>(int n_elements, const REAL* u, REAL* divf)
 *        render.hpp:79-80, launched on n_blocks() x block_threads (layout.hpp:87-90)
 *        -> hf_fused_divergence(): same operands (caller-owned device arrays in
 *           StateField AoSoA order, n_groups*group_words REAL each), but p, d,
 *           group, nu/zeta/T/jac and the D table are runtime arguments instead
 *           of generation-time immediates, and the launch shape is the library's.
 *   (b2) generate_kernel(KernelRequest) + execute(ir, field, grid)
 *        presets.hpp:144-161, simulator.hpp:184-192
 *        -> hf_fused_divergence() with hf_problem.method (auto / planar / planar-managed / lines)
 *   (b1) StateField oracle_divergence(const StateField&, const PhysParams&,
 *                                     const std::array<double,3>& jac, bool with_source)
 *        oracle.hpp:20-21
 *        -> hf_fused_divergence_host() (host buffers in, host buffers out);
 *           include/hexfuse_b200.hpp wraps it with exactly that C++ signature.
 *
 * Error model (mirrors the reference's exception classes and CLI exit codes,
 * cli.hpp:360-368):  HF_EINVAL  <=> std::invalid_argument (exit 2)
 *                    HF_ERUNTIME <=> std::runtime_error / CUDA error (exit 1)
 * The message of the last failure on the calling thread is hf_last_error().
 *
 * Threading: every entry point is reentrant; the operator table travels in the
 * kernel's __grid_constant__ parameters, so there is no per-device state on
 * the launch path and no allocation in hf_fused_divergence().
 */
#ifndef HEXFUSE_B200_H
#define HEXFUSE_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define HF_API __attribute__((visibility("default")))
#else
#define HF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define HF_OK 0
#define HF_ERUNTIME 1 /* runtime_error: CUDA failure, missing device        */
#define HF_EINVAL 2   /* invalid_argument: bad p/d/params/group/method combo */

#define HF_FP32 0 /* Precision::fp32 (core.hpp:10), 4-byte words */
#define HF_FP64 1 /* Precision::fp64, 8-byte words                */

#define HF_METHOD_AUTO 0    /* measured selection table (replaces preset_table, presets.hpp:25-37) */
#define HF_METHOD_PLANAR 1  /* Alg. 1, thread per (element, z-plane)  (codegen_planar.hpp:251-273) */
#define HF_METHOD_LINES 2   /* higher-parallelism, thread per line     (codegen_lines.hpp:299-318)  */
#define HF_METHOD_UNFUSED 3 /* stage 2 + stage 3 (+ stage 6) kernels  (io_model.hpp:32-34)         */
#define HF_METHOD_PLANAR_MANAGED 4 /* Alg. 1 with every operand resident in shared memory
                                      (Method::PlanarManaged, codegen_planar.hpp:276-300) */

/* One fused-divergence problem.  Field layout is StateField's
 * (layout.hpp:104-134): word (e,i,j,k,v) at
 *   (e/group)*group_words + e%group + group*(i + m j + m^2 k + m^d v),
 *   group_words = group * m^d * n_v, m = p+1, n_v = 1+d+d^2,
 * padded to ceil(n_elem/group) groups; padding elements are never read or written. */
typedef struct hf_problem {
    int d;            /* 2 or 3                                       */
    int p;            /* order: 1..7 (d=3), 1..8 (d=2)                */
    int64_t n_elem;   /* real elements                                */
    int group;        /* AoSoA group size (StateField::group), >= 1   */
    int precision;    /* HF_FP32 | HF_FP64                            */
    double nu, zeta, T; /* PhysParams (equations.hpp:14-24)           */
    double jac[3];    /* constant per-axis metric, jac[2] unused for d=2 */
    int with_source;  /* fuse stage 6 (-g/T on the gradient rows)     */
    int method;       /* HF_METHOD_*                                  */
} hf_problem;

/* Static description of the kernel a problem would launch. */
typedef struct hf_kernel_info {
    int method;          /* resolved HF_METHOD_* (never AUTO)            */
    int elems_per_cta;   /* elements one CTA owns (the preferred group)  */
    int block_threads;
    int shared_bytes;    /* dynamic shared memory per CTA                */
    int registers;       /* per thread, from cudaFuncGetAttributes (0 if no device) */
    int64_t grid;        /* CTAs for this problem                        */
    int bulk_path;       /* 1 if full chunks stage through cp.async.bulk */
    int blocks_per_sm;   /* resident CTAs per SM (cudaOccupancy...; 0 if no device) */
    char name[96];
} hf_kernel_info;

/* ---- layout helpers (pure host functions, no device needed) ---- */
HF_API int hf_n_vars(int d);                                   /* equations.hpp:27-30 */
HF_API int64_t hf_field_words(const hf_problem* pr);           /* layout.hpp:115,125  */
HF_API int64_t hf_offset(const hf_problem* pr, int64_t e, int i, int j, int k, int v); /* layout.hpp:128-134 */
HF_API int hf_validate(const hf_problem* pr);                  /* HF_OK or HF_EINVAL  */
/* D on the Gauss-Legendre nodes of order m = p+1, row-major (operators.hpp:17-74); m in [2,9] */
HF_API int hf_derivative_matrix(int m, double* D_out, double* nodes_out);
/* Algorithmic (io_model Fused23) bytes per solution point: 2 * n_v * word bytes. */
HF_API int64_t hf_algorithmic_bytes_per_point(const hf_problem* pr);

/* ---- selection (replaces preset_table / default_lines_n, presets.hpp:25-103) ---- */
HF_API int hf_selected_method(const hf_problem* pr);    /* resolves HF_METHOD_AUTO */
HF_API int hf_preferred_group(const hf_problem* pr);    /* group that enables the bulk-copy path */
HF_API int hf_kernel_info_get(const hf_problem* pr, hf_kernel_info* out);

/* ---- device-buffer entry points (the (b3)/(b2) replacement) ----
 * u_dev, divf_dev: device pointers, hf_field_words(pr) words of the problem's
 * precision each, distinct.  stream: a cudaStream_t (NULL = legacy default).
 * Asynchronous: returns after enqueueing; errors from the launch are reported. */
HF_API int hf_fused_divergence(const hf_problem* pr, const void* u_dev, void* divf_dev, void* stream);

HF_API size_t hf_unfused_workspace_bytes(const hf_problem* pr); /* d*n_v words per padded point */
HF_API int hf_unfused_divergence(const hf_problem* pr, const void* u_dev, void* divf_dev, void* ws_dev, void* stream);

/* ---- extension: elements with a non-constant Jacobian ----
 * Beyond the reference, which fixes a constant per-axis Jacobian (oracle.hpp:47):
 * (bi/tri)linear elements given by their 2^d corners ("linear elements, for which
 * only the element corners need to be loaded").  Conservative FR
 * form out = -(1/|J|) sum_a D_a(sum_b adj(J)_ab F_b) (+ source) at the solution
 * points; pr->jac and pr->method are ignored.  geom_dev: hf_geometry_words(pr)
 * words of the problem's precision, AoSoA with the field's group:
 *   word (e, c, x) = (e/group)*group*2^d*d + e%group + group*(x + d*c),
 * corner c at reference point (bit k of c ? +1 : -1) along xi_k.  For an
 * axis-aligned box of half-widths h this equals hf_fused_divergence with
 * jac = 1/h.  Asynchronous like hf_fused_divergence. */
HF_API int64_t hf_geometry_words(const hf_problem* pr);
HF_API int hf_fused_divergence_mapped(const hf_problem* pr, const void* u_dev, const void* geom_dev, void* divf_dev,
                                      void* stream);
HF_API int hf_mapped_kernel_info(const hf_problem* pr, hf_kernel_info* out);

/* ---- extension: the FR stages either side of the fused kernel ----
 * PAPER.md Table 1 on a periodic structured mesh of dims[0] x dims[1] (x dims[2])
 * elements, element e = ex + dims[0]*(ey + dims[1]*ez), the constant per-axis
 * Jacobian pr->jac (the reference models these stages' I/O only):
 *   hf_fr_project   stage 1: U_f = every a-line extrapolated to xi_a = -1, +1;
 *   hf_fr_correct   stages 4+5: common flux (Rusanov on the
 *                   pressure / velocity rows, wave speed |V_a| + sqrt(V_a^2 + zeta);
 *                   the mean of both sides on the gradient rows) and the DG correction
 *                   -sum_a jac_a (g_L' jump_(-a) + g_R' jump_(+a)) added in place
 *                   to divf_dev, which holds hf_fused_divergence's result;
 *   hf_fr_divergence_faces  stages 1+2+3+6 in one pass: the fused kernel also
 *                   writes the faces from the chunk it has staged (the two
 *                   kernels hf_fused_divergence + hf_fr_project where no fused
 *                   form is built); bit-identical to them;
 *   hf_fr_residual  the whole right-hand side on one device (1+2+3+6, then 4+5).
 * Face layout (AoSoA, the field's group, L = m^(d-1), l = transverse indices,
 * s = 0 at xi = -1, 1 at +1):
 *   word (e, a, s, l, v) = (e/group)*group*2*d*L*n_v + e%group + group*(l + L*(s + 2*(a + d*v))).
 * Partitions (multi-GPU): whole element layers (layer = dims[0]*dims[1], d = 3;
 * dims[0], d = 2), pr->n_elem = mesh->n_local, ghost_lo / ghost_hi = the face
 * arrays (same layout) of the layer below / above the partition (periodic). */
typedef struct hf_mesh {
    int dims[3];
    int64_t e_begin;  /* first element of the partition            */
    int64_t n_local;  /* its elements (== pr->n_elem)               */
    int64_t layer;    /* elements per ghost layer (partitions only) */
} hf_mesh;
HF_API int64_t hf_face_words(const hf_problem* pr);
HF_API int hf_fr_project(const hf_problem* pr, const void* u_dev, void* uf_dev, void* stream);
HF_API int hf_fr_correct(const hf_problem* pr, const hf_mesh* mesh, const void* uf_dev, const void* ghost_lo,
                         const void* ghost_hi, void* divf_dev, void* stream);
HF_API int hf_fr_divergence_faces(const hf_problem* pr, const void* u_dev, void* uf_dev, void* divf_dev, void* stream);
HF_API int hf_fr_residual(const hf_problem* pr, const int* dims, const void* u_dev, void* uf_dev, void* divf_dev,
                          void* stream);

/* ---- peer memory for the FR ghost layers (NVLink / NVSwitch, one process per GPU) ----
 * A rank exports its face array (hf_ipc_handle), its neighbours open it
 * (hf_ipc_open) and pass pointers into it as ghost_lo / ghost_hi of
 * hf_fr_correct: the correction kernel then reads the neighbours' boundary
 * faces straight from their memory over NVLink -- the exchange and the
 * interface kernel are one kernel, no copy.  Thin wrappers over CUDA IPC; the
 * handle names dev_ptr's whole allocation and *offset_out is dev_ptr's byte
 * offset in it (add it to the pointer hf_ipc_open returns). */
#define HF_IPC_HANDLE_BYTES 64
HF_API int hf_ipc_handle(const void* dev_ptr, void* handle_out, int64_t* offset_out);
HF_API int hf_ipc_open(const void* handle, void** dev_ptr_out);
HF_API int hf_ipc_close(void* dev_ptr);

/* ---- host-buffer entry point (the (b1) replacement) ----
 * u_host / divf_host: host arrays of hf_field_words(pr) words of the problem's
 * precision (float for HF_FP32, double for HF_FP64).  Pinned memory is used
 * directly; pageable memory is staged.  The field is streamed through the GPU
 * in group-aligned slices with host->device copy, kernel and device->host copy
 * overlapped on three streams.  Synchronous: returns when divf_host is filled. */
typedef struct hf_context hf_context;
HF_API hf_context* hf_context_create(int device);
HF_API void hf_context_destroy(hf_context* ctx);
HF_API int hf_fused_divergence_host(hf_context* ctx, const hf_problem* pr, const void* u_host, void* divf_host);
/* Several fields (e.g. one per polynomial order of a p-adaptive mesh) through ONE
 * slice pipeline: the copy engines fill once before the first field and drain once
 * after the last, instead of per field.  Same per-field semantics and errors as
 * hf_fused_divergence_host; synchronous. */
HF_API int hf_fused_divergence_host_batch(hf_context* ctx, int n_fields, const hf_problem* prs,
                                          const void* const* u_hosts, void* const* divf_hosts);

/* ---- multi-GPU partition (element-parallel, no collective) ----
 * Part `part` of `n_parts` contiguous, group-aligned slices: elements
 * [*e_begin, *e_begin + *n_elem_part), starting at word *word_offset of the
 * field.  The slice is itself a valid field with the same group. */
HF_API int hf_partition(const hf_problem* pr, int n_parts, int part, int64_t* e_begin, int64_t* n_elem_part,
                 int64_t* word_offset);

/* ---- state blob + sidecar I/O (layout.hpp:155-200) ----
 * The reference's on-disk field: <path> holds the padded field's words little-endian
 * (4 B fp32 / 8 B fp64), <path>.json the sidecar {"byte_order","d","group","n_elem",
 * "p","precision","words"} (field_sidecar, layout.hpp:155-159).  Host only.
 *   hf_blob_info   import_blob's sidecar half (layout.hpp:179-186): fills d, p, n_elem,
 *                  group, precision of *shape_out (other fields untouched)
 *   hf_blob_read   the words into host_words (hf_field_words(pr) words of pr's
 *                  precision); pr's shape must equal the sidecar's
 *   hf_blob_write  export_blob (layout.hpp:161-177), byte-identical blob and sidecar
 *   hf_fused_divergence_blob  in_path -> B200 host path -> out_path: shape from the
 *                  input sidecar, physics / jac / source / method from *params
 * Errors as the reference: missing or short files, word-count mismatch HF_ERUNTIME
 * (std::runtime_error); unknown precision HF_EINVAL (precision_from_string, core.hpp:16-20). */
HF_API int hf_blob_info(const char* path, hf_problem* shape_out);
HF_API int hf_blob_read(const char* path, const hf_problem* pr, void* host_words);
HF_API int hf_blob_write(const char* path, const hf_problem* pr, const void* host_words);
HF_API int hf_fused_divergence_blob(hf_context* ctx, const hf_problem* params, const char* in_path,
                                    const char* out_path);

HF_API const char* hf_last_error(void);
HF_API const char* hf_version(void);

#ifdef __cplusplus
}
#endif

#endif /* HEXFUSE_B200_H */
