/*
 * pdg.h -- C ABI of the B200 (sm_100a) fp64 SIPG assembly engine.
 *
 * Drop-in boundary for polydg's Approach-2 assembly path
 * (/root/reference/pkg/src/polydg/assembly.py:1090-1134).  polydg is pure
 * Python, so the "binding" a maintainer adds is a ctypes stub (see
 * INTEGRATION.md); this package's own shim is
 * paper_2007_04881_b200/_lib.py + assembly.py.
 *
 * Conventions
 *   - every pointer inside the descriptor structs is a DEVICE pointer owned
 *     by the caller; the library never allocates or frees caller memory
 *     (scratch is passed in explicitly, sized by the *_workspace_bytes calls);
 *   - descriptor structs themselves live in host memory and are read at call
 *     time only;
 *   - all work is enqueued on the caller's stream; nothing synchronises;
 *   - return value: PDG_OK or an error code; pdg_last_error() (thread-local)
 *     describes the last failure.  No C++ exception crosses this boundary;
 *   - data-dependent failures found on the device (degenerate simplices,
 *     straddling flow, unclassified faces ...) are OR-ed into a caller
 *     provided uint32 device word as PDG_FLAG_* bits and mapped to polydg's
 *     exception classes by the host shim after the stream is synchronised.
 */
#ifndef PDG_H_
#define PDG_H_

#ifdef __CUDACC_RTC__ /* runtime-compiled (NVRTC) specialisations see only this */
typedef signed char int8_t;
typedef unsigned char uint8_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
typedef unsigned long size_t;
#else
#include <stddef.h>
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define PDG_ABI_VERSION 3

typedef struct CUstream_st* pdg_stream; /* == cudaStream_t */

/* status codes */
enum {
  PDG_OK = 0,
  PDG_ERR_INVALID = 1,     /* bad argument / inconsistent descriptor     -> ValueError */
  PDG_ERR_CUDA = 2,        /* CUDA runtime failure                       -> RuntimeError */
  PDG_ERR_UNSUPPORTED = 3  /* degree / dimension outside compiled range  -> NotImplementedError */
};

/* device error flags (uint32 bitmask written by kernels) */
enum {
  PDG_FLAG_DEGENERATE_SIMPLEX = 1u << 0, /* QuadratureError  quadrature.py:133-134 */
  PDG_FLAG_DEGENERATE_FACET = 1u << 1,   /* QuadratureError  quadrature.py:152-153 */
  PDG_FLAG_STRADDLE = 1u << 2,           /* ClassificationError model.py:128-135   */
  PDG_FLAG_UNCLASSIFIED = 1u << 3,       /* AssemblyError    assembly.py:680-684   */
  PDG_FLAG_NO_ADJACENT_SIMPLEX = 1u << 4,/* MeshError        model.py:224-225,253  */
  PDG_FLAG_STACK = 1u << 5,              /* coefficient program overflow (host bug) */
  PDG_FLAG_NEG_DIFFUSION = 1u << 6       /* isotropic a(x) < 0 met by the sqrt-weighted volume
                                            path: the host re-runs with PDG_OPT_PLAIN_VOLUME */
};

/* boundary tags (polydg mesh.py:40-45) */
enum {
  PDG_TAG_INTERIOR = 0,
  PDG_TAG_DIRICHLET = 1,
  PDG_TAG_NEUMANN = 2,
  PDG_TAG_INFLOW = 3,
  PDG_TAG_OUTFLOW = 4
};

/* Flattened polytopic mesh (polydg PolytopicMesh, mesh.py:107-188). */
typedef struct pdg_mesh {
  int32_t dim;                           /* 2 or 3 */
  int64_t n_vertices, n_simplices, n_elements, n_faces, n_facets, n_interfaces;
  const double* vertices;                /* [n_vertices][dim] */
  const int32_t* simplices;              /* [n_simplices][dim+1], post-reorientation order */
  const double* simplex_volumes;         /* [n_simplices] */
  const int64_t* elem_ptr;               /* [n_elements+1] -> elem_simplices */
  const int32_t* elem_simplices;         /* ascending within an element */
  const double* elem_volumes;            /* [n_elements] */
  const int32_t* face_owner;             /* [n_faces] */
  const int32_t* face_neighbor;          /* [n_faces], -1 on the boundary */
  const int8_t* face_tag;                /* [n_faces] PDG_TAG_* */
  const double* face_normal;             /* [n_faces][dim], outward from owner */
  const double* face_measure;            /* [n_faces] */
  const int64_t* face_ptr;               /* [n_faces+1] -> facets */
  const int32_t* facet_vertices;         /* [n_facets][dim] */
  const int32_t* facet_owner_simplex;    /* [n_facets] */
  const int32_t* facet_neighbor_simplex; /* [n_facets], -1 on the boundary */
  const int32_t* iface_owner;            /* [n_interfaces] owner < neighbor, sorted */
  const int32_t* iface_neighbor;         /* [n_interfaces] */
  const int64_t* iface_ptr;              /* [n_interfaces+1] -> iface_faces */
  const int32_t* iface_faces;
  const int64_t* elem_bface_ptr;         /* [n_elements+1] -> elem_bfaces */
  const int32_t* elem_bfaces;
} pdg_mesh;

/* Per-element basis (polydg BasisSpec, basis.py:36-71; family P only). */
typedef struct pdg_basis {
  int32_t max_degree;          /* selects the compiled kernel instantiation */
  const int32_t* degree;       /* [n_elements] */
  const double* box;           /* [n_elements][2][dim] spec boxes */
  const int64_t* dof_offset;   /* [n_elements+1] DofMap.offsets (assembly.py:64-89) */
} pdg_basis;

/* Coefficient fields compiled to stack bytecode (paper_2007_04881_b200/model.py). */
#define PDG_MAX_CODE 448
#define PDG_MAX_CONST 96
#define PDG_MAX_STACK 8
typedef struct pdg_prog {
  int32_t offset, length;      /* into code[] */
  int32_t is_const, pad_;
  double value;                /* valid when is_const */
} pdg_prog;

enum { PDG_DIFF_NONE = 0, PDG_DIFF_ISO = 1, PDG_DIFF_FULL = 2 };

typedef struct pdg_coeffs {
  int32_t diffusion_kind;      /* PDG_DIFF_* */
  int32_t diffusion_symmetric; /* 1 if A == A^T for all x */
  int32_t has_advection, has_reaction, has_source, has_dirichlet, has_neumann, pad_;
  pdg_prog diffusion[9];       /* ISO: [0] = a(x); FULL: row-major A_ij */
  pdg_prog advection[3];
  pdg_prog reaction, source, dirichlet, neumann;
  int32_t n_code, n_const;
  int32_t code[PDG_MAX_CODE];  /* op | (arg << 8) */
  double consts[PDG_MAX_CONST];
} pdg_coeffs;

/* Reference quadrature tables (polydg quadrature.py:69-103), uploaded once. */
typedef struct pdg_rules {
  int32_t max_order;
  const double* points;        /* [n][3] (unused coordinates zero) */
  const double* weights;       /* [n] */
  const int32_t* vol_offset;   /* [max_order+1] dim-simplex rule of that order, -1 absent */
  const int32_t* vol_count;
  const int32_t* face_offset;  /* [max_order+1] interval (2D) / triangle (3D) rule */
  const int32_t* face_count;
  const double* sqrt_weights;  /* [n] sqrt(weights) (sqrt-weighted symmetric volume tables) */
  int32_t n_points;            /* n (small tables are staged in shared memory by the kernels) */
  int32_t pad_;
} pdg_rules;

typedef struct pdg_params {
  int32_t quad_increment;      /* AssemblyConfig.quad_increment (assembly.py:347) */
  int32_t include_gradient_terms;
  double penalty_constant;     /* PenaltyConfig.constant (model.py:66) */
  const uint8_t* coverable;    /* [n_elements] or NULL (model.py:67) */
  int32_t options;             /* PDG_OPT_* bits (kernel variants; 0 = default) */
  int32_t pad_;
} pdg_params;

/* pdg_params.options */
enum {
  PDG_OPT_PLAIN_VOLUME = 1 /* isotropic volume term as (w a dphi) dphi^T instead of the
                              symmetric sqrt(w a) dphi table (needed when a(x) < 0) */
};

/* Per adjacency entry (row element e, sorted neighbour j) of the rows of one
 * assembly: the block position and the metadata of the interface's first face,
 * flattened by pdg_iface_records so the element kernel stages a window of
 * neighbours with one contiguous asynchronous copy instead of chains of
 * dependent gathers (nbr -> interface -> face -> sigma / normal / frame).
 * 80 bytes.  Self entry: j == e, fa == fb. */
typedef struct pdg_iface_rec {
  int32_t j;        /* neighbour element (sorted ascending, self included) */
  int32_t nj;       /* its number of basis functions */
  int32_t col;      /* first column of its block within e's rows (assembly.py:316-321) */
  int32_t pj;       /* its degree */
  int32_t fa, fb;   /* face range [fa, fb) of the interface (mesh iface_ptr) */
  int32_t row0;     /* first sub-facet row of face fa */
  int32_t info;     /* bit0: e is face fa's neighbour side; bit1: e is downwind of fa;
                       bit2: single face, single sub-facet, <= 8 face points (paired rounds) */
  double sig;       /* penalty of face fa (model.py:238-257) */
  double nrm[3];    /* owner normal of face fa */
  int64_t dof;      /* first global DoF of j (= first column index of its block) */
  int32_t nrows0;   /* sub-facet rows of face fa */
  int32_t pad_;
} pdg_iface_rec;

/* Block pattern of the rows owned by one assembly (assembly.py:209-340). */
typedef struct pdg_pattern {
  int64_t n_row_elements;
  const int32_t* row_elements; /* ascending element ids, or NULL = all elements */
  const int64_t* nbr_ptr;      /* [n_elements+1] from pdg_adjacency */
  const int32_t* nbr_elem;     /* sorted neighbour ids incl. self */
  const int32_t* nbr_iface;    /* interface id per entry, -1 for self */
  int64_t* row_len;            /* [n_row_elements] columns per row of the element */
  int64_t* elem_val_offset;    /* [n_row_elements+1] first value slot of the element */
  int64_t* elem_row_offset;    /* [n_row_elements+1] first local row of the element */
  int64_t* row_ptr;            /* [n_local_rows+1] */
  int64_t* col_idx;            /* [nnz] */
  pdg_iface_rec* nbr_rec;      /* [nbr_ptr[n_elements]] from pdg_iface_records (entries of owned rows) */
  const int64_t* col_dof;      /* [n_elements] first GLOBAL column of each element's block, or NULL =
                                  dof_offset.  Set when the mesh is a rank's sub-mesh (owned elements
                                  + one-ring halo, monotone relabelling): the rows then carry the
                                  global columns of the whole mesh (distribute.py:200-232) */
} pdg_pattern;

/* Affine frames, produced once per assembly by pdg_frames_build and read by
 * the element kernel (one broadcast load per quadrature point):
 *   simplex [n_simplices][W] in ELEMENT order (row elem_ptr[e]+k is the k-th
 *           simplex of element e): v0, E rows (v_k - v_0), |det E|
 *           (quadrature.py:118-136);
 *   facet   [n_facets][W]: v0, E rows, sqrt(det(E E^T)) (quadrature.py:139-156);
 *   element [n_elements][W]: box centre, 1/half-width, 1/sqrt(width) per axis
 *           (basis.py:139-152).
 * W = 8 doubles in 2D, 16 in 3D. */
typedef struct pdg_frames {
  double* simplex;
  double* facet;
  double* element;
} pdg_frames;

/* One space-time slab (polydg spacetime.py:84-104, 133-388): the spatial mesh
 * x (t0, t1), with prism bases (pdg_basis.box is [n_elements][2][3], time
 * last) and the time-jump data of the bottom facets. */
typedef struct pdg_slab {
  double t0, t1;
  const int8_t* lateral_tag;      /* [n_faces] PDG_TAG_* of the lateral boundary faces
                                     (SlabGeometry._classify_lateral, spacetime.py:229-246) */
  const double* prev_values;      /* previous slab's coefficient vector, or NULL: the initial
                                     data field of the policy (spacetime.py:367-388) */
  const int64_t* prev_dof_offset; /* [n_elements+1] previous slab DofMap (same degree/family) */
  const double* prev_box;         /* [n_elements][2][3] previous slab prism boxes */
  int32_t family;                 /* basis family of the slab: 0 = P, 1 = PQ (basis.py:21-26) */
  int32_t table_rows;             /* shared table rows of the coefficient set (model.slab_policy) */
  pdg_rules time_rules;           /* interval rules (in the face tables) of the time axis */
} pdg_slab;

/* Approach-1 work items (see pdg_a1_emit). */
typedef struct pdg_a1_items {
  int64_t n_volume, n_interior, n_boundary;
  int64_t n_cols;                /* global DoFs (key = row * n_cols + col) */
  const int32_t* volume_element; /* [n_volume] element of the i-th simplex (element order) */
  const int32_t* face;           /* [n_interior + n_boundary] face of the item */
  const int64_t* facet_row;      /* [n_interior + n_boundary] its sub-facet row */
  const int64_t* stripe_offset;  /* [n_items + 1] triplet stripe offsets (widths of assembly.py:733-745) */
  const int64_t* load_offset;    /* [n_items + 1] load (RHS) entry offsets */
} pdg_a1_items;

#ifndef __CUDACC_RTC__ /* the runtime-compiled kernels need the types only */
int pdg_abi_version(void);
const char* pdg_last_error(void);

/* Number of kernels this library has launched in this process (benchmark
 * accounting: the driver compares it with the profiler's launch list). */
int64_t pdg_launch_count(void);

/* Page-locked host memory for result buffers a caller keeps across
 * assemblies (device->host copies at the link's DMA rate; the host side of
 * polydg's returned CSRMatrix, assembly.py:1117-1134).  *out = NULL for 0 bytes. */
int pdg_host_alloc(size_t bytes, void** out);
int pdg_host_free(void* p);

/* col_idx crosses the link once per element: every row of an element's block
 * row has the same columns (assembly.py:316-324).  pdg_pack_block_cols gathers
 * each element's first row, packed[pack_offset[k] ..] (pack_offset = exclusive
 * scan of row_len, device arrays); pdg_expand_block_cols writes it back into
 * every row of a host col_idx (host arrays: elem_row_offset [n+1] local first
 * rows, row_ptr, packed; n_threads host threads). */
int pdg_pack_block_cols(const int64_t* col_idx, const int64_t* elem_val_offset, const int64_t* row_len,
                        const int64_t* pack_offset, int64_t n_row_elements, int64_t* packed, pdg_stream stream);
int pdg_expand_block_cols(int64_t n_row_elements, const int64_t* elem_row_offset, const int64_t* row_ptr,
                          const int64_t* packed, int64_t* col_idx, int32_t n_threads);

/* Bytes of device scratch needed by pdg_adjacency / pdg_pattern_offsets. */
size_t pdg_workspace_bytes(int64_t n_elements, int64_t n_interfaces);

/* Index phase 1: sorted per-element neighbour lists from the interface pairs
 * (replaces the adjacency sets of _pattern_from_adjacency, assembly.py:301-313).
 * nbr_ptr [n_elements+1], nbr_elem / nbr_iface [n_elements + 2*n_interfaces]. */
int pdg_adjacency(const pdg_mesh* mesh, int64_t* nbr_ptr, int32_t* nbr_elem,
                  int32_t* nbr_iface, void* workspace, size_t workspace_bytes,
                  pdg_stream stream);

/* Index phase 2: row lengths, value/row offsets and row_ptr of the owned rows
 * (assembly.py:312-329).  When nnz_host != NULL it receives the number of
 * stored entries (that call synchronises the stream once, to size
 * col_idx/values); pass NULL to re-run on preallocated buffers, no sync. */
int pdg_pattern_offsets(const pdg_mesh* mesh, const pdg_basis* basis, pdg_pattern* pattern,
                        int64_t n_local_rows, int64_t* nnz_host, void* workspace,
                        size_t workspace_bytes, pdg_stream stream);

/* Index phase 3: col_idx (assembly.py:319-324); pdg_assemble can fuse it. */
int pdg_pattern_fill(const pdg_mesh* mesh, const pdg_basis* basis,
                     const pdg_pattern* pattern, pdg_stream stream);

/* Face pre-pass: penalty sigma (model.py:196-257, assembly.py:613-626) and the
 * flow side (model.py:176-191, assembly.py:596-611) of every face.
 * face_flow: interior -> downwind side (0 owner, 1 neighbour, -1 none);
 * Dirichlet -> 1 if the owner sees inflow.  elem_abar: [n_elements] scratch. */
int pdg_face_prepass(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_coeffs* coeffs,
                     const pdg_rules* rules, const pdg_params* params, double* sigma,
                     int8_t* face_flow, double* elem_abar, uint32_t* err_flags,
                     pdg_stream stream);

/* Interface records of the owned rows (pdg_iface_rec), after pdg_adjacency and
 * pdg_face_prepass (sigma, flow side).  Fills pattern->nbr_rec. */
int pdg_iface_records(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_coeffs* coeffs,
                      const pdg_rules* rules, const pdg_params* params, const pdg_pattern* pattern,
                      const double* sigma, const int8_t* face_flow, pdg_stream stream);

/* Geometry pre-pass: fills pdg_frames; degenerate simplices / facets raise
 * PDG_FLAG_DEGENERATE_* (quadrature.py:133-134,152-153). */
int pdg_frames_build(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_frames* frames,
                     uint32_t* err_flags, pdg_stream stream);

/* Main kernel: every owned element computes its volume term, the traces of
 * all its faces (both sides, one-sided emission), its boundary terms and its
 * load, and writes its n_e rows of the CSR values (exclusive writer, no
 * atomics) -- plus col_idx when write_col_idx != 0 -- and its RHS segment
 * (rhs indexed by global DoF).  Replaces _execute_plan + sink
 * (assembly.py:912-972,1117-1122). */
int pdg_assemble(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_coeffs* coeffs,
                 const pdg_rules* rules, const pdg_params* params,
                 const pdg_pattern* pattern, const pdg_frames* frames, const double* sigma,
                 const int8_t* face_flow, double* values, int32_t write_col_idx, double* rhs,
                 uint32_t* err_flags, pdg_stream stream);

/* Same as pdg_assemble, but with the coefficient fields given as CUDA source
 * of a policy class (generated by paper_2007_04881_b200/model.py from the
 * same expressions as pdg_coeffs): the element kernel is specialised at run
 * time with NVRTC for sm_100a (fields inlined, kind flags compile-time
 * constants) and cached per (source, dim, degree).  `coeffs` is still
 * required (kind flags for the launch geometry). */
int pdg_assemble_jit(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_coeffs* coeffs,
                     const char* policy_source, const pdg_rules* rules, const pdg_params* params,
                     const pdg_pattern* pattern, const pdg_frames* frames, const double* sigma,
                     const int8_t* face_flow, double* values, int32_t write_col_idx, double* rhs,
                     uint32_t* err_flags, pdg_stream stream);

/* pdg_face_prepass with the coefficient fields inlined (the NVRTC module of
 * pdg_assemble_jit carries the pre-pass kernels). */
int pdg_face_prepass_jit(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_coeffs* coeffs,
                         const char* policy_source, const pdg_rules* rules, const pdg_params* params,
                         double* sigma, int8_t* face_flow, double* elem_abar, uint32_t* err_flags,
                         pdg_stream stream);

/* Compile (or fetch from the cache) the specialisation pdg_assemble_jit would
 * use; lets callers pay the NVRTC cost outside timed regions. */
int pdg_jit_prepare(const pdg_coeffs* coeffs, const char* policy_source, int32_t dim,
                    int32_t max_degree);

/* ---- space-time slabs (polydg spacetime.py; runtime-specialised, NVRTC) ----
 * The index phase is shared with the spatial path (pdg_adjacency /
 * pdg_pattern_offsets with the slab basis), as are the spatial affine frames
 * (pdg_frames_build).  policy_source: model.slab_policy (coefficients in
 * (x, y[, z], t) + initial data).  Spatial dimension 2 or 3, degree
 * <= PDG_SLAB_MAX_DEGREE (family P) / PDG_SLAB_MAX_DEGREE_PQ, uniform degree
 * for family PQ. */
#define PDG_SLAB_MAX_DEGREE 5
#define PDG_SLAB_MAX_DEGREE_PQ 4

/* Compile (or fetch) the slab kernels of one coefficient set / degree / family. */
int pdg_slab_prepare(const char* policy_source, int32_t spatial_dim, int32_t max_degree, int32_t family);

/* Lateral face pre-pass: penalty sigma with the slab's side data
 * (spacetime.py:301-351) and the flow side (spacetime.py:287-309) of every
 * spatial face; replaces SlabGeometry.face_sigma / upwind_side /
 * dirichlet_inflow. */
int pdg_slab_prepass(const pdg_mesh* mesh, const pdg_basis* basis, const char* policy_source,
                     const pdg_rules* rules, const pdg_params* params, const pdg_slab* slab,
                     const pdg_frames* frames, double* sigma, int8_t* face_flow,
                     uint32_t* err_flags, pdg_stream stream);

/* Slab element kernel: every owned prism writes its n_e CSR rows (values and
 * col_idx) and its RHS segment: volume, lateral faces, bottom facet
 * (replaces assemble_slab's _assemble_approach2 over SlabGeometry,
 * spacetime.py:391-413). */
int pdg_slab_assemble(const pdg_mesh* mesh, const pdg_basis* basis, const char* policy_source,
                      const pdg_rules* rules, const pdg_params* params, const pdg_slab* slab,
                      const pdg_pattern* pattern, const pdg_frames* frames, const double* sigma,
                      const int8_t* face_flow, double* values, double* rhs, uint32_t* err_flags,
                      pdg_stream stream);

/* ---- Approach 1: stage-and-sort (polydg assembly.py:158-174, 977-1087) ----
 * Work items in polydg's plan order (volume sub-simplices, interior
 * sub-facets, boundary sub-facets; uniform-degree meshes reproduce
 * build_work_plan's order exactly), each writing its dense local blocks into a
 * triplet stripe (key = row * n_cols + col; unused slots keep the sentinel
 * key ~0), then a stable radix sort + reduce-by-key into CSR. */

/* Emit every item's triplets + load pairs (NVRTC-specialised like pdg_assemble_jit);
 * sigma / face_flow from pdg_face_prepass, frames from pdg_frames_build. */
int pdg_a1_emit(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_coeffs* coeffs,
                const char* policy_source, const pdg_rules* rules, const pdg_params* params,
                const pdg_frames* frames, const double* sigma, const int8_t* face_flow,
                const pdg_a1_items* items, uint64_t* keys, double* vals, uint64_t* load_keys,
                double* load_vals, uint32_t* err_flags, pdg_stream stream);

/* Scratch bytes of pdg_triplets_to_csr / pdg_triplets_to_vector for n triplets. */
size_t pdg_triplets_workspace_bytes(int64_t n_triplets);

/* triplets_to_csr (assembly.py:1002-1031): stable sort by key, sum duplicates in
 * input order, CSR of n_rows x n_cols.  Sentinel keys (~0) are dropped.  Outputs
 * have capacity n_triplets; *nnz_device receives the number of entries. */
int pdg_triplets_to_csr(const uint64_t* keys, const double* vals, int64_t n_triplets, int64_t n_rows,
                        int64_t n_cols, int64_t* row_ptr, int64_t* col_idx, double* values,
                        int64_t* nnz_device, void* workspace, size_t workspace_bytes, pdg_stream stream);

/* Load pairs (row, value) -> dense vector[n_rows] (the RHS sink, assembly.py:966-970). */
int pdg_triplets_to_vector(const uint64_t* keys, const double* vals, int64_t n, int64_t n_rows,
                           double* out, void* workspace, size_t workspace_bytes, pdg_stream stream);

/* ---- mesh preprocessing: agglomeration (polydg mesh.py:328-473) ----
 * Simplicial mesh + element map -> the polytopic mesh arrays of pdg_mesh
 * (same element / face / facet / interface order and conventions, bit for
 * bit).  Caller-allocated device outputs with capacities: elem_ptr [nel+1],
 * elem_simplices [ns], boxes [nel][2][dim], elem_volumes [nel]; every
 * face / facet array [ns*(dim+1)] (+1 for face_ptr), interface arrays
 * [ns*(dim+1)] (+1 for iface_ptr), elem_bface_ptr [nel+1].  The call
 * synchronises the stream (output sizes are data dependent) and fills the
 * counts.  iface_faces = 0..n_interior_faces-1, elem_bfaces = the rest. */
typedef struct pdg_agg_out {
  int64_t* elem_ptr;
  int32_t* elem_simplices;
  double* boxes;
  double* elem_volumes;
  int32_t* face_owner;
  int32_t* face_neighbor;
  double* face_normal;
  double* face_measure;
  int64_t* face_ptr;
  int32_t* facet_vertices;
  int32_t* facet_owner_simplex;
  int32_t* facet_neighbor_simplex;
  double* facet_measures;
  int32_t* iface_owner;
  int32_t* iface_neighbor;
  int64_t* iface_ptr;
  int64_t* elem_bface_ptr;
  int64_t n_faces, n_facets, n_interfaces, n_interior_faces; /* outputs */
} pdg_agg_out;

size_t pdg_agglomerate_workspace_bytes(int32_t dim, int64_t n_simplices, int64_t n_elements);

int pdg_agglomerate(int32_t dim, int64_t n_vertices, int64_t n_simplices, const double* vertices,
                    const int32_t* simplices, const double* simplex_volumes, const int64_t* agg,
                    int64_t n_elements, int32_t check_connected, pdg_agg_out* out, void* workspace,
                    size_t workspace_bytes, pdg_stream stream);

/* ---- consumers of the device CSR (polydg solver.py:30-118) ----
 * The element-block structure of the assembled CSR (every row of element e
 * holds the same column list) is exploited: the column list is read once
 * per element.  err_flags bits: 2 = missing diagonal block, 4 = singular diagonal block. */
int pdg_spmv_blocked(const int64_t* dof_offset, int64_t n_elements, const int64_t* row_ptr,
                     const int64_t* col_idx, const double* values, const double* x, double* y,
                     uint32_t* err_flags, pdg_stream stream);

/* Inverses of the element diagonal blocks (inverses[inv_offset[e] ...] row-major n_e x n_e). */
int pdg_block_jacobi_setup(const int64_t* dof_offset, int64_t n_elements, int32_t max_block,
                           const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                           const int64_t* inv_offset, double* inverses, uint32_t* err_flags,
                           pdg_stream stream);

/* z = blockdiag(inverses) r. */
int pdg_block_jacobi_apply(const int64_t* dof_offset, int64_t n_elements, const int64_t* inv_offset,
                           const double* inverses, const double* r, double* z, pdg_stream stream);

/* ---- unit-level entry points (tests / debugging) ---- */

/* Mapped volume quadrature of simplices (quadrature.py:118-136):
 * points [n][nq][dim], weights [n][nq] for rule `order`. */
int pdg_map_simplices(const pdg_mesh* mesh, const pdg_rules* rules, int32_t order,
                      const int32_t* simplex_ids, int64_t n, double* points, double* weights,
                      uint32_t* err_flags, pdg_stream stream);

/* Basis values [n][nb] and gradients [n][dim][nb] at points [n][dim] for the
 * basis of `element` (basis.py:129-164). */
int pdg_tabulate(const pdg_mesh* mesh, const pdg_basis* basis, int32_t element,
                 const double* points, int64_t n, double* values, double* grads,
                 pdg_stream stream);

/* One face item of the unit face kernels (pdg_face_blocks). */
enum { PDG_UNIT_INTERIOR = 0, PDG_UNIT_DIRICHLET = 1, PDG_UNIT_INFLOW = 2, PDG_UNIT_NEUMANN = 3 };
typedef struct pdg_face_item {
  int32_t face;   /* mesh face id */
  int32_t kind;   /* PDG_UNIT_* */
  int32_t upwind; /* interior: downwind (inflow) side 0 = owner, 1 = neighbour, -1 none
                     (assembly.py:455-462); Dirichlet: 1 = owner inflow (with_inflow) */
  int32_t pad_;
  double sigma;   /* penalty (interior / Dirichlet) */
} pdg_face_item;

/* Unit face kernels (assembly.py:1160-1234): per item the four dense blocks
 * (oo, on, no, nn) [n][4][nb][nb] of an interior face, or block [0] + load
 * [n][nb] of a Dirichlet / inflow / Neumann face, summed over the face's
 * sub-facets; nb = num_basis(max_degree), unused entries zero.  Rules must
 * hold the face orders 2*max(p_o, p_n) + quad_increment.  Coefficients are
 * interpreted (bytecode, numpy-identical trigonometry). */
int pdg_face_blocks(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_coeffs* coeffs,
                    const pdg_rules* rules, const pdg_params* params, const pdg_face_item* items,
                    int64_t n, double* blocks, double* loads, uint32_t* err_flags, pdg_stream stream);

/* Every coefficient field at n points [n][dim] -> out [n][dim*dim + dim + 4]:
 * A (row-major; an isotropic a(x) on the diagonal), b, c, f, g_D, g_N; absent
 * fields are 0 (model.py:38-55; the a_bar input of penalty_side_data,
 * model.py:196-235). */
int pdg_eval_coeffs(int32_t dim, const pdg_coeffs* coeffs, const double* points, int64_t n, double* out,
                    pdg_stream stream);

/* Dense per-element volume blocks [n][nb][nb] and loads [n][nb]
 * (assembly.py:1139-1152); nb = num_basis(max_degree). */
int pdg_element_blocks(const pdg_mesh* mesh, const pdg_basis* basis, const pdg_coeffs* coeffs,
                       const pdg_rules* rules, const pdg_params* params, const pdg_frames* frames,
                       const int32_t* elements, int64_t n, double* blocks, double* loads,
                       uint32_t* err_flags, pdg_stream stream);

#endif /* __CUDACC_RTC__ */

#ifdef __cplusplus
}
#endif

#endif /* PDG_H_ */
