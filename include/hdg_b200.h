/*
 * hdg_b200.h — C ABI of the B200-native element-local HDG engine.
 *
 * Drop-in boundary for the element-local half of the reference HDG library
 * (/root/reference/proj, namespace hdg). Every entry point below names the
 * reference interface it replaces (file:line). Conventions:
 *   - plain pointers and sizes, no C++ or torch types; no exceptions cross;
 *   - every call returns HDG_OK or an HDG_E* status; hdg_b200_last_error()
 *     holds the message of the calling thread's last failure;
 *   - d_* arguments are caller-owned DEVICE buffers, h_* are HOST buffers;
 *   - arrays keep the reference (Eigen, column-major) layouts: an Nelt x c
 *     matrix stores entry (K, j) at j*Nelt + K; Batch3 slice K of an r x c
 *     batch starts at K*r*c (proj/include/hdg/batch.hpp:14-38);
 *   - indices are 0-based, permutation codes 1..6 (proj/include/hdg/mesh.hpp:6-9);
 *   - device work is stream-ordered on the context's stream.
 */
#ifndef HDG_B200_H
#define HDG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HDG_B200_ABI_VERSION 1

/* status codes */
#define HDG_OK 0
#define HDG_ESINGULAR 1 /* singular local system; *bad_element = lowest index (LocalSolverError, local_solver.hpp:45-49) */
#define HDG_EINVAL 2    /* bad argument (std::invalid_argument in the reference) */
#define HDG_ECUDA 3     /* CUDA runtime failure */
#define HDG_ENCCL 4     /* NCCL failure */
#define HDG_EMESH 5     /* MeshError (mesh.hpp:75-78) */
#define HDG_ESTATE 6    /* call order (e.g. no degree set) */
#define HDG_ESOLVE 7    /* GlobalSolverError (global_system.hpp:44-46) */

/* boundary classifiers for generated box meshes (mesh.cpp:173-183) */
#define HDG_BC_ALL_DIRICHLET 0
#define HDG_BC_DIRICHLET_TOP_BOTTOM 1
#define HDG_BC_DIRICHLET_X 2 /* |nu_x| > 0.5 */

/* ---------------------------------------------------------------- fields
 * Coefficient fields replace the reference ScalarField callbacks
 * (proj/include/hdg/coefficient.hpp:13-14): either a constant, samples at the
 * physical quadrature nodes (what the callback returns, nq x nelt, element's
 * nodes contiguous, device memory), or a postfix program over (x,y,z) the
 * kernels evaluate at each node.                                           */
#define HDG_FIELD_CONST 0
#define HDG_FIELD_SAMPLED 1
#define HDG_FIELD_PROGRAM 2
#define HDG_FIELD_MAX_OPS 128
#define HDG_FIELD_MAX_CONSTS 48
#define HDG_FIELD_MAX_STACK 16
enum {
  HDG_OP_X = 0, HDG_OP_Y, HDG_OP_Z, HDG_OP_CONST, HDG_OP_ADD, HDG_OP_SUB, HDG_OP_MUL,
  HDG_OP_DIV, HDG_OP_NEG, HDG_OP_SIN, HDG_OP_COS, HDG_OP_EXP, HDG_OP_SQRT, HDG_OP_ABS,
  HDG_OP_LT, HDG_OP_POW
};
typedef struct {
  int kind;               /* HDG_FIELD_* */
  double value;           /* CONST */
  const double* samples;  /* SAMPLED: device, nq x nelt */
  const int* ops;         /* PROGRAM: host, nops opcodes (copied at call) */
  int nops;
  const double* consts;   /* PROGRAM: host, nconst literals in order of HDG_OP_CONST */
  int nconst;
} hdg_field;

typedef struct hdg_ctx hdg_ctx;   /* device, stream, reference tables */
typedef struct hdg_mesh hdg_mesh; /* host mesh (setup layer) */

const char* hdg_b200_version(void);
const char* hdg_b200_last_error(void);

/* ------------------------------------------------------------ host mesh
 * Replaces box_mesh (mesh.cpp:185-253) and expand (mesh.cpp:74-171): the
 * face numbering (Dirichlet rows, Neumann rows, then interior faces in
 * sorted-vertex-triple order) is bit-exact with the reference.            */
int hdg_b200_mesh_box(int nx, int ny, int nz, int bc_rule, double perturb_frac, uint64_t seed,
                      double keep_plane_z, hdg_mesh** out);
int hdg_b200_mesh_create(int nver, const double* h_coords, int nelt, const int* h_elements,
                         int ndir, const int* h_dirichlet, int nneu, const int* h_neumann,
                         hdg_mesh** out);
int hdg_b200_mesh_expand(hdg_mesh* m);
/* dims: nver, nelt, nfc, ndir, nneu, expanded */
int hdg_b200_mesh_dims(const hdg_mesh* m, int64_t dims[6]);
#define HDG_MESH_COORDS 0    /* double nver x 3 */
#define HDG_MESH_ELEMENTS 1  /* int nelt x 4 */
#define HDG_MESH_DIRICHLET 2 /* int ndir x 3 */
#define HDG_MESH_NEUMANN 3   /* int nneu x 3 */
#define HDG_MESH_FACES 4     /* int nfc x 3 */
#define HDG_MESH_FACETYPE 5  /* uint8 nfc (0 interior, 1 Dirichlet, 2 Neumann) */
#define HDG_MESH_FACEBYELE 6 /* int nelt x 4 */
int hdg_b200_mesh_copy(const hdg_mesh* m, int what, void* h_dst);
void hdg_b200_mesh_free(hdg_mesh* m);

/* Skeleton sparsity (global_system.cpp:31-56): per face the sorted faces it
 * couples to, and per element the slot of each (l1,l2) pair in row-face l1's
 * list. nnbr_total = sum of list lengths; nnz = nnbr_total * d2 * d2.      */
int hdg_b200_pattern_dims(const hdg_mesh* m, int64_t* nnbr_total);
int hdg_b200_pattern_build(const hdg_mesh* m, int64_t* h_facebase /* nfc+1 */,
                           int* h_nbr /* nfc x 8 row-major, -1 padded */,
                           uint8_t* h_slot /* nelt x 16 */);
/* Same from a bare facebyele (nelt x 4, faces numbered 0..nfc-1), e.g. a
 * slab's locally renumbered faces in multi-GPU runs. Any output may be NULL. */
int hdg_b200_pattern_build_raw(int nelt, int nfc, const int* h_facebyele, int64_t* nnbr_total,
                               int64_t* h_facebase, int* h_nbr, uint8_t* h_slot);

/* ------------------------------------------------------------- context */
int hdg_b200_create(int device, void* cuda_stream, hdg_ctx** out);
void hdg_b200_destroy(hdg_ctx* ctx);
int hdg_b200_set_stream(hdg_ctx* ctx, void* cuda_stream);
/* Tables for degree k on tet_rule(tet_deg) / tri_rule(tri_deg)
 * (quadrature.cpp:43-90, basis.cpp:151-165; study.cpp:13-15 uses 2k+2).   */
int hdg_b200_set_degree(hdg_ctx* ctx, int k, int tet_deg, int tri_deg);
/* Degree k+1 tables on tet_rule(tet_deg) for postprocess_star (study.cpp:33-34). */
int hdg_b200_set_postprocess_rule(hdg_ctx* ctx, int tet_deg);
/* dims: k, d3, d2, nq, nqd, factor_doubles_per_element, nq_post, d3_post */
int hdg_b200_dims(const hdg_ctx* ctx, int64_t dims[8]);
#define HDG_TABLE_TET_BARY 0
#define HDG_TABLE_TET_W 1
#define HDG_TABLE_P 2
#define HDG_TABLE_CHAT 3
#define HDG_TABLE_WLM 4
#define HDG_TABLE_PP 5
#define HDG_TABLE_DD 6
#define HDG_TABLE_TRI_BARY 7
#define HDG_TABLE_TRI_W 8
int hdg_b200_copy_table(const hdg_ctx* ctx, int which, double* h_dst, int64_t capacity);
/* Same tables built on the host only (no device needed). */
int hdg_b200_host_table(int k, int tet_deg, int tri_deg, int which, double* h_dst, int64_t capacity);

/* ------------------------------------------------------ K1: geometry
 * Replaces geometry (mesh.cpp:43-66), the per-element part of expand
 * (mesh.cpp:153-169), piola_coefficients (element_matrices.cpp:48-57),
 * normal_weights (:59-64) and StabilizationField::scaled (:31-36).        */
typedef struct {
  double* volume;  /* nelt */
  double* piola;   /* nelt x 9: a_xx a_xy a_xz a_yx ... (detB * B^{-T}) */
  double* normals; /* nelt x 12: outward n_l, |n_l| = |e_l| */
  int* perm;       /* nelt x 4, 1..6 */
  double* T;       /* nelt x 4: tau(K,l) * |e_{f(K,l)}| */
  double* verts;   /* nelt x 12: vertex coordinates x1..x4, y1..y4, z1..z4 */
  double* area;    /* nfc */
} hdg_geometry;
int hdg_b200_geometry(hdg_ctx* ctx, int nver, int nelt, int nfc, const double* d_coords,
                      const int* d_elements, const int* d_faces, const int* d_facebyele,
                      const double* d_tau /* nelt x 4 or NULL */, double tau_const,
                      hdg_geometry* g);
/* tau(K,l) = 1 + |beta(x_e) . nu_{K,l}| at face centroids (config C4 upwinding). */
int hdg_b200_upwind_tau(hdg_ctx* ctx, int nelt, const hdg_geometry* g, hdg_field bx,
                        hdg_field by, hdg_field bz, double* d_tau);

/* --------------------------------------------- K2+K3: build + condense
 * Replaces build_element_matrices (element_matrices.cpp:282-309) ->
 * local_blocks (local_solver.cpp:124-126) -> condense (local_solver.cpp:71-100)
 * as one call returning the same CondensedSystem: C (m x m x nelt Batch3) and
 * Cf (m x nelt), m = 4*d2. d_factors (nullable) receives the per-element
 * recovery cache used by hdg_b200_recover (dims[5] doubles per element:
 * M^-1 packed lower, Vs = S^-1 V (d3 x m), fs = S^-1 f, padded to 16 bytes;
 * the reference refactorises A1 in local_recover instead).
 * d_work: scratch of hdg_b200_work_size() bytes.                           */
int64_t hdg_b200_work_size(const hdg_ctx* ctx, int nelt);
int hdg_b200_build_condense(hdg_ctx* ctx, int nelt, const hdg_geometry* g, hdg_field kappa,
                            hdg_field c, hdg_field f, double* d_C, double* d_Cf,
                            double* d_factors, void* d_work, int64_t* bad_element);

/* ------------------------------------------ K5: gather + local recover
 * Replaces gather_traces (global_system.cpp:167-175) + local_recover
 * (local_solver.cpp:102-135): [q;u] = A1^{-1}(Af - A2 lambda_K) with lambda_K
 * gathered from the skeleton vector uhat (dof = face*d2 + i). Uses the cache
 * written by build_condense. Outputs d3 x nelt each.                         */
int hdg_b200_recover(hdg_ctx* ctx, int nelt, const hdg_geometry* g, const int* d_facebyele,
                     const double* d_factors, const double* d_uhat, double* d_qx, double* d_qy,
                     double* d_qz, double* d_u);

/* ------------------------------------------------------ K4: scatter
 * Replaces assemble (global_system.cpp:31-56): CSR values of H (pattern from
 * hdg_b200_pattern_fill; structurally symmetric so CSR == Eigen's CSC
 * pattern) and b += Cf. d_vals and d_b must be zeroed by the caller.       */
int hdg_b200_pattern_fill(hdg_ctx* ctx, int nfc, int d2, const int64_t* d_facebase,
                          const int* d_nbr, int64_t* d_rowptr, int* d_colidx);
int hdg_b200_scatter(hdg_ctx* ctx, int nelt, int d2, const int* d_facebyele,
                     const uint8_t* d_slot, const int64_t* d_facebase, const double* d_C,
                     const double* d_Cf, double* d_vals, double* d_b);
/* Face-ordered K4 (same result as hdg_b200_scatter, bit for bit): each face's
 * block row of H is one contiguous run, gathered from its elements' C
 * (symmetric: the contiguous column block l is the transposed row block) and
 * written once; the interior diagonal blocks and b sum the two sides in
 * registers. Every entry of d_vals and d_b is written (no zeroing needed).
 * d_sides (nfc x 2) comes from hdg_b200_face_sides: e*4 + l of the face's
 * elements, lower element first, -1 for a one-sided face.                  */
int hdg_b200_face_sides(hdg_ctx* ctx, int nelt, int nfc, const int* d_facebyele, int* d_sides);
int hdg_b200_scatter_faces(hdg_ctx* ctx, int nfc, int d2, const int* d_sides,
                           const uint8_t* d_slot, const int64_t* d_facebase, const double* d_C,
                           const double* d_Cf, double* d_vals, double* d_b);

/* --------------------------------------------------- K6: postprocess
 * Replaces postprocess_star (postprocess.cpp:33-74) with stiffness_matrices
 * (element_matrices.cpp:258-280): u* of degree k+1, d3(k+1) x nelt.        */
int hdg_b200_postprocess(hdg_ctx* ctx, int nelt, const hdg_geometry* g, hdg_field kappa,
                         const double* d_qx, const double* d_qy, const double* d_qz,
                         const double* d_u, double* d_ustar);

/* ------------------------------------- interface exchange (multi-GPU)
 * Elements are split into contiguous z-slabs, one per rank; each rank
 * scatters its slab into a slab-local CSR (faces it touches, global order).
 * Two tets share at most one face, so the only entries two slabs share are
 * the interface faces' d2 x d2 diagonal blocks of H and their d2 entries of b:
 * the reference's assemble sums both sides' triplets (global_system.cpp:
 * 31-56, setFromTriplets at :53-54). A plan lists, per neighbour rank, the
 * interface faces (slab-local ids, ascending global order, so both sides pair
 * entry by entry); exchange_interface gathers those entries, runs one grouped
 * ncclSend/ncclRecv per neighbour on the context stream and adds what it
 * receives: both ranks end with a + b == b + a, bit-identical to one GPU.
 * NCCL failures return HDG_ENCCL. NCCL is loaded at run time (libnccl.so.2).
 * exchange_positions: the plan's positions for one face list (host only):
 *   nfaces*d2*d2 value positions (face-major, block row-major), then
 *   nfaces*d2 positions in b.
 * exchange_pack / unpack_add: the gather and the add of one peer's entries
 *   (what exchange_interface does around the transport), for callers with
 *   their own transport.                                                  */
typedef struct hdg_exchange hdg_exchange;
int hdg_b200_exchange_positions(int nfc, int d2, const int64_t* h_facebase, const int* h_nbr, int nfaces,
                                const int* h_faces, int64_t* h_pos);
int hdg_b200_exchange_plan(hdg_ctx* ctx, int nfc, int d2, const int64_t* h_facebase, const int* h_nbr,
                           int npeers, const int* h_peer_rank, const int* h_peer_nfaces,
                           const int* h_faces /* concatenated per peer */, hdg_exchange** out);
void hdg_b200_exchange_free(hdg_exchange* plan);
int hdg_b200_exchange_pack(hdg_ctx* ctx, const hdg_exchange* plan, int peer, const double* d_vals,
                           const double* d_b, double* d_buf);
int hdg_b200_exchange_unpack_add(hdg_ctx* ctx, const hdg_exchange* plan, int peer, const double* d_buf,
                                 double* d_vals, double* d_b);
/* nccl_comm: an ncclComm_t (from hdg_b200_nccl_comm_init or the caller's own). */
int hdg_b200_exchange_interface(hdg_ctx* ctx, const hdg_exchange* plan, void* nccl_comm, double* d_vals,
                                double* d_b);
/* NCCL communicator plumbing without NCCL types: rank 0 makes the 128-byte
 * unique id, the caller broadcasts it (e.g. torch.distributed), every rank
 * initialises on the context's device.                                     */
int hdg_b200_nccl_get_unique_id(unsigned char id[128]);
int hdg_b200_nccl_comm_init(hdg_ctx* ctx, int nranks, int rank, const unsigned char id[128], void** comm);
int hdg_b200_nccl_comm_destroy(void* comm);

/* ------------------------------------------------ device mesh setup
 * expand_device: mesh.cpp:74-171 on the GPU, bit-exact with
 * hdg_b200_mesh_expand (face numbering, parametrisation, facetype,
 * facebyele; same MeshError conditions and messages). Inputs and outputs are
 * device arrays in the host-mesh layouts (column-major: coords nver x 3,
 * elements nelt x 4, dirichlet/neumann rows x 3, faces nfc x 3, facebyele
 * nelt x 4). d_faces/d_facetype hold nfc = (4 nelt + ndir + nneu) / 2 rows,
 * returned in *nfc_out. Vertex ids must fit 21 bits (nver < 2^21).
 * pattern_device: hdg_b200_pattern_build_raw on the GPU from a device
 * facebyele (facebase nfc + 1, nbr nfc x 8, slot nelt x 16).
 * Both synchronise the context stream once to report errors.           */
int hdg_b200_expand_device(hdg_ctx* ctx, int nver, const double* d_coords, int nelt,
                           const int* d_elements, int ndir, const int* d_dirichlet, int nneu,
                           const int* d_neumann, int* d_faces, uint8_t* d_facetype,
                           int* d_facebyele, int* nfc_out);
int hdg_b200_pattern_device(hdg_ctx* ctx, int nelt, int nfc, const int* d_facebyele,
                            int64_t* d_facebase, int* d_nbr, uint8_t* d_slot, int* maxnbr);

/* ------------------------------------------- K8: skeleton boundary data
 * Face moments of a field against the trace basis, over the face's global
 * vertex triple (face_quad_points, global_system.cpp:9-29). Boundary faces
 * are numbered first (Dirichlet [0, ndir), then Neumann [ndir, ndir+nneu)),
 * mesh.cpp:99-116. A SAMPLED field holds nqd x (faces in the set) samples.
 *  dirichlet_project  replaces dirichlet_project (global_system.cpp:58-70):
 *                     d_out (ndir x d2) = 1/2 sum_r w_r D_i g.
 *  skeleton_project   replaces l2_project_skeleton (postprocess.cpp:84-93):
 *                     d_out (nfc x d2), same moments on every face.
 *  neumann_load       replaces neumann_load (global_system.cpp:72-104):
 *                     d_b[f d2 + i] += alpha sum_r w_r D_i (g . n) on the
 *                     Neumann faces only, n = area-scaled normal of the face's
 *                     element (g->normals). alpha = -1 on the assembled b is
 *                     study.cpp:25 "b -= neumann_load(...)"; alpha = 1 on a
 *                     zeroed vector reproduces the reference's return value. */
int hdg_b200_dirichlet_project(hdg_ctx* ctx, int nver, const double* d_coords, int nfc,
                               const int* d_faces, int ndir, hdg_field g, double* d_out);
int hdg_b200_skeleton_project(hdg_ctx* ctx, int nver, const double* d_coords, int nfc,
                              const int* d_faces, hdg_field g, double* d_out);
int hdg_b200_neumann_load(hdg_ctx* ctx, int nver, const double* d_coords, int nfc,
                          const int* d_faces, int nelt, const int* d_facebyele,
                          const hdg_geometry* g, int ndir, int nneu, hdg_field gx,
                          hdg_field gy, hdg_field gz, double alpha, double* d_b);

/* ------------------------------------------------- K9: skeleton solve
 * Replaces solve_skeleton (global_system.cpp:106-165): Dirichlet dofs (faces
 * [0, ndir)) fixed to d_ub (ndir x d2, hdg_b200_dirichlet_project), the free
 * dofs from H_ff x = b_f - H_fD u_D on the block CSR of hdg_b200_scatter,
 * iterated until ||r|| <= rtol ||r_0|| or maxit. A system passing the
 * reference's symmetry test (sum|H - H^T| < 1e-12 sum|H| over the free block,
 * :144-148) is solved by block-Jacobi preconditioned CG (the SimplicialLDLT
 * branch); any other by block-Jacobi preconditioned BiCGStab restarted on the
 * true residual (the SparseLU branch, :155-162). A non-SPD (CG) or singular
 * (BiCGStab) diagonal block, or no convergence, returns HDG_ESOLVE
 * (GlobalSolverError). d_uhat: nfc x d2.                                   */
typedef struct {
  int iterations;
  int converged;
  double relres;  /* ||r|| / ||r_0|| at exit */
  double asym;    /* sum |H_ij - H_ji| over the free block */
  double scale;   /* sum |H_ij| over the free block */
} hdg_solve_info;
int hdg_b200_solve_skeleton(hdg_ctx* ctx, int nfc, int d2, const int64_t* d_facebase,
                            const int* d_nbr, const double* d_vals, const double* d_b, int ndir,
                            const double* d_ub, double rtol, int maxit, double* d_uhat,
                            hdg_solve_info* info);

/* ------------------------------------------ error functionals (§8(f)4)
 * set_error_rule: tables of degree k and k+1 on tet/tri_rule(deg) (deg < 0:
 * 2k+4, postprocess.cpp:182-183); call after set_degree.
 * hdg_project replaces hdg_project (postprocess.cpp:95-176): the HDG
 * projection of (q, u) into P_k, d3 x nelt each; element matrices from the
 * level's tables, data moments on the error rule; HDG_ESINGULAR + element.
 * compute_errors replaces compute_errors (postprocess.cpp:178-250): relative
 * L2 errors of q, u, u* (d_ustar may be NULL), the skeleton error of uhat,
 * and the superconvergence measures against the HDG (or, tau == 0, L2)
 * projection and l2_project_skeleton. Fields must be CONST or PROGRAM.     */
typedef struct {
  double e_q, e_u, e_uhat, eps_u, eps_uhat, e_star;
} hdg_error_report;
int hdg_b200_set_error_rule(hdg_ctx* ctx, int deg);
int hdg_b200_hdg_project(hdg_ctx* ctx, int nelt, const hdg_geometry* g, hdg_field qx, hdg_field qy,
                         hdg_field qz, hdg_field u, double* d_qx, double* d_qy, double* d_qz,
                         double* d_u, int64_t* bad_element);
int hdg_b200_compute_errors(hdg_ctx* ctx, int nelt, const hdg_geometry* g, int nver,
                            const double* d_coords, int nfc, const int* d_faces, hdg_field qx,
                            hdg_field qy, hdg_field qz, hdg_field u, const double* d_uhat,
                            const double* d_qx, const double* d_qy, const double* d_qz,
                            const double* d_u, const double* d_ustar, hdg_error_report* out);

/* --------------------------------------------- K7: convection block
 * Replaces convection_bilinear_matrices (convdiff.cpp:5-28): vol d3 x d3,
 * dp 4d2 x d3, dd 4d2 x 4d2 per element (Batch3 layout).                   */
int hdg_b200_convection_block(hdg_ctx* ctx, int nelt, const hdg_geometry* g, hdg_field bx,
                              hdg_field by, hdg_field bz, double* d_vol, double* d_dp,
                              double* d_dd);

/* ----------------------------------- materialised element matrices
 * The ElementMatrixSet of build_element_matrices (element_matrices.hpp:86-93)
 * in Batch3 layout, for matrix-level parity; any output may be NULL.       */
typedef struct {
  double *Mkinv, *Mc, *Cx, *Cy, *Cz, *tauPP; /* d3 x d3 x nelt */
  double *tauDP, *nxDP, *nyDP, *nzDP;        /* 4d2 x d3 x nelt */
  double* tauDD;                             /* 4d2 x 4d2 x nelt */
  double* fvec;                              /* d3 x nelt */
} hdg_element_matrices;
int hdg_b200_element_matrices(hdg_ctx* ctx, int nelt, const hdg_geometry* g, hdg_field kappa,
                              hdg_field c, hdg_field f, hdg_element_matrices* out);

/* Physical images of the volume quadrature nodes (quad_points_physical,
 * element_matrices.cpp:66-70), nq x nelt each — for callers that sample
 * their own callbacks into HDG_FIELD_SAMPLED arrays. which: 0 = degree-k
 * rule, 1 = postprocess rule.                                              */
int hdg_b200_quad_points(hdg_ctx* ctx, int nelt, const hdg_geometry* g, int which, double* d_X,
                         double* d_Y, double* d_Z);

/* Per-kernel timing with CUDA events recorded on the context stream around each
 * stage. Stages: 0 geometry (K1), 1 node build (K2), 2 condense (K3),
 * 3 recover (K5), 4 scatter (K4), 5 postprocess (K6), 6 rescue screen (K3b,
 * kernels_rescue.cuh). stage_times waits for
 * the last recorded event of each stage and returns its duration in ms (-1 if
 * the stage did not run since the previous query).                        */
#define HDG_NSTAGES 7
int hdg_b200_set_timing(hdg_ctx* ctx, int enabled);
int hdg_b200_stage_times(hdg_ctx* ctx, double ms[HDG_NSTAGES]);

/* Program fields are compiled into K2 at run time (NVRTC, cached per field
 * set); disable to force the in-kernel field interpreter. jit_status returns
 * the last JIT failure ("" if none; on failure the interpreter runs).      */
int hdg_b200_set_jit(hdg_ctx* ctx, int enabled);
/* k = 1..3 recovery kernel: 3 = TMA-streamed cache records (default), 2 = one warp
 * per element with direct loads (equivalent; kept for comparison). */
int hdg_b200_set_recover_variant(hdg_ctx* ctx, int variant);
/* K3 (k >= 2) skips the operand blocks of the reference convection matrices
 * Chat_# (element_matrices.cpp:117-122) that vanish structurally in the
 * degree-graded orthonormal basis (rows of top-degree modes, the lower
 * triangle). set_degree verifies the pattern on the tables it builds and
 * otherwise (a tet rule too coarse for it) runs the dense kernel; this knob
 * forces the dense kernel (enabled = 0) for comparison. Call after
 * set_degree; returns the setting through *active if not NULL.            */
int hdg_b200_set_chat_sparsity(hdg_ctx* ctx, int enabled, int* active);
/* Singular elements. The condensation eliminates A1 by blocks (sweep
 * inverses of M and of its Schur complement S, no pivoting) and records their
 * extreme |pivots|. An element whose combined pivot ratio falls below
 * `screen` (default 1e-12), or whose pivots vanished or overflowed, is
 * re-solved by the reference's own path on the GPU: partial-pivot LU of A1
 * with the 1e-14 test of factor_checked (local_solver.cpp:50-57), C, Cf from
 * the LU solve (local_solver.cpp:71-100), recovery cache from partial-pivot
 * inverses. So indefinite (c < 0) and ill-conditioned elements get the
 * reference's verdict (HDG_ESINGULAR + lowest element) and values. screen >= 1
 * sends every element through that path (testing). rescued_elements returns
 * how many elements the last build_condense re-solved (synchronises).     */
int hdg_b200_set_rescue_screen(hdg_ctx* ctx, double screen);
int hdg_b200_rescued_elements(hdg_ctx* ctx, int64_t* count);
/* StabilizationField::allow_zero (element_matrices.hpp:24): build_condense
 * validates tau like StabilizationField::validate (element_matrices.cpp:38-46,
 * called at :287) before any factorisation: a negative tau(K,l) returns
 * HDG_EINVAL, and so does tau vanishing on all four faces of an element
 * unless allow_zero is set (the reference's study sets it for BDM,
 * study.cpp:18). Validation and the singular test are reported when
 * build_condense gets a non-NULL bad_element, otherwise by the next
 * hdg_b200_synchronize.                                                   */
int hdg_b200_set_tau_allow_zero(hdg_ctx* ctx, int enabled);
/* BDM variant (bdm_blocks, local_solver.cpp:65-69): the scalar space of the
 * local solve is truncated to its first d3 - d2 modes (P_{k-1}) and tau is
 * ignored (tauPP, tauDP and tauDD dropped); build_condense then returns the
 * condensed system of the BDM blocks and recover returns u zero-padded to
 * d3, as the reference. k = 1..5 (k = 0 is rejected as in the reference). */
int hdg_b200_set_bdm(hdg_ctx* ctx, int enabled);
const char* hdg_b200_jit_status(const hdg_ctx* ctx);

/* Block until the context's stream is idle and report any deferred error. */
int hdg_b200_synchronize(hdg_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* HDG_B200_H */
