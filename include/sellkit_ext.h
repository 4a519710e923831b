/*
 * sellkit_ext.h -- additive B200 extensions to the reference C ABI (sellkit.h).
 * None of these exist in /root/reference/proj/include/sellkit.h; a program that
 * uses only sellkit.h never needs them.  SURVEY §8(b) "Additive extensions".
 */
#ifndef SELLKIT_EXT_H
#define SELLKIT_EXT_H

#include "sellkit.h"

#ifdef __cplusplus
extern "C" {
#endif

/* the library is built with hidden visibility; export exactly this API */
#if defined(SELLKIT_BUILD) && defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* ------------------------------------------------------ execution control --
 * sync = 1 (default): every call returns with its results visible (reference
 * semantics).  sync = 0: calls that do not return data to the host only
 * enqueue work on the library stream of their device; sellkit_ext_synchronize
 * waits for it.  The stream is a cudaStream_t (non-blocking). */
/* Message of the last call on this thread that returned an error ("" if none). */
const char* sellkit_ext_last_error(void);
sellkit_error sellkit_ext_set_sync(int sync);
sellkit_error sellkit_ext_synchronize(void);
sellkit_error sellkit_ext_stream(void** stream);
sellkit_error sellkit_ext_device_info(int* device, int* num_sms, size_t* l2_bytes);
/* Device memory the library keeps for reuse -- freed SELL storage (up to 1/8 of each
 * device's memory, reused by the next matrix of the same size) and the build-temporary
 * pool -- is returned to the driver on every device the library has used. */
sellkit_error sellkit_ext_release_cached(void);

/* ------------------------------------------------------------ CRS input -- */
/* Same as sellkit_crs_create with device (or any UVA) pointers. */
sellkit_error sellkit_ext_crs_create_device(sellkit_datatype dt, sellkit_gidx nrows, sellkit_gidx ncols,
                                            const sellkit_gidx* rowptr, const sellkit_gidx* col,
                                            const void* val, sellkit_crs** out);
/* Synthetic Laplacian stencils generated on the device:
 * points = 5: 2-D grid n x n, row = y*n + x, diagonal 4;
 * points = 7: 3-D grid n x n x n, row = (z*n + y)*n + x, diagonal 6;
 * neighbours -1, Dirichlet boundaries, columns ascending.  Only rows
 * [row_begin, row_end) are generated (global column indices), so each rank of
 * a distributed run can build its own block.  The result has
 * row_end - row_begin rows and n^2 (or n^3) columns. */
sellkit_error sellkit_ext_crs_stencil(sellkit_datatype dt, int points, sellkit_gidx n,
                                      sellkit_gidx row_begin, sellkit_gidx row_end, sellkit_crs** out);

/* Synthetic topological-insulator Hamiltonian: 4 orbitals per site
 * of a periodic Lx x Ly x Lz lattice, 13 nonzeros per row (on-site 2*G1 + V*I, six
 * hoppings (G1 -/+ i*G_{a+2})/2 with Dirac matrices G1 = tau_z(x)I, G2..G4 =
 * tau_x(x)sigma_{x,y,z}); V uniform in [-disorder/2, disorder/2) from a site hash.
 * Real datatypes get the real parts (same sparsity pattern).  Rows [row_begin, row_end). */
sellkit_error sellkit_ext_crs_ti(sellkit_datatype dt, sellkit_gidx lx, sellkit_gidx ly, sellkit_gidx lz,
                                 double disorder, sellkit_gidx row_begin, sellkit_gidx row_end, sellkit_crs** out);

/* -------------------------------------------------------- layout export -- */
sellkit_error sellkit_ext_mat_info(const sellkit_mat* m, int* chunk_height, int* sigma,
                                   sellkit_lidx* nrows_padded, sellkit_gidx* nchunks,
                                   sellkit_gidx* slots, int* cols_permuted);
/* Copies the SELL arrays to host buffers; any pointer may be NULL.
 * Sizes: row_perm_inv/row_perm [nrows], rowlen [nrows_padded], chunk_len
 * [nchunks], chunk_offset [nchunks+1], val/col [slots]. */
sellkit_error sellkit_ext_mat_export(const sellkit_mat* m, int32_t* row_perm_inv, int32_t* row_perm,
                                     int32_t* rowlen, int32_t* chunk_len, int64_t* chunk_offset,
                                     void* val, int32_t* col);

/* Sweep order for SpMV/SpMMV over the whole matrix (results are independent of it;
 * dot products may differ in the last bits): the stored rows are split into blocks
 * of block_rows (a multiple of 32) and swept in the order order[0..nblocks) (a
 * permutation of the block indices, nblocks = ceil(nrows_padded / block_rows)).
 * Used to keep the RHS reuse window small for matrices whose coupling distance is
 * long in row order (e.g. a pencil order over a 3-D lattice).
 * By default (and after order == NULL with block_rows == 0) the library picks the
 * order itself: when the coupling distance (median farthest |column - row|) times the
 * bytes a row streams exceeds half the L2, rows are swept in slabs walked along that
 * distance (SELLKIT_AUTO_ORDER=0 disables it).  order == NULL with block_rows > 0
 * forces the natural row order. */
sellkit_error sellkit_ext_mat_set_sweep_order(sellkit_mat* m, sellkit_lidx block_rows, const int32_t* order,
                                              sellkit_gidx nblocks);

/* Matrix-free operator (reference SellMatrix::apply_override, sellcs.hpp:116-119;
 * spmv.hpp:131-135): once set, sellkit_spmv on this matrix validates its arguments as
 * usual and then calls fn(y, x, opts, stream, ctx) instead of the built-in multiply.
 * y and x are in storage index space; opts is the caller's (or the defaults when the
 * caller passed NULL) and the override must honour the full fused contract.  `stream`
 * is the library's cudaStream_t of the matrix's device: device work the override
 * enqueues there (its own kernels, or library calls, which use that stream) is ordered
 * with the caller's other library calls, and sellkit_spmv synchronises it before
 * returning in the default synchronous mode.  A non-OK return is passed through.
 * fn == NULL removes the override. */
typedef sellkit_error (*sellkit_ext_apply_fn)(sellkit_densemat* y, const sellkit_densemat* x,
                                              const sellkit_spmv_opts* opts, void* stream, void* ctx);
sellkit_error sellkit_ext_mat_set_apply_override(sellkit_mat* m, sellkit_ext_apply_fn fn, void* ctx);

/* ------------------------------------------------------- dense matrices -- */
sellkit_error sellkit_ext_densemat_storage(const sellkit_densemat* m, void** data, sellkit_lidx* stride,
                                           int* order, int* device, int* on_device);
/* m(i, j) = U(-1,1) from splitmix64(seed ^ (i*ncols + j)), mapped by
 * (h >> 11) * 2^-53 * 2 - 1 (complex: re from seed, im from seed+1).
 * Row index i is the storage row. */
sellkit_error sellkit_ext_densemat_fill_hash(sellkit_densemat* m, uint64_t seed);

/* Timeline of the single-process distributed SpMV (sellkit_dist_spmv / _nocomm): with
 * trace on, each call records per rank 5 times in ms after the call's start --
 * exchange start and end (the rank's communication stream: packing its send lists into
 * the receivers' halo blocks), local-sweep start and end, remote-sweep end (the main
 * stream) -- and synchronises.  sellkit_ext_ctx_timeline copies min(*nvalues, 5 k)
 * values (rank-major) and sets *nvalues = 5 k; -1 marks an event not recorded (no
 * exchange, or a rank on another device than rank 0). */
sellkit_error sellkit_ext_ctx_set_trace(sellkit_ctx* ctx, int on);
sellkit_error sellkit_ext_ctx_timeline(const sellkit_ctx* ctx, double* out, int* nvalues);

/* ------------------------------------------ one process per GPU (NCCL) --
 * The multi-process counterpart of sellkit_ctx (which drives all ranks from one
 * process).  Each process owns rank `rank` of a BY_ROWS / BY_NNZ partition
 * (row_offsets[nranks+1], e.g. from sellkit_partition_compute) and passes the
 * CRS of ITS rows only, with global column indices (sellkit_ext_crs_stencil can
 * generate such a block on the device).  Setup protocol:
 *   1. sellkit_ext_rankctx_create             -> local/remote SELL parts on this GPU
 *   2. for q < recv_count: sellkit_ext_rankctx_recv -> (owner, global columns)
 *      the caller ships each request to its owner (any transport, e.g.
 *      torch.distributed); the owner calls sellkit_ext_rankctx_set_sends(to, cols)
 *   3. rank 0: sellkit_ext_nccl_unique_id; broadcast; all: sellkit_ext_rankctx_connect
 *   4. sellkit_ext_rank_spmv(y, rc, x, opts, z, nocomm) -- x, y, z hold this rank's
 *      rows in its stored (sigma-permuted) order (sellkit_ext_rankctx_row_perm).
 * The halo travels as NCCL send/recv pairs on a communication stream, overlapped
 * with the local sweep; dots are all-gathered and summed in rank order. */
typedef struct sellkit_rankctx sellkit_rankctx;
sellkit_error sellkit_ext_nccl_unique_id(void* id128);
sellkit_error sellkit_ext_rankctx_create(const sellkit_crs* rows, const sellkit_gidx* row_offsets, int nranks, int rank,
                                         int chunk_height, int sigma, sellkit_rankctx** out);
sellkit_error sellkit_ext_rankctx_recv_count(const sellkit_rankctx* rc, int* nowners);
sellkit_error sellkit_ext_rankctx_recv(const sellkit_rankctx* rc, int q, int* owner, sellkit_lidx* count,
                                       sellkit_gidx* cols);
sellkit_error sellkit_ext_rankctx_set_sends(sellkit_rankctx* rc, int to, const sellkit_gidx* cols, sellkit_lidx count);
sellkit_error sellkit_ext_rankctx_send(const sellkit_rankctx* rc, int s, int* to, sellkit_lidx* count,
                                       sellkit_lidx* local_rows);
sellkit_error sellkit_ext_rankctx_connect(sellkit_rankctx* rc, const void* id128);
/* CUDA-IPC transport (all ranks on one node; replaces step 3 above).  Each rank
 * exports its send slots (sized for blocks of up to max_width columns), its dot slot
 * and its flag block; blob == NULL queries *blob_bytes.  The caller all-gathers the
 * blobs (any transport) and passes all nranks of them, in rank order, to
 * sellkit_ext_rankctx_ipc_connect.  Halo slots are pulled by the receiver with
 * copy-engine peer copies; ranks signal each other with stream memory operations
 * (no kernel waits on another rank). */
sellkit_error sellkit_ext_rankctx_ipc_export(sellkit_rankctx* rc, int max_width, void* blob, size_t* blob_bytes);
sellkit_error sellkit_ext_rankctx_ipc_connect(sellkit_rankctx* rc, const void* blobs, size_t blob_bytes);
/* 0 = not connected (world size 1), 1 = NCCL, 2 = IPC */
sellkit_error sellkit_ext_rankctx_transport(const sellkit_rankctx* rc, int* transport);
/* graphs: 1 = capture each repeated step (same vectors, flags and scalars) in a CUDA
 * graph on its second use and replay it (default; SELLKIT_GRAPHS=0 disables),
 * 0 = always enqueue eagerly; reserve_sms: SMs the local sweep leaves free for the
 * concurrent halo pack (default SELLKIT_COMM_RESERVE_SMS or 0).  -1 keeps a setting. */
sellkit_error sellkit_ext_rankctx_set_options(sellkit_rankctx* rc, int graphs, int reserve_sms);
sellkit_error sellkit_ext_rank_spmv(sellkit_densemat* y, sellkit_rankctx* rc, const sellkit_densemat* x,
                                    const sellkit_spmv_opts* opts, sellkit_densemat* z, int nocomm);
sellkit_error sellkit_ext_rankctx_stats(const sellkit_rankctx* rc, uint64_t* bytes, uint64_t* msgs,
                                        sellkit_lidx* n_halo, uint64_t* boundary_rows, sellkit_gidx* local_nnz,
                                        sellkit_gidx* remote_nnz);
sellkit_error sellkit_ext_rankctx_row_perm(const sellkit_rankctx* rc, sellkit_lidx* row_perm);
/* Destroy only after EVERY rank has finished its last sellkit_ext_rank_spmv (e.g. after a
 * barrier): the other ranks map this rank's IPC slots / share its NCCL communicator. */
void sellkit_ext_rankctx_destroy(sellkit_rankctx* rc);

/* Host-only planning of one rank (no GPU needed): the partition.hpp:136-220 split
 * metadata, for tests of the setup protocol on machines without a GPU. */
typedef struct sellkit_rankplan sellkit_rankplan;
sellkit_error sellkit_ext_rankplan_create(sellkit_datatype dt, const sellkit_gidx* rowptr, const sellkit_gidx* col,
                                          const void* val, sellkit_lidx nrows, const sellkit_gidx* row_offsets,
                                          int nranks, int rank, sellkit_rankplan** out);
sellkit_error sellkit_ext_rankplan_recv_count(const sellkit_rankplan* rp, int* nowners);
sellkit_error sellkit_ext_rankplan_recv(const sellkit_rankplan* rp, int q, int* owner, sellkit_lidx* count,
                                        sellkit_gidx* cols);
sellkit_error sellkit_ext_rankplan_set_sends(sellkit_rankplan* rp, int to, const sellkit_gidx* cols,
                                             sellkit_lidx count);
sellkit_error sellkit_ext_rankplan_nsends(const sellkit_rankplan* rp, int* nsends);
sellkit_error sellkit_ext_rankplan_send(const sellkit_rankplan* rp, int s, int* to, sellkit_lidx* count,
                                        sellkit_lidx* local_rows);
void sellkit_ext_rankplan_destroy(sellkit_rankplan* rp);

#if defined(SELLKIT_BUILD) && defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* SELLKIT_EXT_H */
