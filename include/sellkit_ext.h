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
sellkit_error sellkit_ext_set_sync(int sync);
sellkit_error sellkit_ext_synchronize(void);
sellkit_error sellkit_ext_stream(void** stream);
sellkit_error sellkit_ext_device_info(int* device, int* num_sms, size_t* l2_bytes);

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

/* ------------------------------------------------------- dense matrices -- */
sellkit_error sellkit_ext_densemat_storage(const sellkit_densemat* m, void** data, sellkit_lidx* stride,
                                           int* order, int* device, int* on_device);
/* m(i, j) = U(-1,1) from splitmix64(seed ^ (i*ncols + j)), mapped by
 * (h >> 11) * 2^-53 * 2 - 1 (complex: re from seed, im from seed+1).
 * Row index i is the storage row. */
sellkit_error sellkit_ext_densemat_fill_hash(sellkit_densemat* m, uint64_t seed);

#if defined(SELLKIT_BUILD) && defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* SELLKIT_EXT_H */
