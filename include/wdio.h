/*
 * wdio.h -- C ABI of libwdio.so: the corpus / stop-file / output formats of
 * the LDA path at configs[2]-[4] scale, host side.
 *
 * Paths are relative to the reference package source
 * (/root/reference/pkg/src/warpdraw).  Every call is thread-safe, takes
 * plain pointers and sizes, and returns 0 on success, 1 (WDIO_FALLBACK) when
 * the input needs the reference's own Python semantics (the Python wrapper
 * then re-reads it with that logic, so errors keep the reference's
 * messages), or -errno.  Buffers are caller-owned except the scan handles,
 * which wdio_release / wdio_release_floats free.
 */
#ifndef WDIO_H
#define WDIO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* lda.load_corpus (lda.py:66-110): text corpus from byte `start` (after the
 * optional "#M V" header) -> counts; wdio_fill_corpus writes offsets
 * int64 [n_docs + 1] and words int32 [n_tokens]. */
int wdio_scan_corpus(const char* path, int64_t start, int threads, void** handle, int64_t* n_docs,
                     int64_t* n_tokens, int32_t* max_word);
int wdio_fill_corpus(void* handle, int64_t* offsets, int32_t* words);
void wdio_release(void* handle);

/* np.loadtxt of the stop-inject file (cli.py:213-230, kernels.py:74-83):
 * one float64 per line. */
int wdio_scan_floats(const char* path, int threads, void** handle, int64_t* n);
int wdio_fill_floats(void* handle, double* out);
void wdio_release_floats(void* handle);

/* Binary CSR corpus (.wdc) reads: nbytes at file offset `off` into dst
 * (pinned host memory), split over `threads` concurrent preads. */
int wdio_pread(const char* path, int64_t off, int64_t nbytes, void* dst, int threads);

/* lda.save_corpus (lda.py:113-118). */
int wdio_write_corpus_text(const char* path, const int32_t* words, const int64_t* offsets, int64_t n_docs,
                           int64_t header_m, int64_t header_v, int threads);

/* cmd_lda's z.csv (cli.py:259-264) from CSR-order z (elem_bytes 2/4/8). */
int wdio_write_z_csv(const char* path, const void* z, int elem_bytes, const int64_t* offsets, int64_t n_docs,
                     int threads);

/* _write_matrix_csv (cli.py:232-236): rows of repr(float(x)) (elem_bytes 4/8,
 * row stride ld elements). */
int wdio_write_matrix_csv(const char* path, const void* m, int elem_bytes, int64_t rows, int64_t cols, int64_t ld,
                          int threads);

/* repr(float(x)) into out (>= 32 bytes); returns the length. */
int wdio_repr(double x, char* out);

#ifdef __cplusplus
}
#endif

#endif /* WDIO_H */
