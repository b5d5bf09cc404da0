/*
 * gts_b200.h -- C ABI of the B200 stencil backend (drop-in for the
 * reference "gen" engine of stencilforge, arXiv 2311.08322 reproduction).
 *
 * Two kinds of shared objects implement this header:
 *
 *  1. libgts_b200.so (paper_2311_08322_b200/libgts_b200.so, built by
 *     __graft_entry__.build()): device, memory, stream and event services,
 *     the L2 flush used by the benchmark, and the halo pack/unpack kernels of
 *     the horizontal domain decomposition.  Every gts_b200_* function below.
 *
 *  2. One generated module per compiled stencil
 *     (<cache>/<fingerprint>/module.so), exporting GTS_B200_ENTRY below plus
 *     the four gts_b200_module_* functions.
 *
 * All functions return 0 on success, otherwise a cudaError_t value or one of
 * the GTS_B200_ERR_* codes; gts_b200_error_string() renders either.
 * No torch or C++ types cross this boundary.
 */
#ifndef GTS_B200_H
#define GTS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GTS_B200_ABI_VERSION 1

#define GTS_B200_ERR_K_MIN 1001       /* nk below the stencil's k_min (runtime.py:178-183) */
#define GTS_B200_ERR_ALLOC 1002       /* device arena allocation failed */
#define GTS_B200_ERR_UNSUPPORTED 1003 /* domain exceeds 2^30 points per axis */

/* ------------------------------------------------------------------------
 * Generated per-stencil entry.
 *
 * Replaces the reference's generated C entry
 *   void gts_run_<name>_<digest8>(int64 ni, nj, nk,
 *        {T* base, int64 s_i, s_j, s_k, int64 o_i, o_j, o_k} per api field,
 *        {double|float} per api scalar)
 * (stencilforge backends/gen.py:5-14 and 269-284, pkg/README.md:142-156;
 * bound by ctypes at gen.py:500-510) with:
 *   - device pointers (element strides / origins unchanged: element (i,j,k)
 *     is base[(i+o_i)*s_i + (j+o_j)*s_j + (k+o_k)*s_k]);
 *   - every scalar passed as double (the debug/vec engines' semantics,
 *     runtime.py:113; gen narrows f32 scalars, gen.py:276-277);
 *   - a trailing cudaStream_t (as void*); the call is asynchronous on it;
 *   - an int status instead of void.
 * Symbol name: gts_run_<stencil name>_<first 8 hex digits of the
 * fingerprint>, the gen mangling (gen.py:184-185).  Api pointers may alias.
 * ---------------------------------------------------------------------- */
typedef int (*gts_b200_entry_fn)(int64_t ni, int64_t nj, int64_t nk, ...);

/* Exported by every generated module (one static CUDA runtime per module). */
int gts_b200_module_set_device(int device);
int gts_b200_module_abi(void);
int gts_b200_module_release(void); /* frees the module's temporary arenas */
/* Kernels the module's entry has enqueued since load (fallback and helper
 * kernels included): the launch count bench.py reports. */
unsigned long long gts_b200_module_launch_count(void);

/* Optional per-module entries (named like the entry: gts_<kind>_<stencil
 * name>_<digest8>), present when the plan allows them:
 *   int gts_frame_<..>(int ilo, int ihi, int jlo, int jhi) -- the calling
 *       thread's next call runs only the frame tiles touching the band of
 *       width ilo / ihi / jlo / jhi along the low-i / high-i / low-j / high-j
 *       side (0: no band on that side, e.g. no neighbour there) (single fused
 *       PARALLEL kernel with idempotent recomputation);
 *   int gts_frametile_<..>(void)            -- the frame tile shape,
 *       rows << 16 | columns (sizes the complementary interior launch);
 *   int gts_mirror_<..>(int n, const int64_t* boxes) -- up to 8 halo-mirror
 *       boxes {i0, i1, j0, j1, base, s_i, s_j, s_k} for the calling thread's
 *       next call (gen_options mirror). */
typedef int (*gts_b200_frame_fn)(int ilo, int ihi, int jlo, int jhi);
typedef int (*gts_b200_frametile_fn)(void);
typedef int (*gts_b200_mirror_fn)(int n, const int64_t* boxes);

/* ------------------------------------------------------------------------
 * libgts_b200.so: runtime services.
 * ---------------------------------------------------------------------- */
int gts_b200_abi_version(void);
const char* gts_b200_error_string(int status);

int gts_b200_device_count(int* count);
/* NVTX ranges (header-only NVTX v3; no-ops without an attached tool): the
 * backend wraps each call in "b200 <stencil>" when GTS_B200_NVTX=1. */
int gts_b200_nvtx_push(const char* name);
int gts_b200_nvtx_pop(void);
int gts_b200_set_device(int device);
int gts_b200_get_device(int* device);
/* SM count, L2 bytes, compute capability (major*10+minor), HBM bytes. */
int gts_b200_device_info(int device, int* sm_count, int* l2_bytes, int* cc, size_t* hbm_bytes);

/* Device memory for field storages (replaces the host numpy buffers of
 * stencilforge storage.py:130-160 for device-resident fields). */
int gts_b200_malloc(void** ptr, size_t bytes);
int gts_b200_free(void* ptr);
int gts_b200_host_alloc(void** ptr, size_t bytes); /* pinned host memory */
int gts_b200_host_free(void* ptr);
/* page-lock / release an existing host buffer in place (mirror mode on the
 * reference's pageable storages); *registered = 0 if it was already pinned */
int gts_b200_host_register(void* ptr, size_t bytes, int* registered);
int gts_b200_host_unregister(void* ptr);
int gts_b200_memset(void* dst, int value, size_t bytes, void* stream);
int gts_b200_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream);
int gts_b200_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream);
int gts_b200_memcpy_d2d(void* dst, const void* src, size_t bytes, void* stream);

int gts_b200_stream_create(void** stream);
int gts_b200_stream_destroy(void* stream);
int gts_b200_stream_synchronize(void* stream);

int gts_b200_event_create(void** event);
int gts_b200_event_destroy(void* event);
int gts_b200_event_record(void* event, void* stream);
/* Plain record for cross-stream ordering: inside a stream capture it is an
 * intra-graph dependency (fork / join), not an event-record node. */
int gts_b200_event_record_dep(void* event, void* stream);
int gts_b200_event_synchronize(void* event);
int gts_b200_event_elapsed_ms(float* ms, void* start, void* end);

/* Evict L2 between timed iterations by writing a buffer of 2x the L2 size
 * on the given stream (SURVEY.md 8(d) timing protocol). */
int gts_b200_l2_flush(void* stream);
/* read-only eviction of the L2 (2x L2 bytes of loads; *bytes_read = that size):
 * appended to a kernel inside a profiled range so the range's DRAM write bytes
 * include the kernel's write-back */
int gts_b200_l2_evict_read(void* stream, size_t* bytes_read);
/* cudaProfilerStart / Stop: the profiled range of ncu --replay-mode range */
int gts_b200_profiler_start(void);
int gts_b200_profiler_stop(void);

/* Halo exchange support for the horizontal decomposition:
 * copy the box [i0,i0+ni) x [j0,j0+nj) x [k0,k0+nk) (storage coordinates,
 * element strides s_i/s_j/s_k, itemsize 4 or 8) of a strided field to / from
 * a contiguous buffer laid out (k, i, j) with j fastest. */
int gts_b200_pack_box(void* buf, const void* base, int64_t s_i, int64_t s_j, int64_t s_k,
                      int64_t i0, int64_t j0, int64_t k0, int64_t ni, int64_t nj, int64_t nk,
                      int itemsize, void* stream);
int gts_b200_unpack_box(void* base, const void* buf, int64_t s_i, int64_t s_j, int64_t s_k,
                        int64_t i0, int64_t j0, int64_t k0, int64_t ni, int64_t nj, int64_t nk,
                        int itemsize, void* stream);

/* Pipelined mirror mode (host FieldStorages): strided 2-D copies (``height``
 * rows of ``width`` bytes, pitches in bytes) and cross-stream ordering. */
int gts_b200_memcpy2d_h2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                          size_t height, void* stream);
int gts_b200_memcpy2d_d2h(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                          size_t height, void* stream);
int gts_b200_stream_wait_event(void* stream, void* event);

/* CUDA graphs: capture everything enqueued on ``stream`` between begin and
 * end (including generated-module entries and event records) into an
 * executable graph; replay it with one launch.  Used for multi-step loops
 * (the dycore step, the benchmark's timed region). */
int gts_b200_graph_begin(void* stream);
int gts_b200_graph_end(void* stream, void** exec);
int gts_b200_graph_launch(void* exec, void* stream);
int gts_b200_graph_destroy(void* exec);

/* Peer-memory halo exchange between the processes of one node (no NCCL on
 * the data path; decomp.PeerHaloExchanger).  Replaces the reference's absent
 * multi-process path (stencilforge SPEC.md:12) the way gen's entry
 * (gen.py:5-14) is replaced above: plain pointers, element strides, a stream.
 *  - ipc_get_handle / ipc_open / ipc_close: share a device allocation (64-B
 *    opaque handle + the byte offset of ``dptr`` from the allocation base,
 *    which ipc_open returns) with another process; opened with lazy peer
 *    access, so the pointer is P2P over NVLink / NVSwitch when the owner is
 *    another GPU;
 *  - copy_box: strided 3-D box -> strided 3-D box (dst / src point at the
 *    boxes' first elements; either side may be a peer pointer);
 *  - flag_signal: after everything earlier on ``stream``, store ``value`` to
 *    a (possibly peer) 64-bit flag with system-scope release;
 *  - flag_wait: ``stream`` waits until the flag is >= ``value``
 *    (system-scope acquire spin). */
int gts_b200_ipc_get_handle(const void* dptr, void* handle64, size_t* offset);
int gts_b200_ipc_open(const void* handle64, void** dptr);
int gts_b200_ipc_close(void* dptr);
int gts_b200_copy_box(void* dst, int64_t d_i, int64_t d_j, int64_t d_k, const void* src,
                      int64_t s_i, int64_t s_j, int64_t s_k, int64_t ni, int64_t nj, int64_t nk,
                      int itemsize, void* stream);
/* n (<= 8) flags at once: add 1 to each (system-scope release, after a
 * system fence), and wait until each reaches its next expected count (one
 * device-resident u64 per flag).  decomp.PeerFusedStep: one launch per step
 * for all neighbours. */
int gts_b200_flags_add(void* const* flags, int n, void* stream);
int gts_b200_flags_wait_next(void* const* flags, void* expected, int n, void* stream);

int gts_b200_flag_signal(void* flag, uint64_t value, void* stream);
/* Graph-capturable forms: flag_add adds 1 (system-scope release);
 * flag_wait_next bumps the consumer's own expected count (a 64-bit word in
 * device memory) and waits until the flag reaches it. */
int gts_b200_flag_add(void* flag, void* stream);
int gts_b200_flag_wait_next(const void* flag, void* expected, void* stream);
int gts_b200_flag_wait(const void* flag, uint64_t value, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GTS_B200_H */
