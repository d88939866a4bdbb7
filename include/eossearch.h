/* eossearch.h -- C ABI of the B200-native batched table lookup.
 *
 * The hot path of arXiv 2112.03229 ("vectorized search over small,
 * logarithmically distributed sorted tables", EOSPAC case study), rebuilt for
 * sm_100a.  Citations: P:<n> = line n of the paper text; the
 * readings R<n> are listed in DESIGN.md.
 *
 * Conventions for every call:
 *   - Returns eos_status (EOS_OK = 0) unless noted.  Argument errors are
 *     detected synchronously, before any device work is queued, and no
 *     output is written.  Asynchronous kernel faults surface as EOS_ERR_CUDA
 *     from a later call or at the caller's stream synchronisation.
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *     Device work is queued on it and the call returns without waiting
 *     (except the *_host entry points, see below).
 *   - "_dev" pointers are device memory of the device the handle was created
 *     on (any allocator: cudaMalloc, torch, ...), owned by the caller.
 *     "_host" pointers are host memory owned by the caller (pinned memory
 *     gives overlapped copies; pageable memory works, slower).
 *   - Any alignment is accepted (vectorised interior + scalar peel / tail).
 *   - count == 0 is an EOS_OK no-op; count must be <= 2^62.
 *   - Handles are immutable after create: concurrent calls on one handle
 *     from several host threads / streams are safe.  destroy must not race
 *     with in-flight work (it synchronises the device before freeing).
 */
#ifndef EOSSEARCH_H
#define EOSSEARCH_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define EOS_API __attribute__((visibility("default")))
#else
#define EOS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define EOS_MAX_TABLE 16384 /* table entries staged in shared memory (fp64) */
#define EOS_MAX_TABLE_TIERED (1 << 29) /* entries of a tiered table */
#define EOS_LEVELS_AUTO (-1)           /* eos_search_create_levels: choose the structure */
#define EOS_LEVELS_PACKED (-2)         /* eos_search_create_levels: packed nodes, the fewest levels that fit */
#define EOS_LEVELS_PACKED_DEPTH(d) (-16 - (d)) /* ... packed nodes, exactly d = 1..4 levels */
#define EOS_MAX_K 19        /* mantissa bits appended to the exponent hash */
#define EOS_K_AUTO (-1)     /* let eos_search_create_ex choose the hash */

/* Bin hash of the directory (eos_search_create_hash / eos_plan_table_hash). */
#define EOS_HASH_AUTO 0     /* choose kind and parameter by the cost rule */
#define EOS_HASH_EXPONENT 1 /* param = k: binary exponent + k mantissa bits */
#define EOS_HASH_LOG 2      /* param = |H|: logarithm hash with |H| bins (Eqs. 1-3) */
#define EOS_N_COUNTERS 8

typedef enum {
  EOS_OK = 0,
  EOS_ERR_NULL = 1,        /* a required pointer / handle is NULL */
  EOS_ERR_SIZE = 2,        /* n or count out of range */
  EOS_ERR_NONFINITE = 3,   /* a table / grid value is NaN or +-inf */
  EOS_ERR_UNSORTED = 4,    /* table not non-decreasing (axes: not strictly increasing) */
  EOS_ERR_DEVICE = 5,      /* no CUDA device, or current device differs from the handle's */
  EOS_ERR_CUDA = 6,        /* a CUDA runtime call failed (incl. earlier async faults) */
  EOS_ERR_NOMEM = 7,       /* host or device allocation failed */
  EOS_ERR_UNSUPPORTED = 8, /* valid request this build does not support (e.g. k > EOS_MAX_K) */
  EOS_ERR_ALIAS = 9        /* output overlaps an input */
} eos_status;

typedef struct eos_table_s* eos_table;
typedef struct eos_grid2d_s* eos_grid2d;

/* Description of a built table (see eos_plan_table for the meaning). */
typedef struct {
  int64_t n;           /* table entries */
  int32_t key_mode;    /* 0: X[0] >= 0, key = |bits| (sign masked); 1: negatives, order-preserving key */
  int32_t k;           /* exponent hash: mantissa bits appended (k = 0: the paper's exponent hash); log hash: -1 */
  int32_t bins;        /* B: number of bins of the directory */
  int32_t max_occ;     /* largest number of table entries in one bin */
  int32_t steps;       /* S = ceil(log2(max_occ + 1)): fixed in-bin search steps */
  int32_t base;        /* hb: key of the lowest binned entry (aligned for the exponent hash) */
  int64_t image_bytes; /* shared-memory image: X fp64[n] (16-B padded) + directory u32[B] */
  int32_t device;      /* CUDA device of the handle (-1 for eos_plan_table) */
  int32_t ctas_per_sm; /* resident CTAs per SM of the search kernel (0 for plan) */
  int32_t hash_kind;   /* EOS_HASH_EXPONENT or EOS_HASH_LOG */
  uint32_t hash_mult;  /* M of the bin function below */
  /* tiered tables (eos_search_create_levels); levels == 0: the fields above
   * describe the whole table.  levels = D >= 1: the fields above (except n)
   * describe the shared-memory sample table T1 of top_n entries. */
  int32_t levels;      /* D: levels of nodes in global memory */
  int32_t node_width;  /* entries per node: 8 (8-ary key levels), 15 (packed), 0 (D = 0) */
  int64_t top_n;       /* n1 = ceil(n / 8^D), or ceil(n / 15) packed (image_bytes then counts
                        * 4 B, packed 2 B, per T1 entry) */
  int64_t level_bytes; /* device bytes of the levels (0 when D == 0) */
  /* lifting layout of the search kernel (ABI >= 3): directory entries of 2 B
   * (8 lo | occ) or 4 B (lo | occ << 16) in the image; fast_steps = the
   * fixed binary-lifting steps SF (0: all S steps in a runtime loop);
   * rare_steps = 1 if some bin holds >= 2^SF entries (its larger strides run
   * in a branch taken only by lanes that land in such a bin); ring_stages =
   * shared-memory stages of the streaming ring that large launches use (0:
   * none; eos_table_info only). */
  int32_t dir_entry_bytes;
  int32_t fast_steps;
  int32_t rare_steps;
  int32_t ring_stages;
  /* 2-D grid axes (eos_grid2d_info, ABI >= 5): how the kernels find a cell.
   * 0: through the directory above; 1: fitted log map -- the cell of x is
   * floor(a log2(x) + b) or the one below, a and b fitted to the axis at create
   * and checked at every node against the device's error bound (fp32,
   * lg2.approx); 2: the same with x in place of log2(x).  Maps are used when
   * both axes have one and the grid has bank-pinned records (not with
   * EOS_GRID_EXACT or EOS_GRID_DIRECTORY).  Same results either way.  0 for
   * 1-D tables. */
  int32_t cell_map;
} eos_table_info_t;

/* ---------------------------------------------------------------------------
 * Host-only planning (no device needed).
 *
 * eos_plan_table: validates a table and builds its exponent-hash bin
 * directory on the host, exactly as eos_search_create does, without touching
 * a device.  Used by the host-logic tests and for inspection.
 *   table_host : fp64[n], finite, non-decreasing (duplicates allowed, P:54-56
 *                "monotonically increasing"; -0.0 is canonicalised to +0.0)
 *   n          : 1 <= n <= EOS_MAX_TABLE (single-level tables; tiered ones:
 *                eos_plan_table_levels)
 *   k          : EOS_K_AUTO (any hash, see eos_plan_table_hash) or 0..EOS_MAX_K
 *                (exponent hash).  The bin of a value v is
 *                  b(v) = min( (max(key(v), hb) - hb) * M >> 32, B-1 ),
 *                key = the upper 32 bits of the IEEE-754 binary64 pattern,
 *                sign masked (mode 0): a fixed-point log2 of v.
 *                Exponent hash, M = 2^(12+k), hb aligned: b = the binary
 *                exponent plus the top k mantissa bits; k = 0 is exactly the
 *                paper's "Exponent Hash Search".  Logarithm hash,
 *                M = |H| 2^32 / span: |H| bins of equal width in log2 (Eqs.
 *                1-2, with the fixed-point log2; R22).
 *                Both are monotone, so every bin is a value interval and the
 *                answer never depends on the hash (R10/R13).
 *   dir_out    : optional (may be NULL) u32[cap]; receives the packed count
 *                directory, entry b = lo_b | (occ_b << 16) with
 *                lo_b = #{j : b(X_j) < b} and occ_b = #{j : b(X_j) == b}
 *                (P:150 and Eq. 3 re-formulated as counts, R10/R11).
 *                EOS_ERR_SIZE if cap < bins.
 *   info       : required, filled on success.
 * ------------------------------------------------------------------------- */
EOS_API eos_status eos_plan_table(const double* table_host, int64_t n, int32_t k, eos_table_info_t* info,
                          uint32_t* dir_out, int64_t cap);

/* Same with an explicit hash: kind EOS_HASH_AUTO (param ignored),
 * EOS_HASH_EXPONENT (param = k, 0..EOS_MAX_K) or EOS_HASH_LOG (param = |H|,
 * 1..2^22, the paper's H_size).  EOS_ERR_UNSUPPORTED if the image would not
 * fit in shared memory (> 200 KB). */
EOS_API eos_status eos_plan_table_hash(const double* table_host, int64_t n, int32_t kind, int64_t param,
                               eos_table_info_t* info, uint32_t* dir_out, int64_t cap);

/* ---------------------------------------------------------------------------
 * 1-D search ("Each algorithm takes a targets array (Y, of size m), and
 * a data array (X, of size n).  They perform a lower-bounds search, returning
 * an array of size m containing the index of the last element of X which is
 * less than or equal to each element of Y.  If X contains no such lower bound
 * for a given y in Y, the index 0 is chosen.  In the case that the element is
 * higher than the highest of X, the index n-1 is chosen.")
 *
 * Result per target y: idx = max(0, #{j : X[j] <= y} - 1) with IEEE "<=".
 * Hence ties -> that entry, duplicates -> the last one, y < X[0] -> 0,
 * NaN -> 0 (R4), +inf -> n-1, -inf -> 0, -0.0 == +0.0 (R6).
 * ------------------------------------------------------------------------- */

/* Setup once per table ("the search setup [is] performed only once"):
 * validates, builds the directory (k chosen by the cost model, EOS_K_AUTO)
 * and uploads the device image to the CURRENT CUDA device.  The table is
 * copied; the caller may free table_host on return.  1 <= n <=
 * EOS_MAX_TABLE_TIERED: tables above EOS_MAX_TABLE are tiered
 * (eos_search_create_levels with EOS_LEVELS_AUTO). */
EOS_API eos_status eos_search_create(const double* table_host, int64_t n, eos_table* out);

/* Same with an explicit k (EOS_K_AUTO or 0..EOS_MAX_K).  Results do not
 * depend on k (tested); only speed does. */
EOS_API eos_status eos_search_create_ex(const double* table_host, int64_t n, int32_t k, eos_table* out);

/* Same with an explicit hash (kind/param as in eos_plan_table_hash). */
EOS_API eos_status eos_search_create_hash(const double* table_host, int64_t n, int32_t kind, int64_t param,
                                  eos_table* out);

/* Tables of any size ("tables larger than smem"), 1 <= n <=
 * EOS_MAX_TABLE_TIERED.  Same result for every n and structure;
 * eos_search_create* call this with levels = EOS_LEVELS_AUTO, so they accept
 * the same n.
 *   levels = D: 0 = the whole table (and directory) in shared memory
 *     (n <= EOS_MAX_TABLE); D >= 1 (<= 5) = a two-level structure: the
 *     sample table T1[j] = X[j 8^D], j < n1 = ceil(n/8^D) <= 32768, held as
 *     the 32-bit keys of its values with its hash directory in shared
 *     memory (equal keys settled from the fp64 values), and D 8-ary levels in device
 *     memory, level d (d = D-1..0) holding F_d[j] = X[j 8^d] (fp64) and the
 *     32-bit order-preserving keys of those values (upper words), padded to
 *     n1 8^(D-d) entries (~1.7 x 8n bytes in all).  A level step reads the
 *     8 keys of a node (one 32-byte sector): c = #{t : key_t < key(y)}, and
 *     the node's fp64 values only when a key equals key(y); b = 8b + c - 1.
 *   levels = EOS_LEVELS_PACKED / EOS_LEVELS_PACKED_DEPTH(D): D = 1..4 levels
 *     of packed nodes (info: levels = D, node_width = 15; EOS_LEVELS_PACKED
 *     takes the smallest D that fits).  Node j of level d (d = D-1..0) is one
 *     32-byte sector covering X[15^(d+1) j + 15^d t], t = 0..14: the upper
 *     key word of its first entry rounded down to a multiple of 64 (B, its low
 *     6 bits a shift s) and the 16-bit residuals ((key64(entry t) - (B << 32))
 *     >> s) + 0x400, t = 1..14 (<= 0x7BFF: positive normal fp16 patterns;
 *     0x7C00 past n), key64 the 64-bit order-preserving key.  The sample table
 *     T1[j] = X[15^D j], j < n1 = ceil(n/15^D), is held in shared memory as the
 *     16 key bits below its bin bits (binned by the key's upper bits: the
 *     exponent hash with k = 20 - sh), with one 32-bit directory entry per pair
 *     of bins.  A lookup reads D nodes from L2; equal residuals are settled
 *     from the fp64 table in device memory (8n + ~34 n / 15 bytes in all).
 *     The sample table and its directory must fit 224 KB (D = 1: n up to
 *     ~1.5e6 for log-spread tables; D = 4 covers 2^29); otherwise
 *     EOS_ERR_UNSUPPORTED.  kind/param ignored.
 *     EOS_LEVELS_AUTO: D = 0 if n <= EOS_MAX_TABLE; else packed if n > 8 x
 *     32768 (where 8-ary levels need D >= 2), kind is EOS_HASH_AUTO and the
 *     packed depth that fits is not larger than the 8-ary depth; else the
 *     smallest 8-ary D with n1 <= 32768.
 *   kind/param: the hash of the shared-memory table (T1 when D >= 1), as in
 *     eos_search_create_hash.
 * Errors: EOS_ERR_SIZE (n out of range, or n1 too large for the given D:
 * > EOS_MAX_TABLE at D = 0, > 32768 at D >= 1), EOS_ERR_UNSUPPORTED (D > 5,
 * or a packed table that does not fit), EOS_ERR_NOMEM, plus the table errors
 * of eos_plan_table. */
EOS_API eos_status eos_search_create_levels(const double* table_host, int64_t n, int32_t levels,
                                            int32_t kind, int64_t param, eos_table* out);

/* Host-only planning of eos_search_create_levels (no device): fills info
 * (levels, top_n, level_bytes and the plan of the shared-memory table). */
EOS_API eos_status eos_plan_table_levels(const double* table_host, int64_t n, int32_t levels,
                                         int32_t kind, int64_t param, eos_table_info_t* info);

/* idx_out_dev[i] = lower bound of targets_dev[i], i in [0, count).
 *   targets_dev : fp64[count] device, read once (streaming)
 *   idx_out_dev : int32[count] device, written once; must not overlap targets
 * Asynchronous on `stream`. */
EOS_API eos_status eos_search(eos_table t, const double* targets_dev, int64_t count, int32_t* idx_out_dev,
                      void* stream);

/* eos_search plus optional validation counters.
 *   global_offset : global position of targets_dev[0] in a sharded stream
 *   counters_dev  : NULL, or device u64[8] that is ACCUMULATED into (+=,
 *                   modulo 2^64; zero it first):
 *       c0 #targets            c1 sum idx
 *       c2 sum mix64((global_position << 20) | idx)   (splitmix64 finalizer)
 *       c3 #(!(y >= X[0]))     c4 #(y > X[n-1])
 *       c5 #NaN                c6 #(y == X[idx])      c7 reserved (0)
 *   With counters_dev == NULL this is exactly eos_search. */
EOS_API eos_status eos_search_ex(eos_table t, const double* targets_dev, int64_t count,
                         int32_t* idx_out_dev, int64_t global_offset, uint64_t* counters_dev,
                         void* stream);

/* End-to-end form with HOST buffers: the targets are copied host->device in
 * chunks, searched, and the indices copied device->host, with the copies of
 * one chunk overlapping the search/copies of the next (two internal streams,
 * stream-ordered device staging allocated on `stream`).  Ordered after prior
 * work on `stream`; returns once the work is queued -- the indices are valid
 * after `stream` is synchronised.  Pinned host memory is required for
 * overlap (pageable memory is accepted). */
EOS_API eos_status eos_search_host(eos_table t, const double* targets_host, int64_t count,
                           int32_t* idx_out_host, void* stream);

/* Zero-setup search ("algorithms with zero setup
 * cost may be a better choice" when tables are not known in advance): no
 * handle, no host work.  Each CTA stages table_dev into shared memory and
 * builds a logarithm-hash count directory there (<= 8192 bins) before
 * streaming the targets.  Same results as eos_search.
 *   table_dev  : device fp64[n], 1 <= n <= 4096 (EOS_DIRECT_MAX_TABLE); it must
 *                be finite and non-decreasing -- this is checked on the device:
 *                if violated, *status_dev (nullable, device int32) receives
 *                EOS_ERR_NONFINITE / EOS_ERR_UNSORTED and the indices are
 *                unspecified.  May be written by earlier work on `stream`.
 *   other arguments as eos_search; asynchronous on `stream`. */
#define EOS_DIRECT_MAX_TABLE 4096
EOS_API eos_status eos_search_direct(const double* table_dev, int64_t n, const double* targets_dev,
                             int64_t count, int32_t* idx_out_dev, int32_t* status_dev,
                             void* stream);

EOS_API eos_status eos_table_info(eos_table t, eos_table_info_t* out);
EOS_API eos_status eos_search_destroy(eos_table t);

/* ---------------------------------------------------------------------------
 * 2-D EOSPAC-style interpolation (EOSPAC "provides interpolation
 * mechanisms" over a SESAME density x temperature table; the paper gives no
 * formula -- bilinear reading R14):
 *   i = lower bound of rho in R, j = lower bound of T in Tax
 *   ci = min(i, nR-2), cj = min(j, nT-2)
 *   tx = clamp01((rho - R[ci]) / (R[ci+1] - R[ci])), ty likewise (NaN kept)
 *   P = (1-tx)((1-ty) G[ci][cj] + ty G[ci][cj+1])
 *     +    tx ((1-ty) G[ci+1][cj] + ty G[ci+1][cj+1])
 * The weights may be evaluated as (rho - R[ci]) * (1/(R[ci+1] - R[ci])) with
 * the inverse precomputed at create (a few ulp of t from the divide): then
 * |P - formula| <= 1e-12 (|G00| + |G01| + |G10| + |G11|) of the cell corners,
 * i.e. within 1e-12 relative of P wherever the corners share a sign (the
 * BASELINE.json bar; grids whose P changes sign inside a cell can cancel, and
 * only the corner-scaled bound holds there).  EOS_GRID_EXACT divides exactly
 * as the formula does.
 * ------------------------------------------------------------------------- */

/* rho_host fp64[n_rho], T_host fp64[n_T]: strictly increasing, finite,
 * 2 <= n <= EOS_MAX_TABLE (negative axis values allowed: key mode 1);
 * P_host fp64[n_rho * n_T] row-major (T fastest), finite, n_rho n_T <=
 * EOS_MAX_GRID_CELLS.  P lives in shared memory when it fits (~200 KB with
 * the axes), else in device memory (see EOS_GRID_GLOBAL); the axes must fit
 * in shared memory (their images <= ~220 KB, else EOS_ERR_UNSUPPORTED).
 * Copied; bound to the current device.  A grid held in shared memory is also
 * kept in device memory as 32-byte cell quads (4x its size, <= ~1 MB): small
 * launches read their corners from there, so that their many CTAs do not each
 * stage the whole grid (same results). */
EOS_API eos_status eos_grid2d_create(const double* rho_host, int64_t n_rho, const double* T_host,
                             int64_t n_T, const double* P_host, eos_grid2d* out);

/* Interpolation variant of a grid (eos_grid2d_create_ex flags). */
#define EOS_GRID_LINEAR 0 /* bilinear in (rho, T) on P -- the formula above (R14) */
#define EOS_GRID_LOGLOG 1 /* bilinear in (ln rho, ln T) on ln P, P = exp(.) (R24):
                           *   tx = clamp01((ln rho - ln R[ci]) / (ln R[ci+1] - ln R[ci])), ty
                           *   likewise, P = exp(bilinear of ln G); exact for power laws.
                           *   Needs R, T, P > 0 (else EOS_ERR_UNSUPPORTED).  Brackets are
                           *   the same P:54 lower bounds.  Derivatives (eos_interp2d_ex):
                           *   dP/drho = P (d ln P / d ln rho) / rho on the cell. */
#define EOS_GRID_GLOBAL 2 /* flag bit: keep the grid in device memory even if it would fit in
                           * shared memory (grids whose P does not fit, n_rho n_T 8 B >
                           * ~200 KB, always live there) as cell quads (the 4 corners of a
                           * cell, 32 B, read with one load per pair; 4x the grid); the axes
                           * stay in shared memory (their images must fit: ~220 KB).  Same
                           * results. */
#define EOS_GRID_EXACT 4  /* flag bit: weights t = (x - X[c]) / (X[c+1] - X[c]) with the fp64
                           * divide, in the formula's order: P bit-identical to the formula
                           * evaluated in fp64 without contraction (linear grids).  Without it
                           * the default layout multiplies by a precomputed 1/(X[c+1] - X[c])
                           * (conflict-free bank-pinned cell records, no divides): a few ulp of
                           * t, i.e. |dP| <= ~1e-15 (|G| summed over the cell corners). */
#define EOS_GRID_DIRECTORY 8 /* flag bit: find the cells through the axis directories even
                            * where both axes follow a fitted map (eos_table_info_t
                            * cell_map); same results */
#define EOS_MAX_GRID_CELLS ((int64_t)1 << 28) /* n_rho n_T (EOS_ERR_SIZE above) */
EOS_API eos_status eos_grid2d_create_ex(const double* rho_host, int64_t n_rho, const double* T_host,
                                int64_t n_T, const double* P_host, int32_t flags, eos_grid2d* out);

/* P_out_dev[q] = interpolated value at (rho_dev[q], T_dev[q]);
 * irho_out_dev / iT_out_dev (nullable) receive the brackets i, j.
 * All device arrays of length count; outputs must not overlap inputs. */
EOS_API eos_status eos_interp2d(eos_grid2d g, const double* rho_dev, const double* T_dev, int64_t count,
                        double* P_out_dev, int32_t* irho_out_dev, int32_t* iT_out_dev,
                        void* stream);

/* eos_interp2d plus the partial derivatives of the interpolant (EOSPAC
 * returns F, dF/dx, dF/dy; reading R23):
 *   dP/drho = ((1-ty)(G[ci+1][cj]-G[ci][cj]) + ty(G[ci+1][cj+1]-G[ci][cj+1])) / (R[ci+1]-R[ci])
 *   dP/dT   = ((1-tx)(G[ci][cj+1]-G[ci][cj]) + tx(G[ci+1][cj+1]-G[ci+1][cj])) / (T[cj+1]-T[cj])
 * inside the axis range; 0 outside it (the clamped interpolant is constant
 * there); NaN for a NaN coordinate.  dPdrho_out_dev / dPdT_out_dev: device
 * fp64[count] or NULL (both NULL: exactly eos_interp2d). */
EOS_API eos_status eos_interp2d_ex(eos_grid2d g, const double* rho_dev, const double* T_dev, int64_t count,
                           double* P_out_dev, int32_t* irho_out_dev, int32_t* iT_out_dev,
                           double* dPdrho_out_dev, double* dPdT_out_dev, void* stream);

/* End-to-end form with host buffers (see eos_search_host): EOS_ERR_ALIAS if
 * an output overlaps an input or another output (checked before any copy). */
EOS_API eos_status eos_interp2d_host(eos_grid2d g, const double* rho_host, const double* T_host,
                             int64_t count, double* P_out_host, int32_t* irho_out_host,
                             int32_t* iT_out_host, void* stream);

/* info of the two axis tables (either pointer may be NULL) */
EOS_API eos_status eos_grid2d_info(eos_grid2d g, eos_table_info_t* rho_info, eos_table_info_t* T_info);
EOS_API eos_status eos_grid2d_destroy(eos_grid2d g);

/* ---------------------------------------------------------------------------
 * Misc
 * ------------------------------------------------------------------------- */
EOS_API const char* eos_status_str(eos_status s); /* static string, never NULL */
EOS_API int32_t eos_abi_version(void);            /* 5 */
/* Kernel launches issued by this library since load (all entry points). */
EOS_API int64_t eos_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* EOSSEARCH_H */
