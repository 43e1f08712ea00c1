/*
 * ntt_b200.h -- C ABI of the B200-native batched NTT engine (libntt_b200.so).
 *
 * The reference (nttkit, /root/reference/pkg/src/nttkit) is a pure-Python
 * package with no FFI: its drop-in surface is the functional API exported by
 * nttkit/__init__.py:27-43.  This header is the boundary *behind* that API:
 * paper_2405_11353_b200 (Python) binds it with ctypes exactly as
 * INTEGRATION.md shows, and any other host language can bind the same
 * symbols.  No torch types cross this boundary: plain integers, pointers and
 * sizes only.  Device pointers are CUDA device pointers; `stream` is a
 * cudaStream_t passed as void* (NULL = legacy default stream).
 *
 * Each entry point cites the reference function it replaces.
 */
#ifndef NTT_B200_H
#define NTT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NTT_B200_ABI_VERSION 1

/* Status codes: one per nttkit.errors class (errors.py:4-37), plus the
 * ValueError conditions of the reference and device-side failures. */
typedef enum {
    NTT_OK = 0,
    NTT_E_NOT_PRIME = 1,            /* errors.NotPrime            (modmath.py:68-69,93-94) */
    NTT_E_NOT_POWER_OF_TWO = 2,     /* errors.NotPowerOfTwo       (algorithms.py:46-49,333-334) */
    NTT_E_SIZE_NOT_SUPPORTED = 3,   /* errors.SizeNotSupported    (twiddle.py:45-46) */
    NTT_E_SIZE_MISMATCH = 4,        /* errors.SizeMismatch        (algorithms.py:41-43,428-429) */
    NTT_E_BAD_FACTORIZATION = 5,    /* errors.BadFactorization    (algorithms.py:346-347,361-362) */
    NTT_E_UNSUPPORTED_VARIANT = 6,  /* errors.UnsupportedVariant  (algorithms.py:331-332,410-411) */
    NTT_E_INVALID = 7,              /* ValueError: bad field/direction/inverse-table misuse
                                       (modmath.py:95-102, twiddle.py:63-64, algorithms.py:417-418) */
    NTT_E_CUDA = 8,                 /* CUDA runtime error (message in ntt_last_error) */
    NTT_E_NCCL = 9,                 /* collective failure on the distributed four-step path */
    NTT_E_NO_MEMORY = 10,
    NTT_E_INVALID_SIZE = 11,        /* errors.InvalidSize (cli.py:128-129) */
    NTT_E_NO_DEVICE = 12            /* no CUDA device: the engine has no CPU fallback */
} ntt_status_t;

/* Variant ids, in the order of algorithms.VARIANTS (algorithms.py:34). */
typedef enum {
    NTT_NAIVE = 0, NTT_DIT = 1, NTT_DIF = 2, NTT_FLAT = 3, NTT_PEASE = 4,
    NTT_PEASE_NC = 5, NTT_STOCKHAM = 6, NTT_SIXSTEP = 7
} ntt_variant_t;

/* twiddle.FORWARD / twiddle.INVERSE (twiddle.py:15-16). */
typedef enum { NTT_FORWARD = 0, NTT_INVERSE = 1 } ntt_direction_t;

/* ntt_exec flags. */
#define NTT_FLAG_SCALE 1u   /* multiply by n_inv (intt, algorithms.py:415-423); needs an INVERSE plan */
#define NTT_FLAG_HOST_ASYNC 2u  /* ntt_exec_host only: enqueue and return; completion is ordered on `stream`
                                   (synchronise it before touching h_out or reusing h_in; h_in must be
                                   ready on the host at the call).  Successive calls pipeline: the
                                   copy-out of one overlaps the copy-in of the next. */
#define NTT_FLAG_INDEPENDENT 4u /* ntt_exec: the caller guarantees that nothing it enqueued on `stream` since its
                                   previous call into this library on that stream produces this call's input or
                                   touches its output (inputs resident, or produced by earlier library calls).
                                   Consecutive single-pass calls with disjoint buffers may then overlap in time
                                   (programmatic dependent launch, dependency wait at the kernel's end; the
                                   library itself checks the buffers of its own calls that may still be running).
                                   Calls still take effect and complete in stream order. */

typedef struct ntt_plan_s* ntt_plan_t;

/* Validation of FieldParams(p, g, w) -- modmath.py:92-102. */
int ntt_field_check(uint64_t p, uint64_t g, int w_bits);
/* find_primitive_root -- modmath.py:63-77 (smallest generator). */
int ntt_find_primitive_root(uint64_t p, uint64_t* g_out);
/* root_of_unity -- twiddle.py:41-50. */
int ntt_root_of_unity(uint64_t p, uint64_t g, uint64_t n, uint64_t* omega_out);

/* build_table -- twiddle.py:57-88, computed natively on the host:
 * w_pow[i] = omega^i, w_shoup[i] = floor(w_pow[i] * 2^w / p), i < n;
 * for INVERSE also n_inv = n^(p-2) and its Shoup word.  Bit-identical to
 * the reference tables.  Arrays hold n uint64 entries each.  For w > 64
 * (accepted, like the reference, whenever p < 2^w) the Shoup words do not
 * fit 64 bits: w_shoup / n_inv_shoup are written as 0 and the caller derives
 * them (the device arithmetic never uses the plan's w). */
int ntt_table_build(uint64_t p, uint64_t g, int w_bits, uint64_t n, int direction,
                    uint64_t* w_pow, uint64_t* w_shoup, uint64_t* n_inv, uint64_t* n_inv_shoup);

/* make_plan -- algorithms.py:322-352.  Builds the device twiddle tables on
 * `device` (cached per (p,g,w,n,direction) like twiddle.py:65).  word_bytes
 * is the residue storage width of the buffers passed to ntt_exec: 4 (uint32,
 * needs p < 2^32) or 8 (uint64).  n1/n2 are the six-step split (0 = default
 * 2^ceil(L/2) x rest, algorithms.py:339-341); ignored by other variants. */
int ntt_plan_create(uint64_t p, uint64_t g, int w_bits, uint64_t n, int variant, int direction,
                    uint64_t n1, uint64_t n2, int word_bytes, int device, ntt_plan_t* plan_out);
int ntt_plan_destroy(ntt_plan_t plan);

typedef struct {
    uint64_t p, g, n, n1, n2;
    int w_bits, variant, direction, word_bytes, device;
    int field_kind;      /* 0: u32 p<2^31, 1: u32 p<2^32, 2: Goldilocks u64, 3: generic u64 */
    int passes;          /* HBM passes per transform (1 = shared-memory resident) */
    uint64_t n_inv, n_inv_shoup;
    uint64_t device_table_bytes;
} ntt_plan_info_t;
int ntt_plan_info(ntt_plan_t plan, ntt_plan_info_t* info);

/* run_plan / ntt / intt -- algorithms.py:402-434, batched: transforms
 * `batch` independent rows of n residues from d_in to d_out (device
 * pointers, row-major, contiguous, canonical residues in [0,p)).
 * Out-of-place; d_in == d_out is allowed.  Asynchronous on `stream`.
 * Inputs are never modified when d_in != d_out (the reference is pure,
 * algorithms.py:119,137,174,238,255,277). */
int ntt_exec(ntt_plan_t plan, const void* d_in, void* d_out, uint64_t batch, unsigned flags,
             void* stream);

/* Same with HOST buffers: H2D copy, transform, D2H copy, synchronise (the
 * path a list[int] / numpy caller takes; `stream` is unused -- the call is
 * synchronous -- unless flags has NTT_FLAG_HOST_ASYNC).  Large batches of shared-memory-resident plans are cut into
 * chunks pipelined over three internal streams so the copies in both
 * directions overlap the transforms (use pinned host memory for overlap). */
int ntt_exec_host(ntt_plan_t plan, const void* h_in, void* h_out, uint64_t batch, unsigned flags,
                  void* stream);

/* Batch scheduler over several devices -- the reference's batch path
 * (NttTransform._apply, estimator.py:61-65: one transform per row, "may run
 * fully in parallel") sharded with NO collective
 * (SURVEY.md sec.8e row 1): plans[i] (one plan per device, all of the same
 * field / size / variant / direction) transforms the contiguous row block
 * [batch*i/nplans, batch*(i+1)/nplans) of the HOST batch, every device's
 * copy-in / transform / copy-out pipeline running concurrently.  Synchronous
 * (returns when every row is back in h_out).  Flags: NTT_FLAG_SCALE. */
int ntt_exec_host_sharded(const ntt_plan_t* plans, int nplans, const void* h_in, void* h_out, uint64_t batch,
                          unsigned flags);

/* Bytes of device scratch ntt_exec needs for `batch` rows (0 for
 * shared-memory-resident plans); the library allocates and caches it. */
uint64_t ntt_plan_workspace_bytes(ntt_plan_t plan, uint64_t batch);

/* Distributed four-step of a six-step plan (algorithms.py:355-389 split
 * across `world` ranks).  Rank g owns input columns
 * i in [g*n1/G, (g+1)*n1/G) as the slab x_local[j][i_local] (n2 x n1/G) and
 * produces output columns k2 in [g*n2/G, ...) as out_local[k1][k2_local]
 * (n1 x n2/G), i.e. out[k1*n2 + k2].  step 0 (A): strided size-n2 DITs +
 * correction twiddles, written packed for the exchange as
 * send[h][i_local][k2_local] (h = destination rank); the caller then runs ONE
 * equal-split all-to-all (NCCL) of n1*n2/G^2 residues per peer; step 1 (B):
 * size-n1 DITs of the received recv[i][k2_local].  world must be a power of
 * two dividing n1 and n2. */
int ntt_sixstep_dist_step(ntt_plan_t plan, int step, int rank, int world, const void* d_in, void* d_out,
                          void* stream);

/* Step A of ntt_sixstep_dist_step with the exchange fused into its pack: the
 * per-destination blocks are stored straight into every rank's receive
 * buffer over NVLink (P2P stores; d_peer_recv[h] = rank h's receive buffer,
 * mapped into this process, e.g. torch symmetric memory buffer_ptrs), block h
 * at offset rank * n1*n2/G^2 residues -- the layout the all-to-all would have
 * produced, so step B (ntt_sixstep_dist_step, step 1) runs unchanged.  The
 * caller orders the ranks: a barrier before (no rank still reads its receive
 * buffer) and after (every block has landed) on the stream.  world <= 8.
 * Replaces the reference's serial ntt_sixstep (algorithms.py:355-389); no
 * reference counterpart for the exchange itself. */
int ntt_sixstep_dist_step_a_peer(ntt_plan_t plan, int rank, int world, const void* d_in, void* const* d_peer_recv,
                                 void* stream);

/* The second half of polymul.cyclic_mul_ntt (polymul.py:61-63, intt of the
 * pointwise product) as ONE call: d_out = intt(d_a .* d_b) for `batch` rows,
 * d_a / d_b the forward transforms of the operands.  `plan` must be an
 * inverse-direction plan.  Shared-memory-resident u32 plans (p < 2^30, N =
 * 2^9..2^13) run one fused kernel: the product is taken (Montgomery) as the
 * inverse's first group loads its input and n^-1 (times 2^32) is applied in
 * its last group's stores; every other plan runs the pointwise kernel + intt. */
int ntt_exec_pointwise_inverse(ntt_plan_t plan, const void* d_a, const void* d_b, void* d_out, uint64_t batch,
                               void* stream);

/* polymul.pointwise_mul -- polymul.py:45-49: c[i] = a[i]*b[i] mod p over
 * `count` residues (device pointers, plan's field/word). */
int ntt_pointwise_mul(ntt_plan_t plan, const void* d_a, const void* d_b, void* d_c,
                      uint64_t count, void* stream);

/* Structural counters (the B200 analogue of the reference's monkeypatch
 * tests, test_algorithms.py:116-141): incremented on the device by the
 * kernels themselves when enabled. */
typedef struct {
    uint64_t kernel_launches;     /* host-side count of engine kernel launches */
    uint64_t transforms;          /* rows transformed (device-side count) */
    uint64_t bitrev_passes;       /* bit-reverse permutations performed (per row) */
    uint64_t stage_copies;        /* Pease copy-back passes (per row); 0 for Pease_nc */
    uint64_t hbm_passes;          /* global-memory passes (per row) */
} ntt_counters_t;
int ntt_counters_enable(int enable);
int ntt_counters_read(ntt_counters_t* out);   /* synchronises the device */
int ntt_counters_reset(void);

/* Thread-local message for the last non-OK status. */
const char* ntt_last_error(void);
int ntt_abi_version(void);
/* Number of CUDA devices visible (0 on a CPU-only host). */
int ntt_device_count(void);

#ifdef __cplusplus
}
#endif
#endif /* NTT_B200_H */
