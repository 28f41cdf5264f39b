// cheb_logdet.cu -- host side of the C ABI (include/cheb_logdet.h): validation,
// fp64 coefficient routine, workspace planning, stream-ordered launch sequence,
// kernel accounting.  Device kernels live in cheb_kernels.cuh.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include "cheb_logdet.h"
#include "cheb_kernels.cuh"

using namespace chebld;

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CL_CUDA(call)                                                                 \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess)                                                        \
            return fail(CL_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_),    \
                        __FILE__, __LINE__);                                          \
    } while (0)

// ---- step-kernel profiling (CUDA events on the launching stream) ------------
struct Profiler {
    std::mutex mu;
    bool on = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[3];  // [0] single step, [1] B^T B spmm
                                                               // (Y = B w), [2] persistent (all n steps)
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pool;
    double ms[3] = {0.0, 0.0, 0.0};
    int64_t n[3] = {0, 0, 0};
} g_prof;

int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}
// schedule controls (process-wide; the CHEB_* env vars set the initial value)
std::atomic<int> g_persistent{env_int("CHEB_PERSISTENT", 1)};  // 0 off, 1 auto (default), 2 forced
std::atomic<int> g_small_tiles{env_int("CHEB_SMALL_TILES", 1)};  // 1 auto (default), 0 standard geometry
std::atomic<int> g_doubling{env_int("CHEB_DOUBLING", 0)};      // 0 off (default), 1 moment doubling
thread_local int g_last_schedule = -1;  // cheb_last_schedule(): 0 per-step, 1 persistent, 2 resident
std::atomic<int> g_resident{env_int("CHEB_RESIDENT", 1)};     // 0 off, 1 auto (default): shared-memory-resident kernel

struct ProfScope {
    cudaStream_t s;
    int kind;
    std::pair<cudaEvent_t, cudaEvent_t> pr{nullptr, nullptr};
    explicit ProfScope(cudaStream_t st, int k = 0) : s(st), kind(k) {
        std::lock_guard<std::mutex> lk(g_prof.mu);
        if (!g_prof.on) return;
        if (!g_prof.pool.empty()) {
            pr = g_prof.pool.back();
            g_prof.pool.pop_back();
        } else {
            cudaEventCreate(&pr.first);
            cudaEventCreate(&pr.second);
        }
        cudaEventRecord(pr.first, s);
    }
    ~ProfScope() {
        if (!pr.first) return;
        cudaEventRecord(pr.second, s);
        std::lock_guard<std::mutex> lk(g_prof.mu);
        g_prof.ev[kind].push_back(pr);
    }
};

int sm_count() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
}

constexpr int kMaxCtasPerSm = 8;  // partial buffers are sized for this

struct DevBuf {  // owning device allocation (freed on scope exit)
    void* p = nullptr;
    ~DevBuf() { if (p) cudaFree(p); }
};

// Grow-only device arenas reused across the synchronous entry points (cheb_logdet,
// cheb_logdet_host) of a host thread: repeated estimates do not pay cudaMalloc/cudaFree of a
// multi-GB workspace every call.  [0]: workspace + result buffers, [1]: the host operator's
// device copy.  cheb_release_cache() frees them.
struct Arena {
    int dev = -1;
    void* p = nullptr;
    size_t cap = 0;
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        dev = -1;
    }
    ~Arena() { release(); }
};
thread_local Arena g_arena[2];

int arena_get(int slot, size_t bytes, void** out) {
    Arena& A = g_arena[slot];
    int dev = 0;
    cudaGetDevice(&dev);
    if (A.p && (A.cap < bytes || A.dev != dev)) A.release();
    if (!A.p) {
        cudaError_t e = cudaMalloc(&A.p, bytes);
        if (e != cudaSuccess) {
            A.p = nullptr;
            return fail(CL_ENOMEM, "cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
        }
        A.cap = bytes;
        A.dev = dev;
    }
    *out = A.p;
    return CL_OK;
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

bool valid_k(int k) { return k == 8 || k == 16 || k == 32 || k == 64 || k == 128; }

// rows per tile: Geo<K, R4>::TILE; the workspace is planned for the larger of the two geometries
int tile_rows(int k, int r4 = CHEB_RPG) { return r4 * kThreads * 4 / k; }
int tile_rows_max(int k) { return tile_rows(k, std::max(CHEB_RPG, CHEB_RPG_DBL)); }

struct Layout {
    size_t misc, w0, w1, y, sbits, part, gpart, sbuf, ticket;
    size_t cv_meta, cv_tab, cv_dc, cv_vi;  // compressed gather matrix (csr / rank-1)
    size_t rp2, ci2, va2, u2, fcoef, cnt64, scan, total;
    size_t scan_bytes;
    int64_t rp2_len;
};

// Status word at the start of every cheb_moments workspace (workspace offset kStatusOff, see
// cheb_workspace_status): bit 0 = a spin wait of the persistent kernel gave up (timeout),
// bit 1 = a moment written by the last call is not finite; bit 8 (informational, not an error) =
// the per-step kernels read the compressed matrix copy.
constexpr size_t kStatusOff = 8;

// Workspace of cheb_moments for dimension d, gather-matrix nnz, probe block k.
Layout plan(int64_t d, int64_t nnz, int k, int kind, int sms) {
    Layout L{};
    size_t off = 0;
    L.misc = off; off += 256;  // [8] u32 status (kStatusOff), [16] persistent-kernel grid barrier
    const size_t wbytes = align256((size_t)d * k * sizeof(double));
    const int words = k >= 32 ? k / 32 : 1;
    const size_t maxgrid = (size_t)sms * kMaxCtasPerSm;
    const int64_t ntiles = (d + tile_rows_max(k) - 1) / tile_rows_max(k);
    L.w0 = off; off += wbytes;
    L.w1 = off; off += wbytes;
    L.y = off; if (kind == CL_OP_BTB) off += wbytes;
    L.sbits = off; off += align256((size_t)d * words * sizeof(uint32_t) + 16);
    // per-CTA partials: up to 3 channels (doubling + rank-1) x 2 step parities (persistent kernel)
    L.part = off; off += align256(3 * maxgrid * k * sizeof(double));
    // reduction-group sums: up to 3 channels x 2 step parities (persistent kernel)
    L.gpart = off; off += align256(6 * (maxgrid / 2 + 1) * k * sizeof(double));  // groups of >= 2 CTAs
    L.sbuf = off; off += align256(2 * (size_t)k * sizeof(double));
    L.ticket = off; off += 256;
    L.rp2_len = ntiles * tile_rows_max(k) + 2;
    L.rp2 = off; off += align256((size_t)L.rp2_len * sizeof(int64_t));
    // rows padded to a multiple of the gather chunk: at most (U - 1) extra entries per row
    // (a row with no stored diagonal gets one extra (i, -beta) entry: at most U more per row)
    const size_t pnnz = (size_t)nnz + (size_t)CHEB_NNZ_UNROLL * (size_t)d;
    L.ci2 = off; off += align256((pnnz + 8) * sizeof(int32_t));
    L.va2 = off; off += align256((pnnz + 4) * sizeof(double));
    L.cnt64 = off; off += align256(((size_t)d + 1) * sizeof(int64_t));  // padded row lengths
    L.scan_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, L.scan_bytes, (const int64_t*)nullptr, (int64_t*)nullptr, (int)(d + 1));
    L.scan = off; off += align256(L.scan_bytes);
    L.u2 = off; if (kind == CL_OP_CSR_RANK1 || kind == CL_OP_FAMILY) off += align256(((size_t)d + 2) * sizeof(double));
    // compressed copy (CV format, cv_values_kernel / cv_encode_kernel): U entries per row, 16 bytes
    // of tail padding for the last tile's bulk copies
    const bool cvk = kind == CL_OP_CSR || kind == CL_OP_CSR_RANK1;
    const size_t ucv = (size_t)CHEB_NNZ_UNROLL * (size_t)d;
    L.cv_meta = off; if (cvk) off += 256;
    L.cv_tab = off; if (cvk) off += align256(kCvSlots * sizeof(double));
    L.cv_dc = off; if (cvk) off += align256(ucv * 2 + 64);
    L.cv_vi = off; if (cvk) off += align256(ucv + 64);
    L.fcoef = off; if (kind == CL_OP_FAMILY) off += align256(3 * (size_t)k * sizeof(double));
    L.total = off;
    return L;
}

int64_t gather_nnz(const cl_operator* op) { return op->kind == CL_OP_BTB ? op->At.nnz : op->A.nnz; }

int check_csr(const cl_csr& A, const char* name) {
    if (A.n_rows < 0 || A.n_cols < 0 || A.nnz < 0)
        return fail(CL_EINVAL, "%s: negative dimension", name);
    if (A.n_rows > 0 && (!A.row_ptr || (A.nnz > 0 && (!A.col_idx || !A.val))))
        return fail(CL_EINVAL, "%s: NULL pointer", name);
    if (A.n_cols >= (int64_t(1) << 31) || A.n_rows >= (int64_t(1) << 31))
        return fail(CL_EDIM, "%s: dimension >= 2^31 (int32 column indices)", name);
    return CL_OK;
}

int check_op(const cl_operator* op) {
    if (!op) return fail(CL_EINVAL, "operator is NULL");
    if (op->kind != CL_OP_CSR && op->kind != CL_OP_CSR_RANK1 && op->kind != CL_OP_BTB && op->kind != CL_OP_FAMILY)
        return fail(CL_EINVAL, "unknown operator kind %d", op->kind);
    int rc = check_csr(op->A, "A");
    if (rc) return rc;
    if (op->A.n_rows == 0) return fail(CL_EDIM, "empty operator (d = 0)");
    if (op->A.n_rows != op->A.n_cols) return fail(CL_EDIM, "A must be square (%lld x %lld)",
                                                  (long long)op->A.n_rows, (long long)op->A.n_cols);
    if (op->kind == CL_OP_BTB) {
        if ((rc = check_csr(op->At, "At"))) return rc;
        if (op->At.n_rows != op->A.n_cols || op->At.n_cols != op->A.n_rows || op->At.nnz != op->A.nnz)
            return fail(CL_EDIM, "At is not shaped as the transpose of B");
    }
    if (op->kind == CL_OP_CSR_RANK1 && !std::isfinite(op->r1_c))
        return fail(CL_EINVAL, "rank-1 weight is not finite");
    return CL_OK;
}

int check_ab(double a, double b, int32_t degree) {
    if (!std::isfinite(a) || !std::isfinite(b) || !(a > 0.0) || !(b > a))
        return fail(CL_EINVAL, "need finite 0 < a < b (got a=%g b=%g)", a, b);
    if (degree < 0) return fail(CL_EINVAL, "degree < 0");
    return CL_OK;
}

// Tiles per CTA below which a step-kernel grid is shrunk (small operators: fewer CTAs mean a
// deeper per-CTA pipeline and cheaper grid-wide reductions/barriers).  CHEB_MIN_TILES tunes it.
int min_tiles_per_cta() {
    static int v = [] {
        const char* e = getenv("CHEB_MIN_TILES");
        const int x = e ? atoi(e) : 1;
        return x < 1 ? 1 : x;
    }();
    return v;
}

// Cap on resident CTAs per SM for the staged step kernels (CHEB_STEP_OCC; 0 = occupancy limit).
int step_occ_cap() {
    static int v = [] {
        const char* e = getenv("CHEB_STEP_OCC");
        return e ? atoi(e) : 0;
    }();
    return v;
}

template <typename Kern>
int grid_for(Kern kern, int64_t ntiles, int sms, size_t dyn_smem = 0) {
    int occ = 0;
    if (dyn_smem > 0) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, dyn_smem);
    if (dyn_smem > 0 && step_occ_cap() > 0 && occ > step_occ_cap()) occ = step_occ_cap();
    if (occ < 1) occ = 1;
    if (occ > kMaxCtasPerSm) occ = kMaxCtasPerSm;
    int64_t g = (int64_t)sms * occ;
    if (dyn_smem > 0) {  // staged step kernels: keep >= min_tiles_per_cta() tiles per CTA
        const int64_t cap = (ntiles + min_tiles_per_cta() - 1) / min_tiles_per_cta();
        if (g > cap) g = cap;
    }
    if (g > ntiles) g = ntiles;
    // staged step / persistent kernels: a multiple of the reduction group (cluster) size, so the
    // persistent kernel's clusters tile the grid and both schedules share one canonical order
    if (dyn_smem > 0 && g >= kRedGroup) g -= g % kRedGroup;
    return (int)(g < 1 ? 1 : g);
}

// ---- operator prep (once per cheb_moments call): scaled/padded gather matrix ---------
template <int MODE>
void run_prep(const cl_operator* op, double alpha, double beta, char* ws, const Layout& L,
              cudaStream_t st, int sms) {
    const cl_csr& G2 = (MODE == MODE_BTB) ? op->At : op->A;
    const int64_t d = G2.n_rows;
    int grid = (int)std::min<int64_t>((d + kThreads) / kThreads, (int64_t)sms * 8);
    if (grid < 1) grid = 1;
    // padded row pointer: lengths rounded up to the gather chunk, exclusive scan (CUB)
    prep_count_kernel<<<grid, kThreads, 0, st>>>(d, G2.row_ptr, G2.col_idx, MODE != MODE_BTB ? 1 : 0,
                                                 (int64_t*)(ws + L.cnt64));
    size_t sb = L.scan_bytes;
    cub::DeviceScan::ExclusiveSum(ws + L.scan, sb, (const int64_t*)(ws + L.cnt64), (int64_t*)(ws + L.rp2),
                                  (int)(d + 1), st);
    g_launches += 1;  // prep_count_kernel (the CUB scan kernels are library code, not counted)
    prep_kernel<MODE><<<grid, kThreads, 0, st>>>(
        d, G2.row_ptr, G2.col_idx, G2.val, alpha, beta, (int64_t*)(ws + L.rp2), L.rp2_len,
        (int32_t*)(ws + L.ci2), (double*)(ws + L.va2),
        MODE == MODE_RANK1 ? op->r1_u : nullptr,
        MODE == MODE_RANK1 || MODE == MODE_FAM ? (double*)(ws + L.u2) : nullptr);
    g_launches++;
}

// Schedule of one cheb_moments call (chosen on the host before any launch).
struct Schedule {
    bool persistent = false;  // all steps of a probe block in one persistent cooperative launch
    bool power = false;       // power basis (Taylor baseline): w_j = Ã w_{j-1}, every step "FIRST"
    bool doubling = false;    // moment doubling: ceil(n/2) applications of Ã give mu_0..mu_n
    bool vbits = false;       // per-step csr/rank-1: v = w_0 lives only as sign bits (steps 1, 2)
    bool small = false;       // 16-row tiles for the Algorithm-1 kernels (RP = 1)
    bool l2res = false;       // csr / rank-1 working set within half of L2 (persistent schedule's home)
    bool resident = false;    // shared-memory-resident kernel (cheb_resident_kernel), plan below
    bool cv = false;          // per-step kernels may use the compressed matrix (device-checked)
    int res_grid = 0, res_rg = 1, res_nr = 0, res_cap = 0;
    int res_maxc = 1;         // single-cluster geometry: co-resident clusters (probe blocks per launch)
    size_t res_smem = 0;
    int fam_kp = 0, fam_r = 0;  // family: probes per member per block, members with output rows
    int64_t fam_rstride = 0;    // family: doubles between consecutive members' mu rows
};

// Launch of one step-kernel variant.  The dynamic shared-memory opt-in is a per-device,
// per-function attribute, so it is set on every launch (a few hundred ns, host side only).
template <int K, int MODE, bool FIRST, bool DBL, int VB, int RP = 0>
void launch_step(int grid, size_t smem, cudaStream_t st, const StepArgs& a) {
    cudaFuncSetAttribute(cheb_step_kernel<K, MODE, FIRST, DBL, VB, RP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cheb_step_kernel<K, MODE, FIRST, DBL, VB, RP><<<grid, kThreads, smem, st>>>(a);
}

// Launch configuration of the persistent kernel: clusters of rg CTAs (attribute 0).
void cluster_config(cudaLaunchConfig_t* cfg, cudaLaunchAttribute* at, int grid, int rg, size_t smem,
                    cudaStream_t st, int threads = kThreads) {
    cfg->gridDim = dim3(grid);
    cfg->blockDim = dim3(threads);
    cfg->dynamicSmemBytes = smem;
    cfg->stream = st;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)rg;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg->attrs = at;
    cfg->numAttrs = 1;
}

// Grid and reduction-group (cluster) size of the persistent kernel.  After each step's barrier the
// rank-1 s_j is summed over the ng = G / RG group sums, so large clusters (few groups) pay; but
// clusters strand CTAs on GPCs of 16/18/20 SMs.  16 (non-portable), 8, 4 and 2 are tried, and the
// largest cluster whose co-resident grid is within 15 % of the best grid wins (configs[1], rank-1
// at 3 CTAs/SM: 8 -> 384 CTAs, 4 -> 416, 2 -> 440; 14.9 us per step at 8 vs 15.9 at 4).
template <typename Kern>
int persist_grid(Kern pk, int64_t ntiles, int sms, size_t smem, int* grid_out, int* rg_out) {
    const int g0 = grid_for(pk, ntiles, sms, smem);
    const int force_rg = env_int("CHEB_RG", 0);  // tuning: one cluster size only
    int gs[5] = {0, 0, 0, 0, 0}, rgs[5] = {16, 8, 4, 2, 1};
    int best = 0;
    for (int x = 0; x < 5; x++) {
        const int rg = rgs[x];
        if (force_rg && rg != force_rg) continue;
        const int r = red_group(g0, rg);
        if (r != rg && r != g0) continue;
        if (rg == 16) cudaFuncSetAttribute(pk, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        cluster_config(&cfg, at, g0 - g0 % r, r, smem, 0);
        int maxc = 0;
        if (cudaOccupancyMaxActiveClusters(&maxc, pk, &cfg) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        gs[x] = (int)std::min<int64_t>(g0 - g0 % r, (int64_t)maxc * r);
        best = std::max(best, gs[x]);
    }
    for (int x = 0; x < 5; x++) {
        if (gs[x] >= 1 && gs[x] >= 0.85 * best) {
            *grid_out = gs[x];
            *rg_out = red_group(gs[x], rgs[x]);
            return CL_OK;
        }
    }
    return fail(CL_ECUDA, "persistent kernel: no co-resident cluster configuration");
}

// ---- shared-memory-resident schedule (cheb_resident_kernel) ------------------------
// One CTA of kResThreads per SM, all dynamic shared memory (the staged-matrix capacity takes what
// the vectors leave).  A single cluster (16, else 8 CTAs) when its CTAs hold the whole probe block
// with at most CHEB_RES_SINGLE_MAX (default 8192) row-probes per CTA: no grid-wide barrier at all
// (configs[0]); otherwise clusters of 16/8/4/2 over the co-resident SMs, the largest cluster whose
// grid is within 15 % of the best (configs[1] at k <= 16).  false: the block does not fit.
template <int K, int MODE, bool DBL>
bool resident_plan(int64_t d, int64_t nnz, bool has_u, Schedule* fp) {
    auto kern = cheb_resident_kernel<K, MODE, DBL>;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    const size_t dyn_max = ((size_t)optin - fa.sharedSizeBytes) & ~size_t(127);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_max) != cudaSuccess ||
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    auto cap_for = [&](int64_t nr) -> int {  // staged nonzero capacity, -1: the vectors do not fit
        if (nr < 1 || nr > 65535) return -1;
        const ResLayout l0 = res_layout<K>((int)nr, 0, has_u);
        if (l0.total + 64 > dyn_max) return -1;
        return (int)(((dyn_max - l0.total - 64) / 12) & ~size_t(3));
    };
    const int force_rg = env_int("CHEB_RG", 0);
    const int64_t single_max = env_int("CHEB_RES_SINGLE_MAX", 8192);
    auto take = [&](int grid, int rg) {
        const int64_t nr = (d + grid - 1) / grid;
        fp->res_grid = grid;
        fp->res_rg = rg;
        fp->res_nr = (int)nr;
        // staged capacity: the expected padded slice (rows padded to the gather chunk, plus a
        // missing diagonal) with room to spare, not all of shared memory
        const int64_t want = nr * ((nnz + d - 1) / d + CHEB_NNZ_UNROLL);
        fp->res_cap = (int)std::min<int64_t>(cap_for(nr), (want + 3) & ~int64_t(3));
        fp->res_smem = res_layout<K>((int)nr, fp->res_cap, has_u).total;
        const int cap_env = env_int("CHEB_RES_CAP", -1);  // tests: force the unstaged-matrix path
        if (cap_env >= 0) fp->res_cap = std::min(fp->res_cap, cap_env & ~3);
        return true;
    };
    // one cluster of 16 (non-portable), else 8 CTAs
    for (int rg : {16, 8}) {
        if (force_rg && rg != force_rg) continue;
        const int64_t nr = (d + rg - 1) / rg;
        if (nr * K > single_max || cap_for(nr) < 0) continue;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        cluster_config(&cfg, at, rg, rg, dyn_max, 0, kResThreads);
        int maxc = 0;
        if (cudaOccupancyMaxActiveClusters(&maxc, kern, &cfg) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        if (maxc >= 1) {
            fp->res_maxc = env_int("CHEB_RES_MULTI", 1) ? maxc : 1;  // 0: one probe block per launch
            return take(rg, rg);
        }
    }
    // flat grid: one CTA per SM, every SM (no cluster stranding), at most kResThreads CTAs
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kResThreads, dyn_max) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    const int grid = std::min(occ * sm_count(), kResThreads);  // CTA p reduces probe p's moments
    if (grid >= 2 && grid >= K && cap_for((d + grid - 1) / grid) >= 0) return take(grid, 1);
    return false;
}

template <int K>
int resident_setup(const cl_operator* op, char* ws, const Layout& L, cudaStream_t st, int sms, Schedule* fp) {
    const int64_t d = op->A.n_cols;
    const bool has_u = op->r1_u != nullptr;
    const bool ok = op->kind == CL_OP_CSR
                        ? (fp->doubling ? resident_plan<K, MODE_CSR, true>(d, op->A.nnz, false, fp)
                                        : resident_plan<K, MODE_CSR, false>(d, op->A.nnz, false, fp))
                        : (fp->doubling ? resident_plan<K, MODE_RANK1, true>(d, op->A.nnz, has_u, fp)
                                        : resident_plan<K, MODE_RANK1, false>(d, op->A.nnz, has_u, fp));
    if (!ok) return CL_OK;
    fp->resident = true;
    uint8_t* exp = (uint8_t*)(ws + L.cnt64);  // the prep's row-length scratch is free again
    CL_CUDA(cudaMemsetAsync(exp, 0, (size_t)d, st));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((d + kThreads - 1) / kThreads, (int64_t)sms * 8));
    resident_prep_kernel<<<grid, kThreads, 0, st>>>(d, (const int64_t*)(ws + L.rp2), (int32_t*)(ws + L.ci2),
                                                    fp->res_nr, fp->res_rg, fp->res_grid == fp->res_rg ? 1 : 0, exp);
    g_launches++;
    if (getenv("CHEB_DEBUG"))
        fprintf(stderr, "[chebld] resident grid %d, clusters of %d, %d rows per CTA, cap %d nnz, smem %zu\n",
                fp->res_grid, fp->res_rg, fp->res_nr, fp->res_cap, fp->res_smem);
    return CL_OK;
}

// ---- compressed copy of the prepped gather matrix (CV format) --------------
// Launches the device check + encode after the prep when the per-step kernels' tile geometry can
// stage it (U * TILE % 16 == 0); the kernels read the verdict word and fall back to the plain copy.
// CHEB_CV=0 disables.  Graph-capturable (memsets and kernels only).
int cv_setup(int64_t d, int32_t probe_block, char* ws, const Layout& L, cudaStream_t st, int sms, Schedule* fp) {
    const int r4 = fp->small ? 1 : (fp->doubling ? CHEB_RPG_DBL : CHEB_RPG);  // the step kernels' geometry
    if (!CHEB_CV_KERNEL || probe_block > 16 || tile_rows(probe_block, r4) % 16 != 0 || env_int("CHEB_CV", 1) == 0)
        return CL_OK;  // (the kernels' CAN_CV rule)
    // meta = {ok = 1, count = 0} by memsets (no host source: the call stays graph-capturable)
    CL_CUDA(cudaMemsetAsync(ws + L.cv_meta, 0, 2 * sizeof(int32_t), st));
    CL_CUDA(cudaMemsetAsync(ws + L.cv_meta, 1, 1, st));
    CL_CUDA(cudaMemsetAsync(ws + L.cv_tab, 0xFF, kCvSlots * sizeof(double), st));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((d + kThreads - 1) / kThreads, (int64_t)sms * 8));
    cv_values_kernel<<<grid, kThreads, 0, st>>>((int64_t)CHEB_NNZ_UNROLL * d, (const double*)(ws + L.va2),
                                                (unsigned long long*)(ws + L.cv_tab), (int32_t*)(ws + L.cv_meta));
    cv_encode_kernel<<<grid, kThreads, 0, st>>>(d, (const int64_t*)(ws + L.rp2), (const int32_t*)(ws + L.ci2),
                                                (const double*)(ws + L.va2), (const unsigned long long*)(ws + L.cv_tab),
                                                (int16_t*)(ws + L.cv_dc), (uint8_t*)(ws + L.cv_vi),
                                                (int32_t*)(ws + L.cv_meta));
    g_launches += 2;
    fp->cv = true;
    return CL_OK;
}

// ---- one probe block: K1, then n x ([K3] K2) --------------------------------
// RP: tile geometry of the Algorithm-1 kernels (0: CHEB_RPG; 1: 16-row tiles, Schedule::small)
// nblk > 1 (single-cluster resident geometry only): nblk consecutive probe blocks of K probes in
// one launch, one cluster each; kvalid counts the probes of all of them.
template <int K, int MODE, int RP = 0>
int run_block(const cl_operator* op, double alpha, double beta, int32_t n, uint64_t seed,
              int64_t p0, int kvalid, char* ws, const Layout& L, double* mu_rows,
              int64_t mu_stride, cudaStream_t st, int sms, const Schedule& fp, int nblk = 1) {
    constexpr int R4S = RP ? RP : CHEB_RPG;
    constexpr int R4D = RP ? RP : CHEB_RPG_DBL;  // doubling kernels: same RP rule
    using G = Geo<K, R4S>;  // Algorithm-1 geometry; the doubling kernels use Geo<K, R4D>
    using GD = Geo<K, R4D>;
    using SL = StageLayout<K, MODE, false, R4S>;
    using SLD = StageLayout<K, MODE, false, R4D>;
    const int64_t d = op->A.n_cols;
    double* w[2] = {(double*)(ws + L.w0), (double*)(ws + L.w1)};
    double* y = (double*)(ws + L.y);
    uint32_t* sbits = (uint32_t*)(ws + L.sbits);
    double* sbuf = (double*)(ws + L.sbuf);

    int rc_persist = CL_OK;
    StepArgs a{};
    a.d = d;
    a.rp = (const int64_t*)(ws + L.rp2);
    a.ci = (const int32_t*)(ws + L.ci2);
    a.va = (const double*)(ws + L.va2);
    a.sbits = sbits;
    a.beta = beta;
    a.r1c_alpha = alpha * op->r1_c;
    a.r1u = ((MODE == MODE_RANK1 && op->r1_u) || MODE == MODE_FAM) ? (const double*)(ws + L.u2) : nullptr;
    a.fam_kp = MODE == MODE_FAM ? fp.fam_kp : 0;
    a.fam_r = fp.fam_r;
    a.fam_rstride = fp.fam_rstride;
    a.fam_coef = MODE == MODE_FAM ? (const double*)(ws + L.fcoef) : nullptr;
    a.part = (double*)(ws + L.part);
    a.gpart = (double*)(ws + L.gpart);
    a.ticket = (unsigned int*)(ws + L.ticket);
    a.mu_out = mu_rows;
    a.mu_stride = mu_stride;
    a.kvalid = kvalid;
    if (fp.cv) {
        a.cv_ok = (const int32_t*)(ws + L.cv_meta);
        a.cv_dc = (const int16_t*)(ws + L.cv_dc);
        a.cv_vi = (const uint8_t*)(ws + L.cv_vi);
        a.cv_tab = (const double*)(ws + L.cv_tab);
    }

    // several blocks per launch: their sign bits and s_0 in the exported-row buffers, which the
    // single-cluster geometry never uses (every gathered row is a cluster row)
    const int64_t sb_stride = ((int64_t)d * words_for(K) + 3) & ~int64_t(3);
    uint32_t* sb_multi = (uint32_t*)(ws + L.w0);
    double* s0_multi = (double*)(ws + L.w1);
    // K1
    for (int b = 0; b < nblk; b++) {
        constexpr int groups = kThreads / (K <= 64 ? K / 2 : K / 4);
        const int64_t niter = (d + groups - 1) / groups;
        constexpr size_t init_smem = red_scratch_bytes<K, MODE == MODE_RANK1 ? 2 : 1>();
        cudaFuncSetAttribute(probe_init_kernel<K, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)init_smem);
        const int grid = grid_for(probe_init_kernel<K, MODE>, niter, sms);
        a.mu_col = 0;
        a.s_next = nblk > 1 ? s0_multi + (size_t)b * K : sbuf;
        a.mu_out = mu_rows + (size_t)b * K * mu_stride;
        a.kvalid = std::min(K, kvalid - b * K);
        if (nblk > 1)
            probe_init_kernel<K, MODE><<<grid, kThreads, init_smem, st>>>(a, seed, (uint64_t)(p0 + (int64_t)b * K),
                                                                        nullptr, sb_multi + (size_t)b * sb_stride);
        else
            probe_init_kernel<K, MODE><<<grid, kThreads, init_smem, st>>>(a, seed, (uint64_t)p0,
                                                                        fp.vbits ? nullptr : w[0], sbits);
        g_launches++;
    }
    a.mu_out = mu_rows;
    a.kvalid = kvalid;
    if (n < 1) return CL_OK;

    if constexpr ((MODE == MODE_CSR || MODE == MODE_RANK1) && K <= 64) if (fp.resident) {
        ResArgs ra{};
        ra.g0 = w[0];
        ra.g1 = w[1];
        ra.n = fp.doubling ? (n + 1) / 2 : n;
        ra.nr = fp.res_nr;
        ra.cap = fp.res_cap;
        ra.power = fp.power ? 1 : 0;
        ra.exp = (const uint8_t*)(ws + L.cnt64);
        ra.gpart = (double*)(ws + L.gpart);
        ra.s_buf = nblk > 1 ? s0_multi : sbuf;
        ra.nblk = nblk;
        ra.sb_stride = sb_stride;
        if (nblk > 1) a.sbits = sb_multi;
        ra.bar_count = (unsigned int*)(ws + L.misc + 16);
        ra.err = (unsigned int*)(ws + L.misc + kStatusOff);
        a.rg = fp.res_rg;
        CL_CUDA(cudaMemsetAsync(ws + L.misc + 16, 0, 16, st));
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[2];
        cluster_config(&cfg, at, fp.res_grid * nblk, fp.res_rg, fp.res_smem, st, kResThreads);
        at[1].id = cudaLaunchAttributeCooperative;  // a single cluster is co-scheduled anyway
        at[1].val.cooperative = 1;
        // (CHEB_RES_NOCOOP=1: profiling only -- ncu cannot replay cooperative cluster launches; the
        // grid is the co-resident capacity, so the CTAs are co-scheduled in practice)
        cfg.numAttrs = fp.res_grid > fp.res_rg && !env_int("CHEB_RES_NOCOOP", 0) ? 2 : 1;
        ProfScope ps(st, 2);
        if (fp.doubling) CL_CUDA(cudaLaunchKernelEx(&cfg, cheb_resident_kernel<K, MODE, true>, a, ra));
        else CL_CUDA(cudaLaunchKernelEx(&cfg, cheb_resident_kernel<K, MODE, false>, a, ra));
        g_launches++;
        return CL_OK;
    }

    const int tile = fp.doubling ? GD::TILE : G::TILE;
    a.ntiles = (d + tile - 1) / tile;
    // dynamic shared memory: the staged tiles, reused as the reduction scratch at the end
    const size_t smem = std::max<size_t>(fp.doubling ? SLD::SMEM : SL::SMEM, red_scratch_bytes<K, 2>());  // persistent
    const size_t smem_step = std::max<size_t>(
        (size_t)kStepStages * (fp.doubling ? StageLayout<K, MODE, CHEB_DBL_STAGE_WC, R4D>::BYTES : SL::BYTES),
        red_scratch_bytes<K, 3>());  // cheb_step_kernel
    constexpr bool CAN_DBL = MODE != MODE_FAM;  // the family mode runs Algorithm 1 only
    int grid_first = grid_for(cheb_step_kernel<K, MODE, true, false, 0, RP>, a.ntiles, sms, smem_step);
    int grid_step = grid_for(cheb_step_kernel<K, MODE, false, false, 0, RP>, a.ntiles, sms, smem_step);
    if constexpr (CAN_DBL) {
        if (fp.doubling) {
            grid_first = grid_for(cheb_step_kernel<K, MODE, true, true, 0, RP>, a.ntiles, sms, smem_step);
            grid_step = grid_for(cheb_step_kernel<K, MODE, false, true, 0, RP>, a.ntiles, sms, smem_step);
        }
    }
    // L2-resident csr / rank-1 operators: the persistent schedule's grid and reduction groups
    // (clusters) are used by the per-step launches too, so both schedules reduce identically
    int grid_p = 0;
    a.rg = 0;  // default reduction groups (red_group(G))
    if constexpr (MODE == MODE_CSR || MODE == MODE_RANK1) if (fp.persistent || fp.l2res) {
        auto pkern = fp.doubling ? cheb_persist_kernel<K, MODE, true, RP> : cheb_persist_kernel<K, MODE, false, RP>;
        int rg = 1;
        if ((rc_persist = persist_grid(pkern, a.ntiles, sms, smem, &grid_p, &rg))) return rc_persist;
        a.rg = rg;
        if (!fp.persistent) grid_first = grid_step = grid_p;
        if (getenv("CHEB_DEBUG")) fprintf(stderr, "[chebld] persistent grid %d, reduction groups of %d\n", grid_p, rg);
    }
    int grid_spmm = 1;
    if (MODE == MODE_BTB) {
        const int64_t ng = (op->A.n_rows + SpmmGeo<K>::GROUPS - 1) / SpmmGeo<K>::GROUPS;
        grid_spmm = grid_for(spmm_kernel<K>, ng, sms);
    }
    // moment doubling (reading G25): steps j = 1..ceil(n/2); the epilogue of step j writes
    // mu_{2j-1} and mu_{2j} (indices <= n) from w_j^T w_{j-1} and w_j^T w_j
    const int32_t nsteps = fp.doubling ? (n + 1) / 2 : n;
    if constexpr (MODE == MODE_CSR || MODE == MODE_RANK1) if (fp.persistent) {
        auto pkern = fp.doubling ? cheb_persist_kernel<K, MODE, true, RP> : cheb_persist_kernel<K, MODE, false, RP>;
        PersistArgs pp{};
        pp.w0 = w[0];
        pp.w1 = w[1];
        pp.n = nsteps;
        pp.gpart = (double*)(ws + L.gpart);
        pp.s_buf = sbuf;
        pp.bar_count = (unsigned int*)(ws + L.misc + 16);
        pp.err = (unsigned int*)(ws + L.misc + kStatusOff);
        pp.power = fp.power ? 1 : 0;
        CL_CUDA(cudaMemsetAsync(ws + L.misc + 16, 0, 16, st));
        // clusters of a.rg CTAs (the reduction groups), all co-resident (cooperative launch)
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[2];
        cluster_config(&cfg, at, grid_p, a.rg, smem, st);
        at[1].id = cudaLaunchAttributeCooperative;
        at[1].val.cooperative = 1;
        cfg.numAttrs = 2;
        ProfScope ps(st, 2);
        CL_CUDA(cudaLaunchKernelEx(&cfg, pkern, a, pp));
        g_launches++;
        return CL_OK;
    }
    for (int32_t j = 1; j <= nsteps; j++) {
        const double* cur = w[(j - 1) & 1];
        double* nxt = w[j & 1];
        if (MODE == MODE_BTB) {
            ProfScope ps(st, 1);
            spmm_kernel<K><<<grid_spmm, kThreads, 0, st>>>(op->A.n_rows, op->A.row_ptr, op->A.col_idx,
                                                          op->A.val, cur, y);
            g_launches++;
        }
        a.xg = (MODE == MODE_BTB) ? y : cur;
        a.wcur = cur;
        a.wnext = nxt;
        a.s_cur = sbuf + ((j - 1) & 1) * K;
        a.s_next = sbuf + (j & 1) * K;
        a.mu_col = j;
        ProfScope ps(st);
        // steps 1 and 2 read v = w_0 from the sign bits when it was not materialised (fp.vbits);
        // same grids as the plain kernels, so the moments are bit-identical either way
        constexpr int V1 = MODE != MODE_BTB ? 1 : 0, V2 = MODE != MODE_BTB ? 2 : 0;
        const bool vb1 = fp.vbits && j == 1, vb2 = fp.vbits && j == 2 && !fp.power;
        bool done = false;
        if constexpr (CAN_DBL) {
            if (fp.doubling) {
                if (j == 1) {
                    if (vb1) launch_step<K, MODE, true, true, V1, RP>(grid_first, smem_step, st, a);
                    else launch_step<K, MODE, true, true, 0, RP>(grid_first, smem_step, st, a);
                } else {
                    if (vb2) launch_step<K, MODE, false, true, V2, RP>(grid_step, smem_step, st, a);
                    else launch_step<K, MODE, false, true, 0, RP>(grid_step, smem_step, st, a);
                }
                done = true;
            }
        }
        if (done) {
        } else if (j == 1 || fp.power) {  // power basis: w_j = Ã w_{j-1} (no w_{j-2} term), ping-pong
            if (vb1) launch_step<K, MODE, true, false, V1, RP>(grid_first, smem_step, st, a);
            else launch_step<K, MODE, true, false, 0, RP>(grid_first, smem_step, st, a);
        } else {
            if (vb2) launch_step<K, MODE, false, false, V2, RP>(grid_step, smem_step, st, a);
            else launch_step<K, MODE, false, false, 0, RP>(grid_step, smem_step, st, a);
        }
        g_launches++;
    }
    return CL_OK;
}

template <int K>
int run_block_mode(const cl_operator* op, double alpha, double beta, int32_t n, uint64_t seed,
                   int64_t p0, int kvalid, char* ws, const Layout& L, double* mu_rows,
                   int64_t mu_stride, cudaStream_t st, int sms, const Schedule& fp, int nblk = 1) {
    switch (op->kind) {
        case CL_OP_CSR:
            if (fp.small) return run_block<K, MODE_CSR, 1>(op, alpha, beta, n, seed, p0, kvalid, ws, L, mu_rows, mu_stride, st, sms, fp, nblk);
            return run_block<K, MODE_CSR>(op, alpha, beta, n, seed, p0, kvalid, ws, L, mu_rows, mu_stride, st, sms, fp, nblk);
        case CL_OP_CSR_RANK1:
            if (fp.small) return run_block<K, MODE_RANK1, 1>(op, alpha, beta, n, seed, p0, kvalid, ws, L, mu_rows, mu_stride, st, sms, fp, nblk);
            return run_block<K, MODE_RANK1>(op, alpha, beta, n, seed, p0, kvalid, ws, L, mu_rows, mu_stride, st, sms, fp, nblk);
        case CL_OP_FAMILY:
            if constexpr (K >= 16) {  // >= 2 probes per member of an 8-member block
                if (fp.small) return run_block<K, MODE_FAM, 1>(op, alpha, beta, n, seed, p0, kvalid, ws, L, mu_rows, mu_stride, st, sms, fp);
                return run_block<K, MODE_FAM>(op, alpha, beta, n, seed, p0, kvalid, ws, L, mu_rows, mu_stride, st, sms, fp);
            }
            return fail(CL_EINVAL, "family moments need probe_block >= 16");
        default:
            return run_block<K, MODE_BTB>(op, alpha, beta, n, seed, p0, kvalid, ws, L, mu_rows, mu_stride, st, sms, fp);
    }
}

void prep_mode(const cl_operator* op, double alpha, double beta, char* ws, const Layout& L,
               cudaStream_t st, int sms) {
    switch (op->kind) {
        case CL_OP_CSR: run_prep<MODE_CSR>(op, alpha, beta, ws, L, st, sms); break;
        case CL_OP_CSR_RANK1: run_prep<MODE_RANK1>(op, alpha, beta, ws, L, st, sms); break;
        case CL_OP_FAMILY: run_prep<MODE_FAM>(op, alpha, beta, ws, L, st, sms); break;
        default: run_prep<MODE_BTB>(op, alpha, beta, ws, L, st, sms); break;
    }
}

int pick_k(int64_t m) {
    // One block when m <= 64 (smallest k >= m: the matrix is read once per step);
    // otherwise blocks of 64 (measured faster than 128 on B200 at config 3).
    if (m > 32) return 64;
    if (m > 16) return 32;
    if (m > 8) return 16;
    return 8;
}

}  // namespace

// ============================================================================
extern "C" {

int cheb_version(void) { return 100; }

int cheb_release_cache(void) {
    for (auto& A : g_arena) A.release();
    return CL_OK;
}

const char* cheb_last_error(void) { return g_err.c_str(); }

int64_t cheb_launch_count(void) { return g_launches.load(); }

int cheb_profile_begin(void) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    for (int k = 0; k < 3; k++) {
        for (auto& p : g_prof.ev[k]) g_prof.pool.push_back(p);
        g_prof.ev[k].clear();
        g_prof.ms[k] = 0.0;
        g_prof.n[k] = 0;
    }
    g_prof.on = true;
    return CL_OK;
}

int cheb_profile_end(double* step_ms, int64_t* step_launches) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.on = false;
    for (int k = 0; k < 3; k++) {
        double tot = 0.0;
        for (auto& p : g_prof.ev[k]) {
            cudaError_t e = cudaEventSynchronize(p.second);
            if (e != cudaSuccess) return fail(CL_ECUDA, "event sync: %s", cudaGetErrorString(e));
            float ms = 0.f;
            cudaEventElapsedTime(&ms, p.first, p.second);
            tot += ms;
        }
        g_prof.ms[k] = tot;
        g_prof.n[k] = (int64_t)g_prof.ev[k].size();
        for (auto& p : g_prof.ev[k]) g_prof.pool.push_back(p);
        g_prof.ev[k].clear();
    }
    if (step_ms) *step_ms = g_prof.ms[0];
    if (step_launches) *step_launches = g_prof.n[0];
    return CL_OK;
}

int cheb_profile_spmm(double* ms, int64_t* launches) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    if (ms) *ms = g_prof.ms[1];
    if (launches) *launches = g_prof.n[1];
    return CL_OK;
}

int cheb_profile_persistent(double* ms, int64_t* launches) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    if (ms) *ms = g_prof.ms[2];
    if (launches) *launches = g_prof.n[2];
    return CL_OK;
}

int cheb_set_persistent(int32_t mode) {
    if (mode < 0 || mode > 2) return fail(CL_EINVAL, "persistent mode must be 0, 1 or 2");
    g_persistent = mode;
    return CL_OK;
}

int cheb_set_small_tiles(int32_t mode) {
    if (mode < 0 || mode > 1) return fail(CL_EINVAL, "small-tiles mode must be 0 or 1");
    g_small_tiles = mode;
    return CL_OK;
}

int cheb_get_small_tiles(void) { return g_small_tiles.load(); }

int cheb_set_doubling(int32_t on) {
    if (on < 0 || on > 1) return fail(CL_EINVAL, "doubling mode must be 0 or 1");
    g_doubling = on;
    return CL_OK;
}

int cheb_get_doubling(void) { return g_doubling.load(); }

int cheb_set_resident(int32_t mode) {
    if (mode < 0 || mode > 1) return fail(CL_EINVAL, "resident mode must be 0 or 1");
    g_resident = mode;
    return CL_OK;
}

int cheb_get_resident(void) { return g_resident.load(); }

int cheb_last_schedule(void) { return g_last_schedule; }

#if CHEB_RES_PROF
// timing builds only (not in the header): per-CTA phase cycles of the last resident launch
int cheb_res_prof_read(long long* out, int n) {
    CL_CUDA(cudaMemcpyFromSymbol(out, chebld::g_res_prof, sizeof(long long) * (size_t)std::min(n, 1024 * 8)));
    return CL_OK;
}
#endif

// Host fp64 coefficient routine: accumulate, node by node, f(x_k)
// times T_j(x_k) for all j with the scalar recurrence, then scale.
int cheb_coeffs_log(double a, double b, int32_t degree, double* c_out) {
    int rc = check_ab(a, b, degree);
    if (rc) return rc;
    if (!c_out) return fail(CL_EINVAL, "c_out is NULL");
    const int n = degree;
    std::vector<double> acc((size_t)n + 1, 0.0);
    const double half_w = 0.5 * (b - a), mid = 0.5 * (b + a);
    for (int k = 0; k <= n; k++) {
        const double x = std::cos(M_PI * (k + 0.5) / (n + 1.0));
        const double f = std::log(half_w * x + mid);
        double tm1 = 1.0, t = x;
        acc[0] += f;
        if (n >= 1) acc[1] += f * x;
        for (int j = 2; j <= n; j++) {
            const double tn = 2.0 * x * t - tm1;
            acc[j] += f * tn;
            tm1 = t;
            t = tn;
        }
    }
    const double s0 = 1.0 / (n + 1.0), s1 = 2.0 / (n + 1.0);
    for (int j = 0; j <= n; j++) {
        const double cj = (j == 0 ? s0 : s1) * acc[j];
        if (!std::isfinite(cj)) return fail(CL_ENONFINITE, "coefficient %d not finite", j);
        c_out[j] = cj;
    }
    return CL_OK;
}

size_t cheb_workspace_bytes(const cl_operator* op, int32_t probe_block) {
    if (check_op(op)) return 0;
    if (!valid_k(probe_block)) {
        fail(CL_EINVAL, "probe_block must be 8, 16, 32, 64 or 128 (got %d)", probe_block);
        return 0;
    }
    return plan(op->A.n_cols, gather_nnz(op), probe_block, op->kind, sm_count()).total;
}

namespace {
int moments_impl(const cl_operator* op, double alpha, double beta, bool power, int32_t degree,
                 int64_t probe_begin, int64_t probe_end, uint64_t seed, int32_t probe_block,
                 void* workspace, size_t ws_bytes, double* mu_out, void* stream);
}

int cheb_moments(const cl_operator* op, double a, double b, int32_t degree,
                 int64_t probe_begin, int64_t probe_end, uint64_t seed, int32_t probe_block,
                 void* workspace, size_t ws_bytes, double* mu_out, void* stream) {
    int rc;
    if ((rc = check_op(op))) return rc;
    if ((rc = check_ab(a, b, degree))) return rc;
    return moments_impl(op, 2.0 / (b - a), (b + a) / (b - a), false, degree, probe_begin, probe_end, seed,
                        probe_block, workspace, ws_bytes, mu_out, stream);
}

int cheb_power_moments(const cl_operator* op, double s, int32_t degree, int64_t probe_begin,
                       int64_t probe_end, uint64_t seed, int32_t probe_block, void* workspace,
                       size_t ws_bytes, double* mu_out, void* stream) {
    int rc;
    if ((rc = check_op(op))) return rc;
    if (!std::isfinite(s) || !(s > 0.0)) return fail(CL_EINVAL, "need finite s > 0");
    if (degree < 0) return fail(CL_EINVAL, "degree < 0");
    // A = I - M/s = alpha*M - beta*I with alpha = -1/s, beta = -1
    return moments_impl(op, -1.0 / s, -1.0, true, degree, probe_begin, probe_end, seed, probe_block,
                        workspace, ws_bytes, mu_out, stream);
}

int cheb_affine_power_moments(const cl_operator* op, double alpha, double beta, int32_t degree,
                              int64_t probe_begin, int64_t probe_end, uint64_t seed, int32_t probe_block,
                              void* workspace, size_t ws_bytes, double* mu_out, void* stream) {
    int rc;
    if ((rc = check_op(op))) return rc;
    if (!std::isfinite(alpha) || !std::isfinite(beta)) return fail(CL_EINVAL, "alpha/beta not finite");
    if (degree < 0) return fail(CL_EINVAL, "degree < 0");
    return moments_impl(op, alpha, beta, true, degree, probe_begin, probe_end, seed, probe_block, workspace,
                        ws_bytes, mu_out, stream);
}

namespace {
double unkey(unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double x;
    memcpy(&x, &b, sizeof(x));
    return x;
}
}  // namespace

int cheb_norm_bound(const cl_operator* op, double* s_out, void* stream) {
    int rc;
    if ((rc = check_op(op))) return rc;
    if (op->kind == CL_OP_FAMILY) return fail(CL_EINVAL, "family operators: use cheb_family_moments");
    if (!s_out) return fail(CL_EINVAL, "s_out is NULL");
    if (op->kind == CL_OP_BTB) {
        double ab[2];
        // ||B||_1 ||B||_inf bounds sigma_max(B)^2; Johnson's bound is not needed here
        cudaStream_t st = (cudaStream_t)stream;
        DevBuf buf;
        CL_CUDA(cudaMalloc(&buf.p, 3 * sizeof(unsigned long long)));
        unsigned long long init[3] = {~0ull, 0ull, 0ull};
        CL_CUDA(cudaMemcpyAsync(buf.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
        const int64_t d = op->A.n_rows;
        int grid = (int)std::min<int64_t>((d + kThreads - 1) / kThreads, (int64_t)sm_count() * 8);
        bounds_btb_kernel<<<grid, kThreads, 0, st>>>(d, op->A.row_ptr, op->A.col_idx, op->A.val,
                                                      op->At.row_ptr, op->At.col_idx, op->At.val,
                                                      (unsigned long long*)buf.p);
        g_launches++;
        CL_CUDA(cudaGetLastError());
        unsigned long long h[3];
        CL_CUDA(cudaMemcpyAsync(h, buf.p, sizeof(h), cudaMemcpyDeviceToHost, st));
        CL_CUDA(cudaStreamSynchronize(st));
        ab[1] = unkey(h[1]) * unkey(h[2]);
        *s_out = ab[1];
        return CL_OK;
    }
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf buf;
    CL_CUDA(cudaMalloc(&buf.p, 3 * sizeof(unsigned long long)));
    unsigned long long init[3] = {0ull, 0ull, ~0ull};
    CL_CUDA(cudaMemcpyAsync(buf.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
    const int64_t d = op->A.n_rows;
    int grid = (int)std::min<int64_t>((d + kThreads - 1) / kThreads, (int64_t)sm_count() * 8);
    const double* u = op->kind == CL_OP_CSR_RANK1 ? op->r1_u : nullptr;
    gershgorin_kernel<<<grid, kThreads, 0, st>>>(d, op->A.row_ptr, op->A.col_idx, op->A.val, u,
                                                  (unsigned long long*)buf.p);
    g_launches++;
    CL_CUDA(cudaGetLastError());
    unsigned long long h[3];
    CL_CUDA(cudaMemcpyAsync(h, buf.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    CL_CUDA(cudaStreamSynchronize(st));
    double s = unkey(h[0]);
    if (op->kind == CL_OP_CSR_RANK1) {
        const double umax = op->r1_u ? unkey(h[1]) : 1.0;
        s += std::fabs(op->r1_c) * umax * umax * (double)d;  // |c| |u_i| sum_j |u_j| <= |c| umax^2 d
    }
    *s_out = s;
    return CL_OK;
}

int cheb_gershgorin(const cl_csr* A, double* lo_hi, void* stream) {
    int rc;
    if (!A || !lo_hi) return fail(CL_EINVAL, "NULL pointer");
    if ((rc = check_csr(*A, "A"))) return rc;
    if (A->n_rows != A->n_cols || A->n_rows < 1) return fail(CL_EDIM, "A must be square and non-empty");
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf buf;
    CL_CUDA(cudaMalloc(&buf.p, 3 * sizeof(unsigned long long)));
    unsigned long long init[3] = {0ull, 0ull, ~0ull};
    CL_CUDA(cudaMemcpyAsync(buf.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
    const int64_t d = A->n_rows;
    int grid = (int)std::min<int64_t>((d + kThreads - 1) / kThreads, (int64_t)sm_count() * 8);
    gershgorin_kernel<<<grid, kThreads, 0, st>>>(d, A->row_ptr, A->col_idx, A->val, nullptr,
                                                  (unsigned long long*)buf.p);
    g_launches++;
    CL_CUDA(cudaGetLastError());
    unsigned long long h[3];
    CL_CUDA(cudaMemcpyAsync(h, buf.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    CL_CUDA(cudaStreamSynchronize(st));
    lo_hi[0] = unkey(h[2]);
    lo_hi[1] = unkey(h[0]);
    return CL_OK;
}

namespace {
int quadform_impl(const cl_csr* A, const double* x, double* out, bool split, void* stream) {
    int rc;
    if (!A || !x || !out) return fail(CL_EINVAL, "NULL pointer");
    if ((rc = check_csr(*A, "A"))) return rc;
    if (A->n_rows != A->n_cols || A->n_rows < 1) return fail(CL_EDIM, "A must be square and non-empty");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t d = A->n_rows;
    const int nout = split ? 2 : 1;
    const int grid = (int)std::min<int64_t>((d + kThreads - 1) / kThreads, (int64_t)sm_count() * 8);
    DevBuf buf;
    CL_CUDA(cudaMalloc(&buf.p, sizeof(double) * ((size_t)grid * nout + nout)));
    double* part = (double*)buf.p;
    if (split) quadform_kernel<true><<<grid, kThreads, 0, st>>>(d, A->row_ptr, A->col_idx, A->val, x, part);
    else quadform_kernel<false><<<grid, kThreads, 0, st>>>(d, A->row_ptr, A->col_idx, A->val, x, part);
    quadform_final_kernel<<<1, 32, 0, st>>>(part, grid, nout, part + (size_t)grid * nout);
    g_launches += 2;
    CL_CUDA(cudaGetLastError());
    CL_CUDA(cudaMemcpyAsync(out, part + (size_t)grid * nout, sizeof(double) * nout, cudaMemcpyDeviceToHost, st));
    CL_CUDA(cudaStreamSynchronize(st));
    return CL_OK;
}
}  // namespace

int cheb_quadform(const cl_csr* A, const double* x, double* out, void* stream) {
    return quadform_impl(A, x, out, false, stream);
}

int cheb_quadform_split(const cl_csr* A, const double* x, double* out2, void* stream) {
    return quadform_impl(A, x, out2, true, stream);
}

int cheb_family_gershgorin(const cl_csr* base, int32_t R, const double* theta, double* lo_hi, void* stream) {
    int rc;
    if (!base || !theta || !lo_hi) return fail(CL_EINVAL, "NULL pointer");
    if ((rc = check_csr(*base, "base"))) return rc;
    if (base->n_rows != base->n_cols || base->n_rows < 1) return fail(CL_EDIM, "base must be square and non-empty");
    if (R < 1) return fail(CL_EINVAL, "R < 1");
    for (int r = 0; r < R; r++)
        if (!std::isfinite(theta[r])) return fail(CL_EINVAL, "theta[%d] not finite", r);
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf buf;
    CL_CUDA(cudaMalloc(&buf.p, 3 * sizeof(unsigned long long) * R));
    std::vector<unsigned long long> init(3 * (size_t)R);
    for (int r = 0; r < R; r++) {
        init[3 * r] = 0ull;
        init[3 * r + 1] = 0ull;
        init[3 * r + 2] = ~0ull;
    }
    CL_CUDA(cudaMemcpyAsync(buf.p, init.data(), sizeof(unsigned long long) * init.size(), cudaMemcpyHostToDevice, st));
    const int64_t d = base->n_rows;
    const int grid = (int)std::min<int64_t>((d + kThreads - 1) / kThreads, (int64_t)sm_count() * 8);
    for (int r = 0; r < R; r++)
        gershgorin_kernel<<<grid, kThreads, 0, st>>>(d, base->row_ptr, base->col_idx, base->val, nullptr,
                                                      (unsigned long long*)buf.p + 3 * r, std::fabs(theta[r]));
    g_launches += R;
    CL_CUDA(cudaGetLastError());
    CL_CUDA(cudaMemcpyAsync(init.data(), buf.p, sizeof(unsigned long long) * init.size(), cudaMemcpyDeviceToHost, st));
    CL_CUDA(cudaStreamSynchronize(st));
    for (int r = 0; r < R; r++) {
        lo_hi[2 * r] = unkey(init[3 * r + 2]);
        lo_hi[2 * r + 1] = unkey(init[3 * r]);
    }
    return CL_OK;
}

int cheb_family_moments(const cl_csr* base, int32_t R, const double* theta, const double* ab, int32_t degree,
                        int64_t probe_begin, int64_t probe_end, uint64_t seed, int32_t probe_block,
                        void* workspace, size_t ws_bytes, double* mu_out, void* stream) {
    int rc;
    if (!base || !theta || !ab) return fail(CL_EINVAL, "NULL pointer");
    cl_operator fop{};
    fop.kind = CL_OP_FAMILY;
    fop.A = *base;
    if ((rc = check_op(&fop))) return rc;
    if (R < 1) return fail(CL_EINVAL, "R < 1");
    for (int r = 0; r < R; r++) {
        if (!std::isfinite(theta[r])) return fail(CL_EINVAL, "theta[%d] not finite", r);
        if ((rc = check_ab(ab[2 * r], ab[2 * r + 1], degree))) return rc;
    }
    if (probe_begin < 0 || probe_end <= probe_begin) return fail(CL_EINVAL, "need 0 <= probe_begin < probe_end");
    if (!valid_k(probe_block)) return fail(CL_EINVAL, "probe_block must be 8, 16, 32, 64 or 128");
    int rpad = 1;
    while (rpad < R) rpad *= 2;
    const int kp = probe_block / rpad;
    if (kp < 2) return fail(CL_EINVAL, "probe_block %d too small for %d family members (need >= 2 probes each)",
                            probe_block, R);
    if (!workspace || !mu_out) return fail(CL_EINVAL, "NULL workspace or mu_out");
    const int sms = sm_count();
    const Layout L = plan(base->n_cols, base->nnz, probe_block, CL_OP_FAMILY, sms);
    if (ws_bytes < L.total) return fail(CL_ENOMEM, "workspace too small: %zu < %zu", ws_bytes, L.total);
    if ((uintptr_t)workspace & 255) return fail(CL_EINVAL, "workspace must be 256-byte aligned");
    cudaStream_t st = (cudaStream_t)stream;
    char* ws = (char*)workspace;
    const int64_t stride = (int64_t)degree + 1, mrows = probe_end - probe_begin;
    CL_CUDA(cudaGetLastError());
    CL_CUDA(cudaMemsetAsync(ws + L.ticket, 0, 256, st));
    CL_CUDA(cudaMemsetAsync(ws + L.misc, 0, 256, st));
    prep_mode(&fop, 0.0, 0.0, ws, L, st, sms);
    // per column c: member r = c / kp (padding columns repeat the last member), its map of
    // [a_r, b_r] onto [-1, 1] and theta_r
    std::vector<double> coef(3 * (size_t)probe_block);
    for (int c = 0; c < probe_block; c++) {
        const int r = std::min(c / kp, R - 1);
        const double a = ab[2 * r], b = ab[2 * r + 1];
        const double alpha = 2.0 / (b - a), beta = (b + a) / (b - a);
        coef[c] = alpha;
        coef[probe_block + c] = beta;
        coef[2 * probe_block + c] = alpha * theta[r];
    }
    CL_CUDA(cudaMemcpyAsync(ws + L.fcoef, coef.data(), sizeof(double) * coef.size(), cudaMemcpyHostToDevice, st));
    Schedule fp;
    int l2 = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    const double wset = 2.0 * base->n_cols * probe_block * 8.0 + 12.0 * base->nnz + 8.0 * base->n_cols;
    fp.small = g_small_tiles.load() != 0 && (wset <= 0.5 * (double)l2 || probe_block <= 16);
    fp.vbits = env_int("CHEB_VBITS", 1) != 0;
    fp.fam_kp = kp;
    fp.fam_r = R;
    fp.fam_rstride = mrows * stride;
    for (int64_t p0 = probe_begin; p0 < probe_end; p0 += kp) {
        const int kvalid = (int)std::min<int64_t>(kp, probe_end - p0);
        double* rows = mu_out + (size_t)(p0 - probe_begin) * stride;
        switch (probe_block) {
            case 16: rc = run_block_mode<16>(&fop, 0.0, 0.0, degree, seed, p0, kvalid, ws, L, rows, stride, st, sms, fp); break;
            case 32: rc = run_block_mode<32>(&fop, 0.0, 0.0, degree, seed, p0, kvalid, ws, L, rows, stride, st, sms, fp); break;
            case 64: rc = run_block_mode<64>(&fop, 0.0, 0.0, degree, seed, p0, kvalid, ws, L, rows, stride, st, sms, fp); break;
            case 128: rc = run_block_mode<128>(&fop, 0.0, 0.0, degree, seed, p0, kvalid, ws, L, rows, stride, st, sms, fp); break;
            default: rc = fail(CL_EINVAL, "family moments need probe_block >= 16"); break;
        }
        if (rc) return rc;
    }
    {
        const int64_t nmu = (int64_t)R * mrows * stride;
        const int grid = (int)std::min<int64_t>((nmu + kThreads - 1) / kThreads, 64);
        moments_status_kernel<<<grid, kThreads, 0, st>>>((unsigned int*)(ws + L.misc + kStatusOff), mu_out, nmu,
                                                         fp.cv ? (const int32_t*)(ws + L.cv_meta) : nullptr);
        g_launches++;
    }
    CL_CUDA(cudaGetLastError());
    return CL_OK;
}

int cheb_taylor_coeffs(double s, int32_t degree, double* c_out) {
    if (!std::isfinite(s) || !(s > 0.0)) return fail(CL_EINVAL, "need finite s > 0");
    if (degree < 0 || !c_out) return fail(CL_EINVAL, "bad degree or NULL c_out");
    c_out[0] = std::log(s);  // log det M = d log s + log det(M/s), log det(M/s) = tr log(I - A)
    for (int32_t k = 1; k <= degree; k++) c_out[k] = -1.0 / (double)k;  // log(1-x) = -sum x^k/k
    return CL_OK;
}

namespace {
int moments_impl(const cl_operator* op, double alpha, double beta, bool power, int32_t degree,
                 int64_t probe_begin, int64_t probe_end, uint64_t seed, int32_t probe_block,
                 void* workspace, size_t ws_bytes, double* mu_out, void* stream) {
    int rc;
    if (op->kind == CL_OP_FAMILY) return fail(CL_EINVAL, "family operators: use cheb_family_moments");
    if (probe_begin < 0 || probe_end <= probe_begin)
        return fail(CL_EINVAL, "need 0 <= probe_begin < probe_end");
    if (!valid_k(probe_block)) return fail(CL_EINVAL, "probe_block must be 8, 16, 32, 64 or 128");
    if (!workspace || !mu_out) return fail(CL_EINVAL, "NULL workspace or mu_out");
    const int sms = sm_count();
    const Layout L = plan(op->A.n_cols, gather_nnz(op), probe_block, op->kind, sms);
    if (ws_bytes < L.total)
        return fail(CL_ENOMEM, "workspace too small: %zu < %zu", ws_bytes, L.total);
    if ((uintptr_t)workspace & 255) return fail(CL_EINVAL, "workspace must be 256-byte aligned");
    cudaStream_t st = (cudaStream_t)stream;
    char* ws = (char*)workspace;
    const int64_t stride = (int64_t)degree + 1;
    CL_CUDA(cudaGetLastError());
    CL_CUDA(cudaMemsetAsync(ws + L.ticket, 0, 256, st));
    CL_CUDA(cudaMemsetAsync(ws + L.misc, 0, 256, st));
    prep_mode(op, alpha, beta, ws, L, st, sms);
    Schedule fp;
    fp.power = power;
    fp.doubling = !power && g_doubling.load() == 1;
    if (op->kind != CL_OP_BTB) {
        // L2-resident working set (two probe-block buffers + matrix): the per-step launch and
        // drain gaps dominate, so run all steps in one launch; small tiles either way (the per-step
        // and persistent schedules keep one geometry, hence bit-identical moments)
        int l2 = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
        const double wset = 2.0 * op->A.n_cols * probe_block * 8.0 + 12.0 * op->A.nnz + 8.0 * op->A.n_cols;
        // 16-row-per-group tiles also pay for Algorithm 1 at k <= 16 (configs[3], k = 16: 1565 vs
        // 1608 ms per estimate), where a standard tile has 128+ rows
        fp.small = g_small_tiles.load() != 0 && (wset <= 0.5 * (double)l2 || (probe_block <= 16 && !fp.doubling));
        fp.l2res = wset <= 0.5 * (double)l2;
        if (g_persistent.load() > 0 && degree >= 1) fp.persistent = g_persistent.load() == 2 || fp.l2res;
        if (getenv("CHEB_DEBUG")) fprintf(stderr, "[chebld] L2=%d working set=%.0f\n", l2, wset);
    }
    // shared-memory-resident kernel: csr / rank-1 (Algorithm 1, moment doubling, power basis) when
    // a probe block fits in the SMs' shared memory; only in the automatic persistent mode
    if (op->kind != CL_OP_BTB && degree >= 1 && probe_block <= 64 && g_persistent.load() == 1 &&
        g_resident.load() > 0) {
        switch (probe_block) {
            case 8: rc = resident_setup<8>(op, ws, L, st, sms, &fp); break;
            case 16: rc = resident_setup<16>(op, ws, L, st, sms, &fp); break;
            case 32: rc = resident_setup<32>(op, ws, L, st, sms, &fp); break;
            default: rc = resident_setup<64>(op, ws, L, st, sms, &fp); break;
        }
        if (rc) return rc;
        if (fp.resident) fp.persistent = false;
    }
    g_last_schedule = fp.resident ? 2 : (fp.persistent ? 1 : 0);
    // per-step csr/rank-1: v = w_0 only as sign bits (CHEB_VBITS=0 disables)
    fp.vbits = !fp.persistent && !fp.resident && op->kind != CL_OP_BTB && env_int("CHEB_VBITS", 1) != 0;
    // per-step csr/rank-1: the compressed matrix copy, if the operator admits it (checked on the
    // device; the kernels fall back to the plain copy otherwise).  CHEB_CV=0 disables.
    if (!fp.persistent && !fp.resident && (op->kind == CL_OP_CSR || op->kind == CL_OP_CSR_RANK1))
        if ((rc = cv_setup(op->A.n_cols, probe_block, ws, L, st, sms, &fp))) return rc;
    if (getenv("CHEB_DEBUG"))
        fprintf(stderr, "[chebld] d=%lld nnz=%lld k=%d kind=%d persistent=%d doubling=%d small=%d\n",
                (long long)op->A.n_cols, (long long)op->A.nnz, probe_block, op->kind, (int)fp.persistent,
                (int)fp.doubling, (int)fp.small);
    // single-cluster resident geometry: up to res_maxc probe blocks run concurrently in one launch
    // (one cluster each; configs[0] at k = 16: 4 blocks in one launch), as many as the exported-row
    // buffers hold sign bits and s_0 for
    int64_t group = 1;
    if (fp.resident && fp.res_grid == fp.res_rg && fp.res_maxc > 1) {
        const int64_t wb = (int64_t)(L.w1 - L.w0);
        const int64_t sbs = (((int64_t)op->A.n_cols * words_for(probe_block) + 3) & ~int64_t(3)) * 4;
        group = std::min<int64_t>({(int64_t)fp.res_maxc, wb / sbs, wb / ((int64_t)probe_block * 8)});
        group = std::max<int64_t>(group, 1);
    }
    for (int64_t p0 = probe_begin; p0 < probe_end;) {
        const int64_t nb = std::min<int64_t>(group, (probe_end - p0 + probe_block - 1) / probe_block);
        const int kvalid = (int)std::min<int64_t>(probe_block * nb, probe_end - p0);
        const int nbi = (int)nb;
        double* rows = mu_out + (size_t)(p0 - probe_begin) * stride;
        const int64_t pb = p0;
        p0 += probe_block * nb;
        switch (probe_block) {
            case 8: rc = run_block_mode<8>(op, alpha, beta, degree, seed, pb, kvalid, ws, L, rows, stride, st, sms, fp, nbi); break;
            case 16: rc = run_block_mode<16>(op, alpha, beta, degree, seed, pb, kvalid, ws, L, rows, stride, st, sms, fp, nbi); break;
            case 32: rc = run_block_mode<32>(op, alpha, beta, degree, seed, pb, kvalid, ws, L, rows, stride, st, sms, fp, nbi); break;
            case 64: rc = run_block_mode<64>(op, alpha, beta, degree, seed, pb, kvalid, ws, L, rows, stride, st, sms, fp, nbi); break;
            default: rc = run_block_mode<128>(op, alpha, beta, degree, seed, pb, kvalid, ws, L, rows, stride, st, sms, fp); break;
        }
        if (rc) return rc;
    }
    // status epilogue: a timed-out spin wait poisons this call's moment rows with NaN (so every
    // finiteness check downstream fires); a non-finite moment sets status bit 1.
    // CHEB_INJECT_TIMEOUT=1 (tests only) raises bit 0 as a timed-out wait would: the call then
    // fails loudly (NaN moments, CL_ECUDA from cheb_logdet), it can never return wrong numbers.
    if (getenv("CHEB_INJECT_TIMEOUT")) CL_CUDA(cudaMemsetAsync(ws + L.misc + kStatusOff, 1, 1, st));
    {
        const int64_t nmu = (probe_end - probe_begin) * stride;
        const int grid = (int)std::min<int64_t>((nmu + kThreads - 1) / kThreads, 64);
        moments_status_kernel<<<grid, kThreads, 0, st>>>((unsigned int*)(ws + L.misc + kStatusOff), mu_out, nmu,
                                                         fp.cv ? (const int32_t*)(ws + L.cv_meta) : nullptr);
        g_launches++;
    }
    CL_CUDA(cudaGetLastError());
    return CL_OK;
}
}  // namespace

int cheb_finalize(const double* mu, const double* c, int64_t m, int32_t degree,
                  double* gamma_p, double* stats, void* stream) {
    if (!mu || !c || !gamma_p || !stats) return fail(CL_EINVAL, "NULL pointer");
    if (m < 1 || degree < 0) return fail(CL_EINVAL, "need m >= 1, degree >= 0");
    finalize_kernel<<<1, kThreads, 0, (cudaStream_t)stream>>>(mu, c, m, degree, gamma_p, stats);
    g_launches++;
    CL_CUDA(cudaGetLastError());
    return CL_OK;
}

int cheb_workspace_status(const void* workspace, uint32_t* status, void* stream) {
    if (!workspace || !status) return fail(CL_EINVAL, "NULL pointer");
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t h = 0;
    CL_CUDA(cudaMemcpyAsync(&h, (const char*)workspace + kStatusOff, sizeof(h), cudaMemcpyDeviceToHost, st));
    CL_CUDA(cudaStreamSynchronize(st));
    *status = h;
    return CL_OK;
}

namespace {

int logdet_device(const cl_operator* op, double a, double b, int32_t degree, int32_t num_probes,
                  uint64_t seed, int32_t probe_block, cl_result* out, cudaStream_t st) {
    const int k = probe_block ? probe_block : pick_k(num_probes);
    if (!valid_k(k)) return fail(CL_EINVAL, "probe_block must be 0, 8, 16, 32, 64 or 128");
    const size_t ws_bytes = plan(op->A.n_cols, gather_nnz(op), k, op->kind, sm_count()).total;
    const size_t mu_n = (size_t)num_probes * (degree + 1);
    const size_t aux_bytes = sizeof(double) * (mu_n + (degree + 1) + num_probes + 4);
    struct { void* p; } ws, aux;
    int rc0 = arena_get(0, align256(ws_bytes) + aux_bytes, &ws.p);
    if (rc0) return rc0;
    aux.p = (char*)ws.p + align256(ws_bytes);
    double* mu = (double*)aux.p;
    double* c = mu + mu_n;
    double* gp = c + degree + 1;
    double* stats = gp + num_probes;
    std::vector<double> ch((size_t)degree + 1);
    int rc = cheb_coeffs_log(a, b, degree, ch.data());
    if (rc) return rc;
    CL_CUDA(cudaMemcpyAsync(c, ch.data(), ch.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    rc = cheb_moments(op, a, b, degree, 0, num_probes, seed, k, ws.p, ws_bytes, mu, st);
    if (rc) return rc;
    rc = cheb_finalize(mu, c, num_probes, degree, gp, stats, st);
    if (rc) return rc;
    double hstats[3];
    unsigned int ferr = 0;
    CL_CUDA(cudaMemcpyAsync(hstats, stats, sizeof(hstats), cudaMemcpyDeviceToHost, st));
    CL_CUDA(cudaMemcpyAsync(&ferr, (char*)ws.p + kStatusOff, sizeof(ferr), cudaMemcpyDeviceToHost, st));
    if (out->per_probe)
        CL_CUDA(cudaMemcpyAsync(out->per_probe, gp, sizeof(double) * num_probes, cudaMemcpyDeviceToHost, st));
    if (out->moments)
        CL_CUDA(cudaMemcpyAsync(out->moments, mu, sizeof(double) * mu_n, cudaMemcpyDeviceToHost, st));
    CL_CUDA(cudaStreamSynchronize(st));
    out->logdet = hstats[0];
    out->stderr_ = hstats[1];
    out->num_probes = num_probes;
    out->degree = degree;
    out->probe_block = k;
    if (ferr & 1u) return fail(CL_ECUDA, "persistent-kernel grid wait timed out (CTAs not co-resident?)");
    if (hstats[2] != 1.0 || !std::isfinite(hstats[0]))
        return fail(CL_ENONFINITE, "non-finite estimate: [a,b]=[%g,%g] likely does not enclose the spectrum", a, b);
    return CL_OK;
}

}  // namespace

int cheb_logdet(const cl_operator* op, double a, double b, int32_t degree, int32_t num_probes,
                uint64_t seed, int32_t probe_block, cl_result* out) {
    auto t0 = std::chrono::steady_clock::now();
    int rc;
    if ((rc = check_op(op))) return rc;
    if (op->kind == CL_OP_FAMILY) return fail(CL_EINVAL, "family operators: use cheb_family_moments");
    if ((rc = check_ab(a, b, degree))) return rc;
    if (num_probes < 1) return fail(CL_EINVAL, "num_probes < 1");
    if (!out) return fail(CL_EINVAL, "out is NULL");
    cudaStream_t st;
    CL_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    rc = logdet_device(op, a, b, degree, num_probes, seed, probe_block, out, st);
    cudaStreamDestroy(st);
    out->elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return rc;
}

namespace {
// Device copy of a HOST operator in the calling thread's operator arena (slot 1), enqueued on st.
int upload_operator(const cl_operator* op, cl_operator* dop, cudaStream_t st) {
    *dop = *op;
    // one arena block holds the device copy of every operator array
    auto csr_bytes = [](const cl_csr& A) {
        return align256(sizeof(int64_t) * (A.n_rows + 1)) + align256(sizeof(int32_t) * A.nnz) +
               align256(sizeof(double) * A.nnz);
    };
    size_t need = csr_bytes(op->A);
    if (op->kind == CL_OP_BTB) need += csr_bytes(op->At);
    if (op->kind == CL_OP_CSR_RANK1 && op->r1_u) need += align256(sizeof(double) * op->A.n_cols);
    void* blk = nullptr;
    int rc;
    if ((rc = arena_get(1, need, &blk))) return rc;
    size_t used = 0;
    auto up = [&](const void* h, size_t bytes, const void** dptr) -> int {
        if (!h || bytes == 0) return CL_OK;
        char* d = (char*)blk + used;
        used += align256(bytes);
        CL_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
        *dptr = d;
        return CL_OK;
    };
    auto up_csr = [&](cl_csr& A) -> int {
        int r;
        if ((r = up(A.row_ptr, sizeof(int64_t) * (A.n_rows + 1), (const void**)&A.row_ptr))) return r;
        if ((r = up(A.col_idx, sizeof(int32_t) * A.nnz, (const void**)&A.col_idx))) return r;
        return up(A.val, sizeof(double) * A.nnz, (const void**)&A.val);
    };
    rc = up_csr(dop->A);
    if (!rc && dop->kind == CL_OP_BTB) rc = up_csr(dop->At);
    if (!rc && dop->kind == CL_OP_CSR_RANK1 && dop->r1_u)
        rc = up(dop->r1_u, sizeof(double) * dop->A.n_cols, (const void**)&dop->r1_u);
    return rc;
}
}  // namespace

int cheb_logdet_host(const cl_operator* op, double a, double b, int32_t degree, int32_t num_probes,
                     uint64_t seed, int32_t probe_block, cl_result* out) {
    auto t0 = std::chrono::steady_clock::now();
    int rc;
    if ((rc = check_op(op))) return rc;
    if (op->kind == CL_OP_FAMILY) return fail(CL_EINVAL, "family operators: use cheb_family_moments");
    if ((rc = check_ab(a, b, degree))) return rc;
    if (num_probes < 1) return fail(CL_EINVAL, "num_probes < 1");
    if (!out) return fail(CL_EINVAL, "out is NULL");
    cudaStream_t st;
    CL_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cl_operator dop;
    const double t_h2d = now_s();
    rc = upload_operator(op, &dop, st);
    if (getenv("CHEB_DEBUG")) {
        cudaStreamSynchronize(st);
        fprintf(stderr, "[chebld] host call: arena + H2D %.1f ms\n", (now_s() - t_h2d) * 1e3);
    }
    const double t_est = now_s();
    if (!rc) rc = logdet_device(&dop, a, b, degree, num_probes, seed, probe_block, out, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    if (getenv("CHEB_DEBUG")) fprintf(stderr, "[chebld] host call: estimate %.1f ms\n", (now_s() - t_est) * 1e3);
    out->elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return rc;
}

int cheb_moments_host(const cl_operator* op, double a, double b, int32_t degree, int64_t probe_begin,
                      int64_t probe_end, uint64_t seed, int32_t probe_block, double* mu_out) {
    int rc;
    if ((rc = check_op(op))) return rc;
    if ((rc = check_ab(a, b, degree))) return rc;
    if (probe_begin < 0 || probe_end <= probe_begin) return fail(CL_EINVAL, "need 0 <= probe_begin < probe_end");
    if (!valid_k(probe_block)) return fail(CL_EINVAL, "probe_block must be 8, 16, 32, 64 or 128");
    if (!mu_out) return fail(CL_EINVAL, "mu_out is NULL");
    cudaStream_t st;
    CL_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cl_operator dop;
    rc = upload_operator(op, &dop, st);
    const size_t ws_bytes = plan(op->A.n_cols, gather_nnz(op), probe_block, op->kind, sm_count()).total;
    const size_t mu_bytes = sizeof(double) * (size_t)(probe_end - probe_begin) * ((size_t)degree + 1);
    void* ws = nullptr;
    if (!rc) rc = arena_get(0, align256(ws_bytes) + mu_bytes, &ws);
    uint32_t status = 0;
    if (!rc) {
        double* mu = (double*)((char*)ws + align256(ws_bytes));
        rc = moments_impl(&dop, 2.0 / (b - a), (b + a) / (b - a), false, degree, probe_begin, probe_end, seed,
                          probe_block, ws, ws_bytes, mu, st);
        if (!rc) {
            cudaError_t e1 = cudaMemcpyAsync(&status, (char*)ws + kStatusOff, sizeof(status), cudaMemcpyDeviceToHost, st);
            cudaError_t e2 = cudaMemcpyAsync(mu_out, mu, mu_bytes, cudaMemcpyDeviceToHost, st);
            cudaError_t e3 = cudaStreamSynchronize(st);
            if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess)
                rc = fail(CL_ECUDA, "D2H of moments: %s",
                          cudaGetErrorString(e1 != cudaSuccess ? e1 : (e2 != cudaSuccess ? e2 : e3)));
        }
    }
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    if (rc) return rc;
    if (status & 1u) return fail(CL_ECUDA, "persistent-kernel grid wait timed out (CTAs not co-resident?)");
    if (status & 2u)
        return fail(CL_ENONFINITE, "non-finite moment: [a,b]=[%g,%g] likely does not enclose the spectrum", a, b);
    return CL_OK;
}

namespace {
// Eigen-decomposition of the symmetric tridiagonal matrix (diag d[0..n-1], off-diagonal e[0..n-2])
// by the implicit QL method with Wilkinson shifts, accumulating the eigenvectors in z (row-major
// n x n, z[r*n + c] = component r of eigenvector c).  d is overwritten by the eigenvalues.
int tridiag_ql(std::vector<double>& d, std::vector<double> e, std::vector<double>& z, bool vectors = true) {
    const int n = (int)d.size();
    z.assign(vectors ? (size_t)n * n : 0, 0.0);
    for (int i = 0; vectors && i < n; i++) z[(size_t)i * n + i] = 1.0;
    e.resize(n, 0.0);
    if (n > 0) e[n - 1] = 0.0;
    for (int l = 0; l < n; l++) {
        int iter = 0, m;
        do {
            for (m = l; m < n - 1; m++) {
                const double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
                if (std::fabs(e[m]) <= 1e-16 * dd) break;
            }
            if (m != l) {
                if (++iter > 60) return fail(CL_ENONFINITE, "tridiagonal QL did not converge");
                double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
                double r = std::hypot(g, 1.0);
                g = d[m] - d[l] + e[l] / (g + (g >= 0 ? r : -r));
                double s = 1.0, c = 1.0, p = 0.0;
                int i;
                for (i = m - 1; i >= l; i--) {
                    double f = s * e[i], b = c * e[i];
                    r = std::hypot(f, g);
                    e[i + 1] = r;
                    if (r == 0.0) {
                        d[i + 1] -= p;
                        e[m] = 0.0;
                        break;
                    }
                    s = f / r;
                    c = g / r;
                    g = d[i + 1] - p;
                    r = (d[i] - g) * s + 2.0 * c * b;
                    p = s * r;
                    d[i + 1] = g + p;
                    g = c * r - b;
                    for (int k = 0; vectors && k < n; k++) {
                        f = z[(size_t)k * n + i + 1];
                        z[(size_t)k * n + i + 1] = s * z[(size_t)k * n + i] + c * f;
                        z[(size_t)k * n + i] = c * z[(size_t)k * n + i] - s * f;
                    }
                }
                if (r == 0.0 && i >= l) continue;
                d[l] -= p;
                e[l] = g;
                e[m] = 0.0;
            }
        } while (m != l);
    }
    return CL_OK;
}
}  // namespace

extern "C++" {
namespace {
// ---- spectral interval (reading G26) ----------------------
// N Lanczos steps for the k probes of one block (columns of [d][k] buffers), on the device;
// hist receives alpha_j (row 2j) and beta_{j+1} (row 2j+1), j < N, k doubles per row.
template <int K>
int lanczos_block(const cl_operator* op, int N, uint64_t seed, int64_t p0, char* ws, size_t wbytes,
                  double* hist_d, cudaStream_t st, int sms) {
    const int64_t d = op->A.n_cols;
    double* Q = (double*)ws;
    double* Pb = (double*)(ws + wbytes);
    double* Z = (double*)(ws + 2 * wbytes);
    double* T = (double*)(ws + 3 * wbytes);  // B^T B: Y = B q
    double* part = (double*)(ws + 4 * wbytes);
    const int gv = (int)std::min<int64_t>((d * (K / 2) + kThreads - 1) / kThreads, (int64_t)sms * 8);
    double* s_d = part + (size_t)gv * K;
    double* beta0 = s_d + K;                  // [K] sqrt(d) (normalises the probe), then zeros
    unsigned int* ticket = (unsigned int*)(beta0 + 2 * K);
    const int64_t ngs = (std::max(op->A.n_rows, op->At.n_rows) + SpmmGeo<K>::GROUPS - 1) / SpmmGeo<K>::GROUPS;
    const int gs = grid_for(spmm_kernel<K>, ngs, sms);
    const int gp = (int)std::min<int64_t>((d * K + kThreads - 1) / kThreads, (int64_t)sms * 8);
    std::vector<double> hb(2 * K);
    for (int c = 0; c < K; c++) {
        hb[c] = std::sqrt((double)d);  // |v| for a +-1 probe
        hb[K + c] = 0.0;
    }
    CL_CUDA(cudaMemcpyAsync(beta0, hb.data(), sizeof(double) * 2 * K, cudaMemcpyHostToDevice, st));
    CL_CUDA(cudaMemsetAsync(ticket, 0, 256, st));
    lanczos_probe_kernel<K><<<gp, kThreads, 0, st>>>(d, seed, (uint64_t)p0, Pb);
    LzArgs a{};
    a.d = d;
    a.u = op->kind == CL_OP_CSR_RANK1 ? op->r1_u : nullptr;
    a.r1c = op->kind == CL_OP_CSR_RANK1 ? op->r1_c : 0.0;
    a.s = s_d;
    a.part = part;
    a.ticket = ticket;
    // q_0 = v / |v|, s = u^T q_0
    a.qp = Pb;
    a.beta = beta0;
    a.out = s_d;
    lanczos_vec_kernel<K, LZ_NRM><<<gv, kThreads, 0, st>>>(a);
    std::swap(Q, Pb);
    CL_CUDA(cudaMemsetAsync(Pb, 0, wbytes, st));  // q_{-1} = 0 (beta_0 = 0: row K.. of beta0)
    g_launches += 2;
    for (int j = 0; j < N; j++) {
        double* al = hist_d + (size_t)(2 * j) * K;
        double* bn = hist_d + (size_t)(2 * j + 1) * K;
        const double* bj = j == 0 ? beta0 + K : hist_d + (size_t)(2 * j - 1) * K;
        if (op->kind == CL_OP_BTB) {
            spmm_kernel<K><<<gs, kThreads, 0, st>>>(op->A.n_rows, op->A.row_ptr, op->A.col_idx, op->A.val, Q, T);
            spmm_kernel<K><<<gs, kThreads, 0, st>>>(op->At.n_rows, op->At.row_ptr, op->At.col_idx, op->At.val, T, Z);
            g_launches += 2;
        } else {
            spmm_kernel<K><<<gs, kThreads, 0, st>>>(op->A.n_rows, op->A.row_ptr, op->A.col_idx, op->A.val, Q, Z);
            g_launches++;
        }
        a.q = Q;
        a.qp = Pb;
        a.z = Z;
        a.out = al;
        lanczos_vec_kernel<K, LZ_DOT><<<gv, kThreads, 0, st>>>(a);
        a.alpha = al;
        a.beta = bj;
        a.out = bn;
        lanczos_vec_kernel<K, LZ_UPD><<<gv, kThreads, 0, st>>>(a);
        a.beta = bn;
        a.out = s_d;
        lanczos_vec_kernel<K, LZ_NRM><<<gv, kThreads, 0, st>>>(a);
        g_launches += 3;
        std::swap(Q, Pb);
    }
    CL_CUDA(cudaGetLastError());
    return CL_OK;
}

size_t lanczos_ws_bytes(int64_t d, int k, int sms) {
    const size_t wbytes = align256((size_t)d * k * sizeof(double));
    return 4 * wbytes + align256(((size_t)sms * 8 + 3) * k * sizeof(double) + 256);
}
}  // namespace
}  // extern "C++"

int cheb_spectrum_bounds(const cl_operator* op, int32_t lanczos_steps, int32_t num_probes, uint64_t seed,
                         cl_spectrum* out, double* jacobi_out) {
    int rc;
    if ((rc = check_op(op))) return rc;
    if (op->kind == CL_OP_FAMILY) return fail(CL_EINVAL, "family operators: not supported here");
    if (!out) return fail(CL_EINVAL, "out is NULL");
    if (lanczos_steps < 1 || lanczos_steps > 2000) return fail(CL_EINVAL, "lanczos_steps must be in [1, 2000]");
    if (num_probes < 1 || num_probes > 4096) return fail(CL_EINVAL, "num_probes must be in [1, 4096]");
    cudaStream_t st;
    CL_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard { cudaStream_t s; ~StreamGuard() { cudaStreamSynchronize(s); cudaStreamDestroy(s); } } guard{st};
    double hi = 0.0;  // a guaranteed upper bound of the spectrum from the matrix
    if ((rc = cheb_norm_bound(op, &hi, st))) return rc;
    const int N = lanczos_steps, k = pick_k(num_probes), sms = sm_count();
    const int64_t d = op->A.n_cols;
    const size_t wbytes = align256((size_t)d * k * sizeof(double));
    const size_t ws_bytes = lanczos_ws_bytes(d, k, sms);
    const size_t hist_n = (size_t)2 * N * k;
    void* ws = nullptr;
    if ((rc = arena_get(0, ws_bytes + sizeof(double) * hist_n, &ws))) return rc;
    double* hist_d = (double*)((char*)ws + ws_bytes);
    std::vector<double> hist(hist_n), dd, ee, z;
    double lmin = INFINITY, lmax = -INFINITY, rmin = 0.0, rmax = 0.0;
    int used = N;
    for (int64_t p0 = 0; p0 < num_probes; p0 += k) {
        const int kvalid = (int)std::min<int64_t>(k, num_probes - p0);
        switch (k) {
            case 8: rc = lanczos_block<8>(op, N, seed, p0, (char*)ws, wbytes, hist_d, st, sms); break;
            case 16: rc = lanczos_block<16>(op, N, seed, p0, (char*)ws, wbytes, hist_d, st, sms); break;
            case 32: rc = lanczos_block<32>(op, N, seed, p0, (char*)ws, wbytes, hist_d, st, sms); break;
            case 64: rc = lanczos_block<64>(op, N, seed, p0, (char*)ws, wbytes, hist_d, st, sms); break;
            default: rc = lanczos_block<128>(op, N, seed, p0, (char*)ws, wbytes, hist_d, st, sms); break;
        }
        if (rc) return rc;
        CL_CUDA(cudaMemcpyAsync(hist.data(), hist_d, sizeof(double) * hist_n, cudaMemcpyDeviceToHost, st));
        CL_CUDA(cudaStreamSynchronize(st));
        for (int c = 0; c < kvalid; c++) {
            // T_Nv: diagonal alpha_0..alpha_{Nv-1}, off-diagonal beta_1..beta_{Nv-1}, residual beta_Nv;
            // the process stops early at an invariant subspace (beta = 0) or a non-finite value
            int Nv = 0;
            double bmax = 0.0;
            for (int j = 0; j < N; j++) {
                const double al = hist[(size_t)(2 * j) * k + c], bn = hist[(size_t)(2 * j + 1) * k + c];
                if (!std::isfinite(al) || !std::isfinite(bn)) break;
                Nv = j + 1;
                bmax = std::max(bmax, bn);
                if (!(bn > 1e-14 * bmax)) break;
            }
            if (Nv < 1) return fail(CL_ENONFINITE, "Lanczos step 1 not finite (probe %lld)", (long long)(p0 + c));
            used = std::min(used, Nv);
            if (jacobi_out) {
                double* row = jacobi_out + (size_t)(p0 + c) * 2 * N;
                for (int j = 0; j < N; j++) {
                    row[j] = j < Nv ? hist[(size_t)(2 * j) * k + c] : NAN;
                    row[N + j] = j < Nv ? hist[(size_t)(2 * j + 1) * k + c] : NAN;
                }
            }
            dd.resize(Nv);
            ee.resize(Nv > 1 ? Nv - 1 : 0);
            for (int j = 0; j < Nv; j++) dd[j] = hist[(size_t)(2 * j) * k + c];
            for (int j = 0; j + 1 < Nv; j++) ee[j] = hist[(size_t)(2 * j + 1) * k + c];
            const double bN = hist[(size_t)(2 * (Nv - 1) + 1) * k + c];
            if ((rc = tridiag_ql(dd, ee, z))) return rc;
            int imin = 0, imax = 0;
            for (int i = 1; i < Nv; i++) {
                if (dd[i] < dd[imin]) imin = i;
                if (dd[i] > dd[imax]) imax = i;
            }
            // Ritz value and Kahan residual bound beta_Nv |s_Nv| (an eigenvalue of M lies within it)
            const double r0 = bN * std::fabs(z[(size_t)(Nv - 1) * Nv + imin]);
            const double r1 = bN * std::fabs(z[(size_t)(Nv - 1) * Nv + imax]);
            if (dd[imin] < lmin) { lmin = dd[imin]; rmin = r0; }
            if (dd[imax] > lmax) { lmax = dd[imax]; rmax = r1; }
        }
    }
    out->lambda_min = lmin;
    out->lambda_max = lmax;
    out->res_min = rmin;
    out->res_max = rmax;
    out->a = std::max(lmin - rmin, 0.0);
    out->b = std::min(lmax + rmax, hi);
    out->hi_bound = hi;
    out->lanczos_steps = used;
    out->num_probes = num_probes;
    return CL_OK;
}

int cheb_bounds_btb(const cl_operator* op, double* ab_out, void* stream) {
    int rc;
    if ((rc = check_op(op))) return rc;
    if (op->kind != CL_OP_BTB) return fail(CL_EINVAL, "cheb_bounds_btb needs a CL_OP_BTB operator");
    if (!ab_out) return fail(CL_EINVAL, "ab_out is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf buf;
    CL_CUDA(cudaMalloc(&buf.p, 3 * sizeof(unsigned long long)));
    unsigned long long init[3] = {~0ull, 0ull, 0ull};
    CL_CUDA(cudaMemcpyAsync(buf.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
    const int64_t d = op->A.n_rows;
    int grid = (int)std::min<int64_t>((d + kThreads - 1) / kThreads, (int64_t)sm_count() * 8);
    bounds_btb_kernel<<<grid, kThreads, 0, st>>>(d, op->A.row_ptr, op->A.col_idx, op->A.val,
                                                  op->At.row_ptr, op->At.col_idx, op->At.val,
                                                  (unsigned long long*)buf.p);
    g_launches++;
    CL_CUDA(cudaGetLastError());
    unsigned long long h[3];
    CL_CUDA(cudaMemcpyAsync(h, buf.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    CL_CUDA(cudaStreamSynchronize(st));
    auto unkey = [](unsigned long long k) {
        unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
        double x;
        memcpy(&x, &b, sizeof(x));
        return x;
    };
    const double smin = unkey(h[0]), rmax = unkey(h[1]), cmax = unkey(h[2]);
    if (!(smin > 0.0))
        return fail(CL_EINVAL, "Johnson lower bound on sigma_min is not positive (%g); supply [a,b]", smin);
    ab_out[0] = smin * smin;
    ab_out[1] = cmax * rmax;
    return CL_OK;
}

int cheb_probes(int64_t d, uint64_t seed, int64_t probe_begin, int32_t probe_block,
                double* v_out, void* stream) {
    if (d < 1 || d >= (int64_t(1) << 31)) return fail(CL_EDIM, "bad d");
    if (probe_begin < 0 || !valid_k(probe_block) || !v_out) return fail(CL_EINVAL, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    cl_operator op{};
    op.kind = CL_OP_CSR;
    op.A.n_rows = op.A.n_cols = d;
    const int sms = sm_count();
    const Layout L = plan(d, 0, probe_block, CL_OP_CSR, sms);
    DevBuf ws, mu;
    CL_CUDA(cudaMalloc(&ws.p, L.total));
    CL_CUDA(cudaMalloc(&mu.p, sizeof(double) * probe_block));
    CL_CUDA(cudaMemsetAsync((char*)ws.p + L.ticket, 0, 256, st));
    int rc;
    switch (probe_block) {
        case 8: rc = run_block<8, MODE_CSR>(&op, 1.0, 0.0, 0, seed, probe_begin, 8, (char*)ws.p, L, (double*)mu.p, 1, st, sms, Schedule()); break;
        case 16: rc = run_block<16, MODE_CSR>(&op, 1.0, 0.0, 0, seed, probe_begin, 16, (char*)ws.p, L, (double*)mu.p, 1, st, sms, Schedule()); break;
        case 32: rc = run_block<32, MODE_CSR>(&op, 1.0, 0.0, 0, seed, probe_begin, 32, (char*)ws.p, L, (double*)mu.p, 1, st, sms, Schedule()); break;
        case 64: rc = run_block<64, MODE_CSR>(&op, 1.0, 0.0, 0, seed, probe_begin, 64, (char*)ws.p, L, (double*)mu.p, 1, st, sms, Schedule()); break;
        default: rc = run_block<128, MODE_CSR>(&op, 1.0, 0.0, 0, seed, probe_begin, 128, (char*)ws.p, L, (double*)mu.p, 1, st, sms, Schedule()); break;
    }
    if (rc) return rc;
    CL_CUDA(cudaMemcpyAsync(v_out, (char*)ws.p + L.w0, sizeof(double) * d * probe_block,
                            cudaMemcpyDeviceToDevice, st));
    CL_CUDA(cudaStreamSynchronize(st));
    return CL_OK;
}

}  // extern "C"
