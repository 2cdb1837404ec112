// symgs_sweep on the device (inc/kernels.hpp:44-48) and CG preconditioned with it
// (inc/solver.hpp:40-46).
//
// The reference's sweep is sequential by definition: natural order, every row uses the latest values.  For the matrix
// of a grid (27-point couplings or a subset of them) the same result comes out of a hyperplane schedule: the row of
// node (ix, iy, iz) depends, in the forward sweep, on the rows with a smaller index among its neighbours, and every one
// of those lies on a lower plane  level = ix + 2 iy + 4 iz  (the smallest integer weights with that property for
// couplings dx, dy, dz in {-1, 0, 1}); the backward sweep walks the levels downwards.  Rows of one level do not read
// one another, so a level is one kernel launch, and a sweep is 2 * ((nx-1) + 2 (ny-1) + 4 (nz-1) + 1) launches whose
// results are bit-identical to the sequential loop (same per-row expression: entries in ascending column order,
// products and sums rounded separately, one subtraction, one division).  The schedule is checked against the matrix on
// the device before the first sweep (every off-diagonal column must lie on the side of the level order that its index
// order says): a matrix that does not fit -- explicit rows with other couplings -- is refused, not swept wrongly.
// It is launch-bound (256^3: 3570 launches per sweep), far from the SpMV's rate, and far ahead of a sequential sweep.
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "device_utils.cuh"
#include "spmv_internal.cuh"

namespace spmvb {

__device__ __forceinline__ int level_of(int64_t row, int nx, int ny) {
    const int ix = (int)(row % nx), iy = (int)((row / nx) % ny), iz = (int)(row / ((int64_t)nx * ny));
    return ix + 2 * iy + 4 * iz;
}

// flags[0]: a row without a non-zero diagonal; flags[1]: a coupling the hyperplane schedule does not order
__global__ void symgs_check_kernel(const int64_t *__restrict__ row_start, const int32_t *__restrict__ cols, const double *__restrict__ vals,
                                   int n, int nx, int ny, int *__restrict__ flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int li = level_of(i, nx, ny);
    bool diag = false, fits = true;
    for (int64_t t = row_start[i]; t < row_start[i + 1]; t++) {
        const int j = cols[t];
        if (j == i) {
            diag = vals[t] != 0.0;
            continue;
        }
        const int lj = level_of(j, nx, ny);
        fits = fits && (j < i ? lj < li : lj > li);
    }
    if (!diag) atomicOr(&flags[0], 1);
    if (!fits) atomicOr(&flags[1], 1);
}

// the rows of one level: a thread per (iy, iz) with iz in [iz_lo, iz_lo + n_iz)
__global__ void symgs_level_kernel(const int64_t *__restrict__ row_start, const int32_t *__restrict__ cols, const double *__restrict__ vals,
                                   double *x, const double *__restrict__ b, int nx, int ny, int level, int iz_lo, int n_iz) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ny * n_iz) return;
    const int iy = t % ny, iz = iz_lo + t / ny;
    const int ix = level - 2 * iy - 4 * iz;
    if (ix < 0 || ix >= nx) return;
    const int i = ix + nx * (iy + ny * iz);
    // Entries in ascending column order; the loads of a batch (columns, values, then the gathers of x) are issued together
    // before the ordered sums consume them: a row costs a few memory latencies instead of one per entry (the launch of a
    // level lasts as long as its slowest row).
    constexpr int B = 27;  // a 27-point row in one batch: row_start -> columns, values -> x -> sum, four dependent latencies
    const int64_t k0 = row_start[i];
    const int cnt = (int)(row_start[i + 1] - k0);
    double sum = 0.0, diag = 0.0;
    for (int base = 0; base < cnt; base += B) {
        int c[B];
        double v[B], xv[B];
#pragma unroll
        for (int j = 0; j < B; j++) {
            const bool in = base + j < cnt;
            c[j] = in ? cols[k0 + base + j] : i;
            v[j] = in ? vals[k0 + base + j] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < B; j++) xv[j] = c[j] != i ? x[c[j]] : 0.0;
#pragma unroll
        for (int j = 0; j < B; j++) {
            if (base + j >= cnt) continue;
            if (c[j] == i) diag = v[j];
            else sum = __dadd_rn(sum, __dmul_rn(v[j], xv[j]));
        }
    }
    x[i] = __ddiv_rn(__dsub_rn(b[i], sum), diag);  // inc/kernels.hpp:46
}

// ---- the whole sweep in ONE launch ---------------------------------------------------------------------------------
// A level holds ~10^4 rows (256^3: 16.8 M rows over 1786 levels) -- microseconds of work -- so a sweep of per-level launches
// is launch latency, 3572 times.  The persistent kernel keeps one CTA per SM resident (cooperative launch) and walks the
// levels itself, a grid-wide barrier between them.  What a row needs besides x does not depend on the sweep, so it is
// fetched ahead, into registers: a thread holds the head of the row it will own two levels on (row_start pair, b[row]) and
// requests the entries of its next row before it arrives at the barrier.  After the barrier only the gathers of x
// (ld.global.cg: the values were written by other SMs a level ago; one L2 round trip), the ordered sum and the store remain.
// 256 threads per CTA so that nothing spills (the barrier's acquire invalidates L1, and spill reloads then miss: 384 threads
// at 168 registers ran 40 % slower; staging the entries in shared memory with cp.async instead: 2.3 x slower).
// Same per-row expression as the level kernel: bit-identical.
constexpr int kSymgsThreads = 256;  // one CTA per SM
constexpr int kSymgsRow = 27;       // entries of a row fetched ahead (longer rows read the rest in place)

__device__ __forceinline__ void symgs_level_rect(int level, int nx, int ny, int nz, int *iz_lo, int *n_iz) {
    const int rest = level - (nx - 1) - 2 * (ny - 1);
    const int lo = rest > 0 ? (rest + 3) / 4 : 0;
    const int hi = min(nz - 1, level / 4);
    *iz_lo = lo;
    *n_iz = hi >= lo ? hi - lo + 1 : 0;
}

// Entry t of a level's enumeration: plane iz = iz_lo + t / w, and the (t % w)-th node of that plane's part of the level --
// iy from max(0, ceil((level - 4 iz - (nx-1)) / 2)) upwards while ix = level - 2 iy - 4 iz stays >= 0.  A plane holds at most
// w = min(ny, nx/2 + 2) nodes of a level, so the enumeration has w * n_iz entries (half of the (iy, iz) rectangle).
__device__ __forceinline__ int symgs_width(int nx, int ny) { return min(ny, nx / 2 + 2); }
__device__ __forceinline__ int symgs_row_of(int t, int level, int nx, int ny, int iz_lo, int n_iz) {
    const int w = symgs_width(nx, ny);
    if (t >= w * n_iz) return -1;
    const int iz = iz_lo + t / w;
    const int rest = level - 4 * iz;               // = ix + 2 iy
    const int lo = rest - (nx - 1);                // 2 iy >= lo
    const int iy = (lo > 0 ? (lo + 1) / 2 : 0) + t % w;
    const int ix = rest - 2 * iy;
    if (iy >= ny || ix < 0 || ix >= nx) return -1;
    return ix + nx * (iy + ny * iz);
}

struct SymgsHead {  // what is known of a row before its entries: the row, its first entry, its length, b[row]
    int i, cnt;
    int64_t k0;
    double bi;
};
struct SymgsBody {  // the first 27 entries
    int c[kSymgsRow];
    double v[kSymgsRow];
};

__device__ __forceinline__ SymgsHead symgs_head(int i, const int64_t *__restrict__ row_start, const double *__restrict__ b) {
    SymgsHead h{i, 0, 0, 0.0};
    if (i >= 0) {
        h.k0 = __ldg(row_start + i);
        h.cnt = (int)(__ldg(row_start + i + 1) - h.k0);
        h.bi = __ldg(b + i);
    }
    return h;
}

__device__ __forceinline__ void symgs_body(SymgsBody &r, const SymgsHead &h, const int32_t *__restrict__ cols, const double *__restrict__ vals) {
#pragma unroll
    for (int j = 0; j < kSymgsRow; j++) {
        const bool in = j < h.cnt;
        r.c[j] = in ? __ldg(cols + h.k0 + j) : h.i;
        r.v[j] = in ? __ldg(vals + h.k0 + j) : 0.0;
    }
}

// the row's new value from the latest x (entries in ascending column order, inc/kernels.hpp:46)
__device__ __forceinline__ void symgs_relax(const SymgsHead &h, const SymgsBody &r, const int32_t *__restrict__ cols,
                                            const double *__restrict__ vals, double *x) {
    const int i = h.i;
    double xv[kSymgsRow];
#pragma unroll
    for (int j = 0; j < kSymgsRow; j++) xv[j] = (j < h.cnt && r.c[j] != i) ? __ldcg(x + r.c[j]) : 0.0;
    double sum = 0.0, diag = 0.0;
#pragma unroll
    for (int j = 0; j < kSymgsRow; j++) {
        if (j >= h.cnt) continue;
        if (r.c[j] == i) diag = r.v[j];
        else sum = __dadd_rn(sum, __dmul_rn(r.v[j], xv[j]));
    }
    for (int j = kSymgsRow; j < h.cnt; j++) {  // longer rows (explicit matrices): the rest entry by entry
        const int cj = __ldg(cols + h.k0 + j);
        const double v = __ldg(vals + h.k0 + j);
        if (cj == i) diag = v;
        else sum = __dadd_rn(sum, __dmul_rn(v, __ldcg(x + cj)));
    }
    __stcg(x + i, __ddiv_rn(__dsub_rn(h.bi, sum), diag));
}

// grid-wide barrier: one arrival per CTA on a monotonically increasing counter (release / acquire at gpu scope)
__device__ __forceinline__ void symgs_grid_barrier(unsigned int *counter, unsigned int target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(counter, 1u);
        unsigned int seen;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(counter) : "memory");
        } while ((int)(seen - target) < 0);
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kSymgsThreads, 1) symgs_sweep_persistent_kernel(const int64_t *__restrict__ row_start, const int32_t *__restrict__ cols,
                                                                                  const double *__restrict__ vals, double *x, const double *__restrict__ b,
                                                                                  int nx, int ny, int nz, int levels, unsigned int *counter,
                                                                                  unsigned int epoch) {
    // rows of a level are dealt out across the SMs first (entry t of the level's rectangle -> CTA t % grid): a level holds
    // fewer rows than the machine has threads, and an SM sustains only so many outstanding gathers
    const int t0 = blockIdx.x + gridDim.x * threadIdx.x;
    const int steps = 2 * levels;
    auto level_of_step = [&](int s) { return s < levels ? s : 2 * levels - 1 - s; };
    auto head_of_step = [&](int s) {
        if (s >= steps) return SymgsHead{-1, 0, 0, 0.0};
        int iz_lo, n_iz;
        symgs_level_rect(level_of_step(s), nx, ny, nz, &iz_lo, &n_iz);
        return symgs_head(symgs_row_of(t0, level_of_step(s), nx, ny, iz_lo, n_iz), row_start, b);
    };
    SymgsHead cur = head_of_step(0), nxt = head_of_step(1);
    SymgsBody body;
    symgs_body(body, cur, cols, vals);
    for (int s = 0; s < steps; s++) {
        if (cur.i >= 0) symgs_relax(cur, body, cols, vals, x);
        if (s + 1 < steps) {
            cur = nxt;
            symgs_body(body, cur, cols, vals);  // the next level's entries (its head arrived a level ago) ...
            nxt = head_of_step(s + 2);          // ... and the head of the level after it: all in flight across the barrier
            symgs_grid_barrier(counter, epoch + (unsigned int)(s + 1) * gridDim.x);
        }
    }
}

// ---- the pipelined sweep: a plane per CTA, operands through shared memory ---------------------------------------------
// What a level costs in the kernels above is neither the barrier nor DRAM: a thread reading its own CSR row touches a cache
// line per load (54 loads of entries, 26 gathers of x), and the L1 tag stage looks up one line per clock.  For matrices
// whose rows are sub-boxes of their node's 27 neighbours (the stencil matrix, 7-point matrices, user values -- anything the
// plan kernel below accepts) none of those loads is needed:
//  * a row is its 27-bit box mask (one word, derived once per matrix) and its values in column order: the columns are never
//    read, and the values of a warp's 32 rows are fetched a row at a time with the lanes on consecutive entries (coalesced),
//    a step ahead, and handed over through the warp's shared-memory buffer;
//  * a CTA owns plane iz, thread t = line iy, and step k relaxes u = k - 2t (the plane's own levels; in-plane dependences are
//    met by the lockstep of the CTA's barriers).  Every thread keeps a 16-deep window of its line of x for the plane below, its
//    own plane and the plane above in shared memory -- one load per plane and step, four to six positions ahead of its own -- and a row
//    takes all 26 operands from those rings: new values behind the front, old values ahead of it, exactly what the sequential
//    sweep would read;
//  * the plane below is another CTA's: it publishes its step count (release) and this plane's step k waits until that count
//    is k + 5 -- the level function's 4 iz plus the one step the ring of that plane runs ahead.  Planes are dealt round-robin to the
//    co-resident CTAs (cooperative launch), each CTA taking its planes in sweep order, so the waits form no cycle; the backward
//    sweep is the mirror image (u, t and the plane order reversed: thread t = line ny-1-t, u = nx-1-ix) and its first plane
//    waits for the forward sweep's last.  Two extra warps poll and publish, so that no compute thread ever executes a gpu-scope
//    fence (which waits for the issuing thread's outstanding loads -- a compute thread always has some).
// Per row the same expression in the same order as the kernels above (ascending column = ascending box position, products
// and sums rounded separately, one subtraction, one division): bit-identical.
constexpr int kBoxRing = 16;       // positions of a line kept per plane
constexpr int kBoxPitch = 17;      // doubles between two lines of a ring (odd: the lanes of a warp, two positions apart on neighbouring lines, spread over the banks)
constexpr int kBoxAhead = 6;       // own plane and the plane above (old values): a thread loads position u + 6 and hands it to the ring a step later
constexpr int kBoxBelow = 4;       // the plane below (new values): position u + 4, requested behind the step's acquire, in the ring by the step's end
constexpr int kBoxLag = 5;         // steps a plane trails the one below: the level function's 4 iz and the one step the ring runs ahead

// plan: bit (dz+1)*9 + (dy+1)*3 + (dx+1) for every entry; flags[0] set when a row is not a sub-box of its node's neighbours
__global__ void symgs_box_plan_kernel(const int64_t *__restrict__ row_start, const int32_t *__restrict__ cols, int n, int nx, int ny, int nz,
                                      uint32_t *__restrict__ mask, int *__restrict__ flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int ix = i % nx, iy = (i / nx) % ny, iz = i / (nx * ny);
    const int64_t nxny = (int64_t)nx * ny;
    uint32_t m = 0;
    bool ok = true;
    int last = -1;
    for (int64_t t = row_start[i]; t < row_start[i + 1]; t++) {
        const int64_t u = (int64_t)cols[t] - i + nxny + nx + 1;  // (dx+1) + nx (dy+1) + nx ny (dz+1)
        if (u < 0 || u >= 3 * nxny) {
            ok = false;
            break;
        }
        const int dzp = (u >= 2 * nxny) + (u >= nxny);
        const int64_t rem = u - dzp * nxny;
        const int dyp = (rem >= 2 * (int64_t)nx) + (rem >= nx);
        const int64_t dxp = rem - (int64_t)dyp * nx;
        const int bit = dzp * 9 + dyp * 3 + (int)dxp;
        if (dxp > 2 || ix + dxp - 1 < 0 || ix + dxp - 1 >= nx || iy + dyp - 1 < 0 || iy + dyp - 1 >= ny || iz + dzp - 1 < 0 || iz + dzp - 1 >= nz ||
            bit <= last) {
            ok = false;
            break;
        }
        last = bit;
        m |= 1u << bit;
    }
    mask[i] = m;
    if (!ok) atomicOr(&flags[0], 1);
}

__device__ __forceinline__ int ld_acquire_gpu(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int *p, int v) { asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }

struct BoxHead {  // what a thread knows of a row before its values: index, first entry, mask, b[row]
    int i;
    uint32_t mask;
    int64_t k0;
    double bi;
};

template <int THREADS>
__global__ void __launch_bounds__(THREADS + 64, 1) symgs_box_pipeline_kernel(const int64_t *__restrict__ row_start, const double *__restrict__ vals,
                                                                             const uint32_t *__restrict__ mask, double *x, const double *__restrict__ b,
                                                                             int nx, int ny, int nz, int lag, int *clock_f, int *clock_b) {
    extern __shared__ __align__(16) unsigned char symgs_smem[];
    constexpr int LINES = THREADS + 2;
    double *ring = reinterpret_cast<double *>(symgs_smem);                                  // [3 planes][LINES][kBoxRing]
    double *stage = ring + 3 * LINES * kBoxPitch;                                           // [THREADS / 32 warps][32 rows][27 values]
    const int t = threadIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int role = threadIdx.x < THREADS ? 0 : threadIdx.x < THREADS + 32 ? 1 : 2;        // compute / poll / publish
    const int G = gridDim.x, c = blockIdx.x;
    const int K = nx + 2 * (ny - 1);                       // levels of a plane
    const int KT = K + kBoxAhead;                          // steps of a plane: the rings are filled six steps ahead of the first row
    const int R = c < nz ? (nz - 1 - c) / G + 1 : 0;       // this CTA's planes: c, c + G, ...
    const int ticks = 2 * R * KT;
    const int64_t nxny = (int64_t)nx * ny;
    if (role != 0) {  // the whole warp walks the steps and meets its barrier; lane 0 does the memory operations
        int seen = 0, r = 0, kt = 0;
        bool back = false;
        for (int tick = 0; tick < ticks; tick++) {
            const int p = back ? c + (R - 1 - r) * G : c + r * G;
            const int k = kt - kBoxAhead;  // level (negative: filling the rings)
            if (role == 1) {
                if (kt == 0) seen = 0;
                int need = min(k + lag, K);
                const int *src = nullptr;
                if (!back) {
                    if (p > 0) src = clock_f + (p - 1);
                } else if (p < nz - 1) {
                    src = clock_b + (p + 1);
                } else {
                    src = clock_f + (nz - 1), need = K;  // the backward sweep begins when the forward sweep has ended
                }
                if (src && lane == 0)
                    while (seen < need) seen = ld_acquire_gpu(src);
                asm volatile("bar.sync 1, %0;" ::"r"(THREADS + 32) : "memory");  // the step may begin
            } else {
                asm volatile("bar.sync 2, %0;" ::"r"(THREADS + 32) : "memory");  // the step's stores are issued (cumulative release below)
                if (lane == 0 && k >= 0) st_release_gpu((back ? clock_b : clock_f) + p, k + 1);
            }
            if (++kt == KT) {
                kt = 0;
                if (++r == R) r = 0, back = true;
            }
        }
        return;
    }
    // ---- compute threads
    // position of a step: (direction, plane, this thread's u = k - 2t); memory coordinates follow from the direction
    struct Pos {
        bool back, valid;
        int p, u;
    };
    // (the step counter is kept as (direction, plane round, step of the plane) and advanced by one: no divisions in the loop)
    struct Cursor {
        int tick, r, kt;
        bool back;
    };
    auto advance = [&](Cursor &cu) {
        cu.tick++;
        if (++cu.kt == KT) {
            cu.kt = 0;
            if (++cu.r == R) cu.r = 0, cu.back = true;
        }
    };
    auto pos_of = [&](const Cursor &cu) -> Pos {
        Pos q{false, false, 0, 0};
        if (cu.tick >= ticks) return q;
        q.back = cu.back;
        q.p = cu.back ? c + (R - 1 - cu.r) * G : c + cu.r * G;
        q.u = cu.kt - kBoxAhead - 2 * t;
        q.valid = t < ny;
        return q;
    };
    auto head_of = [&](const Cursor &cu) -> BoxHead {
        BoxHead h{-1, 0u, 0, 0.0};
        const Pos q = pos_of(cu);
        if (q.valid && q.u >= 0 && q.u < nx) {
            const int ix = q.back ? nx - 1 - q.u : q.u, iy = q.back ? ny - 1 - t : t;
            const int64_t i = ix + (int64_t)nx * iy + nxny * q.p;
            h.i = (int)i;
            h.k0 = __ldg(row_start + i);
            h.mask = __ldg(mask + i);
            h.bi = __ldg(b + i);
        }
        return h;
    };
    double *my_stage = stage + warp * (32 * kSymgsRow);
    double pv[32];
    unsigned pany = 0;
    auto fetch_rows = [&](const BoxHead &h) {  // the values of the warp's 32 rows, a row at a time, lanes on consecutive entries
        pany = __ballot_sync(0xffffffffu, h.i >= 0);
#pragma unroll
        for (int r = 0; r < 32; r++) {
            const int64_t k0 = __shfl_sync(0xffffffffu, h.k0, r);
            const int cnt = __popc(__shfl_sync(0xffffffffu, h.mask, r));
            pv[r] = ((pany >> r & 1u) && lane < cnt) ? __ldg(vals + k0 + lane) : 0.0;
        }
    };
    auto store_rows = [&]() {
#pragma unroll
        for (int r = 0; r < 32; r++)
            if ((pany >> r & 1u) && lane < kSymgsRow) my_stage[r * kSymgsRow + lane] = pv[r];
    };
    // ring loads: position u + 6 of this thread's line in the plane below / own plane / plane above (logical), one step in flight
    double rl[3] = {0.0, 0.0, 0.0};
    bool rl_on[3] = {false, false, false};
    int rl_slot = 0;
    auto ring_loads = [&](const Pos &q) {
        const int u6 = q.u + kBoxAhead;
        rl_slot = u6 & (kBoxRing - 1);
#pragma unroll
        for (int d = 1; d < 3; d++) {
            const int pp = q.p + (q.back ? 1 - d : d - 1);  // this plane / the one logically above
            rl_on[d] = q.valid && u6 >= 0 && u6 < nx && pp >= 0 && pp < nz;
            if (rl_on[d]) {
                const int ix = q.back ? nx - 1 - u6 : u6, iy = q.back ? ny - 1 - t : t;
                rl[d] = __ldcg(x + (ix + (int64_t)nx * iy + nxny * pp));
            }
        }
    };
    double *my_line = ring + (t + 1) * kBoxPitch;  // + d * LINES * kBoxPitch for plane d
    Cursor now{0, 0, 0, false}, ahead{0, 0, 0, false};  // this step / the step whose row is being requested (two ahead)
    BoxHead h0 = head_of(ahead);
    advance(ahead);
    BoxHead h1 = head_of(ahead);
    advance(ahead);
    fetch_rows(h0);
    store_rows();
    __syncwarp();
    for (int tick = 0; tick < ticks; tick++) {
        const Pos q = pos_of(now);
        const BoxHead h2 = head_of(ahead);  // requested two steps ahead of its row
        fetch_rows(h1);                              // the next step's values, in flight across this step
        asm volatile("bar.sync 1, %0;" ::"r"(THREADS + 32) : "memory");
        // (the ring loads of the previous step have had a step to arrive; this step's are requested now, behind the clock's acquire)
        const double prev[3] = {rl[0], rl[1], rl[2]};
        const bool prev_on[3] = {rl_on[0], rl_on[1], rl_on[2]};
        const int prev_slot = rl_slot;
        const bool first = now.kt == 0;  // a new plane: nothing carried over
        ring_loads(q);
        // the plane below: the newest value any neighbour can ask for in the next step, u + 4 (its level there is k + 4: complete, the
        // clock says so); one L2 round trip, hidden behind this step's sums
        const int u4 = q.u + kBoxBelow, pb = q.p + (q.back ? 1 : -1);
        const bool below_on = q.valid && u4 >= 0 && u4 < nx && pb >= 0 && pb < nz;
        double below = 0.0;
        if (below_on) below = __ldcg(x + ((q.back ? nx - 1 - u4 : u4) + (int64_t)nx * (q.back ? ny - 1 - t : t) + nxny * pb));
        if (h0.i >= 0) {
            const double *v = my_stage + lane * kSymgsRow;
            const int s = q.back ? -1 : 1;
            int wc[3];
#pragma unroll
            for (int dx = 0; dx < 3; dx++) wc[dx] = (q.u + s * (dx - 1)) & (kBoxRing - 1);
            double sum = 0.0, diag = 0.0;
            int j = 0;
#pragma unroll
            for (int bz = 0; bz < 3; bz++)
#pragma unroll
                for (int by = 0; by < 3; by++) {
                    const double *line = my_line + ((1 + s * (bz - 1)) * LINES + s * (by - 1)) * kBoxPitch;
#pragma unroll
                    for (int bx = 0; bx < 3; bx++) {
                        const int bit = bz * 9 + by * 3 + bx;
                        if (h0.mask >> bit & 1u) {
                            const double a = v[j++];
                            if (bit == 13) diag = a;
                            else sum = __dadd_rn(sum, __dmul_rn(a, line[wc[bx]]));
                        }
                    }
                }
            const double xn = __ddiv_rn(__dsub_rn(h0.bi, sum), diag);  // inc/kernels.hpp:46
            __stcg(x + h0.i, xn);
            my_line[LINES * kBoxPitch + (q.u & (kBoxRing - 1))] = xn;  // own plane, own line: the new value
        }
        if (!first) {
#pragma unroll
            for (int d = 1; d < 3; d++)
                if (prev_on[d]) my_line[d * LINES * kBoxPitch + prev_slot] = prev[d];
        }
        if (below_on) my_line[u4 & (kBoxRing - 1)] = below;
        asm volatile("bar.sync 2, %0;" ::"r"(THREADS + 32) : "memory");  // the step's x is on its way: the clock may be published
        store_rows();  // (every lane has read its row's values: the buffer takes the next step's, behind the barrier and off the clock's path)
        h0 = h1, h1 = h2;
        advance(now);
        advance(ahead);
    }
}

static int check_schedule(const spmvb_matrix *a, const spmvb_grid *g, cudaStream_t st) {
    if (a->symgs_checked[0] == g->nx && a->symgs_checked[1] == g->ny && a->symgs_checked[2] == g->nz) return SPMVB_OK;
    int *flags = nullptr;
    SPMVB_CUDA(cudaMalloc(&flags, 2 * sizeof(int)));
    int h[2] = {0, 0};
    cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(h), st);
    if (e == cudaSuccess) {
        symgs_check_kernel<<<(a->n + 255) / 256, 256, 0, st>>>(static_cast<const int64_t *>(a->s[SPMVB_S_CSR_ROW_START]),
                                                              static_cast<const int32_t *>(a->s[SPMVB_S_CSR_COLS]),
                                                              static_cast<const double *>(a->s[SPMVB_S_CSR_VALS]), a->n, g->nx, g->ny, flags);
        e = cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, st);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(flags);
    if (e != cudaSuccess) return fail(SPMVB_ERR_CUDA, "symgs_sweep: schedule check failed: %s", cudaGetErrorString(e));
    if (h[0]) return fail(SPMVB_ERR_INVALID_ARGUMENT, "symgs_sweep: a row has a zero or missing diagonal (singular)");
    if (h[1])
        return fail(SPMVB_ERR_INVALID_ARGUMENT,
                    "symgs_sweep: the matrix has couplings the %dx%dx%d hyperplane schedule does not order; the sweep is sequential for it",
                    g->nx, g->ny, g->nz);
    a->symgs_checked[0] = g->nx, a->symgs_checked[1] = g->ny, a->symgs_checked[2] = g->nz;
    return SPMVB_OK;
}

static void launch_levels(const spmvb_matrix *a, const spmvb_grid *g, double *x, const double *b, cudaStream_t st) {
    const int nx = g->nx, ny = g->ny, nz = g->nz;
    const int levels = (nx - 1) + 2 * (ny - 1) + 4 * (nz - 1) + 1;
    const auto *rs = static_cast<const int64_t *>(a->s[SPMVB_S_CSR_ROW_START]);
    const auto *cols = static_cast<const int32_t *>(a->s[SPMVB_S_CSR_COLS]);
    const auto *vals = static_cast<const double *>(a->s[SPMVB_S_CSR_VALS]);
    for (int dir = 0; dir < 2; dir++)
        for (int k = 0; k < levels; k++) {
            const int level = dir == 0 ? k : levels - 1 - k;
            // planes that hold a node of this level: 0 <= level - 4 iz - 2 iy - ix with iy <= ny-1, ix <= nx-1
            const int rest = level - (nx - 1) - 2 * (ny - 1);
            const int iz_lo = rest > 0 ? (rest + 3) / 4 : 0;
            const int iz_hi = std::min(nz - 1, level / 4);
            if (iz_hi < iz_lo) continue;
            const int n_iz = iz_hi - iz_lo + 1;
            const int threads = 128;
            symgs_level_kernel<<<(ny * n_iz + threads - 1) / threads, threads, 0, st>>>(rs, cols, vals, x, b, nx, ny, level, iz_lo, n_iz);
        }
}

// Scratch words for a sweep's synchronisation (barrier counter, plane clocks), one buffer per (device, stream): sweeps on one stream
// are ordered and share it, sweeps on other streams -- other host threads, other handles -- have their own.
static int *sweep_scratch(cudaStream_t st, size_t words) {
    struct Buf {
        int *p = nullptr;
        size_t cap = 0;
    };
    static PerDevice<std::map<cudaStream_t, Buf>> pools;
    static std::mutex lock;
    std::lock_guard<std::mutex> g(lock);
    Buf &b = pools.get()[st];
    if (b.cap < words) {
        if (b.p) cudaFree(b.p);
        b.p = nullptr, b.cap = 0;
        if (cudaMalloc(&b.p, words * sizeof(int)) != cudaSuccess) {
            (void)cudaGetLastError();
            return nullptr;
        }
        b.cap = words;
    }
    return b.p;
}

// A sweep is thousands of tiny dependent launches: they are recorded once into a CUDA graph (kept on the handle, keyed by
// the vectors and the grid) and replayed, which takes the host's per-launch cost out of every sweep after the first
// (the preconditioner applies the sweep to the same two vectors in every iteration).  "symgs_graph" = 0 launches directly.
// one cooperative launch per sweep; 1 = not available here (the caller launches level by level)
static int sweep_persistent(const spmvb_matrix *a, const spmvb_grid *g, double *x, const double *b, cudaStream_t st) {
    struct State {
        int coop = -1, n_sm = 0;
    };
    static PerDevice<State> state;
    State &sd = state.get();
    if (sd.coop < 0) {
        int dev = 0, coop = 0, per_sm = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&sd.n_sm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, symgs_sweep_persistent_kernel, kSymgsThreads, 0) != cudaSuccess || per_sm < 1)
            coop = 0;
        (void)cudaGetLastError();
        sd.coop = coop ? 1 : 0;
    }
    if (!sd.coop) return 1;
    int nx = g->nx, ny = g->ny, nz = g->nz;
    {   // a thread owns at most one row per level: the widest level's (iy, iz) rectangle must fit the grid's threads
        // (256^3: 130 x 193 = 25 k entries against 37,888 threads)
        const int64_t span = std::min<int64_t>(nz, ((int64_t)(nx - 1) + 2 * (int64_t)(ny - 1)) / 4 + 2);
        const int64_t width = std::min<int64_t>(ny, nx / 2 + 2);  // symgs_width
        if (width * span > (int64_t)sd.n_sm * kSymgsThreads) return 1;
    }
    int levels = (nx - 1) + 2 * (ny - 1) + 4 * (nz - 1) + 1;
    const auto *rs = static_cast<const int64_t *>(a->s[SPMVB_S_CSR_ROW_START]);
    const auto *cols = static_cast<const int32_t *>(a->s[SPMVB_S_CSR_COLS]);
    const auto *vals = static_cast<const double *>(a->s[SPMVB_S_CSR_VALS]);
    // the barrier counter: this stream's scratch word, zeroed in front of the launch
    unsigned int *counter = reinterpret_cast<unsigned int *>(sweep_scratch(st, 1));
    unsigned int epoch = 0;
    if (!counter) return 1;
    void *args[] = {&rs, &cols, &vals, &x, &b, &nx, &ny, &nz, &levels, &counter, &epoch};
    if (cudaMemsetAsync(counter, 0, sizeof(unsigned int), st) != cudaSuccess ||
        cudaLaunchCooperativeKernel((const void *)symgs_sweep_persistent_kernel, dim3(sd.n_sm), dim3(kSymgsThreads), args, 0, st) != cudaSuccess) {
        (void)cudaGetLastError();
        return 1;
    }
    return 0;
}

// the pipelined sweep; 1 = not served (rows that are not sub-boxes, lines longer than a CTA, no cooperative launch)
static int sweep_pipeline(const spmvb_matrix *a, const spmvb_grid *g, double *x, const double *b, cudaStream_t st) {
    struct State {
        int coop = -1, n_sm = 0;
    };
    static PerDevice<State> state;
    State &sd = state.get();
    if (sd.coop < 0) {
        int dev = 0, coop = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&sd.n_sm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            coop = 0;
        (void)cudaGetLastError();
        sd.coop = coop ? 1 : 0;
    }
    int nx = g->nx, ny = g->ny, nz = g->nz;
    if (!sd.coop || nx < 3 || ny < 3 || ny > 256) return 1;
    const auto *rs = static_cast<const int64_t *>(a->s[SPMVB_S_CSR_ROW_START]);
    const auto *cols = static_cast<const int32_t *>(a->s[SPMVB_S_CSR_COLS]);
    const auto *vals = static_cast<const double *>(a->s[SPMVB_S_CSR_VALS]);
    if (a->symgs_box[0] != nx || a->symgs_box[1] != ny || a->symgs_box[2] != nz) {  // the plan: once per matrix and grid
        if (a->symgs_mask) cudaFree(a->symgs_mask);
        a->symgs_mask = nullptr;
        a->symgs_box_ok = 0;
        a->symgs_box[0] = nx, a->symgs_box[1] = ny, a->symgs_box[2] = nz;
        int *flags = nullptr;
        int h = 1;
        if (cudaMalloc(&a->symgs_mask, (size_t)a->n * sizeof(uint32_t)) == cudaSuccess && cudaMalloc(&flags, sizeof(int)) == cudaSuccess &&
            cudaMemsetAsync(flags, 0, sizeof(int), st) == cudaSuccess) {
            symgs_box_plan_kernel<<<(a->n + 255) / 256, 256, 0, st>>>(rs, cols, a->n, nx, ny, nz, a->symgs_mask, flags);
            if (cudaMemcpyAsync(&h, flags, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) h = 1;
        }
        if (flags) cudaFree(flags);
        (void)cudaGetLastError();
        a->symgs_box_ok = h == 0;
        if (!a->symgs_box_ok && a->symgs_mask) {
            cudaFree(a->symgs_mask);
            a->symgs_mask = nullptr;
        }
    }
    if (!a->symgs_box_ok) return 1;
    // the planes' clocks: this stream's scratch words, zeroed in front of the launch
    int *clocks = sweep_scratch(st, 1 + (size_t)2 * nz) ;
    if (!clocks) return 1;
    clocks += 1;  // (word 0 is the grid-barrier kernel's counter)
    if (cudaMemsetAsync(clocks, 0, (size_t)2 * nz * sizeof(int), st) != cudaSuccess) {
        (void)cudaGetLastError();
        return 1;
    }
    int *clock_f = clocks, *clock_b = clocks + nz;
    int lag = std::max(kBoxLag, options().symgs_lag);
    const uint32_t *mask = a->symgs_mask;
    const int threads = ny <= 64 ? 64 : 256;
    const void *fn = threads == 64 ? (const void *)symgs_box_pipeline_kernel<64> : (const void *)symgs_box_pipeline_kernel<256>;
    const size_t smem = (size_t)3 * (threads + 2) * kBoxPitch * 8 + (size_t)(threads / 32) * 32 * kSymgsRow * 8;
    const int grid = std::min(sd.n_sm, nz);
    void *args[] = {&rs, &vals, &mask, &x, &b, &nx, &ny, &nz, &lag, &clock_f, &clock_b};
    const bool launched = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess &&
                          cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(threads + 64), args, smem, st) == cudaSuccess;
    if (!launched) {
        (void)cudaGetLastError();
        return 1;
    }
    return 0;
}

static int sweep_device(const spmvb_matrix *a, const spmvb_grid *g, double *x, const double *b, cudaStream_t st) {
    if (options().symgs_pipeline) {
        const int rc = sweep_pipeline(a, g, x, b, st);
        if (rc == 0) {
            options().last_symgs_kernel = 2;
            return SPMVB_OK;
        }
    }
    if (options().symgs_persistent) {
        const int rc = sweep_persistent(a, g, x, b, st);
        if (rc == 0) {
            options().last_symgs_kernel = 1;
            return SPMVB_OK;
        }
    }
    options().last_symgs_kernel = 0;
    SymgsGraph &c = a->symgs_graph;
    const bool hit = c.exec && c.x == x && c.b == b && c.nx == g->nx && c.ny == g->ny && c.nz == g->nz;
    if (options().symgs_graph && !hit) {
        if (c.exec) cudaGraphExecDestroy(c.exec), c.exec = nullptr;
        if (!c.capture_stream && cudaStreamCreateWithFlags(&c.capture_stream, cudaStreamNonBlocking) != cudaSuccess) c.capture_stream = nullptr;
        cudaGraph_t graph = nullptr;
        if (c.capture_stream && cudaStreamBeginCapture(c.capture_stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
            launch_levels(a, g, x, b, c.capture_stream);
            if (cudaStreamEndCapture(c.capture_stream, &graph) == cudaSuccess && graph &&
                cudaGraphInstantiate(&c.exec, graph, nullptr, nullptr, 0) == cudaSuccess) {
                c.x = x, c.b = b, c.nx = g->nx, c.ny = g->ny, c.nz = g->nz;
            } else {
                c.exec = nullptr;
            }
            if (graph) cudaGraphDestroy(graph);
        }
        (void)cudaGetLastError();  // a failed capture falls back to direct launches below
    }
    if (options().symgs_graph && c.exec) {
        SPMVB_CUDA(cudaGraphLaunch(c.exec, st));
        return SPMVB_OK;
    }
    launch_levels(a, g, x, b, st);
    return check_launch("symgs_level");
}

}  // namespace spmvb

using namespace spmvb;

extern "C" {

int spmvb_symgs_sweep(const spmvb_matrix *csr, const spmvb_grid *grid, double *x_dev, const double *b_dev, void *stream) {
    if (!csr || !grid || !x_dev || !b_dev) return fail(SPMVB_ERR_INVALID_ARGUMENT, "symgs_sweep: NULL argument");
    if (csr->format != SPMVB_FMT_CSR || csr->row_offset != 0 || csr->n_cols != csr->n)
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "symgs_sweep: needs the whole square matrix as a CSR handle (inc/kernels.hpp:48)");
    if (grid->nx < 1 || grid->ny < 1 || grid->nz < 1 || (int64_t)grid->nx * grid->ny * grid->nz != csr->n)
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "symgs_sweep: the grid does not have the matrix's %d rows", csr->n);
    if ((int64_t)grid->nx + 2LL * grid->ny + 4LL * grid->nz > INT32_MAX / 2) return fail(SPMVB_ERR_INVALID_ARGUMENT, "symgs_sweep: grid too large");
    if (csr->n == 0) return SPMVB_OK;
    cudaStream_t st = as_stream(stream);
    SPMVB_TRY(check_schedule(csr, grid, st));
    return sweep_device(csr, grid, x_dev, b_dev, st);
}

int spmvb_pcg_solve(const spmvb_matrix *a, const spmvb_matrix *csr, const spmvb_grid *grid, int32_t symgs_sweeps, const double *b_dev,
                    double *x_dev, int32_t max_iterations, double tolerance, int32_t *iterations, int32_t *converged,
                    double *residual_history, void *stream) {
    if (!a || !csr || !grid || !b_dev || !x_dev || !iterations || !converged) return fail(SPMVB_ERR_INVALID_ARGUMENT, "pcg_solve: NULL argument");
    if (max_iterations < 1 || !(tolerance > 0.0) || symgs_sweeps < 1)
        return fail(SPMVB_ERR_INVALID_ARGUMENT, "pcg_solve: need max_iterations >= 1, tolerance > 0 and symgs_sweeps >= 1");
    if (a->row_offset != 0 || a->n != csr->n) return fail(SPMVB_ERR_INVALID_ARGUMENT, "pcg_solve: backend and matrix must be the same whole matrix");
    cudaStream_t st = as_stream(stream);
    const int64_t n = a->n;
    *iterations = 0;
    *converged = 0;
    // the schedule check (and the singularity error) before anything is written
    if (csr->format != SPMVB_FMT_CSR) return fail(SPMVB_ERR_INVALID_ARGUMENT, "pcg_solve: the preconditioner needs the CSR handle");
    if ((int64_t)grid->nx * grid->ny * grid->nz != n) return fail(SPMVB_ERR_INVALID_ARGUMENT, "pcg_solve: the grid does not have the matrix's rows");
    if (n > 0) SPMVB_TRY(check_schedule(csr, grid, st));
    const int64_t n_pad = (n + 63) / 64 * 64;
    double *ws = nullptr;
    SPMVB_CUDA(cudaMalloc(&ws, (size_t)std::max<int64_t>(n_pad, 64) * 4 * sizeof(double)));
    double *r = ws, *z = ws + n_pad, *p = ws + 2 * n_pad, *ap = ws + 3 * n_pad;
    auto done = [&](int code) {
        cudaStreamSynchronize(st);
        cudaFree(ws);
        return code;
    };
    auto precondition = [&]() -> int {  // z <- M^-1 r: sweeps from a zero initial guess
        if (cudaMemsetAsync(z, 0, (size_t)n * 8, st) != cudaSuccess) return fail(SPMVB_ERR_CUDA, "pcg_solve: memset failed");
        for (int s = 0; s < symgs_sweeps; s++) SPMVB_TRY(sweep_device(csr, grid, z, r, st));
        return SPMVB_OK;
    };
    int rc = cudaMemsetAsync(x_dev, 0, (size_t)n * 8, st) == cudaSuccess ? SPMVB_OK : fail(SPMVB_ERR_CUDA, "pcg_solve: memset failed");
    if (rc == SPMVB_OK) rc = spmvb_waxpby(1.0, b_dev, 0.0, b_dev, r, n, stream);
    if (rc == SPMVB_OK) rc = precondition();
    if (rc == SPMVB_OK) rc = spmvb_waxpby(1.0, z, 0.0, z, p, n, stream);
    double bb = 0.0, rz = 0.0;
    if (rc == SPMVB_OK) rc = spmvb_dot(b_dev, b_dev, n, &bb, stream);
    if (rc == SPMVB_OK) rc = spmvb_dot(r, z, n, &rz, stream);
    if (rc != SPMVB_OK) return done(rc);
    const double bnorm = std::sqrt(bb);
    if (residual_history) residual_history[0] = 1.0;
    if (bnorm == 0.0) {
        *converged = 1;
        return done(SPMVB_OK);
    }
    for (int it = 1; it <= max_iterations; it++) {
        double pap = 0.0, rr = 0.0, rz_new = 0.0;
        rc = spmvb_spmv(a, p, 0, n, ap, 0, (int32_t)n, stream);                 // 1 SpMV
        if (rc == SPMVB_OK) rc = spmvb_dot(p, ap, n, &pap, stream);              // dot 1
        if (rc != SPMVB_OK) return done(rc);
        const double alpha = rz / pap;
        rc = spmvb_waxpby(1.0, x_dev, alpha, p, x_dev, n, stream);              // waxpby 1
        if (rc == SPMVB_OK) rc = spmvb_waxpby(1.0, r, -alpha, ap, r, n, stream); // waxpby 2
        if (rc == SPMVB_OK) rc = spmvb_dot(r, r, n, &rr, stream);                // dot 2
        if (rc != SPMVB_OK) return done(rc);
        const double rel = std::sqrt(rr) / bnorm;
        *iterations = it;
        if (residual_history) residual_history[it] = rel;
        if (!std::isfinite(alpha) || !std::isfinite(rel)) {
            done(SPMVB_OK);
            return fail(SPMVB_ERR_DIVERGENCE, "pcg_solve: non-finite value in iteration %d", it);
        }
        if (rel <= tolerance) {
            *converged = 1;
            break;
        }
        rc = precondition();                                                    // z = M^-1 r
        if (rc == SPMVB_OK) rc = spmvb_dot(r, z, n, &rz_new, stream);            // dot 3
        if (rc != SPMVB_OK) return done(rc);
        const double beta = rz_new / rz;
        rz = rz_new;
        rc = spmvb_waxpby(1.0, z, beta, p, p, n, stream);                       // waxpby 3
        if (rc != SPMVB_OK) return done(rc);
    }
    return done(SPMVB_OK);
}

}  // extern "C"
