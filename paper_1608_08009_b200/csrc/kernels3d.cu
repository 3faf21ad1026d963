// 3D fused collision / step kernel (a3-a9) for hard spheres on an N^3 velocity grid.
//
// A group of P co-resident CTAs (cooperative launch, one CTA per SM) owns one cell at a time,
// persistent over cells.  The cell's N^3 spectrum does not fit one SM (N = 32: 512 KiB per
// complex transform), so the 3D inverse FFT of each direction is split by planes:
//   CTA r owns NP = N/P spectrum planes l_y (mirror pairs l_y, -l_y; f^ resident in TMEM) and
//   the output planes j_z in [r NP, (r+1) NP) (gain accumulator in registers).
// Per direction p the CTA
//   z group : forms X = (alpha~_p + i alpha'~_p) f^ on its pencils and IFFTs along z in
//             registers, then writes the pencils to the group's L2 exchange ring (the transpose);
//   xy group: bulk-copies its own j_z planes back (cp.async.bulk, async proxy), IFFTs along x and
//             y and accumulates G += Re z * Im z -- two real transforms packed in one complex
//             IFFT, exact because the symmetrised tables are real and even (reading #10).
// The loss is the (A+1)-th exchange with table (D~, 0); Q = G - f* Re z(loss),
// projection to zero moments (5-sum group reduction through L2) and
// F^{n+1} = f* + (dt/tau) Pi Q, or Q in collide mode.
// Synchronisation is by per-group counters in L2 (GroupSync below), not cluster barriers: the z
// group runs up to NBUF-1 exchange items ahead of the xy group and computes the next cell's
// forward transform (a3 + a4) while the xy group finishes the previous cell.  The exchange goes
// through L2 (bulk reads ~54 B/clk/SM) rather than DSMEM (~7 B/clk/SM, profiles/r01_microbench.txt).
// Tables are pre-folded on the host: alpha~ = s w_p alpha_p / n, alpha'~ = alpha'_p / n,
// D~ = s D / n (s = Btilde kappa^-(d+gamma)); layout T3[p][rank][row][l_x] (Cfg3::SLABR).
#include <cstdlib>

#include "common.cuh"
#include "fft.cuh"
#include "kernels.cuh"

namespace fks {

// Development instrumentation: per-phase clock64 stamps of cluster 0 / CTA 0 (FKS_TIMING builds only).
#ifdef FKS_TIMING
__device__ long long g_tstamp[4096];
#ifndef FKS_TIMING_ROUND
#define FKS_TIMING_ROUND 2  // stamp the group's third cell (steady state)
#endif
#define TSTAMP(slot) do { if (cid == 0 && rank == 0 && (tg == 0) && it == FKS_TIMING_ROUND * c.ncl) g_tstamp[(slot)] = clock64(); } while (0)
// cell boundary: the first cell's epilogue and the second cell's forward (slots 1024..)
#define TSTAMPB(slot) do { if (cid == 0 && rank == 0 && (tg == 0) && (it == 0 || it == c.ncl)) g_tstamp[1024 + (it != 0) * 16 + (slot)] = clock64(); } while (0)
#else
#define TSTAMP(slot) do { } while (0)
#define TSTAMPB(slot) do { } while (0)
#endif

template <int N, int P>
struct Cfg3 {
  static constexpr int NP = N / P;        // planes per CTA
  static constexpr int GT = N * NP;       // threads per warp group (one pencil / row / column each)
  static constexpr int THREADS = 2 * GT;  // z group + xy group (warp-specialised)
  // Planes (SMEM and the L2 exchange buffer) are XOR-swizzled instead of padded: element
  // (row r, column c) lives at r*N + (c ^ (r & 7)), conflict-free for row and column sweeps.
  // z-side plane ownership pairs every l_y plane with its mirror sigma(l_y) = -l_y mod N: the
  // planes in the order 0, N/2, 1, N-1, 2, N-2, ... are dealt out NP per CTA.  The tables are
  // even, T(l) = T(-l) exactly (reading #10), so T(l_x, -a, l_z) = T(-l_x, a, -l_z):
  // a CTA stores only the first plane of each pair and the rows l_z <= N/2 of the self-mirror
  // planes 0 and N/2 -- SLABR rows of N complex entries (halves the table traffic).
  static constexpr int SLABR = (N + 2) + (NP - 2) / 2 * N;  // rows per CTA table slab (rank 0 = max)
  static constexpr int SLAB = SLABR * N;      // complex elements of a table slab
  static constexpr int PSLAB = NP * N * N;    // complex elements of a plane slab
  static constexpr int WPLANE = N * N;        // plane in the exchange buffer
  static constexpr size_t WBUF = (size_t)N * WPLANE;  // one exchange buffer (all N j_z planes)
#ifndef FKS_NBUF
#define FKS_NBUF 5  // C2: 4 slots 19.39 ms / 552 KB DRAM per cell, 5: 19.17 / 724 KB, 6: 19.16 / 2.5 MB (the ring spills), 8: 20.3 ms
#endif
  static constexpr int NBUF = FKS_NBUF;  // exchange ring slots: the z group runs up to NBUF-1 items ahead
  static constexpr int FHAT_COLS = 4 * N;     // one f^ pencil (N complex fp64) per lane (z group)
  // f* column cache (xy group, N >= 16): column (l_x = tx, j_z) of f* (N fp64 = 2N columns),
  // read back by the loss term and the Euler update instead of re-gathering f from HBM.
  // The z group writes it, so z warp w and xy warp w + 4 must share a TMEM lane quarter (GT = 128).
  static constexpr bool FS_TMEM = N >= 16 && N * (N / P) == 128;
  static constexpr int USED_COLS = FHAT_COLS + (FS_TMEM ? 2 * 2 * N : 0);  // two cache parities
  static constexpr int TMEM_COLS = USED_COLS <= 32 ? 32 : USED_COLS <= 64 ? 64 : USED_COLS <= 128 ? 128
                                 : USED_COLS <= 256 ? 256 : 512;
  static constexpr size_t TBUF_BYTES = ((size_t)SLAB * 16 + 127) / 128 * 128;
  static constexpr size_t OFF_TBUF = 0;                       // two table slabs (double-buffered)
  static constexpr size_t OFF_PLN = OFF_TBUF + 2 * TBUF_BYTES;  // two plane slabs
  // Per-warp pipelines: warp w of a group handles the planes tl in [w WPL, (w+1) WPL); the
  // table slab is loaded per table group (TGW warps that share mirror-pair rows).
  static constexpr int NW = GT / 32;                   // warps per group
  static constexpr int WPL = NP / NW;                  // planes per warp
  static constexpr int TGW = NW >= 2 ? 2 : 1;          // warps per table group
  static constexpr int NTG = NW / TGW;                 // table groups
  // mbarriers: tbar[2][NTG], wbar[2][NW], fsb[2] (f* cache written), fse[2] (f* cache read)
  static constexpr int NMBAR = 2 * NTG + 2 * NW + 4 + 2 * NTG;  // ... + tempty[2][NTG]
  static constexpr size_t OFF_MBAR = OFF_PLN + 2 * (size_t)PSLAB * 16;
  static constexpr size_t OFF_TMEM = OFF_MBAR + 8 * NMBAR;
  static constexpr size_t OFF_PART = OFF_TMEM + 8;           // lambda[5] + warp partials [4][5]
  static constexpr size_t OFF_SBASE = OFF_PART + 32 * 8;  // [27] transport sources of the cell
  static constexpr size_t OFF_SFLIP = OFF_SBASE + 27 * 8;  // int8 [27] mirrored components
  static constexpr size_t OFF_DELTA = OFF_SFLIP + 32;      // int8 [3][kMaxN] shift table
  static constexpr size_t SMEM = OFF_DELTA + 3 * kMaxN;
  static_assert(GT % 32 == 0, "warp groups must be whole warps");
  static_assert(NP % 2 == 0, "mirror pairs stay within a CTA");
  static_assert(NP % NW == 0 && (NW == 1 || WPL == 1), "whole planes per warp");
  static_assert(2 * ((SLAB * 16 + 127) / 128 * 128) >= (size_t)NP * N * N * 16,
                "the two table buffers hold one plane slab (z-group forward)");
  static_assert(GT <= 128, "one TMEM lane per z-group thread");
  static_assert(TMEM_COLS >= 32 && (TMEM_COLS & (TMEM_COLS - 1)) == 0, "TMEM allocation: power of two >= 32");
};

__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// TMEM (tcgen05) helpers: 32 columns (32-bit each) of this thread's lane.
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n" : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]) : "r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }


__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// Bulk async copy global -> shared (UBLKCP), completion counted on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  constexpr uint32_t chunk = 32768;
  mbar_expect_tx(bar, bytes);
  for (uint32_t off = 0; off < bytes; off += chunk)
    bulk_g2s(reinterpret_cast<char*>(dst) + off, reinterpret_cast<const char*>(src) + off,
             bytes - off < chunk ? bytes - off : chunk, bar);
}

__device__ __forceinline__ int swz(int r, int c) { return c ^ (r & 7); }

// l_y plane at position q of the order 0, N/2, 1, N-1, 2, N-2, ... (z-side plane ownership).
template <int N>
__device__ __forceinline__ int plane_of(int q) {
  return q == 0 ? 0 : q == 1 ? N / 2 : (q & 1) ? N - q / 2 : q / 2;
}

// Where the z thread of local plane tl finds its table pencil in the CTA's table slab
// (host layout: fks_api.cu upload_tables): first row and how rows/columns map.
struct TabMap {
  int base;  // first slab row of the stored plane
  int mode;  // 0: stored plane; 1: mirror of the stored plane (row -l_z, column -l_x);
             // 2: self-mirror plane, rows l_z <= N/2 stored, the others mirrored
};
template <int N, int NP>
__device__ __forceinline__ TabMap tab_map(int rank, int tl) {
  int base = 0;
  for (int e = 0; e < tl; ++e) {  // rows taken by the entries before tl
    const int ly = plane_of<N>(rank * NP + e);
    if (ly == 0 || ly == N / 2) base += N / 2 + 1;
    else if ((e & 1) == 0) base += N;
  }
  const int ly = plane_of<N>(rank * NP + tl);
  TabMap m;
  if (ly == 0 || ly == N / 2) m = {base, 2};
  else if ((tl & 1) == 0) m = {base, 0};
  else m = {base - N, 1};  // the pair's first plane, stored just before
  return m;
}

// z group: X = T (x) f^ for pencil (l_x = tx, local l_y = tl) of one direction (f^ from this
// thread's TMEM lane, T from the SMEM table slab), then the IFFT along z, in registers.
template <int N, int P>
__device__ __forceinline__ void zpass_compute(uint32_t taddr, const double2* tbuf, int tx, const TabMap& tm,
                                              double2 (&x)[N]) {
  const double2* td = tbuf + tm.base * N + tx;             // stored rows, own column
  const double2* tr = tbuf + tm.base * N + ((N - tx) & (N - 1));  // mirrored column
#pragma unroll
  for (int ch = 0; ch < N / 8; ++ch) {  // 8 complex fp64 = 32 TMEM columns per chunk
    double2 tt[8];  // table entries first: their shared-memory latency overlaps the TMEM load's
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int lz = ch * 8 + i;
      const int lzm = (N - lz) & (N - 1);
      const bool mir = tm.mode == 1 || (tm.mode == 2 && lz > N / 2);
      tt[i] = mir ? tr[lzm * N] : td[lz * N];
    }
    uint32_t v[32];
    tmem_ld32(taddr + ch * 32, v);
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int lz = ch * 8 + i;
      const double Fx = __hiloint2double(v[4 * i + 1], v[4 * i + 0]);
      const double Fy = __hiloint2double(v[4 * i + 3], v[4 * i + 2]);
      const double2 T = tt[i];
      x[lz] = make_double2(fma(T.x, Fx, -T.y * Fy), fma(T.x, Fy, T.y * Fx));
    }
  }
  fft<N, +1>(x);
}


// z-pass output -> this CTA's rows of the exchange buffer (L2): 32 coalesced 512-byte warp stores.
// L2 write bandwidth (~7.8 TB/s chip-wide, tools/microbench/mb_store.cu) bounds the exchange;
// staging through SMEM + bulk (TMA) stores was measured slower: the TMA engine reads the staging
// buffer only as fast as it drains to L2, so the staging slot is not freed any earlier.
template <int N, int P>
__device__ __forceinline__ void zpass_store(const double2 (&x)[N], double2* Wb, int ly, int tx) {
  using C = Cfg3<N, P>;
  double2* w = Wb + (size_t)ly * N + swz(ly, tx);
#pragma unroll
  for (int jz = 0; jz < N; ++jz) w[(size_t)jz * C::WPLANE] = x[jz];
}

// Group synchronisation through L2 (the P CTAs of a cell group are co-resident: cooperative
// launch, one CTA per SM).  Every exchange buffer use is an item of a per-group sequence
// (per cell: the forward xy transform, then z(0) .. z(D-1)); item s lives in ring slot s % NBUF.
// Counts are in warps: each of the NW * P producing warps adds 1 to prod[slot] after writing its
// part (release), each of the NW * P consuming warps adds 1 to cons[slot] once its read has
// completed; a producer of item s first waits for cons[slot] >= NW P (s / NBUF), a consumer for
// prod[slot] >= NW P (s / NBUF + 1).  The counters are zeroed before every launch.
struct GroupSync {
  static constexpr int NB = FKS_NBUF;  // = Cfg3::NBUF
  unsigned prod[NB];
  unsigned cons[NB];
  unsigned part;                // projection partial sums published (cumulative, P per cell)
  unsigned pad[32 - 2 * NB - 1];
  double partial[2][16][5];     // [cell parity][rank][moment]
};

__device__ __forceinline__ void sync_signal(unsigned* ctr) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(ctr) : "memory");
}

__device__ __forceinline__ void sync_signal_n(unsigned* ctr, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(ctr), "r"(v) : "memory");
}

__device__ __forceinline__ void sync_signal_relaxed_n(unsigned* ctr, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;\n" ::"l"(ctr), "r"(v) : "memory");
}

// Consumer-side signal: the reads it announces have completed (their data is in registers or
// SMEM), so no ordering is needed and the thread does not wait for a fence.
__device__ __forceinline__ void sync_signal_relaxed(unsigned* ctr) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;\n" ::"l"(ctr) : "memory");
}

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* ctr) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ctr) : "memory");
  return v;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* ctr) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ctr) : "memory");
  return v;
}

// Spin until *ctr >= target.  A group member that never arrives would otherwise hang the GPU:
// after ~2^24 polls (seconds) the kernel traps and the launch fails loudly.
__device__ __forceinline__ void sync_wait(const unsigned* ctr, unsigned target) {
  unsigned spins = 0;
  while ((int)(ld_acquire(ctr) - target) < 0) {
    if (++spins == (1u << 24)) __trap();
  }
}

// Same for a slot that is only going to be overwritten (its readers signalled after their reads
// completed): a relaxed poll; `seen` is a value loaded earlier, often already sufficient.
__device__ __forceinline__ void sync_wait_free(const unsigned* ctr, unsigned target, unsigned seen) {
  unsigned spins = 0;
  while ((int)(seen - target) < 0) {
    seen = ld_relaxed(ctr);
    if (++spins == (1u << 24)) __trap();
  }
}

// Shared-memory carve-up and per-thread coordinates of the 3D kernel.
template <int N, int P>
struct Ctx3 {
  using C = Cfg3<N, P>;
  double2* tbuf;   // 2 x table slab [SLABR rows][N l_x] (direction g in buffer g & 1)
  double2* pln0;   // 2 x [NP j_z][N y][N x] plane slabs (swizzled)
  uint64_t* tbar;  // [2][NTG] table rows of a table group landed
  uint64_t* wbar;  // [2][NW] plane(s) of a warp landed
  uint64_t* fsb;   // [2] f* cache of parity b written (z group, GT arrivals)
  uint64_t* fse;   // [2] f* cache of parity b read for the last time (xy group, GT arrivals)
  uint64_t* tempty;  // [2][NTG] table buffer b of a table group read by its warps (TGW arrivals)
  double* part;    // [8] epilogue scratch (moment sums, lambda)
  const int8_t (*delta)[kMaxN];  // shift table (SMEM copy)
  const double** sbase;          // [27] per-cell transport sources (forward gather, dx > 0)
  int8_t* sflip;                 // [27] their mirrored velocity components (specular reflection)
  double2* W;      // [NBUF][N j_z][N l_y][N l_x] exchange buffers of this group (L2, swizzled)
  GroupSync* gs;   // this group's counters
  int rank, cid, ncl, tg, tx, tl;
};

// ---- z group: per cell the forward transform, then z(j) for every direction --------------
// Forward (a3 + a4): this CTA's j_z planes of f* are gathered into the table buffers (idle
// between cells), transformed along x and y and published as the forward item; the f* column
// (tx, ., j_z) goes to the xy thread's TMEM lane (cache parity = cell parity).  Then the z
// transform of the CTA's l_y pencils (the forward item of every CTA) into TMEM, and the z passes.
// Doing the forward here lets it overlap the xy group's last directions and epilogue.
template <int N, int P>
__device__ __forceinline__ void z_group(const StepParams& p, const Ctx3<N, P>& c, uint32_t taddr) {
  using C = Cfg3<N, P>;
  constexpr int NP = C::NP, GT = C::GT, NB = C::NBUF;
  constexpr int n = N * N * N;
  const int D = p.A + 1;
  const int rank = c.rank, cid = c.cid, tg = c.tg, tx = c.tx, tl = c.tl;
  GroupSync* gs = c.gs;
  const int ly = plane_of<N>(rank * NP + tl);  // this thread's pencil (l_x = tx, l_y)
  const TabMap tm = tab_map<N, NP>(rank, tl);
  constexpr int NW = C::NW, NTG = C::NTG, TGW = C::TGW;
  constexpr unsigned WP = NW * P;  // signals per exchange item
  const int w = tg >> 5, lane = tg & 31;
  // table group of this warp and its rows of the CTA's table slab: [trow0, trow1)
  const int tgi = w / TGW;
  const bool tg_leader = (w % TGW) == 0 && lane == 0;
  auto rows_end = [&](int tl_last) {
    const TabMap m = tab_map<N, NP>(rank, tl_last);
    return m.mode == 1 ? m.base + N : m.mode == 2 ? m.base + N / 2 + 1 : m.base + N;
  };
  const int trow0 = tab_map<N, NP>(rank, tgi * TGW * C::WPL).base;
  const int trow1 = rows_end((tgi + 1) * TGW * C::WPL - 1);
  const double2* tab_rank = p.tables + (size_t)rank * C::SLAB;  // + direction * P * SLAB
  constexpr size_t TB = C::TBUF_BYTES / 16;  // complex elements per table buffer
  auto load_tab = [&](int j) {  // tg_leader: this group's rows of direction j -> table buffer j & 1
    FKS_CHECK(j >= 0 && j < D && (int64_t)((size_t)j * P * C::SLAB + (size_t)rank * C::SLAB + (size_t)trow1 * N) <= p.table_elems);
    FKS_CHECK(trow0 >= 0 && trow1 <= C::SLABR && (size_t)trow1 * N <= TB);
    bulk_load(c.tbuf + (j & 1) * TB + (size_t)trow0 * N, tab_rank + (size_t)j * P * C::SLAB + (size_t)trow0 * N,
              (uint32_t)(trow1 - trow0) * N * 16, c.tbar + (j & 1) * NTG + tgi);
  };
  uint32_t tphase = 0;  // bit b: parity of this group's table buffer b
  uint32_t tephase = 0;  // bit b: parity of tempty of this group's buffer b
  unsigned pub = 0;     // this warp's first z item not yet published
  unsigned seq = 0;     // exchange-buffer sequence index of the next item
  unsigned ncell = 0;   // cells done by this group
  for (int it = cid; it < p.ncells; it += c.ncl, ++ncell) {
    const int64_t cell = p.cell_list ? p.cell_list[it] : it;
    FKS_CHECK(cell >= 0 && cell < p.tp.ncells_total);
    const CellCoord cc_cell = cell_coord(p.tp, cell);
    const int zpl = rank * NP + tl;  // forward: this thread's j_z plane
    const unsigned par = ncell & 1;
    const uint32_t fs_addr = taddr + C::FHAT_COLS + par * 2 * N;  // xy lane's f* cache (same lane)
    // this CTA's planes of the next cell (homogeneous case: contiguous) -> L2
    if (p.tp.dx == 0 && tg == 0 && !p.cell_list && it + c.ncl < p.ncells)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p.f_in + (int64_t)(it + c.ncl) * n +
                                                                        (int64_t)rank * NP * N * N),
                   "r"((uint32_t)(NP * N * N * sizeof(double)))
                   : "memory");
    const unsigned s_fwd = seq;
    TSTAMPB(0);
    {  // a3 + a4: gather f* (own j_z planes), forward FFT in x and y -> W[s_fwd % NB]
      double2* pln = c.tbuf;  // both table buffers: one plane slab
      constexpr int PER = NP * N * N / GT;  // = N elements per thread
#ifndef FKS_PUB
#define FKS_PUB 1  // z items published per release fence (batches of 2 measured slower: the xy group waits)
#endif
#ifndef FKS_GATHER_B
#define FKS_GATHER_B 32  // f* loads in flight per thread in the forward gather (one L2 round trip)
#endif
      constexpr int B = PER < FKS_GATHER_B ? PER : FKS_GATHER_B;
#pragma unroll 1
      for (int b0 = 0; b0 < PER; b0 += B) {
        double v[B];
        if (p.tp.dx == 0) {  // this CTA's planes are contiguous: every load in flight at once
          const double* src = p.f_in + cell * (int64_t)n + (int64_t)rank * NP * N * N;
#pragma unroll
          for (int j = 0; j < B; ++j) v[j] = __ldg(src + tg + (b0 + j) * GT);
        } else if (p.tp.cfl1) {  // sources per shift combination resolved once per cell, then lookups
          if (b0 == 0) {
            if (tg < 27) {
              int d[3] = {tg % 3 - 1, (tg / 3) % 3 - 1, tg / 9 - 1};
              int flip = 0;
              c.sbase[tg] = source_resolve(p.f_in, p.tp, cc_cell, d, n, flip);
              c.sflip[tg] = (int8_t)flip;
            }
            named_bar(1, GT);
          }
#pragma unroll
          for (int j = 0; j < B; ++j) {
            const int e = tg + (b0 + j) * GT;
            const int x = e % N, y = (e / N) % N, zz = rank * NP + e / (N * N);
            const int combo = (c.delta[0][x] + 1) + 3 * (c.delta[1][y] + 1) + 9 * (c.delta[2][zz] + 1);
            const int k = x + N * (y + N * zz);
            FKS_CHECK(combo >= 0 && combo < 27 && k < n);
            v[j] = c.sbase[combo][c.sflip[combo] ? mirror_k(k, x, y, zz, c.sflip[combo], N) : k];
          }
        } else {
#pragma unroll
          for (int j = 0; j < B; ++j) {
            const int e = tg + (b0 + j) * GT;
            const int x = e % N, y = (e / N) % N, zz = rank * NP + e / (N * N);
            v[j] = gather_fstar(p.f_in, p.tp, cc_cell, x + N * (y + N * zz), x, y, zz, n, c.delta);
          }
        }
#pragma unroll
        for (int j = 0; j < B; ++j) {
          const int e = tg + (b0 + j) * GT;
          const int x = e % N, y = (e / N) % N, zl = e / (N * N);
          pln[zl * N * N + y * N + swz(y, x)] = make_double2(v[j], 0.0);
        }
      }
      named_bar(1, GT);
      if constexpr (C::FS_TMEM) {  // column (tx, ., tl) of f* -> the xy thread's TMEM cache
        if (ncell >= 2) {           // the xy group has finished with this parity (cell ncell - 2)
          mbar_wait(c.fse + par, ((ncell >> 1) - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        }
        const double2* col = pln + tl * N * N;
#pragma unroll
        for (int ch = 0; ch < N / 16; ++ch) {
          uint32_t v[32];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int y = ch * 16 + i;
            const double f = col[y * N + swz(y, tx)].x;
            v[2 * i] = __double2loint(f);
            v[2 * i + 1] = __double2hiint(f);
          }
          tmem_st32(fs_addr + ch * 32, v);
        }
        tmem_wait_st();
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        mbar_arrive(c.fsb + par);
        named_bar(1, GT);  // every column read before the rows are transformed in place
      }
      {
        double2 r[N];
        double2* row = pln + tl * N * N + tx * N;  // row y = tx of plane tl
#pragma unroll
        for (int x = 0; x < N; ++x) r[x] = row[swz(tx, x)];
        fft<N, -1>(r);
#pragma unroll
        for (int x = 0; x < N; ++x) row[swz(tx, x)] = r[x];
        TSTAMPB(1);
      }
      named_bar(1, GT);
      {
        double2 cc[N];
        const double2* col = pln + tl * N * N;  // column l_x = tx of plane tl
#pragma unroll
        for (int y = 0; y < N; ++y) cc[y] = col[y * N + swz(y, tx)];
        fft<N, -1>(cc);
        // the slot's previous item must have been read by every consumer
        if (tg == 0 && s_fwd / NB > 0) sync_wait_free(&gs->cons[s_fwd % NB], WP * (s_fwd / NB), 0u);
        named_bar(1, GT);  // also: every plane read, the table buffers may be refilled
        if (tg_leader) {
          load_tab(0);
          if (D > 1) load_tab(1);
        }
        FKS_CHECK(zpl >= 0 && zpl < N && tx < N);
        double2* Wb = c.W + (s_fwd % NB) * C::WBUF + (size_t)zpl * C::WPLANE;
#pragma unroll
        for (int l = 0; l < N; ++l) Wb[l * N + swz(l, tx)] = cc[l];
      }
      named_bar(1, GT);
      if (tg == 0) sync_signal_n(&gs->prod[s_fwd % NB], NW);
      TSTAMPB(2);
    }
    {  // z transform of the forward item of every CTA -> f^ pencil in TMEM
      const unsigned slot = s_fwd % NB, use = s_fwd / NB;
      if (tg == 0) sync_wait(&gs->prod[slot], WP * (use + 1));
      TSTAMPB(9);
      named_bar(1, GT);
      double2 x[N];
      const double2* Wb = c.W + slot * C::WBUF + (size_t)ly * N + swz(ly, tx);
#pragma unroll
      for (int zz = 0; zz < N; ++zz) x[zz] = __ldcg(Wb + (size_t)zz * C::WPLANE);
      fft<N, -1>(x);
#pragma unroll
      for (int ch = 0; ch < N / 8; ++ch) {
        uint32_t v[32];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          v[4 * i + 0] = __double2loint(x[ch * 8 + i].x);
          v[4 * i + 1] = __double2hiint(x[ch * 8 + i].x);
          v[4 * i + 2] = __double2loint(x[ch * 8 + i].y);
          v[4 * i + 3] = __double2hiint(x[ch * 8 + i].y);
        }
        tmem_st32(taddr + ch * 32, v);
      }
      tmem_wait_st();
      named_bar(1, GT);  // every column of the forward item read
      TSTAMPB(10);
      if (tg == 0) sync_signal_relaxed_n(&gs->cons[slot], NW);
      seq = s_fwd + 1;
      pub = seq;  // first z item of this cell
    }
#pragma unroll 1
    for (int j = 0; j < D; ++j) {
      TSTAMP(2048 + j * 8);
      const unsigned slot = seq % NB, use = seq / NB;
      double2 x[N];
      // slot free once its previous item has been read by every consumer (polled early)
      const unsigned cons_seen = lane == 0 && use > 0 ? ld_relaxed(&gs->cons[slot]) : 0u;
      const int tb = j & 1;
      mbar_wait(c.tbar + tb * NTG + tgi, (tphase >> tb) & 1u);
      tphase ^= 1u << tb;
      TSTAMP(2048 + j * 8 + 1);
      zpass_compute<N, P>(taddr, c.tbuf + tb * TB, tx, tm, x);
      TSTAMP(2048 + j * 8 + 2);
      __syncwarp();  // the warp's reads of table buffer tb and its z(j-1) stores precede this
      if constexpr (TGW == 2) {
        // the partner warp only announces it is done; the loading lane waits for it (mbarrier)
        if (lane == 0) mbar_arrive(c.tempty + tb * NTG + tgi);
        if (tg_leader && j + 2 < D) {
          mbar_wait(c.tempty + tb * NTG + tgi, (tephase >> tb) & 1u);
          load_tab(j + 2);  // into the buffer just freed
        }
        tephase ^= 1u << tb;
      } else {
        if (tg_leader && j + 2 < D) load_tab(j + 2);  // into the buffer just freed
      }
      if (lane == 0) {
        if (use > 0) sync_wait_free(&gs->cons[slot], WP * use, cons_seen);
        // Publish this warp's z items in batches of FKS_PUB: one release fence (which waits for the
        // SM's outstanding stores, ~1-2k cycles) per batch, then relaxed adds.
        if (seq - pub >= FKS_PUB) {
          asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
          for (; pub < seq; ++pub) sync_signal_relaxed(&gs->prod[pub % NB]);
        }
      }
      __syncwarp();
      zpass_store<N, P>(x, c.W + slot * C::WBUF, ly, tx);
      TSTAMP(2048 + j * 8 + 3);
      ++seq;
    }
    __syncwarp();  // this warp's last stores precede the release
    if (lane == 0) {
      asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
      for (; pub < seq; ++pub) sync_signal_relaxed(&gs->prod[pub % NB]);
    }
    named_bar(1, GT);  // every warp done with the tables before the next forward reuses them
  }
}

// ---- xy group: xy(j) and the gain accumulation, epilogue ---------------------------------
template <int N, int P>
__device__ __forceinline__ void xy_group(const StepParams& p, const Ctx3<N, P>& c, uint32_t taddr) {
  using C = Cfg3<N, P>;
  constexpr int NP = C::NP, GT = C::GT, NB = C::NBUF;
  constexpr int n = N * N * N;
  constexpr uint32_t kPlaneBytes = C::PSLAB * 16;
  const int D = p.A + 1;
  const int rank = c.rank, cid = c.cid, tg = c.tg, tx = c.tx, tl = c.tl;
  GroupSync* gs = c.gs;
  uint32_t wphase = 0;  // bit b = parity of plane buffer b
  unsigned seq = 0;     // exchange-buffer sequence index of the next item
  unsigned ncell = 0;   // cells done by this group
  constexpr int NW = C::NW, WPL = C::WPL;
  constexpr unsigned WP = NW * P;  // signals per exchange item
  const int w = tg >> 5, lane = tg & 31;
  // lane 0 of each warp: its planes of W(item s) -> plane buffer b, once every producer has
  // published the item (`seen`: an earlier relaxed read of the counter)
  auto issue_load = [&](unsigned s, int b, unsigned seen) {
    const unsigned* ctr = &gs->prod[s % NB];
    const unsigned target = WP * (s / NB + 1);
    // The producers' release put their stores in L2 before the counter moved, and the bulk copy
    // reads L2 after the (control-dependent) check, so a relaxed observation is enough here.
    if ((int)(seen - target) < 0) sync_wait(ctr, target);
    asm volatile("fence.proxy.async.global;\n" ::: "memory");  // generic-proxy stores -> bulk reads
    bulk_load(c.pln0 + b * C::PSLAB + (size_t)w * WPL * N * N,
              c.W + (s % NB) * C::WBUF + (size_t)(rank * NP + w * WPL) * N * N, kPlaneBytes / NW,
              c.wbar + b * NW + w);
  };
  for (int it = cid; it < p.ncells; it += c.ncl, ++ncell) {
    const int64_t cell = p.cell_list ? p.cell_list[it] : it;
    const CellCoord cc_cell = cell_coord(p.tp, cell);
    const int z = rank * NP + tl;
    const unsigned par = ncell & 1;
    const uint32_t saddr = taddr + C::FHAT_COLS + par * 2 * N;  // f* column cache of this cell
    // f*(tx, y, z) for y in [16 ch, 16 ch + 16) from the column cache
    auto fs_chunk = [&](int ch, double (&fs)[16]) {
      uint32_t v[32];
      tmem_ld32(saddr + ch * 32, v);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 16; ++i) fs[i] = __hiloint2double(v[2 * i + 1], v[2 * i]);
    };
    auto fs_acquire = [&]() {  // the z group wrote this cell's f* cache
      if constexpr (C::FS_TMEM) {
        mbar_wait(c.fsb + par, (ncell >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      }
    };
    auto fs_release = [&]() {  // last read of this cell's f* cache done
      if constexpr (C::FS_TMEM) {
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        mbar_arrive(c.fse + par);
      }
    };
    seq += 1;  // the forward item (z group's)
    TSTAMPB(3);
    if (lane == 0) issue_load(seq, 0, 0u);  // z(0): both plane buffers are free here
    double q[N];  // gain accumulator of column (tx, tl), then Q
#pragma unroll
    for (int y = 0; y < N; ++y) q[y] = 0.0;
#pragma unroll 1
    for (int d = 0; d < D; ++d) {
      TSTAMP(d * 8);
      const int pb = d & 1;
      FKS_CHECK(tl >= 0 && tl < NP && tx < N && d <= p.A);
      double2* pln = c.pln0 + pb * C::PSLAB;
      mbar_wait(c.wbar + pb * NW + w, (wphase >> pb) & 1u);
      wphase ^= 1u << pb;
      unsigned prod_seen = 0;
      if (lane == 0) {
        sync_signal_relaxed(&gs->cons[seq % NB]);  // this warp's planes of W(d) read
        if (d + 1 < D) prod_seen = ld_relaxed(&gs->prod[(seq + 1) % NB]);  // checked after pass 0
      }
      TSTAMP(d * 8 + 1);
      // x pass (rows, in place) then y pass (columns, accumulate): one FFT body for both
      // passes keeps the hot loop's instruction footprint small.
#pragma unroll 1
      for (int pass = 0; pass < 2; ++pass) {
        double2* pl = pln + tl * N * N;  // pass 0: row y = tx; pass 1: column x = tx
        auto at = [&](int i) { return pass == 0 ? tx * N + swz(tx, i) : i * N + swz(i, tx); };
        double2 cc[N];
#pragma unroll
        for (int x = 0; x < N; ++x) cc[x] = pl[at(x)];
        fft<N, +1>(cc);
        if (pass == 0) {
#pragma unroll
          for (int x = 0; x < N; ++x) pl[at(x)] = cc[x];
          __syncwarp();  // rows done; this warp has also finished xy(d-1): its buffer pb^1 is free
          if (lane == 0 && d + 1 < D) issue_load(seq + 1, pb ^ 1, prod_seen);
          TSTAMP(d * 8 + 2);
        } else if (d < p.A) {
#pragma unroll
          for (int y = 0; y < N; ++y) q[y] = fma(cc[y].x, cc[y].y, q[y]);
        } else if constexpr (C::FS_TMEM) {
          fs_acquire();
#pragma unroll
          for (int ch = 0; ch < N / 16; ++ch) {
            double fs[16];
            fs_chunk(ch, fs);
#pragma unroll
            for (int i = 0; i < 16; ++i) q[ch * 16 + i] = q[ch * 16 + i] - fs[i] * cc[ch * 16 + i].x;
          }  // Q = G - f* c
        } else {
#pragma unroll
          for (int y = 0; y < N; ++y) {
            const double fs = gather_fstar(p.f_in, p.tp, cc_cell, tx + N * (y + N * z), tx, y, z, n, c.delta);
            q[y] = q[y] - fs * cc[y].x;  // Q = G - f* c
          }
        }
      }
      TSTAMP(d * 8 + 3);
      ++seq;
    }
    TSTAMPB(4);
    // a8 + a9: projection and Euler (or write Q)
    FKS_CHECK(cell >= 0 && cell < p.tp.ncells_total && z < N);
    double* out = p.f_out + cell * (int64_t)n;
    if (p.mode == 0) {
      fs_release();
#pragma unroll
      for (int y = 0; y < N; ++y) out[tx + N * (y + N * z)] = q[y];
    } else {
      const double vx = node_v(tx, p.L, p.dv), vz = node_v(z, p.L, p.dv);
      double lam[5] = {0, 0, 0, 0, 0};
      if (p.project) {
        double m[5] = {0, 0, 0, 0, 0};
#pragma unroll
        for (int y = 0; y < N; ++y) {
          const double vy = node_v(y, p.L, p.dv);
          m[0] += q[y];
          m[1] += vx * q[y];
          m[2] += vy * q[y];
          m[3] += vz * q[y];
          m[4] += (vx * vx + vy * vy + vz * vz) * q[y];
        }
        // group reduction of the 5 moments in a fixed order (warps, then ranks): deterministic
#pragma unroll
        for (int k = 0; k < 5; ++k) {
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) m[k] += __shfl_xor_sync(0xffffffffu, m[k], o);
        }
        double* wpart = c.part + 8;  // [NW][5]
        constexpr int NW = GT / 32;
        if ((tg & 31) == 0) {
#pragma unroll
          for (int k = 0; k < 5; ++k) wpart[(tg >> 5) * 5 + k] = m[k];
        }
        named_bar(2, GT);
        double* gpart = gs->partial[ncell & 1][rank];
        if (tg < 5) {
          double sum = 0.0;
          for (int w = 0; w < NW; ++w) sum += wpart[w * 5 + tg];
          __stcg(gpart + tg, sum);
        }
        named_bar(2, GT);
        if (tg == 0) {
          TSTAMPB(5);
          sync_signal(&gs->part);
          sync_wait(&gs->part, P * (ncell + 1));
          double mu[5] = {0, 0, 0, 0, 0};
          for (int r = 0; r < P; ++r) {
#pragma unroll
            for (int k = 0; k < 5; ++k) mu[k] += __ldcg(&gs->partial[ncell & 1][r][k]);
          }
#pragma unroll
          for (int a = 0; a < 5; ++a) {
            double sacc = 0.0;
#pragma unroll
            for (int b = 0; b < 5; ++b) sacc = fma(p.Ginv[a * 5 + b], mu[b], sacc);
            c.part[a] = sacc;
          }
        }
        named_bar(2, GT);
        TSTAMPB(6);
#pragma unroll
        for (int a = 0; a < 5; ++a) lam[a] = c.part[a];
      }
      bool bad = false;
      const double* base = p.mode == 2 ? p.f_base + cell * (int64_t)n : nullptr;
      auto euler = [&](int y, double fs) {
        const double vy = node_v(y, p.L, p.dv);
        const int k = tx + N * (y + N * z);
        const double corr = lam[0] + lam[1] * vx + lam[2] * vy + lam[3] * vz + lam[4] * (vx * vx + vy * vy + vz * vz);
        double o = fma(p.dt_tau, q[y] - corr, fs);
        if (base) o = 0.5 * (o + __ldcs(base + k));  // Heun: (f* + E(f1)) / 2 (NEXT-4)
        bad |= !isfinite(o);
        out[k] = o;
      };
      if constexpr (C::FS_TMEM) {
#pragma unroll
        for (int ch = 0; ch < N / 16; ++ch) {
          double fs[16];
          fs_chunk(ch, fs);
#pragma unroll
          for (int i = 0; i < 16; ++i) euler(ch * 16 + i, fs[i]);
        }
        fs_release();
      } else {
#pragma unroll
        for (int y = 0; y < N; ++y)
          euler(y, gather_fstar(p.f_in, p.tp, cc_cell, tx + N * (y + N * z), tx, y, z, n, c.delta));
      }
      if (bad) atomicOr(p.nonfinite, 1);
    }
    named_bar(2, GT);  // c.part / plane buffers free for the next cell
    TSTAMPB(7);
  }
}

template <int N, int P>
__global__ void __launch_bounds__(Cfg3<N, P>::THREADS, 1) k_step3d(const StepParams p) {
  using C = Cfg3<N, P>;
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEM);
  Ctx3<N, P> c;
  c.tbuf = reinterpret_cast<double2*>(smem + C::OFF_TBUF);
  c.pln0 = reinterpret_cast<double2*>(smem + C::OFF_PLN);
  c.tbar = reinterpret_cast<uint64_t*>(smem + C::OFF_MBAR);
  c.wbar = c.tbar + 2 * C::NTG;
  c.fsb = c.wbar + 2 * C::NW;
  c.fse = c.fsb + 2;
  c.tempty = c.fse + 2;
  c.part = reinterpret_cast<double*>(smem + C::OFF_PART);
  c.sbase = reinterpret_cast<const double**>(smem + C::OFF_SBASE);
  c.sflip = reinterpret_cast<int8_t*>(smem + C::OFF_SFLIP);
  int8_t (*sdelta)[kMaxN] = reinterpret_cast<int8_t (*)[kMaxN]>(smem + C::OFF_DELTA);
  load_delta(p.tp, sdelta);
  c.delta = sdelta;
  c.rank = (int)(blockIdx.x % P);
  c.cid = blockIdx.x / P;
  c.ncl = gridDim.x / P;
  const int t = threadIdx.x;
  const bool zg = t < C::GT;
  c.tg = zg ? t : t - C::GT;
  c.tx = c.tg % N;
  c.tl = c.tg / N;
  c.W = p.scratch + (size_t)c.cid * C::NBUF * C::WBUF;
  c.gs = reinterpret_cast<GroupSync*>(p.sync) + c.cid;
  FKS_CHECK(P <= 16 && C::SMEM <= 232448);

  if (t < 32) {  // warp 0 owns the TMEM allocation
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "n"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  if (t == 0) {
    for (int i = 0; i < 2 * C::NTG; ++i) mbar_init(c.tbar + i, 1);
    for (int i = 0; i < 2 * C::NW; ++i) mbar_init(c.wbar + i, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(c.fsb + i, C::GT);
      mbar_init(c.fse + i, C::GT);
      for (int g = 0; g < C::NTG; ++g) mbar_init(c.tempty + i * C::NTG + g, C::TGW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tbase = *tmem_slot;
  FKS_CHECK((tbase & 0xffffu) + C::TMEM_COLS <= 512u && C::USED_COLS <= C::TMEM_COLS);
  // this thread's TMEM lane: warp quarter base + lane in warp (row field = bits 31..16)
  const uint32_t taddr = tbase + ((uint32_t)(32 * ((t >> 5) & 3)) << 16);
  if (zg) z_group<N, P>(p, c, taddr);
  else xy_group<N, P>(p, c, taddr);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "n"(C::TMEM_COLS) : "memory");
}

template <int N, int P>
static cudaError_t prep() {
  using C = Cfg3<N, P>;
  return cudaFuncSetAttribute(k_step3d<N, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
}

// Cooperative launch: all P * ngroups CTAs are co-resident (one per SM), which the group
// synchronisation through L2 requires.
template <int N, int P>
static cudaError_t launch3(const StepParams& p, int ngroups, cudaStream_t s) {
  using C = Cfg3<N, P>;
  cudaError_t e = prep<N, P>();
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ngroups * P);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_step3d<N, P>, p);
}

template <int N, int P>
static int max_groups3() {
  if (prep<N, P>() != cudaSuccess) return 0;
  int per_sm = 0, dev = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step3d<N, P>, Cfg3<N, P>::THREADS, Cfg3<N, P>::SMEM) !=
      cudaSuccess)
    return 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return per_sm * sms / P;
}

cudaError_t launch_step3d(int N, const StepParams& p, int ngroups, cudaStream_t s) {
  switch (N) {
    case 8: return launch3<8, 2>(p, ngroups, s);
    case 16: return launch3<16, 8>(p, ngroups, s);
    case 32: return launch3<32, 8>(p, ngroups, s);
    default: return cudaErrorInvalidValue;
  }
}

int max_active_clusters3d(int N) {
  switch (N) {
    case 8: return max_groups3<8, 2>();
    case 16: return max_groups3<16, 8>();
    case 32: return max_groups3<32, 8>();
    default: return 0;
  }
}

size_t scratch_elems3d(int N) { return (size_t)Cfg3<32, 8>::NBUF * N * N * N; }

size_t sync_bytes3d() { return sizeof(GroupSync); }

// Host-side table layout of the 3D kernel for N: T3[p][rank][row][l_x] (see Cfg3::SLABR).
int table_layout3d(int N, int* P_out, int* NP_out, int* slabr_out) {
  switch (N) {
    case 8: *P_out = 2; *NP_out = Cfg3<8, 2>::NP; *slabr_out = Cfg3<8, 2>::SLABR; return 0;
    case 16: *P_out = 8; *NP_out = Cfg3<16, 8>::NP; *slabr_out = Cfg3<16, 8>::SLABR; return 0;
    case 32: *P_out = 8; *NP_out = Cfg3<32, 8>::NP; *slabr_out = Cfg3<32, 8>::SLABR; return 0;
    default: return -1;
  }
}

#ifdef FKS_TIMING
extern "C" int fks_debug_tstamps(long long* out, int count) {
  return (int)cudaMemcpyFromSymbol(out, g_tstamp, sizeof(long long) * count);
}
#endif

}  // namespace fks
