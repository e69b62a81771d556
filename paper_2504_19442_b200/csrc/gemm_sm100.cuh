// Persistent, warp-specialised tcgen05 GEMM for sm_100a with the two fused
// tensor-parallel epilogues of the hot path:
//
//   MODE_AG : C[m, n] = concat_r(A_shard_r) @ B.  The TMA-producer warp gates
//             every A tile of chunk c on the per-source flag ready[c] (set
//             by the owner's push), so tiles of the local shard start at
//             once and remote chunks are consumed as they land.
//             Reference: pipelines.py:97-150 (ag_gemm), collectives.py:83-102.
//   MODE_RS : rows of chunk d of (A @ B) are written as bf16 straight into
//             rank d's staging slot `rank` (peer TMA store over NVLink) and
//             a release-add on d's per-source counter publishes them.
//             Reference: pipelines.py:179-216 (gemm_rs) + collectives.py:153-161.
//
// Layout: A is K-major (row-major m x k), B is MN-major (row-major k x n, the
// reference's argument layout, pipelines.py:112).  Both are staged by TMA with
// 128-byte swizzle.  A CTA pair (cta_group::2) computes a 256 x BN tile; each
// CTA owns 128 rows of A and BN/2 columns of B in shared memory and 128 x BN
// fp32 accumulator columns in TMEM (double buffered across tiles).
//
// Warp roles (224 threads): warp 0 TMA producer, warp 1 MMA issuer (leader
// CTA), warps 2..5 epilogue (TMEM -> regs -> bf16 -> swizzled smem -> TMA
// store; warp 2 allocates TMEM), warp 6 own-slot copier (AG).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "ptx.cuh"

namespace shb {

constexpr int kMaxWorld = 16;
constexpr int MODE_AG = 0;
constexpr int MODE_RS = 1;

// Flags a kernel releases when its last CTA retires, in place of stream
// memory operations after the launch.  Both users are write-after-read
// flags -- AG done[rank] ("finished reading my gather buffer") and RS
// producer[rank] ("finished reading my staging slots"): the peer overwrites
// memory of THIS GPU once it sees them, so what must precede the flag are
// reads served by this GPU's L2, all of them consumed (values used, bulk
// loads completed on their mbarriers) before the CTA retires.  The last CTA
// therefore orders them at gpu scope (acq_rel counting + fence) and stores
// the flags relaxed at system scope; a system-scope release would also wait
// for every earlier write of the kernel to become visible system-wide.
// TP=8 proxy, M=1024, preset flags, per call: AG 73.0 us with the 7 stream
// memory ops (~2.8 us each in the GPU front end), 60.4 with st.release.sys
// here (or a one-warp store kernel after the GEMM), 53.8 with this form =
// the call without any flag store (profiles/r2_exit_release/).
// SHB_EXIT_SYS_RELEASE=1 selects the system-scope release stores.
struct ExitRelease {
  uint64_t* ptr[kMaxWorld];
  uint64_t value;
  unsigned int* ctr;  // CTAs retired so far; the last one resets it to 0
  int count;          // 0: nothing to release
  int sys_release;    // 1: st.release.sys (see above)
};

// One thread per CTA, after a CTA-wide barrier that follows every read the
// flags vouch for.  The counter reset is ordered before the next launch on
// the stream (the GEMM's main body starts after griddepcontrol.wait, the
// reduction after its GEMM's prologue).
__device__ __forceinline__ void exit_release(const ExitRelease& r) {
  if (r.count <= 0) return;
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(r.ctr) : "memory");
  if (old + 1 == gridDim.x) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(r.ctr) : "memory");
    for (int i = 0; i < r.count; ++i) {
      if (r.sys_release)
        st_release_sys(r.ptr[i], r.value);
      else
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(r.ptr[i]), "l"(r.value) : "memory");
    }
  }
}

struct TileParams {
  int rows;       // rows per chunk (m / world)
  int n, k;
  int world, rank;
  int mblk, nblk;  // m-blocks per chunk, n-blocks
  int num_tiles;   // world * mblk * nblk
  int group_m;     // raster group (m-blocks) for L2 reuse
  // raster regions: consecutive chunk positions [reg_s0[r], reg_s0[r+1])
  // whose m-blocks form one raster (group reg_gm[r]; reg_g0[r] groups come
  // before it).  nreg = 0: one region per position with group_m.
  int nreg;
  // chunks of <= 128 rows (TP=8 at M=1024): the two CTAs of a pair tile
  // take two consecutive chunk positions (128 rows each) instead of 1-CTA
  // tiles (a 256-row tile would be half padding); one raster over the pairs
  int pair_chunks;
  int reg_s0[kMaxWorld + 1];
  int reg_gm[kMaxWorld];
  int reg_g0[kMaxWorld];
  int serpentine;  // odd raster groups walk n backwards (2: parity continues across chunks)
  int kserp;       // every other data-parallel tile of a cluster walks K backwards
  int order[kMaxWorld];  // chunk visit order (reference swizzle.py)
  uint64_t epoch;
  const uint64_t* ready;              // AG: my pad, ready[src] (written by src)
  int ag_sub;                         // AG: row ranges per pushed shard (ready counts them)
  int ag_sub_rows;                    // AG: rows per range (multiple of 256)
  uint64_t* rs_count[kMaxWorld];      // RS: &pad_d[reduction + rank]
  uint32_t rs_gpu_scope;              // RS: bit d -> chunk d's counter released at gpu scope
                                      // (my own chunk: staging and its reducer are on this GPU)
  const uint64_t* rs_free;            // RS: my pad, producer[d] >= epoch-1: d reduced last call
  const uint64_t* rs_mine;            // RS: my pad, reduction[s] (elements delivered by s)
  uint64_t rs_target;                 // RS: epoch * rows * n, a chunk fully delivered
  const uint16_t* staging_local;      // RS: my staging buffer (W slots of rows x n)
  int fuse_reduce;                    // RS: reduce my chunk in the epilogue of its tiles
  int red_help;                       // RS fused: idle warps share the own-chunk reduction
  uint16_t* out_rows;                 // RS: the reduced output rows (rows x n, row-major)
  int copy_own;                       // AG: store own-chunk A stages into gathered[rank]
  // optional timeline: per CTA `trace_cap` records of 4 u64 {kind|aux, t0, t1, tile}
  // (%globaltimer ns); producer records fill from the front, epilogue (warp 2)
  // records from the middle.  Kinds: 1 chunk-flag wait (AG), 2 tile
  // epilogue (t0 = accumulator ready, t1 = stores issued), 3 peer-arrival
  // wait (fused RS), 4 CTA lifetime, 5 MMA accumulator wait (aux = summed
  // operand-stage waits of the item, ns; MMA warp, last quarter of the slots).
  uint64_t* trace;
  int trace_cap;
  uint64_t l2_hint_a, l2_hint_b;      // TMA L2 cache policies of the operand loads
  uint64_t l2_hint_store;             // RS: L2 policy of the staging / output stores
  uint64_t l2_hint_own;               // AG: L2 policy of the own-slot stores; RS: of the
                                      // own chunk's staging stores (fused, W > 1)
  // stream-K tail: tiles [0, dp_tiles) are data-parallel (one cluster each);
  // the k-blocks of tiles [dp_tiles, num_tiles) are split evenly over all
  // clusters.  A cluster's range is walked backwards, so the partial head of a
  // tile is produced first and the cluster finishing its tail (k_end = K)
  // reduces the partials from the fp32 workspace.
  int dp_tiles;
  // AG at W>1: the clusters whose first tile belongs to a remote chunk (the
  // last sk_late clusters when the own chunk has fewer tiles than clusters)
  // start ~one chunk transfer late; they get sk_late_units fewer stream-K
  // units so that every cluster finishes together.  0: even partition.
  int sk_late;
  int sk_late_units;
  // dynamic scheduling of the data-parallel tiles: the leader CTA's producer
  // claims tile ids from a global counter (zeroed before the launch) and
  // broadcasts them through a small smem ring to every role of the pair, so
  // the tiles in flight stay a compact window in launch order (L2 reuse) and
  // faster clusters take more tiles.  The stream-K tail stays static.
  int* tile_counter;                  // null: static stride schedule
  float* ws;                          // clusters x (CG*128) x BN fp32 partials
  uint64_t* ws_flags;                 // clusters x CG x 4 epilogue warps
  uint64_t ws_epoch;                  // launch counter of this workspace
  ExitRelease rel;                    // AG: done[rank] on every peer; fused RS: producer[rank]
  // Wave lockstep: cluster c runs data-parallel tiles c, c+C, c+2C, ...; the
  // i-th of them forms wave i.  When K is long, the operand reuse between the
  // tiles of a wave comes only from their walking K together (a block's
  // k-slice must still be in L2 when the next tile asks for it), and clusters
  // drift apart over many waves.  The leader producer publishes
  // wave_tag | tiles_issued in wave_flags[cluster] and, before issuing wave i,
  // waits (bounded, a hint -- never an error) until every cluster that has a
  // wave i-1 tile has issued it.  MMA and epilogue are not gated, so the wait
  // is absorbed by the smem stages.  null: off.
  uint64_t* wave_flags;
  uint64_t wave_tag;
  int* err;                           // host-mapped error word
  uint64_t timeout_ns;
};

// RS: publish `cnt` more elements of chunk d delivered (data before count:
// the caller completed the tile's bulk stores and fenced the async proxy)
__device__ __forceinline__ void rs_publish(const TileParams& p, int d, uint64_t cnt) {
  if ((p.rs_gpu_scope >> d) & 1u)
    red_add_release_gpu(p.rs_count[d], cnt);
  else
    red_add_release_sys(p.rs_count[d], cnt);
}

__device__ __forceinline__ void trace_rec(const TileParams& p, int slot, uint64_t kind_aux,
                                          uint64_t t0, uint64_t t1, uint64_t tile) {
  if (slot >= p.trace_cap) return;
  uint64_t* r = p.trace + ((size_t)blockIdx.x * p.trace_cap + slot) * 4;
  r[0] = kind_aux;
  r[1] = t0;
  r[2] = t1;
  r[3] = tile;
}

// Warp-wide: wait until every cluster d holding a data-parallel tile of wave
// i-1 (d + (i-1)*C < dp_tiles) has published >= i issued tiles.  Bounded to
// 2 ms: the lockstep is a locality hint, a straggler must never stall a call.
__device__ __forceinline__ void wave_wait(const uint64_t* flags, uint64_t tag, int i, int C,
                                          int dp_tiles) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t want = tag | (uint64_t)i;
  const long long first = (long long)(i - 1) * C;
  uint64_t t0 = 0;
  for (;;) {
    bool ok = true;
    for (int d = (int)lane; d < C; d += 32)
      if (first + d < dp_tiles && ld_relaxed_gpu(flags + d) < want) ok = false;
    if (__all_sync(0xffffffffu, ok)) return;
    const uint64_t now = globaltimer();
    if (t0 == 0) t0 = now;
    else if (now - t0 > 2000000ull) return;
    __nanosleep(64);
  }
}

struct WorkItem {
  int t, kb0, kb1, kind;  // kind: 0 whole tile, 1 partial head (to workspace), 2 finishing tail
};

constexpr int kRing = 4;

// Tile-id ring of the dynamic scheduler (one per CTA, same smem offset in
// both CTAs of a pair; `empty` is only used in the leader CTA).
struct TileRing {
  int ids[kRing];
  uint64_t full[kRing];
  uint64_t empty[kRing];
};

// Identical sequence of work items for the producer, MMA and epilogue roles.
// role: 0 = fetcher (leader producer), 1 = consumer warp, 2 = not a ring user
struct WorkIter {
  int t, C, KB, dp;
  long long u0, u, U;
  // weighted stream-K partition: the last L clusters (late starters) own
  // y = x - d units each, the others x (see TileParams::sk_late)
  int L;
  long long x, y;
  __device__ __forceinline__ long long start(int i) const {
    if (L == 0) return U * i / C;
    const int F = C - L;
    const long long s = i <= F ? (long long)i * x : (long long)F * x + (long long)(i - F) * y;
    return s < U ? s : U;
  }
  // dynamic phase
  TileRing* ring;
  int* counter;
  int role, rslot, cg, pending;
  uint32_t rphase;
  bool dyn;
  __device__ __forceinline__ void init(const TileParams& p, int cid, int nclusters, int kb,
                                       TileRing* r = nullptr, int ring_role = 2, int cgs = 1) {
    C = nclusters;
    KB = kb;
    dp = p.dp_tiles;
    t = cid;
    U = (long long)(p.num_tiles - dp) * KB;
    L = (p.sk_late > 0 && p.sk_late < nclusters && U > 0) ? p.sk_late : 0;
    if (L) {
      const long long d = p.sk_late_units;
      x = (U + (long long)L * d + C - 1) / C;
      y = x - d;
      if (y < 1) { L = 0; }  // host clamps d; never an empty or negative share
    }
    u0 = start(cid);
    u = start(cid + 1);
    ring = r;
    counter = p.tile_counter;
    role = ring_role;
    cg = cgs;
    rslot = 0;
    rphase = 0;
    dyn = counter != nullptr && dp > 0;
    // the first tile of every cluster is static (cid); later ones come from
    // the counter, fetched one tile ahead so the atomic's latency is hidden
    pending = cid;
  }
  // next data-parallel tile id from the ring (-1: exhausted); warp-wide call
  __device__ __forceinline__ int ring_next() {
    const uint32_t lane = threadIdx.x & 31;
    int id = -1;
    if (role == 0) {
      mbar_wait_cluster(&ring->empty[rslot], rphase ^ 1);
      if (lane == 0) {
        id = pending < dp ? pending : -1;
        if (id >= 0) pending = C + atomicAdd(counter, 1);
        ring->ids[rslot] = id;
        if (cg == 2) {
          asm volatile(
              "{\n\t.reg .b32 ra;\n\t"
              "mapa.shared::cluster.u32 ra, %0, 1;\n\t"
              "st.shared::cluster.u32 [ra], %1;\n\t}" ::"r"(smem_u32(&ring->ids[rslot])),
              "r"(id)
              : "memory");
          mbar_arrive_cluster(&ring->full[rslot], 1);
        }
        mbar_arrive(&ring->full[rslot]);
      }
      id = __shfl_sync(0xffffffffu, id, 0);
    } else {
      mbar_wait_cluster(&ring->full[rslot], rphase);
      id = *reinterpret_cast<volatile int*>(&ring->ids[rslot]);
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&ring->empty[rslot], 0);
    }
    if (++rslot == kRing) { rslot = 0; rphase ^= 1; }
    return id;
  }
  __device__ __forceinline__ bool next(WorkItem& w) {
    if (dyn) {
      const int id = ring_next();
      if (id >= 0) {
        w.t = id; w.kb0 = 0; w.kb1 = KB; w.kind = 0;
        return true;
      }
      dyn = false;
      t = dp;  // data-parallel tiles exhausted: continue with the stream-K range
    } else if (t < dp) {
      w.t = t; w.kb0 = 0; w.kb1 = KB; w.kind = 0;
      t += C;
      return true;
    }
    if (u > u0) {
      const long long tile = (u - 1) / KB;
      const long long ts = tile * KB;
      const long long sb = u0 > ts ? u0 : ts;
      w.t = dp + (int)tile;
      w.kb0 = (int)(sb - ts);
      w.kb1 = (int)(u - ts);
      w.kind = (w.kb0 == 0 && w.kb1 == KB) ? 0 : (w.kb1 == KB ? 2 : 1);
      u = sb;
      return true;
    }
    return false;
  }
  // first cluster whose range [start(i), start(i+1)) contains stream-K unit v
  __device__ __forceinline__ int owner(long long v) const {
    int i;
    if (L == 0) {
      i = (int)(v * C / U);
    } else {
      const int F = C - L;
      i = v < (long long)F * x ? (int)(v / x) : F + (int)((v - (long long)F * x) / y);
      if (i > C - 1) i = C - 1;
    }
    while (i + 1 < C && start(i + 1) <= v) ++i;
    while (i > 0 && start(i) > v) --i;
    return i;
  }
};

struct TensorMaps {
  CUtensorMap a_own;  // AG: a_shard {k, rows}
  CUtensorMap a_all;  // AG: gathered {k, rows, W}; RS: a {k, rows, W}
  CUtensorMap b;      // {n, k}
  CUtensorMap c;      // AG: C {n, rows, W}
  CUtensorMap out[kMaxWorld];  // RS: dest d's staging slot `rank`, {n, rows}
  CUtensorMap own_slot;        // AG: my gather slot `rank`, {k, rows} (box = one A stage)
};

// Tile t -> (chunk, m-block, n-block).  Tiles are enumerated position by
// position of the chunk order.  Consecutive positions may form ONE raster
// region whose m-blocks are those of all its chunks (RS: every chunk no
// epilogue waits behind; AG: pairs of chunks that have landed by the time
// the consumer gets there), so a raster group spans several chunks and B is
// streamed once per group instead of once per chunk.
__device__ __forceinline__ void decode_tile(const TileParams& p, int t, int& chunk, int& mb,
                                            int& nb, uint32_t cta_rank = 0) {
  if (p.pair_chunks) {
    // one region of W/2 chunk pairs; group_m counts pairs
    const int vblk = p.world / 2;
    const int gm = p.group_m;
    const int span = gm * p.nblk;
    const int group = t / span;
    const int first_m = group * gm;
    const int gsize = min(vblk - first_m, gm);
    const int in = t - group * span;
    const int vm = first_m + in % gsize;
    nb = in / gsize;
    if (p.serpentine && (group & 1)) nb = p.nblk - 1 - nb;
    chunk = p.order[2 * vm + (int)cta_rank];
    mb = 0;
    return;
  }
  const int per_chunk = p.mblk * p.nblk;
  const int s = t / per_chunk;
  int s0, np, gm, g0;  // region's first position, positions, raster group, groups before
  if (p.nreg > 0) {
    int r = 0;
    while (r + 1 < p.nreg && p.reg_s0[r + 1] <= s) ++r;
    s0 = p.reg_s0[r];
    np = p.reg_s0[r + 1] - s0;
    gm = p.reg_gm[r];
    g0 = p.reg_g0[r];
  } else {
    s0 = s;
    np = 1;
    gm = p.group_m;
    g0 = s * ((p.mblk + gm - 1) / gm);
  }
  const int w = t - s0 * per_chunk;
  const int vblk = np * p.mblk;
  const int span = gm * p.nblk;
  const int group = w / span;
  const int first_m = group * gm;
  const int gsize = min(vblk - first_m, gm);
  const int in = w - group * span;
  const int vm = first_m + in % gsize;
  nb = in / gsize;
  const int vs = vm / p.mblk;  // position inside the region
  chunk = p.order[s0 + vs];
  mb = vm - vs * p.mblk;
  // serpentine: odd groups walk the n-blocks backwards, so a group starts on
  // the B columns its predecessor finished with (still in L2).  2: the parity
  // runs on across chunks / regions, so the next chunk opens on the columns
  // the previous one touched last instead of the ones it touched first
  const int gidx = p.serpentine == 2 ? g0 + group : group;
  if (p.serpentine && (gidx & 1)) nb = p.nblk - 1 - nb;
}

template <int BN, int CG>
struct GemmCfg {
  static constexpr int BM = 128;  // rows per CTA (UMMA M per CTA)
  static constexpr int BK = 64;   // 128 bytes of bf16: one swizzle atom row
  static constexpr int BNC = BN / CG;  // B columns the MMA reads per CTA
  static constexpr int B_BOXES = (BNC + 63) / 64;  // 64-column TMA boxes staged per CTA
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = B_BOXES * 64 * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SUB = 32;                     // epilogue sub-tile: 32 columns
  static constexpr int NSUB = BN / SUB;
  static constexpr int EPI_BUF = 32 * SUB * 2;       // 32 rows x 64 B (SWIZZLE_64B)
  static constexpr int EPI_NBUF = 4;                 // staging buffers per epilogue warp
  static constexpr int EPI_BYTES = 4 * EPI_NBUF * EPI_BUF;
  static constexpr uint32_t TMEM_COLS = (2 * BN <= 256) ? 256 : 512;
  // BN = 512 (pair tiles only): two N = 256 MMAs per K step into one
  // accumulator of all 512 TMEM columns -- no second buffer, so the epilogue
  // is not overlapped with the next tile; chosen only for long-K grids of
  // about one tile per cluster (e.g. C5 RS at M=1024), where the wide tile
  // halves the B re-reads and the single epilogue is noise
  static constexpr int UMMA_N = BN > 256 ? 256 : BN;
  static constexpr int NACC = 2 * BN <= 512 ? 2 : 1;  // TMEM accumulator buffers
  static_assert(BNC % 16 == 0 && BN % SUB == 0 && (BN <= 256 || (BN == 512 && CG == 2)), "BN");
  static_assert(CG == 2 || BN % 64 == 0, "1-CTA tiles stage whole 64-column boxes");
  // 227 KB of dynamic smem per CTA, minus alignment slack and barriers
  static constexpr int stages_for_smem() {
    return (227 * 1024 - 1024 - 512 - EPI_BYTES) / STAGE_BYTES;
  }
  static constexpr int STAGES = stages_for_smem() > 8 ? 8 : stages_for_smem();
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + EPI_BYTES + 512;
};

__device__ __forceinline__ float2 unpack2(uint32_t w, bool fp16) {
  if (fp16) return __half22float2(*reinterpret_cast<const __half2*>(&w));
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w));
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi, bool fp16) {
  if (fp16) {
    __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Fused ReduceScatter reduction of one epilogue warp's 32 rows x BN columns
// of my own chunk (see the MODE_RS epilogue): lane l owns columns
// [n0 + 8l, n0 + 8l + 8) of every row, so one warp-wide load reads 512
// contiguous bytes of one source's row; kRedRows rows x up to 8 sources are
// in flight per lane before the first add.  Sum in ascending source order
// from +0.0f in fp32, rounded once (reference collectives.py:163-171).
template <int BN, bool FP16, int NROWS = 32>
__device__ __forceinline__ void reduce_rows(const TileParams& p, int row0, int n0, uint32_t lane) {
  constexpr int kRedRows = 4;
  constexpr int kGroup = 8;
  static_assert(NROWS % kRedRows == 0, "rows per call");
  const size_t slot_elems = (size_t)p.rows * p.n;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 256) {
  const int col = n0 + c0 + (int)lane * 8;
  if (c0 + (int)lane * 8 >= BN || col + 8 > p.n) continue;
#pragma unroll 1
  for (int r0 = 0; r0 < NROWS; r0 += kRedRows) {
    float acc[kRedRows][8];
#pragma unroll
    for (int r = 0; r < kRedRows; ++r)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[r][e] = 0.f;
#pragma unroll 1
    for (int s0 = 0; s0 < p.world; s0 += kGroup) {
      uint4 v[kRedRows][kGroup];
#pragma unroll
      for (int r = 0; r < kRedRows; ++r) {
        const int grow = row0 + r0 + r;
#pragma unroll
        for (int g = 0; g < kGroup; ++g) {
          const int s = s0 + g;
          v[r][g] = (grow < p.rows && s < p.world)
                        ? __ldcg(reinterpret_cast<const uint4*>(
                              p.staging_local + (size_t)s * slot_elems + (size_t)grow * p.n + col))
                        : make_uint4(0u, 0u, 0u, 0u);
        }
      }
#pragma unroll
      for (int r = 0; r < kRedRows; ++r)
#pragma unroll
        for (int g = 0; g < kGroup; ++g) {
          if (s0 + g >= p.world) break;
          const uint32_t wv[4] = {v[r][g].x, v[r][g].y, v[r][g].z, v[r][g].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = unpack2(wv[e], FP16);
            acc[r][2 * e] += f.x;
            acc[r][2 * e + 1] += f.y;
          }
        }
    }
#pragma unroll
    for (int r = 0; r < kRedRows; ++r) {
      const int grow = row0 + r0 + r;
      if (grow < p.rows)
        *reinterpret_cast<uint4*>(p.out_rows + (size_t)grow * p.n + col) =
            make_uint4(pack2(acc[r][0], acc[r][1], FP16), pack2(acc[r][2], acc[r][3], FP16),
                       pack2(acc[r][4], acc[r][5], FP16), pack2(acc[r][6], acc[r][7], FP16));
    }
  }
  }
}

// Cooperative own-chunk reduction (MODE_RS, fused, W > 1).  The 128 rows a
// CTA holds of an own-chunk tile are reduced in kRedUnits units of 8 rows,
// numbered globally (unit g belongs to the CTA's (g / kRedUnits)-th own tile).
// The four epilogue warps store their rows into staging[rank], bump
// `stored`, and claim units of that tile; warps with nothing else to do --
// the copier warp (idle in RS), the non-leader CTA's MMA warp, and the
// producer / MMA warps once their loops end -- walk the same own tiles and
// claim units too.  At the tail of the launch (the last own tile, which no
// MMA overlaps) six or seven warps share the reduction instead of four.
// Counters are monotone smem words: ctr[0] units claimed, ctr[1] epilogue
// warps that finished storing (tile o stored <=> ctr[1] >= 4 (o + 1)).
constexpr int kRedUnits = 16;

// lane 0: claim the next unit of own tile o, -1 when all of its units are taken
__device__ __forceinline__ int claim_unit(uint32_t* next, int o) {
  const uint32_t limit = (uint32_t)(o + 1) * kRedUnits;
  uint32_t cur = *reinterpret_cast<volatile uint32_t*>(next);
  while (cur < limit) {
    const uint32_t prev = atomicCAS(next, cur, cur + 1);
    if (prev == cur) return (int)(cur - (uint32_t)o * kRedUnits);
    cur = prev;
  }
  return -1;
}

// warp-wide: reduce every unit of own tile o this warp can claim
template <int BN, int CG, bool FP16>
__device__ __forceinline__ void reduce_own_units(const TileParams& p, uint32_t* ctr, int o, int mb,
                                                 int nb, uint32_t cta_rank, uint32_t lane) {
  for (;;) {
    int u = 0;
    if (lane == 0) {
      u = claim_unit(&ctr[0], o);
      if (u >= 0) {
        // every epilogue warp's rows of tile o are in staging[rank]
        // (the epilogue warps always get there, also after a failed peer
        // wait; bounded all the same, like every other spin)
        const uint32_t want = 4u * (uint32_t)(o + 1);
        uint64_t t0 = 0;
        while (*reinterpret_cast<volatile uint32_t*>(&ctr[1]) < want) {
          __nanosleep(128);
          const uint64_t now = globaltimer();
          if (t0 == 0) t0 = now;
          else if (now - t0 > p.timeout_ns) {
            if (p.err) atomicCAS(p.err, 0, 6);
            u = -1;
            break;
          }
        }
        __threadfence_block();
      }
    }
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u < 0) return;
    reduce_rows<BN, FP16, 128 / kRedUnits>(p, mb * (128 * CG) + (int)cta_rank * 128 + u * 8,
                                           nb * BN, lane);
  }
}

constexpr int kThreads = 224;  // 7 warps: producer, MMA, 4 epilogue, own-slot copier

template <int BN, int CG, int MODE, bool FP16>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tp_kernel(const __grid_constant__ TensorMaps maps, const __grid_constant__ TileParams p) {
  using C = GemmCfg<BN, CG>;
  constexpr int BM = C::BM, BK = C::BK, BNC = C::BNC, STAGES = C::STAGES;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + STAGES * C::A_BYTES;
  uint8_t* sEpi = sB + STAGES * C::B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + C::EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* stored_bar = tempty + 2;        // AG own copy: copier done with stage s
  uint64_t* alanded_bar = stored_bar + STAGES;  // AG own copy: this CTA's A half landed
  TileRing* ring = reinterpret_cast<TileRing*>(alanded_bar + STAGES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + 1);
  uint32_t* red_ctr = tmem_slot + 1;  // cooperative own-chunk reduction (2 words)

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t cta_rank = (CG == 2) ? cluster_ctarank() : 0;
  const bool leader = cta_rank == 0;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&maps.a_all);
    prefetch_tmap(&maps.b);
    prefetch_tmap(&maps.c);
    if (MODE == MODE_AG) {
      prefetch_tmap(&maps.a_own);
      if (p.copy_own) prefetch_tmap(&maps.own_slot);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], CG * 4);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&stored_bar[s], 1);
      mbar_init(&alanded_bar[s], 1);
    }
    // ring consumers per CTA: 4 epilogue warps + (MMA warp in the leader /
    // producer warp in the peer) + the own-slot copier when it runs
    const int per_cta = 5 + ((MODE == MODE_AG && p.copy_own) ? 1 : 0);
    for (int r = 0; r < kRing; ++r) {
      mbar_init(&ring->full[r], 1);
      mbar_init(&ring->empty[r], per_cta * CG);
    }
    red_ctr[0] = 0;
    red_ctr[1] = 0;
    fence_mbarrier_init();
  }
  if (warp == 2) tmem_alloc<CG>(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // everything above (barrier init, TMEM allocation, descriptor prefetch)
  // overlaps the previous grid's tail under programmatic dependent launch;
  // every global-memory access comes after this point
  grid_dependency_wait();
  grid_launch_dependents();

  const int cluster_id = blockIdx.x / CG;
  const int num_clusters = gridDim.x / CG;
  const int num_kb = (p.k + BK - 1) / BK;

  if (warp == 0) {
    // ===================== TMA producer =====================
    // The whole warp walks the loop (warp-uniform values stay in uniform
    // registers); one elected lane issues the barrier/TMA instructions.
    {
      uint32_t stage = 0, phase = 0;
      // row ranges of each chunk this CTA has observed landed (ready[c] counts
      // ranges: (epoch-1)*ag_sub + ranges landed so far)
      int landed[kMaxWorld];
#pragma unroll
      for (int c = 0; c < kMaxWorld; ++c) landed[c] = 0;
      int trace_slot = 1;   // slot 0: CTA lifetime (written by the epilogue)
      uint32_t copy_mask = 0, stored_phase = 0;  // stages holding an own-slot copy
      const uint64_t b_hint = p.l2_hint_b, a_hint = p.l2_hint_a;
      WorkIter wi;
      wi.init(p, cluster_id, num_clusters, num_kb, ring, leader ? 0 : 1, CG);
      WorkItem w;
      int waves_issued = 0;  // data-parallel tiles this cluster has issued
      int dp_seen = 0;       // data-parallel tiles seen (K-direction parity)
      const bool wave_lead = p.wave_flags != nullptr && leader;
      while (wi.next(w)) {
        int chunk, mb, nb;
        decode_tile(p, w.t, chunk, mb, nb, cta_rank);
        const bool dp_item = w.t < p.dp_tiles;
        if (wave_lead && dp_item && waves_issued > 0)
          wave_wait(p.wave_flags, p.wave_tag, waves_issued, num_clusters, p.dp_tiles);
        const bool own = (MODE == MODE_AG) && chunk == p.rank;
        const bool copying = own && p.copy_own;
        const int row0 = p.pair_chunks ? 0 : mb * (BM * CG) + (int)cta_rank * BM;
        const int col0 = nb * BN + (int)cta_rank * BNC;
        // global column of this CTA's B box j: for BN <= 256 the CTA holds
        // the contiguous half [col0, col0 + BNC); for BN = 512 it holds the
        // half of each N = 256 MMA (boxes 0-1 and 2-3 = its 128 columns of
        // the tile's first and second 256)
        auto bcol = [&](int j) {
          return BN > 256 ? nb * BN + (j >> 1) * 256 + (int)cta_rank * 128 + (j & 1) * 64
                          : col0 + j * 64;
        };
        if (MODE == MODE_AG && !own) {
          // wait(ready[chunk]) of pipelines.py:130-141, as an acquire spin on
          // the range holding this CTA's last row of the tile
          const int need = (min(row0 + BM, p.rows) - 1) / p.ag_sub_rows + 1;
          if (landed[chunk] < need) {
            if (lane == 0) {
              const uint64_t tw0 = p.trace ? globaltimer() : 0;
              spin_geq(p.ready + chunk, (p.epoch - 1) * (uint64_t)p.ag_sub + need, p.err,
                       p.timeout_ns, 1);
              fence_proxy_async_global();
              if (p.trace)
                trace_rec(p, trace_slot++, (1ull << 56) | ((uint64_t)need << 32) | chunk, tw0,
                          globaltimer(), w.t);
            }
            __syncwarp();
            landed[chunk] = need;
          }
        }
        // K direction: every other data-parallel tile of this cluster walks K
        // backwards, so it opens on the k-slices the previous wave touched last
        const bool rev = p.kserp && w.kind == 0 && dp_item && (dp_seen & 1);
        if (dp_item) ++dp_seen;
        // (kb - nb) mod nblk, stepped with kb: a division per k-block on the
        // producer's path between the empty wait and the TMA issue cost 25 %
        int cr = copying ? ((((rev ? w.kb1 - 1 : w.kb0) - nb) % p.nblk) + p.nblk) % p.nblk : 1;
        for (int i = 0, nk = w.kb1 - w.kb0; i < nk; ++i) {
          const int kb = rev ? w.kb1 - 1 - i : w.kb0 + i;
          mbar_wait(&empty[stage], phase ^ 1);
          if ((copy_mask >> stage) & 1u) {
            // the own-slot store of the previous occupant must have read it
            mbar_wait(&stored_bar[stage], (stored_phase >> stage) & 1u);
            stored_phase ^= 1u << stage;
            copy_mask &= ~(1u << stage);
          }
          // k-block kb of n-block nb goes to the own slot iff kb == nb (mod nblk):
          // each k-block of each m-block exactly once.  Its A half lands on a
          // CTA-local barrier; the copier forwards the bytes to the leader's
          // full barrier and keeps the stage until its store has read it.
          bool copy_kb = false;
          if (copying) {
            copy_kb = cr == 0;
            if (rev) cr = cr == 0 ? p.nblk - 1 : cr - 1;
            else cr = cr + 1 == p.nblk ? 0 : cr + 1;
            if (copy_kb) copy_mask |= 1u << stage;
          }
          uint8_t* a_dst = sA + stage * C::A_BYTES;
          uint8_t* b_dst = sB + stage * C::B_BYTES;
          const int kx = kb * BK;
          if (elect_one()) {
            if (leader) mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES * CG);
            if (copy_kb) {
              mbar_arrive_expect_tx(&alanded_bar[stage], C::A_BYTES);
              tma_load_2d(&maps.a_own, &alanded_bar[stage], a_dst, kx, row0, a_hint);
#pragma unroll
              for (int j = 0; j < C::B_BOXES; ++j) {
                if constexpr (CG == 1)
                  tma_load_2d(&maps.b, &full[stage], b_dst + j * 64 * BK * 2, bcol(j), kx,
                              b_hint);
                else
                  tma_load_2d_pair(&maps.b, &full[stage], b_dst + j * 64 * BK * 2, bcol(j),
                                   kx, b_hint);
              }
            } else if constexpr (CG == 1) {
              if (own) tma_load_2d(&maps.a_own, &full[stage], a_dst, kx, row0, a_hint);
              else tma_load_3d(&maps.a_all, &full[stage], a_dst, kx, row0, chunk, a_hint);
#pragma unroll
              for (int j = 0; j < C::B_BOXES; ++j)
                tma_load_2d(&maps.b, &full[stage], b_dst + j * 64 * BK * 2, bcol(j), kx,
                            b_hint);
            } else {
              if (own) tma_load_2d_pair(&maps.a_own, &full[stage], a_dst, kx, row0, a_hint);
              else tma_load_3d_pair(&maps.a_all, &full[stage], a_dst, kx, row0, chunk, a_hint);
#pragma unroll
              for (int j = 0; j < C::B_BOXES; ++j)
                tma_load_2d_pair(&maps.b, &full[stage], b_dst + j * 64 * BK * 2, bcol(j), kx,
                                 b_hint);
            }
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (wave_lead && dp_item) {
          ++waves_issued;
          if (lane == 0) st_relaxed_gpu(p.wave_flags + cluster_id, p.wave_tag | waves_issued);
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA) =====================
    // Warp-wide loop, one elected lane issues tcgen05.mma / commit.
    // Descriptors are precomputed and advanced by plain adds:
    //   A (K-major SW128): +32 B per 16-element K step -> +2 in addr>>4
    //   B (MN-major SW128): +2 KB per 16-row K step   -> +128 in addr>>4
    if (leader) {
      constexpr uint32_t IDESC = umma_idesc_f16(BM * CG, C::UMMA_N, FP16 ? 0 : 1, /*a K-major*/ 0,
                                                /*b MN-major*/ 1);
      const uint64_t a_desc0 = umma_desc(smem_u32(sA), 16, 1024, 2);
      // B: 64-column atoms 8 KB apart (LBO), 8-row K groups 1 KB apart (SBO)
      const uint64_t b_desc0 = umma_desc(smem_u32(sB), 64 * BK * 2, 1024, 2);
      uint32_t stage = 0, phase = 0;
      int it = 0;
      // optional timeline (kind 5, last quarter of the CTA's records): per
      // work item, the wait for a free accumulator [t0, t1) and the summed
      // time spent waiting for operand stages (aux, ns)
      const bool mtrace = p.trace != nullptr && lane == 0;
      int mslot = p.trace_cap * 3 / 4;
      WorkIter wi;
      wi.init(p, cluster_id, num_clusters, num_kb, ring, 1, CG);
      WorkItem w;
      for (; wi.next(w); ++it) {
        const int as = C::NACC == 2 ? (it & 1) : 0;
        const uint32_t aphase = C::NACC == 2 ? ((it >> 1) & 1) : (it & 1);
        const uint64_t tw0 = mtrace ? globaltimer() : 0;
        mbar_wait_cluster(&tempty[as], aphase ^ 1);
        const uint64_t tw1 = mtrace ? globaltimer() : 0;
        uint64_t full_wait = 0;
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * BN;
        // stages arrive in the producer's order (either K direction); only
        // the first MMA of the item starts a fresh accumulator
        for (int i = 0, nk = w.kb1 - w.kb0; i < nk; ++i) {
          if (mtrace) {
            const uint64_t tf = globaltimer();
            mbar_wait(&full[stage], phase);
            full_wait += globaltimer() - tf;
          } else {
            mbar_wait(&full[stage], phase);
          }
          tc_fence_after();
          const uint64_t ad = a_desc0 + (uint64_t)((stage * C::A_BYTES) >> 4);
          const uint64_t bd = b_desc0 + (uint64_t)((stage * C::B_BYTES) >> 4);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              umma_f16<CG>(d_tmem, ad + 2 * kk, bd + 128 * kk, IDESC, (i != 0) || (kk != 0));
              if constexpr (BN > 256)  // second 256 columns: B boxes 2-3 (16 KB on)
                umma_f16<CG>(d_tmem + 256, ad + 2 * kk, bd + 1024 + 128 * kk, IDESC,
                             (i != 0) || (kk != 0));
            }
            umma_commit<CG>(&empty[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) umma_commit<CG>(&tfull[as]);
        __syncwarp();
        if (mtrace && mslot < p.trace_cap)
          trace_rec(p, mslot++, (5ull << 56) | (full_wait & 0xFFFFFFFFull), tw0, tw1, w.t);
      }
    }
  } else if (warp == 6) {
    // ===================== own-slot copier (AG) =====================
    // Own slot of the gather buffer (allgather_push_intra pushes to self too,
    // collectives.py:95-97): every A stage of the own chunk is already in
    // smem for the MMA, so 1/nblk of them (k-block kb of n-block kb mod nblk
    // -- each k-block of each m-block exactly once) are copied from smem into
    // gathered[rank] once the MMAs consumed them.  No extra HBM or L2 reads.
    if (MODE == MODE_AG && p.copy_own) {  // whole warp walks the items, lane 0 copies
      uint32_t stage = 0, landed_phase = 0;
      int dp_seen = 0;
      WorkIter wi;
      wi.init(p, cluster_id, num_clusters, num_kb, ring, 1, CG);
      WorkItem w;
      while (wi.next(w)) {
        int chunk, mb, nb;
        decode_tile(p, w.t, chunk, mb, nb, cta_rank);
        const bool copying = chunk == p.rank;
        const int row0 = p.pair_chunks ? 0 : mb * (BM * CG) + (int)cta_rank * BM;
        const bool dp_item = w.t < p.dp_tiles;
        const bool rev = p.kserp && w.kind == 0 && dp_item && (dp_seen & 1);
        if (dp_item) ++dp_seen;
        int cr = copying ? ((((rev ? w.kb1 - 1 : w.kb0) - nb) % p.nblk) + p.nblk) % p.nblk : 1;
        for (int i = 0, nk = w.kb1 - w.kb0; i < nk; ++i) {
          const int kb = rev ? w.kb1 - 1 - i : w.kb0 + i;
          if (copying) {
            const bool cr0 = cr == 0;
            if (rev) cr = cr == 0 ? p.nblk - 1 : cr - 1;
            else cr = cr + 1 == p.nblk ? 0 : cr + 1;
            if (cr0 && lane == 0) {
              // uses of a stage for copies alternate with `stored` acks, so
              // this parity wait is never more than one phase away
              mbar_wait(&alanded_bar[stage], (landed_phase >> stage) & 1u);
              mbar_complete_tx_cluster(&full[stage], 0, C::A_BYTES);  // hand to the MMA
              // evict-first: 1 B written per 2 B the GEMM keeps reading from
              // L2; don't let the copy push the operands out
              tma_store_2d_hint(&maps.own_slot, sA + stage * C::A_BYTES, kb * BK, row0,
                                p.l2_hint_own);
              bulk_commit();
              bulk_wait_read<0>();
              mbar_arrive(&stored_bar[stage]);
            }
            if (cr0) landed_phase ^= 1u << stage;
          }
          if (++stage == STAGES) stage = 0;
        }
        __syncwarp();
      }
      if (lane == 0) bulk_wait<0>();
    }
  } else {
    // ===================== epilogue (warps 2..5) =====================
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    uint8_t* stg = sEpi + (warp - 2) * C::EPI_NBUF * C::EPI_BUF;
    int buf = 0;
    int it = 0;
    uint32_t freed = 0;    // RS: destinations observed free for this epoch
    bool peers_in = false;  // RS fused: every peer's contribution to my chunk landed
    int pend_chunk = -1;    // RS: tile whose stores still have to be published
    uint64_t pend_count = 0;
    int own_o = 0;          // RS fused: own-chunk tiles reduced so far (unit numbering)
    const size_t slot_elems = (size_t)p.rows * p.n;
    const bool tracer = p.trace != nullptr && warp == 2 && lane == 0;
    const uint64_t t_cta0 = tracer ? globaltimer() : 0;
    int trace_slot = p.trace_cap / 2;
    WorkIter wi;
    wi.init(p, cluster_id, num_clusters, num_kb, ring, 1, CG);
    WorkItem w;
    for (; wi.next(w); ++it) {
      int chunk, mb, nb;
      decode_tile(p, w.t, chunk, mb, nb, cta_rank);
      const int as = C::NACC == 2 ? (it & 1) : 0;
      const uint32_t aphase = C::NACC == 2 ? ((it >> 1) & 1) : (it & 1);
      const int cta_row0 = p.pair_chunks ? 0 : mb * (BM * CG) + (int)cta_rank * BM;
      const int row = cta_row0 + q * 32;  // first row of this warp's slab
      const int n0 = nb * BN;
      const bool fused_own = (MODE == MODE_RS) && p.fuse_reduce && chunk == p.rank;
      if (MODE == MODE_RS && !((freed >> chunk) & 1u)) {
        // dest must have reduced the previous call before its slot is reused
        if (lane == 0 && p.epoch > 1 && chunk != p.rank)  // own slot: stream-ordered
          spin_geq(p.rs_free + chunk, p.epoch - 1, p.err, p.timeout_ns, 2);
        __syncwarp();
        freed |= 1u << chunk;
      }
      if (MODE == MODE_RS && fused_own && lane == 0 && pend_chunk >= 0) {
        // publish before waiting on the peers: they may be waiting on it
        bulk_wait<0>();
        fence_proxy_async_global();
        rs_publish(p, pend_chunk, pend_count);
        pend_chunk = -1;
      }
      if (fused_own && !peers_in) {
        // the reduce side of rs_intra_streams (collectives.py:163-171) for my
        // own chunk: every other source's rows must have landed; every lane
        // acquires so its own loads below are ordered after the releases
        const uint64_t tw0 = tracer ? globaltimer() : 0;
        for (int s = 0; s < p.world; ++s)
          if (s != p.rank) spin_geq(p.rs_mine + s, p.rs_target, p.err, p.timeout_ns, 3);
        __syncwarp();
        if (tracer) trace_rec(p, trace_slot++, (3ull << 56) | chunk, tw0, globaltimer(), w.t);
        peers_in = true;
      }
      if (MODE == MODE_RS && fused_own && p.world > 1) {
        // Peers' rows of this tile are in memory (peers_in): pull this
        // warp's 32 rows of every peer slot into L2 while the tile's MMA is
        // still running, so the reduction below reads L2 instead of waiting
        // on DRAM (one bulk prefetch per row and source, lanes in parallel).
        const int cols = min(BN, p.n - n0);
        for (int i = (int)lane; i < 32 * p.world; i += 32) {
          const int s = i >> 5, r = row + (i & 31);
          if (s != p.rank && r < p.rows && cols > 0)
            prefetch_l2_bulk(p.staging_local + (size_t)s * slot_elems + (size_t)r * p.n + n0,
                             (uint32_t)cols * 2u);
        }
      }
      mbar_wait(&tfull[as], aphase);
      tc_fence_after();
      const uint64_t t_acc = tracer ? globaltimer() : 0;
      const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + as * BN;
      // Stream-K partials are kept warp-interleaved: the (cluster, CTA, warp)
      // slab is NSUB x 8 x 32 float4 with lane fastest, so every store and the
      // finisher's matching load is one contiguous 512-byte warp access.
      constexpr int kSlab = C::NSUB * 8 * 32;  // float4 per warp slab
      const size_t my_slab = (((size_t)cluster_id * CG + cta_rank) * 4 + q) * kSlab;
      if (w.kind == 1) {
        // partial head of a stream-K tile: fp32 to this cluster's workspace
        // slot, then a release flag per epilogue warp
        float4* dst = reinterpret_cast<float4*>(p.ws) + my_slab + lane;
#pragma unroll 1
        for (int j = 0; j < C::NSUB; ++j) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(t_row + j * C::SUB, v);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 8; ++c)
            __stcg(dst + (j * 8 + c) * 32,
                   make_float4(__uint_as_float(v[4 * c]), __uint_as_float(v[4 * c + 1]),
                               __uint_as_float(v[4 * c + 2]), __uint_as_float(v[4 * c + 3])));
        }
        tc_fence_before();
        __threadfence();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) mbar_arrive_cluster(&tempty[as], 0);
          else mbar_arrive(&tempty[as]);
          st_release_sys(p.ws_flags + ((size_t)cluster_id * CG + cta_rank) * 4 + q, p.ws_epoch);
        }
        __syncwarp();
        if (tracer)
          trace_rec(p, trace_slot++, (2ull << 56) | (1ull << 32) | (uint64_t)chunk, t_acc,
                    globaltimer(), w.t);
        continue;
      }
      int c_lo = 0, c_hi = -1;  // clusters holding this tile's earlier k-blocks
      if (w.kind == 2) {
        const long long ts = (long long)(w.t - p.dp_tiles) * num_kb;
        c_lo = wi.owner(ts);
        c_hi = wi.owner(ts + w.kb0 - 1);
        for (int c = c_lo; c <= c_hi; ++c)
          spin_geq(p.ws_flags + ((size_t)c * CG + cta_rank) * 4 + q, p.ws_epoch, p.err,
                   p.timeout_ns, 5);
        __syncwarp();
      }
      // 32-column sub-tiles: one tcgen05.ld (32 lanes x 32 fp32), bf16 pack,
      // a 64-byte swizzled row per lane, one 32x32 TMA store
#pragma unroll 1
      for (int j = 0; j < C::NSUB; ++j) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_row + j * C::SUB, v);
        tmem_ld_wait();
        for (int c = c_lo; c <= c_hi; ++c) {
          const float4* s4 = reinterpret_cast<const float4*>(p.ws) +
                             (((size_t)c * CG + cta_rank) * 4 + q) * kSlab + j * 8 * 32 + lane;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float4 f = __ldcg(s4 + e * 32);
            v[4 * e] = __float_as_uint(__uint_as_float(v[4 * e]) + f.x);
            v[4 * e + 1] = __float_as_uint(__uint_as_float(v[4 * e + 1]) + f.y);
            v[4 * e + 2] = __float_as_uint(__uint_as_float(v[4 * e + 2]) + f.z);
            v[4 * e + 3] = __float_as_uint(__uint_as_float(v[4 * e + 3]) + f.w);
          }
        }
        if (j == C::NSUB - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 2) mbar_arrive_cluster(&tempty[as], 0);
            else mbar_arrive(&tempty[as]);
          }
        }
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e)
          pk[e] = pack2(__uint_as_float(v[2 * e]), __uint_as_float(v[2 * e + 1]), FP16);
        const int xcol = n0 + j * C::SUB;
        const int swz = (lane >> 1) & 3;  // SWIZZLE_64B: 16-byte chunk ^= row bits 1..2
        // a world of one reduces a single slot: out == staging[0] bit for bit,
        // so both stores are issued from one staging buffer; at W > 1 my own
        // chunk's tile goes to staging[rank] like any other chunk's and is
        // reduced below, once its rows are in memory
        const bool dual = fused_own && p.world == 1;
        {
          // 4-deep ring of staging buffers: at most 3 stores still reading smem
          if (lane == 0) bulk_wait_read<C::EPI_NBUF - 1>();
          __syncwarp();
          uint8_t* sb = stg + buf * C::EPI_BUF;
          uint8_t* rowp = sb + lane * 64;
#pragma unroll
          for (int c = 0; c < 4; ++c)
            *reinterpret_cast<uint4*>(rowp + ((c ^ swz) << 4)) =
                make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if constexpr (MODE == MODE_AG) {
              tma_store_3d_hint(&maps.c, sb, xcol, row, chunk, p.l2_hint_store);
            } else {
              // own chunk at W > 1: re-read by the reduction (the fused
              // epilogue's right away, the reduction kernel's at the end)
              tma_store_2d_hint(&maps.out[chunk], sb, xcol, row,
                                chunk == p.rank && p.world > 1 ? p.l2_hint_own
                                                               : p.l2_hint_store);
              if (dual) tma_store_3d_hint(&maps.c, sb, xcol, row, 0, p.l2_hint_store);
            }
            bulk_commit();
          }
          buf = (buf + 1) % C::EPI_NBUF;
        }
      }
      if (MODE == MODE_RS && fused_own && p.world > 1) {
        // the reduce side of rs_intra_streams (collectives.py:163-171) for
        // this warp's 32 rows of the tile: out = sum_{s ascending} slot_s in
        // fp32, slot_rank being the bf16 rows just stored -- the arithmetic
        // of the separate reduction kernel and of the reference's ascending
        // `acc +=`.  Row-contiguous 16-byte loads (a warp reads 512 B of one
        // row per source) with kRedRows rows x every source in flight: the
        // per-lane-row loads of the accumulator layout were DRAM-latency
        // bound (~48 us per 256x256 tile at W=8).
        const uint64_t tr0 = tracer ? globaltimer() : 0;
        if (lane == 0) {
          bulk_wait<0>();
          fence_proxy_async_global();
          __threadfence_block();
          atomicAdd(&red_ctr[1], 1u);  // this warp's rows of own tile own_o are stored
        }
        __syncwarp();
        const uint64_t tr1 = tracer ? globaltimer() : 0;
        // units of this tile, shared with the helper warps (cta_row0 = the
        // CTA's 128 rows; the units span all four epilogue warps' rows)
        reduce_own_units<BN, CG, FP16>(p, red_ctr, own_o, mb, nb, cta_rank, lane);
        ++own_o;
        if (tracer)  // kind 6: own-chunk reduction, aux = store-drain part (ns)
          trace_rec(p, trace_slot++, (6ull << 56) | ((tr1 - tr0) & 0xFFFFFFFFull), tr0, globaltimer(),
                    w.t);
      }
      if (tracer)
        trace_rec(p, trace_slot++, (2ull << 56) | ((uint64_t)w.kind << 32) | (uint64_t)chunk, t_acc,
                  globaltimer(), w.t);
      if constexpr (MODE == MODE_RS) {
        // Publish the previous tile of a peer chunk now that this tile's
        // stores are queued behind it (keeps the store-completion wait off
        // the accumulator's critical path); my own fused chunk needs no
        // counter -- its reduction happened right here.
        if (lane == 0) {
          if (pend_chunk >= 0) {
            bulk_wait<C::NSUB>();
            fence_proxy_async_global();
            rs_publish(p, pend_chunk, pend_count);
          }
          pend_chunk = -1;
          // count the elements this warp actually delivered (TMA clips the
          // ragged edges), so a chunk is complete at exactly rows*n per call
          const int vr = max(0, min(32, p.rows - row));
          const int vc = max(0, min(BN, p.n - n0));
          if (!fused_own) {
            pend_chunk = chunk;
            pend_count = (uint64_t)vr * (uint64_t)vc;
          } else {
            // nobody waits on my own chunk's counter in the fused path, but it
            // advances all the same, so the counters mean the same thing in
            // both modes (a later unfused call targets epoch * rows * n, and
            // is stream-ordered after this kernel: no release fence needed)
            red_add_relaxed_gpu(p.rs_count[chunk], (uint64_t)vr * (uint64_t)vc);
          }
        }
        __syncwarp();
      }
    }
    if (tracer) trace_rec(p, 0, (4ull << 56) | blockIdx.x, t_cta0, globaltimer(), 0);
    if (lane == 0) {
      bulk_wait<0>();
      if (MODE == MODE_RS && pend_chunk >= 0) {
        fence_proxy_async_global();
        rs_publish(p, pend_chunk, pend_count);
      }
    }
    __syncwarp();
  }

  if constexpr (MODE == MODE_RS) {
    // helper warps of the cooperative own-chunk reduction (see kRedUnits):
    // the copier warp and the non-leader MMA warp from the start, the
    // producer and the leader's MMA warp once their loops are done.  They
    // walk the same static schedule (not with the dynamic tile counter).
    if ((warp == 0 || warp == 1 || warp == 6) && p.fuse_reduce && p.red_help && p.world > 1 &&
        p.tile_counter == nullptr) {
      WorkIter wi;
      wi.init(p, cluster_id, num_clusters, num_kb);
      WorkItem w;
      int o = 0;
      while (wi.next(w)) {
        int chunk, mb, nb;
        decode_tile(p, w.t, chunk, mb, nb);
        if (chunk != p.rank || w.kind == 1) continue;  // kind 1: partial head, no epilogue
        reduce_own_units<BN, CG, FP16>(p, red_ctr, o, mb, nb, cta_rank, lane);
        ++o;
      }
    }
  }

  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<CG>(tmem_base, C::TMEM_COLS);
  }
  if (threadIdx.x == 0) exit_release(p.rel);
}

// ---------------------------------------------------------------------------
// ReduceScatter reduction: out = sum_{s ascending} staging[s] in fp32, stored
// as bf16/fp16 (reference collectives.py:163-171; fixed ascending source
// order keeps the float result reproducible).  Each CTA waits
// for every source's element counter to reach epoch*rows*n first.
// HBM-bound: (W + 1) * rows * n * 2 bytes.  Every source's 16-byte vector of
// an element group is loaded before the first add (8 loads in flight per
// thread): the per-source load -> add loop ran at 4.3 TB/s on the C4/TP=8
// layout (ncu, 31.4 us), this form at ~7 TB/s (scripts/probe/reduce_bw.cu:
// 20.8 us; the slot stride -- exactly 16 MB there -- makes no difference).
template <bool FP16>
__global__ void __launch_bounds__(256) rs_reduce_kernel(const uint16_t* __restrict__ staging,
                                                        uint16_t* __restrict__ out,
                                                        size_t slot_elems, int world,
                                                        const uint64_t* counters, uint64_t target,
                                                        int* err, uint64_t timeout_ns,
                                                        uint64_t* trace, int trace_cap,
                                                        int trace_grid,
                                                        const __grid_constant__ ExitRelease rel) {
  constexpr int kGroup = 8;
  const bool tracer = trace != nullptr && threadIdx.x == 0 && (int)blockIdx.x < trace_grid &&
                      trace_cap >= 2;
  const uint64_t t0 = tracer ? globaltimer() : 0;
  // one thread per source acquires its counter (8 acquires in a row by one
  // thread cost ~3 us per CTA at the kernel start: ncu 30.5 -> 27.4 us)
  if ((int)threadIdx.x < world) spin_geq(counters + threadIdx.x, target, err, timeout_ns, 3);
  __syncthreads();
  if (tracer) {  // kind 3: waiting for the peers' rows (the exposed part of the RS)
    uint64_t* r = trace + (size_t)blockIdx.x * trace_cap * 4;
    r[0] = 3ull << 56;
    r[1] = t0;
    r[2] = globaltimer();
    r[3] = 0;
  }
  // 16-byte vectors only when every slot starts 16-byte aligned
  const size_t nvec = (slot_elems % 8 == 0) ? slot_elems / 8 : 0;
  const uint4* st = reinterpret_cast<const uint4*>(staging);
  uint4* o = reinterpret_cast<uint4*>(out);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nvec;
       i += (size_t)gridDim.x * blockDim.x) {
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    for (int s0 = 0; s0 < world; s0 += kGroup) {
      uint4 v[kGroup];
#pragma unroll
      for (int g = 0; g < kGroup; ++g)
        v[g] = s0 + g < world ? __ldcs(st + (size_t)(s0 + g) * nvec + i) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int g = 0; g < kGroup; ++g) {
        if (s0 + g >= world) break;
        const uint32_t w[4] = {v[g].x, v[g].y, v[g].z, v[g].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = unpack2(w[e], FP16);
          acc[2 * e] += f.x;
          acc[2 * e + 1] += f.y;
        }
      }
    }
    __stcs(o + i, make_uint4(pack2(acc[0], acc[1], FP16), pack2(acc[2], acc[3], FP16),
                             pack2(acc[4], acc[5], FP16), pack2(acc[6], acc[7], FP16)));
  }
  // scalar remainder (every element when the slots are not 16-byte aligned)
  const size_t tail0 = nvec * 8;
  for (size_t i = tail0 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < slot_elems;
       i += (size_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < world; ++s) {
      uint16_t h = staging[s * slot_elems + i];
      acc += FP16 ? __half2float(__ushort_as_half(h)) : __bfloat162float(__ushort_as_bfloat16(h));
    }
    out[i] = FP16 ? __half_as_ushort(__float2half_rn(acc))
                  : __bfloat16_as_ushort(__float2bfloat16_rn(acc));
  }
  if (tracer) {  // kind 4: the CTA's lifetime
    uint64_t* r = trace + ((size_t)blockIdx.x * trace_cap + 1) * 4;
    r[0] = (4ull << 56) | blockIdx.x;
    r[1] = t0;
    r[2] = globaltimer();
    r[3] = 0;
  }
  // producer[rank] on every peer: this rank has read its staging slots
  if (rel.count > 0) {
    __syncthreads();
    if (threadIdx.x == 0) exit_release(rel);
  }
}

// The same reduction with the W source slots staged by bulk copies (the DMA
// path of TMA, no tensor map): each step a CTA pulls 4 KB of every source
// into shared memory (kRbStages-deep ring on mbarriers), and each thread sums
// one 16-byte vector across the sources in ascending order -- the load side
// becomes a few large DMA requests instead of W x 256 16-byte loads per step.
constexpr int kRbChunk = 4096;  // bytes of one source per step (256 threads x 16 B)

template <bool FP16>
__global__ void __launch_bounds__(256) rs_reduce_bulk_kernel(
    const uint16_t* __restrict__ staging, uint16_t* __restrict__ out, size_t slot_elems, int world,
    int stages, const uint64_t* counters, uint64_t target, int* err, uint64_t timeout_ns,
    uint64_t* trace, int trace_cap, int trace_grid, const __grid_constant__ ExitRelease rel) {
  extern __shared__ uint8_t rb_raw[];
  uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(rb_raw) + 127) &
                                            ~uintptr_t(127));
  uint64_t* bars = reinterpret_cast<uint64_t*>(buf + (size_t)stages * world * kRbChunk);
  const bool tracer = trace != nullptr && threadIdx.x == 0 && (int)blockIdx.x < trace_grid &&
                      trace_cap >= 2;
  const uint64_t t0 = tracer ? globaltimer() : 0;
  if (threadIdx.x == 0) {
    for (int st = 0; st < stages; ++st) mbar_init(&bars[st], 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if ((int)threadIdx.x < world) spin_geq(counters + threadIdx.x, target, err, timeout_ns, 3);
  __syncthreads();
  if (tracer) {  // kind 3: waiting for the peers' rows
    uint64_t* r = trace + (size_t)blockIdx.x * trace_cap * 4;
    r[0] = 3ull << 56;
    r[1] = t0;
    r[2] = globaltimer();
    r[3] = 0;
  }
  const size_t slot_bytes = slot_elems * 2;
  const long long nchunks = (long long)((slot_bytes + kRbChunk - 1) / kRbChunk);
  const char* src0 = reinterpret_cast<const char*>(staging);
  auto issue = [&](long long i) {  // thread 0: step i of this CTA into stage i % stages
    const long long c = blockIdx.x + i * (long long)gridDim.x;
    if (c >= nchunks) return;
    const int st = (int)(i % stages);
    const uint32_t bytes = (uint32_t)min((size_t)kRbChunk, slot_bytes - (size_t)c * kRbChunk);
    mbar_arrive_expect_tx(&bars[st], bytes * (uint32_t)world);
    for (int s = 0; s < world; ++s)
      bulk_load_g2s(buf + ((size_t)st * world + s) * kRbChunk,
                    src0 + (size_t)s * slot_bytes + (size_t)c * kRbChunk, bytes, &bars[st]);
  };
  const long long steps = nchunks > (long long)blockIdx.x
                              ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0)
    for (long long i = 0; i < stages && i < steps; ++i) issue(i);
  for (long long i = 0; i < steps; ++i) {
    const int st = (int)(i % stages);
    mbar_wait(&bars[st], (uint32_t)((i / stages) & 1));
    const long long c = blockIdx.x + i * (long long)gridDim.x;
    const size_t off = (size_t)c * kRbChunk + (size_t)threadIdx.x * 16;
    if (off < slot_bytes) {
      float acc[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = 0.f;
      for (int s = 0; s < world; ++s) {
        const uint4 v = *reinterpret_cast<const uint4*>(buf + ((size_t)st * world + s) * kRbChunk +
                                                        threadIdx.x * 16);
        const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = unpack2(w4[e], FP16);
          acc[2 * e] += f.x;
          acc[2 * e + 1] += f.y;
        }
      }
      __stcs(reinterpret_cast<uint4*>(reinterpret_cast<char*>(out) + off),
             make_uint4(pack2(acc[0], acc[1], FP16), pack2(acc[2], acc[3], FP16),
                        pack2(acc[4], acc[5], FP16), pack2(acc[6], acc[7], FP16)));
    }
    __syncthreads();  // stage st is read by every thread: refill it
    if (threadIdx.x == 0 && i + stages < steps) issue(i + stages);
  }
  if (tracer) {  // kind 4: the CTA's lifetime
    uint64_t* r = trace + ((size_t)blockIdx.x * trace_cap + 1) * 4;
    r[0] = (4ull << 56) | blockIdx.x;
    r[1] = t0;
    r[2] = globaltimer();
    r[3] = 0;
  }
  // producer[rank] on every peer: this rank has read its staging slots
  if (rel.count > 0) {
    __syncthreads();
    if (threadIdx.x == 0) exit_release(rel);
  }
}

// Generic slot reduction for the standalone ReduceScatter (any element
// type): out[i] = sum_{s ascending} slot_s[i], accumulated in Acc.
template <typename T, typename Acc>
__global__ void __launch_bounds__(256) slots_reduce_kernel(const T* __restrict__ staging,
                                                           T* __restrict__ out, size_t slot_elems,
                                                           int nslots) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < slot_elems;
       i += (size_t)gridDim.x * blockDim.x) {
    Acc acc = Acc(0);
    for (int s = 0; s < nslots; ++s) acc += Acc(staging[(size_t)s * slot_elems + i]);
    out[i] = T(acc);
  }
}

// ---------------------------------------------------------------------------
// Node-scope multimem (reference primitives.py:291-315).  The symmetric slabs
// of the node's ranks are mapped into this rank's address space (peer access
// / CUDA IPC), so both are SM-driven NVLink transfers: multimem_st reads the
// caller's bytes once and stores them into every other replica (P2P stores),
// multimem_ld_reduce loads every replica (P2P loads) and sums them in
// ascending rank order with numpy's `out += replica` arithmetic: the sum
// starts from +0 and every step rounds to the element type (floats) or wraps
// (integers).

struct PeerList {
  uint8_t* p[kMaxWorld];
};

struct AddBF16 {
  using S = uint16_t;
  __device__ static S add(S a, S b) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(__bfloat162float(__ushort_as_bfloat16(a)) +
                                                    __bfloat162float(__ushort_as_bfloat16(b))));
  }
};
struct AddFP16 {
  using S = uint16_t;
  __device__ static S add(S a, S b) {
    return __half_as_ushort(
        __float2half_rn(__half2float(__ushort_as_half(a)) + __half2float(__ushort_as_half(b))));
  }
};
struct AddF32 {
  using S = float;
  __device__ static S add(S a, S b) { return a + b; }
};
template <typename T, typename U>
struct AddWrap {  // two's-complement wrap-around through the unsigned type
  using S = T;
  __device__ static S add(S a, S b) { return (S)(U)((U)a + (U)b); }
};

template <typename Op>
__global__ void __launch_bounds__(256) peers_reduce_kernel(const __grid_constant__ PeerList src,
                                                           int npeers, typename Op::S* out,
                                                           size_t elems, int vec) {
  using S = typename Op::S;
  constexpr int E = 16 / sizeof(S);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t nvec = vec ? elems / E : 0;
  for (size_t i = tid; i < nvec; i += stride) {
    S acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = S(0);
    for (int r = 0; r < npeers; ++r) {
      const uint4 w = reinterpret_cast<const uint4*>(src.p[r])[i];
      const S* x = reinterpret_cast<const S*>(&w);
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] = Op::add(acc[e], x[e]);
    }
    reinterpret_cast<uint4*>(out)[i] = *reinterpret_cast<const uint4*>(acc);
  }
  for (size_t i = nvec * E + tid; i < elems; i += stride) {
    S acc = S(0);
    for (int r = 0; r < npeers; ++r) acc = Op::add(acc, reinterpret_cast<const S*>(src.p[r])[i]);
    out[i] = acc;
  }
}

__global__ void __launch_bounds__(256) multimem_st_kernel(const __grid_constant__ PeerList dst,
                                                          int ndst, const uint8_t* src,
                                                          size_t nbytes, int vec) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t nvec = vec ? nbytes / 16 : 0;
  for (size_t i = tid; i < nvec; i += stride) {
    const uint4 v = reinterpret_cast<const uint4*>(src)[i];
    for (int d = 0; d < ndst; ++d) reinterpret_cast<uint4*>(dst.p[d])[i] = v;
  }
  for (size_t i = nvec * 16 + tid; i < nbytes; i += stride) {
    const uint8_t v = src[i];
    for (int d = 0; d < ndst; ++d) dst.p[d][i] = v;
  }
}

// Bounded spin for the wait conditions the front end cannot evaluate.
__global__ void flag_wait_cond_kernel(const uint64_t* flag, int cond, uint64_t value, int* err,
                                      uint64_t timeout_ns) {
  if (threadIdx.x != 0) return;
  uint64_t t0 = globaltimer();
  for (uint32_t i = 1;; ++i) {
    const uint64_t v = ld_acquire_sys(flag);
    const bool ok = cond == 0 ? v == value : cond == 1 ? v != value : cond == 2 ? v >= value
                  : cond == 3 ? v > value : cond == 4 ? v <= value : v < value;
    if (ok) return;
    if ((i & 255) == 0 && err && *reinterpret_cast<volatile int*>(err) != 0) return;
    if (globaltimer() - t0 > timeout_ns) {
      if (err) atomicCAS(err, 0, 4);
      return;
    }
    __nanosleep(256);
  }
}

__global__ void flag_add_kernel(uint64_t* flag, uint64_t value) {
  if (threadIdx.x == 0) {
    __threadfence_system();
    red_add_release_sys(flag, value);
  }
}

// Flag publication: one release store per peer (the signal_op(SET) of
// reference collectives.py:97 / :161 for a whole chunk).
__global__ void flag_store_kernel(uint64_t* const* ptrs, int count, uint64_t value) {
  int i = threadIdx.x;
  if (i < count) {
    __threadfence_system();
    st_release_sys(ptrs[i], value);
  }
}

struct FlagList {
  uint64_t* ptr[kMaxWorld];
};

__global__ void flag_store_list_kernel(const __grid_constant__ FlagList l, int count,
                                       uint64_t value) {
  int i = threadIdx.x;
  if (i < count) {
    __threadfence_system();
    st_release_sys(l.ptr[i], value);
  }
}

// Release-store `value` into `count` consecutive signal words (recovery of a
// world whose stream waits on flags nobody will release).
__global__ void flag_fill_kernel(uint64_t* words, int count, uint64_t value) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x)
    st_release_sys(words + i, value);
}

// Stream-side wait on a local flag (used only when stream memory operations
// are unavailable).
__global__ void flag_wait_kernel(const uint64_t* flag, uint64_t target, int* err,
                                 uint64_t timeout_ns) {
  if (threadIdx.x == 0) spin_geq(flag, target, err, timeout_ns, 4);
}

}  // namespace shb
