// Host side of the C ABI (include/shmem_b200.h): symmetric heap, flag/epoch
// protocol, tensor-map construction and kernel launch for the fused
// AllGather+GEMM and GEMM+ReduceScatter paths.
//
// Heap layout is the reference's (core.py:159-160, 242-261): every rank owns a
// slab of `heap_bytes + 8*signal_count` bytes; symmetric handles are offsets
// valid in every slab; signal word `sig` lives at slab + heap_bytes + 8*sig.
// Here each slab is device memory on the rank's GPU and every other rank holds
// a peer mapping of it (cudaDeviceEnablePeerAccess in one process, CUDA IPC
// across processes), so a "remote write" is an NVLink store.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/shmem_b200.h"
#include "gemm_sm100.cuh"

using namespace shb;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      return fail(SH_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),   \
                  __FILE__, __LINE__);                                                    \
  } while (0)

// ---------------------------------------------------------------------------
// driver entry points (no link-time dependency on libcuda)

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*PFN_streamWaitValue64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
typedef CUresult (*PFN_writeValue64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);

struct Driver {
  PFN_encodeTiled encode = nullptr;
  PFN_streamWaitValue64 wait64 = nullptr;
  PFN_writeValue64 write64 = nullptr;
  bool ok = false;
  std::string why;
};

Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess && fn) {
      d.encode = reinterpret_cast<PFN_encodeTiled>(fn);
      d.ok = true;
    } else {
      d.why = "cuTensorMapEncodeTiled unavailable";
    }
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess && fn)
      d.wait64 = reinterpret_cast<PFN_streamWaitValue64>(fn);
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess && fn)
      d.write64 = reinterpret_cast<PFN_writeValue64>(fn);
  });
  return d;
}

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

// ---------------------------------------------------------------------------
// tile configuration

std::atomic<int> g_force_bn{0};
std::atomic<int> g_force_cg{0};
std::atomic<int> g_stream_k{-2};  // -2: not set (env SHB_SK or auto), -1 auto, 0 off, 1 on
std::atomic<int> g_group_m{-1};   // -1: not set (env SHB_GROUP_M or auto), 0 auto, >0 fixed

int num_sms(int dev) {
  static int cache[64] = {0};
  if (dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = v > 0 ? v : 148;
  }
  return cache[dev];
}

struct Cfg {
  int bn, cg, grid, mblk, nblk, tiles;
};

// Stream-K tail: when the last wave of tiles would leave many CTA pairs idle,
// the last full wave plus the partial one are split by k-block over all
// clusters (the rest stays one-tile-per-cluster).  Returns dp_tiles.
int stream_k_split(const Cfg& c, int num_kb) {
  const int clusters = c.grid / c.cg;
  int mode = g_stream_k.load();  // -1 auto, 0 off, 1 on
  if (mode == -2) {
    const char* env = getenv("SHB_SK");
    mode = env ? (atoi(env) != 0 ? 1 : 0) : -1;
  }
  if (mode == 0) return c.tiles;
  // wide tiles: one wave by construction, and splitting K would put the
  // m-blocks of a column block at different k (B re-read from DRAM)
  if (c.bn == 512 && mode != 1) return c.tiles;
  const int waves = (c.tiles + clusters - 1) / clusters;
  const double eff = double(c.tiles) / double(waves * clusters);
  // long K only: the split's fp32 partials and fixups cost a fixed amount
  // per tile; measured on the TP proxy at M=1024 (ncu): RS k=3584 (56
  // k-blocks) 72 -> 62 us and k=7168 104 -> 97 us without it, AG k=8192
  // (128 k-blocks) 187 -> 162 us with it
  const bool want = mode == 1 || (eff < 0.92 && num_kb >= 128);
  if (!want || c.tiles <= 0) return c.tiles;
  const int full = c.tiles / clusters;
  return full > 1 ? (full - 1) * clusters : 0;
}

// Weighted stream-K partition for the AG GEMM at W>1 (TileParams::sk_late):
// with the own chunk first in the order, clusters [tiles_first, clusters)
// open on the next chunk and wait for its push -- about chunk_bytes over
// NVLink (770 GB/s measured) -- so their stream-K share shrinks by that many
// k-block units.  SHB_SK_LATE="L,d" forces the partition (tests at W=1).
void sk_late_partition(const Cfg& c, TileParams& p, int world, size_t chunk_bytes, int sms) {
  const int clusters = c.grid / c.cg;
  const int num_kb = (p.k + 63) / 64;
  const long long U = (long long)(p.num_tiles - p.dp_tiles) * num_kb;
  long long L = 0, d = 0;
  if (const char* e = getenv("SHB_SK_LATE")) {
    if (sscanf(e, "%lld,%lld", &L, &d) != 2) L = d = 0;
  } else if (world > 1) {
    const int tiles_first = p.mblk * p.nblk;
    if (tiles_first < clusters) {
      L = clusters - tiles_first;
      // one k-block of a cluster tile at ~1.4 PFLOP/s spread over the SMs
      const double t_kb = 2.0 * (128.0 * c.cg) * c.bn * 64.0 / (1.4e15 * c.cg / sms);
      d = (long long)(chunk_bytes / 770e9 / t_kb);
    }
  }
  const long long cap = U / clusters / 2;  // never more than half a share
  if (d > cap) d = cap;
  if (L <= 0 || L >= clusters || d <= 0) return;
  p.sk_late = (int)L;
  p.sk_late_units = (int)d;
}

// Sub-chunk count of the AG pushes (see sh_ag_gemm_ex): S > 1 splits every
// pushed shard into S row ranges, each released by its own flag write.  Off
// by default: measured on the TP=8 proxy (tp_proxy.py), every stream memory
// op with its memory barrier costs ~7 us of front-end time, so 4 ranges per
// shard stretch the push pipeline by ~3x that per chunk, while the clusters
// that open on a remote chunk need rows from all of its m-blocks anyway (the
// raster walks the chunk's m-blocks first).  SHB_AG_SUB=S forces S.
int ag_subchunks(int rows, int k, int world) {
  (void)rows;
  (void)k;
  if (world <= 1) return 1;
  if (const char* e = getenv("SHB_AG_SUB")) return std::max(1, std::min(64, atoi(e)));
  return 1;
}

// fp32 partial workspace for the stream-K tail of one stream of launches.
struct SkWorkspace {
  float* ws = nullptr;
  uint64_t* flags = nullptr;
  size_t ws_bytes = 0;
  uint64_t epoch = 0;
};

int sk_reserve(SkWorkspace& w, int clusters, int cg, int bn) {
  const size_t need = (size_t)clusters * cg * 128 * bn * sizeof(float);
  const size_t nflags = (size_t)clusters * cg * 4;
  if (w.ws && w.ws_bytes >= need) return SH_OK;
  if (w.ws) {
    cudaDeviceSynchronize();
    cudaFree(w.ws);
    cudaFree(w.flags);
    w.ws = nullptr;
  }
  const size_t cap_clusters = 128;  // >= any B200 SM count / 2
  const size_t bytes = std::max(need, cap_clusters * 2 * 128 * 256 * sizeof(float));
  CUDA_TRY(cudaMalloc(&w.ws, bytes));
  CUDA_TRY(cudaMalloc(&w.flags, cap_clusters * 2 * 4 * sizeof(uint64_t)));
  CUDA_TRY(cudaMemset(w.flags, 0, cap_clusters * 2 * 4 * sizeof(uint64_t)));
  CUDA_TRY(cudaDeviceSynchronize());
  (void)nflags;
  w.ws_bytes = bytes;
  w.epoch = 0;
  return SH_OK;
}

// Raster group (m-blocks walked before moving to the next n-block).  Two
// regimes:
//  * short K: a group of m-blocks whose A rows fit in ~32 MB of L2 stays
//    resident while B streams through once per group (B200's L2 behaves like
//    ~2 x 63 MB for data that every SM touches, so budget well under 63 MB);
//  * long K (the A rows of even a few m-blocks exceed the budget): nothing
//    stays resident across tiles; the reuse comes from the clusters of one
//    wave walking K in near lockstep, so each k-slice of a block is fetched
//    once per wave.  DRAM reads per wave ~ (distinct m-blocks + distinct
//    n-blocks), minimised by a square wave: group ~ sqrt(clusters).
// Less DRAM traffic = less power = higher clocks under the 1 kW cap.
int raster_group(int rows, int k, int mblk, int bm, int clusters) {
  const int forced = g_group_m.load();
  if (forced > 0) return std::max(1, std::min(mblk, forced));
  if (const char* e = getenv("SHB_GROUP_M"); e && forced < 0)
    return std::max(1, std::min(mblk, atoi(e)));
  const double budget = 32.0 * (1 << 20);
  const double a_blk = (double)bm * k * 2;
  if (a_blk * mblk <= budget) return std::max(1, mblk);
  const int resident = (int)(budget / a_blk);
  int square = 1;
  while ((square + 1) * (square + 1) <= clusters) ++square;
  const int g = std::max(1, std::min(mblk, std::max(resident, square)));
  // equal-sized groups (C4: 16 + 16 instead of 17 + 15; DRAM 216 -> 200 MB)
  const int ngroups = (mblk + g - 1) / g;
  return (mblk + ngroups - 1) / ngroups;
}

// Raster regions of a launch (TileParams::reg_*): starts[0..nreg] are the
// first chunk positions of each region, starts[nreg] = world.
void set_regions(TileParams& p, const int* starts, int nreg, int bm, int clusters) {
  p.nreg = nreg;
  int g0 = 0;
  for (int r = 0; r < nreg; ++r) {
    const int np = starts[r + 1] - starts[r];
    p.reg_s0[r] = starts[r];
    p.reg_gm[r] = raster_group(p.rows * np, p.k, p.mblk * np, bm, clusters);
    p.reg_g0[r] = g0;
    g0 += (p.mblk * np + p.reg_gm[r] - 1) / p.reg_gm[r];
  }
  p.reg_s0[nreg] = starts[nreg];
}

// Pair-chunk tiles (chunks of <= 128 rows, TileParams::pair_chunks): a CTA
// pair's two CTAs take two consecutive chunk positions, one cluster per
// tile.  Tile width 256 or 224, whichever needs less (waves x BN) of MMA
// time per cluster: RS at TP=8, M=1024 (n=8192) is 128 tiles of 256 = 2
// waves of 74 clusters at 86 % fill, or 148 tiles of 224 = 2 full waves
// (TP=8 proxy, preset: 76.3 -> 73.4 us per call).  A stream-K split over
// every cluster for the AG's partial wave (56 tiles on 74 clusters, 128
// k-blocks) measured slower (73 -> 79 us) and is not offered.
// SHB_PAIR_BN=256|224 forces the width.
Cfg pair_chunk_cfg(int W, int n, int sms) {
  const int clusters = sms / 2;
  const int forced = env_int("SHB_PAIR_BN", 0);
  auto make = [&](int bn) {
    const int nblk = (n + bn - 1) / bn, tiles = (W / 2) * nblk;
    return Cfg{bn, 2, std::min(tiles, clusters) * 2, 1, nblk, tiles};
  };
  if (forced == 224 || forced == 256) return make(forced);
  const Cfg wide = make(256), narrow = make(224);
  auto cost = [&](const Cfg& c) { return (double)((c.tiles + clusters - 1) / clusters) * c.bn; };
  // narrow tiles stage more operand bytes per flop: 224 only for a clear gain
  return cost(narrow) < 0.95 * cost(wide) ? narrow : wide;
}

Cfg choose_cfg(int rows, int world, int n, int sms, int share = 1, int k = 0) {
  // ranks sharing one GPU split its SMs, so that all their persistent GEMMs
  // are co-resident (their epilogues wait on each other's stores)
  if (share > 1) sms = std::max(2, (sms / share) & ~1);
  // Wide 256 x 512 pair tiles for long-K grids of at most one tile per
  // cluster: every cluster then streams its own 512 B columns once, all
  // m-blocks of a column block walk K together (B leaves DRAM once), and the
  // single-buffered accumulator's epilogue happens once.  C5 RS at M=1024
  // (k=28672): 256x256 stream-K read 1.85 GB from DRAM for a 0.53 GB
  // problem (ncu, profiles/README.md); cuBLAS picks 256x512 there too.
  if (g_force_bn == 512 ||
      (!g_force_bn && k >= 8192 && rows > 128 && g_force_cg != 1 && n % 512 == 0)) {
    const int mblk = (rows + 255) / 256, nblk = (n + 511) / 512, tiles = world * mblk * nblk;
    if (g_force_bn == 512 || (tiles <= sms / 2 && tiles * 2 > sms / 2)) {
      const int clusters = std::min(tiles, sms / 2);
      return Cfg{512, 2, clusters * 2, mblk, nblk, tiles};
    }
  }
  int cgs[2] = {2, 1};
  int bns[3] = {256, 224, 128};
  Cfg best{};
  double best_score = -1;
  for (int ci = 0; ci < 2; ++ci) {
    int cg = cgs[ci];
    if (g_force_cg && g_force_cg != cg) continue;
    // single-CTA tiles stage 1.5x the operand bytes per flop of a pair tile;
    // they win only where a 256-row pair tile would be mostly padding (a
    // chunk of <= 128 rows: TP=8 at M=1024)
    if (!g_force_cg && cg == 1 && rows > 128) continue;
    for (int bi = 0; bi < 3; ++bi) {
      int bn = bns[bi];
      if (g_force_bn && g_force_bn != bn) continue;
      if (cg == 2 && bn < 128) continue;
      if (cg == 1 && bn % 64) continue;
      int bm = 128 * cg;
      int mblk = (rows + bm - 1) / bm;
      int nblk = (n + bn - 1) / bn;
      int tiles = world * mblk * nblk;
      int max_clusters = sms / cg;
      int clusters = tiles < max_clusters ? tiles : max_clusters;
      int waves = (tiles + clusters - 1) / clusters;
      double eff = double(tiles) / double(waves * clusters) * double(clusters * cg) / sms;
      // useful-work fraction (ragged edges compute padding) times wave fill,
      // with a small penalty for narrow tiles (more operand traffic per flop)
      double useful = double(rows) * n / (double(mblk) * bm * nblk * bn);
      // measured on B200: a 256x128 pair tile runs at ~0.6x the per-flop rate
      // of 256x256 (operand smem traffic per MMA doubles), so narrow tiles
      // only win when they avoid a large amount of padding
      double score = eff * useful * (bn == 256 ? 1.0 : bn == 224 ? 0.85 : 0.6) *
                     (cg == 1 ? 0.8 : 1.0);
      if (score > best_score) {
        best_score = score;
        best = Cfg{bn, cg, clusters * cg, mblk, nblk, tiles};
      }
    }
  }
  if (best_score < 0) {  // an override with no legal tile: use the default pair tile
    int mblk = (rows + 255) / 256, nblk = (n + 255) / 256, tiles = world * mblk * nblk;
    int clusters = std::min(tiles, sms / 2);
    best = Cfg{256, 2, clusters * 2, mblk, nblk, tiles};
  }
  return best;
}

// ---------------------------------------------------------------------------
// tensor maps

// L2 sector promotion of the TMA fetches (SHB_L2_PROMO 0 none, 1 64 B,
// 2 128 B, 3 256 B = default)
CUtensorMapL2promotion l2_promotion() {
  switch (env_int("SHB_L2_PROMO", 3)) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 2: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
}

// Per-thread cache of encoded tensor maps: a call's maps are identical to the
// previous call's whenever the tensors are (the caching allocator hands the
// same outputs back), and each encode is host time on every launch.
struct MapKey {
  const void* ptr;
  uint64_t dims[3], strides[2];
  uint32_t box[3];
  int rank, dtype, swz, promo;
  bool operator==(const MapKey& o) const { return std::memcmp(this, &o, sizeof(MapKey)) == 0; }
};
constexpr int kMapCache = 32;
struct MapCache {
  MapKey key[kMapCache];
  CUtensorMap map[kMapCache];
  int used = 0, next = 0;
};

int make_map(CUtensorMap* m, int dtype, const void* ptr, int rank, const uint64_t* dims,
             const uint64_t* strides_bytes, const uint32_t* box,
             CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  static thread_local MapCache cache;
  static const CUtensorMapL2promotion promo = l2_promotion();
  MapKey key;
  std::memset(&key, 0, sizeof(key));
  key.ptr = ptr;
  for (int i = 0; i < rank; ++i) {
    key.dims[i] = dims[i];
    key.box[i] = box[i];
  }
  for (int i = 0; i < rank - 1; ++i) key.strides[i] = strides_bytes[i];
  key.rank = rank;
  key.dtype = dtype;
  key.swz = (int)swz;
  key.promo = (int)promo;
  for (int i = 0; i < cache.used; ++i)
    if (cache.key[i] == key) {
      *m = cache.map[i];
      return SH_OK;
    }
  Driver& d = driver();
  if (!d.ok) return fail(SH_ERR_CUDA, "%s", d.why.c_str());
  cuuint64_t gd[3];
  cuuint64_t gs[2];
  cuuint32_t bx[3];
  cuuint32_t es[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) {
    gd[i] = dims[i];
    bx[i] = box[i];
  }
  for (int i = 0; i < rank - 1; ++i) gs[i] = strides_bytes[i];
  CUresult r = d.encode(m, dtype == SH_DTYPE_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                  : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                        rank, const_cast<void*>(ptr), gd, gs, bx, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, promo,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(SH_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) ptr=%p dims=%llu,%llu", (int)r,
                ptr, (unsigned long long)dims[0], (unsigned long long)dims[1]);
  const int slot = cache.used < kMapCache ? cache.used++ : (cache.next++ % kMapCache);
  cache.key[slot] = key;
  cache.map[slot] = *m;
  return SH_OK;
}

// ---------------------------------------------------------------------------
// kernel dispatch

template <int BN, int CG, int MODE, bool FP16>
int launch_one(const TensorMaps& maps, const TileParams& p, int grid, cudaStream_t s, bool pdl) {
  using C = GemmCfg<BN, CG>;
  auto kern = gemm_tp_kernel<BN, CG, MODE, FP16>;
  // smem attribute + carveout are set per device by preload_kernels()
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, maps, p));
  return SH_OK;
}

template <int MODE, bool FP16>
int launch_mode(const Cfg& c, const TensorMaps& maps, const TileParams& p, cudaStream_t s,
                bool pdl) {
  if (c.cg == 2) {
    if (c.bn == 512) return launch_one<512, 2, MODE, FP16>(maps, p, c.grid, s, pdl);
    if (c.bn == 256) return launch_one<256, 2, MODE, FP16>(maps, p, c.grid, s, pdl);
    if (c.bn == 224) return launch_one<224, 2, MODE, FP16>(maps, p, c.grid, s, pdl);
    return launch_one<128, 2, MODE, FP16>(maps, p, c.grid, s, pdl);
  }
  if (c.bn == 256) return launch_one<256, 1, MODE, FP16>(maps, p, c.grid, s, pdl);
  return launch_one<128, 1, MODE, FP16>(maps, p, c.grid, s, pdl);
}

uint64_t l2_policy(const char* env, uint64_t dflt) {
  const char* v = getenv(env);
  if (!v) return dflt;
  if (!strcmp(v, "first")) return kEvictFirst;
  if (!strcmp(v, "last")) return kEvictLast;
  return kEvictNormal;
}

// Programmatic dependent launch of back-to-back GEMMs on one stream (the
// next grid's prologue overlaps this grid's tail).  Off for ranks that share
// a GPU: their persistent grids must stay co-resident.  SHB_PDL=0 disables.
template <int MODE>
int launch_gemm(int dtype, const Cfg& c, const TensorMaps& maps, const TileParams& pin,
                cudaStream_t s, bool shares_gpu = false) {
  const bool pdl = !shares_gpu && env_int("SHB_PDL", 1) != 0;
  TileParams p = pin;
  p.l2_hint_a = l2_policy("SHB_HINT_A", kEvictNormal);
  p.l2_hint_b = l2_policy("SHB_HINT_B", kEvictNormal);
  if (MODE == MODE_RS) {  // per-op overrides for the RS operands
    p.l2_hint_a = l2_policy("SHB_HINT_A_RS", p.l2_hint_a);
    p.l2_hint_b = l2_policy("SHB_HINT_B_RS", p.l2_hint_b);
  }
  // RS staging / output stores are evict-first: nothing re-reads them during
  // the launch, and keeping them out of L2 spares the A/B rows the GEMM still
  // reuses (C4: DRAM reads 259 -> 229 MB per launch)
  p.l2_hint_store = MODE == MODE_RS ? l2_policy("SHB_HINT_STORE", kEvictFirst)
                                     : l2_policy("SHB_HINT_STORE_AG", kEvictNormal);
  p.l2_hint_own = MODE == MODE_RS ? l2_policy("SHB_HINT_OWN_RS", kEvictNormal)
                                   : l2_policy("SHB_HINT_OWN", kEvictFirst);
  // 2: the serpentine parity continues across chunks (TP=8 proxy, ncu: RS DRAM
  // reads 579 -> 505 MB, 349 -> 345 us; AG 423 -> 411 MB); = 1 at W = 1
  p.serpentine = env_int("SHB_SERPENTINE", 2);
  p.red_help = env_int("SHB_RED_HELP", 1);
  // K serpentine: AG C3 DRAM reads 484 -> 427 MB per launch; the RS grid
  // (C4: K = 3584, 17 tiles per cluster) reads more with it, so AG only
  p.kserp = env_int("SHB_KSERP", MODE == MODE_AG ? 1 : 0);
  if (env_int("SHB_TRACE", 0))
    fprintf(stderr,
            "[shb] mode=%d bn=%d cg=%d grid=%d rows=%d n=%d k=%d W=%d rank=%d mblk=%d nblk=%d "
            "tiles=%d dp=%d group_m=%d epoch=%llu copy_own=%d fuse=%d err=%p ws=%p "
            "late=%d/%d\n",
            MODE, c.bn, c.cg, c.grid, p.rows, p.n, p.k, p.world, p.rank, p.mblk, p.nblk,
            p.num_tiles, p.dp_tiles, p.group_m, (unsigned long long)p.epoch, p.copy_own,
            p.fuse_reduce, (void*)p.err, (void*)p.ws, p.sk_late, p.sk_late_units);
  if (dtype == SH_DTYPE_FP16) return launch_mode<MODE, true>(c, maps, p, s, pdl);
  return launch_mode<MODE, false>(c, maps, p, s, pdl);
}

// Load every kernel of this library on `dev` now.  With CUDA lazy loading a
// first launch may need a context-wide synchronisation, which deadlocks
// against a kernel of another rank that is spinning on a flag this launch
// is supposed to set (ranks sharing one GPU).
template <int BN, int CG, int MODE, bool FP16>
cudaError_t preload_one() {
  cudaFuncAttributes a;
  auto kern = gemm_tp_kernel<BN, CG, MODE, FP16>;
  cudaError_t e = cudaFuncGetAttributes(&a, kern);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              GemmCfg<BN, CG>::SMEM_BYTES);
}

template <int MODE, bool FP16>
cudaError_t preload_mode() {
  cudaError_t e;
  if ((e = preload_one<512, 2, MODE, FP16>())) return e;
  if ((e = preload_one<256, 2, MODE, FP16>())) return e;
  if ((e = preload_one<224, 2, MODE, FP16>())) return e;
  if ((e = preload_one<128, 2, MODE, FP16>())) return e;
  if ((e = preload_one<256, 1, MODE, FP16>())) return e;
  return preload_one<128, 1, MODE, FP16>();
}

int preload_kernels(int dev) {
  CUDA_TRY(cudaSetDevice(dev));
  CUDA_TRY((preload_mode<MODE_AG, false>()));
  CUDA_TRY((preload_mode<MODE_AG, true>()));
  CUDA_TRY((preload_mode<MODE_RS, false>()));
  CUDA_TRY((preload_mode<MODE_RS, true>()));
  // Small kernels that may spin (or sit next to a spinning kernel) ask for
  // the max-shared-memory carveout: an SM configured for L1 cannot take a
  // GEMM CTA (~225 KB smem) until it drains, and a drained SM is exactly
  // what a spinning reduction would be waiting for.
  const void* small[] = {reinterpret_cast<const void*>(slots_reduce_kernel<__nv_bfloat16, float>),
                         reinterpret_cast<const void*>(slots_reduce_kernel<__half, float>),
                         reinterpret_cast<const void*>(slots_reduce_kernel<float, float>),
                         reinterpret_cast<const void*>(slots_reduce_kernel<int32_t, int32_t>),
                         reinterpret_cast<const void*>(slots_reduce_kernel<long long, long long>),
                         reinterpret_cast<const void*>(peers_reduce_kernel<AddBF16>),
                         reinterpret_cast<const void*>(peers_reduce_kernel<AddFP16>),
                         reinterpret_cast<const void*>(peers_reduce_kernel<AddF32>),
                         reinterpret_cast<const void*>(peers_reduce_kernel<AddWrap<int32_t, uint32_t>>),
                         reinterpret_cast<const void*>(
                             peers_reduce_kernel<AddWrap<long long, unsigned long long>>),
                         reinterpret_cast<const void*>(peers_reduce_kernel<AddWrap<uint8_t, uint8_t>>),
                         reinterpret_cast<const void*>(peers_reduce_kernel<AddWrap<int8_t, uint8_t>>),
                         reinterpret_cast<const void*>(multimem_st_kernel),
                         reinterpret_cast<const void*>(flag_wait_cond_kernel),
                         reinterpret_cast<const void*>(flag_add_kernel),
                         reinterpret_cast<const void*>(rs_reduce_kernel<false>),
                         reinterpret_cast<const void*>(rs_reduce_kernel<true>),
                         reinterpret_cast<const void*>(flag_store_kernel),
                         reinterpret_cast<const void*>(flag_store_list_kernel),
                         reinterpret_cast<const void*>(flag_wait_kernel),
                         reinterpret_cast<const void*>(flag_fill_kernel)};
  for (const void* f : small) {
    cudaFuncAttributes a;
    CUDA_TRY(cudaFuncGetAttributes(&a, f));
    CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
  }
  // the bulk-staged reduction's ring: stages x sources x 4 KB, up to 220 KB
  for (const void* f : {reinterpret_cast<const void*>(rs_reduce_bulk_kernel<false>),
                        reinterpret_cast<const void*>(rs_reduce_bulk_kernel<true>)}) {
    cudaFuncAttributes a;
    CUDA_TRY(cudaFuncGetAttributes(&a, f));
    CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  220 * 1024 + 256));
    CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
  }
  return SH_OK;
}

int ensure_preloaded(int dev) {
  static std::mutex mu;
  static bool done[64] = {false};
  if (dev < 0 || dev >= 64) return fail(SH_ERR_ARG, "device %d", dev);
  std::lock_guard<std::mutex> g(mu);
  if (done[dev]) return SH_OK;
  int cur = 0;
  CUDA_TRY(cudaGetDevice(&cur));
  int rc = preload_kernels(dev);
  CUDA_TRY(cudaSetDevice(cur));
  if (rc) return rc;
  done[dev] = true;
  return SH_OK;
}

std::atomic<int> g_dynamic{-1};  // -1: not set (env SHB_DYN, default off), 0 off, 1 on

// Dynamic (atomic-counter) hand-out of the data-parallel tiles.  Off by
// default: for uniform tiles the static stride schedule gives every cluster
// exactly the same tile count, which the static stream-K split after it
// assumes; measured on C3 the dynamic variant reads ~2% less DRAM but loses
// ~3% tensor-pipe utilisation to the uneven per-cluster tile counts.
bool dynamic_tiles() {
  const int forced = g_dynamic.load();
  if (forced >= 0) return forced != 0;
  const char* e = getenv("SHB_DYN");
  return e ? atoi(e) != 0 : false;
}

// Zero the tile counter on the stream.  A stream memory write runs on the GPU
// front end (no SM): a memset kernel could be starved by spinning GEMMs of
// sibling ranks sharing the GPU, which wait on this very launch.
int zero_counter(int* counter, cudaStream_t s) {
  Driver& d = driver();
  if (d.write64 && d.write64(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(counter),
                             0, CU_STREAM_WRITE_VALUE_DEFAULT) == CUDA_SUCCESS)
    return SH_OK;
  CUDA_TRY(cudaMemsetAsync(counter, 0, 8, s));
  return SH_OK;
}

// Wave lockstep of the data-parallel tiles (see TileParams::wave_flags):
// opt-in (SHB_WAVE=1); not with the dynamic scheduler (no fixed waves).
// Measured on B200 (RS M=16384 K=28672, one launch under ncu): DRAM reads
// 15.0 -> 8.1 GB, 5.50 -> 5.15 ms; but in back-to-back power-capped runs
// the same kernel is 17% slower with it (5.67 -> 6.61 ms median of 5
// interleaved rounds), and C3/C4 lose 3%, so it stays off by default.
constexpr int kWaveFlags = 256;
bool wave_sync_on() { return env_int("SHB_WAVE", 0) != 0; }

template <typename RS>
void attach_wave(RS& rs, TileParams& p) {
  if (!wave_sync_on() || p.tile_counter || !rs.wave) return;
  p.wave_flags = rs.wave;
  p.wave_tag = (++rs.wave_epoch) << 32;
}

// Next slot of the rank's trace ring for a launch of `mode` (0 AG GEMM, 1 RS
// GEMM, 2 RS reduction kernel), cleared on the launch stream first so a
// reused slot holds no records of an older launch.  nullptr: not tracing.
template <typename RS>
uint64_t* trace_slot(RS& rs, int mode, cudaStream_t s) {
  if (!rs.trace) return nullptr;
  const int slot = (int)(rs.trace_count % rs.trace_launches);
  uint64_t* base = rs.trace + (size_t)slot * rs.trace_grid * rs.trace_cap * 4;
  cudaMemsetAsync(base, 0, (size_t)rs.trace_grid * rs.trace_cap * 4 * 8, s);
  rs.trace_modes[slot] = mode;
  ++rs.trace_count;
  return base;
}

template <typename RS>
void attach_trace(RS& rs, TileParams& p, int mode, cudaStream_t s) {
  p.trace = trace_slot(rs, mode, s);
  p.trace_cap = p.trace ? rs.trace_cap : 0;
}

int check_shape(int m, int n, int k, int world, int dtype) {
  if (m < 1 || n < 1 || k < 1) return fail(SH_ERR_ARG, "m, n, k must be >= 1");
  if (world < 1 || world > SH_MAX_WORLD)
    return fail(SH_ERR_ARG, "world %d outside 1..%d", world, SH_MAX_WORLD);
  if (m % world) return fail(SH_ERR_ARG, "M=%d not divisible by world %d", m, world);
  if (dtype != SH_DTYPE_BF16 && dtype != SH_DTYPE_FP16)
    return fail(SH_ERR_ARG, "dtype %d not supported (bf16/fp16 only)", dtype);
  if (n % 8 || k % 8)
    return fail(SH_ERR_ARG, "n (%d) and k (%d) must be multiples of 8 (16-byte TMA rows)", n, k);
  return SH_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Where the W-slot reduction runs.  At W = 1 it is fused into the epilogue
// (one staging buffer feeds both stores).  At W > 1 the default is the
// north star's "GEMM with a scattering epilogue, followed by a vectorised
// in-HBM reduction": on the TP=8 proxy (ncu, one launch each) the GEMM with
// every chunk in one raster region takes 292 us and the separate reduction
// ~21 us, against 338 us for the GEMM whose own-chunk epilogues reduce --
// those reductions compete with the last waves' operand streams and run at
// a few warps per SM.  Ranks of one process that share a GPU run the same
// form (their stream waits for the counters before the reduction launches,
// so no reduction CTA can hold an SM a sibling's persistent GEMM needs).
// Phased calls (serialising tools) are never fused.  SHB_RS_UNFUSED=1 / =0
// forces either form.
bool rs_fused(int phase, int world, bool shares_gpu) {
  (void)shares_gpu;
  if (phase != SH_PHASE_ALL) return false;
  if (const char* e = getenv("SHB_RS_UNFUSED")) return atoi(e) == 0;
  return world == 1;
}

}  // namespace

// ---------------------------------------------------------------------------
// world

struct RankState {
  int rank = -1;
  int device = -1;
  void* slab = nullptr;      // own slab (device memory on `device`)
  bool own_alloc = false;
  void* peer[SH_MAX_WORLD] = {nullptr};  // every slab as seen from this rank's device
  bool ipc_opened[SH_MAX_WORLD] = {false};
  cudaStream_t comm = nullptr;
  cudaEvent_t ev_in = nullptr, ev_done = nullptr;
  int* err_host = nullptr;
  int* err_dev = nullptr;
  bool shares_gpu = false;  // another rank of this process uses the same device
  int ranks_on_device = 1;  // ranks of this process on `device` (incl. this one)
  SkWorkspace sk;           // stream-K partials of this rank's AG launches
  int* tile_counter = nullptr;  // dynamic tile scheduler counter (zeroed per launch)
  unsigned int* exit_ctr = nullptr;  // retired-CTA counts (ExitRelease): AG, RS GEMM, reduction
  uint64_t* wave = nullptr;     // per-cluster wave progress flags (epoch-tagged)
  uint64_t wave_epoch = 0;
  uint64_t* trace = nullptr;  // [max_launches][grid_max][cap][4] timeline records
  int trace_cap = 0, trace_launches = 0, trace_grid = 0;
  long long trace_count = 0;  // launches recorded so far
  std::vector<int> trace_modes;
};

struct sh_world {
  int world = 0;
  size_t heap_bytes = 0;
  int signal_count = 0;
  size_t stride = 0;
  uint64_t timeout_ns = 0;
  bool member = false;
  int member_rank = -1;
  std::mutex mu;
  size_t heap_cursor = 0;
  int sig_cursor = 0;
  RankState r[SH_MAX_WORLD];
};

namespace {

int init_rank_common(sh_world* w, RankState& rs) {
  int rc = ensure_preloaded(rs.device);
  if (rc) return rc;
  CUDA_TRY(cudaSetDevice(rs.device));
  // sized for the widest tile up front: a later growth would synchronise
  // the device, i.e. wait for a sibling rank's spinning GEMM
  if ((rc = sk_reserve(rs.sk, num_sms(rs.device) / 2, 2, 512))) return rc;
  CUDA_TRY(cudaMalloc(&rs.tile_counter, 256));
  CUDA_TRY(cudaMemset(rs.tile_counter, 0, 256));
  CUDA_TRY(cudaMalloc(&rs.exit_ctr, 4 * sizeof(unsigned int)));
  CUDA_TRY(cudaMemset(rs.exit_ctr, 0, 4 * sizeof(unsigned int)));
  CUDA_TRY(cudaMalloc(&rs.wave, kWaveFlags * sizeof(uint64_t)));
  CUDA_TRY(cudaMemset(rs.wave, 0, kWaveFlags * sizeof(uint64_t)));
  CUDA_TRY(cudaStreamCreateWithFlags(&rs.comm, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&rs.ev_in, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&rs.ev_done, cudaEventDisableTiming));
  CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&rs.err_host), sizeof(int), cudaHostAllocMapped));
  *rs.err_host = 0;
  CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&rs.err_dev), rs.err_host, 0));
  (void)w;
  return SH_OK;
}

int validate_world_args(int world_size, size_t heap_bytes, int* signal_count) {
  if (world_size < 1 || world_size > SH_MAX_WORLD)
    return fail(SH_ERR_CONFIG, "world_size %d outside 1..%d", world_size, SH_MAX_WORLD);
  if (heap_bytes == 0) return fail(SH_ERR_CONFIG, "heap_bytes must be > 0");
  if (*signal_count <= 0) *signal_count = (4 * world_size > 64) ? 4 * world_size : 64;
  if (*signal_count < world_size) return fail(SH_ERR_CONFIG, "signal_count must be >= world_size");
  return SH_OK;
}

RankState* rank_of(sh_world* w, int rank) {
  if (!w || rank < 0 || rank >= w->world) return nullptr;
  if (w->member && rank != w->member_rank) return nullptr;
  return &w->r[rank];
}

inline uint64_t* sig_addr(sh_world* w, const RankState& rs, int peer, int sig) {
  return reinterpret_cast<uint64_t*>(static_cast<char*>(rs.peer[peer]) + w->heap_bytes +
                                     8 * (size_t)sig);
}


int stream_wait_geq(RankState& rs, cudaStream_t s, const uint64_t* flag, uint64_t target,
                    uint64_t timeout_ns) {
  if (target == 0) return SH_OK;  // every flag is >= 0
  Driver& d = driver();
  if (env_int("SHB_WAIT_KERNEL", 0)) {
    flag_wait_kernel<<<1, 32, 0, s>>>(flag, target, rs.err_dev, timeout_ns);
    CUDA_TRY(cudaGetLastError());
    return SH_OK;
  }
  if (d.wait64) {
    CUresult r = d.wait64(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag),
                          target, CU_STREAM_WAIT_VALUE_GEQ);
    if (r == CUDA_SUCCESS) return SH_OK;
  }
  flag_wait_kernel<<<1, 32, 0, s>>>(flag, target, rs.err_dev, timeout_ns);
  CUDA_TRY(cudaGetLastError());
  return SH_OK;
}

int store_flags(cudaStream_t s, uint64_t* const* ptrs, int count, uint64_t value) {
  if (count <= 0) return SH_OK;
  // Stream memory operation (executed by the GPU front end, no SM needed,
  // implicit memory barrier before the write = data-before-flag); the
  // one-warp release-store kernel is the fallback.
  // Writes are idempotent SETs, so flags a stream write could not take (e.g.
  // a peer mapping the front end rejects) simply go to the kernel as well.
  static std::atomic<bool> write_value_broken{false};
  Driver& d = driver();
  FlagList l;
  int nk = 0;
  const bool try_wv = d.write64 && !write_value_broken.load() && !env_int("SHB_FLAG_KERNEL", 0);
  for (int i = 0; i < count; ++i) {
    if (try_wv && d.write64(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(ptrs[i]),
                            value, CU_STREAM_WRITE_VALUE_DEFAULT) == CUDA_SUCCESS)
      continue;
    if (try_wv) write_value_broken = true;
    l.ptr[nk++] = ptrs[i];
  }
  if (nk == 0) return SH_OK;
  cudaGetLastError();  // a rejected stream write may leave a sticky-free error behind
  flag_store_list_kernel<<<1, 32, 0, s>>>(l, nk, value);
  CUDA_TRY(cudaGetLastError());
  return SH_OK;
}

// Flags released by the last retiring CTA of the kernel that does the
// reads they vouch for (ExitRelease) instead of stream memory operations
// after it.  SHB_EXIT_RELEASE=0: the stream operations (store_flags).
bool exit_release_on() { return env_int("SHB_EXIT_RELEASE", 1) != 0; }

ExitRelease make_release(uint64_t* const* ptrs, int count, uint64_t value, unsigned int* ctr) {
  ExitRelease r;
  memset(&r, 0, sizeof(r));
  if (env_int("SHB_DIAG_NOFLAGS", 0)) return r;  // diagnostic (see the AG tail)
  for (int i = 0; i < count; ++i) r.ptr[i] = ptrs[i];
  r.count = count;
  r.value = value;
  r.ctr = ctr;
  r.sys_release = env_int("SHB_EXIT_SYS_RELEASE", 0) != 0 ? 1 : 0;
  return r;
}

// Copies of the push / put / get paths.  Across devices (peer access over
// NVLink) cudaMemcpyAsync runs on the copy engines and overlaps a persistent
// GEMM.  Within one device the driver may run it as a copy kernel on the SMs
// (measured with the TP proxy: a feeder copy stalled behind a persistent GEMM
// whose CTAs left no register room for it), which is why ranks sharing a GPU
// push on the caller's stream ahead of their GEMM.
cudaError_t ce_copy(void* dst, const void* src, size_t nbytes, cudaStream_t s) {
  if (nbytes == 0) return cudaSuccess;
  return cudaMemcpyAsync(dst, src, nbytes, cudaMemcpyDefault, s);
}

// Each call bakes its epoch (and the stream-K workspace epoch) into the
// launch parameters; a captured CUDA graph would replay them with the same
// epochs and race on its flags, so capture is refused, not silently recorded.
int refuse_capture(void* stream) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  CUDA_TRY(cudaStreamIsCapturing(static_cast<cudaStream_t>(stream), &st));
  if (st != cudaStreamCaptureStatusNone)
    return fail(SH_ERR_STATE,
                "CUDA graph capture is not supported: epochs are host values baked into "
                "each launch, a replay would reuse them");
  return SH_OK;
}

}  // namespace

extern "C" {

int sh_version(void) { return 1; }

const char* sh_last_error(void) { return g_err.c_str(); }

int sh_world_create(int world_size, const int* devices, size_t heap_bytes, int signal_count,
                    double timeout_s, sh_world** out) {
  if (!out) return fail(SH_ERR_ARG, "out is NULL");
  int rc = validate_world_args(world_size, heap_bytes, &signal_count);
  if (rc) return rc;
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  auto* w = new sh_world();
  w->world = world_size;
  w->heap_bytes = heap_bytes;
  w->signal_count = signal_count;
  w->stride = (heap_bytes + 8 * (size_t)signal_count + 255) & ~size_t(255);
  w->timeout_ns = (uint64_t)(timeout_s > 0 ? timeout_s * 1e9 : 5e9);
  for (int r = 0; r < world_size; ++r) {
    RankState& rs = w->r[r];
    rs.rank = r;
    rs.device = devices ? devices[r] : (ndev ? r % ndev : 0);
    if (rs.device < 0 || rs.device >= ndev) {
      delete w;
      return fail(SH_ERR_CONFIG, "rank %d: device %d not present (%d GPUs)", r, rs.device, ndev);
    }
    if ((rc = init_rank_common(w, rs))) { delete w; return rc; }
    cudaError_t e = cudaMalloc(&rs.slab, w->stride);
    if (e != cudaSuccess) {
      delete w;
      return fail(SH_ERR_ALLOC, "cudaMalloc(%zu) for rank %d slab: %s", w->stride, r,
                  cudaGetErrorString(e));
    }
    rs.own_alloc = true;
    CUDA_TRY(cudaMemset(rs.slab, 0, w->stride));
  }
  // peer mappings: all devices that host ranks see each other over NVLink
  for (int a = 0; a < world_size; ++a)
    for (int b = 0; b < world_size; ++b) {
      int da = w->r[a].device, db = w->r[b].device;
      if (da != db) {
        int can = 0;
        CUDA_TRY(cudaDeviceCanAccessPeer(&can, da, db));
        if (!can) {
          delete w;
          return fail(SH_ERR_CONFIG, "device %d cannot access peer %d", da, db);
        }
        CUDA_TRY(cudaSetDevice(da));
        cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
          delete w;
          return fail(SH_ERR_CUDA, "enable peer %d->%d: %s", da, db, cudaGetErrorString(e));
        }
        cudaGetLastError();
      }
      w->r[a].peer[b] = w->r[b].slab;
    }
  for (int r = 0; r < world_size; ++r) {
    for (int q = 0; q < world_size; ++q)
      if (q != r && w->r[q].device == w->r[r].device) {
        w->r[r].shares_gpu = true;
        w->r[r].ranks_on_device++;
      }
    CUDA_TRY(cudaSetDevice(w->r[r].device));
    CUDA_TRY(cudaDeviceSynchronize());
  }
  *out = w;
  return SH_OK;
}

int sh_world_create_member(int world_size, int rank, int device, size_t heap_bytes,
                           int signal_count, double timeout_s, sh_world** out) {
  if (!out) return fail(SH_ERR_ARG, "out is NULL");
  int rc = validate_world_args(world_size, heap_bytes, &signal_count);
  if (rc) return rc;
  if (rank < 0 || rank >= world_size) return fail(SH_ERR_CONFIG, "rank %d outside world", rank);
  auto* w = new sh_world();
  w->world = world_size;
  w->heap_bytes = heap_bytes;
  w->signal_count = signal_count;
  w->stride = (heap_bytes + 8 * (size_t)signal_count + 255) & ~size_t(255);
  w->timeout_ns = (uint64_t)(timeout_s > 0 ? timeout_s * 1e9 : 5e9);
  w->member = true;
  w->member_rank = rank;
  RankState& rs = w->r[rank];
  rs.rank = rank;
  rs.device = device;
  if ((rc = init_rank_common(w, rs))) { delete w; return rc; }
  cudaError_t e = cudaMalloc(&rs.slab, w->stride);
  if (e != cudaSuccess) {
    delete w;
    return fail(SH_ERR_ALLOC, "cudaMalloc(%zu): %s", w->stride, cudaGetErrorString(e));
  }
  rs.own_alloc = true;
  CUDA_TRY(cudaMemset(rs.slab, 0, w->stride));
  CUDA_TRY(cudaDeviceSynchronize());
  rs.peer[rank] = rs.slab;
  *out = w;
  return SH_OK;
}

int sh_ipc_handle_size(void) { return (int)sizeof(cudaIpcMemHandle_t); }

int sh_export_ipc_handle(sh_world* w, void* handle_out) {
  if (!w || !w->member || !handle_out) return fail(SH_ERR_ARG, "export needs a member world");
  RankState& rs = w->r[w->member_rank];
  CUDA_TRY(cudaSetDevice(rs.device));
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, rs.slab));
  memcpy(handle_out, &h, sizeof(h));
  return SH_OK;
}

int sh_import_ipc_handles(sh_world* w, const void* handles) {
  if (!w || !w->member || !handles) return fail(SH_ERR_ARG, "import needs a member world");
  RankState& rs = w->r[w->member_rank];
  CUDA_TRY(cudaSetDevice(rs.device));
  const char* hp = static_cast<const char*>(handles);
  for (int p = 0; p < w->world; ++p) {
    if (p == w->member_rank) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, hp + p * sizeof(h), sizeof(h));
    void* ptr = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    rs.peer[p] = ptr;
    rs.ipc_opened[p] = true;
  }
  return SH_OK;
}

int sh_world_destroy(sh_world* w) {
  if (!w) return SH_OK;
  for (int r = 0; r < w->world; ++r) {
    RankState& rs = w->r[r];
    if (rs.device < 0) continue;
    cudaSetDevice(rs.device);
    cudaDeviceSynchronize();
    for (int p = 0; p < w->world; ++p)
      if (rs.ipc_opened[p] && rs.peer[p]) cudaIpcCloseMemHandle(rs.peer[p]);
    if (rs.own_alloc && rs.slab) cudaFree(rs.slab);
    if (rs.comm) cudaStreamDestroy(rs.comm);
    if (rs.ev_in) cudaEventDestroy(rs.ev_in);
    if (rs.ev_done) cudaEventDestroy(rs.ev_done);
    if (rs.err_host) cudaFreeHost(rs.err_host);
    if (rs.trace) cudaFree(rs.trace);
    if (rs.tile_counter) cudaFree(rs.tile_counter);
    if (rs.exit_ctr) cudaFree(rs.exit_ctr);
    if (rs.wave) cudaFree(rs.wave);
    if (rs.sk.ws) cudaFree(rs.sk.ws);
    if (rs.sk.flags) cudaFree(rs.sk.flags);
  }
  delete w;
  return SH_OK;
}

int sh_alloc(sh_world* w, size_t nbytes, size_t align, size_t* offset) {
  if (!w || !offset) return fail(SH_ERR_ARG, "null argument");
  if (align < 1 || (align & (align - 1)))
    return fail(SH_ERR_ARG, "alignment %zu is not a power of two", align);
  std::lock_guard<std::mutex> g(w->mu);
  size_t off = (w->heap_cursor + align - 1) & ~(align - 1);
  if (off + nbytes > w->heap_bytes)
    return fail(SH_ERR_ALLOC, "heap exhausted: need %zu at %zu, slab is %zu", nbytes, off,
                w->heap_bytes);
  w->heap_cursor = off + nbytes;
  *offset = off;
  return SH_OK;
}

int sh_alloc_signals(sh_world* w, int count, int* base) {
  if (!w || !base) return fail(SH_ERR_ARG, "null argument");
  if (count < 0) return fail(SH_ERR_ARG, "negative signal allocation");
  std::lock_guard<std::mutex> g(w->mu);
  if (w->sig_cursor + count > w->signal_count)
    return fail(SH_ERR_ALLOC, "signal pad exhausted: need %d at %d, pad is %d", count,
                w->sig_cursor, w->signal_count);
  *base = w->sig_cursor;
  w->sig_cursor += count;
  return SH_OK;
}

int sh_heap_ptr(sh_world* w, int rank, int peer, size_t offset, void** ptr) {
  RankState* rs = rank_of(w, rank);
  if (!rs || !ptr) return fail(SH_ERR_ARG, "bad rank %d", rank);
  if (peer < 0 || peer >= w->world || !rs->peer[peer])
    return fail(SH_ERR_ARG, "peer %d out of range (world %d)", peer, w->world);
  if (offset > w->heap_bytes) return fail(SH_ERR_ARG, "offset %zu outside heap", offset);
  *ptr = static_cast<char*>(rs->peer[peer]) + offset;
  return SH_OK;
}

int sh_signal_ptr(sh_world* w, int rank, int peer, int sig, void** ptr) {
  RankState* rs = rank_of(w, rank);
  if (!rs || !ptr) return fail(SH_ERR_ARG, "bad rank %d", rank);
  if (peer < 0 || peer >= w->world || !rs->peer[peer])
    return fail(SH_ERR_ARG, "peer %d out of range (world %d)", peer, w->world);
  if (sig < 0 || sig >= w->signal_count)
    return fail(SH_ERR_ARG, "signal %d out of pad of %d", sig, w->signal_count);
  *ptr = sig_addr(w, *rs, peer, sig);
  return SH_OK;
}

int sh_read_signals(sh_world* w, int rank, int base, int count, uint64_t* out_host) {
  RankState* rs = rank_of(w, rank);
  if (!rs || !out_host) return fail(SH_ERR_ARG, "bad rank %d", rank);
  if (base < 0 || count < 0 || base + count > w->signal_count)
    return fail(SH_ERR_ARG, "signals [%d, %d) outside pad of %d", base, base + count,
                w->signal_count);
  CUDA_TRY(cudaSetDevice(rs->device));
  CUDA_TRY(cudaMemcpy(out_host, sig_addr(w, *rs, rank, base), 8 * (size_t)count,
                      cudaMemcpyDeviceToHost));
  return SH_OK;
}

int sh_reset_signals(sh_world* w, int rank, int base, int count, void* stream) {
  RankState* rs = rank_of(w, rank);
  if (!rs) return fail(SH_ERR_ARG, "bad rank %d", rank);
  if (base < 0 || count < 0 || base + count > w->signal_count)
    return fail(SH_ERR_ARG, "signals [%d, %d) outside pad of %d", base, base + count,
                w->signal_count);
  CUDA_TRY(cudaSetDevice(rs->device));
  CUDA_TRY(cudaMemsetAsync(sig_addr(w, *rs, rank, base), 0, 8 * (size_t)count,
                           static_cast<cudaStream_t>(stream)));
  return SH_OK;
}

int sh_fill_signals(sh_world* w, int rank, int base, int count, uint64_t value, void* stream) {
  RankState* rs = rank_of(w, rank);
  if (!rs) return fail(SH_ERR_ARG, "bad rank %d", rank);
  if (base < 0 || count < 0 || base + count > w->signal_count)
    return fail(SH_ERR_ARG, "signals [%d, %d) outside pad of %d", base, base + count,
                w->signal_count);
  if (count == 0) return SH_OK;
  CUDA_TRY(cudaSetDevice(rs->device));
  // a kernel of this (preloaded) module: a first launch of a lazily loaded
  // kernel would synchronise the context -- against the very stream that is
  // blocked on these words
  flag_fill_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(sig_addr(w, *rs, rank, base),
                                                                     count, value);
  CUDA_TRY(cudaGetLastError());
  return SH_OK;
}

int sh_poll_error(sh_world* w, int rank, int* code) {
  RankState* rs = rank_of(w, rank);
  if (!rs || !code) return fail(SH_ERR_ARG, "bad rank %d", rank);
  *code = *reinterpret_cast<volatile int*>(rs->err_host);
  return SH_OK;
}

int sh_clear_error(sh_world* w, int rank) {
  RankState* rs = rank_of(w, rank);
  if (!rs) return fail(SH_ERR_ARG, "bad rank %d", rank);
  *reinterpret_cast<volatile int*>(rs->err_host) = 0;
  // a kernel that bailed out on a timeout may have left a retired-CTA count
  // behind (ExitRelease); the caller has drained the device (World.recover)
  if (rs->exit_ctr) {
    CUDA_TRY(cudaSetDevice(rs->device));
    CUDA_TRY(cudaMemset(rs->exit_ctr, 0, 4 * sizeof(unsigned int)));
  }
  return SH_OK;
}

int sh_set_tile_config(int bn, int cta_group) {
  if (bn != 0 && bn != 128 && bn != 224 && bn != 256 && bn != 512)
    return fail(SH_ERR_ARG, "bn must be 0, 128, 224, 256 or 512");
  if (bn == 512 && cta_group == 1) return fail(SH_ERR_ARG, "bn 512 needs cta_group 2");
  if (cta_group < 0 || cta_group > 2) return fail(SH_ERR_ARG, "cta_group must be 0, 1 or 2");
  g_force_bn = bn;
  g_force_cg = cta_group;
  return SH_OK;
}

int sh_trace_enable(sh_world* w, int rank, int records_per_cta, int max_launches) {
  RankState* rs = rank_of(w, rank);
  if (!rs) return fail(SH_ERR_ARG, "bad rank %d", rank);
  CUDA_TRY(cudaSetDevice(rs->device));
  CUDA_TRY(cudaDeviceSynchronize());
  if (rs->trace) cudaFree(rs->trace);
  rs->trace = nullptr;
  rs->trace_count = 0;
  if (records_per_cta <= 0 || max_launches <= 0) return SH_OK;
  rs->trace_cap = records_per_cta;
  rs->trace_launches = max_launches;
  rs->trace_grid = num_sms(rs->device);
  rs->trace_modes.assign(max_launches, -1);
  const size_t bytes = (size_t)max_launches * rs->trace_grid * records_per_cta * 4 * 8;
  CUDA_TRY(cudaMalloc(&rs->trace, bytes));
  CUDA_TRY(cudaMemset(rs->trace, 0, bytes));
  return SH_OK;
}

int sh_trace_read(sh_world* w, int rank, uint64_t* out_host, size_t out_words, int* info) {
  RankState* rs = rank_of(w, rank);
  if (!rs) return fail(SH_ERR_ARG, "bad rank %d", rank);
  if (!rs->trace) return fail(SH_ERR_STATE, "tracing is not enabled on rank %d", rank);
  const size_t words = (size_t)rs->trace_launches * rs->trace_grid * rs->trace_cap * 4;
  if (out_words < words) return fail(SH_ERR_ARG, "need %zu words", words);
  CUDA_TRY(cudaSetDevice(rs->device));
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(out_host, rs->trace, words * 8, cudaMemcpyDeviceToHost));
  if (info) {  // {launches recorded, slots, grid, cap, mode of slot 0..}
    info[0] = (int)rs->trace_count;
    info[1] = rs->trace_launches;
    info[2] = rs->trace_grid;
    info[3] = rs->trace_cap;
    for (int i = 0; i < rs->trace_launches; ++i) info[4 + i] = rs->trace_modes[i];
  }
  return SH_OK;
}

int sh_set_schedule_config(int stream_k, int group_m) {
  if (stream_k < -2 || stream_k > 1) return fail(SH_ERR_ARG, "stream_k must be -2, -1, 0 or 1");
  if (group_m < -1) return fail(SH_ERR_ARG, "group_m must be >= -1");
  g_stream_k = stream_k;
  g_group_m = group_m;
  return SH_OK;
}

int sh_set_dynamic_tiles(int mode) {
  if (mode < -1 || mode > 1) return fail(SH_ERR_ARG, "mode must be -1, 0 or 1");
  g_dynamic = mode;
  return SH_OK;
}

int sh_set_rank_solo(sh_world* w, int rank, int solo) {
  RankState* rs = rank_of(w, rank);
  if (!rs) return fail(SH_ERR_ARG, "bad rank %d", rank);
  if (solo) {
    rs->shares_gpu = false;
    rs->ranks_on_device = 1;
    return SH_OK;
  }
  rs->ranks_on_device = 1;
  rs->shares_gpu = false;
  for (int q = 0; q < w->world; ++q)
    if (q != rank && w->r[q].device == rs->device && w->r[q].rank >= 0) {
      rs->shares_gpu = true;
      rs->ranks_on_device++;
    }
  return SH_OK;
}

// Stream memory operations on an arbitrary 8-byte word (device, or pinned
// host memory under UVA): executed by the GPU front end, no SM involved.
int sh_stream_write_word(void* word, uint64_t value, void* stream) {
  if (!word || (reinterpret_cast<uintptr_t>(word) & 7))
    return fail(SH_ERR_ARG, "word must be 8-byte aligned");
  Driver& d = driver();
  if (!d.write64) return fail(SH_ERR_CUDA, "cuStreamWriteValue64 unavailable");
  CUresult r = d.write64(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(word),
                         value, CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) return fail(SH_ERR_CUDA, "cuStreamWriteValue64: error %d", (int)r);
  return SH_OK;
}

int sh_stream_wait_word(const void* word, uint64_t value, void* stream) {
  if (!word || (reinterpret_cast<uintptr_t>(word) & 7))
    return fail(SH_ERR_ARG, "word must be 8-byte aligned");
  Driver& d = driver();
  if (!d.wait64) return fail(SH_ERR_CUDA, "cuStreamWaitValue64 unavailable");
  CUresult r = d.wait64(reinterpret_cast<CUstream>(stream),
                        reinterpret_cast<CUdeviceptr>(const_cast<void*>(word)), value,
                        CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return fail(SH_ERR_CUDA, "cuStreamWaitValue64: error %d", (int)r);
  return SH_OK;
}

// Host pacer of the TP proxy (tp_proxy.py): spin until a stream has written
// `origin_value` (or more) into the pinned word `origin` -- the moment a
// paced call starts -- then store tick_base + i + 1 into the pinned word
// `tick` at origin + deltas_ns[i] on the host's monotonic clock.  A feeder
// stream gates each flag release on its tick (sh_stream_wait_word): no SM
// and no copy engine is involved, so the kernel under test shares nothing
// with the pacing.  Blocking; call it from its own thread (ctypes drops the
// GIL around the call).
int sh_pace_host(const void* origin, uint64_t origin_value, void* tick, uint64_t tick_base,
                 const uint64_t* deltas_ns, int n, double timeout_s) {
  if (!origin || !tick || n < 0 || (n > 0 && !deltas_ns)) return fail(SH_ERR_ARG, "null pacer argument");
  auto* o = static_cast<const volatile uint64_t*>(origin);
  auto* t = static_cast<volatile uint64_t*>(tick);
  auto now = [] {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (uint64_t)ts.tv_sec * 1000000000ull + (uint64_t)ts.tv_nsec;
  };
  const uint64_t limit = (uint64_t)((timeout_s > 0 ? timeout_s : 10.0) * 1e9);
  const uint64_t t_in = now();
  while (*o < origin_value)
    if (now() - t_in > limit) return fail(SH_ERR_TIMEOUT, "pacer origin never written");
  const uint64_t t0 = now();
  for (int i = 0; i < n; ++i) {
    while (now() - t0 < deltas_ns[i]) {
    }
    std::atomic_thread_fence(std::memory_order_release);
    *t = tick_base + (uint64_t)i + 1;
  }
  return SH_OK;
}


int sh_query_tile_config(int rows, int world, int n, int* bn, int* cta_group, int* grid) {
  int dev = 0;
  cudaGetDevice(&dev);
  Cfg c = choose_cfg(rows, world, n, num_sms(dev));
  // chunks of <= 128 rows in an even world: both ops launch pair-chunk tiles
  // (the RS unless its reduction is forced into the GEMM, SHB_RS_UNFUSED=0)
  if (world % 2 == 0 && rows <= 128 && c.cg == 1 && !g_force_bn && !g_force_cg)
    c = pair_chunk_cfg(world, n, num_sms(dev));
  if (bn) *bn = c.bn;
  if (cta_group) *cta_group = c.cg;
  if (grid) *grid = c.grid;
  return SH_OK;
}

// ---------------------------------------------------------------------------
// plain GEMM core (TP = 1)

// Caller-provided stream-K workspace: fp32 partial slabs + one flag word per
// (cluster, CTA, epilogue warp), zeroed per launch on the caller's stream.
size_t sk_workspace_bytes(const Cfg& c) {
  const size_t clusters = c.grid / c.cg;
  return clusters * c.cg * 128 * (size_t)c.bn * sizeof(float) + clusters * c.cg * 4 * 8;
}

// front of the caller's workspace: dynamic tile counter (256 B), then the
// wave progress flags (kWaveFlags u64)
constexpr size_t kCounterBytes = 256 + kWaveFlags * sizeof(uint64_t);

int sh_gemm_workspace_bytes(int m, int n, int k, size_t* bytes) {
  if (!bytes) return fail(SH_ERR_ARG, "null argument");
  if (m < 1 || n < 1 || k < 1) return fail(SH_ERR_ARG, "m, n, k must be >= 1");
  int dev = 0;
  cudaGetDevice(&dev);
  Cfg cfg = choose_cfg(m, 1, n, num_sms(dev), 1, k);
  *bytes = kCounterBytes +
           (stream_k_split(cfg, (k + 63) / 64) < cfg.tiles ? sk_workspace_bytes(cfg) : 0);
  return SH_OK;
}

int sh_gemm(const void* a, const void* b, void* c, int m, int n, int k, int dtype, void* workspace,
            size_t workspace_bytes, void* stream) {
  int rc = check_shape(m, n, k, 1, dtype);
  if (rc) return rc;
  if (!a || !b || !c) return fail(SH_ERR_ARG, "null tensor");
  if (!aligned16(a) || !aligned16(b) || !aligned16(c))
    return fail(SH_ERR_ARG, "tensors must be 16-byte aligned");
  if ((rc = refuse_capture(stream))) return rc;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if ((rc = ensure_preloaded(dev))) return rc;
  Cfg cfg = choose_cfg(m, 1, n, num_sms(dev), 1, k);
  TensorMaps maps;
  memset(&maps, 0, sizeof(maps));
  const uint64_t es = 2;
  {
    uint64_t d[2] = {(uint64_t)k, (uint64_t)m}, s[1] = {(uint64_t)k * es};
    uint32_t bx[2] = {64, 128};
    if ((rc = make_map(&maps.a_own, dtype, a, 2, d, s, bx))) return rc;
    uint64_t d3[3] = {(uint64_t)k, (uint64_t)m, 1}, s3[2] = {(uint64_t)k * es, (uint64_t)m * k * es};
    uint32_t bx3[3] = {64, 128, 1};
    if ((rc = make_map(&maps.a_all, dtype, a, 3, d3, s3, bx3))) return rc;
  }
  {
    uint64_t d[2] = {(uint64_t)n, (uint64_t)k}, s[1] = {(uint64_t)n * es};
    uint32_t bx[2] = {64, 64};
    if ((rc = make_map(&maps.b, dtype, b, 2, d, s, bx))) return rc;
  }
  {
    uint64_t d3[3] = {(uint64_t)n, (uint64_t)m, 1}, s3[2] = {(uint64_t)n * es, (uint64_t)m * n * es};
    uint32_t bx3[3] = {32, 32, 1};
    if ((rc = make_map(&maps.c, dtype, c, 3, d3, s3, bx3, CU_TENSOR_MAP_SWIZZLE_64B))) return rc;
  }
  TileParams p;
  memset(&p, 0, sizeof(p));
  p.rows = m;
  p.n = n;
  p.k = k;
  p.world = 1;
  p.rank = 0;
  p.mblk = cfg.mblk;
  p.nblk = cfg.nblk;
  p.num_tiles = cfg.tiles;
  p.dp_tiles = stream_k_split(cfg, (k + 63) / 64);
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  const bool have_ws = workspace && aligned16(workspace) && workspace_bytes >= kCounterBytes;
  if (have_ws && dynamic_tiles()) {
    p.tile_counter = static_cast<int*>(workspace);
    if ((rc = zero_counter(p.tile_counter, cs))) return rc;
  }
  if (have_ws && !p.tile_counter && wave_sync_on()) {
    p.wave_flags = reinterpret_cast<uint64_t*>(static_cast<char*>(workspace) + 256);
    p.wave_tag = 1ull << 32;
    CUDA_TRY(cudaMemsetAsync(p.wave_flags, 0, kWaveFlags * sizeof(uint64_t), cs));
  }
  if (p.dp_tiles < p.num_tiles) {
    const size_t need = sk_workspace_bytes(cfg);
    if (!have_ws || workspace_bytes < kCounterBytes + need) {
      p.dp_tiles = p.num_tiles;  // no (or too small a) workspace: plain tiles
    } else {
      char* base = static_cast<char*>(workspace) + kCounterBytes;
      const size_t slabs = need - (size_t)(cfg.grid / cfg.cg) * cfg.cg * 4 * 8;
      p.ws = reinterpret_cast<float*>(base);
      p.ws_flags = reinterpret_cast<uint64_t*>(base + slabs);
      p.ws_epoch = 1;
      CUDA_TRY(cudaMemsetAsync(p.ws_flags, 0, need - slabs, cs));
    }
  }
  p.group_m = raster_group(p.rows, p.k, p.mblk, 128 * cfg.cg, cfg.grid / cfg.cg);
  p.order[0] = 0;
  p.epoch = 1;
  p.timeout_ns = 5000000000ull;
  return launch_gemm<MODE_AG>(dtype, cfg, maps, p, static_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------------------
// fused AllGather + GEMM

int sh_ag_subchunks(int m, int k, int world, int* subchunks) {
  if (!subchunks) return fail(SH_ERR_ARG, "null argument");
  if (m < 1 || k < 1 || world < 1 || m % world) return fail(SH_ERR_ARG, "bad shape");
  *subchunks = ag_subchunks(m / world, k, world);
  return SH_OK;
}

int sh_ag_gemm(sh_world* w, int rank, const void* a_shard, const void* b, void* c,
               size_t gathered_off, int ready_base, int done_base, int m, int n, int k, int dtype,
               const int* chunk_order, uint64_t epoch, void* stream) {
  return sh_ag_gemm_ex(w, rank, a_shard, b, c, gathered_off, ready_base, done_base, m, n, k, dtype,
                       chunk_order, epoch, 0, SH_PHASE_ALL, stream);
}

int sh_ag_gemm_ex(sh_world* w, int rank, const void* a_shard, const void* b, void* c,
                  size_t gathered_off, int ready_base, int done_base, int m, int n, int k,
                  int dtype, const int* chunk_order, uint64_t epoch, int subchunks, int phase,
                  void* stream) {
  RankState* rs = rank_of(w, rank);
  if (!rs) return fail(SH_ERR_ARG, "bad rank %d", rank);
  const int W = w->world;
  int rc = check_shape(m, n, k, W, dtype);
  if (rc) return rc;
  if (!a_shard || !b || !c || !chunk_order) return fail(SH_ERR_ARG, "null argument");
  if (!aligned16(a_shard) || !aligned16(b) || !aligned16(c))
    return fail(SH_ERR_ARG, "tensors must be 16-byte aligned");
  if (epoch < 1) return fail(SH_ERR_ARG, "epoch must be >= 1");
  if (phase < SH_PHASE_ALL || phase > SH_PHASE_COMPUTE)
    return fail(SH_ERR_ARG, "unknown phase %d", phase);
  if ((rc = refuse_capture(stream))) return rc;
  const int rows = m / W;
  const uint64_t es = 2;
  const size_t chunk_bytes = (size_t)rows * k * es;
  if (gathered_off % 16) return fail(SH_ERR_ARG, "gather buffer must be 16-byte aligned");
  if (gathered_off + (size_t)W * chunk_bytes > w->heap_bytes)
    return fail(SH_ERR_ARG, "gather buffer [%zu, +%zu) outside heap of %zu", gathered_off,
                (size_t)W * chunk_bytes, w->heap_bytes);
  if (ready_base < 0 || ready_base + W > w->signal_count || done_base < 0 ||
      done_base + W > w->signal_count)
    return fail(SH_ERR_ARG, "signal sets outside pad");
  {
    unsigned seen = 0;
    for (int i = 0; i < W; ++i) {
      int ch = chunk_order[i];
      if (ch < 0 || ch >= W || (seen >> ch & 1u))
        return fail(SH_ERR_ARG, "chunk order is not a permutation of 0..%d", W - 1);
      seen |= 1u << ch;
    }
  }
  // Sub-chunk flags: the push of a shard is split into S row ranges of
  // sub_rows rows (a multiple of 256, so every m-block of either tile height
  // lies in one range); after range j lands, ready[src] = (epoch-1)*S + j+1.
  // One monotone word per source, so S=1 is the plain per-chunk flag.
  if (subchunks < 0 || subchunks > 64) return fail(SH_ERR_ARG, "subchunks %d outside 0..64", subchunks);
  const int S = W == 1 ? 1 : (subchunks ? subchunks : ag_subchunks(rows, k, W));
  const int sub_rows = S > 1 ? ((rows + S - 1) / S + 255) / 256 * 256 : rows;
  const int S_eff = (rows + sub_rows - 1) / sub_rows;  // a rounding may merge ranges
  CUDA_TRY(cudaSetDevice(rs->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int dev = rs->device;
  Cfg cfg = choose_cfg(rows, W, n, num_sms(dev), rs->ranks_on_device, k);
  // chunks of <= 128 rows: pair tiles over two chunk positions (as in the
  // RS, TileParams::pair_chunks); the own chunk shares its pairs' first
  // tiles with the first remote chunk.  SHB_AG_PAIR_CHUNKS=0: off.
  const bool pair_chunks = W % 2 == 0 && rows <= 128 && cfg.cg == 1 && !g_force_bn &&
                           !g_force_cg && env_int("SHB_AG_PAIR_CHUNKS", 1) != 0;
  if (pair_chunks) {
    int sms = num_sms(dev);
    if (rs->ranks_on_device > 1) sms = std::max(2, (sms / rs->ranks_on_device) & ~1);
    cfg = pair_chunk_cfg(W, n, sms);
  }
  const bool own_by_ce = env_int("SHB_OWN_COPY_CE", 0) != 0;
  const bool do_comm = phase != SH_PHASE_COMPUTE;
  const bool do_compute = phase != SH_PHASE_COMM;

  // ---- comm half: push own shard into every rank's slot `rank`
  // (allgather_push_intra, collectives.py:95-97).  Copy engine, in the order
  // peers consume it under the ring schedule (peer p wants chunk `rank` at
  // step (rank-p) mod W), after p finished reading the previous call.
  // Ranks with a GPU of their own push on a side stream (copy engine), so
  // the GEMM starts on the local shard while the pushes are in flight.
  // Ranks sharing a GPU push on the caller's stream ahead of the GEMM: a
  // side stream's copies could otherwise be queued behind another rank's
  // spinning GEMM on the same device (measured: 13/30 W=8 runs stalled).
  // A phased call (SH_PHASE_COMM) pushes on the caller's stream too, so
  // draining that stream means the pushes and their flags have landed.
  const bool push_on_main =
      rs->shares_gpu || phase != SH_PHASE_ALL || env_int("SHB_PUSH_ON_MAIN", 0) != 0;
  // nothing to push (TP=1, own slot written by the GEMM): keep the side
  // stream out of it entirely -- cross-stream event pairs measured to
  // serialise the caller's pinned copies on other streams at TP=1
  const bool use_comm = do_comm && !push_on_main && (W > 1 || own_by_ce);
  cudaStream_t cs = use_comm ? rs->comm : s;
  if (use_comm) {
    CUDA_TRY(cudaEventRecord(rs->ev_in, s));
    CUDA_TRY(cudaStreamWaitEvent(rs->comm, rs->ev_in, 0));
  }
  char* own_gathered = static_cast<char*>(rs->peer[rank]) + gathered_off;
  if (do_comm) {
    const size_t row_bytes = (size_t)k * es;
    for (int step = 1; step < W; ++step) {
      int p = (rank - step + W) % W;
      if ((rc = stream_wait_geq(*rs, cs, sig_addr(w, *rs, rank, done_base + p), epoch - 1,
                                w->timeout_ns)))
        return rc;
      char* dst = static_cast<char*>(rs->peer[p]) + gathered_off + (size_t)rank * chunk_bytes;
      uint64_t* f = sig_addr(w, *rs, p, ready_base + rank);
      for (int j = 0; j < S_eff; ++j) {
        const size_t r0 = (size_t)j * sub_rows;
        const size_t nr = std::min<size_t>(sub_rows, rows - r0);
        CUDA_TRY(ce_copy(dst + r0 * row_bytes, static_cast<const char*>(a_shard) + r0 * row_bytes,
                         nr * row_bytes, cs));
        if ((rc = store_flags(cs, &f, 1, (epoch - 1) * (uint64_t)S_eff + j + 1))) return rc;
      }
    }
    // own slot: written by the GEMM's idle epilogue warps from L2-hot rows
    // (own_dst below); the copy-engine path stays available for A/B checks
    if (own_by_ce)
      CUDA_TRY(ce_copy(own_gathered + (size_t)rank * chunk_bytes, a_shard, chunk_bytes, cs));
  }
  if (!do_compute) return SH_OK;

  // ---- compute half on the caller's stream
  TensorMaps maps;
  memset(&maps, 0, sizeof(maps));
  {
    uint64_t d[2] = {(uint64_t)k, (uint64_t)rows}, st[1] = {(uint64_t)k * es};
    uint32_t bx[2] = {64, 128};
    if ((rc = make_map(&maps.a_own, dtype, a_shard, 2, d, st, bx))) return rc;
    uint64_t d3[3] = {(uint64_t)k, (uint64_t)rows, (uint64_t)W},
             s3[2] = {(uint64_t)k * es, (uint64_t)chunk_bytes};
    uint32_t bx3[3] = {64, 128, 1};
    if ((rc = make_map(&maps.a_all, dtype, own_gathered, 3, d3, s3, bx3))) return rc;
  }
  {
    uint64_t d[2] = {(uint64_t)n, (uint64_t)k}, st[1] = {(uint64_t)n * es};
    uint32_t bx[2] = {64, 64};
    if ((rc = make_map(&maps.b, dtype, b, 2, d, st, bx))) return rc;
  }
  {
    uint64_t d3[3] = {(uint64_t)n, (uint64_t)rows, (uint64_t)W},
             s3[2] = {(uint64_t)n * es, (uint64_t)rows * n * es};
    uint32_t bx3[3] = {32, 32, 1};
    if ((rc = make_map(&maps.c, dtype, c, 3, d3, s3, bx3, CU_TENSOR_MAP_SWIZZLE_64B))) return rc;
  }
  TileParams p;
  memset(&p, 0, sizeof(p));
  p.rows = rows;
  p.n = n;
  p.k = k;
  p.world = W;
  p.rank = rank;
  p.mblk = cfg.mblk;
  p.nblk = cfg.nblk;
  p.num_tiles = cfg.tiles;
  p.group_m = pair_chunks ? raster_group(p.rows * W, p.k, W / 2, 256, cfg.grid / cfg.cg)
                          : raster_group(p.rows, p.k, p.mblk, 128 * cfg.cg, cfg.grid / cfg.cg);
  p.pair_chunks = pair_chunks ? 1 : 0;
  {
    // Raster regions: the own chunk (position 0) and the first remote one
    // alone, then SHB_AG_MERGE consecutive remote chunks per region (B
    // streamed once per region).  The pushes run ahead of the consumer from
    // the second remote chunk on (C3/TP=8: a 16 MB chunk lands every ~21 us,
    // one chunk position of GEMM takes ~38 us), so a region's later chunks
    // have landed when it opens.  Measured neutral on the TP=8 proxy (ncu:
    // DRAM reads 412 / 408 / 445 MB, 305 / 305 / 306 us for 1 / 2 / 3; the
    // cross-chunk serpentine already keeps B in L2), so default 1: regions
    // are single chunks, and a chunk's tiles never wait on a later push.
    const int mg = std::max(1, env_int("SHB_AG_MERGE", 1));
    int starts[SH_MAX_WORLD + 1], nreg = 0;
    for (int s0 = 0; s0 < W; s0 += (s0 < 2 ? 1 : mg)) starts[nreg++] = s0;
    starts[nreg] = W;
    set_regions(p, starts, nreg, 128 * cfg.cg, cfg.grid / cfg.cg);
  }
  for (int i = 0; i < W; ++i) p.order[i] = chunk_order[i];
  p.epoch = epoch;
  p.ready = sig_addr(w, *rs, rank, ready_base);
  p.ag_sub = S_eff;
  p.ag_sub_rows = sub_rows;
  attach_trace(*rs, p, MODE_AG, s);
  if (dynamic_tiles()) {
    p.tile_counter = rs->tile_counter;
    if ((rc = zero_counter(rs->tile_counter, s))) return rc;
  }
  attach_wave(*rs, p);
  // pair tiles keep one cluster per tile (a stream-K split over every
  // cluster measured slower on the TP=8 proxy, pair_chunk_cfg)
  p.dp_tiles = pair_chunks ? cfg.tiles : stream_k_split(cfg, (k + 63) / 64);
  if (p.dp_tiles < p.num_tiles) {
    if ((rc = sk_reserve(rs->sk, cfg.grid / cfg.cg, cfg.cg, cfg.bn))) return rc;
    p.ws = rs->sk.ws;
    p.ws_flags = rs->sk.flags;
    p.ws_epoch = ++rs->sk.epoch;
    // with sub-chunk flags the late clusters wait for the first range only
    if (!p.tile_counter)
      sk_late_partition(cfg, p, W, chunk_bytes * (S_eff + 1) / (2 * S_eff), num_sms(dev));
  }
  p.copy_own = own_by_ce ? 0 : 1;
  if (p.copy_own) {
    uint64_t d[2] = {(uint64_t)k, (uint64_t)rows}, st[1] = {(uint64_t)k * es};
    uint32_t bx[2] = {64, 128};
    if ((rc = make_map(&maps.own_slot, dtype, own_gathered + (size_t)rank * chunk_bytes, 2, d, st,
                       bx)))
      return rc;
  }
  p.err = rs->err_dev;
  p.timeout_ns = w->timeout_ns;
  // ---- publish "finished reading my gather buffer" to every peer: done[rank]
  // on each, released by the GEMM's last retiring CTA (or stream operations
  // after it); then join the comm stream so the call completes only when
  // a_shard is free.
  uint64_t* fl[SH_MAX_WORLD];
  int cnt = 0;
  for (int q = 0; q < W; ++q)
    if (q != rank) fl[cnt++] = sig_addr(w, *rs, q, done_base + rank);
  const bool in_kernel = exit_release_on();
  if (in_kernel) p.rel = make_release(fl, cnt, epoch, rs->exit_ctr + 0);
  if ((rc = launch_gemm<MODE_AG>(dtype, cfg, maps, p, s, rs->shares_gpu || phase != SH_PHASE_ALL)))
    return rc;
  // (SHB_DIAG_NOFLAGS: diagnostic only, what these stores cost a call on the
  // TP proxy with preset flags)
  if (!in_kernel && cnt > 0 && !env_int("SHB_DIAG_NOFLAGS", 0) &&
      (rc = store_flags(s, fl, cnt, epoch)))
    return rc;
  if (use_comm) {
    CUDA_TRY(cudaEventRecord(rs->ev_done, rs->comm));
    CUDA_TRY(cudaStreamWaitEvent(s, rs->ev_done, 0));
  }
  return SH_OK;
}

// ---------------------------------------------------------------------------
// fused GEMM + ReduceScatter

int sh_gemm_rs(sh_world* w, int rank, const void* a, const void* b, void* out,
               size_t staging_off, int producer_base, int reduction_base, int m, int n, int k,
               int dtype, const int* chunk_order, uint64_t epoch, void* stream) {
  return sh_gemm_rs_ex(w, rank, a, b, out, staging_off, producer_base, reduction_base, m, n, k,
                       dtype, chunk_order, epoch, SH_PHASE_ALL, stream);
}

int sh_gemm_rs_ex(sh_world* w, int rank, const void* a, const void* b, void* out,
                  size_t staging_off, int producer_base, int reduction_base, int m, int n, int k,
                  int dtype, const int* chunk_order, uint64_t epoch, int rs_phase, void* stream) {
  if (rs_phase < SH_PHASE_ALL || rs_phase > SH_PHASE_COMPUTE)
    return fail(SH_ERR_ARG, "unknown phase %d", rs_phase);
  RankState* rs = rank_of(w, rank);
  if (!rs) return fail(SH_ERR_ARG, "bad rank %d", rank);
  const int W = w->world;
  int rc = check_shape(m, n, k, W, dtype);
  if (rc) return rc;
  if (!a || !b || !out || !chunk_order) return fail(SH_ERR_ARG, "null argument");
  if (!aligned16(a) || !aligned16(b) || !aligned16(out))
    return fail(SH_ERR_ARG, "tensors must be 16-byte aligned");
  if (epoch < 1) return fail(SH_ERR_ARG, "epoch must be >= 1");
  if ((rc = refuse_capture(stream))) return rc;
  const int rows = m / W;
  const uint64_t es = 2;
  const size_t slot_bytes = (size_t)rows * n * es;
  if (staging_off % 16) return fail(SH_ERR_ARG, "staging buffer must be 16-byte aligned");
  if (staging_off + (size_t)W * slot_bytes > w->heap_bytes)
    return fail(SH_ERR_ARG, "staging [%zu, +%zu) outside heap of %zu", staging_off,
                (size_t)W * slot_bytes, w->heap_bytes);
  if (producer_base < 0 || producer_base + W > w->signal_count || reduction_base < 0 ||
      reduction_base + W > w->signal_count)
    return fail(SH_ERR_ARG, "signal sets outside pad");
  {
    unsigned seen = 0;
    for (int i = 0; i < W; ++i) {
      int ch = chunk_order[i];
      if (ch < 0 || ch >= W || (seen >> ch & 1u))
        return fail(SH_ERR_ARG, "chunk order is not a permutation of 0..%d", W - 1);
      seen |= 1u << ch;
    }
  }
  CUDA_TRY(cudaSetDevice(rs->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Cfg cfg = choose_cfg(rows, W, n, num_sms(rs->device), rs->ranks_on_device, k);
  const bool fuse = rs_fused(rs_phase, W, rs->shares_gpu);
  // Chunks of <= 128 rows (TP=8 at M=1024) with every chunk in one raster
  // region (no fused reduction): a pair tile's two CTAs take two consecutive
  // chunk positions, 128 rows each, instead of 1-CTA tiles (ncu, RS
  // 1024x8192x3584 at TP=8: see DESIGN).  SHB_RS_PAIR_CHUNKS=0: off.
  const bool pair_chunks = !fuse && W % 2 == 0 && rows <= 128 && cfg.cg == 1 &&
                           !g_force_bn && !g_force_cg && env_int("SHB_RS_PAIR_CHUNKS", 1) != 0;
  if (pair_chunks) {
    int sms = num_sms(rs->device);
    if (rs->ranks_on_device > 1) sms = std::max(2, (sms / rs->ranks_on_device) & ~1);
    cfg = pair_chunk_cfg(W, n, sms);
  }
  // With the reduction fused, the tiles of my own chunk wait for every peer's
  // rows; a cluster that reached them before finishing its peer-chunk tiles
  // would hold back rows a peer is waiting for, on every rank at once.  The
  // own chunk therefore always runs last (the result does not depend on the
  // order: the reduction is ascending by source whatever the schedule).
  int order[SH_MAX_WORLD];
  {
    int j = 0;
    for (int i = 0; i < W; ++i)
      if (!fuse || chunk_order[i] != rank) order[j++] = chunk_order[i];
    if (fuse) order[j++] = rank;
  }
  chunk_order = order;

  TensorMaps maps;
  memset(&maps, 0, sizeof(maps));
  {
    uint64_t d3[3] = {(uint64_t)k, (uint64_t)rows, (uint64_t)W},
             s3[2] = {(uint64_t)k * es, (uint64_t)rows * k * es};
    uint32_t bx3[3] = {64, 128, 1};
    if ((rc = make_map(&maps.a_all, dtype, a, 3, d3, s3, bx3))) return rc;
  }
  {
    uint64_t d[2] = {(uint64_t)n, (uint64_t)k}, st[1] = {(uint64_t)n * es};
    uint32_t bx[2] = {64, 64};
    if ((rc = make_map(&maps.b, dtype, b, 2, d, st, bx))) return rc;
  }
  {
    // reduced output rows (written by the fused epilogue of my own chunk)
    uint64_t d3[3] = {(uint64_t)n, (uint64_t)rows, 1},
             s3[2] = {(uint64_t)n * es, (uint64_t)rows * n * es};
    uint32_t bx3[3] = {32, 32, 1};
    if ((rc = make_map(&maps.c, dtype, out, 3, d3, s3, bx3, CU_TENSOR_MAP_SWIZZLE_64B))) return rc;
  }
  for (int d = 0; d < W; ++d) {
    // rank d's staging slot `rank` (collectives.py:160: dst_off = rank*chunk_bytes)
    char* dst = static_cast<char*>(rs->peer[d]) + staging_off + (size_t)rank * slot_bytes;
    uint64_t dd[2] = {(uint64_t)n, (uint64_t)rows}, st[1] = {(uint64_t)n * es};
    uint32_t bx[2] = {32, 32};
    if ((rc = make_map(&maps.out[d], dtype, dst, 2, dd, st, bx, CU_TENSOR_MAP_SWIZZLE_64B)))
      return rc;
  }
  TileParams p;
  memset(&p, 0, sizeof(p));
  p.rows = rows;
  p.n = n;
  p.k = k;
  p.world = W;
  p.rank = rank;
  p.mblk = cfg.mblk;
  p.nblk = cfg.nblk;
  p.num_tiles = cfg.tiles;
  p.group_m = pair_chunks ? raster_group(p.rows * W, p.k, W / 2, 256, cfg.grid / cfg.cg)
                          : raster_group(p.rows, p.k, p.mblk, 128 * cfg.cg, cfg.grid / cfg.cg);
  p.pair_chunks = pair_chunks ? 1 : 0;
  // One raster region over every chunk that no epilogue waits behind (fused:
  // the peer chunks, the own chunk stays last; unfused: all of them), so B
  // is streamed once per raster group rather than once per chunk (C4 at
  // TP=8: 8 x 58 MB of B).  The peers' chunks then complete together near the
  // end of the region instead of one by one -- the owner waits for the last
  // of them either way, at the start of its own chunk.  SHB_RS_MERGE=0: off.
  {
    const int merge = env_int("SHB_RS_MERGE", 1) ? (fuse ? W - 1 : W) : 1;
    int starts[SH_MAX_WORLD + 1], nreg = 0;
    for (int s0 = 0; s0 < W; s0 += (s0 == 0 ? std::max(1, merge) : 1)) starts[nreg++] = s0;
    starts[nreg] = W;
    set_regions(p, starts, nreg, 128 * cfg.cg, cfg.grid / cfg.cg);
  }
  for (int i = 0; i < W; ++i) p.order[i] = chunk_order[i];
  p.epoch = epoch;
  for (int d = 0; d < W; ++d) p.rs_count[d] = sig_addr(w, *rs, d, reduction_base + rank);
  // my own chunk's staging slot and its reducer (the separate kernel or the
  // fused epilogue) are on this GPU: gpu-scope release for its counter.
  // SHB_RS_OWN_GPU=0: system scope; SHB_DIAG_RS_GPU_SCOPE=1: every chunk at
  // gpu scope (diagnostic, valid only when every rank shares this GPU).
  p.rs_gpu_scope = env_int("SHB_RS_OWN_GPU", 1) ? (1u << rank) : 0u;
  if (env_int("SHB_DIAG_RS_GPU_SCOPE", 0)) {
    bool all_here = true;  // honoured only when every rank's staging is on this GPU
    for (int q = 0; q < W; ++q) all_here = all_here && w->r[q].device == rs->device;
    if (all_here) p.rs_gpu_scope = ~0u;
  }
  p.rs_free = sig_addr(w, *rs, rank, producer_base);
  const uint16_t* staging =
      reinterpret_cast<const uint16_t*>(static_cast<char*>(rs->peer[rank]) + staging_off);
  const size_t slot_elems = (size_t)rows * n;
  const uint64_t target = epoch * (uint64_t)slot_elems;
  // Stream-K tail as in the AG GEMM.  A cluster's stream-K pieces come after
  // its data-parallel tiles; with the reduction fused, an own-chunk tile
  // waits for every peer's contribution, so a peer-chunk piece queued behind
  // it could close a wait cycle across ranks.  The split is therefore only
  // taken when the whole stream-K range lies inside my own chunk, scheduled
  // last (rs_inter_order), or when nothing waits on peers.
  p.dp_tiles = p.num_tiles;
  {
    const int dp = pair_chunks ? cfg.tiles : stream_k_split(cfg, (k + 63) / 64);
    const int per_chunk = cfg.mblk * cfg.nblk;
    const bool safe = !fuse || W == 1 ||
                      (chunk_order[W - 1] == rank && p.num_tiles - dp <= per_chunk);
    if (dp < p.num_tiles && safe) {
      if ((rc = sk_reserve(rs->sk, cfg.grid / cfg.cg, cfg.cg, cfg.bn))) return rc;
      p.dp_tiles = dp;
      p.ws = rs->sk.ws;
      p.ws_flags = rs->sk.flags;
      p.ws_epoch = ++rs->sk.epoch;
    }
  }
  attach_trace(*rs, p, MODE_RS, s);
  if (dynamic_tiles()) {
    p.tile_counter = rs->tile_counter;
    if ((rc = zero_counter(rs->tile_counter, s))) return rc;
  }
  attach_wave(*rs, p);
  p.rs_mine = sig_addr(w, *rs, rank, reduction_base);
  p.rs_target = target;
  p.staging_local = staging;
  p.out_rows = static_cast<uint16_t*>(out);
  p.fuse_reduce = fuse ? 1 : 0;
  p.err = rs->err_dev;
  p.timeout_ns = w->timeout_ns;
  // reduction of my W staging slots in ascending source order: fused into the
  // epilogue of my own chunk's tiles (scheduled last, rs_inter_order), or a
  // separate vectorised pass.  Then publish "reduced epoch" to every peer:
  // frees my staging slots for their next call (the join of
  // collectives.py:1-10, made a flag), released by the last retiring CTA of
  // the kernel that reads the slots (or stream operations after it).  My own
  // slot is rewritten only by my own next call, stream-ordered, so no self flag.
  uint64_t* fl[SH_MAX_WORLD];
  int nfl = 0;
  for (int q = 0; q < W; ++q)
    if (q != rank) fl[nfl++] = sig_addr(w, *rs, q, producer_base + rank);
  const bool in_kernel = exit_release_on();
  if (fuse && in_kernel) p.rel = make_release(fl, nfl, epoch, rs->exit_ctr + 1);
  // the separate reduction's timeline slot is cleared (a memset on the
  // stream) before the GEMM, so a traced call keeps the programmatic
  // dependent launch between the two kernels
  uint64_t* red_tr = (!fuse && rs_phase != SH_PHASE_COMM) ? trace_slot(*rs, 2, s) : nullptr;
  if (rs_phase != SH_PHASE_COMPUTE &&
      (rc = launch_gemm<MODE_RS>(dtype, cfg, maps, p, s, rs->shares_gpu || rs_phase != SH_PHASE_ALL)))
    return rc;
  if (rs_phase == SH_PHASE_COMM) return SH_OK;  // scatter only: reduce in a later phase call
  const bool host_flags = !in_kernel && nfl > 0 && !env_int("SHB_DIAG_NOFLAGS", 0);
  if (fuse) return host_flags ? store_flags(s, fl, nfl, epoch) : SH_OK;
  ExitRelease rel;
  memset(&rel, 0, sizeof(rel));
  if (in_kernel) rel = make_release(fl, nfl, epoch, rs->exit_ctr + 2);
  int sms = num_sms(rs->device);
  size_t nvec = (slot_elems + 7) / 8;
  int grid = (int)std::min<size_t>((nvec + 255) / 256, (size_t)sms * 4);
  if (grid < 1) grid = 1;
  const uint64_t* counters = sig_addr(w, *rs, rank, reduction_base);
  if (rs->shares_gpu && rs_phase == SH_PHASE_ALL) {
    // Ranks sharing a GPU (the separate form forced): the stream waits for
    // every source's counter in the GPU front end before the reduction is
    // launched, so no reduction CTA can occupy an SM that a sibling rank's
    // persistent GEMM still needs (a forced-separate fuzz on one GPU
    // deadlocked 40 % of its W >= 3 cases without this)
    for (int q = 0; q < W; ++q)
      if ((rc = stream_wait_geq(*rs, s, counters + q, target, w->timeout_ns))) return rc;
  }
  // Programmatic dependent launch: the reduction's CTAs may start while the
  // GEMM still runs (it allows dependents right after its prologue) and
  // take SMs as its CTAs retire.  No griddepcontrol.wait: every byte the
  // reduction reads is covered by the element counters it acquires (the own
  // slot's too), and the GEMM never touches `out` in this form.  Not for
  // ranks sharing a GPU or phased calls (SHB_RED_PDL=0 / SHB_PDL=0: off).
  const bool red_pdl = !rs->shares_gpu && rs_phase == SH_PHASE_ALL &&
                       env_int("SHB_PDL", 1) != 0 && env_int("SHB_RED_PDL", 1) != 0;
  {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid, 1, 1);
    lc.blockDim = dim3(256, 1, 1);
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = red_pdl ? 1 : 0;
    uint16_t* o16 = static_cast<uint16_t*>(out);
    // timeline: per CTA (< trace grid) its counter wait (kind 3) and life (kind 4)
    uint64_t* tr = red_tr;
    const int tcap = tr ? rs->trace_cap : 0, tgrid = tr ? rs->trace_grid : 0;
    if (env_int("SHB_RED_BULK", 1) && slot_elems % 8 == 0 && !rs->shares_gpu) {
      // bulk-DMA staged form: W x 4 KB per step in a 3-deep (W > 8: 2-deep)
      // shared-memory ring, two CTAs per SM at W <= 8 (one rank per GPU
      // only: its full-size grid spinning on sibling ranks' counters would
      // hold the SMs their GEMMs still need -- the forced-separate tests on
      // one GPU timed out)
      // SHB_RB_CTAS (CTAs per SM) / SHB_RB_STAGES: A/B knobs, clamped to the
      // shared memory per SM.  TP=8 proxy RS (C4, preset, medians of 4 x 20
      // calls): 2 x 3 stages 342.1 us, 1 x 6 347.9, 1 x 4 356.6, 2 x 2 355.0
      // (scripts/probe/rb_stages.sh)
      const int per_sm = std::max(1, std::min(2, env_int("SHB_RB_CTAS", W > 8 ? 1 : 2)));
      int stages = env_int("SHB_RB_STAGES", W > 8 ? 2 : 3);
      const int max_st = (int)((220 * 1024 / per_sm) / ((size_t)W * kRbChunk));
      stages = std::max(1, std::min(stages, std::max(1, max_st)));
      lc.dynamicSmemBytes = (size_t)stages * W * kRbChunk + 128 + 8 * stages;
      lc.gridDim = dim3(sms * per_sm, 1, 1);
      if (dtype == SH_DTYPE_FP16)
        CUDA_TRY(cudaLaunchKernelEx(&lc, rs_reduce_bulk_kernel<true>, staging, o16, slot_elems,
                                    W, stages, counters, target, rs->err_dev, w->timeout_ns, tr,
                                    tcap, tgrid, rel));
      else
        CUDA_TRY(cudaLaunchKernelEx(&lc, rs_reduce_bulk_kernel<false>, staging, o16, slot_elems,
                                    W, stages, counters, target, rs->err_dev, w->timeout_ns, tr,
                                    tcap, tgrid, rel));
    } else if (dtype == SH_DTYPE_FP16) {
      CUDA_TRY(cudaLaunchKernelEx(&lc, rs_reduce_kernel<true>, staging, o16, slot_elems, W,
                                  counters, target, rs->err_dev, w->timeout_ns, tr, tcap, tgrid,
                                  rel));
    } else {
      CUDA_TRY(cudaLaunchKernelEx(&lc, rs_reduce_kernel<false>, staging, o16, slot_elems, W,
                                  counters, target, rs->err_dev, w->timeout_ns, tr, tcap, tgrid,
                                  rel));
    }
  }

  return host_flags ? store_flags(s, fl, nfl, epoch) : SH_OK;
}

// ---------------------------------------------------------------------------
// one-sided primitives + slot reduction (standalone collectives)

int sh_putmem(sh_world* w, int rank, int peer, size_t dst_off, const void* src, size_t nbytes,
              void* stream) {
  RankState* rs = rank_of(w, rank);
  if (!rs) return fail(SH_ERR_ARG, "bad rank %d", rank);
  if (peer < 0 || peer >= w->world || !rs->peer[peer])
    return fail(SH_ERR_ARG, "peer %d out of range (world %d)", peer, w->world);
  if (dst_off + nbytes > w->heap_bytes)
    return fail(SH_ERR_ARG, "put [%zu, %zu) outside heap of %zu", dst_off, dst_off + nbytes,
                w->heap_bytes);
  if (nbytes == 0) return SH_OK;
  if (!src) return fail(SH_ERR_ARG, "null source");
  CUDA_TRY(cudaSetDevice(rs->device));
  CUDA_TRY(ce_copy(static_cast<char*>(rs->peer[peer]) + dst_off, src, nbytes,
                   static_cast<cudaStream_t>(stream)));
  return SH_OK;
}

int sh_getmem(sh_world* w, int rank, void* dst, int peer, size_t src_off, size_t nbytes,
              void* stream) {
  RankState* rs = rank_of(w, rank);
  if (!rs) return fail(SH_ERR_ARG, "bad rank %d", rank);
  if (peer < 0 || peer >= w->world || !rs->peer[peer])
    return fail(SH_ERR_ARG, "peer %d out of range (world %d)", peer, w->world);
  if (src_off + nbytes > w->heap_bytes)
    return fail(SH_ERR_ARG, "get [%zu, %zu) outside heap of %zu", src_off, src_off + nbytes,
                w->heap_bytes);
  if (nbytes == 0) return SH_OK;
  if (!dst) return fail(SH_ERR_ARG, "null destination");
  CUDA_TRY(cudaSetDevice(rs->device));
  CUDA_TRY(ce_copy(dst, static_cast<char*>(rs->peer[peer]) + src_off, nbytes,
                   static_cast<cudaStream_t>(stream)));
  return SH_OK;
}

int sh_signal_op(sh_world* w, int rank, int peer, int sig, int op, uint64_t value, void* stream) {
  RankState* rs = rank_of(w, rank);
  if (!rs) return fail(SH_ERR_ARG, "bad rank %d", rank);
  if (peer < 0 || peer >= w->world || !rs->peer[peer])
    return fail(SH_ERR_ARG, "peer %d out of range (world %d)", peer, w->world);
  if (sig < 0 || sig >= w->signal_count)
    return fail(SH_ERR_ARG, "signal %d out of pad of %d", sig, w->signal_count);
  CUDA_TRY(cudaSetDevice(rs->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint64_t* f = sig_addr(w, *rs, peer, sig);
  if (op == SH_SIG_SET) return store_flags(s, &f, 1, value);
  if (op != SH_SIG_ADD) return fail(SH_ERR_ARG, "unknown signal op %d", op);
  flag_add_kernel<<<1, 32, 0, s>>>(f, value);
  CUDA_TRY(cudaGetLastError());
  return SH_OK;
}

int sh_signal_wait(sh_world* w, int rank, int sig, int cond, uint64_t value, void* stream) {
  RankState* rs = rank_of(w, rank);
  if (!rs) return fail(SH_ERR_ARG, "bad rank %d", rank);
  if (sig < 0 || sig >= w->signal_count)
    return fail(SH_ERR_ARG, "signal %d out of pad of %d", sig, w->signal_count);
  if (cond < 0 || cond > 5) return fail(SH_ERR_ARG, "unknown wait condition %d", cond);
  CUDA_TRY(cudaSetDevice(rs->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t* f = sig_addr(w, *rs, rank, sig);
  // A user-level wait must honour the world's timeout (a peer that never
  // signals is a SynchronizationFault, not a hung stream): bounded one-thread
  // spin that records the timeout in the error word.  The front-end wait
  // (no SM, no timeout) stays available as SHB_WAIT_MEMOP=1.
  Driver& d = driver();
  if (env_int("SHB_WAIT_MEMOP", 0) && d.wait64 && (cond == 0 || cond == 2)) {
    CUresult r = d.wait64(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(f), value,
                          cond == 0 ? CU_STREAM_WAIT_VALUE_EQ : CU_STREAM_WAIT_VALUE_GEQ);
    if (r == CUDA_SUCCESS) return SH_OK;
  }
  flag_wait_cond_kernel<<<1, 32, 0, s>>>(f, cond, value, rs->err_dev, w->timeout_ns);
  CUDA_TRY(cudaGetLastError());
  return SH_OK;
}

int sh_reduce_slots(sh_world* w, int rank, size_t staging_off, int nslots, size_t slot_elems,
                    int dtype, void* out, void* stream) {
  RankState* rs = rank_of(w, rank);
  if (!rs) return fail(SH_ERR_ARG, "bad rank %d", rank);
  static const size_t esize[] = {2, 2, 4, 4, 8};
  if (dtype < 0 || dtype > 4) return fail(SH_ERR_ARG, "dtype %d not supported", dtype);
  if (nslots < 1) return fail(SH_ERR_ARG, "need at least one slot");
  if (staging_off + (size_t)nslots * slot_elems * esize[dtype] > w->heap_bytes)
    return fail(SH_ERR_ARG, "staging outside heap");
  if (slot_elems == 0) return SH_OK;
  if (!out) return fail(SH_ERR_ARG, "null output");
  CUDA_TRY(cudaSetDevice(rs->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const void* st = static_cast<char*>(rs->peer[rank]) + staging_off;
  int grid = (int)std::min<size_t>((slot_elems + 255) / 256, (size_t)num_sms(rs->device) * 4);
  switch (dtype) {
    case SH_DTYPE_BF16:
      slots_reduce_kernel<__nv_bfloat16, float><<<grid, 256, 0, s>>>(
          static_cast<const __nv_bfloat16*>(st), static_cast<__nv_bfloat16*>(out), slot_elems,
          nslots);
      break;
    case SH_DTYPE_FP16:
      slots_reduce_kernel<__half, float><<<grid, 256, 0, s>>>(
          static_cast<const __half*>(st), static_cast<__half*>(out), slot_elems, nslots);
      break;
    case SH_DTYPE_FP32:
      slots_reduce_kernel<float, float><<<grid, 256, 0, s>>>(
          static_cast<const float*>(st), static_cast<float*>(out), slot_elems, nslots);
      break;
    case SH_DTYPE_I32:
      slots_reduce_kernel<int32_t, int32_t><<<grid, 256, 0, s>>>(
          static_cast<const int32_t*>(st), static_cast<int32_t*>(out), slot_elems, nslots);
      break;
    default:
      slots_reduce_kernel<long long, long long><<<grid, 256, 0, s>>>(
          static_cast<const long long*>(st), static_cast<long long*>(out), slot_elems, nslots);
  }
  CUDA_TRY(cudaGetLastError());
  return SH_OK;
}

namespace {

int node_peers(sh_world* w, RankState* rs, int rank, int first, int count, size_t offset,
               size_t nbytes, PeerList& pl, int& n, bool skip_self) {
  if (first < 0 || count < 1 || first + count > w->world || rank < first || rank >= first + count)
    return fail(SH_ERR_ARG, "node ranks [%d, %d) do not hold rank %d (world %d)", first,
                first + count, rank, w->world);
  if (offset + nbytes > w->heap_bytes || offset + nbytes < offset)
    return fail(SH_ERR_ARG, "range [%zu, %zu) outside heap of %zu", offset, offset + nbytes,
                w->heap_bytes);
  n = 0;
  for (int q = first; q < first + count; ++q) {
    if (skip_self && q == rank) continue;
    if (!rs->peer[q]) return fail(SH_ERR_ARG, "rank %d has no mapping of rank %d", rank, q);
    pl.p[n++] = static_cast<uint8_t*>(rs->peer[q]) + offset;
  }
  return SH_OK;
}

bool all16(const PeerList& pl, int n, const void* extra) {
  for (int i = 0; i < n; ++i)
    if (reinterpret_cast<uintptr_t>(pl.p[i]) & 15) return false;
  return (reinterpret_cast<uintptr_t>(extra) & 15) == 0;
}

}  // namespace

int sh_multimem_st(sh_world* w, int rank, int first, int count, size_t offset, size_t nbytes,
                   void* stream) {
  RankState* rs = rank_of(w, rank);
  if (!rs) return fail(SH_ERR_ARG, "bad rank %d", rank);
  PeerList pl;
  memset(&pl, 0, sizeof(pl));
  int n = 0;
  int rc = node_peers(w, rs, rank, first, count, offset, nbytes, pl, n, true);
  if (rc) return rc;
  if (nbytes == 0 || n == 0) return SH_OK;
  CUDA_TRY(cudaSetDevice(rs->device));
  const uint8_t* src = static_cast<const uint8_t*>(rs->peer[rank]) + offset;
  const int vec = all16(pl, n, src) ? 1 : 0;
  const size_t work = vec ? nbytes / 16 + 1 : nbytes;
  const int grid = (int)std::max<size_t>(1, std::min<size_t>((work + 255) / 256,
                                                             (size_t)num_sms(rs->device) * 4));
  multimem_st_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(pl, n, src, nbytes,
                                                                          vec);
  CUDA_TRY(cudaGetLastError());
  return SH_OK;
}

int sh_multimem_ld_reduce(sh_world* w, int rank, int first, int count, size_t offset,
                          size_t nbytes, int dtype, void* out, void* stream) {
  RankState* rs = rank_of(w, rank);
  if (!rs) return fail(SH_ERR_ARG, "bad rank %d", rank);
  static const size_t esize[] = {2, 2, 4, 4, 8, 1, 1};
  if (dtype < 0 || dtype > SH_DTYPE_I8) return fail(SH_ERR_ARG, "dtype %d not supported", dtype);
  if (nbytes % esize[dtype])
    return fail(SH_ERR_ARG, "%zu bytes not a multiple of %zu-byte elements", nbytes, esize[dtype]);
  PeerList pl;
  memset(&pl, 0, sizeof(pl));
  int n = 0;
  int rc = node_peers(w, rs, rank, first, count, offset, nbytes, pl, n, false);
  if (rc) return rc;
  if (nbytes == 0) return SH_OK;
  if (!out) return fail(SH_ERR_ARG, "null output");
  CUDA_TRY(cudaSetDevice(rs->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t elems = nbytes / esize[dtype];
  const int vec = all16(pl, n, out) ? 1 : 0;
  const size_t work = vec ? nbytes / 16 + 1 : elems;
  const int grid = (int)std::max<size_t>(1, std::min<size_t>((work + 255) / 256,
                                                             (size_t)num_sms(rs->device) * 4));
  switch (dtype) {
    case SH_DTYPE_BF16:
      peers_reduce_kernel<AddBF16><<<grid, 256, 0, s>>>(pl, n, static_cast<uint16_t*>(out), elems, vec);
      break;
    case SH_DTYPE_FP16:
      peers_reduce_kernel<AddFP16><<<grid, 256, 0, s>>>(pl, n, static_cast<uint16_t*>(out), elems, vec);
      break;
    case SH_DTYPE_FP32:
      peers_reduce_kernel<AddF32><<<grid, 256, 0, s>>>(pl, n, static_cast<float*>(out), elems, vec);
      break;
    case SH_DTYPE_I32:
      peers_reduce_kernel<AddWrap<int32_t, uint32_t>><<<grid, 256, 0, s>>>(
          pl, n, static_cast<int32_t*>(out), elems, vec);
      break;
    case SH_DTYPE_I64:
      peers_reduce_kernel<AddWrap<long long, unsigned long long>><<<grid, 256, 0, s>>>(
          pl, n, static_cast<long long*>(out), elems, vec);
      break;
    case SH_DTYPE_U8:
      peers_reduce_kernel<AddWrap<uint8_t, uint8_t>><<<grid, 256, 0, s>>>(
          pl, n, static_cast<uint8_t*>(out), elems, vec);
      break;
    default:
      peers_reduce_kernel<AddWrap<int8_t, uint8_t>><<<grid, 256, 0, s>>>(
          pl, n, static_cast<int8_t*>(out), elems, vec);
  }
  CUDA_TRY(cudaGetLastError());
  return SH_OK;
}

}  // extern "C"
