// claw_host.cpp -- C ABI of libclaw.so (include/claw.h): validation, level
// planning (owner map, ghost-source tables, tiles, halo plan), the device
// patch pool and the per-step driver around the sm_100a kernels.
//
// Paper map: patch hierarchy P:97-106; ghost cells and their three
// sources P:125-132; level-by-level advance P:113-118; CFL P:227-233,
// P:282-288; GPU memory pool P:422-426; one merged launch per level instead of
// per-patch kernels P:296-299; per-patch max-speed array reduced to
// a level max P:417-420.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: ranges cost nothing unless a tool is attached
#include <unistd.h>
#include <nccl.h>

#include <algorithm>
#include <functional>
#include <condition_variable>
#include <climits>
#include <chrono>
#include <array>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <string>
#include <thread>
#include <vector>

#include "../../include/claw.h"
#include "claw_internal.h"

using claw::DevInterp;
using claw::DevPatch;
using claw::DevRect;

namespace {

constexpr int kMaxLevel = 8;
constexpr int kBucket = 16;
constexpr int kBandEdge = 4;   // band split: rows of each edge tile (a multiple of 4)

// ---------------------------------------------------------------------------
// NCCL through dlopen: the library loads without NCCL; world > 1 needs it.
// ---------------------------------------------------------------------------
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  // optional (introspection only): the communicator's own view
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommCuDevice)(const ncclComm_t, int*) = nullptr;
  bool load(std::string& err) {
    if (h) return true;
    // CLAW_NCCL_LIB: an explicit library (tests load a stand-in that runs
    // the same calls between processes sharing one GPU, which NCCL refuses)
    if (const char* lib = std::getenv("CLAW_NCCL_LIB")) {
      h = dlopen(lib, RTLD_NOW | RTLD_LOCAL);
      if (!h) {
        err = std::string("CLAW_NCCL_LIB=") + lib + " could not be loaded";
        return false;
      }
    }
    // prefer the NCCL already in the process (torch's), else load one locally
    // so it cannot interpose on another library's NCCL symbols
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      if (h) break;
      h = dlopen(n, RTLD_NOW | RTLD_NOLOAD);
    }
    for (const char* n : names) {
      if (h) break;
      h = dlopen(n, RTLD_NOW | RTLD_LOCAL);
    }
    if (!h) {
      err = "NCCL (libnccl.so.2) could not be loaded";
      return false;
    }
#define SYM(f)                                                   \
  f = reinterpret_cast<decltype(f)>(dlsym(h, "nccl" #f));        \
  if (!f) {                                                      \
    err = "NCCL symbol nccl" #f " missing";                      \
    return false;                                                \
  }
    SYM(GetUniqueId) SYM(CommInitRank) SYM(CommDestroy) SYM(AllReduce) SYM(Send) SYM(Recv)
    SYM(GroupStart) SYM(GroupEnd) SYM(GetErrorString)
#undef SYM
    CommCount = reinterpret_cast<decltype(CommCount)>(dlsym(h, "ncclCommCount"));
    CommUserRank = reinterpret_cast<decltype(CommUserRank)>(dlsym(h, "ncclCommUserRank"));
    CommCuDevice = reinterpret_cast<decltype(CommCuDevice)>(dlsym(h, "ncclCommCuDevice"));
    return true;
  }
};
Nccl g_nccl;

// ---------------------------------------------------------------------------
// Device memory pool (the paper's GPU memory pool: cudaMalloc per
// patch "can even dominate" with small patches; the paper's pool "allocates a
// huge chunk of memory at a time and allocates more chunks when needed").
// Every device buffer of the library comes from here: per device, chunks of
// >= 1 GiB (growing geometrically up to 2 GiB) from cudaMalloc, carved
// best-fit (512-byte granules) with free ranges coalesced on release, so regrids and re-set levels of varying sizes
// reuse memory without calling cudaMalloc.  Releases happen only after the
// owning context's stream is synchronised (set_level, regrid, destroy), so a
// range is never reused while a kernel may still touch it.  Wholly free chunks
// beyond CLAW_POOL_LIMIT_MB (default 16384) of free memory go back to the
// driver, and a failing cudaMalloc first returns every free chunk and retries.
// ---------------------------------------------------------------------------
// A context created with claw_config.arena (device memory the caller owns,
// e.g. a torch tensor's storage) allocates from that arena only: the arena is
// one borrowed chunk of its own key (device, arena id), carved by the same
// best-fit / coalescing rules, never grown and never freed to the driver
// (a request that does not fit fails with ENOMEM); the thread's current arena
// is the one of the context whose API call is running (set by check_ctx).
thread_local int64_t t_arena = 0;
struct Pool {
  static constexpr size_t kGrain = 512;
  static constexpr size_t kChunk = size_t{1} << 30;  // first chunk (cudaMalloc of a chunk: 15-100 ms)
  struct Dev {
    std::map<char*, size_t> chunks;        // start -> size
    std::map<char*, size_t> free_at;       // free ranges by address
    std::multimap<size_t, char*> free_sz;  // the same by size (best fit)
    size_t free_bytes = 0;
    bool borrowed = false;                 // a caller's arena: no growth, never cudaFree'd
  };
  using Key = std::pair<int, int64_t>;     // (device, arena id; 0 = the library's own chunks)
  std::mutex mu;
  std::map<Key, Dev> devs;
  std::unordered_map<void*, std::pair<Key, size_t>> live;
  int64_t next_arena = 1;
  size_t limit = 0;
  int64_t hits = 0, misses = 0;
  Pool() {
    const char* s = std::getenv("CLAW_POOL_LIMIT_MB");
    limit = static_cast<size_t>(s ? std::atoll(s) : 16384) << 20;
  }
  static bool is_chunk_start(const Dev& d, char* p) { return d.chunks.count(p) != 0; }
  void erase_free(Dev& d, char* p, size_t n) {
    d.free_at.erase(p);
    auto r = d.free_sz.equal_range(n);
    for (auto it = r.first; it != r.second; ++it)
      if (it->second == p) {
        d.free_sz.erase(it);
        break;
      }
    d.free_bytes -= n;
  }
  void insert_free(Dev& d, char* p, size_t n) {
    d.free_at[p] = n;
    d.free_sz.emplace(n, p);
    d.free_bytes += n;
  }
  void release_free_chunks(Dev& d, size_t keep) {
    if (d.borrowed) return;
    for (auto it = d.chunks.begin(); it != d.chunks.end() && d.free_bytes > keep;) {
      auto f = d.free_at.find(it->first);
      if (f != d.free_at.end() && f->second == it->second) {  // chunk entirely free
        erase_free(d, it->first, it->second);
        cudaFree(it->first);
        it = d.chunks.erase(it);
      } else {
        ++it;
      }
    }
  }
  cudaError_t alloc(void** out, size_t bytes) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const size_t n = (std::max<size_t>(bytes, 1) + kGrain - 1) / kGrain * kGrain;
    std::lock_guard<std::mutex> g(mu);
    const Key key{dev, t_arena};
    if (t_arena != 0 && devs.find(key) == devs.end()) {
      *out = nullptr;
      return cudaErrorInvalidValue;  // the arena lives on another device
    }
    Dev& d = devs[key];
    auto it = d.free_sz.lower_bound(n);
    if (it == d.free_sz.end() && d.borrowed) {
      *out = nullptr;
      return cudaErrorMemoryAllocation;  // arena exhausted
    }
    if (it == d.free_sz.end()) {
      // geometric growth (a new chunk at least as large as all chunks so far):
      // cudaMalloc of a few hundred MB costs 15-50 ms on B200, so a growing
      // workload (the paper's regrids) misses O(log) times, not once per size
      // (capped at 2 GiB; if that much is not free, just the request)
      size_t have = 0;
      for (const auto& ch : d.chunks) have += ch.second;
      size_t cs = std::max({n, kChunk, std::min(have, size_t{2} << 30)});
      void* c = nullptr;
      e = cudaMalloc(&c, cs);
      if (e == cudaErrorMemoryAllocation && cs > std::max(n, kChunk)) {
        cudaGetLastError();
        cs = std::max(n, kChunk);
        e = cudaMalloc(&c, cs);
      }
      if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        release_free_chunks(d, 0);
        e = cudaMalloc(&c, cs);
      }
      if (e != cudaSuccess) {
        *out = nullptr;
        return e;
      }
      d.chunks[static_cast<char*>(c)] = cs;
      insert_free(d, static_cast<char*>(c), cs);
      ++misses;
      it = d.free_sz.lower_bound(n);
    } else if (!d.borrowed) {
      ++hits;   // (hits / misses count the library's own chunks, not arenas)
    }
    char* p = it->second;
    const size_t fs = it->first;
    erase_free(d, p, fs);
    if (fs > n) insert_free(d, p + n, fs - n);
    live[p] = {key, n};
    *out = p;
    return cudaSuccess;
  }
  // adopt [base, base + bytes) of device `dev` as a new arena; returns its id
  int64_t add_arena(int dev, void* base, size_t bytes) {
    std::lock_guard<std::mutex> g(mu);
    char* b = static_cast<char*>(base);
    const size_t skip = (kGrain - reinterpret_cast<uintptr_t>(b) % kGrain) % kGrain;
    if (bytes <= skip + kGrain) return 0;
    b += skip;
    const size_t n = (bytes - skip) / kGrain * kGrain;
    const int64_t id = next_arena++;
    Dev& d = devs[Key{dev, id}];
    d.borrowed = true;
    d.chunks[b] = n;
    insert_free(d, b, n);
    return id;
  }
  // forget an arena (every buffer carved from it must have been released)
  void remove_arena(int64_t id) {
    std::lock_guard<std::mutex> g(mu);
    for (auto it = devs.begin(); it != devs.end();)
      it = (it->first.second == id) ? devs.erase(it) : std::next(it);
  }
  size_t arena_free(int64_t id) {
    std::lock_guard<std::mutex> g(mu);
    size_t f = 0;
    for (auto& kv : devs)
      if (kv.first.second == id) f += kv.second.free_bytes;
    return f;
  }
  void release(void* vp) {
    std::lock_guard<std::mutex> g(mu);
    auto lv = live.find(vp);
    if (lv == live.end()) return;
    Dev& d = devs[lv->second.first];
    char* p = static_cast<char*>(vp);
    size_t n = lv->second.second;
    live.erase(lv);
    // coalesce with the free neighbours inside the same chunk
    auto nx = d.free_at.find(p + n);
    if (nx != d.free_at.end() && !is_chunk_start(d, p + n)) {
      const size_t m = nx->second;
      erase_free(d, p + n, m);
      n += m;
    }
    auto pv = d.free_at.lower_bound(p);
    if (pv != d.free_at.begin() && !is_chunk_start(d, p)) {
      --pv;
      if (pv->first + pv->second == p) {
        char* q = pv->first;
        const size_t m = pv->second;
        erase_free(d, q, m);
        p = q;
        n += m;
      }
    }
    insert_free(d, p, n);
    if (d.free_bytes > limit) release_free_chunks(d, limit);
  }
  void trim_all() {
    std::lock_guard<std::mutex> g(mu);
    for (auto& kv : devs) release_free_chunks(kv.second, 0);
  }
  size_t cached() {
    size_t c = 0;
    for (auto& kv : devs)
      if (!kv.second.borrowed) c += kv.second.free_bytes;
    return c;
  }
};
Pool& pool() {
  static Pool* p = new Pool();  // never destroyed: no cudaFree after the driver is torn down
  return *p;
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      reset();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { reset(); }
  void reset() {
    if (p) pool().release(p);
    p = nullptr;
    n = 0;
  }
  cudaError_t alloc(size_t count) {
    reset();
    if (count == 0) return cudaSuccess;
    void* v = nullptr;
    cudaError_t e = pool().alloc(&v, count * sizeof(T));
    if (e == cudaSuccess) {
      p = static_cast<T*>(v);
      n = count;
    }
    return e;
  }
};

// Per-cell ghost source (host side of the planner).
struct Src {
  int kind;        // 0 local same-level interior, 1 frame (coarse / remote), -1 unset
  int64_t base;    // element offset (p component) in the level buffer / frame
  int64_t cs;      // component stride
};

struct Level {
  bool set = false;
  int npatch = 0;
  std::vector<claw_patch_desc> desc;
  std::vector<int64_t> i0, j0;
  int64_t nx = 0, ny = 0;
  int ratio = 0;  // to the coarser level
  double dx = 0, dy = 0;
  std::vector<int32_t> owner;
  std::vector<int32_t> local;       // global patch -> owned index or -1
  std::vector<int32_t> owned;       // owned index -> global patch
  std::vector<int64_t> off;         // owned index -> element offset
  int64_t buf_elems = 0;
  bool gapless = true;
  int64_t cells_owned = 0;
  // bucket grid
  int64_t nbx = 0, nby = 0;
  std::vector<int64_t> bstart;
  std::vector<int32_t> blist;
  // host tables
  std::vector<DevPatch> hpatch;
  std::vector<DevRect> hrect;
  int64_t ncellrect = 0;           // entries of the ghost-cell rectangle map (DevPatch::crect)
  std::vector<int4> htile;
  int lane_tiles = 0;         // generic tiles: 30-column strips for step_lane_kernel
  std::vector<DevInterp> hinterp;
  // debug: per owned patch, per padded cell, donor code
  std::vector<std::vector<int64_t>> dbg_src, dbg_remote;
  // halo plan (per peer)
  std::vector<std::vector<int64_t>> send_off, send_cs;
  std::vector<std::vector<int64_t>> send_dbg;  // patch<<32 | j<<16 | i
  std::vector<int64_t> nrecv, recv_frame_off;
  int64_t frame_elems = 0;
  int nslice = 1;                // frame slices (the R substeps of a fine level inside a coarse step)
  int fsel = 0;                  // slice the next step reads
  int64_t coarse_frame_off = 0, ncoarse = 0;
  // device
  DevBuf<double> q[2];
  int cur = 0;
  DevBuf<double> frame;
  DevBuf<DevPatch> dpatch;
  DevBuf<DevRect> drect;
  DevBuf<int32_t> dcellrect;
  DevBuf<int4> dtile;
  DevBuf<DevInterp> dinterp;
  DevBuf<unsigned long long> pcfl;  // per owned patch
  DevBuf<unsigned long long> lcfl;  // level slot
  std::vector<std::unique_ptr<DevBuf<int64_t>>> dsend_off, dsend_cs;
  // world > 1: this level is the partitioned one (claw_config.dist_level);
  // otherwise every rank holds all of it (replicated, or world = 1)
  bool dist = false;
  // update exchange of the partitioned level (dist, level > 1): the
  // level-(L-1) cells this rank averages (send) and those each peer
  // averages (recv), as (offset in the coarse level buffer, component stride)
  std::vector<int64_t> upd_send_off, upd_send_cs;
  std::vector<std::vector<int64_t>> upd_recv_off, upd_recv_cs;
  DevBuf<int64_t> dupd_send_off, dupd_send_cs;
  DevBuf<double> dupd_send_buf;
  std::vector<std::unique_ptr<DevBuf<int64_t>>> dupd_recv_off, dupd_recv_cs;
  std::vector<std::unique_ptr<DevBuf<double>>> dupd_recv_buf;
  std::vector<std::unique_ptr<DevBuf<double>>> dsend_buf;
  double t_old = 0, t_new = 0;
  bool stepped_once = false;
  int64_t device_bytes = 0;
  bool uniform = false;  // every patch shares (c, Z): step constants as kernel params
  bool grid = false;     // one uniform grid of equal patches: table-free grid kernel
  int th = 64;           // rows per tile for this level
  bool band = false;     // world > 1 band partition of a uniform grid (grid kernel per rank)
  int gnpx = 0, gnpy = 0;  // grid layout of the whole level
  int64_t Y0 = 0, Y1 = 0;  // this rank's band of level rows
  int64_t hoff[4] = {-1, -1, -1, -1};  // frame offset (column 0) of halo rows Y0-2, Y0-1, Y1, Y1+1; -1 local
  int64_t hcs[4] = {0, 0, 0, 0};       // their component strides
  // updating table (this fine level onto level-1): covered coarse cells and
  // their R*R children
  std::vector<claw::DevUpdate> hu;
  std::vector<claw::DevUpdateRect> hur;  // rectangles of coarse cells inside one fine patch
  DevBuf<claw::DevUpdateRect> dur;
  DevBuf<int32_t> dur_chunk;
  std::vector<int32_t> hur_chunk;        // work chunk -> rectangle (claw::kUpdChunk cells per chunk)
  std::vector<int64_t> hu_src, hu_scs;   // slow entries: R*R (offset, cs) each
  DevBuf<claw::DevUpdate> du;
  DevBuf<int64_t> du_src, du_scs;
  // conservation-fix registers of this fine level against level-1 (reflux on)
  std::vector<claw::DevReflux> hreg;
  std::vector<int32_t> hheads;           // first register of each coarse cell, + end
  DevBuf<claw::DevReflux> dreg;
  DevBuf<int32_t> dheads;
  DevBuf<double> racc;                   // [nreg][3]
  int gen = 0;           // level CFL slot generation (lcfl[gen] is the last step's)
  unsigned long long* hier = nullptr;  // coarse-step slot while claw_advance_hierarchy runs

  // variable media (claw_set_aux; grid mode, single rank): (Z, c) per cell in
  // q's patch layout, and per owned patch the max sound speed over its cells
  // and 1-deep ghost frame (the cells its faces touch) for claw_patch_cfl
  DevBuf<double> aux;
  DevBuf<double> aux_halo;            // band mode: (Z, c) of the four halo rows, [4][2][nx]
  bool vc = false;
  std::vector<double> vc_pcmax;
  double last_r = 0.0, last_s = 0.0;  // dt/dx, dt/dy of the last step

  int npx = 0;
  int64_t ngrid_tiles = 0;
  int64_t ngrid_blocks = 0;   // row blocks of the band (grid mode)
  int grid_th = 0;            // rows per grid tile (> my: tiles span patch rows)
  int grid_th_base = 0;       // single-rank makespan choice: the th it started from (0: not auto)
  int band_te = 0;            // band split (world > 1): rows of each edge tile (0: row blocks)
  int grid_th_int = 0;        // band split: rows per interior tile
  int64_t ngrid_blocks_int = 0;
  bool use_side = false;      // generic kernel: side records by a side_kernel ahead of the step
  bool sparse = false;        // grid kernel on a sparse lattice of equal patches
  std::vector<int32_t> hslots;  // lattice slot -> patch (>= 0) or -1-v (virtual slot v)
  int32_t nvirt = 0;
  std::vector<int4> hgtile;   // sparse lattice: (strip, row block) tiles
  DevBuf<int32_t> dslots;
  DevBuf<int4> dgtile;
  int64_t frame_cs = 0;       // component stride of the coarse frame cells (interp_kernel)
  DevBuf<double> side;
  int64_t ntile_interior = 0; // generic tiles [0, n) read no remote ghost cell
  bool halo_pending = false;  // NCCL halo in flight on the comm stream

  int find(int64_t I, int64_t J) const {
    if (I < 0 || J < 0 || I >= nx || J >= ny) return -1;
    const int64_t b = (J / kBucket) * nbx + (I / kBucket);
    for (int64_t k = bstart[b]; k < bstart[b + 1]; ++k) {
      const int p = blist[k];
      if (I >= i0[p] && I < i0[p] + desc[p].mx && J >= j0[p] && J < j0[p] + desc[p].my) return p;
    }
    return -1;
  }
};

// One captured coarse step of claw_advance_hierarchy (the
// per-step launch sequence replayed as a CUDA graph).  Valid for the key it
// was captured under: context epoch, dt, flags, profiling, and every level's
// ping-pong buffer / CFL-slot parity.
struct HierGraph {
  std::vector<uint64_t> key;
  cudaGraphExec_t exec = nullptr;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_step, ev_ghost;  // timing nodes (profiling)
};
constexpr int kMaxAlpha = 4096;  // interpolation launches per coarse step

}  // namespace

struct claw_ctx {
  claw_config cfg{};
  bool host_only = false;
  bool dead = false;       // sticky CUDA / NCCL failure
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ncclComm_t comm = nullptr;
  Level lev[kMaxLevel + 1];
  Level stash[kMaxLevel + 1];  // levels discarded by a regrid: copy sources for the
                               // regrid that re-creates them (R18), until time moves
  bool stashed = false;
  double* h_cfl = nullptr;  // pinned 8 bytes
  std::string err;
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_step, ev_ghost, ev_pool;
  claw_stats stats{};
  int tile_rows = 64;
  int nsm = 148;            // SM count of the device (queried at create; B200: 148)
  unsigned long long* hier_slot = nullptr;  // set while claw_advance_hierarchy runs
  cudaStream_t comm_stream = nullptr;       // world > 1: halo pack + NCCL send/recv
  cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
  cudaEvent_t ev_int = nullptr, ev_edge = nullptr;   // split step: q^n ready for, and end of, the edge launch
  DevBuf<unsigned long long> hier_buf;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_free;  // event pool
  uint8_t* h_stage = nullptr;  // pinned staging for flag maps (regrid)
  size_t h_stage_bytes = 0;
  // CUDA graphs of the hierarchy's coarse step
  std::vector<HierGraph> graphs;
  uint64_t epoch = 0;          // bumped whenever levels are (re)defined
  bool graphs_on = false;      // CLAW_GRAPH=1 enables
  bool in_hier = false;        // inside claw_advance_hierarchy (alpha through d_alpha)
  bool dry = false;            // host bookkeeping only: the graph launches the work
  bool capturing = false;
  int alpha_n = 0;
  double* h_alpha = nullptr;   // pinned [kMaxAlpha], copied to d_alpha by the graph
  DevBuf<double> d_alpha;
  DevBuf<unsigned long long> hier_many;  // claw_advance_hierarchy_n: one CFL slot per coarse step
  double* h_many = nullptr;    // pinned copy
  int h_many_n = 0;
  int64_t arena_id = 0;        // claw_config.arena adopted by the pool (0: library chunks)
  DevBuf<int32_t> nf_flag;     // claw_config.check_finite: non-finite flag of the last step
  int32_t* h_nf = nullptr;     // pinned copy
  int nf_level = 0;            // level whose step set it
};

namespace {

int fail(claw_ctx* c, int code, const char* fmt, ...) {
  if (c) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    c->err = buf;
  }
  return code;
}

int cuda_fail(claw_ctx* c, cudaError_t e, const char* where) {
  if (e == cudaErrorMemoryAllocation) {  // pool / arena exhausted: not sticky
    cudaGetLastError();
    return fail(c, CLAW_ENOMEM, "%s: out of device memory%s", where, c->arena_id ? " (arena full)" : "");
  }
  c->dead = true;
  return fail(c, CLAW_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define CUDA_TRY(expr)                                 \
  do {                                                 \
    cudaError_t e_ = (expr);                           \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #expr); \
  } while (0)

// NVTX range over one API call / phase (tracing): named ranges for
// ghost fill, level step, halo exchange, CFL all-reduce, updating, regrid and
// the hierarchy drivers, visible in nsys / ncu timelines
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  Nvtx(const char* fmt, int a) {
    char b[64];
    std::snprintf(b, sizeof b, fmt, a);
    nvtxRangePushA(b);
  }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

int nccl_fail(claw_ctx* c, ncclResult_t r, const char* where) {
  c->dead = true;
  return fail(c, CLAW_ENCCL, "%s: %s", where,
              g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "nccl error");
}

int64_t map_axis(int64_t I, int64_t n, int bc_lo, int bc_hi) {
  if (I < 0) return (bc_lo == CLAW_BC_PERIODIC) ? ((I % n) + n) % n : 0;
  if (I >= n) return (bc_hi == CLAW_BC_PERIODIC) ? I % n : n - 1;
  return I;
}

uint64_t morton(uint32_t x, uint32_t y) {
  auto spread = [](uint64_t v) {
    v &= 0xffffffffull;
    v = (v | (v << 16)) & 0x0000ffff0000ffffull;
    v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
    v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
    v = (v | (v << 2)) & 0x3333333333333333ull;
    v = (v | (v << 1)) & 0x5555555555555555ull;
    return v;
  };
  return spread(x) | (spread(y) << 1);
}

// A uniform grid of equal patches in row-major order filling a rectangle of
// the index space (relative to the minimum corner): returns npx, npy.
bool grid_layout(int npatch, const claw_patch_desc* d, const std::vector<int64_t>& i0,
                 const std::vector<int64_t>& j0, int* npx_out, int* npy_out) {
  const int mx = d[0].mx, my = d[0].my;
  int64_t imin = i0[0], jmin = j0[0], imax = i0[0], jmax = j0[0];
  for (int p = 1; p < npatch; ++p) {
    imin = std::min(imin, i0[p]);
    jmin = std::min(jmin, j0[p]);
    imax = std::max(imax, i0[p]);
    jmax = std::max(jmax, j0[p]);
  }
  const int64_t npx = (imax - imin) / mx + 1, npy = (jmax - jmin) / my + 1;
  if (npx * npy != npatch) return false;
  for (int p = 0; p < npatch; ++p)
    if (d[p].mx != mx || d[p].my != my || i0[p] - imin != (p % npx) * mx || j0[p] - jmin != (p / npx) * my)
      return false;
  *npx_out = static_cast<int>(npx);
  *npy_out = static_cast<int>(npy);
  return true;
}

// Owner map.  A uniform grid with at least `world` patch rows is cut into
// horizontal bands of whole patch rows (rank r: rows [r npy / world, (r+1) npy
// / world)), so every rank advances a rectangle with the table-free grid
// kernel and exchanges only full halo rows.  Anything else: patches in Morton
// order of their lower-left index, split contiguously by cell count.
void partition_impl(int npatch, const claw_patch_desc* d, const std::vector<int64_t>& i0,
                    const std::vector<int64_t>& j0, int world, int32_t* owner) {
  if (world <= 1) {
    for (int p = 0; p < npatch; ++p) owner[p] = 0;
    return;
  }
  int npx, npy;
  if (grid_layout(npatch, d, i0, j0, &npx, &npy) && npy >= world &&
      static_cast<int64_t>(d[0].my) * (npy / world) >= 4) {
    for (int p = 0; p < npatch; ++p) {
      const int64_t pr = p / npx;
      // band cut r: rows [floor(r npy / world), floor((r+1) npy / world))
      int r = static_cast<int>((pr * world) / npy);
      while (r + 1 < world && (static_cast<int64_t>(r + 1) * npy) / world <= pr) ++r;
      while (r > 0 && (static_cast<int64_t>(r) * npy) / world > pr) --r;
      owner[p] = r;
    }
    return;
  }
  std::vector<int> order(npatch);
  for (int p = 0; p < npatch; ++p) order[p] = p;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return morton(static_cast<uint32_t>(i0[a]), static_cast<uint32_t>(j0[a])) <
           morton(static_cast<uint32_t>(i0[b]), static_cast<uint32_t>(j0[b]));
  });
  int64_t total = 0;
  for (int p = 0; p < npatch; ++p) total += static_cast<int64_t>(d[p].mx) * d[p].my;
  // greedy contiguous split: rank r takes patches until its running total
  // reaches the (r+1)/world quantile (closest boundary)
  int r = 0;
  int64_t acc = 0;
  for (int k = 0; k < npatch; ++k) {
    const int p = order[k];
    const int64_t w = static_cast<int64_t>(d[p].mx) * d[p].my;
    const double target = static_cast<double>(total) * (r + 1) / world;
    if (r < world - 1 && acc > 0 &&
        std::fabs(static_cast<double>(acc + w) - target) > std::fabs(static_cast<double>(acc) - target))
      ++r;
    owner[p] = r;
    acc += w;
  }
}

int validate_config(claw_ctx* c, const claw_config* cfg) {
  if (!(cfg->xhi > cfg->xlo) || !(cfg->yhi > cfg->ylo)) return fail(c, CLAW_EINVAL, "domain: xhi>xlo, yhi>ylo required");
  for (int k = 0; k < 4; ++k)
    if (cfg->bc[k] != CLAW_BC_EXTRAP && cfg->bc[k] != CLAW_BC_PERIODIC)
      return fail(c, CLAW_EINVAL, "bc[%d]=%d: must be 1 (extrapolation) or 2 (periodic)", k, cfg->bc[k]);
  if ((cfg->bc[0] == CLAW_BC_PERIODIC) != (cfg->bc[1] == CLAW_BC_PERIODIC) ||
      (cfg->bc[2] == CLAW_BC_PERIODIC) != (cfg->bc[3] == CLAW_BC_PERIODIC))
    return fail(c, CLAW_EINVAL, "bc: periodic boundaries must come in pairs");
  if (cfg->limiter < 0 || cfg->limiter > 4) return fail(c, CLAW_EINVAL, "limiter=%d: must be 0..4", cfg->limiter);
  if (cfg->order_trans < 0 || cfg->order_trans > 2)
    return fail(c, CLAW_EINVAL, "order_trans=%d: must be 0..2", cfg->order_trans);
  if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world)
    return fail(c, CLAW_EINVAL, "rank=%d world=%d", cfg->rank, cfg->world);
  if (cfg->exchange != 0 && cfg->exchange != 1) return fail(c, CLAW_EINVAL, "exchange=%d: must be 0 or 1", cfg->exchange);
  if (cfg->world > 1 && cfg->exchange == 0 && !cfg->nccl_unique_id && cfg->device >= 0)
    return fail(c, CLAW_EINVAL, "world>1 needs nccl_unique_id");
  if (cfg->reflux != 0 && cfg->reflux != 1) return fail(c, CLAW_EINVAL, "reflux=%d: must be 0 or 1", cfg->reflux);
  if (cfg->dist_level < 0 || cfg->dist_level == 1 || cfg->dist_level > kMaxLevel)
    return fail(c, CLAW_EINVAL, "dist_level=%d: 0 (level 1) or 2..%d", cfg->dist_level, kMaxLevel);
  if (cfg->reflux && cfg->world > 1)
    return fail(c, CLAW_EINVAL, "reflux: the conservation fix is single-rank in this version (world=%d)", cfg->world);
  if (cfg->tile_rows < 0 || cfg->tile_rows > claw::max_tile_rows())
    return fail(c, CLAW_EINVAL, "tile_rows=%d: must be 0..%d", cfg->tile_rows, claw::max_tile_rows());
  if (cfg->check_finite != 0 && cfg->check_finite != 1)
    return fail(c, CLAW_EINVAL, "check_finite=%d: must be 0 or 1", cfg->check_finite);
  if (cfg->arena && (cfg->device < 0 || cfg->arena_bytes == 0))
    return fail(c, CLAW_EINVAL, "arena needs a device context and arena_bytes > 0");
  return CLAW_OK;
}

// Validate descriptors and integer boxes of a level (S:51-style messages).
int build_geometry(claw_ctx* c, int level, int npatch, const claw_patch_desc* d, Level& L) {
  const claw_config& cfg = c->cfg;
  L.npatch = npatch;
  L.desc.assign(d, d + npatch);
  L.dx = d[0].dx;
  L.dy = d[0].dy;
  if (!(L.dx > 0) || !(L.dy > 0)) return fail(c, CLAW_EINVAL, "patch 0: dx, dy must be > 0");
  L.nx = std::llround((cfg.xhi - cfg.xlo) / L.dx);
  L.ny = std::llround((cfg.yhi - cfg.ylo) / L.dy);
  if (std::fabs((cfg.xhi - cfg.xlo) / L.dx - L.nx) > 1e-6 || std::fabs((cfg.yhi - cfg.ylo) / L.dy - L.ny) > 1e-6)
    return fail(c, CLAW_EINVAL, "level %d: dx/dy do not divide the domain", level);
  if (level > 1) {
    const Level& C = c->lev[level - 1];
    const double rx = C.dx / L.dx, ry = C.dy / L.dy;
    L.ratio = static_cast<int>(std::llround(rx));
    if (L.ratio < 1 || std::fabs(rx - L.ratio) > 1e-9 || std::fabs(ry - L.ratio) > 1e-9)
      return fail(c, CLAW_EINVAL, "level %d: refinement ratio must be an integer, equal in x and y", level);
  }
  L.i0.resize(npatch);
  L.j0.resize(npatch);
  int64_t cells = 0;
  for (int p = 0; p < npatch; ++p) {
    const claw_patch_desc& q = d[p];
    if (q.mx < 1 || q.my < 1) return fail(c, CLAW_EINVAL, "patch %d: mx=%d my=%d must be >= 1", p, q.mx, q.my);
    if (q.mx > 65535 || q.my > 65535) return fail(c, CLAW_EINVAL, "patch %d: mx, my must be < 65536", p);
    if (q.mbc != 2) return fail(c, CLAW_EINVAL, "patch %d: mbc=%d must be 2", p, q.mbc);
    if (!(q.rho > 0) || !(q.K > 0)) return fail(c, CLAW_EINVAL, "patch %d: rho and K must be > 0", p);
    if (q.dx != L.dx || q.dy != L.dy) return fail(c, CLAW_EINVAL, "patch %d: dx/dy differ within level %d", p, level);
    const double fi = (q.xlower - cfg.xlo) / L.dx, fj = (q.ylower - cfg.ylo) / L.dy;
    L.i0[p] = std::llround(fi);
    L.j0[p] = std::llround(fj);
    if (std::fabs(fi - L.i0[p]) > 1e-6 || std::fabs(fj - L.j0[p]) > 1e-6)
      return fail(c, CLAW_EINVAL, "patch %d: xlower/ylower not on the level grid", p);
    if (L.i0[p] < 0 || L.j0[p] < 0 || L.i0[p] + q.mx > L.nx || L.j0[p] + q.my > L.ny)
      return fail(c, CLAW_EINVAL, "patch %d: outside the domain", p);
    cells += static_cast<int64_t>(q.mx) * q.my;
  }
  // bucket grid
  L.nbx = (L.nx + kBucket - 1) / kBucket;
  L.nby = (L.ny + kBucket - 1) / kBucket;
  const int64_t nb = L.nbx * L.nby;
  L.bstart.assign(nb + 1, 0);
  for (int pass = 0; pass < 2; ++pass) {
    std::vector<int64_t> fill;
    if (pass == 1) {
      for (int64_t b = 0; b < nb; ++b) L.bstart[b + 1] += L.bstart[b];
      L.blist.assign(L.bstart[nb], 0);
      fill.assign(L.bstart.begin(), L.bstart.end() - 1);
    }
    for (int p = 0; p < npatch; ++p) {
      const int64_t bx0 = L.i0[p] / kBucket, bx1 = (L.i0[p] + d[p].mx - 1) / kBucket;
      const int64_t by0 = L.j0[p] / kBucket, by1 = (L.j0[p] + d[p].my - 1) / kBucket;
      for (int64_t by = by0; by <= by1; ++by)
        for (int64_t bx = bx0; bx <= bx1; ++bx) {
          const int64_t b = by * L.nbx + bx;
          if (pass == 0) L.bstart[b + 1]++;
          else L.blist[fill[b]++] = p;
        }
    }
  }
  for (int64_t b = 0; b < nb; ++b)
    for (int64_t k = L.bstart[b]; k < L.bstart[b + 1]; ++k)
      for (int64_t k2 = k + 1; k2 < L.bstart[b + 1]; ++k2) {
        const int p = L.blist[k], q = L.blist[k2];
        if (L.i0[p] < L.i0[q] + d[q].mx && L.i0[q] < L.i0[p] + d[p].mx && L.j0[p] < L.j0[q] + d[q].my &&
            L.j0[q] < L.j0[p] + d[p].my)
          return fail(c, CLAW_EINVAL, "patches %d and %d overlap on level %d", p, q, level);
      }
  if (level == 1 && cells != L.nx * L.ny) return fail(c, CLAW_EINVAL, "level 1 does not tile the domain");
  return CLAW_OK;
}

// Index of ghost cell (i, j) of an mx x my patch in its frame ring of
// 4(mx+my)+16 cells: the two rows below, the two rows above (full padded
// width), then 4 cells per interior row.
inline int64_t frame_index(int i, int j, int mx, int my) {
  const int64_t PX = mx + 4;
  if (j < 0) return (j + 2) * PX + (i + 2);
  if (j >= my) return 2 * PX + (j - my) * PX + (i + 2);
  return 4 * PX + 4ll * j + (i < 0 ? i + 2 : 2 + (i - mx));
}
inline int64_t frame_size(int mx, int my) { return 4ll * (mx + my) + 16; }

// Compress per-cell sources of a patch's ghost frame (frame_index order)
// into rectangles.
void compress_rects(const std::vector<Src>& cell, int mx, int my, std::vector<DevRect>& out) {
  auto at = [&](int i, int j) -> const Src& { return cell[frame_index(i, j, mx, my)]; };
  struct Run {
    int i0, i1, j0, j1;  // [i0, i1) x [j0, j1)
    int kind;
    int64_t base, sx, sy, cs;
    bool open;
  };
  std::vector<Run> runs;
  std::vector<Run> prev;  // runs of the previous row that can still grow
  std::vector<Run> row, next;
  for (int j = -2; j <= my + 1; ++j) {
    row.clear();
    auto emit_segment = [&](int a, int b) {  // ghost cells [a, b) of row j
      int i = a;
      while (i < b) {
        const Src& s = at(i, j);
        Run r{i, i + 1, j, j + 1, s.kind, s.base, 0, 0, s.cs, true};
        int k = i + 1;
        if (k < b) {
          const Src& t = at(k, j);
          if (t.kind == s.kind && t.cs == s.cs) {
            r.sx = t.base - s.base;
            while (k < b) {
              const Src& u = at(k, j);
              if (u.kind != s.kind || u.cs != s.cs || u.base != s.base + (k - i) * r.sx) break;
              ++k;
            }
          }
        }
        r.i1 = k;
        row.push_back(r);
        i = k;
      }
    };
    if (j < 0 || j >= my) {
      emit_segment(-2, mx + 2);
    } else {
      emit_segment(-2, 0);
      emit_segment(mx, mx + 2);
    }
    // vertical merge with runs ending at row j
    next.clear();
    for (Run& r : row) {
      bool merged = false;
      for (Run& p : prev) {
        if (!p.open || p.i0 != r.i0 || p.i1 != r.i1 || p.kind != r.kind || p.cs != r.cs) continue;
        if (p.i1 - p.i0 > 1 && p.sx != r.sx) continue;
        const int64_t step = r.base - (p.base + (int64_t)(p.j1 - 1 - p.j0) * p.sy);
        if (p.j1 - p.j0 > 1 && step != p.sy) continue;
        // compatible: also need x steps equal when width 1 is ambiguous (both 0)
        if (p.j1 - p.j0 == 1) p.sy = step;
        p.j1 = j + 1;
        next.push_back(p);
        p.open = false;
        merged = true;
        break;
      }
      if (!merged) next.push_back(r);
    }
    for (Run& p : prev)
      if (p.open) runs.push_back(p);
    prev.swap(next);
    for (Run& p : prev) p.open = true;
  }
  for (Run& p : prev) runs.push_back(p);
  for (const Run& r : runs) {
    DevRect d{};
    d.i0 = r.i0;
    d.j0 = r.j0;
    d.w = r.i1 - r.i0;
    d.h = r.j1 - r.j0;
    d.kind = r.kind;
    d.base = r.base;
    d.sx = r.sx;
    d.sy = r.sy;
    d.cs = r.cs;
    out.push_back(d);
  }
}

// The composite ghost rule (R1, R8-R10) for every padded
// cell of every owned patch, the halo plan, coarse-interpolation specs, and
// device tables.
// Phase timer for CLAW_TRACE_PLAN=1 (stderr), host wall clock.
struct PhaseTrace {
  bool on;
  const char* tag;
  int level;
  std::chrono::steady_clock::time_point t;
  PhaseTrace(const char* tg, int lv)
      : on(std::getenv("CLAW_TRACE_PLAN") != nullptr), tag(tg), level(lv), t(std::chrono::steady_clock::now()) {}
  void operator()(const char* what) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[%s L%d] %-10s %8.2f ms\n", tag, level, what,
                 std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

// Persistent host workers for parallel_for: a regrid runs ~10 parallel loops
// of the planner and clusterer, and creating and joining 16 std::threads per
// loop cost milliseconds.  The caller takes part as thread 0; thread t runs
// indices t, t + nthr, ...; jobs are serialised; a loop body that itself calls
// parallel_for runs that loop serially.
class HostPool {
 public:
  static HostPool& get() {
    // never destroyed (workers detached at exit); a forked child has none of
    // the parent's workers, so it starts its own pool
    static HostPool* p = nullptr;
    static pid_t owner = 0;
    static std::mutex mk;
    std::lock_guard<std::mutex> g(mk);
    if (!p || owner != getpid()) {
      p = new HostPool();
      owner = getpid();
    }
    return *p;
  }
  static bool& in_worker() {
    thread_local bool w = false;
    return w;
  }
  void run(int nthr, int n, const std::function<void(int)>& f) {
    std::lock_guard<std::mutex> one(run_mu_);
    nthr = std::min(nthr, 1 + static_cast<int>(workers_.size()));
    {
      std::lock_guard<std::mutex> g(mu_);
      job_ = &f;
      n_ = n;
      nthr_ = nthr;
      pending_ = nthr - 1;
      ++gen_;
    }
    cv_.notify_all();
    in_worker() = true;
    for (int k = 0; k < n; k += nthr) f(k);
    in_worker() = false;
    std::unique_lock<std::mutex> g(mu_);
    done_.wait(g, [&] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  HostPool() {
    const int nw = std::max(0, std::min(31, static_cast<int>(std::thread::hardware_concurrency()) - 1));
    for (int t = 1; t <= nw; ++t) workers_.emplace_back([this, t] { loop(t); });
    for (auto& w : workers_) w.detach();
  }
  void loop(int t) {
    in_worker() = true;
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* f;
      int n, nthr;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return gen_ != seen; });
        seen = gen_;
        f = job_;
        n = n_;
        nthr = nthr_;
      }
      if (t >= nthr) continue;
      for (int k = t; k < n; k += nthr) (*f)(k);
      std::lock_guard<std::mutex> g(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex run_mu_, mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int n_ = 0, nthr_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
};

// Host threads for the planner's per-patch loops (results are assembled in
// patch order, so they do not depend on the thread count).
int host_threads(int nwork) {
  static const int hw = [] {
    const char* e = std::getenv("CLAW_HOST_THREADS");
    const int n = e ? std::atoi(e) : static_cast<int>(std::thread::hardware_concurrency());
    return std::max(1, std::min(n, 32));
  }();
  return std::max(1, std::min(hw, nwork / 64));
}

template <class F>
void parallel_for(int nthr, int n, F&& f) {
  if (nthr <= 1 || HostPool::in_worker()) {
    for (int k = 0; k < n; ++k) f(k);
    return;
  }
  const std::function<void(int)> fn = [&](int k) { f(k); };
  HostPool::get().run(nthr, n, fn);
}

// grid tiles spanning whole patch rows: w rows, a multiple of the patch
// height my (the row pointers step across patch-row boundaries)
bool span_rows_ok(int w, int my) { return w > my && w % my == 0 && my % 4 == 0 && my >= 8 && w <= 512; }

// Tile height of a large single-rank grid level by the makespan of the
// launch: ceil(tiles / slots) waves of (th + 4) row steps each (the 4 halo
// rows are the per-tile prologue); slots = resident warps of the kernel
// that runs the level.  Ties go to the taller tile; a sub-wave candidate is
// skipped (latency-bound levels keep th0).
// (grid-kernel heights capped at kSpanAutoMax rows: re-swept on the final
// kernel, C5 measured 129.5 G at 192-row tiles against 126.4 G at the 384
// the uncapped rule picked, C4 unchanged at 192; the vc kernel and the van
// Leer limiter keep the uncapped rule -- 384-row tiles on c5vc, 2% faster
// than 192 -- profiles/r02_grid_tile_rows_final.txt)
#ifndef CLAW_SPAN_AUTO_MAX
#define CLAW_SPAN_AUTO_MAX 192
#endif
constexpr int kSpanAutoMax = CLAW_SPAN_AUTO_MAX;
int makespan_th(int64_t nstrip, int64_t rows, int my, int64_t slots, int th0, int cap = kSpanAutoMax) {
  int th = th0;
  double best = -1.0;
  for (int w = my; w <= cap; w += my) {
    if (!(w == my || span_rows_ok(w, my))) continue;
    const int64_t tiles = nstrip * ((rows + w - 1) / w);
    if (tiles < slots) continue;
    const double cost = static_cast<double>((tiles + slots - 1) / slots) * (w + 4);
    if (best < 0 || cost <= best) {
      best = cost;
      th = w;
    }
  }
  return th;
}

// Interior tile height of a band-split level: any
// multiple of 4 from 16 to 256 rows, by the same makespan rule.
int band_int_th(int64_t nstrip, int64_t rows, int my, int64_t slots) {
  int thi = my;
  double best = -1.0;
  for (int w = 16; w <= 256; w += 4) {
    const int64_t tiles = nstrip * ((rows + w - 1) / w);
    if (tiles < slots && w > my) continue;
    const double cost = static_cast<double>((tiles + slots - 1) / slots) * (w + 4);
    if (best < 0 || cost <= best) {
      best = cost;
      thi = w;
    }
  }
  return thi;
}

int plan_level(claw_ctx* c, int level, Level& L) {
  static const bool trace = std::getenv("CLAW_TRACE_PLAN") != nullptr;
  auto tnow = [] { return std::chrono::steady_clock::now(); };
  auto t_last = tnow();
  auto lap = [&](const char* what) {
    if (!trace) return;
    const auto t = tnow();
    std::fprintf(stderr, "[plan L%d] %-10s %8.2f ms\n", level,
                 what, std::chrono::duration<double, std::milli>(t - t_last).count());
    t_last = t;
  };
  const claw_config& cfg = c->cfg;
  // the partitioned level (world > 1): level 1, or claw_config.dist_level;
  // any other level is replicated -- every rank owns every patch and plans
  // it as a one-rank level
  L.dist = cfg.world > 1 && level == (cfg.dist_level >= 2 ? cfg.dist_level : 1);
  const int me = cfg.rank, world = L.dist ? cfg.world : 1;
  const int np = L.npatch;
  if (L.dist) {
    // (indices relative to the level's minimum corner, as claw_partition
    // computes them from the descriptors alone: the Morton order is not
    // shift-invariant, and callers slice their data with claw_partition)
    L.owner.assign(np, 0);
    const int64_t mi = np ? *std::min_element(L.i0.begin(), L.i0.end()) : 0;
    const int64_t mj = np ? *std::min_element(L.j0.begin(), L.j0.end()) : 0;
    std::vector<int64_t> ri(L.i0), rj(L.j0);
    for (auto& v : ri) v -= mi;
    for (auto& v : rj) v -= mj;
    partition_impl(np, L.desc.data(), ri, rj, world, L.owner.data());
  } else {
    L.owner.assign(np, me);
  }
  L.local.assign(np, -1);
  L.owned.clear();
  L.off.clear();
  int64_t off = 0;
  L.gapless = true;
  L.cells_owned = 0;
  for (int p = 0; p < np; ++p) {
    if (L.owner[p] != me) continue;
    L.local[p] = static_cast<int32_t>(L.owned.size());
    L.owned.push_back(p);
    const int64_t n = 3ll * L.desc[p].mx * L.desc[p].my;
    const int64_t aligned = (off + 31) / 32 * 32;  // 256-byte aligned patch start
    if (aligned != off) L.gapless = false;
    off = aligned;
    L.off.push_back(off);
    off += n;
    L.cells_owned += n / 3;
  }
  L.buf_elems = off;

  const Level* C = (level > 1) ? &c->lev[level - 1] : nullptr;

  L.send_off.assign(world, {});
  L.send_cs.assign(world, {});
  L.send_dbg.assign(world, {});
  L.nrecv.assign(world, 0);
  L.recv_frame_off.assign(world, 0);

  // ---- band mode: a uniform grid over the whole domain cut into bands of
  // patch rows by partition_impl; halo = two full rows below and above
  L.band = false;
  if (world > 1 && grid_layout(np, L.desc.data(), L.i0, L.j0, &L.gnpx, &L.gnpy)) {
    const int mx = L.desc[0].mx, my = L.desc[0].my;
    const bool whole = L.gnpx * static_cast<int64_t>(mx) == L.nx && L.gnpy * static_cast<int64_t>(my) == L.ny;
    if (whole && L.gnpy >= world && static_cast<int64_t>(my) * (L.gnpy / world) >= 4 && !L.owned.empty()) {
      L.band = true;
      const int npx = L.gnpx;
      auto band_of = [&](int r, int64_t& y0, int64_t& y1) {
        y0 = (static_cast<int64_t>(r) * L.gnpy / world) * my;
        y1 = (static_cast<int64_t>(r + 1) * L.gnpy / world) * my;
      };
      auto row_owner = [&](int64_t J) { return L.owner[static_cast<size_t>((J / my) * npx)]; };
      auto halo_rows = [&](int r, int64_t* J) {
        int64_t y0, y1;
        band_of(r, y0, y1);
        const int64_t raw[4] = {y0 - 2, y0 - 1, y1, y1 + 1};
        for (int k = 0; k < 4; ++k) J[k] = map_axis(raw[k], L.ny, cfg.bc[2], cfg.bc[3]);
      };
      band_of(me, L.Y0, L.Y1);
      if (L.owned.front() != static_cast<int>((L.Y0 / my) * npx)) return fail(c, CLAW_EINVAL, "band mismatch");
      int64_t Jme[4];
      halo_rows(me, Jme);
      int64_t fo = 0;
      for (int srank = 0; srank < world; ++srank) {
        if (srank == me) continue;
        int cnt = 0;
        for (int k = 0; k < 4; ++k)
          if (row_owner(Jme[k]) == srank && !(Jme[k] >= L.Y0 && Jme[k] < L.Y1)) ++cnt;
        if (!cnt) continue;
        L.recv_frame_off[srank] = fo;
        L.nrecv[srank] = static_cast<int64_t>(cnt) * L.nx;
        int idx = 0;
        for (int k = 0; k < 4; ++k)
          if (row_owner(Jme[k]) == srank && !(Jme[k] >= L.Y0 && Jme[k] < L.Y1)) {
            L.hoff[k] = fo + static_cast<int64_t>(idx++) * L.nx;
            L.hcs[k] = L.nrecv[srank];
          }
        fo += 3 * L.nrecv[srank];
      }
      L.coarse_frame_off = fo;
      L.ncoarse = 0;
      L.frame_elems = fo;
      // send lists: for every other rank, its halo rows that I own, in its k order
      for (int r = 0; r < world; ++r) {
        if (r == me) continue;
        int64_t Jr[4], y0r, y1r;
        halo_rows(r, Jr);
        band_of(r, y0r, y1r);
        for (int k = 0; k < 4; ++k) {
          if (row_owner(Jr[k]) != me || (Jr[k] >= y0r && Jr[k] < y1r)) continue;
          const int64_t prow = Jr[k] / my, lj = Jr[k] % my;
          for (int64_t Cc = 0; Cc < L.nx; ++Cc) {
            const int gp = static_cast<int>(prow * npx + Cc / mx);
            const int lq = L.local[gp];
            const int64_t li = Cc % mx;
            L.send_off[r].push_back(L.off[lq] + lj * mx + li);
            L.send_cs[r].push_back(static_cast<int64_t>(mx) * my);
            L.send_dbg[r].push_back((static_cast<int64_t>(gp) << 32) | (lj << 16) | li);
          }
        }
      }
    }
  }

  // which patches need resolving: owned ones (receive side) and, for world>1,
  // patches of other ranks whose ghost frame may read my cells (send side)
  std::vector<char> need(np, 0);
  int64_t bx0 = INT64_MAX, by0 = INT64_MAX, bx1 = INT64_MIN, by1 = INT64_MIN;
  for (int p : L.owned) {
    need[p] = 1;
    bx0 = std::min(bx0, L.i0[p]);
    by0 = std::min(by0, L.j0[p]);
    bx1 = std::max(bx1, L.i0[p] + L.desc[p].mx);
    by1 = std::max(by1, L.j0[p] + L.desc[p].my);
  }
  const bool periodic = cfg.bc[0] == CLAW_BC_PERIODIC || cfg.bc[2] == CLAW_BC_PERIODIC;
  if (world > 1 && !L.band)
    for (int p = 0; p < np; ++p) {
      if (need[p]) continue;
      const int64_t a0 = L.i0[p] - 2, a1 = L.i0[p] + L.desc[p].mx + 2;
      const int64_t b0 = L.j0[p] - 2, b1 = L.j0[p] + L.desc[p].my + 2;
      bool touch = a0 < bx1 && bx0 < a1 && b0 < by1 && by0 < b1;
      if (periodic && (a0 < 0 || b0 < 0 || a1 > L.nx || b1 > L.ny)) touch = true;
      need[p] = touch;
    }

  // (L.hinterp keeps its previous contents here: the one-rank path below
  // overwrites every entry it keeps, so a regrid does not zero-fill tens of
  // MB of interpolation specs first)
  L.dbg_src.assign(L.owned.size(), {});
  L.dbg_remote.assign(L.owned.size(), {});

  struct Pending {  // frame cells of owned patches before slot assignment
    int lp;         // owned index
    int cellidx;
    int kind;       // 1 remote, 2 coarse
    int src_rank;
    int64_t Ic, Jc, I, J;  // coarse spec inputs (kind 2)
  };
  std::vector<std::vector<Src>> cells(L.owned.size());

  auto ghost_patch = [&](int p, std::vector<Pending>& pend, std::string& emsg) -> int {
    const int dst_owner = L.owner[p];
    const bool mine = dst_owner == me;
    const int mx = L.desc[p].mx, my = L.desc[p].my, PX = mx + 4;
    const int lp = mine ? L.local[p] : -1;
    if (mine) {
      const size_t nf = static_cast<size_t>(frame_size(mx, my));
      cells[lp].assign(nf, Src{-1, 0, 0});
      L.dbg_src[lp].assign(nf, 0);
      L.dbg_remote[lp].assign(nf, 0);
    }
    (void)PX;
    int qlast = -1;
    for (int j = -2; j <= my + 1; ++j)
      for (int i = -2; i <= mx + 1; ++i) {
        if (i >= 0 && i < mx && j >= 0 && j < my) {  // interior: the kernels address it directly
          i = mx - 1;
          continue;
        }
        const int idx = static_cast<int>(frame_index(i, j, mx, my));
        const int64_t I = map_axis(L.i0[p] + i, L.nx, cfg.bc[0], cfg.bc[1]);
        const int64_t J = map_axis(L.j0[p] + j, L.ny, cfg.bc[2], cfg.bc[3]);
        // neighbouring ghost cells usually share their donor patch
        if (!(qlast >= 0 && I >= L.i0[qlast] && I < L.i0[qlast] + L.desc[qlast].mx && J >= L.j0[qlast] &&
              J < L.j0[qlast] + L.desc[qlast].my))
          qlast = L.find(I, J);
        const int q = qlast;
        if (q >= 0) {
          const int li = static_cast<int>(I - L.i0[q]), lj = static_cast<int>(J - L.j0[q]);
          const int src_owner = L.owner[q];
          const int64_t code = (static_cast<int64_t>(q) << 32) | (static_cast<int64_t>(lj) << 16) | li;
          if (mine) {
            if (src_owner == me) {
              const int lq = L.local[q];
              cells[lp][idx] = Src{0, L.off[lq] + static_cast<int64_t>(lj) * L.desc[q].mx + li,
                                   static_cast<int64_t>(L.desc[q].mx) * L.desc[q].my};
              L.dbg_src[lp][idx] = code;
            } else {
              if (L.band) {  // full halo rows in the band frame
                int kk = -1;
                const int64_t raw[4] = {L.Y0 - 2, L.Y0 - 1, L.Y1, L.Y1 + 1};
                for (int k2 = 0; k2 < 4; ++k2)
                  if (L.hoff[k2] >= 0 && map_axis(raw[k2], L.ny, cfg.bc[2], cfg.bc[3]) == J) kk = k2;
                if (kk < 0) {
                  emsg = "band halo row not planned";
                  return CLAW_EINVAL;
                }
                cells[lp][idx] = Src{1, L.hoff[kk] + I, L.hcs[kk]};
              } else {
                pend.push_back(Pending{lp, idx, 1, src_owner, 0, 0, 0, 0});
              }
              L.dbg_src[lp][idx] = -2;
              L.dbg_remote[lp][idx] = code;
            }
          } else if (src_owner == me) {
            // p belongs to dst_owner; I supply this cell (send list order =
            // dst patch ascending, cell row-major: identical on both sides)
            const int lq = L.local[q];
            L.send_off[dst_owner].push_back(L.off[lq] + static_cast<int64_t>(lj) * L.desc[q].mx + li);
            L.send_cs[dst_owner].push_back(static_cast<int64_t>(L.desc[q].mx) * L.desc[q].my);
            L.send_dbg[dst_owner].push_back(code);
          }
          continue;
        }
        if (!mine) continue;
        if (!C) {
          char b[160];
          std::snprintf(b, sizeof b, "level %d patch %d: ghost cell (%d,%d) has no donor", level, p, i, j);
          emsg = b;
          return CLAW_ENEST;
        }
        const int R = L.ratio;
        const int64_t Ic = I / R, Jc = J / R;
        pend.push_back(Pending{lp, idx, 2, -1, Ic, Jc, I, J});
        L.dbg_src[lp][idx] = -1;
      }
      return CLAW_OK;
  };
  // sparse lattice (grid kernel on a level of equal, lattice-aligned patches
  // that does not cover the domain, e.g. C3's level 3): one rank, one medium,
  // level > 1; the frame is laid out as the lattice's empty slots ("virtual
  // patches"), so coarse ghost values sit where the grid kernel's arithmetic
  // addressing looks for them (CLAW_SPARSE=0 disables)
  L.sparse = false;
  L.hslots.clear();
  {
    const char* e = std::getenv("CLAW_SPARSE");
    bool ok = !(e && e[0] == '0') && world == 1 && cfg.path == 0 && level > 1 && np > 0 && L.gapless;
    const int mx = np ? L.desc[0].mx : 0, my = np ? L.desc[0].my : 0;
    if (ok) ok = L.nx % mx == 0 && L.ny % my == 0 && L.nx < (1ll << 30) && L.ny < (1ll << 30);
    for (int p = 0; ok && p < np; ++p)
      ok = L.desc[p].mx == mx && L.desc[p].my == my && L.i0[p] % mx == 0 && L.j0[p] % my == 0 &&
           L.desc[p].rho == L.desc[0].rho && L.desc[p].K == L.desc[0].K &&
           L.off[L.local[p]] == static_cast<int64_t>(L.local[p]) * 3 * mx * my;
    const int64_t npx = ok ? L.nx / mx : 0, npy = ok ? L.ny / my : 0;
    ok = ok && npx * npy > np && npx * npy <= 4ll * np && npx * npy < (1ll << 30);
    if (ok) {
      L.sparse = true;
      L.npx = static_cast<int>(npx);
      L.hslots.assign(static_cast<size_t>(npx * npy), INT32_MIN);
      for (int p = 0; p < np; ++p) L.hslots[(L.j0[p] / my) * npx + L.i0[p] / mx] = L.local[p];
      int32_t v = 0;
      for (auto& x : L.hslots)
        if (x == INT32_MIN) x = -1 - v++;
      L.nvirt = v;
    }
  }
  lap("pre");
  // per patch; in parallel on one rank (every patch is owned, nothing is
  // sent), the pending frame cells concatenated in patch order afterwards
  std::vector<std::vector<Pending>> pend_p(np);
  std::vector<int> rc_p(np, CLAW_OK);
  std::vector<std::string> msg_p(np);
  const int nthr = world == 1 ? host_threads(np) : 1;
  parallel_for(nthr, np, [&](int p) {
    if (need[p]) rc_p[p] = ghost_patch(p, pend_p[p], msg_p[p]);
  });
  lap("ghost-par");
  for (int p = 0; p < np; ++p)
    if (rc_p[p]) return fail(c, rc_p[p], "%s", msg_p[p].c_str());
  std::vector<Pending> pend;
  if (world > 1)
    for (int p = 0; p < np; ++p) pend.insert(pend.end(), pend_p[p].begin(), pend_p[p].end());
  lap("ghosts");
  // coarse donors of a frame slot: centre, x-, x+, y-, y+ (coarse composite
  // via clamp/wrap)
  // (hint: the coarse patch of the previous donor -- a ghost cell's five
  // donors and the next ghost cell's are nearly always in one coarse patch,
  // so most lookups skip the bucket search; same result as C->find)
  auto make_spec = [&](const Pending& pd, int64_t slot, DevInterp& sp, std::string& emsg, int& hint) -> int {
    sp = DevInterp{};
    const int64_t cI[5] = {pd.Ic, map_axis(pd.Ic - 1, C->nx, cfg.bc[0], cfg.bc[1]),
                           map_axis(pd.Ic + 1, C->nx, cfg.bc[0], cfg.bc[1]), pd.Ic, pd.Ic};
    const int64_t cJ[5] = {pd.Jc, pd.Jc, pd.Jc, map_axis(pd.Jc - 1, C->ny, cfg.bc[2], cfg.bc[3]),
                           map_axis(pd.Jc + 1, C->ny, cfg.bc[2], cfg.bc[3])};
    for (int d = 0; d < 5; ++d) {
      const int h = hint;
      const bool in_h = h >= 0 && cI[d] >= C->i0[h] && cI[d] < C->i0[h] + C->desc[h].mx && cJ[d] >= C->j0[h] &&
                        cJ[d] < C->j0[h] + C->desc[h].my;
      const int q = in_h ? h : C->find(cI[d], cJ[d]);
      if (q >= 0) hint = q;
      if (q < 0 || C->local[q] < 0) {
        char b[200];
        std::snprintf(b, sizeof b, "level %d: coarse cell (%lld,%lld) needed for interpolation is not on level %d",
                      level, (long long)cI[d], (long long)cJ[d], level - 1);
        emsg = b;
        return CLAW_ENEST;
      }
      const int lq = C->local[q];
      sp.off[d] = C->off[lq] + (cJ[d] - C->j0[q]) * C->desc[q].mx + (cI[d] - C->i0[q]);
      sp.cs[d] = static_cast<int64_t>(C->desc[q].mx) * C->desc[q].my;
    }
    const int R = L.ratio;
    sp.xi = (static_cast<double>(pd.I % R) + 0.5) / static_cast<double>(R) - 0.5;
    sp.eta = (static_cast<double>(pd.J % R) + 0.5) / static_cast<double>(R) - 0.5;
    sp.dst = L.coarse_frame_off + slot;
    return CLAW_OK;
  };
  if (world == 1) {
    // one rank: every frame cell is coarse-interpolated; slots in patch order,
    // specs built per patch in parallel
    std::vector<int64_t> cstart(np + 1, 0);
    for (int p = 0; p < np; ++p) cstart[p + 1] = cstart[p] + static_cast<int64_t>(pend_p[p].size());
    L.coarse_frame_off = 0;
    L.ncoarse = cstart[np];
    L.frame_elems = 3 * L.ncoarse;
    L.frame_cs = L.ncoarse;
    const int smx = np ? L.desc[0].mx : 1, smy = np ? L.desc[0].my : 1;
    if (L.sparse) {  // frame = the lattice's virtual slots, [slot][3][my][mx]
      L.frame_elems = static_cast<int64_t>(L.nvirt) * 3 * smx * smy;
      L.frame_cs = static_cast<int64_t>(smx) * smy;
    }
    L.hinterp.resize(static_cast<size_t>(L.ncoarse));   // every entry is written below
    parallel_for(host_threads(np), np, [&](int p) {
      int hint = -1;
      for (size_t k = 0; k < pend_p[p].size() && !rc_p[p]; ++k) {
        const Pending& pd = pend_p[p][k];
        const int64_t slot = cstart[p] + static_cast<int64_t>(k);
        DevInterp& sp = L.hinterp[static_cast<size_t>(slot)];
        rc_p[p] = make_spec(pd, slot, sp, msg_p[p], hint);
        if (L.sparse) {
          const int32_t sl = L.hslots[(pd.J / smy) * L.npx + pd.I / smx];
          if (sl >= 0) {
            rc_p[p] = CLAW_EINVAL;
            msg_p[p] = "sparse lattice: a coarse ghost cell inside a patch slot";
          }
          sp.dst = static_cast<int64_t>(-1 - sl) * 3 * smx * smy + (pd.J % smy) * smx + pd.I % smx;
        }
        cells[pd.lp][pd.cellidx] = Src{1, sp.dst, L.frame_cs};
      }
    });
    for (int p = 0; p < np; ++p)
      if (rc_p[p]) return fail(c, rc_p[p], "%s", msg_p[p].c_str());
  } else {
  // frame layout: [peer 0 segment][peer 1 segment]...[coarse segment], each [3][n]
  // (band mode: planned above, full halo rows per source rank)
  int64_t fo = L.band ? L.frame_elems : 0;
  if (!L.band) {
    for (const Pending& pd : pend)
      if (pd.kind == 1) L.nrecv[pd.src_rank]++;
    for (int r = 0; r < world; ++r) {
      L.recv_frame_off[r] = fo;
      fo += 3 * L.nrecv[r];
    }
  }
  L.coarse_frame_off = fo;
  L.ncoarse = 0;
  for (const Pending& pd : pend)
    if (pd.kind == 2) L.ncoarse++;
  L.frame_elems = fo + 3 * L.ncoarse;
  L.frame_cs = L.ncoarse;
  std::vector<int64_t> rk(world, 0);
  int64_t ck = 0;
  int hint = -1;
  L.hinterp.clear();
  for (const Pending& pd : pend) {
    if (pd.kind == 1) {
      const int64_t k = rk[pd.src_rank]++;
      cells[pd.lp][pd.cellidx] = Src{1, L.recv_frame_off[pd.src_rank] + k, L.nrecv[pd.src_rank]};
    } else {
      const int64_t k = ck++;
      cells[pd.lp][pd.cellidx] = Src{1, L.coarse_frame_off + k, L.ncoarse};
      DevInterp sp;
      std::string emsg;
      if (int rc = make_spec(pd, k, sp, emsg, hint)) return fail(c, rc, "%s", emsg.c_str());
      L.hinterp.push_back(sp);
    }
  }

  }
  lap("frame");
  // rectangles (per patch, in parallel) and device patch records
  std::vector<std::vector<DevRect>> rects_p(L.owned.size());
  parallel_for(world == 1 ? host_threads(static_cast<int>(L.owned.size())) : 1, static_cast<int>(L.owned.size()),
               [&](int lp) {
                 compress_rects(cells[lp], L.desc[L.owned[lp]].mx, L.desc[L.owned[lp]].my, rects_p[lp]);
               });
  L.hpatch.clear();
  L.hrect.clear();
  for (size_t lp = 0; lp < L.owned.size(); ++lp) {
    const int p = L.owned[lp];
    DevPatch d{};
    d.off = L.off[lp];
    d.cs = static_cast<int64_t>(L.desc[p].mx) * L.desc[p].my;
    d.mx = L.desc[p].mx;
    d.my = L.desc[p].my;
    d.rect_begin = static_cast<int32_t>(L.hrect.size());
    L.hrect.insert(L.hrect.end(), rects_p[lp].begin(), rects_p[lp].end());
    d.rect_end = static_cast<int32_t>(L.hrect.size());
    d.crect = -1;   // (set below for levels the halo-lane kernel steps)
    // regions: strips W (i in [-2,0), j in [0,my)), E, S, N and 2x2 corners
    // SW, SE, NW, NE, each covered by one rectangle (or -1)
    const int X0 = -2, X1 = 0, X2 = d.mx, X3 = d.mx + 2, Y0 = -2, Y1 = 0, Y2 = d.my, Y3 = d.my + 2;
    const int sb[8][4] = {{X0, X1, Y1, Y2}, {X2, X3, Y1, Y2}, {X1, X2, Y0, Y1}, {X1, X2, Y2, Y3},
                          {X0, X1, Y0, Y1}, {X2, X3, Y0, Y1}, {X0, X1, Y2, Y3}, {X2, X3, Y2, Y3}};
    for (int e = 0; e < 8; ++e) {
      d.region[e] = -1;
      for (int k = d.rect_begin; k < d.rect_end; ++k) {
        const DevRect& r = L.hrect[k];
        if (r.i0 <= sb[e][0] && r.i0 + r.w >= sb[e][1] && r.j0 <= sb[e][2] && r.j0 + r.h >= sb[e][3]) {
          d.region[e] = k;
          break;
        }
      }
    }
    d.dx = L.desc[p].dx;
    d.dy = L.desc[p].dy;
    d.c = std::sqrt(L.desc[p].K / L.desc[p].rho);
    d.Z = L.desc[p].rho * d.c;
    L.hpatch.push_back(d);
  }
  lap("rects");
  // tiles: strips of <= 32 columns x <= tile_rows rows, largest first
  L.uniform = true;
  for (size_t lp = 1; lp < L.hpatch.size(); ++lp)
    if (L.hpatch[lp].c != L.hpatch[0].c || L.hpatch[lp].Z != L.hpatch[0].Z) L.uniform = false;
  // rows per tile: the configured value, or (auto) the largest power of two
  // <= 64 that still gives ~half a tile per resident warp of the GPU (SMs
  // x 16 warps); small, latency-bound levels get short tiles (>= 4) so the
  // serial row march of each warp stays short (measured: C3's level 3 runs
  // 2.5% faster with 32-row tiles at 0.7 tiles per warp than with 16-row
  // ones, profiles/r01_tile_rows_c123.txt; a floor of 4 rows instead of 8:
  // C2 0.061 -> 0.056 ms, C1 0.0089 -> 0.0084 ms per step, C3 and the paper
  // workload unchanged, profiles/r02_min_tile_rows.txt)
  if (c->cfg.tile_rows > 0) {
    L.th = c->tile_rows;
  } else {
    const int64_t want = static_cast<int64_t>(c->nsm) * 8;
    int min_th = 4;
    if (const char* e = std::getenv("CLAW_MIN_TH"))   // tuning: smallest auto tile height (2, 4 or 8)
      if (std::atoi(e) == 2 || std::atoi(e) == 4 || std::atoi(e) == 8) min_th = std::atoi(e);
    int th = 64;
    while (th > min_th && L.cells_owned / (32ll * th) < want) th /= 2;
    L.th = th;
  }
  // grid mode: whole domain tiled by equal patches in row-major order, gapless
  L.grid = false;
  if (L.sparse && L.uniform) {
    // sparse lattice: the grid kernel over listed (strip, row block) tiles that
    // hold at least one patch cell; tiles stay inside one patch row
    const int mx = L.desc[0].mx, my = L.desc[0].my;
    L.grid = true;
    L.Y0 = 0;
    L.Y1 = L.ny;
    int th = std::min(L.th, my);
    if (const char* e = std::getenv("CLAW_SPARSE_TH")) {  // tuning: rows per sparse-lattice tile
      const int v = std::atoi(e);
      if (v >= 4 && v <= my && my % v == 0) th = v;
    }
    L.grid_th = th;
    const int nbr = (my + th - 1) / th;
    const int64_t npy = L.ny / my, nstrip = claw::grid_nstrip(L.nx);
    L.hgtile.clear();
    for (int64_t pr = 0; pr < npy; ++pr)
      for (int rb = 0; rb < nbr; ++rb)
        for (int64_t st = 0; st < nstrip; ++st) {
          int64_t c0, c1;
          claw::grid_strip_cols(st, L.nx, c0, c1);
          bool any = false;
          for (int64_t pc = c0 / mx; pc <= (c1 - 1) / mx && !any; ++pc) any = L.hslots[pr * L.npx + pc] >= 0;
          if (any) L.hgtile.push_back(make_int4(static_cast<int>(st), static_cast<int>(pr * nbr + rb), 0, 0));
        }
    L.ngrid_tiles = static_cast<int64_t>(L.hgtile.size());
    L.ngrid_blocks = npy * nbr;
  } else if (L.uniform && c->cfg.path == 0 && (world == 1 || L.band) && L.gapless && !L.owned.empty() &&
             !L.sparse) {
    const int mx = L.desc[0].mx, my = L.desc[0].my;
    bool ok = (L.nx % mx == 0) && (L.ny % my == 0) &&
              static_cast<int64_t>(np) == (L.nx / mx) * (L.ny / my);
    const int npx = ok ? static_cast<int>(L.nx / mx) : 0;
    for (int p = 0; ok && p < np; ++p)
      ok = L.desc[p].mx == mx && L.desc[p].my == my && L.i0[p] == static_cast<int64_t>(p % npx) * mx &&
           L.j0[p] == static_cast<int64_t>(p / npx) * my;
    // owned patches: whole patch rows, back to back in the buffer
    const int p0 = L.owned.front();
    for (size_t lp = 0; ok && lp < L.owned.size(); ++lp)
      ok = L.owned[lp] == p0 + static_cast<int>(lp) && L.off[lp] == static_cast<int64_t>(lp) * 3 * mx * my;
    ok = ok && (p0 % npx == 0) && (L.owned.size() % npx == 0);
    if (ok && L.nx < (1ll << 30) && L.ny < (1ll << 30)) {
      L.grid = true;
      L.npx = npx;
      if (!L.band) {
        L.Y0 = 0;
        L.Y1 = L.ny;
      }
      // rows per grid tile: within one patch row (th <= my), or spanning
      // several whole patch rows (the kernel steps its row pointers across
      // patch-row boundaries), which halves the per-tile prologue on 32-row
      // patches; CLAW_GRID_TH overrides (tuning)
      int th = std::min(L.th, my);
      L.grid_th_base = 0;
      const int64_t nstrip0 = claw::grid_nstrip(L.nx);
      auto span_ok = [&](int w) { return span_rows_ok(w, my); };
      if (const char* e = std::getenv("CLAW_GRID_TH")) {
        if (span_ok(std::atoi(e))) th = std::atoi(e);
      } else if (c->cfg.tile_rows > 0) {
        if (span_ok(c->cfg.tile_rows)) th = c->cfg.tile_rows;
      } else if (L.th == 64) {
        // large level: tiles spanning whole patch rows, height chosen by the
        // makespan of the launch -- ceil(tiles / resident warps) waves of
        // (th + 4) row steps each (the 4 halo rows are the per-tile
        // prologue); the tail of a partly filled last wave is what one-
        // patch-row or fixed 256-row tiles lose on C4 (3.7 waves of 256-row
        // tiles: the last wave 70% full).  Ties go to the taller tile.
        L.grid_th_base = L.band ? 0 : th;
        // (the cap for the MC limiter only: the paper workload's van Leer
        // levels measured 3% slower per coarse step with it)
        th = makespan_th(nstrip0, L.Y1 - L.Y0, my, static_cast<int64_t>(c->nsm) * claw::grid_resident_warps(), th,
                         c->cfg.limiter == 4 ? kSpanAutoMax : 512);
      }
      L.grid_th = th;
      const int64_t nstrip = claw::grid_nstrip(L.nx);
      L.ngrid_blocks = th > my ? ((L.Y1 - L.Y0) + th - 1) / th : ((L.Y1 - L.Y0) / my) * ((my + th - 1) / th);
      L.ngrid_tiles = nstrip * L.ngrid_blocks;
      // band split (world > 1): every step is an interior launch, which runs
      // while the halo is in flight, and an edge launch after it lands.  The
      // edge launch takes only the kBandEdge rows at each end of the band
      // (the rows whose stencil reaches a halo row), so nearly all the work
      // is in the interior launch, whose tile height is chosen by the same
      // makespan rule over the band minus its edges (split into row blocks
      // instead, the edge launch would hold a third of the band as a second,
      // sub-wave launch: DESIGN.md section 9).  Tiles of the interior start
      // kBandEdge rows into a patch row, so my >= 16 keeps a tile's first
      // ring rows inside one patch row (the kernels' prologue).
      L.band_te = 0;
      if (L.band && my >= 16 && my % 4 == 0 && L.Y1 - L.Y0 >= 4 * kBandEdge) {
        L.band_te = kBandEdge;
        const int64_t slots = static_cast<int64_t>(c->nsm) * claw::grid_resident_warps();
        const int64_t rows = L.Y1 - L.Y0 - 2 * kBandEdge;
        // (interior tiles start 4 rows into a patch row and may start
        // anywhere in one after that: heights are multiples of 4 -- the
        // kernels cross patch rows at rows congruent to Y0 mod 4 -- so the
        // makespan can pick near-integral waves; e.g. N = 8 on C5: 547
        // strips x 17 blocks of 120 rows = 3.93 waves instead of 8 blocks of
        // 256 = 1.85 waves: per-rank step 0.295 -> 0.279 ms)
        // (heights capped at 256: the makespan model does not see a tall
        // tile's longer tail -- N = 2 on C5 picked 484-row tiles at 3.9 waves
        // and measured 6% slower than 192-row ones at 9.9 waves)
        auto int_ok = [&](int w) { return w >= 16 && w % 4 == 0 && w <= 512; };
        int thi = band_int_th(nstrip, rows, my, slots);
        if (const char* e = std::getenv("CLAW_GRID_TH")) {
          if (int_ok(std::atoi(e))) thi = std::atoi(e);
        } else if (c->cfg.tile_rows > 0 && int_ok(c->cfg.tile_rows)) {
          thi = c->cfg.tile_rows;
        }
        L.grid_th_int = thi;
        L.ngrid_blocks_int = (rows + thi - 1) / thi;
      }
    }
  }
  // generic tiles: strips of 30 columns for the halo-lane kernel (default;
  // CLAW_LANE=0 selects the side-pass kernel and 32-column strips)
  // (auto: where 30-column strips need at most 20% more warps than 32-column
  // ones -- measured 9% faster per coarse step on the paper workload's mixed
  // widths and 13% on C2, but 21% slower on uniform 64-wide patches, which
  // take 3 strips instead of 2; profiles/r01_lane_kernel.txt)
  {
    const char* e = std::getenv("CLAW_LANE");
    if (e && (e[0] == '0' || e[0] == '1')) {
      L.lane_tiles = e[0] == '1';
    } else {
      // lane tiles take the rows the tile loop below gives them (gth)
      const int lth = c->cfg.tile_rows == 0 ? std::min(L.th, 32) : L.th;
      int64_t n30 = 0, n32 = 0, t30 = 0;
      for (size_t lp = 0; lp < L.owned.size(); ++lp) {
        n30 += (L.hpatch[lp].mx + 29) / 30;
        n32 += (L.hpatch[lp].mx + 31) / 32;
        t30 += static_cast<int64_t>((L.hpatch[lp].mx + 29) / 30) * ((L.hpatch[lp].my + lth - 1) / lth);
      }
      // a level whose lane tiles fit in one wave of resident warps (SMs x
      // 16) is latency-bound: the extra warps are free and the march without
      // side passes is shorter
      L.lane_tiles = (5 * n30 <= 6 * n32 || t30 <= static_cast<int64_t>(c->nsm) * 16) ? 1 : 0;
    }
  }
  // each ghost cell's rectangle (the rectangles partition the frame ring),
  // for the levels the halo-lane kernel steps: it resolves a column segment
  // with one table load instead of searching the patch's rectangle list
  // (ragged levels whose ghost strips have several donors have no single
  // region rectangle; the search was the paper workload's top stall)
  // (offsets here; the map itself is written on the device from the
  // rectangle list, launch_cellrect in alloc_level: building it on the host
  // cost the paper workload ~1.5 ms per regrid)
  L.ncellrect = 0;
  if (L.lane_tiles && !L.grid)
    for (size_t lp = 0; lp < L.owned.size(); ++lp) {
      L.hpatch[lp].crect = L.ncellrect;
      L.ncellrect += frame_size(L.hpatch[lp].mx, L.hpatch[lp].my);
    }
  const int tstrip = L.lane_tiles ? 30 : 32;
  // halo-lane tiles take at most 32 rows: measured 1.3% faster per coarse
  // step on the paper workload's fine levels than 64 (more, shorter marches
  // over its ragged patches; profiles/r01_lane_kernel.txt); an equal split of
  // a patch's rows (50 + 50 instead of 64 + 36) measured no better
  const int gth = (L.lane_tiles && c->cfg.tile_rows == 0) ? std::min(L.th, 32) : L.th;
  L.htile.clear();
  for (size_t lp = 0; lp < L.owned.size(); ++lp) {
    const int mx = L.hpatch[lp].mx, my = L.hpatch[lp].my;
    for (int j0 = 0; j0 < my; j0 += gth)
      for (int i0 = 0; i0 < mx; i0 += tstrip) {
        const int tw = std::min(tstrip, mx - i0), th = std::min(gth, my - j0);
        L.htile.push_back(make_int4(static_cast<int>(lp), i0, j0, tw | (th << 16)));
      }
  }
  // tiles of patches that read remote (other-rank) ghost cells go last, so a
  // step can run the others while the halo is in flight
  std::vector<char> remote(L.owned.size(), 0);
  for (size_t lp = 0; lp < L.owned.size() && world > 1; ++lp)
    for (const int64_t code : L.dbg_src[lp])
      if (code == -2) {
        remote[lp] = 1;
        break;
      }
  std::stable_sort(L.htile.begin(), L.htile.end(), [&](const int4& a, const int4& b) {
    if (remote[a.x] != remote[b.x]) return remote[a.x] < remote[b.x];
    return (a.w & 0xffff) * (a.w >> 16) > (b.w & 0xffff) * (b.w >> 16);
  });
  L.ntile_interior = 0;
  while (L.ntile_interior < static_cast<int64_t>(L.htile.size()) && !remote[L.htile[L.ntile_interior].x])
    ++L.ntile_interior;
  lap("tiles");
  // updating table: coarse cells (level-1) whose R x R children are all
  // interior cells of this level
  L.hu.clear();
  L.hur.clear();
  L.hur_chunk.clear();
  L.hu_src.clear();
  L.hu_scs.clear();
  L.upd_send_off.clear();
  L.upd_send_cs.clear();
  L.upd_recv_off.assign(world, {});
  L.upd_recv_cs.assign(world, {});
  if (C && (world == 1 || L.dist)) {
    // (partitioned level: the coarse level is replicated, so every fine
    // patch's rectangles are computed -- the device tables take the owned
    // ones, the exchange lists every rank's -- and the level must be aligned
    // to the coarse cells: no per-cell entries)
    const int R = L.ratio;
    // per fine patch in parallel (host workers), concatenated in patch order:
    // the tables are the sequential ones
    struct UpdPart {
      std::vector<claw::DevUpdateRect> rects;
      std::vector<claw::DevUpdate> cells;
      std::vector<int64_t> so, sc;  // slow entries (src = index into this part's R*R groups)
    };
    std::vector<UpdPart> parts(np);
    parallel_for(host_threads(np), np, [&](int fp) {
      UpdPart& P = parts[fp];
      const int64_t ic0 = L.i0[fp] / R, ic1 = (L.i0[fp] + L.desc[fp].mx - 1) / R;
      const int64_t jc0 = L.j0[fp] / R, jc1 = (L.j0[fp] + L.desc[fp].my - 1) / R;
      const int64_t fi0 = L.i0[fp], fi1 = L.i0[fp] + L.desc[fp].mx, fj0 = L.j0[fp], fj1 = L.j0[fp] + L.desc[fp].my;
      // coarse cells whose R x R children all lie in this patch: rectangles
      // (one per overlapping coarse patch), averaged by one CTA each
      const int64_t ia = (fi0 + R - 1) / R, ib = fi1 / R, ja = (fj0 + R - 1) / R, jb = fj1 / R;
      if (ia < ib && ja < jb) {
        std::vector<int> cand;
        for (int64_t by = ja / kBucket; by <= (jb - 1) / kBucket && by < C->nby; ++by)
          for (int64_t bx = ia / kBucket; bx <= (ib - 1) / kBucket && bx < C->nbx; ++bx)
            for (int64_t k = C->bstart[by * C->nbx + bx]; k < C->bstart[by * C->nbx + bx + 1]; ++k)
              cand.push_back(C->blist[k]);
        std::sort(cand.begin(), cand.end());
        cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
        for (int cq : cand) {
          const int64_t x0 = std::max(ia, C->i0[cq]), x1 = std::min(ib, C->i0[cq] + C->desc[cq].mx);
          const int64_t y0 = std::max(ja, C->j0[cq]), y1 = std::min(jb, C->j0[cq] + C->desc[cq].my);
          if (x0 >= x1 || y0 >= y1) continue;
          const int lc = C->local[cq];
          claw::DevUpdateRect r{};
          r.dst = C->off[lc] + (y0 - C->j0[cq]) * C->desc[cq].mx + (x0 - C->i0[cq]);
          r.src = L.local[fp] >= 0 ? L.off[L.local[fp]] + (y0 * R - fj0) * L.desc[fp].mx + (x0 * R - fi0) : 0;
          r.dcs = static_cast<int64_t>(C->desc[cq].mx) * C->desc[cq].my;
          r.fcs = static_cast<int64_t>(L.desc[fp].mx) * L.desc[fp].my;
          r.cmx = C->desc[cq].mx;
          r.fmx = L.desc[fp].mx;
          r.w = static_cast<int32_t>(x1 - x0);
          r.h = static_cast<int32_t>(y1 - y0);
          P.rects.push_back(r);
        }
      }
      // the rest of the footprint (patches not aligned to the coarse cells):
      // cell by cell
      int cq = -1;
      for (int64_t Jc = jc0; Jc <= jc1; ++Jc)
        for (int64_t Ic = ic0; Ic <= ic1; ++Ic) {
          if (Jc >= ja && Jc < jb && Ic >= ia && Ic < ib) {
            Ic = ib - 1;
            continue;
          }
          if (cq < 0 || Ic < C->i0[cq] || Ic >= C->i0[cq] + C->desc[cq].mx || Jc < C->j0[cq] ||
              Jc >= C->j0[cq] + C->desc[cq].my)
            cq = C->find(Ic, Jc);
          if (cq < 0) continue;
          const int lc = C->local[cq];
          // each coarse cell once: only from the fine patch holding its first child
          if (L.find(Ic * R, Jc * R) != fp) continue;
          bool all = true, one = true;
          std::vector<int64_t> so, sc;
          for (int b = 0; b < R && all; ++b)
            for (int a = 0; a < R && all; ++a) {
              const int q = L.find(Ic * R + a, Jc * R + b);
              if (q < 0) {
                all = false;
                break;
              }
              if (q != fp) one = false;
              const int lq = L.local[q];
              so.push_back(L.off[lq] + (Jc * R + b - L.j0[q]) * L.desc[q].mx + (Ic * R + a - L.i0[q]));
              sc.push_back(static_cast<int64_t>(L.desc[q].mx) * L.desc[q].my);
            }
          if (!all) continue;
          if (L.dist) {   // (unaligned fine patches: rejected below)
            P.cells.push_back(claw::DevUpdate{});
            continue;
          }
          claw::DevUpdate u{};
          u.dst = C->off[lc] + (Jc - C->j0[cq]) * C->desc[cq].mx + (Ic - C->i0[cq]);
          u.dcs = C->desc[cq].mx * C->desc[cq].my;
          if (one) {
            u.src = so[0];
            u.fcs = L.desc[fp].mx * L.desc[fp].my;
            u.fmx = L.desc[fp].mx;
            u.slow = 0;
          } else {
            u.src = static_cast<int64_t>(P.so.size()) / (R * R);
            u.slow = 1;
            P.so.insert(P.so.end(), so.begin(), so.end());
            P.sc.insert(P.sc.end(), sc.begin(), sc.end());
          }
          P.cells.push_back(u);
        }
    });
    for (int fp = 0; fp < np && L.dist; ++fp) {
      if (!parts[fp].cells.empty())
        return fail(c, CLAW_EINVAL,
                    "level %d is partitioned across ranks (dist_level): patch %d is not aligned to the level-%d "
                    "cells (R=%d)", level, fp, level - 1, R);
      // every rank's averaged coarse cells, in patch, rectangle, row-major
      // order (the same lists on every rank)
      const int ow = L.owner[fp];
      for (const claw::DevUpdateRect& r : parts[fp].rects)
        for (int y = 0; y < r.h; ++y)
          for (int x = 0; x < r.w; ++x) {
            const int64_t o = r.dst + static_cast<int64_t>(y) * r.cmx + x;
            if (ow == me) {
              L.upd_send_off.push_back(o);
              L.upd_send_cs.push_back(r.dcs);
            } else {
              L.upd_recv_off[ow].push_back(o);
              L.upd_recv_cs[ow].push_back(r.dcs);
            }
          }
    }
    for (int fp = 0; fp < np; ++fp) {
      if (L.local[fp] < 0) continue;   // (partitioned level: owned patches only)
      UpdPart& P = parts[fp];
      for (claw::DevUpdateRect r : P.rects) {
        r.chunk0 = static_cast<int32_t>(L.hur_chunk.size());
        L.hur_chunk.insert(L.hur_chunk.end(), (r.w * r.h + claw::kUpdChunk - 1) / claw::kUpdChunk,
                           static_cast<int32_t>(L.hur.size()));
        L.hur.push_back(r);
      }
      const int64_t base = static_cast<int64_t>(L.hu_src.size()) / (R * R);
      for (claw::DevUpdate u : P.cells) {
        if (u.slow) u.src += base;
        L.hu.push_back(u);
      }
      L.hu_src.insert(L.hu_src.end(), P.so.begin(), P.so.end());
      L.hu_scs.insert(L.hu_scs.end(), P.sc.begin(), P.sc.end());
    }
  }
  lap("update");
  // conservation-fix registers (same order as the oracle's: coarse patch, row,
  // column, then neighbours x-, x+, y-, y+)
  L.hreg.clear();
  L.hheads.clear();
  if (C && cfg.reflux) {
    const int R = L.ratio;
    for (int p = 0; p < np; ++p)
      if (L.i0[p] % R || L.j0[p] % R || L.desc[p].mx % R || L.desc[p].my % R)
        return fail(c, CLAW_EINVAL, "reflux: level %d patch %d is not aligned to the level-%d cells (R=%d)", level, p,
                    level - 1, R);
    auto covered = [&](int64_t Ic, int64_t Jc) {
      for (int b = 0; b < R; ++b)
        for (int a = 0; a < R; ++a)
          if (L.find(Ic * R + a, Jc * R + b) < 0) return false;
      return true;
    };
    for (int cq = 0; cq < C->npatch; ++cq) {
      const int lc = C->local[cq];
      for (int lj = 0; lj < C->desc[cq].my; ++lj)
        for (int li = 0; li < C->desc[cq].mx; ++li) {
          const int64_t Ic = C->i0[cq] + li, Jc = C->j0[cq] + lj;
          if (covered(Ic, Jc)) continue;
          bool head = true;
          for (int e = 0; e < 4; ++e) {
            const int dir = e / 2, side = (e % 2 == 0) ? 1 : 0;
            int64_t In = Ic + (dir == 0 ? (e % 2 ? 1 : -1) : 0);
            int64_t Jn = Jc + (dir == 1 ? (e % 2 ? 1 : -1) : 0);
            const int64_t nax = dir == 0 ? C->nx : C->ny, v = dir == 0 ? In : Jn;
            if (v < 0 || v >= nax) {
              if (cfg.bc[2 * dir] != CLAW_BC_PERIODIC) continue;
              if (dir == 0) In = (In + C->nx) % C->nx;
              else Jn = (Jn + C->ny) % C->ny;
            }
            if (!covered(In, Jn)) continue;
            int64_t I, J;
            if (dir == 0) {
              I = In * R + (side == 0 ? 0 : R - 1);
              J = Jc * R;
            } else {
              I = Ic * R;
              J = Jn * R + (side == 0 ? 0 : R - 1);
            }
            const int fq = L.find(I, J);
            claw::DevReflux r{};
            r.cp = lc;
            r.ci = li;
            r.cj = lj;
            r.ds = dir | (side << 1);
            r.fp = L.local[fq];
            r.fi = static_cast<int32_t>(I - L.i0[fq]);
            r.fj = static_cast<int32_t>(J - L.j0[fq]);
            if (head) L.hheads.push_back(static_cast<int32_t>(L.hreg.size()));
            head = false;
            L.hreg.push_back(r);
          }
        }
    }
    L.hheads.push_back(static_cast<int32_t>(L.hreg.size()));
  }
  return CLAW_OK;
}

// Host twin of the kernel's make_consts (same operations, same order; x86-64
// without FMA contraction, so every result is the same IEEE double).
void fill_step_consts(const DevPatch& pt, double dt, double LS, int ot, claw::StepConsts& k) {
  volatile double c = pt.c, Z = pt.Z;  // volatile: keep each operation separately rounded
  k.Z = Z;
  k.r = dt / pt.dx;
  k.s = dt / pt.dy;
  k.h = 0.5 * c;
  k.hz = k.h / Z;
  volatile double cr = c * k.r, cs = c * k.s;
  volatile double omx = 1.0 - cr, omy = 1.0 - cs;
  const double kx = c * omx, ky = c * omy;
  k.kx4 = kx / (4.0 * LS);
  k.ky4 = ky / (4.0 * LS);
  k.kx2 = (ot == 2) ? kx / (2.0 * LS) : 0.0;
  k.ky2 = (ot == 2) ? ky / (2.0 * LS) : 0.0;
  k.kx4z = k.kx4 / Z;
  k.ky4z = k.ky4 / Z;
  volatile double rs = k.r * k.s;
  volatile double rsc = rs * c;
  k.T = (ot != 0) ? 0.25 * rsc : 0.0;
  k.TZ = (ot != 0) ? k.T / Z : 0.0;
  const double a = k.r * c, b = k.s * c;
  k.cfl = a > b ? a : b;
  k.mr = -k.r;
  k.ms = -k.s;
  k.mT = -k.T;
}

template <class T>
int upload(claw_ctx* ctx, DevBuf<T>& b, const std::vector<T>& v) {
  CUDA_TRY(b.alloc(v.size()));
  if (!v.empty()) CUDA_TRY(cudaMemcpy(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return CLAW_OK;
}

// Device pool of a planned level: two ping-pong buffers, the frame, every
// table (allocated once per set_level / regrid; no per-step allocation, cf.
// the paper's memory pool P:422-426; blocks come from the caching Pool).
int alloc_level(claw_ctx* ctx, int level, Level& L) {
  for (int b = 0; b < 2; ++b) {
    cudaError_t e = L.q[b].alloc(std::max<int64_t>(L.buf_elems, 1));
    if (e != cudaSuccess) {
      const long long bytes = 2ll * L.buf_elems * 8;
      L = Level();
      cudaGetLastError();
      return fail(ctx, CLAW_ENOMEM, "level %d: cannot allocate %lld bytes of device pool", level, bytes);
    }
  }
  // a fine level's coarse ghost values for all R substeps of a coarse step
  // are interpolated by one launch into R slices (claw_advance_hierarchy)
  L.nslice = (level > 1 && L.ncoarse > 0 && !L.dist && L.ratio >= 2 &&
              L.ratio <= claw::kMaxInterpAlphas) ? L.ratio : 1;
  CUDA_TRY(L.frame.alloc(std::max<int64_t>(L.frame_elems, 1) * L.nslice));
  if (int r2 = upload(ctx, L.dpatch, L.hpatch)) return r2;
  if (int r2 = upload(ctx, L.drect, L.hrect)) return r2;
  if (L.ncellrect > 0) {
    // (on the legacy stream, after the pageable uploads of the patch and
    // rectangle tables it reads, and waited for: the step kernels on the
    // library's stream read the map)
    CUDA_TRY(L.dcellrect.alloc(static_cast<size_t>(L.ncellrect)));
    CUDA_TRY(static_cast<cudaError_t>(claw::launch_cellrect(L.dpatch.p, static_cast<int32_t>(L.hpatch.size()),
                                                            L.drect.p, L.dcellrect.p, nullptr)));
    CUDA_TRY(cudaStreamSynchronize(nullptr));
  }
  if (int r2 = upload(ctx, L.dtile, L.htile)) return r2;
  if (int r2 = upload(ctx, L.dinterp, L.hinterp)) return r2;
  if (int r2 = upload(ctx, L.du, L.hu)) return r2;
  if (int r2 = upload(ctx, L.dur, L.hur)) return r2;
  if (int r2 = upload(ctx, L.dur_chunk, L.hur_chunk)) return r2;
  if (int r2 = upload(ctx, L.dslots, L.hslots)) return r2;
  if (int r2 = upload(ctx, L.dgtile, L.hgtile)) return r2;
  if (int r2 = upload(ctx, L.du_src, L.hu_src)) return r2;
  if (int r2 = upload(ctx, L.du_scs, L.hu_scs)) return r2;
  if (int r2 = upload(ctx, L.dreg, L.hreg)) return r2;
  if (int r2 = upload(ctx, L.dheads, L.hheads)) return r2;
  CUDA_TRY(L.racc.alloc(std::max<size_t>(3 * L.hreg.size(), 1)));
  CUDA_TRY(cudaMemset(L.racc.p, 0, L.racc.n * 8));
  CUDA_TRY(L.pcfl.alloc(std::max<size_t>(L.owned.size(), 1)));
  CUDA_TRY(L.lcfl.alloc(2));
  CUDA_TRY(cudaMemset(L.pcfl.p, 0, L.pcfl.n * 8));
  CUDA_TRY(cudaMemset(L.lcfl.p, 0, 16));
  L.gen = 0;
  const int world = static_cast<int>(L.send_off.size());   // (1 unless the level is partitioned)
  L.dsend_off.clear();
  L.dsend_cs.clear();
  L.dsend_buf.clear();
  if (int r2 = upload(ctx, L.dupd_send_off, L.upd_send_off)) return r2;
  if (int r2 = upload(ctx, L.dupd_send_cs, L.upd_send_cs)) return r2;
  CUDA_TRY(L.dupd_send_buf.alloc(std::max<size_t>(3 * L.upd_send_off.size(), 1)));
  L.dupd_recv_off.clear();
  L.dupd_recv_cs.clear();
  L.dupd_recv_buf.clear();
  for (size_t r = 0; r < L.upd_recv_off.size(); ++r) {
    L.dupd_recv_off.emplace_back(new DevBuf<int64_t>());
    L.dupd_recv_cs.emplace_back(new DevBuf<int64_t>());
    L.dupd_recv_buf.emplace_back(new DevBuf<double>());
    if (int r2 = upload(ctx, *L.dupd_recv_off[r], L.upd_recv_off[r])) return r2;
    if (int r2 = upload(ctx, *L.dupd_recv_cs[r], L.upd_recv_cs[r])) return r2;
    CUDA_TRY(L.dupd_recv_buf[r]->alloc(std::max<size_t>(3 * L.upd_recv_off[r].size(), 1)));
  }
  for (int r = 0; r < world; ++r) {
    L.dsend_off.emplace_back(new DevBuf<int64_t>());
    L.dsend_cs.emplace_back(new DevBuf<int64_t>());
    L.dsend_buf.emplace_back(new DevBuf<double>());
    if (int r2 = upload(ctx, *L.dsend_off[r], L.send_off[r])) return r2;
    if (int r2 = upload(ctx, *L.dsend_cs[r], L.send_cs[r])) return r2;
    CUDA_TRY(L.dsend_buf[r]->alloc(3 * L.send_off[r].size()));
  }
  // generic levels with many tall tiles (one rank): side records computed
  // ahead of the step kernel by a side_kernel -- measured 10% faster on the
  // paper workload's level 3 (64-row tiles), 4% slower on C3's level 3
  // (16-row tiles), so only for th >= 64 (CLAW_SIDE=0/1 overrides)
  {
    const char* e = std::getenv("CLAW_SIDE");
    const bool want = e ? e[0] == '1' : (L.htile.size() >= 1024 && L.th >= 64);
    L.use_side = want && !L.grid && !L.lane_tiles && !L.dist && !L.htile.empty();
    if (L.use_side) CUDA_TRY(L.side.alloc(L.htile.size() * static_cast<size_t>(claw::side_stride())));
  }
  L.device_bytes = 2 * L.buf_elems * 8 + L.frame_elems * 8 +
                   static_cast<int64_t>(L.hpatch.size() * sizeof(DevPatch) + L.hrect.size() * sizeof(DevRect) +
                                        L.htile.size() * sizeof(int4) + L.hinterp.size() * sizeof(DevInterp));
  return CLAW_OK;
}

int check_ctx(claw_ctx* c) {
  if (!c) return CLAW_EINVAL;
  t_arena = c->arena_id;   // this call's allocations come from the context's arena, if any
  if (c->dead) return fail(c, CLAW_ECUDA, "context unusable after an earlier CUDA/NCCL error");
  return CLAW_OK;
}

// claw_config.check_finite: the flag the steps since the last read raised
// (h_nf copied by the caller's synchronising read); ENONFINITE names the level
int take_nonfinite(claw_ctx* ctx) {
  if (!ctx->cfg.check_finite || *ctx->h_nf == 0) return CLAW_OK;
  const int lv = *ctx->h_nf;
  *ctx->h_nf = 0;
  CUDA_TRY(cudaMemset(ctx->nf_flag.p, 0, 4));
  return fail(ctx, CLAW_ENONFINITE, "non-finite value (NaN / Inf) in q after a step of level %d", lv);
}

int check_level(claw_ctx* c, int level) {
  if (level < 1 || level > kMaxLevel || !c->lev[level].set)
    return fail(c, CLAW_ESTATE, "level %d is not set", level);
  return CLAW_OK;
}

void record(claw_ctx* c, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v, bool start) {
  if (!c->profiling || c->dry) return;
  const unsigned fl = c->capturing ? cudaEventRecordExternal : cudaEventRecordDefault;
  if (start) {
    std::pair<cudaEvent_t, cudaEvent_t> e;
    if (!c->ev_free.empty()) {
      e = c->ev_free.back();
      c->ev_free.pop_back();
    } else {
      cudaEventCreate(&e.first);
      cudaEventCreate(&e.second);
    }
    v.push_back(e);
    cudaEventRecordWithFlags(e.first, c->stream, fl);
  } else {
    cudaEventRecordWithFlags(v.back().second, c->stream, fl);
  }
}

void drop_graphs(claw_ctx* c) {
  for (HierGraph& g : c->graphs) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    for (auto& e : g.ev_step) c->ev_free.push_back(e);
    for (auto& e : g.ev_ghost) c->ev_free.push_back(e);
  }
  c->graphs.clear();
  c->epoch++;
}

double drain(claw_ctx* c, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v) {
  double ms = 0;
  for (auto& e : v) {
    float t = 0;
    cudaEventSynchronize(e.second);
    cudaEventElapsedTime(&t, e.first, e.second);
    ms += t;
    c->ev_free.push_back(e);
  }
  v.clear();
  return ms;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* claw_version(void) { return "libclaw 0.1 (sm_100a, fp64, acoustics 2D)"; }

int claw_partition(int32_t npatch, const claw_patch_desc* d, int32_t world, int32_t* owner) {
  if (npatch < 1 || !d || !owner || world < 1) return CLAW_EINVAL;
  // integer boxes relative to the minimum corner (no domain needed)
  double xmin = d[0].xlower, ymin = d[0].ylower;
  for (int p = 1; p < npatch; ++p) {
    xmin = std::min(xmin, d[p].xlower);
    ymin = std::min(ymin, d[p].ylower);
  }
  std::vector<int64_t> i0(npatch), j0(npatch);
  for (int p = 0; p < npatch; ++p) {
    if (!(d[p].dx > 0) || !(d[p].dy > 0)) return CLAW_EINVAL;
    i0[p] = std::llround((d[p].xlower - xmin) / d[p].dx);
    j0[p] = std::llround((d[p].ylower - ymin) / d[p].dy);
  }
  partition_impl(npatch, d, i0, j0, world, owner);
  return CLAW_OK;
}

int claw_create(const claw_config* cfg, claw_ctx** out) {
  if (!cfg || !out) return CLAW_EINVAL;
  *out = nullptr;
  auto* ctx = new claw_ctx();
  ctx->cfg = *cfg;
  int rc = validate_config(ctx, cfg);
  if (rc) {
    // keep the context so the caller can read the message
    *out = ctx;
    ctx->dead = true;
    return rc;
  }
  ctx->tile_rows = cfg->tile_rows > 0 ? cfg->tile_rows : claw::max_tile_rows();
  ctx->host_only = cfg->device < 0;
  {
    const char* pd = std::getenv("CLAW_PDL");  // programmatic dependent launches (default on)
    claw::set_pdl(pd ? std::atoi(pd) : 1);
    const char* rc = std::getenv("CLAW_ROWCOPY");  // grid-kernel row copies: 3 auto
    claw::set_rowcopy(rc ? std::atoi(rc) : 3);
  }
  {
    // opt-in (CLAW_GRAPH=1): measured slower than the asynchronous launch
    // sequence, which never starves the GPU inside a coarse step
    const char* gv = std::getenv("CLAW_GRAPH");
    ctx->graphs_on = gv && gv[0] == '1';
  }
  *out = ctx;
  if (ctx->host_only) return CLAW_OK;
  CUDA_TRY(cudaSetDevice(cfg->device));
  CUDA_TRY(cudaDeviceGetAttribute(&ctx->nsm, cudaDevAttrMultiProcessorCount, cfg->device));
  claw::set_grid_wave(ctx->nsm * claw::grid_resident_warps());
  t_arena = 0;
  if (cfg->arena) {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, cfg->arena) != cudaSuccess || pa.type != cudaMemoryTypeDevice ||
        pa.device != cfg->device) {
      cudaGetLastError();
      ctx->dead = true;
      return fail(ctx, CLAW_EINVAL, "arena %p is not device memory of device %d", cfg->arena, cfg->device);
    }
    ctx->arena_id = pool().add_arena(cfg->device, cfg->arena, static_cast<size_t>(cfg->arena_bytes));
    if (!ctx->arena_id) {
      ctx->dead = true;
      return fail(ctx, CLAW_EINVAL, "arena_bytes=%llu: too small", static_cast<unsigned long long>(cfg->arena_bytes));
    }
    t_arena = ctx->arena_id;
  }
  if (cfg->stream) {
    ctx->stream = static_cast<cudaStream_t>(cfg->stream);
  } else {
    CUDA_TRY(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    ctx->own_stream = true;
  }
  CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_cfl), sizeof(double)));
  if (cfg->check_finite) {
    CUDA_TRY(ctx->nf_flag.alloc(1));
    CUDA_TRY(cudaMemset(ctx->nf_flag.p, 0, 4));
    CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_nf), sizeof(int32_t)));
    *ctx->h_nf = 0;
  }
  if (cfg->world > 1) {
    CUDA_TRY(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_ready, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_halo, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_int, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_edge, cudaEventDisableTiming));
  }
  if (cfg->world > 1 && cfg->exchange == 0) {
    if (!g_nccl.load(ctx->err)) {
      ctx->dead = true;
      return CLAW_ENCCL;
    }
    ncclUniqueId id;
    std::memcpy(&id, cfg->nccl_unique_id, sizeof id);
    ncclResult_t r = g_nccl.CommInitRank(&ctx->comm, cfg->world, id, cfg->rank);
    if (r != ncclSuccess) return nccl_fail(ctx, r, "ncclCommInitRank");
  }
  return CLAW_OK;
}

int claw_comm_info(const claw_ctx* ctx, int32_t* nranks, int32_t* rank, int32_t* cuda_device) {
  if (!ctx || !nranks || !rank || !cuda_device) return CLAW_EINVAL;
  if (!ctx->comm || !g_nccl.CommCount || !g_nccl.CommUserRank || !g_nccl.CommCuDevice) return CLAW_ESTATE;
  int n = 0, r = 0, d = 0;
  if (g_nccl.CommCount(ctx->comm, &n) != ncclSuccess || g_nccl.CommUserRank(ctx->comm, &r) != ncclSuccess ||
      g_nccl.CommCuDevice(ctx->comm, &d) != ncclSuccess)
    return CLAW_ENCCL;
  *nranks = n;
  *rank = r;
  *cuda_device = d;
  return CLAW_OK;
}

int claw_nccl_unique_id(void* out128) {
  std::string err;
  if (!out128 || !g_nccl.load(err)) return CLAW_ENCCL;
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return CLAW_ENCCL;
  std::memcpy(out128, &id, sizeof id);
  return CLAW_OK;
}

int claw_destroy(claw_ctx* ctx) {
  if (!ctx) return CLAW_EINVAL;
  if (!ctx->host_only && !ctx->dead) cudaStreamSynchronize(ctx->stream);
  drain(ctx, ctx->ev_step);
  drain(ctx, ctx->ev_ghost);
  drop_graphs(ctx);
  if (ctx->h_alpha) cudaFreeHost(ctx->h_alpha);
  ctx->d_alpha.reset();
  for (auto& L : ctx->lev) L = Level();
  for (auto& L : ctx->stash) L = Level();
  for (auto& e : ctx->ev_free) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  ctx->hier_buf.reset();
  if (ctx->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(ctx->comm);
  if (ctx->h_cfl) cudaFreeHost(ctx->h_cfl);
  if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  if (ctx->ev_ready) cudaEventDestroy(ctx->ev_ready);
  if (ctx->ev_halo) cudaEventDestroy(ctx->ev_halo);
  if (ctx->ev_int) cudaEventDestroy(ctx->ev_int);
  if (ctx->ev_edge) cudaEventDestroy(ctx->ev_edge);
  ctx->nf_flag.reset();
  ctx->hier_many.reset();
  if (ctx->h_nf) cudaFreeHost(ctx->h_nf);
  if (ctx->h_many) cudaFreeHost(ctx->h_many);
  const int64_t arena = ctx->arena_id;
  delete ctx;                                  // (every buffer is back in the pool)
  if (arena) pool().remove_arena(arena);
  t_arena = 0;
  return CLAW_OK;
}

const char* claw_last_error(const claw_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int claw_set_level(claw_ctx* ctx, int32_t level, int32_t npatch, const claw_patch_desc* descs,
                   const double* q0) {
  Nvtx nv_("claw_set_level L%d", level);
  if (int rc = check_ctx(ctx)) return rc;
  if (level < 1 || level > kMaxLevel) return fail(ctx, CLAW_EINVAL, "level=%d: must be 1..%d", level, kMaxLevel);
  if (npatch < 1 || !descs) return fail(ctx, CLAW_EINVAL, "npatch=%d: need >= 1 patch descriptors", npatch);
  if (level > 1 && !ctx->lev[level - 1].set) return fail(ctx, CLAW_ESTATE, "level %d set before level %d", level, level - 1);
  if (level > 1 && ctx->cfg.world > 1 && level > ctx->cfg.dist_level)
    return fail(ctx, CLAW_EINVAL,
                "level %d with world=%d: a multi-rank hierarchy needs claw_config.dist_level >= %d (the partitioned, "
                "finest level; the levels below it are replicated)", level, ctx->cfg.world, level);
  if (level > 1 && ctx->lev[1].vc)
    return fail(ctx, CLAW_EINVAL, "level %d: variable media (claw_set_aux) are single-level (DESIGN.md R20)", level);
  if (!ctx->host_only) CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  drop_graphs(ctx);
  for (int l = level; l <= kMaxLevel; ++l) {
    ctx->lev[l] = Level();
    ctx->stash[l] = Level();
  }
  Level& L = ctx->lev[level];
  int rc = build_geometry(ctx, level, npatch, descs, L);
  if (!rc) rc = plan_level(ctx, level, L);
  if (rc) {
    L = Level();
    return rc;
  }
  L.t_old = L.t_new = (level > 1) ? ctx->lev[level - 1].t_old : 0.0;
  if (ctx->host_only) {
    L.set = true;
    return CLAW_OK;
  }
  if (int r2 = alloc_level(ctx, level, L)) return r2;
  L.cur = 0;
  if (q0) {
    if (L.gapless) {
      CUDA_TRY(cudaMemcpy(L.q[0].p, q0, L.buf_elems * 8, cudaMemcpyHostToDevice));
    } else {
      // alignment gaps between patches are never read; zero them so the
      // whole-buffer copy below moves initialised bytes only
      CUDA_TRY(cudaMemset(L.q[0].p, 0, L.buf_elems * 8));
      int64_t src = 0;
      for (size_t lp = 0; lp < L.owned.size(); ++lp) {
        const int64_t n = 3ll * L.hpatch[lp].mx * L.hpatch[lp].my;
        CUDA_TRY(cudaMemcpy(L.q[0].p + L.off[lp], q0 + src, n * 8, cudaMemcpyHostToDevice));
        src += n;
      }
    }
  } else {
    CUDA_TRY(cudaMemset(L.q[0].p, 0, L.buf_elems * 8));
  }
  CUDA_TRY(cudaMemcpy(L.q[1].p, L.q[0].p, L.buf_elems * 8, cudaMemcpyDeviceToDevice));
  CUDA_TRY(cudaMemset(L.frame.p, 0, L.frame.n * 8));
  // the copies above ran on the legacy stream; the library's stream is
  // non-blocking, so finish them before any kernel can read the level
  CUDA_TRY(cudaStreamSynchronize(nullptr));
  L.set = true;
  return CLAW_OK;
}

int claw_set_aux(claw_ctx* ctx, int32_t level, const double* aux) {
  Nvtx nv_("claw_set_aux L%d", level);
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_level(ctx, level)) return rc;
  Level& L = ctx->lev[level];
  if (level != 1 || ctx->lev[2].set)
    return fail(ctx, CLAW_EINVAL, "set_aux(level %d): variable media are single-level (level 1, no finer level)", level);
  if (!L.grid || L.sparse)
    return fail(ctx, CLAW_EINVAL, "set_aux: the level must be one uniform grid of equal patches (claw_level_mode 1; "
                "with world > 1 the band partition)");
  if (!aux) return fail(ctx, CLAW_EINVAL, "aux is NULL");
  const int mx = L.desc[0].mx, my = L.desc[0].my;
  const int64_t plane = static_cast<int64_t>(mx) * my;
  const int64_t n = static_cast<int64_t>(L.npatch) * 2 * plane;
  for (int64_t k = 0; k < n; ++k)
    if (!(aux[k] > 0.0) || !std::isfinite(aux[k]))
      return fail(ctx, CLAW_EINVAL, "aux: patch %lld %s at cell %lld is %g (must be finite and > 0)",
                  static_cast<long long>(k / (2 * plane)), (k / plane) % 2 ? "K" : "rho",
                  static_cast<long long>(k % plane), aux[k]);
  // (Z, c) per cell, the oracle's operation order: c = sqrt(K / rho), Z = rho c
  std::vector<double> zc(static_cast<size_t>(n));
  std::vector<double> cl(static_cast<size_t>(L.nx * L.ny));   // c on the level index grid
  for (int p = 0; p < L.npatch; ++p) {
    const double* a = aux + static_cast<int64_t>(p) * 2 * plane;
    double* o = zc.data() + static_cast<int64_t>(p) * 2 * plane;
    for (int64_t k = 0; k < plane; ++k) {
      const double c = std::sqrt(a[plane + k] / a[k]);
      o[k] = a[k] * c;
      o[plane + k] = c;
      cl[static_cast<size_t>((L.j0[p] + k / mx) * L.nx + L.i0[p] + k % mx)] = c;
    }
  }
  // per patch: max c over its cells and 1-deep ghost frame (BC-mapped)
  const bool px = ctx->cfg.bc[0] == CLAW_BC_PERIODIC, py = ctx->cfg.bc[2] == CLAW_BC_PERIODIC;
  auto mapi = [](int64_t I, int64_t nn, bool per) { return I < 0 ? (per ? I + nn : 0) : (I >= nn ? (per ? I - nn : nn - 1) : I); };
  L.vc_pcmax.assign(L.owned.size(), 0.0);
  for (size_t lp = 0; lp < L.owned.size(); ++lp) {
    const int p = L.owned[lp];
    double m = 0.0;
    for (int64_t J = L.j0[p] - 1; J <= L.j0[p] + my; ++J)
      for (int64_t I = L.i0[p] - 1; I <= L.i0[p] + mx; ++I)
        m = std::max(m, cl[static_cast<size_t>(mapi(J, L.ny, py) * L.nx + mapi(I, L.nx, px))]);
    L.vc_pcmax[lp] = m;
  }
  // band mode (world > 1): the medium of the four halo rows Y0-2, Y0-1, Y1,
  // Y1+1 (BC-mapped) as [4][2][nx]; the medium is static, so no exchange
  std::vector<double> halo(static_cast<size_t>(8 * L.nx), 1.0);
  for (int kk = 0; kk < 4 && L.band; ++kk) {
    const int64_t J = kk < 2 ? L.Y0 - 2 + kk : L.Y1 + kk - 2;
    const int64_t Jm = mapi(J, L.ny, py);
    for (int64_t I = 0; I < L.nx; ++I) {
      const int64_t pc = I / mx, pr = Jm / my, p = pr * (L.nx / mx) + pc;
      const int64_t k = (Jm - pr * my) * mx + (I - pc * mx);
      halo[static_cast<size_t>((2 * kk) * L.nx + I)] = zc[static_cast<size_t>(p * 2 * plane + k)];
      halo[static_cast<size_t>((2 * kk + 1) * L.nx + I)] = zc[static_cast<size_t>(p * 2 * plane + plane + k)];
    }
  }
  if (!ctx->host_only) {
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    drop_graphs(ctx);
    // the owned patches: whole patch rows, consecutive (grid / band mode)
    const int64_t p0 = L.owned.front(), nown = static_cast<int64_t>(L.owned.size());
    CUDA_TRY(L.aux.alloc(static_cast<size_t>(nown * 2 * plane)));
    CUDA_TRY(cudaMemcpy(L.aux.p, zc.data() + p0 * 2 * plane, static_cast<size_t>(nown * 2 * plane) * 8,
                        cudaMemcpyHostToDevice));
    if (L.band) {
      CUDA_TRY(L.aux_halo.alloc(halo.size()));
      CUDA_TRY(cudaMemcpy(L.aux_halo.p, halo.data(), halo.size() * 8, cudaMemcpyHostToDevice));
    }
  }
  L.vc = true;
  if (L.grid && L.grid_th_base > 0 && !L.sparse) {
    // the vc kernel measured faster with the uncapped makespan rule's taller
    // tiles (c5vc 384 rows: 76.9 G against 75.4 G at 192)
    const int my = L.desc[0].my;
    const int th = makespan_th(claw::grid_nstrip(L.nx), L.Y1 - L.Y0, my,
                               static_cast<int64_t>(ctx->nsm) * claw::grid_resident_warps(), L.grid_th_base, 512);
    if (th != L.grid_th) {
      if (!ctx->host_only) drop_graphs(ctx);
      L.grid_th = th;
      L.ngrid_blocks = th > my ? ((L.Y1 - L.Y0) + th - 1) / th : ((L.Y1 - L.Y0) / my) * ((my + th - 1) / th);
      L.ngrid_tiles = claw::grid_nstrip(L.nx) * L.ngrid_blocks;
    }
  }
  return CLAW_OK;
}

namespace {
// Coarse-to-fine interpolation (R10) of level `level`'s frame cells at
// the times ts[0..nts) into frame slices 0..nts-1, one launch; slice 0 is
// what the next step reads.
int interp_frames(claw_ctx* ctx, int32_t level, const double* ts, int nts) {
  Level& L = ctx->lev[level];
  L.fsel = 0;
  if (!(level > 1 && L.ncoarse > 0)) return CLAW_OK;
  const Level& C = ctx->lev[level - 1];
  const double span = C.t_new - C.t_old;
  const double tol = 1e-12 * std::max(1.0, std::fabs(C.t_new));
  double alpha[claw::kMaxInterpAlphas];
  for (int k = 0; k < nts; ++k) {
    const double t = ts[k];
    if (t < C.t_old - tol || t > C.t_new + tol)
      return fail(ctx, CLAW_ESTATE, "fill_ghost(level %d, t=%.17g): outside level %d's [%.17g, %.17g]", level, t,
                  level - 1, C.t_old, C.t_new);
    alpha[k] = (span > 0) ? (t - C.t_old) / span : 0.0;
  }
  // inside claw_advance_hierarchy's graph path alpha goes through device
  // memory, so a replayed graph interpolates at this step's times
  const double* adev = nullptr;
  if (ctx->in_hier) {
    if (ctx->alpha_n + nts > kMaxAlpha) return fail(ctx, CLAW_EINVAL, "more than %d interpolations per coarse step", kMaxAlpha);
    for (int k = 0; k < nts; ++k) ctx->h_alpha[ctx->alpha_n + k] = alpha[k];
    adev = ctx->d_alpha.p + ctx->alpha_n;
    ctx->alpha_n += nts;
  }
  // C.q[C.cur] holds t_new, the other buffer t_old; DevInterp.dst is a frame
  // offset inside a slice, components are frame_cs apart
  if (!ctx->dry)
    CUDA_TRY(static_cast<cudaError_t>(claw::launch_interp(C.q[1 - C.cur].p, C.q[C.cur].p, alpha, nts, adev,
                                                          L.dinterp.p, L.ncoarse, L.frame.p, L.frame_cs,
                                                          L.frame_elems, ctx->stream)));
  ctx->stats.ghost_launches++;
  return CLAW_OK;
}
}  // namespace

int claw_fill_ghost(claw_ctx* ctx, int32_t level, double t) {
  Nvtx nv_("claw_fill_ghost L%d", level);
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_level(ctx, level)) return rc;
  if (ctx->host_only) return fail(ctx, CLAW_ENODEV, "host-only context");
  Level& L = ctx->lev[level];
  record(ctx, ctx->ev_ghost, true);
  if (int rc = interp_frames(ctx, level, &t, 1)) return rc;
  if (L.dist && ctx->cfg.exchange == 0) {
    // halo on the comm stream: starts when q^n is complete on the main
    // stream; claw_advance_level runs the interior tiles meanwhile and waits
    // for it only before the edge tiles
    const int world = ctx->cfg.world;
    cudaStream_t cst = ctx->comm_stream;
    CUDA_TRY(cudaEventRecord(ctx->ev_ready, ctx->stream));
    CUDA_TRY(cudaStreamWaitEvent(cst, ctx->ev_ready, 0));
    for (int r = 0; r < world; ++r) {
      const int64_t n = static_cast<int64_t>(L.send_off[r].size());
      if (n == 0) continue;
      CUDA_TRY(static_cast<cudaError_t>(claw::launch_pack(L.q[L.cur].p, L.dsend_off[r]->p, L.dsend_cs[r]->p, n,
                                                          L.dsend_buf[r]->p, cst)));
      ctx->stats.ghost_launches++;
    }
    Nvtx nv_halo("claw_halo_exchange");
    ncclResult_t nr = g_nccl.GroupStart();
    if (nr != ncclSuccess) return nccl_fail(ctx, nr, "ncclGroupStart");
    for (int r = 0; r < world; ++r) {
      const size_t ns = L.send_off[r].size();
      if (ns) {
        nr = g_nccl.Send(L.dsend_buf[r]->p, 3 * ns, ncclFloat64, r, ctx->comm, cst);
        if (nr != ncclSuccess) return nccl_fail(ctx, nr, "ncclSend");
        ctx->stats.halo_bytes_sent += static_cast<int64_t>(24 * ns);
      }
      if (L.nrecv[r]) {
        nr = g_nccl.Recv(L.frame.p + L.recv_frame_off[r], 3 * L.nrecv[r], ncclFloat64, r, ctx->comm, cst);
        if (nr != ncclSuccess) return nccl_fail(ctx, nr, "ncclRecv");
      }
    }
    nr = g_nccl.GroupEnd();
    if (nr != ncclSuccess) return nccl_fail(ctx, nr, "ncclGroupEnd");
    CUDA_TRY(cudaEventRecord(ctx->ev_halo, cst));
    L.halo_pending = true;
  }
  record(ctx, ctx->ev_ghost, false);
  return CLAW_OK;
}

int claw_advance_level_async(claw_ctx* ctx, int32_t level, double dt) {
  Nvtx nv_("claw_step L%d", level);
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_level(ctx, level)) return rc;
  if (ctx->host_only) return fail(ctx, CLAW_ENODEV, "host-only context");
  if (!(dt >= 0) || !std::isfinite(dt)) return fail(ctx, CLAW_EINVAL, "dt=%g: must be finite and >= 0", dt);
  if (ctx->stashed) {  // discarded levels are stale once time moves (no kernel reads them)
    for (auto& X : ctx->stash) X = Level();
    ctx->stashed = false;
  }
  Level& L = ctx->lev[level];
  // CFL slots: this step accumulates into lcfl[g] (zeroed by the previous
  // step's kernel, or at set_level) and zeroes lcfl[1-g] for the next step
  const int g = 1 - L.gen;
  claw::StepParams P{};
  P.q = L.q[L.cur].p;
  P.qn = L.q[1 - L.cur].p;
  P.frame = L.frame.p + static_cast<int64_t>(L.fsel) * L.frame_elems;
  P.patches = L.dpatch.p;
  P.rects = L.drect.p;
  P.tiles = L.dtile.p;
  P.cellrect = L.ncellrect > 0 ? L.dcellrect.p : nullptr;
  P.ntiles = static_cast<int32_t>(L.htile.size());
  P.lane_tiles = L.lane_tiles;
  P.limiter = ctx->cfg.limiter;
  P.order_trans = ctx->cfg.order_trans;
  P.dt = dt;
  P.patch_cfl = L.pcfl.p;
  P.level_cfl = L.lcfl.p + g;
  P.level_cfl_reset = L.lcfl.p + (1 - g);
  P.hier_cfl = ctx->hier_slot;
  P.blk_first = 0;
  P.blk_stride = 1;
  P.tile_offset = 0;
  P.uniform = (L.uniform && !L.hpatch.empty()) ? 1 : 0;
  if (P.uniform) fill_step_consts(L.hpatch[0], dt, ctx->cfg.limiter == 4 ? 2.0 : 1.0, ctx->cfg.order_trans, P.k);
  if (L.grid) {
    P.grid = 1;
    P.NX = static_cast<int32_t>(L.nx);
    P.NY = static_cast<int32_t>(L.ny);
    P.mx = L.desc[0].mx;
    P.my = L.desc[0].my;
    P.npx = L.npx;
    P.th = L.grid_th;
    P.per_x = ctx->cfg.bc[0] == CLAW_BC_PERIODIC;
    P.per_y = ctx->cfg.bc[2] == CLAW_BC_PERIODIC;
    P.ntiles = static_cast<int32_t>(L.ngrid_tiles);
    if (L.sparse) {
      P.slots = L.dslots.p;
      P.tiles = L.dgtile.p;
    }
    P.Y0 = static_cast<int32_t>(L.Y0);
    P.Y1 = static_cast<int32_t>(L.Y1);
    P.span = L.grid_th > L.desc[0].my ? 1 : 0;
    P.R0 = P.Y0;
    P.R1 = P.Y1;
    for (int k = 0; k < 4; ++k) {
      P.hoff[k] = L.hoff[k];
      P.hcs[k] = L.hcs[k];
    }
  }
  if (L.vc) {
    P.aux = L.aux.p;
    P.aux_halo = L.aux_halo.p;
    L.last_r = P.k.r;
    L.last_s = P.k.s;
  }
  record(ctx, ctx->ev_step, true);
  if (L.dist) {
    // interior tiles (no remote ghost) first, then -- once the halo has
    // landed -- the edge tiles
    claw::StepParams Pi = P, Pe = P;
    int64_t n_int = 0, n_all = 0;
    if (L.grid && L.band_te > 0) {
      // interior: rows [Y0 + te, Y1 - te); edge: the te rows at each end
      const int64_t nstrip = claw::grid_nstrip(L.nx);
      const int te = L.band_te;
      Pi.span = 1;
      Pi.th = L.grid_th_int;
      Pi.R0 = P.Y0 + te;
      Pi.R1 = P.Y1 - te;
      Pi.ntiles = static_cast<int32_t>(nstrip * L.ngrid_blocks_int);
      Pe.span = 1;
      Pe.th = te;
      Pe.blk_first = 0;
      Pe.blk_stride = (P.Y1 - P.Y0) / te - 1;
      Pe.ntiles = static_cast<int32_t>(nstrip * 2);
      n_int = 1;
      n_all = 1;
    } else if (L.grid) {
      const int64_t nstrip = claw::grid_nstrip(L.nx);
      const int64_t nb = L.ngrid_blocks;
      if (nb >= 3) {
        Pi.blk_first = 1;
        Pi.blk_stride = 1;
        Pi.ntiles = static_cast<int32_t>(nstrip * (nb - 2));
        Pe.blk_first = 0;
        Pe.blk_stride = static_cast<int32_t>(nb - 1);
        Pe.ntiles = static_cast<int32_t>(nstrip * 2);
        n_int = 1;
      }
      n_all = 1;
    } else {
      Pi.tile_offset = 0;
      Pi.ntiles = static_cast<int32_t>(L.ntile_interior);
      Pe.tile_offset = static_cast<int32_t>(L.ntile_interior);
      Pe.ntiles = static_cast<int32_t>(L.htile.size() - L.ntile_interior);
      n_int = L.ntile_interior;
      n_all = 1;
    }
    if (n_int > 0 && Pi.ntiles > 0 && n_all && Pe.ntiles > 0 && !ctx->dry) {
      // the edge tiles on the comm stream, behind the halo there, so they
      // fill the SMs the interior launch's last wave leaves idle; they read
      // q^n and the frame (ready: ev_int, recorded after this level's ghost
      // fill), write cells the interior tiles do not, and max into the same
      // CFL slot; the library stream waits for them before anything else
      Pe.level_cfl_reset = nullptr;  // reset once (by the interior launch)
      CUDA_TRY(cudaEventRecord(ctx->ev_int, ctx->stream));
      CUDA_TRY(static_cast<cudaError_t>(claw::launch_step(Pi, ctx->stream)));
      CUDA_TRY(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_int, 0));
      CUDA_TRY(static_cast<cudaError_t>(claw::launch_step(Pe, ctx->comm_stream)));
      CUDA_TRY(cudaEventRecord(ctx->ev_edge, ctx->comm_stream));
      CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->ev_edge, 0));
      L.halo_pending = false;
      ctx->stats.step_launches += 2;
    } else {
      if (n_int > 0 && Pi.ntiles > 0) {
        Pe.level_cfl_reset = nullptr;  // reset once (by the interior launch)
        if (!ctx->dry) CUDA_TRY(static_cast<cudaError_t>(claw::launch_step(Pi, ctx->stream)));
        ctx->stats.step_launches++;
      } else {
        Pe = P;                        // no split: one launch after the halo
      }
      if (L.halo_pending) {
        CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->ev_halo, 0));
        L.halo_pending = false;
      }
      if (n_all && Pe.ntiles > 0) {
        if (!ctx->dry) CUDA_TRY(static_cast<cudaError_t>(claw::launch_step(Pe, ctx->stream)));
        ctx->stats.step_launches++;
      }
    }
  } else {
    P.side = L.use_side ? L.side.p : nullptr;
    if (!ctx->dry) CUDA_TRY(static_cast<cudaError_t>(claw::launch_step(P, ctx->stream)));
    ctx->stats.step_launches++;
    if (P.side) ctx->stats.ghost_launches++;  // the side_kernel ahead of it
  }
  record(ctx, ctx->ev_step, false);
  if (ctx->cfg.check_finite && !ctx->dry)  // debug check: every new value finite
    CUDA_TRY(static_cast<cudaError_t>(claw::launch_nonfinite(P.qn, L.buf_elems, level, ctx->nf_flag.p, ctx->stream)));
  ctx->stats.cells_advanced += L.cells_owned;
  if (ctx->cfg.reflux) {
    // conservation fix: fine part of this level's registers (q^n of this level
    // and of level-1, which advanced first), coarse part of level+1's
    if (level > 1 && !L.hreg.empty()) {
      const Level& C = ctx->lev[level - 1];
      if (!ctx->dry) CUDA_TRY(static_cast<cudaError_t>(claw::launch_reflux(1, P, C.q[1 - C.cur].p, C.dpatch.p, L.dreg.p,
                                                            static_cast<int64_t>(L.hreg.size()), L.ratio, L.racc.p,
                                                            ctx->stream)));
      ctx->stats.ghost_launches++;
    }
    if (level < kMaxLevel && ctx->lev[level + 1].set && !ctx->lev[level + 1].hreg.empty()) {
      Level& F = ctx->lev[level + 1];
      if (!ctx->dry) CUDA_TRY(static_cast<cudaError_t>(claw::launch_reflux(0, P, nullptr, nullptr, F.dreg.p,
                                                            static_cast<int64_t>(F.hreg.size()), F.ratio, F.racc.p,
                                                            ctx->stream)));
      ctx->stats.ghost_launches++;
    }
  }
  // the level's CFL all-reduce; inside a hierarchy call the step's Courant
  // number also lands in the hierarchy slot, reduced once for the whole call
  // (one all-reduce per claw_advance_hierarchy[_n] instead of one per level
  // step, which nothing overlaps), so the level slot stays rank-local there
  if (L.dist && ctx->cfg.exchange == 0 && !ctx->hier_slot) {
    Nvtx nv_red("claw_cfl_allreduce");
    ncclResult_t nr = g_nccl.AllReduce(L.lcfl.p + g, L.lcfl.p + g, 1, ncclFloat64, ncclMax, ctx->comm, ctx->stream);
    if (nr != ncclSuccess) return nccl_fail(ctx, nr, "ncclAllReduce(cfl, max)");
  }
  L.gen = g;
  L.cur = 1 - L.cur;
  L.t_old = L.t_new;
  L.t_new = L.t_new + dt;
  return CLAW_OK;
}

int claw_wait_cfl(claw_ctx* ctx, int32_t level, double* cfl_max) {
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_level(ctx, level)) return rc;
  if (ctx->host_only) return fail(ctx, CLAW_ENODEV, "host-only context");
  if (!cfl_max) return fail(ctx, CLAW_EINVAL, "cfl_max is NULL");
  Level& L = ctx->lev[level];
  CUDA_TRY(cudaMemcpyAsync(ctx->h_cfl, L.lcfl.p + L.gen, 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (ctx->cfg.check_finite)
    CUDA_TRY(cudaMemcpyAsync(ctx->h_nf, ctx->nf_flag.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  *cfl_max = *ctx->h_cfl;
  return take_nonfinite(ctx);
}

int claw_advance_level(claw_ctx* ctx, int32_t level, double dt, double* cfl_max) {
  if (!cfl_max) return fail(ctx, CLAW_EINVAL, "cfl_max is NULL");
  if (int rc = claw_advance_level_async(ctx, level, dt)) return rc;
  return claw_wait_cfl(ctx, level, cfl_max);
}

static int owned_index(claw_ctx* ctx, int level, int patch, int* lp) {
  if (int rc = check_level(ctx, level)) return rc;
  const Level& L = ctx->lev[level];
  if (patch < 0 || patch >= L.npatch) return fail(ctx, CLAW_EINVAL, "patch %d out of range", patch);
  if (L.local[patch] < 0) return fail(ctx, CLAW_EINVAL, "patch %d is owned by rank %d", patch, L.owner[patch]);
  *lp = L.local[patch];
  return CLAW_OK;
}

int claw_read(claw_ctx* ctx, int32_t level, int32_t patch, double* q_out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (ctx->host_only) return fail(ctx, CLAW_ENODEV, "host-only context");
  int lp;
  if (int rc = owned_index(ctx, level, patch, &lp)) return rc;
  if (!q_out) return fail(ctx, CLAW_EINVAL, "q_out is NULL");
  Level& L = ctx->lev[level];
  const int64_t n = 3ll * L.hpatch[lp].mx * L.hpatch[lp].my;
  CUDA_TRY(cudaMemcpyAsync(q_out, L.q[L.cur].p + L.off[lp], n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return CLAW_OK;
}

int claw_write(claw_ctx* ctx, int32_t level, int32_t patch, const double* q_in) {
  if (int rc = check_ctx(ctx)) return rc;
  if (ctx->host_only) return fail(ctx, CLAW_ENODEV, "host-only context");
  int lp;
  if (int rc = owned_index(ctx, level, patch, &lp)) return rc;
  if (!q_in) return fail(ctx, CLAW_EINVAL, "q_in is NULL");
  Level& L = ctx->lev[level];
  const int64_t n = 3ll * L.hpatch[lp].mx * L.hpatch[lp].my;
  CUDA_TRY(cudaMemcpyAsync(L.q[L.cur].p + L.off[lp], q_in, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return CLAW_OK;
}

int claw_read_level(claw_ctx* ctx, int32_t level, double* q_out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_level(ctx, level)) return rc;
  if (ctx->host_only) return fail(ctx, CLAW_ENODEV, "host-only context");
  if (!q_out) return fail(ctx, CLAW_EINVAL, "q_out is NULL");
  Level& L = ctx->lev[level];
  if (L.gapless) {
    CUDA_TRY(cudaMemcpyAsync(q_out, L.q[L.cur].p, L.buf_elems * 8, cudaMemcpyDeviceToHost, ctx->stream));
  } else {
    int64_t dst = 0;
    for (size_t lp = 0; lp < L.owned.size(); ++lp) {
      const int64_t n = 3ll * L.hpatch[lp].mx * L.hpatch[lp].my;
      CUDA_TRY(cudaMemcpyAsync(q_out + dst, L.q[L.cur].p + L.off[lp], n * 8, cudaMemcpyDeviceToHost, ctx->stream));
      dst += n;
    }
  }
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return CLAW_OK;
}

int claw_write_level(claw_ctx* ctx, int32_t level, const double* q_in) {
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_level(ctx, level)) return rc;
  if (ctx->host_only) return fail(ctx, CLAW_ENODEV, "host-only context");
  if (!q_in) return fail(ctx, CLAW_EINVAL, "q_in is NULL");
  Level& L = ctx->lev[level];
  if (L.gapless) {
    CUDA_TRY(cudaMemcpyAsync(L.q[L.cur].p, q_in, L.buf_elems * 8, cudaMemcpyHostToDevice, ctx->stream));
  } else {
    int64_t src = 0;
    for (size_t lp = 0; lp < L.owned.size(); ++lp) {
      const int64_t n = 3ll * L.hpatch[lp].mx * L.hpatch[lp].my;
      CUDA_TRY(cudaMemcpyAsync(L.q[L.cur].p + L.off[lp], q_in + src, n * 8, cudaMemcpyHostToDevice, ctx->stream));
      src += n;
    }
  }
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return CLAW_OK;
}

int claw_read_padded(claw_ctx* ctx, int32_t level, int32_t patch, double* q_out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (ctx->host_only) return fail(ctx, CLAW_ENODEV, "host-only context");
  int lp;
  if (int rc = owned_index(ctx, level, patch, &lp)) return rc;
  if (!q_out) return fail(ctx, CLAW_EINVAL, "q_out is NULL");
  Level& L = ctx->lev[level];
  const int64_t n = 3ll * (L.hpatch[lp].mx + 4) * (L.hpatch[lp].my + 4);
  DevBuf<double> tmp;
  CUDA_TRY(tmp.alloc(n));
  CUDA_TRY(static_cast<cudaError_t>(claw::launch_gather_padded(L.q[L.cur].p, L.frame.p + static_cast<int64_t>(L.fsel) * L.frame_elems, L.dpatch.p, L.drect.p, lp,
                                                               tmp.p, ctx->stream)));
  CUDA_TRY(cudaMemcpyAsync(q_out, tmp.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return CLAW_OK;
}

int claw_patch_cfl(claw_ctx* ctx, int32_t level, int32_t patch, double* cfl) {
  if (int rc = check_ctx(ctx)) return rc;
  if (ctx->host_only) return fail(ctx, CLAW_ENODEV, "host-only context");
  int lp;
  if (int rc = owned_index(ctx, level, patch, &lp)) return rc;
  if (!cfl) return fail(ctx, CLAW_EINVAL, "cfl is NULL");
  const Level& Lv = ctx->lev[level];
  if (Lv.vc) {
    // variable media: max over the patch's faces of max(c_l, c_r) dt/dx (dt/dy)
    // = max(dt/dx, dt/dy) times the max c over the cells those faces touch
    // (its cells and 1-deep ghost frame); the medium is static
    const double m = Lv.vc_pcmax[static_cast<size_t>(lp)];
    *cfl = std::max(Lv.last_r * m, Lv.last_s * m);
    return CLAW_OK;
  }
  unsigned long long bits = 0;
  // grid mode: every patch shares dt, dx, dy and c, so its max Courant number
  // is the level's (the grid kernel only maintains the level slot)
  const unsigned long long* src =
      ctx->lev[level].grid ? ctx->lev[level].lcfl.p + ctx->lev[level].gen : ctx->lev[level].pcfl.p + lp;
  CUDA_TRY(cudaMemcpyAsync(ctx->h_cfl, src, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  std::memcpy(&bits, ctx->h_cfl, 8);
  std::memcpy(cfl, &bits, 8);
  return CLAW_OK;
}

int claw_owner(const claw_ctx* ctx, int32_t level, int32_t patch, int32_t* rank) {
  if (!ctx || !rank || level < 1 || level > kMaxLevel || !ctx->lev[level].set) return CLAW_EINVAL;
  const Level& L = ctx->lev[level];
  if (patch < 0 || patch >= L.npatch) return CLAW_EINVAL;
  *rank = L.owner[patch];
  return CLAW_OK;
}

int claw_level_mode(const claw_ctx* ctx, int32_t level, int32_t* mode) {
  if (!ctx || !mode || level < 1 || level > kMaxLevel || !ctx->lev[level].set) return CLAW_EINVAL;
  *mode = ctx->lev[level].grid ? (ctx->lev[level].sparse ? 2 : 1) : 0;
  return CLAW_OK;
}

int claw_update_level(claw_ctx* ctx, int32_t level) {
  Nvtx nv_("claw_update L%d", level);
  if (int rc = check_ctx(ctx)) return rc;
  if (level < 2 || level > kMaxLevel || !ctx->lev[level].set || !ctx->lev[level - 1].set)
    return fail(ctx, CLAW_ESTATE, "update needs level %d and level %d set", level, level - 1);
  if (ctx->host_only) return fail(ctx, CLAW_ENODEV, "host-only context");
  Level& F = ctx->lev[level];
  Level& C = ctx->lev[level - 1];
  if (C.dist) return fail(ctx, CLAW_EINVAL, "update: level %d is partitioned across ranks", level - 1);
  if (std::fabs(F.t_new - C.t_new) > 1e-12 * std::max(1.0, std::fabs(C.t_new)))
    return fail(ctx, CLAW_ESTATE, "update: level %d (t=%.17g) has not caught up with level %d (t=%.17g)", level,
                F.t_new, level - 1, C.t_new);
  const int64_t n = static_cast<int64_t>(F.hu.size());
  if (!ctx->dry) CUDA_TRY(static_cast<cudaError_t>(claw::launch_update_rects(C.q[C.cur].p, F.q[F.cur].p, F.dur.p,
                                                              F.dur_chunk.p,
                                                              static_cast<int32_t>(F.hur_chunk.size()), F.ratio,
                                                              ctx->stream)));
  if (!ctx->dry) CUDA_TRY(static_cast<cudaError_t>(claw::launch_update(C.q[C.cur].p, F.q[F.cur].p, F.du.p, n, F.ratio,
                                                        F.du_src.p, F.du_scs.p, ctx->stream)));
  ctx->stats.ghost_launches += (F.hur.empty() ? 0 : 1) + (n > 0 ? 1 : 0);
  if (F.dist && ctx->cfg.exchange == 0 && !ctx->dry) {
    // the replicated coarse level takes every rank's averages: each rank
    // sends the cells its patches averaged to every peer, receives theirs,
    // and writes them into its replica (grouped NCCL send/recv)
    Nvtx nv_x("claw_update_exchange");
    const int world = ctx->cfg.world, me = ctx->cfg.rank;
    const int64_t ns = static_cast<int64_t>(F.upd_send_off.size());
    if (ns)
      CUDA_TRY(static_cast<cudaError_t>(claw::launch_pack(C.q[C.cur].p, F.dupd_send_off.p, F.dupd_send_cs.p, ns,
                                                          F.dupd_send_buf.p, ctx->stream)));
    ncclResult_t nr = g_nccl.GroupStart();
    if (nr != ncclSuccess) return nccl_fail(ctx, nr, "ncclGroupStart");
    for (int r = 0; r < world; ++r) {
      if (r == me) continue;
      if (ns) {
        nr = g_nccl.Send(F.dupd_send_buf.p, 3 * ns, ncclFloat64, r, ctx->comm, ctx->stream);
        if (nr != ncclSuccess) return nccl_fail(ctx, nr, "ncclSend");
      }
      const size_t nrv = F.upd_recv_off[r].size();
      if (nrv) {
        nr = g_nccl.Recv(F.dupd_recv_buf[r]->p, 3 * nrv, ncclFloat64, r, ctx->comm, ctx->stream);
        if (nr != ncclSuccess) return nccl_fail(ctx, nr, "ncclRecv");
      }
    }
    nr = g_nccl.GroupEnd();
    if (nr != ncclSuccess) return nccl_fail(ctx, nr, "ncclGroupEnd");
    for (int r = 0; r < world; ++r) {
      const int64_t nrv = static_cast<int64_t>(F.upd_recv_off[r].size());
      if (r != me && nrv)
        CUDA_TRY(static_cast<cudaError_t>(claw::launch_scatter(F.dupd_recv_buf[r]->p, F.dupd_recv_off[r]->p,
                                                               F.dupd_recv_cs[r]->p, nrv, C.q[C.cur].p,
                                                               ctx->stream)));
    }
    ctx->stats.ghost_launches += 1 + (world - 1);
  }
  if (ctx->cfg.reflux && !F.hreg.empty()) {
    if (!ctx->dry) CUDA_TRY(static_cast<cudaError_t>(claw::launch_reflux_apply(C.q[C.cur].p, C.dpatch.p, F.dreg.p, F.dheads.p,
                                                                static_cast<int64_t>(F.hheads.size()) - 1, F.racc.p,
                                                                ctx->stream)));
    ctx->stats.ghost_launches++;
  }
  return CLAW_OK;
}

int claw_reflux_registers(claw_ctx* ctx, int32_t level, int64_t* n, int32_t* edges, double* acc) {
  if (int rc = check_ctx(ctx)) return rc;
  if (level < 2 || level > kMaxLevel || !ctx->lev[level].set) return fail(ctx, CLAW_ESTATE, "level %d is not set", level);
  if (!n) return fail(ctx, CLAW_EINVAL, "n is NULL");
  const Level& F = ctx->lev[level];
  const Level& C = ctx->lev[level - 1];
  *n = static_cast<int64_t>(F.hreg.size());
  if (edges)
    for (size_t e = 0; e < F.hreg.size(); ++e) {
      const claw::DevReflux& r = F.hreg[e];
      int32_t* o = edges + 8 * e;
      o[0] = C.owned[r.cp];
      o[1] = r.ci;
      o[2] = r.cj;
      o[3] = r.ds & 1;
      o[4] = r.ds >> 1;
      o[5] = F.owned[r.fp];
      o[6] = r.fi;
      o[7] = r.fj;
    }
  if (acc && !F.hreg.empty()) {
    if (ctx->host_only) return fail(ctx, CLAW_ENODEV, "host-only context");
    CUDA_TRY(cudaMemcpyAsync(acc, F.racc.p, 3 * F.hreg.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  }
  return CLAW_OK;
}

// Recursive subcycled advance without host synchronisation; every
// step kernel also folds its Courant number into the coarse-step slot.
// sub_ts / sub_k / sub_n: this level is substep sub_k of sub_n at the times
// sub_ts (set by the parent); a level with that many frame slices gets the
// coarse ghost values of all its substeps from one interpolation launch at
// substep 0, and later substeps only select their slice
static int advance_rec(claw_ctx* ctx, int level, double t, double dt, int nlev, int flags,
                       const double* sub_ts = nullptr, int sub_k = 0, int sub_n = 1) {
  Level& L = ctx->lev[level];
  if (sub_ts && sub_n > 1 && L.nslice >= sub_n && L.ncoarse > 0) {
    if (sub_k == 0) {
      if (int rc = check_ctx(ctx)) return rc;
      record(ctx, ctx->ev_ghost, true);
      if (int rc = interp_frames(ctx, level, sub_ts, sub_n)) return rc;
      record(ctx, ctx->ev_ghost, false);
    }
    L.fsel = sub_k;
  } else {
    if (int rc = claw_fill_ghost(ctx, level, t)) return rc;
  }
  if (int rc = claw_advance_level_async(ctx, level, dt)) return rc;
  if (level < nlev) {
    const int R = ctx->lev[level + 1].ratio;
    const double dtf = dt / R;
    double ts[claw::kMaxInterpAlphas];
    const bool multi = R <= claw::kMaxInterpAlphas;
    for (int k = 0; k < R && multi; ++k) ts[k] = t + k * dtf;
    for (int k = 0; k < R; ++k)
      if (int rc = advance_rec(ctx, level + 1, t + k * dtf, dtf, nlev, flags, multi ? ts : nullptr, k, R)) return rc;
    if (flags & CLAW_HIER_UPDATE)
      if (int rc = claw_update_level(ctx, level + 1)) return rc;
  }
  return CLAW_OK;
}

int claw_advance_hierarchy(claw_ctx* ctx, double t, double dt, int32_t flags, double* cfl_max) {
  Nvtx nv_("claw_advance_hierarchy");
  if (int rc = check_ctx(ctx)) return rc;
  if (ctx->host_only) return fail(ctx, CLAW_ENODEV, "host-only context");
  if (!cfl_max) return fail(ctx, CLAW_EINVAL, "cfl_max is NULL");
  int nlev = 0;
  while (nlev < kMaxLevel && ctx->lev[nlev + 1].set) ++nlev;
  if (nlev == 0) return fail(ctx, CLAW_ESTATE, "no level set");
  if (!ctx->hier_buf.p) CUDA_TRY(ctx->hier_buf.alloc(1));
  const bool graph = ctx->graphs_on && ctx->cfg.world == 1 && !ctx->cfg.check_finite;
  if (!graph) {
    CUDA_TRY(cudaMemsetAsync(ctx->hier_buf.p, 0, 8, ctx->stream));
    ctx->hier_slot = ctx->hier_buf.p;
    const int rc = advance_rec(ctx, 1, t, dt, nlev, flags);
    ctx->hier_slot = nullptr;
    if (rc) return rc;
    if (ctx->cfg.world > 1 && ctx->cfg.exchange == 0) {
      ncclResult_t nr = g_nccl.AllReduce(ctx->hier_buf.p, ctx->hier_buf.p, 1, ncclFloat64, ncclMax, ctx->comm,
                                         ctx->stream);
      if (nr != ncclSuccess) return nccl_fail(ctx, nr, "ncclAllReduce(cfl, max)");
    }
    CUDA_TRY(cudaMemcpyAsync(ctx->h_cfl, ctx->hier_buf.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (ctx->cfg.check_finite)
      CUDA_TRY(cudaMemcpyAsync(ctx->h_nf, ctx->nf_flag.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    *cfl_max = *ctx->h_cfl;
    return take_nonfinite(ctx);
  }
  // CUDA-graph path: the whole coarse step -- every fill,
  // step, reflux and update launch -- is captured once per key and replayed;
  // the host only redoes its bookkeeping (times, buffer parity) and the
  // interpolation weights, which reach the graph through pinned memory.
  if (!ctx->h_alpha) {
    CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_alpha), kMaxAlpha * sizeof(double)));
    CUDA_TRY(ctx->d_alpha.alloc(kMaxAlpha));
  }
  std::vector<uint64_t> key = {ctx->epoch, 0, static_cast<uint64_t>(flags), ctx->profiling ? 1u : 0u,
                               static_cast<uint64_t>(nlev)};
  std::memcpy(&key[1], &dt, 8);
  for (int l = 1; l <= nlev; ++l) key.push_back(static_cast<uint64_t>(ctx->lev[l].cur | (ctx->lev[l].gen << 1)));
  HierGraph* hg = nullptr;
  for (HierGraph& g : ctx->graphs)
    if (g.key == key) hg = &g;
  ctx->in_hier = true;
  ctx->alpha_n = 0;
  ctx->hier_slot = ctx->hier_buf.p;
  int rc = CLAW_OK;
  if (hg) {
    ctx->dry = true;
    rc = advance_rec(ctx, 1, t, dt, nlev, flags);
    ctx->dry = false;
    if (!rc) {
      cudaError_t e = cudaGraphLaunch(hg->exec, ctx->stream);
      if (e != cudaSuccess) rc = cuda_fail(ctx, e, "cudaGraphLaunch");
    }
  } else {
    const size_t s0 = ctx->ev_step.size(), g0 = ctx->ev_ghost.size();
    cudaError_t e = cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) rc = cuda_fail(ctx, e, "cudaStreamBeginCapture");
    if (!rc) {
      ctx->capturing = true;
      cudaMemcpyAsync(ctx->d_alpha.p, ctx->h_alpha, kMaxAlpha * sizeof(double), cudaMemcpyHostToDevice, ctx->stream);
      cudaMemsetAsync(ctx->hier_buf.p, 0, 8, ctx->stream);
      rc = advance_rec(ctx, 1, t, dt, nlev, flags);
      cudaMemcpyAsync(ctx->h_cfl, ctx->hier_buf.p, 8, cudaMemcpyDeviceToHost, ctx->stream);
      ctx->capturing = false;
      cudaGraph_t gr = nullptr;
      e = cudaStreamEndCapture(ctx->stream, &gr);
      if (!rc && e != cudaSuccess) rc = cuda_fail(ctx, e, "cudaStreamEndCapture");
      if (!rc) {
        HierGraph ng;
        ng.key = key;
        e = cudaGraphInstantiate(&ng.exec, gr, 0);
        if (e != cudaSuccess) rc = cuda_fail(ctx, e, "cudaGraphInstantiate");
        ng.ev_step.assign(ctx->ev_step.begin() + s0, ctx->ev_step.end());
        ng.ev_ghost.assign(ctx->ev_ghost.begin() + g0, ctx->ev_ghost.end());
        ctx->ev_step.resize(s0);
        ctx->ev_ghost.resize(g0);
        if (!rc) {
          ctx->graphs.push_back(std::move(ng));
          hg = &ctx->graphs.back();
          e = cudaGraphLaunch(hg->exec, ctx->stream);
          if (e != cudaSuccess) rc = cuda_fail(ctx, e, "cudaGraphLaunch");
        }
      }
      if (gr) cudaGraphDestroy(gr);
    }
  }
  ctx->in_hier = false;
  ctx->hier_slot = nullptr;
  if (rc) return rc;
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  *cfl_max = *ctx->h_cfl;
  if (ctx->profiling) {  // this replay's timing nodes
    for (auto& p : hg->ev_step) {
      float ms = 0;
      cudaEventElapsedTime(&ms, p.first, p.second);
      ctx->stats.step_ms += ms;
    }
    for (auto& p : hg->ev_ghost) {
      float ms = 0;
      cudaEventElapsedTime(&ms, p.first, p.second);
      ctx->stats.ghost_ms += ms;
    }
  }
  return CLAW_OK;
}

int claw_advance_hierarchy_n(claw_ctx* ctx, double t, double dt, int32_t nsteps, int32_t flags, double* cfl_out) {
  Nvtx nv_("claw_advance_hierarchy_n %d", nsteps);
  if (int rc = check_ctx(ctx)) return rc;
  if (ctx->host_only) return fail(ctx, CLAW_ENODEV, "host-only context");
  if (nsteps < 1 || !cfl_out) return fail(ctx, CLAW_EINVAL, "nsteps=%d, cfl_out=%p", nsteps, static_cast<void*>(cfl_out));
  int nlev = 0;
  while (nlev < kMaxLevel && ctx->lev[nlev + 1].set) ++nlev;
  if (nlev == 0) return fail(ctx, CLAW_ESTATE, "no level set");
  // one CFL slot per coarse step, zeroed by one memset for the batch; the
  // launches of all nsteps coarse steps are queued back to back on the
  // stream (the host runs ahead of the GPU), one synchronisation at the end
  if (ctx->hier_many.n < static_cast<size_t>(nsteps)) CUDA_TRY(ctx->hier_many.alloc(static_cast<size_t>(nsteps)));
  if (ctx->h_many_n < nsteps) {
    if (ctx->h_many) cudaFreeHost(ctx->h_many);
    ctx->h_many = nullptr;
    CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_many), static_cast<size_t>(nsteps) * sizeof(double)));
    ctx->h_many_n = nsteps;
  }
  CUDA_TRY(cudaMemsetAsync(ctx->hier_many.p, 0, static_cast<size_t>(nsteps) * 8, ctx->stream));
  for (int k = 0; k < nsteps; ++k) {
    ctx->hier_slot = ctx->hier_many.p + k;
    const int rc = advance_rec(ctx, 1, t + k * dt, dt, nlev, flags);
    ctx->hier_slot = nullptr;
    if (rc) return rc;
  }
  if (ctx->cfg.world > 1 && ctx->cfg.exchange == 0) {
    ncclResult_t nr = g_nccl.AllReduce(ctx->hier_many.p, ctx->hier_many.p, static_cast<size_t>(nsteps), ncclFloat64,
                                       ncclMax, ctx->comm, ctx->stream);
    if (nr != ncclSuccess) return nccl_fail(ctx, nr, "ncclAllReduce(cfl, max)");
  }
  CUDA_TRY(cudaMemcpyAsync(ctx->h_many, ctx->hier_many.p, static_cast<size_t>(nsteps) * 8, cudaMemcpyDeviceToHost,
                           ctx->stream));
  if (ctx->cfg.check_finite)
    CUDA_TRY(cudaMemcpyAsync(ctx->h_nf, ctx->nf_flag.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  std::memcpy(cfl_out, ctx->h_many, static_cast<size_t>(nsteps) * sizeof(double));
  return take_nonfinite(ctx);
}

int claw_level_owned(const claw_ctx* ctx, int32_t level, int32_t* npatch_owned, int64_t* cells_owned,
                     int64_t* device_bytes) {
  if (!ctx || level < 1 || level > kMaxLevel || !ctx->lev[level].set) return CLAW_EINVAL;
  const Level& L = ctx->lev[level];
  if (npatch_owned) *npatch_owned = static_cast<int32_t>(L.owned.size());
  if (cells_owned) *cells_owned = L.cells_owned;
  if (device_bytes) *device_bytes = L.device_bytes;
  return CLAW_OK;
}

int claw_debug_ghost_sources(const claw_ctx* ctx, int32_t level, int32_t patch, int64_t* out, int64_t* out2) {
  if (!ctx || !out || level < 1 || level > kMaxLevel || !ctx->lev[level].set) return CLAW_EINVAL;
  const Level& L = ctx->lev[level];
  if (patch < 0 || patch >= L.npatch || L.local[patch] < 0) return CLAW_EINVAL;
  const auto& v = L.dbg_src[L.local[patch]];
  const auto& w = L.dbg_remote[L.local[patch]];
  const int mx = L.desc[patch].mx, my = L.desc[patch].my, PX = mx + 4;
  for (int j = -2; j <= my + 1; ++j)
    for (int i = -2; i <= mx + 1; ++i) {
      const int64_t o = static_cast<int64_t>(j + 2) * PX + (i + 2);
      const bool interior = i >= 0 && i < mx && j >= 0 && j < my;
      const int64_t f = interior ? -1 : frame_index(i, j, mx, my);
      out[o] = interior ? (static_cast<int64_t>(patch) << 32) | (static_cast<int64_t>(j) << 16) | i : v[f];
      if (out2) out2[o] = interior ? 0 : w[f];
    }
  return CLAW_OK;
}

int claw_halo_pack(claw_ctx* ctx, int32_t level, int32_t peer, double* host_out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_level(ctx, level)) return rc;
  if (ctx->host_only) return fail(ctx, CLAW_ENODEV, "host-only context");
  if (peer < 0 || peer >= ctx->cfg.world || !host_out) return fail(ctx, CLAW_EINVAL, "bad peer or buffer");
  Level& L = ctx->lev[level];
  if (!L.dist) return CLAW_OK;   // (a replicated level has no halo)
  const int64_t n = static_cast<int64_t>(L.send_off[peer].size());
  if (n == 0) return CLAW_OK;
  CUDA_TRY(static_cast<cudaError_t>(claw::launch_pack(L.q[L.cur].p, L.dsend_off[peer]->p, L.dsend_cs[peer]->p, n,
                                                      L.dsend_buf[peer]->p, ctx->stream)));
  CUDA_TRY(cudaMemcpyAsync(host_out, L.dsend_buf[peer]->p, 3 * n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return CLAW_OK;
}

int claw_halo_unpack(claw_ctx* ctx, int32_t level, int32_t peer, const double* host_in) {
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_level(ctx, level)) return rc;
  if (ctx->host_only) return fail(ctx, CLAW_ENODEV, "host-only context");
  if (peer < 0 || peer >= ctx->cfg.world || !host_in) return fail(ctx, CLAW_EINVAL, "bad peer or buffer");
  Level& L = ctx->lev[level];
  if (!L.dist) return CLAW_OK;
  const int64_t n = L.nrecv[peer];
  if (n == 0) return CLAW_OK;
  CUDA_TRY(cudaMemcpyAsync(L.frame.p + L.recv_frame_off[peer], host_in, 3 * n * 8, cudaMemcpyHostToDevice,
                           ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return CLAW_OK;
}

int claw_debug_halo_counts(const claw_ctx* ctx, int32_t level, int32_t peer, int64_t* nsend, int64_t* nrecv) {
  if (!ctx || level < 1 || level > kMaxLevel || !ctx->lev[level].set) return CLAW_EINVAL;
  const Level& L = ctx->lev[level];
  if (peer < 0 || peer >= ctx->cfg.world) return CLAW_EINVAL;
  if (nsend) *nsend = L.dist ? static_cast<int64_t>(L.send_off[peer].size()) : 0;
  if (nrecv) *nrecv = L.dist ? L.nrecv[peer] : 0;
  return CLAW_OK;
}

int claw_update_pack(claw_ctx* ctx, int32_t level, double* host_out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_level(ctx, level)) return rc;
  if (ctx->host_only) return fail(ctx, CLAW_ENODEV, "host-only context");
  if (level < 2 || !ctx->lev[level].dist || !host_out)
    return fail(ctx, CLAW_EINVAL, "update_pack: level %d is not the partitioned level, or no buffer", level);
  Level& F = ctx->lev[level];
  Level& C = ctx->lev[level - 1];
  const int64_t n = static_cast<int64_t>(F.upd_send_off.size());
  if (n == 0) return CLAW_OK;
  CUDA_TRY(static_cast<cudaError_t>(claw::launch_pack(C.q[C.cur].p, F.dupd_send_off.p, F.dupd_send_cs.p, n,
                                                      F.dupd_send_buf.p, ctx->stream)));
  CUDA_TRY(cudaMemcpyAsync(host_out, F.dupd_send_buf.p, 3 * n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return CLAW_OK;
}

int claw_update_unpack(claw_ctx* ctx, int32_t level, int32_t peer, const double* host_in) {
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_level(ctx, level)) return rc;
  if (ctx->host_only) return fail(ctx, CLAW_ENODEV, "host-only context");
  if (level < 2 || !ctx->lev[level].dist || peer < 0 || peer >= ctx->cfg.world || peer == ctx->cfg.rank ||
      !host_in)
    return fail(ctx, CLAW_EINVAL, "update_unpack: level %d / peer %d / buffer", level, peer);
  Level& F = ctx->lev[level];
  Level& C = ctx->lev[level - 1];
  const int64_t n = static_cast<int64_t>(F.upd_recv_off[peer].size());
  if (n == 0) return CLAW_OK;
  CUDA_TRY(cudaMemcpyAsync(F.dupd_recv_buf[peer]->p, host_in, 3 * n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CUDA_TRY(static_cast<cudaError_t>(claw::launch_scatter(F.dupd_recv_buf[peer]->p, F.dupd_recv_off[peer]->p,
                                                         F.dupd_recv_cs[peer]->p, n, C.q[C.cur].p, ctx->stream)));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return CLAW_OK;
}

int claw_debug_update_counts(const claw_ctx* ctx, int32_t level, int32_t peer, int64_t* nsend, int64_t* nrecv) {
  if (!ctx || level < 2 || level > kMaxLevel || !ctx->lev[level].set) return CLAW_EINVAL;
  const Level& F = ctx->lev[level];
  if (peer < 0 || peer >= ctx->cfg.world) return CLAW_EINVAL;
  if (nsend) *nsend = F.dist ? static_cast<int64_t>(F.upd_send_off.size()) : 0;
  if (nrecv) *nrecv = (F.dist && peer != ctx->cfg.rank) ? static_cast<int64_t>(F.upd_recv_off[peer].size()) : 0;
  return CLAW_OK;
}

int claw_debug_halo_send(const claw_ctx* ctx, int32_t level, int32_t peer, int64_t k, int32_t* patch, int32_t* i,
                         int32_t* j) {
  if (!ctx || level < 1 || level > kMaxLevel || !ctx->lev[level].set) return CLAW_EINVAL;
  const Level& L = ctx->lev[level];
  if (peer < 0 || peer >= ctx->cfg.world || k < 0 || k >= static_cast<int64_t>(L.send_dbg[peer].size()))
    return CLAW_EINVAL;
  const int64_t code = L.send_dbg[peer][k];
  if (patch) *patch = static_cast<int32_t>(code >> 32);
  if (j) *j = static_cast<int32_t>((code >> 16) & 0xffff);
  if (i) *i = static_cast<int32_t>(code & 0xffff);
  return CLAW_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Regridding (NEXT-3; "every K time steps ... cells are flagged
// ... clustered into new rectangular grid patches"; DESIGN.md
// R18).  Flagging and the new level's data stay on the device; only the flag
// map crosses to the host for clustering, as in the paper (the CPU owns the
// patch structure).
// ---------------------------------------------------------------------------
namespace {

// Berger-Rigoutsos box splitter over a summed-area table (each box costs
// O(w + h) instead of O(w h)).  Rules (R18): shrink to the flags'
// bounding box; accept if efficiency >= cutoff and both sides <= max_dim;
// else cut at (a) the hole of the signature closest to the centre (longer
// side first), (b) the strongest sign change of the signature's second
// difference (largest |jump|, then closest to the centre, longer side first),
// (c) the middle of the longer side -- every cut leaving >= min_dim on both
// sides; no admissible cut: accept.  Low part before high part.
struct Clusterer {
  int64_t nx, ny;
  std::vector<int32_t> own;
  std::vector<int32_t>& sat;  // (ny+1) x (nx+1) prefix counts (maps < 2^31 cells)
  const int32_t* S = nullptr; // the table count() reads (sat's data, or a table built on the GPU)
  double cutoff;
  int maxd, mind;
  std::vector<int32_t> out;  // (x0, y0, w, h) quadruples

  // a table computed elsewhere (launch_sat on the device, copied back)
  Clusterer(const int32_t* table, int64_t nx_, int64_t ny_, double c, int mx, int mn)
      : nx(nx_), ny(ny_), sat(own), S(table), cutoff(c), maxd(mx), mind(mn) {}
  // scratch: a caller-kept buffer for the table (no fresh pages per regrid)
  Clusterer(const uint8_t* f, int64_t nx_, int64_t ny_, double c, int mx, int mn,
            std::vector<int32_t>* scratch = nullptr)
      : nx(nx_), ny(ny_), sat(scratch ? *scratch : own), cutoff(c), maxd(mx), mind(mn) {
    sat.resize(static_cast<size_t>((nx + 1) * (ny + 1)));
    const int64_t W = nx + 1;
    const int nt = host_threads(static_cast<int>(std::min<int64_t>(ny, 1 << 20)) * 4);
    // row prefix sums (rows in parallel), then running sums down each column
    // (column blocks in parallel)
    std::fill(sat.begin(), sat.begin() + W, 0);
    parallel_for(nt, static_cast<int>(ny), [&](int J) {
      int32_t run = 0;
      int32_t* row = sat.data() + (J + 1) * W;
      row[0] = 0;
      const uint8_t* fr = f + static_cast<int64_t>(J) * nx;
      for (int64_t I = 0; I < nx; ++I) {
        run += fr[I] ? 1 : 0;
        row[I + 1] = run;
      }
    });
    const int64_t blk = 256;
    const int nb = static_cast<int>((W + blk - 1) / blk);
    parallel_for(std::min(nt, nb), nb, [&](int b) {
      const int64_t a0 = b * blk, a1 = std::min(W, a0 + blk);
      for (int64_t J = 1; J <= ny; ++J) {
        int32_t* r = sat.data() + J * W;
        const int32_t* q = r - W;
        for (int64_t I = a0; I < a1; ++I) r[I] += q[I];
      }
    });
    S = sat.data();
  }
  int64_t count(int64_t x0, int64_t y0, int64_t x1, int64_t y1) const {  // [x0,x1) x [y0,y1)
    const int64_t W = nx + 1;
    return static_cast<int64_t>(S[y1 * W + x1]) - S[y0 * W + x1] - S[y1 * W + x0] + S[y0 * W + x0];
  }
  void emit(int64_t x0, int64_t y0, int64_t w, int64_t h) {
    out.push_back(static_cast<int32_t>(x0));
    out.push_back(static_cast<int32_t>(y0));
    out.push_back(static_cast<int32_t>(w));
    out.push_back(static_cast<int32_t>(h));
  }
  bool admissible(int64_t k, int64_t n) const { return k >= mind && n - k >= mind; }

  struct Box { int64_t x0, y0, x1, y1; };
  // Berger-Rigoutsos, depth first with the low part of every cut first (the
  // oracle's order).  The first cuts are expanded breadth first into an
  // ordered frontier (a cut box is replaced by its low and high parts, so each
  // entry's subtree output stays contiguous in the depth-first order) until
  // it holds enough open boxes; their subtrees are then clustered by host
  // workers and all outputs concatenated in frontier order: the result is the
  // sequential one for any thread count.
  void run() {
    struct Ent {
      Box b;
      bool open;
      std::vector<int32_t> out;
    };
    std::vector<int64_t> sig[2];
    const int nthr = host_threads(64 * 64);
    const size_t want = static_cast<size_t>(4 * nthr);
    std::vector<Ent> fr;
    fr.push_back(Ent{Box{0, 0, nx, ny}, true, {}});
    size_t nopen = 1;
    std::vector<Box> st;
    while (nthr > 1 && nopen > 0 && nopen < want) {
      std::vector<Ent> nxt;
      nopen = 0;
      for (Ent& e : fr) {
        if (!e.open) {
          nxt.push_back(std::move(e));
          continue;
        }
        st.clear();
        std::vector<int32_t> o;
        process(e.b, st, o, sig);
        if (!o.empty()) nxt.push_back(Ent{e.b, false, std::move(o)});
        if (st.size() == 2) {  // pushed hi, then lo
          nxt.push_back(Ent{st[1], true, {}});
          nxt.push_back(Ent{st[0], true, {}});
          nopen += 2;
        }
      }
      fr.swap(nxt);
    }
    parallel_for(nthr, static_cast<int>(fr.size()), [&](int i) {
      Ent& e = fr[i];
      if (!e.open) return;
      std::vector<Box> stk{e.b};
      std::vector<int64_t> sg[2];
      while (!stk.empty()) {
        Box bx = stk.back();
        stk.pop_back();
        process(bx, stk, e.out, sg);
      }
    });
    for (auto& e : fr) out.insert(out.end(), e.out.begin(), e.out.end());
  }
  static void emit_to(std::vector<int32_t>& o, int64_t x0, int64_t y0, int64_t w, int64_t h) {
    o.push_back(static_cast<int32_t>(x0));
    o.push_back(static_cast<int32_t>(y0));
    o.push_back(static_cast<int32_t>(w));
    o.push_back(static_cast<int32_t>(h));
  }
  // one popped box: emit it, or push its two parts
  void process(Box b, std::vector<Box>& stack, std::vector<int32_t>& o, std::vector<int64_t>* sig) const {
    {
      if (count(b.x0, b.y0, b.x1, b.y1) == 0) return;
      // shrink: first / last non-empty column and row
      while (count(b.x0, b.y0, b.x0 + 1, b.y1) == 0) ++b.x0;
      while (count(b.x1 - 1, b.y0, b.x1, b.y1) == 0) --b.x1;
      while (count(b.x0, b.y0, b.x1, b.y0 + 1) == 0) ++b.y0;
      while (count(b.x0, b.y1 - 1, b.x1, b.y1) == 0) --b.y1;
      const int64_t w = b.x1 - b.x0, h = b.y1 - b.y0;
      const int64_t nf = count(b.x0, b.y0, b.x1, b.y1);
      if (static_cast<double>(nf) / static_cast<double>(w * h) >= cutoff && w <= maxd && h <= maxd) {
        emit_to(o, b.x0, b.y0, w, h);
        return;
      }
      sig[0].resize(w);
      sig[1].resize(h);
      for (int64_t k = 0; k < w; ++k) sig[0][k] = count(b.x0 + k, b.y0, b.x0 + k + 1, b.y1);
      for (int64_t k = 0; k < h; ++k) sig[1][k] = count(b.x0, b.y0 + k, b.x1, b.y0 + k + 1);
      const int order[2] = {w >= h ? 0 : 1, w >= h ? 1 : 0};
      const int64_t len[2] = {w, h};
      int dir = -1;
      int64_t cut = 0;
      // (a) holes
      for (int t = 0; t < 2 && dir < 0; ++t) {
        const int d = order[t];
        const int64_t n = len[d];
        int64_t best = -1, bd = 0;
        for (int64_t k = 1; k < n; ++k) {
          if (sig[d][k] != 0 || !admissible(k, n)) continue;
          const int64_t dist = std::llabs(2 * k - n);
          if (best < 0 || dist < bd) {
            best = k;
            bd = dist;
          }
        }
        if (best >= 0) {
          dir = d;
          cut = best;
        }
      }
      // (b) inflections of the second difference
      if (dir < 0) {
        int64_t bv = -1, bd = 0;
        for (int t = 0; t < 2; ++t) {
          const int d = order[t];
          const int64_t n = len[d];
          const std::vector<int64_t>& g = sig[d];
          for (int64_t k = 2; k + 2 <= n; ++k) {
            const int64_t lap0 = g[k - 2] - 2 * g[k - 1] + g[k];
            const int64_t lap1 = g[k - 1] - 2 * g[k] + g[k + 1];
            const bool flip = (lap0 < 0 && lap1 > 0) || (lap0 > 0 && lap1 < 0);
            if (!flip || !admissible(k, n)) continue;
            const int64_t v = std::llabs(lap1 - lap0), dist = std::llabs(2 * k - n);
            if (v > bv || (v == bv && dist < bd)) {
              bv = v;
              bd = dist;
              dir = d;
              cut = k;
            }
          }
        }
      }
      // (c) bisect the longer side
      if (dir < 0 && admissible(len[order[0]] / 2, len[order[0]])) {
        dir = order[0];
        cut = len[order[0]] / 2;
      }
      if (dir < 0) {
        emit_to(o, b.x0, b.y0, w, h);
        return;
      }
      Box lo = b, hi = b;
      if (dir == 0) lo.x1 = hi.x0 = b.x0 + cut;
      else lo.y1 = hi.y0 = b.y0 + cut;
      stack.push_back(hi);  // LIFO: the low part is processed (entirely) first
      stack.push_back(lo);
    }
  }
};

}  // namespace

extern "C" {

int claw_level_extent(const claw_ctx* ctx, int32_t level, int64_t* nx, int64_t* ny) {
  if (!ctx || level < 1 || level > kMaxLevel || !ctx->lev[level].set) return CLAW_EINVAL;
  if (nx) *nx = ctx->lev[level].nx;
  if (ny) *ny = ctx->lev[level].ny;
  return CLAW_OK;
}

int claw_level_count(const claw_ctx* ctx, int32_t level, int32_t* npatch) {
  if (!ctx || !npatch || level < 1 || level > kMaxLevel) return CLAW_EINVAL;
  *npatch = ctx->lev[level].set ? ctx->lev[level].npatch : 0;
  return CLAW_OK;
}

int claw_level_descs(const claw_ctx* ctx, int32_t level, claw_patch_desc* out) {
  if (!ctx || !out || level < 1 || level > kMaxLevel || !ctx->lev[level].set) return CLAW_EINVAL;
  const Level& L = ctx->lev[level];
  std::memcpy(out, L.desc.data(), sizeof(claw_patch_desc) * L.desc.size());
  return CLAW_OK;
}

int claw_cluster(const uint8_t* flags, int64_t nx, int64_t ny, double cutoff, int32_t max_dim, int32_t min_dim,
                 int32_t* boxes, int32_t cap, int32_t* nbox) {
  if (!flags || nx < 1 || ny < 1 || !(cutoff > 0.0) || cutoff > 1.0 || max_dim < 1 || min_dim < 1 ||
      2 * min_dim > max_dim || !nbox || nx >= (1ll << 31) || ny >= (1ll << 31) || nx * ny >= (1ll << 31))
    return CLAW_EINVAL;
  Clusterer cl(flags, nx, ny, cutoff, max_dim, min_dim);
  cl.run();
  const int64_t n = static_cast<int64_t>(cl.out.size() / 4);
  *nbox = static_cast<int32_t>(n);
  if (boxes) std::memcpy(boxes, cl.out.data(), sizeof(int32_t) * 4 * std::min<int64_t>(n, cap));
  return (boxes && n > cap) ? CLAW_ENOMEM : CLAW_OK;
}

}  // extern "C"

namespace {

// Flag map of `level` on the device: raw flags, the level's own cells, and
// (nest > 0) the nesting mask M = cells whose in-domain neighbours within
// Chebyshev distance `nest` all belong to the level; then the dilation by
// `buffer` clipped to (clip: the level's cells / M).  Leaves the result in
// `out` (device) and its count in *nflag.
int flag_device(claw_ctx* ctx, int level, double tol, int buffer, int clip, DevBuf<uint8_t>& out,
                DevBuf<uint8_t>& on, int64_t* nflag) {
  Level& L = ctx->lev[level];
  const int64_t n = L.nx * L.ny;
  DevBuf<uint8_t> raw, tmp;
  DevBuf<int2> orig;
  DevBuf<unsigned long long> cnt;
  CUDA_TRY(raw.alloc(n));
  CUDA_TRY(tmp.alloc(n));
  CUDA_TRY(out.alloc(n));
  CUDA_TRY(on.alloc(n));
  CUDA_TRY(cnt.alloc(1));
  std::vector<int2> ho(L.owned.size());
  for (size_t lp = 0; lp < L.owned.size(); ++lp)
    ho[lp] = make_int2(static_cast<int>(L.i0[L.owned[lp]]), static_cast<int>(L.j0[L.owned[lp]]));
  if (int rc = upload(ctx, orig, ho)) return rc;
  CUDA_TRY(cudaMemsetAsync(raw.p, 0, n, ctx->stream));
  CUDA_TRY(cudaMemsetAsync(on.p, 0, n, ctx->stream));
  CUDA_TRY(cudaMemsetAsync(cnt.p, 0, 8, ctx->stream));
  claw::StepParams P{};
  P.q = L.q[L.cur].p;
  P.frame = L.frame.p + static_cast<int64_t>(L.fsel) * L.frame_elems;
  P.patches = L.dpatch.p;
  P.rects = L.drect.p;
  P.cellrect = L.ncellrect > 0 ? L.dcellrect.p : nullptr;
  int64_t max_cells = 1;
  for (const DevPatch& d : L.hpatch) max_cells = std::max<int64_t>(max_cells, static_cast<int64_t>(d.mx) * d.my);
  CUDA_TRY(static_cast<cudaError_t>(claw::launch_flag(P, orig.p, static_cast<int32_t>(L.owned.size()), L.nx, tol,
                                                      raw.p, on.p, max_cells, ctx->stream)));
  const uint8_t* mask = nullptr;
  if (clip == 1) mask = on.p;
  if (clip == 2) {
    // M = on & ~dilate(~on, 2): the complement, dilated (clipped to the
    // domain, so out-of-domain cells never veto), then inverted
    DevBuf<uint8_t> off, offd;
    DevBuf<unsigned long long> c2;
    CUDA_TRY(off.alloc(n));
    CUDA_TRY(offd.alloc(n));
    CUDA_TRY(c2.alloc(1));
    CUDA_TRY(static_cast<cudaError_t>(claw::launch_not(on.p, off.p, n, ctx->stream)));
    CUDA_TRY(static_cast<cudaError_t>(claw::launch_dilate(off.p, tmp.p, offd.p, nullptr, L.nx, L.ny, 2, c2.p,
                                                          ctx->stream)));
    CUDA_TRY(static_cast<cudaError_t>(claw::launch_not(offd.p, on.p, n, ctx->stream)));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));  // off / offd go back to the pool
    mask = on.p;
  }
  CUDA_TRY(static_cast<cudaError_t>(claw::launch_dilate(raw.p, tmp.p, out.p, mask, L.nx, L.ny, buffer, cnt.p,
                                                        ctx->stream)));
  unsigned long long c = 0;
  CUDA_TRY(cudaMemcpyAsync(&c, cnt.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (nflag) *nflag = static_cast<int64_t>(c);
  return CLAW_OK;
}

}  // namespace

extern "C" {

int claw_flag(claw_ctx* ctx, int32_t level, double tol, int32_t buffer, int32_t clip, uint8_t* flags_out,
              int64_t* nflag) {
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_level(ctx, level)) return rc;
  if (ctx->host_only) return fail(ctx, CLAW_ENODEV, "host-only context");
  if (ctx->cfg.world > 1) return fail(ctx, CLAW_EINVAL, "flagging is single-rank in this version");
  if (buffer < 0 || clip < 0 || clip > 2) return fail(ctx, CLAW_EINVAL, "buffer=%d clip=%d", buffer, clip);
  DevBuf<uint8_t> out, on;
  if (int rc = flag_device(ctx, level, tol, buffer, clip, out, on, nflag)) return rc;
  const Level& L = ctx->lev[level];
  if (flags_out) {
    CUDA_TRY(cudaMemcpyAsync(flags_out, out.p, L.nx * L.ny, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  }
  return CLAW_OK;
}

int claw_regrid(claw_ctx* ctx, int32_t level, int32_t nbox, const int32_t* boxes, int32_t R) {
  Nvtx nv_("claw_regrid L%d", level + 1);
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_level(ctx, level)) return rc;
  if (level >= kMaxLevel) return fail(ctx, CLAW_EINVAL, "regrid: level %d has no finer level", level);
  if (ctx->cfg.world > 1) return fail(ctx, CLAW_EINVAL, "regridding is single-rank in this version");
  if (ctx->lev[1].vc) return fail(ctx, CLAW_EINVAL, "regrid: variable media (claw_set_aux) are single-level (DESIGN.md R20)");
  if (nbox < 0 || (nbox > 0 && !boxes) || R < 1) return fail(ctx, CLAW_EINVAL, "regrid: nbox=%d R=%d", nbox, R);
  Level& C = ctx->lev[level];
  for (int b = 0; b < nbox; ++b) {
    const int32_t* x = boxes + 4 * b;
    if (x[2] < 1 || x[3] < 1 || x[0] < 0 || x[1] < 0 || x[0] + x[2] > C.nx || x[1] + x[3] > C.ny)
      return fail(ctx, CLAW_EINVAL, "regrid: box %d (%d,%d,%d,%d) outside level %d's index space", b, x[0], x[1],
                  x[2], x[3], level);
  }
  // the old fine level: the current level+1, else the one a regrid of a
  // coarser level discarded just before (R18)
  Level& src = ctx->lev[level + 1].set ? ctx->lev[level + 1] : ctx->stash[level + 1];
  if (src.set && nbox > 0 && src.ratio != R)
    return fail(ctx, CLAW_EINVAL, "regrid: R=%d differs from the old level %d's ratio %d", R, level + 1, src.ratio);
  PhaseTrace lap("regrid", level);
  if (!ctx->host_only) CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  drop_graphs(ctx);
  Level old = std::move(src);
  ctx->lev[level + 1] = Level();
  ctx->stash[level + 1] = Level();
  for (int l = level + 2; l <= kMaxLevel; ++l)  // discarded levels become copy sources
    if (ctx->lev[l].set) {
      ctx->stash[l] = std::move(ctx->lev[l]);
      ctx->lev[l] = Level();
      ctx->stashed = true;
    }
  if (nbox == 0) return CLAW_OK;
  // descriptors of the new level: boxes refined by R
  const double dxf = C.dx / R, dyf = C.dy / R;
  std::vector<claw_patch_desc> d(nbox);
  for (int b = 0; b < nbox; ++b) {
    d[b].mx = boxes[4 * b + 2] * R;
    d[b].my = boxes[4 * b + 3] * R;
    d[b].dx = dxf;
    d[b].dy = dyf;
    d[b].xlower = ctx->cfg.xlo + static_cast<double>(boxes[4 * b + 0] * R) * dxf;
    d[b].ylower = ctx->cfg.ylo + static_cast<double>(boxes[4 * b + 1] * R) * dyf;
    d[b].mbc = 2;
    d[b].rho = C.desc[0].rho;
    d[b].K = C.desc[0].K;
  }
  Level& L = ctx->lev[level + 1];
  L.hinterp.swap(old.hinterp);  // reuse the old table's pages (plan_level reassigns it)
  int rc = build_geometry(ctx, level + 1, nbox, d.data(), L);
  if (!rc) rc = plan_level(ctx, level + 1, L);
  if (rc) {
    L = Level();
    return rc;
  }
  lap("plan");
  L.t_old = L.t_new = C.t_new;
  lap("tables");
  if (ctx->host_only) {
    L.set = true;
    return CLAW_OK;
  }
  if (int r2 = alloc_level(ctx, level + 1, L)) return r2;
  lap("alloc");
  L.cur = 0;
  CUDA_TRY(cudaStreamSynchronize(nullptr));  // alloc_level's legacy-stream memsets
  // patch-id maps (coarse level; old fine level) and origins, all on the
  // device: no per-cell host work (P:373 runs regridding on the GPU)
  auto origins = [](const Level& X) {
    std::vector<int2> o(X.owned.size());
    for (size_t lp = 0; lp < X.owned.size(); ++lp)
      o[lp] = make_int2(static_cast<int>(X.i0[X.owned[lp]]), static_cast<int>(X.j0[X.owned[lp]]));
    return o;
  };
  DevBuf<int32_t> cmap, omap, err;
  DevBuf<int2> corig, oorig, norig;
  if (int r2 = upload(ctx, corig, origins(C))) return r2;
  if (int r2 = upload(ctx, norig, origins(L))) return r2;
  CUDA_TRY(cmap.alloc(C.nx * C.ny));
  CUDA_TRY(err.alloc(1));
  CUDA_TRY(cudaMemsetAsync(cmap.p, 0xff, C.nx * C.ny * 4, ctx->stream));
  CUDA_TRY(cudaMemsetAsync(err.p, 0, 4, ctx->stream));
  CUDA_TRY(static_cast<cudaError_t>(claw::launch_paint(cmap.p, C.nx, corig.p, C.dpatch.p,
                                                       static_cast<int32_t>(C.owned.size()), ctx->stream)));
  claw::RegridParams P{};
  if (old.set) {
    if (int r2 = upload(ctx, oorig, origins(old))) return r2;
    CUDA_TRY(omap.alloc(old.nx * old.ny));
    CUDA_TRY(cudaMemsetAsync(omap.p, 0xff, old.nx * old.ny * 4, ctx->stream));
    CUDA_TRY(static_cast<cudaError_t>(claw::launch_paint(omap.p, old.nx, oorig.p, old.dpatch.p,
                                                         static_cast<int32_t>(old.owned.size()), ctx->stream)));
    P.qf_old = old.q[old.cur].p;
    P.oldmap = omap.p;
    P.opatch = old.dpatch.p;
    P.oorig = oorig.p;
  }
  P.qc_old = C.q[1 - C.cur].p;
  P.qc_new = C.q[C.cur].p;
  P.cmap = cmap.p;
  P.cpatch = C.dpatch.p;
  P.corig = corig.p;
  P.cnx = C.nx;
  P.cny = C.ny;
  P.fnx = L.nx;
  P.qf = L.q[0].p;
  P.npatch = L.dpatch.p;
  P.norig = norig.p;
  P.R = R;
  P.per_x = ctx->cfg.bc[0] == CLAW_BC_PERIODIC;
  P.per_y = ctx->cfg.bc[2] == CLAW_BC_PERIODIC;
  P.err = err.p;
  if (!L.gapless) CUDA_TRY(cudaMemsetAsync(L.q[0].p, 0, L.buf_elems * 8, ctx->stream));  // alignment gaps
  CUDA_TRY(static_cast<cudaError_t>(claw::launch_regrid(P, static_cast<int32_t>(L.owned.size()), ctx->stream)));
  int32_t herr = 0;
  CUDA_TRY(cudaMemcpyAsync(&herr, err.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(cudaMemcpyAsync(L.q[1].p, L.q[0].p, L.buf_elems * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  CUDA_TRY(cudaMemsetAsync(L.frame.p, 0, L.frame.n * 8, ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));  // the old level and the maps go back to the pool
  if (herr) {
    L = Level();
    return fail(ctx, CLAW_ENEST, "regrid: a new level-%d cell to interpolate has a coarse donor that is not on "
                "level %d", level + 1, level);
  }
  lap("kernels");
  ctx->stats.ghost_launches += old.set ? 3 : 2;
  L.set = true;
  return CLAW_OK;
}

int claw_regrid_auto(claw_ctx* ctx, int32_t level, double tol, int32_t buffer, double cutoff, int32_t max_dim,
                     int32_t min_dim, int32_t R, int32_t* nbox_out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = check_level(ctx, level)) return rc;
  if (ctx->host_only) return fail(ctx, CLAW_ENODEV, "host-only context");
  if (ctx->cfg.world > 1) return fail(ctx, CLAW_EINVAL, "regridding is single-rank in this version");
  if (buffer < 0) return fail(ctx, CLAW_EINVAL, "buffer=%d", buffer);
  const Level& C = ctx->lev[level];
  const int64_t n = C.nx * C.ny;
  PhaseTrace lap("auto", level);
  DevBuf<uint8_t> out, on;
  int64_t nflag = 0;
  if (int rc = flag_device(ctx, level, tol, buffer, 2, out, on, &nflag)) return rc;
  lap("flag");
  // the clusterer reads only the flags' summed-area table: built on the
  // device (launch_sat) and copied back with the nesting mask, instead of
  // copying the flag map and summing it on the host (4 ms for 2000^2 cells)
  const size_t satb = static_cast<size_t>((C.nx + 1) * (C.ny + 1)) * sizeof(int32_t);
  const size_t need = satb + static_cast<size_t>(n);
  if (ctx->h_stage_bytes < need) {
    if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
    ctx->h_stage = nullptr;
    ctx->h_stage_bytes = 0;
    CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&ctx->h_stage), need));
    ctx->h_stage_bytes = need;
  }
  const int32_t* hsat = reinterpret_cast<const int32_t*>(ctx->h_stage);
  const uint8_t* m = ctx->h_stage + satb;
  {
    DevBuf<int32_t> dsat;
    if (nflag > 0) {
      CUDA_TRY(dsat.alloc(static_cast<size_t>((C.nx + 1) * (C.ny + 1))));
      CUDA_TRY(static_cast<cudaError_t>(claw::launch_sat(out.p, C.nx, C.ny, dsat.p, ctx->stream)));
      if (lap.on) {
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        lap("sat");
      }
      CUDA_TRY(cudaMemcpyAsync(ctx->h_stage, dsat.p, satb, cudaMemcpyDeviceToHost, ctx->stream));
    }
    CUDA_TRY(cudaMemcpyAsync(ctx->h_stage + satb, on.p, n, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  }
  lap("d2h");
  std::vector<int32_t> boxes;
  if (nflag > 0) {
    if (!(cutoff > 0.0) || cutoff > 1.0 || max_dim < 1 || min_dim < 1 || 2 * min_dim > max_dim)
      return fail(ctx, CLAW_EINVAL, "cluster: cutoff=%g max_dim=%d min_dim=%d", cutoff, max_dim, min_dim);
    if (n >= (1ll << 31)) return fail(ctx, CLAW_EINVAL, "regrid_auto: flag map of %lld cells", (long long)n);
    Clusterer cl(hsat, C.nx, C.ny, cutoff, max_dim, min_dim);
    cl.run();
    lap("BR");
    // nesting: split each box into row-run rectangles of the nesting mask M
    // (runs identical in consecutive rows merge), drop pieces without flags;
    // boxes in parallel, pieces concatenated in box order
    const int nbx = static_cast<int>(cl.out.size() / 4);
    std::vector<std::vector<int32_t>> piece(nbx);
    parallel_for(host_threads(nbx * 16), nbx, [&](int bi) {
      const size_t b = 4 * static_cast<size_t>(bi);
      const int64_t x0 = cl.out[b], y0 = cl.out[b + 1], x1 = x0 + cl.out[b + 2], y1 = y0 + cl.out[b + 3];
      struct Open { int64_t a, e, y; };
      std::vector<Open> open, next;
      std::vector<std::array<int64_t, 4>> done;
      std::vector<std::pair<int64_t, int64_t>> runs;
      for (int64_t J = y0; J <= y1; ++J) {
        runs.clear();
        if (J < y1)
          for (int64_t I = x0; I < x1;) {
            if (!m[J * C.nx + I]) {
              ++I;
              continue;
            }
            int64_t e = I;
            while (e < x1 && m[J * C.nx + e]) ++e;
            runs.emplace_back(I, e);
            I = e;
          }
        next.clear();
        for (const Open& o : open) {
          bool cont = false;
          for (auto& r : runs)
            if (r.first == o.a && r.second == o.e) cont = true;
          if (cont) next.push_back(o);
          else done.push_back({o.a, o.y, o.e, J});
        }
        for (auto& r : runs) {
          bool had = false;
          for (const Open& o : open)
            if (o.a == r.first && o.e == r.second) had = true;
          if (!had) next.push_back(Open{r.first, r.second, J});
        }
        std::sort(next.begin(), next.end(), [](const Open& a, const Open& b) { return a.a < b.a; });
        open.swap(next);
      }
      std::stable_sort(done.begin(), done.end(), [](const std::array<int64_t, 4>& a, const std::array<int64_t, 4>& b) {
        return a[1] != b[1] ? a[1] < b[1] : a[0] < b[0];
      });
      for (auto& r : done)
        if (cl.count(r[0], r[1], r[2], r[3]) > 0) {
          piece[bi].push_back(static_cast<int32_t>(r[0]));
          piece[bi].push_back(static_cast<int32_t>(r[1]));
          piece[bi].push_back(static_cast<int32_t>(r[2] - r[0]));
          piece[bi].push_back(static_cast<int32_t>(r[3] - r[1]));
        }
    });
    for (auto& pc : piece) boxes.insert(boxes.end(), pc.begin(), pc.end());
  }
  const int32_t nb = static_cast<int32_t>(boxes.size() / 4);
  lap("nest-split");
  if (nbox_out) *nbox_out = nb;
  const int rc = claw_regrid(ctx, level, nb, boxes.data(), R);
  lap("regrid");
  return rc;
}

int claw_pool_stats(int64_t* hits, int64_t* misses, int64_t* cached_bytes) {
  Pool& P = pool();
  std::lock_guard<std::mutex> g(P.mu);
  if (hits) *hits = P.hits;
  if (misses) *misses = P.misses;
  if (cached_bytes) *cached_bytes = static_cast<int64_t>(P.cached());
  return CLAW_OK;
}

int claw_pool_trim(void) {
  pool().trim_all();
  return CLAW_OK;
}

int claw_set_profiling(claw_ctx* ctx, int32_t on) {
  if (int rc = check_ctx(ctx)) return rc;
  ctx->profiling = on != 0;
  return CLAW_OK;
}

int claw_get_stats(claw_ctx* ctx, claw_stats* out) {
  if (int rc = check_ctx(ctx)) return rc;
  if (!out) return CLAW_EINVAL;
  ctx->stats.step_ms += drain(ctx, ctx->ev_step);
  ctx->stats.ghost_ms += drain(ctx, ctx->ev_ghost);
  *out = ctx->stats;
  return CLAW_OK;
}

int claw_reset_stats(claw_ctx* ctx) {
  if (int rc = check_ctx(ctx)) return rc;
  drain(ctx, ctx->ev_step);
  drain(ctx, ctx->ev_ghost);
  ctx->stats = claw_stats{};
  return CLAW_OK;
}

int claw_synchronize(claw_ctx* ctx) {
  if (int rc = check_ctx(ctx)) return rc;
  if (ctx->host_only) return CLAW_OK;
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return CLAW_OK;
}

}  // extern "C"
