/* Test-only stand-in for libnccl.so.2 (loaded by libclaw.so through
 * CLAW_NCCL_LIB): the few NCCL calls libclaw makes -- unique id, communicator
 * init/destroy, grouped point-to-point send/recv and a max/sum all-reduce --
 * implemented between PROCESSES ON ONE GPU through a memory-mapped file,
 * with synchronous device<->host copies (CUDA driver API).  Real NCCL refuses
 * two ranks on one GPU ("Duplicate GPU detected"), so this is how the
 * library's NCCL call sequence (pack kernel, group of sends and receives into
 * the frame on the comm stream, events, edge tiles, CFL all-reduce) runs in a
 * multi-process test on a 1-GPU box.  Not used by the product. */
#define _GNU_SOURCE
#include <dlfcn.h>
#include <fcntl.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

typedef enum { ncclSuccess = 0, ncclUnhandledCudaError = 1, ncclSystemError = 2, ncclInternalError = 3,
               ncclInvalidArgument = 4, ncclInvalidUsage = 5 } ncclResult_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclDataType_t;  /* NCCL: ncclFloat64 = 8, ncclUint64 = 5, ncclInt64 = 4 */
typedef int ncclRedOp_t;     /* NCCL: ncclSum = 0, ncclMax = 2 */

#define MAXW 8
#define MBOX (16u << 20)   /* bytes per ordered rank pair */
#define SLOT 4096          /* bytes per rank for all-reduce */

typedef struct {
  volatile uint64_t bar_count, bar_gen;
  volatile uint64_t seq[MAXW][MAXW];   /* messages posted src -> dst */
  volatile uint64_t ack[MAXW][MAXW];   /* messages src -> dst copied out by dst */
  volatile uint64_t size[MAXW][MAXW];
} Hdr;

typedef struct Comm {
  int rank, world;
  char path[256];
  unsigned char* base;
  size_t bytes;
  Hdr* h;
  uint64_t got[MAXW];   /* messages received from each src */
} Comm;
typedef Comm* ncclComm_t;

/* ---- CUDA driver API (dlopen: no link dependency) */
typedef int (*fn_sync)(void*);
typedef int (*fn_d2h)(void*, unsigned long long, size_t, void*);
typedef int (*fn_h2d)(unsigned long long, const void*, size_t, void*);
static fn_sync p_sync;
static fn_d2h p_d2h;
static fn_h2d p_h2d;
static int cuda_load(void) {
  if (p_sync) return 0;
  void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_LOCAL);
  if (!h) return -1;
  p_sync = (fn_sync)dlsym(h, "cuStreamSynchronize");
  p_d2h = (fn_d2h)dlsym(h, "cuMemcpyDtoHAsync_v2");
  p_h2d = (fn_h2d)dlsym(h, "cuMemcpyHtoDAsync_v2");
  return (p_sync && p_d2h && p_h2d) ? 0 : -1;
}
static int d2h(void* dst, const void* src, size_t n, void* st) {
  if (p_d2h(dst, (unsigned long long)(uintptr_t)src, n, st)) return -1;
  return p_sync(st) ? -1 : 0;
}
static int h2d(void* dst, const void* src, size_t n, void* st) {
  if (p_h2d((unsigned long long)(uintptr_t)dst, src, n, st)) return -1;
  return p_sync(st) ? -1 : 0;
}

static void nap(void) {
  struct timespec ts = {0, 20000};
  nanosleep(&ts, NULL);
}
static size_t dsize(ncclDataType_t t) {
  switch (t) {
    case 0: case 1: return 1;          /* int8, uint8 */
    case 2: case 3: case 9: return 4;  /* int32, uint32, float32 */
    case 6: return 2;                  /* float16 */
    default: return 8;                 /* int64, uint64, float64 */
  }
}
static unsigned char* mbox(Comm* c, int src, int dst) {
  return c->base + sizeof(Hdr) + (size_t)(src * MAXW + dst) * MBOX;
}
static unsigned char* slot(Comm* c, int r) {
  return c->base + sizeof(Hdr) + (size_t)MAXW * MAXW * MBOX + (size_t)r * SLOT;
}
static void barrier(Comm* c) {
  const uint64_t gen = __atomic_load_n(&c->h->bar_gen, __ATOMIC_ACQUIRE);
  if (__atomic_add_fetch(&c->h->bar_count, 1, __ATOMIC_ACQ_REL) == (uint64_t)c->world) {
    __atomic_store_n(&c->h->bar_count, 0, __ATOMIC_RELEASE);
    __atomic_add_fetch(&c->h->bar_gen, 1, __ATOMIC_ACQ_REL);
  } else {
    while (__atomic_load_n(&c->h->bar_gen, __ATOMIC_ACQUIRE) == gen) nap();
  }
}

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  memset(id, 0, sizeof *id);
  struct timespec ts;
  clock_gettime(CLOCK_REALTIME, &ts);
  snprintf(id->internal, sizeof id->internal, "/tmp/claw_ncclshim_%d_%ld_%ld", (int)getpid(), (long)ts.tv_sec,
           (long)ts.tv_nsec);
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int world, ncclUniqueId id, int rank) {
  if (world < 1 || world > MAXW || rank < 0 || rank >= world) return ncclInvalidArgument;
  if (cuda_load()) return ncclUnhandledCudaError;
  Comm* c = (Comm*)calloc(1, sizeof(Comm));
  c->rank = rank;
  c->world = world;
  snprintf(c->path, sizeof c->path, "%s", id.internal);
  c->bytes = sizeof(Hdr) + (size_t)MAXW * MAXW * MBOX + (size_t)MAXW * SLOT;
  int fd = open(c->path, O_RDWR | O_CREAT, 0600);
  if (fd < 0) return ncclSystemError;
  if (ftruncate(fd, (off_t)c->bytes)) return ncclSystemError;  /* sparse file, zero-filled */
  c->base = (unsigned char*)mmap(NULL, c->bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (c->base == MAP_FAILED) return ncclSystemError;
  c->h = (Hdr*)c->base;
  barrier(c);  /* every rank mapped the file */
  *comm = c;
  return ncclSuccess;
}

/* introspection (claw_comm_info); the stand-in has no device of its own: the
 * caller's current device */
ncclResult_t ncclCommCount(const ncclComm_t c, int* n) {
  *n = c->world;
  return ncclSuccess;
}
ncclResult_t ncclCommUserRank(const ncclComm_t c, int* r) {
  *r = c->rank;
  return ncclSuccess;
}
ncclResult_t ncclCommCuDevice(const ncclComm_t c, int* d) {
  (void)c;
  *d = -1;
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t c) {
  if (!c) return ncclSuccess;
  barrier(c);
  if (c->rank == 0) unlink(c->path);
  munmap(c->base, c->bytes);
  free(c);
  return ncclSuccess;
}

/* ---- groups: operations are queued and run at ncclGroupEnd (sends first) */
typedef struct { int send; void* buf; size_t bytes; int peer; Comm* c; void* st; } Op;
static Op ops[256];
static int nops, depth;

static ncclResult_t run_ops(void) {
  for (int k = 0; k < nops; ++k) {
    Op* o = &ops[k];
    if (!o->send) continue;
    Comm* c = o->c;
    if (o->bytes > MBOX) return ncclInvalidArgument;
    /* the peer must have copied out the previous message on this pair */
    while (__atomic_load_n(&c->h->ack[c->rank][o->peer], __ATOMIC_ACQUIRE) !=
           __atomic_load_n(&c->h->seq[c->rank][o->peer], __ATOMIC_ACQUIRE))
      nap();
    if (d2h(mbox(c, c->rank, o->peer), o->buf, o->bytes, o->st)) return ncclUnhandledCudaError;
    c->h->size[c->rank][o->peer] = o->bytes;
    __atomic_add_fetch(&c->h->seq[c->rank][o->peer], 1, __ATOMIC_ACQ_REL);
  }
  for (int k = 0; k < nops; ++k) {
    Op* o = &ops[k];
    if (o->send) continue;
    Comm* c = o->c;
    const uint64_t want = c->got[o->peer] + 1;
    while (__atomic_load_n(&c->h->seq[o->peer][c->rank], __ATOMIC_ACQUIRE) < want) nap();
    if (c->h->size[o->peer][c->rank] != o->bytes) return ncclInvalidUsage;
    if (h2d(o->buf, mbox(c, o->peer, c->rank), o->bytes, o->st)) return ncclUnhandledCudaError;
    c->got[o->peer] = want;
    __atomic_add_fetch(&c->h->ack[o->peer][c->rank], 1, __ATOMIC_ACQ_REL);
  }
  nops = 0;
  return ncclSuccess;
}

ncclResult_t ncclGroupStart(void) {
  ++depth;
  return ncclSuccess;
}
ncclResult_t ncclGroupEnd(void) {
  if (depth <= 0) return ncclInvalidUsage;
  if (--depth) return ncclSuccess;
  return run_ops();
}
static ncclResult_t post(int send, void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t c, void* st) {
  if (nops >= 256 || !c || peer < 0 || peer >= c->world) return ncclInvalidArgument;
  ops[nops++] = (Op){send, buf, count * dsize(t), peer, c, st};
  return depth ? ncclSuccess : run_ops();
}
ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t c, void* st) {
  return post(1, (void*)buf, count, t, peer, c, st);
}
ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t c, void* st) {
  return post(0, buf, count, t, peer, c, st);
}

ncclResult_t ncclAllReduce(const void* sb, void* rb, size_t count, ncclDataType_t t, ncclRedOp_t op,
                           ncclComm_t c, void* st) {
  if (t != 8 || (op != 0 && op != 2) || count * 8 > SLOT) return ncclInvalidArgument;  /* float64 sum / max */
  double* mine = (double*)slot(c, c->rank);
  if (d2h(mine, sb, count * 8, st)) return ncclUnhandledCudaError;
  barrier(c);
  double acc[SLOT / 8];
  for (size_t k = 0; k < count; ++k) {
    double a = ((double*)slot(c, 0))[k];
    for (int r = 1; r < c->world; ++r) {
      const double v = ((double*)slot(c, r))[k];
      a = op == 2 ? (v > a ? v : a) : a + v;
    }
    acc[k] = a;
  }
  barrier(c);  /* every rank read the slots */
  if (h2d(rb, acc, count * 8, st)) return ncclUnhandledCudaError;
  return ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t r) {
  (void)r;
  return "ncclshim error";
}
