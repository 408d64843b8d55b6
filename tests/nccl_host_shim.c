/* Test infrastructure: a stand-in for the four NCCL entry points
 * plq_solve_parallel_sharded binds (PLQ_NCCL_LIB), for running its exchange
 * logic across several ranks that are processes sharing ONE GPU.  Every
 * collective is staged through a POSIX shared-memory buffer on the host and
 * completed with process-shared barriers, after the caller's stream has
 * drained -- so no kernel of one rank ever waits on another rank's kernel.
 * Not NCCL, not part of the product. */
#include <cuda_runtime.h>
#include <fcntl.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <unistd.h>

typedef struct {
  pthread_barrier_t bar;
  unsigned long long calls;   /* collectives completed (rank 0 counts) */
  char data[];
} shared_t;

typedef struct {
  int rank, world;
  size_t cap;
  shared_t* sh;
} comm_t;

static size_t elem_bytes(int dtype) { return dtype == 2 ? 4 : 8; } /* ncclInt32 : ncclFloat64 */

/* parent: create and initialise the shared block */
int shim_create(const char* name, int world, size_t cap) {
  int fd = shm_open(name, O_CREAT | O_RDWR, 0600);
  if (fd < 0) return -1;
  if (ftruncate(fd, sizeof(shared_t) + cap)) return -2;
  shared_t* sh = mmap(NULL, sizeof(shared_t) + cap, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (sh == MAP_FAILED) return -3;
  pthread_barrierattr_t a;
  pthread_barrierattr_init(&a);
  pthread_barrierattr_setpshared(&a, PTHREAD_PROCESS_SHARED);
  pthread_barrier_init(&sh->bar, &a, world);
  sh->calls = 0;
  munmap(sh, sizeof(shared_t) + cap);
  return 0;
}

int shim_destroy(const char* name) { return shm_unlink(name); }

/* rank: attach; the returned pointer is passed as the ncclComm_t */
void* shim_attach(const char* name, int rank, int world, size_t cap) {
  int fd = shm_open(name, O_RDWR, 0600);
  if (fd < 0) return NULL;
  shared_t* sh = mmap(NULL, sizeof(shared_t) + cap, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (sh == MAP_FAILED) return NULL;
  comm_t* c = malloc(sizeof(comm_t));
  c->rank = rank;
  c->world = world;
  c->cap = cap;
  c->sh = sh;
  return c;
}

unsigned long long shim_calls(void* comm) { return ((comm_t*)comm)->sh->calls; }

int ncclGroupStart(void) { return 0; }
int ncclGroupEnd(void) { return 0; }
const char* ncclGetErrorString(int e) { return e ? "shim error" : "ok"; }

int ncclBroadcast(const void* send, void* recv, size_t count, int dtype, int root, void* comm, cudaStream_t s) {
  comm_t* c = comm;
  const size_t bytes = count * elem_bytes(dtype);
  if (bytes > c->cap) return 2;
  if (cudaStreamSynchronize(s) != cudaSuccess) return 1;
  if (c->rank == root && cudaMemcpy(c->sh->data, send, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
  pthread_barrier_wait(&c->sh->bar);
  if (c->rank != root && cudaMemcpy(recv, c->sh->data, bytes, cudaMemcpyHostToDevice) != cudaSuccess) return 1;
  if (c->rank == 0) c->sh->calls++;
  pthread_barrier_wait(&c->sh->bar);
  return 0;
}

int ncclAllGather(const void* send, void* recv, size_t sendcount, int dtype, void* comm, cudaStream_t s) {
  comm_t* c = comm;
  const size_t bytes = sendcount * elem_bytes(dtype);
  if (bytes * c->world > c->cap) return 2;
  if (cudaStreamSynchronize(s) != cudaSuccess) return 1;
  if (cudaMemcpy(c->sh->data + c->rank * bytes, send, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
  pthread_barrier_wait(&c->sh->bar);
  if (cudaMemcpy(recv, c->sh->data, bytes * c->world, cudaMemcpyHostToDevice) != cudaSuccess) return 1;
  if (c->rank == 0) c->sh->calls++;
  pthread_barrier_wait(&c->sh->bar);
  return 0;
}
