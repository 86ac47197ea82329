/*
 * c_multiproc_demo.c -- one process per pool, in plain C (no Python, no torch).
 *
 * N processes (fork) each own one paged KV pool (cudaMalloc) and a 128-byte
 * line of barrier counters.  They exchange CUDA IPC handles of both through a
 * MAP_SHARED page, build identical caches and identical source tables
 * (kv_alloc is deterministic), then switch six DP requests DP_N -> TP_N and
 * back, each process switching its own pool in one call: plan, push of its
 * atoms into the peers' pools, the group barrier (a5), remap of its pool,
 * read-back.  With >= N GPUs process r runs on device r and the barrier is
 * the device-side kv_group_barrier inside kv_switch_range.  With fewer GPUs
 * the processes share cuda:0 and call kv_switch_range_host with a host
 * barrier callback: separate launches of different processes that spin on
 * one another are not co-scheduled on one device.  Check: every source block
 * of every layer a process owned is back, byte for byte, in the blocks of its
 * final DP tables.  Exit code 0 on success.
 *
 * Build: gcc -std=c99 -o c_multiproc_demo c_multiproc_demo.c -I../include -lflykv -lcudart
 */
#define _GNU_SOURCE
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/wait.h>
#include <unistd.h>

#include <cuda_runtime_api.h>

#include "flykv.h"

#define CHECK(x)                                                                               \
    do {                                                                                       \
        kv_status s_ = (x);                                                                    \
        if (s_ != KV_OK) {                                                                     \
            fprintf(stderr, "rank %d: %s:%d %s -> %s: %s\n", rank, __FILE__, __LINE__, #x,     \
                    kv_strerror(s_), kv_last_error());                                         \
            return 1;                                                                          \
        }                                                                                      \
    } while (0)

#define CUDA(x)                                                                                \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            fprintf(stderr, "rank %d: %s -> %s\n", rank, #x, cudaGetErrorString(e_));          \
            return 1;                                                                          \
        }                                                                                      \
    } while (0)

enum { MAXN = 8, L = 2, NB = 96, NREQ = 6, LINE = 16 };

/* the page every process maps: IPC handles and a host barrier for the setup */
typedef struct {
    uint8_t pool_handle[MAXN][64];
    uint64_t pool_off[MAXN];
    uint8_t flag_handle[MAXN][64];
    uint64_t flag_off[MAXN];
    volatile int arrived;
    volatile int failed;
} shared_t;

static void host_barrier(shared_t* sh, int n, int* gen) {
    *gen += 1;
    __atomic_fetch_add(&sh->arrived, 1, __ATOMIC_SEQ_CST);
    while (__atomic_load_n(&sh->arrived, __ATOMIC_SEQ_CST) < n * *gen && !sh->failed) usleep(100);
}

/* kv_switch_range_host's callback: the host barrier over the processes */
typedef struct {
    shared_t* sh;
    int n;
    int* gen;
} hb_ctx;

static int32_t host_barrier_cb(void* ctx) {
    hb_ctx* h = (hb_ctx*)ctx;
    host_barrier(h->sh, h->n, h->gen);
    return h->sh->failed ? 1 : 0;
}

static int run_rank(int rank, int n, shared_t* sh) {
    const kv_geometry geo = {L, 8, 64, 16, 2};
    int64_t M = 0;
    int32_t hl = 0, bt = 0, gen = 0;
    CHECK(kv_layout(&geo, 1, &hl, &bt, &M));
    const size_t pool_bytes = (size_t)L * NB * (size_t)M;
    int n_dev = 0;
    CUDA(cudaGetDeviceCount(&n_dev));
    const int own_gpu = n_dev >= n; /* one GPU per process: device barrier */
    CUDA(cudaSetDevice(own_gpu ? rank : 0));
    uint8_t* pool = NULL;
    uint64_t* flags = NULL;
    CUDA(cudaMalloc((void**)&pool, pool_bytes));
    CUDA(cudaMalloc((void**)&flags, LINE * sizeof(uint64_t)));
    CUDA(cudaMemset(flags, 0, LINE * sizeof(uint64_t)));
    uint8_t* host = (uint8_t*)malloc(pool_bytes);
    for (size_t i = 0; i < pool_bytes; ++i) host[i] = (uint8_t)(i * 131u + (size_t)rank * 17u + (i >> 13));
    CUDA(cudaMemcpy(pool, host, pool_bytes, cudaMemcpyHostToDevice));
    CHECK(kv_ipc_export(pool, sh->pool_handle[rank], &sh->pool_off[rank]));
    CHECK(kv_ipc_export(flags, sh->flag_handle[rank], &sh->flag_off[rank]));
    host_barrier(sh, n, &gen);

    /* every pool's layers and every member's counters, as seen from this process */
    void* bases[MAXN * L];
    uint64_t* ctr[MAXN];
    int32_t nb[MAXN];
    for (int g = 0; g < n; ++g) {
        uint8_t* b = pool;
        uint64_t* f = flags;
        if (g != rank) {
            void* p = NULL;
            CHECK(kv_ipc_import(sh->pool_handle[g], sh->pool_off[g], &p));
            b = (uint8_t*)p;
            CHECK(kv_ipc_import(sh->flag_handle[g], sh->flag_off[g], &p));
            f = (uint64_t*)p;
        }
        for (int l = 0; l < L; ++l) bases[g * L + l] = b + (size_t)l * NB * (size_t)M;
        ctr[g] = f;
        nb[g] = NB;
    }
    const int32_t degrees[3] = {2, 4, 8};
    kv_cache* c = NULL;
    CHECK(kv_cache_create(&geo, n, nb, (void* const*)bases, degrees, 3, &c));

    /* identical source tables on every process: DP request i on engine i % n */
    const int32_t T[NREQ] = {40, 200, 17, 96, 130, 65};
    int32_t src_ids[NREQ][NB];
    kv_request fwd[NREQ], back[NREQ];
    for (int i = 0; i < NREQ; ++i) {
        int32_t nblk = 0;
        kv_group g = {i % n, 1};
        CHECK(kv_blocks_for(&geo, T[i], 1, &nblk));
        CHECK(kv_alloc(c, g, nblk, src_ids[i]));
        kv_request r = {(int64_t)i, T[i], g, src_ids[i], nblk, {0, n}, NULL, NULL};
        fwd[i] = r;
    }

    cudaStream_t stream;
    CUDA(cudaStreamCreate(&stream));
    const int64_t timeout_ns = 30000000000LL;
    int32_t* status = NULL;
    CUDA(cudaMalloc((void**)&status, sizeof(int32_t)));
    CUDA(cudaMemset(status, 0, sizeof(int32_t)));

    /* DP_n -> TP_n, this process's share in one call (device barrier: the
     * 1st on these counters, target n) */
    hb_ctx hb = {sh, n, &gen};
    kv_plan* p1 = NULL;
    if (own_gpu)
        CHECK(kv_switch_range(c, fwd, NREQ, rank, rank + 1, ctr, n, rank, (uint64_t)n, timeout_ns, status, stream,
                              &p1));
    else
        CHECK(kv_switch_range_host(c, fwd, NREQ, rank, rank + 1, host_barrier_cb, &hb, stream, &p1));
    int32_t ptr[NREQ + 1], tp_ids[NREQ * NB];
    CHECK(kv_plan_dst_tables(p1, ptr, tp_ids));
    for (int i = 0; i < NREQ; ++i) {
        kv_request r = {(int64_t)i, T[i], {0, n}, tp_ids + ptr[i], ptr[i + 1] - ptr[i], {i % n, 1}, NULL, NULL};
        back[i] = r;
    }
    /* and back, TP_n -> DP_n (2nd barrier: target 2n) */
    kv_plan* p2 = NULL;
    if (own_gpu)
        CHECK(kv_switch_range(c, back, NREQ, rank, rank + 1, ctr, n, rank, 2 * (uint64_t)n, timeout_ns, status,
                              stream, &p2));
    else
        CHECK(kv_switch_range_host(c, back, NREQ, rank, rank + 1, host_barrier_cb, &hb, stream, &p2));
    int32_t st = 0;
    CUDA(cudaMemcpy(&st, status, sizeof st, cudaMemcpyDeviceToHost));
    if (st) {
        fprintf(stderr, "rank %d: device barrier timed out\n", rank);
        return 1;
    }
    int32_t ptr2[NREQ + 1], dp_ids[NREQ * NB];
    CHECK(kv_plan_dst_tables(p2, ptr2, dp_ids));

    /* round trip: this process's requests, every layer, whole blocks */
    uint8_t* now = (uint8_t*)malloc(pool_bytes);
    CUDA(cudaMemcpy(now, pool, pool_bytes, cudaMemcpyDeviceToHost));
    int bad = 0, checked = 0;
    for (int i = 0; i < NREQ; ++i) {
        if (i % n != rank) continue;
        for (int k = 0; k < ptr2[i + 1] - ptr2[i]; ++k)
            for (int l = 0; l < L; ++l) {
                const size_t a = ((size_t)l * NB + (size_t)src_ids[i][k]) * (size_t)M;
                const size_t b = ((size_t)l * NB + (size_t)dp_ids[ptr2[i] + k]) * (size_t)M;
                bad += memcmp(host + a, now + b, (size_t)M) != 0;
                ++checked;
            }
    }
    /* nobody unmaps a peer's pool while another process may still touch it */
    host_barrier(sh, n, &gen);
    kv_plan_destroy(p1);
    kv_plan_destroy(p2);
    kv_cache_destroy(c);
    for (int g = 0; g < n; ++g)
        if (g != rank) {
            CHECK(kv_ipc_close((uint8_t*)bases[g * L] , sh->pool_off[g]));
            CHECK(kv_ipc_close(ctr[g], sh->flag_off[g]));
        }
    host_barrier(sh, n, &gen);
    printf("rank %d: %d blocks checked, %d differ\n", rank, checked, bad);
    return bad ? 1 : 0;
}

int main(int argc, char** argv) {
    int n = argc > 1 ? atoi(argv[1]) : 2;
    if (n < 2 || n > MAXN || (n & (n - 1))) {
        fprintf(stderr, "usage: %s [2|4|8]\n", argv[0]);
        return 2;
    }
    shared_t* sh = (shared_t*)mmap(NULL, sizeof(shared_t), PROT_READ | PROT_WRITE, MAP_SHARED | MAP_ANONYMOUS, -1, 0);
    if (sh == MAP_FAILED) return 2;
    memset(sh, 0, sizeof *sh);
    pid_t pids[MAXN];
    for (int r = 0; r < n; ++r) {  /* fork before any CUDA call: each child makes its own context */
        pids[r] = fork();
        if (pids[r] == 0) {
            int rc = run_rank(r, n, sh);
            if (rc) sh->failed = 1;
            fflush(stdout);
            _exit(rc);
        }
    }
    int ok = 1;
    for (int r = 0; r < n; ++r) {
        int status = 0;
        waitpid(pids[r], &status, 0);
        ok = ok && WIFEXITED(status) && WEXITSTATUS(status) == 0;
    }
    printf(ok ? "multi-process round-trip byte-exact (%d processes, kv_switch_range / kv_switch_range_host)\n"
              : "FAILED (%d processes)\n", n);
    return ok ? 0 : 1;
}
