/*
 * c_switch_demo.c -- the C ABI used from plain C (no Python, no torch).
 *
 * Allocates two paged KV pools with cudaMalloc (virtual ranks on one GPU),
 * registers three live DP requests, switches them DP2 -> TP2 with
 * kv_plan_switch / kv_reshard / kv_remap_block_tables and back with the
 * one-call kv_switch, then DP2 -> TP2 -> DP2 again through kv_switch_waves
 * (a memory-bounded switch in one call, one request per wave), and checks
 * the round trip: every source block of every layer is back, byte for byte, in the
 * blocks of the final DP tables (a DP block holds B tokens of all heads, so
 * whole blocks round-trip).  Exit code 0 on success.
 *
 * Build: nvcc -O2 -o c_switch_demo c_switch_demo.c -I../include -L../paper_2602_22593_b200/lib -lflykv
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "flykv.h"

#define CHECK(x)                                                                  \
    do {                                                                          \
        kv_status s_ = (x);                                                       \
        if (s_ != KV_OK) {                                                        \
            fprintf(stderr, "%s:%d %s -> %s: %s\n", __FILE__, __LINE__, #x,       \
                    kv_strerror(s_), kv_last_error());                            \
            return 1;                                                             \
        }                                                                         \
    } while (0)

#define CUDA(x)                                                                   \
    do {                                                                          \
        cudaError_t e_ = (x);                                                     \
        if (e_ != cudaSuccess) {                                                  \
            fprintf(stderr, "%s -> %s\n", #x, cudaGetErrorString(e_));            \
            return 1;                                                             \
        }                                                                         \
    } while (0)

enum { L = 3, NB = 64, NREQ = 3 };

static int switch_all(kv_cache* c, kv_request* r, int n, int32_t** out_tabs, int32_t* out_len) {
    kv_plan* p = NULL;
    int g, i;
    CHECK(kv_plan_switch(c, r, n, &p));
    CHECK(kv_reshard(p, -1, NULL));
    for (g = 0; g < 2; ++g) {
        int32_t nres = 0, nids = 0;
        int32_t *rp, *ids, *meta;
        CHECK(kv_plan_resident(p, g, &nres, &nids));
        CUDA(cudaMalloc((void**)&rp, (nres + 1) * 4));
        CUDA(cudaMalloc((void**)&ids, (nids + 1) * 4));
        CUDA(cudaMalloc((void**)&meta, (4 * nres + 1) * 4));
        CHECK(kv_remap_block_tables(p, g, rp, ids, meta, NULL));
        CUDA(cudaDeviceSynchronize());
        cudaFree(rp);
        cudaFree(ids);
        cudaFree(meta);
    }
    {
        int32_t ptr[NREQ + 1];
        int32_t all[4 * NB];
        CHECK(kv_plan_dst_tables(p, ptr, all));
        for (i = 0; i < n; ++i) {
            out_len[i] = ptr[i + 1] - ptr[i];
            memcpy(out_tabs[i], all + ptr[i], (size_t)out_len[i] * 4);
        }
    }
    kv_plan_destroy(p);
    return 0;
}

/* The same switch through kv_switch: one call plans, moves, remaps and
 * reads every pool's new table back; kv_plan_tables exposes them. */
static int switch_one_call(kv_cache* c, kv_request* r, int n, int32_t** out_tabs, int32_t* out_len) {
    kv_plan* p = NULL;
    int g, i;
    CHECK(kv_switch(c, r, n, NULL, &p));
    for (g = 0; g < 2; ++g) {
        const int32_t *rp, *ids, *meta;
        int32_t nres = 0, nids = 0;
        CHECK(kv_plan_resident(p, g, &nres, &nids));
        CHECK(kv_plan_tables(p, g, 0, &rp, &ids, &meta));
        if (rp[0] != 0 || rp[nres] != nids) {
            fprintf(stderr, "GPU %d: bad CSR table from kv_switch\n", g);
            return 1;
        }
        for (i = 0; i < nres; ++i)  /* meta: plan index, B(p), H_loc, first head */
            if (meta[4 * i + 1] != 16 || meta[4 * i + 2] != 4) {
                fprintf(stderr, "GPU %d: bad per-request meta\n", g);
                return 1;
            }
    }
    {
        int32_t ptr[NREQ + 1];
        int32_t all[4 * NB];
        CHECK(kv_plan_dst_tables(p, ptr, all));
        for (i = 0; i < n; ++i) {
            out_len[i] = ptr[i + 1] - ptr[i];
            memcpy(out_tabs[i], all + ptr[i], (size_t)out_len[i] * 4);
        }
    }
    kv_plan_destroy(p);
    return 0;
}

/* A memory-bounded switch in one call: kv_switch_waves schedules the waves
 * (max_wave_bytes = 1: one request per wave; split: the cap also cuts each
 * request into block-aligned token pieces, a few waves each) and runs
 * them back to back; a request's table is the concatenation of its pieces'
 * tables in wave order. */
static int switch_waves(kv_cache* c, kv_request* r, int n, int split, int32_t** out_tabs, int32_t* out_len) {
    kv_piece pcs[64];
    kv_plan* plans[64];
    int32_t np = 0, nw = 0, w, i, k = 0;
    CHECK(kv_switch_waves(c, r, n, 1, split, NULL, 64, pcs, &np, plans, &nw));
    if (split ? nw < n : nw != n) {  /* split: the byte cap also cuts requests into pieces */
        fprintf(stderr, "unexpected wave count %d for %d requests\n", nw, n);
        return 1;
    }
    for (i = 0; i < n; ++i) out_len[i] = 0;
    for (w = 0; w < nw; ++w) {
        int32_t ptr[65], cnt = 0, j;
        int32_t* all;
        while (k + cnt < np && pcs[k + cnt].wave == w) ++cnt;
        CHECK(kv_plan_dst_tables(plans[w], ptr, NULL));
        all = (int32_t*)malloc((size_t)(ptr[cnt] > 0 ? ptr[cnt] : 1) * 4);
        CHECK(kv_plan_dst_tables(plans[w], ptr, all));
        for (j = 0; j < cnt; ++j) {
            const int q = pcs[k + j].req;
            memcpy(out_tabs[q] + out_len[q], all + ptr[j], (size_t)(ptr[j + 1] - ptr[j]) * 4);
            out_len[q] += ptr[j + 1] - ptr[j];
        }
        free(all);
        kv_plan_destroy(plans[w]);
        k += cnt;
    }
    return 0;
}

int main(void) {
    kv_geometry geo = {L, 4, 64, 16, 2};
    int64_t M = 0;
    int32_t hl, bt;
    void* pool[2];
    void* bases[2 * L];
    int32_t nb[2] = {NB, NB};
    int32_t degrees[1] = {2};
    kv_cache* c = NULL;
    int g, l, i, k;
    const int32_t T[NREQ] = {40, 129, 7};
    int32_t tab0_store[NREQ][NB], tab1_store[NREQ][NB], tab2_store[NREQ][NB], tab3_store[NREQ][NB],
        tab4_store[NREQ][NB];
    int32_t* tab0[NREQ];
    int32_t* tab1[NREQ];
    int32_t* tab2[NREQ];
    int32_t* tab3[NREQ];
    int32_t* tab4[NREQ];
    int32_t len0[NREQ], len1[NREQ], len2[NREQ], len3[NREQ], len4[NREQ];
    uint8_t *before, *after;
    size_t bytes;
    kv_request req[NREQ];

    CHECK(kv_layout(&geo, 1, &hl, &bt, &M));
    bytes = (size_t)L * NB * M;
    for (g = 0; g < 2; ++g) {
        uint8_t* h = (uint8_t*)malloc(bytes);
        size_t b;
        for (b = 0; b < bytes; ++b) h[b] = (uint8_t)(b * 2654435761u >> 13) ^ (uint8_t)(g * 77);
        CUDA(cudaMalloc(&pool[g], bytes));
        CUDA(cudaMemcpy(pool[g], h, bytes, cudaMemcpyHostToDevice));
        free(h);
        for (l = 0; l < L; ++l) bases[g * L + l] = (char*)pool[g] + (size_t)l * NB * M;
    }
    CHECK(kv_cache_create(&geo, 2, nb, bases, degrees, 1, &c));
    for (i = 0; i < NREQ; ++i) {  /* DP: request i lives on GPU i % 2 */
        kv_group src = {i % 2, 1};
        tab0[i] = tab0_store[i];
        tab1[i] = tab1_store[i];
        tab2[i] = tab2_store[i];
        tab3[i] = tab3_store[i];
        tab4[i] = tab4_store[i];
        CHECK(kv_blocks_for(&geo, T[i], 1, &len0[i]));
        CHECK(kv_alloc(c, src, len0[i], tab0[i]));
    }
    before = (uint8_t*)malloc(2 * bytes);
    after = (uint8_t*)malloc(2 * bytes);
    for (g = 0; g < 2; ++g) CUDA(cudaMemcpy(before + g * bytes, pool[g], bytes, cudaMemcpyDeviceToHost));

    for (i = 0; i < NREQ; ++i) {  /* DP2 -> TP2 */
        kv_group src = {i % 2, 1}, dst = {0, 2};
        kv_request r = {100 + i, T[i], src, tab0[i], len0[i], dst};
        req[i] = r;
    }
    if (switch_all(c, req, NREQ, tab1, len1)) return 1;
    for (i = 0; i < NREQ; ++i) {  /* TP2 -> DP2 */
        kv_group src = {0, 2}, dst = {i % 2, 1};
        kv_request r = {100 + i, T[i], src, tab1[i], len1[i], dst};
        req[i] = r;
    }
    if (switch_one_call(c, req, NREQ, tab2, len2)) return 1;
    for (i = 0; i < NREQ; ++i) {  /* DP2 -> TP2 again, one request per wave */
        kv_group src = {i % 2, 1}, dst = {0, 2};
        kv_request r = {100 + i, T[i], src, tab2[i], len2[i], dst};
        req[i] = r;
    }
    if (switch_waves(c, req, NREQ, 0, tab3, len3)) return 1;
    for (i = 0; i < NREQ; ++i) {  /* and back, pieces allowed */
        kv_group src = {0, 2}, dst = {i % 2, 1};
        kv_request r = {100 + i, T[i], src, tab3[i], len3[i], dst};
        req[i] = r;
    }
    if (switch_waves(c, req, NREQ, 1, tab4, len4)) return 1;  /* tables = concatenated pieces */

    for (g = 0; g < 2; ++g) CUDA(cudaMemcpy(after + g * bytes, pool[g], bytes, cudaMemcpyDeviceToHost));
    for (i = 0; i < NREQ; ++i) {
        g = i % 2;
        if (len4[i] != len0[i]) { fprintf(stderr, "length mismatch\n"); return 1; }
        for (l = 0; l < L; ++l)
            for (k = 0; k < len0[i]; ++k) {
                const uint8_t* a = before + g * bytes + ((size_t)l * NB + tab0[i][k]) * M;
                const uint8_t* b = after + g * bytes + ((size_t)l * NB + tab4[i][k]) * M;
                if (memcmp(a, b, (size_t)M)) {
                    fprintf(stderr, "request %d layer %d block %d differs\n", i, l, k);
                    return 1;
                }
            }
    }
    {
        int32_t f0, f1;
        CHECK(kv_free_count(c, 0, &f0));
        CHECK(kv_free_count(c, 1, &f1));
        printf("c_switch_demo ok: %d requests DP2->TP2 (step by step) ->DP2 (kv_switch) ->TP2 ->DP2 (kv_switch_waves) "
               "round-trip byte-exact; free blocks %d/%d; "
               "%lld kernel launches\n", NREQ, f0, f1, (long long)kv_launch_count());
    }
    kv_cache_destroy(c);
    cudaFree(pool[0]);
    cudaFree(pool[1]);
    free(before);
    free(after);
    return 0;
}
