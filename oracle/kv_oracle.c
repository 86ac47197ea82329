/*
 * kv_oracle.c -- ORACLE: plain, slow, obviously-correct CPU re-layout of a
 * paged KV cache between DP and TP layouts (Flying Serving, arXiv 2602.22593).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, the
 * smoke() check in __graft_entry__.py and bench.py's cpu_baseline /
 * --impl reference legs may load it.  It shares no code, header, table or
 * constant generator with the CUDA path under paper_2602_22593_b200/ and
 * include/; it does not include flykv.h.
 *
 * Citations: P:n = line n of the paper's LaTeX; R<n> = reading n
 * listed in DESIGN.md section 3 ("Readings of the paper").
 *
 * What it computes:
 *   for each request, in caller order:
 *     1. allocate n1 = ceil(T / B(p1)) block IDs: the lowest IDs that are
 *        free on EVERY GPU of the destination group (R6 uniform IDs, R8
 *        lowest-first, Alg.1 "KVCacheMgr.Allocate" P:493);
 *     2. for every layer l, kv in {K,V}, head h and token slot
 *        t in [0, ceil(T/B)*B) (R9 whole B-token atoms) copy the d*e bytes
 *        of (l,kv,h,t) from the lowest source replica of head h to every
 *        destination replica of head h;
 *   then free every source block ID (R13: after all copies).
 *   Requests whose src group == dst group are no-ops (R12).
 *
 * Layout of one block of one layer at degree p (R4, north_star):
 *   [K/V][H_loc(p)][B(p)][d] elements of e bytes, K first;
 *   H_loc(p) = H/p if p <= H else 1                (Eq.3, R2)
 *   B(p)     = B * H / H_loc(p)  (= p*B when p | H) (Eq.2, R2)
 *   M        = 2 * H_loc(p) * B(p) * d * e  = 2*H*B*d*e for every p
 *                                               (M_block eq. P:338-340, R1)
 * Head ownership at degree p in group [g0, g0+p) (Eq.1, R3):
 *   p <= H: head h lives on rank h / H_loc(p), local index h % H_loc(p)
 *   p >  H: head h lives on ranks h*(p/H) ... h*(p/H)+p/H-1, local index 0
 * Pools (test-harness convention): GPU g's pool is one host buffer laid out
 * [L][num_blocks[g]][M] bytes.
 *
 * Build: gcc -O2 -shared -fPIC -o liboracle_kv.so kv_oracle.c
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int32_t L;  /* layers */
    int32_t H;  /* KV heads */
    int32_t d;  /* head_dim */
    int32_t B;  /* B_base: tokens per block in DP mode */
    int32_t e;  /* bytes per element (2 = bf16) */
} or_geom;

/* ---------------- layout parameters (Eq.2, Eq.3, M_block eq.) ---------- */

/* H_loc(p): heads held per rank.  Eq.3 H_req = H_base / N_eng;
 * GQA replication when p > H keeps one head per rank (R2). */
int32_t or_h_loc(const or_geom* g, int32_t p) {
    if (p <= g->H) return g->H / p;
    return 1;
}

/* B(p): tokens per block.  Eq.2 B(p) = p * B_base when p | H;
 * under replication B(p) = H * B_base so that M stays constant (R2). */
int32_t or_block_tokens(const or_geom* g, int32_t p) {
    return g->B * (g->H / or_h_loc(g, p));
}

/* M: bytes of one block of one layer; K and V halves (R1). */
int64_t or_block_bytes(const or_geom* g) {
    return (int64_t)2 * g->H * g->B * g->d * g->e;
}

/* Number of blocks a T-token request occupies at degree p (SPEC allocate:
 * ceil(tokens / B(p))). */
int32_t or_num_blocks(const or_geom* g, int32_t T, int32_t p) {
    int32_t bp = or_block_tokens(g, p);
    return (T + bp - 1) / bp;
}

/* How many ranks of a degree-p group hold head h. */
int32_t or_replicas(const or_geom* g, int32_t p) {
    if (p <= g->H) return 1;
    return p / g->H;
}

/* j-th rank (0 <= j < replicas) of a degree-p group that holds head h. */
int32_t or_owner_rank(const or_geom* g, int32_t p, int32_t h, int32_t j) {
    if (p <= g->H) return h / or_h_loc(g, p);
    return h * (p / g->H) + j;
}

/* Index of head h inside its owner's block. */
int32_t or_local_head(const or_geom* g, int32_t p, int32_t h) {
    if (p <= g->H) return h % or_h_loc(g, p);
    return 0;
}

/* First global head held by rank r of a degree-p group. */
int32_t or_first_head(const or_geom* g, int32_t p, int32_t r) {
    if (p <= g->H) return r * or_h_loc(g, p);
    return r / (p / g->H);
}

/* Rank-ID assignment ("the Manager assigns each engine a unique
 * rank ID r in [0, m-1]"): rid[m] is the rank ID of member engine g0 + m of
 * the group; NULL means the identity (R3).  The member holding rank ID r. */
int32_t or_member(const int32_t* rid, int32_t p, int32_t r) {
    int32_t m;
    if (!rid) return r;
    for (m = 0; m < p; m++)
        if (rid[m] == r) return m;
    return -1;
}

/* Where the d*e bytes of (kv, h, token t) of a request live, for replica j:
 * GPU index and byte offset inside that GPU's layer region (add
 * l * num_blocks * M for layer l).  tab = the request's block table at
 * degree p, group starting at GPU g0, rank IDs rid (NULL = identity). */
void or_locate_rid(const or_geom* g, int32_t g0, int32_t p, const int32_t* rid, const int32_t* tab,
                   int32_t kv, int32_t h, int32_t t, int32_t j,
                   int32_t* gpu, int64_t* off) {
    int32_t bp = or_block_tokens(g, p);
    int32_t hl = or_h_loc(g, p);
    int64_t row = (int64_t)g->d * g->e;           /* bytes of one token of one head */
    int64_t M = or_block_bytes(g);
    int32_t block = tab[t / bp];
    int32_t slot = t % bp;
    int32_t lh = or_local_head(g, p, h);
    *gpu = g0 + or_member(rid, p, or_owner_rank(g, p, h, j));
    *off = (int64_t)block * M                   /* block                   */
         + (int64_t)kv * (M / 2)                /* K half, then V half     */
         + ((int64_t)lh * bp + slot) * row;     /* [H_loc][B(p)][d]        */
    (void)hl;
}

void or_locate(const or_geom* g, int32_t g0, int32_t p, const int32_t* tab,
               int32_t kv, int32_t h, int32_t t, int32_t j,
               int32_t* gpu, int64_t* off) {
    or_locate_rid(g, g0, p, NULL, tab, kv, h, t, j, gpu, off);
}

/* ---------------- the switch ------------------------------------------- */

/* A request is a no-op only if it stays in the same group with the same
 * rank IDs (R12, R19). */
static int same_layout(int32_t g0a, int32_t pa, const int32_t* ra, int32_t g0b, int32_t pb, const int32_t* rb) {
    int32_t m;
    if (g0a != g0b || pa != pb) return 0;
    for (m = 0; m < pa; m++)
        if ((ra ? ra[m] : m) != (rb ? rb[m] : m)) return 0;
    return 1;
}

enum { OR_OK = 0, OR_OUT_OF_BLOCKS = 6, OR_INVALID = 1 };

/*
 * or_switch: re-lay-out every listed request from its source group/layout
 * to its destination group/layout.
 *
 *   pools[gpu]       host buffer [L][num_blocks[gpu]][M] bytes, modified
 *   do_copy          0: allocation and release only (pools may be NULL)
 *   held[gpu][b]     1 if block b of gpu is held by any live request
 *                    (moving or not); updated: dst IDs set, src IDs cleared
 *   request i: T[i] tokens, source group [src_g0[i], +src_p[i]) with table
 *              src_ids[src_ptr[i] .. src_ptr[i+1]), destination group
 *              [dst_g0[i], +dst_p[i])
 *   out: dst_ptr[n+1], dst_ids[<= dst_cap]
 * Returns OR_OK, or OR_OUT_OF_BLOCKS (state then partially modified -- the
 * oracle is not transactional; callers discard it).
 */
int32_t or_switch(const or_geom* g, int32_t n_gpus, const int32_t* num_blocks,
                  uint8_t** pools, int32_t do_copy, uint8_t** held, int32_t n_reqs,
                  const int32_t* T, const int32_t* src_g0, const int32_t* src_p,
                  const int32_t* src_ptr, const int32_t* src_ids,
                  const int32_t* dst_g0, const int32_t* dst_p,
                  const int32_t* const* src_rid, const int32_t* const* dst_rid,
                  int32_t* dst_ptr, int32_t* dst_ids, int32_t dst_cap) {
    int64_t M = or_block_bytes(g);
    int64_t row = (int64_t)g->d * g->e;
    int32_t i, l, kv, h, t, j, b, k;
    (void)n_gpus;

    /* step 1 and 2, request by request */
    dst_ptr[0] = 0;
    for (i = 0; i < n_reqs; i++) {
        const int32_t* tab0 = src_ids + src_ptr[i];
        int32_t* tab1 = dst_ids + dst_ptr[i];
        const int32_t* rid0 = src_rid ? src_rid[i] : NULL;
        const int32_t* rid1 = dst_rid ? dst_rid[i] : NULL;
        int same = same_layout(src_g0[i], src_p[i], rid0, dst_g0[i], dst_p[i], rid1);
        int32_t n1 = same ? (src_ptr[i + 1] - src_ptr[i])
                          : or_num_blocks(g, T[i], dst_p[i]);
        if (dst_ptr[i] + n1 > dst_cap) return OR_INVALID;
        dst_ptr[i + 1] = dst_ptr[i] + n1;
        if (same) {                                   /* no-op (R12) */
            for (k = 0; k < n1; k++) tab1[k] = tab0[k];
            continue;
        }
        /* 1. allocate: lowest IDs free on every destination GPU (R6, R8) */
        int32_t nb = num_blocks[dst_g0[i]];
        for (k = 1; k < dst_p[i]; k++)
            if (num_blocks[dst_g0[i] + k] < nb) nb = num_blocks[dst_g0[i] + k];
        k = 0;
        for (b = 0; b < nb && k < n1; b++) {
            int free_everywhere = 1;
            int32_t r;
            for (r = 0; r < dst_p[i]; r++)
                if (held[dst_g0[i] + r][b]) free_everywhere = 0;
            if (free_everywhere) {
                for (r = 0; r < dst_p[i]; r++) held[dst_g0[i] + r][b] = 1;
                tab1[k++] = b;
            }
        }
        if (k < n1) return OR_OUT_OF_BLOCKS;

        /* 2. copy, token by token (R9: whole B-token atoms) */
        if (!do_copy) continue;  /* tables-only mode (full-size sampled checks) */
        int32_t t_end = ((T[i] + g->B - 1) / g->B) * g->B;
        int32_t reps = or_replicas(g, dst_p[i]);
        for (l = 0; l < g->L; l++)
            for (kv = 0; kv < 2; kv++)
                for (h = 0; h < g->H; h++)
                    for (t = 0; t < t_end; t++) {
                        int32_t sg, dg;
                        int64_t so, dof;
                        /* lowest source replica (R10) */
                        or_locate_rid(g, src_g0[i], src_p[i], rid0, tab0, kv, h, t, 0, &sg, &so);
                        const uint8_t* src = pools[sg] + (int64_t)l * num_blocks[sg] * M + so;
                        for (j = 0; j < reps; j++) {
                            or_locate_rid(g, dst_g0[i], dst_p[i], rid1, tab1, kv, h, t, j, &dg, &dof);
                            uint8_t* dst = pools[dg] + (int64_t)l * num_blocks[dg] * M + dof;
                            memcpy(dst, src, (size_t)row);
                        }
                    }
    }

    /* release every source block (after all copies, R13) */
    for (i = 0; i < n_reqs; i++) {
        int same = same_layout(src_g0[i], src_p[i], src_rid ? src_rid[i] : NULL,
                               dst_g0[i], dst_p[i], dst_rid ? dst_rid[i] : NULL);
        int32_t r;
        if (same) continue;
        for (k = src_ptr[i]; k < src_ptr[i + 1]; k++)
            for (r = 0; r < src_p[i]; r++) held[src_g0[i] + r][src_ids[k]] = 0;
    }
    return OR_OK;
}

/*
 * or_tables: the per-GPU block table after the switch ("request -> block
 * IDs" logical table, with per-request capacity/stride P:365).
 * For GPU gpu, list the requests whose destination group contains gpu, in
 * request order:
 *   req_ptr[0..n_res], ids[...]: CSR of their destination tables
 *   meta[4*r .. 4*r+3] = { request index, B(p1), H_loc(p1), first head }
 * Returns n_res.
 */
int32_t or_tables(const or_geom* g, int32_t gpu, int32_t n_reqs,
                  const int32_t* dst_g0, const int32_t* dst_p, const int32_t* const* dst_rid,
                  const int32_t* dst_ptr, const int32_t* dst_ids,
                  int32_t* req_ptr, int32_t* ids, int32_t* meta) {
    int32_t i, k, n = 0, pos = 0;
    req_ptr[0] = 0;
    for (i = 0; i < n_reqs; i++) {
        if (gpu < dst_g0[i] || gpu >= dst_g0[i] + dst_p[i]) continue;
        for (k = dst_ptr[i]; k < dst_ptr[i + 1]; k++) ids[pos++] = dst_ids[k];
        meta[4 * n + 0] = i;
        meta[4 * n + 1] = or_block_tokens(g, dst_p[i]);
        meta[4 * n + 2] = or_h_loc(g, dst_p[i]);
        {
            const int32_t* rid = dst_rid ? dst_rid[i] : NULL;
            int32_t m = gpu - dst_g0[i];
            meta[4 * n + 3] = or_first_head(g, dst_p[i], rid ? rid[m] : m);
        }
        n++;
        req_ptr[n] = pos;
    }
    return n;
}

/*
 * or_atom_map: every (layer, kv, head, chunk, replica) atom of one request
 * as (source GPU, source byte offset in that GPU's pool, destination GPU,
 * destination byte offset), offsets including the layer region
 * (l * num_blocks * M).  Enumerates exactly the copies or_switch performs,
 * one B-token atom per entry (R9), in the order l, kv, h, c, j.  Used for
 * full-size checks of the device result.  Returns the number of entries.
 */
int64_t or_atom_map(const or_geom* g, const int32_t* num_blocks, int32_t T,
                    int32_t src_g0, int32_t src_p, const int32_t* rid0, const int32_t* tab0,
                    int32_t dst_g0, int32_t dst_p, const int32_t* rid1, const int32_t* tab1,
                    int32_t* src_gpu, int64_t* src_off, int32_t* dst_gpu, int64_t* dst_off) {
    int64_t M = or_block_bytes(g);
    int32_t C = (T + g->B - 1) / g->B;
    int32_t reps = or_replicas(g, dst_p);
    int64_t n = 0;
    int32_t l, kv, h, c, j;
    for (l = 0; l < g->L; l++)
        for (kv = 0; kv < 2; kv++)
            for (h = 0; h < g->H; h++)
                for (c = 0; c < C; c++)
                    for (j = 0; j < reps; j++) {
                        int32_t sg, dg;
                        int64_t so, dof;
                        or_locate_rid(g, src_g0, src_p, rid0, tab0, kv, h, c * g->B, 0, &sg, &so);
                        or_locate_rid(g, dst_g0, dst_p, rid1, tab1, kv, h, c * g->B, j, &dg, &dof);
                        src_gpu[n] = sg;
                        src_off[n] = (int64_t)l * num_blocks[sg] * M + so;
                        dst_gpu[n] = dg;
                        dst_off[n] = (int64_t)l * num_blocks[dg] * M + dof;
                        n++;
                    }
    return n;
}
