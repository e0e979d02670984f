// stage_kernels.cuh -- one kernel per stage of the TOF loop, state in HBM.
//
// Used by (a) the stage entry points of the C ABI (sf_init_swarm, sf_step,
// sf_eval_path_rows, sf_eval_bench_rows, sf_update_bests), which let the
// parity tests check every stage on identical inputs, and (b) the large-swarm
// driver (big_swarm.cu) for swarms that do not fit a cluster's shared memory
// (config 4: 65,536 particles x 128 dims x 4,096 obstacle edges).
//
// Arrays are T = float (FP32 engine) or double (FP64 parity engine); `fp64`
// selects the instantiation.  Rows are the device's slice
// [row_begin, row_begin + rows) of the reference's row-major (g, n) order;
// every random draw is indexed by the GLOBAL row so a sharded swarm draws
// exactly what the unsharded one draws.
#pragma once
#include <cstddef>
#include <cstdint>

namespace sepso {

struct StageShape {
    int G, N, D;
    int row_begin, rows;
};

// Iteration state shared by the bests/finish kernels (device resident).
struct IterState {
    double tbest_f;          // population best fitness (as double)
    int tbest_q;             // Q of the population best
    int tbest_group;         // group of the population best
    int stop, truncated, status, k_done;
    int nonfinite_row;       // INT_MAX when all finite
    int win_len, win_head;
    int pad[2];
};

// words != nullptr: draw i is words[i - wbase] (a pre-generated mt19937_64
// window, stage_mt_fill); otherwise the Philox word of index i.
int stage_init(bool fp64, const StageShape& s, const double* hypers, const void* lo,
               const void* hi, uint64_t seed, uint64_t first_draw, const double* prev, int warm,
               double pi_radius, void* x, void* v, void* pbest_x, void* stream,
               const unsigned long long* words = nullptr, long long wbase = 0);

// imp != nullptr: rows with imp[row] set improved their pbest this iteration
// and their pbest_x copy was deferred (stage_pbest_partials with imp): the
// step reads pbest_x from x and writes it to pbest_x.
int stage_step(bool fp64, const StageShape& s, const double* hypers, const void* lo,
               const void* hi, void* x, void* v, void* pbest_x, const void* gbest_x,
               const void* tbest_x, uint64_t seed, uint64_t first_draw, int k, int total,
               const IterState* gate, void* stream, const unsigned long long* words = nullptr,
               long long wbase = 0, const unsigned char* imp = nullptr);

// Persisted mt19937_64 generator for the staged path (device memory).
struct MtPersist {
    unsigned long long st[624];     // the two latest blocks (mt19937.cuh MtState pair)
    long long blocks;
};
// Generate words [from, upto) of the stream, untempered (consumers apply
// mt_temper), into out[w - from] (one CTA);
// earlier words are skipped.  reseed restarts the generator from `seed`.
int stage_mt_fill(MtPersist* g, unsigned long long seed, bool reseed, long long from,
                  long long upto, unsigned long long* out, void* stream);
// The same fill of [0, upto) from a fresh seed in 2^levels parallel segments of
// Q words (Q a multiple of 624, Q * 2^levels >= upto) started from jumped
// states (mt_jump.cpp); terms = level j's polynomial mt_jump_ladder(Q, levels)[j]
// as the sorted list of its nterms[j] (host array) exponents, at terms + j *
// kMtDegree on the device; states = scratch for 2^levels x 312 words.
// Identical words and final g.
int stage_mt_fill_parallel(MtPersist* g, unsigned long long seed, long long upto, unsigned long long* out,
                           unsigned long long* states, const unsigned short* terms, const int* nterms, int levels,
                           long long Q, void* stream);

int stage_eval_path(bool fp64, const unsigned char* world, int max_obs, int max_verts,
                    int off_offsets, int off_verts, int D, int rows, const void* x,
                    double alpha, double beta, void* fit, int* q, const IterState* gate,
                    void* stream);

int stage_eval_bench(bool fp64, int kind, int D, int rows, const void* x, void* fit,
                     int* q, const IterState* gate, void* stream);

// pbest update + per-group partial (value, global row, q) for the local groups.
// imp != nullptr: improved rows are flagged in imp instead of copying x into
// pbest_x (the copy happens in the next stage_step / stage_group_bests with imp).
int stage_pbest_partials(bool fp64, const StageShape& s, const void* x, const void* fit,
                         const int* q, void* pbest_x, void* pbest_f, int* pbest_q,
                         IterState* st, void* part_f, int* part_row, int* part_q,
                         const IterState* gate, void* stream, unsigned char* imp = nullptr);

// gbest (local groups) from the partials; writes this device's tbest
// candidate: best local group (value, q, global group) + its x.
int stage_group_bests(bool fp64, const StageShape& s, const void* part_f, const int* part_row,
                      const int* part_q, const void* pbest_x, void* gbest_x, void* gbest_f,
                      int* gbest_q, void* cand /*packed candidate*/, const IterState* gate,
                      void* stream, const IterState* st = nullptr, const void* x = nullptr,
                      const unsigned char* imp = nullptr);

// Scan n_cand candidates (ascending group order) for tbest, push the window,
// evaluate AT; trace[k-1] = tbest_f.  cand layout: see big_swarm.cu.
int stage_finish(bool fp64, int D, const void* cands, int n_cand, void* tbest_x, IterState* st,
                 double* win, int tw, int auto_truncate, double delta, int k, int cap,
                 double* trace, void* stream);

size_t cand_bytes(bool fp64, int D);

} // namespace sepso
