/*
 * llama_ref — CPU oracle of the chunked-prefill compute side (TEST
 * INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this).
 *
 * The reference has no transformer — its compute side sleeps for a modeled
 * latency (reference proj/src/compute.cpp:48-49). This file is
 * the standard Llama-3 block restated in plain C, fp32 arithmetic over the
 * same seeded bf16 weights the GPU generates (weight_value() is bit-identical
 * to paper_2410_03065_b200/csrc/cuda/elementwise.cuh), at the same rounding
 * points (bf16 activations into each projection, bf16 K/V/Q after RoPE).
 * Transformer arithmetic is PARITY UNPINNED by the reference;
 * tolerances are stated in tests/test_gpu_parity.py.
 *
 * KV cache layout (fp32 values of the bf16 cache): [layer][K|V][kv_head][pos][head_dim].
 */
#ifndef LLAMA_REF_H_
#define LLAMA_REF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ref_config {
  int n_layers, hidden, n_heads, n_kv_heads, head_dim, ffn, vocab;
  float rope_theta, rms_eps;
  unsigned long long seed;
  int threads; /* OpenMP threads, 0 = default */
} ref_config;

typedef struct ref_model ref_model;

ref_model* ref_create(const ref_config* cfg, long long max_tokens, long long cache_weight_bytes);
void ref_destroy(ref_model* m);

/* One chunk: tokens[len] at absolute positions [start, start+len). */
int ref_begin_chunk(ref_model* m, const int32_t* tokens, long long start, int len);
int ref_run_layers(ref_model* m, int layer_begin, int layer_end);
/* Final RMSNorm of hidden row `row` of the current chunk + LM head -> logits[vocab]. */
int ref_final_logits(ref_model* m, int row, float* logits);
/* First-token step when the tail was loaded: q-only pass of token at pos T-1
 * over the cache (its own K/V already cached), then the LM head. */
int ref_last_token_logits(ref_model* m, int32_t token, long long T, float* logits);
/* Install a loaded chunk from the cache-tier bf16 bytes [layer][K|V][kv_head][token][head_dim]. */
int ref_load_chunk(ref_model* m, const uint16_t* tier_bf16, long long start, int len);

float* ref_kv(ref_model* m); /* [L][2][nkv][max_tokens][hd] */
long long ref_max_tokens(const ref_model* m);

/* Exact generator shared with the GPU (bf16 bits of one weight). */
uint16_t ref_weight_bits(unsigned long long seed, uint32_t tensor_id, uint64_t logical_index, float scale);
/* rows x cols block of tensor `tensor_id` (row-major, logical index r*cols+k) as bf16 bits,
 * OpenMP-parallel — the weight source of the numpy oracle (oracle/llama_np.py). */
void ref_weight_matrix_bits(unsigned long long seed, uint32_t tensor_id, long long rows, long long cols, float scale,
                            uint16_t* out);
/* Row `row` of a (*, cols) tensor: logical indices [row*cols, (row+1)*cols). */
void ref_weight_row_bits(unsigned long long seed, uint32_t tensor_id, long long row, long long cols, float scale,
                         uint16_t* out);
/* bf16 rounding (nearest-even) of n floats in place. */
void ref_round_bf16(float* x, long long n);
uint16_t ref_bf16_from_float(float f);
float ref_bf16_to_float(uint16_t b);

#ifdef __cplusplus
}
#endif
#endif
