/*
 * hipprune_b200 developer hooks — NOT part of the product ABI. Exported only by the
 * dev builds of the kernel library (HP_TRACE=1 / HP_VARIANT builds of
 * paper_2502_08910_b200/build.py, which define HP_TRACE or HP_DEV); the product
 * libhipprune_b200.so has none of these symbols. Used by scripts/ (timelines, phase cuts).
 */
#ifndef HIPPRUNE_B200_DEV_H
#define HIPPRUNE_B200_DEV_H

#ifdef __cplusplus
extern "C" {
#endif

/* per-CTA %globaltimer / clock64 stamps of the fused decode kernels (kernel_id 10 + l_c =
 * stage descent, 3 = top-k, 2 = BSA) into buf [16384][8] u64; NULL disables */
int hp_trace_enable(unsigned long long* buf, int kernel_id);
/* the same for hp_decode_layer's kernel (trace ids 20-22) */
int hp_layer_trace_enable(unsigned long long* buf, int kernel_id);
/* kernel `kernel_id` returns early at its cut point `at` (-1 disables) */
int hp_debug_cut(int kernel_id, int at);
/* the tcgen05 prefill's thread 0 writes progress codes to this mapped host word */
int hp_debug_prefill_progress(int* mapped_word);

#ifdef __cplusplus
}
#endif
#endif
