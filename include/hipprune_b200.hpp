// hipprune_b200 C++ host API — the reference hipprune operator surface, served by
// the sm_100a kernels behind include/hipprune_b200.h.
//
// The declarations live in headers named as the reference's
// (/root/reference/proj/include/hipprune/*.hpp), so existing callers that
// `#include "hipprune/pruning.hpp"` etc. compile unchanged against this library:
//   errors.hpp           ContractViolation
//   tensor.hpp           DenseMatrix, RopeTable, build_rope_table, apply_rope, dot_f32, block_scores
//   workload.hpp         AttentionWorkload, SyntheticConfig, generate_synthetic, plant_needle,
//                        save_dump / load_dump / dump_checksum (HIPW v1), FormatError
//   rope_policy.hpp      RopePolicyId, RopePolicySet, PositionContext, query/key_position,
//                        streaming_positions
//   key_source.hpp       KeySource, DirectKeySource
//   pruning.hpp          StageConfig, PruningPlan, ChunkPartition, partition_chunks,
//                        SparseBlockMask, StageContext, select_rep, run_pruning_stage,
//                        StageTrace, build_mask
//   sparse_attention.hpp AttentionOutput, dense_attention, block_sparse_attention,
//                        attention_row, selected_indices, exact_topk, attention_recall,
//                        chunk_sparsity_histogram
//   kv_store.hpp         BankId, BankStats, CostModel, modeled_latency, PartialCommitError,
//                        TieredKvStore, KvView
//   decode.hpp           StoreConfig, TokenInput, StepTelemetry, StepResult, PrefillResult,
//                        refresh_due, DecodeEngine
//   config.hpp           preset_plan
//
// Pruning stages, block-sparse attention and the decode step run on the GPU (no CPU
// fallback: without a CUDA device they throw std::runtime_error). Data formats,
// page accounting and the quality checkers are host code, as in the reference.
#pragma once

#include "hipprune/config.hpp"
#include "hipprune/decode.hpp"
#include "hipprune/errors.hpp"
#include "hipprune/key_source.hpp"
#include "hipprune/kv_store.hpp"
#include "hipprune/pruning.hpp"
#include "hipprune/rope_policy.hpp"
#include "hipprune/sparse_attention.hpp"
#include "hipprune/tensor.hpp"
#include "hipprune/workload.hpp"
