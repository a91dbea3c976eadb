// Internal interface between the C ABI (engine.cu) and the 3D engine
// (engine3.cu).  Not part of include/tmg.h: every function returns a TMG_*
// status and writes its message into err.
#pragma once

#include <cstdint>
#include <string>

#include "tmg.h"

struct Engine3;

int e3_create(const tmg_tree3* t, const tmg_config* cfg, Engine3** out, std::string& err);
int e3_rebuild(Engine3* e, const tmg_tree3* t, std::string& err);
void e3_destroy(Engine3* e);
int e3_set_rhs(Engine3* e, int level, const double* rhs, std::string& err);
int e3_set_u(Engine3* e, int level, const double* u, std::string& err);
int e3_get_u(Engine3* e, int level, double* u, std::string& err);
int e3_update_fas_state(Engine3* e, std::string& err);
int e3_cycle(Engine3* e, int ncycles, tmg_stats* stats, std::string& err);
int e3_residual_stats(Engine3* e, tmg_stats* out, std::string& err);
int e3_levels(Engine3* e, int32_t* lmin, int32_t* ltop);
int e3_level_counts(Engine3* e, int level, int64_t* dof, int64_t* composite, int64_t* hanging,
                    std::string& err);
int e3_get_kinds(Engine3* e, int level, int8_t* out, std::string& err);
int e3_get_table(Engine3* e, int which, int level, double* out, std::string& err);
int e3_time_cycles(Engine3* e, int ncycles, int64_t flush_bytes, float* ms, std::string& err);
int e3_profile_cycles(Engine3* e, int ncycles, int cap, const char** names, float* ms,
                      int32_t* launches, int32_t* nk, std::string& err);
int e3_launches_per_cycle(Engine3* e, int32_t* n, std::string& err);
int e3_shard(Engine3* e, int ls, const int32_t* lo, const int32_t* hi, std::string& err);
int e3_phase(Engine3* e, int phase, int level, std::string& err);
int e3_phase_range(Engine3* e, int phase, int level, int lo, int hi, int first, int last, std::string& err);
int e3_field(Engine3* e, int field, int level, uint64_t* ptr, int64_t* count, std::string& err);
int e3_storage(Engine3* e, int level, int64_t* out, std::string& err);
int e3_fused(Engine3* e, int level, int32_t* out, std::string& err);
int e3_stream(Engine3* e, uint64_t* s);
int e3_history(Engine3* e, int count, tmg_stats* out, std::string& err);
int e3_cycle_state(Engine3* e, int64_t* count, int32_t* parity, int set, std::string& err);
