// gt_api_internal.h — helpers shared by libgt.so's translation units (not ABI).
#pragma once
#include <cstdint>

#include "../../include/gt.h"

int gt_internal_set_err(int code, const char* msg);
int gt_set_errf(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int gt_internal_shard_geometry(uint64_t V, uint64_t E, gt_shard_geom* g);
