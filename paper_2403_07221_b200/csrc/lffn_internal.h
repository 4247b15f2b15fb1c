// lffn_internal.h -- shared declarations of the lffn_gpu library (not part of
// the C-ABI; see include/lffn_gpu.h for that).
#pragma once

#include <cstdint>
#include <string>

#include "lffn_gpu.h"

namespace lffn_gpu {

// Thread-local last-error message (lffn_last_error) + status passthrough.
int fail(int status, const std::string& msg);

int64_t next_pow2(int64_t n);
int64_t transform_width(const lffn_proj* p);
int64_t blob_size(const lffn_proj* p);
int validate_cfg(const lffn_cfg* c);
int validate_proj(const lffn_proj* p);

// Host tables [k0, k0+nk) of a context's slice -> device (checkpoint.cpp
// streams through this).
int tables_upload_range(lffn_ctx* c, const void* host, int host_dtype, int store_dtype, int64_t k0,
                        int64_t nk);

// Device non-finite flag bits; each names the reference stage that would
// throw NumericError (lookup.cpp:204,269; projection.cpp:172,264).
enum : int {
  kFlagInput = 1,   // "projection forward input"
  kFlagHash = 2,    // "hash stage"
  kFlagGather = 4,  // "gather stage"
  kFlagBwdInput = 8,    // "lookup backward input" / "projection backward input"
  kFlagBwdOutput = 16,  // "projection backward output"
  kFlagBwdTables = 32,  // "lookup backward tables"
  kFlagStream = 64,     // a bounded device-side wait timed out (fused kernel ring)
};

}  // namespace lffn_gpu
