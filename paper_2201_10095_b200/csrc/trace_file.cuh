// rs_trace_file: a trace loaded by rs_trace_read (trace_io.cu), device-resident.
#pragma once

#include <vector>

#include "../../include/shardplan_gpu.h"

struct rs_trace_file {
  std::vector<rs_table_spec> tables;
  uint64_t num_samples = 0;
  uint64_t nrec = 0, nids = 0;
  uint64_t rec_cap = 0, ids_cap = 0;
  uint64_t* rec_sample = nullptr;
  uint32_t* rec_table = nullptr;
  uint64_t* rec_offset = nullptr;
  uint32_t* rec_len = nullptr;
  uint32_t* ids = nullptr;
  ~rs_trace_file() {
    for (void* p : {(void*)rec_sample, (void*)rec_table, (void*)rec_offset, (void*)rec_len, (void*)ids})
      if (p) cudaFree(p);
  }
};

