// The extern "C" boundary (include/shardplan_gpu.h): validation, error
// mapping and dispatch into the host orchestration of each hot path.
#include <cmath>
#include <string>

#include "../../include/shardplan_gpu.h"
#include "context.cuh"
#include "trace_file.cuh"

struct rs_profile;
struct rs_emb;

namespace rs {
rs_profile* profile_run(rs_context*, const rs_trace*, double, uint64_t);
void hash_ids(rs_context*, const uint64_t*, uint64_t, uint64_t, uint32_t*, int);
void build_icdf(rs_context*, const uint64_t*, uint64_t, int, uint64_t*);
void count_distinct_raw(rs_context*, const rs_trace*, uint64_t*);
void build_remap(rs_context*, uint32_t, uint64_t, uint64_t, const uint32_t*, uint64_t, int, int,
                 int32_t*, int, uint64_t*);
void simulate(rs_context*, const rs_trace*, uint32_t, const rs_plan_entry*, uint32_t,
              const rs_remap_view*, const rs_system_spec*, uint64_t, rs_sim_report*);
rs_emb* emb_create(rs_context*, uint32_t, const rs_emb_table*, uint64_t, uint64_t, int, float);
void emb_unbacked(rs_emb*, uint64_t*, uint64_t*, int);
void emb_init_weights(rs_emb*, uint64_t, float);
void emb_forward(rs_emb*, uint64_t, const uint32_t*, const uint32_t*, float*, uint64_t*);
void emb_backward(rs_emb*, uint64_t, const uint32_t*, const uint32_t*, const float*, float);
void emb_read_rows(rs_emb*, uint32_t, const uint32_t*, uint64_t, float*, float*);
void emb_enable_cache(rs_emb*, uint32_t);
void emb_prefetch(rs_emb*, uint64_t, const uint32_t*, const uint32_t*);
void emb_flush(rs_emb*);
void emb_memory(const rs_emb*, uint64_t*, uint64_t*);
void remap_write(rs_context*, const char*, uint32_t, uint64_t, uint64_t, const int32_t*, int);
void remap_read_header(const char*, uint32_t*, uint64_t*, uint64_t*);
void remap_read(rs_context*, const char*, int32_t*, int, uint64_t, uint64_t*);
rs_trace_file* trace_read(rs_context*, const char*, uint64_t);
void trace_write(rs_context*, const rs_trace*, const char*, const char* const*, uint32_t, uint64_t);
void emb_kernel_times(rs_emb*, double*, uint64_t*, double*, uint64_t*, int);
void profile_view(const rs_profile*, uint32_t, rs_feature_stats*);
uint32_t profile_tables(const rs_profile*);
uint64_t profile_selected(const rs_profile*);
void profile_free(rs_profile*);
void emb_free(rs_emb*);
rs_exchange* exchange_create(rs_context*, int, uint32_t, uint32_t, uint64_t, uint32_t, const uint32_t*,
                             const uint32_t*);
void exchange_blob(rs_exchange*, void*);
void exchange_connect(rs_exchange*, const void*);
void exchange_info(const rs_exchange*, uint64_t*, uint64_t*, uint64_t*, float**);
void exchange_free(rs_exchange*);
float* exchange_forward(rs_exchange*, rs_emb*, const uint32_t*, const uint32_t*, uint64_t*);
void exchange_backward(rs_exchange*, rs_emb*, const uint32_t*, const uint32_t*, const float*, float);
void alltoall_fwd(rs_exchange*, const float*, float*);
void alltoall_bwd(rs_exchange*, const float*, float*);
}  // namespace rs

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return RS_OK;
  } catch (const rs::Error& e) {
    g_err = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return RS_ERR_INTERNAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RS_ERR_INTERNAL;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw rs::InvalidArgument(std::string(what) + " is null");
}
}  // namespace

namespace rs {
void set_error(const std::string& m) { g_err = m; }
uint64_t& launch_counter() {
  static uint64_t n = 0;
  return n;
}
}  // namespace rs

extern "C" {

int rs_abi_version(void) { return RS_ABI_VERSION; }
uint64_t rs_launch_counter(void) { return rs::launch_counter(); }
const char* rs_last_error(void) { return g_err.c_str(); }

int rs_context_create(int device, void* stream, int flags, rs_context** out) {
  return guarded([&] {
    need(out, "out");
    RS_CUDA(cudaSetDevice(device));
    auto* c = new rs_context;
    c->device = device;
    if (!(flags & RS_CTX_PRIVATE_STREAM)) {
      c->stream = static_cast<cudaStream_t>(stream);
    } else {
      cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
      if (e != cudaSuccess) {
        delete c;
        throw rs::CudaError(std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
      }
      c->own_stream = true;
    }
    *out = c;
  });
}

int rs_context_destroy(rs_context* c) {
  return guarded([&] {
    if (!c) return;
    cudaStreamSynchronize(c->stream);
    if (c->arena) cudaFree(c->arena);
    if (c->pinned) cudaFreeHost(c->pinned);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
  });
}

int rs_context_synchronize(rs_context* c) {
  return guarded([&] {
    need(c, "ctx");
    c->sync();
  });
}

int rs_hash_value(uint64_t raw, uint64_t hash_size, uint32_t* out) {
  return guarded([&] {
    need(out, "out");
    if (hash_size == 0) throw rs::InvalidArgument("hash_value: hash_size must be >= 1");
    *out = static_cast<uint32_t>(rs::mix64(raw) % hash_size);  // inc/workload.hpp:28-31
  });
}

int rs_hash_ids(rs_context* c, const uint64_t* raw, uint64_t n, uint64_t H, uint32_t* out, int loc) {
  return guarded([&] {
    need(c, "ctx");
    if (n) {
      need(raw, "raw");
      need(out, "out");
    }
    rs::hash_ids(c, raw, n, H, out, loc);
  });
}

int rs_profile_run(rs_context* c, const rs_trace* tr, double rate, uint64_t seed, rs_profile** out) {
  return guarded([&] {
    need(c, "ctx");
    need(out, "out");
    *out = rs::profile_run(c, tr, rate, seed);
  });
}

int rs_profile_num_tables(const rs_profile* p, uint32_t* out) {
  return guarded([&] {
    need(p, "profile");
    *out = rs::profile_tables(p);
  });
}

int rs_profile_get(const rs_profile* p, uint32_t j, rs_feature_stats* out) {
  return guarded([&] {
    need(p, "profile");
    need(out, "out");
    rs::profile_view(p, j, out);
  });
}

int rs_profile_selected(const rs_profile* p, uint64_t* out) {
  return guarded([&] {
    need(p, "profile");
    *out = rs::profile_selected(p);
  });
}

int rs_profile_destroy(rs_profile* p) {
  return guarded([&] { rs::profile_free(p); });
}

int rs_build_icdf(rs_context* c, const uint64_t* counts, uint64_t n, int loc, uint64_t* out101) {
  return guarded([&] {
    need(c, "ctx");
    need(out101, "out");
    if (n) need(counts, "counts");
    rs::build_icdf(c, counts, n, loc, out101);
  });
}

int rs_count_distinct_raw(rs_context* c, const rs_trace* tr, uint64_t* out) {
  return guarded([&] {
    need(c, "ctx");
    need(tr, "trace");
    need(out, "out");
    rs::count_distinct_raw(c, tr, out);
  });
}

int rs_hash_utilization(uint64_t distinct, uint64_t hash_size, uint64_t distinct_raw, double* sp,
                        double* col) {
  return guarded([&] {
    need(sp, "sparsity");
    need(col, "collisions");
    // core/src/profiler.cpp:163-174
    const double h = static_cast<double>(hash_size);
    *sp = static_cast<double>(hash_size - distinct) / h;
    *col = (static_cast<double>(distinct_raw) - static_cast<double>(distinct)) / h;
  });
}

int rs_build_remap(rs_context* c, uint32_t table_id, uint64_t H, uint64_t hbm_rows,
                   const uint32_t* rows_by_rank, uint64_t distinct, int rows_loc, int omit,
                   int32_t* entries, int out_loc, uint64_t* slow_alloc) {
  return guarded([&] {
    need(c, "ctx");
    if (H) need(entries, "entries");
    rs::build_remap(c, table_id, H, hbm_rows, rows_by_rank, distinct, rows_loc, omit, entries, out_loc,
                    slow_alloc);
  });
}

int rs_simulate(rs_context* c, const rs_trace* tr, uint32_t ne, const rs_plan_entry* entries,
                uint32_t nr, const rs_remap_view* remaps, const rs_system_spec* sys, uint64_t B,
                rs_sim_report* out) {
  return guarded([&] {
    need(c, "ctx");
    need(tr, "trace");
    need(sys, "system");
    need(out, "out");
    rs::simulate(c, tr, ne, entries, nr, remaps, sys, B, out);
  });
}

int rs_emb_create(rs_context* c, uint32_t T, const rs_emb_table* tabs, uint64_t max_batch,
                  uint64_t max_lookups, int opt, float eps, rs_emb** out) {
  return guarded([&] {
    need(c, "ctx");
    need(tabs, "tables");
    need(out, "out");
    *out = rs::emb_create(c, T, tabs, max_batch, max_lookups, opt, eps);
  });
}

int rs_emb_destroy(rs_emb* e) {
  return guarded([&] { rs::emb_free(e); });
}

int rs_emb_unbacked(rs_emb* e, uint64_t* lookups, uint64_t* rows, int reset) {
  return guarded([&] {
    need(e, "emb");
    rs::emb_unbacked(e, lookups, rows, reset);
  });
}

int rs_emb_init_weights(rs_emb* e, uint64_t seed, float scale) {
  return guarded([&] {
    need(e, "emb");
    rs::emb_init_weights(e, seed, scale);
  });
}

int rs_emb_forward(rs_emb* e, uint64_t B, const uint32_t* off, const uint32_t* idx, float* pooled,
                   uint64_t* hits) {
  return guarded([&] {
    need(e, "emb");
    need(off, "offsets");
    need(pooled, "pooled");
    rs::emb_forward(e, B, off, idx, pooled, hits);
  });
}

int rs_emb_backward(rs_emb* e, uint64_t B, const uint32_t* off, const uint32_t* idx,
                    const float* grad, float lr) {
  return guarded([&] {
    need(e, "emb");
    need(off, "offsets");
    need(grad, "grad");
    rs::emb_backward(e, B, off, idx, grad, lr);
  });
}

int rs_emb_enable_uvm_cache(rs_emb* e, uint32_t nslots) {
  return guarded([&] {
    need(e, "emb");
    rs::emb_enable_cache(e, nslots);
  });
}

int rs_emb_prefetch(rs_emb* e, uint64_t B, const uint32_t* off, const uint32_t* idx) {
  return guarded([&] {
    need(e, "emb");
    need(off, "offsets");
    rs::emb_prefetch(e, B, off, idx);
  });
}

int rs_emb_flush(rs_emb* e) {
  return guarded([&] {
    need(e, "emb");
    rs::emb_flush(e);
  });
}

int rs_emb_read_rows(rs_emb* e, uint32_t t, const uint32_t* rows, uint64_t n, float* out, float* mom) {
  return guarded([&] {
    need(e, "emb");
    if (n) {
      need(rows, "rows");
      need(out, "out");
    }
    rs::emb_read_rows(e, t, rows, n, out, mom);
  });
}

int rs_radix_sort_pairs(rs_context* c, uint32_t* keys, uint32_t* vals, uint64_t n, int end_bit) {
  return guarded([&] {
    need(c, "ctx");
    if (n) need(keys, "keys");
    if (end_bit < 0 || end_bit > 32) throw rs::InvalidArgument("radix_sort: end_bit in [0, 32]");
    rs::Scratch scr = c->scratch(rs::radix_sort_scratch_bytes(n) + (4 << 20));
    rs::radix_sort_pairs(keys, vals, n, end_bit, scr, c->stream);
  });
}

int rs_remap_write(rs_context* c, const char* path, uint32_t table_id, uint64_t H, uint64_t hbm_rows,
                   const int32_t* entries, int loc) {
  return guarded([&] {
    need(path, "path");
    if (H) need(entries, "entries");
    if (loc == RS_MEM_DEVICE) need(c, "ctx");
    rs::remap_write(c, path, table_id, H, hbm_rows, entries, loc);
  });
}

int rs_remap_read_header(const char* path, uint32_t* table_id, uint64_t* H, uint64_t* hbm_rows) {
  return guarded([&] {
    need(path, "path");
    need(table_id, "table_id");
    need(H, "hash_size");
    need(hbm_rows, "hbm_rows");
    rs::remap_read_header(path, table_id, H, hbm_rows);
  });
}

int rs_remap_read(rs_context* c, const char* path, int32_t* out, int loc, uint64_t capacity, uint64_t* slow) {
  return guarded([&] {
    need(path, "path");
    need(out, "out");
    if (loc == RS_MEM_DEVICE) need(c, "ctx");
    rs::remap_read(c, path, out, loc, capacity, slow);
  });
}

int rs_emb_kernel_times(rs_emb* e, double* fwd_ms, uint64_t* n_fwd, double* bwd_ms, uint64_t* n_bwd, int reset) {
  return guarded([&] {
    need(e, "emb");
    rs::emb_kernel_times(e, fwd_ms, n_fwd, bwd_ms, n_bwd, reset);
  });
}

int rs_trace_read(rs_context* c, const char* path, uint64_t chunk_bytes, rs_trace_file** out) {
  return guarded([&] {
    need(c, "ctx");
    need(path, "path");
    need(out, "out");
    *out = rs::trace_read(c, path, chunk_bytes);
  });
}

int rs_trace_file_view(const rs_trace_file* f, rs_trace* v) {
  return guarded([&] {
    need(f, "trace_file");
    need(v, "view");
    *v = rs_trace{};
    v->num_tables = uint32_t(f->tables.size());
    v->tables = f->tables.data();
    v->num_samples = f->num_samples;
    v->num_records = f->nrec;
    v->rec_sample = f->rec_sample;
    v->rec_table = f->rec_table;
    v->rec_offset = f->rec_offset;
    v->rec_len = f->rec_len;
    v->num_ids = f->nids;
    v->ids = f->ids;
    v->raw_ids = nullptr;
    v->location = RS_MEM_DEVICE;
  });
}

int rs_trace_file_export(rs_context* c, const rs_trace_file* f, uint64_t* rs_, uint32_t* rt, uint64_t* ro,
                         uint32_t* rl, uint32_t* ids, int loc) {
  return guarded([&] {
    need(c, "ctx");
    need(f, "trace_file");
    const cudaMemcpyKind k = loc == RS_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) RS_CUDA(cudaMemcpyAsync(dst, src, bytes, k, c->stream));
    };
    cp(rs_, f->rec_sample, f->nrec * 8);
    cp(rt, f->rec_table, f->nrec * 4);
    cp(ro, f->rec_offset, f->nrec * 8);
    cp(rl, f->rec_len, f->nrec * 4);
    cp(ids, f->ids, f->nids * 4);
    c->sync();
  });
}

int rs_trace_file_destroy(rs_trace_file* f) {
  return guarded([&] { delete f; });
}

int rs_trace_write(rs_context* c, const rs_trace* tr, const char* path, const char* const* comments,
                   uint32_t n_comments) {
  return guarded([&] {
    need(c, "ctx");
    need(tr, "trace");
    need(path, "path");
    if (n_comments) need(comments, "comments");
    if (tr->num_tables) need(tr->tables, "tables");
    rs::trace_write(c, tr, path, comments, n_comments, 0);
  });
}

int rs_emb_memory(const rs_emb* e, uint64_t* hbm, uint64_t* host) {
  return guarded([&] {
    need(e, "emb");
    rs::emb_memory(e, hbm, host);
  });
}

// ---------------------------------------------------------------- K6 exchange
int rs_exchange_create(rs_context* c, int transport, uint32_t nranks, uint32_t rank, uint64_t batch,
                       uint32_t num_tables, const uint32_t* dims, const uint32_t* owner, rs_exchange** out) {
  return guarded([&] {
    need(c, "ctx");
    need(out, "out");
    *out = rs::exchange_create(c, transport, nranks, rank, batch, num_tables, dims, owner);
  });
}

int rs_exchange_blob(rs_exchange* x, void* blob) {
  return guarded([&] {
    need(x, "exchange");
    need(blob, "blob");
    rs::exchange_blob(x, blob);
  });
}

int rs_exchange_connect(rs_exchange* x, const void* blobs) {
  return guarded([&] {
    need(x, "exchange");
    need(blobs, "blobs");
    rs::exchange_connect(x, blobs);
  });
}

int rs_exchange_info(const rs_exchange* x, uint64_t* bl, uint64_t* d_total, uint64_t* d_local, float** owned) {
  return guarded([&] {
    need(x, "exchange");
    rs::exchange_info(x, bl, d_total, d_local, owned);
  });
}

int rs_exchange_destroy(rs_exchange* x) {
  return guarded([&] { rs::exchange_free(x); });
}

int rs_emb_forward_to_owners(rs_emb* e, rs_exchange* x, const uint32_t* offsets, const uint32_t* indices,
                             uint64_t* hit_counts, float** owned) {
  return guarded([&] {
    need(e, "emb");
    need(x, "exchange");
    need(offsets, "offsets");
    float* o = rs::exchange_forward(x, e, offsets, indices, hit_counts);
    if (owned) *owned = o;
  });
}

int rs_emb_backward_from_owners(rs_emb* e, rs_exchange* x, const uint32_t* offsets, const uint32_t* indices,
                                const float* grad_owned, float lr) {
  return guarded([&] {
    need(e, "emb");
    need(x, "exchange");
    need(offsets, "offsets");
    rs::exchange_backward(x, e, offsets, indices, grad_owned, lr);
  });
}

int rs_emb_alltoall_fwd(rs_exchange* x, const float* pooled_local, float* pooled_owned) {
  return guarded([&] {
    need(x, "exchange");
    need(pooled_owned, "pooled_owned");
    rs::alltoall_fwd(x, pooled_local, pooled_owned);
  });
}

int rs_emb_alltoall_bwd(rs_exchange* x, const float* grad_owned, float* grad_local) {
  return guarded([&] {
    need(x, "exchange");
    need(grad_owned, "grad_owned");
    rs::alltoall_bwd(x, grad_owned, grad_local);
  });
}

}  // extern "C"
