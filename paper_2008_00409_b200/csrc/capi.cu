// capi.cu — the extern "C" boundary (include/weft_gpu.h). Every entry
// point converts exceptions into a weft_status plus a thread-local message
// worded like the reference's exception.
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "cr_atan2.cuh"
#include "ctx.cuh"

namespace {
thread_local std::string g_last_error;

template <class F>
weft_status guard(weft_gpu_ctx* ctx, F&& f) {
  try {
    if (ctx) WG_CUDA(cudaSetDevice(ctx->c.device));
    f();
    return WEFT_OK;
  } catch (const weft_gpu::Error& e) {
    g_last_error = e.what();
    return e.status;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return WEFT_ERR_INVALID;
  }
}

void need(bool ok, weft_status s, const char* msg) {
  if (!ok) throw weft_gpu::Error(s, msg);
}

bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

// generate_work_queues (proj/src/topology.cpp:34-89).
void gen_range(int lo, int hi, std::vector<std::vector<int>>& peer, std::vector<std::vector<int>>& vec) {
  const int size = hi - lo;
  if (size == 1) return;
  const int half = size / 2, mid = lo + half;
  gen_range(lo, mid, peer, vec);
  gen_range(mid, hi, peer, vec);
  const size_t child = peer[static_cast<size_t>(lo)].size();
  for (int i = lo; i < mid; ++i) {
    peer[i].push_back(i + half);
    vec[i].push_back(i + half);
  }
  for (int j = mid; j < hi; ++j) {
    peer[j].push_back(j - half);
    vec[j].push_back(j - half);
  }
  for (int i = lo; i < hi; ++i) {
    const int off = i < mid ? half : -half;
    for (size_t k = 0; k < child; ++k) {
      peer[i].push_back(peer[i][k]);
      vec[i].push_back(vec[i][k] + off);
    }
  }
}

__global__ void k_hinge_atan2(const double* __restrict__ y, const double* __restrict__ x, double* __restrict__ out,
                              int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = weft_gpu::cr::atan2(y[i], x[i]);
}

}  // namespace

extern "C" {

const char* weft_gpu_last_error(void) { return g_last_error.c_str(); }

weft_status weft_gpu_internal_set_error(const char* msg, weft_status s) {
  g_last_error = msg;
  return s;
}

weft_status weft_hinge_atan2_host(int64_t n, const double* y, const double* x, double* out) {
  return guard(nullptr, [&] {
    need(n >= 0, WEFT_ERR_DIMENSION, "negative count");
    for (int64_t i = 0; i < n; ++i) out[i] = weft_gpu::cr::atan2(y[i], x[i]);
  });
}

weft_status weft_gpu_hinge_atan2(weft_gpu_ctx* ctx, int64_t n, const double* y, const double* x, double* out) {
  return guard(ctx, [&] {
    need(n >= 0, WEFT_ERR_DIMENSION, "negative count");
    if (n == 0) return;
    auto& c = ctx->c;
    weft_gpu::DBuf<double> buf;
    buf.resize(static_cast<size_t>(3 * n));
    WG_CUDA(cudaMemcpyAsync(buf.data(), y, sizeof(double) * n, cudaMemcpyDefault, c.stream));
    WG_CUDA(cudaMemcpyAsync(buf.data() + n, x, sizeof(double) * n, cudaMemcpyDefault, c.stream));
    k_hinge_atan2<<<static_cast<unsigned>((n + 255) / 256), 256, 0, c.stream>>>(buf.data(), buf.data() + n,
                                                                               buf.data() + 2 * n, n);
    WG_CUDA(cudaGetLastError());
    WG_CUDA(cudaMemcpyAsync(out, buf.data() + 2 * n, sizeof(double) * n, cudaMemcpyDefault, c.stream));
    WG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

weft_status weft_make_partitions(int32_t p, int32_t n, int32_t* begin, int32_t* end) {
  return guard(nullptr, [&] {
    if (n < 1) throw weft_gpu::Error(WEFT_ERR_TOPOLOGY, "device count must be >= 1");
    if (p < 0) throw weft_gpu::Error(WEFT_ERR_DIMENSION, "negative vertex count");
    const auto pm = weft_gpu::PartMap::make(p, n);
    for (int d = 0; d < n; ++d) {
      begin[d] = pm.begin(d);
      end[d] = pm.end(d);
    }
  });
}

weft_status weft_work_queues(int32_t n, int32_t* peer, int32_t* vec) {
  return guard(nullptr, [&] {
    if (!is_pow2(n))
      throw weft_gpu::Error(WEFT_ERR_TOPOLOGY,
                            "work queue generation requires power-of-two devices, got " + std::to_string(n));
    std::vector<std::vector<int>> pr(static_cast<size_t>(n)), vc(static_cast<size_t>(n));
    gen_range(0, n, pr, vc);
    for (int d = 0; d < n; ++d)
      for (int k = 0; k < n - 1; ++k) {
        peer[d * (n - 1) + k] = pr[d][k];
        vec[d * (n - 1) + k] = vc[d][k];
      }
  });
}

weft_status weft_split_workload(int64_t total, int32_t devices, int64_t* begin, int64_t* end) {
  return guard(nullptr, [&] {
    need(devices >= 1, WEFT_ERR_TOPOLOGY, "device count must be >= 1");
    const int64_t base = total / devices, extra = total % devices;
    int64_t cursor = 0;
    for (int d = 0; d < devices; ++d) {
      const int64_t size = base + (d < extra ? 1 : 0);
      begin[d] = cursor;
      end[d] = cursor + size;
      cursor += size;
    }
  });
}

weft_status weft_gpu_create(const weft_gpu_options* opts, weft_gpu_ctx** out) {
  *out = nullptr;
  auto* ctx = new weft_gpu_ctx();
  const weft_status st = guard(nullptr, [&] {
    auto& c = ctx->c;
    c.device = opts ? opts->cuda_device : 0;
    c.nparts = opts ? opts->partitions : 1;
    c.part_begin = opts ? opts->part_begin : 0;
    c.part_end = opts ? opts->part_end : c.nparts;
    if (c.nparts < 1 || c.nparts > weft_gpu::kMaxParts)
      throw weft_gpu::Error(WEFT_ERR_TOPOLOGY, "partition count must be in [1, 8]");
    if (!is_pow2(c.nparts))
      throw weft_gpu::Error(WEFT_ERR_TOPOLOGY,
                            "fat-tree requires a power-of-two device count, got " + std::to_string(c.nparts));
    const int span = c.part_end - c.part_begin;
    if (span < 1 || c.part_begin < 0 || c.part_end > c.nparts || c.nparts % span != 0 || c.part_begin % span != 0)
      throw weft_gpu::Error(WEFT_ERR_TOPOLOGY, "partition range [" + std::to_string(c.part_begin) + ", " +
                                                   std::to_string(c.part_end) +
                                                   ") is not one of equal contiguous rank ranges of " +
                                                   std::to_string(c.nparts) + " partitions");
    c.world = c.nparts / span;
    c.rank = c.part_begin / span;
    int count = 0;
    WG_CUDA(cudaGetDeviceCount(&count));
    if (c.device < 0 || c.device >= count)
      throw weft_gpu::Error(WEFT_ERR_EXEC, "device " + std::to_string(c.device) + " failed: no such CUDA device");
    WG_CUDA(cudaSetDevice(c.device));
    WG_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    WG_CUDA(cudaStreamCreateWithFlags(&c.side, cudaStreamNonBlocking));
    c.cur = c.stream;
    for (auto& e : c.ev) WG_CUDA(cudaEventCreate(&e));
    for (auto& e : c.ev_side) WG_CUDA(cudaEventCreate(&e));
    c.scalars.resize(64);
    if (const char* e = std::getenv("WEFT_SPMV_PAIR")) c.spmv_pair = std::atoi(e) != 0;
    if (const char* e = std::getenv("WEFT_NO_GRAPHS")) c.use_graphs = std::atoi(e) == 0;
    if (const char* e = std::getenv("WEFT_PCG_PERSISTENT")) c.use_persistent = std::atoi(e) != 0;
    // accumulation group order from the work queues
    const int n = c.nparts;
    c.go.n = n;
    std::memset(c.go.qpos, 0, sizeof(c.go.qpos));
    c.queue_vec.assign(static_cast<size_t>(n * (n > 1 ? n - 1 : 0)), 0);
    if (n > 1) {
      std::vector<std::vector<int>> pr(static_cast<size_t>(n)), vc(static_cast<size_t>(n));
      gen_range(0, n, pr, vc);
      for (int d = 0; d < n; ++d)
        for (int k = 0; k < n - 1; ++k) {
          c.queue_vec[static_cast<size_t>(d * (n - 1) + k)] = vc[d][k];
          c.go.qpos[d][vc[d][k]] = static_cast<int8_t>(k + 1);
        }
    }
  });
  if (st != WEFT_OK) {
    delete ctx;
    return st;
  }
  *out = ctx;
  return WEFT_OK;
}

weft_status weft_gpu_destroy(weft_gpu_ctx* ctx) {
  if (!ctx) return WEFT_OK;
  const weft_status st = guard(ctx, [&] {
    auto& c = ctx->c;
    weft_gpu::pcg_free(c);
    WG_CUDA(cudaStreamSynchronize(c.stream));
    weft_gpu::comm_free(c);
    WG_CUDA(cudaStreamSynchronize(c.side));
    for (auto& e : c.ev) cudaEventDestroy(e);
    for (auto& e : c.ev_side) cudaEventDestroy(e);
    if (c.map_host) cudaFreeHost(c.map_host);
    cudaStreamDestroy(c.side);
    cudaStreamDestroy(c.stream);
  });
  delete ctx;
  return st;
}

weft_status weft_gpu_set_matrix(weft_gpu_ctx* ctx, int32_t rows, const int64_t* row_ptr, const int32_t* cols,
                                const double* vals) {
  return guard(ctx, [&] {
    need(row_ptr != nullptr, WEFT_ERR_INVALID, "set_matrix: row_ptr is NULL");
    // The CSR is read on the host; copy device inputs first.
    std::vector<int64_t> rp(static_cast<size_t>(rows) + 1);
    WG_CUDA(cudaMemcpy(rp.data(), row_ptr, rp.size() * sizeof(int64_t), cudaMemcpyDefault));
    const int64_t nnzb = rp.back();
    std::vector<int32_t> cl(static_cast<size_t>(nnzb));
    std::vector<double> vl(9 * static_cast<size_t>(nnzb));
    if (nnzb) {
      WG_CUDA(cudaMemcpy(cl.data(), cols, cl.size() * sizeof(int32_t), cudaMemcpyDefault));
      WG_CUDA(cudaMemcpy(vl.data(), vals, vl.size() * sizeof(double), cudaMemcpyDefault));
    }
    weft_gpu::set_matrix_csr(ctx->c, rows, rp.data(), cl.data(), vl.data());
  });
}

// ---- Precision::Single (driver.hpp:13; Real = float), one rank
weft_status weft_gpu_set_matrix_f32(weft_gpu_ctx* ctx, int32_t rows, const int64_t* row_ptr, const int32_t* cols,
                                    const float* vals) {
  return guard(ctx, [&] {
    need(row_ptr != nullptr, WEFT_ERR_INVALID, "set_matrix: row_ptr is NULL");
    need(ctx->c.world == 1, WEFT_ERR_INVALID, "set_matrix: Precision::Single runs on one rank");
    std::vector<int64_t> rp(static_cast<size_t>(rows) + 1);
    WG_CUDA(cudaMemcpy(rp.data(), row_ptr, rp.size() * sizeof(int64_t), cudaMemcpyDefault));
    const int64_t nnzb = rp.back();
    std::vector<int32_t> cl(static_cast<size_t>(nnzb));
    std::vector<float> vl(9 * static_cast<size_t>(nnzb));
    if (nnzb) {
      WG_CUDA(cudaMemcpy(cl.data(), cols, cl.size() * sizeof(int32_t), cudaMemcpyDefault));
      WG_CUDA(cudaMemcpy(vl.data(), vals, vl.size() * sizeof(float), cudaMemcpyDefault));
    }
    weft_gpu::set_matrix_csr_f32(ctx->c, rows, rp.data(), cl.data(), vl.data());
  });
}

weft_status weft_gpu_spmv_f32(weft_gpu_ctx* ctx, const float* x, float* y) {
  return guard(ctx, [&] {
    auto& c = ctx->c;
    need(c.has_matrix && c.A.f32, WEFT_ERR_INVALID, "spmv: no single-precision matrix");
    const size_t len = 3 * static_cast<size_t>(c.pm.p);
    c.q.resize(len);
    c.r.resize(len);
    float* xd = reinterpret_cast<float*>(c.r.data());
    float* yd = reinterpret_cast<float*>(c.q.data());
    WG_CUDA(cudaMemcpyAsync(xd, x, len * sizeof(float), cudaMemcpyDefault, c.stream));
    weft_gpu::spmv_f32(c, xd, yd);
    WG_CUDA(cudaMemcpyAsync(y, yd, len * sizeof(float), cudaMemcpyDefault, c.stream));
    WG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

weft_status weft_gpu_pcg_f32(weft_gpu_ctx* ctx, const float* b, float* x, const weft_pcg_config* config,
                             weft_pcg_report* report) {
  return guard(ctx, [&] {
    auto& c = ctx->c;
    need(c.has_matrix && c.A.f32, WEFT_ERR_INVALID, "pcg: no single-precision matrix");
    need(config != nullptr, WEFT_ERR_INVALID, "pcg: config is NULL");
    const size_t len = 3 * static_cast<size_t>(c.pm.p);
    const float* bdev = nullptr;
    if (b) {
      c.bvec.resize(len);
      WG_CUDA(cudaMemcpyAsync(c.bvec.data(), b, len * sizeof(float), cudaMemcpyDefault, c.stream));
      bdev = reinterpret_cast<const float*>(c.bvec.data());
    } else {
      need(c.has_rhs, WEFT_ERR_INVALID, "pcg: b is NULL and no assembled rhs");
      bdev = reinterpret_cast<const float*>(c.rhs.data());
    }
    weft_gpu::PcgResult r;
    try {
      r = weft_gpu::pcg_solve_f32(c, bdev, *config, report ? report->residual_history : nullptr,
                                  report ? report->precond_norm_history : nullptr);
    } catch (...) {
      if (report) report->iterations = 0;
      throw;
    }
    if (report) {
      report->iterations = r.iterations;
      report->converged = r.converged;
      report->rel_residual = r.rel_residual;
    }
    if (x) {
      float* xs = reinterpret_cast<float*>(c.xs.data());
      if (r.iterations == 0) WG_CUDA(cudaMemsetAsync(xs, 0, len * sizeof(float), c.stream));
      WG_CUDA(cudaMemcpyAsync(x, xs, len * sizeof(float), cudaMemcpyDefault, c.stream));
      WG_CUDA(cudaStreamSynchronize(c.stream));
    }
  });
}

weft_status weft_gpu_download_matrix_f32(weft_gpu_ctx* ctx, int64_t* row_ptr, int32_t* cols, float* vals) {
  return guard(ctx, [&] {
    need(ctx->c.has_matrix, WEFT_ERR_INVALID, "download_matrix: no matrix");
    weft_gpu::download_csr_f32(ctx->c, row_ptr, cols, vals);
  });
}

weft_status weft_gpu_spmv(weft_gpu_ctx* ctx, const double* x, double* y) {
  return guard(ctx, [&] {
    auto& c = ctx->c;
    need(c.has_matrix, WEFT_ERR_INVALID, "spmv: no matrix");
    const size_t len = 3 * static_cast<size_t>(c.pm.p);
    c.q.resize(len);
    if (c.world == 1) {
      c.r.resize(len);
      WG_CUDA(cudaMemcpyAsync(c.r.data(), x, len * sizeof(double), cudaMemcpyDefault, c.stream));
      if (c.profile) WG_CUDA(cudaEventRecord(c.ev[6], c.stream));
      weft_gpu::spmv(c, c.r.data(), c.q.data());
      if (c.profile) {  // the kernel alone (the copies of x and y are outside the events)
        WG_CUDA(cudaEventRecord(c.ev[7], c.stream));
        WG_CUDA(cudaEventSynchronize(c.ev[7]));
        float ms = 0.f;
        WG_CUDA(cudaEventElapsedTime(&ms, c.ev[6], c.ev[7]));
        c.spmv_ms += ms;
        ++c.spmv_launches;
      }
      WG_CUDA(cudaMemcpyAsync(y, c.q.data(), len * sizeof(double), cudaMemcpyDefault, c.stream));
    } else {
      // own rows of x into the window; peers gather the rest from their owners
      weft_gpu::comm_need(c, "spmv");
      const size_t o = 3 * static_cast<size_t>(c.row0), m = 3 * static_cast<size_t>(c.A.rows);
      WG_CUDA(cudaMemcpyAsync(c.z.data() + o, x + o, m * sizeof(double), cudaMemcpyDefault, c.stream));
      weft_gpu::publish_vectors(c);
      weft_gpu::spmv(c, c.z.data(), c.q.data());
      weft_gpu::rank_barrier(c);  // peers finished reading this rank's x rows
      WG_CUDA(cudaMemcpyAsync(y + o, c.q.data() + o, m * sizeof(double), cudaMemcpyDefault, c.stream));
    }
    WG_CUDA(cudaStreamSynchronize(c.stream));
    weft_gpu::comm_check(c);
  });
}

weft_status weft_gpu_matrix_info(weft_gpu_ctx* ctx, weft_matrix_info* info) {
  return guard(ctx, [&] {
    auto& c = ctx->c;
    need(c.has_matrix, WEFT_ERR_INVALID, "matrix_info: no matrix");
    info->block_rows = c.A.rows;
    info->max_row_blocks = c.A.max_len;
    info->nnzb = c.A.nnzb;
    info->padded_slots = c.A.total;
  });
}

weft_status weft_gpu_download_matrix(weft_gpu_ctx* ctx, int64_t* row_ptr, int32_t* cols, double* vals) {
  return guard(ctx, [&] {
    need(ctx->c.has_matrix, WEFT_ERR_INVALID, "download_matrix: no matrix");
    weft_gpu::download_csr(ctx->c, row_ptr, cols, vals);
  });
}

weft_status weft_gpu_download_rhs(weft_gpu_ctx* ctx, double* rhs) {
  return guard(ctx, [&] {
    auto& c = ctx->c;
    need(c.has_rhs, WEFT_ERR_INVALID, "download_rhs: no assembled system");
    need(!c.A.f32, WEFT_ERR_INVALID, "download_rhs: single-precision system (use the f32 entry)");
    WG_CUDA(cudaMemcpyAsync(rhs, c.rhs.data() + 3 * static_cast<size_t>(c.row0), 3 * sizeof(double) * c.A.rows,
                            cudaMemcpyDefault, c.stream));
    WG_CUDA(cudaStreamSynchronize(c.stream));
  });
}

weft_status weft_gpu_pcg(weft_gpu_ctx* ctx, const double* b, double* x, const weft_pcg_config* config,
                         weft_pcg_report* report) {
  return guard(ctx, [&] {
    auto& c = ctx->c;
    need(c.has_matrix, WEFT_ERR_INVALID, "pcg: no matrix");
    need(config != nullptr, WEFT_ERR_INVALID, "pcg: config is NULL");
    const size_t len = 3 * static_cast<size_t>(c.pm.p);
    const double* bdev = nullptr;
    if (b) {
      c.bvec.resize(len);
      WG_CUDA(cudaMemcpyAsync(c.bvec.data(), b, len * sizeof(double), cudaMemcpyDefault, c.stream));
      bdev = c.bvec.data();
    } else {
      need(c.has_rhs, WEFT_ERR_INVALID, "pcg: b is NULL and no assembled rhs");
      bdev = c.rhs.data();
    }
    weft_gpu::PcgResult r;
    try {
      r = weft_gpu::pcg_solve(c, bdev, *config, report ? report->residual_history : nullptr,
                              report ? report->precond_norm_history : nullptr);
    } catch (...) {
      if (report) report->iterations = 0;
      throw;
    }
    if (report) {
      report->iterations = r.iterations;
      report->converged = r.converged;
      report->rel_residual = r.rel_residual;
    }
    if (x) {
      const size_t o = 3 * static_cast<size_t>(c.row0), m = 3 * static_cast<size_t>(c.A.rows);
      if (r.iterations == 0) WG_CUDA(cudaMemsetAsync(c.xs.data() + o, 0, m * sizeof(double), c.stream));
      WG_CUDA(cudaMemcpyAsync(x + o, c.xs.data() + o, m * sizeof(double), cudaMemcpyDefault, c.stream));
      WG_CUDA(cudaStreamSynchronize(c.stream));
    }
  });
}

weft_status weft_gpu_comm_export(weft_gpu_ctx* ctx, void* handle_out) {
  return guard(ctx, [&] {
    need(handle_out != nullptr, WEFT_ERR_INVALID, "comm_export: handle_out is NULL");
    weft_gpu::comm_export(ctx->c, handle_out);
  });
}

weft_status weft_gpu_comm_attach(weft_gpu_ctx* ctx, const void* handles) {
  return guard(ctx, [&] {
    need(handles != nullptr, WEFT_ERR_INVALID, "comm_attach: handles is NULL");
    weft_gpu::comm_attach(ctx->c, handles);
  });
}

weft_status weft_gpu_rank_info(weft_gpu_ctx* ctx, weft_rank_info* info) {
  return guard(ctx, [&] {
    auto& c = ctx->c;
    info->world = c.world;
    info->rank = c.rank;
    info->first_row = c.row0;
    info->rows = c.row1 - c.row0;
    info->global_rows = c.pm.p;
  });
}

weft_status weft_gpu_profile(weft_gpu_ctx* ctx, int32_t enable) {
  return guard(ctx, [&] {
    ctx->c.profile = enable != 0;
    ctx->c.spmv_launches = 0;
    ctx->c.spmv_ms = 0.0;
    ctx->c.pcg_solves = 0;
    ctx->c.pcg_iterations = 0;
    ctx->c.pcg_ms = 0.0;
    ctx->c.pcg_bytes = 0.0;
  });
}

weft_status weft_gpu_set_instrument(weft_gpu_ctx* ctx, int32_t on) {
  return guard(ctx, [&] {
    ctx->c.instrument = on != 0;
    if (!on) ctx->c.log.clear();
  });
}

weft_status weft_gpu_take_log(weft_gpu_ctx* ctx, char* buf, int64_t cap, int64_t* len) {
  return guard(ctx, [&] {
    std::string& l = ctx->c.log;
    if (len) *len = static_cast<int64_t>(l.size());
    if (!buf || cap < static_cast<int64_t>(l.size()) + 1) return;
    std::memcpy(buf, l.data(), l.size());
    buf[l.size()] = '\0';
    l.clear();
  });
}

weft_status weft_gpu_stats(weft_gpu_ctx* ctx, weft_gpu_stats_t* out) {
  return guard(ctx, [&] {
    out->launches = ctx->c.launches;
    out->spmv_launches = ctx->c.spmv_launches;
    out->spmv_ms = ctx->c.spmv_ms;
    out->pcg_solves = ctx->c.pcg_solves;
    out->pcg_iterations = ctx->c.pcg_iterations;
    out->pcg_ms = ctx->c.pcg_ms;
    out->pcg_bytes = ctx->c.pcg_bytes;
  });
}

weft_status weft_gpu_test_serial_sum(weft_gpu_ctx* ctx, int32_t n, const double* d, int32_t fast,
                                     double* mean_exact, double* sum_naive) {
  return guard(ctx, [&] { weft_gpu::serial_sum(ctx->c, n, d, mean_exact, sum_naive, fast); });
}

weft_status weft_gpu_get_stream(weft_gpu_ctx* ctx, void** stream) {
  return guard(ctx, [&] { *stream = static_cast<void*>(ctx->c.stream); });
}

}  // extern "C"
