// Multi-device ensembles behind the C-ABI (include/pbn_b200.h "device group";
// SURVEY §8e): trajectories are independent, so a job's global trajectory ids
// are split into contiguous per-rank ranges (one rank per device), the plan is
// replicated, and the ONLY collective is one NCCL all-reduce (sum) of the
// pooled counts — plus the pooled per-node one-counts when asked — over
// NVLink. Every draw is keyed by (seed, global trajectory id, step), so the
// totals are identical for any device count.
//
// Built on the public single-device entry points (pbn_gpu_create /
// pbn_gpu_run_device). NCCL is bound at run time (dlopen of libnccl.so.2:
// the copy a host process already loaded — e.g. PyTorch's — or the system
// one), so the library itself keeps loading on machines without NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pbn_b200.h"

namespace pbn_b200 {
void set_last_error(const std::string& msg);  // capi.cpp: what pbn_last_error() returns
cudaError_t launch_pool(const std::uint64_t* d_counts, const std::uint64_t* d_nc, std::uint32_t n,
                        std::uint32_t cols, unsigned long long* d_out, cudaStream_t stream);
}

namespace {

struct group_error : std::runtime_error {
  int code;
  group_error(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};

template <class F>
int gguard(F&& f) {
  try {
    f();
    return PBN_OK;
  } catch (const group_error& e) {
    pbn_b200::set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    pbn_b200::set_last_error("out of host memory");
    return PBN_ERESOURCE;
  } catch (const std::exception& e) {
    pbn_b200::set_last_error(e.what());
    return PBN_EUSAGE;
  }
}

void gck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw group_error(PBN_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// status of a single-device entry point -> exception (keeps its message)
void pck(int rc) {
  if (rc != PBN_OK) throw group_error(rc, pbn_last_error());
}

struct nccl_api {
  void* h = nullptr;
  std::string why;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const nccl_api& nccl() {
  static nccl_api api = [] {
    nccl_api a;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (a.h) break;
    }
    if (!a.h) {
      a.why = std::string("NCCL not loadable: ") + dlerror();
      return a;
    }
    auto sym = [&](auto& fp, const char* n) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(a.h, n));
      if (!fp && a.why.empty()) a.why = std::string("NCCL symbol missing: ") + n;
    };
    sym(a.get_unique_id, "ncclGetUniqueId");
    sym(a.comm_init_all, "ncclCommInitAll");
    sym(a.comm_init_rank, "ncclCommInitRank");
    sym(a.comm_destroy, "ncclCommDestroy");
    sym(a.all_reduce, "ncclAllReduce");
    sym(a.group_start, "ncclGroupStart");
    sym(a.group_end, "ncclGroupEnd");
    sym(a.error_string, "ncclGetErrorString");
    return a;
  }();
  if (!api.why.empty()) throw group_error(PBN_ERESOURCE, api.why);
  return api;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw group_error(PBN_ECUDA, std::string(what) + ": " + nccl().error_string(r));
}

// Contiguous [begin, begin + count) of n_total ids for `rank` of `world`
// (the same rule as paper_1605_00854_b200/ensemble.py shard_range).
void shard(std::uint64_t n_total, std::uint32_t world, std::uint32_t rank, std::uint64_t& begin,
           std::uint64_t& count) {
  const std::uint64_t base = n_total / world, extra = n_total % world;
  begin = rank * base + std::min<std::uint64_t>(rank, extra);
  count = base + (rank < extra ? 1 : 0);
}

template <class T>
struct dbuf {
  T* p = nullptr;
  std::size_t n = 0;
  void need(std::size_t want) {
    if (want <= n) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    gck(cudaMalloc(&p, sizeof(T) * (want ? want : 1)), "cudaMalloc group buffer");
    n = want;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

}  // namespace

struct pbn_group {
  struct member {
    int device = 0;
    pbn_gpu* eng = nullptr;
    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;
    dbuf<std::uint64_t> states, counts, nc;
    dbuf<unsigned long long> pool;
  };
  std::vector<member> m;
  std::uint32_t nranks = 1, first_rank = 0;
  std::uint32_t n_kept = 0;

  ~pbn_group() {
    for (auto& x : m) {
      cudaSetDevice(x.device);
      if (x.comm) nccl().comm_destroy(x.comm);
      if (x.stream) cudaStreamDestroy(x.stream);
      x.states.release();
      x.counts.release();
      x.nc.release();
      x.pool.release();
      if (x.eng) pbn_gpu_destroy(x.eng);
    }
  }
};

namespace {

std::unique_ptr<pbn_group> make_members(const pbn_plan_view* view, const std::vector<int>& devs,
                                        std::uint32_t lpt) {
  if (!view) throw std::invalid_argument("null argument: view");
  auto gr = std::make_unique<pbn_group>();
  gr->n_kept = view->n_kept;
  gr->m.resize(devs.size());
  for (std::size_t i = 0; i < devs.size(); ++i) {
    auto& x = gr->m[i];
    x.device = devs[i];
    pck(pbn_gpu_create(view, devs[i], lpt, &x.eng));
    gck(cudaSetDevice(devs[i]), "cudaSetDevice");
    gck(cudaStreamCreateWithFlags(&x.stream, cudaStreamNonBlocking), "cudaStreamCreate");
  }
  return gr;
}

}  // namespace

extern "C" {

int pbn_nccl_unique_id(uint8_t* id_out) {
  return gguard([&] {
    if (!id_out) throw std::invalid_argument("null argument: id_out");
    ncclUniqueId id;
    nck(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(id_out, id.internal, NCCL_UNIQUE_ID_BYTES);
  });
}

int pbn_group_create(const pbn_plan_view* view, const int* devices, uint32_t n_devices,
                     uint32_t lanes_per_traj, pbn_group** out) {
  return gguard([&] {
    if (!out) throw std::invalid_argument("null argument: out");
    if (n_devices == 0) throw std::invalid_argument("a device group needs at least one device");
    std::vector<int> devs(n_devices);
    for (uint32_t i = 0; i < n_devices; ++i) devs[i] = devices ? devices[i] : static_cast<int>(i);
    auto gr = make_members(view, devs, lanes_per_traj);
    gr->nranks = n_devices;
    gr->first_rank = 0;
    std::vector<ncclComm_t> comms(n_devices);
    nck(nccl().comm_init_all(comms.data(), static_cast<int>(n_devices), devs.data()),
        "ncclCommInitAll");
    for (uint32_t i = 0; i < n_devices; ++i) gr->m[i].comm = comms[i];
    *out = gr.release();
  });
}

int pbn_group_create_rank(const pbn_plan_view* view, int device, uint32_t nranks, uint32_t rank,
                          const uint8_t* nccl_id, uint32_t lanes_per_traj, pbn_group** out) {
  return gguard([&] {
    if (!out || !nccl_id) throw std::invalid_argument("null argument: out / nccl_id");
    if (nranks == 0 || rank >= nranks) throw std::invalid_argument("rank must be < nranks");
    auto gr = make_members(view, {device}, lanes_per_traj);
    gr->nranks = nranks;
    gr->first_rank = rank;
    ncclUniqueId id;
    std::memcpy(id.internal, nccl_id, NCCL_UNIQUE_ID_BYTES);
    gck(cudaSetDevice(device), "cudaSetDevice");
    nck(nccl().comm_init_rank(&gr->m[0].comm, static_cast<int>(nranks), id, static_cast<int>(rank)),
        "ncclCommInitRank");
    *out = gr.release();
  });
}

int pbn_group_info(const pbn_group* gr, uint32_t* n_members, uint32_t* nranks,
                   uint32_t* first_rank) {
  return gguard([&] {
    if (!gr) throw std::invalid_argument("null argument: group");
    if (n_members) *n_members = static_cast<uint32_t>(gr->m.size());
    if (nranks) *nranks = gr->nranks;
    if (first_rank) *first_rank = gr->first_rank;
  });
}

int pbn_group_shard(const pbn_group* gr, uint64_t n_total, uint32_t rank, uint64_t* begin,
                    uint64_t* count) {
  return gguard([&] {
    if (!gr || !begin || !count) throw std::invalid_argument("null argument");
    if (rank >= gr->nranks) throw std::invalid_argument("rank out of range");
    shard(n_total, gr->nranks, rank, *begin, *count);
  });
}

int pbn_group_member(const pbn_group* gr, uint32_t i, pbn_gpu** eng) {
  return gguard([&] {
    if (!gr || !eng) throw std::invalid_argument("null argument");
    if (i >= gr->m.size()) throw std::invalid_argument("member out of range");
    *eng = gr->m[i].eng;
  });
}

int pbn_group_run(pbn_group* gr, const pbn_run_args* a, uint64_t* states_inout,
                  uint64_t* counts_out, uint64_t* totals_out, uint64_t* node_totals_out) {
  return gguard([&] {
    if (!gr || !a || !states_inout || !totals_out)
      throw std::invalid_argument("null argument: group / args / states / totals");
    if (a->series || a->tprev)
      throw std::invalid_argument("group runs take no series / tprev buffers (use a member engine)");
    const bool nc = (a->flags & PBN_RUN_NODE_COUNTS) != 0;
    if (nc != (node_totals_out != nullptr))
      throw std::invalid_argument("PBN_RUN_NODE_COUNTS and node_totals_out go together");
    const std::size_t words = pbn_state_words(gr->n_kept);
    const std::size_t cols = gr->n_kept;
    const std::size_t pool_len = 8 + (nc ? cols : 0);
    std::uint64_t row0 = 0, dummy = 0;  // first global row of this process
    shard(a->n_traj, gr->nranks, gr->first_rank, row0, dummy);
    // 1) per member: its rows host -> device, the ensemble launch, the pooling
    //    kernels — asynchronous on the member's stream, members back to back
    std::vector<std::uint64_t> rb(gr->m.size()), rc(gr->m.size());
    for (std::size_t i = 0; i < gr->m.size(); ++i) {
      auto& x = gr->m[i];
      shard(a->n_traj, gr->nranks, gr->first_rank + static_cast<uint32_t>(i), rb[i], rc[i]);
      if (rc[i] > 0xFFFFFFFFull) throw std::invalid_argument("shard too large");
      gck(cudaSetDevice(x.device), "cudaSetDevice");
      x.states.need(rc[i] * words);
      x.counts.need(rc[i] * PBN_COUNT_FIELDS);
      x.pool.need(pool_len);
      if (nc) x.nc.need(rc[i] * cols);
      const std::uint64_t* src = states_inout + (rb[i] - row0) * words;
      gck(cudaMemcpyAsync(x.states.p, src, 8 * words * rc[i], cudaMemcpyHostToDevice, x.stream),
          "H2D states");
      if (nc) gck(cudaMemsetAsync(x.nc.p, 0, 8 * cols * rc[i], x.stream), "memset node counts");
      pbn_run_args la = *a;
      la.traj_begin = a->traj_begin + rb[i];
      la.n_traj = static_cast<uint32_t>(rc[i]);
      if (rc[i]) pck(pbn_gpu_run_device(x.eng, &la, x.states.p, x.counts.p, nc ? x.nc.p : nullptr, x.stream));
      gck(pbn_b200::launch_pool(x.counts.p, nc ? x.nc.p : nullptr, static_cast<uint32_t>(rc[i]),
                                static_cast<uint32_t>(cols), x.pool.p, x.stream),
          "pool kernels");
    }
    // 2) the single collective: sum of the pooled vectors over every rank
    nck(nccl().group_start(), "ncclGroupStart");
    for (auto& x : gr->m)
      nck(nccl().all_reduce(x.pool.p, x.pool.p, pool_len, ncclUint64, ncclSum, x.comm, x.stream),
          "ncclAllReduce");
    nck(nccl().group_end(), "ncclGroupEnd");
    // 3) results back: this process's rows, the job-wide totals from member 0
    std::vector<unsigned long long> tot(pool_len);
    for (std::size_t i = 0; i < gr->m.size(); ++i) {
      auto& x = gr->m[i];
      gck(cudaSetDevice(x.device), "cudaSetDevice");
      std::uint64_t* dst = states_inout + (rb[i] - row0) * words;
      gck(cudaMemcpyAsync(dst, x.states.p, 8 * words * rc[i], cudaMemcpyDeviceToHost, x.stream),
          "D2H states");
      if (counts_out)
        gck(cudaMemcpyAsync(counts_out + (rb[i] - row0) * PBN_COUNT_FIELDS, x.counts.p,
                            8 * PBN_COUNT_FIELDS * rc[i], cudaMemcpyDeviceToHost, x.stream),
            "D2H counts");
      if (i == 0)
        gck(cudaMemcpyAsync(tot.data(), x.pool.p, 8 * pool_len, cudaMemcpyDeviceToHost, x.stream),
            "D2H totals");
    }
    for (auto& x : gr->m) {
      gck(cudaSetDevice(x.device), "cudaSetDevice");
      gck(cudaStreamSynchronize(x.stream), "group run");
    }
    for (int f = 0; f < PBN_COUNT_FIELDS; ++f) totals_out[f] = tot[f];
    if (nc)
      for (std::size_t c = 0; c < cols; ++c) node_totals_out[c] = tot[8 + c];
  });
}

void pbn_group_destroy(pbn_group* gr) { delete gr; }

}  // extern "C"
