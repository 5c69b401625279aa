// Multi-GPU z-slab transport of the host runtime: the NCCL / in-process hub
// window, halo exchange of boundary planes (overlapped with interior work)
// and the device / host all-reductions. Part of the capi.cu translation unit.
#pragma once
// ------------------------------------------------- multi-GPU z-slab comm

static int setup_window(isc_ctx* ctx, int32_t rank, int32_t nranks, int32_t has_lo,
                        int32_t has_hi, int32_t kw_lo, int32_t kw_hi) {
  if (kw_lo < 0 || kw_hi > ctx->g.nz || kw_lo >= kw_hi || (has_lo && kw_lo < 1) ||
      (has_hi && kw_hi > ctx->g.nz - 1)) {
    g_err = "bad owned plane window";
    return ISC_BAD_ARGUMENT;
  }
  if (ctx->precond == ISC_PRECOND_RAS || ctx->precond == ISC_PRECOND_BJACOBI) {
    g_err = "multi-rank solves use mcilu or none (rank-local block-Jacobi of the multicolour ILU)";
    return ISC_UNSUPPORTED;
  }
  ctx->g.kw_lo = kw_lo;
  ctx->g.kw_hi = kw_hi;
  ctx->g.tw_lo = ctx->g.colored ? (int64_t)kw_lo * ctx->g.ph : 0;
  ctx->g.tw_hi = ctx->g.colored ? (int64_t)kw_hi * ctx->g.ph : ctx->g.half;
  ctx->comm.rank = rank;
  ctx->comm.nranks = nranks;
  ctx->comm.has_lo = has_lo != 0;
  ctx->comm.has_hi = has_hi != 0;
  // one plane of up to NB rows (vectors: NU; boundary blocks for the factor: NB)
  const size_t bytes = (size_t)NB * ctx->g.nxny * 8;
  if (!ctx->halo_send_lo) {
    ALLOC(ctx->halo_send_lo, bytes);
    ALLOC(ctx->halo_send_hi, bytes);
    ALLOC(ctx->halo_recv_lo, bytes);
    ALLOC(ctx->halo_recv_hi, bytes);
  }
  return ISC_OK;
}

extern "C" int isc_comm_nccl(isc_ctx* ctx, const void* unique_id, int32_t rank, int32_t nranks,
                             int32_t has_lo, int32_t has_hi, int32_t kw_lo, int32_t kw_hi) {
  int s = setup_window(ctx, rank, nranks, has_lo, has_hi, kw_lo, kw_hi);
  if (s) return s;
  // ISC_NCCL_SINGLE=1: a one-rank communicator is created and used as well
  // (the slab code path with no neighbours: every all-reduce goes through
  // NCCL) -- the transport check that one GPU allows
  const char* single_env = std::getenv("ISC_NCCL_SINGLE");
  ctx->comm.single = nranks == 1 && single_env && std::atoi(single_env) != 0;
  if (nranks > 1 || ctx->comm.single) {
    NcclApi& api = nccl_api();
    if (!api.ok) { g_err = "libnccl.so.2 not available in this process"; return ISC_UNSUPPORTED; }
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    const int r = api.CommInitRank(&ctx->comm.nccl, nranks, id, rank);
    if (r != ncclSuccess_) {
      g_err = std::string("ncclCommInitRank: ") + (api.GetErrorString ? api.GetErrorString(r) : "");
      return ISC_CUDA_ERROR;
    }
  }
  return ISC_OK;
}

extern "C" int isc_comm_is_nccl(isc_ctx* ctx) {
  return ctx->comm.active() && ctx->comm.nccl != nullptr ? 1 : 0;
}

extern "C" int isc_nccl_unique_id(void* out128) {
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) { g_err = "libnccl.so.2 not found"; return ISC_UNSUPPORTED; }
  auto fn = (int (*)(ncclUniqueId*))dlsym(h, "ncclGetUniqueId");
  if (!fn) { g_err = "ncclGetUniqueId not found"; return ISC_UNSUPPORTED; }
  ncclUniqueId id;
  if (fn(&id) != ncclSuccess_) { g_err = "ncclGetUniqueId failed"; return ISC_CUDA_ERROR; }
  std::memcpy(out128, &id, sizeof(id));
  return ISC_OK;
}

extern "C" void* isc_hub_create(int32_t nranks) {
  Hub* h = new Hub();
  h->nranks = nranks;
  h->send_lo.assign(nranks, nullptr);
  h->send_hi.assign(nranks, nullptr);
  h->ready.assign(nranks, nullptr);
  h->red.assign((size_t)nranks * 64, 0.0);
  return h;
}
extern "C" int isc_hub_destroy(void* hub) {
  delete (Hub*)hub;
  return ISC_OK;
}

extern "C" int isc_comm_hub(isc_ctx* ctx, void* hub, int32_t rank, int32_t has_lo, int32_t has_hi,
                            int32_t kw_lo, int32_t kw_hi) {
  Hub* h = (Hub*)hub;
  int s = setup_window(ctx, rank, h->nranks, has_lo, has_hi, kw_lo, kw_hi);
  if (s) return s;
  ctx->comm.hub = h;
  h->send_lo[rank] = ctx->halo_send_lo;
  h->send_hi[rank] = ctx->halo_send_hi;
  CK(cudaEventCreateWithFlags(&h->ready[rank], cudaEventDisableTiming));
  return ISC_OK;
}

// one-plane halo of a storage-order vector (rows x n)
// Halo exchange in two halves so that work not touching the ghost planes
// can run in between: halo_start packs the boundary planes on the main
// stream; halo_finish moves them on the copy stream (NCCL send/recv, or
// device copies between hub contexts), unpacks into the ghost planes there
// and makes the main stream wait for it.
static int halo_start(isc_ctx* ctx, double* v, int rows) {
  Comm& cm = ctx->comm;
  if (!cm.active()) return ISC_OK;
  const Dims& g = ctx->g;
  cudaStream_t st = ctx->stream;
  const int64_t cnt = (int64_t)rows * g.nxny;
  const int bl = grid1d(cnt, 256);
  if (cm.has_lo) k_pack_plane<<<bl, 256, 0, st>>>(g, rows, g.kw_lo, v, ctx->halo_send_lo);
  if (cm.has_hi) k_pack_plane<<<bl, 256, 0, st>>>(g, rows, g.kw_hi - 1, v, ctx->halo_send_hi);
  ctx->launches += (cm.has_lo ? 1 : 0) + (cm.has_hi ? 1 : 0);
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->halo_ev[0], st));
  return ISC_OK;
}

static int halo_finish(isc_ctx* ctx, double* v, int rows) {
  Comm& cm = ctx->comm;
  if (!cm.active()) return ISC_OK;
  const Dims& g = ctx->g;
  cudaStream_t st = ctx->stream, cs = ctx->cstream;
  const int64_t cnt = (int64_t)rows * g.nxny;
  const int bl = grid1d(cnt, 256);
  CK(cudaStreamWaitEvent(cs, ctx->halo_ev[0], 0));
  if (cm.nccl) {
    NcclApi& api = nccl_api();
    api.GroupStart();
    if (cm.has_lo) {
      api.Send(ctx->halo_send_lo, cnt, ncclFloat64_, cm.rank - 1, cm.nccl, cs);
      api.Recv(ctx->halo_recv_lo, cnt, ncclFloat64_, cm.rank - 1, cm.nccl, cs);
    }
    if (cm.has_hi) {
      api.Send(ctx->halo_send_hi, cnt, ncclFloat64_, cm.rank + 1, cm.nccl, cs);
      api.Recv(ctx->halo_recv_hi, cnt, ncclFloat64_, cm.rank + 1, cm.nccl, cs);
    }
    const int r = api.GroupEnd();
    if (r != ncclSuccess_) { g_err = "NCCL halo exchange failed"; return ISC_CUDA_ERROR; }
  } else if (cm.hub) {
    Hub* h = cm.hub;
    CK(cudaEventRecord(h->ready[cm.rank], cs));   // after the pack (cs waited for it)
    h->barrier();
    if (cm.has_lo) {
      CK(cudaStreamWaitEvent(cs, h->ready[cm.rank - 1], 0));
      CK(cudaMemcpyAsync(ctx->halo_recv_lo, h->send_hi[cm.rank - 1], cnt * 8,
                         cudaMemcpyDeviceToDevice, cs));
    }
    if (cm.has_hi) {
      CK(cudaStreamWaitEvent(cs, h->ready[cm.rank + 1], 0));
      CK(cudaMemcpyAsync(ctx->halo_recv_hi, h->send_lo[cm.rank + 1], cnt * 8,
                         cudaMemcpyDeviceToDevice, cs));
    }
    CK(cudaStreamSynchronize(cs));
    h->barrier();   // neighbours may now reuse their send buffers
  }
  if (cm.has_lo) k_unpack_plane<<<bl, 256, 0, cs>>>(g, rows, g.kw_lo - 1, ctx->halo_recv_lo, v);
  if (cm.has_hi) k_unpack_plane<<<bl, 256, 0, cs>>>(g, rows, g.kw_hi, ctx->halo_recv_hi, v);
  ctx->launches += (cm.has_lo ? 1 : 0) + (cm.has_hi ? 1 : 0);
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->halo_ev[1], cs));
  CK(cudaStreamWaitEvent(st, ctx->halo_ev[1], 0));
  return ISC_OK;
}

static int halo_exchange(isc_ctx* ctx, double* v, int rows) {
  int s = halo_start(ctx, v, rows);
  if (s) return s;
  return halo_finish(ctx, v, rows);
}

// sum `count` consecutive device scalars over the ranks (in place)
static int allreduce_dev(isc_ctx* ctx, double* d, int count) {
  Comm& cm = ctx->comm;
  if (!cm.active()) return ISC_OK;
  if (cm.nccl) {
    const int r = nccl_api().AllReduce(d, d, count, ncclFloat64_, ncclSum_, cm.nccl, ctx->stream);
    if (r != ncclSuccess_) { g_err = "NCCL allreduce failed"; return ISC_CUDA_ERROR; }
    return ISC_OK;
  }
  Hub* h = cm.hub;
  double loc[64];
  CK(cudaMemcpyAsync(loc, d, count * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  std::memcpy(&h->red[(size_t)cm.rank * 64], loc, count * 8);
  h->barrier();
  for (int i = 0; i < count; ++i) {
    double s = 0.0;
    for (int q = 0; q < h->nranks; ++q) s += h->red[(size_t)q * 64 + i];   // rank order
    loc[i] = s;
  }
  h->barrier();
  CK(cudaMemcpyAsync(d, loc, count * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return ISC_OK;
}

// host-side reductions over ranks: op 0 sum, 1 max (NaN propagates)
extern "C" int isc_comm_allreduce_host(isc_ctx* ctx, double* vals, int32_t count, int32_t op) {
  Comm& cm = ctx->comm;
  if (!cm.active() || count <= 0) return ISC_OK;
  if (count > 64) { g_err = "too many values"; return ISC_BAD_ARGUMENT; }
  if (cm.nccl) {
    // NCCL's max on doubles drops NaN (fmax semantics), so a NaN norm on one
    // rank would vanish behind the others' finite values. For op max the
    // values go as (NaN -> +inf, NaN flag) pairs in one reduction and NaN is
    // restored wherever any rank had one (the hub path below propagates it).
    double buf[128];
    const int len = op ? 2 * count : count;
    for (int i = 0; i < count; ++i) {
      const bool nan = vals[i] != vals[i];
      buf[i] = (op && nan) ? INFINITY : vals[i];
      if (op) buf[count + i] = nan ? 1.0 : 0.0;
    }
    double* d = ctx->partial;   // scratch
    CK(cudaMemcpyAsync(d, buf, len * 8, cudaMemcpyHostToDevice, ctx->stream));
    const int r = nccl_api().AllReduce(d, d, len, ncclFloat64_, op ? ncclMax_ : ncclSum_,
                                       cm.nccl, ctx->stream);
    if (r != ncclSuccess_) { g_err = "NCCL allreduce failed"; return ISC_CUDA_ERROR; }
    CK(cudaMemcpyAsync(buf, d, len * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < count; ++i) vals[i] = (op && buf[count + i] > 0.0) ? NAN : buf[i];
    return ISC_OK;
  }
  Hub* h = cm.hub;
  std::memcpy(&h->red[(size_t)cm.rank * 64], vals, count * 8);
  h->barrier();
  for (int i = 0; i < count; ++i) {
    double s = op ? h->red[i] : 0.0;
    for (int q = op ? 1 : 0; q < h->nranks; ++q) {
      const double v = h->red[(size_t)q * 64 + i];
      s = op ? ((v != v || s != s) ? v + s : std::max(s, v)) : s + v;
    }
    vals[i] = s;
  }
  h->barrier();
  return ISC_OK;
}

