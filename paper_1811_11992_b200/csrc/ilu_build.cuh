// Host-side structure of the reference-exact subdomain ILU(0) (ras /
// bjacobi): the slab partition, the per-subdomain slot and level order and
// the lower / upper coupling lists that k_ilu_factor / k_ilu_apply walk
// (grid.py:148-186, linsolve.py:262-358). Part of the capi.cu translation unit.
#pragma once
// ------------------------------------------------------ ILU structure
// Subdomains exactly as the reference: count min(64, max(1, n // 2048))
// (linsolve.py:34-42), slabs along the first longest axis with the
// remainder on the leading slabs (grid.py:148-166); RAS extends each slab
// by its one-plane halo (linsolve.py:341-345), bjacobi does not.
static int build_ilu(isc_ctx* ctx) {
  const Dims& g = ctx->g;
  const int64_t n = g.n;
  const int nsub = (int)std::min<int64_t>(64, std::max<int64_t>(1, n / 2048));
  const int dims[3] = {g.nx, g.ny, g.nz};
  int axis = 0;
  for (int a = 1; a < 3; ++a)
    if (dims[a] > dims[axis]) axis = a;
  const int na = dims[axis];
  const int base = na / nsub, extra = na % nsub;
  struct Box { int lo[3], hi[3], olo, ohi; };
  std::vector<Box> boxes;
  int pos = 0;
  for (int s = 0; s < nsub; ++s) {
    const int size = base + (s < extra ? 1 : 0);
    Box b;
    for (int a = 0; a < 3; ++a) { b.lo[a] = 0; b.hi[a] = dims[a]; }
    b.olo = pos;
    b.ohi = pos + size;
    b.lo[axis] = pos;
    b.hi[axis] = pos + size;
    if (ctx->precond == ISC_PRECOND_RAS && nsub > 1) {
      b.lo[axis] = std::max(0, pos - 1);
      b.hi[axis] = std::min(na, pos + size + 1);
    }
    pos += size;
    boxes.push_back(b);
  }
  // slots: subdomain-major, level-major inside a subdomain box; the level
  // of a cell is (i-x0)+(j-y0)+(k-z0) (its dependencies sit one level lower)
  int maxlev = 0;
  for (auto& b : boxes)
    maxlev = std::max(maxlev, (b.hi[0] - b.lo[0] - 1) + (b.hi[1] - b.lo[1] - 1) + (b.hi[2] - b.lo[2] - 1));
  const int nlev = maxlev + 1;
  std::vector<int64_t> lvl_ptr((size_t)nsub * (nlev + 1), 0);
  int64_t total = 0;
  for (int s = 0; s < nsub; ++s) {
    const Box& b = boxes[s];
    std::vector<int64_t> cnt(nlev, 0);
    for (int k = b.lo[2]; k < b.hi[2]; ++k)
      for (int j = b.lo[1]; j < b.hi[1]; ++j)
        for (int i = b.lo[0]; i < b.hi[0]; ++i) cnt[(i - b.lo[0]) + (j - b.lo[1]) + (k - b.lo[2])]++;
    int64_t* lp = lvl_ptr.data() + (size_t)s * (nlev + 1);
    lp[0] = total;
    for (int l = 0; l < nlev; ++l) lp[l + 1] = lp[l] + cnt[l];
    total = lp[nlev];
  }
  const int64_t ns = total;
  std::vector<int64_t> cell(ns), lo(3 * ns, -1), up(3 * ns, -1);
  std::vector<int8_t> owned(ns, 0);
  for (int sidx = 0; sidx < nsub; ++sidx) {
    const Box& b = boxes[sidx];
    std::vector<int64_t> fill(lvl_ptr.begin() + (size_t)sidx * (nlev + 1),
                              lvl_ptr.begin() + (size_t)sidx * (nlev + 1) + nlev);
    const int wx = b.hi[0] - b.lo[0], wy = b.hi[1] - b.lo[1], wz = b.hi[2] - b.lo[2];
    std::vector<int64_t> slot((size_t)wx * wy * wz);
    for (int k = b.lo[2]; k < b.hi[2]; ++k)
      for (int j = b.lo[1]; j < b.hi[1]; ++j)
        for (int i = b.lo[0]; i < b.hi[0]; ++i) {
          const int li = i - b.lo[0], lj = j - b.lo[1], lk = k - b.lo[2];
          const int64_t s = fill[li + lj + lk]++;
          slot[((size_t)lk * wy + lj) * wx + li] = s;
          cell[s] = pos_of(g, i + (int64_t)g.nx * (j + (int64_t)g.ny * k));
          const int ijk[3] = {i, j, k};
          owned[s] = (ijk[axis] >= b.olo && ijk[axis] < b.ohi) ? 1 : 0;
        }
    for (int lk = 0; lk < wz; ++lk)
      for (int lj = 0; lj < wy; ++lj)
        for (int li = 0; li < wx; ++li) {
          const int64_t s = slot[((size_t)lk * wy + lj) * wx + li];
          auto at = [&](int a, int bb, int c) { return slot[((size_t)c * wy + bb) * wx + a]; };
          // lower in ascending neighbour index: -z, -y, -x
          if (lk > 0) lo[0 * ns + s] = at(li, lj, lk - 1);
          if (lj > 0) lo[1 * ns + s] = at(li, lj - 1, lk);
          if (li > 0) lo[2 * ns + s] = at(li - 1, lj, lk);
          // upper ascending: +x, +y, +z
          if (li + 1 < wx) up[0 * ns + s] = at(li + 1, lj, lk);
          if (lj + 1 < wy) up[1 * ns + s] = at(li, lj + 1, lk);
          if (lk + 1 < wz) up[2 * ns + s] = at(li, lj, lk + 1);
        }
  }
  ctx->nsub = nsub;
  int64_t *cell_d, *lo_d, *up_d;
  int8_t* owned_d;
  ALLOC(cell_d, ns * 8);
  ALLOC(lo_d, 3 * ns * 8);
  ALLOC(up_d, 3 * ns * 8);
  ALLOC(owned_d, ns);
  ALLOC(ctx->lvl_ptr_d, lvl_ptr.size() * 8);
  CK(cudaMemcpy(cell_d, cell.data(), ns * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(lo_d, lo.data(), 3 * ns * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(up_d, up.data(), 3 * ns * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(owned_d, owned.data(), ns, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ctx->lvl_ptr_d, lvl_ptr.data(), lvl_ptr.size() * 8, cudaMemcpyHostToDevice));
  double *lblk, *uinv, *zs, *aup;
  ALLOC(aup, (size_t)3 * NB * ns * 8);
  ALLOC(lblk, (size_t)3 * NB * ns * 8);
  ALLOC(uinv, (size_t)NB * ns * 8);
  ALLOC(zs, (size_t)NU * ns * 8);
  ctx->ilu = IluDev{ns, cell_d, owned_d, lo_d, up_d, lblk, uinv, zs, aup};
  ctx->nlev = nlev;
  return ISC_OK;
}

