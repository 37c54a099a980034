// pack_gpu.cu -- the packer's slot and variable phases on the GPU (SURVEY §8(f)
// f2; FDOG_GPU_PACK=1): canonical slots, J_i as CSR over the variables in the
// order of their first device slot, and every variable's device slots in
// ascending j (A1).  The same construction as plan.cpp's host phases, so the
// arrays are identical (tests/test_gpu_compile.py compares plan digests):
//   * canonical slot q of (local row r, hop h): q = q0[r] + h, q0 = exclusive
//     scan of the row lengths; device slot row_slot[j] + h row_L[j];
//   * each variable's first device slot by atomic min; the device slots that
//     are a first occurrence, compacted in device-slot order, give var_list;
//   * var_ptr = exclusive scan of the local degrees in var_list order;
//   * var_slots: the canonical slots stably sorted by their variable's
//     position in var_list (radix sort: within a variable ascending q, i.e.
//     ascending j), mapped to device slots.
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <climits>
#include <vector>

#include "internal.h"

namespace fdog {
namespace {

__global__ void row_len_kernel(int64_t nr, const int32_t *rows, const int64_t *row_ptr, int64_t *len) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r < nr) len[r] = row_ptr[rows[r] + 1] - row_ptr[rows[r]];
}

__global__ void canon_kernel(int64_t nr, const int32_t *rows, const int64_t *row_ptr, const int32_t *col_var,
                             const int64_t *row_slot, const int32_t *row_L, const int64_t *q0, int64_t *canon_slot,
                             int32_t *canon_con, int32_t *canon_pos, int32_t *canon_var, int32_t *cnt) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= nr) return;
  const int32_t j = rows[r];
  const int64_t a = row_ptr[j];
  const int32_t k = (int32_t)(row_ptr[j + 1] - a);
  for (int32_t h = 0; h < k; ++h) {
    const int64_t q = q0[r] + h;
    const int32_t v = col_var[a + h];
    canon_slot[q] = row_slot[j] + (int64_t)h * row_L[j];
    canon_con[q] = j;
    canon_pos[q] = h;
    canon_var[q] = v;
    atomicAdd(cnt + v, 1);
  }
}

__global__ void first_kernel(int64_t ns, const int32_t *slot_var, int32_t *first) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d < ns && slot_var[d] >= 0) atomicMin(first + slot_var[d], (int32_t)d);
}

__global__ void flag_kernel(int64_t ns, const int32_t *slot_var, const int32_t *first, int32_t *flag) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d < ns) flag[d] = (slot_var[d] >= 0 && first[slot_var[d]] == (int32_t)d) ? 1 : 0;
}

__global__ void compact_kernel(int64_t ns, const int32_t *slot_var, const int32_t *flag, const int32_t *pos,
                               int32_t *var_list, int32_t *where) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d < ns && flag[d]) {
    var_list[pos[d]] = slot_var[d];
    where[slot_var[d]] = pos[d];
  }
}

__global__ void degree_kernel(int64_t nv, const int32_t *var_list, const int32_t *cnt, int64_t *deg) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < nv) deg[k] = cnt[var_list[k]];
}

__global__ void key_kernel(int64_t nq, const int32_t *canon_var, const int32_t *where, int32_t *key, int32_t *idx) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q < nq) {
    key[q] = where[canon_var[q]];
    idx[q] = (int32_t)q;
  }
}

__global__ void slots_kernel(int64_t nq, const int32_t *sorted_q, const int64_t *canon_slot, int32_t *var_slots) {
  const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x < nq) var_slots[x] = (int32_t)canon_slot[sorted_q[x]];
}

unsigned grid_of(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + 255) / 256); }

struct DevBufs {
  std::vector<void *> p;
  ~DevBufs() {
    for (void *x : p) cudaFree(x);
  }
  template <typename V>
  V *get(size_t n) {
    void *x = nullptr;
    if (cudaMalloc(&x, std::max<size_t>(n, 1) * sizeof(V)) != cudaSuccess) return nullptr;
    p.push_back(x);
    return (V *)x;
  }
};

}  // namespace

fdog_status gpu_pack_slots(Plan &P, const std::vector<int64_t> &row_slot, const std::vector<int32_t> &row_L,
                           int device) {
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return FDOG_ECUDA;
  const int64_t nr = (int64_t)P.local_rows.size(), ns = (int64_t)P.slot_var.size();
  const int64_t n_cons = (int64_t)P.row_ptr.size() - 1, nnz = P.row_ptr.back();
  const int32_t n_vars = P.n_vars;
  DevBufs B;
  int32_t *d_rows = B.get<int32_t>(nr), *d_col = B.get<int32_t>(nnz), *d_rowL = B.get<int32_t>(n_cons);
  int64_t *d_rp = B.get<int64_t>(n_cons + 1), *d_rslot = B.get<int64_t>(n_cons);
  int32_t *d_svar = B.get<int32_t>(ns);
  int64_t *d_len = B.get<int64_t>(nr + 1), *d_q0 = B.get<int64_t>(nr + 1);
  if (!d_rows || !d_col || !d_rowL || !d_rp || !d_rslot || !d_svar || !d_len || !d_q0) return FDOG_ENOMEM;
  auto up = [&](void *dst, const void *src, size_t bytes) {
    return bytes ? cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice) : cudaSuccess;
  };
  if (up(d_rows, P.local_rows.data(), nr * 4) || up(d_col, P.col_var.data(), nnz * 4) ||
      up(d_rowL, row_L.data(), n_cons * 4) || up(d_rp, P.row_ptr.data(), (n_cons + 1) * 8) ||
      up(d_rslot, row_slot.data(), n_cons * 8) || up(d_svar, P.slot_var.data(), ns * 4))
    return FDOG_ECUDA;
  // q0: exclusive scan of the local row lengths
  row_len_kernel<<<grid_of(nr), 256>>>(nr, d_rows, d_rp, d_len);
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_len, d_q0, (int)nr + 1);
  void *d_tmp = B.get<unsigned char>(tmp_bytes);
  if (!d_tmp) return FDOG_ENOMEM;
  if (cudaMemset(d_len + nr, 0, 8)) return FDOG_ECUDA;
  cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_len, d_q0, (int)nr + 1);
  const int64_t nq = P.n_slots;
  int64_t *d_cslot = B.get<int64_t>(nq);
  int32_t *d_ccon = B.get<int32_t>(nq), *d_cpos = B.get<int32_t>(nq), *d_cvar = B.get<int32_t>(nq);
  int32_t *d_cnt = B.get<int32_t>(n_vars), *d_first = B.get<int32_t>(n_vars), *d_where = B.get<int32_t>(n_vars);
  int32_t *d_flag = B.get<int32_t>(ns + 1), *d_pos = B.get<int32_t>(ns + 1);
  if (!d_cslot || !d_ccon || !d_cpos || !d_cvar || !d_cnt || !d_first || !d_where || !d_flag || !d_pos)
    return FDOG_ENOMEM;
  if (cudaMemset(d_cnt, 0, (size_t)std::max(n_vars, 1) * 4) || cudaMemset(d_first, 0x7f, (size_t)std::max(n_vars, 1) * 4))
    return FDOG_ECUDA;
  canon_kernel<<<grid_of(nr), 256>>>(nr, d_rows, d_rp, d_col, d_rslot, d_rowL, d_q0, d_cslot, d_ccon, d_cpos, d_cvar,
                                     d_cnt);
  first_kernel<<<grid_of(ns), 256>>>(ns, d_svar, d_first);
  flag_kernel<<<grid_of(ns), 256>>>(ns, d_svar, d_first, d_flag);
  if (cudaMemset(d_flag + ns, 0, 4)) return FDOG_ECUDA;
  size_t t2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t2, d_flag, d_pos, (int)ns + 1);
  void *d_tmp2 = B.get<unsigned char>(t2);
  if (!d_tmp2) return FDOG_ENOMEM;
  cub::DeviceScan::ExclusiveSum(d_tmp2, t2, d_flag, d_pos, (int)ns + 1);
  int32_t nv = 0;
  if (cudaMemcpy(&nv, d_pos + ns, 4, cudaMemcpyDeviceToHost)) return FDOG_ECUDA;
  int32_t *d_vlist = B.get<int32_t>(nv);
  int64_t *d_deg = B.get<int64_t>((int64_t)nv + 1), *d_vptr = B.get<int64_t>((int64_t)nv + 1);
  if (!d_vlist || !d_deg || !d_vptr) return FDOG_ENOMEM;
  compact_kernel<<<grid_of(ns), 256>>>(ns, d_svar, d_flag, d_pos, d_vlist, d_where);
  degree_kernel<<<grid_of(nv), 256>>>(nv, d_vlist, d_cnt, d_deg);
  if (cudaMemset(d_deg + nv, 0, 8)) return FDOG_ECUDA;
  size_t t3 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t3, d_deg, d_vptr, nv + 1);
  void *d_tmp3 = B.get<unsigned char>(t3);
  if (!d_tmp3) return FDOG_ENOMEM;
  cub::DeviceScan::ExclusiveSum(d_tmp3, t3, d_deg, d_vptr, nv + 1);
  // canonical slots stably sorted by their variable's position in var_list
  int32_t *d_key = B.get<int32_t>(nq), *d_idx = B.get<int32_t>(nq), *d_key2 = B.get<int32_t>(nq),
          *d_idx2 = B.get<int32_t>(nq), *d_vslots = B.get<int32_t>(nq);
  if (!d_key || !d_idx || !d_key2 || !d_idx2 || !d_vslots) return FDOG_ENOMEM;
  key_kernel<<<grid_of(nq), 256>>>(nq, d_cvar, d_where, d_key, d_idx);
  int bits = 1;
  while (bits < 31 && (int64_t(1) << bits) < (int64_t)nv) ++bits;
  size_t t4 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t4, d_key, d_key2, d_idx, d_idx2, (int)nq, 0, bits);
  void *d_tmp4 = B.get<unsigned char>(t4);
  if (!d_tmp4) return FDOG_ENOMEM;
  cub::DeviceRadixSort::SortPairs(d_tmp4, t4, d_key, d_key2, d_idx, d_idx2, (int)nq, 0, bits);
  slots_kernel<<<grid_of(nq), 256>>>(nq, d_idx2, d_cslot, d_vslots);
  if ((e = cudaGetLastError()) != cudaSuccess) return FDOG_ECUDA;
  P.canon_slot.resize(nq);
  P.canon_con.resize(nq);
  P.canon_pos.resize(nq);
  P.var_list.resize(nv);
  P.var_ptr.resize((size_t)nv + 1);
  P.var_slots.resize(nq);
  auto down = [&](void *dst, const void *src, size_t bytes) {
    return bytes ? cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost) : cudaSuccess;
  };
  if (down(P.canon_slot.data(), d_cslot, nq * 8) || down(P.canon_con.data(), d_ccon, nq * 4) ||
      down(P.canon_pos.data(), d_cpos, nq * 4) || down(P.var_list.data(), d_vlist, (size_t)nv * 4) ||
      down(P.var_ptr.data(), d_vptr, ((size_t)nv + 1) * 8) || down(P.var_slots.data(), d_vslots, nq * 4))
    return FDOG_ECUDA;
  return FDOG_OK;
}

}  // namespace fdog
