// Mesh preprocessing on the device: agglomeration of a simplicial mesh into
// the polytopic mesh (polydg agglomerate, mesh.py:328-473) -- SURVEY §8f-2.
//
// Same element / face / facet / interface order and the same geometric
// conventions as polydg (and as this package's vectorised numpy
// agglomerate, mesh.py), bit for bit:
//   1. elements: stable sort of the simplices by element id (elem_ptr,
//      elem_simplices ascending), boxes (min / max), volumes (np.add.reduceat's
//      order -- first + pairwise sum of the rest -- so the floats match);
//   2. facets: facet k of simplex s omits local vertex k (row s*(d+1)+k);
//      sorted vertex ids -> 64-bit key; stable radix sort; equal keys pair
//      two simplices (more than two: non-manifold); a pair inside one
//      element is internal and dropped;
//   3. connectivity check (mesh.py:419-425): union-find over the internal
//      pairs (atomic hooking), every element's simplices one component;
//   4. kept facets (key order): owner = lower element, the facet's vertex
//      order is the lower simplex row's, unit normal + measure from the
//      coordinates, flipped to point away from the owner simplex centroid;
//   5. interfaces: interior kept facets stable-sorted by (owner, neighbour),
//      boundary facets by owner; each set with more than one facet is split
//      into co-hyperplanar faces greedily in order (_group_by_hyperplane,
//      mesh.py:294-325: normal within 1e-9, distance to the first facet's
//      plane within 1e-9 of the running bounding-box diameter);
//   6. faces: owner / neighbour / normal of the first member, measure = the
//      members' sum in order, boundary faces per element.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <vector>

#include "pdg_internal.cuh"

namespace pdg {
namespace {

constexpr double NORMAL_TOL = 1e-9;  // polydg mesh.py:28-29
constexpr double PLANE_TOL = 1e-9;
constexpr int GREEDY_MAX = 64;       // facets of one (owner, neighbour) set handled by the greedy split

struct Bump {
  char* p;
  size_t left;
  bool ok = true;
  template <class T>
  T* take(int64_t n) {
    const size_t b = ((size_t)std::max<int64_t>(n, 1) * sizeof(T) + 255) & ~size_t(255);
    if (b > left) {
      ok = false;
      return nullptr;
    }
    T* r = reinterpret_cast<T*>(p);
    p += b;
    left -= b;
    return r;
  }
};

__global__ void iota_i64(int64_t* a, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = i;
}

__global__ void count_elems(const int64_t* agg, int64_t ns, int64_t nel, int64_t* cnt, uint32_t* flags) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = agg[i];
    if (e < 0 || e >= nel) {
      atomicOr(flags, 1u);
      continue;
    }
    atomicAdd(reinterpret_cast<unsigned long long*>(cnt + e), 1ull);
  }
}

__global__ void check_counts(const int64_t* cnt, int64_t nel, uint32_t* flags) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nel; e += (int64_t)gridDim.x * blockDim.x)
    if (cnt[e] == 0) atomicOr(flags, 1u);  // not surjective
}

// numpy's pairwise summation of a contiguous run (n <= 128: 8 partial sums)
__device__ double np_sum(const double* v, const int64_t* idx, int64_t n) {
  if (n < 8) {
    double s = -0.0;
    for (int64_t i = 0; i < n; ++i) s += v[idx[i]];
    return s;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = v[idx[j]];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] += v[idx[i + j]];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += v[idx[i]];
  return res;
}

template <int D>
__global__ void elem_geometry(const double* verts, const int32_t* simp, const double* svol, const int64_t* order,
                              const int64_t* eptr, int64_t nel, double* boxes, double* vols, int32_t* esimp) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nel; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = eptr[e], b = eptr[e + 1];
    double lo[D], hi[D];
    for (int k = 0; k < D; ++k) {
      lo[k] = PDG_INF;
      hi[k] = -PDG_INF;
    }
    for (int64_t i = a; i < b; ++i) {
      const int64_t s = order[i];
      esimp[i] = (int32_t)s;
      for (int v = 0; v <= D; ++v) {
        const double* x = verts + (int64_t)simp[s * (D + 1) + v] * D;
        for (int k = 0; k < D; ++k) {
          lo[k] = fmin(lo[k], x[k]);
          hi[k] = fmax(hi[k], x[k]);
        }
      }
    }
    for (int k = 0; k < D; ++k) {
      boxes[e * 2 * D + k] = lo[k];
      boxes[e * 2 * D + D + k] = hi[k];
    }
    // np.add.reduceat over a segment = first + pairwise sum of the rest
    vols[e] = b - a > 1 ? svol[order[a]] + np_sum(svol, order + a + 1, b - a - 1) : svol[order[a]];
  }
}

template <int D>
__device__ __forceinline__ void facet_ids(const int32_t* simp, int64_t row, int32_t* v) {
  const int64_t s = row / (D + 1);
  const int k = (int)(row - s * (D + 1));
  int c = 0;
  for (int j = 0; j <= D; ++j)
    if (j != k) v[c++] = simp[s * (D + 1) + j];
}

template <int D>
__global__ void facet_keys(const int32_t* simp, int64_t nrows, uint64_t* keys) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    int32_t v[D];
    facet_ids<D>(simp, r, v);
    // sort the d ids ascending
    for (int i = 1; i < D; ++i)
      for (int j = i; j > 0 && v[j] < v[j - 1]; --j) {
        const int32_t t = v[j];
        v[j] = v[j - 1];
        v[j - 1] = t;
      }
    uint64_t k = 0;
    const int bits = D == 2 ? 32 : 21;
    for (int i = 0; i < D; ++i) k = (k << bits) | (uint64_t)(uint32_t)v[i];
    keys[r] = k;
  }
}

// per sorted position: 1 where a new key starts
__global__ void head_flags(const uint64_t* ks, int64_t n, int64_t* head) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    head[i] = (i == 0 || ks[i] != ks[i - 1]) ? 1 : 0;
}

// per segment (facet): simplices on both sides, elements, internal flag
template <int D>
__global__ void segments(const uint64_t* ks, const int64_t* order, const int64_t* head_scan, int64_t n,
                         const int64_t* agg, int64_t* seg_r0, int64_t* seg_s1, uint8_t* seg_internal,
                         uint32_t* flags) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (!(i == 0 || ks[i] != ks[i - 1])) continue;
    int64_t size = 1;
    while (i + size < n && ks[i + size] == ks[i]) ++size;
    if (size > 2) atomicOr(flags, 2u);  // non-manifold
    const int64_t seg = head_scan[i];
    const int64_t r0 = order[i];
    seg_r0[seg] = r0;
    int64_t s1 = -1;
    if (size == 2) s1 = order[i + 1] / (D + 1);
    seg_s1[seg] = s1;
    seg_internal[seg] = (s1 >= 0 && agg[r0 / (D + 1)] == agg[s1]) ? 1 : 0;
  }
}

__device__ int64_t uf_find(int64_t* parent, int64_t x) {
  while (true) {
    const int64_t p = parent[x];
    if (p == x) return x;
    const int64_t gp = parent[p];
    if (gp != p) atomicCAS(reinterpret_cast<unsigned long long*>(parent + x), (unsigned long long)p,
                           (unsigned long long)gp);
    x = p;
  }
}

template <int D>
__global__ void uf_union(const int64_t* seg_r0, const int64_t* seg_s1, const uint8_t* internal, int64_t nseg,
                         int64_t* parent) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < nseg; g += (int64_t)gridDim.x * blockDim.x) {
    if (!internal[g]) continue;
    int64_t a = seg_r0[g] / (D + 1), b = seg_s1[g];
    while (true) {
      a = uf_find(parent, a);
      b = uf_find(parent, b);
      if (a == b) break;
      if (a < b) {
        const int64_t t = a;
        a = b;
        b = t;
      }
      if ((int64_t)atomicCAS(reinterpret_cast<unsigned long long*>(parent + a), (unsigned long long)a,
                             (unsigned long long)b) == a)
        break;
    }
  }
}

__global__ void uf_check(int64_t* parent, const int64_t* order, const int64_t* eptr, int64_t nel,
                         unsigned long long* bad_elem) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nel; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = uf_find(parent, order[eptr[e]]);
    for (int64_t i = eptr[e] + 1; i < eptr[e + 1]; ++i)
      if (uf_find(parent, order[i]) != r) {
        atomicMin(bad_elem, (unsigned long long)e);
        break;
      }
  }
}

__global__ void kept_flags(const uint8_t* internal, int64_t nseg, int64_t* kf) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < nseg; g += (int64_t)gridDim.x * blockDim.x)
    kf[g] = internal[g] ? 0 : 1;
}

// kept facet data (key order): owner orientation, vertex ids, normal, measure
template <int D>
__global__ void kept_facets(const int64_t* seg_r0, const int64_t* seg_s1, const uint8_t* internal,
                            const int64_t* kscan, int64_t nseg, const int64_t* agg, const int32_t* simp,
                            const double* verts, int64_t* own_s, int64_t* nbr_s, int64_t* own_e, int64_t* nbr_e,
                            int32_t* vids, double* normal, double* measure) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < nseg; g += (int64_t)gridDim.x * blockDim.x) {
    if (internal[g]) continue;
    const int64_t k = kscan[g];
    const int64_t r0 = seg_r0[g], s0 = r0 / (D + 1), s1 = seg_s1[g];
    const int64_t e0 = agg[s0], e1 = s1 >= 0 ? agg[s1] : -1;
    const bool swap = s1 >= 0 && e0 > e1;
    own_s[k] = swap ? s1 : s0;
    nbr_s[k] = swap ? s0 : s1;
    own_e[k] = swap ? e1 : e0;
    nbr_e[k] = swap ? e0 : e1;
    int32_t v[D];
    facet_ids<D>(simp, r0, v);
    double c[D][D];
    for (int i = 0; i < D; ++i) {
      vids[k * D + i] = v[i];
      for (int j = 0; j < D; ++j) c[i][j] = verts[(int64_t)v[i] * D + j];
    }
    // numpy's operation order, every product rounded (no FMA contraction):
    // the normals and measures are stored, so they must match bit for bit
    double n[D], meas;
    if (D == 2) {
      const double tx = c[1][0] - c[0][0], ty = c[1][1] - c[0][1];
      const double len = sqrt(__dadd_rn(__dmul_rn(tx, tx), __dmul_rn(ty, ty)));
      n[0] = ty / len;
      n[1] = -tx / len;
      meas = len;
    } else {
      const double ax = c[1][0] - c[0][0], ay = c[1][1] - c[0][1], az = c[1][2] - c[0][2];
      const double bx = c[2][0] - c[0][0], by = c[2][1] - c[0][1], bz = c[2][2] - c[0][2];
      const double cx = __dsub_rn(__dmul_rn(ay, bz), __dmul_rn(az, by));
      const double cy = __dsub_rn(__dmul_rn(az, bx), __dmul_rn(ax, bz));
      const double cz = __dsub_rn(__dmul_rn(ax, by), __dmul_rn(ay, bx));
      const double a2 = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(cx, cx), __dmul_rn(cy, cy)), __dmul_rn(cz, cz)));
      n[0] = cx / a2;
      n[1] = cy / a2;
      n[2] = cz / a2;
      meas = __dmul_rn(0.5, a2);
    }
    // centroid of the owner simplex and of the facet (numpy mean: sequential sum / count)
    const int64_t os = own_s[k];
    double dot = 0.0;
    for (int j = 0; j < D; ++j) {
      double sc = 0.0, fc = 0.0;
      for (int v2 = 0; v2 <= D; ++v2) sc += verts[(int64_t)simp[os * (D + 1) + v2] * D + j];
      for (int i = 0; i < D; ++i) fc += c[i][j];
      sc /= (double)(D + 1);
      fc /= (double)D;
      dot += n[j] * (fc - sc);
    }
    const bool flip = dot < 0.0;
    for (int j = 0; j < D; ++j) normal[k * D + j] = flip ? -n[j] : n[j];
    measure[k] = meas;
  }
}

__global__ void iface_keys(const int64_t* own_e, const int64_t* nbr_e, int64_t nk, int64_t nel, uint64_t* key) {
  // interior facets: owner * nel + neighbour; boundary facets after all interior ones: nel^2 + owner
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nk; k += (int64_t)gridDim.x * blockDim.x)
    key[k] = nbr_e[k] >= 0 ? (uint64_t)own_e[k] * (uint64_t)nel + (uint64_t)nbr_e[k]
                           : (uint64_t)nel * (uint64_t)nel + (uint64_t)own_e[k];
}

// greedy co-hyperplanar split of each multi-facet set; members are permuted
// within the set's range so faces are contiguous; fstart marks face starts
template <int D>
__global__ void greedy_faces(const uint64_t* skey, const int64_t* sidx, int64_t nk, const double* normal,
                             const int32_t* vids, const double* verts, int64_t* members, int64_t* fstart,
                             uint32_t* flags) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nk; i += (int64_t)gridDim.x * blockDim.x) {
    if (!(i == 0 || skey[i] != skey[i - 1])) continue;
    int64_t n = 1;
    while (i + n < nk && skey[i + n] == skey[i]) ++n;
    if (n == 1) {
      members[i] = sidx[i];
      fstart[i] = 1;
      continue;
    }
    if (n > GREEDY_MAX) {
      atomicOr(flags, 4u);
      continue;
    }
    double gn[GREEDY_MAX][D], gp[GREEDY_MAX][D], glo[GREEDY_MAX][D], ghi[GREEDY_MAX][D];
    int gid[GREEDY_MAX];
    int ng = 0;
    for (int64_t m = 0; m < n; ++m) {
      const int64_t idx = sidx[i + m];
      double v[D][D], vlo[D], vhi[D];
      for (int a = 0; a < D; ++a) {
        vlo[a] = PDG_INF;
        vhi[a] = -PDG_INF;
      }
      for (int r = 0; r < D; ++r)
        for (int a = 0; a < D; ++a) {
          v[r][a] = verts[(int64_t)vids[idx * D + r] * D + a];
          vlo[a] = fmin(vlo[a], v[r][a]);
          vhi[a] = fmax(vhi[a], v[r][a]);
        }
      int found = -1;
      for (int q = 0; q < ng && found < 0; ++q) {
        double dn = 0.0;
        for (int a = 0; a < D; ++a) dn = fmax(dn, fabs(normal[idx * D + a] - gn[q][a]));
        if (dn > NORMAL_TOL) continue;
        double lo[D], hi[D], diam2 = 0.0;
        for (int a = 0; a < D; ++a) {
          lo[a] = fmin(glo[q][a], vlo[a]);
          hi[a] = fmax(ghi[q][a], vhi[a]);
          diam2 += (hi[a] - lo[a]) * (hi[a] - lo[a]);
        }
        double diam = sqrt(diam2);
        if (diam == 0.0) diam = 1.0;
        double dmax = 0.0;
        for (int r = 0; r < D; ++r) {
          double s = 0.0;
          for (int a = 0; a < D; ++a) s += (v[r][a] - gp[q][a]) * gn[q][a];
          dmax = fmax(dmax, fabs(s));
        }
        if (dmax <= PLANE_TOL * diam) {
          found = q;
          for (int a = 0; a < D; ++a) {
            glo[q][a] = lo[a];
            ghi[q][a] = hi[a];
          }
        }
      }
      if (found < 0) {
        found = ng++;
        for (int a = 0; a < D; ++a) {
          gn[found][a] = normal[idx * D + a];
          gp[found][a] = v[0][a];
          glo[found][a] = vlo[a];
          ghi[found][a] = vhi[a];
        }
      }
      gid[m] = found;
    }
    int64_t w = i;
    for (int q = 0; q < ng; ++q)
      for (int64_t m = 0; m < n; ++m)
        if (gid[m] == q) members[w++] = sidx[i + m];
    // face starts: first member of every group
    w = i;
    for (int q = 0; q < ng; ++q) {
      int cnt = 0;
      for (int64_t m = 0; m < n; ++m) cnt += gid[m] == q;
      fstart[w] = 1;
      for (int c2 = 1; c2 < cnt; ++c2) fstart[w + c2] = 0;
      w += cnt;
    }
  }
}

// per face (position of its first member in the member order)
template <int D>
__global__ void faces_out(const int64_t* members, const int64_t* fstart, const int64_t* fscan, int64_t nk,
                          const int64_t* own_s, const int64_t* nbr_s, const int64_t* own_e, const int64_t* nbr_e,
                          const int32_t* vids, const double* normal, const double* measure, int32_t* face_owner,
                          int32_t* face_nbr, double* face_normal, double* face_measure, int64_t* face_ptr,
                          int32_t* fvert, int32_t* fos, int32_t* fns, double* fmeas) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nk; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = members[i];
    for (int a = 0; a < D; ++a) fvert[i * D + a] = vids[m * D + a];
    fos[i] = (int32_t)own_s[m];
    fns[i] = (int32_t)nbr_s[m];
    fmeas[i] = measure[m];
    if (!fstart[i]) continue;
    const int64_t f = fscan[i];
    face_ptr[f] = i;
    face_owner[f] = (int32_t)own_e[m];
    face_nbr[f] = (int32_t)nbr_e[m];
    for (int a = 0; a < D; ++a) face_normal[f * D + a] = normal[m * D + a];
    int64_t cnt = 1;
    while (i + cnt < nk && !fstart[i + cnt]) ++cnt;
    face_measure[f] = np_sum(measure, members + i, cnt);  // numpy's sum of the face's facet measures
  }
}

// interfaces: one per distinct interior key; per-interface face counts
__global__ void iface_out(const uint64_t* skey, const int64_t* sidx, const int64_t* fstart, const int64_t* fscan,
                          const int64_t* ihead_scan, int64_t n_int, const int64_t* own_e, const int64_t* nbr_e,
                          int32_t* iface_owner, int32_t* iface_nbr, int64_t* iface_ptr) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_int; i += (int64_t)gridDim.x * blockDim.x) {
    if (!(i == 0 || skey[i] != skey[i - 1])) continue;
    const int64_t q = ihead_scan[i];
    iface_owner[q] = (int32_t)own_e[sidx[i]];
    iface_nbr[q] = (int32_t)nbr_e[sidx[i]];
    iface_ptr[q] = fscan[i];  // first face of the interface
  }
}

__global__ void bface_count(const int32_t* face_owner, int64_t f0, int64_t nf, int64_t* cnt) {
  for (int64_t f = f0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(cnt + face_owner[f]), 1ull);
}

}  // namespace
}  // namespace pdg

using namespace pdg;

extern "C" size_t pdg_agglomerate_workspace_bytes(int32_t dim, int64_t n_simplices, int64_t n_elements) {
  const int64_t nr = n_simplices * (dim + 1);
  size_t cub_b = 0, t = 0;
  cub::DoubleBuffer<uint64_t> kb(nullptr, nullptr);
  cub::DoubleBuffer<int64_t> vb(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, t, kb, vb, std::max<int64_t>(nr, 1), 0, 64);
  cub_b = std::max(cub_b, t);
  cub::DeviceScan::ExclusiveSum(nullptr, t, (int64_t*)nullptr, (int64_t*)nullptr, std::max<int64_t>(nr + 1, 1));
  cub_b = std::max(cub_b, t);
  const size_t per = 256;
  // keys x4, idx x4, heads/scans x4, per-kept arrays (~12 words + dim ints + dim doubles), element arrays
  return (size_t)(nr + 2) * (8 * 16 + 12 * 8 + 4 * dim + 8 * dim) + (size_t)(n_elements + 2) * 8 * 4 +
         (size_t)n_simplices * 8 * 3 + cub_b + 64 * per;
}

extern "C" int pdg_agglomerate(int32_t dim, int64_t n_vertices, int64_t n_simplices, const double* vertices,
                               const int32_t* simplices, const double* simplex_volumes, const int64_t* agg,
                               int64_t n_elements, int32_t check_connected, pdg_agg_out* out, void* workspace,
                               size_t workspace_bytes, pdg_stream stream) {
  PDG_TRY {
    if (!vertices || !simplices || !simplex_volumes || !agg || !out || !workspace)
      return fail(PDG_ERR_INVALID, "null argument");
    if (dim != 2 && dim != 3) return fail(PDG_ERR_UNSUPPORTED, "dim must be 2 or 3");
    if (dim == 3 && n_vertices >= (1ll << 21)) return fail(PDG_ERR_UNSUPPORTED, "3D agglomeration needs < 2^21 vertices");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t ns = n_simplices, nel = n_elements, nr = ns * (dim + 1);
    Bump bp{static_cast<char*>(workspace), workspace_bytes};
    uint32_t* flags = bp.take<uint32_t>(4);
    unsigned long long* bad = bp.take<unsigned long long>(1);
    int64_t* cnt = bp.take<int64_t>(nel + 1);
    int64_t* sidx = bp.take<int64_t>(std::max(nr, ns));
    int64_t* sidx2 = bp.take<int64_t>(std::max(nr, ns));
    uint64_t* k1 = bp.take<uint64_t>(std::max(nr, ns));
    uint64_t* k2 = bp.take<uint64_t>(std::max(nr, ns));
    int64_t* head = bp.take<int64_t>(nr + 1);
    int64_t* hscan = bp.take<int64_t>(nr + 1);
    int64_t* seg_r0 = bp.take<int64_t>(nr);
    int64_t* seg_s1 = bp.take<int64_t>(nr);
    uint8_t* seg_int = bp.take<uint8_t>(nr);
    int64_t* kf = bp.take<int64_t>(nr + 1);
    int64_t* kscan = bp.take<int64_t>(nr + 1);
    int64_t* own_s = bp.take<int64_t>(nr);
    int64_t* nbr_s = bp.take<int64_t>(nr);
    int64_t* own_e = bp.take<int64_t>(nr);
    int64_t* nbr_e = bp.take<int64_t>(nr);
    int32_t* vids = bp.take<int32_t>(nr * dim);
    double* normal = bp.take<double>(nr * dim);
    double* measure = bp.take<double>(nr);
    int64_t* members = bp.take<int64_t>(nr);
    int64_t* fstart = bp.take<int64_t>(nr + 1);
    int64_t* fscan = bp.take<int64_t>(nr + 1);
    int64_t* parent = bp.take<int64_t>(ns);
    int64_t* order = bp.take<int64_t>(ns);
    size_t cub_b = 0;
    {
      size_t t = 0;
      cub::DoubleBuffer<uint64_t> kb(nullptr, nullptr);
      cub::DoubleBuffer<int64_t> vb(nullptr, nullptr);
      cub::DeviceRadixSort::SortPairs(nullptr, t, kb, vb, std::max<int64_t>(std::max(nr, ns), 1), 0, 64);
      cub_b = std::max(cub_b, t);
      cub::DeviceScan::ExclusiveSum(nullptr, t, (int64_t*)nullptr, (int64_t*)nullptr, nr + 1);
      cub_b = std::max(cub_b, t);
    }
    void* cubtmp = bp.take<char>((int64_t)cub_b);
    if (!bp.ok) return fail(PDG_ERR_INVALID, "agglomerate workspace too small (pdg_agglomerate_workspace_bytes)");
    auto G = [](int64_t n) { return grid_for(std::max<int64_t>(n, 1), 256); };
    auto scan = [&](const int64_t* in, int64_t* o, int64_t n) -> cudaError_t {
      size_t t = cub_b;
      return cub::DeviceScan::ExclusiveSum(cubtmp, t, in, o, n, st);
    };
    int nb = 0;
    auto launched = [&]() { ++nb; note_launch(); };
    PDG_CUDA(cudaMemsetAsync(flags, 0, 16, st));
    PDG_CUDA(cudaMemsetAsync(bad, 0xff, 8, st));
    PDG_CUDA(cudaMemsetAsync(cnt, 0, (size_t)(nel + 1) * 8, st));

    // 1. elements
    iota_i64<<<G(ns), 256, 0, st>>>(sidx, ns);
    launched();
    {
      // stable sort of simplex ids by element id (agg as key)
      PDG_CUDA(cudaMemcpyAsync(k1, agg, (size_t)ns * 8, cudaMemcpyDeviceToDevice, st));
      cub::DoubleBuffer<uint64_t> kb(k1, k2);
      cub::DoubleBuffer<int64_t> vb(sidx, sidx2);
      size_t t = cub_b;
      int bits = 1;
      while (bits < 63 && ((uint64_t)nel >> bits)) ++bits;
      PDG_CUDA(cub::DeviceRadixSort::SortPairs(cubtmp, t, kb, vb, ns, 0, bits, st));
      launched();
      PDG_CUDA(cudaMemcpyAsync(order, vb.Current(), (size_t)ns * 8, cudaMemcpyDeviceToDevice, st));
    }
    count_elems<<<G(ns), 256, 0, st>>>(agg, ns, nel, cnt, flags);
    launched();
    check_counts<<<G(nel), 256, 0, st>>>(cnt, nel, flags);
    launched();
    PDG_CUDA(scan(cnt, out->elem_ptr, nel + 1));
    if (dim == 2)
      elem_geometry<2><<<G(nel), 256, 0, st>>>(vertices, simplices, simplex_volumes, order, out->elem_ptr, nel,
                                               out->boxes, out->elem_volumes, out->elem_simplices);
    else
      elem_geometry<3><<<G(nel), 256, 0, st>>>(vertices, simplices, simplex_volumes, order, out->elem_ptr, nel,
                                               out->boxes, out->elem_volumes, out->elem_simplices);
    launched();

    // 2. facet keys + stable sort
    if (dim == 2) facet_keys<2><<<G(nr), 256, 0, st>>>(simplices, nr, k1);
    else facet_keys<3><<<G(nr), 256, 0, st>>>(simplices, nr, k1);
    launched();
    iota_i64<<<G(nr), 256, 0, st>>>(sidx, nr);
    launched();
    uint64_t* ks;
    int64_t* ko;
    {
      cub::DoubleBuffer<uint64_t> kb(k1, k2);
      cub::DoubleBuffer<int64_t> vb(sidx, sidx2);
      size_t t = cub_b;
      int bits = 1;
      const uint64_t maxk = dim == 2 ? (((uint64_t)n_vertices) << 32) : (((uint64_t)n_vertices) << 42);
      while (bits < 64 && (maxk >> bits)) ++bits;
      PDG_CUDA(cub::DeviceRadixSort::SortPairs(cubtmp, t, kb, vb, nr, 0, bits, st));
      launched();
      ks = kb.Current();
      ko = vb.Current();
    }
    head_flags<<<G(nr), 256, 0, st>>>(ks, nr, head);
    launched();
    PDG_CUDA(scan(head, hscan, nr + 1));  // hscan[nr] = number of facets (segments)
    int64_t nseg = 0;
    PDG_CUDA(cudaMemcpyAsync(&nseg, hscan + nr, 8, cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    if (dim == 2)
      segments<2><<<G(nr), 256, 0, st>>>(ks, ko, hscan, nr, agg, seg_r0, seg_s1, seg_int, flags);
    else
      segments<3><<<G(nr), 256, 0, st>>>(ks, ko, hscan, nr, agg, seg_r0, seg_s1, seg_int, flags);
    launched();

    // 3. connectivity
    if (check_connected) {
      iota_i64<<<G(ns), 256, 0, st>>>(parent, ns);
      launched();
      if (dim == 2) uf_union<2><<<G(nseg), 256, 0, st>>>(seg_r0, seg_s1, seg_int, nseg, parent);
      else uf_union<3><<<G(nseg), 256, 0, st>>>(seg_r0, seg_s1, seg_int, nseg, parent);
      launched();
      uf_check<<<G(nel), 256, 0, st>>>(parent, order, out->elem_ptr, nel, bad);
      launched();
    }

    // 4. kept facets
    kept_flags<<<G(nseg), 256, 0, st>>>(seg_int, nseg, kf);
    launched();
    PDG_CUDA(scan(kf, kscan, nseg + 1));
    int64_t nk = 0;
    PDG_CUDA(cudaMemcpyAsync(&nk, kscan + nseg, 8, cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    if (dim == 2)
      kept_facets<2><<<G(nseg), 256, 0, st>>>(seg_r0, seg_s1, seg_int, kscan, nseg, agg, simplices, vertices, own_s,
                                              nbr_s, own_e, nbr_e, vids, normal, measure);
    else
      kept_facets<3><<<G(nseg), 256, 0, st>>>(seg_r0, seg_s1, seg_int, kscan, nseg, agg, simplices, vertices, own_s,
                                              nbr_s, own_e, nbr_e, vids, normal, measure);
    launched();

    // 5. interfaces / boundary sets: stable sort of kept facets by (owner, neighbour) | boundary owner
    iface_keys<<<G(nk), 256, 0, st>>>(own_e, nbr_e, nk, nel, k1);
    launched();
    iota_i64<<<G(nk), 256, 0, st>>>(sidx, nk);
    launched();
    uint64_t* sk;
    int64_t* so;
    {
      cub::DoubleBuffer<uint64_t> kb(k1, k2);
      cub::DoubleBuffer<int64_t> vb(sidx, sidx2);
      size_t t = cub_b;
      const uint64_t maxk = (uint64_t)nel * (uint64_t)nel + (uint64_t)nel;
      int bits = 1;
      while (bits < 64 && (maxk >> bits)) ++bits;
      PDG_CUDA(cub::DeviceRadixSort::SortPairs(cubtmp, t, kb, vb, nk, 0, bits, st));
      launched();
      sk = kb.Current();
      so = vb.Current();
    }
    // number of interior kept facets (their keys are < nel^2)
    if (dim == 2)
      greedy_faces<2><<<G(nk), 256, 0, st>>>(sk, so, nk, normal, vids, vertices, members, fstart, flags);
    else
      greedy_faces<3><<<G(nk), 256, 0, st>>>(sk, so, nk, normal, vids, vertices, members, fstart, flags);
    launched();
    PDG_CUDA(scan(fstart, fscan, nk + 1));
    int64_t nf = 0;
    PDG_CUDA(cudaMemcpyAsync(&nf, fscan + nk, 8, cudaMemcpyDeviceToHost, st));
    // interior facet count = first position whose key >= nel^2 (counted by a head scan over interior keys)
    head_flags<<<G(nk), 256, 0, st>>>(sk, nk, head);
    launched();
    PDG_CUDA(scan(head, hscan, nk + 1));
    uint32_t hflags = 0;
    unsigned long long hbad = 0;
    PDG_CUDA(cudaMemcpyAsync(&hflags, flags, 4, cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaMemcpyAsync(&hbad, bad, 8, cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
    if (hflags & 1u) return fail(PDG_ERR_INVALID, "agglomeration map must be surjective onto 0..max");
    if (hflags & 2u) return fail(PDG_ERR_INVALID, "non-manifold facet shared by more than two simplices");
    if (hflags & 4u) return fail(PDG_ERR_UNSUPPORTED, "more than 64 facets between one element pair");
    if (check_connected && hbad != ~0ull)
      return fail(PDG_ERR_INVALID, "element " + std::to_string(hbad) +
                                       " is not facet-connected; refine the agglomeration map");
    // interior kept facets: binary search not needed -- copy own/nbr to find the split on the host side
    int64_t n_int_facets = 0;
    {
      // count interior facets: nbr_e >= 0 ; reuse kf as flags
      // (kept order already groups interior keys first in the sorted order)
      std::vector<uint64_t> tail(1);
      int64_t lo = 0, hi = nk;
      const uint64_t lim = (uint64_t)nel * (uint64_t)nel;
      while (lo < hi) {  // lower_bound on the sorted keys (device reads, log2(nk) syncs)
        const int64_t mid = (lo + hi) >> 1;
        PDG_CUDA(cudaMemcpyAsync(tail.data(), sk + mid, 8, cudaMemcpyDeviceToHost, st));
        PDG_CUDA(cudaStreamSynchronize(st));
        if (tail[0] < lim) lo = mid + 1;
        else hi = mid;
      }
      n_int_facets = lo;
    }
    int64_t n_iface = 0, n_int_faces = 0;
    if (n_int_facets > 0) {
      PDG_CUDA(cudaMemcpyAsync(&n_iface, hscan + n_int_facets, 8, cudaMemcpyDeviceToHost, st));
      PDG_CUDA(cudaMemcpyAsync(&n_int_faces, fscan + n_int_facets, 8, cudaMemcpyDeviceToHost, st));
      PDG_CUDA(cudaStreamSynchronize(st));
    }

    // 6. faces, facets, interfaces, boundary faces per element
    if (dim == 2)
      faces_out<2><<<G(nk), 256, 0, st>>>(members, fstart, fscan, nk, own_s, nbr_s, own_e, nbr_e, vids, normal,
                                          measure, out->face_owner, out->face_neighbor, out->face_normal,
                                          out->face_measure, out->face_ptr, out->facet_vertices,
                                          out->facet_owner_simplex, out->facet_neighbor_simplex, out->facet_measures);
    else
      faces_out<3><<<G(nk), 256, 0, st>>>(members, fstart, fscan, nk, own_s, nbr_s, own_e, nbr_e, vids, normal,
                                          measure, out->face_owner, out->face_neighbor, out->face_normal,
                                          out->face_measure, out->face_ptr, out->facet_vertices,
                                          out->facet_owner_simplex, out->facet_neighbor_simplex, out->facet_measures);
    launched();
    PDG_CUDA(cudaMemcpyAsync(out->face_ptr + nf, &nk, 8, cudaMemcpyHostToDevice, st));
    iface_out<<<G(n_int_facets), 256, 0, st>>>(sk, so, fstart, fscan, hscan, n_int_facets, own_e, nbr_e,
                                               out->iface_owner, out->iface_neighbor, out->iface_ptr);
    launched();
    PDG_CUDA(cudaMemcpyAsync(out->iface_ptr + n_iface, &n_int_faces, 8, cudaMemcpyHostToDevice, st));
    PDG_CUDA(cudaMemsetAsync(cnt, 0, (size_t)(nel + 1) * 8, st));
    bface_count<<<G(nf - n_int_faces), 256, 0, st>>>(out->face_owner, n_int_faces, nf, cnt);
    launched();
    PDG_CUDA(scan(cnt, out->elem_bface_ptr, nel + 1));
    PDG_CUDA(cudaStreamSynchronize(st));
    PDG_CUDA(cudaGetLastError());
    out->n_faces = nf;
    out->n_facets = nk;
    out->n_interfaces = n_iface;
    out->n_interior_faces = n_int_faces;
    return PDG_OK;
  }
  PDG_CATCH
}
