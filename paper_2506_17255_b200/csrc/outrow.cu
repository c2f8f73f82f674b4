// outrow.cu -- K4o: the decode sketch-GEMV of OUTPUT-ROW units (L31).
//
// Unit (l, o) holds the weights W[o, :] at positions p = j ("each row of the weight
// matrix corresponds to an independent AbsMaxMin sketch instance").  A row's dot product
//     y[o] = sum_j x[j] * w'(o, j),  w'(o, j) = the bonded cell of max |.| over rows i < M_u (Eq. 5)
// then needs only that unit's M_u * N_u cells, so a CTA that owns a block of rows owns their whole
// reduction: ONE kernel per call, no split-K partials, no second (reduce) kernel.
//
//   * CTA = 64 RB threads (2 RB warps) x RB consecutive rows of the launch, RB in {2, 4, 8} the
//     largest that still gives >= 3 CTAs per SM (grid = row blocks, several CTAs per SM).  The 8 units' cells are one contiguous byte range: one TMA bulk copy
//     (cp.async.bulk, mbarrier) into a raw buffer, issued before griddepcontrol.wait (the sketch
//     does not depend on the previous kernel), then converted into the bank-private rho layout
//     cell (i, k) of lane column L at word (i * maxN + k) * 32 + L, lane column L holding unit
//     L mod RB (32 / RB copies): every gather of a warp stays in the lane's own bank.
//   * lane L of warp w: unit r = L mod RB, slice z = L / RB + (32 / RB) w in [0, 64); it visits the
//     positions j = 4 (z + 64 s) + t, t < 4, s = 0, 1, ...: 4 consecutive x values per load (8 B bf16 / 16 B fp32) and the position
//     mixes R_0..R_2(j) mod 2^23 from the plan's table (one 16-B load per j and lane); per weight and sketch row one LOP3 + FFMA.RZ + IMAD + LDS, the
//     Eq. 5 select as an integer max, rotr(rho, 1) = bits of -w' times -x into a per-lane sum.
//   * a row's 64 slice sums go through shared memory and are added in slice order: deterministic,
//     and a row's value does not depend on RB or the launch (an output shard or a grouped call
//     reproduces the rows bit for bit).
#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"

namespace usk {
namespace {

constexpr int kORSlices = 64;    // lanes per row: row o's positions are summed in 64 fixed slices
constexpr int kORMaxRows = 8;    // rows (units) per CTA: RB in {2, 4, 8}, chosen per launch; 64 RB threads
constexpr int kORMaxBatch = 8;

struct ORLayer {
  int64_t unit0;      // global unit id of the layer's first launched row (unit_begin + o_begin)
  int64_t rows;       // launched rows
  int32_t blk_begin;  // first CTA of the layer
  int32_t pad;
  void* y;
};

struct ORArgs {
  ORLayer layer[kORMaxBatch];
  int32_t n_layers;
  int32_t maxN;       // slot row stride (cells): max N over the launch's units
  int64_t in;
  const void* sketch;
  const int32_t* ncols;
  const uint8_t* nrows;
  const int64_t* offsets;
  const uint32_t* ukeys;
  const uint4* R4;    // {R_0, R_1, R_2, 0} mod 2^23 per position p < max(max_out, max_in)
  HashConsts hc;
  const void* x;
  int32_t x_bf16;
  int32_t y_bf16;
};

constexpr int kORCellsByte = 2304;  // [mbarrier][copy shift][8 x 64 slice sums][cells][raw]

__device__ __forceinline__ uint32_t lds_u32(uint32_t saddr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}

template <typename E, int MT, typename XT, int RB, bool PF>
__global__ void __launch_bounds__(kORSlices * RB) k_gemv_outrow(const __grid_constant__ ORArgs A) {
  constexpr int ES = sizeof(E);
  extern __shared__ __align__(128) uint8_t osm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(osm);
  uint32_t* shift = reinterpret_cast<uint32_t*>(osm + 8);
  float* wpart = reinterpret_cast<float*>(osm + 128);  // [RB rows][64 slices]
  uint32_t* cells = reinterpret_cast<uint32_t*>(osm + kORCellsByte);
  const int maxN = A.maxN;
  unsigned char* raw = osm + kORCellsByte + (size_t)32 * MT * maxN * 4;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int li = 0;
  while (li + 1 < A.n_layers && A.layer[li + 1].blk_begin <= (int)blockIdx.x) ++li;
  const ORLayer& Ly = A.layer[li];
  const int64_t rb0 = (int64_t)(blockIdx.x - Ly.blk_begin) * RB;  // first row of the block (launch-relative)
  const int nb = (int)min((int64_t)RB, Ly.rows - rb0);
  const int64_t u0 = Ly.unit0 + rb0;

  // ---- stage the block's cells (contiguous) with one bulk copy, before the PDL wait
  const int r = lane & (RB - 1);
  const bool valid = r < nb;
  const int64_t ur = u0 + (valid ? r : 0);
  const uint32_t N = valid ? (uint32_t)A.ncols[ur] : 1u;
  const int Mu = valid ? (int)A.nrows[ur] : 0;
  const int64_t cell0 = A.offsets[u0];
  const int64_t coff = A.offsets[ur] - cell0;  // the unit's first cell, relative to the block's
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    const uint64_t g0 = (uint64_t)cell0 * ES, g1 = (uint64_t)A.offsets[u0 + nb] * ES;
    const uint64_t a0 = g0 & ~uint64_t(15), a1 = (g1 + 15) & ~uint64_t(15);
    *shift = (uint32_t)(g0 - a0);
    mbar_arrive_expect_tx(bar, (uint32_t)(a1 - a0));
    bulk_g2s(raw, reinterpret_cast<const unsigned char*>(A.sketch) + a0, (uint32_t)(a1 - a0), bar);
  }
  // lane state (overlaps the copy): FFMA key / addend per sketch row, 4N, bank-private base
  uint32_t fk[MT], cb[MT];
  const uint32_t Ku = valid ? A.ukeys[ur] : 0u;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    fk[i] = short_fkey(row_key(Ku, A.hc.kap[i]));
    cb[i] = short_cbits(N, (uint32_t)(i * maxN));
  }
  const float Nf = (float)(4u * N);
  const uint32_t B = smem_u32(cells) + 4u * (uint32_t)lane;
  __syncthreads();  // barrier initialised, shift visible
  mbar_wait(bar, 0);
  {
    // convert: lane column L (this thread's lane) of sketch row i, columns k = warp, warp + 8, ...
    // (rows >= M_u and missing units hold rho = 0, the identity of the max)
    const unsigned char* src = raw + *shift + coff * ES;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      for (int k = warp; k < maxN; k += 2 * RB) {
        uint32_t v = 0u;
        if (i < Mu && k < (int)N) {
          const uint32_t b = ES == 2 ? ((uint32_t)reinterpret_cast<const uint16_t*>(src)[i * N + k] << 16)
                                     : reinterpret_cast<const uint32_t*>(src)[i * N + k];
          v = rotl1(b) ^ 1u;
        }
        cells[(i * maxN + k) * 32 + lane] = v;
      }
    }
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");               // x may come from the previous kernel
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // ---- the row dot products: full groups of 4 positions, then one guarded tail group
  constexpr int Q = 32 / RB;   // lanes of a warp per unit
  const int q = lane / RB;
  const int z = q + Q * warp;  // the lane's slice: position groups g = j / 4 with g mod 64 = z
  const int in = (int)A.in;
  constexpr int kStep = 4 * kORSlices;  // positions per loop trip of a lane
  const int jf = 4 * z;                 // this lane's first position
  const int n_full = jf + 4 <= in ? (in - 4 - jf) / kStep + 1 : 0;
  float acc0 = 0.f, acc1 = 0.f;
  const uint4* Rp = A.R4 + jf;
  const XT* xp = reinterpret_cast<const XT*>(A.x) + jf;
  auto weight = [&](const uint4& R, float xv, float& acc) {
    const uint32_t Ri[3] = {R.x, R.y, R.z};
    uint32_t best = 0u;
#pragma unroll
    for (int i = 0; i < MT; ++i) best = max(best, lds_u32(short_fma_bits(Ri[i], fk[i], Nf, cb[i]) * 128u + B));
    acc = fmaf(-xv, __uint_as_float(rotr1(best)), acc);  // rotr(rho, 1) = bits of -w'
  };
  auto trip = [&](const uint4& R0, const uint4& R1, const uint4& R2, const uint4& R3, const float (&xv)[4]) {
    weight(R0, xv[0], acc0);
    weight(R1, xv[1], acc1);
    weight(R2, xv[2], acc0);
    weight(R3, xv[3], acc1);
  };
  using XV = typename std::conditional<sizeof(XT) == 2, uint2, float4>::type;
  auto unpack = [](const XV& v, float (&xv)[4]) {
    if constexpr (sizeof(XT) == 2) {
      xv[0] = __uint_as_float(v.x << 16);
      xv[1] = __uint_as_float(v.x & 0xFFFF0000u);
      xv[2] = __uint_as_float(v.y << 16);
      xv[3] = __uint_as_float(v.y & 0xFFFF0000u);
    } else {
      xv[0] = v.x;
      xv[1] = v.y;
      xv[2] = v.z;
      xv[3] = v.w;
    }
  };
  if constexpr (PF) {
    // wide layers: the 16 B x in position-mix table does not stay in L1, so its loads see L2
    // latency -- software pipeline: the next trip's mixes and x are loaded before this trip's math
    uint4 Rn0, Rn1, Rn2, Rn3;
    XV xn;
    if (n_full > 0) {
      Rn0 = __ldg(Rp), Rn1 = __ldg(Rp + 1), Rn2 = __ldg(Rp + 2), Rn3 = __ldg(Rp + 3);
      xn = __ldg(reinterpret_cast<const XV*>(xp));
    }
    for (int it = 0; it < n_full; ++it) {
      const uint4 R0 = Rn0, R1 = Rn1, R2 = Rn2, R3 = Rn3;
      const XV xc = xn;
      if (it + 1 < n_full) {
        Rp += kStep;
        xp += kStep;
        Rn0 = __ldg(Rp), Rn1 = __ldg(Rp + 1), Rn2 = __ldg(Rp + 2), Rn3 = __ldg(Rp + 3);
        xn = __ldg(reinterpret_cast<const XV*>(xp));
      }
      float xv[4];
      unpack(xc, xv);
      trip(R0, R1, R2, R3, xv);
    }
  } else {
#pragma unroll 2
    for (int it = 0; it < n_full; ++it, Rp += kStep, xp += kStep) {
      float xv[4];
      unpack(__ldg(reinterpret_cast<const XV*>(xp)), xv);
      trip(__ldg(Rp), __ldg(Rp + 1), __ldg(Rp + 2), __ldg(Rp + 3), xv);
    }
  }
  {
    const int j0 = jf + n_full * kStep;  // the tail group (fewer than 4 positions left), if any
    if (j0 < in) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int j = j0 + t;
        if (j < in) {
          const float xv = sizeof(XT) == 2 ? __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(A.x)[j] << 16)
                                           : reinterpret_cast<const float*>(A.x)[j];
          weight(__ldg(A.R4 + j), xv, (t & 1) ? acc1 : acc0);
        }
      }
    }
  }
  // the row's 64 slice sums in slice order: the same bits whatever RB, batch or output range
  wpart[r * kORSlices + z] = acc0 + acc1;
  __syncthreads();
  if (tid < nb) {
    float y = 0.f;
#pragma unroll 8
    for (int k = 0; k < kORSlices; ++k) y += wpart[tid * kORSlices + k];
    if (A.y_bf16) {
      const uint32_t b = __float_as_uint(y);
      reinterpret_cast<uint16_t*>(Ly.y)[rb0 + tid] = (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
    } else {
      reinterpret_cast<float*>(Ly.y)[rb0 + tid] = y;
    }
  }
}

}  // namespace

// OUTROW units with the fast hash form (M <= 3, USK-X), raw states, no side table, and the block's
// cells + raw copy within shared memory
bool outrow_fast_ok(const usk_plan* pl, const int32_t* layers, int n) {
  if (pl->gran != USK_GRAN_OUTROW || pl->variant != USK_ABSMAXMIN || pl->q || pl->topk || pl->hash != USK_HASH_X ||
      pl->M > 3 || n > kORMaxBatch)
    return false;
  int maxN = 0;
  for (int k = 0; k < n; ++k) maxN = std::max(maxN, pl->layers[layers[k]].max_ncols);
  const size_t smem = kORCellsByte + (size_t)32 * pl->M * maxN * 4 + (size_t)kORMaxRows * pl->M * maxN * pl->cell_bytes() + 64;
  return smem <= 200 * 1024;
}

usk_status launch_gemv_outrow(const usk_plan* pl, const void* sketch, const int32_t* layers, const int64_t* o0,
                              const int64_t* o1, int n, const void* x, int32_t x_dtype, void* const* y, int32_t y_dtype,
                              cudaStream_t st) {
  ORArgs A{};
  int maxN = 1;
  int blocks = 0;
  // rows per CTA: the largest RB that still gives >= 3 CTAs per SM (the CTAs of a small call are
  // few and long otherwise: too few warps to hide the gather latency)
  int64_t total_rows = 0;
  for (int k = 0; k < n; ++k) total_rows += std::max<int64_t>(0, o1[k] - o0[k]);
  // (wide layers keep RB = 8: their position-mix table, 16 B x in, must stay L1-resident beside the
  // CTAs' shared memory, which grows with the CTAs per SM)
  const int64_t in = pl->layers[layers[0]].in;
  int RB = kORMaxRows;
  while (RB > 2 && total_rows / RB < 3 * 148 && in < 4096) RB /= 2;
  for (int k = 0; k < n; ++k) {
    const int64_t rows = o1[k] - o0[k];
    if (rows <= 0) continue;
    const LayerGeom& L = pl->layers[layers[k]];
    ORLayer& Ly = A.layer[A.n_layers++];
    Ly.unit0 = L.unit_begin + o0[k];
    Ly.rows = rows;
    Ly.blk_begin = blocks;
    Ly.y = y[k];
    blocks += (int)((rows + RB - 1) / RB);
    maxN = std::max(maxN, L.max_ncols);
  }
  if (!A.n_layers) return USK_OK;
  A.maxN = maxN;
  A.in = in;
  A.sketch = sketch;
  A.ncols = pl->d_ncols;
  A.nrows = pl->d_nrows;
  A.offsets = pl->d_offsets;
  A.ukeys = pl->d_keys;
  A.R4 = pl->d_R4;
  A.hc = pl->hc;
  A.x = x;
  A.x_bf16 = x_dtype == USK_BF16;
  A.y_bf16 = y_dtype == USK_BF16;
  const int es = pl->cell_bytes();
  const size_t smem = kORCellsByte + (size_t)32 * pl->M * maxN * 4 + (((size_t)RB * pl->M * maxN * es + 47) / 16) * 16;
  (void)es;
  void* kern = nullptr;
  const bool bf16 = pl->dtype == USK_BF16;
  const bool xb = x_dtype == USK_BF16;
  auto pick_rb = [&](auto e, auto xt, auto mt) -> void* {
    using E = decltype(e);
    using XT = decltype(xt);
    constexpr int MT = decltype(mt)::value;
    // software-pipelined loads for wide layers (L2-latency table reads) and for calls with few CTAs
    // (few warps to hide even L1 latency); the many short CTAs of a large call keep more CTAs
    // resident instead (fewer registers)
    if (in >= 4096) return (void*)k_gemv_outrow<E, MT, XT, 8, true>;  // (RB = 8 for wide layers)
    if (blocks < 640)
      return RB == 8 ? (void*)k_gemv_outrow<E, MT, XT, 8, true>
                     : RB == 4 ? (void*)k_gemv_outrow<E, MT, XT, 4, true> : (void*)k_gemv_outrow<E, MT, XT, 2, true>;
    return RB == 8 ? (void*)k_gemv_outrow<E, MT, XT, 8, false>
                   : RB == 4 ? (void*)k_gemv_outrow<E, MT, XT, 4, false> : (void*)k_gemv_outrow<E, MT, XT, 2, false>;
  };
  auto pick = [&](auto e, auto xt) -> void* {
    switch (pl->M) {
      case 1: return pick_rb(e, xt, std::integral_constant<int, 1>{});
      case 2: return pick_rb(e, xt, std::integral_constant<int, 2>{});
      default: return pick_rb(e, xt, std::integral_constant<int, 3>{});
    }
  };
  kern = bf16 ? (xb ? pick(uint16_t{}, uint16_t{}) : pick(uint16_t{}, float{}))
              : (xb ? pick(uint32_t{}, uint16_t{}) : pick(uint32_t{}, float{}));
  USK_CUDA(ensure_smem(kern, 200 * 1024));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(kORSlices * RB);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {&A};
  USK_CUDA(cudaLaunchKernelExC(&cfg, kern, args));
  count_launch();
  return USK_OK;
}

}  // namespace usk
