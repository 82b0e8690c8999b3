// Device memory of a prepared plan (ed_plan_h::allocate): one chunk arena,
// refinement tables, TMA tensor maps and the descriptor tables of every
// grouped launch, resolved to device pointers once.
#include "runtime.h"

namespace edrt {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    CUDA_OK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p) throw ed_error(ED_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

void make_map(CUtensorMap* m, const void* base, bool bf16, int64_t inner, int64_t outer, int64_t outer_stride,
              int64_t batch, int64_t batch_stride, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz) {
  const int es = bf16 ? 2 : 4;
  cuuint64_t dims[3] = {cuuint64_t(inner), cuuint64_t(outer), cuuint64_t(batch)};
  auto fix = [&](int64_t s, int64_t prev_bytes) -> cuuint64_t {
    int64_t b = s * es;
    if (b <= 0 || b % 16) b = ((prev_bytes + 15) / 16) * 16;  // unit extent: stride unused
    return cuuint64_t(b);
  };
  cuuint64_t s1 = fix(outer > 1 ? outer_stride : 0, inner * es);
  cuuint64_t s2 = fix(batch > 1 ? batch_stride : 0, int64_t(s1) * outer);
  cuuint64_t strides[2] = {s1, s2};
  cuuint32_t box[3] = {box_inner, box_outer, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                           const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw ed_error(ED_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
}

}  // namespace edrt

void ed_plan_h::allocate() {
  const int ne = int(X.size());
  CUDA_OK(cudaMalloc(&arena, arena_bytes));
  char* base = static_cast<char*>(arena);
  for (int id = 0; id < ne; ++id) {
    if (buf[id].off_main != SIZE_MAX) buf[id].main = base + buf[id].off_main;
    if (buf[id].off_16 != SIZE_MAX) buf[id].b16 = base + buf[id].off_16;
    if (buf[id].off_lo != SIZE_MAX) buf[id].lo = base + buf[id].off_lo;
  }
  CUDA_OK(cudaMalloc(&d_err, sizeof(int)));
  CUDA_OK(cudaMemset(d_err, 0, sizeof(int)));
  CUDA_OK(cudaMalloc(&d_ptrs, sizeof(void*) * 2 * std::max(1, ne)));

  // refinement dependency tables, one contiguous device array
  host_deps.clear();
  std::map<int, size_t> dep_off;
  for (auto& s : srcs_) {
    if (!dep_off.count(s.ref)) dep_off[s.ref] = host_deps.size();
    DepRect r{};
    r.src = buf[s.src].main;
    for (size_t i = 0; i < s.r0.size(); ++i) {
      r.r0[i] = s.r0[i];
      r.ext[i] = s.ext[i];
    }
    host_deps.push_back(r);
  }
  if (!host_deps.empty()) {
    CUDA_OK(cudaMalloc(&d_deps, sizeof(DepRect) * host_deps.size()));
    CUDA_OK(cudaMemcpy(d_deps, host_deps.data(), sizeof(DepRect) * host_deps.size(), cudaMemcpyHostToDevice));
  }

  auto resolve = [&](int dep) { return local[dep] ? owner[dep] : dep; };
  const bool x3 = opt.precision == ED_PREC_F32X3;
  const bool lo_epi = x3 && x3_lo_by_producer();
  size_t gemm_maps_total = 0, gemm_regions_total = 0, jptrs_total = 0, rect_total = 0;
  size_t attn_maps_total = 0, attn_regions_total = 0, rowseg_total = 0;
  for (auto& op : ops) {
    const int id = int(reinterpret_cast<intptr_t>(op.ptr));
    switch (op.kind) {
      case OpKind::GEMM: {
        const Ex& u = X[id];
        const GemmMap& g = gmap_.at(u.producer);
        GemmLaunch& p = op.gemm;
        const bool b16 = op.bf16;
        p.bf16 = b16;
        p.M = int(g.am.ext);
        p.N = int(g.bn.ext);
        p.K = int(kseg_.count(u.producer) ? kseg_.at(u.producer).kseg : g.ak.ext);
        p.batch = int(g.ab.ext);
        p.a_mn = g.a_mn;
        p.b_mn = g.b_mn;
        p.c_sm = g.cm.ext > 1 ? g.cm.stride : 0;
        p.c_sb = g.cb.ext > 1 ? g.cb.stride : 0;
        p.vec_ok = (p.c_sm % 8 == 0) && (p.c_sb % 8 == 0);
        p.epi_map = -1;
        if (epi_.count(u.producer)) {
          p.epi_map = epi_.at(u.producer).first;
          p.epi_c = float(epi_.at(u.producer).second);
          op.name += "+map";
        }
        p.bn = gemm_pick_bn(p.M, p.N, p.batch, int(op.heads.size()), ctx->num_sms);
        p.x3 = opt.precision == ED_PREC_F32X3;
        p.mc = gemm_use_mc(p.M, p.N, p.bn);
        p.group_m = 8;
        p.chunk = 0;
        if (p.x3) {  // promoted accumulation (gemm_x3_kernel); ED_GEMM_X3_CHUNK=0 keeps one TMEM accumulator
          p.chunk = 4;  // 4 K blocks: 1.5% slower than no promotion on hoc, 2 drains too often (18% slower)
          if (const char* ch = std::getenv("ED_GEMM_X3_CHUNK")) p.chunk = std::max(0, std::atoi(ch));
        }
        if (const char* gm = std::getenv("ED_GEMM_GROUP_M")) p.group_m = std::max(1, std::atoi(gm));  // experiments
        // serpentine K (gemm_sm100.cu) in the bf16 / tf32 kernels; the x3 kernel keeps
        // the forward order: its promoted fp32 sums then round exactly as validated
        // (reversed sums are as accurate on average, but move individual sampled
        // outputs near zero past the reference's own f32 error: FFNN C slice 4.2e-5
        // vs 1.4e-5). ED_GEMM_SERP=0 / 1 forces it off / on.
        p.serp = p.x3 ? 0 : 1;
        if (const char* e = std::getenv("ED_GEMM_SERP")) p.serp = std::atoi(e) != 0;
        const uint32_t BK = uint32_t(gemm_bk(b16)), BM = uint32_t(gemm_bm());
        const uint32_t ATOM = 128u / (b16 ? 2u : 4u);
        op.maps.clear();
        op.regions.clear();
        int total_sib = 0;
        std::vector<const void*> b_src;  // each region's B operand buffer
        for (int head : op.heads) {
          const auto& sibs = region_sibs_.at(head);
          GemmRegion r{};
          r.n_sib = int(sibs.size());
          r.map0 = int(op.maps.size());
          const KSeg* ks = kseg_.count(u.producer) ? &kseg_.at(u.producer) : nullptr;
          const int nseg = ks ? int(ks->segs.at(sibs[0]).size()) : 1;
          r.n_sib = int(sibs.size()) * nseg;
          // MN-major fp32 operands need the 32-byte-atom swizzle (see gemm_sm100.cu)
          const CUtensorMapSwizzle mn_swz = b16 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
          const int es_op = b16 ? 2 : 4;
          // batch-segmented operand: one set of sibling maps per segment, the
          // tiles of batch b use set b / bseg (gemm_sm100.cu)
          const BSeg* bs = bseg_.count(u.producer) ? &bseg_.at(u.producer) : nullptr;
          const int nbs = bs ? int(bs->segs.at(sibs[0]).size()) : 1;
          r.bseg = bs ? int(bs->bseg) : 0;
          r.bseg_b = bs ? bs->role : 0;
          for (int bsi = 0; bsi < nbs; ++bsi)
          for (int pseudo = 0; pseudo < r.n_sib; ++pseudo) {
            const int sidx = sibs[pseudo / nseg];
            const int seg = pseudo % nseg;
            const Ex& j = X[sidx];
            int da = resolve(j.deps[g.a_slot]), db = resolve(j.deps[g.b_slot]);
            Dim am = g.am, ak = g.ak, ab = g.ab, bn = g.bn, bk = g.bk, bb = g.bb;
            int64_t aoff = 0, boff = 0;
            if (bs) {
              const Seg& sg = bs->segs.at(sidx)[size_t(bsi)];
              if (bs->role == 0) {
                da = sg.owner;
                am = sg.mn;
                ak = sg.k;
                ab = sg.b;
                aoff = sg.off;
              } else {
                db = sg.owner;
                bn = sg.mn;
                bk = sg.k;
                bb = sg.b;
                boff = sg.off;
              }
            }
            if (ks) {
              const Seg& sg = ks->segs.at(sidx)[seg];
              if (ks->role == 0) {
                da = sg.owner;
                am = sg.mn;
                ak = sg.k;
                ab = sg.b;
                bk.ext = sg.kext;
                boff = sg.k0 * g.bk.stride;
              } else {
                db = sg.owner;
                bn = sg.mn;
                bk = sg.k;
                bb = sg.b;
                ak.ext = sg.kext;
                aoff = sg.k0 * g.ak.stride;
              }
            }
            // F32X3: A, B, then their lo copies (x - tf32(x)); the kernel feeds
            // hi*hi + hi*lo + lo*hi from one stage into the accumulator
            for (int part = 0; part < (x3 ? 2 : 1); ++part) {
              const char* pa = static_cast<const char*>(b16 ? buf[da].b16 : part ? buf[da].lo : buf[da].main);
              const char* pb = static_cast<const char*>(b16 ? buf[db].b16 : part ? buf[db].lo : buf[db].main);
              if (!pa || !pb) throw ed_error(ED_ERR_PLAN, "GEMM operand buffer missing");
              pa += aoff * es_op;
              pb += boff * es_op;
              if (bsi == 0 && pseudo == 0 && part == 0) b_src.push_back(pb);
              CUtensorMap ma, mb;
              if (!g.a_mn)
                make_map(&ma, pa, b16, ak.ext, am.ext, am.stride, ab.ext, ab.stride, BK, uint32_t(gemm_a_box_rows(p.mc)));
              else make_map(&ma, pa, b16, am.ext, ak.ext, ak.stride, ab.ext, ab.stride, ATOM, BK, mn_swz);
              if (!g.b_mn)
                make_map(&mb, pb, b16, bk.ext, bn.ext, bn.stride, bb.ext, bb.stride, BK, uint32_t(gemm_b_box(p.M, p.bn)));
              else make_map(&mb, pb, b16, bn.ext, bk.ext, bk.stride, bb.ext, bb.stride, ATOM, BK, mn_swz);
              op.maps.push_back(ma);
              op.maps.push_back(mb);
            }
            total_sib += x3 ? 2 : 1;
          }
          r.c32 = static_cast<float*>(buf[head].main);
          r.c16 = p.x3 ? (lo_epi ? buf[head].lo : nullptr) : buf[head].b16;  // x3: the epilogue writes the lo shadow
          // output tensor maps for the TMA-store epilogue (16-byte strides only)
          auto out_map = [&](void* base, bool o16) {
            const int oes = o16 ? 2 : 4;
            bool ok = base && (g.cm.ext == 1 || (g.cm.stride * oes) % 16 == 0) &&
                      (g.cb.ext == 1 || (g.cb.stride * oes) % 16 == 0);
            if (!ok) return -1;
            CUtensorMap mc;
            make_map(&mc, base, o16, g.bn.ext, g.am.ext, g.cm.stride, g.ab.ext, g.cb.stride, o16 ? 64u : 32u,
                     uint32_t(kStoreRows));
            op.maps.push_back(mc);
            return int(op.maps.size()) - 1;
          };
          r.cmap32 = out_map(r.c32, false);
          r.cmap16 = out_map(r.c16, !p.x3);
          op.regions.push_back(r);
        }
        p.n_regions = int(op.regions.size());
        // regions that all read one B operand per batch: order tiles batch-major
        p.region_inner = p.n_regions > 1 && p.batch > 1 &&
                         std::all_of(b_src.begin(), b_src.end(), [&](const void* q) { return q == b_src[0]; });
        const double ab = double(g.am.ext) * g.ak.ext * g.ab.ext + double(g.bn.ext) * g.bk.ext * g.bb.ext;
        const double cbytes = double(g.am.ext) * g.bn.ext * g.ab.ext *
                              ((op.regions[0].c32 ? 4 : 0) + (op.regions[0].c16 ? (p.x3 ? 4 : 2) : 0));
        op.bytes = ab * (b16 ? 2 : 4) * total_sib + cbytes * p.n_regions;
        gemm_maps_total += op.maps.size();
        gemm_regions_total += op.regions.size();
        break;
      }
      case OpKind::GENERIC: {
        const Ex& u = X[id];
        const Vtx& w = V[u.producer];
        GenericParams& p = op.gen;
        std::memset(&p, 0, sizeof(p));
        shape lxy = local_xy(u.producer);
        std::map<int, int64_t> ext;
        for (size_t i = 0; i < w.lxy.size(); ++i) ext.emplace(w.lxy[i], lxy[i]);
        auto strides_of = [&](const labels& ls) {
          std::map<int, int64_t> st;
          int64_t s = 1;
          for (int i = int(ls.size()) - 1; i >= 0; --i) {
            st[ls[i]] = s;
            s *= ext.at(ls[i]);
          }
          return st;
        };
        auto xs = strides_of(w.lx);
        auto ys = w.arity == 2 ? strides_of(w.ly) : std::map<int, int64_t>{};
        auto get = [](const std::map<int, int64_t>& m, int l) {
          auto it = m.find(l);
          return it == m.end() ? int64_t(0) : it->second;
        };
        p.nz = int(w.lz.size());
        for (int i = 0; i < p.nz; ++i) {
          p.zext[i] = ext.at(w.lz[i]);
          p.xs_z[i] = get(xs, w.lz[i]);
          p.ys_z[i] = get(ys, w.lz[i]);
        }
        p.na = 0;
        for (auto l : w.dls)
          if (std::find(w.lz.begin(), w.lz.end(), l) == w.lz.end()) {
            p.aext[p.na] = ext.at(l);
            p.xs_a[p.na] = get(xs, l);
            p.ys_a[p.na] = get(ys, l);
            ++p.na;
          }
        p.join = w.join;
        p.map = w.map;
        p.agg = w.agg;
        p.c = w.c;
        p.x = buf[resolve(u.deps[0])].main;
        p.y = w.arity == 2 ? buf[resolve(u.deps[1])].main : nullptr;
        p.out = buf[id].main;
        p.out16 = buf[id].b16;
        p.n_out = u.sz;
        p.err = d_err;
        int64_t xin = prod(pick(lxy, positions(w.lx, w.lxy)));
        int64_t yin = w.arity == 2 ? prod(pick(lxy, positions(w.ly, w.lxy))) : 0;
        op.bytes = double(xin + yin + u.sz) * es;
        break;
      }
      case OpKind::REFINE: {
        const Ex& u = X[id];
        const Vtx& w = V[u.producer];
        RefineParams& p = op.ref;
        std::memset(&p, 0, sizeof(p));
        const shape& bound = w.bound;
        shape dc = region_partition(id);
        p.rank = int(bound.size());
        p.agg = w.arity == 0 ? -1 : w.agg;
        for (int i = 0; i < p.rank; ++i) {
          p.cext[i] = u.cb[i];
          p.c0[i] = u.key[i] * (bound[i] / dc[i]);
        }
        p.n_out = u.sz;
        size_t first = dep_off.at(id), n = 0;
        for (auto& s : srcs_) n += s.ref == id;
        p.deps = d_deps + first;
        p.n_deps = int(n);
        p.out = buf[id].main;
        p.out16 = x3 ? (lo_epi ? buf[id].lo : nullptr) : buf[id].b16;  // x3: the lo shadow a later fp32x3 contraction reads
        p.lo = x3;
        op.bytes = double(u.sz) * (es + (p.out16 ? (x3 ? 4 : 2) : 0));
        double rd = 0;
        for (auto& s : srcs_)
          if (s.ref == id) {
            double vol = 1;
            for (int i = 0; i < p.rank; ++i)
              vol *= double(std::max<int64_t>(0, std::min(s.r0[i] + s.ext[i], p.c0[i] + p.cext[i]) -
                                                     std::max(s.r0[i], p.c0[i])));
            rd += vol;
          }
        op.bytes += rd * es;
        // fast path: group sources by region (siblings fold in dep order)
        op.groups.clear();
        op.max_rows = 0;
        bool fast = true;
        std::vector<std::pair<shape, std::vector<const void*>>> regions;
        std::vector<const SrcRec*> firsts;
        for (auto& sr : srcs_) {
          if (sr.ref != id) continue;
          auto it = std::find_if(regions.begin(), regions.end(), [&](auto& q) { return q.first == sr.r0; });
          if (it == regions.end()) {
            regions.push_back({sr.r0, {}});
            firsts.push_back(&sr);
            it = regions.end() - 1;
          }
          it->second.push_back(buf[sr.src].main);
        }
        const int V = int(16 / es);
        bool vec = true;
        for (size_t gi = 0; gi < regions.size() && fast; ++gi) {
          const SrcRec& f = *firsts[gi];
          if (int(regions[gi].second.size()) > kRectSrc) {
            fast = false;
            break;
          }
          RectGroup rg{};
          rg.n_src = int(regions[gi].second.size());
          for (int k = 0; k < rg.n_src; ++k) rg.src[k] = regions[gi].second[k];
          int64_t ss = 1, ds = 1;
          for (int i = p.rank - 1; i >= 0; --i) {
            rg.sstr[i] = ss;
            rg.dstr[i] = ds;
            ss *= f.ext[i];
            ds *= p.cext[i];
          }
          rg.src_off = rg.dst_off = 0;
          rg.rows = 1;
          for (int i = 0; i < p.rank; ++i) {
            int64_t lo = std::max(f.r0[i], p.c0[i]);
            int64_t hi = std::min(f.r0[i] + f.ext[i], p.c0[i] + p.cext[i]);
            rg.ext[i] = hi - lo;
            rg.src_off += (lo - f.r0[i]) * rg.sstr[i];
            rg.dst_off += (lo - p.c0[i]) * rg.dstr[i];
            if (i < p.rank - 1) rg.rows *= rg.ext[i];
          }
          if (std::any_of(rg.ext, rg.ext + p.rank, [](int64_t e) { return e <= 0; })) continue;
          vec = vec && rg.ext[p.rank - 1] % V == 0 && rg.src_off % V == 0 && rg.dst_off % V == 0 &&
                (p.rank == 1 || (f.ext[p.rank - 1] % V == 0 && p.cext[p.rank - 1] % V == 0));
          op.max_rows = std::max(op.max_rows, rg.rows);
          op.groups.push_back(rg);
        }
        if (fast && !op.groups.empty() && p.rank >= 1) {
          op.rect.rank = p.rank;
          op.rect.agg = p.agg;
          op.rect.vec = vec;
          const int64_t inner = op.groups[0].ext[p.rank - 1];
          // ~32 KiB of output per block
          op.rect.rows_per_block = int(std::max<int64_t>(1, (32768 / int64_t(es)) / std::max<int64_t>(1, inner)));
          op.rect.out = p.out;
          op.rect.out16 = p.out16;
          op.rect.lo = p.lo;
          rect_total += op.groups.size();
        } else {
          op.groups.clear();
        }
        break;
      }
      case OpKind::SPLIT:
        op.gen.x = buf[id].main;
        op.gen.out = buf[id].lo;
        op.gen.n_out = X[id].sz;
        break;
      case OpKind::CORRUPT:
        op.dt = buf[id].main ? store : DT::BF16;
        op.ptr = buf[id].main ? buf[id].main : buf[id].b16;
        break;
      case OpKind::SEND:
        op.ptr = buf[resolve(id)].main;
        break;
      case OpKind::RECV:
        op.ptr = buf[id].main;
        break;
      case OpKind::CONVERT:
        op.gen.x = buf[id].main;
        op.gen.out16 = buf[id].b16;
        op.gen.n_out = X[id].sz;
        break;
      case OpKind::FLASH: {
        const Flash& f = flash_.at(X[id].producer);
        const GemmMap& gs = gmap_.at(f.t1);
        const GemmMap& go = gmap_.at(f.o);
        AttnLaunch& a = op.attn;
        a.H = int(gs.ab.ext);
        a.S = int(gs.am.ext);
        a.T = int(gs.bn.ext);
        a.D = int(gs.ak.ext);
        a.scale = f.scale;
        op.maps.clear();
        op.aregions.clear();
        a.x3 = x3;
        for (auto& r : f.regions) {
          AttnRegion ar{};
          // bf16: the operands' bf16 shadows; fp32x3: fp32 values (+ lo shadows)
          auto opnd = [&](int id2) { return x3 ? buf[id2].main : buf[id2].b16; };
          const void* q = opnd(resolve(r[0]));
          const void* k = f.ktiles[size_t(&r - f.regions.data())].tiled ? nullptr : opnd(resolve(r[1]));
          const void* v = f.vtiles[size_t(&r - f.regions.data())].tiled ? nullptr : opnd(resolve(r[2]));
          if (!q || (x3 && !buf[resolve(r[0])].lo)) throw ed_error(ED_ERR_PLAN, "attention operand buffer missing");
          CUtensorMap m;
          if (x3) make_map(&m, buf[resolve(r[0])].lo, false, gs.ak.ext, gs.am.ext, gs.am.stride, gs.ab.ext, gs.ab.stride, 32, 128);
          else make_map(&m, q, true, gs.ak.ext, gs.am.ext, gs.am.stride, gs.ab.ext, gs.ab.stride, 64, 128);
          ar.q = int(op.maps.size());
          op.maps.push_back(m);
          if (x3) {  // maps[q + 1]: Q itself (read by the MMA as Q_hi)
            make_map(&m, q, false, gs.ak.ext, gs.am.ext, gs.am.stride, gs.ab.ext, gs.ab.stride, 32, 128);
            op.maps.push_back(m);
            ar.q_tm = static_cast<const float*>(q);
            ar.q_rs = gs.am.stride;
            ar.q_hs = gs.ab.ext > 1 ? gs.ab.stride : 0;
          }
          const size_t ri = size_t(&r - f.regions.data());
          // K: {d, keys, h}; V: {d, keys, h} — from the pasted chunk, or from each
          // source region of the grid with that region's own strides
          // x3 boxes: K {32, 64} K-major; V {32, 32} MN-major (32-byte-atom swizzle);
          // the lo twins follow the hi maps (AttnSrc::lo)
          auto kv_map = [&](const void* base, int64_t dext, int64_t kext, int64_t kstr, int64_t hext, int64_t hstr,
                            bool is_v) {
            if (!x3) make_map(&m, base, true, dext, kext, kstr, hext, hstr, 64, 128);
            else if (!is_v) make_map(&m, base, false, dext, kext, kstr, hext, hstr, 32, uint32_t(128 / attn_x3_cta(a.S)));
            else make_map(&m, base, false, dext, kext, kstr, hext, hstr, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
            op.maps.push_back(m);
          };
          auto kv_maps = [&](const KVTiles& t, int chunk_id, const Dim& dk, const Dim& keys, const Dim& hb,
                             const labels& lop, int keyl, int hl, bool is_v, AttnSrc& out) {
            out.base = int(op.maps.size());
            out.lo = 0;
            if (!t.tiled) {
              kv_map(opnd(chunk_id), dk.ext, keys.ext, keys.stride, hb.ext, hb.stride, is_v);
              if (x3) {
                if (!buf[chunk_id].lo) throw ed_error(ED_ERR_PLAN, "attention operand lo shadow missing");
                kv_map(buf[chunk_id].lo, dk.ext, keys.ext, keys.stride, hb.ext, hb.stride, is_v);
                out.lo = 1;
              }
              out.nd = 1;
              out.keys = int(keys.ext);
              out.dw = int(dk.ext);
              out.hoff = 0;
              return;
            }
            const int kd = int(std::find(lop.begin(), lop.end(), keyl) - lop.begin());
            const int hd = int(std::find(lop.begin(), lop.end(), hl) - lop.begin());
            shape st(3, 1);
            for (int i = 1; i >= 0; --i) st[i] = st[i + 1] * t.ext[i + 1];
            for (int part = 0; part < (x3 ? 2 : 1); ++part)
              for (int o2 : t.owners) {
                const void* b = part ? buf[o2].lo : opnd(o2);
                if (!b) throw ed_error(ED_ERR_PLAN, "attention source buffer missing");
                kv_map(b, t.ext[2], t.ext[kd], st[kd], t.ext[hd], st[hd], is_v);
              }
            out.lo = x3 ? int(t.owners.size()) : 0;
            out.nd = t.nd;
            out.keys = int(t.keys);
            out.dw = int(t.dw);
            out.hoff = int(t.hoff);
          };
          const labels& lk = gs.b_slot == 0 ? V[f.t1].lx : V[f.t1].ly;
          const labels& lv = go.b_slot == 0 ? V[f.o].lx : V[f.o].ly;
          (void)k;
          (void)v;
          kv_maps(f.ktiles[ri], resolve(r[1]), gs.bk, gs.bn, gs.bb, lk, gs.Nc.empty() ? -1 : gs.Nc[0],
                  gs.Bc.empty() ? -1 : gs.Bc[0], false, ar.k);
          kv_maps(f.vtiles[ri], resolve(r[2]), go.bn, go.bk, go.bb, lv, go.Kc.empty() ? -1 : go.Kc[0],
                  go.Bc.empty() ? -1 : go.Bc[0], true, ar.v);
          auto out_map = [&](void* base, bool o16) {
            const int oes = o16 ? 2 : 4;
            bool ok = base && (go.cm.ext == 1 || (go.cm.stride * oes) % 16 == 0) &&
                      (go.cb.ext == 1 || (go.cb.stride * oes) % 16 == 0);
            if (!ok) return -1;
            CUtensorMap mc;
            make_map(&mc, base, o16, go.bn.ext, go.am.ext, go.cm.stride, go.ab.ext, go.cb.stride, o16 ? 64u : 32u,
                     uint32_t(kStoreRows));
            op.maps.push_back(mc);
            return int(op.maps.size()) - 1;
          };
          if (x3) {
            // row-per-thread float4 stores: d contiguous, 16-byte row / head strides
            ar.o32 = ar.o16 = -1;
            ar.o = static_cast<float*>(buf[r[3]].main);
            ar.o_lo = static_cast<float*>(buf[r[3]].lo);
            ar.o_rs = go.cm.stride;
            ar.o_hs = go.cb.ext > 1 ? go.cb.stride : 0;
            if (!ar.o || ar.o_rs % 4 || ar.o_hs % 4 || ar.q_rs % 4 || ar.q_hs % 4)
              throw ed_error(ED_ERR_UNSUPPORTED, "attention output not 16-byte aligned");
          } else {
            ar.o32 = out_map(buf[r[3]].main, false);
            ar.o16 = out_map(buf[r[3]].b16, true);
            if ((buf[r[3]].main && ar.o32 < 0) || (buf[r[3]].b16 && ar.o16 < 0))
              throw ed_error(ED_ERR_UNSUPPORTED, "attention output not 16-byte aligned");
          }
          op.aregions.push_back(ar);
        }
        a.n_regions = int(op.aregions.size());
        op.bytes = 0;
        for (auto& r : f.regions)
          op.bytes += double(X[r[0]].sz + X[r[1]].sz + X[r[2]].sz) * (x3 ? 8 : 2) +
                      double(X[r[3]].sz) * (buf[r[3]].main ? 4 : 0) + double(X[r[3]].sz) * (buf[r[3]].b16 ? 2 : 0) +
                      double(X[r[3]].sz) * (x3 && buf[r[3]].lo ? 4 : 0);
        attn_maps_total += op.maps.size();
        attn_regions_total += op.aregions.size();
        break;
      }
      case OpKind::SOFTMAX: {
        const Softmax& sm = softmax_.at(X[id].producer);
        op.jptrs.clear();
        for (size_t k = 0; k < sm.pairs.size(); ++k) {
          const int yj = sm.pairs[k].first, xr = sm.pairs[k].second;
          JoinPtrs jp{};
          jp.x = buf[resolve(xr)].main;
          jp.y = sm.m_refs.empty() ? nullptr : buf[resolve(sm.m_refs[k])].main;
          jp.out = buf[yj].main;
          jp.out16 = x3 ? (lo_epi ? buf[yj].lo : nullptr) : buf[yj].b16;  // x3: the lo shadow a later fp32x3 contraction reads
          op.jptrs.push_back(jp);
          op.bytes += double(X[yj].sz) * (es + (jp.out ? es : 0) + (jp.out16 ? (x3 ? 4 : 2) : 0));
        }
        op.sm.lo = x3;
        op.sm.rows = X[sm.pairs[0].first].sz / sm.len;
        op.sm.len = int(sm.len);
        op.rowsegs.clear();
        if (!sm.xsegs.empty()) {
          op.sm.n_seg = int(sm.xsegs[0].size());
          op.sm.seg_w = sm.seg_w;
          for (auto& v : sm.xsegs)
            for (auto& xs : v) op.rowsegs.push_back(RowSeg{static_cast<const float*>(buf[xs.owner].main), xs.row0, xs.stride});
          rowseg_total += op.rowsegs.size();
        }
        jptrs_total += op.jptrs.size();
        break;
      }
      case OpKind::EWISE:
      case OpKind::ROWREDUCE: {
        const Ex& u = X[id];
        const Vtx& w = V[u.producer];
        const MemMap& mm = memmap_.at(u.producer);
        op.jptrs.clear();
        double in_el = 0;
        shape lxy = local_xy(u.producer);
        int64_t xin = prod(pick(lxy, positions(w.lx, w.lxy)));
        int64_t yin = w.arity == 2 ? prod(pick(lxy, positions(w.ly, w.lxy))) : 0;
        for (int h : op.heads) {
          const Ex& j = X[h];
          JoinPtrs jp{};
          jp.x = buf[resolve(j.deps[0])].main;
          jp.y = w.arity == 2 ? buf[resolve(j.deps[1])].main : nullptr;
          jp.out = buf[h].main;
          jp.out16 = buf[h].b16;
          op.jptrs.push_back(jp);
          in_el += double(xin + yin);
          op.bytes += double(j.sz) * ((jp.out ? es : 0) + (jp.out16 ? 2 : 0));
        }
        op.bytes += in_el * es;
        if (mm.kind == OpKind::EWISE) {
          EwiseParams& p = op.ew;
          p.n = u.sz;
          p.binary = w.arity == 2;
          p.y_mode = mm.y_mode;
          p.inner = mm.inner;
          p.join = w.join;
          p.map = w.map;
          p.c = w.c;
          p.err = d_err;
        } else {
          RowReduceParams& p = op.rr;
          p.rows = mm.rows;
          p.len = mm.len;
          p.map = w.map;
          p.agg = w.agg;
          p.c = w.c;
        }
        jptrs_total += op.jptrs.size();
        break;
      }
    }
  }
  if (rowseg_total) {
    CUDA_OK(cudaMalloc(&d_rowsegs, sizeof(RowSeg) * rowseg_total));
    size_t o = 0;
    for (auto& op : ops) {
      if (op.rowsegs.empty()) continue;
      RowSeg* d = static_cast<RowSeg*>(d_rowsegs) + o;
      CUDA_OK(cudaMemcpy(d, op.rowsegs.data(), sizeof(RowSeg) * op.rowsegs.size(), cudaMemcpyHostToDevice));
      op.sm.segs = d;
      o += op.rowsegs.size();
    }
  }
  if (attn_maps_total) {
    CUDA_OK(cudaMalloc(&d_attn, sizeof(CUtensorMap) * attn_maps_total + sizeof(AttnRegion) * attn_regions_total));
    size_t mo = 0, ro = 0;
    CUtensorMap* maps = static_cast<CUtensorMap*>(d_attn);
    AttnRegion* regs = reinterpret_cast<AttnRegion*>(maps + attn_maps_total);
    for (auto& op : ops) {
      if (op.kind != OpKind::FLASH) continue;
      CUDA_OK(cudaMemcpy(maps + mo, op.maps.data(), sizeof(CUtensorMap) * op.maps.size(), cudaMemcpyHostToDevice));
      CUDA_OK(cudaMemcpy(regs + ro, op.aregions.data(), sizeof(AttnRegion) * op.aregions.size(),
                         cudaMemcpyHostToDevice));
      op.attn.maps = maps + mo;
      op.attn.regions = regs + ro;
      mo += op.maps.size();
      ro += op.aregions.size();
    }
  }
  if (rect_total) {
    CUDA_OK(cudaMalloc(&d_rects, sizeof(RectGroup) * rect_total));
    size_t o = 0;
    for (auto& op : ops) {
      if (op.groups.empty()) continue;
      RectGroup* d = static_cast<RectGroup*>(d_rects) + o;
      CUDA_OK(cudaMemcpy(d, op.groups.data(), sizeof(RectGroup) * op.groups.size(), cudaMemcpyHostToDevice));
      op.rect.groups = d;
      o += op.groups.size();
    }
  }
  if (jptrs_total) {
    CUDA_OK(cudaMalloc(&d_joinptrs, sizeof(JoinPtrs) * jptrs_total));
    size_t o = 0;
    for (auto& op : ops) {
      if (op.jptrs.empty()) continue;
      JoinPtrs* d = static_cast<JoinPtrs*>(d_joinptrs) + o;
      CUDA_OK(cudaMemcpy(d, op.jptrs.data(), sizeof(JoinPtrs) * op.jptrs.size(), cudaMemcpyHostToDevice));
      op.ew.joins = d;
      op.rr.joins = d;
      op.sm.joins = d;
      o += op.jptrs.size();
    }
  }
  // tensor maps and region tables of every GEMM launch, in device memory
  if (gemm_maps_total) {
    CUDA_OK(cudaMalloc(&d_maps, sizeof(CUtensorMap) * gemm_maps_total));
    CUDA_OK(cudaMalloc(&d_regions, sizeof(GemmRegion) * gemm_regions_total));
    size_t mo = 0, ro = 0;
    for (auto& op : ops) {
      if (op.kind != OpKind::GEMM) continue;
      CUtensorMap* dm = static_cast<CUtensorMap*>(d_maps) + mo;
      GemmRegion* dr = static_cast<GemmRegion*>(d_regions) + ro;
      CUDA_OK(cudaMemcpy(dm, op.maps.data(), sizeof(CUtensorMap) * op.maps.size(), cudaMemcpyHostToDevice));
      CUDA_OK(cudaMemcpy(dr, op.regions.data(), sizeof(GemmRegion) * op.regions.size(), cudaMemcpyHostToDevice));
      op.gemm.maps = dm;
      op.gemm.regions = dr;
      mo += op.maps.size();
      ro += op.regions.size();
    }
    // loose producer lockstep (GemmLaunch::sync) of the fp32x3 kernel: epochs of 16
    // K blocks, lag 2 (hoc 3%, FFNN 7% faster); ED_GEMM_SYNC="g,lag" overrides,
    // "0,0" turns it off. Launches that run as parallel graph branches skip it.
    int sg = 16, slag = 2;
    if (const char* e = std::getenv("ED_GEMM_SYNC")) std::sscanf(e, "%d,%d", &sg, &slag);
    if (sg > 0 && slag > 0) {
      size_t words = 0;
      for (auto& op : ops) {
        // fp32x3 only: the bf16 kernel's 64-deep K blocks go by too fast to
        // wait on a global counter (hoc bf16 4.9 -> 6.3 ms with it)
        if (op.kind != OpKind::GEMM || !op.gemm.x3 || op.gemm.chunk <= 0) continue;
        int max_sib = 1;
        for (auto& r : op.regions) max_sib = std::max(max_sib, r.n_sib);
        op.gemm.sync_g = sg;
        op.gemm.sync_lag = slag;
        op.gemm.sync_epochs = gemm_sync_epochs(op.gemm, ctx->num_sms, max_sib);
        words += size_t(op.gemm.sync_epochs) + 1;
      }
      if (words) {
        CUDA_OK(cudaMalloc(&d_sync, words * sizeof(unsigned int)));
        CUDA_OK(cudaMemset(d_sync, 0, words * sizeof(unsigned int)));
        size_t o = 0;
        for (auto& op : ops) {
          if (op.kind != OpKind::GEMM || op.gemm.sync_g <= 0) continue;
          op.gemm.sync = static_cast<unsigned int*>(d_sync) + o;
          o += size_t(op.gemm.sync_epochs) + 1;
        }
      }
    }
  }
  // x3 tail split-K: per launch, the first halves' running sums and one counter per split tile
  {
    size_t floats = 0, counters = 0;
    for (auto& op : ops) {
      if (op.kind != OpKind::GEMM) continue;
      op.gemm.split = gemm_x3_split(op.gemm, ctx->num_sms);
      const size_t tile = size_t(gemm_bm()) * (gemm_paired(op.gemm.M) ? 2 : 1) * size_t(op.gemm.bn);
      floats += size_t(op.gemm.split) * tile;
      counters += size_t(op.gemm.split);
    }
    if (counters) {
      CUDA_OK(cudaMalloc(&d_split, floats * sizeof(float) + counters * sizeof(unsigned int)));
      CUDA_OK(cudaMemset(static_cast<char*>(d_split) + floats * sizeof(float), 0, counters * sizeof(unsigned int)));
      size_t fo = 0, co = 0;
      for (auto& op : ops) {
        if (op.kind != OpKind::GEMM || !op.gemm.split) continue;
        const size_t tile = size_t(gemm_bm()) * (gemm_paired(op.gemm.M) ? 2 : 1) * size_t(op.gemm.bn);
        op.gemm.split_ws = static_cast<float*>(d_split) + fo;
        op.gemm.split_cnt = reinterpret_cast<unsigned int*>(static_cast<float*>(d_split) + floats) + co;
        fo += size_t(op.gemm.split) * tile;
        co += size_t(op.gemm.split);
      }
    }
  }
  if (peer) {
    CUDA_OK(cudaMalloc(&d_epoch, sizeof(int)));
    CUDA_OK(cudaMemset(d_epoch, 0, sizeof(int)));
    CUDA_OK(cudaMalloc(&d_pflags, sizeof(int) * (X.size() + 2)));
    CUDA_OK(cudaMemset(d_pflags, 0, sizeof(int) * (X.size() + 2)));
    CUDA_OK(cudaMalloc(&d_perr, sizeof(int)));
    CUDA_OK(cudaMemset(d_perr, 0, sizeof(int)));
  }
}

// Direct receives (peer transport, prefetched): a received chunk that only
// refinement folds read is not copied — the folds' source pointers (the
// DepRect table and the rect groups) are rebound to the producer's chunk, and
// the receive becomes the wait for its ready flag. Called once the peers'
// arenas are known (ed_prepare over several ranks, ed_peer_import).
void ed_plan_h::bind_direct() {
  if (!peer || !peer_ready || !prefetch_ok || !peer_prefetch()) return;
  if (const char* e = std::getenv("ED_PEER_DIRECT"))
    if (e[0] == '0') return;  // A/B: copy every received chunk
  std::map<const void*, const void*> remap;
  for (Op& op : ops) {
    if (op.kind != OpKind::RECV || !direct[size_t(op.exec)]) continue;
    const int64_t off = peer_off[size_t(op.peer)][size_t(op.exec)];
    if (off < 0) continue;
    remap[buf[size_t(op.exec)].main] = peer_arena[size_t(op.peer)] + off;
    op.direct = true;
  }
  if (remap.empty()) return;
  direct_bound = true;
  bool deps_changed = false;
  for (DepRect& r : host_deps) {
    auto it = remap.find(r.src);
    if (it != remap.end()) {
      r.src = it->second;
      deps_changed = true;
    }
  }
  if (deps_changed)
    CUDA_OK(cudaMemcpy(d_deps, host_deps.data(), sizeof(DepRect) * host_deps.size(), cudaMemcpyHostToDevice));
  for (Op& op : ops) {
    if (op.kind != OpKind::REFINE || op.groups.empty()) continue;
    bool changed = false;
    for (RectGroup& g : op.groups)
      for (int k = 0; k < g.n_src; ++k) {
        auto it = remap.find(g.src[k]);
        if (it != remap.end()) {
          g.src[k] = it->second;
          changed = true;
        }
      }
    if (changed)
      CUDA_OK(cudaMemcpy(const_cast<RectGroup*>(op.rect.groups), op.groups.data(), sizeof(RectGroup) * op.groups.size(),
                         cudaMemcpyHostToDevice));
  }
}
