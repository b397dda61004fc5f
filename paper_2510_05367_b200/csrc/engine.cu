// GPU execution engine; see engine.hpp.
#include "engine.hpp"

#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include <chrono>
#include <thread>

namespace lc {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw LcError(kCudaError, std::string("CUDA error ") + cudaGetErrorString(e) + " at " + what);
}

// ---------------------------------------------------------------- ledger
double Ledger::now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
void Ledger::record(int kind, int tier, int64_t bytes, uint64_t id) {
    events.push_back(
        {kind, bytes, tier, stage, id, static_cast<uint64_t>(events.size()), virt >= 0 ? virt : now() - t0});
    ++events_per_stage[stage];
}
void Ledger::enter(int s) {
    stage = s;
    for (int t = 0; t < 2; ++t) peak[s][t] = std::max(peak[s][t], occ[t]);
    record(4, 0, 0, 0);
}
void Ledger::check_budget(int64_t extra) const {
    if (budget_fast > 0 && occ[0] + extra > budget_fast) {
        static const char* names[4] = {"setup", "encode", "denoise", "decode"};
        throw LcError(kBudgetError,
                      std::string("fast-tier budget exceeded in stage ") + names[stage] + ": " +
                          std::to_string(occ[0]) + " + " + std::to_string(extra) + " > " +
                          std::to_string(budget_fast) + " bytes",
                      stage);
    }
}
uint64_t Ledger::alloc(int tier, int64_t bytes) {
    if (tier == 0) check_budget(bytes);
    occ[tier] += bytes;
    peak[stage][tier] = std::max(peak[stage][tier], occ[tier]);
    const uint64_t id = next_id++;
    record(0, tier, bytes, id);
    return id;
}
void Ledger::free(int tier, int64_t bytes, uint64_t id) {
    occ[tier] -= bytes;
    record(1, tier, bytes, id);
}
uint64_t Ledger::region_alloc(int tier, int64_t bytes) {
    const uint64_t id = alloc(tier, bytes);
    live[id] = Live{bytes, tier, false, tier};
    return id;
}
void Ledger::region_free(uint64_t id) {
    auto it = live.find(id);
    if (it == live.end()) throw_invariant("ledger: free of unknown region " + std::to_string(id));
    if (it->second.moving) throw_invariant("ledger: free of a region while its tier move is in flight");
    const Live r = it->second;
    live.erase(it);
    free(r.tier, r.bytes, id);
}
int Ledger::region_tier(uint64_t id) const {
    auto it = live.find(id);
    return it == live.end() ? -1 : it->second.tier;
}
// Double residency (ledger.cpp:93-123): the destination's occupancy rises at
// the start of the move, the source's falls only at its end.
void Ledger::move_start(uint64_t id, int dst) {
    auto it = live.find(id);
    if (it == live.end()) throw_invariant("ledger: tier move of unknown region");
    if (it->second.moving) throw_invariant("ledger: tier move already in flight");
    if (it->second.tier == dst) throw_invariant("ledger: tier move to the region's own tier");
    if (dst == 0) check_budget(it->second.bytes);
    it->second.moving = true;
    it->second.dst = dst;
    occ[dst] += it->second.bytes;
    peak[stage][dst] = std::max(peak[stage][dst], occ[dst]);
    record(2, dst, it->second.bytes, id);
}
void Ledger::move_end(uint64_t id) {
    auto it = live.find(id);
    if (it == live.end() || !it->second.moving) throw_invariant("ledger: tier move end without start");
    const int src = it->second.tier;
    it->second.tier = it->second.dst;
    it->second.moving = false;
    occ[src] -= it->second.bytes;
    record(3, src, it->second.bytes, id);
}

DevBuf& DevBuf::operator=(DevBuf&& o) noexcept {
    if (this != &o) {
        reset();
        p = o.p;
        bytes = o.bytes;
        ledger = o.ledger;
        tier = o.tier;
        id = o.id;
        o.p = nullptr;
        o.bytes = 0;
    }
    return *this;
}
void DevBuf::reset() {
    if (p) {
        if (tier == 0) cudaFree(p);
        else cudaFreeHost(p);
        if (ledger) ledger->free(tier, bytes, id);
    }
    p = nullptr;
    bytes = 0;
}
DevBuf dev_alloc(Ledger* l, int64_t bytes, bool zero) {
    DevBuf b;
    if (bytes <= 0) return b;
    if (l) b.id = l->alloc(0, bytes);
    LC_CUDA(cudaMalloc(&b.p, static_cast<size_t>(bytes)));
    if (zero) {
        // zero channel padding (TMA 64-channel blocks read it): complete
        // before any non-blocking-stream kernel can touch the buffer
        LC_CUDA(cudaMemset(b.p, 0, static_cast<size_t>(bytes)));
        LC_CUDA(cudaStreamSynchronize(nullptr));
    }
    b.bytes = bytes;
    b.ledger = l;
    b.tier = 0;
    return b;
}
void h2d_blocking(void* dst, const void* src, size_t bytes) {
    LC_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
    LC_CUDA(cudaStreamSynchronize(nullptr));
}

DevBuf host_alloc(Ledger* l, int64_t bytes) {
    DevBuf b;
    if (bytes <= 0) return b;
    if (l) b.id = l->alloc(1, bytes);
    LC_CUDA(cudaHostAlloc(&b.p, static_cast<size_t>(bytes), cudaHostAllocDefault));
    b.bytes = bytes;
    b.ledger = l;
    b.tier = 1;
    return b;
}

namespace {

int round_up(int v, int m) { return (v + m - 1) / m * m; }

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        LC_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p)
            throw LcError(kCudaError, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

void encode_map(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* base,
                const uint64_t* dims, const uint64_t* strides_bytes, const uint32_t* box,
                const uint32_t* estr, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    const CUresult r = encode_fn()(m, dt, static_cast<cuuint32_t>(rank), const_cast<void*>(base), dims,
                                   strides_bytes, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw LcError(kCudaError, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
}

// LC_CLEAN_EVICT=0 moves every eviction's bytes, clean or not (A/B timing)
bool clean_evict_enabled() {
    static const bool on = !(std::getenv("LC_CLEAN_EVICT") && std::atoi(std::getenv("LC_CLEAN_EVICT")) == 0);
    return on;
}

// LC_SPLIT_STORE=0 runs the cache-producing up path on the whole CFG batch (A/B timing)
bool split_store_enabled() {
    static const bool on = !(std::getenv("LC_SPLIT_STORE") && std::atoi(std::getenv("LC_SPLIT_STORE")) == 0);
    return on;
}

// LC_TAP_GATHER=0 keeps the thin-output convs as direct k x k GEMMs (A/B timing)
bool tap_gather_enabled() {
    static const bool on = !(std::getenv("LC_TAP_GATHER") && std::atoi(std::getenv("LC_TAP_GATHER")) == 0);
    return on;
}

// LC_SUBPIX_FUSED=0 runs the decoder's last stage as tap-to-N conv + gather (A/B)
bool subpix_fused_enabled() {
    static const bool on = !(std::getenv("LC_SUBPIX_FUSED") && std::atoi(std::getenv("LC_SUBPIX_FUSED")) == 0);
    return on;
}

// LC_TMA_STORE=0 turns the TMA-store epilogue off (A/B timing)
bool tma_store_enabled() {
    static const bool on = !(std::getenv("LC_TMA_STORE") && std::atoi(std::getenv("LC_TMA_STORE")) == 0);
    return on;
}

// Border-class geometry: lattice window length L and position Y with the
// requested distances (capped at rc) to the low/high window edges.
void class_geom(int d_lo, int d_hi, int rc, int* L, int* Y) {
    if (rc == 0) {
        *L = 1, *Y = 0;
    } else if (d_lo < rc && d_hi < rc) {
        *L = d_lo + d_hi + 1, *Y = d_lo;
    } else if (d_lo < rc) {
        *Y = d_lo, *L = d_lo + rc + 2;
    } else if (d_hi < rc) {
        *Y = rc + 1, *L = rc + 2 + d_hi;
    } else {
        *Y = rc + 1, *L = 2 * rc + 3;
    }
}

}  // namespace

// ------------------------------------------------------- layer packing
// Pixel tile of a launch: TI x TH x TW <= 128 (one UMMA M) with the fewest
// tiles, i.e. the least padded M; ties keep the widest rows.  Full-width rows
// first (TW = w), then powers of two.  E.g. the 9x16 lattices of config C
// (mid, u2): 16x8 tiles leave a 1-row tail per image (56 % useful M); 16x1x8
// tiles (one row of 8 images) are 89 % useful.
void choose_tile(int n, int h, int w, int* TW, int* TH, int* TI) {
    int best = -1, bw = 1, bh = 1, bi = 1;
    auto consider = [&](int tw) {
        if (tw < 1 || tw > 128) return;
        for (int th = std::min(h, 128 / tw); th >= 1; --th) {
            const int ti = std::max(1, std::min(n, 128 / (tw * th)));
            const int tiles = ((n + ti - 1) / ti) * ((h + th - 1) / th) * ((w + tw - 1) / tw);
            if (best < 0 || tiles < best) {
                best = tiles;
                bw = tw, bh = th, bi = ti;
            }
        }
    };
    consider(std::min(w, 128));
    for (int tw = 128; tw >= 1; tw /= 2)
        if (tw < std::min(w, 128)) consider(tw);
    *TW = bw, *TH = bh, *TI = bi;
}

int est_m_tiles(int n, int h, int w) {
    int TW, TH, TI;
    choose_tile(n, h, w, &TW, &TH, &TI);
    return ((n + TI - 1) / TI) * ((h + TH - 1) / TH) * ((w + TW - 1) / TW);
}

std::unique_ptr<TcLayer> pack_tc_layer(Ledger* l, const Bank& b, int c_split, int mode, int m_tiles_hint) {
    auto L = std::make_unique<TcLayer>();
    L->mode = mode;
    L->k = static_cast<int>(b.k);
    L->r = (L->k - 1) / 2;
    L->c_out = static_cast<int>(b.c_out);
    const int c_in = static_cast<int>(b.c_in), k = L->k, r = L->r;
    if (k * k > kMaxTaps) throw_config("unet.kernel larger than 15 is not supported on the GPU path");
    int ch0 = 0;  // first input channel of each segment
    int seg_ch0[2] = {0, 0};
    if (mode == 0) {
        L->P = 1;
        L->rc = r;
        if (c_split > 0 && c_split < c_in) {
            L->nseg = 2;
            L->seg_c[0] = c_split;
            L->seg_c[1] = c_in - c_split;
        } else {
            L->nseg = 1;
            L->seg_c[0] = c_in;
        }
        for (int s = 0; s < L->nseg; ++s) {
            L->seg_ntaps[s] = k * k;
            L->seg_m[s] = 1;
            for (int t = 0; t < k * k; ++t) {
                L->ox[s][0][t] = static_cast<int8_t>(t % k - r);
                L->oy[s][0][t] = static_cast<int8_t>(t / k - r);
            }
        }
    } else {
        if (k != 3) throw_invariant("sub-pixel packing needs k == 3");
        L->P = 4;
        L->rc = 1;
        int s = 0;
        if (c_split > 0) {  // full-res skip, stride-2 taps
            L->seg_c[s] = c_split;
            L->seg_ntaps[s] = 9;
            L->seg_m[s] = 2;
            for (int p = 0; p < 4; ++p)
                for (int t = 0; t < 9; ++t) {
                    L->oy[s][p][t] = static_cast<int8_t>(p / 2 + t / 3 - 1);
                    L->ox[s][p][t] = static_cast<int8_t>(p % 2 + t % 3 - 1);
                }
            ++s;
        }
        L->seg_c[s] = c_in - c_split;  // low-res operand, merged 2x2 taps
        L->seg_ntaps[s] = 4;
        L->seg_m[s] = 1;
        for (int p = 0; p < 4; ++p)
            for (int t = 0; t < 4; ++t) {
                L->oy[s][p][t] = static_cast<int8_t>(t / 2 - 1 + p / 2);
                L->ox[s][p][t] = static_cast<int8_t>(t % 2 - 1 + p % 2);
            }
        L->nseg = s + 1;
    }
    for (int s = 0; s < L->nseg; ++s) {
        seg_ch0[s] = ch0;
        ch0 += L->seg_c[s];
        L->seg_cpad[s] = round_up(L->seg_c[s], 64);
        L->seg_kbase[s] = L->k_total;
        L->k_total += L->seg_ntaps[s] * L->seg_cpad[s];
    }
    // N tiling: fewest N tiles of <= 256 columns (largest BN: least A
    // re-reading, best MMA/smem ratio) by default.  With the run geometry
    // known (m_tiles_hint), BN minimises a wave-quantisation cost model of
    // the persistent schedule: waves = ceil(units / slots) (148 CTAs, or 74
    // CTA pairs of M = 256 when conv_tc_cta_group would pick pairs), each
    // wave costing BN + 32 (per-tile fixed overhead ~ 32 columns; pairs 5%
    // cheaper: half the weight staging per CTA; single CTAs on long K loops
    // 35% dearer: measured, they are shared-memory-bandwidth bound).
    // E.g. d2/u2 at 16x16 (1280 out): BN 256 -> 160 units = 3 waves of
    // pairs, BN 160 -> 256 units = 4 shorter waves (-11%).
    int nt = 1;
    while (round_up((L->c_out + nt - 1) / nt, 16) > 256) ++nt;
    L->BN = round_up((L->c_out + nt - 1) / nt, 16);
    if (m_tiles_hint > 0 && L->c_out > 64) {
        const int kb = L->k_total / 64;
        double best = 1e30;
        int best_bn = L->BN;
        for (int bn = 256; bn >= 48; bn -= 16) {
            const int n_t = (L->c_out + bn - 1) / bn;
            if (n_t * bn - L->c_out >= bn) continue;  // an empty N tile
            if (static_cast<double>(n_t) * bn > 1.125 * round_up(L->c_out, 16)) continue;  // > 12.5% padding
            const int64_t tiles = static_cast<int64_t>(m_tiles_hint) * n_t * L->P;
            const int64_t pair_units = static_cast<int64_t>((m_tiles_hint + 1) / 2) * n_t * L->P;
            // pairs as conv_tc_cta_group picks them (>= 2 waves, or a long K
            // loop filling >= 3/4 of the pair slots)
            const bool pair = bn % 32 == 0 && m_tiles_hint >= 2 && kb >= 32 &&
                              (tiles >= 2 * 148 || (kb >= 64 && 4 * pair_units >= 3 * 74));
            const int64_t units = pair ? pair_units : tiles;
            const int slots = pair ? 74 : 148;
            static const double ovh = std::getenv("LC_BN_OVERHEAD") ? std::atof(std::getenv("LC_BN_OVERHEAD")) : 32.0;
            const double cost = static_cast<double>((units + slots - 1) / slots) *
                                (pair ? 0.95 : (kb >= 32 ? 1.35 : 1.0)) * (bn + ovh);
            if (cost < best - 1e-9) {
                best = cost;
                best_bn = bn;
            }
        }
        L->BN = best_bn;
        nt = (L->c_out + L->BN - 1) / L->BN;
    }
    L->n_pad = nt * L->BN;
    // power-of-two weight scale ~ sqrt(fan_in): exact to undo in fp32
    const double fan_in = static_cast<double>(k) * k * c_in;
    L->wscale = std::ldexp(1.0f, static_cast<int>(std::lround(0.5 * std::log2(fan_in))));

    // fp32 packed weights [P][n_pad][k_total]
    const size_t nW = static_cast<size_t>(L->P) * L->n_pad * L->k_total;
    std::vector<float> wf(nW, 0.0f);
    auto tap = [&](int oc, int ic, int ky, int kx) {
        return b.taps[((static_cast<size_t>(oc) * c_in + ic) * k + ky) * k + kx];
    };
    // merged-row sets of the sub-pixel decomposition: rows(py, dy)
    auto rows = [](int par, int d, int* lo, int* hi) {
        if (par == 0) {
            *lo = d == 0 ? 0 : 1;
            *hi = d == 0 ? 1 : 3;
        } else {
            *lo = d == 0 ? 0 : 2;
            *hi = d == 0 ? 2 : 3;
        }
    };
    for (int p = 0; p < L->P; ++p)
        for (int oc = 0; oc < L->c_out; ++oc) {
            float* row = wf.data() + (static_cast<size_t>(p) * L->n_pad + oc) * L->k_total;
            for (int s = 0; s < L->nseg; ++s) {
                const bool merged = mode == 1 && L->seg_ntaps[s] == 4;
                for (int t = 0; t < L->seg_ntaps[s]; ++t)
                    for (int c = 0; c < L->seg_c[s]; ++c) {
                        const int ic = seg_ch0[s] + c;
                        float v;
                        if (!merged) {
                            v = tap(oc, ic, t / k, t % k);
                        } else {
                            int y0, y1, x0, x1;
                            rows(p / 2, t / 2, &y0, &y1);
                            rows(p % 2, t % 2, &x0, &x1);
                            double acc = 0.0;
                            for (int ky = y0; ky < y1; ++ky)
                                for (int kx = x0; kx < x1; ++kx) acc += tap(oc, ic, ky, kx);
                            v = static_cast<float>(acc);
                        }
                        row[L->seg_kbase[s] + t * L->seg_cpad[s] + c] = v;
                    }
            }
        }
    std::vector<__half> wh(nW);
    for (size_t i = 0; i < nW; ++i) wh[i] = __float2half_rn(wf[i] * L->wscale);
    L->w = dev_alloc(l, static_cast<int64_t>(nW * sizeof(__half)), false);
    h2d_blocking(L->w.p, wh.data(), nW * sizeof(__half));

    std::vector<float> bias(static_cast<size_t>(L->n_pad), 0.0f);
    for (int oc = 0; oc < L->c_out; ++oc) bias[oc] = b.bias[oc];
    L->bias = dev_alloc(l, L->n_pad * 4, false);
    h2d_blocking(L->bias.p, bias.data(), bias.size() * 4);

    // conditioning-shift tables: sum of in-bound tap weights per class
    const int rc = L->rc, rr = rc + 1, ncls = rr * rr * rr * rr;
    std::vector<float> corr(static_cast<size_t>(L->P) * ncls * L->n_pad, 0.0f);
    for (int p = 0; p < L->P; ++p)
        for (int cls = 0; cls < ncls; ++cls) {
            const int dt = cls / (rr * rr * rr), db = (cls / (rr * rr)) % rr;
            const int dl = (cls / rr) % rr, dr = cls % rr;
            int Ly, Y, Lx, X;
            class_geom(dt, db, rc, &Ly, &Y);
            class_geom(dl, dr, rc, &Lx, &X);
            for (int oc = 0; oc < L->c_out; ++oc) {
                const float* row = wf.data() + (static_cast<size_t>(p) * L->n_pad + oc) * L->k_total;
                double acc = 0.0;
                for (int s = 0; s < L->nseg; ++s) {
                    const int m = L->seg_m[s];
                    for (int t = 0; t < L->seg_ntaps[s]; ++t) {
                        const int sy = Y * m + L->oy[s][p][t], sx = X * m + L->ox[s][p][t];
                        if (sy < 0 || sy >= Ly * m || sx < 0 || sx >= Lx * m) continue;
                        for (int c = 0; c < L->seg_c[s]; ++c) acc += row[L->seg_kbase[s] + t * L->seg_cpad[s] + c];
                    }
                }
                corr[(static_cast<size_t>(p) * ncls + cls) * L->n_pad + oc] = static_cast<float>(acc);
            }
        }
    L->corr = dev_alloc(l, static_cast<int64_t>(corr.size() * 4), false);
    h2d_blocking(L->corr.p, corr.data(), corr.size() * 4);
    return L;
}

std::unique_ptr<ThinLayer> pack_thin_layer(Ledger* l, const Bank& b) {
    auto L = std::make_unique<ThinLayer>();
    L->c_in = static_cast<int>(b.c_in);
    L->c_out = static_cast<int>(b.c_out);
    L->k = static_cast<int>(b.k);
    L->w = dev_alloc(l, static_cast<int64_t>(b.taps.size() * 4), false);
    h2d_blocking(L->w.p, b.taps.data(), b.taps.size() * 4);
    L->bias = dev_alloc(l, static_cast<int64_t>(b.bias.size() * 4), false);
    h2d_blocking(L->bias.p, b.bias.data(), b.bias.size() * 4);
    return L;
}

// ------------------------------------------------------- conv launch
Bank patch_bank(const Bank& b) {
    Bank p;
    const int64_t kk = b.c_in * b.k * b.k;
    p.c_in = (kk + 63) / 64 * 64;
    p.c_out = b.c_out;
    p.k = 1;
    p.taps.assign(static_cast<size_t>(p.c_out * p.c_in), 0.0f);
    for (int64_t oc = 0; oc < b.c_out; ++oc)
        for (int64_t t = 0; t < kk; ++t) p.taps[oc * p.c_in + t] = b.taps[oc * kk + t];
    p.bias = b.bias;
    return p;
}

// Tap-to-N bank of a thin-output k x k conv: a 1x1 conv whose output
// channel t*C + c carries tap t of channel c (no bias; the gather adds it).
Bank tap_bank(const Bank& b) {
    Bank t;
    const int64_t kk = b.k * b.k;
    t.c_in = b.c_in;
    t.c_out = kk * b.c_out;
    t.k = 1;
    t.taps.assign(static_cast<size_t>(t.c_out * t.c_in), 0.0f);
    for (int64_t tp = 0; tp < kk; ++tp)
        for (int64_t c = 0; c < b.c_out; ++c)
            for (int64_t ic = 0; ic < b.c_in; ++ic)
                t.taps[static_cast<size_t>((tp * b.c_out + c) * t.c_in + ic)] = b.taps[(c * b.c_in + ic) * kk + tp];
    t.bias.assign(static_cast<size_t>(t.c_out), 0.0f);
    return t;
}

// K8 operand: a tap bank's rows as fp16 [round_up(rows, 16)][kb * 64], zero
// padded, times the power-of-two scale pack_tc_layer gives the same bank
// (fan_in = c_in for a 1x1 tap bank), so K8 rounds the weights and the
// accumulator exactly as the tap-to-N GEMM it replaces; the epilogue
// multiplies by scale / wscale.
DevBuf pack_tap_w16(Ledger* l, const Bank& tb, int* kb_out, int* n_out, float* wscale_out) {
    const int kb = static_cast<int>((tb.c_in + 63) / 64);
    const int n = static_cast<int>((tb.c_out + 15) / 16 * 16);
    const int kp = 64 * kb;
    const float wscale = std::ldexp(1.0f, static_cast<int>(std::lround(0.5 * std::log2(static_cast<double>(tb.c_in)))));
    std::vector<__half> w16(static_cast<size_t>(n) * kp, __float2half_rn(0.0f));
    for (int64_t r = 0; r < tb.c_out; ++r)
        for (int64_t ic = 0; ic < tb.c_in; ++ic)
            w16[static_cast<size_t>(r * kp + ic)] =
                __float2half_rn(tb.taps[static_cast<size_t>(r * tb.c_in + ic)] * wscale);
    *wscale_out = wscale;
    DevBuf b = dev_alloc(l, static_cast<int64_t>(w16.size() * 2), false);
    h2d_blocking(b.p, w16.data(), w16.size() * 2);
    *kb_out = kb;
    *n_out = n;
    return b;
}

// Sub-pixel tap-to-N bank of nearest-upsample + 3x3 (the last decoder conv):
// output channel (p*4 + t)*C + c = merged weights of parity p = (py, px) and
// low-res tap t = (dy, dx) (see launch_subpix_gather; written channel-planar).
Bank subpix_tap_bank(const Bank& b) {
    if (b.k != 3) throw_invariant("sub-pixel tap bank needs k == 3");
    Bank t;
    t.c_in = b.c_in;
    if (b.c_out > 4) throw_invariant("sub-pixel tap bank needs c_out <= 4");
    t.c_out = 16 * b.c_out;
    t.k = 1;
    t.taps.assign(static_cast<size_t>(t.c_out * t.c_in), 0.0f);
    t.bias.assign(static_cast<size_t>(t.c_out), 0.0f);
    const int lo[2][2] = {{0, 1}, {0, 2}}, hi[2][2] = {{1, 3}, {2, 3}};  // rows(parity, d)
    for (int p = 0; p < 4; ++p)
        for (int tp = 0; tp < 4; ++tp) {
            const int py = p / 2, px = p % 2, dy = tp / 2, dx = tp % 2;
            for (int64_t c = 0; c < b.c_out; ++c)
                for (int64_t ic = 0; ic < b.c_in; ++ic) {
                    double acc = 0.0;
                    for (int ky = lo[py][dy]; ky < hi[py][dy]; ++ky)
                        for (int kx = lo[px][dx]; kx < hi[px][dx]; ++kx)
                            acc += b.taps[((c * b.c_in + ic) * 3 + ky) * 3 + kx];
                    t.taps[static_cast<size_t>(((p * 4 + tp) * b.c_out + c) * t.c_in + ic)] = static_cast<float>(acc);
                }
        }
    return t;
}

// K8 decoder operand (row-summed sub-pixel form): rows (py, px, dx, c) --
// ((py*2 + px)*2 + dx)*C + c -- and K blocks (o, channel block) with o the
// window-row offset dy + py of the merged 2x2 tap (dy = o - py in {0, 1},
// zero otherwise), fp16 times the power-of-two scale of the tap bank
// (fan_in = c_in), padded to [round_up(8C, 16)][3 * kb * 64].
DevBuf pack_rowsum_w16(Ledger* l, const Bank& b, int* kb_out, int* n_out, float* wscale_out) {
    if (b.k != 3 || b.c_out > 4) throw_invariant("row-summed sub-pixel bank needs k == 3, c_out <= 4");
    const Bank t = subpix_tap_bank(b);  // rows (p*4 + tp)*C + c, tp = dy*2 + dx
    const int C = static_cast<int>(b.c_out), kb = static_cast<int>((b.c_in + 63) / 64);
    const int n = (8 * C + 15) / 16 * 16, kp = 3 * kb * 64;
    const float wscale = std::ldexp(1.0f, static_cast<int>(std::lround(0.5 * std::log2(static_cast<double>(b.c_in)))));
    std::vector<__half> w16(static_cast<size_t>(n) * kp, __float2half_rn(0.0f));
    for (int py = 0; py < 2; ++py)
        for (int px = 0; px < 2; ++px)
            for (int dx = 0; dx < 2; ++dx)
                for (int c = 0; c < C; ++c) {
                    const int row = ((py * 2 + px) * 2 + dx) * C + c;
                    for (int o = 0; o < 3; ++o) {
                        const int dy = o - py;
                        if (dy < 0 || dy > 1) continue;
                        const int trow = ((py * 2 + px) * 4 + dy * 2 + dx) * C + c;
                        for (int64_t ic = 0; ic < b.c_in; ++ic)
                            w16[static_cast<size_t>(row) * kp + o * kb * 64 + ic] =
                                __float2half_rn(t.taps[static_cast<size_t>(trow * t.c_in + ic)] * wscale);
                    }
                }
    *wscale_out = wscale;
    DevBuf buf = dev_alloc(l, static_cast<int64_t>(w16.size() * 2), false);
    h2d_blocking(buf.p, w16.data(), w16.size() * 2);
    *kb_out = kb;
    *n_out = n;
    return buf;
}

Bank subpixel_shuffle_bank(const Bank& b) {
    if (b.k != 3) throw_invariant("sub-pixel shuffle needs k == 3");
    Bank s;
    s.c_in = b.c_in;
    s.c_out = 4 * b.c_out;
    s.k = 3;
    s.taps.assign(static_cast<size_t>(s.c_out * s.c_in * 9), 0.0f);
    s.bias.resize(static_cast<size_t>(s.c_out));
    // rows(parity, d): merged source rows of the 3x3 kernel
    const int lo[2][2] = {{0, 1}, {0, 2}}, hi[2][2] = {{1, 3}, {2, 3}};
    for (int p = 0; p < 4; ++p) {
        const int py = p / 2, px = p % 2;
        for (int64_t o = 0; o < b.c_out; ++o) {
            s.bias[p * b.c_out + o] = b.bias[o];
            for (int64_t c = 0; c < b.c_in; ++c)
                for (int ry = 0; ry < 3; ++ry)
                    for (int rx = 0; rx < 3; ++rx) {
                        const int dy = ry - py, dx = rx - px;  // low-res row Y+ry-1 = Y+dy-1+py
                        if (dy < 0 || dy > 1 || dx < 0 || dx > 1) continue;
                        double acc = 0.0;
                        for (int ky = lo[py][dy]; ky < hi[py][dy]; ++ky)
                            for (int kx = lo[px][dx]; kx < hi[px][dx]; ++kx)
                                acc += b.taps[((o * b.c_in + c) * 3 + ky) * 3 + kx];
                        s.taps[(((p * b.c_out + o) * s.c_in + c) * 3 + ry) * 3 + rx] = static_cast<float>(acc);
                    }
        }
    }
    return s;
}

// Halo operand staging (ConvParams::halo) for layers that qualify: one
// segment at source scale 1, several taps, one-row tiles of 128 pixels, and
// either the weight-stationary schedule with >= 2 halo stages or (any CTA
// group) 2 halo stages beside a ring of >= 3 weight stages.  The activation map is
// re-encoded with the halo box {64, hw, hh, 1}; LC_HALO=0 disables it.
void plan_halo(const TcLayer& L, ConvParams* p, const __half* base, const uint64_t* dims, const uint64_t* strides) {
    static const int env = std::getenv("LC_HALO") ? std::atoi(std::getenv("LC_HALO")) : 1;
    p->halo = 0;
    if (!env || L.nseg != 1 || L.seg_m[0] != 1 || L.seg_ntaps[0] < 2) return;
    if (p->TW != 128 || p->TH != 1 || p->TI != 1) return;
    int dxr = 0, dyr = 0;
    for (int q = 0; q < L.P; ++q) {
        int x0 = 127, x1 = -128, y0 = 127, y1 = -128;
        for (int t = 0; t < L.seg_ntaps[0]; ++t) {
            x0 = std::min(x0, static_cast<int>(L.ox[0][q][t]));
            x1 = std::max(x1, static_cast<int>(L.ox[0][q][t]));
            y0 = std::min(y0, static_cast<int>(L.oy[0][q][t]));
            y1 = std::max(y1, static_cast<int>(L.oy[0][q][t]));
        }
        p->hox[q] = x0;
        p->hoy[q] = y0;
        dxr = std::max(dxr, x1 - x0);
        dyr = std::max(dyr, y1 - y0);
    }
    p->hw = p->TW + dxr;
    p->hh = 1 + dyr;
    if (p->hw > 256 || p->hh > 8) return;
    p->halo = 1;
    if (!conv_tc_halo_fits(*p, L.P)) {
        p->halo = 0;
        return;
    }
    const uint32_t box[4] = {64, static_cast<uint32_t>(p->hw), static_cast<uint32_t>(p->hh), 1};
    const uint32_t estr[4] = {1, 1, 1, 1};
    encode_map(&p->tmA[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, base, dims, strides, box, estr);
}

void run_tc_conv(const TcLayer& L, const Act* srcs, const Act& out, const Window& win, float s,
                 float o, bool silu, cudaStream_t st, float* out32, int shuffle_c, bool nhwc32, bool planar) {
    ConvParams p{};
    const int sub = L.mode == 1 ? 2 : 1;
    // per parity class q = (py, px): output pixels 2Y+py in [oy0, oy1)
    int Lh = 0, Lw = 0;
    for (int q = 0; q < 4; ++q) {
        const int py = sub == 2 ? q / 2 : 0, px = sub == 2 ? q % 2 : 0;
        p.ly0[q] = (win.oy0 - py + sub - 1) / sub;
        p.ly1[q] = (win.oy1 - py + sub - 1) / sub;
        p.lx0[q] = (win.ox0 - px + sub - 1) / sub;
        p.lx1[q] = (win.ox1 - px + sub - 1) / sub;
        Lh = std::max(Lh, p.ly1[q] - p.ly0[q]);
        Lw = std::max(Lw, p.lx1[q] - p.lx0[q]);
    }
    p.cy0 = win.vy0 / sub;
    p.cy1 = win.vy1 / sub;
    p.cx0 = win.vx0 / sub;
    p.cx1 = win.vx1 / sub;
    p.n_img = out.n;
    choose_tile(out.n, Lh, Lw, &p.TW, &p.TH, &p.TI);
    p.tiles_x = (Lw + p.TW - 1) / p.TW;
    p.tiles_y = (Lh + p.TH - 1) / p.TH;
    p.tiles_i = (out.n + p.TI - 1) / p.TI;
    p.nseg = L.nseg;
    const __half* seg0_base = nullptr;
    uint64_t seg0_dims[4] = {}, seg0_strides[3] = {};
    for (int sgi = 0; sgi < L.nseg; ++sgi) {
        const Act& a = srcs[sgi];
        const int m = L.seg_m[sgi];
        // operand window in its own coordinates
        const int scale_num = (L.mode == 1) ? m : 1;  // full-res skip: x2 of lattice, low-res: x1
        const int wy0 = p.cy0 * scale_num, wy1 = p.cy1 * scale_num;
        const int wx0 = p.cx0 * scale_num, wx1 = p.cx1 * scale_num;
        const int wy0s = L.mode == 1 ? wy0 : win.vy0, wy1s = L.mode == 1 ? wy1 : win.vy1;
        const int wx0s = L.mode == 1 ? wx0 : win.vx0, wx1s = L.mode == 1 ? wx1 : win.vx1;
        const __half* base = a.p + (static_cast<int64_t>(wy0s) * a.w + wx0s) * a.cs;
        const uint64_t dims[4] = {static_cast<uint64_t>(a.cs), static_cast<uint64_t>(wx1s - wx0s),
                                  static_cast<uint64_t>(wy1s - wy0s), static_cast<uint64_t>(a.n)};
        const uint64_t strides[3] = {static_cast<uint64_t>(a.cs) * 2,
                                     static_cast<uint64_t>(a.w) * a.cs * 2,
                                     static_cast<uint64_t>(a.h) * a.w * a.cs * 2};
        const uint32_t box[4] = {64, static_cast<uint32_t>(p.TW * m), static_cast<uint32_t>(p.TH * m),
                                 static_cast<uint32_t>(p.TI)};
        const uint32_t estr[4] = {1, static_cast<uint32_t>(m), static_cast<uint32_t>(m), 1};
        encode_map(&p.tmA[sgi], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, base, dims, strides, box, estr);
        if (sgi == 0) {
            seg0_base = base;
            std::memcpy(seg0_dims, dims, sizeof(dims));
            std::memcpy(seg0_strides, strides, sizeof(strides));
        }
        ConvSegDev& sd = p.seg[sgi];
        sd.ntaps = L.seg_ntaps[sgi];
        sd.ncb = L.seg_cpad[sgi] / 64;
        sd.kbase = L.seg_kbase[sgi];
        sd.mx = sd.my = m;
        sd.wx0 = wx0s;
        sd.wy0 = wy0s;
        std::memcpy(sd.ox, L.ox[sgi], sizeof(sd.ox));
        std::memcpy(sd.oy, L.oy[sgi], sizeof(sd.oy));
    }
    {
        const uint64_t dims[3] = {static_cast<uint64_t>(L.k_total), static_cast<uint64_t>(L.n_pad),
                                  static_cast<uint64_t>(L.P)};
        const uint64_t strides[2] = {static_cast<uint64_t>(L.k_total) * 2,
                                     static_cast<uint64_t>(L.n_pad) * L.k_total * 2};
        p.cg = conv_tc_cta_group(L.BN, p.tiles_x * p.tiles_y * p.tiles_i, L.n_pad / L.BN, L.P, L.k_total / 64);
        p.nparity = L.P;
        {
            const double wbytes = 2.0 * L.n_pad * L.k_total * L.P;
            double abytes = 0;
            for (int sgi = 0; sgi < L.nseg; ++sgi) abytes += 2.0 * srcs[sgi].elems();
            p.m_fastest = wbytes > abytes ? 1 : 0;
        }
        const uint32_t box[3] = {64, static_cast<uint32_t>(L.BN / p.cg), 1};
        const uint32_t estr[3] = {1, 1, 1};
        encode_map(&p.tmB, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, L.w.p, dims, strides, box, estr);
    }
    p.BN = L.BN;
    p.n_pad = L.n_pad;
    p.c_out = L.c_out;
    p.cs_out = out.cs;
    p.out_h = out.h;
    p.out_w = out.w;
    p.sy = p.sx = sub;
    for (int q = 0; q < 4; ++q) {
        p.py[q] = L.mode == 1 ? q / 2 : 0;
        p.px[q] = L.mode == 1 ? q % 2 : 0;
    }
    p.out = out.p;
    p.out32 = out32;
    p.nhwc32 = out32 && nhwc32 ? 1 : 0;
    p.planar32 = p.nhwc32 && planar ? 1 : 0;
    if (p.planar32 && sub != 1) throw_invariant("planar raw output needs a non-sub-pixel layer");
    if ((!out32 || p.nhwc32) && tma_store_enabled()) {
        // TMA-store epilogue: each warp's 32 pixels must form one box in
        // (x, y, img) of the tile, and every parity class a non-empty window
        uint32_t bxd = 0, byd = 0, bid = 0;
        const int tp = p.TH * p.TW;
        if (p.TW % 32 == 0) {
            bxd = 32, byd = 1, bid = 1;
        } else if (32 % p.TW == 0 && tp % 32 == 0) {
            bxd = p.TW, byd = 32 / p.TW, bid = 1;
        } else if (32 % p.TW == 0 && 32 % tp == 0 && (p.TI * tp) % 32 == 0) {
            bxd = p.TW, byd = p.TH, bid = 32 / tp;
        }
        bool ok = bxd != 0 && (!p.planar32 || bxd >= 4);  // planar fp32 boxes need >= 16 B rows
        for (int q = 0; q < L.P; ++q) ok = ok && p.ly1[q] > p.ly0[q] && p.lx1[q] > p.lx0[q];
        if (ok) {
            p.tma_out = 1;
            for (int q = 0; q < L.P; ++q) {
                const int py = p.py[q], px = p.px[q];
                const int esz = p.nhwc32 ? 4 : 2;
                if (p.planar32) {
                    // [channel][img][y][x]: dims {x, y, img, channel}
                    const char* pbase = reinterpret_cast<const char*>(out32) +
                                        (static_cast<int64_t>(p.ly0[q]) * out.w + p.lx0[q]) * 4;
                    const uint64_t pdims[4] = {static_cast<uint64_t>(p.lx1[q] - p.lx0[q]),
                                               static_cast<uint64_t>(p.ly1[q] - p.ly0[q]),
                                               static_cast<uint64_t>(out.n), static_cast<uint64_t>(out.cs)};
                    const uint64_t pstr[3] = {static_cast<uint64_t>(out.w) * 4,
                                              static_cast<uint64_t>(out.h) * out.w * 4,
                                              static_cast<uint64_t>(out.n) * out.h * out.w * 4};
                    const uint32_t pbox[4] = {bxd, byd, bid, 16};
                    const uint32_t pestr[4] = {1, 1, 1, 1};
                    encode_map(&p.tmO[q], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, pbase, pdims, pstr, pbox, pestr,
                               CU_TENSOR_MAP_SWIZZLE_NONE);
                    continue;
                }
                const char* base = (p.nhwc32 ? reinterpret_cast<const char*>(out32) : reinterpret_cast<const char*>(out.p)) +
                                   (static_cast<int64_t>(p.ly0[q] * sub + py) * out.w + (p.lx0[q] * sub + px)) * out.cs * esz;
                const uint64_t dims[4] = {static_cast<uint64_t>(out.cs), static_cast<uint64_t>(p.lx1[q] - p.lx0[q]),
                                          static_cast<uint64_t>(p.ly1[q] - p.ly0[q]), static_cast<uint64_t>(out.n)};
                const uint64_t strides[3] = {static_cast<uint64_t>(sub) * out.cs * esz,
                                             static_cast<uint64_t>(sub) * out.w * out.cs * esz,
                                             static_cast<uint64_t>(out.h) * out.w * out.cs * esz};
                const uint32_t box[4] = {16, bxd, byd, bid};
                const uint32_t estr[4] = {1, 1, 1, 1};
                // fp16: the 32 px x 16 ch staging box has 32 B rows, swizzled so the
                // epilogue's 16-byte stores of 8 consecutive pixels hit distinct banks
                // (the staging slots are 256 B aligned, the 32B-swizzle atom)
                encode_map(&p.tmO[q], p.nhwc32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4,
                           base, dims, strides, box, estr,
                           p.nhwc32 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_32B);
            }
        }
    }
    p.shuffle_c = shuffle_c;
    p.bias = L.bias.as<float>();
    p.corr = L.corr.as<float>();
    p.rc = L.rc;
    p.scale = s / L.wscale;
    p.shift = o;
    static const bool silu_exact = std::getenv("LC_SILU_EXACT") && std::atoi(std::getenv("LC_SILU_EXACT")) != 0;
    p.silu = silu ? (silu_exact ? 2 : 1) : 0;
    plan_halo(L, &p, seg0_base, seg0_dims, seg0_strides);
    ConvProfiler* prof = conv_profiler();
    if (prof) {
        // algorithmic work of the reference op (conv2d over the concat,
        // tensor.cpp:194-195 count_macs) vs the MMA work actually issued
        int64_t pix = 0;
        for (int q = 0; q < L.P; ++q)
            pix += static_cast<int64_t>(std::max(0, p.ly1[q] - p.ly0[q])) * std::max(0, p.lx1[q] - p.lx0[q]);
        int64_t cin = 0;
        for (int sgi = 0; sgi < L.nseg; ++sgi) cin += L.seg_c[sgi];
        ConvProfiler::Rec r;
        r.alg_flops = 2.0 * static_cast<double>(pix) * out.n * L.c_out * L.k * L.k * cin;
        r.exec_flops = 2.0 * static_cast<double>(p.tiles_x) * p.tiles_y * p.tiles_i * L.P * 128.0 *
                       L.n_pad * L.k_total;
        {
            const int mt = p.tiles_x * p.tiles_y * p.tiles_i;
            r.desc = "P" + std::to_string(L.P) + " M" + std::to_string(mt) + "x128 tile " + std::to_string(p.TI) +
                     "x" + std::to_string(p.TH) + "x" + std::to_string(p.TW) + " N" + std::to_string(L.n_pad) +
                     "/BN" + std::to_string(L.BN) + " K" + std::to_string(L.k_total) + " cg" + std::to_string(p.cg) +
                     (out32 ? (nhwc32 ? " raw32" : " f32") : (silu ? " silu" : "")) + (p.tma_out ? " tma" : "") +
                     (p.halo ? " halo" : "");
        }
        LC_CUDA(cudaEventCreate(&r.e0));
        LC_CUDA(cudaEventCreate(&r.e1));
        LC_CUDA(cudaEventRecord(r.e0, st));
        LC_CUDA(launch_conv_tc(p, L.P, st));
        LC_CUDA(cudaEventRecord(r.e1, st));
        prof->recs.push_back(r);
        return;
    }
    LC_CUDA(launch_conv_tc(p, L.P, st));
}

static std::vector<Window> block_windows(const RunConfig& c, const std::string& name, int h, int w);

// ---------------------------------------------------------------- engine
Engine::Engine(int device) : device_(device) {
    LC_CUDA(cudaSetDevice(device));
    LC_CUDA(cudaStreamCreateWithFlags(&s_compute_, cudaStreamNonBlocking));
    LC_CUDA(cudaStreamCreateWithFlags(&s_d2h_, cudaStreamNonBlocking));
    LC_CUDA(cudaStreamCreateWithFlags(&s_h2d_, cudaStreamNonBlocking));
    LC_CUDA(cudaStreamCreateWithFlags(&s_comm_, cudaStreamNonBlocking));
    LC_CUDA(cudaEventCreate(&ev_base_));
    for (int b = 0; b < 2; ++b) {
        LC_CUDA(cudaEventCreateWithFlags(&ev_evict_[b], cudaEventDisableTiming));
        LC_CUDA(cudaEventCreateWithFlags(&ev_prefetch_[b], cudaEventDisableTiming));
        LC_CUDA(cudaEventCreateWithFlags(&ev_prefetch_part_[b], cudaEventDisableTiming));
    }
    for (int b = 0; b < 2; ++b) LC_CUDA(cudaEventCreateWithFlags(&ev_cache_ready_[b], cudaEventDisableTiming));
    LC_CUDA(cudaEventCreate(&ev_start_));
    for (int b = 0; b < 2; ++b) LC_CUDA(cudaEventCreateWithFlags(&ev_join_[b], cudaEventDisableTiming));
    LC_CUDA(cudaEventCreateWithFlags(&ev_vid_done_, cudaEventDisableTiming));
    LC_CUDA(cudaStreamCreateWithFlags(&s_vid_, cudaStreamNonBlocking));
    LC_CUDA(cudaEventCreateWithFlags(&ev_dl_gate_, cudaEventDisableTiming));
    LC_CUDA(cudaEventCreateWithFlags(&ev_dl_done_, cudaEventDisableTiming));
    LC_CUDA(cudaEventCreateWithFlags(&ev_dl_src_, cudaEventDisableTiming));
    if (const char* e = std::getenv("LC_NO_GRAPH")) use_graphs = (e[0] == '0');
    // LC_DL_GATE = "<step>:<stem|d0|up|head>" or "off" (download right
    // after the decode, per slice, as the synchronous run does)
    if (const char* e = std::getenv("LC_DL_GATE")) {
        const std::string g = e;
        const auto colon = g.find(':');
        if (g == "off" || colon == std::string::npos) dl_gate_step_ = -1;
        else {
            dl_gate_step_ = std::atoi(g.substr(0, colon).c_str());
            dl_gate_where_ = g.substr(colon + 1);
        }
    }
}

Engine::~Engine() {
    cudaDeviceSynchronize();
    for (auto e : ev_pool_) cudaEventDestroy(e);
    for (int b = 0; b < 3; ++b)
        for (auto e : ev_chunk_[b]) cudaEventDestroy(e);
    cudaEventDestroy(ev_base_);
    for (int b = 0; b < 2; ++b) {
        cudaEventDestroy(ev_evict_[b]);
        cudaEventDestroy(ev_prefetch_[b]);
        cudaEventDestroy(ev_prefetch_part_[b]);
    }
    for (int b = 0; b < 2; ++b) cudaEventDestroy(ev_cache_ready_[b]);
    cudaEventDestroy(ev_start_);
    for (int b = 0; b < 2; ++b) cudaEventDestroy(ev_join_[b]);
    cudaEventDestroy(ev_vid_done_);
    cudaEventDestroy(ev_dl_gate_);
    cudaEventDestroy(ev_dl_done_);
    cudaEventDestroy(ev_dl_src_);
    if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
    if (graph_) cudaGraphDestroy(graph_);
    cudaStreamDestroy(s_vid_);
    cudaStreamDestroy(s_compute_);
    cudaStreamDestroy(s_d2h_);
    cudaStreamDestroy(s_h2d_);
    cudaStreamDestroy(s_comm_);
}

cudaEvent_t Engine::next_event() {
    if (ev_next_ == ev_pool_.size()) {
        cudaEvent_t e;
        LC_CUDA(cudaEventCreate(&e));
        ev_pool_.push_back(e);
    }
    return ev_pool_[ev_next_++];
}

// Timing event record: inside a stream capture it must become an event
// record NODE (cudaEventRecordExternal) so graph replays re-record it; a
// plain record would only express a capture dependency.
void record_timing(cudaEvent_t e, cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    LC_CUDA(cudaStreamIsCapturing(st, &cs));
    if (cs == cudaStreamCaptureStatusActive) LC_CUDA(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal));
    else LC_CUDA(cudaEventRecord(e, st));
}

void Engine::record(int kind, int step, int64_t bytes, cudaStream_t st) {
    cudaEvent_t e = next_event();
    record_timing(e, st);
    marks_.push_back({kind, step, bytes, e});
}

static std::string weights_key(const RunConfig& c) {
    return std::to_string(c.depth) + "/" + std::to_string(c.base_channels) + "/" + std::to_string(c.kernel) +
           "/" + std::to_string(c.cache_depth) + "/" + std::to_string(c.in_channels) + "/" +
           std::to_string(c.unet_seed) + "/" + std::to_string(c.stages) + "/" + std::to_string(c.codec_width) +
           "/" + std::to_string(c.codec_seed) +
           // geometry steers the N tiling of the packed layers
           "/" + std::to_string(c.frames) + "x" + std::to_string(c.height) + "x" + std::to_string(c.width);
}

void Engine::configure(const RunConfig& cfg) {
    const double t_cfg = Ledger::now();
    struct SetupTimer {  // StageWall::setup: weight init + packing of this configure
        Engine* e;
        double t0;
        ~SetupTimer() { e->configure_s_ = Ledger::now() - t0; }
    } setup_timer{this, t_cfg};
    cfg.validate();
    if (async_pending_) (void)wait();
    const std::string key = weights_key(cfg);
    const bool same_weights = configured_ && key == cfg_key_;
    const bool same_geom = configured_ && cfg.frames == cfg_.frames && cfg.height == cfg_.height &&
                           cfg.width == cfg_.width && same_weights &&
                           cfg.cache_enabled == cfg_.cache_enabled &&
                           // alloc_activations: the pinned slow-tier entry and the
                           // separate upsample buffers depend on these
                           (cfg.swap_mode != SwapMode::Off) == (cfg_.swap_mode != SwapMode::Off) &&
                           cfg.chunk_enabled == cfg_.chunk_enabled && cfg.halo == cfg_.halo;
    cfg_ = cfg;
    ledger_.budget_fast = 0;  // budget applies to runs, see run()
    sim_tl_.clear();
    sim_step_s_.assign(static_cast<size_t>(cfg.steps), 0.0);
    sim_decode_s_ = 0;
    if (cfg.swap_simulate) {
        sim_tl_ = simulate_timeline(cfg);
        for (const SimEvent& e : sim_tl_)
            if (e.kind == 0) sim_step_s_[static_cast<size_t>(e.step)] = e.clock_ns * 1e-9;
        sim_decode_s_ = sim_denoise_end_ns(cfg) * 1e-9;
    }
    ledger_.virt = cfg.swap_simulate ? 0.0 : -1.0;
    if (!same_weights) {
        ledger_.enter(kSetup);
        uw_ = init_unet(cfg);
        cw_ = init_codec(cfg);
        const auto plan = block_plans(cfg);
        tc_.clear();
        tc_.resize(plan.size());
        tc_fb_.clear();
        tc_fb_.resize(plan.size());
        // Evicting full steps run the blocks below the seam level per CFG
        // branch (forward_dev, branch_deep_): their tile-count hints then see
        // T images, not 2T (the wave model picks BN for the half batch).
        const char* bde = std::getenv("LC_BRANCH_DEEP");
        const int bmode = bde ? std::atoi(bde) : 1;
        const bool evicting = cfg.cache_enabled && cfg.swap_mode == SwapMode::Async &&
                              cfg.cache_depth + 1 < cfg.depth && bmode != 0;
        for (size_t j = 0; j < plan.size(); ++j) {
            const auto& bp = plan[j];
            if (bp.name == "stem" || bp.name == "head") continue;
            // M-tile hints from the run geometry (2T images at the block's level)
            const bool half_batch = evicting && bp.level > cfg.cache_depth &&
                                    (bmode == 1 || bp.name[0] == 'u');
            const int n2 = static_cast<int>((half_batch ? 1 : 2) * cfg.frames);
            const int hl = static_cast<int>(cfg.latent_h() >> bp.level), wl = static_cast<int>(cfg.latent_w() >> bp.level);
            if (bp.name[0] == 'u') {
                const int i = std::stoi(bp.name.substr(1));
                const int c_skip = static_cast<int>(cfg.base_channels << i);
                if (cfg.kernel == 3)
                    tc_[j] = pack_tc_layer(&ledger_, uw_.banks[j], c_skip, 1,
                                           est_m_tiles(n2, std::max(1, hl / 2), std::max(1, wl / 2)));
            } else {
                tc_[j] = pack_tc_layer(&ledger_, uw_.banks[j], static_cast<int>(bp.c_in), 0, est_m_tiles(n2, hl, wl));
            }
        }
        stem_ = pack_thin_layer(&ledger_, uw_.banks.front());
        head_ = pack_thin_layer(&ledger_, uw_.banks.back());
        dec0_ = pack_thin_layer(&ledger_, cw_.dec[0]);
        dec_last_ = pack_thin_layer(&ledger_, cw_.dec[static_cast<size_t>(cfg.stages)]);
        head_tc_ = pack_tc_layer(&ledger_, uw_.banks.back(), static_cast<int>(cfg.base_channels), 0);
        {
            const Bank& hb = uw_.banks.back();
            head_tap_tc_.reset();
            head_w16_.reset();
            head_kb_ = head_n_ = 0;
            if (hb.c_out <= 4 && hb.k * hb.k * hb.c_out <= 256) {
                const Bank tb = tap_bank(hb);
                head_tap_tc_ = pack_tc_layer(&ledger_, tb, static_cast<int>(hb.c_in), 0);
                if (hb.k == 3 && tap_tc_supported(kTapConv3, static_cast<int>(hb.c_out),
                                                  static_cast<int>((tb.c_in + 63) / 64),
                                                  static_cast<int>((tb.c_out + 15) / 16 * 16)))
                    head_w16_ = pack_tap_w16(&ledger_, tb, &head_kb_, &head_n_, &head_wscale_);
                const int64_t kk = hb.k * hb.k;
                std::vector<float> ws(static_cast<size_t>(kk * hb.c_out));
                for (int64_t tp = 0; tp < kk; ++tp)
                    for (int64_t c = 0; c < hb.c_out; ++c) {
                        double acc = 0.0;
                        for (int64_t ic = 0; ic < hb.c_in; ++ic) acc += hb.taps[(c * hb.c_in + ic) * kk + tp];
                        ws[static_cast<size_t>(tp * hb.c_out + c)] = static_cast<float>(acc);
                    }
                head_wsum_ = dev_alloc(&ledger_, static_cast<int64_t>(ws.size() * 4), false);
                h2d_blocking(head_wsum_.p, ws.data(), ws.size() * 4);
                head_bias_ = dev_alloc(&ledger_, static_cast<int64_t>(hb.bias.size() * 4), false);
                h2d_blocking(head_bias_.p, hb.bias.data(), hb.bias.size() * 4);
            }
            const Bank& db = cw_.dec[static_cast<size_t>(cfg.stages)];
            dec_last_tap_tc_.reset();
            dec_last_w16_.reset();
            dec_last_kb_ = 0;
            if (db.k == 3 && db.c_out <= 4) {
                const Bank tb = subpix_tap_bank(db);
                dec_last_tap_tc_ = pack_tc_layer(&ledger_, tb, static_cast<int>(db.c_in), 0);
                if (tap_tc_supported(kTapSubpix, static_cast<int>(db.c_out), static_cast<int>((db.c_in + 63) / 64),
                                     static_cast<int>((8 * db.c_out + 15) / 16 * 16))) {
                    dec_last_w16_ = pack_rowsum_w16(&ledger_, db, &dec_last_kb_, &dec_last_n_, &dec_last_wscale_);
                }
                dec_last_bias_ = dev_alloc(&ledger_, static_cast<int64_t>(db.bias.size() * 4), false);
                h2d_blocking(dec_last_bias_.p, db.bias.data(), db.bias.size() * 4);
            }
        }
        {
            const Bank sp = patch_bank(uw_.banks.front());
            stem_kp_ = static_cast<int>(sp.c_in);
            stem_tc_ = pack_tc_layer(&ledger_, sp, stem_kp_, 0);
            const Bank dp = patch_bank(cw_.dec[0]);
            dec0_kp_ = static_cast<int>(dp.c_in);
            dec0_tc_ = pack_tc_layer(&ledger_, dp, dec0_kp_, 0);
            const Bank ds = subpixel_shuffle_bank(cw_.dec[static_cast<size_t>(cfg.stages)]);
            dec_last_tc_ = pack_tc_layer(&ledger_, ds, static_cast<int>(ds.c_in), 0);
            const Bank ep = patch_bank(cw_.enc[0]);
            enc0_kp_ = static_cast<int>(ep.c_in);
            enc0_tc_ = pack_tc_layer(&ledger_, ep, enc0_kp_, 0);
            enc_tc_.clear();
            for (int64_t i = 1; i <= cfg.stages; ++i)
                enc_tc_.push_back(pack_tc_layer(&ledger_, cw_.enc[static_cast<size_t>(i)],
                                                static_cast<int>(cw_.enc[static_cast<size_t>(i)].c_in), 0));
            img_key_.clear();
        }
        if (cw_.dec[static_cast<size_t>(cfg.stages)].c_out > 4)
            throw_config("codec image channels > 4 not supported on the GPU decoder");
        dec_tc_.clear();
        for (int64_t i = 1; i < cfg.stages; ++i) dec_tc_.push_back(pack_tc_layer(&ledger_, cw_.dec[i], 0, 1));
        cfg_key_ = key;
        T_alloc_ = -1;
    }
    {
        // materialised-upsample fallbacks of the up blocks (2-segment 3x3
        // convs over the upsampled input): only where the fused sub-pixel
        // form cannot run -- kernels other than 3x3, or chunk tiles whose
        // readable windows are not parity-aligned (halos below the radius)
        // -- so their weights (86 MB at base 320) are not resident otherwise
        const auto plan = block_plans(cfg);
        for (size_t j = 0; j < plan.size(); ++j) {
            const auto& bp = plan[j];
            if (bp.name[0] != 'u' || tc_fb_[j]) continue;
            const int hl = static_cast<int>(cfg.latent_h() >> bp.level), wl = static_cast<int>(cfg.latent_w() >> bp.level);
            bool need = cfg.kernel != 3;
            for (const Window& wd : block_windows(cfg, bp.name, hl, wl))
                if ((wd.vy0 | wd.vy1 | wd.vx0 | wd.vx1) & 1) need = true;
            if (!need) continue;
            const int i = std::stoi(bp.name.substr(1));
            ledger_.enter(kSetup);
            tc_fb_[j] = pack_tc_layer(&ledger_, uw_.banks[j], static_cast<int>(cfg.base_channels << i), 0,
                                      est_m_tiles(static_cast<int>(2 * cfg.frames), hl, wl));
        }
    }
    if (!same_geom || cfg.mode != cfg_prev_mode_ || cfg.slice_decode != cfg_prev_sliced_) T_alloc_ = -1;
    cfg_prev_mode_ = cfg.mode;
    cfg_prev_sliced_ = cfg.slice_decode;
    invalidate_graph();  // any config change re-records the body
    dec_bufs_op_.clear();  // operator-level decode workspace follows the geometry
    dec_ws_op_.G = 0;
    configured_ = true;
}

int64_t Engine::latent_elems() const {
    return cfg_.frames * cfg_.latent_channels * cfg_.latent_h() * cfg_.latent_w();
}
int64_t Engine::video_elems() const { return cfg_.frames * cfg_.image_channels * cfg_.height * cfg_.width; }

// Host-link bandwidth per direction with D2H and H2D concurrent (the swap's
// evict / prefetch pattern): 64 MB each way on the swap's copy streams,
// once per device and process.
double Engine::probe_link_gbs() {
    static double cached[64] = {};
    const int dev = device_ >= 0 && device_ < 64 ? device_ : 0;
    if (cached[dev] > 0) return cached[dev];
    const size_t bytes = size_t{64} << 20;
    DevBuf hd = host_alloc(nullptr, 2 * static_cast<int64_t>(bytes));
    DevBuf dd = dev_alloc(nullptr, 2 * static_cast<int64_t>(bytes), false);
    char* h = hd.as<char>();
    char* d = dd.as<char>();
    cudaEvent_t e[4];
    for (auto& x : e) LC_CUDA(cudaEventCreate(&x));
    double best = 0;
    for (int rep = 0; rep < 3; ++rep) {
        LC_CUDA(cudaEventRecord(e[0], s_d2h_));
        LC_CUDA(cudaEventRecord(e[2], s_h2d_));
        LC_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s_d2h_));
        LC_CUDA(cudaMemcpyAsync(d + bytes, h + bytes, bytes, cudaMemcpyHostToDevice, s_h2d_));
        LC_CUDA(cudaEventRecord(e[1], s_d2h_));
        LC_CUDA(cudaEventRecord(e[3], s_h2d_));
        LC_CUDA(cudaEventSynchronize(e[1]));
        LC_CUDA(cudaEventSynchronize(e[3]));
        float a = 0, b = 0;
        LC_CUDA(cudaEventElapsedTime(&a, e[0], e[1]));
        LC_CUDA(cudaEventElapsedTime(&b, e[2], e[3]));
        if (rep > 0) best = std::max(best, static_cast<double>(bytes) / (std::max(a, b) * 1e-3) / 1e9);
    }
    for (auto& x : e) cudaEventDestroy(x);
    cached[dev] = best;
    return best;
}

// The per-branch deep path starts the swap's transfers half a deep path
// earlier and lets entry 1's eviction start before entry 0's has finished
// queueing on the link.  Measured on C, same box back to back: 241.4
// frames/s with it, 239.7 without (42 GB/s link, no cost); on a 32 GB/s
// host link the whole-batch path left 12 ms of seam stall per video.  On by
// default (LC_BRANCH_DEEP=0 turns it off); the host link is probed once
// (reported as swap_schedule.link_gbs_probe) for swaps of >= 32 MB entries.
void Engine::decide_branch_deep() {
    branch_deep_ = 0;
    branch_seam_ = true;
    link_gbs_ = 0;
    const bool swap_async = cfg_.cache_enabled && cfg_.swap_mode == SwapMode::Async &&
                            cfg_.cache_depth + 1 < cfg_.depth;
    if (!swap_async) return;
    const char* env = std::getenv("LC_BRANCH_DEEP");
    branch_deep_ = env ? std::atoi(env) : 1;
    if (cache_.elems() * 2 >= (int64_t{32} << 20)) link_gbs_ = probe_link_gbs();
    // The branch-wise seam (the cached step's seam block per entry, first
    // half of its images as soon as they landed) only pays when the prefetch
    // is still in flight at the seam.  On a host link that moves a step's
    // entries well inside the compute window the whole-batch seam block is
    // one launch instead of four: C, one box, 3 interleaved runs each:
    // 248.3 vs 246.9 frames/s at a 48-50 GB/s probe.  LC_BRANCH_SEAM=0/1
    // forces it.
    const char* bs = std::getenv("LC_BRANCH_SEAM");
    branch_seam_ = bs ? std::atoi(bs) != 0 : !(link_gbs_ >= 45.0);
}

int64_t Engine::run_dec_group() const {
    const int64_t T = cfg_.frames;
    return std::max<int64_t>(1, std::min<int64_t>(cfg_.slice_decode ? decode_slice : T, T));
}

// Bytes of a decode workspace for slices of G frames (DecWs); every part
// 256-byte aligned as the arena carves it.
int64_t Engine::dec_ws_bytes(int G, bool want_y) const {
    auto al = [](int64_t b) { return (b + 255) / 256 * 256; };
    const int S = static_cast<int>(cfg_.stages);
    const int64_t lh = cfg_.latent_h(), lw = cfg_.latent_w();
    const int64_t cs = round_up(static_cast<int>(cfg_.codec_width), 64);
    int64_t b = 0;
    for (int i = 0; i < S; ++i) b += al(G * (lh << i) * (lw << i) * cs * 2);
    b += al(G * lh * lw * dec0_kp_ * 2);
    if (want_y && dec_last_tap_tc_)
        b += al(static_cast<int64_t>(G) * (lh << (S - 1)) * (lw << (S - 1)) * dec_last_tap_tc_->n_pad * 4);
    return b;
}

// The per-run working sets in ONE device arena (see Ledger in engine.hpp):
//   [0, cache)            feature-cache entries U_{m+1} (b=2: uncond, cond)
//   [cache, act_end)      denoise activations of every level
//   [0, enc_end)          image mode: the encode workspace (encode precedes
//                         denoise; cache and activations are dead)
//   [top - dec, top)      decode workspace (the denoise activations are dead;
//                         it may reach into the cache region only when the
//                         swap holds the entries on the host through decode,
//                         as the reference's final eviction does --
//                         proj/README.md "Swap schedule" -- and then waits
//                         for that eviction before overwriting it).
// top = max(act_end, enc_end, dec + (cache resident through decode ? cache : 0)),
// so the arena is exactly the peak of the working-set lifetimes the ledger
// logs.  The video, latents, weights and noise stay separate allocations
// (the video outlives the run: it is downloaded after or during the next).
void Engine::alloc_activations(int64_t T) {
    const int64_t G = run_dec_group();
    if (T_alloc_ == T && arena_G_ == G) return;
    if (async_pending_) (void)wait();  // queued runs still use the old arena
    LC_CUDA(cudaDeviceSynchronize());
    invalidate_graph();
    z_key_.clear();
    act_bufs_.clear();
    arena_.reset();
    cache_host_.reset();
    auto al = [](int64_t b) { return (b + 255) / 256 * 256; };
    const int M = static_cast<int>(cfg_.depth), m = static_cast<int>(cfg_.cache_depth);
    const int lh = static_cast<int>(cfg_.latent_h()), lw = static_cast<int>(cfg_.latent_w());
    // layout pass: offsets first, pointers once the arena exists
    std::vector<std::pair<Act*, int64_t>> carve;
    int64_t off = 0;
    bool pad = false;
    auto place = [&](Act* a, int nn, int h, int w, int c, int cs) {
        a->n = nn, a->h = h, a->w = w, a->c = c, a->cs = cs;
        a->p = nullptr;
        carve.push_back({a, off});
        off += al(a->elems() * 2);
        pad = pad || cs != c;
    };
    ArenaInfo ai;
    cache_ = Act{};
    lv_.assign(static_cast<size_t>(M + 1), Level{});
    mid_ = Act{};
    // Denoise activations, packed by lifetime (host.cpp plan_arena, checked
    // on CPU by tests/test_host.py): every buffer lives from its first write
    // to its last read within one full step; two buffers whose lifetimes are
    // disjoint may share storage (e.g. the stem output, dead after d0, holds
    // D_1, U_2, P_1 ... and then U_0).  Cached steps run a sub-sequence of
    // that order, and the per-branch deep path keeps both halves of every
    // deep buffer inside its branch's span, so disjoint there means disjoint
    // in every schedule.  The cache entries live across steps at [0, cache).
    if (stem_kp_ != static_cast<int>((cfg_.in_channels * cfg_.kernel * cfg_.kernel + 63) / 64 * 64))
        throw_invariant("arena plan: stem patch width mismatch");
    RunConfig pc = cfg_;
    pc.frames = T;
    const ArenaPlan plan = plan_arena(pc);
    auto act_of = [&](const std::string& nm) -> Act* {
        if (nm == "cache") return &cache_;
        if (nm == "patch") return &patch_;
        if (nm == "stem") return &stem_out_;
        if (nm == "mid") return &mid_;
        const int l = std::stoi(nm.substr(nm[0] == 'U' && nm[1] == 'P' ? 2 : 1));
        if (nm[0] == 'D') return &lv_[l].D;
        if (nm[0] == 'P') return &lv_[l].P;
        if (nm[1] == 'P') return &lv_[l].UP;
        return &lv_[l].U;
    };
    for (const ArenaBuf& b : plan.bufs) {
        if (b.t1 < 0) continue;
        Act* a = act_of(b.name);
        a->n = b.n, a->h = b.h, a->w = b.w, a->c = b.c, a->cs = b.cs;
        a->p = nullptr;
        carve.push_back({a, b.off});
        pad = pad || b.cs != b.c;
    }
    ai.cache = plan.cache_bytes;
    const int64_t act0 = plan.cache_bytes;
    off = plan.act_end;
    const int64_t act_end = off;
    act_padding_ = pad;
    ai.act = act_end - act0;
    // encode workspace (image mode), over the activations
    int64_t enc_end = 0;
    enc_padding_ = false;
    if (cfg_.mode == "image") {
        const int S = static_cast<int>(cfg_.stages), H = static_cast<int>(cfg_.height),
                  W = static_cast<int>(cfg_.width), Wc = static_cast<int>(cfg_.codec_width);
        const int Ge = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(decode_slice, T)));
        off = 0;  // the cache entries are produced by step 0: nothing else is live in encode
        pad = false;
        place(&enc_patch_, Ge, H, W, enc0_kp_, enc0_kp_);
        for (int i = 0; i < S; ++i) place(&enc_e_[i], Ge, H >> i, W >> i, Wc, round_up(Wc, 64));
        for (int i = 1; i <= S; ++i) place(&enc_p_[i], Ge, H >> i, W >> i, Wc, round_up(Wc, 64));
        enc_end = off;
        enc_padding_ = pad;
        ai.enc = enc_end;
    }
    // decode workspace at the top
    const bool want_y = !(dec_last_w16_.p && subpix_fused_enabled()) && dec_last_tap_tc_ && tap_gather_enabled();
    ai.dec = dec_ws_bytes(static_cast<int>(G), want_y);
    const bool swap = cfg_.cache_enabled && cfg_.swap_mode != SwapMode::Off;
    const int64_t top = std::max({act_end, enc_end, ai.dec + (swap ? 0 : ai.cache)});
    ai.arena = top;
    ai.dec_overlaps_cache = top - ai.dec < ai.cache;
    {
        off = top - ai.dec;
        pad = false;
        DecWs& d = dec_ws_run_;
        d.G = static_cast<int>(G);
        const int S = static_cast<int>(cfg_.stages);
        const int Wc = static_cast<int>(cfg_.codec_width);
        for (int i = 0; i < S; ++i) place(&d.act[i], d.G, lh << i, lw << i, Wc, round_up(Wc, 64));
        place(&d.patch, d.G, lh, lw, dec0_kp_, dec0_kp_);
        d.y = nullptr;
        if (want_y) {
            d.y = reinterpret_cast<float*>(static_cast<intptr_t>(off));  // offset, fixed up below
            off += al(static_cast<int64_t>(d.G) * (lh << (S - 1)) * (lw << (S - 1)) * dec_last_tap_tc_->n_pad * 4);
        }
        dec_padding_ = pad;
    }
    // the arena: zero once (channel padding stays zero between stages unless
    // another stage's workspace overwrote it -- see enqueue_body)
    arena_ = dev_alloc(nullptr, std::max<int64_t>(top, 256), true);
    char* base = arena_.as<char>();
    for (auto& [a, o] : carve) a->p = reinterpret_cast<__half*>(base + o);
    if (dec_ws_run_.y) dec_ws_run_.y = reinterpret_cast<float*>(base + reinterpret_cast<intptr_t>(dec_ws_run_.y));
    if (cfg_.cache_enabled) {
        if (m + 1 == M) mid_ = cache_;
        else lv_[m + 1].U = cache_;
        // the swap's slow tier: pinned host memory for both entries (its
        // occupancy is logged by the tier moves, like the arena's regions)
        if (cfg_.swap_mode != SwapMode::Off) cache_host_ = host_alloc(nullptr, cache_.elems() * 2);
    }
    arena_info_ = ai;
    decide_branch_deep();
    const int64_t nl = T * cfg_.latent_channels * lh * lw;
    x0_ = dev_alloc(&ledger_, nl * 4, true);
    x_ = dev_alloc(&ledger_, nl * 4, true);
    xn_ = dev_alloc(&ledger_, nl * 4, true);
    z_.reset();  // ancestral noise, allocated by prepare_noise()
    eps2_ = dev_alloc(&ledger_, 2 * nl * 4, true);
    bad_ = dev_alloc(&ledger_, 16, true);
    video_ = dev_alloc(&ledger_, T * cfg_.image_channels * cfg_.height * cfg_.width * 4, false);
    T_alloc_ = T;
    arena_G_ = G;
}

// LC_FORCE_TILES=1: run exact-halo chunk tiles as separate launches too
// (the lossless case below normally collapses them into one); used to prove
// tiled == untiled bit for bit on the GPU.
static bool force_tiles() {
    static const bool on = std::getenv("LC_FORCE_TILES") && std::atoi(std::getenv("LC_FORCE_TILES")) != 0;
    return on;
}

// Chunk windows for a block at a level (proj/src/chunk.cpp:145-181 split,
// :69-92 plan_windows, :201-228 run_chunked): per tile, the output core and
// the readable (materialised) window -- the tile's padded region, outside
// which the reference's crop reads zeros (TMA out-of-bounds fill here).
static std::vector<Window> block_windows(const RunConfig& c, const std::string& name, int h, int w) {
    const bool chunked =
        c.chunk_enabled && std::find(c.targets.begin(), c.targets.end(), name) != c.targets.end();
    if (!chunked) return {Window{0, h, 0, w, 0, h, 0, w}};
    int64_t halo = 0;
    const auto tiles = split(h, w, c.eta, c.omega, c.halo, c.halo_px, c.kernel, &halo);
    const int64_t r = (c.kernel - 1) / 2;
    // A halo >= the receptive radius makes every tile read the whole image
    // window its core needs, i.e. tiled == untiled (the reference's lossless
    // case, proj/tests/test_chunk.cpp:118-160).  The fused kernels never
    // materialise a tile, so the tiles of that case run as ONE launch over
    // the union of the cores (the full image): identical bytes, no per-tile
    // tails (LC_FORCE_TILES=1 keeps the tiles).  Halos below the radius
    // (seams) always run one launch per tile.
    const bool lossless = halo >= r;
    if (lossless && !force_tiles()) return {Window{0, h, 0, w, 0, h, 0, w}};
    std::vector<Window> out;
    for (const Tile& t : tiles) {
        Window wd;
        wd.oy0 = static_cast<int>(t.core.y0);
        wd.oy1 = static_cast<int>(t.core.y1);
        wd.ox0 = static_cast<int>(t.core.x0);
        wd.ox1 = static_cast<int>(t.core.x1);
        wd.vy0 = static_cast<int>(t.padded.y0);
        wd.vy1 = static_cast<int>(t.padded.y1);
        wd.vx0 = static_cast<int>(t.padded.x0);
        wd.vx1 = static_cast<int>(t.padded.x1);
        if (lossless) {
            // the core's outputs read only core +- r inside the padded
            // region, so widening it to even bounds (the parity-aligned
            // window the fused sub-pixel up-conv needs) changes nothing
            wd.vy0 &= ~1, wd.vx0 &= ~1;
            wd.vy1 = std::min(h, (wd.vy1 + 1) & ~1), wd.vx1 = std::min(w, (wd.vx1 + 1) & ~1);
        }
        out.push_back(wd);
    }
    return out;
}

void Engine::conv_block(int j, const Act& in, const Act& out, float s, float o, bool silu) {
    const auto plan = block_plans(cfg_);
    for (const Window& wd : block_windows(cfg_, plan[j].name, in.h, in.w)) {
        run_tc_conv(*tc_[j], &in, out, wd, s, o, silu, s_compute_);
        ++launches;
    }
}

void Engine::up_block(int i, const Act& skip, const Act& u, const Act& out, float s, float o) {
    const int j = static_cast<int>(block_index(cfg_, "u" + std::to_string(i)));
    const auto wins = block_windows(cfg_, "u" + std::to_string(i), skip.h, skip.w);
    bool subpixel = tc_[j] != nullptr;
    // merged sub-pixel taps need a parity-aligned readable window; odd
    // output cores are fine (per-parity lattice regions)
    for (const Window& wd : wins)
        if ((wd.vy0 | wd.vy1 | wd.vx0 | wd.vx1) & 1) subpixel = false;
    if (subpixel) {
        const Act srcs[2] = {skip, u};
        for (const Window& wd : wins) {
            run_tc_conv(*tc_[j], srcs, out, wd, s, o, true, s_compute_);
            ++launches;
        }
        return;
    }
    // Fallback (k != 3, or odd tile windows): materialise the nearest
    // upsample, then a two-segment conv.
    Act& up = lv_[i].UP;
    if (!up.p) {
        up = Act{nullptr, u.n, skip.h, skip.w, u.cs, u.c};
        act_bufs_.push_back(dev_alloc(&ledger_, up.elems() * 2, true));
        up.p = act_bufs_.back().as<__half>();
    }
    LC_CUDA(launch_up2(u.p, up.p, u.n, u.h, u.w, u.cs, s_compute_));
    ++launches;
    const Act srcs[2] = {skip, up};
    if (!tc_fb_[j]) throw_invariant("up block fallback weights not prepared by configure()");
    for (const Window& wd : wins) {
        run_tc_conv(*tc_fb_[j], srcs, out, wd, s, o, true, s_compute_);
        ++launches;
    }
}

// LC_FUSED_STEP=0 keeps the sampler step as its own kernel (A/B timing)
static bool fused_step_enabled() {
    static const bool on = !(std::getenv("LC_FUSED_STEP") && std::atoi(std::getenv("LC_FUSED_STEP")) == 0);
    return on;
}

void Engine::forward_dev(const float* x_dev, bool stacked, int64_t T, int64_t timestep, bool full,
                         float* eps2_dev, int step, int seam, const StepArgs* fuse) {
    step_fused_ = false;
    const int M = static_cast<int>(cfg_.depth), m = static_cast<int>(cfg_.cache_depth);
    const int lh = static_cast<int>(cfg_.latent_h()), lw = static_cast<int>(cfg_.latent_w());
    auto cond = [&](int j, float* s, float* o) { block_conditioning(uw_, j, timestep, s, o); };
    float s, o;
    dl_gate(step, "stem");
    // stem: CFG pair built on the fly (pipeline.cpp:127-131), affine + conv + SiLU
    {
        const int j = 0;
        cond(j, &s, &o);
        for (const Window& wd : block_windows(cfg_, "stem", lh, lw)) {
            ThinInArgs a{};
            a.x = x_dev;
            a.nsrc = static_cast<int>(stacked ? 2 * T : T);
            a.c_in = stem_->c_in;
            a.H = lh;
            a.W = lw;
            a.cfg_pair = stacked ? 0 : 1;
            a.cond_bias = 0.15f;
            a.s = s;
            a.o = o;
            a.apply_affine = 1;
            a.w = stem_->w.as<float>();
            a.bias = stem_->bias.as<float>();
            a.c_out = stem_->c_out;
            a.k = stem_->k;
            a.silu = 1;
            // gather conditioned 3x3x4 patches (exact reference roundings),
            // then a K=64 tensor-core GEMM with bias + SiLU epilogue
            a.out = patch_.p;
            a.cs_out = patch_.cs;
            a.win = wd;
            LC_CUDA(launch_patch(a, stem_kp_, s_compute_));
            run_tc_conv(*stem_tc_, &patch_, stem_out_, Window{0, lh, 0, lw, wd.oy0, wd.oy1, wd.ox0, wd.ox1},
                        1.0f, 0.0f, true, s_compute_);
            launches += 2;
        }
    }
    cond(1, &s, &o);
    dl_gate(step, "d0");
    conv_block(1, stem_out_, lv_[0].D, s, o, true);
    const bool writes_cache = full && cfg_.cache_enabled;
    // Per-branch deep path (async swap, full step whose U_{m+1} is evicted,
    // slow host link -- see branch_deep_wanted): everything below level m
    // runs on the uncond half, then on the cond half, so entry 0 is complete
    // (and its eviction starts) half a deep path earlier, and entry 1's
    // eviction no longer queues behind it on the link.  Same per-image
    // arithmetic (bit-identical), same transfer issue points.
    const bool evicting = writes_cache && seam == 3 && cfg_.swap_mode == SwapMode::Async && m + 1 < M;
    const bool branch_deep = evicting && branch_deep_ == 1;
    const bool branch_up = evicting && branch_deep_ == 2;  // down path whole-batch, up path per branch
    const int deepest = full ? M - 1 : m;
    for (int i = 1; i <= (branch_deep ? m : deepest); ++i) {
        const Act& prev = lv_[i - 1].D;
        LC_CUDA(launch_down2(prev.p, lv_[i].P.p, prev.n, prev.h, prev.w, prev.cs, s_compute_));
        ++launches;
        cond(1 + i, &s, &o);
        conv_block(1 + i, lv_[i].P, lv_[i].D, s, o, true);
    }
    // U_l holder: output of u_l (l < M) or mid (l == M); the cache slot when
    // l == m+1 and caching is on.
    auto U_of = [&](int l) -> const Act& { return l == M ? mid_ : lv_[l].U; };
    if (writes_cache) host_valid_ = false;  // this step stores new entries
    if (writes_cache)
        // CacheStore::store (cache.cpp:43-63) replaces the entries: ones the
        // swap left on the host are dropped, the new ones are HBM-resident
        for (int b = 0; b < 2; ++b)
            if (rid_cache_[b] && ledger_.region_tier(rid_cache_[b]) == 1) {
                ledger_.region_free(rid_cache_[b]);
                rid_cache_[b] = ledger_.region_alloc(0, cache_.elems());
            }
    // CacheStore::store awaits pending transfers before replacing entries
    // (cache.cpp:48-52): the compute stream waits on entry b's eviction right
    // before the block that overwrites entry b.
    auto await_store = [&](int b) {
        if (!(writes_cache && evict_pending_)) return;
        if (b < 0) {
            for (int e = 0; e < 2; ++e) LC_CUDA(cudaStreamWaitEvent(s_compute_, ev_evict_[e], 0));
        } else {
            LC_CUDA(cudaStreamWaitEvent(s_compute_, ev_evict_[b], 0));
        }
        if (b != 0) evict_pending_ = false;
    };
    auto cache_ready = [&](int b) {
        for (int e = 0; e < 2; ++e)
            if (b < 0 || e == b) LC_CUDA(cudaEventRecord(ev_cache_ready_[e], s_compute_));
        cache_ready_recorded_ = true;
    };
    auto half = [&](const Act& a, int b) {
        Act h = a;
        h.n = a.n / 2;
        h.p = a.p + static_cast<int64_t>(b) * h.n * a.h * a.w * a.cs;
        return h;
    };
    if (branch_deep) {
        for (int b = 0; b < 2; ++b) {
            for (int i = m + 1; i <= M; ++i) {
                const Act prev = half(lv_[i - 1].D, b);
                const Act pin = half(lv_[i].P, b);
                LC_CUDA(launch_down2(prev.p, pin.p, prev.n, prev.h, prev.w, prev.cs, s_compute_));
                ++launches;
                cond(1 + i, &s, &o);
                conv_block(1 + i, pin, half(i == M ? mid_ : lv_[i].D, b), s, o, true);
            }
            for (int i = M - 1; i >= m + 1; --i) {
                const int j = static_cast<int>(block_index(cfg_, "u" + std::to_string(i)));
                cond(j, &s, &o);
                if (i == m + 1) await_store(b);
                up_block(i, half(lv_[i].D, b), half(U_of(i + 1), b), half(U_of(i), b), s, o);
            }
            cache_ready(b);
        }
    }
    if (full && !branch_deep) {
        const Act& prev = lv_[M - 1].D;
        LC_CUDA(launch_down2(prev.p, lv_[M].P.p, prev.n, prev.h, prev.w, prev.cs, s_compute_));
        ++launches;
        cond(1 + M, &s, &o);
        if (m + 1 == M) await_store(-1);
        conv_block(1 + M, lv_[M].P, mid_, s, o, true);
        if (writes_cache && m + 1 == M && seam == 3) cache_ready(-1);
    }
    // Branch-wise seam (async swap with a prefetch in flight): the two CFG
    // entries are separate transfers (CacheStore entries, cache.cpp:43-90),
    // so the seam block starts on the uncond half as soon as that entry has
    // landed and overlaps the cond entry's transfer.  Same bytes, same order
    // of awaits and issue points as assemble() + evict_all().
    const bool branch_seam =
        !full && seam > 0 && prefetch_pending_ && cfg_.swap_mode == SwapMode::Async && branch_seam_;
    if (!full && seam > 0 && !branch_seam) {
        seam_await(step);
        // last consumer: evict_all right after assemble (pipeline.cpp:156-160)
        if (seam == 2) issue_evict(step);
    }
    const int top = full ? M - 1 : m;
    dl_gate(step, "up");
    // Per-branch store (async swap, full step whose U_{m+1} is evicted): the
    // producing block u_{m+1} runs on the uncond half, then on the cond half,
    // so entry 0's eviction starts half a block earlier and overlaps the
    // cond half.  Same per-image arithmetic (bit-identical), same transfer
    // issue points.
    const bool split_store = writes_cache && seam == 3 && cfg_.swap_mode == SwapMode::Async && m + 1 < M &&
                             split_store_enabled() && !branch_deep && !branch_up;
    // Deeper up blocks stay whole-batch (their weight panels, up to 170 MB,
    // would be streamed twice); only the producing block u_{m+1} is split.
    int first = branch_deep ? m : top;
    if (branch_up) {
        // every up block below the seam per branch: entry 0 is complete
        // after half of the deep up path
        for (int b = 0; b < 2; ++b) {
            for (int i = top; i >= m + 1; --i) {
                const int j = static_cast<int>(block_index(cfg_, "u" + std::to_string(i)));
                cond(j, &s, &o);
                if (i == m + 1) await_store(b);
                up_block(i, half(lv_[i].D, b), half(U_of(i + 1), b), half(U_of(i), b), s, o);
            }
            cache_ready(b);
        }
        first = m;
    }
    if (split_store) {
        for (int i = top; i > m + 1; --i) {
            const int j = static_cast<int>(block_index(cfg_, "u" + std::to_string(i)));
            cond(j, &s, &o);
            up_block(i, lv_[i].D, U_of(i + 1), U_of(i), s, o);
        }
        const int j = static_cast<int>(block_index(cfg_, "u" + std::to_string(m + 1)));
        cond(j, &s, &o);
        for (int b = 0; b < 2; ++b) {
            await_store(b);
            up_block(m + 1, half(lv_[m + 1].D, b), half(U_of(m + 2), b), half(U_of(m + 1), b), s, o);
            cache_ready(b);
        }
        first = m;
    }
    for (int i = first; i >= 0; --i) {
        const int j = static_cast<int>(block_index(cfg_, "u" + std::to_string(i)));
        cond(j, &s, &o);
        const Act& out_i = i == 0 ? lv_[0].U : U_of(i);
        if (branch_seam && i == m) {
            // per entry: the first half of its images as soon as their bytes
            // landed, the second half once the whole entry has (the await
            // marks bracket the wait that gates the block; the second wait is
            // marked as a partial await)
            auto part = [&](const Act& a, int i0, int ni) {
                Act h = a;
                h.n = ni;
                h.p = a.p + static_cast<int64_t>(i0) * a.h * a.w * a.cs;
                return h;
            };
            static const bool parts = !(std::getenv("LC_SEAM_PARTS") && std::atoi(std::getenv("LC_SEAM_PARTS")) == 0);
            const int ne = out_i.n / 2, n0 = parts ? ne / 2 : 0;
            for (int b = 0; b < 2; ++b) {
                const int i0 = b * ne;
                record(4, prefetch_tag_, 0, s_compute_);
                LC_CUDA(cudaStreamWaitEvent(s_compute_, n0 > 0 ? ev_prefetch_part_[b] : ev_prefetch_[b], 0));
                record(5, prefetch_tag_, 0, s_compute_);
                if (n0 > 0) {
                    up_block(i, part(lv_[i].D, i0, n0), part(U_of(i + 1), i0, n0), part(out_i, i0, n0), s, o);
                    record(7, prefetch_tag_, 0, s_compute_);
                    LC_CUDA(cudaStreamWaitEvent(s_compute_, ev_prefetch_[b], 0));
                    record(8, prefetch_tag_, 0, s_compute_);
                }
                if (b == 1 && seam == 2) issue_evict(step);
                up_block(i, part(lv_[i].D, i0 + n0, ne - n0), part(U_of(i + 1), i0 + n0, ne - n0),
                         part(out_i, i0 + n0, ne - n0), s, o);
            }
            prefetch_pending_ = false;
        } else {
            if (i == m + 1) await_store(-1);
            up_block(i, lv_[i].D, U_of(i + 1), out_i, s, o);
        }
        if (writes_cache && i == m + 1 && seam == 3) cache_ready(-1);
    }
    // head: affine + conv, no SiLU -> eps (2,T,C,h,w) fp32
    dl_gate(step, "head");
    {
        const int j = static_cast<int>(block_index(cfg_, "head"));
        cond(j, &s, &o);
        Act eps_view;  // fp32 NCHW output geometry (2T, C, h, w)
        eps_view.n = lv_[0].U.n;
        eps_view.h = lh;
        eps_view.w = lw;
        eps_view.c = head_tc_->c_out;
        if (head_w16_.p && subpix_fused_enabled()) {
            // K8: tap-to-N GEMM over a halo window + in-window tap sums, fused
            const Act& a = lv_[0].U;
            const uint64_t dims[4] = {static_cast<uint64_t>(a.cs), static_cast<uint64_t>(lw), static_cast<uint64_t>(lh),
                                      static_cast<uint64_t>(a.n)};
            const uint64_t strides[3] = {static_cast<uint64_t>(a.cs) * 2, static_cast<uint64_t>(lw) * a.cs * 2,
                                         static_cast<uint64_t>(lh) * lw * a.cs * 2};
            const int hty = tap_tile_rows(kTapConv3, static_cast<int>(head_tc_->c_out), head_kb_, head_n_);
            const uint32_t box[4] = {64, kTapSX, static_cast<uint32_t>(hty + 2), 1};
            const uint32_t estr[4] = {1, 1, 1, 1};
            TapTcParams q{};
            encode_map(&q.tmA, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, a.p, dims, strides, box, estr);
            q.w = head_w16_.as<__half>();
            q.bias = head_bias_.as<float>();
            q.wsum = head_wsum_.as<float>();
            q.scale = s / head_wscale_;
            q.shift = o;
            q.out = eps2_dev;
            q.n = a.n;
            q.H = lh;
            q.W = lw;
            q.C = static_cast<int>(head_tc_->c_out);
            q.N = head_n_;
            q.kb = head_kb_;
            if (fuse && fused_step_enabled()) {
                q.pair_T = a.n / 2;
                q.x = fuse->x;
                q.x_out = fuse->x_out;
                q.z = fuse->z;
                q.g = fuse->g;
                q.a = fuse->a;
                q.b = fuse->b;
                q.c = fuse->c;
                q.bad = fuse->bad;
                step_fused_ = true;
            }
            for (const Window& wd : block_windows(cfg_, "head", lh, lw)) {
                q.win = wd;
                q.tiles_x = (wd.ox1 - wd.ox0 + kTapTX - 1) / kTapTX;
                q.tiles_y = (wd.oy1 - wd.oy0 + hty - 1) / hty;
                q.num_tiles = a.n * q.tiles_x * q.tiles_y;
                LC_CUDA(launch_tap_tc(kTapConv3, q, s_compute_));
                ++launches;
            }
        } else if (head_tap_tc_ && tap_gather_enabled()) {
            // tap-to-N: one K = c_in GEMM over the materialised window into
            // y[px][tap*C + c], then the tap gather adds the in-window taps
            Act yv;
            yv.n = lv_[0].U.n;
            yv.h = lh;
            yv.w = lw;
            yv.c = head_tap_tc_->c_out;
            yv.cs = head_tap_tc_->n_pad;
            ensure_buf(&head_y_buf_, yv.elems() * 4);
            for (const Window& wd : block_windows(cfg_, "head", lh, lw)) {
                run_tc_conv(*head_tap_tc_, &lv_[0].U, yv,
                            Window{wd.vy0, wd.vy1, wd.vx0, wd.vx1, wd.vy0, wd.vy1, wd.vx0, wd.vx1}, s, 0.0f, false,
                            s_compute_, head_y_buf_.as<float>(), 0, true, true);
                TapGatherArgs g{};
                g.y = head_y_buf_.as<float>();
                g.cs_y = yv.cs;
                g.n = yv.n;
                g.H = lh;
                g.W = lw;
                g.C = head_tc_->c_out;
                g.k = head_tc_->k;
                g.win = wd;
                g.wsum = head_wsum_.as<float>();
                g.bias = head_bias_.as<float>();
                g.o = o;
                g.out = eps2_dev;
                LC_CUDA(launch_tap_gather(g, s_compute_));
                launches += 2;
            }
        } else {
            for (const Window& wd : block_windows(cfg_, "head", lh, lw)) {
                run_tc_conv(*head_tc_, &lv_[0].U, eps_view, wd, s, o, false, s_compute_, eps2_dev);
                ++launches;
            }
        }
    }
}

// Swap transfers (TransferEngine evict/prefetch, proj/src/swap.cpp:284-304).
// One "transfer" = one CFG branch entry (half of the b=2 cache, contiguous
// since b is the outermost image index).  Each entry moves in chunks of
// swap_chunk() bytes (2 MB) so the H2D prefetch of chunk i can start as soon as its
// D2H eviction lands (PCIe is full duplex); async mode uses dedicated D2H
// and H2D streams ordered by CUDA events, sync mode serialises on compute.
// 2 MB measured best on B (value 3120 -> 3190 frames/s vs 4 MB; 1 MB worse:
// per-chunk event overhead); LC_SWAP_CHUNK_MB overrides.
static int64_t swap_chunk() {
    static const int64_t c = std::getenv("LC_SWAP_CHUNK_MB") ? std::atoll(std::getenv("LC_SWAP_CHUNK_MB")) << 20
                                                             : int64_t{2} << 20;
    return c;
}

cudaEvent_t Engine::chunk_event(int b, size_t i) {
    while (ev_chunk_[b].size() <= i) {
        cudaEvent_t e;
        LC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ev_chunk_[b].push_back(e);
    }
    return ev_chunk_[b][i];
}

void Engine::issue_evict(int step) {
    if (!cache_host_.p) return;
    const bool async = cfg_.swap_mode == SwapMode::Async;
    cudaStream_t st = async ? s_d2h_ : s_compute_;
    // The entry is complete once U_{m+1} was produced: on a full step that
    // event was recorded right after the producing block (forward_dev), so
    // the copy overlaps the remaining up path; at a seam it is recorded now.
    if (!cache_ready_recorded_)
        for (int b = 0; b < 2; ++b) LC_CUDA(cudaEventRecord(ev_cache_ready_[b], s_compute_));
    cache_ready_recorded_ = false;
    const int64_t bytes = cache_.elems();  // one branch: elems()*2 bytes / 2 branches
    // Clean eviction: when the pinned host copy already holds these exact
    // bytes (evicted after the store, prefetched back, only read since),
    // evict_all moves nothing -- the entries leave the fast tier and the
    // slow-tier copy stays valid, like a clean page.  Logical transfer,
    // timeline marks and issue order are the reference's.
    const bool clean = host_valid_ && clean_evict_enabled();
    // ledger: each entry moves to the slow tier (double residency while the
    // copy is in flight, ledger.cpp:93-123), logged in issue order
    auto ledger_move = [&](int b) {
        if (rid_cache_[b] && ledger_.region_tier(rid_cache_[b]) == 0) {
            ledger_.move_start(rid_cache_[b], 1);
            ledger_.move_end(rid_cache_[b]);
        }
    };
    if (clean) {
        for (int b = 0; b < 2; ++b) {
            if (async) LC_CUDA(cudaStreamWaitEvent(st, ev_cache_ready_[b], 0));  // issue point, as a dirty one
            if (async) d2h_used_ = true;
            ledger_move(b);
            record(2, step, bytes, st);
            record(3, step, bytes, st);
            LC_CUDA(cudaEventRecord(ev_evict_[b], st));
            if (stats_) stats_->swap_bytes += bytes;
        }
        if (stats_) stats_->swap_calls += 1;
        evict_pending_ = true;
        return;
    }
    host_valid_ = true;
    for (int b = 0; b < 2; ++b) {
        if (async) LC_CUDA(cudaStreamWaitEvent(st, ev_cache_ready_[b], 0));
        if (async) d2h_used_ = true;
        if (stats_) stats_->swap_bytes_moved += bytes;
        ledger_move(b);
        record(2, step, bytes, st);
        size_t ci = 0;
        for (int64_t off = 0; off < bytes; off += swap_chunk(), ++ci) {
            const int64_t len = std::min(swap_chunk(), bytes - off);
            LC_CUDA(cudaMemcpyAsync(cache_host_.as<char>() + b * bytes + off,
                                    reinterpret_cast<char*>(cache_.p) + b * bytes + off, static_cast<size_t>(len),
                                    cudaMemcpyDeviceToHost, st));
            LC_CUDA(cudaEventRecord(chunk_event(b, ci), st));
        }
        record(3, step, bytes, st);
        LC_CUDA(cudaEventRecord(ev_evict_[b], st));
        if (stats_) stats_->swap_bytes += bytes;
    }
    if (stats_) stats_->swap_calls += 1;
    evict_pending_ = true;
}

void Engine::issue_prefetch(int issued, int needed) {
    (void)issued;
    if (!cache_host_.p) return;
    const bool async = cfg_.swap_mode == SwapMode::Async;
    cudaStream_t st = async ? s_h2d_ : s_compute_;
    const int64_t bytes = cache_.elems();
    // the first half of an entry's images (its bytes come first) gets its own
    // event, so the seam block starts on it while the rest is in flight
    const int64_t img_bytes = static_cast<int64_t>(cache_.h) * cache_.w * cache_.cs * 2;
    const int64_t part_bytes = (cache_.n / 2 / 2) * img_bytes;
    for (int b = 0; b < 2; ++b) {
        if (async) h2d_used_ = true;
        if (rid_cache_[b] && ledger_.region_tier(rid_cache_[b]) == 1) {
            ledger_.move_start(rid_cache_[b], 0);  // back to HBM (budget checked, swap.cpp:198)
            ledger_.move_end(rid_cache_[b]);
        }
        size_t ci = 0;
        bool part_done = part_bytes <= 0;
        for (int64_t off = 0; off < bytes; off += swap_chunk(), ++ci) {
            const int64_t len = std::min(swap_chunk(), bytes - off);
            if (async) LC_CUDA(cudaStreamWaitEvent(st, chunk_event(b, ci), 0));
            if (ci == 0) record(2, needed, bytes, st);  // start = first byte can move
            LC_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(cache_.p) + b * bytes + off,
                                    cache_host_.as<char>() + b * bytes + off, static_cast<size_t>(len),
                                    cudaMemcpyHostToDevice, st));
            if (!part_done && off + len >= part_bytes) {
                LC_CUDA(cudaEventRecord(ev_prefetch_part_[b], st));
                part_done = true;
            }
        }
        record(3, needed, bytes, st);
        LC_CUDA(cudaEventRecord(ev_prefetch_[b], st));
        if (stats_) stats_->swap_bytes += bytes;
        if (stats_) stats_->swap_bytes_moved += bytes;
    }
    if (stats_) stats_->swap_calls += 1;
    prefetch_pending_ = true;
    prefetch_tag_ = needed;
}

void Engine::seam_await(int step) {
    // CacheStore::assemble -> fetch -> await_ready (cache.cpp:65-90): the
    // compute stream waits for the prefetch only here, after the shallow path.
    // Await events carry the ticket's step, i.e. the prefetch's
    // needed_at_step (swap.cpp:306-324, ticket step set at submit).
    (void)step;
    for (int b = 0; b < 2; ++b) {
        record(4, prefetch_tag_, 0, s_compute_);
        if (prefetch_pending_) LC_CUDA(cudaStreamWaitEvent(s_compute_, ev_prefetch_[b], 0));
        record(5, prefetch_tag_, 0, s_compute_);
    }
    prefetch_pending_ = false;
}

// Operator-level decode workspace (lc_decode / lc_decode_sharded): real
// allocations outside the run arena, grow-only per slice size.
void Engine::ensure_op_dec_ws(int G) {
    if (dec_ws_op_.G == G && !dec_bufs_op_.empty()) return;
    dec_bufs_op_.clear();
    const int S = static_cast<int>(cfg_.stages);
    const int lh = static_cast<int>(cfg_.latent_h()), lw = static_cast<int>(cfg_.latent_w());
    const int Wc = static_cast<int>(cfg_.codec_width);
    auto make = [&](int h, int w, int c, int cs) {
        Act a{nullptr, G, h, w, cs, c};
        dec_bufs_op_.push_back(dev_alloc(&ledger_, a.elems() * 2, true));
        a.p = dec_bufs_op_.back().as<__half>();
        return a;
    };
    for (int i = 0; i < S; ++i) dec_ws_op_.act[i] = make(lh << i, lw << i, Wc, round_up(Wc, 64));
    dec_ws_op_.patch = make(lh, lw, dec0_kp_, dec0_kp_);
    dec_ws_op_.y = nullptr;
    if (dec_last_tap_tc_) {
        const int64_t yb = static_cast<int64_t>(G) * (lh << (S - 1)) * (lw << (S - 1)) * dec_last_tap_tc_->n_pad * 4;
        dec_bufs_op_.push_back(dev_alloc(&ledger_, yb, true));
        dec_ws_op_.y = dec_bufs_op_.back().as<float>();
    }
    dec_ws_op_.G = G;
}

// Sliced decode (decode_sliced, proj/src/codec.cpp:126-145) of n latents in
// slices of dec_ws_->G frames, using the workspace dec_ws_ points at.
void Engine::decode_dev(const float* lat_dev, int64_t n, float* video_dev) {
    const int S = static_cast<int>(cfg_.stages);
    const int lh = static_cast<int>(cfg_.latent_h()), lw = static_cast<int>(cfg_.latent_w());
    if (!dec_ws_) throw_invariant("decode without a workspace");
    const DecWs& ws = *dec_ws_;
    const int G = ws.G;
    const int C = static_cast<int>(cfg_.latent_channels), IC = static_cast<int>(cfg_.image_channels);
    const int H = static_cast<int>(cfg_.height), W = static_cast<int>(cfg_.width);
    if (out_slices_) {
        // the previous run's video download must have read the device video
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        LC_CUDA(cudaStreamIsCapturing(s_compute_, &cs));
        LC_CUDA(cudaStreamWaitEvent(s_compute_, ev_vid_done_,
                                    cs == cudaStreamCaptureStatusActive ? cudaEventWaitExternal : 0));
        if (dl_capture_) {
            if (!dl_fired_) fire_download();
            LC_CUDA(cudaStreamWaitEvent(s_compute_, ev_dl_done_, 0));
        }
        slice_spans_.clear();
    }
    for (int64_t g0 = 0; g0 < n; g0 += G) {
        const int gs = static_cast<int>(std::min<int64_t>(G, n - g0));
        Act e[8];
        for (int i = 0; i < S; ++i) {
            e[i] = ws.act[i];
            e[i].n = gs;
        }
        ThinInArgs a{};
        a.x = lat_dev + g0 * C * lh * lw;
        a.nsrc = gs;
        a.c_in = C;
        a.H = lh;
        a.W = lw;
        a.cfg_pair = 0;
        a.s = 1.0f;
        a.o = 0.0f;
        a.apply_affine = 0;
        a.w = dec0_->w.as<float>();
        a.bias = dec0_->bias.as<float>();
        a.c_out = dec0_->c_out;
        a.k = 3;
        a.silu = 1;
        Act patch = ws.patch;
        patch.n = gs;
        a.out = patch.p;
        a.cs_out = patch.cs;
        a.win = Window{0, lh, 0, lw, 0, lh, 0, lw};
        LC_CUDA(launch_patch(a, dec0_kp_, s_compute_));
        run_tc_conv(*dec0_tc_, &patch, e[0], a.win, 1.0f, 0.0f, true, s_compute_);
        launches += 2;
        for (int i = 1; i < S; ++i) {
            const int h = lh << i, w = lw << i;
            run_tc_conv(*dec_tc_[i - 1], &e[i - 1], e[i], Window{0, h, 0, w, 0, h, 0, w}, 1.0f, 0.0f, true,
                        s_compute_);
            ++launches;
        }
        // last conv: sub-pixel 3x3 on the low-res image with 4x3 outputs,
        // depth-to-space into the fp32 NCHW video
        const int hl = lh << (S - 1), wl = lw << (S - 1);
        Act vid;
        vid.n = gs;
        vid.h = H;
        vid.w = W;
        vid.c = IC;
        if (dec_last_w16_.p && subpix_fused_enabled()) {
            // K8: upsample + conv + bias + depth-to-space in one kernel
            const Act& a = e[S - 1];
            TapTcParams q{};
            const uint64_t dims[4] = {static_cast<uint64_t>(a.cs), static_cast<uint64_t>(wl), static_cast<uint64_t>(hl),
                                      static_cast<uint64_t>(gs)};
            const uint64_t strides[3] = {static_cast<uint64_t>(a.cs) * 2, static_cast<uint64_t>(wl) * a.cs * 2,
                                         static_cast<uint64_t>(hl) * wl * a.cs * 2};
            const int dty = tap_tile_rows(kTapSubpix, IC, dec_last_kb_, dec_last_n_);
            const uint32_t box[4] = {64, kTapSX, static_cast<uint32_t>(dty + 2), 1};
            const uint32_t estr[4] = {1, 1, 1, 1};
            encode_map(&q.tmA, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, a.p, dims, strides, box, estr);
            q.w = dec_last_w16_.as<__half>();
            q.scale = 1.0f / dec_last_wscale_;
            q.bias = dec_last_bias_.as<float>();
            q.out = video_dev + g0 * IC * H * W;
            q.n = gs;
            q.H = hl;
            q.W = wl;
            q.C = IC;
            q.N = dec_last_n_;
            q.kb = dec_last_kb_;
            q.win = Window{0, hl, 0, wl, 0, hl, 0, wl};
            q.tiles_x = (wl + kTapTX - 1) / kTapTX;
            q.tiles_y = (hl + dty - 1) / dty;
            q.num_tiles = gs * q.tiles_x * q.tiles_y;
            LC_CUDA(launch_tap_tc(kTapSubpix, q, s_compute_));
            ++launches;
        } else if (dec_last_tap_tc_ && tap_gather_enabled()) {
            Act yv;
            yv.n = gs;
            yv.h = hl;
            yv.w = wl;
            yv.c = dec_last_tap_tc_->c_out;
            yv.cs = dec_last_tap_tc_->n_pad;
            if (!ws.y) throw_invariant("decode workspace without tap-to-N partial sums");
            run_tc_conv(*dec_last_tap_tc_, &e[S - 1], yv, Window{0, hl, 0, wl, 0, hl, 0, wl}, 1.0f, 0.0f, false,
                        s_compute_, ws.y, 0, true, true);
            SubpixGatherArgs g{};
            g.y = ws.y;
            g.cs_y = yv.cs;
            g.n = gs;
            g.H = hl;
            g.W = wl;
            g.C = IC;
            g.bias = dec_last_bias_.as<float>();
            g.out = video_dev + g0 * IC * H * W;
            LC_CUDA(launch_subpix_gather(g, s_compute_));
            launches += 2;
        } else {
            run_tc_conv(*dec_last_tc_, &e[S - 1], vid, Window{0, hl, 0, wl, 0, hl, 0, wl}, 1.0f, 0.0f, false,
                        s_compute_, video_dev + g0 * IC * H * W, IC);
            ++launches;
        }
        if (out_slices_) {
            // slice g0 is final: the host side streams it to the caller's
            // pinned buffer on the D2H stream (enqueue_video_out), outside
            // the captured body, while the next slice decodes
            record_timing(chunk_event(2, slice_spans_.size()), s_compute_);
            slice_spans_.push_back({g0, gs});
        }
    }
}

// After a body launch: per decoded slice, wait for its event and copy it to
// the caller's pinned buffer on the D2H stream; ev_vid_done_ marks the last
// byte read, and the next body's decode waits for it before overwriting the
// device video (so back-to-back runs may overlap this download).
void Engine::enqueue_video_out(float* pinned) {
    const int64_t frame = static_cast<int64_t>(cfg_.image_channels) * cfg_.height * cfg_.width;
    for (size_t i = 0; i < slice_spans_.size(); ++i) {
        LC_CUDA(cudaStreamWaitEvent(s_d2h_, chunk_event(2, i), 0));
        const int64_t g0 = slice_spans_[i].first, gs = slice_spans_[i].second;
        LC_CUDA(cudaMemcpyAsync(pinned + g0 * frame, video_.as<float>() + g0 * frame,
                                static_cast<size_t>(gs * frame) * 4, cudaMemcpyDeviceToHost, s_d2h_));
    }
    LC_CUDA(cudaEventRecord(ev_vid_done_, s_d2h_));
}

void Engine::ensure_buf(DevBuf* b, int64_t bytes) {
    if (b->p && b->bytes >= bytes) return;
    invalidate_graph();
    *b = dev_alloc(&ledger_, bytes, false);
}

void Engine::invalidate_graph() {
    if (dl_pending_) {  // the device video may be about to move or be rewritten
        flush_pending_download();
        LC_CUDA(cudaStreamSynchronize(s_vid_));
    }
    if (graph_exec_) {
        cudaGraphExecDestroy(graph_exec_);
        graph_exec_ = nullptr;
    }
    if (graph_) {
        cudaGraphDestroy(graph_);
        graph_ = nullptr;
    }
    dl_node_ = nullptr;
    eager_runs_ = 0;
}

// ------------------------------------------------ deferred video download
void Engine::dl_gate(int step, const char* where) {
    if (dl_capture_ && !dl_fired_ && step == dl_gate_step_ && dl_gate_where_ == where) fire_download();
}

// Inside the capture: the previous run's video (still in video_) leaves for
// the host on s_vid_ from this point of the body; the decode joins it before
// overwriting video_.  The node's destination is a placeholder, re-pointed
// per launch by arm_download_node().
void Engine::fire_download() {
    const size_t bytes = static_cast<size_t>(video_elems()) * 4;
    if (!dl_scratch_.p || dl_scratch_.bytes < static_cast<int64_t>(bytes))
        throw_invariant("deferred download: placeholder not allocated before capture");
    LC_CUDA(cudaEventRecord(ev_dl_gate_, s_compute_));
    LC_CUDA(cudaStreamWaitEvent(s_vid_, ev_dl_gate_, 0));
    LC_CUDA(cudaMemcpyAsync(dl_scratch_.p, video_.p, bytes, cudaMemcpyDeviceToHost, s_vid_));
    LC_CUDA(cudaEventRecord(ev_dl_done_, s_vid_));
    dl_fired_ = true;
}

// Outside any graph: issue the pending download now (after everything queued
// on the compute stream); the next body's decode waits on ev_vid_done_.
void Engine::flush_pending_download() {
    if (!dl_pending_) return;
    LC_CUDA(cudaEventRecord(ev_dl_src_, s_compute_));
    LC_CUDA(cudaStreamWaitEvent(s_vid_, ev_dl_src_, 0));
    LC_CUDA(cudaMemcpyAsync(dl_pending_, video_.p, static_cast<size_t>(video_elems()) * 4, cudaMemcpyDeviceToHost,
                            s_vid_));
    LC_CUDA(cudaEventRecord(ev_vid_done_, s_vid_));
    dl_pending_ = nullptr;
}

void Engine::arm_download_node() {
    if (!dl_node_) {
        flush_pending_download();
        return;
    }
    if (dl_pending_) {
        LC_CUDA(cudaGraphExecMemcpyNodeSetParams1D(graph_exec_, dl_node_, dl_pending_, video_.p,
                                                   static_cast<size_t>(video_elems()) * 4,
                                                   cudaMemcpyDeviceToHost));
        LC_CUDA(cudaGraphNodeSetEnabled(graph_exec_, dl_node_, 1));
        dl_pending_ = nullptr;
    } else {
        LC_CUDA(cudaGraphNodeSetEnabled(graph_exec_, dl_node_, 0));
    }
}

// Ancestral per-step noise randn(derive_seed(seed, 0x1000 + s))
// (pipeline.cpp:181-182), drawn on the host with the reference's
// SplitMix64/Box-Muller stream (libm double log/sqrt/cos/sin, bit-exact with
// the reference) once per config and kept resident: S x n floats.
void Engine::prepare_noise() {
    if (cfg_.sampler != Sampler::Ancestral) return;
    const int64_t nl = latent_elems(), S = cfg_.steps;
    const std::string key = std::to_string(cfg_.seed) + "/" + std::to_string(S) + "/" + std::to_string(nl) +
                            "/" + std::to_string(cfg_.train_steps);
    if (key == z_key_) return;
    invalidate_graph();
    z_ = dev_alloc(&ledger_, S * nl * 4, true);
    const Schedule sc = make_schedule(cfg_);
    std::vector<float> z(static_cast<size_t>(nl));
    for (int64_t s = 0; s < S; ++s) {
        const StepCoeffs k = step_coeffs(cfg_, sc, s);
        if (!k.has_noise) continue;
        randn(k.noise_seed, nl, z.data());
        h2d_blocking(z_.as<float>() + s * nl, z.data(), static_cast<size_t>(nl) * 4);
    }
    z_key_ = key;
}

// Image mode inputs (pipeline.cpp:22-37, :108-114): the deterministic
// synthetic frames and the forward-noise draw randn(derive_seed(seed, 2)),
// generated on the host with the reference's double-precision formulas
// once per config and kept resident in HBM.
void Engine::prepare_image() {
    const int64_t T = cfg_.frames, IC = cfg_.image_channels, H = cfg_.height, W = cfg_.width;
    const std::string key = std::to_string(cfg_.seed) + "/" + std::to_string(T) + "x" + std::to_string(H) + "x" +
                            std::to_string(W);
    if (key == img_key_ && frames_dev_.p) return;
    invalidate_graph();
    std::vector<float> fr(static_cast<size_t>(T * IC * H * W));
    for (int64_t t = 0; t < T; ++t)
        for (int64_t c = 0; c < IC; ++c)
            for (int64_t y = 0; y < H; ++y)
                for (int64_t x = 0; x < W; ++x) {
                    const double phase = 0.25 * static_cast<double>(t) + 0.5 * static_cast<double>(c);
                    fr[static_cast<size_t>(((t * IC + c) * H + y) * W + x)] = static_cast<float>(
                        0.5 + 0.5 * std::sin(phase + 6.0 * static_cast<double>(y) / static_cast<double>(H)) *
                                  std::cos(phase + 6.0 * static_cast<double>(x) / static_cast<double>(W)));
                }
    frames_dev_ = dev_alloc(&ledger_, static_cast<int64_t>(fr.size()) * 4, false);
    h2d_blocking(frames_dev_.p, fr.data(), fr.size() * 4);
    const int64_t nl = latent_elems();
    std::vector<float> e(static_cast<size_t>(nl));
    randn(derive_seed(cfg_.seed, 2), nl, e.data());
    eps0_dev_ = dev_alloc(&ledger_, nl * 4, false);
    h2d_blocking(eps0_dev_.p, e.data(), e.size() * 4);
    img_key_ = key;
}

// encode (codec.cpp:64-81), frame slices of decode_slice frames:
// conv_silu(frames, enc0) -> [downsample2 -> conv(_silu)] x S -> latent
// (fp32 NCHW into lat_dev).
void Engine::encode_dev(float* lat_dev) {
    const int S = static_cast<int>(cfg_.stages);
    const int T = static_cast<int>(cfg_.frames), IC = static_cast<int>(cfg_.image_channels);
    const int H = static_cast<int>(cfg_.height), W = static_cast<int>(cfg_.width);
    const int Wc = static_cast<int>(cfg_.codec_width), C = static_cast<int>(cfg_.latent_channels);
    const int G = enc_patch_.n;  // slice of the arena's encode workspace (alloc_activations)
    if (G < 1 || !enc_patch_.p) throw_invariant("encode without a workspace");
    (void)Wc;
    const int lh = H >> S, lw = W >> S;
    for (int g0 = 0; g0 < T; g0 += G) {
        const int gs = std::min(G, T - g0);
        Act patch = enc_patch_, e[8], pl[8];
        patch.n = gs;
        for (int i = 0; i < S; ++i) (e[i] = enc_e_[i]).n = gs;
        for (int i = 1; i <= S; ++i) (pl[i] = enc_p_[i]).n = gs;
        ThinInArgs a{};
        a.x = frames_dev_.as<float>() + static_cast<int64_t>(g0) * IC * H * W;
        a.nsrc = gs;
        a.c_in = IC;
        a.H = H;
        a.W = W;
        a.cfg_pair = 0;
        a.apply_affine = 0;
        a.k = 3;
        a.out = patch.p;
        a.cs_out = patch.cs;
        a.win = Window{0, H, 0, W, 0, H, 0, W};
        LC_CUDA(launch_patch(a, enc0_kp_, s_compute_));
        run_tc_conv(*enc0_tc_, &patch, e[0], a.win, 1.0f, 0.0f, true, s_compute_);
        launches += 2;
        for (int i = 1; i <= S; ++i) {
            const Act& prev = e[i - 1];
            LC_CUDA(launch_down2(prev.p, pl[i].p, gs, prev.h, prev.w, prev.cs, s_compute_));
            const int h = H >> i, w = W >> i;
            if (i < S) {
                run_tc_conv(*enc_tc_[i - 1], &pl[i], e[i], Window{0, h, 0, w, 0, h, 0, w}, 1.0f, 0.0f, true,
                            s_compute_);
            } else {
                Act latv;
                latv.n = gs;
                latv.h = lh;
                latv.w = lw;
                latv.c = C;
                run_tc_conv(*enc_tc_[i - 1], &pl[i], latv, Window{0, h, 0, w, 0, h, 0, w}, 1.0f, 0.0f, false,
                            s_compute_, lat_dev + static_cast<int64_t>(g0) * C * lh * lw);
            }
            launches += 2;
        }
    }
}

// Denoise loop + decode for the current config, enqueued on the compute
// stream (and the two copy streams).  Fully asynchronous, so it can be
// captured into a CUDA graph and replayed (Engine::run).
void Engine::enqueue_body(RunStats& st) {
    const int64_t T = cfg_.frames;
    const Schedule sc = make_schedule(cfg_);
    const StepPlan plan = cfg_.cache_enabled ? plan_steps(cfg_.steps, cfg_.cache_n)
                                             : StepPlan{std::vector<bool>(static_cast<size_t>(cfg_.steps), true)};
    const int64_t nl = latent_elems();
    const int lh = static_cast<int>(cfg_.latent_h()), lw = static_cast<int>(cfg_.latent_w());
    const bool swap = cfg_.cache_enabled && cfg_.swap_mode != SwapMode::Off;
    evict_pending_ = prefetch_pending_ = false;
    d2h_used_ = h2d_used_ = false;
    {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        LC_CUDA(cudaStreamIsCapturing(s_compute_, &cs));
        dl_capture_ = cs == cudaStreamCaptureStatusActive && dl_gate_step_ >= 0 && dl_gate_step_ < cfg_.steps;
        dl_fired_ = false;
    }
    host_valid_ = false;
    body_enqueued_ = true;
    // regions a previous body left behind (an exception mid-enqueue, e.g.
    // BudgetError) are released so occupancy does not drift
    for (uint64_t* id : {&rid_act_, &rid_dec_, &rid_enc_, &rid_cache_[0], &rid_cache_[1]})
        if (*id) {
            if (ledger_.live.count(*id)) ledger_.region_free(*id);
            *id = 0;
        }
    marks_.clear();
    ev_next_ = 0;
    launches = 0;
    ev_den0_ = next_event();
    ev_den1_ = next_event();
    ev_end_ = next_event();
    record(6, -1, 0, s_compute_);  // timeline origin inside the body

    if (cfg_.mode == "image") {
        // Encode stage: latent = encode(frames); x = forward_noise(latent,
        // S-1, eps0) = sqrt(abar)*latent + sqrt(1-abar)*eps0 (pipeline.cpp:108-114)
        ledger_.enter(kEncode);
        rid_enc_ = ledger_.region_alloc(0, arena_info_.enc);
        // the workspace sits on the last run's activations / decode
        // workspace: channel padding must read zero again
        if (enc_padding_) LC_CUDA(cudaMemsetAsync(arena_.p, 0, static_cast<size_t>(arena_info_.enc), s_compute_));
        encode_dev(xn_.as<float>());
        ledger_.region_free(rid_enc_);
        rid_enc_ = 0;
        const Schedule sc0 = make_schedule(cfg_);
        const double ab = sc0.abar[static_cast<size_t>(cfg_.steps - 1)];
        LC_CUDA(launch_linear(static_cast<float>(std::sqrt(ab)), xn_.as<float>(),
                              static_cast<float>(std::sqrt(1.0 - ab)), eps0_dev_.as<float>(), x_.as<float>(), nl,
                              s_compute_));
        ++launches;
        ledger_.enter(kDenoise);
    }
    // Denoise working set: the activations and the two cache entries (the
    // reference's CacheStore holds one entry per CFG branch, cache.cpp:43-90)
    rid_act_ = ledger_.region_alloc(0, arena_info_.act);
    rid_cache_[0] = rid_cache_[1] = 0;
    if (cfg_.cache_enabled)
        for (int b = 0; b < 2; ++b) rid_cache_[b] = ledger_.region_alloc(0, cache_.elems());  // bytes/2 per branch
    {
        // the previous run's decode (and this run's encode) workspace
        // overwrote part of the arena: re-zero the channel padding the TMA
        // 64-channel blocks read (no padding at base 320: nothing to do)
        const int64_t dec_lo = arena_info_.arena - arena_info_.dec;
        const int64_t act_end = arena_info_.cache + arena_info_.act;
        if (act_padding_ && (dec_lo < act_end || cfg_.mode == "image"))
            LC_CUDA(cudaMemsetAsync(arena_.p, 0, static_cast<size_t>(act_end), s_compute_));
    }
    LC_CUDA(cudaMemsetAsync(bad_.p, 0, 16, s_compute_));
    LC_CUDA(launch_isfinite(x_.as<float>(), nl, bad_.as<int>(), s_compute_));
    ++launches;
    record_timing(ev_den0_, s_compute_);
    st.macs_full = flops_estimate(cfg_, 2, T, lh, lw, false);
    st.macs_cached = flops_estimate(cfg_, 2, T, lh, lw, true);
    const int64_t S = cfg_.steps;
    float* xa = x_.as<float>();
    float* xb = xn_.as<float>();
    for (int64_t s = 0; s < S; ++s) {
        const int64_t j = S - 1 - s;
        const int64_t t_orig = sc.src[j];
        const bool full = plan.is_full(s);
        if (cfg_.swap_simulate) ledger_.virt = sim_step_s_[static_cast<size_t>(s)];
        record(0, static_cast<int>(s), 0, s_compute_);
        // 3: full step whose store will be evicted (mark the cache-ready point)
        const int seam = swap ? (full ? 3 : (plan.is_last_consumer(s) ? 2 : 1)) : 0;
        const StepCoeffs k = step_coeffs(cfg_, sc, s);
        StepArgs a{};
        a.eps2 = eps2_.as<float>();
        a.x = xa;
        a.x_out = xb;
        // ancestral noise randn(derive_seed(seed, 0x1000+s)) (pipeline.cpp:181),
        // drawn on the host once per config (rng.hpp, bit-exact) and resident
        a.z = k.has_noise ? z_.as<float>() + s * nl : nullptr;
        a.n = nl;
        a.g = static_cast<float>(cfg_.guidance);
        a.a = k.a;
        a.b = k.b;
        a.c = k.noise;
        a.bad = bad_.as<int>();
        // the head (K8) applies the step in its epilogue when it can
        forward_dev(xa, false, T, t_orig, full, eps2_.as<float>(), static_cast<int>(s), seam, &a);
        record(1, static_cast<int>(s), 0, s_compute_);
        if (full) {
            st.full_steps++;
            st.denoiser_macs += st.macs_full;
            if (swap) {
                issue_evict(static_cast<int>(s));
                if (plan.has_consumers(s)) issue_prefetch(static_cast<int>(s), static_cast<int>(s + 1));
            }
        } else {
            st.cached_steps++;
            st.denoiser_macs += st.macs_cached;
        }
        if (!step_fused_) {
            LC_CUDA(launch_step(a, s_compute_));
            ++launches;
        }
        std::swap(xa, xb);
    }
    x_final_ = xa;
    record_timing(ev_den1_, s_compute_);
    // the denoise activations die with the loop (x_in / eps of the last step,
    // pipeline.cpp:170-186); the cache entries stay (on the host after the
    // final eviction with the swap on, in HBM without it) until the store's
    // teardown after decode (pipeline.cpp:206)
    ledger_.region_free(rid_act_);
    rid_act_ = 0;
    if (cfg_.swap_simulate) ledger_.virt = sim_decode_s_;
    ledger_.enter(kDecode);
    rid_dec_ = ledger_.region_alloc(0, arena_info_.dec);
    if (arena_info_.dec_overlaps_cache && evict_pending_)
        for (int b = 0; b < 2; ++b) LC_CUDA(cudaStreamWaitEvent(s_compute_, ev_evict_[b], 0));
    if (dec_padding_)
        LC_CUDA(cudaMemsetAsync(arena_.as<char>() + (arena_info_.arena - arena_info_.dec), 0,
                                static_cast<size_t>(arena_info_.dec), s_compute_));
    out_slices_ = true;
    dec_ws_ = &dec_ws_run_;
    decode_dev(xa, T, video_.as<float>());
    dec_ws_ = nullptr;
    out_slices_ = false;
    dl_capture_ = false;
    ledger_.region_free(rid_dec_);
    rid_dec_ = 0;
    for (int b = 0; b < 2; ++b)
        if (rid_cache_[b]) {
            ledger_.region_free(rid_cache_[b]);  // CacheStore::teardown (cache.cpp:110-122)
            rid_cache_[b] = 0;
        }
    // join the copy streams that were used (required to close a graph
    // capture; the last eviction stays in flight through decode as in the
    // reference, proj/README.md "Swap schedule")
    if (d2h_used_) {
        LC_CUDA(cudaEventRecord(ev_join_[0], s_d2h_));
        LC_CUDA(cudaStreamWaitEvent(s_compute_, ev_join_[0], 0));
    }
    if (h2d_used_) {
        LC_CUDA(cudaEventRecord(ev_join_[1], s_h2d_));
        LC_CUDA(cudaStreamWaitEvent(s_compute_, ev_join_[1], 0));
    }
    record_timing(ev_end_, s_compute_);
}

RunStats Engine::run(const float* x0_host, float* video_host, float* latent_host, bool resident_input) {
    if (async_pending_) (void)wait();  // completes queued runs (and resets stats_)
    RunStats st;
    stats_ = &st;
    const int64_t T = cfg_.frames;
    alloc_activations(T);
    ledger_.budget_fast = cfg_.budget_fast_bytes;
    // per-run peaks, as each reference run has a fresh ledger
    // (pipeline.cpp:69); the persistent buffers are the starting occupancy
    for (int s = 0; s < 4; ++s)
        for (int t = 0; t < 2; ++t) ledger_.peak[s][t] = ledger_.occ[t];
    if (cfg_.budget_fast_bytes > 0 && ledger_.occ[0] > cfg_.budget_fast_bytes)
        throw LcError(kBudgetError,
                      "fast-tier budget exceeded in stage denoise: " + std::to_string(ledger_.occ[0]) + " > " +
                          std::to_string(cfg_.budget_fast_bytes) + " bytes",
                      kDenoise);
    const int64_t nl = latent_elems();
    const int lh = static_cast<int>(cfg_.latent_h()), lw = static_cast<int>(cfg_.latent_w());
    prepare_noise();
    const bool image = cfg_.mode == "image";
    if (image) prepare_image();

    if (async_pending_) (void)wait();
    cudaEvent_t t_start = ev_start_;
    LC_CUDA(cudaEventRecord(t_start, s_compute_));
    ledger_.virt = cfg_.swap_simulate ? 0.0 : -1.0;
    ledger_.enter(kEncode);
    if (image) {
        // the latent comes from the encode stage inside the body
    } else if (!resident_input) {
        std::vector<float> gen;
        const float* src = x0_host;
        if (!src) {
            gen.resize(static_cast<size_t>(nl));
            randn(derive_seed(cfg_.seed, 1), nl, gen.data());
            src = gen.data();
        }
        LC_CUDA(cudaMemcpyAsync(x_.p, src, static_cast<size_t>(nl) * 4, cudaMemcpyHostToDevice, s_compute_));
        if (!x0_host) LC_CUDA(cudaStreamSynchronize(s_compute_));
    } else {
        LC_CUDA(cudaMemcpyAsync(x_.p, x0_.p, static_cast<size_t>(nl) * 4, cudaMemcpyDeviceToDevice, s_compute_));
    }

    ledger_.enter(kDenoise);
    // The body is enqueued eagerly on the first run after (re)configuration
    // (allocations, kernel attributes), captured into a CUDA graph on the
    // second, and replayed from then on: the host no longer paces ~70
    // launches per video (tensor-map encoding, parameter setup).
    const bool can_graph = use_graphs && conv_profiler() == nullptr;
    // Pinned destination: the decoded slices stream out inside the body.  A
    // pageable destination (the reference's host RunResult::video) gets a
    // pinned staging buffer that the slices stream into the same way; the
    // host copies it out with several threads once the run completes.
    float* pinned = nullptr;
    if (video_host) {
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, video_host) == cudaSuccess && pa.type == cudaMemoryTypeHost)
            pinned = video_host;
        cudaGetLastError();  // clear a "not a CUDA pointer" status for pageable memory
        if (!pinned) {
            const int64_t vbytes = video_elems() * 4;
            if (!vid_stage_.p || vid_stage_.bytes < vbytes) vid_stage_ = host_alloc(nullptr, vbytes);
            pinned = vid_stage_.as<float>();
        }
    }
    if (graph_exec_ && graph_slice_ != decode_slice) invalidate_graph();
    video_host_pinned_ = pinned;
    graph_slice_ = decode_slice;
    if (can_graph && graph_exec_) {
        arm_download_node();
        LC_CUDA(cudaGraphLaunch(graph_exec_, s_compute_));
        st = graph_stats_;
        stats_ = &st;
    } else if (can_graph && eager_runs_ > 0) {
        cudaGraph_t g = nullptr;
        // placeholder destination of the deferred-download node (no
        // allocation may happen inside the capture); not a ledger buffer:
        // steady-state launches re-point the node at the caller's memory
        const int64_t vbytes = video_elems() * 4;
        if (dl_gate_step_ >= 0 && (!dl_scratch_.p || dl_scratch_.bytes < vbytes))
            dl_scratch_ = host_alloc(nullptr, vbytes);
        LC_CUDA(cudaStreamBeginCapture(s_compute_, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue_body(st);
        } catch (...) {
            cudaStreamEndCapture(s_compute_, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        LC_CUDA(cudaStreamEndCapture(s_compute_, &g));
        // the deferred-download memcpy node (source: the device video)
        dl_node_ = nullptr;
        size_t nn = 0;
        LC_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        if (nn) LC_CUDA(cudaGraphGetNodes(g, nodes.data(), &nn));
        for (cudaGraphNode_t nd : nodes) {
            cudaGraphNodeType ty;
            LC_CUDA(cudaGraphNodeGetType(nd, &ty));
            if (ty != cudaGraphNodeTypeMemcpy) continue;
            cudaMemcpy3DParms mp{};
            LC_CUDA(cudaGraphMemcpyNodeGetParams(nd, &mp));
            if (mp.srcPtr.ptr == video_.p && dl_scratch_.p && mp.dstPtr.ptr == dl_scratch_.p) dl_node_ = nd;
        }
        LC_CUDA(cudaGraphInstantiate(&graph_exec_, g, 0));
        graph_ = g;
        graph_stats_ = st;
        arm_download_node();
        LC_CUDA(cudaGraphLaunch(graph_exec_, s_compute_));
    } else {
        flush_pending_download();
        enqueue_body(st);
        ++eager_runs_;
    }
    if (pinned) enqueue_video_out(pinned);
    if (cfg_.swap_simulate) ledger_.virt = sim_decode_s_;
    ledger_.enter(kDecode);
    RunStats out = finish_run(st, pinned == video_host ? video_host : nullptr, latent_host);
    if (video_host && pinned != video_host) copy_out_parallel(video_host, pinned, video_elems());
    return out;
}

// Pinned staging -> the caller's pageable video: a memory-bound host copy
// split over up to 8 threads (first-touch page faults of a fresh caller
// buffer are spread the same way).
void Engine::copy_out_parallel(float* dst, const float* src, int64_t n) {
    const int64_t kMin = 1 << 20;  // floats per thread at least
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int nt = static_cast<int>(std::min<int64_t>(std::min<unsigned>(hw, 8u), (n + kMin - 1) / kMin));
    if (nt <= 1) {
        std::memcpy(dst, src, static_cast<size_t>(n) * 4);
        return;
    }
    std::vector<std::thread> th;
    const int64_t per = (n + nt - 1) / nt;
    for (int i = 0; i < nt; ++i) {
        const int64_t a = i * per, b = std::min(n, a + per);
        if (a < b) th.emplace_back([=] { std::memcpy(dst + a, src + a, static_cast<size_t>(b - a) * 4); });
    }
    for (auto& t : th) t.join();
}

// Throughput form of run() with pinned host buffers: H2D of the latent, the
// graph, and the per-slice video download are queued without a host round
// trip, so run k+1's denoise overlaps run k's download; wait() completes.
void Engine::run_e2e_async(const float* x0_pinned, float* video_pinned) {
    // page-locked buffers only: the graph's download node and the queued H2D
    // must not see pageable memory (such a call runs synchronously instead)
    auto is_pinned = [](const void* ptr) {
        cudaPointerAttributes pa{};
        const bool ok = ptr && cudaPointerGetAttributes(&pa, ptr) == cudaSuccess && pa.type == cudaMemoryTypeHost;
        cudaGetLastError();
        return ok;
    };
    const bool ready = use_graphs && conv_profiler() == nullptr && graph_exec_ && graph_slice_ == decode_slice &&
                       T_alloc_ == cfg_.frames && cfg_.mode != "image" && is_pinned(x0_pinned) &&
                       is_pinned(video_pinned);
    if (!ready) {
        last_async_ = run(x0_pinned, video_pinned, nullptr, false);
        async_pending_ = false;
        return;
    }
    LC_CUDA(cudaEventRecord(ev_start_, s_compute_));
    LC_CUDA(cudaMemcpyAsync(x_.p, x0_pinned, static_cast<size_t>(latent_elems()) * 4, cudaMemcpyHostToDevice,
                            s_compute_));
    arm_download_node();  // the previous run's video leaves inside this one
    LC_CUDA(cudaGraphLaunch(graph_exec_, s_compute_));
    if (dl_node_) dl_pending_ = video_pinned;
    else enqueue_video_out(video_pinned);
    async_pending_ = true;
}

// Steady-state resident replay without the host round trip: enqueue the
// input copy and the graph, return.  Consecutive calls queue back to back on
// the compute stream (the body joins its copy streams at the end, so runs
// never overlap); wait() completes the last one.  Before the graph exists
// (first two runs after a (re)configuration) this is a synchronous run().
void Engine::run_resident_async() {
    const bool ready = use_graphs && conv_profiler() == nullptr && graph_exec_ && graph_slice_ == decode_slice &&
                       T_alloc_ == cfg_.frames;
    if (!ready) {
        last_async_ = run(nullptr, nullptr, nullptr, true);
        async_pending_ = false;
        return;
    }
    LC_CUDA(cudaEventRecord(ev_start_, s_compute_));
    LC_CUDA(cudaMemcpyAsync(x_.p, x0_.p, static_cast<size_t>(latent_elems()) * 4, cudaMemcpyDeviceToDevice,
                            s_compute_));
    arm_download_node();
    LC_CUDA(cudaGraphLaunch(graph_exec_, s_compute_));
    async_pending_ = true;
}

RunStats Engine::wait() {
    if (!async_pending_) return last_async_;
    async_pending_ = false;
    flush_pending_download();
    video_host_pinned_ = nullptr;
    RunStats st = graph_stats_;
    stats_ = &st;
    if (cfg_.swap_simulate) ledger_.virt = sim_decode_s_;
    ledger_.enter(kDecode);
    last_async_ = finish_run(st, nullptr, nullptr);
    return last_async_;
}

RunStats Engine::finish_run(RunStats st, float* video_host, float* latent_host) {
    const cudaEvent_t t_start = ev_start_;
    const int64_t T = cfg_.frames;
    const int64_t nl = latent_elems();
    const int lh = static_cast<int>(cfg_.latent_h()), lw = static_cast<int>(cfg_.latent_w());
    if (video_host && !video_host_pinned_)
        LC_CUDA(cudaMemcpyAsync(video_host, video_.p, static_cast<size_t>(video_elems()) * 4,
                                cudaMemcpyDeviceToHost, s_compute_));
    if (latent_host)
        LC_CUDA(cudaMemcpyAsync(latent_host, x_final_, static_cast<size_t>(nl) * 4, cudaMemcpyDeviceToHost,
                                s_compute_));
    int bad = 0;
    LC_CUDA(cudaMemcpyAsync(&bad, bad_.p, 4, cudaMemcpyDeviceToHost, s_compute_));
    LC_CUDA(cudaStreamSynchronize(s_compute_));
    LC_CUDA(cudaStreamSynchronize(s_d2h_));
    LC_CUDA(cudaStreamSynchronize(s_h2d_));
    LC_CUDA(cudaStreamSynchronize(s_vid_));
    stats_ = nullptr;
    video_host_pinned_ = nullptr;  // operator-level decode() must not stream to it
    if (bad) throw_shape("denoiser input contains non-finite values");

    float ms = 0;
    LC_CUDA(cudaEventElapsedTime(&ms, ev_den0_, ev_den1_));
    st.ms_denoise = ms;
    LC_CUDA(cudaEventElapsedTime(&ms, ev_den1_, ev_end_));
    st.ms_decode = ms;
    LC_CUDA(cudaEventElapsedTime(&ms, t_start, ev_end_));
    st.ms_total = ms;
    if (!marks_.empty()) {  // body origin (record 6) -> denoise start: the encode stage
        LC_CUDA(cudaEventElapsedTime(&ms, marks_.front().ev, ev_den0_));
        st.ms_encode = ms;
    }
    st.timeline.clear();
    st.stall_ms = 0;
    double open = 0, lo = 1e30, hi = -1e30;
    const cudaEvent_t origin = marks_.empty() ? t_start : marks_.front().ev;
    for (const Mark& mk : marks_) {
        if (mk.kind == 6) continue;
        float t = 0;
        LC_CUDA(cudaEventElapsedTime(&t, origin, mk.ev));
        st.timeline.push_back({static_cast<double>(mk.kind), static_cast<double>(mk.step),
                               static_cast<double>(mk.bytes), static_cast<double>(t)});
        lo = std::min(lo, static_cast<double>(t));
        hi = std::max(hi, static_cast<double>(t));
        if (mk.kind == 4 || mk.kind == 7) open = t;
        if (mk.kind == 5 || mk.kind == 8) st.stall_ms += t - open;
    }
    st.makespan_ms = marks_.empty() ? 0.0 : hi - lo;
    st.simulated = cfg_.swap_simulate;
    if (st.simulated) {
        // swap.simulate: the reported timeline is the simulated transfer
        // engine's virtual one (swap.cpp:141-374, pipeline.cpp:209-212);
        // the device work above is unchanged.
        st.timeline.clear();
        for (const SimEvent& e : sim_tl_)
            st.timeline.push_back({static_cast<double>(e.kind), static_cast<double>(e.step),
                                   static_cast<double>(e.bytes), e.clock_ns * 1e-6});
        st.makespan_ms = sim_makespan_ns(sim_tl_) * 1e-6;
        st.stall_ms = sim_stall_ns(sim_tl_) * 1e-6;
    }
    st.cache_bytes_planned = cfg_.cache_enabled
                                 ? 2 * T * cache_channels(cfg_) * (lh >> cfg_.cache_depth) *
                                       (lw >> cfg_.cache_depth) * 4
                                 : 0;
    st.cache_bytes_physical = cfg_.cache_enabled ? cache_.elems() * 2 : 0;
    // A graph replay logs no ledger events (the body was not enqueued on the
    // host): its peaks are those of the run that enqueued / captured it.
    if (body_enqueued_) std::memcpy(body_peak_, ledger_.peak, sizeof(body_peak_));
    else
        for (int s = 0; s < 4; ++s)
            for (int t = 0; t < 2; ++t) ledger_.peak[s][t] = std::max(ledger_.peak[s][t], body_peak_[s][t]);
    body_enqueued_ = false;
    std::memcpy(st.peak, ledger_.peak, sizeof(st.peak));
    st.hbm_peak = 0;
    for (int s = 0; s < 4; ++s) st.hbm_peak = std::max(st.hbm_peak, ledger_.peak[s][0]);
    st.kernel_launches = launches;
    st.setup_s = configure_s_;
    ledger_.enter(kSetup);
    last_stats_ = st;
    return st;
}

void Engine::forward(const float* x_host, int64_t T, int64_t timestep, const float* deep_in_ref,
                     float* deep_out_ref, float* eps_host) {
    if (async_pending_) (void)wait();
    RunConfig c = cfg_;
    if (c.frames != T) {
        c.frames = T;
        configure(c);
    }
    alloc_activations(T);
    const int lh = static_cast<int>(cfg_.latent_h()), lw = static_cast<int>(cfg_.latent_w());
    const int C = static_cast<int>(cfg_.latent_channels);
    const int64_t n1 = T * C * lh * lw;
    // explicit (2,T,...) input: the stem reads both halves as given.
    invalidate_graph();
    if (act_padding_) {  // a run's decode workspace may have overwritten the channel padding
        LC_CUDA(cudaMemsetAsync(arena_.p, 0, static_cast<size_t>(arena_info_.cache + arena_info_.act), s_compute_));
        LC_CUDA(cudaStreamSynchronize(s_compute_));
    }
    DevBuf xin = dev_alloc(nullptr, 2 * n1 * 4, false);
    h2d_blocking(xin.p, x_host, static_cast<size_t>(2 * n1) * 4);
    const bool full = deep_in_ref == nullptr;
    if (!cfg_.cache_enabled) throw_config("forward(): cache.enabled must be true for seam access");
    if (!full) {
        // reference u_next = upsample2(U_{m+1}); keep every other pixel (exact).
        const int m = static_cast<int>(cfg_.cache_depth);
        const Act& a = cache_;
        std::vector<__half> hbuf(static_cast<size_t>(a.elems()), __float2half_rn(0.0f));
        const int Hr = lh >> m, Wr = lw >> m;
        for (int n = 0; n < a.n; ++n)
            for (int c2 = 0; c2 < a.c; ++c2)
                for (int y = 0; y < a.h; ++y)
                    for (int x = 0; x < a.w; ++x)
                        hbuf[((static_cast<size_t>(n) * a.h + y) * a.w + x) * a.cs + c2] = __float2half_rn(
                            deep_in_ref[((static_cast<size_t>(n) * a.c + c2) * Hr + 2 * y) * Wr + 2 * x]);
        h2d_blocking(a.p, hbuf.data(), hbuf.size() * 2);
    }
    forward_dev(xin.as<float>(), true, T, timestep, full, eps2_.as<float>(), 0, 0);
    LC_CUDA(cudaStreamSynchronize(s_compute_));
    LC_CUDA(cudaMemcpy(eps_host, eps2_.p, static_cast<size_t>(2 * n1) * 4, cudaMemcpyDeviceToHost));
    if (full && deep_out_ref) {
        const int m = static_cast<int>(cfg_.cache_depth);
        const Act& a = cache_;
        std::vector<__half> hbuf(static_cast<size_t>(a.elems()));
        LC_CUDA(cudaMemcpy(hbuf.data(), a.p, hbuf.size() * 2, cudaMemcpyDeviceToHost));
        const int Hr = lh >> m, Wr = lw >> m;
        for (int n = 0; n < a.n; ++n)
            for (int c2 = 0; c2 < a.c; ++c2)
                for (int y = 0; y < Hr; ++y)
                    for (int x = 0; x < Wr; ++x)
                        deep_out_ref[((static_cast<size_t>(n) * a.c + c2) * Hr + y) * Wr + x] = __half2float(
                            hbuf[((static_cast<size_t>(n) * a.h + y / 2) * a.w + x / 2) * a.cs + c2]);
    }
}

// decode_batch / decode_sliced's checks (codec.cpp:117-135): the latent
// channel count must be the codec's; the engine is configured for one
// latent geometry, so a different h x w is a ShapeError too.
static void check_decode_shape(const RunConfig& c, int64_t n, int64_t ch, int64_t h, int64_t w) {
    if (n < 0) throw_shape("decode: negative frame count");
    if (ch != c.latent_channels)
        throw_shape("decode expects " + std::to_string(c.latent_channels) + " latent channels");
    if (h != c.latent_h() || w != c.latent_w())
        throw_shape("decode: latent " + std::to_string(h) + "x" + std::to_string(w) +
                    " does not match the configured geometry " + std::to_string(c.latent_h()) + "x" +
                    std::to_string(c.latent_w()));
}

void Engine::decode(const float* lat_host, int64_t n, int64_t c, int64_t h, int64_t w, float* video_host,
                    int64_t slice) {
    if (async_pending_) (void)wait();
    check_decode_shape(cfg_, n, c, h, w);
    if (n == 0) return;
    const int C = static_cast<int>(cfg_.latent_channels);
    const int64_t nl = n * C * cfg_.latent_h() * cfg_.latent_w();
    const int64_t nv = n * cfg_.image_channels * cfg_.height * cfg_.width;
    invalidate_graph();
    DevBuf lat = dev_alloc(nullptr, nl * 4, false);
    DevBuf vid = dev_alloc(nullptr, nv * 4, false);
    LC_CUDA(cudaMemcpyAsync(lat.p, lat_host, static_cast<size_t>(nl) * 4, cudaMemcpyHostToDevice, s_compute_));
    if (slice < 1) throw_config("decode slice must be >= 1");
    ensure_op_dec_ws(static_cast<int>(std::min(slice, n)));
    dec_ws_ = &dec_ws_op_;
    decode_dev(lat.as<float>(), n, vid.as<float>());
    dec_ws_ = nullptr;
    LC_CUDA(cudaMemcpyAsync(video_host, vid.p, static_cast<size_t>(nv) * 4, cudaMemcpyDeviceToHost, s_compute_));
    LC_CUDA(cudaStreamSynchronize(s_compute_));
}

}  // namespace lc

namespace lc {

void Engine::decode_sharded(const float* lat_host, int64_t T, int64_t c, int64_t h, int64_t w, int64_t slice,
                            float* video_host, bool host_shared, ncclComm_t comm, int world, int rank,
                            float* ms_out) {
    if (async_pending_) (void)wait();
    check_decode_shape(cfg_, T, c, h, w);
    if (slice < 1) throw_config("decode slice must be >= 1");
    if (world > 1 && !comm) throw_config("decode_sharded: no NCCL communicator for world > 1");
    const int64_t lat_frame = cfg_.latent_channels * cfg_.latent_h() * cfg_.latent_w();
    const int64_t vid_frame = cfg_.image_channels * cfg_.height * cfg_.width;
    const ShardSpan me = shard_frames(T, world, rank);
    const std::vector<GatherRow> plan = gather_plan(T, world, slice);
    // shard buffers persist across calls (grow-only), like the run's; only
    // rank 0 holds the whole video (the gather target)
    ensure_buf(&shard_lat_, std::max<int64_t>(1, me.count) * lat_frame * 4);
    ensure_buf(&shard_vid_, std::max<int64_t>(1, rank == 0 ? T : me.count) * vid_frame * 4);
    float* vid = shard_vid_.as<float>();
    // rank 0 decodes its frames in place; the others into [0, count)
    const int64_t own0 = rank == 0 ? me.first : 0;
    cudaEvent_t e0, e1, ej;
    LC_CUDA(cudaEventCreate(&e0));
    LC_CUDA(cudaEventCreate(&e1));
    LC_CUDA(cudaEventCreateWithFlags(&ej, cudaEventDisableTiming));
    LC_CUDA(cudaEventRecord(e0, s_compute_));  // device time: shard H2D, decode, gather (+ host output)
    launches = 0;
    if (me.count > 0)
        LC_CUDA(cudaMemcpyAsync(shard_lat_.p, lat_host + me.first * lat_frame,
                                static_cast<size_t>(me.count * lat_frame) * 4, cudaMemcpyHostToDevice, s_compute_));
    // the comm / copy streams start after the shard buffers are ours
    LC_CUDA(cudaEventRecord(ej, s_compute_));
    LC_CUDA(cudaStreamWaitEvent(s_comm_, ej, 0));
    LC_CUDA(cudaStreamWaitEvent(s_d2h_, ej, 0));
    out_slices_ = true;  // per-slice completion events (chunk_event(2, i))
    slice_spans_.clear();
    if (me.count > 0) {
        ensure_op_dec_ws(static_cast<int>(std::min(slice, me.count)));
        dec_ws_ = &dec_ws_op_;
        decode_dev(shard_lat_.as<float>(), me.count, vid + own0 * vid_frame);
        dec_ws_ = nullptr;
    }
    out_slices_ = false;
    auto nccl = [](ncclResult_t r, const char* what) {
        if (r != ncclSuccess) throw LcError(kCudaError, std::string(what) + ": " + ncclGetErrorString(r));
    };
    const bool host_out = video_host != nullptr;
    if (world > 1) {
        // the gather, slice by slice (gather_plan rounds): senders post slice
        // i as soon as it is decoded; rank 0 receives round i from every peer
        // in one group while its own slices still decode
        int64_t round = -1;
        bool open = false;
        size_t mine = 0;
        for (const GatherRow& g : plan) {
            if (g.rank == 0) continue;
            if (rank == 0) {
                if (g.round != round) {
                    if (open) nccl(ncclGroupEnd(), "ncclGroupEnd");
                    nccl(ncclGroupStart(), "ncclGroupStart");
                    open = true;
                    round = g.round;
                }
                nccl(ncclRecv(vid + g.first * vid_frame, static_cast<size_t>(g.count * vid_frame), ncclFloat,
                              static_cast<int>(g.rank), comm, s_comm_),
                     "ncclRecv");
            } else if (g.rank == rank) {
                LC_CUDA(cudaStreamWaitEvent(s_comm_, chunk_event(2, mine), 0));
                nccl(ncclSend(vid + (g.first - me.first) * vid_frame, static_cast<size_t>(g.count * vid_frame),
                              ncclFloat, 0, comm, s_comm_),
                     "ncclSend");
                ++mine;
            }
        }
        if (open) nccl(ncclGroupEnd(), "ncclGroupEnd");
    }
    if (host_out) {
        // every rank's own slices leave for the host as they are decoded;
        // rank 0 also downloads what it received unless the peers write their
        // frames into the shared host buffer themselves
        for (size_t i = 0; i < slice_spans_.size(); ++i) {
            if (!host_shared && rank != 0) break;
            LC_CUDA(cudaStreamWaitEvent(s_d2h_, chunk_event(2, i), 0));
            const int64_t f = me.first + slice_spans_[i].first, n = slice_spans_[i].second;
            LC_CUDA(cudaMemcpyAsync(video_host + f * vid_frame, vid + (own0 + slice_spans_[i].first) * vid_frame,
                                    static_cast<size_t>(n * vid_frame) * 4, cudaMemcpyDeviceToHost, s_d2h_));
        }
        if (rank == 0 && !host_shared && world > 1) {
            LC_CUDA(cudaEventRecord(ej, s_comm_));
            LC_CUDA(cudaStreamWaitEvent(s_d2h_, ej, 0));
            for (const GatherRow& g : plan)
                if (g.rank != 0)
                    LC_CUDA(cudaMemcpyAsync(video_host + g.first * vid_frame, vid + g.first * vid_frame,
                                            static_cast<size_t>(g.count * vid_frame) * 4, cudaMemcpyDeviceToHost,
                                            s_d2h_));
        }
    }
    for (cudaStream_t st : {s_comm_, s_d2h_}) {
        LC_CUDA(cudaEventRecord(ej, st));
        LC_CUDA(cudaStreamWaitEvent(s_compute_, ej, 0));
    }
    LC_CUDA(cudaEventRecord(e1, s_compute_));
    LC_CUDA(cudaStreamSynchronize(s_compute_));
    float ms = 0;
    LC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (ms_out) *ms_out = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(ej);
}

}  // namespace lc

namespace lc {

namespace {
ConvProfiler* g_conv_prof = nullptr;
}

ConvProfiler* conv_profiler() { return g_conv_prof; }
void set_conv_profiler(ConvProfiler* p) { g_conv_prof = p; }

void ConvProfiler::clear() {
    for (auto& r : recs) {
        cudaEventDestroy(r.e0);
        cudaEventDestroy(r.e1);
    }
    recs.clear();
}

std::string ConvProfiler::records_json() const {
    std::string o = "[";
    for (size_t i = 0; i < recs.size(); ++i) {
        float t = 0;
        LC_CUDA(cudaEventSynchronize(recs[i].e1));
        LC_CUDA(cudaEventElapsedTime(&t, recs[i].e0, recs[i].e1));
        o += (i ? ",{" : "{");
        o += "\"ms\":" + std::to_string(t) + ",\"alg_flops\":" + std::to_string(recs[i].alg_flops) +
             ",\"exec_flops\":" + std::to_string(recs[i].exec_flops) + ",\"desc\":\"" + recs[i].desc + "\"}";
    }
    return o + "]";
}

void ConvProfiler::summarize(int64_t* n, double* ms, double* alg, double* exec) const {
    *n = static_cast<int64_t>(recs.size());
    *ms = *alg = *exec = 0;
    for (const auto& r : recs) {
        float t = 0;
        LC_CUDA(cudaEventSynchronize(r.e1));
        LC_CUDA(cudaEventElapsedTime(&t, r.e0, r.e1));
        *ms += t;
        *alg += r.alg_flops;
        *exec += r.exec_flops;
    }
}

}  // namespace lc
