// Phase-vocoder time stretch on the GPU — the reference's own alignment of the chosen cached
// latent to the requested duration: time_stretch (vocoder.cpp:128-207) with
// its stft / istft (vocoder.cpp:54-124) and radix-2 fft_inplace (vocoder.cpp:18-44).
//
// One CTA per clip, frames processed in order (the synthesis phase of every bin is a running
// sum over frames): per frame a forward FFT of the Hann-windowed analysis frame, per bin the
// magnitude / phase, the phase-increment unwrap around the bin centre and the synthesis-phase
// advance by hop_s, the conjugate-symmetric synthesis frame, the inverse FFT and the
// overlap-add of window * frame and window^2 (acc / wsum in frame order, as istft does).
//
// Every + - * / is the reference's, in its order (complex products as ac - bd, ad + bc; the FFT
// twiddles are the reference's own recurrence w *= wlen, evaluated once on the host with libm;
// the Hann window likewise). Only hypot / atan2 / cos / sin of the per-bin polar conversion use
// CUDA's libm (<= 2 ulp from glibc), so outputs match the reference to ~1e-15 relative before
// the final fp32 rounding (tests/test_gpu_vocoder.py: |d| <= 1e-6, almost all bit-equal).
#include <cmath>
#include <complex>
#include <map>
#include <mutex>

#include "sw_internal.cuh"

namespace sw {

namespace {

constexpr int VT = 64;           // threads per clip (one radix-2 butterfly each at N = 128)
constexpr int kMaxWin = 1024;

struct ClipDesc {
    int64_t in_off, out_off, work_off;
    int32_t in_len, target, hop_s, frames, natural, status;
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {  // (a.x + i a.y)(b.x + i b.y)
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

__device__ __forceinline__ double wrap_phase(double p) {  // vocoder.cpp:126-130
    p = fmod(__dadd_rn(p, M_PI), 2.0 * M_PI);
    if (p < 0) p = __dadd_rn(p, 2.0 * M_PI);
    return __dsub_rn(p, M_PI);
}

// fft_inplace stages on a bit-reversed buffer; tw = the per-stage w_j sequences, concatenated
__device__ void fft_stages(double2* a, int n, const double2* __restrict__ tw) {
    int base = 0;
    for (int len = 2; len <= n; len <<= 1) {
        const int h = len >> 1;
        for (int b = threadIdx.x; b < (n >> 1); b += blockDim.x) {
            const int grp = b / h, j = b - grp * h;
            const int i = grp * len + j;
            const double2 u = a[i];
            const double2 v = cmul(a[i + h], __ldg(&tw[base + j]));
            a[i] = make_double2(__dadd_rn(u.x, v.x), __dadd_rn(u.y, v.y));
            a[i + h] = make_double2(__dsub_rn(u.x, v.x), __dsub_rn(u.y, v.y));
        }
        base += h;
        __syncthreads();
    }
}

__device__ __forceinline__ int bitrev(int i, int logn) { return (int)(__brev((unsigned)i) >> (32 - logn)); }

// One clip's time_stretch by one CTA: x[i * xs] for i < in_len -> y[i * ys] for i < ylim
// (<= target). buf: n complex doubles; acc / wsum: natural doubles each (smem or global).
template <int NB>  // bins per thread: k = threadIdx.x + VT u, u < NB (NB * VT > n / 2)
__device__ void stretch_clip(const float* __restrict__ x, int xs, int in_len, float* __restrict__ y,
                             int ys, int ylim, int target, int hop_s, int frames, int natural,
                             int n, int logn, int hop_a, const double* __restrict__ window,
                             const double2* __restrict__ tw_fwd, const double2* __restrict__ tw_inv,
                             double2* buf, double* acc, double* wsum) {
    const int half = n / 2;
    for (int i = threadIdx.x; i < natural; i += blockDim.x) {
        acc[i] = 0.0;
        wsum[i] = 0.0;
    }
    double prev_phase[NB], synth_phase[NB];
    double2 ob[NB];
#pragma unroll
    for (int u = 0; u < NB; ++u) prev_phase[u] = synth_phase[u] = 0.0;
    for (int m = 0; m < frames; ++m) {
        __syncthreads();
        // stft frame m (vocoder.cpp:80-88): window[i] * padded[m hop_a + i], zero past the clip
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int s = m * hop_a + i;
            const float v = s < in_len ? x[(int64_t)s * xs] : 0.0f;
            buf[bitrev(i, logn)] = make_double2(__dmul_rn(__ldg(&window[i]), (double)v), 0.0);
        }
        __syncthreads();
        fft_stages(buf, n, tw_fwd);
        // per-bin magnitude and phase propagation (vocoder.cpp:174-192)
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const int kk = threadIdx.x + VT * u;
            ob[u] = make_double2(0.0, 0.0);
            if (kk > half) continue;
            const double2 z = buf[kk];
            const double mag = hypot(z.x, z.y);  // std::abs
            const double cur = atan2(z.y, z.x);  // std::arg
            double phase;
            if (m == 0) {
                prev_phase[u] = cur;
                synth_phase[u] = cur;
                phase = cur;
            } else {
                const double omega = __ddiv_rn(__dmul_rn(2.0 * M_PI, (double)kk), (double)n);
                const double expected = __dmul_rn(omega, (double)hop_a);
                const double dev = wrap_phase(__dsub_rn(__dsub_rn(cur, prev_phase[u]), expected));
                const double inst = __dadd_rn(omega, __ddiv_rn(dev, (double)hop_a));
                synth_phase[u] =
                    wrap_phase(__dadd_rn(synth_phase[u], __dmul_rn(inst, (double)hop_s)));
                prev_phase[u] = cur;
                phase = synth_phase[u];
            }
            double sn, cs;
            sincos(phase, &sn, &cs);  // one range reduction for both (polar)
            ob[u] = make_double2(__dmul_rn(mag, cs), __dmul_rn(mag, sn));
        }
        __syncthreads();
        // synthesis frame, conjugate-symmetric, into bit-reversed order for the inverse FFT
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const int kk = threadIdx.x + VT * u;
            if (kk > half) continue;
            buf[bitrev(kk, logn)] = ob[u];
            if (kk >= 1 && kk < half) buf[bitrev(n - kk, logn)] = make_double2(ob[u].x, -ob[u].y);
        }
        __syncthreads();
        fft_stages(buf, n, tw_inv);
        // istft overlap-add (vocoder.cpp:104-111): real part of x / n, frames in order
        const int64_t off = (int64_t)m * hop_s;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const double w = __ldg(&window[i]);
            const double re = __ddiv_rn(buf[i].x, (double)n);
            acc[off + i] = __dadd_rn(acc[off + i], __dmul_rn(w, re));
            wsum[off + i] = __dadd_rn(wsum[off + i], __dmul_rn(w, w));
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ylim; i += blockDim.x) {
        float v = 0.0f;
        if (i < natural && wsum[i] > 1e-9) v = (float)__ddiv_rn(acc[i], wsum[i]);
        y[(int64_t)i * ys] = v;
    }
}

template <int NB>
__global__ void __launch_bounds__(VT) k_time_stretch(const float* __restrict__ in, float* __restrict__ out,
                                                     const ClipDesc* __restrict__ desc, int n,
                                                     int logn, int hop_a,
                                                     const double* __restrict__ window,
                                                     const double2* __restrict__ tw_fwd,
                                                     const double2* __restrict__ tw_inv,
                                                     double* __restrict__ work) {
    extern __shared__ double2 buf[];  // [n]
    const ClipDesc d = desc[blockIdx.x];
    if (d.status != 0) return;
    double* acc = work + d.work_off;
    stretch_clip<NB>(in + d.in_off, 1, d.in_len, out + d.out_off, 1, d.target, d.target, d.hop_s,
                 d.frames, d.natural, n, logn, hop_a, window, tw_fwd, tw_inv, buf, acc,
                 acc + d.natural);
}

// ---- the reference's alignment inside the warm-start path (sw_set_align_mode VOCODER)
struct VocReq {
    int64_t src;      // float offset of (slot, channel 0, frame lo, feature 0) in the latent arena
    int32_t t_seg, target, ylim, hop_s, frames, natural, status;
};

// per request: slice_clip frames (simgen.cpp:116-119) and time_stretch's plan
// (vocoder.cpp:139-157) of the segment clip at the latent frame rate
__global__ void k_voc_plan(const sw_choice* __restrict__ ch, const sw_request* __restrict__ rq,
                           int B, int rank, const int32_t* __restrict__ tsrc, int64_t Lslots,
                           int C, int Tmax, int F, int fps, int t_out_max, int n, int hop_a,
                           VocReq* __restrict__ vr, int32_t* __restrict__ ok) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    VocReq v{};
    v.status = 1;
    const sw_choice c = ch[b];
    if (c.hit && (rank < 0 || c.owner == rank)) {
        const int ts = tsrc[c.slot];
        long long lo = llround(c.segment.start_s * fps);
        long long hi = llround((c.segment.start_s + c.segment.length_s) * fps);
        lo = min(lo, (long long)ts);
        hi = max(min(hi, (long long)ts), lo);
        v.t_seg = (int)(hi - lo);
        const double L = rq[b].duration_s;
        if (v.t_seg > 0 && L > 0.0) {
            const double r = L / ((double)v.t_seg / fps);
            if (r >= 0.4 && r <= 2.5) {  // else the reference throws (pipeline falls back cold)
                v.hop_s = max(1, (int)llround(hop_a * r));
                const long long target = llround(L * fps);
                long long frames_l = 1;
                if (target > n) frames_l = 1 + llround((double)(target - n) / v.hop_s);
                const int frames = (int)max(2LL, frames_l);
                v.target = (int)target;
                v.ylim = min(v.target, t_out_max);
                // frames are causal: output frames [0, ylim) only see frames m with
                // m hop_s < ylim, so the rest (which would write past t_out_max) are skipped
                v.frames = v.ylim > 0 ? min(frames, (v.ylim - 1) / v.hop_s + 1) : 0;
                v.natural = v.frames > 0 ? (v.frames - 1) * v.hop_s + n : 0;
                v.src = ((c.slot % Lslots) * C * (int64_t)Tmax + lo) * F;
                v.status = v.frames > 0 ? 0 : 1;
            }
        }
    }
    vr[b] = v;
    ok[b] = v.status == 0 ? 1 : 0;
}

// one CTA per (request, latent channel (c, f)): the 1-D series latent[c][lo + t][f] stretched to
// llround(L fps) frames -> x0[b][c][t][f]; acc / wsum in dynamic smem after the FFT buffer
template <int NB>
__global__ void __launch_bounds__(VT) k_voc_align(const float* __restrict__ latent,
                                                  const VocReq* __restrict__ vr, int C, int Tmax,
                                                  int F, int t_out_max, float* __restrict__ out,
                                                  int n, int logn, int hop_a,
                                                  const double* __restrict__ window,
                                                  const double2* __restrict__ tw_fwd,
                                                  const double2* __restrict__ tw_inv) {
    extern __shared__ double2 buf[];
    const int b = blockIdx.y, ch = blockIdx.x;
    const VocReq v = vr[b];
    if (v.status != 0) return;
    const int c = ch / F, f = ch % F;
    double* acc = reinterpret_cast<double*>(buf + n);
    const float* x = latent + v.src + (int64_t)c * Tmax * F + f;
    float* y = out + ((int64_t)b * C + c) * t_out_max * F + f;
    stretch_clip<NB>(x, F, v.t_seg, y, F, v.ylim, v.target, v.hop_s, v.frames, v.natural, n, logn,
                 hop_a, window, tw_fwd, tw_inv, buf, acc, acc + v.natural);
}

struct Tables {
    double* window = nullptr;
    double2* tw_fwd = nullptr;
    double2* tw_inv = nullptr;
};

// Hann window and the FFT twiddle recurrences, evaluated on the host exactly as the reference
// does (vocoder.cpp:27-35, 46-52), once per (device, N).
Tables tables_for(int n) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, Tables> cache;
    int dev = 0;
    SW_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({dev, n});
    if (it != cache.end()) return it->second;
    std::vector<double> w((size_t)n);
    for (int i = 0; i < n; ++i) w[(size_t)i] = 0.5 * (1.0 - std::cos(2.0 * M_PI * i / n));
    std::vector<double2> tf, ti;
    for (int dir = 0; dir < 2; ++dir) {
        auto& t = dir ? ti : tf;
        const bool inverse = dir == 1;
        for (int len = 2; len <= n; len <<= 1) {
            const double ang = 2.0 * M_PI / static_cast<double>(len) * (inverse ? 1.0 : -1.0);
            const std::complex<double> wlen(std::cos(ang), std::sin(ang));
            std::complex<double> cw(1.0, 0.0);
            for (int j = 0; j < len / 2; ++j) {
                t.push_back(make_double2(cw.real(), cw.imag()));
                // w *= wlen with the reference's finite-value complex product (ac - bd, ad + bc)
                const double a = cw.real(), b = cw.imag(), c = wlen.real(), e = wlen.imag();
                cw = std::complex<double>(a * c - b * e, a * e + b * c);
            }
        }
    }
    Tables tb;
    SW_CUDA(cudaMalloc(&tb.window, sizeof(double) * n));
    SW_CUDA(cudaMalloc(&tb.tw_fwd, sizeof(double2) * tf.size()));
    SW_CUDA(cudaMalloc(&tb.tw_inv, sizeof(double2) * ti.size()));
    SW_CUDA(cudaMemcpy(tb.window, w.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
    SW_CUDA(cudaMemcpy(tb.tw_fwd, tf.data(), sizeof(double2) * tf.size(), cudaMemcpyHostToDevice));
    SW_CUDA(cudaMemcpy(tb.tw_inv, ti.data(), sizeof(double2) * ti.size(), cudaMemcpyHostToDevice));
    // the legacy-stream copies do not order against the caller's (non-blocking) stream: make
    // the tables complete before any kernel reads them (once per device and window)
    SW_CUDA(cudaDeviceSynchronize());
    cache[{dev, n}] = tb;
    return tb;
}

}  // namespace

// Host-side planning of time_stretch (vocoder.cpp:128-157) for one clip: status 0 or SW_EINVAL
// (the reference throws std::invalid_argument), output length, synthesis hop, frame count.
static ClipDesc plan_clip(int in_len, int rate, double target_s, int n, int hop_a) {
    ClipDesc d{};
    d.in_len = in_len;
    if (in_len <= 0 || !(target_s > 0.0) || rate <= 0) {
        d.status = SW_EINVAL;
        return d;
    }
    const double in_duration = static_cast<double>(in_len) / rate;
    const double r = target_s / in_duration;
    if (r < 0.4 || r > 2.5) {
        d.status = SW_EINVAL;
        return d;
    }
    d.hop_s = std::max(1, static_cast<int>(std::llround(hop_a * r)));
    const long long target = std::llround(target_s * rate);
    long frames_l = 1;
    if (target > n) frames_l = 1 + std::lround(static_cast<double>(target - n) / d.hop_s);
    d.frames = (int)std::max(2L, frames_l);
    d.natural = (d.frames - 1) * d.hop_s + n;
    d.target = (int)target;
    return d;
}

int time_stretch_batch(const float* d_in, const int64_t* in_off, const int32_t* in_len, int B,
                       int rate, const double* target_s, int n, int hop_a, float* d_out,
                       int64_t out_cap, int64_t* out_off, int32_t* out_len, int32_t* status,
                       cudaStream_t st) {
    SW_REQUIRE(n >= 2 && (n & (n - 1)) == 0 && n <= kMaxWin,
               "stft window size must be a power of two >= 2 (at most 1024 here)");  // :9-15
    SW_REQUIRE(hop_a >= 1 && hop_a <= n, "stft hop must be in (0, window_size]");
    std::vector<ClipDesc> desc((size_t)B);
    int64_t o = 0, work = 0;
    for (int b = 0; b < B; ++b) {
        ClipDesc d = plan_clip(in_len[b], rate, target_s[b], n, hop_a);
        d.in_off = in_off[b];
        d.out_off = o;
        d.work_off = work;
        if (d.status == 0) {
            o += d.target;
            work += 2 * (int64_t)d.natural;
        }
        out_off[b] = d.out_off;
        out_len[b] = d.status == 0 ? d.target : 0;
        status[b] = d.status;
        desc[(size_t)b] = d;
    }
    SW_REQUIRE(o <= out_cap, "output buffer too small for the stretched clips");
    if (B == 0) return 0;
    const Tables tb = tables_for(n);
    ClipDesc* d_desc = nullptr;
    double* d_work = nullptr;
    SW_CUDA(cudaMallocAsync(&d_desc, sizeof(ClipDesc) * B, st));
    SW_CUDA(cudaMallocAsync(&d_work, sizeof(double) * std::max<int64_t>(work, 1), st));
    SW_CUDA(cudaMemcpyAsync(d_desc, desc.data(), sizeof(ClipDesc) * B, cudaMemcpyHostToDevice, st));
    int logn = 0;
    while ((1 << logn) < n) ++logn;
    auto go = [&](auto kern) {
        kern<<<B, VT, sizeof(double2) * n, st>>>(d_in, d_out, d_desc, n, logn, hop_a, tb.window,
                                                 tb.tw_fwd, tb.tw_inv, d_work);
    };
    // smallest NB with NB * VT > n / 2 (bins 0..n/2): registers 64 (n <= 254) .. 158 (n = 1024)
    if (n / 2 < 2 * VT) go(k_time_stretch<2>);
    else if (n / 2 < 3 * VT) go(k_time_stretch<3>);
    else if (n / 2 < 5 * VT) go(k_time_stretch<5>);
    else go(k_time_stretch<9>);
    SW_CUDA(cudaGetLastError());
    SW_CUDA(cudaFreeAsync(d_desc, st));
    SW_CUDA(cudaFreeAsync(d_work, st));
    return 1;
}

// The reference's alignment (slice_clip + time_stretch, pipeline.cpp:158-169) of the chosen
// latent to the requested duration, per latent channel, written as x0 into d_out; the caller
// then applies the forward noising in place (align.cu, k_noise_inplace). Requests whose stretch
// ratio falls outside [0.4, 2.5] (the reference throws; its pipeline serves them cold) are
// left untouched. Returns the per-request "aligned" flags (stream-ordered device scratch).
const int32_t* launch_align_vocoder(Ctx& c, const sw_choice* d_ch, const sw_request* d_req,
                                    int B, int rank, float* d_out, int t_out_max,
                                    cudaStream_t st) {
    const int n = c.voc_win, hop_a = c.voc_hop;
    const int fps = (int)llround(c.cfg.latent_fps);
    SW_REQUIRE(std::fabs(c.cfg.latent_fps - fps) < 1e-12,
               "the vocoder alignment needs an integral latent frame rate (AudioClip::sample_rate)");
    const Tables tb = tables_for(n);
    if (!c.d_voc || c.voc_cap < B) {
        cudaFree(c.d_voc);
        c.voc_cap = c.Bmax;
        SW_CUDA(cudaMalloc(&c.d_voc, (sizeof(VocReq) + sizeof(int32_t)) * c.voc_cap));
    }
    VocReq* vr = reinterpret_cast<VocReq*>(c.d_voc);
    int32_t* ok = reinterpret_cast<int32_t*>(vr + c.voc_cap);
    k_voc_plan<<<(B + 127) / 128, 128, 0, st>>>(d_ch, d_req, B, rank, c.tsrc, c.Lslots, c.C, c.Tmax,
                                                c.F, fps, t_out_max, n, hop_a, vr, ok);
    int logn = 0;
    while ((1 << logn) < n) ++logn;
    const size_t nat_bound = (size_t)t_out_max + n + 1;  // natural <= ylim - 1 + n
    const size_t smem = sizeof(double2) * n + 2 * sizeof(double) * nat_bound;
    SW_REQUIRE(smem <= 200 * 1024, "vocoder alignment: stretched latent too long for smem");
    auto go = [&](auto kern) {
        ensure_smem_attr(c, kern, smem);
        kern<<<dim3(c.C * c.F, B), VT, smem, st>>>(c.latent, vr, c.C, c.Tmax, c.F, t_out_max,
                                                    d_out, n, logn, hop_a, tb.window, tb.tw_fwd,
                                                    tb.tw_inv);
    };
    // smallest NB with NB * VT > n / 2 (bins 0..n/2): registers 64 (n <= 254) .. 158 (n = 1024)
    if (n / 2 < 2 * VT) go(k_voc_align<2>);
    else if (n / 2 < 3 * VT) go(k_voc_align<3>);
    else if (n / 2 < 5 * VT) go(k_voc_align<5>);
    else go(k_voc_align<9>);
    SW_CUDA(cudaGetLastError());
    return ok;
}

}  // namespace sw
