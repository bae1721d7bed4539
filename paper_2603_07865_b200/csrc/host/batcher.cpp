// Request batching in front of the warm-start path — SURVEY §8f row 4.
//
// The reference serves one request per client thread: the socket server runs
// Pipeline::handle_request per connection (server.cpp:83, :149), each plan_request a B = 1
// search under a shared lock (pipeline.cpp:216). On the GPU a B = 1 plan streams the whole bf16
// arena for one query (HBM-bound, ~0.28 ms at 1M entries); above B ~ 250 the tcgen05 scoring is
// tensor-bound and a 1024-request batch costs ~1 ms. swb_* turns concurrent callers into
// device batches: swb_submit (thread-safe, blocking) enqueues one request; a worker thread
// takes up to max_batch queued requests — waiting at most max_wait_us after the oldest one
// arrived for the batch to fill — and runs them as ONE device batch (pinned staging,
// H2D, sw_warmstart (plan + align+noise) or sw_plan, D2H of the choices and, if asked, of the
// aligned latents).
//
// Results do not depend on how requests were grouped: every request's selector draw is keyed
// by (seed, request id) (pipeline.cpp:211), its noise by (philox seed, request id), and the
// cache snapshot is shared by all requests of a batch (the batch-vs-sequential semantics of
// SURVEY H5). tests/test_gpu_batcher.py checks concurrent submitters against one sw_plan.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

#include "semwarm_b200.h"

struct swb_batcher {
    struct Item {
        const float* prompt;
        sw_request req;
        sw_choice* choice;
        float* latent;
        std::chrono::steady_clock::time_point t;
        bool done = false;
        int rc = 0;
    };

    sw_ctx* ctx = nullptr;
    int D = 0, C = 0, T = 0, F = 0;
    int max_batch = 0;
    std::chrono::microseconds max_wait{0};
    uint64_t seed = 0, philox_seed = 0;
    sw_selector_config sel{};
    sw_policy pol{};
    int t_out_max = 0;
    bool with_latent = false;

    std::mutex mu;
    std::condition_variable cv_work, cv_done;
    std::deque<Item*> queue;
    bool stop = false;
    std::thread worker;
    int64_t n_batches = 0, n_requests = 0;

    float* h_q = nullptr;            // pinned [max_batch][D]
    sw_request* h_req = nullptr;     // pinned [max_batch]
    sw_choice* h_choice = nullptr;   // pinned [max_batch]
    float* d_q = nullptr;            // device copies of the batch
    sw_request* d_req = nullptr;
    sw_choice* d_choice = nullptr;
    float* d_lat = nullptr;          // device [max_batch][C][t_out_max][F]
    float* h_lat = nullptr;          // pinned copy of d_lat (with_latent)
    cudaStream_t st = nullptr;

    void run() {
        std::vector<Item*> batch;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu);
                cv_work.wait(lk, [&] { return stop || !queue.empty(); });
                if (queue.empty()) return;  // stop requested and drained
                const auto deadline = queue.front()->t + max_wait;
                while (!stop && (int)queue.size() < max_batch &&
                       cv_work.wait_until(lk, deadline) != std::cv_status::timeout) {
                }
                batch.clear();
                while (!queue.empty() && (int)batch.size() < max_batch) {
                    batch.push_back(queue.front());
                    queue.pop_front();
                }
            }
            const int B = (int)batch.size();
            for (int i = 0; i < B; ++i) {
                std::memcpy(h_q + (size_t)i * D, batch[i]->prompt, sizeof(float) * D);
                h_req[i] = batch[i]->req;
            }
            int rc = SW_OK;
            if (cudaMemcpyAsync(d_q, h_q, sizeof(float) * (size_t)B * D, cudaMemcpyHostToDevice,
                                st) != cudaSuccess ||
                cudaMemcpyAsync(d_req, h_req, sizeof(sw_request) * B, cudaMemcpyHostToDevice,
                                st) != cudaSuccess)
                rc = SW_ECUDA;
            const size_t per = (size_t)C * t_out_max * F;
            if (rc == SW_OK && with_latent)
                cudaMemsetAsync(d_lat, 0, sizeof(float) * per * B, st);
            if (rc == SW_OK)
                rc = d_lat ? sw_warmstart(ctx, d_q, d_req, B, seed, &sel, &pol, nullptr,
                                          philox_seed, d_choice, d_lat, t_out_max, st)
                           : sw_plan(ctx, d_q, d_req, B, seed, &sel, &pol, d_choice, st);
            if (rc == SW_OK &&
                cudaMemcpyAsync(h_choice, d_choice, sizeof(sw_choice) * B, cudaMemcpyDeviceToHost,
                                st) != cudaSuccess)
                rc = SW_ECUDA;
            if (rc == SW_OK && with_latent &&
                cudaMemcpyAsync(h_lat, d_lat, sizeof(float) * per * B, cudaMemcpyDeviceToHost,
                                st) != cudaSuccess)
                rc = SW_ECUDA;
            if (cudaStreamSynchronize(st) != cudaSuccess && rc == SW_OK) rc = SW_ECUDA;
            if (rc == SW_OK && with_latent)
                for (int i = 0; i < B; ++i)
                    if (batch[i]->latent)
                        std::memcpy(batch[i]->latent, h_lat + per * i, sizeof(float) * per);
            {
                std::lock_guard<std::mutex> lk(mu);
                for (int i = 0; i < B; ++i) {
                    if (rc == SW_OK) *batch[i]->choice = h_choice[i];
                    batch[i]->rc = rc;
                    batch[i]->done = true;
                }
                ++n_batches;
                n_requests += B;
            }
            cv_done.notify_all();
        }
    }
};

extern "C" {

int swb_create(sw_ctx* ctx, int32_t max_batch, int32_t max_wait_us, uint64_t seed,
               const sw_selector_config* sel, const sw_policy* pol, uint64_t philox_seed,
               int32_t t_out_max, int32_t with_latent, swb_batcher** out) {
    if (!ctx || !sel || !pol || !out || max_batch < 1 || max_wait_us < 0 || t_out_max < 0)
        return SW_EINVAL;
    int32_t D = 0, C = 0, T = 0, F = 0, bmax = 0, dev = 0;
    if (sw_ctx_info(ctx, &D, &C, &T, &F, &bmax, &dev) != SW_OK) return SW_EINVAL;
    if (max_batch > bmax) return SW_EINVAL;
    auto* b = new swb_batcher;
    b->ctx = ctx;
    b->D = D;
    b->C = C;
    b->T = T;
    b->F = F;
    b->max_batch = max_batch;
    b->max_wait = std::chrono::microseconds(max_wait_us);
    b->seed = seed;
    b->philox_seed = philox_seed;
    b->sel = *sel;
    b->pol = *pol;
    b->t_out_max = C > 0 ? t_out_max : 0;
    b->with_latent = with_latent && C > 0 && t_out_max > 0;
    bool ok = cudaSetDevice(dev) == cudaSuccess &&
              cudaStreamCreateWithFlags(&b->st, cudaStreamNonBlocking) == cudaSuccess &&
              cudaHostAlloc(&b->h_q, sizeof(float) * (size_t)max_batch * D, 0) == cudaSuccess &&
              cudaHostAlloc(&b->h_req, sizeof(sw_request) * max_batch, 0) == cudaSuccess &&
              cudaHostAlloc(&b->h_choice, sizeof(sw_choice) * max_batch, 0) == cudaSuccess &&
              cudaMalloc(&b->d_q, sizeof(float) * (size_t)max_batch * D) == cudaSuccess &&
              cudaMalloc(&b->d_req, sizeof(sw_request) * max_batch) == cudaSuccess &&
              cudaMalloc(&b->d_choice, sizeof(sw_choice) * max_batch) == cudaSuccess;
    const size_t lat = (size_t)max_batch * C * b->t_out_max * F;
    if (ok && lat > 0) ok = cudaMalloc(&b->d_lat, sizeof(float) * lat) == cudaSuccess;
    if (ok && b->with_latent) ok = cudaHostAlloc(&b->h_lat, sizeof(float) * lat, 0) == cudaSuccess;
    if (!ok) {
        swb_destroy(b);
        return SW_ENOMEM;
    }
    b->worker = std::thread([b] {
        int d = 0;
        sw_ctx_info(b->ctx, nullptr, nullptr, nullptr, nullptr, nullptr, &d);
        cudaSetDevice(d);
        b->run();
    });
    *out = b;
    return SW_OK;
}

int swb_destroy(swb_batcher* b) {
    if (!b) return SW_EINVAL;
    {
        std::lock_guard<std::mutex> lk(b->mu);
        b->stop = true;
    }
    b->cv_work.notify_all();
    if (b->worker.joinable()) b->worker.join();
    if (b->st) cudaStreamDestroy(b->st);
    cudaFreeHost(b->h_q);
    cudaFreeHost(b->h_req);
    cudaFreeHost(b->h_choice);
    cudaFreeHost(b->h_lat);
    cudaFree(b->d_lat);
    cudaFree(b->d_q);
    cudaFree(b->d_req);
    cudaFree(b->d_choice);
    delete b;
    return SW_OK;
}

int swb_submit(swb_batcher* b, const float* prompt, const sw_request* req, sw_choice* choice,
               float* latent) {
    if (!b || !prompt || !req || !choice) return SW_EINVAL;
    swb_batcher::Item it;
    it.prompt = prompt;
    it.req = *req;
    it.choice = choice;
    it.latent = latent;
    it.t = std::chrono::steady_clock::now();
    std::unique_lock<std::mutex> lk(b->mu);
    if (b->stop) return SW_EINVAL;
    b->queue.push_back(&it);
    if ((int)b->queue.size() == 1 || (int)b->queue.size() >= b->max_batch) b->cv_work.notify_one();
    b->cv_done.wait(lk, [&] { return it.done; });
    return it.rc;
}

int swb_stats(swb_batcher* b, int64_t* batches, int64_t* requests) {
    if (!b) return SW_EINVAL;
    std::lock_guard<std::mutex> lk(b->mu);
    if (batches) *batches = b->n_batches;
    if (requests) *requests = b->n_requests;
    return SW_OK;
}

// Native load generator: `clients` threads (the reference's thread per connection) each submit
// `per_client` blocking requests, prompt/request (t * per_client + j) mod n of the given pools,
// with fresh request ids. Wall-clock throughput and per-request latency percentiles; the Python
// driver's GIL is not in the loop.
int swb_load_test(swb_batcher* b, const float* prompts, const sw_request* reqs, int32_t n,
                  int32_t clients, int32_t per_client, uint64_t first_id, double* req_per_s,
                  double* p50_ms, double* p99_ms, double* mean_batch) {
    if (!b || !prompts || !reqs || n < 1 || clients < 1 || per_client < 1) return SW_EINVAL;
    std::vector<std::vector<double>> lat((size_t)clients);
    std::vector<int> rc((size_t)clients, SW_OK);
    int64_t b0 = 0, r0 = 0, b1 = 0, r1 = 0;
    swb_stats(b, &b0, &r0);
    const auto t0 = std::chrono::steady_clock::now();
    {
        std::vector<std::thread> th;
        th.reserve((size_t)clients);
        for (int t = 0; t < clients; ++t)
            th.emplace_back([&, t] {
                sw_choice ch;
                lat[t].reserve((size_t)per_client);
                for (int j = 0; j < per_client; ++j) {
                    const int64_t k = (int64_t)t * per_client + j;
                    sw_request rq = reqs[k % n];
                    rq.id = first_id + (uint64_t)k;
                    const auto a = std::chrono::steady_clock::now();
                    const int r = swb_submit(b, prompts + (k % n) * b->D, &rq, &ch, nullptr);
                    const auto z = std::chrono::steady_clock::now();
                    if (r != SW_OK) {
                        rc[t] = r;
                        return;
                    }
                    lat[t].push_back(std::chrono::duration<double, std::milli>(z - a).count());
                }
            });
        for (auto& x : th) x.join();
    }
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (int r : rc)
        if (r != SW_OK) return r;
    swb_stats(b, &b1, &r1);
    std::vector<double> all;
    for (auto& v : lat) all.insert(all.end(), v.begin(), v.end());
    std::sort(all.begin(), all.end());
    if (req_per_s) *req_per_s = (double)all.size() / wall;
    if (p50_ms) *p50_ms = all[all.size() / 2];
    if (p99_ms) *p99_ms = all[std::min(all.size() - 1, (size_t)(all.size() * 0.99))];
    if (mean_batch) *mean_batch = b1 > b0 ? (double)(r1 - r0) / (double)(b1 - b0) : 0.0;
    return SW_OK;
}

}  // extern "C"
