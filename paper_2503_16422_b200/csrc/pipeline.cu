// pipeline.cu -- fdgs_pipeline_*: host-side submission of a batch of frames
// over a pipeline of render workspaces (include/fdgs.h).
//
// Frame k of a batch renders in workspace slot k mod depth: its front end on
// the slot's (high-priority) front stream, its blend on the slot's blend
// stream (fdgs_render_split), the slot's next frame ordered after this blend.
// The ~20 launches of a frame cost ~60 us of host time (CUDA API calls), a
// third of the frame's device time at C3.  One call submits the whole batch,
// in frame order on the caller's thread by default; optionally worker threads
// owned by the handle issue it in parallel (one group of slots per thread),
// which cuts the host time but measurably slows the device's scheduling of the
// 12 streams.  Every slot's frames are issued in
// order by one thread, so stream order alone orders their work; threads share
// only the copy streams (independent copies).
#include <algorithm>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include "fdgs_internal.h"

using namespace fdgs;

struct fdgs_pipeline {
    int device = 0;
    int depth = 0;
    std::vector<fdgs_pipeline_slot> slots;
    std::vector<cudaStream_t> copies;
    std::vector<cudaEvent_t> done_ev, fin_ev, split_ev, join_ev;  // per slot (join: per stream)
    cudaEvent_t start_ev = nullptr;
    // worker pool
    int n_threads = 1;
    std::vector<std::thread> workers;
    std::mutex m;
    std::condition_variable cv_work, cv_done;
    uint64_t generation = 0;
    int pending = 0;
    bool stop = false;
    // the batch being submitted
    const fdgs_frame_job *jobs = nullptr;
    int32_t n_jobs = 0;
    void *const *stage_events = nullptr;
    fdgs_status err = FDGS_OK;
    char err_msg[512] = "";
};

namespace {

void record_error(fdgs_pipeline *p, fdgs_status s) {
    std::lock_guard<std::mutex> g(p->m);
    if (p->err == FDGS_OK) {
        p->err = s;
        std::snprintf(p->err_msg, sizeof p->err_msg, "%s", fdgs_last_error());
    }
}

fdgs_status cuda_status(cudaError_t e, const char *where) {
    if (e == cudaSuccess) return FDGS_OK;
    char buf[256];
    std::snprintf(buf, sizeof buf, "%s: %s", where, cudaGetErrorString(e));
    return set_error(FDGS_ERR_CUDA, buf);  // this thread's fdgs_last_error()
}

// Issue every frame of the batch whose slot belongs to worker w (of nw).
fdgs_status submit(fdgs_pipeline *p, int w, int nw) {
    std::vector<int> seen(p->depth, 0);
    for (int32_t k = 0; k < p->n_jobs; ++k) {
        const int s = k % p->depth;
        if (s % nw != w) continue;
        const fdgs_frame_job &J = p->jobs[k];
        const fdgs_pipeline_slot &S = p->slots[s];
        cudaStream_t front = (cudaStream_t)S.front_stream;
        cudaStream_t blend = (cudaStream_t)S.blend_stream;
        cudaStream_t last = blend ? blend : front;
        cudaError_t e;
        if (seen[s]++) {  // the slot's previous frame must have left the workspace
            if ((e = cudaEventRecord(p->done_ev[s], last)) != cudaSuccess) return cuda_status(e, "record");
            if ((e = cudaStreamWaitEvent(front, p->done_ev[s], 0)) != cudaSuccess) return cuda_status(e, "wait");
        }
        void *const *evs = p->stage_events ? p->stage_events + 5 * (size_t)k : nullptr;
        fdgs_status st =
            S.graph != nullptr && J.d_stats == nullptr
                ? fdgs_render_graph_launch_timed(S.graph, &J.scene, J.d_mask_l, J.d_mask_r, &J.cam, J.t, J.d_out_rgb,
                                                 J.d_out_T, S.front_stream, S.blend_stream,
                                                 blend ? (void *)p->split_ev[s] : nullptr, evs)
            : blend ? fdgs_render_split(&J.scene, J.d_mask_l, J.d_mask_r, &J.cam, J.t, J.d_out_rgb,
                                                   J.d_out_T, S.d_ws, S.ws_bytes, S.max_entries, J.d_stats,
                                                   S.front_stream, S.blend_stream, (void *)p->split_ev[s], evs)
                               : fdgs_render_timed(&J.scene, J.d_mask_l, J.d_mask_r, &J.cam, J.t, J.d_out_rgb,
                                                   J.d_out_T, S.d_ws, S.ws_bytes, S.max_entries, J.d_stats,
                                                   S.front_stream, evs);
        if (st != FDGS_OK) return st;
        if (J.d_status != nullptr) {  // the frame's counter block, before the workspace is reused
            fdgs_debug_views v;
            st = fdgs_render_debug_views(S.d_ws, S.ws_bytes, std::max(J.scene.n, J.scene.n_capacity), J.cam.width,
                                         J.cam.height, S.max_entries, &v);
            if (st != FDGS_OK) return st;
            if ((e = cudaMemcpyAsync(J.d_status, v.counters, 16, cudaMemcpyDeviceToDevice, last)) != cudaSuccess)
                return cuda_status(e, "status copy");
        }
        if (J.done_event != nullptr && (e = cudaEventRecord((cudaEvent_t)J.done_event, last)) != cudaSuccess)
            return cuda_status(e, "done event");
        if (J.h_out_rgb != nullptr) {  // D2H of the finished frame on a copy stream
            if (p->copies.empty()) return set_error(FDGS_ERR_INVALID_ARG, "h_out_rgb needs a copy stream");
            cudaStream_t cp = p->copies[k % p->copies.size()];
            if ((e = cudaEventRecord(p->fin_ev[s], last)) != cudaSuccess) return cuda_status(e, "record");
            if ((e = cudaStreamWaitEvent(cp, p->fin_ev[s], 0)) != cudaSuccess) return cuda_status(e, "wait");
            const size_t bytes = sizeof(float) * 3 * (size_t)J.cam.width * J.cam.height;
            if ((e = cudaMemcpyAsync(J.h_out_rgb, J.d_out_rgb, bytes, cudaMemcpyDeviceToHost, cp)) != cudaSuccess)
                return cuda_status(e, "frame copy");
        }
    }
    return FDGS_OK;
}

void worker_main(fdgs_pipeline *p, int w) {
    cudaSetDevice(p->device);
    uint64_t seen = 0;
    for (;;) {
        {
            std::unique_lock<std::mutex> lk(p->m);
            p->cv_work.wait(lk, [&] { return p->stop || p->generation != seen; });
            if (p->stop) return;
            seen = p->generation;
        }
        const fdgs_status st = submit(p, w, p->n_threads);
        if (st != FDGS_OK) record_error(p, st);
        {
            std::lock_guard<std::mutex> g(p->m);
            if (--p->pending == 0) p->cv_done.notify_all();
        }
    }
}

void destroy_events(fdgs_pipeline *p) {
    for (auto *v : {&p->done_ev, &p->fin_ev, &p->split_ev, &p->join_ev})
        for (cudaEvent_t e : *v)
            if (e) cudaEventDestroy(e);
    if (p->start_ev) cudaEventDestroy(p->start_ev);
}

}  // namespace

extern "C" {

fdgs_status fdgs_pipeline_create(const fdgs_pipeline_slot *slots, int32_t depth, void *const *copy_streams,
                                 int32_t n_copy, int32_t n_threads, fdgs_pipeline **out) {
    if (out == nullptr) return set_error(FDGS_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (slots == nullptr || depth < 1 || depth > 64 || n_copy < 0 || (n_copy > 0 && copy_streams == nullptr) ||
        n_threads < 1 || n_threads > 64)
        return set_error(FDGS_ERR_INVALID_ARG, "slots / depth in [1, 64] / copy streams / n_threads in [1, 64]");
    for (int s = 0; s < depth; ++s)
        if (slots[s].d_ws == nullptr || slots[s].front_stream == nullptr)
            return set_error(FDGS_ERR_INVALID_ARG, "a slot without workspace or front stream");
    fdgs_pipeline *p = new (std::nothrow) fdgs_pipeline();
    if (p == nullptr) return set_error(FDGS_ERR_CUDA, "out of host memory");
    cudaGetDevice(&p->device);
    p->depth = depth;
    p->slots.assign(slots, slots + depth);
    for (int c = 0; c < n_copy; ++c) p->copies.push_back((cudaStream_t)copy_streams[c]);
    cudaError_t e = cudaEventCreateWithFlags(&p->start_ev, cudaEventDisableTiming);
    for (auto *v : {&p->done_ev, &p->fin_ev, &p->split_ev}) {
        v->resize(depth, nullptr);
        for (int s = 0; s < depth && e == cudaSuccess; ++s) e = cudaEventCreateWithFlags(&(*v)[s], cudaEventDisableTiming);
    }
    p->join_ev.resize(2 * depth + p->copies.size(), nullptr);
    for (auto &ev : p->join_ev)
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        destroy_events(p);
        delete p;
        return cuda_status(e, "fdgs_pipeline_create");
    }
    p->n_threads = std::min(n_threads, depth);
    if (p->n_threads > 1)
        for (int w = 0; w < p->n_threads; ++w) p->workers.emplace_back(worker_main, p, w);
    *out = p;
    return FDGS_OK;
}

fdgs_status fdgs_pipeline_render(fdgs_pipeline *p, const fdgs_frame_job *jobs, int32_t n_jobs, void *stream,
                                 void *const *stage_events) {
    if (p == nullptr || n_jobs < 0 || (n_jobs > 0 && jobs == nullptr))
        return set_error(FDGS_ERR_INVALID_ARG, "pipeline / jobs");
    cudaStream_t main = (cudaStream_t)stream;
    cudaError_t e = cudaEventRecord(p->start_ev, main);  // every stream starts after the caller's work
    std::vector<cudaStream_t> streams;
    for (const auto &S : p->slots) {
        streams.push_back((cudaStream_t)S.front_stream);
        if (S.blend_stream) streams.push_back((cudaStream_t)S.blend_stream);
    }
    for (cudaStream_t c : p->copies) streams.push_back(c);
    for (cudaStream_t s : streams)
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, p->start_ev, 0);
    if (e != cudaSuccess) return cuda_status(e, "fdgs_pipeline_render");
    p->jobs = jobs;
    p->n_jobs = n_jobs;
    p->stage_events = stage_events;
    p->err = FDGS_OK;
    fdgs_status st = FDGS_OK;
    if (p->workers.empty()) {
        st = submit(p, 0, 1);
    } else {
        {
            std::lock_guard<std::mutex> g(p->m);
            p->pending = (int)p->workers.size();
            ++p->generation;
        }
        p->cv_work.notify_all();
        std::unique_lock<std::mutex> lk(p->m);
        p->cv_done.wait(lk, [&] { return p->pending == 0; });
        st = p->err;
    }
    // the caller's stream waits for every frame and copy of the batch
    for (size_t i = 0; i < streams.size() && e == cudaSuccess; ++i) {
        e = cudaEventRecord(p->join_ev[i], streams[i]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(main, p->join_ev[i], 0);
    }
    if (st != FDGS_OK) return p->workers.empty() ? st : set_error(st, p->err_msg);  // the worker's message
    return e == cudaSuccess ? FDGS_OK : cuda_status(e, "fdgs_pipeline_render");
}

fdgs_status fdgs_pipeline_destroy(fdgs_pipeline *p) {
    if (p == nullptr) return FDGS_OK;
    {
        std::lock_guard<std::mutex> g(p->m);
        p->stop = true;
    }
    p->cv_work.notify_all();
    for (auto &t : p->workers) t.join();
    destroy_events(p);
    delete p;
    return FDGS_OK;
}

}  // extern "C"
