// ss_sched.cu — native batch formation and dispatch (the reference executor's scheduler loop,
// executor.py:162-178 submit, 235-283 _loop / _pick_ready, 285-300 _dispatch) on a C++ thread.
//
// Client threads queue DEVICE-resident requests and block in ss_sched_request / ss_sched_wait
// without the Python GIL; one scheduler thread picks ripe queues under the BatchPolicy, makes
// its stream wait for each request's `ready` event, runs ss_compute_batch (public ABI, which
// holds the context lock) and records one completion event per batch. Waiters make their own
// stream wait for that event, so nothing on the device side is serialised beyond stream order.
// Contract: include/ss_b200.h (ss_sched_*).
#include <cuda_runtime.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/ss_b200.h"

namespace {

using Clock = std::chrono::steady_clock;

constexpr int kDoneEvents = 64;   // completion events, reused round-robin (see dispatch)

struct Pending {
  uint64_t ticket;
  ss_request req;
  Clock::time_point arrived;
  bool notify;
};

struct Queue {
  int block, role, pass;
  std::deque<Pending> q;
};

struct Done {
  int32_t status = 0;
  int64_t aux = 0;
  int ev = -1;         // completion event slot (-1: nothing to wait for: rejected at intake)
};

}  // namespace

struct ss_sched {
  ss_ctx* ctx = nullptr;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ss_sched_policy pol{};
  std::mutex mu;
  std::condition_variable cv_work, cv_done;
  std::vector<Queue> queues;                       // first-seen order (the reference's dict order)
  std::map<std::tuple<int, int, int>, size_t> qidx;
  std::map<uint32_t, bool> clients;                // registered -> sends_backward
  std::unordered_map<uint32_t, uint64_t> last_id;  // submit(): request_id strictly increasing
  std::map<std::pair<int, int>, bool> known_layers; // intake's layer check, cached (no ctx lock)
  std::unordered_map<uint64_t, Done> done;         // completed tickets not yet collected
  std::unordered_map<uint64_t, bool> outstanding;  // ticket -> notify, queued or in flight
  std::deque<uint64_t> notify_done;                // completion order of notify tickets
  std::vector<ss_sched_rec> log;
  cudaEvent_t ev[kDoneEvents] = {};
  int ev_next = 0;
  uint64_t next_ticket = 1;
  uint64_t dispatch_seq = 0;
  int64_t queued = 0;
  bool running = false, drain = true;
  std::string err;
  std::thread th;
};

namespace {

double wait_budget(const ss_sched_policy& p, int64_t min_tokens) {
  const double w = p.wait_per_token * (double)min_tokens;
  return w < p.wait_cap ? w : p.wait_cap;
}

// executor.py:247-283. Returns the index of a queue to dispatch now, or -1 and (in *sleep) the
// time until the earliest opportunistic deadline (negative: nothing queued).
long pick_ready(ss_sched* s, Clock::time_point now, double* sleep) {
  *sleep = -1.0;
  for (size_t i = 0; i < s->queues.size(); ++i) {
    Queue& Q = s->queues[i];
    if (Q.q.empty()) continue;
    if (Q.pass == SS_PASS_NOISE_EFFECT || s->pol.mode == SS_SCHED_NOLOCKSTEP) return (long)i;
    if (s->pol.mode == SS_SCHED_LOCKSTEP) {
      bool all = true;
      for (const auto& c : s->clients) {
        if (Q.pass != SS_PASS_FORWARD && !c.second) continue;
        bool have = false;
        for (const Pending& p : Q.q)
          if (p.req.client_id == c.first) { have = true; break; }
        if (!have) { all = false; break; }
      }
      if (all) return (long)i;
      continue;
    }
    int64_t tokens = 0, min_tokens = INT64_MAX;
    Clock::time_point oldest = Q.q.front().arrived;
    for (const Pending& p : Q.q) {
      tokens += p.req.seg.rows;
      if ((int64_t)p.req.seg.rows < min_tokens) min_tokens = p.req.seg.rows;
      if (p.arrived < oldest) oldest = p.arrived;
    }
    if (tokens >= s->pol.max_batch_tokens) return (long)i;
    const double age = std::chrono::duration<double>(now - oldest).count();
    const double left = wait_budget(s->pol, min_tokens) - age;
    if (left <= 0) return (long)i;
    if (*sleep < 0 || left < *sleep) *sleep = left;
  }
  return -1;
}

// called with s->mu held
void complete(ss_sched* s, const Pending& p, int32_t status, int64_t aux, int ev) {
  Done& d = s->done[p.ticket];
  d.status = status;
  d.aux = aux;
  d.ev = ev;
  auto it = s->outstanding.find(p.ticket);
  if (it != s->outstanding.end()) {
    if (it->second) s->notify_done.push_back(p.ticket);
    s->outstanding.erase(it);
  }
}

void dispatch(ss_sched* s, std::vector<Pending>& batch, Clock::time_point picked) {
  const Pending& first = batch.front();
  const int block = first.req.block, role = first.req.role, pass = (int)first.req.pass_kind;
  std::vector<ss_seg> segs(batch.size());
  std::vector<int32_t> st(batch.size(), 0);
  cudaSetDevice(s->device);
  int rc = SS_OK;
  for (size_t i = 0; i < batch.size(); ++i) {
    segs[i] = batch[i].req.seg;
    segs[i].client_id = batch[i].req.client_id;
    if (batch[i].req.ready &&
        cudaStreamWaitEvent(s->stream, (cudaEvent_t)batch[i].req.ready, 0) != cudaSuccess)
      rc = SS_E_CUDA;
  }
  std::string msg;
  if (rc == SS_OK) {
    rc = ss_compute_batch(s->ctx, pass, block, role, (int)segs.size(), segs.data(), s->stream, st.data());
    if (rc != SS_OK) msg = ss_last_error(s->ctx);
  } else {
    cudaGetLastError();
    msg = "cudaStreamWaitEvent on a request's ready event failed";
  }
  std::lock_guard<std::mutex> g(s->mu);
  // one completion event per batch, recorded under the lock so that a waiter's stream-wait
  // (also under the lock) always sees this record or a later one of the same slot — a later
  // record completes after this batch (same stream), so waiting on it is still correct
  const int ev = s->ev_next;
  s->ev_next = (s->ev_next + 1) % kDoneEvents;
  if (cudaEventRecord(s->ev[ev], s->stream) != cudaSuccess && rc == SS_OK) {
    rc = SS_E_CUDA;
    msg = "cudaEventRecord failed";
  }
  if (rc != SS_OK) s->err = msg;
  const uint64_t seq = ++s->dispatch_seq;
  for (size_t i = 0; i < batch.size(); ++i) {
    const Pending& p = batch[i];
    complete(s, p, rc == SS_OK ? st[i] : SS_REQ_FAILED, rc, ev);
    ss_sched_rec r;
    r.dispatch = seq;
    r.block = block;
    r.role = role;
    r.pass_kind = pass;
    r.rows = (int32_t)p.req.seg.rows;
    r.wait_s = std::chrono::duration<double>(picked - p.arrived).count();
    if (s->log.size() < (1u << 20)) s->log.push_back(r);
  }
  s->queued -= (int64_t)batch.size();
  s->cv_done.notify_all();
}

void loop(ss_sched* s) {
  cudaSetDevice(s->device);
  std::unique_lock<std::mutex> lk(s->mu);
  for (;;) {
    double sleep = -1.0;
    const auto now = Clock::now();
    long qi = pick_ready(s, now, &sleep);
    if (qi < 0 && !s->running) {
      // stopping: a drain dispatches what is left whatever the policy; otherwise fail it
      for (size_t i = 0; i < s->queues.size() && qi < 0; ++i)
        if (!s->queues[i].q.empty()) qi = (long)i;
      if (qi >= 0 && !s->drain) {
        for (Queue& Q : s->queues) {
          for (const Pending& p : Q.q) complete(s, p, SS_REQ_FAILED, 0, -1);
          s->queued -= (int64_t)Q.q.size();
          Q.q.clear();
        }
        s->err = "scheduler stopped";
        s->cv_done.notify_all();
        qi = -1;
      }
      if (qi < 0) return;
    }
    if (qi < 0) {
      if (sleep < 0) s->cv_work.wait(lk);
      else s->cv_work.wait_for(lk, std::chrono::duration<double>(sleep));
      continue;
    }
    Queue& Q = s->queues[(size_t)qi];
    std::vector<Pending> batch;
    if (Q.pass == SS_PASS_NOISE_EFFECT || s->pol.mode == SS_SCHED_NOLOCKSTEP) {
      batch.push_back(Q.q.front());
      Q.q.pop_front();
    } else {
      batch.assign(Q.q.begin(), Q.q.end());
      Q.q.clear();
    }
    lk.unlock();
    dispatch(s, batch, now);
    lk.lock();
  }
}

int wait_locked(ss_sched* s, std::unique_lock<std::mutex>& lk, uint64_t ticket, void* wait_stream,
                int64_t timeout_us, int32_t* status, int64_t* aux) {
  auto ready = [&] { return s->done.count(ticket) != 0; };
  if (!ready()) {
    if (!s->outstanding.count(ticket)) return SS_E_ARG;
    if (timeout_us < 0) s->cv_done.wait(lk, ready);
    else if (!s->cv_done.wait_for(lk, std::chrono::microseconds(timeout_us), ready)) return 1;
  }
  Done d = s->done[ticket];
  s->done.erase(ticket);
  if (d.ev >= 0 && wait_stream) cudaStreamWaitEvent((cudaStream_t)wait_stream, s->ev[d.ev], 0);
  if (status) *status = d.status;
  if (aux) *aux = d.aux;
  return SS_OK;
}

}  // namespace

extern "C" {

int ss_sched_create(ss_ctx* ctx, const ss_sched_policy* policy, void* stream, ss_sched** out) {
  if (!ctx || !policy || !out) return SS_E_ARG;
  *out = nullptr;
  if (policy->mode < 0 || policy->mode > 2) return SS_E_ARG;
  ss_sched* s = new ss_sched();
  s->ctx = ctx;
  s->device = ss_ctx_device(ctx);
  s->pol = *policy;
  cudaSetDevice(s->device);
  if (stream) {
    s->stream = (cudaStream_t)stream;
  } else {
    if (cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete s;
      return SS_E_CUDA;
    }
    s->own_stream = true;
  }
  for (auto& e : s->ev) {
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
      for (auto& f : s->ev) if (f) cudaEventDestroy(f);
      if (s->own_stream) cudaStreamDestroy(s->stream);
      delete s;
      return SS_E_CUDA;
    }
  }
  s->running = true;
  s->th = std::thread(loop, s);
  *out = s;
  return SS_OK;
}

int ss_sched_destroy(ss_sched* s, int drain) {
  if (!s) return SS_E_ARG;
  {
    std::lock_guard<std::mutex> g(s->mu);
    s->running = false;
    s->drain = drain != 0;
    s->cv_work.notify_all();
  }
  s->th.join();
  cudaSetDevice(s->device);
  cudaStreamSynchronize(s->stream);
  for (auto& e : s->ev) cudaEventDestroy(e);
  if (s->own_stream) cudaStreamDestroy(s->stream);
  delete s;
  return SS_OK;
}

int ss_sched_set_policy(ss_sched* s, const ss_sched_policy* policy) {
  if (!s || !policy || policy->mode < 0 || policy->mode > 2) return SS_E_ARG;
  std::lock_guard<std::mutex> g(s->mu);
  s->pol = *policy;
  s->cv_work.notify_all();
  return SS_OK;
}

int ss_sched_register(ss_sched* s, uint32_t client_id, int sends_backward) {
  if (!s) return SS_E_ARG;
  std::lock_guard<std::mutex> g(s->mu);
  s->clients[client_id] = sends_backward != 0;
  s->cv_work.notify_all();
  return SS_OK;
}

int ss_sched_deregister(ss_sched* s, uint32_t client_id) {
  if (!s) return SS_E_ARG;
  std::lock_guard<std::mutex> g(s->mu);
  s->clients.erase(client_id);
  s->cv_work.notify_all();   // lockstep: a queue may now be complete
  return SS_OK;
}

int ss_sched_submit(ss_sched* s, const ss_request* req, int notify, uint64_t* ticket) {
  if (!s || !req || !ticket) return SS_E_ARG;
  const std::pair<int, int> lk_key(req->block, req->role);
  bool known = false, cached = false;
  {
    std::lock_guard<std::mutex> g(s->mu);
    auto it = s->known_layers.find(lk_key);
    if (it != s->known_layers.end()) cached = true, known = it->second;
  }
  if (!cached) {   // the context lock is taken only the first time a layer is seen
    int d_in = 0, d_out = 0;
    known = ss_layer_dims(s->ctx, req->block, req->role, &d_in, &d_out) == SS_OK;
    std::lock_guard<std::mutex> g(s->mu);
    s->known_layers[lk_key] = known;
  }
  std::lock_guard<std::mutex> g(s->mu);
  Pending p;
  p.ticket = s->next_ticket++;
  p.req = *req;
  p.arrived = Clock::now();
  p.notify = notify != 0;
  *ticket = p.ticket;
  s->outstanding[p.ticket] = p.notify;
  // submit() checks, in the reference's order (executor.py:162-178)
  if (req->pass_kind > SS_PASS_NOISE_EFFECT) {
    complete(s, p, SS_REQ_BAD_PASS, 0, -1);
  } else {
    auto it = s->last_id.find(req->client_id);
    if (it != s->last_id.end() && req->request_id <= it->second) {
      complete(s, p, SS_REQ_BAD_ID, (int64_t)it->second, -1);
    } else {
      s->last_id[req->client_id] = req->request_id;
      if (!known) {
        complete(s, p, SS_REQ_NO_LAYER, 0, -1);
      } else {
        const auto key = std::make_tuple((int)req->block, (int)req->role, (int)req->pass_kind);
        auto qi = s->qidx.find(key);
        size_t idx;
        if (qi == s->qidx.end()) {
          idx = s->queues.size();
          s->queues.push_back(Queue{req->block, req->role, (int)req->pass_kind, {}});
          s->qidx[key] = idx;
        } else {
          idx = qi->second;
        }
        s->queues[idx].q.push_back(p);
        s->queued++;
        s->cv_work.notify_all();
        return SS_OK;
      }
    }
  }
  s->cv_done.notify_all();
  return SS_OK;
}

int ss_sched_wait(ss_sched* s, uint64_t ticket, void* wait_stream, int64_t timeout_us,
                  int32_t* status, int64_t* aux) {
  if (!s) return SS_E_ARG;
  std::unique_lock<std::mutex> lk(s->mu);
  return wait_locked(s, lk, ticket, wait_stream, timeout_us, status, aux);
}

int ss_sched_request(ss_sched* s, const ss_request* req, void* wait_stream, int64_t timeout_us,
                     int32_t* status, int64_t* aux) {
  uint64_t ticket = 0;
  int rc = ss_sched_submit(s, req, 0, &ticket);
  if (rc) return rc;
  return ss_sched_wait(s, ticket, wait_stream, timeout_us, status, aux);
}

int ss_sched_next_done(ss_sched* s, void* wait_stream, int64_t timeout_us, uint64_t* ticket,
                       int32_t* status, int64_t* aux) {
  if (!s || !ticket) return SS_E_ARG;
  std::unique_lock<std::mutex> lk(s->mu);
  auto any = [&] { return !s->notify_done.empty(); };
  if (!any()) {
    if (timeout_us < 0) s->cv_done.wait(lk, any);
    else if (!s->cv_done.wait_for(lk, std::chrono::microseconds(timeout_us), any)) return 1;
  }
  *ticket = s->notify_done.front();
  s->notify_done.pop_front();
  return wait_locked(s, lk, *ticket, wait_stream, 0, status, aux);
}

int ss_sched_log(ss_sched* s, ss_sched_rec* out, int cap, int* n) {
  if (!s || !n || (cap > 0 && !out)) return SS_E_ARG;
  std::lock_guard<std::mutex> g(s->mu);
  const size_t k = std::min<size_t>((size_t)(cap > 0 ? cap : 0), s->log.size());
  if (k) std::memcpy(out, s->log.data(), k * sizeof(ss_sched_rec));
  s->log.erase(s->log.begin(), s->log.begin() + (long)k);
  *n = (int)k;
  return SS_OK;
}

int64_t ss_sched_queued(ss_sched* s) {
  if (!s) return -1;
  std::lock_guard<std::mutex> g(s->mu);
  return s->queued;
}

const char* ss_sched_last_error(ss_sched* s) { return s ? s->err.c_str() : "null scheduler"; }

}  // extern "C"
