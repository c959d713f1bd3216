// epp-b200: the per-stage executor behind include/epp_gpu.h.
//
// Runs a contiguous range of transformer layers of one pipeline stage on
// heterogeneous EPP chunks (Batched / Split / Hybrid, proj/include/epp/
// chunk.hpp:16-46), with the memory contract the planner assumes
// (proj/src/cost_model.cpp:47-66):
//   * non-checkpointed layers keep full activations until the chunk's
//     backward;  the first `ckpt_layers` layers of the stage keep only their
//     input and are re-run layer by layer right before their backward;
//   * K/V of a long sequence's slices live in a per-(stage, sequence) buffer
//     that later slices attend to (and that checkpointed layers therefore
//     never drop); dK/dV of those keys accumulate in fp32 across the
//     sequence's chunks, whose backwards run last-slice-first
//     (proj/src/pipeline.cpp:119-131);
//   * the buffers are released after the sequence's first slice (context 0)
//     finishes its backward.
// Memory comes from the CUDA stream-ordered allocator on the stage's stream.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "epp_gpu.h"
#include "kernels.h"
#include "profile.h"

namespace eppk {

long long& launch_counter() {
    static long long n = 0;
    return n;
}

std::string& gpu_error_slot() {
    thread_local std::string err;
    return err;
}

namespace {

// ----------------------------------------------------------- allocation ----
struct Pool {
    long long live = 0;
    long long peak = 0;
};

// Activations come from the device's default stream-ordered pool
// (cudaMallocAsync).  With the default release threshold (0) the driver hands
// freed memory back to the OS at every stream/event synchronisation and must
// re-map it on the next step, which shows up as 100s of ms of idle GPU in
// steps whose chunks are larger than the previous step's; a stage keeps its
// high-water mark reserved instead.
inline void keep_pool_reserved() {
    int dev = 0;
    EPP_CUDA(cudaGetDevice(&dev));
    cudaMemPool_t mp;
    EPP_CUDA(cudaDeviceGetDefaultMemPool(&mp, dev));
    uint64_t thr = ~0ull;
    EPP_CUDA(cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr));
}

// Stream-ordered device buffer.
class Buf {
public:
    Buf() = default;
    Buf(Pool* pool, size_t bytes, cudaStream_t s, bool zero = false) : pool_(pool), bytes_(bytes), s_(s) {
        if (bytes_ == 0) return;
        EPP_CUDA(cudaMallocAsync(&p_, bytes_, s_));
        if (zero) EPP_CUDA(cudaMemsetAsync(p_, 0, bytes_, s_));
        pool_->live += static_cast<long long>(bytes_);
        if (pool_->live > pool_->peak) pool_->peak = pool_->live;
    }
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
    Buf(Buf&& o) noexcept { *this = std::move(o); }
    Buf& operator=(Buf&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_; bytes_ = o.bytes_; s_ = o.s_; pool_ = o.pool_;
            o.p_ = nullptr; o.bytes_ = 0;
        }
        return *this;
    }
    ~Buf() { release(); }
    void release() {
        if (p_) {
            cudaFreeAsync(p_, s_);
            pool_->live -= static_cast<long long>(bytes_);
            p_ = nullptr;
            bytes_ = 0;
        }
    }
    template <typename T = void> T* get() const { return static_cast<T*>(p_); }
    explicit operator bool() const { return p_ != nullptr; }

private:
    Pool* pool_ = nullptr;
    void* p_ = nullptr;
    size_t bytes_ = 0;
    cudaStream_t s_ = nullptr;
};

// Pinned host staging for small per-chunk tables (segment descriptors, token
// maps, work lists): a two-half ring so H2D copies stay asynchronous.  When
// the ring moves into a half, it first waits for the copies that last read
// from that half.
class PinnedRing {
public:
    explicit PinnedRing(size_t bytes) : cap_(bytes) {
        EPP_CUDA(cudaMallocHost(&base_, cap_));
        for (auto& e : done_) EPP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    ~PinnedRing() {
        for (auto& e : done_) cudaEventDestroy(e);
        cudaFreeHost(base_);
    }
    void* stage(const void* src, size_t bytes, cudaStream_t s) {
        const size_t half = cap_ / 2;
        EPP_REQUIRE(bytes <= half, "staging request too large");
        const size_t aligned = (bytes + 255) & ~static_cast<size_t>(255);
        if (off_ + aligned > (cur_ + 1) * half) {
            EPP_CUDA(cudaEventRecord(done_[cur_], s));
            cur_ ^= 1;
            if (used_[cur_]) EPP_CUDA(cudaEventSynchronize(done_[cur_]));
            off_ = cur_ * half;
        }
        used_[cur_] = true;
        void* dst = base_ + off_;
        std::memcpy(dst, src, bytes);
        off_ += aligned;
        return dst;
    }

private:
    char* base_ = nullptr;
    size_t cap_;
    size_t off_ = 0;
    int cur_ = 0;
    bool used_[2] = {false, false};
    cudaEvent_t done_[2];
};

struct Param {
    std::string name;
    long long numel = 0;
    float* master = nullptr;
    void* work = nullptr;
    float* grad = nullptr;
    long long off = 0;      // element offset in the stage's arenas
    float init_std = 0.f;   // 0 -> constant init_val
    float init_val = 0.f;
};

struct LayerParams {
    int ln1_w = -1, ln1_b = -1, wqkv = -1, wo = -1, ln2_w = -1, ln2_b = -1, w1 = -1, w2 = -1;
};

// Saved per-layer activations of one chunk.
struct LayerSaved {
    Buf x_out;        // output of this layer (= next layer's input); last layer -> act_out
    Buf mean1, rstd1, mean2, rstd2;
    Buf q, o, lse, x_mid, h;
    bool full = false;   // q/o/lse/x_mid/h/act present
};

struct ChunkState {
    int T = 0;
    std::vector<AttnSeg> segs;     // host copy
    Buf segs_dev, tok_seg, tok_pos, qwork, kwork, qwork128, kwork128, qwork256, kwork256;
    Buf kv_local;                  // [K|V][layer][T][Hkv*hd] rows of packed segments
    Buf dkv_local;                 // fp32 [dK|dV][T][Hkv*hd], one layer, re-zeroed per layer
    int nqwork = 0, nkwork = 0, nqwork128 = 0, nkwork128 = 0, nqwork256 = 0, nkwork256 = 0;
    double pairs = 0;
    AttnMaps maps{};               // TMA descriptors (K/V per chunk, Q/dO per layer call)
    Buf x_in;                      // stage input (copy of act_in or embedding)
    std::vector<LayerSaved> layers;
    Buf meanf, rstdf, dxf;         // last stage: final-norm stats + d(final norm out)
    int ckpt = 0;
};

struct SeqKV {
    long long len = 0;
    Buf kv;          // [layers][len][Hkv*hd] K then V halves: k at 0, v at layers*len*kvw
    Buf dkv;         // fp32, same layout
};

// Measured per-op trace (epp_stage_trace*): CUDA events on the stage stream
// around every forward / backward call and around each recompute
// layer_forward inside a backward (reference event kinds F / B / R,
// proj/include/epp/pipeline.hpp:43-51).  Events are recycled.
struct TraceOp {
    int chunk = -1;
    int kind = 0;                 // 0 forward, 1 backward (recompute split out at read)
    cudaEvent_t a = nullptr, b = nullptr;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> rec;
    long long live = 0;           // stage bytes held when the op's work was enqueued
};

class Tracer {
public:
    ~Tracer() {
        clear();
        for (cudaEvent_t e : free_) cudaEventDestroy(e);
    }
    bool on() const { return on_; }
    void start(cudaStream_t s) {
        clear();
        origin_ = ev();
        EPP_CUDA(cudaEventRecord(origin_, s));
        on_ = true;
    }
    void stop() { on_ = false; }
    cudaEvent_t record(cudaStream_t s) {
        cudaEvent_t e = ev();
        EPP_CUDA(cudaEventRecord(e, s));
        return e;
    }
    std::vector<TraceOp>& ops() { return ops_; }
    cudaEvent_t origin() const { return origin_; }
    void clear() {
        for (TraceOp& o : ops_) {
            give(o.a);
            give(o.b);
            for (auto& r : o.rec) {
                give(r.first);
                give(r.second);
            }
        }
        ops_.clear();
        give(origin_);
        origin_ = nullptr;
    }

private:
    cudaEvent_t ev() {
        if (!free_.empty()) {
            cudaEvent_t e = free_.back();
            free_.pop_back();
            return e;
        }
        cudaEvent_t e;
        EPP_CUDA(cudaEventCreate(&e));
        return e;
    }
    void give(cudaEvent_t e) {
        if (e) free_.push_back(e);
    }
    bool on_ = false;
    cudaEvent_t origin_ = nullptr;
    std::vector<TraceOp> ops_;
    std::vector<cudaEvent_t> free_;
};

}  // namespace

// ===========================================================================
class StageImpl {
public:
    StageImpl(const epp_model_desc& m, int first, int nl, bool embed, bool head, DType dt)
        : m_(m), first_(first), nl_(nl), has_embed_(embed), has_head_(head), dt_(dt) {
        EPP_REQUIRE(m.heads > 0 && m.kv_heads > 0 && m.heads % m.kv_heads == 0, "bad head counts");
        EPP_REQUIRE(m.head_dim * m.heads == m.hidden, "head_dim * heads must equal hidden");
        EPP_REQUIRE(first >= 0 && nl >= 0 && first + nl <= m.layers, "bad layer range");
        EPP_REQUIRE(m.hidden % 64 == 0 && m.ffn % 64 == 0 && m.vocab % 64 == 0,
                    "hidden/ffn/vocab must be multiples of 64");
        EPP_REQUIRE(dt == DType::F32 || m.head_dim == 64 || m.head_dim == 128,
                    "bf16 attention supports head_dim 64 or 128");
        keep_pool_reserved();
        if (const char* e = getenv("EPP_DEFER_WGRAD"); e && e[0] == '0') defer_wgrad_ = false;   // A/B switch
        if (const char* e = getenv("EPP_SMEM_PREF"); e && e[0] == '1')
            EPP_CUDA(cudaDeviceSetCacheConfig(cudaFuncCachePreferShared));
        D_ = m.hidden;
        H_ = m.heads;
        Hkv_ = m.kv_heads;
        hd_ = m.head_dim;
        llama_ = m.arch == EPP_ARCH_LLAMA;
        F_ = m.ffn;
        F1_ = llama_ ? 2 * F_ : F_;
        Nqkv_ = (H_ + 2 * Hkv_) * hd_;
        const float std0 = 0.02f;
        const float std_out = 0.02f / std::sqrt(2.0f * m.layers);
        if (has_embed_) emb_ = add("embed.weight", static_cast<long long>(m.vocab) * D_, std0);
        for (int j = 0; j < nl; ++j) {
            const std::string pre = "layers." + std::to_string(first + j) + ".";
            LayerParams lp;
            lp.ln1_w = add(pre + "norm1.weight", D_, 0.f, 1.f);
            if (!llama_) lp.ln1_b = add(pre + "norm1.bias", D_, 0.f, 0.f);
            lp.wqkv = add(pre + "attn.wqkv", static_cast<long long>(Nqkv_) * D_, std0);
            lp.wo = add(pre + "attn.wo", static_cast<long long>(D_) * H_ * hd_, std_out);
            lp.ln2_w = add(pre + "norm2.weight", D_, 0.f, 1.f);
            if (!llama_) lp.ln2_b = add(pre + "norm2.bias", D_, 0.f, 0.f);
            lp.w1 = add(pre + (llama_ ? "mlp.w13" : "mlp.w1"), static_cast<long long>(F1_) * D_, std0);
            lp.w2 = add(pre + "mlp.w2", static_cast<long long>(D_) * F_, std_out);
            lps_.push_back(lp);
        }
        if (has_head_) {
            lnf_w_ = add("final_norm.weight", D_, 0.f, 1.f);
            if (!llama_) lnf_b_ = add("final_norm.bias", D_, 0.f, 0.f);
            lm_ = add("lm_head.weight", static_cast<long long>(m.vocab) * D_, std0);
        }
        // One arena per kind (fp32 masters, fp32 grads, working copies),
        // parameters in creation order, each 64-element aligned; buckets
        // (embedding | one per layer | head) padded to 4096 elements, so a
        // bucket is one contiguous range for the data-parallel collectives
        // and splits evenly over up to 16 replicas (ZeRO-1 slices).
        {
            long long off = 0;
            int bucket_of_next = -1;
            auto close_bucket = [&] {
                off = (off + kBucketAlign - 1) / kBucketAlign * kBucketAlign;
                bucket_off_.push_back(off);
            };
            bucket_off_.push_back(0);
            for (size_t i = 0; i < params_.size(); ++i) {
                const int b = bucket_index(static_cast<int>(i));
                if (bucket_of_next >= 0 && b != bucket_of_next) close_bucket();
                bucket_of_next = b;
                params_[i].off = off;
                off += (params_[i].numel + 63) / 64 * 64;
            }
            close_bucket();
            arena_n_ = off;
        }
        EPP_CUDA(cudaMalloc(&master_arena_, sizeof(float) * arena_n_));
        EPP_CUDA(cudaMalloc(&grad_arena_, sizeof(float) * arena_n_));
        EPP_CUDA(cudaMemset(master_arena_, 0, sizeof(float) * arena_n_));
        EPP_CUDA(cudaMemset(grad_arena_, 0, sizeof(float) * arena_n_));
        if (dt_ == DType::F32) {
            work_arena_ = master_arena_;
        } else {
            EPP_CUDA(cudaMalloc(&work_arena_, dtype_size(dt_) * arena_n_));
            EPP_CUDA(cudaMemset(work_arena_, 0, dtype_size(dt_) * arena_n_));
        }
        for (Param& p : params_) {
            p.master = master_arena_ + p.off;
            p.grad = grad_arena_ + p.off;
            p.work = static_cast<char*>(work_arena_) + dtype_size(dt_) * p.off;
        }
        set_opt_shard(0, 1);
        // fp64 loss records: [0..1] the stage accumulator, then one
        // (sum, #targets) slot per chunk id forwarded since the last reset
        EPP_CUDA(cudaMalloc(&loss_acc_, sizeof(double) * 2 * (1 + kLossSlots)));
        EPP_CUDA(cudaMemset(loss_acc_, 0, sizeof(double) * 2 * (1 + kLossSlots)));
        // Keep freed chunk memory in the pool instead of returning it to the OS.
        int dev = 0;
        EPP_CUDA(cudaGetDevice(&dev));
        cudaMemPool_t mp;
        EPP_CUDA(cudaDeviceGetDefaultMemPool(&mp, dev));
        uint64_t thresh = UINT64_MAX;
        EPP_CUDA(cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thresh));
    }

    ~StageImpl() {
        chunks_.clear();
        seqs_.clear();
        cudaDeviceSynchronize();
        cudaFree(master_arena_);
        cudaFree(grad_arena_);
        if (work_arena_ != master_arena_) cudaFree(work_arena_);
        cudaFree(m_arena_);
        cudaFree(v_arena_);
        cudaFree(adam_segs_dev_);
        for (cudaEvent_t e : bucket_ev_) cudaEventDestroy(e);
        cudaFree(loss_acc_);
    }

    std::vector<Param>& params() { return params_; }
    Pool& pool() { return pool_; }

    void init_weights(unsigned long long seed, cudaStream_t s) {
        for (size_t i = 0; i < params_.size(); ++i) {
            Param& p = params_[i];
            if (p.init_std > 0.f) {
                // Seed folds in the global parameter name so stages agree
                // irrespective of how layers are partitioned.
                unsigned long long h = seed * 0x100000001b3ULL;
                for (char c : p.name) h = (h ^ static_cast<unsigned char>(c)) * 0x100000001b3ULL;
                init_normal(p.master, p.numel, p.init_std, h, s);
            } else {
                init_const(p.master, p.numel, p.init_val, s);
            }
        }
        sync_weights(s);
    }

    void sync_weights(cudaStream_t s) {
        if (dt_ == DType::F32) return;
        cast_f32_to(dt_, master_arena_, work_arena_, arena_n_, s);
    }

    void zero_grads(cudaStream_t s) { fill_zero(grad_arena_, sizeof(float) * arena_n_, s); }

    // One multi-tensor launch over the optimizer segments (this replica's
    // slice of every parameter; no weight decay on norms / biases); zeroes
    // every gradient.  With a ZeRO-1 shard the masters outside the slice are
    // left for the caller's all-gather.
    void adamw_step(float lr, float b1, float b2, float eps, float wd, int step, cudaStream_t s) {
        EPP_REQUIRE(step >= 1, "adamw step must be >= 1");
        const float bc1 = 1.f - std::pow(b1, static_cast<float>(step));
        const float bc2 = 1.f - std::pow(b2, static_cast<float>(step));
        adamw_multi(adam_segs_dev_, adam_nseg_, adam_total4_, master_arena_, work_arena_, dt_, grad_arena_,
                    m_arena_, v_arena_, lr, b1, b2, eps, wd, bc1, bc2, s);
        if (opt_nranks_ > 1) zero_grads(s);
    }

    // ZeRO-1: Adam state only for this rank's 1/nranks slice of every bucket.
    void set_opt_shard(int rank, int nranks) {
        EPP_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "bad optimizer shard");
        EPP_REQUIRE(kBucketAlign % (64 * nranks) == 0 || nranks == 1, "too many optimizer shards");
        std::vector<AdamSeg> segs;
        long long mv = 0;
        for (size_t b = 0; b + 1 < bucket_off_.size(); ++b) {
            const long long n = (bucket_off_[b + 1] - bucket_off_[b]) / nranks;
            const long long lo = bucket_off_[b] + rank * n, hi = lo + n;
            for (const Param& p : params_) {
                const long long a = std::max(lo, p.off), e = std::min(hi, p.off + p.numel);
                if (a >= e) continue;
                segs.push_back(AdamSeg{a, e - a, mv + (a - lo), p.init_std > 0.f ? 1 : 0, 0});
            }
            mv += n;
        }
        // prefix of float4 groups (segment lengths are multiples of 4)
        long long acc = 0;
        for (AdamSeg& g : segs) {
            EPP_REQUIRE(g.n % 4 == 0 && g.off % 4 == 0, "optimizer segment not float4-aligned");
            g.start4 = acc;
            acc += g.n / 4;
        }
        cudaFree(m_arena_);
        cudaFree(v_arena_);
        cudaFree(adam_segs_dev_);
        m_arena_ = v_arena_ = nullptr;
        adam_segs_dev_ = nullptr;
        EPP_CUDA(cudaMalloc(&m_arena_, sizeof(float) * std::max<long long>(mv, 4)));
        EPP_CUDA(cudaMalloc(&v_arena_, sizeof(float) * std::max<long long>(mv, 4)));
        EPP_CUDA(cudaMemset(m_arena_, 0, sizeof(float) * std::max<long long>(mv, 4)));
        EPP_CUDA(cudaMemset(v_arena_, 0, sizeof(float) * std::max<long long>(mv, 4)));
        if (!segs.empty()) {
            EPP_CUDA(cudaMalloc(&adam_segs_dev_, sizeof(AdamSeg) * segs.size()));
            EPP_CUDA(cudaMemcpy(adam_segs_dev_, segs.data(), sizeof(AdamSeg) * segs.size(), cudaMemcpyHostToDevice));
        }
        adam_nseg_ = static_cast<int>(segs.size());
        adam_total4_ = acc;
        opt_rank_ = rank;
        opt_nranks_ = nranks;
        opt_state_n_ = mv;
    }

    // --- data-parallel buckets -------------------------------------------
    long long arena_numel() const { return arena_n_; }
    float* master_arena() const { return master_arena_; }
    void* work_arena() const { return work_arena_; }
    float* grad_arena() const { return grad_arena_; }
    long long opt_state_numel() const { return opt_state_n_; }
    const std::vector<long long>& buckets() const { return bucket_off_; }
    void grad_events(bool on) {
        grad_events_ = on;
        if (on && bucket_ev_.empty()) {
            bucket_ev_.resize(bucket_off_.size() - 1);
            for (auto& e : bucket_ev_) EPP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
    }
    void bucket_wait(int b, cudaStream_t s) {
        EPP_REQUIRE(b >= 0 && b + 1 < static_cast<int>(bucket_off_.size()), "bucket index out of range");
        EPP_REQUIRE(!bucket_ev_.empty(), "bucket events were never enabled");
        EPP_CUDA(cudaStreamWaitEvent(s, bucket_ev_[b], 0));
    }

    void loss(double out[2], bool reset, cudaStream_t s) {
        EPP_CUDA(cudaMemcpyAsync(out, loss_acc_, sizeof(double) * 2, cudaMemcpyDeviceToHost, s));
        EPP_CUDA(cudaStreamSynchronize(s));
        if (reset) reset_loss(s);
    }

    // Stream-ordered copy of the accumulator into caller memory (pinned host
    // or device), optional reset; no synchronisation.
    void loss_async(double* out2, bool reset, cudaStream_t s) {
        EPP_CUDA(cudaMemcpyAsync(out2, loss_acc_, sizeof(double) * 2, cudaMemcpyDefault, s));
        if (reset) reset_loss(s);
    }

    // (sum of token losses, #targets) of the latest forward of `chunk_id`
    // since the last reset (a plan's chunk ids repeat from step to step).
    void read_chunk_loss(int chunk_id, double out[2], cudaStream_t s) {
        EPP_REQUIRE(has_head_, "chunk loss: not the last stage");
        auto it = loss_slot_.find(chunk_id);
        EPP_REQUIRE(it != loss_slot_.end(), "chunk loss: chunk not forwarded since the last reset");
        EPP_CUDA(cudaMemcpyAsync(out, loss_acc_ + 2 * (1 + it->second), sizeof(double) * 2,
                                 cudaMemcpyDeviceToHost, s));
        EPP_CUDA(cudaStreamSynchronize(s));
    }

    void reset_loss(cudaStream_t s) {
        EPP_CUDA(cudaMemsetAsync(loss_acc_, 0, sizeof(double) * 2, s));
        loss_slot_.clear();
    }

    void release_seq(int seq) { seqs_.erase(seq); }

    // ------------------------------------------------------------------
    void forward(const epp_chunk_desc& c, const void* act_in, void* act_out, cudaStream_t s) {
        EPP_REQUIRE(chunks_.find(c.id) == chunks_.end(), "chunk already in flight on this stage");
        EPP_REQUIRE(c.ckpt_layers >= 0 && c.ckpt_layers <= nl_, "ckpt_layers out of range");
        ChunkState& cs = chunks_[c.id];
        TraceOp* tr = trace_begin(c.id, 0, s);
        try {
            setup_chunk(cs, c, s);
            cs.ckpt = c.ckpt_layers;
            const size_t act_bytes = static_cast<size_t>(cs.T) * D_ * esz();
            cs.x_in = Buf(&pool_, act_bytes, s);
            if (has_embed_) {
                EPP_REQUIRE(c.token_ids != nullptr, "embedding stage needs token_ids");
                embed_fwd(dt_, c.token_ids, work(emb_), cs.x_in.get(), cs.T, D_, s);
            } else {
                EPP_REQUIRE(act_in != nullptr, "act_in is null");
                ProfScope pc(kProfCopy, 2.0 * act_bytes, s);
                EPP_CUDA(cudaMemcpyAsync(cs.x_in.get(), act_in, act_bytes, cudaMemcpyDeviceToDevice, s));
            }
            cs.layers.resize(nl_);
            const void* x = cs.x_in.get();
            for (int j = 0; j < nl_; ++j) {
                LayerSaved& L = cs.layers[j];
                // the last layer of a non-head stage writes its output straight
                // into act_out (the caller's buffer, e.g. the next stage's P2P
                // mailbox in peer memory): its backward never reads it
                void* out = nullptr;
                if (j == nl_ - 1 && !has_head_) {
                    EPP_REQUIRE(act_out != nullptr, "act_out is null");
                    out = act_out;
                } else {
                    L.x_out = Buf(&pool_, act_bytes, s);
                    out = L.x_out.get();
                }
                layer_forward(cs, j, x, L, out, /*skip_out=*/false, s);
                if (j < cs.ckpt) drop_full(L);
                x = out;
            }
            if (has_head_) {
                head_forward(cs, c, x, s);
            } else if (nl_ == 0) {
                EPP_REQUIRE(act_out != nullptr, "act_out is null");
                EPP_CUDA(cudaMemcpyAsync(act_out, x, act_bytes, cudaMemcpyDeviceToDevice, s));
            }
        } catch (...) {
            chunks_.erase(c.id);
            throw;
        }
        trace_end(tr, s);
    }

    void backward(const epp_chunk_desc& c, const void* grad_in, void* grad_out, cudaStream_t s) {
        auto it = chunks_.find(c.id);
        EPP_REQUIRE(it != chunks_.end(), "backward of a chunk that was not forwarded");
        ChunkState& cs = it->second;
        TraceOp* tr = trace_begin(c.id, 1, s);
        const size_t act_bytes = static_cast<size_t>(cs.T) * D_ * esz();
        // d(stage output): the head's final-norm backward, or grad_in used in
        // place (read by the last layer's backward only; the caller keeps it
        // valid until this call's work has run)
        Buf dy;
        const void* dy_ptr = grad_in;
        if (has_head_) {
            dy = Buf(&pool_, act_bytes, s);
            const void* xl = nl_ > 0 ? cs.layers[nl_ - 1].x_out.get() : cs.x_in.get();
            norm_bwd(dt_, llama_, xl, work(lnf_w_), cs.dxf.get(), cs.meanf.get<float>(),
                     cs.rstdf.get<float>(), nullptr, dy.get(), grad(lnf_w_),
                     lnf_b_ >= 0 ? grad(lnf_b_) : nullptr, cs.T, D_, s);
            cs.dxf.release();
            dy_ptr = dy.get();
            bucket_ready(head_bucket(), s);   // lm_head (forward) + final norm grads
        } else {
            EPP_REQUIRE(grad_in != nullptr, "grad_in is null");
        }
        attach_dkv(cs, c, s);

        for (int j = nl_ - 1; j >= 0; --j) {
            LayerSaved& L = cs.layers[j];
            const void* x = j == 0 ? cs.x_in.get() : cs.layers[j - 1].x_out.get();
            if (!L.full) {   // recompute
                flush_wgrad(false, s);
                cudaEvent_t ra = tr ? tracer_.record(s) : nullptr;
                layer_forward(cs, j, x, L, nullptr, /*skip_out=*/true, s);
                if (tr) tr->rec.emplace_back(ra, tracer_.record(s));
            }
            // the first layer of a non-embedding stage writes d(stage input)
            // straight into grad_out (e.g. the previous stage's P2P mailbox)
            Buf dx;
            void* dx_ptr = nullptr;
            if (j == 0 && !has_embed_) {
                EPP_REQUIRE(grad_out != nullptr, "grad_out is null");
                dx_ptr = grad_out;
            } else {
                dx = Buf(&pool_, act_bytes, s);
                dx_ptr = dx.get();
            }
            layer_backward(cs, j, x, L, dy_ptr, dx_ptr, s);
            if (pending_.live) pending_.bucket = layer_bucket(j);   // its dWqkv is still pending
            else bucket_ready(layer_bucket(j), s);
            drop_full(L);
            L.x_out.release();
            dy = std::move(dx);
            dy_ptr = dx_ptr;
        }
        flush_wgrad(false, s);
        if (has_embed_) {
            embed_bwd(dt_, c.token_ids, dy_ptr, grad(emb_), cs.T, D_, s);
            bucket_ready(0, s);
        } else if (nl_ == 0) {
            EPP_REQUIRE(grad_out != nullptr, "grad_out is null");
            EPP_CUDA(cudaMemcpyAsync(grad_out, dy_ptr, act_bytes, cudaMemcpyDeviceToDevice, s));
        }
        dy.release();
        const bool first_slice = c.seq >= 0 && c.context == 0;
        const int seq = c.seq;
        chunks_.erase(it);
        if (first_slice) seqs_.erase(seq);
        trace_end(tr, s);
    }

    // ------------------------------------------------------------ tracing
    void trace(bool on, cudaStream_t s) {
        if (on) tracer_.start(s);
        else tracer_.stop();
    }

    // Resolves the recorded events (synchronises on the last one).  Per
    // backward with recompute, an R event [start, start + sum of the
    // recompute intervals) precedes the B event, as the reference simulator
    // lays them out (proj/src/pipeline.cpp:246-257).
    int trace_read(epp_trace_event* out, int cap) {
        auto& ops = tracer_.ops();
        for (auto it = ops.rbegin(); it != ops.rend(); ++it)
            if (it->b) {
                EPP_CUDA(cudaEventSynchronize(it->b));
                break;
            }
        auto since = [&](cudaEvent_t e) {
            float ms = 0.f;
            EPP_CUDA(cudaEventElapsedTime(&ms, tracer_.origin(), e));
            return static_cast<double>(ms) * 1e-3;
        };
        int n = 0;
        auto put = [&](int chunk, int op, double a, double b, long long live) {
            if (out && n < cap) out[n] = epp_trace_event{chunk, op, a, b, live};
            ++n;
        };
        for (const TraceOp& o : ops) {
            if (!o.b) continue;   // a call that failed
            const double a = since(o.a), b = since(o.b);
            double rec = 0.0;
            for (const auto& r : o.rec) {
                float ms = 0.f;
                EPP_CUDA(cudaEventElapsedTime(&ms, r.first, r.second));
                rec += static_cast<double>(ms) * 1e-3;
            }
            if (o.kind == 1 && rec > 0.0) {
                put(o.chunk, 2, a, a + rec, o.live);
                put(o.chunk, 1, a + rec, b, o.live);
            } else {
                put(o.chunk, o.kind, a, b, o.live);
            }
        }
        return n;
    }

private:
    int add(const std::string& name, long long numel, float std, float val = 0.f) {
        Param p;
        p.name = name;
        p.numel = numel;
        p.init_std = std;
        p.init_val = val;
        params_.push_back(p);
        return static_cast<int>(params_.size()) - 1;
    }
    // bucket of parameter i: [embedding] [layer 0] ... [layer n-1] [head]
    int bucket_index(int i) const {
        if (i == emb_) return 0;
        const int e = has_embed_ ? 1 : 0;
        if (i == lnf_w_ || i == lnf_b_ || i == lm_) return e + nl_;
        for (int j = 0; j < nl_; ++j) {
            const LayerParams& lp = lps_[j];
            for (int q : {lp.ln1_w, lp.ln1_b, lp.wqkv, lp.wo, lp.ln2_w, lp.ln2_b, lp.w1, lp.w2})
                if (q == i) return e + j;
        }
        throw std::logic_error("parameter without a bucket");
    }
    int layer_bucket(int j) const { return (has_embed_ ? 1 : 0) + j; }
    int head_bucket() const { return (has_embed_ ? 1 : 0) + nl_; }
    void bucket_ready(int b, cudaStream_t s) {
        if (grad_events_) EPP_CUDA(cudaEventRecord(bucket_ev_[b], s));
    }
    void* work(int i) const { return params_[i].work; }
    float* grad(int i) const { return params_[i].grad; }
    size_t esz() const { return dtype_size(dt_); }
    long long kvw() const { return static_cast<long long>(Hkv_) * hd_; }

    void drop_full(LayerSaved& L) {
        L.q.release(); L.o.release(); L.lse.release(); L.x_mid.release(); L.h.release();
        L.full = false;
    }

    // Segment table, token maps and attention work lists of one chunk.
    void setup_chunk(ChunkState& cs, const epp_chunk_desc& c, cudaStream_t s) {
        EPP_REQUIRE(c.nslices >= 1 && c.slices != nullptr, "chunk has no slices");
        long long T = 0;
        for (int i = 0; i < c.nslices; ++i) {
            EPP_REQUIRE(c.slices[i] > 0, "slice length must be positive");
            T += c.slices[i];
        }
        EPP_REQUIRE(T < (1LL << 31), "chunk too large");
        cs.T = static_cast<int>(T);
        const bool seq_chunk = c.seq >= 0;
        if (seq_chunk) {
            EPP_REQUIRE(c.seq_len >= c.context + c.slices[0], "seq_len shorter than the slice");
            SeqKV& sk = seqs_[c.seq];
            if (!sk.kv) {
                sk.len = c.seq_len;
                // bf16: no zero fill (the chunk's TMA maps end at its last
                // visible key, rows past it load as zeros); fp32 parity
                // kernels never read past a query's position either, but
                // keep the buffer defined for them
                sk.kv = Buf(&pool_, 2 * static_cast<size_t>(nl_) * sk.len * kvw() * esz(), s,
                            /*zero=*/dt_ != DType::BF16);
            }
            EPP_REQUIRE(sk.len == c.seq_len, "seq_len changed between slices");
        } else {
            EPP_REQUIRE(c.context == 0, "context without a sequence");
        }
        // chunk-local K/V of packed documents: every row a kernel reads is
        // written by the layer's QKV epilogue first (rows past T load as
        // zeros through the TMA map), so bf16 skips the zero fill (~8 GB per
        // 15K-token GPT-7B chunk)
        cs.kv_local = Buf(&pool_, 2 * static_cast<size_t>(nl_) * T * kvw() * esz(), s, /*zero=*/dt_ != DType::BF16);
        int max_pos = 0;
        long long q_start = 0;
        cs.segs.clear();
        for (int i = 0; i < c.nslices; ++i) {
            AttnSeg sg{};
            sg.q_start = static_cast<int>(q_start);
            sg.q_len = static_cast<int>(c.slices[i]);
            if (i == 0 && seq_chunk) {
                SeqKV& sk = seqs_[c.seq];
                sg.kv_ctx = static_cast<int>(c.context);
                sg.tma_map = 0;
                sg.kv_row0 = 0;
                sg.k = sk.kv.get<uint8_t>();
                sg.v = sk.kv.get<uint8_t>() + static_cast<size_t>(nl_) * sk.len * kvw() * esz();
                sg.kv_layer_stride = sk.len * kvw();
                sg.dkv_layer_stride = sk.len * kvw();
                // the tail slice's backward is the sequence's first (later
                // slices run first, pipeline.cpp:121-131): it WRITES every
                // context row of the fp32 dK/dV buffer and has no partials for
                // its own rows (2); earlier slices read-add (1)
                sg.dkv_accum = (c.tail && dt_ == DType::BF16) ? 2 : 1;
            } else {
                // Packed document: K/V rows in the chunk-local buffer (layer
                // strided like the sequence buffers); dK/dV in a one-layer
                // scratch (dkv stride 0), bound at backward.
                sg.kv_ctx = 0;
                sg.tma_map = 1;
                sg.kv_row0 = static_cast<int>(q_start);
                const size_t row0 = static_cast<size_t>(q_start) * kvw();
                sg.k = cs.kv_local.get<uint8_t>() + row0 * esz();
                sg.v = cs.kv_local.get<uint8_t>() + (static_cast<size_t>(nl_) * T * kvw() + row0) * esz();
                sg.kv_layer_stride = T * kvw();
                sg.dkv_layer_stride = 0;
                sg.dkv_accum = 0;
            }
            max_pos = std::max(max_pos, sg.kv_ctx + sg.q_len);
            cs.segs.push_back(sg);
            q_start += c.slices[i];
        }
        rope_reserve(max_pos, hd_, m_.rope_theta, s);
        if (dt_ == DType::BF16) {
            if (seq_chunk) {
                const SeqKV& sk = seqs_[c.seq];
                // rows end at the chunk's last visible key: tiles past it read zeros
                attn_maps_kv(cs.maps, 0, sk.kv.get(),
                             sk.kv.get<uint8_t>() + static_cast<size_t>(nl_) * sk.len * kvw() * esz(),
                             c.context + c.slices[0], nl_, Hkv_, hd_, sk.len);
            }
            attn_maps_kv(cs.maps, 1, cs.kv_local.get(),
                         cs.kv_local.get<uint8_t>() + static_cast<size_t>(nl_) * T * kvw() * esz(), T, nl_,
                         Hkv_, hd_);
        }
        std::vector<int> tseg(cs.T), tpos(cs.T);
        std::vector<AttnWork> qw, kw, qw128, kw128, qw256, kw256;
        for (int i = 0; i < static_cast<int>(cs.segs.size()); ++i) {
            const AttnSeg& sg = cs.segs[i];
            for (int t = 0; t < sg.q_len; ++t) {
                tseg[sg.q_start + t] = i;
                tpos[sg.q_start + t] = sg.kv_ctx + t;
            }
            for (int b = 0; b * kAttnBlock < sg.q_len; ++b) qw.push_back({i, b});
            for (int b = 0; b * kAttnBlock < sg.kv_ctx + sg.q_len; ++b) kw.push_back({i, b});
            for (int b = 0; b * 128 < sg.q_len; ++b) qw128.push_back({i, b});
            for (int b = 0; b * 128 < sg.kv_ctx + sg.q_len; ++b) kw128.push_back({i, b});
            for (int b = 0; b * 256 < sg.q_len; ++b) qw256.push_back({i, b});
            for (int b = 0; b * 256 < sg.kv_ctx + sg.q_len; ++b) kw256.push_back({i, b});
        }
        cs.pairs = 0;
        for (const AttnSeg& sg : cs.segs)
            cs.pairs += static_cast<double>(sg.q_len) * sg.kv_ctx +
                        0.5 * static_cast<double>(sg.q_len) * (sg.q_len + 1);
        // Longest-processing-time first: blocks with the most keys (or the
        // most query blocks, for the key-parallel backward) are dispatched
        // first so long-context slices do not form the tail of the grid.
        auto qcost = [&](const AttnWork& w, int blk) {
            const AttnSeg& sg = cs.segs[w.seg];
            return sg.kv_ctx + std::min(sg.q_len, (w.block + 1) * blk);
        };
        auto kcost = [&](const AttnWork& w, int blk) {
            const AttnSeg& sg = cs.segs[w.seg];
            return sg.q_len - std::max(0, w.block * blk - sg.kv_ctx);   // queries seeing the block
        };
        auto by = [](auto cost, int blk) {
            return [cost, blk](const AttnWork& a, const AttnWork& b) {
                const int ca = cost(a, blk), cb = cost(b, blk);
                if (ca != cb) return ca > cb;
                return a.seg != b.seg ? a.seg < b.seg : a.block < b.block;
            };
        };
        std::sort(qw.begin(), qw.end(), by(qcost, kAttnBlock));
        std::sort(kw.begin(), kw.end(), by(kcost, kAttnBlock));
        std::sort(qw128.begin(), qw128.end(), by(qcost, 128));
        std::sort(kw128.begin(), kw128.end(), by(kcost, 128));
        std::sort(qw256.begin(), qw256.end(), by(qcost, 256));
        std::sort(kw256.begin(), kw256.end(), by(kcost, 256));
        cs.nqwork = static_cast<int>(qw.size());
        cs.nkwork = static_cast<int>(kw.size());
        cs.tok_seg = upload(tseg.data(), tseg.size() * sizeof(int), s);
        cs.tok_pos = upload(tpos.data(), tpos.size() * sizeof(int), s);
        cs.qwork = upload(qw.data(), qw.size() * sizeof(AttnWork), s);
        cs.kwork = upload(kw.data(), kw.size() * sizeof(AttnWork), s);
        cs.nqwork128 = static_cast<int>(qw128.size());
        cs.nkwork128 = static_cast<int>(kw128.size());
        cs.qwork128 = upload(qw128.data(), qw128.size() * sizeof(AttnWork), s);
        cs.kwork128 = upload(kw128.data(), kw128.size() * sizeof(AttnWork), s);
        cs.nqwork256 = static_cast<int>(qw256.size());
        cs.qwork256 = upload(qw256.data(), qw256.size() * sizeof(AttnWork), s);
        cs.nkwork256 = static_cast<int>(kw256.size());
        cs.kwork256 = upload(kw256.data(), kw256.size() * sizeof(AttnWork), s);
        cs.segs_dev = upload(cs.segs.data(), cs.segs.size() * sizeof(AttnSeg), s);
    }

    Buf upload(const void* host, size_t bytes, cudaStream_t s) {
        Buf b(&pool_, bytes, s);
        if (bytes) copy_h2d(b.get(), host, bytes, s);
        return b;
    }
    void copy_h2d(void* dst, const void* host, size_t bytes, cudaStream_t s) {
        const void* src = ring_.stage(host, bytes, s);
        EPP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    }

    // Bind dK/dV accumulators into the segment table: the sequence's
    // persistent fp32 buffer for segment 0 of a Split/Hybrid chunk, a
    // one-layer chunk-local scratch for packed documents.
    void attach_dkv(ChunkState& cs, const epp_chunk_desc& c, cudaStream_t s) {
        const size_t half = static_cast<size_t>(cs.T) * kvw();
        cs.dkv_local = Buf(&pool_, 2 * half * sizeof(float), s);
        for (size_t i = 0; i < cs.segs.size(); ++i) {
            AttnSeg& sg = cs.segs[i];
            if (i == 0 && c.seq >= 0) {
                SeqKV& sk = seqs_[c.seq];
                if (!sk.dkv)   // bf16: the tail slice writes it first (dkv_accum 2), no zero fill
                    sk.dkv = Buf(&pool_, 2 * static_cast<size_t>(nl_) * sk.len * kvw() * sizeof(float),
                                 s, /*zero=*/dt_ != DType::BF16);
                sg.dk = sk.dkv.get<float>();
                sg.dv = sk.dkv.get<float>() + static_cast<size_t>(nl_) * sk.len * kvw();
            } else {
                const size_t row0 = static_cast<size_t>(sg.q_start) * kvw();
                sg.dk = cs.dkv_local.get<float>() + row0;
                sg.dv = cs.dkv_local.get<float>() + half + row0;
            }
        }
        copy_h2d(cs.segs_dev.get(), cs.segs.data(), cs.segs.size() * sizeof(AttnSeg), s);
    }

    AttnArgs attn_args(ChunkState& cs, int j) const {
        AttnArgs a;
        a.segs = cs.segs_dev.get<AttnSeg>();
        a.nseg = static_cast<int>(cs.segs.size());
        a.qwork = cs.qwork.get<AttnWork>();
        a.nqwork = cs.nqwork;
        a.kwork = cs.kwork.get<AttnWork>();
        a.nkwork = cs.nkwork;
        a.qwork128 = cs.qwork128.get<AttnWork>();
        a.nqwork128 = cs.nqwork128;
        a.kwork128 = cs.kwork128.get<AttnWork>();
        a.nkwork128 = cs.nkwork128;
        a.kwork256 = cs.kwork256.get<AttnWork>();
        a.nkwork256 = cs.nkwork256;
        a.qwork256 = cs.qwork256.get<AttnWork>();
        a.nqwork256 = cs.nqwork256;
        a.T = cs.T;
        a.H = H_;
        a.Hkv = Hkv_;
        a.hd = hd_;
        a.layer = j;
        a.scale = 1.f / std::sqrt(static_cast<float>(hd_));
        a.dtype = dt_;
        a.pairs = cs.pairs;
        return a;
    }

    // Forward of stage layer j on input x.  Writes the saved activations into
    // L (q, o, lse, x_mid, h, kv_local, norm stats) and, unless skip_out, the
    // layer output to `out`.
    void layer_forward(ChunkState& cs, int j, const void* x, LayerSaved& L, void* out, bool skip_out,
                       cudaStream_t s) {
        const LayerParams& P = lps_[j];
        const int T = cs.T;
        const size_t e = esz();
        if (!L.mean1) {
            L.mean1 = Buf(&pool_, sizeof(float) * T, s);
            L.rstd1 = Buf(&pool_, sizeof(float) * T, s);
            L.mean2 = Buf(&pool_, sizeof(float) * T, s);
            L.rstd2 = Buf(&pool_, sizeof(float) * T, s);
        }
        L.q = Buf(&pool_, static_cast<size_t>(T) * H_ * hd_ * e, s);
        L.o = Buf(&pool_, static_cast<size_t>(T) * H_ * hd_ * e, s);
        L.lse = Buf(&pool_, sizeof(float) * H_ * T, s);
        L.x_mid = Buf(&pool_, static_cast<size_t>(T) * D_ * e, s);
        L.h = Buf(&pool_, static_cast<size_t>(T) * F1_ * e, s);
        L.full = true;

        Buf xn(&pool_, static_cast<size_t>(T) * D_ * e, s);
        norm_fwd(dt_, llama_, x, work(P.ln1_w), P.ln1_b >= 0 ? work(P.ln1_b) : nullptr, xn.get(),
                 llama_ ? nullptr : L.mean1.get<float>(), L.rstd1.get<float>(), T, D_,
                 m_.norm_eps, s);
        if (dt_ == DType::BF16) {
            // QKV projection with RoPE and the q / K / V scatter in its epilogue
            RopeScatterArgs ra;
            ra.q_out = L.q.get();
            ra.segs = cs.segs_dev.get<AttnSeg>();
            ra.tok_seg = cs.tok_seg.get<int>();
            ra.tok_pos = cs.tok_pos.get<int>();
            ra.cs = rope_table_ptr(hd_, m_.rope_theta, s);
            ra.H = H_;
            ra.Hkv = Hkv_;
            ra.hd = hd_;
            ra.layer = j;
            GemmArgs g = mk(T, Nqkv_, D_, xn.get(), D_, true, work(P.wqkv), D_, true, nullptr, Nqkv_);
            g.epi = Epi::RopeScatter;
            g.rope = &ra;
            gemm(g, s);
        } else {
            Buf qkv(&pool_, static_cast<size_t>(T) * Nqkv_ * e, s);
            gemm(mk(T, Nqkv_, D_, xn.get(), D_, true, work(P.wqkv), D_, true, qkv.get(), Nqkv_), s);
            rope_qkv_scatter(dt_, qkv.get(), L.q.get(), cs.segs_dev.get<AttnSeg>(),
                             static_cast<int>(cs.segs.size()), cs.tok_seg.get<int>(),
                             cs.tok_pos.get<int>(), T, H_, Hkv_, hd_, j, m_.rope_theta, s);
        }
        AttnArgs a = attn_args(cs, j);
        a.q = L.q.get();
        a.o = L.o.get();
        a.lse = L.lse.get<float>();
        if (dt_ == DType::BF16) {
            attn_maps_q(cs.maps, L.q.get(), nullptr, T, H_, hd_);
            a.maps = &cs.maps;
        }
        attn_fwd(a, s);
        // x_mid = x + o Wo^T
        GemmArgs g = mk(T, D_, H_ * hd_, L.o.get(), H_ * hd_, true, work(P.wo), H_ * hd_, true,
                        L.x_mid.get(), D_);
        g.epi = Epi::AddRes;
        g.R = x;
        g.ldr = D_;
        gemm(g, s);
        norm_fwd(dt_, llama_, L.x_mid.get(), work(P.ln2_w), P.ln2_b >= 0 ? work(P.ln2_b) : nullptr,
                 xn.get(), llama_ ? nullptr : L.mean2.get<float>(), L.rstd2.get<float>(), T, D_,
                 m_.norm_eps, s);
        // The MLP activation is only W2's operand here: transient (the
        // backward re-creates it from h for dW2), so a layer keeps 14 -> 10
        // hidden-widths of activations per token (GPT) and the planner's
        // checkpoint ladder has to recompute fewer layers.  A recompute
        // (skip_out) only restores h.
        Buf act;
        if (!skip_out) act = Buf(&pool_, static_cast<size_t>(T) * F_ * e, s);
        GemmArgs up = mk(T, F1_, D_, xn.get(), D_, true, work(P.w1), D_, true, L.h.get(), F1_);
        if (!llama_ && !skip_out) {   // GELU fused into the up-projection epilogue
            up.epi = Epi::StoreGelu;
            up.C2 = act.get();
            up.ldc2 = F_;
        } else if (llama_ && !skip_out) {   // SwiGLU fused (CTA-pair tiles pair gate and up rows)
            up.epi = Epi::SwiGlu;
            up.C2 = act.get();
            up.ldc2 = F_;
            if (!gemm_swiglu_fusable(up)) {
                up.epi = Epi::Store;
                up.C2 = nullptr;
            }
        }
        gemm(up, s);
        xn.release();
        if (!skip_out) {
            if (llama_ && up.epi != Epi::SwiGlu) act_fwd(dt_, 1, L.h.get(), act.get(), T, F_, s);
            GemmArgs g2 = mk(T, D_, F_, act.get(), F_, true, work(P.w2), F_, true, out, D_);
            g2.epi = Epi::AddRes;
            g2.R = L.x_mid.get();
            g2.ldr = D_;
            gemm(g2, s);
        }
    }

    void layer_backward(ChunkState& cs, int j, const void* x, LayerSaved& L, const void* dy,
                        void* dx, cudaStream_t s) {
        const LayerParams& P = lps_[j];
        const int T = cs.T;
        const size_t e = esz();
        const int Dq = H_ * hd_;
        // ---- MLP ----
        // The activation A = act(h) that dW2 needs is not kept from the
        // forward: GPT re-creates it in the W2 data-gradient epilogue (which
        // reads h for gelu' anyway), Llama in a pass over h.
        Buf act(&pool_, static_cast<size_t>(T) * F_ * e, s);
        Buf dh(&pool_, static_cast<size_t>(T) * F1_ * e, s);
        GemmArgs swb = mk(T, F_, D_, dy, D_, true, work(P.w2), F_, false, dh.get(), F1_);   // dA = dY W2
        swb.epi = Epi::SwiGluBwd;   // -> dh = [dA u silu'(g) | dA silu(g)], A = silu(g) u
        swb.R = L.h.get();
        swb.ldr = F1_;
        swb.C2 = act.get();
        swb.ldc2 = F_;
        Buf dxn(&pool_, static_cast<size_t>(T) * D_ * e, s);
        auto dgrad_w1 = [&] {
            gemm(mk(T, D_, F1_, dh.get(), F1_, true, work(P.w1), D_, false, dxn.get(), D_), s);  // dXn2
        };
        // Where the W2 data-gradient epilogue forms A, dW2 runs after the
        // (independent) W1 data gradient and fills that GEMM's last wave.
        bool w1_done = false;
        if (llama_ && gemm_swiglu_fusable(swb)) {
            gemm(swb, s);
            flush_wgrad(true, s);   // the previous layer's dWqkv
            dgrad_w1();
            w1_done = true;
            wgrad(D_, F_, T, dy, D_, act.get(), F_, grad(P.w2), s, true);              // dW2 += dY^T A
            act.release();
        } else if (llama_) {
            flush_wgrad(false, s);
            act_fwd(dt_, 1, L.h.get(), act.get(), T, F_, s);
            wgrad(D_, F_, T, dy, D_, act.get(), F_, grad(P.w2), s);                    // dW2 += dY^T A
            act.release();
            Buf da(&pool_, static_cast<size_t>(T) * F_ * e, s);
            gemm(mk(T, F_, D_, dy, D_, true, work(P.w2), F_, false, da.get(), F_), s);    // dA = dY W2
            act_bwd(dt_, 1, L.h.get(), da.get(), dh.get(), T, F_, s);
        } else {
            // dH = (dY W2) * gelu'(H) and A = gelu(H), fused into the
            // data-gradient epilogue
            GemmArgs g = mk(T, F_, D_, dy, D_, true, work(P.w2), F_, false, dh.get(), F_);
            g.epi = Epi::GeluBwd;
            g.R = L.h.get();
            g.ldr = F_;
            g.C2 = act.get();
            g.ldc2 = F_;
            gemm(g, s);
            flush_wgrad(true, s);   // the previous layer's dWqkv
            dgrad_w1();
            w1_done = true;
            wgrad(D_, F_, T, dy, D_, act.get(), F_, grad(P.w2), s, true);              // dW2 += dY^T A
            act.release();
        }
        if (!w1_done) dgrad_w1();
        // norm backward also re-creates xn = norm(x_mid) (one pass over x_mid)
        // for the dW1 weight gradient
        Buf xn(&pool_, static_cast<size_t>(T) * D_ * e, s);
        Buf dxm(&pool_, static_cast<size_t>(T) * D_ * e, s);
        norm_bwd(dt_, llama_, L.x_mid.get(), work(P.ln2_w), dxn.get(),
                 llama_ ? nullptr : L.mean2.get<float>(), L.rstd2.get<float>(), dy, dxm.get(),
                 grad(P.ln2_w), P.ln2_b >= 0 ? grad(P.ln2_b) : nullptr, T, D_, s,
                 P.ln2_b >= 0 ? work(P.ln2_b) : nullptr, xn.get());
        // ---- attention ----
        // dW1 and dWo do not depend on the out-projection's data gradient:
        // they follow it and fill its last wave (and each other's)
        Buf dout(&pool_, static_cast<size_t>(T) * Dq * e, s);
        gemm(mk(T, Dq, D_, dxm.get(), D_, true, work(P.wo), Dq, false, dout.get(), Dq), s);  // dO
        wgrad(F1_, D_, T, dh.get(), F1_, xn.get(), D_, grad(P.w1), s, true);               // dW1
        dh.release();
        wgrad(D_, Dq, T, dxm.get(), D_, L.o.get(), Dq, grad(P.wo), s, true);               // dWo
        Buf delta(&pool_, sizeof(float) * static_cast<size_t>(H_) * T, s);
        Buf dqkv(&pool_, static_cast<size_t>(T) * Nqkv_ * e, s);
        AttnArgs a = attn_args(cs, j);
        // bf16 (tcgen05): the dK/dV kernel writes every key row of a packed
        // segment exactly once (dkv_accum = 0), and the dQ and dK/dV kernels
        // write un-rotated bf16 dQ / dK / dV straight into dqkv.  fp32 parity
        // kernels: accumulate into zeroed buffers, fp32 dQ, then the RoPE
        // gather pass.
        const bool tc_bwd = dt_ == DType::BF16;
        if (!tc_bwd) fill_zero(cs.dkv_local.get(), 2 * static_cast<size_t>(T) * kvw() * sizeof(float), s);
        a.q = L.q.get();
        a.o = L.o.get();
        a.lse = L.lse.get<float>();
        a.dout = dout.get();
        a.delta = delta.get<float>();
        Buf dq;
        if (tc_bwd) {
            a.dqkv_out = dqkv.get();
            a.tok_pos = cs.tok_pos.get<int>();
            a.rope_cs = rope_table_ptr(hd_, m_.rope_theta, s);
            attn_maps_q(cs.maps, L.q.get(), dout.get(), T, H_, hd_);
            a.maps = &cs.maps;
        } else {
            dq = Buf(&pool_, sizeof(float) * static_cast<size_t>(T) * Dq, s);
            a.dq = dq.get<float>();
        }
        attn_bwd(a, s);
        dout.release();
        delta.release();
        if (!tc_bwd)
            rope_qkv_gather_grad(dt_, dq.get<float>(), cs.segs_dev.get<AttnSeg>(), cs.tok_seg.get<int>(),
                                 cs.tok_pos.get<int>(), dqkv.get(), T, H_, Hkv_, hd_, j, m_.rope_theta, s);
        dq.release();
        gemm(mk(T, D_, Nqkv_, dqkv.get(), Nqkv_, true, work(P.wqkv), D_, false, dxn.get(), D_), s);
        norm_bwd(dt_, llama_, x, work(P.ln1_w), dxn.get(), llama_ ? nullptr : L.mean1.get<float>(),
                 L.rstd1.get<float>(), dxm.get(), dx, grad(P.ln1_w),
                 P.ln1_b >= 0 ? grad(P.ln1_b) : nullptr, T, D_, s,
                 P.ln1_b >= 0 ? work(P.ln1_b) : nullptr, xn.get());
        // dWqkv waits for the next kernel that does not touch its operands
        // (the next layer's first data gradient): flush_wgrad()
        GemmArgs wq = mk(Nqkv_, D_, T, dqkv.get(), Nqkv_, false, xn.get(), D_, false, grad(P.wqkv), D_);
        wq.epi = Epi::AccumF32;
        pending_ = PendingWgrad{wq, std::move(dqkv), std::move(xn), -1, true};
    }

    // A weight gradient held back until an independent GEMM has been
    // enqueued; it then follows that GEMM with a deferred dependency wait
    // (GemmArgs::defer_wait) and fills its last wave.  `bucket`: the DP
    // bucket whose gradients it completes (recorded after it runs).
    struct PendingWgrad {
        GemmArgs g;
        Buf a, b;
        int bucket = -1;
        bool live = false;
    };
    PendingWgrad pending_;
    void flush_wgrad(bool defer, cudaStream_t s) {
        if (!pending_.live) return;
        pending_.g.defer_wait = defer && defer_wgrad_;
        gemm(pending_.g, s);
        pending_.a.release();
        pending_.b.release();
        pending_.live = false;
        if (pending_.bucket >= 0) bucket_ready(pending_.bucket, s);
        pending_.bucket = -1;
    }

    // Last stage: final norm, LM head, cross-entropy and its backward through
    // the head, in row blocks so the [rows, vocab] logits stay bounded.
    void head_forward(ChunkState& cs, const epp_chunk_desc& c, const void* x, cudaStream_t s) {
        EPP_REQUIRE(c.target_ids != nullptr, "last stage needs target_ids");
        const int T = cs.T;
        const size_t e = esz();
        const int V = m_.vocab;
        cs.meanf = Buf(&pool_, sizeof(float) * T, s);
        cs.rstdf = Buf(&pool_, sizeof(float) * T, s);
        Buf xf(&pool_, static_cast<size_t>(T) * D_ * e, s);
        norm_fwd(dt_, llama_, x, work(lnf_w_), lnf_b_ >= 0 ? work(lnf_b_) : nullptr, xf.get(),
                 llama_ ? nullptr : cs.meanf.get<float>(), cs.rstdf.get<float>(), T, D_, m_.norm_eps,
                 s);
        cs.dxf = Buf(&pool_, static_cast<size_t>(T) * D_ * e, s);
        const int rows = std::max(1, std::min(T, static_cast<int>((512LL << 20) / (static_cast<long long>(V) * e))));
        Buf logits(&pool_, static_cast<size_t>(rows) * V * e, s);
        Buf row_loss(&pool_, sizeof(float) * T, s);
        for (int r0 = 0; r0 < T; r0 += rows) {
            const int n = std::min(rows, T - r0);
            const uint8_t* xr = xf.get<uint8_t>() + static_cast<size_t>(r0) * D_ * e;
            gemm(mk(n, V, D_, xr, D_, true, work(lm_), D_, true, logits.get(), V), s);
            cross_entropy(dt_, logits.get(), c.target_ids + r0, row_loss.get<float>() + r0, n, V, c.loss_scale, s);
            // dXf = dLogits Wlm ; dWlm += dLogits^T Xf
            gemm(mk(n, D_, V, logits.get(), V, true, work(lm_), D_, false,
                    cs.dxf.get<uint8_t>() + static_cast<size_t>(r0) * D_ * e, D_), s);
            wgrad(V, D_, n, logits.get(), V, xr, D_, grad(lm_), s, true);   // independent of dXf
        }
        auto slot = loss_slot_.find(c.id);
        if (slot == loss_slot_.end()) {
            EPP_REQUIRE(loss_slot_.size() < static_cast<size_t>(kLossSlots),
                        "chunk loss: too many chunks since the last loss reset");
            slot = loss_slot_.emplace(c.id, static_cast<int>(loss_slot_.size())).first;
        }
        chunk_loss(row_loss.get<float>(), c.target_ids, T, loss_acc_ + 2 * (1 + slot->second), loss_acc_, s);
    }

    GemmArgs mk(int M, int N, int K, const void* A, long long lda, bool ak, const void* B,
                long long ldb, bool bk, void* C, long long ldc) const {
        GemmArgs g;
        g.M = M; g.N = N; g.K = K;
        g.A = A; g.lda = lda; g.a_kmajor = ak;
        g.B = B; g.ldb = ldb; g.b_kmajor = bk;
        g.C = C; g.ldc = ldc;
        g.dtype = dt_;
        return g;
    }
    // dW[M,N] += sum_t dY[t, m] X[t, n]  (both operands MN-major)
    // defer: the previous kernel in the stream is independent of this one
    // (GemmArgs::defer_wait): the weight gradient fills its last wave.
    void wgrad(int M, int N, int T, const void* dy, long long ldy, const void* x, long long ldx,
               float* dw, cudaStream_t s, bool defer = false) const {
        GemmArgs g = mk(M, N, T, dy, ldy, false, x, ldx, false, dw, N);
        g.epi = Epi::AccumF32;
        g.defer_wait = defer && defer_wgrad_;
        gemm(g, s);
    }

    epp_model_desc m_;
    int first_, nl_;
    bool has_embed_, has_head_;
    DType dt_;
    int D_ = 0, H_ = 0, Hkv_ = 0, hd_ = 0, F_ = 0, F1_ = 0, Nqkv_ = 0;
    bool llama_ = false;
    bool defer_wgrad_ = true;
    std::vector<Param> params_;
    static constexpr long long kBucketAlign = 4096;
    std::vector<long long> bucket_off_;
    long long arena_n_ = 0;
    float* master_arena_ = nullptr;
    float* grad_arena_ = nullptr;
    void* work_arena_ = nullptr;
    float* m_arena_ = nullptr;
    float* v_arena_ = nullptr;
    AdamSeg* adam_segs_dev_ = nullptr;
    int adam_nseg_ = 0;
    long long adam_total4_ = 0;
    int opt_rank_ = 0, opt_nranks_ = 1;
    long long opt_state_n_ = 0;
    bool grad_events_ = false;
    std::vector<cudaEvent_t> bucket_ev_;
    std::vector<LayerParams> lps_;
    int emb_ = -1, lnf_w_ = -1, lnf_b_ = -1, lm_ = -1;
    static constexpr int kLossSlots = 1 << 16;
    double* loss_acc_ = nullptr;
    std::map<int, int> loss_slot_;   // chunk id -> loss record
    Pool pool_;
    TraceOp* trace_begin(int chunk, int kind, cudaStream_t s) {
        if (!tracer_.on()) return nullptr;
        TraceOp op;
        op.chunk = chunk;
        op.kind = kind;
        op.a = tracer_.record(s);
        tracer_.ops().push_back(std::move(op));
        return &tracer_.ops().back();
    }
    void trace_end(TraceOp* tr, cudaStream_t s) {
        if (!tr) return;
        tr->b = tracer_.record(s);
        tr->live = pool_.live;
    }

    Tracer tracer_;
    PinnedRing ring_{32u << 20};
    std::map<int, ChunkState> chunks_;
    std::map<int, SeqKV> seqs_;
};

}  // namespace eppk

// ===========================================================================
// C ABI
// ===========================================================================
struct epp_stage {
    std::unique_ptr<eppk::StageImpl> impl;
};

namespace {

template <typename F>
int guard(F&& f) {
    eppk::gpu_error_slot().clear();
    try {
        f();
        return EPP_GPU_OK;
    } catch (const eppk::CudaError& e) {
        eppk::gpu_error_slot() = e.what();
        return EPP_GPU_ECUDA;
    } catch (const std::invalid_argument& e) {
        eppk::gpu_error_slot() = e.what();
        return EPP_GPU_EARG;
    } catch (const std::exception& e) {
        eppk::gpu_error_slot() = e.what();
        return EPP_GPU_EOTHER;
    }
}

cudaStream_t S(void* p) { return static_cast<cudaStream_t>(p); }

}  // namespace

extern "C" {

int epp_gpu_set_device(int device) {
    return guard([&] { EPP_CUDA(cudaSetDevice(device)); });
}

int epp_stage_create(const epp_model_desc* model, int first_layer, int num_layers, int has_embed,
                     int has_head, int dtype, epp_stage** out) {
    return guard([&] {
        EPP_REQUIRE(model && out, "null argument");
        EPP_REQUIRE(dtype == EPP_DTYPE_F32 || dtype == EPP_DTYPE_BF16, "bad dtype");
        auto* st = new epp_stage;
        try {
            st->impl = std::make_unique<eppk::StageImpl>(*model, first_layer, num_layers, has_embed != 0,
                                                         has_head != 0, static_cast<eppk::DType>(dtype));
        } catch (...) {
            delete st;
            throw;
        }
        *out = st;
    });
}

int epp_stage_destroy(epp_stage* st) {
    return guard([&] { delete st; });
}

int epp_stage_init_weights(epp_stage* st, uint64_t seed, void* stream) {
    return guard([&] { st->impl->init_weights(seed, S(stream)); });
}

int epp_stage_num_params(epp_stage* st, int32_t* n) {
    return guard([&] { *n = static_cast<int32_t>(st->impl->params().size()); });
}

int epp_stage_param(epp_stage* st, int32_t idx, epp_param_info* info) {
    return guard([&] {
        auto& ps = st->impl->params();
        EPP_REQUIRE(idx >= 0 && idx < static_cast<int32_t>(ps.size()), "param index out of range");
        const auto& p = ps[idx];
        info->name = p.name.c_str();
        info->numel = p.numel;
        info->master = p.master;
        info->work = p.work;
        info->grad = p.grad;
    });
}

int epp_stage_sync_weights(epp_stage* st, void* stream) {
    return guard([&] { st->impl->sync_weights(S(stream)); });
}

int epp_stage_forward(epp_stage* st, const epp_chunk_desc* chunk, const void* act_in, void* act_out,
                      void* stream) {
    return guard([&] { st->impl->forward(*chunk, act_in, act_out, S(stream)); });
}

int epp_stage_backward(epp_stage* st, const epp_chunk_desc* chunk, const void* grad_in,
                       void* grad_out, void* stream) {
    return guard([&] { st->impl->backward(*chunk, grad_in, grad_out, S(stream)); });
}

int epp_seq_release(epp_stage* st, int32_t seq) {
    return guard([&] { st->impl->release_seq(seq); });
}

int epp_stage_loss(epp_stage* st, double out[2], int32_t reset, void* stream) {
    return guard([&] { st->impl->loss(out, reset != 0, S(stream)); });
}

int epp_stage_chunk_loss(epp_stage* st, int32_t chunk_id, double out[2], void* stream) {
    return guard([&] {
        EPP_REQUIRE(out != nullptr, "out is null");
        st->impl->read_chunk_loss(chunk_id, out, S(stream));
    });
}

int epp_stage_loss_async(epp_stage* st, double* out2, int32_t reset, void* stream) {
    return guard([&] {
        EPP_REQUIRE(out2 != nullptr, "out2 is null");
        st->impl->loss_async(out2, reset != 0, S(stream));
    });
}

int epp_gpu_pool_reserve(uint64_t bytes, void* stream) {
    return guard([&] {
        eppk::keep_pool_reserved();
        if (bytes == 0) return;
        cudaStream_t s = S(stream);
        void* p = nullptr;
        EPP_CUDA(cudaMallocAsync(&p, bytes, s));
        EPP_CUDA(cudaFreeAsync(p, s));
        EPP_CUDA(cudaStreamSynchronize(s));
    });
}

int epp_stage_zero_grads(epp_stage* st, void* stream) {
    return guard([&] { st->impl->zero_grads(S(stream)); });
}

int epp_stage_adamw_step(epp_stage* st, float lr, float beta1, float beta2, float eps,
                         float weight_decay, int32_t step, void* stream) {
    return guard([&] { st->impl->adamw_step(lr, beta1, beta2, eps, weight_decay, step, S(stream)); });
}

int epp_stage_memory(epp_stage* st, int64_t* live_bytes, int64_t* peak_bytes) {
    return guard([&] {
        if (live_bytes) *live_bytes = st->impl->pool().live;
        if (peak_bytes) *peak_bytes = st->impl->pool().peak;
    });
}

int epp_stage_arena(epp_stage* st, float** master, void** work, float** grad, int64_t* numel) {
    return guard([&] {
        if (master) *master = st->impl->master_arena();
        if (work) *work = st->impl->work_arena();
        if (grad) *grad = st->impl->grad_arena();
        if (numel) *numel = st->impl->arena_numel();
    });
}

int epp_stage_buckets(epp_stage* st, int64_t* offsets, int32_t cap, int32_t* nbuckets) {
    return guard([&] {
        EPP_REQUIRE(nbuckets != nullptr, "nbuckets is null");
        const auto& b = st->impl->buckets();
        *nbuckets = static_cast<int32_t>(b.size()) - 1;
        for (int32_t i = 0; offsets && i < cap && i < static_cast<int32_t>(b.size()); ++i) offsets[i] = b[i];
    });
}

int epp_stage_grad_events(epp_stage* st, int32_t enable) {
    return guard([&] { st->impl->grad_events(enable != 0); });
}

int epp_stage_bucket_wait(epp_stage* st, int32_t bucket, void* stream) {
    return guard([&] { st->impl->bucket_wait(bucket, S(stream)); });
}

int epp_stage_opt_shard(epp_stage* st, int32_t rank, int32_t nranks, int64_t* state_numel) {
    return guard([&] {
        st->impl->set_opt_shard(rank, nranks);
        if (state_numel) *state_numel = st->impl->opt_state_numel();
    });
}

int epp_stage_trace(epp_stage* st, int32_t enable, void* stream) {
    return guard([&] { st->impl->trace(enable != 0, S(stream)); });
}

int epp_stage_trace_read(epp_stage* st, epp_trace_event* out, int32_t cap, int32_t* n) {
    return guard([&] {
        EPP_REQUIRE(n != nullptr, "n is null");
        *n = st->impl->trace_read(out, cap);
    });
}

const char* epp_gpu_last_error(void) { return eppk::gpu_error_slot().c_str(); }

int64_t epp_gpu_kernel_launches(void) { return eppk::launch_counter(); }

}  // extern "C"
