// pa_alloc.cpp -- host block allocator: the paper's KV block manager (P:249-256,
// P:295-332), used only to generate block tables, slot mappings and
// copy-on-write pairs.  Plain C++ on the host; no CUDA.
//
//  * physical blocks handed out from a FIFO free list seeded with `initial_order`;
//    freed blocks join the back (Fig.9: after freeing 2,4,5,8 the new blocks are 9-12,
//    P:330);
//  * allocate fills logical blocks left to right (Fig.6);
//  * append_slot: in place / new block / copy-on-write of a shared partial last block
//    (P:302-304);
//  * fork shares every block (refcount + 1); free releases blocks whose count drops to 0.
#include "../../include/pa.h"

#include <deque>
#include <string>
#include <vector>

namespace {
thread_local std::string g_alloc_err;
}

struct pa_alloc {
    struct Entry {
        int block;
        int filled;
    };
    struct Seq {
        bool live = false;
        std::vector<Entry> entries;
    };
    int num_blocks = 0;
    int B = 0;
    std::deque<int> free_list;
    std::vector<int> ref;
    std::vector<Seq> seqs;

    int pop() {
        const int b = free_list.front();
        free_list.pop_front();
        ref[b] = 1;
        return b;
    }
    bool valid(int s) const { return s >= 0 && s < (int)seqs.size() && seqs[s].live; }
};

extern "C" {

pa_alloc_t* pa_alloc_create(int num_blocks, int block_size, const int32_t* initial_order) {
    if (num_blocks <= 0 || block_size <= 0) return nullptr;
    pa_alloc* a = new pa_alloc();
    a->num_blocks = num_blocks;
    a->B = block_size;
    a->ref.assign(num_blocks, 0);
    if (initial_order) {
        std::vector<char> seen(num_blocks, 0);
        for (int i = 0; i < num_blocks; ++i) {
            const int b = initial_order[i];
            if (b < 0 || b >= num_blocks || seen[b]) {
                delete a;
                return nullptr;
            }
            seen[b] = 1;
            a->free_list.push_back(b);
        }
    } else {
        for (int i = 0; i < num_blocks; ++i) a->free_list.push_back(i);
    }
    return a;
}

void pa_alloc_destroy(pa_alloc_t* a) { delete a; }

pa_status_t pa_alloc_allocate(pa_alloc_t* a, int num_tokens, int* seq_out) {
    if (!a || !seq_out || num_tokens <= 0) return PA_ERR_INVALID_ARG;
    const int n = (num_tokens + a->B - 1) / a->B;
    if (n > (int)a->free_list.size()) return PA_ERR_OUT_OF_BLOCKS;
    pa_alloc::Seq s;
    s.live = true;
    int left = num_tokens;
    for (int i = 0; i < n; ++i) {
        const int f = left < a->B ? left : a->B;
        s.entries.push_back({a->pop(), f});
        left -= f;
    }
    a->seqs.push_back(std::move(s));
    *seq_out = (int)a->seqs.size() - 1;
    return PA_OK;
}

pa_status_t pa_alloc_append_slot(pa_alloc_t* a, int seq, int64_t* slot_out, int* cow_src_out, int* cow_dst_out) {
    if (!a || !a->valid(seq) || !slot_out || !cow_src_out || !cow_dst_out) return PA_ERR_INVALID_ARG;
    auto& e = a->seqs[seq].entries;
    *cow_src_out = *cow_dst_out = -1;
    if (e.empty() || e.back().filled == a->B) {  // last block full: new block (Fig.6 step 3)
        if (a->free_list.empty()) return PA_ERR_OUT_OF_BLOCKS;
        const int b = a->pop();
        e.push_back({b, 1});
        *slot_out = (int64_t)b * a->B;
        return PA_OK;
    }
    pa_alloc::Entry& last = e.back();
    if (a->ref[last.block] == 1) {  // sole owner: write in place (Fig.6 step 2)
        *slot_out = (int64_t)last.block * a->B + last.filled;
        ++last.filled;
        return PA_OK;
    }
    // shared partial block: copy-on-write
    if (a->free_list.empty()) return PA_ERR_OUT_OF_BLOCKS;
    const int dst = a->pop();
    --a->ref[last.block];
    *cow_src_out = last.block;
    *cow_dst_out = dst;
    last.block = dst;
    *slot_out = (int64_t)dst * a->B + last.filled;
    ++last.filled;
    return PA_OK;
}

pa_status_t pa_alloc_fork(pa_alloc_t* a, int parent, int* child_out) {
    if (!a || !a->valid(parent) || !child_out) return PA_ERR_INVALID_ARG;
    pa_alloc::Seq c;
    c.live = true;
    c.entries = a->seqs[parent].entries;
    for (const auto& en : c.entries) ++a->ref[en.block];
    a->seqs.push_back(std::move(c));
    *child_out = (int)a->seqs.size() - 1;
    return PA_OK;
}

pa_status_t pa_alloc_free(pa_alloc_t* a, int seq, int* freed_out) {
    if (!a || !a->valid(seq)) return PA_ERR_INVALID_ARG;  // unknown handle or double free
    int freed = 0;
    for (const auto& en : a->seqs[seq].entries) {
        if (a->ref[en.block] <= 0) return PA_ERR_INVALID_ARG;  // refcount underflow
        if (--a->ref[en.block] == 0) {
            a->free_list.push_back(en.block);
            ++freed;
        }
    }
    a->seqs[seq].live = false;
    a->seqs[seq].entries.clear();
    if (freed_out) *freed_out = freed;
    return PA_OK;
}

pa_status_t pa_alloc_export(const pa_alloc_t* a, const int* seqs, int n, int W, int32_t* block_tables_out,
                            int32_t* context_lens_out) {
    if (!a || n < 0 || W <= 0 || (n > 0 && (!seqs || !block_tables_out || !context_lens_out))) return PA_ERR_INVALID_ARG;
    for (int i = 0; i < n; ++i) {
        if (!a->valid(seqs[i])) return PA_ERR_INVALID_ARG;
        const auto& e = a->seqs[seqs[i]].entries;
        if ((int)e.size() > W) return PA_ERR_INVALID_ARG;
        int32_t tokens = 0;
        for (int j = 0; j < W; ++j) {
            if (j < (int)e.size()) {
                block_tables_out[(int64_t)i * W + j] = e[j].block;
                tokens += e[j].filled;
            } else {
                block_tables_out[(int64_t)i * W + j] = -1;
            }
        }
        context_lens_out[i] = tokens;
    }
    return PA_OK;
}

int pa_alloc_refcount(const pa_alloc_t* a, int block) {
    if (!a || block < 0 || block >= a->num_blocks) return -1;
    return a->ref[block];
}

int pa_alloc_num_free(const pa_alloc_t* a) { return a ? (int)a->free_list.size() : -1; }

int pa_alloc_num_blocks_of(const pa_alloc_t* a, int seq) {
    if (!a || !a->valid(seq)) return -1;
    return (int)a->seqs[seq].entries.size();
}

}  // extern "C"
