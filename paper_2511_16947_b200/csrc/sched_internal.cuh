// sched_internal.cuh — layout of the opaque hep_sched handle (shared by the
// scheduler and the dispatch kernels; not part of the C ABI).
#pragma once
#include <stdint.h>

#include <vector>

struct hep_sched {
    int G, E, nnz, gpn;
    int64_t Q, max_ranges;
    int32_t *d_grp_off = nullptr;    // [E+1]
    int32_t *d_grp_gpu = nullptr;    // [nnz]  EDP list order
    int32_t *d_sorted = nullptr;     // [nnz]  nnz index of the k-th arc of expert e in gpu-id order
    uint32_t *d_mask = nullptr;      // [E]
    int32_t *d_slots = nullptr;      // [E]
    int32_t *d_hosted_off = nullptr; // [G+1] segment offsets per destination GPU
    int32_t *d_seg_nnz = nullptr;    // [nnz]  nnz index of segment position p ([dst][expert asc])
    int32_t *d_nnz_exp = nullptr;    // [nnz]  expert of each nnz entry
    int8_t *d_kidx = nullptr;        // [E*G]  list position of GPU g in expert e's group (-1: absent)
    size_t smem_set = 0;             // dynamic smem opt-in already granted
    cudaEvent_t ev_fork = nullptr;   // pipelined split: forks the static phase onto its stream
    std::vector<int32_t> h_grp_off, h_grp_gpu, h_slots, h_hosted_off;
};
