// The persistent-executor kernel variants (tile-shape x occupancy x small
// block), instantiated in parallel translation units (tc_persist_inst.cu,
// one group each) and declared extern in tc_device.cu.
#pragma once
#define TC_PERSIST_VARIANTS(X)                                              \
    X(0, 64, 64, 2, 2, 2, 1, 0) X(1, 64, 64, 2, 2, 2, 2, 0)                 \
    X(2, 64, 64, 2, 2, 2, 1, 24) X(3, 64, 64, 2, 2, 2, 2, 24)               \
    X(4, 64, 64, 2, 2, 2, 1, 32) X(5, 64, 64, 2, 2, 2, 2, 32)               \
    X(6, 80, 48, 2, 2, 2, 1, 24) X(7, 80, 48, 2, 2, 2, 2, 24)               \
    X(0, 80, 40, 2, 1, 4, 1, 0) X(1, 80, 40, 2, 1, 4, 2, 0)                 \
    X(2, 80, 40, 2, 1, 4, 1, 32) X(3, 80, 40, 2, 1, 4, 2, 32)               \
    X(4, 40, 40, 1, 1, 8, 1, 0) X(5, 40, 40, 1, 1, 8, 2, 0)                 \
    X(6, 40, 40, 1, 1, 8, 1, 24) X(7, 40, 40, 1, 1, 8, 2, 24)               \
    X(0, 32, 32, 2, 2, 2, 1, 0) X(1, 32, 32, 2, 2, 2, 2, 0)                 \
    X(2, 128, 64, 4, 2, 1, 1, 32) X(3, 128, 128, 2, 4, 1, 1, 32)
#define TC_PERSIST_GROUPS 8
