// NCCL status -> moe::Error(MOE_ERR_NCCL, "<call>: <nccl message>").
#pragma once

#include <nccl.h>

#include <string>

#include "common.cuh"

#define MOE_NCCL(expr)                                                                  \
  do {                                                                                  \
    ncclResult_t _r = (expr);                                                           \
    if (_r != ncclSuccess)                                                              \
      ::moe::fail(MOE_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(_r));    \
  } while (0)
