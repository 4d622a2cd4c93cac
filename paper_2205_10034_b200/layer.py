"""Host-side MoE-layer operator over the C-ABI (moe_layer_* in include/moe_b200.h).

PyTorch is used only for device memory, streams and torch.distributed; every
compute step runs in libmoe_b200.so.  Parameter / input generation follows the
SplitMix64 substream convention of the reference (rng.hpp:19-42) so the CPU
oracle reproduces the same tensors bit for bit.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

import torch

from . import _lib
from ._lib import LayerDesc, LayerGrads, LayerParams, RoutingOut, call, lib

MASK64 = (1 << 64) - 1

# tensor ids for substream_seed(seed, tensor_id, index)
T_WG, T_BG, T_W1, T_B1, T_W2, T_B2, T_X, T_DY = range(8)


def substream_seed(seed: int, step: int, rank: int) -> int:
    """rng.hpp:40-42."""
    return (seed ^ ((0x9E3779B97F4A7C15 * (step + 1)) & MASK64)
            ^ ((0xC2B2AE3D27D4EB4F * (rank + 1)) & MASK64)) & MASK64


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _p(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()


def dtype_code(dtype: torch.dtype) -> int:
    if dtype == torch.bfloat16:
        return _lib.MOE_DTYPE_BF16
    if dtype == torch.float32:
        return _lib.MOE_DTYPE_F32
    raise _lib.ConfigError("layer.dtype: must be torch.bfloat16 or torch.float32")


def fill_uniform(t: torch.Tensor, seed: int, lo: float, hi: float, stream=None) -> torch.Tensor:
    """t[i] = lo + (hi-lo) * u_i, u_i = i-th SplitMix64(seed) draw (device kernel)."""
    assert t.is_cuda and t.is_contiguous()
    call("moe_fill_uniform", t.data_ptr(), t.numel(), dtype_code(t.dtype), seed, lo, hi,
         _stream(stream))
    return t


def capacity(top_k: int, capacity_factor: float, tokens: int, experts: int) -> int:
    """C = ceil(k * cf * T / E) (DESIGN.md Appendix A §5)."""
    return int(math.ceil(top_k * capacity_factor * tokens / experts))


@dataclass
class MoEConfig:
    num_experts: int
    top_k: int
    d_model: int
    d_ff: int
    capacity_factor: float
    tokens: int
    dtype: torch.dtype = torch.bfloat16
    gate_bias: bool = False
    exchange: str = "p2p"  # EP token exchange: "p2p" (NVLink peer stores) or "nccl"
    placement: str = "contiguous"  # expert placement over ranks: "contiguous" or "round_robin"
    gate_grad_reduce: str = "layer"  # EP gate-gradient sum: "layer" (in backward) or "caller"


class EPGroup:
    """NCCL communicator for expert parallelism; the 128-byte unique id travels
    over torch.distributed (any backend)."""

    def __init__(self, world_size: int, rank: int, pg=None):
        import torch.distributed as dist
        self.world_size, self.rank = world_size, rank
        idbuf = (C.c_uint8 * 128)()
        if rank == 0:
            call("moe_comm_unique_id", C.cast(idbuf, C.c_void_p))
        obj = [bytes(idbuf)]
        dist.broadcast_object_list(obj, src=0, group=pg)
        uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        comm = C.c_void_p()
        call("moe_comm_create", C.cast(uid, C.c_void_p), world_size, rank, C.byref(comm))
        self.comm = comm

    def alltoall_packed(self, send: torch.Tensor, recv: torch.Tensor, bytes_per_peer: int,
                        slices_per_peer: int = 1, fused: bool = True, stream=None) -> None:
        call("moe_alltoall_packed", self.comm, send.data_ptr(), recv.data_ptr(), bytes_per_peer,
             slices_per_peer, 1 if fused else 0, _stream(stream))

    def close(self):
        if self.comm:
            call("moe_comm_destroy", self.comm)
            self.comm = None


class MoELayer:
    """One MoE layer (gate + E experts) over T tokens per call.

    Parameters (nn.Linear-style [out, in] layouts): wg [E,d], bg [E] fp32,
    w1 [El,d_ff,d], b1 [El,d_ff] fp32, w2 [El,d,d_ff], b2 [El,d] fp32, where
    El = E / ep_size local experts of this rank.
    """

    def __init__(self, cfg: MoEConfig, ep: Optional[EPGroup] = None, device=None):
        self.cfg = cfg
        self.ep = ep
        self.P = ep.world_size if ep else 1
        self.rank = ep.rank if ep else 0
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        desc = LayerDesc()
        desc.num_experts = cfg.num_experts
        desc.top_k = cfg.top_k
        desc.d_model = cfg.d_model
        desc.d_ff = cfg.d_ff
        desc.capacity_factor = cfg.capacity_factor
        desc.tokens = cfg.tokens
        desc.dtype = dtype_code(cfg.dtype)
        desc.has_gate_bias = 1 if cfg.gate_bias else 0
        desc.ep_size = self.P
        desc.ep_rank = self.rank
        desc.nccl_comm = ep.comm if ep else None
        if cfg.exchange not in ("p2p", "nccl"):
            raise _lib.ConfigError("layer.exchange: must be 'p2p' or 'nccl'")
        desc.exchange = 0 if cfg.exchange == "p2p" else 1
        if cfg.placement not in ("contiguous", "round_robin"):
            raise _lib.ConfigError("layer.placement: must be 'contiguous' or 'round_robin'")
        desc.placement = 0 if cfg.placement == "contiguous" else 1
        if cfg.gate_grad_reduce not in ("layer", "caller"):
            raise _lib.ConfigError("layer.gate_grad_reduce: must be 'layer' or 'caller'")
        desc.gate_grad_reduce = 0 if cfg.gate_grad_reduce == "layer" else 1
        h = C.c_void_p()
        if self.device.type == "cuda":
            with torch.cuda.device(self.device):
                call("moe_layer_create", C.byref(desc), C.byref(h))
        else:  # validation only (raises before any device work)
            call("moe_layer_create", C.byref(desc), C.byref(h))
        self._h = h
        self.capacity = int(lib.moe_layer_capacity(h))
        self.El = cfg.num_experts // self.P
        # global expert id of each local expert (include/moe_b200.h placement)
        if cfg.placement == "round_robin":
            self.local_experts = [j * self.P + self.rank for j in range(self.El)]
        else:
            self.local_experts = [self.rank * self.El + j for j in range(self.El)]
        self.params: Dict[str, torch.Tensor] = {}
        self.grads: Dict[str, torch.Tensor] = {}

    # ------------------------------------------------------------- params --
    def init_params(self, seed: int, gate_bias: Optional[torch.Tensor] = None) -> None:
        c, dev = self.cfg, self.device
        E, d, f, El = c.num_experts, c.d_model, c.d_ff, self.El
        dt = c.dtype
        bd, bf = 1.0 / math.sqrt(d), 1.0 / math.sqrt(f)
        p = {
            "wg": torch.empty(E, d, dtype=dt, device=dev),
            "bg": torch.zeros(E, dtype=torch.float32, device=dev),
            "w1": torch.empty(El, f, d, dtype=dt, device=dev),
            "b1": torch.empty(El, f, dtype=torch.float32, device=dev),
            "w2": torch.empty(El, d, f, dtype=dt, device=dev),
            "b2": torch.empty(El, d, dtype=torch.float32, device=dev),
        }
        fill_uniform(p["wg"], substream_seed(seed, T_WG, 0), -bd, bd)
        if gate_bias is not None:
            p["bg"].copy_(gate_bias)
        for j in range(El):
            e = self.local_experts[j]  # global expert id: identical weights for any ep_size
            fill_uniform(p["w1"][j], substream_seed(seed, T_W1, e), -bd, bd)
            fill_uniform(p["b1"][j], substream_seed(seed, T_B1, e), -bd, bd)
            fill_uniform(p["w2"][j], substream_seed(seed, T_W2, e), -bf, bf)
            fill_uniform(p["b2"][j], substream_seed(seed, T_B2, e), -bf, bf)
        self.params = p
        self.grads = {
            "dwg": torch.zeros(E, d, dtype=torch.float32, device=dev),
            "dbg": torch.zeros(E, dtype=torch.float32, device=dev),
            "dw1": torch.zeros(El, f, d, dtype=torch.float32, device=dev),
            "db1": torch.zeros(El, f, dtype=torch.float32, device=dev),
            "dw2": torch.zeros(El, d, f, dtype=torch.float32, device=dev),
            "db2": torch.zeros(El, d, dtype=torch.float32, device=dev),
        }

    def _params(self) -> LayerParams:
        p = self.params
        lp = LayerParams()
        lp.wg, lp.bg = _p(p["wg"]), _p(p["bg"]) if self.cfg.gate_bias else None
        lp.w1, lp.b1, lp.w2, lp.b2 = _p(p["w1"]), _p(p["b1"]), _p(p["w2"]), _p(p["b2"])
        return lp

    def _grads(self) -> LayerGrads:
        g = self.grads
        lg = LayerGrads()
        lg.dwg, lg.dbg, lg.dw1 = _p(g["dwg"]), _p(g["dbg"]), _p(g["dw1"])
        lg.db1, lg.dw2, lg.db2 = _p(g["db1"]), _p(g["dw2"]), _p(g["db2"])
        return lg

    def make_input(self, seed: int, tensor_id: int = T_X) -> torch.Tensor:
        c = self.cfg
        x = torch.empty(c.tokens, c.d_model, dtype=c.dtype, device=self.device)
        return fill_uniform(x, substream_seed(seed, tensor_id, self.rank), -1.0, 1.0)

    # ------------------------------------------------------------ compute --
    def forward(self, x: torch.Tensor, logits_override: Optional[torch.Tensor] = None,
                routing: bool = False, stream=None):
        c = self.cfg
        assert x.shape == (c.tokens, c.d_model) and x.dtype == c.dtype and x.is_contiguous()
        y = torch.empty_like(x)
        T, E, k = c.tokens, c.num_experts, c.top_k
        rout = None
        ro = None
        logits = None
        if routing:
            dev = self.device
            rout = {
                "expert": torch.empty(T, k, dtype=torch.int32, device=dev),
                "gate": torch.empty(T, k, dtype=torch.float32, device=dev),
                "position": torch.empty(T, k, dtype=torch.int32, device=dev),
                "keep": torch.empty(T, k, dtype=torch.uint8, device=dev),
                "count1": torch.empty(E, dtype=torch.int32, device=dev),
                "count2": torch.empty(E, dtype=torch.int32, device=dev),
                "kept": torch.empty(E, dtype=torch.int32, device=dev),
                "aux_loss": torch.empty(1, dtype=torch.float32, device=dev),
            }
            ro = RoutingOut(*[rout[n].data_ptr() for n in
                              ("expert", "gate", "position", "keep", "count1", "count2", "kept",
                               "aux_loss")])
            logits = torch.empty(T, E, dtype=torch.float32, device=dev)
            rout["logits"] = logits
        lp = self._params()
        call("moe_layer_forward", self._h, C.byref(lp), x.data_ptr(), y.data_ptr(),
             _p(logits_override), _p(logits), C.byref(ro) if ro is not None else None,
             _stream(stream))
        self._x = x  # the backward's gate GEMM reads x
        return (y, rout) if routing else y

    def backward(self, dy: torch.Tensor, d_aux: float = 0.0, stream=None) -> torch.Tensor:
        c = self.cfg
        assert dy.shape == (c.tokens, c.d_model) and dy.dtype == c.dtype and dy.is_contiguous()
        dx = torch.empty_like(dy)
        lp, lg = self._params(), self._grads()
        call("moe_layer_backward", self._h, C.byref(lp), dy.data_ptr(), float(d_aux),
             dx.data_ptr(), C.byref(lg), _stream(stream))
        return dx

    def train_step_host(self, x_host: torch.Tensor, dy_host: torch.Tensor, y_host: torch.Tensor,
                        dx_host: torch.Tensor, d_aux: float = 0.0, stream=None,
                        deferred: bool = False) -> None:
        """End-to-end step from pinned host buffers (H2D, fwd, bwd, D2H).
        deferred=True: y_host / dx_host are complete once the stream reaches
        the next call or host_sync() (moe_layer_train_step_host_async)."""
        lp, lg = self._params(), self._grads()
        fn = "moe_layer_train_step_host_async" if deferred else "moe_layer_train_step_host"
        call(fn, self._h, C.byref(lp), x_host.data_ptr(), dy_host.data_ptr(), float(d_aux),
             y_host.data_ptr(), dx_host.data_ptr(), C.byref(lg), _stream(stream))

    def host_sync(self, stream=None) -> None:
        call("moe_layer_host_sync", self._h, _stream(stream))

    def set_peer_timeout(self, seconds: float) -> None:
        """Limit of the NVLink exchange's peer waits (0 = wait forever)."""
        call("moe_layer_set_peer_timeout", self._h, float(seconds))

    def comm_status(self) -> int:
        """0, or raises MoEError when a peer missed the peer-wait limit."""
        code = C.c_int32(0)
        call("moe_layer_comm_status", self._h, C.byref(code))
        return code.value

    def set_profiling(self, on: bool) -> None:
        call("moe_layer_set_profiling", self._h, 1 if on else 0)

    def phase_list(self, which: Optional[str] = None) -> List[Tuple[str, float]]:
        """(phase, ms) in launch order (profiling on) of the last call, or of
        the last forward / backward (which = "fwd" / "bwd")."""
        names = (C.c_char_p * 64)()
        ms = (C.c_float * 64)()
        n = C.c_uint32(0)
        if which is None:
            call("moe_layer_phase_times", self._h, names, ms, 64, C.byref(n))
        else:
            call("moe_layer_phase_times_of", self._h, 1 if which == "bwd" else 0, names, ms, 64,
                 C.byref(n))
        return [(names[i].decode(), float(ms[i])) for i in range(n.value)]

    def phase_times(self) -> Dict[str, float]:
        out: Dict[str, float] = {}
        for name, ms in self.phase_list():
            out[name] = out.get(name, 0.0) + ms
        return out

    def close(self):
        if getattr(self, "_h", None):
            call("moe_layer_destroy", self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def route(logits: torch.Tensor, top_k: int, capacity_: int, stream=None) -> Dict[str, torch.Tensor]:
    """Standalone K2 routing on fp32 logits [T,E] (moe_route)."""
    assert logits.dtype == torch.float32 and logits.is_contiguous()
    T, E = logits.shape
    dev = logits.device
    out = {
        "expert": torch.empty(T, top_k, dtype=torch.int32, device=dev),
        "gate": torch.empty(T, top_k, dtype=torch.float32, device=dev),
        "position": torch.empty(T, top_k, dtype=torch.int32, device=dev),
        "keep": torch.empty(T, top_k, dtype=torch.uint8, device=dev),
        "count1": torch.empty(E, dtype=torch.int32, device=dev),
        "count2": torch.empty(E, dtype=torch.int32, device=dev),
        "kept": torch.empty(E, dtype=torch.int32, device=dev),
        "aux_loss": torch.empty(1, dtype=torch.float32, device=dev),
    }
    ro = RoutingOut(*[out[n].data_ptr() for n in ("expert", "gate", "position", "keep", "count1",
                                                  "count2", "kept", "aux_loss")])
    call("moe_route", T, E, top_k, capacity_, logits.data_ptr(), C.byref(ro), _stream(stream))
    return out


def grouped_gemm(problem: _lib.GemmProblem, stream=None) -> None:
    call("moe_grouped_gemm", C.byref(problem), _stream(stream))


def kernel_launch_count() -> int:
    return int(lib.moe_kernel_launch_count())
