"""Strong scaling of one grid over G GPUs.

apply(SystemOperator) (reference src/cie.cpp:56-73 over src/toeplitz.cpp:163-283)
split at its contraction:

  1. every rank owns a depth slab -- all three components of the intervals
     [z0, z1) -- and transforms it laterally (r2 scaling, zero-padded 2-D
     DFTs): S_loc[r][m][c*nzl + z], mode m = mx*ey + my;
  2. all-to-all #1: rank h sends rank g the columns of g's modes (the 1-4
     mirrors of g's quadrant modes, in contraction order) for its planes; g
     scatters them into the full-depth spectrum S[r][m][c*nz + z];
  3. rank g contracts its quadrant modes [q0, q1) with its shard of the
     spectra (1/G of the operator in HBM) -- or, with ShardPlan(octant=True)
     on an x <-> y symmetric operator, the octant items of its rows of
     quadrant modes, reading each block once for a mode and its transpose;
  4. all-to-all #2 returns the columns to the slab owners;
  5. every rank inverse-transforms its slab with the system epilogue.

The per-rank stages are separate methods so the same code runs under NCCL
(one process per GPU), gloo on CPU (tests, NumPy backend) or a loopback that
runs G virtual ranks in one process (one-GPU parity tests). Backends: CUDA
(the C ABI of libemie_cu.so on torch tensors) and NumPy (the restatement of
tests/numpy_backend.py, test infrastructure only).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List, Sequence

import numpy as np


# ------------------------------------------------------------------ plan ----
def _splits(n: int, g: int) -> List[int]:
    return [(i * n) // g for i in range(g + 1)]


def mirror_modes(qm: int, qx: int, ex: int, ey: int) -> List[int]:
    """Full modes m = mx*ey + my of quadrant mode qm in contraction order
    (operator.cu mirror_mode; emie_cu_mode_list)."""
    qmy, qmx = divmod(qm, qx)
    mx_ok = qmx > 0 and (ex - qmx) > ex // 2
    my_ok = qmy > 0 and (ey - qmy) > ey // 2
    out = [qmx * ey + qmy]
    if mx_ok:
        out.append((ex - qmx) * ey + qmy)
    if my_ok:
        out.append(qmx * ey + (ey - qmy))
    if mx_ok and my_ok:
        out.append((ex - qmx) * ey + (ey - qmy))
    return out


def octant_row_splits(qy: int, G: int) -> List[int]:
    """Row boundaries of G octant shards: rank g owns rows [b_g, b_g+1) of
    quadrant modes, i.e. the octant items (qmy, qmx <= qmy) of those rows --
    2 qmy + 1 quadrant modes per row, r^2 over rows [0, r) -- balanced by
    that count (b_g ~ qy sqrt(g / G)), at least one row each."""
    if not 1 <= G <= qy:
        raise ValueError("octant shard plan: need 1 <= G <= qy")
    b = [0] + [int(round(qy * np.sqrt(g / G))) for g in range(1, G)] + [qy]
    for g in range(1, G + 1):  # strictly increasing, room for the ranks after g
        b[g] = min(max(b[g], b[g - 1] + 1), qy - (G - g))
    return b


@dataclass
class ShardPlan:
    """Depth slabs and mode shards of G ranks for one grid.

    octant=False: rank g owns quadrant modes [q_g, q_g+1) and contracts them.
    octant=True (x <-> y symmetric operators, ex == ey): rank g owns whole
    rows [b_g, b_g+1) of quadrant modes (its operator shard, q_g = b_g qx)
    and contracts their octant items: each stored block (qmy, qmx <= qmy) is
    read once and serves that mode and its transpose (qmx, qmy), so the rank's
    modes are every quadrant mode whose larger index is one of its rows (an
    L-shaped set) and its operator reads halve (csrc/operator.cu
    contract_mma_kernel OCT, Operator::shard_octant)."""
    nx: int
    ny: int
    nz: int
    ex: int
    ey: int
    G: int
    octant: bool = False

    def __post_init__(self):
        if not 1 <= self.G <= self.nz:
            raise ValueError("shard plan: need 1 <= G <= nz (every rank owns at least one interval)")
        self.qx, self.qy = self.ex // 2 + 1, self.ey // 2 + 1
        self.E = self.ex * self.ey
        self.z = _splits(self.nz, self.G)
        if self.octant:
            if self.ex != self.ey:
                raise ValueError("octant shard plan: needs a square embedding (ex == ey)")
            self.rows = octant_row_splits(self.qy, self.G)
            self.q = [r * self.qx for r in self.rows]
            self.qmodes = [[qm for r in range(self.rows[g], self.rows[g + 1])
                            for qm in [r * self.qx + c for c in range(r + 1)] + [c * self.qx + r for c in range(r)]]
                           for g in range(self.G)]
        else:
            self.q = _splits(self.qx * self.qy, self.G)
            self.qmodes = [list(range(self.q[g], self.q[g + 1])) for g in range(self.G)]
        self.modes = [np.array([m for qm in self.qmodes[g]
                                for m in mirror_modes(qm, self.qx, self.ex, self.ey)], dtype=np.int32)
                      for g in range(self.G)]

    def nzl(self, g: int) -> int:
        return self.z[g + 1] - self.z[g]

    def slab_cells(self, g: int) -> int:
        return self.nzl(g) * self.ny * self.nx


def slab_of(u: np.ndarray, plan: ShardPlan, g: int, nrhs: int) -> np.ndarray:
    """Rank g's part [nrhs][3][nzl][ny][nx] of nrhs GridVectors (flat)."""
    v = np.asarray(u).reshape(nrhs, 3, plan.nz, plan.ny, plan.nx)
    return np.ascontiguousarray(v[:, :, plan.z[g]:plan.z[g + 1]])


def join_slabs(parts: Sequence[np.ndarray], plan: ShardPlan, nrhs: int) -> np.ndarray:
    """Inverse of slab_of over all ranks: nrhs flat GridVectors."""
    v = np.concatenate([np.asarray(p).reshape(nrhs, 3, plan.nzl(g), plan.ny, plan.nx)
                        for g, p in enumerate(parts)], axis=2)
    return v.reshape(nrhs, -1)


# -------------------------------------------------------- orchestration ----
class ShardedApply:
    """One rank's share of the sharded apply(SystemOperator)."""

    def __init__(self, plan: ShardPlan, rank: int, backend, nrhs: int):
        self.plan, self.rank, self.be, self.nrhs = plan, rank, backend, nrhs
        self.nzl = plan.nzl(rank)
        self.q0, self.q1 = plan.q[rank], plan.q[rank + 1]

    # column descriptors {mapped, planes per column, component stride, depth offset}
    def _slab_desc(self, mapped: bool):
        return (1 if mapped else 0, 3 * self.nzl, self.nzl, 0)

    def stage_forward(self, U):
        """Slab transform and the packed columns for every destination rank."""
        P, be = self.plan, self.be
        S_loc = be.lateral_forward(U, self.nrhs)
        self._U, self._S_loc = U, S_loc
        sends = []
        for g in range(P.G):
            buf = be.empty((self.nrhs, len(P.modes[g]), 3 * self.nzl))
            be.move(S_loc, buf, self.nrhs, g, P.E, self._slab_desc(True), self._slab_desc(False), self.nzl)
            sends.append(buf)
        return sends

    def stage_contract(self, recvs):
        """Scatter the slabs' columns into the full-depth spectrum of this
        rank's modes, contract them, pack the results per slab owner."""
        P, be, me = self.plan, self.be, self.rank
        # only this rank's mode columns are written (all planes, by the scatters
        # below) and read (contraction, packs): no zero fill needed
        S = be.empty((self.nrhs, P.E, 3 * P.nz))
        for h, buf in enumerate(recvs):
            nzh = P.nzl(h)
            be.move(buf, S, self.nrhs, me, P.E, (0, 3 * nzh, nzh, 0), (1, 3 * P.nz, P.nz, P.z[h]), nzh)
        be.contract(S, self.nrhs, self.q0, self.q1)
        sends = []
        for h in range(P.G):
            nzh = P.nzl(h)
            buf = be.empty((self.nrhs, len(P.modes[me]), 3 * nzh))
            be.move(S, buf, self.nrhs, me, P.E, (1, 3 * P.nz, P.nz, P.z[h]), (0, 3 * nzh, nzh, 0), nzh)
            sends.append(buf)
        return sends

    def stage_inverse(self, recvs):
        """Columns back into the slab spectrum, inverse transform + epilogue."""
        P, be = self.plan, self.be
        for g, buf in enumerate(recvs):
            be.move(buf, self._S_loc, self.nrhs, g, P.E, self._slab_desc(False), self._slab_desc(True), self.nzl)
        out = be.lateral_inverse(self._S_loc, self._U, self.nrhs)
        self._S_loc = self._U = None
        return out


def loopback_apply(shards: Sequence[ShardedApply], slabs):
    """G virtual ranks in one process: the all-to-alls are list transposes."""
    s1 = [sh.stage_forward(u) for sh, u in zip(shards, slabs)]
    s2 = [sh.stage_contract([s1[h][g] for h in range(len(shards))]) for g, sh in enumerate(shards)]
    return [sh.stage_inverse([s2[g][h] for g in range(len(shards))]) for h, sh in enumerate(shards)]


def torch_all_to_all(group=None):
    """all_to_all over torch.distributed (NCCL on GPUs, gloo on CPU) on
    complex128 tensors of per-peer shapes known to both sides."""
    import torch
    import torch.distributed as dist

    use_p2p = dist.get_backend(group) != "nccl"  # gloo has no alltoall: pairwise send/recv

    def a2a(sends, recv_shapes):
        ins = [torch.view_as_real(s.contiguous()).reshape(-1) for s in sends]
        dev = ins[0].device
        if use_p2p and dev.type != "cpu":  # gloo point-to-point moves host tensors only
            ins = [t.cpu() for t in ins]
        outs = [torch.empty(int(np.prod(sh)) * 2, dtype=torch.float64, device=ins[0].device) for sh in recv_shapes]
        if use_p2p:
            me = dist.get_rank(group)
            reqs = []
            for h in range(len(ins)):
                if h == me:
                    outs[h].copy_(ins[h])
                else:
                    reqs.append(dist.isend(ins[h], h, group=group))
                    reqs.append(dist.irecv(outs[h], h, group=group))
            for r in reqs:
                r.wait()
        else:
            dist.all_to_all(outs, ins, group=group)
        if outs[0].device != dev:
            outs = [o.to(dev) for o in outs]
        return [torch.view_as_complex(o.view(-1, 2)).view(sh) for o, sh in zip(outs, recv_shapes)]
    return a2a


class DistributedSystem:
    """The sharded apply of one grid on this rank (NCCL / gloo plumbing).
    recv shapes of both exchanges follow from the plan."""

    def __init__(self, shard: ShardedApply, group=None):
        self.sh, self.a2a = shard, torch_all_to_all(group)

    def apply(self, U):
        sh, P = self.sh, self.sh.plan
        me = sh.rank
        s1 = sh.stage_forward(U)
        r1 = self.a2a(s1, [(sh.nrhs, len(P.modes[me]), 3 * P.nzl(h)) for h in range(P.G)])
        s2 = sh.stage_contract(r1)
        r2 = self.a2a(s2, [(sh.nrhs, len(P.modes[g]), 3 * sh.nzl) for g in range(P.G)])
        return sh.stage_inverse(r2)


# ------------------------------------------------- peer-memory exchange ----
class _Buf:
    """A device buffer by address (exchange buffers live outside torch's
    allocator: CUDA IPC maps whole cudaMalloc allocations)."""

    def __init__(self, ptr: int):
        self.ptr = int(ptr)

    def data_ptr(self) -> int:
        return self.ptr


class PeerExchange:
    """The sharded apply with the two column transposes done as peer stores
    (SURVEY.md §8(e).3 over NVLink / NVSwitch; csrc/peer.cu): every rank owns
    two exchange buffers -- its slab spectrum S_loc[r][m][3 nzl] and the
    full-depth spectrum S_full[r][m][3 nz] of its quadrant modes -- plus a
    flag array of G ints, all mapped into every rank through CUDA IPC. A rank
    moves its slab's columns straight into each owner's S_full (one
    move_planes pass per destination, the stores cross NVLink), signals the
    owners, waits for its own G flags, contracts in place, moves the results
    straight into each slab owner's S_loc, signals, waits, and inverse
    transforms. No pack / all-to-all / unpack copies and no NCCL call on the
    data path; the two flag barriers per apply order the buffers' reuse.

    `peers` gives, per rank g, (S_loc, S_full, flags) device addresses as
    seen from this process: the rank's own allocations for itself, IPC
    mappings of the others' (PeerExchange.open_ipc) or, for G virtual ranks
    in one process, the other shards' own buffers (loopback)."""

    def __init__(self, shard: "ShardedApply", peers, own, fused: bool = True):
        self.sh, self.peers, self.own = shard, peers, own
        self.epoch = 0
        self.fused = fused  # contraction + return transpose in one kernel where the backend has it
        # flag arrays: device addresses (None: a host backend, no device flags)
        self._flag_ptrs = (None if own[2] is None else
                           (ctypes.c_void_p * shard.plan.G)(*[p[2] for p in peers]))

    @staticmethod
    def allocate(shard: "ShardedApply"):
        """This rank's exchange buffers: (S_loc, S_full, flags) addresses."""
        from . import lib, _check
        L, P = lib(), shard.plan
        sizes = [shard.nrhs * P.E * 3 * shard.nzl * 16, shard.nrhs * P.E * 3 * P.nz * 16, 4 * P.G]
        out = []
        for b in sizes:
            p = ctypes.c_void_p()
            _check(L.emie_cu_peer_alloc(b, ctypes.byref(p)))
            out.append(p.value)
        return (_Buf(out[0]), _Buf(out[1]), out[2])

    @staticmethod
    def allocate_host(shard: "ShardedApply"):
        """Host tensors for a NumPy-backend shard (CPU tests of the exchange
        plan: same moves and stage order, no device flags)."""
        P, be = shard.plan, shard.be
        return (be.zeros((shard.nrhs, P.E, 3 * shard.nzl)), be.zeros((shard.nrhs, P.E, 3 * P.nz)), None)

    @staticmethod
    def _addrs(own):
        return [own[0].data_ptr(), own[1].data_ptr(), own[2]]

    @staticmethod
    def free(own):
        from . import lib
        for p in PeerExchange._addrs(own):
            lib().emie_cu_peer_free(ctypes.c_void_p(p))

    @staticmethod
    def ipc_handles(own) -> List[bytes]:
        from . import lib, _check
        out = []
        for p in PeerExchange._addrs(own):
            h = ctypes.create_string_buffer(64)
            _check(lib().emie_cu_ipc_handle(ctypes.c_void_p(p), h))
            out.append(h.raw)
        return out

    @staticmethod
    def open_ipc(handles: List[bytes]):
        from . import lib, _check
        out = []
        for h in handles:
            p = ctypes.c_void_p()
            _check(lib().emie_cu_ipc_open(ctypes.create_string_buffer(h, 64), ctypes.byref(p)))
            out.append(p.value)
        return (_Buf(out[0]), _Buf(out[1]), out[2])

    def _stream(self):
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    host_barrier = None  # callable: host-side exchange barrier instead of the flag kernels

    def signal(self):
        """After this rank's pushes (stream order): epoch += 1 into every rank's flag slot."""
        from . import lib, _check
        self.epoch += 1
        if self.host_barrier is not None:  # pushes complete before the host barrier
            import torch
            torch.cuda.current_stream().synchronize()
            return
        if self._flag_ptrs is None:
            return
        P = self.sh.plan
        _check(lib().emie_cu_peer_signal(self._flag_ptrs, P.G, self.sh.rank, self.epoch, self._stream()))

    def wait(self):
        """Before reading this rank's buffer: all G ranks reached the epoch."""
        from . import lib, _check
        if self.host_barrier is not None:
            self.host_barrier()
            return
        if self._flag_ptrs is None:
            return
        _check(lib().emie_cu_peer_wait(ctypes.c_void_p(self.own[2]), self.sh.plan.G, self.epoch, self._stream()))

    # stages (loopback runs each over all virtual ranks before the next)
    def push_forward(self, U):
        sh, P, be = self.sh, self.sh.plan, self.sh.be
        self._U = U
        S_loc = self.own[0]
        if getattr(be, "fused_peer_forward", False) and self.fused:
            # one pass: the slab's y transform stores each mode's column into its owner's S_full
            be.lateral_forward_peer(U, [self.peers[g][1] for g in range(P.G)], sh.nrhs)
            return
        be.lateral_forward_into(U, S_loc, sh.nrhs)
        for g in range(P.G):  # my slab's columns of g's modes -> g's full-depth spectrum
            be.move(S_loc, self.peers[g][1], sh.nrhs, g, P.E, sh._slab_desc(True),
                    (1, 3 * P.nz, P.nz, P.z[sh.rank]), sh.nzl)

    def push_contracted(self):
        sh, P, be = self.sh, self.sh.plan, self.sh.be
        S_full = self.own[1]
        if getattr(be, "fused_peer_contract", False) and self.fused:
            # one kernel: the contraction's epilogue stores into the owners' S_loc
            be.contract_peer(S_full, sh.nrhs, sh.q0, sh.q1, [self.peers[h][0] for h in range(P.G)], P.z)
            return
        be.contract(S_full, sh.nrhs, sh.q0, sh.q1)
        for h in range(P.G):  # my modes' columns of h's planes -> h's slab spectrum
            nzh = P.nzl(h)
            be.move(S_full, self.peers[h][0], sh.nrhs, sh.rank, P.E, (1, 3 * P.nz, P.nz, P.z[h]),
                    (1, 3 * nzh, nzh, 0), nzh)

    def finish(self):
        out = self.sh.be.lateral_inverse(self.own[0], self._U, self.sh.nrhs)
        self._U = None
        return out

    def check(self):
        """Raise if a flag wait of this process gave up on a peer (the sticky
        timeout of emie_cu_peer_wait; synchronises the device)."""
        from . import lib, _check
        t = ctypes.c_int(0)
        _check(lib().emie_cu_peer_status(ctypes.byref(t)))
        if t.value:
            raise RuntimeError("peer exchange: a rank never signalled (flag wait timed out); results are invalid")

    def apply(self, U):
        """One rank per process (all ranks call it with their slabs)."""
        self.push_forward(U)
        self.signal()
        self.wait()
        self.push_contracted()
        self.signal()
        self.wait()
        return self.finish()


def peer_loopback(shards: Sequence["ShardedApply"], host: bool = False, fused: bool = True):
    """G virtual ranks in one process (one GPU, or host tensors with the
    NumPy backend): every rank's exchange buffers allocated here, the 'peer'
    buffers are the other shards' own."""
    owns = [PeerExchange.allocate_host(sh) if host else PeerExchange.allocate(sh) for sh in shards]
    return [PeerExchange(sh, owns, owns[g], fused) for g, sh in enumerate(shards)], owns


def peer_loopback_apply(xs: Sequence[PeerExchange], slabs):
    """Stage by stage over the virtual ranks on one stream: every rank's
    pushes and signals precede every wait (a wait ahead of another virtual
    rank's signal would block the stream that signal is queued on)."""
    for x, u in zip(xs, slabs):
        x.push_forward(u)
        x.signal()
    for x in xs:
        x.wait()
    for x in xs:
        x.push_contracted()
        x.signal()
    for x in xs:
        x.wait()
    return [x.finish() for x in xs]


def peer_exchange_torch(shard: "ShardedApply", group=None) -> PeerExchange:
    """One rank per process: allocate, swap IPC handles over torch.distributed
    (all_gather_object), map the peers' buffers."""
    import torch.distributed as dist
    G, me = shard.plan.G, shard.rank
    own = PeerExchange.allocate(shard)
    hs = [None] * G
    dist.all_gather_object(hs, PeerExchange.ipc_handles(own), group=group)
    peers = [own if g == me else PeerExchange.open_ipc(hs[g]) for g in range(G)]
    dist.barrier(group=group)
    return PeerExchange(shard, peers, own)


# -------------------------------------------------------------- backends ----
class CudaBackend:
    """Stages on the device through the C ABI; tensors are torch complex128
    CUDA tensors (no host fallback: the library raises if it is missing)."""

    def __init__(self, plan: ShardPlan, rank: int, op_shard, sigma_slab, sigma_b_slab, volume_slab):
        import torch
        from . import lib, _check
        self.torch, self.L, self._check = torch, lib(), _check
        self.plan, self.rank = plan, rank
        L = self.L
        nzl = plan.nzl(rank)
        g = ctypes.c_void_p()
        _check(L.emie_cu_geometry_create(plan.nx, plan.ny, nzl, ctypes.byref(g)))
        self.geom = g
        self.op = op_shard  # SpectralOperator holding quadrant modes [q0, q1)
        if plan.octant:  # contract the shard's octant rows (the plan delivers the transposed modes)
            _check(L.emie_cu_operator_shard_octant(op_shard.handle, 1, None))
        # local system diagonals (cie.cpp:24-54) of the slab's cells
        sysh = ctypes.c_void_p()
        sa = np.ascontiguousarray(sigma_slab, dtype=np.complex128)
        sb = np.ascontiguousarray(sigma_b_slab, dtype=np.complex128)
        vol = np.ascontiguousarray(volume_slab, dtype=np.float64)
        _check(L.emie_cu_system_create(g, sa.ctypes.data, sb.ctypes.data, vol.ctypes.data, ctypes.byref(sysh)))
        n = plan.slab_cells(rank)
        s = np.zeros(n, np.complex128)
        r1 = np.zeros(n)
        r2 = np.zeros(n, np.complex128)
        _check(L.emie_cu_system_download(sysh, s.ctypes.data, r1.ctypes.data, r2.ctypes.data))
        L.emie_cu_system_destroy(sysh)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.s = torch.from_numpy(s).to(dev)
        self.r1 = torch.from_numpy(r1).to(dev)
        self.r2 = torch.from_numpy(r2).to(dev)
        self.idx = [torch.from_numpy(m).to(dev) for m in plan.modes]
        self.dev = dev

    def _st(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream().cuda_stream)

    def empty(self, shape):
        return self.torch.empty(shape, dtype=self.torch.complex128, device=self.dev)

    def zeros(self, shape):
        return self.torch.zeros(shape, dtype=self.torch.complex128, device=self.dev)

    def lateral_forward(self, U, nrhs):
        P = self.plan
        S = self.empty((nrhs, P.E, 3 * P.nzl(self.rank)))
        self._check(self.L.emie_cu_lateral_forward(self.geom, ctypes.c_void_p(U.data_ptr()),
                                                   ctypes.c_void_p(self.r2.data_ptr()),
                                                   ctypes.c_void_p(S.data_ptr()), nrhs, self._st()))
        return S

    def lateral_forward_into(self, U, S, nrhs):
        self._check(self.L.emie_cu_lateral_forward(self.geom, ctypes.c_void_p(U.data_ptr()),
                                                   ctypes.c_void_p(self.r2.data_ptr()),
                                                   ctypes.c_void_p(S.data_ptr()), nrhs, self._st()))

    def contract(self, S, nrhs, q0, q1):
        self._check(self.L.emie_cu_contract_modes(self.op.handle, ctypes.c_void_p(S.data_ptr()), nrhs, q0, q1,
                                                  self._st()))

    @property
    def fused_peer_forward(self) -> bool:
        if not hasattr(self, "_fpf"):
            v = ctypes.c_int(0)
            self._check(self.L.emie_cu_lateral_forward_peer_supported(self.geom, ctypes.byref(v)))
            self._fpf = bool(v.value)
            if self._fpf:  # the owners as the plan's splits (rows of the octant, or quadrant-mode ranges)
                P = self.plan
                self.splits = (ctypes.c_int * (P.G + 1))(*(P.rows if P.octant else P.q))
        return self._fpf

    def lateral_forward_peer(self, U, dsts, nrhs):
        P = self.plan
        G = len(dsts)
        dp = (ctypes.c_void_p * G)(*[d.data_ptr() for d in dsts])
        self._check(self.L.emie_cu_lateral_forward_peer_split(self.geom, ctypes.c_void_p(U.data_ptr()),
                                                              ctypes.c_void_p(self.r2.data_ptr()), self.splits,
                                                              1 if P.octant else 0, dp, G, P.nz, P.z[self.rank],
                                                              nrhs, self._st()))

    @property
    def fused_peer_contract(self) -> bool:
        return self.plan.nz in (8, 16, 32, 48, 64)  # the DMMA contractions have the peer epilogue

    def contract_peer(self, S, nrhs, q0, q1, dsts, z):
        G = len(dsts)
        dp = (ctypes.c_void_p * G)(*[d.data_ptr() for d in dsts])
        zz = (ctypes.c_int * (G + 1))(*z)
        self._check(self.L.emie_cu_contract_modes_peer(self.op.handle, ctypes.c_void_p(S.data_ptr()), nrhs, q0, q1,
                                                       dp, zz, G, self._st()))

    def lateral_inverse(self, S, U, nrhs):
        out = self.torch.empty_like(U)
        self._check(self.L.emie_cu_lateral_inverse(self.geom, ctypes.c_void_p(S.data_ptr()),
                                                   ctypes.c_void_p(U.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                                   ctypes.c_void_p(self.s.data_ptr()),
                                                   ctypes.c_void_p(self.r1.data_ptr()), nrhs, self._st()))
        return out

    def move(self, src, dst, nrhs, g, E, sdesc, ddesc, nzh):
        sd = (ctypes.c_int * 4)(*sdesc)
        dd = (ctypes.c_int * 4)(*ddesc)
        idx = self.idx[g]
        self._check(self.L.emie_cu_move_planes(ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()),
                                               nrhs, int(idx.numel()), ctypes.c_void_p(idx.data_ptr()),
                                               ctypes.c_longlong(E), sd, dd, nzh, self._st()))

    def __del__(self):
        try:
            self.L.emie_cu_operator_destroy(self.geom)
        except Exception:  # noqa: BLE001 -- interpreter teardown
            pass


def greens_offset_ranges(n_offsets: int, G: int) -> List[tuple]:
    """Contiguous ranges of the build's computed offsets per rank (every
    offset costs the same: all nz(nz+1)/2 pairs over the same 451 lambdas)."""
    s = _splits(n_offsets, G)
    return [(s[g], s[g + 1]) for g in range(G)]


def sharded_block_arrays(nx, ny, nz, offsets, G: int, ranks: Sequence[int], compute, zeros, reduce_blocks):
    """The offset-sharded half of the Green's build: the
    build's computed offsets are split into G contiguous ranges; each listed
    rank computes its range into a zeroed (ny, nx, 2nz(2nz+1)) block array
    (compute(c0, c1, buf)), and reduce_blocks sums the arrays over all ranks --
    every offset is written by exactly one rank, so the sum is exact -- and
    returns each listed rank's copy. compute / zeros / reduce_blocks are the
    device build, torch CUDA tensors and NCCL in production; the CPU tests
    plug in the numpy oracle, host tensors and gloo."""
    rng = greens_offset_ranges(len(offsets), G)
    nent = 2 * nz * (2 * nz + 1)
    bufs = []
    for g in ranks:
        b = zeros((ny, nx, nent))
        compute(rng[g][0], rng[g][1], b)
        bufs.append(b)
    return reduce_blocks(bufs)


def sharded_greens_build(grid, model, omega: float, plan: ShardPlan, ranks: Sequence[int], reduce_blocks,
                         params=None):
    """The Green's build sharded by offset: each listed
    rank computes its range of the computed offsets into a zeroed block array,
    reduce_blocks sums the arrays over all ranks (every offset is written by
    one rank, so the sum is exact) and returns each listed rank's copy; each
    rank then builds the spectra of its own quadrant-mode shard.
    Returns the per-rank mode-shard operators (SpectralOperator)."""
    import torch
    from . import greens_offsets, greens_blocks, operator_from_greens_blocks
    offs = greens_offsets(grid.nx, grid.ny, grid.hx, grid.hy)
    full = sharded_block_arrays(
        grid.nx, grid.ny, grid.nz, offs, plan.G, ranks,
        lambda c0, c1, b: greens_blocks(grid, model, omega, c0, c1, b, params),
        lambda shape: torch.zeros(shape, dtype=torch.complex128, device="cuda"), reduce_blocks)
    return [operator_from_greens_blocks(grid, omega, full[i], plan.q[g], plan.q[g + 1])
            for i, g in enumerate(ranks)]


def loopback_block_sum(bufs):
    """Virtual ranks in one process: the all-reduce of the block arrays (rank
    order); every rank gets its own copy (the mirror completes it in place)."""
    tot = bufs[0].clone()
    for b in bufs[1:]:
        tot += b
    return [tot.clone() for _ in bufs]


def torch_block_sum(group=None):
    """One rank per process: all-reduce (sum) of the rank's block array."""
    import torch.distributed as dist

    def red(bufs):
        (b,) = bufs
        dist.all_reduce(b, op=dist.ReduceOp.SUM, group=group)
        return [b]
    return red


def cuda_shard(grid, sop_full, plan: ShardPlan, rank: int, nrhs: int, op_shard=None) -> ShardedApply:
    """Rank `rank`'s sharded apply on the current CUDA device: the mode shard
    of sop_full's spectra (or the given op_shard), the lateral geometry and system diagonals of the
    depth slab (build_system, cie.cpp:24-54, restricted to its cells)."""
    from . import restrict_modes
    z0, z1 = plan.z[rank], plan.z[rank + 1]
    if op_shard is None:  # cut from a full operator (or built sharded: sharded_greens_build)
        op_shard = restrict_modes(sop_full, plan.q[rank], plan.q[rank + 1])
    sa = np.asarray(grid.sigma_a)[z0:z1]
    sb = np.asarray(grid.sigma_b)[z0:z1]
    vol = np.array([grid.volume(iz) for iz in range(z0, z1)], dtype=np.float64)
    be = CudaBackend(plan, rank, op_shard, sa, sb, vol)
    return ShardedApply(plan, rank, be, nrhs)
