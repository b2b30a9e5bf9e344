"""Element partitioning and face-halo plans for multi-GPU runs (host logic, no method arithmetic).

A global mesh (meshgen dict) and a part array (element -> rank) become one RankMesh per rank:
  * local elements in ascending global id (Morton order of the global mesh is preserved);
  * EToV with GLOBAL vertex ids (the library reads VX, VY with the same numbering);
  * bc codes, with faces whose neighbour lives on another rank set to IPDG_BC_REMOTE (3);
  * the halo plan: for every neighbour rank q, the local elements sent to q and the ghost
    elements received from q, both sorted by global id, so rank r's send list to q equals
    rank q's receive list from r element by element;
  * per REMOTE face: the ghost index h (position in the concatenated receive lists) and the
    neighbour's local face index f'.
This realises SURVEY section 8.5 (element partition, face-trace halo) and is exercised by
tests/test_partition.py (including a world_size-2 gloo exchange).
"""
from dataclasses import dataclass, field

import numpy as np

REMOTE = 3


@dataclass
class RankMesh:
    rank: int
    nparts: int
    elems: np.ndarray          # (K,) global element ids owned by this rank, ascending
    EToV: np.ndarray           # (K,3) global vertex ids
    bc: np.ndarray             # (K,3) codes, REMOTE on cut faces
    remote: np.ndarray         # (K,3) ghost index h on REMOTE faces, else -1
    remote_face: np.ndarray    # (K,3) neighbour face f' on REMOTE faces, else -1
    ghosts: np.ndarray         # (H,) global ids of the ghost elements (concatenated receive lists)
    ghost_EToV: np.ndarray     # (H,3) their global vertex ids
    nbr_ranks: np.ndarray      # (nnbr,) neighbour ranks, ascending
    send_off: np.ndarray       # (nnbr+1,) offsets into send_elems
    send_elems: np.ndarray     # local ids of the elements sent to each neighbour
    recv_off: np.ndarray       # (nnbr+1,) offsets into ghosts
    VX: np.ndarray = field(repr=False, default=None)
    VY: np.ndarray = field(repr=False, default=None)

    @property
    def K(self):
        return self.elems.size

    @property
    def H(self):
        return self.ghosts.size

    def local_mesh(self):
        return dict(VX=self.VX, VY=self.VY, EToV=self.EToV, bc=self.bc)


def global_connectivity(EToV):
    """EToE, EToF (K,3) from shared vertex pairs (-1 on boundary faces)."""
    K = EToV.shape[0]
    a = EToV[:, [0, 1, 2]].astype(np.int64)
    b = EToV[:, [1, 2, 0]].astype(np.int64)
    nv = int(EToV.max()) + 1
    key = (np.minimum(a, b) * nv + np.maximum(a, b)).ravel()
    order = np.argsort(key, kind="stable")
    ks = key[order]
    EToE = -np.ones(3 * K, dtype=np.int64)
    EToF = -np.ones(3 * K, dtype=np.int64)
    same = np.nonzero(ks[1:] == ks[:-1])[0]
    i1, i2 = order[same], order[same + 1]
    EToE[i1], EToF[i1] = i2 // 3, i2 % 3
    EToE[i2], EToF[i2] = i1 // 3, i1 % 3
    return EToE.reshape(K, 3), EToF.reshape(K, 3)


def local_connectivity(EToV, part, r):
    """EToE, EToF for the rows of rank r's elements only (global element ids), without sorting the whole
    mesh: the candidates are the elements that share a vertex with rank r (every face neighbour shares
    two), and only own + candidates are keyed and sorted.  Returns (elems, EToE_r, EToF_r)."""
    elems = np.nonzero(part == r)[0]
    verts = np.unique(EToV[elems])
    touch = np.isin(EToV, verts).any(axis=1)
    touch[elems] = False
    sub = np.concatenate([elems, np.nonzero(touch)[0]])
    E, F = global_connectivity(EToV[sub])
    Eo, Fo = E[:elems.size], F[:elems.size]
    Eg = np.where(Eo >= 0, sub[np.maximum(Eo, 0)], -1)
    return elems, Eg, Fo


def split(mesh, part, nparts, ranks=None):
    """List of RankMesh, one per rank (or only for `ranks`: then each rank's face connectivity is built
    from its own elements and their vertex neighbours, not from a sort of the whole mesh)."""
    EToV = np.asarray(mesh["EToV"])
    bc = np.asarray(mesh["bc"])
    part = np.asarray(part)
    local = ranks is not None
    if not local:
        EToE, EToF = global_connectivity(EToV)
    out = []
    for r in (range(nparts) if ranks is None else ranks):
        if local:
            elems_l, E_l, F_l = local_connectivity(EToV, part, r)
            EToE = np.full((EToV.shape[0], 3), -1, dtype=np.int64)
            EToF = np.full((EToV.shape[0], 3), -1, dtype=np.int64)
            EToE[elems_l], EToF[elems_l] = E_l, F_l
        elems = np.nonzero(part == r)[0]
        g2l = -np.ones(EToV.shape[0], dtype=np.int64)
        g2l[elems] = np.arange(elems.size)
        nb = EToE[elems]
        cut = (nb >= 0) & (part[np.maximum(nb, 0)] != r)
        lbc = bc[elems].copy()
        lbc[cut] = REMOTE
        nbr_ranks = np.unique(part[nb[cut]]) if np.any(cut) else np.zeros(0, dtype=np.int64)
        ghosts, recv_off, send_elems, send_off = [], [0], [], [0]
        for q in nbr_ranks:
            on_q = cut & (part[np.maximum(nb, 0)] == q)
            g = np.unique(nb[on_q])                     # q's elements adjacent to ours
            s = np.unique(np.repeat(elems[:, None], 3, 1)[on_q])  # our elements adjacent to q
            ghosts.append(g)
            recv_off.append(recv_off[-1] + g.size)
            send_elems.append(g2l[s])
            send_off.append(send_off[-1] + s.size)
        ghosts = np.concatenate(ghosts) if ghosts else np.zeros(0, dtype=np.int64)
        gpos = {int(gid): h for h, gid in enumerate(ghosts)}
        remote = -np.ones((elems.size, 3), dtype=np.int32)
        remote_face = -np.ones((elems.size, 3), dtype=np.int32)
        ee, ff = np.nonzero(cut)
        for e, f in zip(ee, ff):
            remote[e, f] = gpos[int(nb[e, f])]
            remote_face[e, f] = EToF[elems[e], f]
        out.append(RankMesh(rank=r, nparts=nparts, elems=elems, EToV=np.ascontiguousarray(EToV[elems], dtype=np.int32),
                            bc=lbc.astype(np.int8), remote=remote, remote_face=remote_face,
                            ghosts=ghosts.astype(np.int64), ghost_EToV=np.ascontiguousarray(EToV[ghosts], dtype=np.int32),
                            nbr_ranks=nbr_ranks.astype(np.int32), send_off=np.array(send_off, dtype=np.int64),
                            send_elems=(np.concatenate(send_elems) if send_elems else np.zeros(0)).astype(np.int32),
                            recv_off=np.array(recv_off, dtype=np.int64), VX=mesh["VX"], VY=mesh["VY"]))
    return out


def check_plan(ranks):
    """Consistency of a full set of RankMesh plans (send list of r to q == receive list of q from r)."""
    by = {rm.rank: rm for rm in ranks}
    for rm in ranks:
        for j, q in enumerate(rm.nbr_ranks):
            sent = rm.elems[rm.send_elems[rm.send_off[j]:rm.send_off[j + 1]]]
            other = by[int(q)]
            jj = int(np.nonzero(other.nbr_ranks == rm.rank)[0][0])
            recv = other.ghosts[other.recv_off[jj]:other.recv_off[jj + 1]]
            if not np.array_equal(sent, recv):
                raise AssertionError("halo plan mismatch between ranks %d and %d" % (rm.rank, q))
    return True
