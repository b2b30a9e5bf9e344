"""Halo message sizes of the multi-GPU partitions: ghost-ROW exchange (what libipdg
ships: N_p doubles per ghost element) against a face-TRACE exchange (u and sJ n.grad u at the N_fp nodes of
every cut face: 2 N_fp doubles per face), per rank and per PCG iteration, from the real partition plans.

  C4: RCB partitions of the cylinder mesh (N = 6), P = 2, 4, 8 (strong scaling)
  C5: px x py tiles of n x n cells (N = 8), one tile per rank; counted on n = 200 and scaled to n = 1414
      (every quantity is proportional to the tile side)
usage: python tools/halo_sizes.py [--quick]   (prints JSON lines)"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1801_00246_b200 import meshgen, partition  # noqa: E402

NVLINK_GBS = 900.0  # per direction per GPU (NVLink 5)


def sizes(m, part, P, N, scale=1.0):
    Np, Nfp = (N + 1) * (N + 2) // 2, N + 1
    ranks = partition.split(m, part, P)
    worst = None
    for rm in ranks:
        cut_faces = int((rm.bc == partition.REMOTE).sum())
        H = int(rm.H)
        rows_b = H * Np * 8 * scale
        face_b = cut_faces * 2 * Nfp * 8 * scale
        rec = dict(rank=rm.rank, K=int(rm.elems.size * scale * scale), ghosts=int(H * scale), cut_faces=int(cut_faces * scale),
                   neighbours=int(rm.nbr_ranks.size), row_bytes=int(rows_b), face_bytes=int(face_b))
        if worst is None or rows_b > worst["row_bytes"]:
            worst = rec
    worst["row_us_at_nvlink"] = round(worst["row_bytes"] / (NVLINK_GBS * 1e3), 3)
    worst["face_us_at_nvlink"] = round(worst["face_bytes"] / (NVLINK_GBS * 1e3), 3)
    worst["row_over_face"] = round(worst["row_bytes"] / max(1, worst["face_bytes"]), 2)
    return worst


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    for P in (2, 4, 8):
        px = {2: 2, 4: 2, 8: 4}[P]
        n = 60 if a.quick else 200
        m, part = meshgen.tiles(n, px, P // px, jitter=0.2, seed=5)
        print(json.dumps(dict(config="C5", N=8, P=P, tile_cells=1414, counted_on=n, **sizes(m, part, P, 8, 1414.0 / n))), flush=True)
    if not a.quick:
        m = meshgen.cylinder()
        for P in (2, 4, 8):
            part = meshgen.rcb_partition(m["VX"], m["VY"], m["EToV"], P)
            print(json.dumps(dict(config="C4", N=6, P=P, **sizes(m, part, P, 6))), flush=True)


if __name__ == "__main__":
    main()
