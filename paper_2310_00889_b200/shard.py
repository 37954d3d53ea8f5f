"""Target/panel partition for the multi-GPU operator apply.

Each rank owns a contiguous range of source panels; its targets are those panels' coarse
nodes (plus, on rank 0, any off-surface targets), so node targets, their near blocks and the
identity/projector terms are rank-local.  The only exchange is the all-gather of the upsampled
density inside slb_matvec.  Ranges are balanced by panel count; with whole_bodies=True (the
mobility projector needs a body's nodes on one rank) range ends snap to body boundaries.
"""
import numpy as np


def partition_panels(n_panels, nranks, body_of_panel=None, whole_bodies=False):
    if nranks < 1:
        raise ValueError("nranks >= 1")
    cuts = [round(r * n_panels / nranks) for r in range(nranks + 1)]
    if whole_bodies:
        if body_of_panel is None:
            raise ValueError("whole_bodies needs body_of_panel")
        bop = np.asarray(body_of_panel)
        starts = np.concatenate([[0], np.nonzero(np.diff(bop))[0] + 1, [n_panels]])
        snapped = [0]
        for c in cuts[1:-1]:
            j = int(np.argmin(np.abs(starts - c)))
            snapped.append(int(max(starts[j], snapped[-1])))
        snapped.append(n_panels)
        cuts = snapped
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(nranks)]
