"""Parity criteria of the north star (BASELINE.json), applied to GPU output vs oracle output:

  1. primary nearest-hit IDs bit-exact except on pixels the oracle flags as fragile
     (F1-F5 of the primary ray: a competing hit within 1e-4 relative, a primitive
     boundary within the band, grazing, t_min range end) -- DESIGN.md reading 22; on those
     the GPU's ID must be one of the oracle's near-tie candidates (the IDs the band-turned
     ray may hit first, -1 = miss);
  2. RGB (8-bit) within 2/255 on at least 99.9% of pixels (all pixels counted);
  3. max abs error <= 1e-3 of the clamped linear radiance on pixels with no fragile
     decision anywhere in their ray tree.
"""
import numpy as np

from oracle.oracle import CAND_K, ID_FRAGILE_MASK

RGB_TOL = 2
RGB_FRAC = 0.999
RAD_TOL = 1e-3


def compare(ref, ids, rgba8, radiance, label=""):
    """ref: oracle dict (flattened or image-shaped); ids/rgba8/radiance: GPU arrays, same shape."""
    rid = ref["id"].reshape(-1)
    pf = ref["pflags"].reshape(-1)
    tf = ref["tflags"].reshape(-1)
    ids = np.asarray(ids).reshape(-1)
    ok_id = (pf & ID_FRAGILE_MASK) == 0
    id_mism = int((ids[ok_id] != rid[ok_id]).sum())
    # ID-fragile pixels: the GPU ID must be one of the near-tie candidates
    frag = np.flatnonzero(~ok_id)
    nc = ref["ncand"].reshape(-1)[frag] if "ncand" in ref else np.zeros(len(frag), int)
    cand = ref["cand"].reshape(-1, CAND_K)[frag] if "cand" in ref else np.zeros((len(frag), CAND_K), int)
    checkable = (nc >= 1) & (nc <= CAND_K)
    inset = np.array([ids[i] in cand[k, :nc[k]] for k, i in enumerate(frag)], bool) if len(frag) else np.zeros(0, bool)
    cand_viol = int((checkable & ~inset).sum())
    d8 = np.abs(np.asarray(rgba8).reshape(-1, 4)[:, :3].astype(int) - ref["rgba8"].reshape(-1, 4)[:, :3].astype(int)).max(1)
    frac = float((d8 <= RGB_TOL).mean())
    ok = tf == 0
    g = np.clip(np.asarray(radiance).reshape(-1, 4)[:, :3].astype(np.float64), 0, 1)
    o = np.clip(ref["radiance"].reshape(-1, 3), 0, 1)
    err = np.abs(g - o).max(1)
    max_err = float(err[ok].max()) if ok.any() else 0.0
    stats = dict(label=label, n=len(rid), id_excluded=float(1 - ok_id.mean()), id_mismatch=id_mism,
                 rgb_frac=frac, rad_excluded=float(1 - ok.mean()), max_err=max_err,
                 all_id_mismatch=int((ids != rid).sum()),
                 # the oracle's primary boundary margin of every GPU/oracle ID disagreement: the
                 # triangle-edge band eps_edge must stay >= 4x the largest
                 mismatch_margins=sorted(float(x) for x in ref["margin"].reshape(-1)[ids != rid]),
                 id_fragile=int(len(frag)),
                 id_fragile_checked=int(checkable.sum()), id_candidate_violations=cand_viol,
                 id_fragile_unchecked=int((~checkable).sum()))
    return stats


def assert_parity(stats):
    msg = str(stats)
    assert stats["id_mismatch"] == 0, msg
    assert stats["id_candidate_violations"] == 0, msg
    assert stats["rgb_frac"] >= RGB_FRAC, msg
    assert stats["max_err"] <= RAD_TOL, msg
