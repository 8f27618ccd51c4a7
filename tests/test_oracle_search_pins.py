"""Hand-worked pins for the oracle's per-step prune decision (O5; P:L535-541 test m1_d·P_d + β'_d > τ,
P:L582-586 one classifier per projected dimension, R9/R10 step indexing, R11 τ = ∞ before K
results, R13 τ frozen per epoch) and for the centring of the rotation.

Every expected value below is derived by hand in the comments, not by running the oracle: the
candidates have at most three non-zero coordinates (dims 0, 16, 32), the query is the origin and
the rotation is the identity, so every partial distance is a sum of one to three exact squares.
Each plausible slip in `search` changes a number asserted here:
  * P at the wrong index (P[:, d] instead of P[:, d-1]) prunes id 4 at d = 32 (P_33 = 1, 1 + 3 > 3);
  * the wrong calibration row (d = 16 using the d = 32 entry) prunes id 5 at d = 16 instead of 32;
  * τ refreshed inside an epoch (after id 4 enters) prunes id 6 at d = 32;
  * a test at d = D (R10) prunes survivors; `>=` instead of `>` prunes ids 4 and 6 (score = τ)."""
import numpy as np

from oracle import dade_oracle as O

D = 48
# (a, b, c) at dims (0, 16, 32); dist = a² + b² + c², P_16 = a², P_32 = a² + b²
CANDS = [
    (3.0, 0.0, 0.0),   # id 0: 9         epoch 0 (ids 0-3, c0 = 4K = 4): τ = ∞, all survive
    (2.0, 2.0, 0.0),   # id 1: 8
    (1.0, 1.0, 1.0),   # id 2: 3         → top-1 after epoch 0 = (3, id 2): τ_1 = 3
    (4.0, 0.0, 0.0),   # id 3: 16
    (0.0, 0.0, 1.0),   # id 4: 1         epoch 1 (ids 4-7), τ = 3: d16 2·0+1 = 1 ≤ 3, d32 0+3 = 3 ≤ 3 → survives
    (1.0, 0.0, 0.0),   # id 5: 1         d16 2·1+1 = 3 ≤ 3, d32 1+3 = 4 > 3 → pruned at d = 32
    (0.0, 0.0, 1.5),   # id 6: 2.25      d16 1 ≤ 3, d32 3 ≤ 3 → survives (τ is NOT refreshed to 1 by id 4)
    (2.0, 0.0, 0.0),   # id 7: 4         d16 2·4+1 = 9 > 3 → pruned at d = 16
    (0.0, 0.0, 0.5),   # id 8: 0.25      epoch 2 (ids 8-9), τ_2 = 1 (id 4): d16 1 ≤ 1, d32 3 > 1 → pruned at 32
    (0.5, 0.0, 0.0),   # id 9: 0.25      d16 2·0.25+1 = 1.5 > 1 → pruned at d = 16
]
# step table: m1 = (2, 1) at d = (16, 32); with n0 = 1 Label-0 value per step, β'_d = v_d[0] = (1, 3)
CAL = {"m1": np.array([2.0, 1.0]), "v": np.array([[1.0], [3.0]]), "ok": np.array([True, True]),
       "n0": 1, "K": 1, "block": 16}


def hand_case():
    X = np.zeros((len(CANDS), D), np.float32)
    for i, (a, b, c) in enumerate(CANDS):
        X[i, 0], X[i, 16], X[i, 32] = a, b, c
    idx = O.build_index(X, np.zeros((1, D), np.float32), mean=np.zeros(D), R=np.eye(D), cal=CAL)
    return X, idx


def test_hand_worked_prune_decisions():
    X, idx = hand_case()
    Q = np.zeros((1, D), np.float32)
    ids, d, st = O.search(idx, Q, 1, 1, 16, 0.1, log=True)
    assert ids.tolist() == [[4]] and d.tolist() == [[1.0]]            # id 8 (0.25) was pruned at d = 32
    assert st["tested"] == 10 and st["survivors"] == 6                 # ids 0-4, 6
    assert st["pruned_at_step"].tolist() == [0, 2, 2]                  # d16: ids 7, 9; d32: ids 5, 8
    assert st["dims_scanned"] == 6 * 48 + 32 + 16 + 32 + 16            # = 384
    assert st["n_epochs"] == 3                                         # [0,4), [4,8), [8,10)
    pruned = sorted((i, dd, tau) for (_q, i, dd, _s, tau) in st["decisions"])
    assert pruned == [(5, 32, 3.0), (7, 16, 3.0), (8, 32, 1.0), (9, 16, 1.0)]
    scores = {i: s for (_q, i, _d, s, _t) in st["decisions"]}
    assert scores == {5: 4.0, 7: 9.0, 8: 3.0, 9: 1.5}
    # per-candidate log: dims read and the closest call |score − τ| / (|m1 P| + |β'| + τ)
    q_, i_, dims, margin = (np.concatenate(c) for c in zip(*st["candidates"]))
    assert i_.tolist() == list(range(10)) and set(q_.tolist()) == {0}
    assert dims.tolist() == [48, 48, 48, 48, 48, 32, 48, 16, 32, 16]
    assert np.all(np.isinf(margin[:4]))                                # τ = ∞ in epoch 0: never tested
    # id 4: d16 |1−3|/(0+1+3) = 0.5, d32 |3−3|/(0+3+3) = 0 → 0;  id 9: d16 |1.5−1|/(0.5+1+1) = 0.2
    assert margin[4] == 0.0 and margin[6] == 0.0 and abs(margin[9] - 0.2) < 1e-15
    # id 5: d16 |3−3| = 0 → 0;  id 7: d16 |9−3|/(8+1+3) = 0.5;  id 8: d16 |1−1| = 0
    assert margin[5] == 0.0 and abs(margin[7] - 0.5) < 1e-15 and margin[8] == 0.0


def test_hand_worked_sequential_mode_refreshes_tau():
    # the paper's literal heap: τ drops to 1 as soon as id 4 enters, so id 6
    # (d32: 0 + 3 > 1) is pruned at d = 32 — the difference the epoch schedule (R13) makes
    X, idx = hand_case()
    ids, d, st = O.search(idx, np.zeros((1, D), np.float32), 1, 1, 16, 0.1, mode="sequential")
    assert ids.tolist() == [[4]]
    # id 0 enters (τ 9); id 1: d16 2·4+1 = 9 ≤ 9, d32 8+3 = 11 > 9 pruned; id 2: 3 ≤ 9, 5 ≤ 9 → enters (τ 3);
    # id 3: 2·16+1 > 3 pruned d16; id 4 → τ 1; id 5: 3 > 1 d16; id 6: d16 1 ≤ 1, d32 3 > 1; id 7 d16;
    # id 8: d16 1 ≤ 1, d32 3 > 1; id 9: d16 1.5 > 1  → d16: ids 3, 5, 7, 9; d32: ids 1, 6, 8
    assert st["pruned_at_step"].tolist() == [0, 4, 3]
    assert st["survivors"] == 3


def test_hand_worked_alpha0_keeps_everything():
    X, idx = hand_case()
    ids, d, st = O.search(idx, np.zeros((1, D), np.float32), 2, 1, 16, 0.0)
    assert ids.tolist() == [[8, 9]] and d.tolist() == [[0.25, 0.25]]   # tie at 0.25 → lower id first
    assert st["dims_scanned"] == 10 * 48 and st["pruned_at_step"].sum() == 0


def test_rotation_centres_on_the_sample_mean():
    # the data are centred before the rotation. Points (0,1), (4,1), (2,0), (2,2): mean (2,1),
    # centred (∓2,0), (0,∓1) → Σ = diag(2, 0.5) (divisor n): R = I, λ = (2, 0.5). The point (5, 3)
    # rotates to (3, 2), ‖x̃‖² = 13 (uncentred it would be 34).
    X = np.array([[0, 1], [4, 1], [2, 0], [2, 2]], np.float32)
    mean, R, lam = O.fit_rotation(X)
    assert mean.tolist() == [2.0, 1.0] and lam.tolist() == [2.0, 0.5]
    np.testing.assert_array_equal(R, np.eye(2))
    xr = O.rotate(np.array([[5.0, 3.0]]), mean, R)
    assert xr.tolist() == [[3.0, 2.0]] and float((xr ** 2).sum()) == 13.0
