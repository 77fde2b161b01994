"""Pin the CPU oracle against golden vectors recorded from the reference.

The oracle (oracle/) is the checker for every GPU parity test, so it must
reproduce the reference bit for bit: identical operation order in the C
restatement, identical numpy host glue.
"""

import numpy as np
import pytest

from golden_util import load, names
from oracle import oracle as O


@pytest.mark.parametrize("name", names())
def test_forward_backward_bit_exact(name):
    batch, nums, den, leak, z = load(name)
    for side, g in (("num", nums), ("den", den)):
        fb = O.forward_backward(batch, g, leak=leak, keep_trellis=f"{side}_alpha" in z)
        np.testing.assert_array_equal(fb.log_probs, z[f"{side}_log_probs"])
        np.testing.assert_array_equal(fb.posteriors, z[f"{side}_posteriors"])
        np.testing.assert_array_equal(fb.scale_logs, z[f"{side}_scale_logs"])
        np.testing.assert_array_equal(fb.failure_frames, z[f"{side}_failure_frames"])
        if f"{side}_alpha" in z:
            np.testing.assert_array_equal(fb.alpha, z[f"{side}_alpha"])
            np.testing.assert_array_equal(fb.beta, z[f"{side}_beta"])


@pytest.mark.parametrize("name", names())
def test_chain_loss_bit_exact(name):
    batch, nums, den, leak, z = load(name)
    if int(z["all_failed"]):
        with pytest.raises(RuntimeError, match="failed"):
            O.chain_loss(batch, nums, den, leak=leak)
        return
    res = O.chain_loss(batch, nums, den, leak=leak)
    assert res.objective == float(z["objective"])
    assert res.loss == float(z["loss"])
    np.testing.assert_array_equal(res.grad, z["grad"])
    np.testing.assert_array_equal(np.array(res.per_utt), z["per_utt"])
    assert res.num_failed == int(z["num_failed"])


def test_known_answers_in_fixtures():
    # TWO_STATE ln 0.64 and posteriors (0.625, 0.375), (1, 0).
    _, _, _, _, z = load("ka_two_state")
    np.testing.assert_allclose(z["num_log_probs"][0], np.log(0.64), atol=1e-12)
    np.testing.assert_allclose(z["num_posteriors"][0], [[0.625, 0.375], [1.0, 0.0]], atol=1e-12)
    _, _, _, _, z = load("ka_self_loop")
    np.testing.assert_allclose(z["num_log_probs"], [3 * np.log(0.5), 0.0], atol=1e-14)
    _, _, _, _, z = load("ka_failure")
    assert list(z["num_failure_frames"]) == [-1, 0] and int(z["num_failed"]) == 1
