"""Golden-fixture case table (shared by make_golden.py and the tests).

Inputs are dense U(-1, 1) drawn from ``default_rng(seed + 1000)`` per
iteration (x first, then targets); weights are ``Weights.init(net, seed)``.
"""

CASES = {
    "lstm_small": dict(builder="build_lstm", args=(3, 4, 3), S=2, h=6, hp=3, iters=4, lr=0.05, seed=1),
    "lstm_small_seq": dict(builder="build_lstm", args=(3, 4, 3), S=2, h=6, hp=3, iters=3, lr=0.05, seed=1,
                           frame_parallel=False),
    "lstm_nopeep_d1": dict(builder="build_lstm", args=(4, 5, 3),
                           kwargs=dict(output_peephole_delay=1), S=1, h=5, hp=5, iters=3, lr=0.1, seed=2),
    "elman": dict(builder="build_elman", args=(3, 5, 4), S=3, h=4, hp=2, iters=5, lr=0.1, seed=3),
    "elman_mse": dict(builder="build_elman", args=(2, 4, 2), kwargs=dict(output_activation=__import__(
        "paper_1503_02852_b200.netdef", fromlist=["Activation"]).Activation.IDENTITY),
        S=2, h=6, hp=3, iters=4, lr=0.05, seed=4, criterion="mse_identity"),
    "stacked_small": dict(builder="build_stacked_lstm", args=(4, (5, 3), 4), S=2, h=6, hp=3, iters=4, lr=0.05,
                          seed=5),
    "custom_small": dict(builder="build_custom_graph", args=(5, 6, 4), S=2, h=8, hp=4, iters=4, lr=0.05, seed=6),
    "cfg1": dict(builder="build_lstm", args=(39, 128, 39), S=1, h=32, hp=16, iters=3, lr=1e-3, seed=0, compact=True),
}
