"""Cases of the reference-generated golden fixtures (tests/golden/make_golden.py)."""
CASES = {
    # name: (n_envs, steps, EnvConfig overrides, reward mode)
    "pendulum1_m2": (3, 40, dict(episode_horizon=25, rsi=True), 0),
    "arm2_m6": (4, 60, dict(episode_horizon=30, rsi=True), 2),
    "walker5_m16": (4, 40, dict(episode_horizon=1000, rsi=True, termination_body_err=0.3), 0),
    "wb700_fixed": (2, 3, dict(episode_horizon=1000, rsi=True), 0),
    "wb700": (2, 3, dict(episode_horizon=1000, rsi=True), 2),
    "wb700_backflip": (2, 3, dict(episode_horizon=1000, rsi=True), 0),
}
