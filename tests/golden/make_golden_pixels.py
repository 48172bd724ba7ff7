"""Golden vectors for the cartpole pixel observations, produced by the reference.

    python tests/golden/make_golden_pixels.py     (needs /root/reference; CPU)

BatchEnv("cartpole-balance-pixels", visual_randomization, episode_length 6) over
8 worlds for 14 steps (two autoresets per world), recording state and pixel
observations, terminal pixel stacks, the per-world visuals, and batch_render RGB
(with and without brightness_postprocess) for random states and visuals.
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from deskrl import dynamics, envkit, pixelrender

    def pack(v):
        return [*map(float, v.background), *map(float, v.cart_color), *map(float, v.pole_color),
                float(v.camera_offset[0]), float(v.camera_offset[1]), float(v.camera_zoom),
                float(v.brightness)]

    rng = np.random.default_rng(64)
    data = {}
    for name, rand in (("rand", True), ("plain", False)):
        N, T = 8, 14
        env = envkit.BatchEnv(envkit.EnvConfig(task="cartpole-balance-pixels", episode_length=6,
                                               visual_randomization=rand), N)
        obs = env.reset(seed=4)
        st, px, vis = [obs["state"]], [obs["pixels"]], [[pack(e._visuals) for e in env.envs]]
        acts = rng.uniform(-1, 1, (T, N, 1))
        term_px = np.zeros((T, N, 64, 64, 3))
        term_mask = np.zeros((T, N), dtype=np.uint8)
        for t in range(T):
            obs, r, d, tr, infos = env.step(acts[t])
            st.append(obs["state"])
            px.append(obs["pixels"])
            vis.append([pack(e._visuals) for e in env.envs])
            for i in range(N):
                if "terminal_observation" in infos[i]:
                    term_px[t, i] = infos[i]["terminal_observation"]["pixels"]
                    term_mask[t, i] = 1
        data[f"{name}/actions"] = acts
        data[f"{name}/state"] = np.array(st)
        data[f"{name}/pixels"] = np.array(px)
        data[f"{name}/visuals"] = np.array(vis)
        data[f"{name}/term_pixels"] = term_px
        data[f"{name}/term_mask"] = term_mask
    # batch_render on random states / visuals
    n = 64
    q = np.stack([rng.uniform(-2.2, 2.2, n), rng.uniform(-np.pi, np.pi, n)], 1)
    bounds = pixelrender.VisualBounds()
    vps = [pixelrender.randomize_visuals(np.random.default_rng(k), bounds) for k in range(n)]
    states = dynamics.SystemState(q=q, v=np.zeros_like(q))
    img = pixelrender.batch_render(states, vps, 48, 40)
    data["render/q"] = q
    data["render/visuals"] = np.array([pack(v) for v in vps])
    data["render/rgb"] = img
    data["render/bright"] = np.stack([pixelrender.brightness_postprocess(img[i], vps[i].brightness)
                                      for i in range(n)])
    path = os.path.join(OUT, "pixels_golden.npz")
    np.savez_compressed(path, **data)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(data)} arrays)")


if __name__ == "__main__":
    main()
