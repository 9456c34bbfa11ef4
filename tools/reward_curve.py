"""Fig. 4-style learning curve, in spirit: the whole of Alg. 1 on one B200 through the C ABI.

On-GPU acting (dqn_collect: n parallel Snake games, eps-greedy on Q(phi; theta), Store into the replay;
P:113-117) alternates with replica steps (dqn_train_steps: sample, TD target with theta^, RMSProp;
P:119-125). The game and its rules are the paper's Snake as closed in DESIGN.md A34-A36. This script does not
reproduce the paper's numbers (its Fig. 4 used Atari and a CPU cluster); it shows that the built path learns.

Prints one JSON line per window: env steps, gradient steps, episodes, mean reward per episode, mean
episode length, epsilon, wall seconds.

usage: python tools/reward_curve.py [--seconds 180] [--envs 64] [--out gpurun_out/reward_curve.jsonl]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=180.0)
    ap.add_argument("--envs", type=int, default=64)
    ap.add_argument("--grid", type=int, default=12)
    ap.add_argument("--collect", type=int, default=8, help="acting steps per iteration (per game)")
    ap.add_argument("--train", type=int, default=16, help="replica steps per iteration")
    ap.add_argument("--replay", type=int, default=200_000)
    ap.add_argument("--eps-decay-s", type=float, default=60.0, help="seconds for eps 1 -> eps-min")
    ap.add_argument("--eps-min", type=float, default=0.05)
    ap.add_argument("--window", type=int, default=200, help="iterations per logged window")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import torch
    import paper_1508_04186_b200 as D

    torch.cuda.set_device(0)
    cfg = D.Config(convs=((16, 8, 4), (32, 4, 2)), fcs=(256,), n_actions=4, minibatch=args.envs,
                   replay_capacity=args.replay, target_sync=1000, precision=D.BF16, lr=2.5e-4, gamma=0.99)
    g = D.DQN(cfg)
    seed = 0x5AC3
    # warm the replay with uniformly random play before the first gradient step
    while g.replay_size()[1] < 10 * args.envs:
        g.collect(args.envs, args.grid, args.collect, 1.0, seed)
    out = open(args.out, "w") if args.out else None
    t0 = time.time()
    it = env_steps = grad_steps = 0
    win = dict(ep=0, rew=0.0, steps=0)
    while time.time() - t0 < args.seconds:
        el = time.time() - t0
        eps = max(args.eps_min, 1.0 - (1.0 - args.eps_min) * el / args.eps_decay_s)
        c = g.collect(args.envs, args.grid, args.collect, eps, seed)
        st = g.train(args.train, want_loss=True)
        env_steps += c["env_steps"]
        grad_steps += args.train
        win["ep"] += c["episodes"]
        win["rew"] += c["reward_sum"]
        win["steps"] += c["env_steps"]
        it += 1
        if it % args.window == 0:
            line = {"env_steps": env_steps, "grad_steps": grad_steps, "episodes": win["ep"],
                    "reward_per_episode": win["rew"] / win["ep"] if win["ep"] else None,
                    "episode_length": win["steps"] / win["ep"] if win["ep"] else None,
                    "epsilon": round(eps, 3), "loss": float(st["loss_mean"]), "wall_s": round(time.time() - t0, 1)}
            print(json.dumps(line), flush=True)
            if out:
                out.write(json.dumps(line) + "\n")
            win = dict(ep=0, rew=0.0, steps=0)
    g.close()


if __name__ == "__main__":
    main()
