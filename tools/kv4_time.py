"""Time qoq_kv4_decode_attention at the bench size (bench.kv4_measure: B = 64 x 1024 tokens, Llama-3-8B
heads, 4 rotated layer caches, CUDA graph) and print its JSON."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_04532_b200 as qoq  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    qoq.load()
    stream = torch.cuda.Stream(dev)

    def timed(graph, steps, warmup):
        for _ in range(warmup):
            graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            graph.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    print(json.dumps(bench.kv4_measure(qoq, torch, dev, stream, timed)))


if __name__ == "__main__":
    main()
