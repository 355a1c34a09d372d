"""Golden HTTP exchanges of the reference service (service/app.py:74-118).

Run in the build container with the reference importable:
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_service_golden.py
Posts each request below to the reference's own FastAPI app (TestClient) and
records status code and response body bytes in service_exchanges.json;
tests/test_gpu_parity.py posts the same requests to
paper_2302_05176_b200.service and compares the bytes.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def requests():
    rng = np.random.default_rng(11)
    big = {int(i): float(w) for i, w in zip(rng.choice(10**7, 5000, replace=False) + 1, rng.exponential(1.0, 5000))}
    mid = {int(i): float(w) for i, w in zip(rng.choice(10**6, 300, replace=False) + 1, rng.random(300) + 0.01)}
    mid2 = dict(list(mid.items())[:150])
    mid2.update({int(i) + 2_000_000: float(w) for i, w in zip(rng.choice(10**6, 150, replace=False), rng.random(150) + 0.01)})
    small = {"1": 0.5, "2": 1.5, "9": 0.25}
    items = [[int(e), float(w)] for e, w in zip(rng.integers(0, 50, 400), np.ones(400))]
    reqs = [
        ("GET", "/healthz", None),
        ("POST", "/sketches/vector", {"entries": {str(k): v for k, v in mid.items()}, "k": 64, "seed": 9}),
        ("POST", "/sketches/vector", {"entries": {str(k): v for k, v in mid2.items()}, "k": 64, "seed": 9}),
        ("POST", "/sketches/vector", {"entries": small, "k": 16, "seed": 7, "method": "naive"}),
        ("POST", "/sketches/vector", {"entries": small, "k": 16, "seed": 7, "stream_salt": 12345}),
        ("POST", "/sketches/vector", {"entries": {str(k): v for k, v in big.items()}, "k": 256, "seed": 3}),
        ("POST", "/sketches/vector", {"entries": {"0": 1.0}, "k": 4, "seed": 1}),
        ("POST", "/sketches/stream", {"items": items, "k": 32, "seed": 5}),
        ("POST", "/sketches/stream", {"items": [[1, 0.5], [1, 0.75]], "k": 4, "seed": 5}),
    ]
    return reqs


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    from fastapi.testclient import TestClient

    from gmsketch.service import create_app

    client = TestClient(create_app())
    out = []
    bodies = {}
    for method, path, body in requests():
        r = client.get(path) if method == "GET" else client.post(path, json=body)
        out.append({"method": method, "path": path, "request": body, "status": r.status_code, "body": r.text})
        bodies[len(out) - 1] = r.json()
    # merges and estimators over the two 64-register sketches (requests 1 and 2)
    a, b = bodies[1], bodies[2]
    for path, body in [("/sketches/merge", {"sketches": [a, b]}), ("/sketches/merge", {"sketches": [b, a, b]}),
                       ("/estimates/jaccard", {"a": a, "b": b}), ("/estimates/cardinality", {"sketch": a}),
                       ("/estimates/set-algebra", {"a": a, "b": b}),
                       ("/sketches/merge", {"sketches": [a, bodies[3]]})]:
        r = client.post(path, json=body)
        out.append({"method": "POST", "path": path, "request": body, "status": r.status_code, "body": r.text})
    with open(os.path.join(HERE, "service_exchanges.json"), "w") as f:
        json.dump(out, f, indent=0)
    print(len(out), "exchanges")


if __name__ == "__main__":
    main()
