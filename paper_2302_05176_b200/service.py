"""HTTP wiring of the engine: the reference service's sketch and estimator
routes (service/app.py:74-118, request/response layout service/models.py:18-98),
answered by the CUDA engine.

A GPU-built sketch leaves the service in the reference's wire record
(hex-float registers, service/models.py:18-40 = sketch.py:325-339), so
clients of the reference service -- its CLI's ServiceClient, cli.py:29-56,
or any HTTP caller -- switch by pointing at this app.  The experiment and
network-simulation routes of the reference (/experiments/*, /simulate/*) are
its research harness, not the hot path, and are not
served here.

    uvicorn --factory paper_2302_05176_b200.service:create_app
"""

from __future__ import annotations

from typing import Literal

from pydantic import BaseModel, Field

from . import __version__
from .errors import GmSketchError
from .estimate import estimate_cardinality, estimate_jaccard_p, estimate_set_algebra, merge
from .randgen import SeedScheme
from .sketch import SKETCH_FORMAT, GenerationParams, GumbelMaxSketch, WeightedVector, sketch_fast, sketch_naive
from .stream import sketch_stream


class SketchModel(BaseModel):
    """The wire record of one sketch (registers as IEEE-754 hex strings)."""

    format: str = SKETCH_FORMAT
    k: int = Field(ge=1)
    fingerprint: str
    s: list[int]
    y: list[str]

    @classmethod
    def from_sketch(cls, sk: GumbelMaxSketch) -> "SketchModel":
        return cls(k=sk.k, fingerprint=f"{sk.fingerprint:#018x}", s=list(sk.s), y=[float(v).hex() for v in sk.y])

    def to_sketch(self) -> GumbelMaxSketch:
        return GumbelMaxSketch(k=self.k, s=tuple(self.s), y=tuple(float.fromhex(v) for v in self.y),
                               fingerprint=int(self.fingerprint, 16))


class VectorSketchRequest(BaseModel):
    entries: dict[int, float]
    k: int = Field(ge=1)
    seed: int
    stream_salt: int | None = None
    delta: int | None = Field(default=None, ge=1)
    method: Literal["fast", "naive"] = "fast"


class StreamSketchRequest(BaseModel):
    items: list[tuple[int, float]]
    k: int = Field(ge=1)
    seed: int
    stream_salt: int | None = None
    skip_duplicates: bool = True


class MergeRequest(BaseModel):
    sketches: list[SketchModel] = Field(min_length=1)


class SketchPairRequest(BaseModel):
    a: SketchModel
    b: SketchModel


class CardinalityRequest(BaseModel):
    sketch: SketchModel


class SimilarityResponse(BaseModel):
    jaccard_p: float
    k: int
    matches: int


class CardinalityResponse(BaseModel):
    weighted_cardinality: float
    k: int


class SetAlgebraResponse(BaseModel):
    union_w: float
    intersection_w: float
    a_minus_b_w: float
    jaccard_w: float


class HealthResponse(BaseModel):
    status: str
    version: str


def _scheme(seed: int, salt: int | None) -> SeedScheme:
    return SeedScheme(seed) if salt is None else SeedScheme(seed, salt)


def create_app():
    """FastAPI app serving the sketch routes on the CUDA engine; library
    errors answer HTTP 400 {"detail", "error": class name} like the
    reference's (service/app.py:63-68)."""
    from fastapi import FastAPI, Request
    from fastapi.responses import JSONResponse

    app = FastAPI(title="gmsketch (B200 engine)", version=__version__,
                  description="Gumbel-Max sketches built on sm_100a: vectors, streams, merges, estimators.")

    @app.exception_handler(GmSketchError)
    async def _library_error(request: Request, exc: GmSketchError):
        return JSONResponse(status_code=400, content={"detail": str(exc), "error": type(exc).__name__})

    @app.get("/healthz", response_model=HealthResponse)
    def healthz():
        return HealthResponse(status="ok", version=__version__)

    @app.post("/sketches/vector", response_model=SketchModel)
    def sketch_vector(req: VectorSketchRequest):
        params = GenerationParams(k=req.k, scheme=_scheme(req.seed, req.stream_salt), delta=req.delta)
        gen = sketch_naive if req.method == "naive" else sketch_fast
        return SketchModel.from_sketch(gen(WeightedVector(req.entries), params))

    @app.post("/sketches/stream", response_model=SketchModel)
    def sketch_from_stream(req: StreamSketchRequest):
        sk = sketch_stream(req.items, req.k, _scheme(req.seed, req.stream_salt), skip_duplicates=req.skip_duplicates)
        return SketchModel.from_sketch(sk)

    @app.post("/sketches/merge", response_model=SketchModel)
    def merge_sketches(req: MergeRequest):
        return SketchModel.from_sketch(merge([m.to_sketch() for m in req.sketches]))

    @app.post("/estimates/jaccard", response_model=SimilarityResponse)
    def jaccard(req: SketchPairRequest):
        est = estimate_jaccard_p(req.a.to_sketch(), req.b.to_sketch())
        return SimilarityResponse(jaccard_p=est.value, k=est.k, matches=est.matches)

    @app.post("/estimates/cardinality", response_model=CardinalityResponse)
    def cardinality(req: CardinalityRequest):
        est = estimate_cardinality(req.sketch.to_sketch())
        return CardinalityResponse(weighted_cardinality=est.value, k=est.k)

    @app.post("/estimates/set-algebra", response_model=SetAlgebraResponse)
    def set_algebra(req: SketchPairRequest):
        est = estimate_set_algebra(req.a.to_sketch(), req.b.to_sketch())
        return SetAlgebraResponse(union_w=est.union_w, intersection_w=est.intersection_w,
                                  a_minus_b_w=est.a_minus_b_w, jaccard_w=est.jaccard_w)

    return app
