"""HTTP service routed to the GPU path.

Same JSON contract as the reference service (service/app.py:33-59,
service/models.py:8-20 and 53-55): ``GET /health`` and ``POST /transform``
with ``{re, im, algorithm, inverse}`` -> ``{re, im, m, algorithm, inverse}``;
ValueError (including CapacityError) -> HTTP 400, schema violations -> 422.
The transform runs through ``fft_split`` on a device plan cache (the
reference's ``lru_cache`` plan cache, app.py:28-30, moved onto the GPU).
``re``/``im`` may also be lists of equal-length rows: a batch in one call.
The reference's /verify (dense O(4^m) proof tool) and /bench (CPU wall-clock
harness) are out of scope.
"""

from typing import List, Literal, Union

import numpy as np
import torch
from fastapi import FastAPI, HTTPException
from pydantic import BaseModel

from . import __version__


class TransformRequest(BaseModel):
    re: Union[List[float], List[List[float]]]
    im: Union[List[float], List[List[float]]]
    algorithm: Literal["dit", "dif"] = "dit"
    inverse: bool = False


class TransformResponse(BaseModel):
    re: Union[List[float], List[List[float]]]
    im: Union[List[float], List[List[float]]]
    m: int
    algorithm: str
    inverse: bool


class HealthResponse(BaseModel):
    status: str
    version: str
    device: str


def _device_name():
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.get_device_name(torch.cuda.current_device())
    except Exception:
        pass
    return "none"


def create_app() -> FastAPI:
    from .layout import SplitSignal, is_power_of_two
    from .transform import fft_split

    app = FastAPI(title="splitfft-b200", version=__version__)

    @app.get("/health", response_model=HealthResponse)
    def health():
        return HealthResponse(status="ok", version=__version__, device=_device_name())

    @app.post("/transform", response_model=TransformResponse)
    def transform(req: TransformRequest):
        try:
            re = np.asarray(req.re, dtype=np.float64)
            im = np.asarray(req.im, dtype=np.float64)
            # length / shape checks (layout.py:28-37); torch mode keeps the
            # batched [B, N] request rows of this service
            sig = SplitSignal(torch.from_numpy(re), torch.from_numpy(im))
            n = len(sig)
            if not is_power_of_two(n):
                raise ValueError(f"sample count {n} is not a power of two")   # layout.py:96-97
            yr, yi = fft_split(re, im, algorithm=req.algorithm, inverse=req.inverse)
        except ValueError as exc:                      # includes CapacityError
            raise HTTPException(status_code=400, detail=str(exc)) from exc
        except RuntimeError as exc:                    # no GPU / CUDA failure
            raise HTTPException(status_code=503, detail=str(exc)) from exc
        return TransformResponse(re=yr.tolist(), im=yi.tolist(), m=n.bit_length() - 1,
                                 algorithm=req.algorithm, inverse=req.inverse)

    return app
