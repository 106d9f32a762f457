from .session import RunReport, Session

__all__ = ["Session", "RunReport"]
